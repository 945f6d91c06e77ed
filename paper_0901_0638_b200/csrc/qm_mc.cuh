// qm_mc.cuh -- config 5: Philox-fused Monte-Carlo European-call sweep whose
// normal innovations come from the EXPONENTIAL base.
//
// Per sample (the oracle's orc_mc.c states the same recipe):
//   w = Philox word (stream layout of qm_philox_uniform, fp32 grid)
//   v = -log u, u = (2 (w >> 9) + 1) 2^-24       one-sided unit exponential
//   s = +1 if bit 8 of w is set, else -1          two-sided (Laplace) base
//   Z = s Q(v)                                    App C rational, no reflection needed
//   S_T = exp(a + b Z), a = log S0 + (r - sigma^2/2) T, b = sigma sqrt(T)
//   per strike j: (S_T - K_j)^+ and its square.
// Sums: fp32 partials over 64 samples per thread, flushed into fp64
// accumulators in shared memory; one CTA per fixed chunk of QM_MC_CHUNK samples
// of the GLOBAL stream writes one row [sum p_0, sum p_0^2, sum p_1, ...]; rows
// are all-reduced exactly across GPUs and added by qm_reduce_rows (fixed order).
#pragma once
#include "qm_math.cuh"

#define QM_MC_CHUNK (1 << 20)
#define QM_MC_MAXK 32

namespace qm {

struct McParams {
    float a, b;                 // log-price drift and volatility scale
    int nk;                     // number of strikes (<= QM_MC_MAXK)
    float K[QM_MC_MAXK];
};

// row columns 4q..4q+3 = (sum, sq) of strikes 2q and 2q+1, added into the
// thread's fp64 accumulators
QM_DEV void flush_pair(double *acc, int tid, int q, int nk, float2 sum, float2 sq)
{
    if (2 * q < nk) {
        acc[(4 * q) * 256 + tid] = __dadd_rn(acc[(4 * q) * 256 + tid], (double)sum.x);
        acc[(4 * q + 1) * 256 + tid] = __dadd_rn(acc[(4 * q + 1) * 256 + tid], (double)sq.x);
    }
    if (2 * q + 1 < nk) {
        acc[(4 * q + 2) * 256 + tid] = __dadd_rn(acc[(4 * q + 2) * 256 + tid], (double)sum.y);
        acc[(4 * q + 3) * 256 + tid] = __dadd_rn(acc[(4 * q + 3) * 256 + tid], (double)sq.y);
    }
}

// NKMAX: register budget for the per-thread fp32 partials (instantiated for 8, 17, 32)
// MINB: resident blocks per SM the register budget is set for (17 strikes: 3
// blocks at 80 registers, +3.5 % over 2 blocks at 96)
// EXACT: the call has exactly NKMAX strikes, so the strike loop has no run-time
// bounds (a warp-uniform branch per strike pair otherwise)
template <int NKMAX, int VB = 1, int MINB = 1, bool EXACT = false>
__global__ void __launch_bounds__(256, MINB)
k_mc_call(int64_t n, unsigned long long seed, unsigned long long c0, const __grid_constant__ McParams mp,
          double *__restrict__ rows)
{
    extern __shared__ double acc[];            // [2 * nk][256]
    const int nk = mp.nk, tid = threadIdx.x;
    const int nkl = EXACT ? NKMAX : nk;        // the hot loop's strike count
    const PhiloxKeys keys(seed);
    for (int j = 0; j < 2 * nk; ++j) acc[j * 256 + tid] = 0.0;

    const int64_t s0 = (int64_t)blockIdx.x * QM_MC_CHUNK;
    const int64_t s1 = (s0 + QM_MC_CHUNK < n) ? s0 + QM_MC_CHUNK : n;
    const int64_t b0 = s0 >> 2, b1 = (s1 + 3) >> 2;         // Philox blocks of this chunk
    // per-thread fp32 partials: sum and sum of squares of each strike's payoff,
    // strikes paired so that one FADD2 / FFMA2 updates two strikes (the same
    // IEEE operations as one FADD / FFMA per strike: bitwise the same sums)
    constexpr int NP = (NKMAX + 1) / 2;
    float2 sum[NP], sq[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) { sum[q] = make_float2(0.0f, 0.0f); sq[q] = make_float2(0.0f, 0.0f); }
    int inpart = 0;

    for (int64_t blk0 = b0 + tid; blk0 < b1; blk0 += 256 * VB) {
        // VB Philox blocks (4 VB samples) per iteration: all chains first (ILP),
        // then the strikes, which see the samples in stream order
        float ST[4 * VB];
        uint32_t ws[4 * VB];
#pragma unroll
        for (int b = 0; b < VB; ++b) {
            const uint4 w = philox_block(c0 + (unsigned long long)(blk0 + 256 * b), keys);
            ws[4 * b] = w.x; ws[4 * b + 1] = w.y; ws[4 * b + 2] = w.z; ws[4 * b + 3] = w.w;
        }
        float v[4 * VB];
#pragma unroll
        for (int k = 0; k < 4 * VB; k += 2) {
            const float2 vv = neg_log2x_f32x2(u01_f32(ws[k]), u01_f32(ws[k + 1]), -1);   // -log u
            v[k] = vv.x; v[k + 1] = vv.y;
        }
        float zr[4 * VB];
#pragma unroll
        for (int k = 0; k < 4 * VB; k += 2) {
            if (QM_F32_RAT >= 1 && !(QM_F32_RAT == 2 && (k & 2) == 0)) {   // grid u: v on the lattice's range
                const float2 m2 = c55_comp1_x2(make_float2(v[k], v[k + 1]));
                zr[k] = m2.x; zr[k + 1] = m2.y;
            } else {
                zr[k] = rat32<ALG_BREAKLESS>(v[k]);
                zr[k + 1] = rat32<ALG_BREAKLESS>(v[k + 1]);
            }
        }
#pragma unroll
        for (int k = 0; k < 4 * VB; ++k) {
            const int64_t i = 4 * (blk0 + 256 * (k / 4)) + (k % 4);
            float z = zr[k];
            z = ((ws[k] >> 8) & 1u) ? z : -z;
            // past the end of the chunk: S_T = -inf makes every payoff max(-inf, 0) = 0
            ST[k] = (i < s1) ? expf(__fmaf_rn(mp.b, z, mp.a)) : __int_as_float(0xff800000);
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
#pragma unroll
            for (int k = 0; k < 4 * VB; ++k) {
                if (2 * q + 1 < nkl) {
                    const float2 d = add2(make_float2(ST[k], ST[k]), make_float2(-mp.K[2 * q], -mp.K[2 * q + 1]));
                    const float2 p = make_float2(fmaxf(d.x, 0.0f), fmaxf(d.y, 0.0f));
                    sum[q] = add2(sum[q], p);
                    sq[q] = fma2(p, p, sq[q]);
                } else if (2 * q < nkl) {
                    const float p = fmaxf(__fsub_rn(ST[k], mp.K[2 * q]), 0.0f);
                    sum[q].x = __fadd_rn(sum[q].x, p);
                    sq[q].x = __fmaf_rn(p, p, sq[q].x);
                }
            }
        }
        if ((inpart += VB) == 16) {             // 64 samples: flush into fp64
            inpart = 0;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                flush_pair(acc, tid, q, nk, sum[q], sq[q]);
                sum[q] = make_float2(0.0f, 0.0f);
                sq[q] = make_float2(0.0f, 0.0f);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) flush_pair(acc, tid, q, nk, sum[q], sq[q]);
    __syncthreads();
    // fixed tree over the 256 threads, column by column
    for (int w = 128; w > 0; w >>= 1) {
        if (tid < w)
            for (int j = 0; j < 2 * nk; ++j) acc[j * 256 + tid] = __dadd_rn(acc[j * 256 + tid], acc[j * 256 + tid + w]);
        __syncthreads();
    }
    if (tid < 2 * nk) rows[(int64_t)blockIdx.x * 2 * nk + tid] = acc[tid * 256];
}

}  // namespace qm
