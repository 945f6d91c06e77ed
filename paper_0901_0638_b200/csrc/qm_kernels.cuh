// qm_kernels.cuh -- __global__ kernels of the hot path (sm_100a).
//
// Large aligned arrays (>= 2^23 samples) stream through the TMA-in /
// streaming-store pipeline of qm_tma.cuh (`*_tl` kernels: persistent CTAs,
// bulk-copy input ring, per-warp stage release, one warp vote per group of
// samples); everything else, and the remainder of the pipelines, runs the
// register-pipelined LDG kernels below.  The LDG kernels share one shape:
//  * grid = k x (SM count) blocks of 256 threads, a warp-uniform grid-stride
//    loop over warp CHUNKS (32 lanes x V 128-bit vectors), so every branch in
//    the loop body is warp-uniform -- the paper's divergence argument
//    turned into a structural property;
//  * 128-bit streaming loads (ld.global.nc.L1::no_allocate) and stores
//    (st.global.cs), all loads of a chunk issued before any math;
//  * one FSETP-AND per element builds a "normal input" predicate; a single
//    __all_sync vote picks the fast path (no special-value code) or the careful
//    path for the whole warp.  Grid inputs never leave the fast path;
//  * the scalar remainder (n % 4, or a misaligned array) runs the careful
//    scalar code in the same launch.
#pragma once
#include "qm_math.cuh"
#include "qm_tma.cuh"

namespace qm {

constexpr int kThreads = 256;

// ------------------------------------------------------------ fp32 normal
template <int ALG>
__global__ void __launch_bounds__(kThreads, 4)
k_normal_f32(const float *__restrict__ u, float *__restrict__ z, int64_t n, int vec)
{
    pdl_begin();                                          // launched with PDL (qm_lib.cu)
    constexpr int V = 2;                                  // float4 per lane per chunk
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nv = vec ? (n >> 2) : 0;
    const int64_t nchunks = (nv + 32 * V - 1) / (32 * V);
    const float4 *u4 = reinterpret_cast<const float4 *>(u);
    float4 *z4 = reinterpret_cast<float4 *>(z);

    for (int64_t c = gwarp; c < nchunks; c += nwarps) {   // warp-uniform trip count
        float x[4 * V];
        const int64_t base = c * (32 * V) + lane;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = base + 32 * j;
            const float4 a = (i < nv) ? ld_stream_f4(u4 + i) : make_float4(0.5f, 0.5f, 0.5f, 0.5f);
            x[4 * j] = a.x; x[4 * j + 1] = a.y; x[4 * j + 2] = a.z; x[4 * j + 3] = a.w;
        }
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 4 * V; ++k) ok &= (fminf(x[k], __fsub_rn(1.0f, x[k])) >= fast_vv_min_f32<ALG>());
        float y[4 * V];
        if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
            for (int k = 0; k < 4 * V; k += 2) {
                const float oa = __fsub_rn(1.0f, x[k]), ob = __fsub_rn(1.0f, x[k + 1]);
                const float2 lz = neg_log2x_f32x2(fminf(x[k], oa), fminf(x[k + 1], ob));
                y[k] = apply_sign_f32(rat32<fast_alg<ALG>()>(lz.x), x[k], oa);
                y[k + 1] = apply_sign_f32(rat32<fast_alg<ALG>()>(lz.y), x[k + 1], ob);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4 * V; ++k) y[k] = nq_f32_careful<ALG>(x[k]);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = base + 32 * j;
            if (i < nv) st_stream_f4(z4 + i, make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]));
        }
    }
    // scalar remainder
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = 4 * nv + t;
    if (i < n) z[i] = nq_f32_careful<ALG>(u[i]);
    for (int64_t j = i + (int64_t)gridDim.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        z[j] = nq_f32_careful<ALG>(u[j]);
}

// ------------------------------------------------- fp32 normal, TMA pipeline
// pipeline shapes: NC consumer warps (+1 producer), STAGES x TILE floats of
// shared memory per CTA, MINB CTAs per SM
template <int NC_, int STAGES_, int TILE_, int MINB_, int UNROLL_ = 1>
struct TmaCfg {
    static constexpr int NC = NC_, STAGES = STAGES_, TILE = TILE_, MINB = MINB_, THREADS = 32 * (NC_ + 1);
    static constexpr int UNROLL = UNROLL_;
    static_assert(TILE_ % (4 * 32 * NC_ * UNROLL_) == 0, "tile must split evenly over the consumer threads");
};
using TmaCfgB = TmaCfg<16, 3, 8192, 2>;      // 2 CTAs/SM, 32 consumer warps, 2 x 96 KB

// one float4 of u -> one float4 of z: a single vote per warp picks the fast path
// (no special-value code) or the careful path for all 4 x 32 samples
template <int ALG>
QM_DEV float4 normal4_f32(const float4 a)
{
    const float x[4] = {a.x, a.y, a.z, a.w};
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) ok &= (fminf(x[k], __fsub_rn(1.0f, x[k])) >= fast_vv_min_f32<ALG>());
    float y[4];
    if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
        for (int k = 0; k < 4; k += 2) {
            const float oa = __fsub_rn(1.0f, x[k]), ob = __fsub_rn(1.0f, x[k + 1]);
            const float2 lz = neg_log2x_f32x2(fminf(x[k], oa), fminf(x[k + 1], ob));
            y[k] = apply_sign_f32(rat32<fast_alg<ALG>()>(lz.x), x[k], oa);
            y[k + 1] = apply_sign_f32(rat32<fast_alg<ALG>()>(lz.y), x[k + 1], ob);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) y[k] = nq_f32_careful<ALG>(x[k]);
    }
    return make_float4(y[0], y[1], y[2], y[3]);
}

// G float4 (4G samples) per lane under ONE vote: the fast path of all 4G samples
// is one basic block, so the scheduler can interleave their log chains (FFMA2)
// and rational chains (DFMA) -- the fp32 log alone is a 9-deep dependent chain.
template <int ALG, int G>
QM_DEV void normal_group_f32(float4 *a)
{
    constexpr int NS = 4 * G;
    float x[NS];
#pragma unroll
    for (int j = 0; j < G; ++j) { x[4 * j] = a[j].x; x[4 * j + 1] = a[j].y; x[4 * j + 2] = a[j].z; x[4 * j + 3] = a[j].w; }
    // 1 - u two samples per FADD2 (the same IEEE subtraction per lane)
    float om[NS], vv[NS];
#pragma unroll
    for (int k = 0; k < NS; k += 2) {
        const float2 o = add2(make_float2(1.0f, 1.0f), make_float2(-x[k], -x[k + 1]));
        om[k] = o.x; om[k + 1] = o.y;
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) vv[k] = fminf(x[k], om[k]);
    // the whole group is "normal" iff the NaN-propagating minimum of its vv is
    // >= the fast-path threshold: 3-input FMNMX3.NAN, one FSETP per group
    float mn = vv[0];
    int k0 = 1;
#pragma unroll
    for (; k0 + 1 < NS; k0 += 2) mn = min3_nan(mn, vv[k0], vv[k0 + 1]);
    if (k0 < NS) mn = min_nan(mn, vv[k0]);
    constexpr bool COMP = QM_F32_RAT >= 1 && fast_alg<ALG>() == ALG_BREAKLESS;
    bool ok;
    if constexpr (COMP) {
        // the FMA-pipe rational needs every sample on the 24-bit lattice: 1 - (1 - u) == u
        // (1 - u is exact for u >= 1/2, and for u < 1/2 exactly when u is a multiple of 2^-24)
        float dm = 0.0f;
#pragma unroll
        for (int k = 0; k < NS; k += 2) {
            const float2 b = add2(make_float2(1.0f, 1.0f), make_float2(-om[k], -om[k + 1]));
            const float2 d = add2(b, make_float2(-x[k], -x[k + 1]));
            dm = fmaxf(dm, fmaxf(fabsf(d.x), fabsf(d.y)));
        }
        ok = (mn >= QM_LATTICE_MIN) & (dm == 0.0f);
    } else {
        ok = mn >= fast_vv_min_f32<ALG>();
    }
    float y[NS];
    if (__all_sync(0xffffffffu, ok)) {
        float zl[NS];
#pragma unroll
        for (int k = 0; k < NS; k += 2) {
            const float2 lz = neg_log2x_f32x2(vv[k], vv[k + 1]);
            zl[k] = lz.x; zl[k + 1] = lz.y;
        }
        // sign of u - (1-u), two samples per FADD2 (+0 at u = 1/2, as apply_sign_f32)
        float dsg[NS];
#pragma unroll
        for (int k = 0; k < NS; k += 2) {
            const float2 d = add2(make_float2(x[k], x[k + 1]), make_float2(-om[k], -om[k + 1]));
            dsg[k] = d.x; dsg[k + 1] = d.y;
        }
        float mag[NS];
#pragma unroll
        for (int k = 0; k < NS; k += 2) {
            if (COMP && !(QM_F32_RAT == 2 && (k & 2) == 0)) {
                const float2 m2 = c55_comp1_x2(make_float2(zl[k], zl[k + 1]));
                mag[k] = m2.x; mag[k + 1] = m2.y;
            } else {
                mag[k] = rat32<fast_alg<ALG>()>(zl[k]);
                mag[k + 1] = rat32<fast_alg<ALG>()>(zl[k + 1]);
            }
        }
#pragma unroll
        for (int k = 0; k < NS; ++k)
            y[k] = __uint_as_float((__float_as_uint(mag[k]) & 0x7fffffffu) | (__float_as_uint(dsg[k]) & 0x80000000u));
    } else {
#pragma unroll
        for (int k = 0; k < NS; ++k) y[k] = nq_f32_careful<ALG>(x[k]);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) a[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
}

template <int ALG, int G>
struct MapNormalF32 {
    template <int PER>
    QM_DEV void map_slice(float4 *a) const
    {
        static_assert(PER % G == 0, "group size must divide the per-lane vector count");
#pragma unroll
        for (int j = 0; j < PER; j += G) normal_group_f32<ALG, G>(a + j);
    }
};

// TMA-in / STG-out shapes (tma_load_map): NC consumer warps, STAGES x TILE
// floats of shared memory per CTA, MINB CTAs per SM
template <int NC_, int STAGES_, int TILE_, int MINB_, int G_ = 1>
struct TlCfg {
    static constexpr int NC = NC_, STAGES = STAGES_, TILE = TILE_, MINB = MINB_, THREADS = 32 * (NC_ + 1);
    static constexpr int UNROLL = 1, G = G_;
    static_assert(TILE_ % (4 * 32 * NC_) == 0, "tile must split evenly over the consumer warps");
};
using TlCfgJ = TlCfg<16, 4, 8192, 1>;       // 1 CTA/SM, 16 consumer warps, 4 x 32 KB
using TlCfgK = TlCfg<16, 3, 8192, 2>;       // 2 CTAs/SM, 2 x 3 x 32 KB
using TlCfgL = TlCfg<16, 4, 8192, 1, 2>;    // J, 2 float4 per vote
using TlCfgM = TlCfg<8, 3, 8192, 2, 2>;     // 2 CTAs/SM of 8 consumer warps, 2 x 3 x 32 KB

template <int ALG, class CFG>
__global__ void __launch_bounds__(CFG::THREADS, CFG::MINB)
k_normal_f32_tl(const float *__restrict__ u, float *__restrict__ z, int64_t ntiles)
{
    tma_load_map<float4, CFG::TILE / 4, CFG::STAGES, CFG::NC>(reinterpret_cast<const float4 *>(u),
                                                             reinterpret_cast<float4 *>(z), ntiles,
                                                             MapNormalF32<ALG, CFG::G>{});
}

template <int ALG, class CFG>
struct OpNormalF32 {
    QM_DEV void tile(float *t, int ctid, int nct) const
    {
        float4 *t4 = reinterpret_cast<float4 *>(t);
        constexpr int per = CFG::TILE / 4 / (CFG::NC * 32);
#pragma unroll CFG::UNROLL
        for (int j = 0; j < per; ++j) {
            float4 *p = t4 + ctid + j * nct;
            const float4 a = *p;
            const float x[4] = {a.x, a.y, a.z, a.w};
            bool ok = true;
#pragma unroll
            for (int k = 0; k < 4; ++k) ok &= (fminf(x[k], __fsub_rn(1.0f, x[k])) >= fast_vv_min_f32<ALG>());
            float y[4];
            if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
                for (int k = 0; k < 4; k += 2) {
                    const float oa = __fsub_rn(1.0f, x[k]), ob = __fsub_rn(1.0f, x[k + 1]);
                    const float2 lz = neg_log2x_f32x2(fminf(x[k], oa), fminf(x[k + 1], ob));
                    y[k] = apply_sign_f32(rat32<fast_alg<ALG>()>(lz.x), x[k], oa);
                    y[k + 1] = apply_sign_f32(rat32<fast_alg<ALG>()>(lz.y), x[k + 1], ob);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) y[k] = nq_f32_careful<ALG>(x[k]);
            }
            *p = make_float4(y[0], y[1], y[2], y[3]);
        }
    }
};

template <int ALG, class CFG>
__global__ void __launch_bounds__(CFG::THREADS, CFG::MINB)
k_normal_f32_tma(const float *__restrict__ u, float *__restrict__ z, int64_t ntiles)
{
    tma_stream_map<float, CFG::TILE, CFG::STAGES, CFG::NC>(u, z, ntiles, OpNormalF32<ALG, CFG>{});
}

// ------------------------------------------------------------ fp64 normal
template <int ALG>
__global__ void __launch_bounds__(kThreads, 2)
k_normal_f64(const double *__restrict__ u, double *__restrict__ z, int64_t n, int vec)
{
    constexpr int V = 1;                                  // double2 per lane per chunk (FP64-bound:
                                                          // occupancy over ILP)
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nv = vec ? (n >> 1) : 0;
    const int64_t nchunks = (nv + 32 * V - 1) / (32 * V);
    const double2 *u2 = reinterpret_cast<const double2 *>(u);
    double2 *z2 = reinterpret_cast<double2 *>(z);

    for (int64_t c = gwarp; c < nchunks; c += nwarps) {
        double x[2 * V];
        const int64_t base = c * (32 * V) + lane;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = base + 32 * j;
            const double2 a = (i < nv) ? ld_stream_d2(u2 + i) : make_double2(0.5, 0.5);
            x[2 * j] = a.x; x[2 * j + 1] = a.y;
        }
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 2 * V; ++k) ok &= (fmin(x[k], __dadd_rn(1.0, -x[k])) >= fast_vv_min_f64<ALG>());
        double y[2 * V];
        if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
            for (int k = 0; k < 2 * V; ++k) y[k] = nq_f64_fast<ALG>(x[k]);
        } else {
#pragma unroll
            for (int k = 0; k < 2 * V; ++k) y[k] = nq_f64_careful<ALG>(x[k]);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = base + 32 * j;
            if (i < nv) st_stream_d2(z2 + i, make_double2(y[2 * j], y[2 * j + 1]));
        }
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t j = 2 * nv + t; j < n; j += (int64_t)gridDim.x * blockDim.x)
        z[j] = nq_f64_careful<ALG>(u[j]);
}

// fp64 map through the TMA-in / streaming-store pipeline: a lane's slice of PER
// double2 under one vote per double2 (64 samples per warp vote)
#ifndef QM_F64_GROUP
#define QM_F64_GROUP 1
#endif
template <int ALG, int GD = QM_F64_GROUP>   // GD double2 (2 GD samples) per lane per vote
struct MapNormalF64 {
    template <int PER>
    QM_DEV void map_slice(double2 *a) const
    {
        static_assert(PER % GD == 0, "group must divide the slice");
#pragma unroll
        for (int j = 0; j < PER; j += GD) {
            bool ok = true;
#pragma unroll
            for (int g = 0; g < GD; ++g)
                ok &= (fmin(a[j + g].x, __dadd_rn(1.0, -a[j + g].x)) >= fast_vv_min_f64<ALG>()) &
                      (fmin(a[j + g].y, __dadd_rn(1.0, -a[j + g].y)) >= fast_vv_min_f64<ALG>());
            if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
                for (int g = 0; g < GD; ++g)
                    a[j + g] = make_double2(nq_f64_fast<ALG>(a[j + g].x), nq_f64_fast<ALG>(a[j + g].y));
            } else {
#pragma unroll
                for (int g = 0; g < GD; ++g)
                    a[j + g] = make_double2(nq_f64_careful<ALG>(a[j + g].x), nq_f64_careful<ALG>(a[j + g].y));
            }
        }
    }
};

// 1 CTA/SM: producer + NC consumer warps, 4 stages of TILE_VECS double2
template <int NC_, int TILE_VECS_>
struct TlCfgF64 {
    static constexpr int NC = NC_, STAGES = 4, TILE_VECS = TILE_VECS_, THREADS = 32 * (NC_ + 1);
    static constexpr int TILE = 2 * TILE_VECS_;                          // doubles per tile
};
using TlF64A = TlCfgF64<12, 1536>;    // 13 warps, 4 x 24 KB, 4 double2 per lane
using TlF64B = TlCfgF64<16, 2048>;    // 17 warps, 4 x 32 KB, 4 double2 per lane

template <int ALG, class CFG>
__global__ void __launch_bounds__(CFG::THREADS, 1)
k_normal_f64_tl(const double *__restrict__ u, double *__restrict__ z, int64_t ntiles)
{
    tma_load_map<double2, CFG::TILE_VECS, CFG::STAGES, CFG::NC>(reinterpret_cast<const double2 *>(u),
                                                               reinterpret_cast<double2 *>(z), ntiles,
                                                               MapNormalF64<ALG>{});
}

// --------------------------------------------------- Philox uniforms / fused
// MODE 0: write the uniforms; MODE 1: write the normal quantile of them (fused).
template <int MODE, int ALG, int V = 2, int MINB = 1>   // V: Philox blocks per lane per chunk
__global__ void __launch_bounds__(kThreads, MINB)
k_philox_f32(float *__restrict__ z, int64_t n, unsigned long long seed, unsigned long long c0, int vec)
{
    pdl_begin();                                          // launched with PDL (qm_lib.cu)
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nb = (n + 3) >> 2;                      // Philox blocks
    const int64_t nchunks = (nb + 32 * V - 1) / (32 * V);
    for (int64_t c = gwarp; c < nchunks; c += nwarps) {
        const int64_t base = c * (32 * V) + lane;
        // all V blocks (4V samples) in one basic block, stores after the math, so
        // the scheduler can interleave the Philox rounds, logs and rationals
        float r[4 * V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint4 w = philox_block(c0 + (unsigned long long)(base + 32 * j), seed);
            r[4 * j] = u01_f32(w.x); r[4 * j + 1] = u01_f32(w.y);
            r[4 * j + 2] = u01_f32(w.z); r[4 * j + 3] = u01_f32(w.w);
        }
        if (MODE == 1) {
            // 1 - u and the sign subtraction two samples per FADD2 (same IEEE ops)
            float om[4 * V], zl[4 * V], dsg[4 * V];
#pragma unroll
            for (int k = 0; k < 4 * V; k += 2) {
                const float2 o = add2(make_float2(1.0f, 1.0f), make_float2(-r[k], -r[k + 1]));
                om[k] = o.x; om[k + 1] = o.y;
                const float2 l = neg_log2x_f32x2(fminf(r[k], om[k]), fminf(r[k + 1], om[k + 1]));
                zl[k] = l.x; zl[k + 1] = l.y;
                const float2 d = add2(make_float2(r[k], r[k + 1]), make_float2(-om[k], -om[k + 1]));
                dsg[k] = d.x; dsg[k + 1] = d.y;
            }
            constexpr bool COMP = QM_F32_RAT >= 1 && fast_alg<ALG>() == ALG_BREAKLESS;
            float mag[4 * V];
#pragma unroll
            for (int k = 0; k < 4 * V; k += 2) {
                if (COMP && !(QM_F32_RAT == 2 && (k & 2) == 0)) {   // grid inputs: always on the lattice
                    const float2 m2 = c55_comp1_x2(make_float2(zl[k], zl[k + 1]));
                    mag[k] = m2.x; mag[k + 1] = m2.y;
                } else {
                    mag[k] = rat32<fast_alg<ALG>()>(zl[k]);
                    mag[k + 1] = rat32<fast_alg<ALG>()>(zl[k + 1]);
                }
            }
#pragma unroll
            for (int k = 0; k < 4 * V; ++k)
                r[k] = __uint_as_float((__float_as_uint(mag[k]) & 0x7fffffffu) | (__float_as_uint(dsg[k]) & 0x80000000u));
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = 4 * (base + 32 * j);
            if (vec && i + 3 < n) {
                st_stream_f4(reinterpret_cast<float4 *>(z + i), make_float4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]));
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) if (i + k < n) z[i + k] = r[4 * j + k];
            }
        }
    }
}

template <int MODE, int ALG, int V = 1>   // V Philox blocks (2V samples) per lane per chunk
__global__ void __launch_bounds__(kThreads)
k_philox_f64(double *__restrict__ z, int64_t n, unsigned long long seed, unsigned long long c0, int vec)
{
    pdl_begin();                                          // launched with PDL (qm_lib.cu)
    const PhiloxKeys keys(seed);
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nb = (n + 1) >> 1;
    const int64_t nchunks = (nb + 32 * V - 1) / (32 * V);
    for (int64_t c = gwarp; c < nchunks; c += nwarps) {
        double r[2 * V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint4 w = philox_block(c0 + (unsigned long long)(c * 32 * V + 32 * j + lane), keys);
            r[2 * j] = u01_f64(w.x, w.y);
            r[2 * j + 1] = u01_f64(w.z, w.w);
        }
        if (MODE == 1) {
#pragma unroll
            for (int k = 0; k < 2 * V; ++k) r[k] = nq_f64_fast<ALG>(r[k]);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = 2 * (c * 32 * V + 32 * j + lane);
            if (vec && i + 1 < n) {
                st_stream_d2(reinterpret_cast<double2 *>(z + i), make_double2(r[2 * j], r[2 * j + 1]));
            } else {
                if (i < n) z[i] = r[2 * j];
                if (i + 1 < n) z[i + 1] = r[2 * j + 1];
            }
        }
    }
}

// -------------------------------------------------- antithetic
// v = -log u, Z = Q(v); out[2i] = Z, out[2i+1] = -Z.
template <int ALG>
QM_DEV float anti_f32_careful(float u)
{
    const bool sub = u < 1.17549435e-38f;
    const float us = sub ? __fmul_rn(u, 16777216.0f) : u;
    float mag = rat32<ALG>(neg_log2x_f32(us, sub ? -25 : -1));
    mag = (u == 0.0f) ? __int_as_float(0x7f800000) : mag;
    mag = __uint_as_float(__float_as_uint(mag) & 0x7fffffffu);            // +0 at u = 1
    return (u >= 0.0f && u <= 1.0f) ? mag : __int_as_float(0x7fffffff);
}

template <int ALG>
__global__ void __launch_bounds__(kThreads)
k_antithetic_f32(const float *__restrict__ u, float *__restrict__ z, int64_t n, int vec)
{
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nv = vec ? (n >> 2) : 0;
    const int64_t nchunks = (nv + 31) / 32;
    for (int64_t c = gwarp; c < nchunks; c += nwarps) {
        const int64_t i = c * 32 + lane;
        const float4 a = (i < nv) ? ld_stream_f4(reinterpret_cast<const float4 *>(u) + i)
                                  : make_float4(0.5f, 0.5f, 0.5f, 0.5f);
        const float x[4] = {a.x, a.y, a.z, a.w};
        bool ok = true;
#pragma unroll
        // v = -log u < vc for the tail composite: u > e^-37 = 8.5e-17
        for (int k = 0; k < 4; ++k) ok &= (x[k] >= (ALG == ALG_BREAKLESS_TAIL ? 8.6e-17f : 1.17549435e-38f)) & (x[k] <= 1.0f);
        float y[4];
        if (__all_sync(0xffffffffu, ok)) {
            // -log u: eadj = -1 cancels the factor 2 of neg_log2x
            const float2 l01 = neg_log2x_f32x2(x[0], x[1], -1);
            const float2 l23 = neg_log2x_f32x2(x[2], x[3], -1);
            y[0] = fabsf(rat32<fast_alg<ALG>()>(l01.x)); y[1] = fabsf(rat32<fast_alg<ALG>()>(l01.y));
            y[2] = fabsf(rat32<fast_alg<ALG>()>(l23.x)); y[3] = fabsf(rat32<fast_alg<ALG>()>(l23.y));
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) y[k] = anti_f32_careful<ALG>(x[k]);
        }
        if (i < nv) {
            float4 *o = reinterpret_cast<float4 *>(z) + 2 * i;
            st_stream_f4(o, make_float4(y[0], -y[0], y[1], -y[1]));
            st_stream_f4(o + 1, make_float4(y[2], -y[2], y[3], -y[3]));
        }
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t j = 4 * nv + t; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const float y = anti_f32_careful<ALG>(u[j]);
        z[2 * j] = y; z[2 * j + 1] = -y;
    }
}

// antithetic pairs through the TMA pipeline: input float4 u -> two float4
// (Z0, -Z0, Z1, -Z1), (Z2, -Z2, Z3, -Z3); the same arithmetic as k_antithetic_f32
template <int ALG>
struct MapAntithetic {
    template <int PER>
    QM_DEV void map_slice(const float4 *a, float4 *b) const
    {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const float x[4] = {a[j].x, a[j].y, a[j].z, a[j].w};
            bool ok = true;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                ok &= (x[k] >= (ALG == ALG_BREAKLESS_TAIL ? 8.6e-17f : 1.17549435e-38f)) & (x[k] <= 1.0f);
            float y[4];
            if (__all_sync(0xffffffffu, ok)) {
                const float2 l01 = neg_log2x_f32x2(x[0], x[1], -1);
                const float2 l23 = neg_log2x_f32x2(x[2], x[3], -1);
                y[0] = fabsf(rat32<fast_alg<ALG>()>(l01.x)); y[1] = fabsf(rat32<fast_alg<ALG>()>(l01.y));
                y[2] = fabsf(rat32<fast_alg<ALG>()>(l23.x)); y[3] = fabsf(rat32<fast_alg<ALG>()>(l23.y));
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) y[k] = anti_f32_careful<ALG>(x[k]);
            }
            b[2 * j] = make_float4(y[0], -y[0], y[1], -y[1]);
            b[2 * j + 1] = make_float4(y[2], -y[2], y[3], -y[3]);
        }
    }
};

template <int ALG>
__global__ void __launch_bounds__(32 * (16 + 1), 1)
k_antithetic_f32_tl(const float *__restrict__ u, float *__restrict__ z, int64_t ntiles)
{
    tma_load_map<float4, 2048, 4, 16, MapAntithetic<ALG>, 2>(reinterpret_cast<const float4 *>(u),
                                                            reinterpret_cast<float4 *>(z), ntiles,
                                                            MapAntithetic<ALG>{});
}


template <int ALG>
QM_DEV double anti_f64(double u)
{
    const bool sub = u < 2.2250738585072014e-308;
    const double us = sub ? __dmul_rn(u, 18014398509481984.0) : u;
    double mag = rat64<ALG>(neg_log2x_dd(us, sub ? -55 : -1));
    mag = (u == 0.0) ? __longlong_as_double(0x7ff0000000000000LL) : mag;
    mag = fabs(mag);
    return (u >= 0.0 && u <= 1.0) ? mag : __longlong_as_double(0x7fffffffffffffffLL);
}

template <int ALG>
__global__ void __launch_bounds__(kThreads)
k_antithetic_f64(const double *__restrict__ u, double *__restrict__ z, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const double y = anti_f64<ALG>(u[j]);
        z[2 * j] = y;
        z[2 * j + 1] = -y;
    }
}

// ------------------------------------------- exponential (Laplace) -> normal
template <int ALG>
QM_DEV float exp2n_f32(float v)
{
    const float a = fabsf(v);
    float mag = rat32<ALG>(a);
    mag = (a == __int_as_float(0x7f800000)) ? a : mag;
    const float r = __uint_as_float((__float_as_uint(mag) & 0x7fffffffu) | (__float_as_uint(v) & 0x80000000u));
    return (v == v) ? r : v;
}

template <int ALG>
__global__ void __launch_bounds__(kThreads)
k_exp2n_f32(const float *__restrict__ v, float *__restrict__ z, int64_t n, int vec)
{
    pdl_begin();                                          // launched with PDL (qm_lib.cu)
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nv = vec ? (n >> 2) : 0;
    const int64_t nchunks = (nv + 63) / 64;
    for (int64_t c = gwarp; c < nchunks; c += nwarps) {
        const int64_t base = c * 64 + lane;
        float4 a[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int64_t i = base + 32 * j;
            a[j] = (i < nv) ? ld_stream_f4(reinterpret_cast<const float4 *>(v) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int64_t i = base + 32 * j;
            const float4 r = make_float4(exp2n_f32<ALG>(a[j].x), exp2n_f32<ALG>(a[j].y),
                                         exp2n_f32<ALG>(a[j].z), exp2n_f32<ALG>(a[j].w));
            if (i < nv) st_stream_f4(reinterpret_cast<float4 *>(z) + i, r);
        }
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t j = 4 * nv + t; j < n; j += (int64_t)gridDim.x * blockDim.x) z[j] = exp2n_f32<ALG>(v[j]);
}

template <int ALG, class CFG>
struct OpExp2nF32 {
    QM_DEV void tile(float *t, int ctid, int nct) const
    {
        float4 *t4 = reinterpret_cast<float4 *>(t);
        constexpr int per = CFG::TILE / 4 / (CFG::NC * 32);
#pragma unroll 2
        for (int j = 0; j < per; ++j) {
            float4 *p = t4 + ctid + j * nct;
            const float4 a = *p;
            *p = make_float4(exp2n_f32<ALG>(a.x), exp2n_f32<ALG>(a.y), exp2n_f32<ALG>(a.z), exp2n_f32<ALG>(a.w));
        }
    }
};

template <int ALG>
struct MapExp2nF32 {
    template <int PER>
    QM_DEV void map_slice(float4 *a) const
    {
#pragma unroll
        for (int j = 0; j < PER; ++j)
            a[j] = make_float4(exp2n_f32<ALG>(a[j].x), exp2n_f32<ALG>(a[j].y), exp2n_f32<ALG>(a[j].z),
                               exp2n_f32<ALG>(a[j].w));
    }
};

template <int ALG, class CFG>
__global__ void __launch_bounds__(CFG::THREADS, CFG::MINB)
k_exp2n_f32_tl(const float *__restrict__ v, float *__restrict__ z, int64_t ntiles)
{
    tma_load_map<float4, CFG::TILE / 4, CFG::STAGES, CFG::NC>(reinterpret_cast<const float4 *>(v),
                                                             reinterpret_cast<float4 *>(z), ntiles,
                                                             MapExp2nF32<ALG>{});
}

template <int ALG, class CFG>
__global__ void __launch_bounds__(CFG::THREADS, CFG::MINB)
k_exp2n_f32_tma(const float *__restrict__ v, float *__restrict__ z, int64_t ntiles)
{
    tma_stream_map<float, CFG::TILE, CFG::STAGES, CFG::NC>(v, z, ntiles, OpExp2nF32<ALG, CFG>{});
}

// fp64: for |v| >= 2^40 the polynomials would overflow in double; evaluate the
// same rational in reversed form, P(v)/Q(v) = Prev(1/v)/Qrev(1/v).
template <int N>
QM_DEV double ratio_rev(double v, const double *P, const double *Q)
{
    const double w = 1.0 / v;
    double p = P[0], q = Q[0];
#pragma unroll
    for (int i = 1; i < N; ++i) { p = __fma_rn(p, w, P[i]); q = __fma_rn(q, w, Q[i]); }
    return v * (p / q);
}

template <int ALG>
QM_DEV double exp2n_f64(double v)
{
    const double a = fabs(v);
    double mag;
    if (a < 1099511627776.0 || (ALG == ALG_BREAKLESS_TAIL && a < __longlong_as_double(0x7ff0000000000000LL))) {
        mag = rat64<ALG>(dd{a, 0.0});
    } else if (a == __longlong_as_double(0x7ff0000000000000LL)) {
        mag = a;
    } else {
        mag = (ALG == ALG_BREAKLESS77) ? ratio_rev<8>(a, kA77P_d, kA77Q_d) : ratio_rev<14>(a, kD13P, kD13Q);
    }
    const double r = copysign(mag, v);
    return (v == v) ? r : v;
}

template <int ALG>
__global__ void __launch_bounds__(kThreads)
k_exp2n_f64(const double *__restrict__ v, double *__restrict__ z, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const double x = v[j];
        // warp-uniform fast check
        const bool ok = fabs(x) < 1099511627776.0;
        z[j] = __all_sync(__activemask(), ok) ? copysign(rat64<ALG>(dd{fabs(x), 0.0}), x) : exp2n_f64<ALG>(x);
    }
}

}  // namespace qm
