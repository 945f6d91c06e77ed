// qm_student.cuh -- normal -> Student-t recycling kernel.
//
//   central  t = z sum_{k=0}^{K} c_k y^k, y = z^2
//   tail     w = (1 - Phi(|z|)) C_nu, C_nu = nu sqrt(pi) Gamma(nu/2)/Gamma((nu+1)/2),
//            t = sqrt(nu) w^(-1/nu) (1 - (nu+1)/(2(nu+2)) w^(2/nu))
//   composite central for |z| < z*, tail for |z| >= z*, odd in z.
//
// c_0..c_K come from the recurrence of P:178-188, run on the host in __float128
// (qm_student_host.cpp): the recurrence cancels terms of size c_i down to
// c_{i+1}, so double would lose up to 8 digits at nu = 10, K = 16.
//
// Device: the central series is a compensated Horner in y carried as a
// double-double (y = z*z exactly); the tail is evaluated in double-double
// (log, exp) behind a warp-uniform vote, so it costs nothing when no lane of
// the warp is in the tail (P(|z| > 3.9) ~ 1e-4 per sample).
#pragma once
#include "qm_dd.cuh"
#include "qm_tma.cuh"
#include "qm_moments.cuh"

#include "qm_student_params.h"

#ifndef QM_STUDENT_DEFER
// A/B: 1 = one vote per slice and the lane's tails one at a time (below).  Measured
// (same box, Gsamples/s, defer / per-position votes): nu = 3 241 / 237, nu = 4 274 /
// 276, nu = 5 254 / 253, nu = 10 253 / 257, fused moments 234 / 238 -- the tail is
// not what separates nu = 3 from nu = 5 (a caller z* beyond every sample runs nu = 3
// at 250), so the simpler per-position vote stays
#define QM_STUDENT_DEFER 0
#endif
#ifndef QM_STUDENT_PAIR
#define QM_STUDENT_PAIR 1   // 1 = the two samples of a double2 interleaved (+2-4 %); 0 = one by one; 2 = four
#endif

namespace qm {

QM_DEV double student_central(const StudentParams &sp, double a)
{
    const double yh = __dmul_rn(a, a);
    const double yl = __fma_rn(a, a, -yh);
    double s = sp.c[sp.K], c = 0.0;
    int i = sp.K - 1;
    for (; i >= sp.kc; --i) s = __fma_rn(s, yh, sp.c[i]);      // high-order steps: plain
    for (; i >= 0; --i) {                                      // last kc steps: compensated
        const double p = __dmul_rn(s, yh);
        const double pi = __fma_rn(s, yh, -p);
        const double t = __dadd_rn(p, sp.c[i]);
        const double bb = __dadd_rn(t, -p);
        const double sg = __dadd_rn(__dadd_rn(p, -__dadd_rn(t, -bb)), __dadd_rn(sp.c[i], -bb));
        c = __fma_rn(c, yh, __fma_rn(s, yl, __dadd_rn(pi, sg)));
        s = t;
    }
    return __fma_rn(a, s, __dmul_rn(a, c));
}

// the same series with K and the compensated count KC fixed at compile time
// (fully unrolled; bitwise equal to student_central for sp.K == K, sp.kc == KC)
template <int K, int KC>
QM_DEV double student_central_k(const StudentParams &sp, double a)
{
    const double yh = __dmul_rn(a, a);
    const double yl = __fma_rn(a, a, -yh);
    double s = sp.c[K], c = 0.0;
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
        if (i >= KC) {
            s = __fma_rn(s, yh, sp.c[i]);
        } else {
            const double p = __dmul_rn(s, yh);
            const double pi = __fma_rn(s, yh, -p);
            const dd t = two_sum_ord(p, sp.c[i]);            // = TwoSum, bitwise
            c = __fma_rn(c, yh, __fma_rn(s, yl, __dadd_rn(pi, t.lo)));
            s = t.hi;
        }
    }
    return __fma_rn(a, s, __dmul_rn(a, c));
}

// exp(x) in double for -700 < x < 700, ~1 ulp: k = rint(x / ln 2), r = x - k ln 2
// (two-part ln 2), Taylor to r^13 (|r| <= 0.347), 2^k from exponent bits in two
// factors -- branch-free (libdevice exp() measured 2x slower in this kernel)
QM_DEV double exp_plain(double x)
{
    x = fmin(fmax(x, -746.0), 710.0);              // saturate: +0 / +inf through the scaling
    const double k = rint(__dmul_rn(x, 1.4426950408889634));
    double r = __fma_rn(-k, 6.93147180369123816490e-01, x);
    r = __fma_rn(-k, 1.90821492927058770002e-10, r);
    double t = 1.0 / 6227020800.0;                          // 1/13!
    const double f[13] = {1.0, 1.0, 0.5, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
                          1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600};
#pragma unroll
    for (int i = 12; i >= 0; --i) t = __fma_rn(t, r, f[i]);
    const int ki = (int)k, k1 = ki / 2, k2 = ki - k1;
    const double s1 = __longlong_as_double((long long)(k1 + 1023) << 52);
    const double s2 = __longlong_as_double((long long)(k2 + 1023) << 52);
    return t * s1 * s2;
}

#ifndef QM_STUDENT_TAIL_NOINLINE
#define QM_STUDENT_TAIL_NOINLINE 1   // the rarely taken tail out of line: a compact hot loop (A/B same box: nu = 3 240 -> 246, nu = 4 276 -> 281, nu = 5 260 -> 260)
#endif
#if QM_STUDENT_TAIL_NOINLINE
__device__ __noinline__ double student_tail(const StudentParams &sp, double a)
#else
QM_DEV double student_tail(const StudentParams &sp, double a)
#endif
{
    // log w = log(erfc(a/sqrt2)) + log(C_nu/2); erfc(x) = exp(-x^2) erfcx(x)
    const double xh = __dmul_rn(a, 0.70710678118654752440);
    const double xl = __fma_rn(a, 0.70710678118654752440, -xh) + a * (-4.8336466567264567e-17);
    const dd x2 = dd_mul(dd{xh, xl}, dd{xh, xl});
    const dd lx = dd_log(erfcx(xh));
    dd logw = dd_add(dd{-x2.hi, -x2.lo}, lx);
    logw = dd_add(logw, dd{sp.logC_hi, sp.logC_lo});
    // w^(-1/nu) in double-double; w^(2/nu) enters only the correction
    // 1 - (nu+1)/(2(nu+2)) w^(2/nu) (a term << 1 beside the leading 1), so double
    // precision suffices for it: exp of the rounded exponent, relative error
    // ~1e-15 of a term that is itself < 0.1 -> < 1e-16 of t
    const dd e1 = dd_exp(dd_mul(logw, dd{-sp.inv_nu, -sp.inv_nu_lo}));
    const double e2 = exp_plain(__dmul_rn(logw.hi + logw.lo, sp.two_over_nu));
    const dd corr = two_sum(1.0, -__dmul_rn(e2, sp.acoef));
    const dd t = dd_mul(dd_mul(e1, dd{sp.sqrt_nu, sp.sqrt_nu_lo}), corr);
    // beyond the double range w^(-1/nu) = +inf and the dd products give inf - inf =
    // NaN: the value is +inf
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    return (e1.hi == inf) ? inf : t.hi + t.lo;
}

// the composite from a central value tc already computed for |z|
QM_DEV double student_finish(const StudentParams &sp, double z, double tc, bool any_tail)
{
    const double a = fabs(z);
    double t = tc;
    if (any_tail) {
        const double tt = student_tail(sp, fmax(a, sp.zstar));
        t = (a >= sp.zstar) ? tt : t;
    }
    t = (a == __longlong_as_double(0x7ff0000000000000LL)) ? a : t;
    const double r = copysign(t, z);
    return (z == z) ? r : z;
}

template <int K = 0, int KC = 0>   // K = 0: run-time sp.K / sp.kc
QM_DEV double student_map(const StudentParams &sp, double z, bool any_tail)
{
    const double a = fabs(z);
    double t = (K > 0) ? student_central_k<K, KC>(sp, a) : student_central(sp, a);
    if (any_tail) {
        // every lane of the warp evaluates the tail at a >= z* (one erfcx region)
        const double tt = student_tail(sp, fmax(a, sp.zstar));
        t = (a >= sp.zstar) ? tt : t;
    }
    t = (a == __longlong_as_double(0x7ff0000000000000LL)) ? a : t;
    const double r = copysign(t, z);
    return (z == z) ? r : z;
}

__global__ void __launch_bounds__(256)
k_student_f64(const double *__restrict__ z, double *__restrict__ t, int64_t n, const __grid_constant__ StudentParams sp)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) / 32 * 32;                     // warp-uniform trip count
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        const double x = (i < n) ? z[i] : 0.0;
        const bool tail = !(fabs(x) < sp.zstar);                    // NaN votes for the careful path too
        const bool any = __any_sync(0xffffffffu, tail);
        const double r = student_map(sp, x, any);
        if (i < n) t[i] = r;
    }
}

__global__ void __launch_bounds__(256)
k_student_f32(const float *__restrict__ z, float *__restrict__ t, int64_t n, const __grid_constant__ StudentParams sp)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) / 32 * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        const double x = (i < n) ? (double)z[i] : 0.0;
        const bool tail = !(fabs(x) < sp.zstar);
        const bool any = __any_sync(0xffffffffu, tail);
        const double r = student_map(sp, x, any);
        if (i < n) t[i] = (float)r;
    }
}

// fp64 through the TMA-in / streaming-store pipeline (qm_tma.cuh).  One vote per
// 32 samples (one per element position of the lane's slice), as in k_student_f64:
// the tail is expensive, so the vote granularity sets how often a warp pays it
// (32 P(|z| >= z*) ~ 0.3 % of votes at nu = 4).
// One vote per element position (32 samples) for the tail.  (Evaluating the
// central series of all of a lane's 2 PER samples first, to interleave their DFMA
// chains, was measured 5-7 % slower: 3771 vs 3532 us in ncu at nu = 4.)
template <int K, int KC>
struct MapStudentF64 {
    const StudentParams *sp;
    QM_DEV double one(double x) const
    {
        const bool any = __any_sync(0xffffffffu, !(fabs(x) < sp->zstar));
        return student_map<K, KC>(*sp, x, any);
    }
    template <int PER>
    QM_DEV void map_slice(double2 *a) const
    {
#if QM_STUDENT_DEFER
        // The central series of the lane's 2 PER samples (two chains at a time), then
        // the tails: each lane keeps a bit mask of its samples with |z| >= z* (or NaN)
        // and, while any lane of the warp has one left, every lane evaluates the tail
        // for its next one.  One vote per slice (2 PER x 32 samples) instead of one per
        // element position: at nu = 3 a warp meets a tail in 8.8 % of its slices and
        // then pays one tail evaluation, not one per position that has a tail lane.
        // Bitwise the same values as student_map (the tail at max(|z|, z*)).
        constexpr int NS = 2 * PER;
        double z[NS], t[NS];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            z[2 * j] = a[j].x;
            z[2 * j + 1] = a[j].y;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            t[2 * j] = student_central_k<K, KC>(*sp, fabs(z[2 * j]));
            t[2 * j + 1] = student_central_k<K, KC>(*sp, fabs(z[2 * j + 1]));
        }
        uint32_t need = 0;
#pragma unroll
        for (int k = 0; k < NS; ++k) need |= (uint32_t)(!(fabs(z[k]) < sp->zstar)) << k;
        while (__any_sync(0xffffffffu, need != 0)) {
            const int kk = __ffs(need) - 1;                          // -1: this lane has none left
            double zs = 0.0;
#pragma unroll
            for (int k = 0; k < NS; ++k) zs = (kk == k) ? z[k] : zs;
            const double tt = student_tail(*sp, fmax(fabs(zs), sp->zstar));
#pragma unroll
            for (int k = 0; k < NS; ++k) t[k] = (kk == k && fabs(z[k]) >= sp->zstar) ? tt : t[k];
            need &= need - 1;
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) t[k] = student_finish(*sp, z[k], t[k], false);
#pragma unroll
        for (int j = 0; j < PER; ++j) a[j] = make_double2(t[2 * j], t[2 * j + 1]);
#elif QM_STUDENT_PAIR == 2
        // four samples (two double2) interleaved: four independent DFMA chains
        static_assert(PER % 2 == 0, "pairs of double2");
#pragma unroll
        for (int j = 0; j < PER; j += 2) {
            const double c0 = student_central_k<K, KC>(*sp, fabs(a[j].x));
            const double c1 = student_central_k<K, KC>(*sp, fabs(a[j].y));
            const double c2 = student_central_k<K, KC>(*sp, fabs(a[j + 1].x));
            const double c3 = student_central_k<K, KC>(*sp, fabs(a[j + 1].y));
            const bool v0 = __any_sync(0xffffffffu, !(fabs(a[j].x) < sp->zstar));
            const bool v1 = __any_sync(0xffffffffu, !(fabs(a[j].y) < sp->zstar));
            const bool v2 = __any_sync(0xffffffffu, !(fabs(a[j + 1].x) < sp->zstar));
            const bool v3 = __any_sync(0xffffffffu, !(fabs(a[j + 1].y) < sp->zstar));
            a[j] = make_double2(student_finish(*sp, a[j].x, c0, v0), student_finish(*sp, a[j].y, c1, v1));
            a[j + 1] = make_double2(student_finish(*sp, a[j + 1].x, c2, v2), student_finish(*sp, a[j + 1].y, c3, v3));
        }
#elif QM_STUDENT_PAIR
        // the two central series of a double2 in one basic block (two independent
        // DFMA chains), then the two votes and tails
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const double cx = student_central_k<K, KC>(*sp, fabs(a[j].x));
            const double cy = student_central_k<K, KC>(*sp, fabs(a[j].y));
            const bool ax = __any_sync(0xffffffffu, !(fabs(a[j].x) < sp->zstar));
            const bool ay = __any_sync(0xffffffffu, !(fabs(a[j].y) < sp->zstar));
            a[j] = make_double2(student_finish(*sp, a[j].x, cx, ax), student_finish(*sp, a[j].y, cy, ay));
        }
#else
#pragma unroll
        for (int j = 0; j < PER; ++j) a[j] = make_double2(one(a[j].x), one(a[j].y));
#endif
    }
};

// 1 CTA/SM: a producer warp + 16 consumer warps, 4 stages of 32 KB (2048 double2)
// (A/B knobs: QM_STUDENT_NC consumer warps, QM_STUDENT_STAGES, QM_STUDENT_TV double2 per
// tile; measured on one box, nu = 4 K = 10 / nu = 5 K = 16 / nu = 3 K = 16 Gsamples/s:
// one by one 268 / 244 / 228; pairs 275 / 251 / 235 (kept); pairs 3 x 3072 277 / 258 /
// 181 -- a warp in the tail (13 % of a warp's tiles at nu = 3) holds a big stage
// longer; pairs 6 x 2048 276 / 256 / 235; 8 x 1024 268 / 243 / 235; fours 274 / 251 / 231)
#ifndef QM_STUDENT_NC
#define QM_STUDENT_NC 16
#endif
#ifndef QM_STUDENT_STAGES
#define QM_STUDENT_STAGES 4
#endif
#ifndef QM_STUDENT_TV
#define QM_STUDENT_TV 2048
#endif
constexpr int kStudentNC = QM_STUDENT_NC, kStudentStages = QM_STUDENT_STAGES, kStudentTileVecs = QM_STUDENT_TV;
static_assert(kStudentTileVecs % (32 * kStudentNC) == 0, "a tile splits evenly over the consumer lanes");
// the fused-moments kernel keeps 16 consumer warps and 32 KB tiles (a moment chunk of
// 65536 samples is 16 whole tiles)
constexpr int kStudentMomNC = 16, kStudentMomStages = 4, kStudentMomTileVecs = 2048;

template <int K, int KC>
__global__ void __launch_bounds__(32 * (kStudentNC + 1), 1)
k_student_f64_tl(const double *__restrict__ z, double *__restrict__ t, int64_t ntiles,
                 const __grid_constant__ StudentParams sp)
{
    tma_load_map<double2, kStudentTileVecs, kStudentStages, kStudentNC>(
        reinterpret_cast<const double2 *>(z), reinterpret_cast<double2 *>(t), ntiles, MapStudentF64<K, KC>{&sp});
}

// Config 4 with the moments fused into the map (SURVEY §8 d4 "Student-t ... with
// fused moments S_1..S_4"): each CTA owns whole QM_MOMENT_CHUNK chunks (16 tiles
// of 4096 samples, streamed by the TMA producer in order); a consumer warp maps
// its slice of every tile, stores t, and accumulates x, x^2, x^3, x^4 of its
// samples in a fixed order (tile, vector, component; the operations of
// k_moment_rows).  At the chunk's end: a fixed xor-shuffle tree per warp, the
// 16 warp partials added in warp order by warp 0, one row of 4 doubles per
// chunk -- deterministic and independent of the grid, like qm_moment_rows (the
// rows differ from its in summation order only).
template <int K, int KC>
__global__ void __launch_bounds__(32 * (kStudentMomNC + 1), 1)
k_student_moments_tl(const double *__restrict__ z, double *__restrict__ t, int64_t nchunks,
                     const __grid_constant__ StudentParams sp, double *__restrict__ rows)
{
    constexpr int TV = kStudentMomTileVecs, S = kStudentMomStages, NC = kStudentMomNC;
    constexpr int TPC = QM_MOMENT_CHUNK / (2 * TV);                 // tiles per chunk
    constexpr int PER = TV / (32 * NC);
    constexpr uint32_t TILE_BYTES = TV * 16;
    static_assert(TPC * 2 * TV == QM_MOMENT_CHUNK, "a chunk is a whole number of tiles");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *tiles = reinterpret_cast<double2 *>(smem_raw);
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ double part[NC][4];
    const double2 *z2 = reinterpret_cast<const double2 *>(z);
    double2 *t2 = reinterpret_cast<double2 *>(t);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        for (int i = 0; i < S; ++i) { mbar_init_elect(&full[i], 1); mbar_init_elect(&empty[i], NC); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {   // producer: all lanes, one elected lane issues (qm_tma.cuh)
        int st = 0;
        uint32_t ph = 0;
        int64_t k = 0;
        for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x)
            for (int i = 0; i < TPC; ++i, ++k) {
                if (k >= S) mbar_wait(&empty[st], ph ^ 1);
                elect_tma_load(&full[st], tiles + (size_t)st * TV, z2 + (c * TPC + i) * TV, TILE_BYTES);
                if (++st == S) { st = 0; ph ^= 1; }
            }
        return;
    }
    const int w = warp - 1;
    const int off = w * (PER * 32) + lane;
    const MapStudentF64<K, KC> op{&sp};
    int st = 0;
    uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
        for (int i = 0; i < TPC; ++i) {
            mbar_wait(&full[st], ph);
            const double2 *tile = tiles + (size_t)st * TV + off;
            double2 a[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) a[j] = tile[32 * j];
            fence_proxy_async();                                    // generic reads before the next TMA write
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            op.template map_slice<PER>(a);
            double2 *o = t2 + (c * TPC + i) * TV + off;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                st_stream(o + 32 * j, a[j]);
                const double v[2] = {a[j].x, a[j].y};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double v2 = __dmul_rn(v[e], v[e]);
                    s1 = __dadd_rn(s1, v[e]);
                    s2 = __dadd_rn(s2, v2);
                    s3 = __fma_rn(v2, v[e], s3);
                    s4 = __fma_rn(v2, v2, s4);
                }
            }
            if (++st == S) { st = 0; ph ^= 1; }
        }
        // fixed xor tree: every lane ends with the same warp total
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, d));
            s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, d));
            s3 = __dadd_rn(s3, __shfl_xor_sync(0xffffffffu, s3, d));
            s4 = __dadd_rn(s4, __shfl_xor_sync(0xffffffffu, s4, d));
        }
        // every lane holds the warp totals: lane l stores column l & 3 (8 lanes store
        // the same value to each address) -- no lane-dependent branch
        const int col = lane & 3;
        part[w][col] = (col == 0) ? s1 : (col == 1) ? s2 : (col == 2) ? s3 : s4;
        consumer_bar(NC * 32);
        if (w == 0) {                                               // warp-uniform
            double r = 0.0;
            for (int q = 0; q < NC; ++q) r = __dadd_rn(r, part[q][col]);
            rows[c * 4 + col] = r;                                  // same value from 8 lanes
        }
        consumer_bar(NC * 32);                                      // part[] reused by the next chunk
    }
}

}  // namespace qm

