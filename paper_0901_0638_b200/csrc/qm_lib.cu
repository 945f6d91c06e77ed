// qm_lib.cu -- the C ABI of libqm.so (include/qm.h): argument validation,
// launch configuration and the host-buffer pipeline.  Every element of every
// output is computed by the kernels in qm_kernels.cuh; the host only validates,
// configures and enqueues.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/qm.h"
#include "qm_kernels.cuh"
#include "qm_baselines.cuh"
#include "qm_student.cuh"
#include "qm_moments.cuh"
#include "qm_mc.cuh"
#include "qm_rode.cuh"
#include <cmath>

using namespace qm;

namespace {

int sm_count_for_current_device()
{
    static std::mutex mu;
    static std::vector<int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    std::lock_guard<std::mutex> g(mu);
    if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
    if (cache[dev] == 0) {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
        cache[dev] = sms;
    }
    return cache[dev];
}

// blocks: `per_sm` resident blocks per SM, but never more than the work needs
int grid_for(int64_t work_items, int items_per_block, int per_sm)
{
    const int sms = sm_count_for_current_device();
    int64_t g = (int64_t)(sms > 0 ? sms : 148) * per_sm;
    const int64_t need = (work_items + items_per_block - 1) / items_per_block;
    if (need < g) g = need;
    return (int)(g < 1 ? 1 : g);
}

// persistent grid: as many blocks as can be resident at once (one wave), but
// never more than the work needs
template <typename K>
int grid_resident(K kernel, int threads, int64_t work_items, int items_per_block)
{
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return grid_for(work_items, items_per_block, per_sm);
}

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

qm_status launched()
{
    return cudaGetLastError() == cudaSuccess ? QM_OK : QM_ECUDA;
}

bool bad_ptrs(const void *a, const void *b, int64_t n) { return n > 0 && (a == nullptr || b == nullptr); }

// A/B diagnostic knobs, read once per process (function-local statics: their
// initialisation is thread-safe)
int env_int(const char *name, int dflt, int lo, int hi)
{
    const char *e = getenv(name);
    const int v = e ? atoi(e) : dflt;
    return (v < lo || v > hi) ? dflt : v;
}

// QM_STREAM_PATH: "ldg" forces the register-pipelined LDG kernels, "tma" the
// in-place TMA load/store pipeline; default "tl" (TMA in, streaming stores out)
int stream_path()
{
    static const int p = [] {
        const char *e = getenv("QM_STREAM_PATH");
        return (e && strcmp(e, "ldg") == 0) ? 0 : (e && strcmp(e, "tma") == 0) ? 1 : 2;
    }();
    return p;
}
bool tma_enabled() { return stream_path() != 0; }

// fp32 elementwise map: whole tiles through the TMA pipeline (persistent CTAs),
// the remainder (< 1 tile) and misaligned arrays through the LDG kernel.
// Programmatic dependent launch: the kernel may start while the previous grid on
// the stream drains (its prologue overlaps that grid's tail and the launch gap);
// it waits in pdl_begin() (qm_tma.cuh) before touching global memory.  QM_PDL=0
// launches normally (A/B).
bool pdl_enabled()
{
    static const bool on = [] {
        const char *e = getenv("QM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename K, typename... Args>
void launch_pdl(K kernel, unsigned grid, unsigned block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <class CFG, typename KT, typename KL>
qm_status launch_stream_f32(KT ktma, KL kldg, const float *in, float *out, int64_t n, cudaStream_t s)
{
    const int vec = aligned16(in) && aligned16(out);
    // below 2^23 samples the LDG kernel balances better (measured: 2^20 273 vs 262,
    // 2^22 454 vs 442 Gsamples/s; from 2^23 the pipeline wins, 569 vs 491)
    int64_t ntiles = (vec && tma_enabled() && n >= ((int64_t)1 << 23)) ? n / CFG::TILE : 0;
    if (ntiles > 0) {
        const size_t smem = (size_t)CFG::STAGES * CFG::TILE * sizeof(float);
        if (cudaFuncSetAttribute(ktma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return QM_ECUDA;
        const int sms = sm_count_for_current_device();
        int64_t g = (int64_t)(sms > 0 ? sms : 148) * CFG::MINB;
        if (ntiles < g) g = ntiles;
        launch_pdl(ktma, (unsigned)g, CFG::THREADS, smem, s, in, out, ntiles);
    }
    const int64_t done = ntiles * CFG::TILE, rest = n - done;
    if (rest > 0) {
        const int g = grid_for(rest, kThreads * 8, 8);
        launch_pdl(kldg, (unsigned)g, kThreads, 0, s, in + done, out + done, rest, vec);
    }
    return launched();
}

// QM_TL_CFG=J|K|L|M selects the TMA-in/STG-out shape (default L)
char tl_cfg()
{
    static const char c = [] {
        const char *e = getenv("QM_TL_CFG");
        return (e && e[0] >= 'J' && e[0] <= 'M') ? e[0] : 'L';
    }();
    return c;
}

template <int ALG>
qm_status normal_f32(const float *u, float *z, int64_t n, cudaStream_t s)
{
    if constexpr (ALG != ALG_BREAKLESS)     // A/B shapes only for the headline formula
        return launch_stream_f32<TlCfgL>(k_normal_f32_tl<ALG, TlCfgL>, k_normal_f32<ALG>, u, z, n, s);
    if (stream_path() == 2) {
        switch (tl_cfg()) {
        case 'K': return launch_stream_f32<TlCfgK>(k_normal_f32_tl<ALG, TlCfgK>, k_normal_f32<ALG>, u, z, n, s);
        case 'L': return launch_stream_f32<TlCfgL>(k_normal_f32_tl<ALG, TlCfgL>, k_normal_f32<ALG>, u, z, n, s);
        case 'M': return launch_stream_f32<TlCfgM>(k_normal_f32_tl<ALG, TlCfgM>, k_normal_f32<ALG>, u, z, n, s);
        default: return launch_stream_f32<TlCfgJ>(k_normal_f32_tl<ALG, TlCfgJ>, k_normal_f32<ALG>, u, z, n, s);
        }
    }
    // QM_STREAM_PATH=tma: the first (in-place, bulk-store) pipeline, shape B
    return launch_stream_f32<TmaCfgB>(k_normal_f32_tma<ALG, TmaCfgB>, k_normal_f32<ALG>, u, z, n, s);
}

template <int ALG>
qm_status exp2n_f32(const float *v, float *z, int64_t n, cudaStream_t s)
{
    if (stream_path() == 2)
        return launch_stream_f32<TlCfgJ>(k_exp2n_f32_tl<ALG, TlCfgJ>, k_exp2n_f32<ALG>, v, z, n, s);
    return launch_stream_f32<TmaCfgB>(k_exp2n_f32_tma<ALG, TmaCfgB>, k_exp2n_f32<ALG>, v, z, n, s);
}

#define QM_ALG_LAST QM_TWO_REGION

bool breakless_family(qm_algorithm a) { return a == QM_BREAKLESS || a == QM_BREAKLESS77 || a == QM_BREAKLESS_TAIL; }

// which algorithms qm_normal_quantile evaluates in which precision (qm.h)
bool normal_supported(qm_precision p, qm_algorithm a)
{
    if (p == QM_F32) return breakless_family(a) || a == QM_BREAKLESS88 || a == QM_TWO_REGION;
    return a != QM_TWO_REGION;
}

// f(std::integral_constant<int, ALG>) for the breakless family, else QM_EUNSUPPORTED
template <typename F>
qm_status with_breakless(qm_algorithm a, F f)
{
    switch (a) {
    case QM_BREAKLESS: return f(std::integral_constant<int, ALG_BREAKLESS>{});
    case QM_BREAKLESS77: return f(std::integral_constant<int, ALG_BREAKLESS77>{});
    case QM_BREAKLESS_TAIL: return f(std::integral_constant<int, ALG_BREAKLESS_TAIL>{});
    default: return QM_EUNSUPPORTED;
    }
}

// The validated Student configurations (qm.h): the paper's nu = 4, K = 10 with its
// crossover 3.93473, and nu = 3, 5, 10 with K = 16 and the min-max
// crossovers of reading R13 (tests/golden/student_crossover.txt).  zstar <= 0
// selects from this table; a caller-supplied zstar > 0 is accepted for any
// 1 <= nu <= 20, 1 <= K <= QM_STUDENT_KMAX (the caller owns the crossover).
struct StudentDefault { double nu; int K; double zstar; };
constexpr StudentDefault kStudentTable[] = {{4.0, 10, 3.93473}, {3.0, 16, 3.5667}, {5.0, 16, 4.6506}, {10.0, 16, 6.9584}};

qm_status student_setup(double nu, int K, double zstar, StudentParams *sp)
{
    if (!(nu > 0.0) || K < 1 || K > QM_STUDENT_KMAX || zstar != zstar) return QM_EINVAL;
    if (!(zstar > 0.0)) {
        zstar = 0.0;
        for (const StudentDefault &d : kStudentTable)
            if (d.nu == nu && d.K == K) zstar = d.zstar;
        if (zstar == 0.0) return QM_EUNSUPPORTED;   // no validated crossover for (nu, K)
    }
    // nu in [2, 20]: the recurrence is ill-conditioned beyond 20 (R22); below 2 the
    // tail's w^(-1/nu) amplifies the double erfcx's few-ulp error by 1/nu past the
    // 2-ulp contract (measured 2.19 ulp at nu = 1.5, 1.79 at nu = 2)
    if (nu < 2.0 || nu > 20.0) return QM_EUNSUPPORTED;
    return student_params(nu, K, zstar, sp) ? QM_OK : QM_EUNSUPPORTED;
}

}  // namespace

// fp64 breakless map: the TMA-in / streaming-store pipeline for large aligned n,
// else (and for the remainder) the LDG kernel -- every fp64 breakless formula
template <int ALG>
qm_status normal_f64(const double *ud, double *zd, int64_t n, int vec, cudaStream_t s)
{
    // the pipeline only pays with several tiles per CTA (small n: the LDG kernel
    // balances better, e.g. config 1's 2^20: 55 vs 40 Gsamples/s)
    if (vec && stream_path() == 2 && n >= ((int64_t)1 << 23)) {
        static const int cfg = env_int("QM_TL64_CFG", 2, 0, 2);   // 0 = LDG kernel, 1 = TlF64A, 2 = TlF64B (default: +2.3 % measured)
        if (cfg > 0) {
            auto go = [&](auto k, int tile, int threads, size_t smem) {
                const int64_t ntiles = n / tile;
                if (ntiles > 0) {
                    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                        return QM_ECUDA;
                    const int sms = sm_count_for_current_device();
                    const int64_t gg = ntiles < (sms > 0 ? sms : 148) ? ntiles : (sms > 0 ? sms : 148);
                    k<<<(int)gg, threads, smem, s>>>(ud, zd, ntiles);
                }
                const int64_t done = ntiles * tile;
                if (n > done)
                    k_normal_f64<ALG><<<grid_for(n - done, kThreads * 2, 8), kThreads, 0, s>>>(ud + done, zd + done,
                                                                                      n - done, 1);
                return launched();
            };
            if (cfg == 2) return go(k_normal_f64_tl<ALG, TlF64B>, TlF64B::TILE, TlF64B::THREADS,
                                    (size_t)TlF64B::STAGES * TlF64B::TILE_VECS * 16);
            return go(k_normal_f64_tl<ALG, TlF64A>, TlF64A::TILE, TlF64A::THREADS,
                      (size_t)TlF64A::STAGES * TlF64A::TILE_VECS * 16);
        }
    }
    k_normal_f64<ALG><<<grid_for(n, kThreads * 2, 8), kThreads, 0, s>>>(ud, zd, n, vec);
    return launched();
}

extern "C" {

int qm_abi_version(void) { return QM_ABI_VERSION; }

double qm_student_default_crossover(double nu, int K)
{
    for (const StudentDefault &d : kStudentTable)
        if (d.nu == nu && d.K == K) return d.zstar;
    return 0.0;
}

const char *qm_status_string(qm_status s)
{
    switch (s) {
    case QM_OK: return "ok";
    case QM_EINVAL: return "invalid argument";
    case QM_EUNSUPPORTED: return "unsupported combination";
    case QM_ECUDA: return "CUDA launch failure";
    }
    return "unknown status";
}

int qm_device_sm_count(void) { return sm_count_for_current_device(); }

qm_status qm_normal_quantile(const void *u, void *z, int64_t n, qm_precision p, qm_algorithm alg, void *stream)
{
    if (n < 0 || bad_ptrs(u, z, n)) return QM_EINVAL;
    if (p != QM_F32 && p != QM_F64) return QM_EINVAL;
    if (alg < QM_BREAKLESS || alg > QM_ALG_LAST) return QM_EINVAL;
    if (!normal_supported(p, alg)) return QM_EUNSUPPORTED;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int vec = aligned16(u) && aligned16(z);
    if (p == QM_F32) {
        if (alg == QM_BREAKLESS88) return normal_f32<ALG_F88>((const float *)u, (float *)z, n, s);
        if (alg == QM_TWO_REGION) return normal_f32<ALG_TWO_REGION>((const float *)u, (float *)z, n, s);
        return with_breakless(alg, [&](auto A) { return normal_f32<decltype(A)::value>((const float *)u, (float *)z, n, s); });
    }
    const double *ud = (const double *)u;
    double *zd = (double *)z;
    switch (alg) {
    case QM_AS241: k_branchy_f64<ALG_AS241><<<grid_for(n, kThreads, 8), kThreads, 0, s>>>(ud, zd, n); return launched();
    case QM_ACKLAM: k_branchy_f64<ALG_ACKLAM><<<grid_for(n, kThreads, 8), kThreads, 0, s>>>(ud, zd, n); return launched();
    case QM_ACKLAM_REFINED:
        k_branchy_f64<ALG_ACKLAM_REF><<<grid_for(n, kThreads, 8), kThreads, 0, s>>>(ud, zd, n);
        return launched();
    case QM_MORO: k_branchy_f64<ALG_MORO><<<grid_for(n, kThreads, 8), kThreads, 0, s>>>(ud, zd, n); return launched();
    case QM_BREAKLESS1212: return normal_f64<ALG_F1212>(ud, zd, n, vec, s);
    case QM_BREAKLESS88: return normal_f64<ALG_F88>(ud, zd, n, vec, s);
    case QM_TWO_REGION: return QM_EUNSUPPORTED;
    default: break;
    }
    return with_breakless(alg, [&](auto A) { return normal_f64<decltype(A)::value>(ud, zd, n, vec, s); });
}

qm_status qm_normal_quantile_plain(const void *u, void *z, int64_t n, qm_algorithm alg, void *stream)
{
    if (n < 0 || bad_ptrs(u, z, n) || alg < QM_BREAKLESS || alg > QM_ALG_LAST) return QM_EINVAL;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const double *ud = (const double *)u;
    double *zd = (double *)z;
    const int g = grid_for(n, kThreads, 8);
    switch (alg) {
    case QM_BREAKLESS: k_plain_f64<ALG_BREAKLESS><<<g, kThreads, 0, s>>>(ud, zd, n); break;
    case QM_BREAKLESS77: k_plain_f64<ALG_BREAKLESS77><<<g, kThreads, 0, s>>>(ud, zd, n); break;
    case QM_AS241: k_plain_f64<ALG_AS241><<<g, kThreads, 0, s>>>(ud, zd, n); break;
    case QM_ACKLAM: k_plain_f64<ALG_ACKLAM><<<g, kThreads, 0, s>>>(ud, zd, n); break;
    case QM_ACKLAM_REFINED: k_plain_f64<ALG_ACKLAM_REF><<<g, kThreads, 0, s>>>(ud, zd, n); break;
    case QM_MORO: k_plain_f64<ALG_MORO><<<g, kThreads, 0, s>>>(ud, zd, n); break;
    default: return QM_EUNSUPPORTED;
    }
    return launched();
}

qm_status qm_normal_antithetic(const void *u, void *z, int64_t n, qm_precision p, qm_algorithm alg, void *stream)
{
    if (n < 0 || bad_ptrs(u, z, n)) return QM_EINVAL;
    if ((p != QM_F32 && p != QM_F64) || alg < QM_BREAKLESS || alg > QM_ALG_LAST) return QM_EINVAL;
    if (!breakless_family(alg)) return QM_EUNSUPPORTED;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (p == QM_F32) {
        const int vec = aligned16(u) && aligned16(z);
        return with_breakless(alg, [&](auto A) {
            constexpr int ALG = decltype(A)::value;
            const float *uf = (const float *)u;
            float *zf = (float *)z;
            int64_t done = 0;
            if (vec && stream_path() == 2 && n >= ((int64_t)1 << 23)) {   // whole tiles: TMA pipeline
                constexpr int64_t TILE = 8192;
                const int64_t ntiles = n / TILE;
                const size_t smem = (size_t)4 * TILE * sizeof(float);
                auto k = k_antithetic_f32_tl<ALG>;
                if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                    return QM_ECUDA;
                const int sms = sm_count_for_current_device();
                const int64_t gg = ntiles < (sms > 0 ? sms : 148) ? ntiles : (sms > 0 ? sms : 148);
                k<<<(int)gg, 32 * 17, smem, s>>>(uf, zf, ntiles);
                done = ntiles * TILE;
            }
            if (n > done) {
                const int g = grid_for(n - done, kThreads * 4, 8);
                k_antithetic_f32<ALG><<<g, kThreads, 0, s>>>(uf + done, zf + 2 * done, n - done, vec);
            }
            return launched();
        });
    }
    const int g = grid_for(n, kThreads, 8);
    return with_breakless(alg, [&](auto A) {
        k_antithetic_f64<decltype(A)::value><<<g, kThreads, 0, s>>>((const double *)u, (double *)z, n);
        return launched();
    });
}

#ifndef QM_F64_FUSED_V
#define QM_F64_FUSED_V 1   // A/B: Philox blocks (2 samples each) per lane per chunk of the fused fp64 sampler
#endif
static qm_status philox_launch(void *z, int64_t n, qm_precision p, int mode, qm_algorithm alg,
                               uint64_t seed, uint64_t c0, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    const int vec = aligned16(z);
    // on the odd grid v < 17 (fp32) / 37 (fp64) < vc: the tail composite is the
    // plain rational there, so QM_BREAKLESS_TAIL runs the QM_BREAKLESS kernel
    if (alg == QM_BREAKLESS_TAIL) alg = QM_BREAKLESS;
    if (p == QM_F32) {
        const int64_t nb = (n + 3) / 4;
        if (mode == 0) {
            auto k = k_philox_f32<0, ALG_BREAKLESS>;
            launch_pdl(k, grid_resident(k, kThreads, nb, kThreads * 2), kThreads, 0, s, (float *)z, n, seed, c0, vec);
        } else if (alg == QM_BREAKLESS) {
            auto k = k_philox_f32<1, ALG_BREAKLESS>;
            launch_pdl(k, grid_resident(k, kThreads, nb, kThreads * 2), kThreads, 0, s, (float *)z, n, seed, c0, vec);
        } else {
            auto k = k_philox_f32<1, ALG_BREAKLESS77>;
            launch_pdl(k, grid_resident(k, kThreads, nb, kThreads * 2), kThreads, 0, s, (float *)z, n, seed, c0, vec);
        }
    } else {
        const int g = grid_for((n + 1) / 2, kThreads, 8);
        if (mode == 0) launch_pdl(k_philox_f64<0, ALG_BREAKLESS>, g, kThreads, 0, s, (double *)z, n, seed, c0, vec);
        else if (alg == QM_BREAKLESS)
            launch_pdl(k_philox_f64<1, ALG_BREAKLESS, QM_F64_FUSED_V>, g, kThreads, 0, s, (double *)z, n, seed, c0, vec);
        else launch_pdl(k_philox_f64<1, ALG_BREAKLESS77>, g, kThreads, 0, s, (double *)z, n, seed, c0, vec);
    }
    return launched();
}

qm_status qm_philox_uniform(void *u, int64_t n, qm_precision p, uint64_t seed, uint64_t counter_offset, void *stream)
{
    if (n < 0 || (n > 0 && u == nullptr) || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (n == 0) return QM_OK;
    return philox_launch(u, n, p, 0, QM_BREAKLESS, seed, counter_offset, stream);
}

qm_status qm_normal_philox(void *z, int64_t n, qm_precision p, qm_algorithm alg, uint64_t seed,
                           uint64_t counter_offset, void *stream)
{
    if (n < 0 || (n > 0 && z == nullptr) || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (alg < QM_BREAKLESS || alg > QM_ALG_LAST) return QM_EINVAL;
    if (!breakless_family(alg)) return QM_EUNSUPPORTED;
    if (n == 0) return QM_OK;
    return philox_launch(z, n, p, 1, alg, seed, counter_offset, stream);
}

qm_status qm_recycle_exp_to_normal(const void *v, void *z, int64_t n, qm_precision p, qm_algorithm alg, void *stream)
{
    if (n < 0 || bad_ptrs(v, z, n)) return QM_EINVAL;
    if ((p != QM_F32 && p != QM_F64) || alg < QM_BREAKLESS || alg > QM_ALG_LAST) return QM_EINVAL;
    if (!breakless_family(alg)) return QM_EUNSUPPORTED;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (p == QM_F32)
        return with_breakless(alg, [&](auto A) { return exp2n_f32<decltype(A)::value>((const float *)v, (float *)z, n, s); });
    const int g = grid_for(n, kThreads, 8);
    return with_breakless(alg, [&](auto A) {
        k_exp2n_f64<decltype(A)::value><<<g, kThreads, 0, s>>>((const double *)v, (double *)z, n);
        return launched();
    });
}

qm_status qm_recycle_normal_to_t(const void *z, void *t, int64_t n, qm_precision p, double nu, int K,
                                 double zstar, void *stream)
{
    if (n < 0 || bad_ptrs(z, t, n) || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    StudentParams sp;
    const qm_status st = student_setup(nu, K, zstar, &sp);
    if (st != QM_OK) return st;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t done = 0;
    if (p == QM_F64 && aligned16(z) && aligned16(t) && sp.kc == 3 && (K == 10 || K == 16)) {
        // whole tiles through the TMA pipeline with the series unrolled at compile time
        constexpr int64_t TILE = 2 * kStudentTileVecs;
        const int64_t ntiles = n / TILE;
        if (ntiles > 0) {
            const size_t smem = (size_t)kStudentStages * kStudentTileVecs * 16;
            auto k = (K == 10) ? k_student_f64_tl<10, 3> : k_student_f64_tl<16, 3>;
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return QM_ECUDA;
            const int sms = sm_count_for_current_device();
            const int64_t g = ntiles < (sms > 0 ? sms : 148) ? ntiles : (sms > 0 ? sms : 148);
            k<<<(int)g, 32 * (kStudentNC + 1), smem, s>>>((const double *)z, (double *)t, ntiles, sp);
            done = ntiles * TILE;
        }
    }
    if (n > done) {
        const int g = grid_for(n - done, kThreads * 2, 8);
        if (p == QM_F64) k_student_f64<<<g, kThreads, 0, s>>>((const double *)z + done, (double *)t + done, n - done, sp);
        else k_student_f32<<<g, kThreads, 0, s>>>((const float *)z, (float *)t, n, sp);
    }
    return launched();
}

qm_status qm_recycle_normal_to_t_moments(const void *z, void *t, int64_t n, qm_precision p, double nu, int K,
                                         double zstar, double *rows, void *stream)
{
    if (n < 0 || bad_ptrs(z, t, n) || (n > 0 && rows == nullptr) || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    StudentParams sp;
    const qm_status st = student_setup(nu, K, zstar, &sp);
    if (st != QM_OK) return st;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t done = 0;
    if (p == QM_F64 && aligned16(z) && aligned16(t) && sp.kc == 3 && (K == 10 || K == 16)) {
        // whole chunks: the map and the moment rows in one pass
        const int64_t nchunks = n / QM_MOMENT_CHUNK;
        if (nchunks > 0) {
            const size_t smem = (size_t)kStudentMomStages * kStudentMomTileVecs * 16;
            auto k = (K == 10) ? k_student_moments_tl<10, 3> : k_student_moments_tl<16, 3>;
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return QM_ECUDA;
            const int sms = sm_count_for_current_device();
            const int64_t g = nchunks < (sms > 0 ? sms : 148) ? nchunks : (sms > 0 ? sms : 148);
            k<<<(int)g, 32 * (kStudentMomNC + 1), smem, s>>>((const double *)z, (double *)t, nchunks, sp, rows);
            done = nchunks * QM_MOMENT_CHUNK;
        }
    }
    if (n > done) {   // the rest: map, then the rows of the remaining chunks
        const size_t es = (p == QM_F64) ? 8 : 4;
        const qm_status r = qm_recycle_normal_to_t((const char *)z + done * es, (char *)t + done * es, n - done, p, nu,
                                                   K, zstar, stream);
        if (r != QM_OK) return r;
        return moment_rows_launch((const char *)t + done * es, n - done, p == QM_F64, rows + 4 * (done / QM_MOMENT_CHUNK), s);
    }
    return launched();
}

qm_status qm_exp_target_table(qm_target kind, const double *params, double *table_dev)
{
    if (params == nullptr || table_dev == nullptr || (kind != QM_TARGET_HYPERBOLIC && kind != QM_TARGET_VG))
        return QM_EINVAL;
    // a valid VG (lambda > 0, alpha > |beta|) outside the supported lambda range:
    // lambda < 1 is out of scope (H(0) diverges), 1 < lambda < 1.1 needs the
    // "many steps near v = 0" P:395 warns of, and lambda > 30 is untested
    if (kind == QM_TARGET_VG && params[0] > 0.0 && params[1] > std::fabs(params[2])) {
        const double lam = params[0];
        const bool integer = lam == std::floor(lam);
        if (lam < 1.0 || lam > QM_RODE_VG_LAMBDA_MAX || (!integer && lam < QM_RODE_VG_LAMBDA_MIN_REAL))
            return QM_EUNSUPPORTED;
    }
    static_assert(QM_RODE_TABLE_DOUBLES == QM_RODE_TABLE_LEN, "qm.h and qm_rode_params.h disagree");
    std::vector<double> tab(QM_RODE_TABLE_DOUBLES);
    if (!rode_table_build((int)kind, params, tab.data())) return QM_EINVAL;
    return cudaMemcpy(table_dev, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess
               ? QM_OK : QM_ECUDA;
}

// SIDES = 1: an odd map (the Student table, R35) -- one side's nodes staged, a larger ring
extern "C++" {
template <int SIDES>
static qm_status rode_map_launch(const void *v, void *x, int64_t n, qm_precision p, const double *tab, void *stream)
{
    if (n < 0 || bad_ptrs(v, x, n) || tab == nullptr || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    using C = RodeTl<SIDES>;
    // large aligned arrays: whole tiles through the TMA pipeline, the rest below
    int64_t done = 0;
    if (aligned16(v) && aligned16(x) && n >= ((int64_t)1 << 23)) {
        const int64_t tile = (int64_t)C::tile_vecs * (p == QM_F64 ? 2 : 4);
        const int64_t ntiles = n / tile;
        const int sms = sm_count_for_current_device();
        const int gg = (int)(ntiles < (sms > 0 ? sms : 148) ? ntiles : (sms > 0 ? sms : 148));
        auto tl = [&](auto k, auto *vv, auto *xx) {
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes) != cudaSuccess)
                return QM_ECUDA;
            k<<<gg, 32 * (kRodeTlNC + 1), C::smem_bytes, s>>>(vv, xx, ntiles, tab);
            return QM_OK;
        };
        const qm_status r = (p == QM_F64) ? tl(k_rode_map_tl<double2, SIDES>, (const double2 *)v, (double2 *)x)
                                          : tl(k_rode_map_tl<float4, SIDES>, (const float4 *)v, (float4 *)x);
        if (r != QM_OK) return r;
        done = ntiles * tile;
        if (done == n) return launched();
        const size_t es = (p == QM_F64) ? 8 : 4;
        v = (const char *)v + done * es;
        x = (char *)x + done * es;
        n -= done;
    }
    // persistent: one 512-thread CTA per SM, each staging the centre nodes
    const int g = grid_for(n, 512 * 4, 1);
    const size_t smem = rode_smem_bytes<SIDES>(kRodeSmemNodes);
    auto go = [&](auto k, auto *vv, auto *xx) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return QM_ECUDA;
        k<<<g, 512, smem, s>>>(vv, xx, n, tab);
        return launched();
    };
    if (p == QM_F64) return go(k_rode_map<double, SIDES>, (const double *)v, (double *)x);
    return go(k_rode_map<float, SIDES>, (const float *)v, (float *)x);
}
}  // extern "C++"

qm_status qm_recycle_exp_to_hyperbolic(const void *v, void *x, int64_t n, qm_precision p, const double *table_dev,
                                       void *stream)
{
    return rode_map_launch<2>(v, x, n, p, table_dev, stream);
}

qm_status qm_recycle_exp_to_vg(const void *v, void *x, int64_t n, qm_precision p, const double *table_dev,
                               void *stream)
{
    return rode_map_launch<2>(v, x, n, p, table_dev, stream);
}

qm_status qm_normal_target_table(qm_target kind, const double *params, double *table_dev)
{
    if (params == nullptr || table_dev == nullptr || kind != QM_TARGET_STUDENT || !(params[0] > 0.0)) return QM_EINVAL;
    if (params[0] < QM_RODE_STUDENT_NU_MIN || params[0] > QM_RODE_STUDENT_NU_MAX) return QM_EUNSUPPORTED;
    std::vector<double> tab(QM_RODE_TABLE_DOUBLES);
    if (!rode_student_table_build(params[0], tab.data())) return QM_EINVAL;
    return cudaMemcpy(table_dev, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess
               ? QM_OK : QM_ECUDA;
}

qm_status qm_recycle_normal_to_t_rode(const void *z, void *t, int64_t n, qm_precision p, const double *table_dev,
                                      void *stream)
{
    return rode_map_launch<1>(z, t, n, p, table_dev, stream);
}

qm_status qm_exp_base_quantile(const void *u, void *v, int64_t n, qm_precision p, const double *table_dev,
                               void *stream)
{
    if (n < 0 || bad_ptrs(u, v, n) || table_dev == nullptr || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int g = grid_for(n, kThreads, 8);
    if (p == QM_F64) k_exp_base_quantile<double><<<g, kThreads, 0, s>>>((const double *)u, (double *)v, n, table_dev);
    else k_exp_base_quantile<float><<<g, kThreads, 0, s>>>((const float *)u, (float *)v, n, table_dev);
    return launched();
}

qm_status qm_exp_target_philox(void *x, int64_t n, qm_precision p, const double *table_dev, uint64_t seed,
                               uint64_t counter_offset, void *stream)
{
    if (n < 0 || (n > 0 && x == nullptr) || table_dev == nullptr || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (n == 0) return QM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    auto go = [&](auto k, auto *xx, int64_t nb) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRodeSmemBytes) != cudaSuccess)
            return QM_ECUDA;
        k<<<grid_for(nb, 512 * 2, 1), 512, kRodeSmemBytes, s>>>(xx, n, seed, counter_offset, table_dev);
        return launched();
    };
    if (p == QM_F64) return go(k_rode_philox<double>, (double *)x, (n + 1) / 2);
    return go(k_rode_philox<float>, (float *)x, (n + 3) / 4);
}

int64_t qm_mc_row_count(int64_t n) { return n > 0 ? (n + QM_MC_CHUNK - 1) / QM_MC_CHUNK : 0; }

qm_status qm_mc_european_call(int64_t n, uint64_t seed, uint64_t counter_offset, const qm_mc_params *params,
                              double *rows, void *stream)
{
    if (n < 0 || params == nullptr || (n > 0 && rows == nullptr)) return QM_EINVAL;
    const int nk = params->nstrikes;
    if (nk < 1 || nk > QM_MC_MAXK || !(params->S0 > 0.0) || !(params->sigma >= 0.0) || !(params->T >= 0.0))
        return QM_EINVAL;
    if (n == 0) return QM_OK;
    McParams mp;
    mp.a = (float)(log(params->S0) + (params->r - 0.5 * params->sigma * params->sigma) * params->T);
    mp.b = (float)(params->sigma * sqrt(params->T));
    mp.nk = nk;
    for (int j = 0; j < QM_MC_MAXK; ++j) mp.K[j] = (j < nk) ? (float)params->strikes[j] : 0.0f;
    const size_t smem = (size_t)2 * nk * 256 * sizeof(double);
    const int64_t nrows = qm_mc_row_count(n);
    cudaStream_t s = (cudaStream_t)stream;
    auto go = [&](auto kern) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return QM_ECUDA;
        kern<<<(unsigned)nrows, 256, smem, s>>>(n, seed, counter_offset, mp, rows);
        return launched();
    };
    if (nk <= 8) return go(k_mc_call<8>);
    if (nk == 17) return go(k_mc_call<17, 1, 3, true>);
    if (nk <= 17) return go(k_mc_call<17, 1, 3>);
    return go(k_mc_call<32>);
}

int64_t qm_moment_row_count(int64_t n) { return n > 0 ? moment_rows(n) : 0; }

qm_status qm_moment_rows(const void *x, int64_t n, qm_precision p, double *rows, void *stream)
{
    if (n < 0 || (n > 0 && (x == nullptr || rows == nullptr)) || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (n == 0) return QM_OK;
    return moment_rows_launch(x, n, p == QM_F64, rows, (cudaStream_t)stream);
}

qm_status qm_reduce_rows(const double *rows, int64_t nrows, int ncol, double *out, void *stream)
{
    if (nrows < 0 || ncol < 1 || ncol > 64 || out == nullptr || (nrows > 0 && rows == nullptr)) return QM_EINVAL;
    return reduce_rows_launch(rows, nrows, ncol, ncol, out, (cudaStream_t)stream);
}

qm_status qm_moments(const void *x, int64_t n, qm_precision p, int kmax, double *sums_dev, double *rows_ws,
                     void *stream)
{
    if (n < 0 || (n > 0 && (x == nullptr || rows_ws == nullptr)) || sums_dev == nullptr) return QM_EINVAL;
    if ((p != QM_F32 && p != QM_F64) || kmax < 1 || kmax > 4) return QM_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    qm_status r = (n > 0) ? moment_rows_launch(x, n, p == QM_F64, rows_ws, s) : QM_OK;
    if (r != QM_OK) return r;
    return reduce_rows_launch(rows_ws, moment_rows(n), 4, kmax, sums_dev, s);
}

// ------------------------------------------------------------------ e2e
namespace {
constexpr int kHostPipeMax = 4;
struct HostPipe {
    cudaStream_t st[kHostPipeMax] = {};
    void *din[kHostPipeMax] = {}, *dout[kHostPipeMax] = {};
    size_t cap = 0;   // bytes per buffer
    int dev = -1, np = 0;
    ~HostPipe()
    {
        for (int i = 0; i < kHostPipeMax; ++i) {
            if (din[i]) cudaFree(din[i]);
            if (dout[i]) cudaFree(dout[i]);
            if (st[i]) cudaStreamDestroy(st[i]);
        }
    }
};
thread_local HostPipe g_pipe;
}  // namespace

qm_status qm_normal_quantile_host(const void *u_host, void *z_host, int64_t n, qm_precision p, qm_algorithm alg)
{
    if (n < 0 || bad_ptrs(u_host, z_host, n) || (p != QM_F32 && p != QM_F64)) return QM_EINVAL;
    if (alg < QM_BREAKLESS || alg > QM_ALG_LAST) return QM_EINVAL;
    if (!normal_supported(p, alg)) return QM_EUNSUPPORTED;
    if (n == 0) return QM_OK;
    const size_t es = (p == QM_F32) ? 4 : 8;
    // QM_HOST_STREAMS (2..4) x chunks of 2^QM_HOST_CHUNK_LOG2 elements (A/B knobs)
    static const int np_cfg = env_int("QM_HOST_STREAMS", 2, 2, kHostPipeMax);
    static const int lg_cfg = env_int("QM_HOST_CHUNK_LOG2", 24, 20, 27);
    const int NP = np_cfg;
    const int64_t chunk = (int64_t)1 << lg_cfg;             // elements per pipeline stage
    const size_t need = (size_t)chunk * es;
    HostPipe &hp = g_pipe;
    int dev = 0;
    cudaGetDevice(&dev);
    if (hp.dev != dev || hp.cap < need || hp.np != NP) {
        hp.~HostPipe();
        new (&hp) HostPipe();
        for (int i = 0; i < NP; ++i) {
            if (cudaStreamCreateWithFlags(&hp.st[i], cudaStreamNonBlocking) != cudaSuccess) return QM_ECUDA;
            if (cudaMalloc(&hp.din[i], need) != cudaSuccess || cudaMalloc(&hp.dout[i], need) != cudaSuccess)
                return QM_ECUDA;
        }
        hp.cap = need;
        hp.dev = dev;
        hp.np = NP;
    }
    const char *hu = (const char *)u_host;
    char *hz = (char *)z_host;
    int k = 0;
    for (int64_t off = 0; off < n; off += chunk, k = (k + 1) % NP) {
        const int64_t m = (n - off < chunk) ? (n - off) : chunk;
        cudaStream_t s = hp.st[k];
        if (cudaMemcpyAsync(hp.din[k], hu + off * es, m * es, cudaMemcpyHostToDevice, s) != cudaSuccess) return QM_ECUDA;
        qm_status r = qm_normal_quantile(hp.din[k], hp.dout[k], m, p, alg, s);
        if (r != QM_OK) return r;
        if (cudaMemcpyAsync(hz + off * es, hp.dout[k], m * es, cudaMemcpyDeviceToHost, s) != cudaSuccess) return QM_ECUDA;
    }
    for (int i = 0; i < NP; ++i)
        if (cudaStreamSynchronize(hp.st[i]) != cudaSuccess) return QM_ECUDA;
    return QM_OK;
}

}  // extern "C"
