// qm_moments.cuh -- moment sums S_k = sum_i x_i^k (the
// north star's "moment and Monte Carlo price sums" that the multi-GPU harness
// all-reduces).
//
// Determinism across launches, devices AND device counts: the global sample
// stream is cut into fixed chunks of QM_MOMENT_CHUNK elements; one CTA sums
// one chunk in a fixed order (256 strided per-thread partials + a fixed
// shared-memory tree) into one ROW of 4 doubles.  A rank that owns chunks
// [c0, c1) writes rows [c0, c1) of a zero-initialised global row matrix; an
// all-reduce(SUM) of that matrix is exact (every row has one non-zero
// contributor) and qm_reduce_rows adds the rows in a fixed tree.  The result
// is bit-identical for 1 or 8 GPUs.
#pragma once
#include <cuda_runtime.h>

#define QM_MOMENT_CHUNK 65536
#define QM_REDUCE_THREADS 1024

namespace qm {

template <typename T>
__global__ void __launch_bounds__(256)
k_moment_rows(const T *__restrict__ x, int64_t n, double *__restrict__ rows)
{
    const int64_t lo = (int64_t)blockIdx.x * QM_MOMENT_CHUNK;
    const int64_t hi = (lo + QM_MOMENT_CHUNK < n) ? lo + QM_MOMENT_CHUNK : n;
    double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
        const double v = (double)x[i];
        const double v2 = __dmul_rn(v, v);
        s1 = __dadd_rn(s1, v);
        s2 = __dadd_rn(s2, v2);
        s3 = __fma_rn(v2, v, s3);
        s4 = __fma_rn(v2, v2, s4);
    }
    __shared__ double sh[4][256];
    sh[0][threadIdx.x] = s1; sh[1][threadIdx.x] = s2; sh[2][threadIdx.x] = s3; sh[3][threadIdx.x] = s4;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
#pragma unroll
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = __dadd_rn(sh[k][threadIdx.x], sh[k][threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x < 4) rows[blockIdx.x * 4 + threadIdx.x] = sh[threadIdx.x][0];
}

// fixed-order sum of nrows rows of `ncol` doubles (ncol <= 64): thread t adds
// rows t, t+1024, ... in order, then a fixed tree over the 1024 threads; one
// block per column group of 1 column (grid = ncol).
__global__ void __launch_bounds__(QM_REDUCE_THREADS)
k_reduce_rows(const double *__restrict__ rows, int64_t nrows, int ncol, double *__restrict__ out)
{
    const int c = blockIdx.x;
    double a = 0.0;
    for (int64_t r = threadIdx.x; r < nrows; r += QM_REDUCE_THREADS) a = __dadd_rn(a, rows[r * ncol + c]);
    __shared__ double sh[QM_REDUCE_THREADS];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int w = QM_REDUCE_THREADS / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = sh[0];
}

inline int64_t moment_rows(int64_t n) { return (n + QM_MOMENT_CHUNK - 1) / QM_MOMENT_CHUNK; }

inline qm_status moment_rows_launch(const void *x, int64_t n, bool f64, double *rows, cudaStream_t s)
{
    const int64_t nr = moment_rows(n);
    if (nr == 0) return QM_OK;
    if (f64) k_moment_rows<double><<<(unsigned)nr, 256, 0, s>>>((const double *)x, n, rows);
    else k_moment_rows<float><<<(unsigned)nr, 256, 0, s>>>((const float *)x, n, rows);
    return cudaGetLastError() == cudaSuccess ? QM_OK : QM_ECUDA;
}

// sums the first `nout` of `ncol` columns
inline qm_status reduce_rows_launch(const double *rows, int64_t nrows, int ncol, int nout, double *out, cudaStream_t s)
{
    k_reduce_rows<<<nout, QM_REDUCE_THREADS, 0, s>>>(rows, nrows, ncol, out);
    return cudaGetLastError() == cudaSuccess ? QM_OK : QM_ECUDA;
}

}  // namespace qm
