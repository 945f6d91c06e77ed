// qm_moments.cuh -- moment sums S_k = sum_i x_i^k (the
// north star's "moment and Monte Carlo price sums" that the multi-GPU harness
// all-reduces).  Deterministic: the array is cut into QM_MOMENT_PARTS fixed
// contiguous parts (independent of the device and the launch), each part is
// summed in a fixed order (per-thread strided partials + a fixed shared-memory
// tree), and a second single-block kernel adds the part sums in a fixed tree.
#pragma once
#include <cuda_runtime.h>

#define QM_MOMENT_PARTS 1024

namespace qm {

template <typename T>
__global__ void __launch_bounds__(256)
k_moment_parts(const T *__restrict__ x, int64_t n, int kmax, double *__restrict__ parts)
{
    const int64_t b = blockIdx.x;
    const int64_t lo = (n * b) / QM_MOMENT_PARTS, hi = (n * (b + 1)) / QM_MOMENT_PARTS;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double v = (double)x[i];
        const double v2 = v * v;
        s[0] += v;
        s[1] += v2;
        s[2] = __fma_rn(v2, v, s[2]);
        s[3] = __fma_rn(v2, v2, s[3]);
    }
    __shared__ double sh[4][256];
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = s[k];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
#pragma unroll
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x < (unsigned)kmax) parts[b * 4 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void __launch_bounds__(256)
k_moment_final(const double *__restrict__ parts, int kmax, double *__restrict__ out)
{
    __shared__ double sh[4][256];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double a = 0.0;
        for (int j = threadIdx.x; j < QM_MOMENT_PARTS; j += 256) a += (k < kmax) ? parts[j * 4 + k] : 0.0;
        sh[k][threadIdx.x] = a;
    }
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
#pragma unroll
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x < (unsigned)kmax) out[threadIdx.x] = sh[threadIdx.x][0];
}

// sums_dev: QM_MOMENTS_WORKSPACE doubles; results in [0, kmax), scratch after 4
inline qm_status moments_launch(const void *x, int64_t n, bool f64, int kmax, double *sums_dev, cudaStream_t s)
{
    double *parts = sums_dev + 4;
    if (f64) k_moment_parts<double><<<QM_MOMENT_PARTS, 256, 0, s>>>((const double *)x, n, kmax, parts);
    else k_moment_parts<float><<<QM_MOMENT_PARTS, 256, 0, s>>>((const float *)x, n, kmax, parts);
    k_moment_final<<<1, 256, 0, s>>>(parts, kmax, sums_dev);
    return cudaGetLastError() == cudaSuccess ? QM_OK : QM_ECUDA;
}

}  // namespace qm
