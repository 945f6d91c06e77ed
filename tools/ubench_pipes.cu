// ubench_pipes.cu -- issue/dispatch cost of the instruction classes the hot path
// mixes (DFMA, FFMA, FFMA2, F2F, MUFU.RCP64H, integer ALU), alone and in pairs,
// measured on one B200 with every SM full of warps (experiment helper, not product).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_pipes.cu && /tmp/ubench
//
// Each test runs 8 independent dependency chains per thread (latency hidden by
// 16 warps per SMSP) and reports warp-instructions issued per cycle per SMSP
// (clock64 per CTA, one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

template <int T>
__global__ void __launch_bounds__(1024, 1) kern(double *sink, long long *cyc, double a, float af)
{
    double d[8];
    float f[8];
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        d[i] = 1.0 + threadIdx.x * 1e-9 + i;
        f[i] = 1.0f + threadIdx.x * 1e-7f + i;
        u[i] = threadIdx.x * 7 + i;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (T == 0) {   // DFMA
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
            } else if (T == 1) {   // FFMA (register operands)
                asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[i]) : "f"(af));
            } else if (T == 2) {   // FFMA2
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "fma.rn.f32x2 x, x, y, y;\n\tmov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
            } else if (T == 3) {   // F2F f32 -> f64 -> f32 (2 conversions)
                double t;
                asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[i]));
                asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[i]) : "d"(t));
            } else if (T == 4) {   // MUFU.RCP64H
                asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(d[i]));
            } else if (T == 5) {   // integer ALU (IADD3/LOP3)
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
            } else if (T == 6) {   // DFMA + FFMA2 (1:1)
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "fma.rn.f32x2 x, x, y, y;\n\tmov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
            } else if (T == 7) {   // DFMA + ALU (1:1)
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
            } else if (T == 8) {   // DFMA + 2 ALU (1:2)
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(u[(i + 3) & 7]) : "r"((unsigned)it));
            } else if (T == 9) {   // DFMA + F2F pair (1:2)
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
                double t;
                asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[i]));
                asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[i]) : "d"(t));
            } else if (T == 10) {   // FFMA2 + ALU (1:1)
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "fma.rn.f32x2 x, x, y, y;\n\tmov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
            } else if (T == 11) {   // FFMA + ALU (1:1)
                asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[i]) : "f"(af));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
            } else if (T == 12) {   // 2 DFMA + 3 FFMA2 + 2 ALU (the map's mix, roughly)
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[(i + 4) & 7]) : "d"(a));
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "fma.rn.f32x2 x, x, y, y;\n\tfma.rn.f32x2 x, x, y, y;\n\tfma.rn.f32x2 x, x, y, y;\n\t"
                             "mov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(u[(i + 3) & 7]) : "r"((unsigned)it));
            } else if (T == 13) {   // DMUL
                asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(a));
            } else if (T == 14) {   // FMUL2
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "mul.rn.f32x2 x, x, y;\n\tmov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
            } else if (T == 15) {   // FFMA imm (constant operand)
                asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F000000;" : "+f"(f[i]));
            } else if (T == 16) {   // DFMA + MUFU (1:1)
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
                asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(d[(i + 4) & 7]));
            } else if (T == 17) {   // FFMA2 + F2F pair (1:2)
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "fma.rn.f32x2 x, x, y, y;\n\tmov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
                double t;
                asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[(i + 2) & 7]));
                asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[(i + 2) & 7]) : "d"(t));
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i] + f[i] + u[i];
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int T>
void run(const char *name, double inst_per_step)
{
    double *sink;
    long long *cyc;
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&cyc, sms * 8);
    kern<T><<<sms, 1024>>>(sink, cyc, 0.999999, 0.9999f);   // warm
    kern<T><<<sms, 1024>>>(sink, cyc, 0.999999, 0.9999f);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    // warp-instructions per SMSP: 32 warps per CTA / 4 SMSPs x ITERS x 8 x inst_per_step
    const double wi = 8.0 * ITERS * 8 * inst_per_step;
    printf("%-34s %6.3f warp-inst/cycle/SMSP  (%.0f cycles)\n", name, wi / mx, mx);
    cudaFree(sink);
    cudaFree(cyc);
}

int main()
{
    run<0>("DFMA", 1);
    run<13>("DMUL", 1);
    run<1>("FFMA (reg)", 1);
    run<15>("FFMA (imm)", 1);
    run<2>("FFMA2", 1);
    run<14>("FMUL2", 1);
    run<3>("F2F f32->f64->f32", 2);
    run<4>("MUFU.RCP64H", 1);
    run<5>("ALU xor", 1);
    run<6>("DFMA+FFMA2", 2);
    run<7>("DFMA+ALU", 2);
    run<8>("DFMA+2ALU", 3);
    run<9>("DFMA+2F2F", 3);
    run<16>("DFMA+MUFU", 2);
    run<10>("FFMA2+ALU", 2);
    run<11>("FFMA+ALU", 2);
    run<17>("FFMA2+2F2F", 3);
    run<12>("2DFMA+3FFMA2+2ALU", 7);
    return 0;
}
