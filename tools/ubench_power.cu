// ubench_power.cu -- energy per warp-instruction of the instruction classes the
// hot path mixes, measured on one B200 (experiment helper, not product):
// each class runs ~1.5 s on every SM (8 warps per SMSP); the host samples NVML
// power and SM clock meanwhile and prints W, MHz, warp-inst/s and nJ per
// warp-instruction above the idle power.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/upow tools/ubench_power.cu -lnvidia-ml && /tmp/upow
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
#include <nvml.h>

template <int T>
__global__ void __launch_bounds__(1024, 1) kern(double *sink, int iters, double a, float af)
{
    __shared__ float tab[32 * 8];
    double d[8];
    float f[8];
    unsigned u[8];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = 1.0f + i;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        d[i] = 1.0 + threadIdx.x * 1e-9 + i;
        f[i] = 1.0f + threadIdx.x * 1e-7f + i;
        u[i] = threadIdx.x * 7 + i;
    }
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (T == 0) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(a));
            if (T == 1) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[i]) : "f"(af));
            if (T == 2)
                asm volatile("{.reg .b64 x, y;\n\tmov.b64 x, {%0,%1};\n\tmov.b64 y, {%2,%2};\n\t"
                             "fma.rn.f32x2 x, x, y, y;\n\tmov.b64 {%0,%1}, x;}"
                             : "+f"(f[i]), "+f"(f[(i + 4) & 7]) : "f"(af));
            if (T == 3) {
                double t;
                asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[i]));
                asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[i]) : "d"(t));
            }
            if (T == 4) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(d[i]));
            if (T == 5) asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"((unsigned)it));
            if (T == 6) {   // conflict-free LDS.32 gather: lane-dependent row, bank = lane
                unsigned idx = ((u[i] & 7u) << 5) | (threadIdx.x & 31u);
                float v;
                asm volatile("ld.shared.f32 %0, [%1];"
                             : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(tab) + 4 * idx));
                u[i] += __float_as_uint(v);
            }
            if (T == 7) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(a));
            if (T == 8) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i] + f[i] + u[i];
    if (s == 12345.678) sink[0] = s;
}

struct Sampler {
    nvmlDevice_t h;
    std::atomic<bool> stop{false};
    std::vector<double> p, c;
    std::thread th;
    void start()
    {
        stop = false;
        p.clear();
        c.clear();
        th = std::thread([this] {
            while (!stop) {
                unsigned mw = 0, mhz = 0;
                nvmlDeviceGetPowerUsage(h, &mw);
                nvmlDeviceGetClockInfo(h, NVML_CLOCK_SM, &mhz);
                p.push_back(mw / 1e3);
                c.push_back(mhz);
                std::this_thread::sleep_for(std::chrono::milliseconds(5));
            }
        });
    }
    void end(double &pw, double &mhz)
    {
        stop = true;
        th.join();
        double sp = 0, sc = 0;   // mean over the second half (steady state)
        int n = 0;
        for (size_t i = p.size() / 2; i < p.size(); ++i) { sp += p[i]; sc += c[i]; ++n; }
        pw = n ? sp / n : 0;
        mhz = n ? sc / n : 0;
    }
};

template <int T>
void run(const char *name, double inst_per_step, Sampler &S, double idle, int sms)
{
    double *sink;
    cudaMalloc(&sink, 8);
    const int iters = 4096;
    kern<T><<<sms, 1024>>>(sink, 64, 0.999999, 0.9999f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<T><<<sms, 1024>>>(sink, iters, 0.999999, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms1;
    cudaEventElapsedTime(&ms1, e0, e1);
    const int L = (int)(2000.0 / ms1) + 1;
    S.start();
    cudaEventRecord(e0);
    for (int i = 0; i < L; ++i) kern<T><<<sms, 1024>>>(sink, iters, 0.999999, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pw, mhz;
    S.end(pw, mhz);
    const double winst = (double)L * sms * 32 * iters * 8 * inst_per_step;   // warp-instructions
    const double rate = winst / (ms / 1e3);
    printf("%-14s %7.1f W %6.0f MHz %8.3f Twi/s  %6.3f nJ/warp-inst above idle  (%.3f warp-inst/cycle/SMSP)\n", name,
           pw, mhz, rate / 1e12, (pw - idle) / rate * 1e9, rate / (sms * 4 * mhz * 1e6));
    cudaFree(sink);
}

int main()
{
    nvmlInit();
    Sampler S;
    nvmlDeviceGetHandleByIndex(0, &S.h);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFree(0);
    std::this_thread::sleep_for(std::chrono::milliseconds(500));
    S.start();
    std::this_thread::sleep_for(std::chrono::milliseconds(1000));
    double idle, imhz;
    S.end(idle, imhz);
    printf("idle %.1f W at %.0f MHz\n", idle, imhz);
    run<0>("DFMA", 1, S, idle, sms);
    run<7>("DMUL", 1, S, idle, sms);
    run<1>("FFMA", 1, S, idle, sms);
    run<2>("FFMA2", 1, S, idle, sms);
    run<3>("F2F(x2)", 2, S, idle, sms);
    run<4>("MUFU.RCP64H", 1, S, idle, sms);
    run<8>("MUFU.RCP32", 1, S, idle, sms);
    run<5>("ALU", 1, S, idle, sms);
    run<6>("LDS+ALU", 3, S, idle, sms);
    run<0>("DFMA(again)", 1, S, idle, sms);
    return 0;
}
