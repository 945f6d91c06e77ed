// qm_prim.cuh -- the few hardware primitives the sm_100a kernels use directly.
//
// Everything numerically sensitive in qm_math.cuh is written with explicitly
// rounded operations (no FMA contraction left to the compiler), so that the
// result of each device function is a fixed function of its input.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define QM_DEV __device__ __forceinline__

namespace qm {

// MUFU.RCP64H: ~2^-22-accurate reciprocal seed for x >= 1 (no special cases
// are ever fed to it).
QM_DEV double rcp_approx_f64(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

// Streaming 128-bit global accesses: loads bypass L1 allocation (each byte is
// read once), stores are evict-first.
QM_DEV float4 ld_stream_f4(const float4 *p)
{
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
QM_DEV void st_stream_f4(float4 *p, float4 v)
{
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
QM_DEV double2 ld_stream_d2(const double2 *p)
{
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
QM_DEV void st_stream_d2(double2 *p, double2 v)
{
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}

QM_DEV void st_stream(float4 *p, float4 v) { st_stream_f4(p, v); }
QM_DEV void st_stream(double2 *p, double2 v) { st_stream_d2(p, v); }

// NaN-propagating minima (min.NaN: FMNMX.NAN / 3-input FMNMX3.NAN on sm_100a)
QM_DEV float min_nan(float a, float b)
{
    float d;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
QM_DEV float min3_nan(float a, float b, float c)
{
    float d;
    asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// Packed fp32 pair arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100a): two
// independent IEEE round-to-nearest operations per instruction.
// QM_F32X2 (A/B): 1 = packed instructions; 0 = two scalar ones each (bitwise the
// same results); 2 = packed FFMA2 only, scalar adds and multiplies
#ifndef QM_F32X2
#define QM_F32X2 1
#endif
QM_DEV float2 fma2(float2 a, float2 b, float2 c)
{
    if (QM_F32X2 == 0) return make_float2(__fmaf_rn(a.x, b.x, c.x), __fmaf_rn(a.y, b.y, c.y));
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, {%6,%7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0,%1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
QM_DEV float2 mul2(float2 a, float2 b)
{
    if (QM_F32X2 != 1) return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0,%1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
QM_DEV float2 add2(float2 a, float2 b)
{
    if (QM_F32X2 != 1) return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0,%1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

}  // namespace qm
