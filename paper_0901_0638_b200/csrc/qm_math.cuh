// qm_math.cuh -- device numerics of the hot path (sm_100a).
//
// Paper: Shaw & Brickman, "Quantile Mechanics II" (arXiv 0901.0638); P:n are
// PAPER.md line numbers.  The kernels evaluate the paper's formulas; the
// arithmetic SCHEME below (how each formula is evaluated so that the result is
// within 4 ulp (fp32) / 2 ulp (fp64) of the exactly evaluated formula) is ours
// and is described in DESIGN.md "Kernels".
//
//  fp32 breakless (App B/C):  vv = min(u, 1-u) (exact), z = -log(2 vv) by a
//    polynomial log in fp32 (<= 1 ulp), then z P(z)/Q(z) with the
//    float-rounded coefficients evaluated in FP64 (B200 has a full-rate-ish FP64
//    pipe: 64 lanes/SM), one final rounding to float.  Exhaustive CPU emulation
//    over the fp32 grid: <= 1.42 ulp.
//  fp64 breakless (App D):    z = -log(2 vv) as a double-double from a
//    range-reduced atanh series, compensated (error-free transform) Horner for
//    the last K steps of P and Q, a double-double quotient and one final
//    rounding: <= ~0.7 ulp.
#pragma once
#ifndef QM_PRIM_EXTERNAL   // (a development-time CPU emulation supplies its own primitives)
#include "qm_prim.cuh"
#endif

namespace qm {

// ---------------------------------------------------------------- constants
// App C (5,5), P:792-803 -- float-rounded as the listing declares (`const float`),
// held in double for the FP64 evaluation.
__constant__ double kC55P[6] = {
    (double)(float)1.2533136835212087879, (double)(float)1.9797154223229267471,
    (double)(float)0.80002295072483916762, (double)(float)0.087403248265958578062,
    (double)(float)0.0020751409553756572917, (double)(float)4.744820732427972462e-6};
__constant__ double kC55Q[6] = {
    1.0, (double)(float)2.0795584360534589311, (double)(float)1.2499328117341603014,
    (double)(float)0.23668431621373705623, (double)(float)0.0120098270559197768,
    (double)(float)0.00010590620919921025259};
// the same coefficients as floats (for the optional fp32 inner Horner steps)
__constant__ float kC55Pf[6] = {1.2533136835212087879f, 1.9797154223229267471f, 0.80002295072483916762f,
                                0.087403248265958578062f, 0.0020751409553756572917f, 4.744820732427972462e-6f};
__constant__ float kC55Qf[6] = {1.0f, 2.0795584360534589311f, 1.2499328117341603014f,
                                0.23668431621373705623f, 0.0120098270559197768f, 0.00010590620919921025259f};

// App A/B (7,7), P:477-497 / P:755-770: float-rounded (App B) and double (App A)
#define QM_A77P 1.2533141359896652729, 3.0333178251950406994, 2.3884158540184385711, \
    0.73176759583280610539, 0.085838533424158257377, 0.0034424140686962222423,       \
    0.000036313870818023761224, 4.3304513840364031401e-8
#define QM_A77Q 1.0, 2.9202373175993672857, 2.9373357991677046357, 1.2356513216582148689, \
    0.2168237095066675527, 0.014494272424798068406, 0.00030617264753008793976,          \
    1.3141263119543315917e-6
__constant__ double kA77P_d[8] = {QM_A77P};
__constant__ double kA77Q_d[8] = {QM_A77Q};
__constant__ double kA77P_f[8] = {
    (double)(float)1.2533141359896652729, (double)(float)3.0333178251950406994,
    (double)(float)2.3884158540184385711, (double)(float)0.73176759583280610539,
    (double)(float)0.085838533424158257377, (double)(float)0.0034424140686962222423,
    (double)(float)0.000036313870818023761224, (double)(float)4.3304513840364031401e-8};
__constant__ double kA77Q_f[8] = {
    1.0, (double)(float)2.9202373175993672857, (double)(float)2.9373357991677046357,
    (double)(float)1.2356513216582148689, (double)(float)0.2168237095066675527,
    (double)(float)0.014494272424798068406, (double)(float)0.00030617264753008793976,
    (double)(float)1.3141263119543315917e-6};

// App D (13,13), P:821-848 (`const double`)
__constant__ double kD13P[14] = {
    1.2533141373154989811, 5.5870183514814983104, 9.9373788223105148469, 9.11745910783758368,
    4.6865666928347513004, 1.3841649695441184484, 0.23434950424605615377, 0.022306824510199724768,
    0.0011538603964070818722, 0.000030796620691411567563, 3.9115723028719510263e-7,
    2.0589573468131996933e-9, 3.3944224725087481454e-12, 7.3936480912071325978e-16};
__constant__ double kD13Q[14] = {
    1.00000000000000000000, 4.9577956835689939051, 9.9793129245112074476, 10.574454910639356539,
    6.4247521669505779535, 2.3008904864351121026, 0.48545999687461771635, 0.059283082737079006352,
    0.0040618506206078995821, 0.00014919732843986856251, 2.7477061392049947066e-6,
    2.2815008011613816939e-8, 7.0445790305953963457e-11, 5.1535907808963289678e-14};

// Our minimax fits (tests/golden/fit_*.txt, tools/fit_rational.py; SURVEY rows
// f3/f4): the (12,12) on [0, 37] (< 5e-16) and (8,8) on [0, 74] (~6e-10) that
// P:544 says exist, and the (4,4) on [0, 10] below the break of the two-region
// variant.  Double-rounded (fp64) and float-rounded (fp32) as for App A-D.
__constant__ double kF12P[13] = {
    1.25331413731549964304885084933, 5.65670727193097123052913156555, 10.199184028049004645639650354,
    9.49108178418734942631477139003, 4.94304333170547437473236493918, 1.47293406972979776643830812522,
    0.249077147187243284286425789887, 0.0232075251548776468184535573962,
    0.00113211638446441623489197365915, 0.000026638805014702015041938526811,
    0.000000262823263993221383793586115962, 8.20115160731597726774034377471e-10,
    3.4080843072305026219786124261e-13};
__constant__ double kF12Q[13] = {
    1.0, 5.01339939725483198543174978089, 10.2160051129404404259102375667,
    10.9670844662824747543017650822, 6.74844347326083628169062975985, 2.44148341873030012307321591735,
    0.516866979805929966868864954603, 0.0624322209086865620690205639678,
    0.00411740318775822728331972658499, 0.00013852471353158268838850038814,
    0.00000213335696590330667438560151822, 0.0000000123741421877613097338506656296,
    1.71840938834726185281010719498e-11};
__constant__ double kF88P_d[9] = {
    1.25331413659487693200589460544, 3.18279215828640909853465485323, 2.69637013151484046914318369988,
    0.926505960348117503759109131467, 0.130722564999804748080717604434,
    0.00715510742068364856695515828894, 0.000134566885939144919435102866116,
    0.000000669320737492863356757758585237, 3.78894005999045094010072867485e-10};
__constant__ double kF88Q_d[9] = {
    1.0, 3.03950064147177248702038516122, 3.24267820535186536296356820427,
    1.49261049909605991213659399514, 0.302049532338050455259987910733,
    0.0255324575872787421879918341977, 0.000815155781723673184564102970288,
    0.00000817923481671560569243134101007, 0.0000000166707331365471438381381542416};
__constant__ double kF88P_f[9] = {
    (double)(float)1.25331413659487693200589460544, (double)(float)3.18279215828640909853465485323,
    (double)(float)2.69637013151484046914318369988, (double)(float)0.926505960348117503759109131467,
    (double)(float)0.130722564999804748080717604434, (double)(float)0.00715510742068364856695515828894,
    (double)(float)0.000134566885939144919435102866116,
    (double)(float)0.000000669320737492863356757758585237,
    (double)(float)3.78894005999045094010072867485e-10};
__constant__ double kF88Q_f[9] = {
    (double)(float)1.0, (double)(float)3.03950064147177248702038516122,
    (double)(float)3.24267820535186536296356820427, (double)(float)1.49261049909605991213659399514,
    (double)(float)0.302049532338050455259987910733, (double)(float)0.0255324575872787421879918341977,
    (double)(float)0.000815155781723673184564102970288,
    (double)(float)0.00000817923481671560569243134101007,
    (double)(float)0.0000000166707331365471438381381542416};
__constant__ double kF44P_f[5] = {
    (double)(float)1.25331376367946351584057665416, (double)(float)1.90154131297345796677471850561,
    (double)(float)0.692706016566279324284406456679, (double)(float)0.0560005883011708193276104273226,
    (double)(float)0.000448739389131331445037989032119};
__constant__ double kF44Q_f[5] = {
    (double)(float)1.0, (double)(float)2.01718797443210201360154517184,
    (double)(float)1.13309652308639082468928923168, (double)(float)0.179982309491888788965156666547,
    (double)(float)0.0053418912252851127623755674913};

// fp32 log: log1p(f) = f + f^2 R(f), f in [-1/3, 1/3); R: degree-7 Chebyshev fit
// (tools/fit_log.py), |error of R| < 2.1e-7.  Where the log's relative error
// reaches z unscaled (e = 0, f -> -1/3) it is < 0.3 ulp of z; the fp32 map stays
// <= 1.67 ulp over the whole fp32 grid (degree 8 and a two-part ln2: 1.42 ulp,
// one FFMA2 per sample pair more for each).
#define QM_LR0 -0.49999985098838806f
#define QM_LR1 0.33333319425582886f
#define QM_LR2 -0.2500414550304413f
#define QM_LR3 0.20003780722618103f
#define QM_LR4 -0.16483017802238464f
#define QM_LR5 0.14118309319019318f
#define QM_LR6 -0.15040764212608337f
#define QM_LR7 0.1342574954032898f
#define QM_LN2F 0.6931471824645996f          // (float)ln 2

// fp64 log: log1p(f) = 2 atanh(s) = 2s + s^3 T(s^2), s = f/(2+f) in [-0.2, 1/7];
// T: Chebyshev fit on w in [0, 1/25], relative error < 4e-17 (term is < 1.3% of 2s)
__constant__ double kLogT[8] = {0.6666666666666666, 0.400000000000078, 0.2857142856733919,
                                0.22222223037807243, 0.18181738454723026, 0.15388834677801916,
                                0.1321036048513262, 0.13604015707124079};
#define QM_LN2_HI 6.93147180369123816490e-01   // trailing zeros: e*hi exact for |e| < 2^11
#define QM_LN2_LO 1.90821492927058770002e-10

// ------------------------------------------------------------- fp32 pieces
#define QM_LOG_R(r, f, FMA, C)                                                      \
    r = FMA(C(QM_LR7), f, C(QM_LR6));                                               \
    r = FMA(r, f, C(QM_LR5));                                                       \
    r = FMA(r, f, C(QM_LR4));                                                       \
    r = FMA(r, f, C(QM_LR3));                                                       \
    r = FMA(r, f, C(QM_LR2));                                                       \
    r = FMA(r, f, C(QM_LR1));                                                       \
    r = FMA(r, f, C(QM_LR0));
#define QM_C1(x) (x)
#define QM_C2(x) make_float2((x), (x))

// z = -log(2 vv) for vv a normal float in (0, 1/2]; `eadj` adds to the binary
// exponent (used to pre-scale subnormals by 2^24).  <= ~1 ulp.
QM_DEV float neg_log2x_f32(float vv, int eadj)
{
    const int32_t k = (int32_t)(__float_as_uint(vv) - 0x3f2aaaabu);   // 0x3f2aaaab = 2/3
    const int32_t e = (k >> 23) + 1 + eadj;                             // +1: the factor 2
    const float m = __uint_as_float(((uint32_t)k & 0x7fffffu) + 0x3f2aaaabu);   // [2/3, 4/3)
    const float f = __fsub_rn(m, 1.0f);                                 // exact (Sterbenz)
    float r;
    QM_LOG_R(r, f, __fmaf_rn, QM_C1)
    const float f2 = __fmul_rn(f, f);
    const float L = __fmaf_rn(f2, r, f);                                // log1p(f)
    // (float)e without I2F: 1.5*2^23 + e as bits, minus 1.5*2^23 (|e| < 2^22)
    const float ef = __fsub_rn(__int_as_float(0x4B400000 + e), 12582912.0f);
    const float zf = __fmaf_rn(ef, QM_LN2F, L);
    return -zf;
}

// Two samples at once with packed f32x2 arithmetic (bitwise identical to two
// calls of neg_log2x_f32 with the same eadj).
QM_DEV float2 neg_log2x_f32x2(float vva, float vvb, int eadj = 0)
{
    const int32_t ka = (int32_t)(__float_as_uint(vva) - 0x3f2aaaabu);
    const int32_t kb = (int32_t)(__float_as_uint(vvb) - 0x3f2aaaabu);
    const float2 m = make_float2(__uint_as_float(((uint32_t)ka & 0x7fffffu) + 0x3f2aaaabu),
                                 __uint_as_float(((uint32_t)kb & 0x7fffffu) + 0x3f2aaaabu));
    const float2 f = add2(m, make_float2(-1.0f, -1.0f));
    float2 r;
    QM_LOG_R(r, f, fma2, QM_C2)
    const float2 f2 = mul2(f, f);
    const float2 L = fma2(f2, r, f);
    const float2 ef = add2(make_float2(__int_as_float(0x4B400000 + (ka >> 23) + 1 + eadj),
                                       __int_as_float(0x4B400000 + (kb >> 23) + 1 + eadj)),
                           make_float2(-12582912.0f, -12582912.0f));
    const float2 zf = fma2(ef, make_float2(QM_LN2F, QM_LN2F), L);
    return make_float2(-zf.x, -zf.y);
}

// |z P(z)/Q(z)| for the fp32 formulas: coefficients float-rounded, evaluated in
// FP64 (N coefficients each), rcp seed + one quotient correction, one rounding.
#ifndef QM_F32_XU_LITE
#define QM_F32_XU_LITE 0   // A/B: 1 = float<->double conversions by integer ops (XU relief)
#endif
// float -> double by bits for z >= +-0 finite (sign cleared: -0 -> +2^-127, which the
// final multiply by the float z turns back into 0)
QM_DEV double widen_pos(float z)
{
    const uint32_t f = __float_as_uint(z) & 0x7fffffffu;
    return __hiloint2double((int)((f >> 3) + 0x38000000u), (int)(f << 29));
}
// double in [2^-126, 2^127) -> float by truncation (funnel shift + exponent rebias)
QM_DEV float narrow_trunc(double t)
{
    const uint32_t fb = __funnelshift_l((uint32_t)__double2loint(t), (uint32_t)__double2hiint(t), 3) - 0xC0000000u;
    return __uint_as_float(fb);
}

template <int N, bool CORRECT = true>
QM_DEV float rational_f32path(float z, const double *P, const double *Q)
{
    const double zd = QM_F32_XU_LITE ? widen_pos(z) : (double)z;
    double p = P[N - 1], q = Q[N - 1];
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
        p = __fma_rn(p, zd, P[i]);
        q = __fma_rn(q, zd, Q[i]);
    }
    // MUFU.RCP64H seed + one residual correction.  Measured on B200 over the whole
    // fp32 grid: without the correction (2 DFMA) the map is 8 % faster but 16.9 ulp off.
    const double r = rcp_approx_f64(q);
    if (!CORRECT) return (float)__dmul_rn(__dmul_rn(zd, p), r);
    double t = __dmul_rn(p, r);
    const double e = __fma_rn(-q, t, p);
    t = __fma_rn(e, r, t);
#ifdef QM_F32_FINAL_DMUL
    return (float)__dmul_rn(zd, t);
#else
    // z (P/Q) with P/Q rounded to float and the product in fp32: one DMUL fewer
    // on the FP64 pipe (the kernel's co-bottleneck) for +0.5 ulp: <= 2.41 ulp over
    // the fp32 grid in emulation (final DMUL: 1.67)
    return __fmul_rn(QM_F32_XU_LITE ? narrow_trunc(t) : __double2float_rn(t), z);
#endif
}

// ---------------------------------------------- fp32 App C on the FMA pipe
// z P(z)/Q(z) of App C (float coefficients) entirely in fp32, two
// samples per instruction (FFMA2): plain Horner for the first four steps of P
// and Q, the LAST step of each compensated (TwoProd by FMA, Fast2Sum of the
// operands ordered by max/min: both positive, exact error), the quotient from
// MUFU.RCP plus one residual correction (e = P - t Q with P's and Q's low parts)
// folded into the final product z t + z (e r).  Valid for inputs on the 24-bit
// lattice (vv a multiple of 2^-24, vv >= 2^-24, i.e. z <= 15.95): exhaustive CPU
// emulation over every such vv with the kernel's log, rcp seed +-1 ulp: 3.64 ulp
// max (tools/emu_f32map.c; off the lattice it reaches 4.5 ulp, so other inputs
// take the FP64 evaluation).
#define QM_C55P0F 1.2533136835212087879f
#define QM_C55P1F 1.9797154223229267471f
#define QM_C55P2F 0.80002295072483916762f
#define QM_C55P3F 0.087403248265958578062f
#define QM_C55P4F 0.0020751409553756572917f
#define QM_C55P5F 4.744820732427972462e-6f
#define QM_C55Q1F 2.0795584360534589311f
#define QM_C55Q2F 1.2499328117341603014f
#define QM_C55Q3F 0.23668431621373705623f
#define QM_C55Q4F 0.0120098270559197768f
#define QM_C55Q5F 0.00010590620919921025259f
#define QM_LATTICE_MIN 5.9604644775390625e-8f      // 2^-24: the smallest vv on the lattice

QM_DEV float rcp_approx_f32(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

QM_DEV float2 c55_comp1_x2(float2 z)
{
    float2 p = fma2(QM_C2(QM_C55P5F), z, QM_C2(QM_C55P4F));
    float2 q = fma2(QM_C2(QM_C55Q5F), z, QM_C2(QM_C55Q4F));
    p = fma2(p, z, QM_C2(QM_C55P3F));
    q = fma2(q, z, QM_C2(QM_C55Q3F));
    p = fma2(p, z, QM_C2(QM_C55P2F));
    q = fma2(q, z, QM_C2(QM_C55Q2F));
    p = fma2(p, z, QM_C2(QM_C55P1F));
    q = fma2(q, z, QM_C2(QM_C55Q1F));
    // last step: s = p z + a0 with its exact error (TwoProd + ordered Fast2Sum)
    const float2 pp = mul2(p, z), qq = mul2(q, z);
    const float2 ppe = fma2(p, z, make_float2(-pp.x, -pp.y)), qqe = fma2(q, z, make_float2(-qq.x, -qq.y));
    const float2 ps = add2(pp, QM_C2(QM_C55P0F)), qs = add2(qq, QM_C2(1.0f));
    const float2 tp = add2(ps, make_float2(-fmaxf(pp.x, QM_C55P0F), -fmaxf(pp.y, QM_C55P0F)));
    const float2 tq = add2(qs, make_float2(-fmaxf(qq.x, 1.0f), -fmaxf(qq.y, 1.0f)));
    const float2 ep = add2(make_float2(fminf(pp.x, QM_C55P0F), fminf(pp.y, QM_C55P0F)), make_float2(-tp.x, -tp.y));
    const float2 eq = add2(make_float2(fminf(qq.x, 1.0f), fminf(qq.y, 1.0f)), make_float2(-tq.x, -tq.y));
    const float2 lp = add2(ppe, ep), lq = add2(qqe, eq);
    // quotient: t = ps r, e = ps + lp - t (qs + lq), result z t + z e r
    const float2 r = make_float2(rcp_approx_f32(qs.x), rcp_approx_f32(qs.y));
    const float2 t = mul2(ps, r);
    float2 e = fma2(make_float2(-qs.x, -qs.y), t, ps);
    e = add2(e, lp);
    e = fma2(make_float2(-t.x, -t.y), lq, e);
    return fma2(z, mul2(e, r), mul2(t, z));
}

// the same arithmetic for one sample (bitwise equal to a lane of c55_comp1_x2)
QM_DEV float c55_comp1(float z) { return c55_comp1_x2(make_float2(z, z)).x; }

// copysign by the sign of (u - (1-u)): +0 at u = 1/2 (P:773, P:855 sgn = +1)
QM_DEV float apply_sign_f32(float mag, float u, float omu)
{
    const uint32_t s = __float_as_uint(__fsub_rn(u, omu)) & 0x80000000u;
    return __uint_as_float((__float_as_uint(mag) & 0x7fffffffu) | s);
}

// ------------------------------------------------------------- fp64 pieces
struct dd { double hi, lo; };

// -log(2 vv) as a double-double for vv a normal double in (0, 1/2]
QM_DEV dd neg_log2x_dd(double vv, int eadj)
{
    const int64_t k = (int64_t)(__double_as_longlong(vv) - 0x3FE5555555555555LL);   // 2/3
    const int64_t e = (k >> 52) + 1 + eadj;
    const double m = __longlong_as_double((k & 0x000FFFFFFFFFFFFFLL) + 0x3FE5555555555555LL);
    const double f = __dadd_rn(m, -1.0);                     // exact, [-1/3, 1/3)
    // s = f / (2 + f) as sh + sl
    const double dh = __dadd_rn(2.0, f);
    const double dl = __dadd_rn(f, -__dadd_rn(dh, -2.0));   // Fast2Sum, |2| >= |f|
    double r = rcp_approx_f64(dh);
    r = __fma_rn(r, __fma_rn(-dh, r, 1.0), r);               // ~2^-44
    const double s0 = __dmul_rn(f, r);
    double rem = __fma_rn(-s0, dh, f);
    rem = __fma_rn(-s0, dl, rem);
    const double s1 = __dmul_rn(rem, r);
    // renormalise so that |sl| <= ulp(sh)/2: the cubic term below uses sh only
    const double sh = __dadd_rn(s0, s1);
    const double sl = __dadd_rn(s1, -__dadd_rn(sh, -s0));    // Fast2Sum, |s0| >= |s1|
    // log1p(f) = 2 sh + (2 sl + sh^3 T(sh^2))
    const double w = __dmul_rn(sh, sh);
    double T = kLogT[7];
#pragma unroll
    for (int i = 6; i >= 0; --i) T = __fma_rn(T, w, kLogT[i]);
    const double l_hi = 2.0 * sh;
    const double l_lo = __fma_rn(__dmul_rn(sh, w), T, 2.0 * sl);
    // + e ln2:  a = E*LN2_HI (exact); Fast2Sum(a, l_hi) valid: |a| >= ln2 > |l_hi| or a = 0
    const double E = (double)e;
    const double a = __dmul_rn(E, QM_LN2_HI);
    const double S = __dadd_rn(a, l_hi);
    const double err = __dadd_rn(l_hi, -__dadd_rn(S, -a));
    const double lo = __dadd_rn(err, __fma_rn(E, QM_LN2_LO, l_lo));
    const double t = __dadd_rn(S, lo);
    const double tl = __dadd_rn(lo, -__dadd_rn(t, -S));
    return dd{-t, -tl};
}

// Compensated Horner (error-free transforms) of sum a_i z^i at z = zh + zl,
// plain FMA for the first N-1-KC steps, compensated for the last KC steps.
template <int N, int KC>
QM_DEV dd horner_comp(const double *a, double zh, double zl)
{
    double s = a[N - 1], c = 0.0;
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
        if (i >= KC) {
            s = __fma_rn(s, zh, a[i]);
        } else {
            const double p = __dmul_rn(s, zh);
            const double pi = __fma_rn(s, zh, -p);               // TwoProd
            const double t = __dadd_rn(p, a[i]);                 // TwoSum
            const double bb = __dadd_rn(t, -p);
            const double sg = __dadd_rn(__dadd_rn(p, -__dadd_rn(t, -bb)), __dadd_rn(a[i], -bb));
            c = __fma_rn(c, zh, __fma_rn(s, zl, __dadd_rn(pi, sg)));
            s = t;
        }
    }
    return dd{s, c};
}

// The same compensated Horner for POSITIVE coefficients and zh >= 0 (every
// breakless rational: all its coefficients are positive).  Then p = s zh >= 0
// and a_i > 0, so the sum's error is exact with Fast2Sum once the larger
// operand is first; for positive doubles the order of the high words decides it
// (equal high words: equal exponents, either order is exact).  The compare and
// selects run on the integer pipe: 3 DADD + ISETP + 4 SEL per step instead of
// TwoSum's 6 DADD on the FP64 pipe -- bitwise the same result (both errors exact).
QM_DEV dd two_sum_pos(double p, double a)
{
    const bool pa = __double2hiint(p) >= __double2hiint(a);
    const double hi = pa ? p : a, lo = pa ? a : p;
    const double t = __dadd_rn(hi, lo);
    return dd{t, __dadd_rn(lo, -__dadd_rn(t, -hi))};
}

// Fast2Sum with the operands ordered by magnitude (any signs): |x| >= |y| is
// decided on the high words with the sign masked (equal high words: equal
// exponents, exact either way).  Exact like TwoSum, 3 DADD instead of 6.
QM_DEV dd two_sum_ord(double p, double a)
{
    const bool pa = (__double2hiint(p) & 0x7fffffff) >= (__double2hiint(a) & 0x7fffffff);
    const double hi = pa ? p : a, lo = pa ? a : p;
    const double t = __dadd_rn(hi, lo);
    return dd{t, __dadd_rn(lo, -__dadd_rn(t, -hi))};
}

// ZL = false: P(zh) only -- z's low part is left to the caller (rational_dd)
template <int N, int KC, bool ZL = true>
QM_DEV dd horner_comp_pos(const double *a, double zh, double zl)
{
    double s = a[N - 1], c = 0.0;
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
        if (i >= KC) {
            s = __fma_rn(s, zh, a[i]);
        } else {
            const double p = __dmul_rn(s, zh);
            const double pi = __fma_rn(s, zh, -p);               // TwoProd
            const dd t = two_sum_pos(p, a[i]);                   // Fast2Sum, ordered
            const double err = __dadd_rn(pi, t.lo);
            c = __fma_rn(c, zh, ZL ? __fma_rn(s, zl, err) : err);
            s = t.hi;
        }
    }
    return dd{s, c};
}

// z P(z)/Q(z) for a double-double z >= 0, one final rounding (positive
// coefficients: the breakless rationals).
// z's low part zl (|zl| <= 2^-53 zh) enters once, as zl R(zh) in the final sum,
// not in every compensated Horner step (QM_DD_ZL_STEPS=1 restores the per-step
// form): (zh + zl) R(zh + zl) = zh R + zl R + zh zl R' + O(zl^2), and the dropped
// zh zl R' is (zl/zh)(kappa - 1) of the result, kappa = d ln(zR)/d ln z.  Up to
// z = 36.8 (the fp64 grid ends at 36.04) |kappa - 1| < 0.48 for App D, so this adds
// < 0.48 ulp: with the plain steps' W_P + W_Q it stays <= 1.06 + 0.5 (final rounding)
// ulp (tests/test_oracle_normal.py::test_d13_partial_compensation_bound), and it
// saves one DFMA per compensated step (20 of App D's ~211 FP64 operations per sample).
// Off the fp64 grid (z > 36.8: u below the odd grid's 2^-54, only from callers' own
// uniforms, or Laplace |v| > 36.8) App D's plain steps weigh more (W_P + W_Q = 1.55 at
// z = 74, -> 6 as z grows: 3.7 ulp measured at z = 477 with 10 of 13 steps), so there
// rat64 evaluates all 13 steps compensated with zl per step (<= 0.5 + O(u) ulp), per
// lane, out of line and only when a lane of the warp needs it.
#ifndef QM_DD_ZL_STEPS
#define QM_DD_ZL_STEPS 0
#endif
#define QM_DD_ZL_ZMAX 36.8
template <int N, int KC, bool ZL>
QM_DEV double rational_dd_zl(dd z, const double *P, const double *Q)
{
    const dd p = horner_comp_pos<N, KC, ZL>(P, z.hi, z.lo);
    const dd q = horner_comp_pos<N, KC, ZL>(Q, z.hi, z.lo);
    double r = rcp_approx_f64(q.hi);
    r = __fma_rn(r, __fma_rn(-q.hi, r, 1.0), r);
    const double q0 = __dmul_rn(p.hi, r);
    double e = __fma_rn(-q.hi, q0, p.hi);
    e = __fma_rn(-q0, q.lo, __dadd_rn(e, p.lo));
    const double dq = __dmul_rn(e, r);
    return __fma_rn(z.hi, q0, __fma_rn(z.hi, dq, __dmul_rn(z.lo, q0)));
}
template <int N, int KC>
QM_DEV double rational_dd(dd z, const double *P, const double *Q)
{
    return rational_dd_zl<N, KC, QM_DD_ZL_STEPS != 0>(z, P, Q);
}

QM_DEV double apply_sign_f64(double mag, double u, double omu)
{
    const unsigned long long s = (unsigned long long)__double_as_longlong(__dadd_rn(u, -omu)) & 0x8000000000000000ULL;
    return __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(mag) & 0x7fffffffffffffffULL) | s));
}

// ----------------------------------------------------- breakless quantiles
// Algorithm ids for templates (mirror qm_algorithm)
// ALG_BREAKLESS_TAIL (row f2): the breakless rational for v < vc and the §5.1
// supplementary tail model beyond; vc = 37 for App C and
// 86.75 for App D (reading R23).  Its fast path is ALG_BREAKLESS: the warp vote
// sends a warp with any v >= vc to the careful path.
// ALG_F1212 / ALG_F88 / ALG_TWO_REGION: rows f3/f4 (our fits); ALG_F44 is the
// fast path of the two-region variant (every lane of the warp below the break).
enum { ALG_BREAKLESS = 0, ALG_BREAKLESS77 = 1, ALG_BREAKLESS_TAIL = 5, ALG_F1212 = 7, ALG_F88 = 8,
       ALG_TWO_REGION = 9, ALG_F44 = 10 };
#define QM_TWO_BREAK_F32 10.0f
#define QM_VC_F32 37.0f
#define QM_VC_F64 86.75
#ifndef QM_F32_RAT
#define QM_F32_RAT 0     // fp32 App C fast path: 0 FP64 rational, 1 FMA-pipe (c55_comp1), 2 both (pairs alternate)
#endif
#ifndef QM_D13_KC
#define QM_D13_KC 10     // compensated Horner steps of App D's 13 (A/B builds may override)
#endif
#ifndef QM_D13_KC_LO
#define QM_D13_KC_LO 8   // ... for z <= QM_D13_ZSPLIT (written bound in rat64)
#endif
#define QM_D13_ZSPLIT 12.0
#ifndef QM_D13_SPLIT
#define QM_D13_SPLIT 0    // A/B: 1 = the z <= 12 / z > 12 split of rat64 (measured slower, see there)
#endif

template <int ALG> __host__ __device__ constexpr int fast_alg()
{
    return ALG == ALG_BREAKLESS_TAIL ? ALG_BREAKLESS : ALG == ALG_TWO_REGION ? ALG_F44 : ALG;
}
// smallest vv = min(u, 1-u) of the fast path: normal numbers; for the tail
// composite also v = -log(2 vv) < vc (e^-37/2 = 4.2665e-17, e^-86.75/2 = 1.0566e-38)
template <int ALG> __host__ __device__ constexpr float fast_vv_min_f32()
{
    // two-region: z < 10 for every vv >= 2.2705e-5 (e^-10/2 = 2.26999e-5, margin for
    // the fp32 log), so the whole warp is below the break
    return ALG == ALG_BREAKLESS_TAIL ? 4.3e-17f : ALG == ALG_TWO_REGION ? 2.2705e-5f : 1.17549435e-38f;
}
template <int ALG> __host__ __device__ constexpr double fast_vv_min_f64()
{
    return ALG == ALG_BREAKLESS_TAIL ? 1.1e-38 : 2.2250738585072014e-308;
}

QM_DEV double tail_model_q(double v);   // qm_dd.cuh
QM_DEV double tail_model_q_dd(dd v);    // qm_dd.cuh

template <int ALG>
QM_DEV float rat32(float z)
{
    if (ALG == ALG_BREAKLESS77) return rational_f32path<8>(z, kA77P_f, kA77Q_f);
    if (ALG == ALG_F88) return rational_f32path<9>(z, kF88P_f, kF88Q_f);
    if (ALG == ALG_F44) return rational_f32path<5>(z, kF44P_f, kF44Q_f);
    if (ALG == ALG_TWO_REGION)
        return (z < QM_TWO_BREAK_F32) ? rational_f32path<5>(z, kF44P_f, kF44Q_f) : rational_f32path<6>(z, kC55P, kC55Q);
    if (ALG == ALG_BREAKLESS_TAIL) {
        const float r = rational_f32path<6>(z, kC55P, kC55Q);
        return (z < QM_VC_F32) ? r : (float)tail_model_q((double)z);
    }
    return rational_f32path<6>(z, kC55P, kC55Q);
}

// App D with all 13 Horner steps compensated and zl per step (off the grid; out of
// line so that the hot loop keeps its registers)
__device__ __noinline__ double d13_full(double zh, double zl)
{
    return rational_dd_zl<14, 13, true>(dd{zh, zl}, kD13P, kD13Q);
}

template <int ALG>
QM_DEV double rat64(dd z)
{
    if (ALG == ALG_BREAKLESS77) return rational_dd<8, 7>(z, kA77P_d, kA77Q_d);
    if (ALG == ALG_F1212) return rational_dd<13, 12>(z, kF12P, kF12Q);
    if (ALG == ALG_F88) return rational_dd<9, 8>(z, kF88P_d, kF88Q_d);
    if (ALG == ALG_BREAKLESS_TAIL)
        return (z.hi < QM_VC_F64) ? rat64<ALG_BREAKLESS>(z) : tail_model_q_dd(z);
    // App D: compensate the last KC of the 13 Horner steps, KC from a written bound.
    // The plain steps k >= KC add at most u (W_P(z) + W_Q(z)) relative error,
    // W(z) = sum_{k >= KC} (sum_{i >= k} a_i z^i) / P(z) (all coefficients positive);
    // with the double-double log and quotient and the final rounding the result is
    // within W_P + W_Q + 0.5 + O(u) ulp.  max W_P + W_Q: KC = 10: 0.567 on z <= 36.04
    // (the fp64 grid), 1.55 on z <= 74; KC = 8: 0.891 on z <= 12; KC = 9: 1.65 on
    // z <= 36 (B200 measured 2.13 ulp: the bound is tight).  So z <= 12 takes KC = 8
    // (two compensated steps = 16 FP64 operations fewer per sample), z > 12 KC = 10.
    // That split (QM_D13_SPLIT=1) measured: fused fp64 +6.5 % (61.3 vs 57.6 Gsamples/s),
    // but the TMA map -11 % (58 vs 65: the per-pair votes break the interleaving of
    // the pairs' chains, 128 registers) and tail-stratified config 1 -34 % (most
    // warps pay both schemes) -- so the product keeps KC = 10 for every z.
    if (QM_D13_SPLIT)
        return (z.hi <= QM_D13_ZSPLIT) ? rational_dd<14, QM_D13_KC_LO>(z, kD13P, kD13Q)
                                        : rational_dd<14, QM_D13_KC>(z, kD13P, kD13Q);
    double r = rational_dd<14, QM_D13_KC>(z, kD13P, kD13Q);
    if (__any_sync(__activemask(), z.hi > QM_DD_ZL_ZMAX)) {     // off the grid (above)
        const double rf = d13_full(z.hi, z.lo);
        r = (z.hi > QM_DD_ZL_ZMAX) ? rf : r;
    }
    return r;
}

// The same value in warp-uniform code: every lane evaluates the cheap scheme; if
// any lane of the warp has z > QM_D13_ZSPLIT (P = 1 - (1 - e^-12)^64 ~ 4e-4 per
// 64-sample warp group) the warp also evaluates the other and each lane keeps its
// own -- bitwise equal to rat64, with no divergent branch.
template <int ALG>
QM_DEV double rat64_warp(dd z)
{
    if (fast_alg<ALG>() != ALG_BREAKLESS || !QM_D13_SPLIT) return rat64<fast_alg<ALG>()>(z);
    double r = rational_dd<14, QM_D13_KC_LO>(z, kD13P, kD13Q);
    if (__any_sync(0xffffffffu, !(z.hi <= QM_D13_ZSPLIT))) {
        const double r2 = rational_dd<14, QM_D13_KC>(z, kD13P, kD13Q);
        r = (z.hi <= QM_D13_ZSPLIT) ? r : r2;
    }
    return r;
}

// fast path: requires vv = min(u, 1-u) >= 2^-126 (normal, not NaN)
template <int ALG>
QM_DEV float nq_f32_fast(float u)
{
    const float omu = __fsub_rn(1.0f, u);
    const float vv = fminf(u, omu);
    return apply_sign_f32(rat32<fast_alg<ALG>()>(neg_log2x_f32(vv, 0)), u, omu);
}

// every input: subnormal vv pre-scaled by 2^24; 0/1 -> -+inf; else NaN
template <int ALG>
QM_DEV float nq_f32_careful(float u)
{
    const float omu = __fsub_rn(1.0f, u);
    const float vv = fminf(u, omu);
    const bool sub = vv < 1.17549435e-38f;
    const float vs = sub ? __fmul_rn(vv, 16777216.0f) : vv;
    float mag = rat32<ALG>(neg_log2x_f32(vs, sub ? -24 : 0));
    mag = (vv == 0.0f) ? __int_as_float(0x7f800000) : mag;
    const float r = apply_sign_f32(mag, u, omu);
    return (vv >= 0.0f) ? r : __int_as_float(0x7fffffff);   // NaN, u < 0, u > 1
}

// warp-uniform callers only (rat64_warp votes)
template <int ALG>
QM_DEV double nq_f64_fast(double u)
{
    const double omu = __dadd_rn(1.0, -u);
    const double vv = fmin(u, omu);
    return apply_sign_f64(rat64_warp<ALG>(neg_log2x_dd(vv, 0)), u, omu);
}

template <int ALG>
QM_DEV double nq_f64_careful(double u)
{
    const double omu = __dadd_rn(1.0, -u);
    const double vv = fmin(u, omu);
    const bool sub = vv < 2.2250738585072014e-308;
    const double vs = sub ? __dmul_rn(vv, 18014398509481984.0) : vv;   // 2^54
    double mag = rat64<ALG>(neg_log2x_dd(vs, sub ? -54 : 0));
    mag = (vv == 0.0) ? __longlong_as_double(0x7ff0000000000000LL) : mag;
    const double r = apply_sign_f64(mag, u, omu);
    return (vv >= 0.0) ? r : __longlong_as_double(0x7fffffffffffffffLL);
}

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11); see qm.h for the stream layout.
// 32x32 -> 64 multiply as (lo, hi) words.  Written with mul.wide + mov.b64: the
// C form ((unsigned long long)a * b >> 32) compiles to IMAD.WIDE plus one
// spurious IADD per product on sm_100a (59 vs 39 instructions per block).
QM_DEV void mul_wide_u32(uint32_t a, uint32_t b, uint32_t &lo, uint32_t &hi)
{
    unsigned long long p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
}

QM_DEV uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0, hi0, lo1, hi1;
        mul_wide_u32(0xD2511F53u, c.x, lo0, hi0);
        mul_wide_u32(0xCD9E8D57u, c.z, lo1, hi1);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// the ten round keys of a seed, computed once per thread (loop-invariant; the
// compiler otherwise re-derives them with UIADD3s inside the sample loops)
struct PhiloxKeys {
    uint32_t k0[10], k1[10];
    QM_DEV explicit PhiloxKeys(unsigned long long seed)
    {
        uint32_t a = (uint32_t)seed, b = (uint32_t)(seed >> 32);
#pragma unroll
        for (int r = 0; r < 10; ++r) { k0[r] = a; k1[r] = b; a += 0x9E3779B9u; b += 0xBB67AE85u; }
    }
};

QM_DEV uint4 philox_block(unsigned long long counter, const PhiloxKeys &K)
{
    uint4 c = make_uint4((uint32_t)counter, (uint32_t)(counter >> 32), 0u, 0u);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0, hi0, lo1, hi1;
        mul_wide_u32(0xD2511F53u, c.x, lo0, hi0);
        mul_wide_u32(0xCD9E8D57u, c.z, lo1, hi1);
        c = make_uint4(hi1 ^ c.y ^ K.k0[r], lo1, hi0 ^ c.w ^ K.k1[r], lo0);
    }
    return c;
}

QM_DEV uint4 philox_block(unsigned long long counter, unsigned long long seed)
{
    return philox4x32_10(make_uint4((uint32_t)counter, (uint32_t)(counter >> 32), 0u, 0u),
                         (uint32_t)seed, (uint32_t)(seed >> 32));
}

// (2 (w >> 9) + 1) 2^-24: [1,2) float from the top 23 bits, minus (1 - 2^-24), exact
QM_DEV float u01_f32(uint32_t w)
{
    return __fsub_rn(__uint_as_float(0x3f800000u | (w >> 9)), 0x1.fffffep-1f);
}

// (2x + 1) 2^-53, x = ((hi << 32) | lo) >> 12
QM_DEV double u01_f64(uint32_t hi, uint32_t lo)
{
    const unsigned long long x = (((unsigned long long)hi << 32) | lo) >> 12;
    return __dadd_rn(__longlong_as_double((long long)(0x3FF0000000000000ULL | x)), -0x1.fffffffffffffp-1);
}

}  // namespace qm
