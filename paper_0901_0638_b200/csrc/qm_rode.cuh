// qm_rode.cuh -- recycling by a numerically solved Recycling ODE: exponential
// base into hyperbolic / variance-gamma samples (§4 of the
// paper) and Gaussian base into Student-t samples (§3.6, P:282-283;
// reading R35).
//
// The map Q(v) is built on the host (qm_rode_host.cpp) into a table of (Q, Q', Q'')
// at the nodes of a centre (octave levels, R36), a fine and a coarse segment per
// side (qm_rode_params.h).  Per sample the kernel does a quintic Hermite
// interpolation between two nodes (the error is O(h^6), relative accuracy near
// v = 0 from the octave spacing); the centre's nodes are staged in shared memory
// and a warp whose samples all lie there takes a fast path (explicit shared
// loads, the coordinate from the bits of |v|/Wc).  Past the last node (no double
// uniform reaches it) linear extrapolation with the end slope (Q' -> 1 in the
// tails; log-linear for the Student table).  The fused sampler draws u
// from Philox and applies the base quantile Q0 of P:322-329 first.
#pragma once
#include "qm_dd.cuh"
#include "qm_rode_params.h"
#include "qm_tma.cuh"

namespace qm {

// Centre-segment nodes staged in shared memory: (R, R', R'') per node, 3 doubles,
// nodes 0..Nc of both sides (2 x 3585 x 24 B = 172 KB).  The centre covers
// rate |v| <= 10 (99.995 % of the base samples; |z| <= 4.5 = 1 - 7e-6 for the
// Student table; rate |v| <= 2 = 86 % for a real-lambda VG table); the other
// nodes are gathered from the table in global memory (L2-resident).
constexpr int kRodeSmemNodes = QM_RODE_CENTRE_NODES + 1;
// SIDES = 1: an odd map (Student, R35): only side 0 staged, the sign applied at the end
template <int SIDES>
constexpr size_t rode_smem_bytes(int m) { return (size_t)(QM_RODE_HEADER + SIDES * m * 3) * sizeof(double); }
constexpr size_t kRodeSmemBytes = rode_smem_bytes<2>(kRodeSmemNodes);
// with the TMA input pipeline nodes 0..Nc-1 of each side: every centre interval
// but the last
#ifndef QM_RODE_TL_NODES
#define QM_RODE_TL_NODES QM_RODE_CENTRE_NODES
#endif
constexpr int kRodeTlNodes = QM_RODE_TL_NODES;
#ifndef QM_RODE_TL_NC
#define QM_RODE_TL_NC 16   // A/B knob: consumer warps of the RODE pipeline
#endif
constexpr int kRodeTlNC = QM_RODE_TL_NC;
// the TMA ring: 3 x 16 KB beside both sides' nodes (173 KB); 4 x 32 KB beside one side's
#ifndef QM_RODE_SYM_STAGES
#define QM_RODE_SYM_STAGES 4
#endif
#ifndef QM_RODE_SYM_TILE
#define QM_RODE_SYM_TILE 2048
#endif
template <int SIDES> struct RodeTl {
    static constexpr int stages = SIDES == 2 ? 3 : QM_RODE_SYM_STAGES;
    static constexpr int tile_vecs = SIDES == 2 ? 1024 : QM_RODE_SYM_TILE;
    static constexpr size_t ring_bytes = (size_t)stages * tile_vecs * 16;
    static constexpr size_t smem_bytes = ring_bytes + rode_smem_bytes<SIDES>(kRodeTlNodes);
};
static_assert(RodeTl<1>::smem_bytes <= 227 * 1024 && RodeTl<2>::smem_bytes <= 227 * 1024, "shared memory");
constexpr int kRodeTlTileVecs = RodeTl<2>::tile_vecs;
constexpr size_t kRodeTlSmemBytes = RodeTl<2>::smem_bytes;

// shared-memory layout: the table header (segment records, Vmax; 80 doubles),
// then (R, R') pairs of nodes 0..M-1 of side 0 and of side 1 (16 B each: one
// 128-bit load), then R'' of the same nodes (8 B each) -- 24 B per node, 4 loads
// per sample (the two nodes of its interval) instead of 6
constexpr int kRodeSmHdr = QM_RODE_HEADER;

template <int M = kRodeSmemNodes, int SIDES = 2>
QM_DEV void rode_stage_centre(const double *__restrict__ tab, double *sm)
{
    for (int i = threadIdx.x; i < kRodeSmHdr; i += blockDim.x) sm[i] = __ldg(tab + i);
    for (int i = threadIdx.x; i < SIDES * M; i += blockDim.x) {
        const int side = i / (M > 0 ? M : 1), k = i - side * M;
        const double *g = tab + QM_RODE_HEADER + side * 4 * (QM_RODE_NT + 1) + 4 * k;
        double *d = sm + kRodeSmHdr + 2 * i;
        d[0] = __ldg(g); d[1] = __ldg(g + 1);
        sm[kRodeSmHdr + 2 * SIDES * M + i] = __ldg(g + 2);
    }
    __syncthreads();
}

// one sample split in three phases so that a batch of samples has all its node
// gathers in flight together (a warp waits for its slowest lane: one lane with a
// node in L2 stalls the warp for the L2 latency)
struct RodePrep {
    const double *b;     // (R, R') of node k of the sample's side (shared or global memory)
    const double *b2;    // R'' of node k
    int st, st2;         // doubles from node k to node k+1 (shared 2 and 1, global 4 and 4)
    double t, a, vmax;
    // dw/ds and d2w/ds2 at nodes k and k+1 (s = the node coordinate): h and 0 on a
    // uniform segment; on the graded centre segment of a real-lambda VG table
    // (w = Wc (s/n)^4, qm_rode_host.cpp): 4 G s^3 and 12 G s^2, G = Wc/n^4
    double ws0, ws1, wss0, wss1;
    bool lg;             // segment holds log |R| (Student coarse tail): the value is +-exp(q)
    bool neg;            // side 1 (v < 0)
    bool oc;             // on the octave-level centre (j = 0): R'' from the RODE when QM_RODE_ODE_D2
};

// per-side segment boundaries Wc, V and Vmax, held in registers (loaded once
// per thread): the segment choice needs no shared-memory load
struct RodeBounds {
    double wc0, wc1, v0, v1, vm0, vm1;
    double iwc0, iwc1;   // 1/Wc per side (the centre record's 1/h slot when graded or on octaves)
    double nu, nu1;      // Student table: n and n + 1 (table[2]); R'' from the RODE (rode_student_d2)
    double ha, hb, hd2;  // hyperbolic table: alpha, beta, delta^2 (table[3..5]; rode_hyp_d2)
    double rate0, rate1; // base rates per side (table[10 + s])
};
QM_DEV RodeBounds rode_bounds(const double *__restrict__ tab)
{
    const double nu = __ldg(tab + 2);
    return RodeBounds{__ldg(tab + QM_RODE_SEG + 8), __ldg(tab + QM_RODE_SEG + 24 + 8),
                      __ldg(tab + QM_RODE_SEG + 16), __ldg(tab + QM_RODE_SEG + 24 + 16),
                      __ldg(tab + 28), __ldg(tab + 29), __ldg(tab + QM_RODE_SEG + 2), __ldg(tab + QM_RODE_SEG + 24 + 2),
                      nu, nu + 1.0, __ldg(tab + 3), __ldg(tab + 4), __ldg(tab + 5), __ldg(tab + 10), __ldg(tab + 11)};
}

// R'' of the Student table's centre nodes from the RODE itself instead of a third
// shared load (the table stores the same quantity, rounded from long double):
//     R'' = H(R) R'^2 - w R',  H(R) = (n + 1) R / (n + R^2)      (Gaussian base)
// at the node w.  The map was bound by the shared-memory data pipe (89 % of its peak:
// random 8-byte gathers cost ~6 wavefronts per warp for 256 bytes); dropping the R''
// loads trades 2 of the 4 gathers per sample for ~14 FP64 operations.  The second
// derivative enters the quintic with weight ~(h/w)^2 < 1e-5, so the ~2^-45 relative
// error of this evaluation (one Newton step on the reciprocal) is below 1e-19 of R.
// The generic path (rode_map_batch) does the same for centre samples, so a sample's
// bits do not depend on its warp's path; the fine and coarse segments keep the stored
// R''.  (The same for the hyperbolic table, QM_RODE_ODE_D2=2 with a reciprocal square
// root per node, measured -11 % and stays off.)
#ifndef QM_RODE_ODE_D2
#define QM_RODE_ODE_D2 1   // A/B: 0 = the stored R'' on every path; 2 = also the hyperbolic table's
#endif
// the same for the hyperbolic table (exponential base):
//     R'' = H(R) R'^2 - rate_s R',  H(x) = alpha x / sqrt(delta^2 + x^2) - beta
// (1/sqrt from MUFU.RSQ64H and one Newton step: ~2^-46; the weight of R'' is < 1e-5)
QM_DEV double rode_hyp_d2(double r, double rp, double rate, const RodeBounds &bd)
{
    const double s = __fma_rn(r, r, bd.hd2);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    y = __fma_rn(__dmul_rn(0.5, y), __fma_rn(-s, __dmul_rn(y, y), 1.0), y);
    const double H = __fma_rn(__dmul_rn(bd.ha, r), y, -bd.hb);
    return __dmul_rn(rp, __fma_rn(H, rp, -rate));
}
QM_DEV double rode_student_d2(double r, double rp, double w, const RodeBounds &bd)
{
    const double s = __fma_rn(r, r, bd.nu);
    double q = rcp_approx_f64(s);
    q = __fma_rn(q, __fma_rn(-s, q, 1.0), q);
    const double H = __dmul_rn(__dmul_rn(bd.nu1, r), q);
    return __dmul_rn(rp, __fma_rn(rp, H, -w));
}

// one double from shared memory by its 32-bit shared address (an explicit LDS,
// not a generic load)
QM_DEV double lds_f64(uint32_t addr)
{
    double r;
    asm("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(addr));
    return r;
}
// select without a branch (the compiler turned some double selects of the
// octave path into divergent branches)
QM_DEV double sel_f64(bool c, double a, double b)
{
    double r;
    asm("{ .reg .pred p; setp.ne.u32 p, %3, 0; selp.f64 %0, %1, %2, p; }" : "=d"(r) : "d"(a), "d"(b), "r"((unsigned)c));
    return r;
}

// MODE: the table's features, a kernel-level (warp-uniform) dispatch on the header,
// so that each table pays only for its own: bit 0 = centre nodes at Wc (k/n)^4
// (table[32 + 7] = 4), bit 2 = centre on octave levels (= 1), bit 1 = log-valued
// segment 2 (Student, table[31])
// bit 3 = hyperbolic octave table (R'' from the RODE, QM_RODE_ODE_D2 >= 2)
constexpr int kRodeGraded = 1, kRodeLog = 2, kRodeOct = 4, kRodeHyp = 8;
QM_DEV int rode_mode(const double *__restrict__ tab)
{
    const double g = __ldg(tab + QM_RODE_SEG + 7);
    const bool hyp = QM_RODE_ODE_D2 >= 2 && g == 1.0 && __ldg(tab) == (double)QM_RODE_HYPERBOLIC;
    return (g == 4.0 ? kRodeGraded : 0) | (g == 1.0 ? kRodeOct : 0) | (__ldg(tab + 31) != 0.0 ? kRodeLog : 0) |
           (hyp ? kRodeHyp : 0);
}

// octave-level coordinate of x = w/Wc in [0, 1) (R36; L + 1 levels of NB intervals):
// x = 2^e m, level l = e + L + 1 (0 below 2^-L); on levels l >= 1 the node index
// is NB l + the top 9 bits of m's fraction and the local coordinate t the other
// 43 bits (exact, integer operations); level 0 is uniform, s = 2^(9+L) x.  Node
// step h = Wc 2^(max(l,1) - L - 10).  (Computing s = 512 (m - 1) + 512 l in double
// would round t to 41 bits on the upper levels.)
struct OctCoord { int k; double t, h; };
QM_DEV OctCoord oct_coord(double x, double wc)
{
    constexpr int L = QM_RODE_OCT_LEVELS - 1, NB = QM_RODE_OCT_NODES;
    static_assert(NB == 512 && L == 6, "the bit layout below assumes 512 intervals per level, 7 levels");
    const long long xb = __double_as_longlong(x);
    const int l = min(max((int)(xb >> 52) - 1023 + L + 1, 0), L);
    const long long mant = xb & 0x000fffffffffffffLL;
    const int k1 = NB * l + (int)(mant >> 43);
    const double t1 = __longlong_as_double(0x3ff0000000000000LL | ((mant << 9) & 0x000fffffffffffffLL)) - 1.0;
    const double s0 = x * (double)(NB << L);
    const double f0 = floor(s0);
    OctCoord c;
    c.k = (l == 0) ? (int)f0 : k1;
    c.t = sel_f64(l == 0, s0 - f0, t1);
    c.h = wc * __longlong_as_double((long long)(1023 + max(l, 1) - L - 1 - 9) << 52);
    return c;
}

template <int M, int MODE, int SIDES = 2>
QM_DEV RodePrep rode_prep(const double *__restrict__ tab, double v, const double *sm, const RodeBounds &bd)
{
    const int side = (SIDES == 2 && v < 0.0) ? 1 : 0;
    const double a = fabs(v);
    const double wc = side ? bd.wc1 : bd.wc0, vb = side ? bd.v1 : bd.v0;
    // segment j = [a >= Wc] + [a >= V] (selects; NaN lands in j = 0 and is replaced later)
    const int j = (a >= wc) + (a >= vb);
    // the segment record (w0, h | 1/h, k0 | n, w1 | G, graded) as four 16-byte shared loads
    const double2 *r = reinterpret_cast<const double2 *>(sm + QM_RODE_SEG + 24 * side + 8 * j);
    const double2 r01 = r[0], r23 = r[1], r45 = r[2], r67 = r[3];
    double s = (a - r01.x) * r23.x;                             // local coordinate in [0, n]
    // graded centre (r23.x = 1/Wc, r67 = (G, g)): s = n (w/Wc)^(1/g)
    const bool g4 = (MODE & kRodeGraded) && r67.y == 4.0;
    if (MODE & kRodeGraded) s = g4 ? r45.x * sqrt(sqrt(a * r23.x)) : s;
    s = fmin(s, r45.x);
    double fk = fmin(floor(s), r45.x - 1.0), t = s - fk, hoct = 0.0;
    if (MODE & kRodeOct) {                                      // centre on octave levels (R36)
        const bool oc = (j == 0) && r67.y == 1.0;
        const OctCoord c = oct_coord(a * r23.x, r45.y);         // r45.y = w1 = Wc
        fk = oc ? (double)c.k : fk;
        t = sel_f64(oc, c.t, t);
        hoct = oc ? c.h : 0.0;
    }
    const int k = (int)r23.y + (int)fk;
    const bool in_sm = (M > 0) && (j == 0) && (k + 1 < M);
    RodePrep p;
    // (R, R') of node k and its R'': shared (pairs array, R'' array) or global (4-double records)
    p.b = in_sm ? sm + kRodeSmHdr + 2 * (side * M + k) : tab + QM_RODE_HEADER + side * 4 * (QM_RODE_NT + 1) + 4 * k;
    p.b2 = in_sm ? sm + kRodeSmHdr + 2 * SIDES * M + (side * M + k) : p.b + 2;
    p.st = in_sm ? 2 : 4;
    p.st2 = in_sm ? 1 : 4;
    p.t = t;
    p.a = a;
    p.vmax = side ? bd.vm1 : bd.vm0;
    const double k1 = fk + 1.0;
    // dw/ds and d2w/ds2 at the two nodes: h, 0 (uniform); 4 G s^3, 12 G s^2 (graded)
    p.ws0 = g4 ? 4.0 * r67.x * fk * fk * fk : ((MODE & kRodeOct) && hoct != 0.0 ? hoct : r01.y);
    p.ws1 = g4 ? 4.0 * r67.x * k1 * k1 * k1 : ((MODE & kRodeOct) && hoct != 0.0 ? hoct : r01.y);
    p.wss0 = g4 ? 12.0 * r67.x * fk * fk : 0.0;
    p.wss1 = g4 ? 12.0 * r67.x * k1 * k1 : 0.0;
    p.lg = (MODE & kRodeLog) && j == 2;
    p.oc = (MODE & kRodeOct) && j == 0 && r67.y == 1.0;
    p.neg = side != 0;
    return p;
}

struct RodeNodes { double r0, d0, dd0, r1, d1, dd1; };

template <int M>
QM_DEV RodeNodes rode_load(const RodePrep &p)
{
    if constexpr (M == 0) {   // every node from global memory (L1-cached 16-byte gathers)
        const double2 n0 = __ldg(reinterpret_cast<const double2 *>(p.b));
        const double2 n1 = __ldg(reinterpret_cast<const double2 *>(p.b + 4));
        return RodeNodes{n0.x, n0.y, __ldg(p.b + 2), n1.x, n1.y, __ldg(p.b + 6)};
    } else {
        return RodeNodes{p.b[0], p.b[1], p.b2[0], p.b[p.st], p.b[p.st + 1], p.b2[p.st2]};
    }
}

// quintic Hermite in monomial form: R(k h + t h) = p0 + m0 t + a0/2 t^2 + c3 t^3 + c4 t^4 + c5 t^5
// (inside the table; rode_finish adds the extrapolation beyond Vmax)
template <int MODE>
QM_DEV double rode_interp(const RodePrep &p, const RodeNodes &n)
{
    const double t = p.t;
    // derivatives with respect to s: dR/ds = R' w_s, d2R/ds2 = R'' w_s^2 + R' w_ss
    const double m0 = p.ws0 * n.d0, m1 = p.ws1 * n.d1;
    constexpr bool GR = (MODE & kRodeGraded) != 0;
    const double a0 = GR ? __fma_rn(p.ws0 * p.ws0, n.dd0, p.wss0 * n.d0) : p.ws0 * p.ws0 * n.dd0;
    const double a1 = GR ? __fma_rn(p.ws1 * p.ws1, n.dd1, p.wss1 * n.d1) : p.ws1 * p.ws1 * n.dd1;
    const double dp = n.r1 - n.r0;
    const double c3 = 10.0 * dp - 6.0 * m0 - 4.0 * m1 - 1.5 * a0 + 0.5 * a1;
    const double c4 = -15.0 * dp + 8.0 * m0 + 7.0 * m1 + 1.5 * a0 - a1;
    const double c5 = 6.0 * dp - 3.0 * m0 - 3.0 * m1 - 0.5 * a0 + 0.5 * a1;
    return n.r0 + t * (m0 + t * (0.5 * a0 + t * (c3 + t * (c4 + t * c5))));
}
template <int MODE>
QM_DEV double rode_finish(const RodePrep &p, const RodeNodes &n)
{
    const double q = rode_interp<MODE>(p, n);
    const double qx = n.r1 + (p.a - p.vmax) * n.d1;             // beyond Vmax: node k+1 = node NT
    return (p.a <= p.vmax) ? q : qx;
}

// log-valued segment (Student tail, 2e-9 of the normal samples): R = +-exp(q),
// evaluated only when a lane of the (active) warp needs it
template <int MODE>
QM_DEV double rode_unlog(const RodePrep &p, double q)
{
    if ((MODE & kRodeLog) && __any_sync(__activemask(), p.lg)) {
        const double e = exp(q);
        q = p.lg ? (p.neg ? -e : e) : q;
    }
    return q;
}

// IEEE semantics of the map: +-0 -> +-0, +-inf -> +-inf, NaN -> NaN
QM_DEV double rode_special(double v, double q)
{
    const double r = (v == 0.0) ? v : q;
    return (fabs(v) < __longlong_as_double(0x7ff0000000000000LL)) ? r : v;
}

// The centre on octave levels (R36; 99.995 % of the base samples) with every
// node in shared memory: the coordinate of oct_coord, explicit shared loads, no
// segment record.  Bitwise the same k, t and h as rode_prep.
struct RodeFast {
    uint32_t addr, addr2;  // shared addresses of node k's (R, R') and R''
    bool ok;               // a < Wc, node k+1 staged, finite
    RodePrep p;
};
QM_DEV double2 lds_f64x2(uint32_t addr)
{
    double2 r;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(addr));
    return r;
}
template <int M, int SIDES = 2>
QM_DEV RodeFast rode_fast_prep(double v, uint32_t sm_nodes, const RodeBounds &bd)
{
    const int side = (SIDES == 2 && v < 0.0) ? 1 : 0;
    const double a = fabs(v);
    const double wc = side ? bd.wc1 : bd.wc0, iwc = side ? bd.iwc1 : bd.iwc0;
    const OctCoord c = oct_coord(a * iwc, wc);
    RodeFast f;
    f.p.t = c.t;
    f.p.a = a;
    f.p.vmax = side ? bd.vm1 : bd.vm0;
    f.p.ws0 = f.p.ws1 = c.h;
    f.p.wss0 = f.p.wss1 = 0.0;
    f.p.lg = false;
    f.p.oc = true;
    f.p.neg = side != 0;
    f.p.b = f.p.b2 = nullptr;
    f.p.st = 2;
    f.p.st2 = 1;
    f.ok = (a < wc) && (c.k + 1 < M);
    const uint32_t node = (uint32_t)(side * M + min(c.k, M - 2));
    f.addr = sm_nodes + 16u * node;
    f.addr2 = sm_nodes + 16u * SIDES * (uint32_t)M + 8u * node;
    return f;
}

// B samples x[i] = Q(v[i]), in groups of up to 4 whose node gathers are all
// issued before their arithmetic (4 keeps the state in registers)
#ifndef QM_RODE_G
#define QM_RODE_G 4   // A/B knob: samples per gather group
#endif
// SIDES = 1 (odd map): side 0 for |v|, the sign of v at the end
QM_DEV double rode_odd(double v, double q) { return v < 0.0 ? -q : q; }

template <int M, int MODE, int SIDES = 2, int B>
QM_DEV void rode_map_batch(const double *__restrict__ tab, const double *sm, const RodeBounds &bd, const double (&v)[B],
                           double (&x)[B])
{
    constexpr int G = B < QM_RODE_G ? B : QM_RODE_G;
    static_assert(B % G == 0, "batch must split into groups of QM_RODE_G");
#pragma unroll
    for (int g = 0; g < B; g += G) {
        if constexpr ((MODE & kRodeOct) && M > 0) {
            // warp-uniform fast path: every lane's samples on the staged centre
            const uint32_t smn = (uint32_t)__cvta_generic_to_shared(sm + kRodeSmHdr);
            RodeFast f[G];
            bool ok = true;
#pragma unroll
            for (int k = 0; k < G; ++k) {
                f[k] = rode_fast_prep<M, SIDES>(v[g + k], smn, bd);
                ok = ok && f[k].ok;
            }
            if (__all_sync(__activemask(), ok)) {
                RodeNodes nd[G];
#pragma unroll
                for (int k = 0; k < G; ++k) {
                    const double2 n0 = lds_f64x2(f[k].addr), n1 = lds_f64x2(f[k].addr + 16);
                    if constexpr (SIDES == 1 && (MODE & kRodeLog) && QM_RODE_ODE_D2) {   // Student table
                        const double w0 = __fma_rn(-f[k].p.t, f[k].p.ws0, f[k].p.a), w1 = w0 + f[k].p.ws0;
                        nd[k] = RodeNodes{n0.x, n0.y, rode_student_d2(n0.x, n0.y, w0, bd),
                                          n1.x, n1.y, rode_student_d2(n1.x, n1.y, w1, bd)};
                    } else if constexpr (SIDES == 2 && (MODE & kRodeHyp)) {           // hyperbolic table
                        const double rate = f[k].p.neg ? bd.rate1 : bd.rate0;
                        nd[k] = RodeNodes{n0.x, n0.y, rode_hyp_d2(n0.x, n0.y, rate, bd),
                                          n1.x, n1.y, rode_hyp_d2(n1.x, n1.y, rate, bd)};
                    } else {
                        nd[k] = RodeNodes{n0.x, n0.y, lds_f64(f[k].addr2), n1.x, n1.y, lds_f64(f[k].addr2 + 8)};
                    }
                }
#pragma unroll
                for (int k = 0; k < G; ++k) {
                    const double q = rode_interp<MODE>(f[k].p, nd[k]);
                    x[g + k] = rode_special(v[g + k], SIDES == 1 ? rode_odd(v[g + k], q) : q);
                }
                continue;
            }
        }
        RodePrep p[G];
        RodeNodes nd[G];
#pragma unroll
        for (int k = 0; k < G; ++k) p[k] = rode_prep<M, MODE, SIDES>(tab, v[g + k], sm, bd);
#pragma unroll
        for (int k = 0; k < G; ++k) {
            nd[k] = rode_load<M>(p[k]);
            if constexpr (SIDES == 1 && (MODE & kRodeLog) && (MODE & kRodeOct) && QM_RODE_ODE_D2) {
                // the fast path's R'' for centre samples in the generic path too, bit for bit
                const double w0 = __fma_rn(-p[k].t, p[k].ws0, p[k].a), w1 = w0 + p[k].ws0;
                nd[k].dd0 = p[k].oc ? rode_student_d2(nd[k].r0, nd[k].d0, w0, bd) : nd[k].dd0;
                nd[k].dd1 = p[k].oc ? rode_student_d2(nd[k].r1, nd[k].d1, w1, bd) : nd[k].dd1;
            }
            if constexpr (SIDES == 2 && (MODE & kRodeHyp)) {
                const double rate = p[k].neg ? bd.rate1 : bd.rate0;
                nd[k].dd0 = p[k].oc ? rode_hyp_d2(nd[k].r0, nd[k].d0, rate, bd) : nd[k].dd0;
                nd[k].dd1 = p[k].oc ? rode_hyp_d2(nd[k].r1, nd[k].d1, rate, bd) : nd[k].dd1;
            }
        }
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const double q = rode_unlog<MODE>(p[k], rode_finish<MODE>(p[k], nd[k]));
            x[g + k] = rode_special(v[g + k], SIDES == 1 ? rode_odd(v[g + k], q) : q);
        }
    }
}

// kernel-level dispatch on the table's MODE (uniform for the whole grid)
#define QM_RODE_DISPATCH(tab, CALL)                                                 \
    switch (rode_mode(tab)) {                                                       \
    case kRodeOct: CALL(kRodeOct); break;                                           \
    case kRodeOct | kRodeLog: CALL(kRodeOct | kRodeLog); break;                     \
    case kRodeOct | kRodeHyp: CALL(kRodeOct | kRodeHyp); break;                     \
    case kRodeGraded: CALL(kRodeGraded); break;                                     \
    default: CALL(kRodeGraded | kRodeOct | kRodeLog); break;                        \
    }

template <typename T, int MODE, int SIDES>
QM_DEV void rode_map_body(const T *__restrict__ v, T *__restrict__ x, int64_t n, const double *__restrict__ tab,
                          const double *rode_sm, const RodeBounds &bd)
{
    constexpr int U = 4;
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * S) {
        double a[U], r[U];
#pragma unroll
        for (int k = 0; k < U; ++k) a[k] = (i0 + k * S < n) ? (double)v[i0 + k * S] : 0.0;
        rode_map_batch<kRodeSmemNodes, MODE, SIDES>(tab, rode_sm, bd, a, r);
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i0 + k * S < n) x[i0 + k * S] = (T)r[k];
    }
}

template <typename T, int SIDES = 2>
__global__ void __launch_bounds__(512, 1)
k_rode_map(const T *__restrict__ v, T *__restrict__ x, int64_t n, const double *__restrict__ tab)
{
    extern __shared__ __align__(16) double rode_sm[];
    rode_stage_centre<kRodeSmemNodes, SIDES>(tab, rode_sm);
    const RodeBounds bd = rode_bounds(tab);
#define QM_RODE_MAP_CALL(MD) rode_map_body<T, MD, SIDES>(v, x, n, tab, rode_sm, bd)
    QM_RODE_DISPATCH(tab, QM_RODE_MAP_CALL)
#undef QM_RODE_MAP_CALL
}

// the map through the TMA-in / streaming-store pipeline (qm_tma.cuh): the
// input stream no longer waits on registers (the LDG kernel's stalls were on
// the loads of v, not on the table); nodes 0..3599 of the centre in shared memory
template <typename V> struct RodeVec;
template <> struct RodeVec<double2> { using T = double; static constexpr int W = 2; };
template <> struct RodeVec<float4> { using T = float; static constexpr int W = 4; };

template <typename V, int MODE, int SIDES>
struct MapRode {
    const double *tab;
    const double *sm;
    RodeBounds bd;
    template <int PER>
    QM_DEV void map_slice(V *a) const
    {
        using T = typename RodeVec<V>::T;
        constexpr int W = RodeVec<V>::W;
        T *e = reinterpret_cast<T *>(a);
        double in[PER * W], out[PER * W];
#pragma unroll
        for (int k = 0; k < PER * W; ++k) in[k] = (double)e[k];
        rode_map_batch<kRodeTlNodes, MODE, SIDES>(tab, sm, bd, in, out);
#pragma unroll
        for (int k = 0; k < PER * W; ++k) e[k] = (T)out[k];
    }
};

template <typename V, int SIDES = 2>
__global__ void __launch_bounds__(32 * (kRodeTlNC + 1), 1)
k_rode_map_tl(const V *__restrict__ v, V *__restrict__ x, int64_t ntiles, const double *__restrict__ tab)
{
    using C = RodeTl<SIDES>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sm = reinterpret_cast<double *>(smem_raw + C::ring_bytes);
    rode_stage_centre<kRodeTlNodes, SIDES>(tab, sm);
    const RodeBounds bd = rode_bounds(tab);
#define QM_RODE_TL_CALL(MD) \
    tma_load_map<V, C::tile_vecs, C::stages, kRodeTlNC>(v, x, ntiles, MapRode<V, MD, SIDES>{tab, sm, bd})
    QM_RODE_DISPATCH(tab, QM_RODE_TL_CALL)
#undef QM_RODE_TL_CALL
}

// base quantile Q0: u < p- -> log(u/p-)/(a+b); u > p- -> -log((1-u)/p+)/(a-b).
// |v| = (-log t + log p_s)/rate_s with t = u (left) or 1-u (right), exact on the odd grid.
QM_DEV double exp_base_quantile(const double *__restrict__ tab, double u)
{
    const int side = (u < __ldg(tab + 9)) ? 1 : 0;             // tab[9] = p-
    const double t = side ? u : __dadd_rn(1.0, -u);
    const dd L = neg_log_dd(t);                                 // -log t
    const dd m = dd_add(L, dd{__ldg(tab + 16 + side), __ldg(tab + 18 + side)});
    const double av = (m.hi + m.lo) * __ldg(tab + 20 + side);
    return side ? -av : av;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_exp_base_quantile(const T *__restrict__ u, T *__restrict__ v, int64_t n, const double *__restrict__ tab)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double ui = (double)u[i];
        const double r = exp_base_quantile(tab, ui);
        v[i] = (T)((ui > 0.0 && ui < 1.0) ? r : (ui == 0.0 ? -__longlong_as_double(0x7ff0000000000000LL)
                                                  : (ui == 1.0 ? __longlong_as_double(0x7ff0000000000000LL)
                                                               : __longlong_as_double(0x7fffffffffffffffLL))));
    }
}

// fused: Philox uniforms (qm_philox_uniform layout) -> Q0 -> Q
template <typename T, int MODE>
QM_DEV void rode_philox_body(T *__restrict__ x, int64_t n, unsigned long long seed, unsigned long long c0,
                             const double *__restrict__ tab, const double *rode_sm, const RodeBounds &bd)
{
    constexpr int W = (sizeof(T) == 4) ? 4 : 2;                 // samples per Philox block
    const int64_t nb = (n + W - 1) / W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // two Philox blocks per iteration, every sample computed before the stores
    // (the table gathers of all samples in flight together)
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b0 < nb; b0 += 2 * stride) {
        double u[2 * W], r[2 * W];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint4 w = philox_block(c0 + (unsigned long long)(b0 + h * stride), seed);
            if (W == 4) {
                u[4 * h] = u01_f32(w.x); u[4 * h + 1] = u01_f32(w.y); u[4 * h + 2] = u01_f32(w.z); u[4 * h + 3] = u01_f32(w.w);
            } else {
                u[2 * h] = u01_f64(w.x, w.y); u[2 * h + 1] = u01_f64(w.z, w.w);
            }
        }
#pragma unroll
        for (int k = 0; k < 2 * W; ++k) u[k] = exp_base_quantile(tab, u[k]);
        rode_map_batch<kRodeSmemNodes, MODE, 2>(tab, rode_sm, bd, u, r);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t b = b0 + h * stride;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int64_t i = b * W + k;
                if (b < nb && i < n) x[i] = (T)r[W * h + k];
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(512, 1)
k_rode_philox(T *__restrict__ x, int64_t n, unsigned long long seed, unsigned long long c0,
              const double *__restrict__ tab)
{
    extern __shared__ __align__(16) double rode_sm[];
    rode_stage_centre(tab, rode_sm);
    const RodeBounds bd = rode_bounds(tab);
#define QM_RODE_PHILOX_CALL(MD) rode_philox_body<T, MD>(x, n, seed, c0, tab, rode_sm, bd)
    QM_RODE_DISPATCH(tab, QM_RODE_PHILOX_CALL)
#undef QM_RODE_PHILOX_CALL
}

}  // namespace qm
