/*
 * orc_normal.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Everything the normal-quantile rows of SURVEY.md §8 compute, written out in
 * long double in the paper's order:
 *   - the exact quantile w(u), F(w(u)) = u (§1), by bracketed Newton
 *     on erfl/erfcl -- the plain definition, never forming 1 - Phi;
 *   - the exact exponential-coordinate map Q(v) = Phi^-1(1 - e^-v / 2)
 *     (§5);
 *   - the paper's breakless rationals Q(v) = v P(v)/Q(v): (7,7) of App A/B
 *     (P:477-497), (5,5) of App C, (13,13) of App D
 *     (P:821-848), with the coefficients rounded to the target type exactly as
 *     the listings declare them (`const float` / `const double`), or kept as
 *     long-double decimals for the formula-vs-exact bounds;
 *   - the sampling algorithm: vv = min(u, 1-u), z = -log(2 vv), sign flip
 *     (§5; App D);
 *   - the antithetic variant v = -log u -> {Z, -Z};
 *   - the exponential (Laplace) base: Z = sign(v) Q(|v|);
 *   - the Taylor series of Q at v = 0 and the supplementary tail
 *     model (§5.1; reading R1 of DESIGN.md: a = v - 1/2 log pi);
 *   - the comparison quantiles AS241 (Wichura 1988) and Acklam level 1 with the
 *     optional Halley refinement, which the paper benchmarks against
 *     (Table 3).  Their coefficients are NOT in
 *     the paper (P:601-616 point to external code); they are transcribed from
 *     the original publications (reading R17) and pinned by the accuracy the
 *     paper states for them (< 1.15e-9 for Acklam L1).
 */
#include <math.h>
#include <stdlib.h>
#include <stdint.h>
#include <float.h>
#include "orc.h"

/* formula ids (oracle-local; no shared enum with the product) */
#define ORC_C55 55
#define ORC_A77 77
#define ORC_D13 13
#define ORC_F1212 1212   /* (12,12) on [0, 37] */
#define ORC_F88 88       /* (8,8) on [0, 74] */
#define ORC_F44 44       /* (4,4) on [0, 10], first region of the two-region variant */
#define ORC_TWO 410      /* two regions: F44 for v < 10, App C (5,5) for v >= 10 */
/* coefficient precision: 32 = float-rounded, 64 = double-rounded, 0 = decimal */

/* App A / App B (7,7): P:477-497 (numerator), P:485-497 (denominator) */
static const char *A77_P[8] = {
    "1.2533141359896652729", "3.0333178251950406994", "2.3884158540184385711",
    "0.73176759583280610539", "0.085838533424158257377", "0.0034424140686962222423",
    "0.000036313870818023761224", "4.3304513840364031401e-8" };
static const char *A77_Q[8] = {
    "1", "2.9202373175993672857", "2.9373357991677046357", "1.2356513216582148689",
    "0.2168237095066675527", "0.014494272424798068406", "0.00030617264753008793976",
    "1.3141263119543315917e-6" };
/* App C (5,5): P:792-803 */
static const char *C55_P[6] = {
    "1.2533136835212087879", "1.9797154223229267471", "0.80002295072483916762",
    "0.087403248265958578062", "0.0020751409553756572917", "4.744820732427972462e-6" };
static const char *C55_Q[6] = {
    "1.0", "2.0795584360534589311", "1.2499328117341603014", "0.23668431621373705623",
    "0.0120098270559197768", "0.00010590620919921025259" };
/* App D (13,13): P:821-848 */
static const char *D13_P[14] = {
    "1.2533141373154989811", "5.5870183514814983104", "9.9373788223105148469",
    "9.11745910783758368", "4.6865666928347513004", "1.3841649695441184484",
    "0.23434950424605615377", "0.022306824510199724768", "0.0011538603964070818722",
    "0.000030796620691411567563", "3.9115723028719510263e-7", "2.0589573468131996933e-9",
    "3.3944224725087481454e-12", "7.3936480912071325978e-16" };
static const char *D13_Q[14] = {
    "1.00000000000000000000", "4.9577956835689939051", "9.9793129245112074476",
    "10.574454910639356539", "6.4247521669505779535", "2.3008904864351121026",
    "0.48545999687461771635", "0.059283082737079006352", "0.0040618506206078995821",
    "0.00014919732843986856251", "2.7477061392049947066e-6", "2.2815008011613816939e-8",
    "7.0445790305953963457e-11", "5.1535907808963289678e-14" };

/* Our minimax fits (tools/fit_rational.py), transcribed from
 * tests/golden/fit_*.txt: the (12,12) on [0,37] and (8,8) on [0,74] the paper
 * says exist, and the (4,4) on [0,10] of the two-region variant. */
static const char *F1212_P[13] = {
    "1.25331413731549964304885084933", "5.65670727193097123052913156555",
    "10.199184028049004645639650354", "9.49108178418734942631477139003",
    "4.94304333170547437473236493918", "1.47293406972979776643830812522",
    "0.249077147187243284286425789887", "0.0232075251548776468184535573962",
    "0.00113211638446441623489197365915", "0.000026638805014702015041938526811",
    "0.000000262823263993221383793586115962", "8.20115160731597726774034377471e-10",
    "3.4080843072305026219786124261e-13" };
static const char *F1212_Q[13] = {
    "1.0", "5.01339939725483198543174978089", "10.2160051129404404259102375667",
    "10.9670844662824747543017650822", "6.74844347326083628169062975985",
    "2.44148341873030012307321591735", "0.516866979805929966868864954603",
    "0.0624322209086865620690205639678", "0.00411740318775822728331972658499",
    "0.00013852471353158268838850038814", "0.00000213335696590330667438560151822",
    "0.0000000123741421877613097338506656296", "1.71840938834726185281010719498e-11" };
static const char *F88_P[9] = {
    "1.25331413659487693200589460544", "3.18279215828640909853465485323",
    "2.69637013151484046914318369988", "0.926505960348117503759109131467",
    "0.130722564999804748080717604434", "0.00715510742068364856695515828894",
    "0.000134566885939144919435102866116", "0.000000669320737492863356757758585237",
    "3.78894005999045094010072867485e-10" };
static const char *F88_Q[9] = {
    "1.0", "3.03950064147177248702038516122", "3.24267820535186536296356820427",
    "1.49261049909605991213659399514", "0.302049532338050455259987910733",
    "0.0255324575872787421879918341977", "0.000815155781723673184564102970288",
    "0.00000817923481671560569243134101007", "0.0000000166707331365471438381381542416" };
static const char *F44_P[5] = {
    "1.25331376367946351584057665416", "1.90154131297345796677471850561",
    "0.692706016566279324284406456679", "0.0560005883011708193276104273226",
    "0.000448739389131331445037989032119" };
static const char *F44_Q[5] = {
    "1.0", "2.01718797443210201360154517184", "1.13309652308639082468928923168",
    "0.179982309491888788965156666547", "0.0053418912252851127623755674913" };

static ld coef(const char *s, int prec)
{
    if (prec == 32) return (ld)(float)strtod(s, NULL);   /* `const float P1 = <double literal>;` */
    if (prec == 64) return (ld)strtod(s, NULL);          /* `const double P1 = ...;` */
    return strtold(s, NULL);                             /* decimal, for exact-arithmetic bounds */
}

/* one rational, or (two-region formula) a second one used for v >= vb */
typedef struct { int n; ld p[14]; ld q[14]; int n2; ld vb; ld p2[14]; ld q2[14]; } rat_t;
#define ORC_TWO_BREAK 10.0L

static int get_rat(int formula, int prec, rat_t *r)
{
    const char **P, **Q; int n;
    r->n2 = 0;
    if (formula == ORC_TWO) {            /* (4,4) below the break, App C above */
        rat_t hi;
        get_rat(ORC_C55, prec, &hi);
        get_rat(ORC_F44, prec, r);
        r->n2 = hi.n; r->vb = ORC_TWO_BREAK;
        for (int i = 0; i < hi.n; ++i) { r->p2[i] = hi.p[i]; r->q2[i] = hi.q[i]; }
        return 0;
    }
    switch (formula) {
    case ORC_A77: P = A77_P; Q = A77_Q; n = 8; break;
    case ORC_C55: P = C55_P; Q = C55_Q; n = 6; break;
    case ORC_D13: P = D13_P; Q = D13_Q; n = 14; break;
    case ORC_F1212: P = F1212_P; Q = F1212_Q; n = 13; break;
    case ORC_F88: P = F88_P; Q = F88_Q; n = 9; break;
    case ORC_F44: P = F44_P; Q = F44_Q; n = 5; break;
    default: return -1;
    }
    r->n = n;
    for (int i = 0; i < n; ++i) { r->p[i] = coef(P[i], prec); r->q[i] = coef(Q[i], prec); }
    return 0;
}

/* Q(v) = v * P(v) / Q(v), nested (Horner) form as printed. */
static ld rational_Q(const rat_t *r, ld v)
{
    const int second = r->n2 > 0 && v >= r->vb;
    const int n = second ? r->n2 : r->n;
    const ld *p = second ? r->p2 : r->p, *q = second ? r->q2 : r->q;
    ld P = p[n - 1], Q = q[n - 1];
    for (int i = n - 2; i >= 0; --i) { P = p[i] + v * P; Q = q[i] + v * Q; }
    return v * P / Q;
}

/* --------------------------------------------------------------------------
 * Exact quantile: x >= 0 with 1/2 erfc(x/sqrt2) = t, 0 < t <= 1/2.
 * For t > 1/4 solve 1/2 erf(x/sqrt2) = 1/2 - t instead (1/2 - t is exact), so
 * that the relative accuracy of small x is kept.  Bracketed Newton: a Newton
 * step that leaves the bracket is replaced by bisection.
 * ------------------------------------------------------------------------ */
static const ld SQRT1_2L = 0.707106781186547524400844362104849039L;
static const ld INV_SQRT_2PI_L = 0.398942280401432677939946059934381868L;

static ld solve_upper(ld t, ld half_minus_t)
{
    int central = (t > 0.25L);
    ld target = central ? half_minus_t : t;
    ld lo = 0.0L, hi = central ? 0.7L : 40.0L;
    ld x = central ? target * 2.50662827463100050242L : sqrtl(-2.0L * logl(t));
    if (!(x > lo && x < hi)) x = 0.5L * (lo + hi);
    for (int it = 0; it < 400; ++it) {
        ld g = central ? (0.5L * erfl(x * SQRT1_2L) - target)      /* increasing in x */
                       : (target - 0.5L * erfcl(x * SQRT1_2L));    /* increasing in x */
        if (g == 0.0L) return x;
        if (g > 0.0L) hi = x; else lo = x;
        ld phi = INV_SQRT_2PI_L * expl(-0.5L * x * x);
        ld xn = x - g / phi;
        if (!(xn > lo && xn < hi)) xn = 0.5L * (lo + hi);
        if (fabsl(xn - x) <= 2.0L * LDBL_EPSILON * fabsl(x) || hi - lo <= 2.0L * LDBL_EPSILON * hi)
            return xn;
        x = xn;
    }
    return x;
}

ld orc_ndtri_exact_ld(ld u)
{
    if (isnan(u) || u < 0.0L || u > 1.0L) return NAN;
    if (u == 0.0L) return -INFINITY;
    if (u == 1.0L) return INFINITY;
    ld t = (u < 0.5L) ? u : 1.0L - u;      /* exact: u carries <= 64 significant bits */
    if (t == 0.5L) return 0.0L;
    ld x = solve_upper(t, 0.5L - t);     /* 1/2 - t exact (Sterbenz) */
    return (u < 0.5L) ? -x : x;
}

/* Q(v) = Phi^-1(1 - 1/2 e^-v), v >= 0: upper tail mass t = e^-v / 2 */
ld orc_Qexact_ld(ld v)
{
    if (isnan(v) || v < 0.0L) return NAN;
    if (v == 0.0L) return 0.0L;
    if (isinf(v)) return INFINITY;
    /* t = e^-v/2 and 1/2 - t = -expm1(-v)/2, each without cancellation */
    return solve_upper(0.5L * expl(-v), -0.5L * expm1l(-v));
}

/* --------------------------------------------------------------------------
 * Bulk entry points (ctypes).  Inputs are doubles (a float input is passed as
 * the exactly-equal double), outputs long double.
 * ------------------------------------------------------------------------ */
void orc_ndtri_exact(const double *u, ld *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) out[i] = orc_ndtri_exact_ld((ld)u[i]);
}

void orc_Qexact(const ld *v, ld *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) out[i] = orc_Qexact_ld(v[i]);
}

/* the rational alone, Q(v) = v P(v)/Q(v) for v >= 0 */
int orc_rational(const ld *v, ld *out, int64_t n, int formula, int prec)
{
    rat_t r;
    if (get_rat(formula, prec, &r)) return -1;
    for (int64_t i = 0; i < n; ++i) out[i] = rational_Q(&r, v[i]);
    return 0;
}

/* coefficient table as used (for transcription pins) */
int orc_coeffs(int formula, int prec, ld *p, ld *q)
{
    rat_t r;
    if (get_rat(formula, prec, &r)) return -1;
    for (int i = 0; i < r.n; ++i) { p[i] = r.p[i]; q[i] = r.q[i]; }
    return r.n;
}

/* Breakless normal quantile, same formula as the kernels (App D
 * P:855-864).  vv = min(u, 1-u) is exact; z = -log(2 vv); r = z P(z)/Q(z);
 * sign +1 for u >= 1/2.  Endpoint/invalid semantics are the
 * boundary contract (reading R9): u = 0 -> -inf, u = 1 -> +inf, else NaN. */
static ld breakless_one(const rat_t *r, ld u)
{
    if (isnan(u) || u < 0.0L || u > 1.0L) return NAN;
    if (u == 0.0L) return -INFINITY;
    if (u == 1.0L) return INFINITY;
    ld vv = (u < 0.5L) ? u : 1.0L - u;
    ld z = 0.0L - logl(2.0L * vv);       /* 0 - log(1) = +0 at u = 1/2 */
    ld q = rational_Q(r, z);
    return (u >= 0.5L) ? q : -q;
}

int orc_normal_breakless(const double *u, ld *out, int64_t n, int formula, int prec)
{
    rat_t r;
    if (get_rat(formula, prec, &r)) return -1;
    for (int64_t i = 0; i < n; ++i) out[i] = breakless_one(&r, (ld)u[i]);
    return 0;
}

/* Antithetic form ("better, v = -log[u]"): u in (0,1] ->
 * Z = Q(-log u) >= 0; the pair is {Z, -Z}.  out[2i] = Z, out[2i+1] = -Z.
 * u = 0 -> {+inf, -inf}; u outside [0,1] or NaN -> NaN. */
int orc_normal_antithetic(const double *u, ld *out, int64_t n, int formula, int prec)
{
    rat_t r;
    if (get_rat(formula, prec, &r)) return -1;
    for (int64_t i = 0; i < n; ++i) {
        ld ui = (ld)u[i], z;
        if (isnan(ui) || ui < 0.0L || ui > 1.0L) z = NAN;
        else if (ui == 0.0L) z = INFINITY;
        else z = rational_Q(&r, 0.0L - logl(ui));   /* v = -log u >= 0, +0 at u = 1 (Z >= 0) */
        out[2 * i] = z;
        out[2 * i + 1] = -z;
    }
    return 0;
}

/* Exponential (two-sided, Laplace) base -> normal
 * ("If an exponential base is used we are essentially employing the last two
 * steps"): Z = sign(v) Q(|v|).  +-inf -> +-inf, NaN -> NaN, +-0 -> +-0. */
int orc_exp_to_normal(const double *v, ld *out, int64_t n, int formula, int prec)
{
    rat_t r;
    if (get_rat(formula, prec, &r)) return -1;
    for (int64_t i = 0; i < n; ++i) {
        ld vi = (ld)v[i], a = fabsl(vi), q;
        if (isnan(vi)) q = NAN;
        else if (isinf(vi)) q = INFINITY;
        else q = rational_Q(&r, a);
        out[i] = signbit(vi) ? -q : q;
    }
    return 0;
}

/* --------------------------------------------------------------------------
 * Taylor series of Q at v = 0, through v^10 exactly as printed.
 * ------------------------------------------------------------------------ */
static void taylor_coeffs(ld c[11])
{
    const ld pi = 3.14159265358979323846264338327950288L;
    const ld sp = sqrtl(pi), s2 = sqrtl(2.0L);
    const ld p1 = sp, p3 = pi * sp, p5 = pi * pi * sp, p7 = pi * pi * pi * sp, p9 = pi * pi * pi * pi * sp;
    c[0] = 0.0L;
    c[1] = sqrtl(pi / 2.0L);
    c[2] = -0.5L * sqrtl(pi / 2.0L);
    c[3] = (2 * p1 + p3) / (12 * s2);
    c[4] = -(p1 + 3 * p3) / (24 * s2);
    c[5] = (4 * p1 + 50 * p3 + 7 * p5) / (480 * s2);
    c[6] = -(4 * p1 + 180 * p3 + 105 * p5) / (2880 * s2);
    c[7] = (8 * p1 + 1204 * p3 + 1960 * p5 + 127 * p7) / (40320 * s2);
    c[8] = -(2 * p1 + 966 * p3 + 3675 * p5 + 889 * p7) / (80640 * s2);
    c[9] = (16 * p1 + 24200 * p3 + 194628 * p5 + 117348 * p7 + 4369 * p9) / (5806080 * s2);
    c[10] = -(16 * p1 + 74640 * p3 + 1190700 * p5 + 1493520 * p7 + 196605 * p9) / (58060800 * s2);
}

void orc_Q_taylor_coeffs(ld *out)
{
    taylor_coeffs(out);
}

ld orc_Q_taylor_ld(ld v, int terms)
{
    ld c[11];
    taylor_coeffs(c);
    if (terms > 10) terms = 10;
    ld s = 0.0L, vk = 1.0L;
    for (int k = 1; k <= terms; ++k) { vk *= v; s += c[k] * vk; }
    return s;
}

void orc_Q_taylor(const ld *v, ld *out, int64_t n, int terms)
{
    for (int64_t i = 0; i < n; ++i) out[i] = orc_Q_taylor_ld(v[i], terms);
}

/* Supplementary tail model (§5.1): Q = sqrt(2 q(a,b)),
 * a = v - 1/2 log(pi)  (reading R1: the printed "a = log(v - 1/2 log pi)" is
 * a transcription error -- the tail mass e^-v/2 fixes log pi, and only this
 * reading meets the printed 1.06e-9 bound), b = log a. */
ld orc_Q_tail_ld(ld v, int groups)
{
    const ld pi = 3.14159265358979323846264338327950288L;
    ld a = v - 0.5L * logl(pi), b = logl(a);
    ld q = a - b / 2.0L;
    if (groups >= 1) q += (b / 4.0L - 0.5L) / a;
    if (groups >= 2) q += (b * b - 6.0L * b + 14.0L) / (16.0L * a * a);
    if (groups >= 3) q += (2.0L * b * b * b - 21.0L * b * b + 102.0L * b - 214.0L) / (96.0L * a * a * a);
    if (groups >= 4) q += (3.0L * b * b * b * b - 46.0L * b * b * b + 348.0L * b * b - 1488.0L * b + 2978.0L)
                          / (384.0L * a * a * a * a);
    return sqrtl(2.0L * q);
}

void orc_Q_tail(const ld *v, ld *out, int64_t n, int groups)
{
    for (int64_t i = 0; i < n; ++i) out[i] = orc_Q_tail_ld(v[i], groups);
}

/* --------------------------------------------------------------------------
 * AS241 PPND16 (Wichura, Appl. Statist. 37 (1988) 477-484), the "Wichura's
 * AS241: two breaks, at u = 0.925 and u = 1 - e^-25" of P:435.  Coefficients
 * from the publication (not in the paper, reading R17).  Region decisions are
 * taken in double, as the kernel takes them; the arithmetic is long double
 * with double-rounded coefficients.
 * ------------------------------------------------------------------------ */
static const char *AS_A[8] = {
    "3.3871328727963666080e0", "1.3314166789178437745e+2", "1.9715909503065514427e+3",
    "1.3731693765509461125e+4", "4.5921953931549871457e+4", "6.7265770927008700853e+4",
    "3.3430575583588128105e+4", "2.5090809287301226727e+3" };
static const char *AS_B[8] = {
    "1.0", "4.2313330701600911252e+1", "6.8718700749205790830e+2",
    "5.3941960214247511077e+3", "2.1213794301586595867e+4", "3.9307895800092710610e+4",
    "2.8729085735721942674e+4", "5.2264952788528545610e+3" };
static const char *AS_C[8] = {
    "1.42343711074968357734e0", "4.63033784615654529590e0", "5.76949722146069140550e0",
    "3.64784832476320460504e0", "1.27045825245236838258e0", "2.41780725177450611770e-1",
    "2.27238449892691845833e-2", "7.74545014278341407640e-4" };
static const char *AS_D[8] = {
    "1.0", "2.05319162663775882187e0", "1.67638483018380384940e0",
    "6.89767334985100004550e-1", "1.48103976427480074590e-1", "1.51986665636164571966e-2",
    "5.47593808499534494600e-4", "1.05075007164441684324e-9" };
static const char *AS_E[8] = {
    "6.65790464350110377720e0", "5.46378491116411436990e0", "1.78482653991729133580e0",
    "2.96560571828504891230e-1", "2.65321895265761230930e-2", "1.24266094738807843860e-3",
    "2.71155556874348757815e-5", "2.01033439929228813265e-7" };
static const char *AS_F[8] = {
    "1.0", "5.99832206555887937690e-1", "1.36929880922735805310e-1",
    "1.48753612908506148525e-2", "7.86869131145613259100e-4", "1.84631831751005468180e-5",
    "1.42151175831644588870e-7", "2.04426310338993978564e-15" };

static ld poly8(const char **c, int prec, ld x)
{
    ld s = coef(c[7], prec);
    for (int i = 6; i >= 0; --i) s = coef(c[i], prec) + x * s;
    return s;
}

static ld as241_one(ld u, int prec)
{
    if (isnan(u) || u < 0.0L || u > 1.0L) return NAN;
    if (u == 0.0L) return -INFINITY;
    if (u == 1.0L) return INFINITY;
    double qd = (double)u - 0.5;                       /* decision in double */
    ld q = u - 0.5L;
    if (fabs(qd) <= 0.425) {
        ld r = 0.180625L - q * q;
        return q * poly8(AS_A, prec, r) / poly8(AS_B, prec, r);
    }
    ld t = (q < 0.0L) ? u : 1.0L - u;
    double rd = sqrt(-log((double)t));                  /* decision in double */
    ld r = sqrtl(-logl(t)), x;
    if (rd <= 5.0) { r -= 1.6L; x = poly8(AS_C, prec, r) / poly8(AS_D, prec, r); }
    else           { r -= 5.0L; x = poly8(AS_E, prec, r) / poly8(AS_F, prec, r); }
    return (q < 0.0L) ? -x : x;
}

int orc_normal_as241(const double *u, ld *out, int64_t n, int prec)
{
    for (int64_t i = 0; i < n; ++i) out[i] = as241_one((ld)u[i], prec);
    return 0;
}

/* --------------------------------------------------------------------------
 * Acklam level 1 ("breaks at u = 0.97575"; "< 1.15e-9") and the
 * refined variant: one Halley step e = 1/2 erfc(-x/sqrt2) - p,
 * u = e sqrt(2 pi) exp(x^2/2), x <- x - u/(1 + x u/2) ("level one fed once
 * through a Newton-Raphson-Halley method").  Coefficients from Acklam's
 * published algorithm (reading R17).
 * ------------------------------------------------------------------------ */
static const char *AK_A[6] = { "-3.969683028665376e+01", "2.209460984245205e+02",
    "-2.759285104469687e+02", "1.383577518672690e+02", "-3.066479806614716e+01",
    "2.506628277459239e+00" };
static const char *AK_B[5] = { "-5.447609879822406e+01", "1.615858368580409e+02",
    "-1.556989798598866e+02", "6.680131188771972e+01", "-1.328068155288572e+01" };
static const char *AK_C[6] = { "-7.784894002430293e-03", "-3.223964580411365e-01",
    "-2.400758277161838e+00", "-2.549732539343734e+00", "4.374664141464968e+00",
    "2.938163982698783e+00" };
static const char *AK_D[4] = { "7.784695709041462e-03", "3.224671290700398e-01",
    "2.445134137142996e+00", "3.754408661907416e+00" };

/* Horner from the highest coefficient c[0] down to c[n-1] (Acklam's order) */
static ld hornerA(const char **c, int n, int prec, ld x)
{
    ld s = coef(c[0], prec);
    for (int i = 1; i < n; ++i) s = s * x + coef(c[i], prec);
    return s;
}

static ld acklam_one(ld p, int prec, int refine)
{
    if (isnan(p) || p < 0.0L || p > 1.0L) return NAN;
    if (p == 0.0L) return -INFINITY;
    if (p == 1.0L) return INFINITY;
    /* Reflection (reading R19): evaluate on the lower half t = min(p, 1-p)
     * (exact), as the paper's CPU runs do ("samples on [0, 0.5]"), and
     * flip the sign.  Acklam's upper-region formula is the mirror of the lower
     * one, so level 1 is unchanged; the Halley step needs it, because
     * Phi(x) - p cancels catastrophically for p near 1. */
    const double plow = 0.02425;                         /* decision in double */
    ld t = (p < 0.5L) ? p : 1.0L - p;
    ld x;
    if ((double)t < plow) {
        ld q = sqrtl(-2.0L * logl(t));
        x = hornerA(AK_C, 6, prec, q) / (hornerA(AK_D, 4, prec, q) * q + 1.0L);
    } else {
        ld q = t - 0.5L, r = q * q;
        x = hornerA(AK_A, 6, prec, r) * q / (hornerA(AK_B, 5, prec, r) * r + 1.0L);
    }
    if (refine && (double)t >= 2.2250738585072014e-308) {   /* R20: the double-precision step overflows for subnormal t */
        ld e = 0.5L * erfcl(-x * SQRT1_2L) - t;
        ld uu = e * 2.50662827463100050242L * expl(0.5L * x * x);
        x = x - uu / (1.0L + 0.5L * x * uu);
    }
    return (p < 0.5L) ? x : 0.0L - x;                    /* +0 at p = 1/2 */
}

int orc_normal_acklam(const double *u, ld *out, int64_t n, int prec, int refine)
{
    for (int64_t i = 0; i < n; ++i) out[i] = acklam_one((ld)u[i], prec, refine);
    return 0;
}

/* --------------------------------------------------------------------------
 * Moro (1995), the Beasley-Springer central rational with Moro's tail series
 * ("Moro: breaks at u = 0.92"; "In the Moro model a log(log()) operation
 * is carried out in the tail region").  Coefficients are
 * NOT in the paper (reading R17): transcribed from Moro's publication, pinned by
 * its published accuracy (absolute error < 3e-9 for |x| <= 7) in the tests.
 *   y = u - 1/2;  |y| < 0.42:  x = y A(y^2) / B(y^2)   (A cubic, B quartic, B(0) = 1)
 *   else          r = min(u, 1-u), s = log(-log r), x = +-C(s)  (C degree 8),
 *                 negative for u < 1/2.
 * ------------------------------------------------------------------------ */
static const char *MO_A[4] = { "2.50662823884", "-18.61500062529", "41.39119773534", "-25.44106049637" };
static const char *MO_B[5] = { "1", "-8.47351093090", "23.08336743743", "-21.06224101826", "3.13082909833" };
static const char *MO_C[9] = { "0.3374754822726147", "0.9761690190917186", "0.1607979714918209",
    "0.0276438810333863", "0.0038405729373609", "0.0003951896511919", "0.0000321767881768",
    "0.0000002888167364", "0.0000003960315187" };

/* ascending powers: c[0] + c[1] x + ... */
static ld horner_up(const char **c, int n, int prec, ld x)
{
    ld s = coef(c[n - 1], prec);
    for (int i = n - 2; i >= 0; --i) s = s * x + coef(c[i], prec);
    return s;
}

static ld moro_one(ld u, int prec)
{
    if (isnan(u) || u < 0.0L || u > 1.0L) return NAN;
    if (u == 0.0L) return -INFINITY;
    if (u == 1.0L) return INFINITY;
    double yd = (double)u - 0.5;                        /* decision in double */
    ld y = u - 0.5L;
    if (fabs(yd) < 0.42) {
        ld r = y * y;
        return y * horner_up(MO_A, 4, prec, r) / horner_up(MO_B, 5, prec, r);
    }
    ld t = (y < 0.0L) ? u : 1.0L - u;                   /* exact */
    ld x = horner_up(MO_C, 9, prec, logl(-logl(t)));
    return (y < 0.0L) ? -x : x;
}

int orc_normal_moro(const double *u, ld *out, int64_t n, int prec)
{
    for (int64_t i = 0; i < n; ++i) out[i] = moro_one((ld)u[i], prec);
    return 0;
}

/* Q(v) of App C with float-rounded coefficients (for orc_mc.c) */
ld orc_Q_C55_f32coef(ld v)
{
    static rat_t r;
    static int init = 0;
    if (!init) { get_rat(ORC_C55, 32, &r); init = 1; }
    return rational_Q(&r, v);
}
