/*
 * qm.h -- C ABI of the B200-native bulk inverse-CDF sampling library (libqm.so).
 *
 * Paper: W. T. Shaw & N. Brickman, "Quantile Mechanics II: Changes of Variables
 * in Monte Carlo methods and a GPU-Optimized Normal Quantile" (arXiv 0901.0638).
 * Citations "P:n" are PAPER.md line numbers.
 *
 * The problem (§1): given base samples Z with CDF G, produce target
 * samples A(Z) = F^-1(G(Z)) -- for a uniform base the quantile w(U), F(w(u)) = u.
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - Device pointers are caller-owned (allocated by the caller, e.g. torch
 *    tensors passed by data_ptr()); the library never allocates or frees them
 *    and never allocates on the hot path (the _host entry point owns private
 *    staging buffers, see there).
 *  - Layout: contiguous 1-D arrays, unit stride, of float (QM_F32) or double
 *    (QM_F64).  16-byte alignment is NOT required; misaligned or ragged arrays
 *    are handled inside the kernels (128-bit vector body, scalar remainder).
 *  - n is an int64 element count; n == 0 is a no-op returning QM_OK.
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls enqueue asynchronously and return without synchronising, except
 *    qm_*_host which returns after the results are in host memory.
 *  - In-place (output == input) is allowed; partial overlap is undefined.
 *  - Errors are reported synchronously, before any launch: QM_EINVAL for a bad
 *    argument (n < 0, NULL with n > 0, bad enum, nu <= 0, K out of range),
 *    QM_EUNSUPPORTED for a valid but unsupported combination, QM_ECUDA when the
 *    launch fails (cudaGetLastError).  There is no per-element status: element
 *    semantics are IEEE-style (see each function).
 *  - Determinism: results are bitwise reproducible for the same arguments,
 *    independent of launch configuration and device count.
 */
#ifndef QM_H
#define QM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QM_ABI_VERSION 1

typedef enum { QM_OK = 0, QM_EINVAL = 1, QM_EUNSUPPORTED = 2, QM_ECUDA = 3 } qm_status;
typedef enum { QM_F32 = 1, QM_F64 = 2 } qm_precision;

/* Normal-quantile algorithms.
 *  QM_BREAKLESS    the paper's branch-free rational in the exponential
 *                  coordinate: App C (5,5) in fp32 ("the algorithm we
 *                  propose for optimal GPU normal simulation"), App D
 *                  (13,13) in fp64.
 *  QM_BREAKLESS77  the (7,7) rational of App A/B.
 *  QM_AS241, QM_ACKLAM, QM_ACKLAM_REFINED  the branching comparison quantiles of
 *                  the paper's Table 3; fp64 only.
 *  QM_BREAKLESS_TAIL  QM_BREAKLESS below v = vc and the supplementary tail model
 *                  Q = sqrt(2 q(a,b)) of §5.1 above: vc = 37 (fp32,
 *                  App C) or 86.75 (fp64, App D).  Keeps the precision in
 *                  the deep tail (u < 4.3e-17 in fp32, u < 1e-38 in fp64) at no
 *                  cost elsewhere (warp-uniform switch).  Normal quantile,
 *                  antithetic and exponential-base entry points.
 *  QM_MORO         Moro's quantile (Beasley-Springer centre for |u - 1/2| < 0.42,
 *                  a log(log) series beyond; "Moro: breaks at u = 0.92", P:436,
 *                  P:551), a further branching comparison kernel (
 *                  coefficients external, R17); fp64 only, normal
 *                  quantile entry point only.
 *  QM_BREAKLESS1212  (12,12) single patch on v in [0, 37], max relative error
 *                  4.85e-16 ("a (12,12) rational approximation exists ... less than
 *                  5e-16"); fp64 only.
 *  QM_BREAKLESS88  (8,8) single patch on v in [0, 74], 5.75e-10 ("precision about
 *                  6e-10 on the range 0 <= v <= 74"); fp32 and fp64 (row f3).
 *  QM_TWO_REGION   (4,4) below v = 10, App C (5,5) above: the two-region variant of
 *                  P:664 ("shorter rational approximations in two regions"); max
 *                  error 3.62e-7 (App C's); fp32 only (row f4).  The branch is a
 *                  warp-uniform vote: a warp with every lane below the break runs
 *                  the short rational only.
 *  The f3/f4 coefficients are our own minimax fits (the paper does not print
 *  them): tests/golden/fit_12_37.txt, fit_8_74.txt, fit_4_10.txt.  These three
 *  are normal-quantile (qm_normal_quantile, qm_normal_quantile_host) only. */
typedef enum {
    QM_BREAKLESS = 0, QM_BREAKLESS77 = 1, QM_AS241 = 2, QM_ACKLAM = 3, QM_ACKLAM_REFINED = 4,
    QM_BREAKLESS_TAIL = 5, QM_MORO = 6, QM_BREAKLESS1212 = 7, QM_BREAKLESS88 = 8, QM_TWO_REGION = 9
} qm_algorithm;

int         qm_abi_version(void);
const char *qm_status_string(qm_status s);
/* number of SMs of the current device (cached per device); -1 on error */
int         qm_device_sm_count(void);

/* Normal quantile z[i] = w(u[i]), Phi(w(u)) = u.
 * Breakless algorithms: vv = min(u, 1-u), v = -log(2 vv), z = sign(u - 1/2) v P(v)/Q(v)
 * (App D).  u in (0,1) -> finite; u = 0 -> -inf; u = 1 -> +inf;
 * u = 1/2 -> +0; u < 0, u > 1 or NaN -> NaN.  Accuracy: within 4 ulp (fp32) / 2 ulp
 * (fp64) of the same formula evaluated exactly; the formula itself is within
 * 4e-7 (App C), 1.1e-15 (App D), 1.06e-9 ((7,7)) of Phi^-1 for v <= 37 (74 for
 * App D), degrading slowly beyond. */
qm_status qm_normal_quantile(const void *u, void *z, int64_t n, qm_precision p,
                             qm_algorithm alg, void *stream);

/* Config 1 like-for-like (Table 3): the same formulas in PLAIN double,
 * as the paper's codes are written -- FMA Horner, library log/sqrt/erfc/exp, IEEE
 * division, per-element branches, no compensation.  fp64 only; alg in
 * {QM_BREAKLESS (App D), QM_BREAKLESS77, QM_AS241, QM_ACKLAM, QM_ACKLAM_REFINED,
 * QM_MORO}, else QM_EUNSUPPORTED.  Same element semantics as qm_normal_quantile;
 * accuracy that of plain double evaluation (not the 2-ulp contract): a timing
 * comparison, not a product path. */
qm_status qm_normal_quantile_plain(const void *u, void *z, int64_t n, qm_algorithm alg, void *stream);

/* Antithetic pairs ("always work antithetically"): for each
 * u[i] in (0,1]: v = -log u[i] ("better, v = -log[u]"), Z = Q(v) >= 0,
 * z_pairs[2i] = Z, z_pairs[2i+1] = -Z.  2n outputs.  u = 0 -> {+inf, -inf};
 * u outside [0,1] or NaN -> NaN.  Breakless algorithms only. */
qm_status qm_normal_antithetic(const void *u, void *z_pairs, int64_t n, qm_precision p,
                               qm_algorithm alg, void *stream);

/* Counter-based Philox4x32-10 uniforms (row a1; not in the paper, whose rnd()
 * is a placeholder).  key = (lo32(seed), hi32(seed)); block counter c ->
 * ctr = (lo32(c), hi32(c), 0, 0).  fp32: u[i] = (2 (w >> 9) + 1) 2^-24 from word
 * i%4 of block counter_offset + i/4.  fp64: u[i] = (2x + 1) 2^-53 with
 * x = ((w_{2j} << 32) | w_{2j+1}) >> 12, j = i%2, block counter_offset + i/2.
 * Values lie on an odd grid: never 0 or 1, 1-u on the grid. */
qm_status qm_philox_uniform(void *u, int64_t n, qm_precision p, uint64_t seed,
                            uint64_t counter_offset, void *stream);

/* Fused: z[i] = normal quantile of the i-th Philox uniform above, generated in
 * registers (no HBM read).  Bitwise equal to qm_philox_uniform followed by
 * qm_normal_quantile with the same arguments. */
qm_status qm_normal_philox(void *z, int64_t n, qm_precision p, qm_algorithm alg,
                           uint64_t seed, uint64_t counter_offset, void *stream);

/* Recycle standard normal samples into Student-t samples, t = F_nu^-1(Phi(z))
 * (§3): central series t = z sum_{k=0}^{K} c_k z^{2k} for |z| < zstar
 * and the two-term tail
 * t = sqrt(nu) w^(-1/nu)(1 - (nu+1)/(2(nu+2)) w^(2/nu)),
 * w = (1 - Phi(|z|)) nu sqrt(pi) Gamma(nu/2)/Gamma((nu+1)/2) for |z| >= zstar
 * (P:267-272), odd in z.
 * Validated configurations (zstar <= 0 selects the crossover from this table):
 *     nu = 4,  K = 10, zstar = 3.93473 (the paper's; max rel. error 1.36e-5)
 *     nu = 3,  K = 16, zstar = 3.5667  (4.2e-6)
 *     nu = 5,  K = 16, zstar = 4.6506  (6.7e-6)
 *     nu = 10, K = 16, zstar = 6.9584  (4.1e-6)
 * (the last three: min-max crossovers of DESIGN.md reading R13, the paper gives
 * only nu = 4).  zstar <= 0 with any other (nu, K) -> QM_EUNSUPPORTED.  A caller
 * zstar > 0 is accepted for 2 <= nu <= 20, 1 <= K <= 24: the kernel then
 * evaluates the same composite with the caller's crossover and its error is the
 * caller's choice (tools/student_crossover.py computes min-max crossovers; the
 * tests cover nu in {2, 2.5, 7, 20} x K in {10, 16, 24} that way).  nu outside
 * [2, 20] -> QM_EUNSUPPORTED (beyond 20 the coefficient recurrence is
 * ill-conditioned; below 2 the tail's w^(-1/nu) amplifies the double erfcx's
 * few-ulp error past the 2-ulp contract);
 * nu <= 0, K outside [1, 24] or a NaN zstar -> QM_EINVAL.
 * +-inf -> +-inf, NaN -> NaN; tail values beyond the double range -> +-inf. */
qm_status qm_recycle_normal_to_t(const void *z, void *t, int64_t n, qm_precision p,
                                 double nu, int K, double zstar, void *stream);
/* the crossover qm_recycle_normal_to_t uses for zstar <= 0, or 0 if (nu, K) is
 * not a validated configuration (host-only, no CUDA call) */
double qm_student_default_crossover(double nu, int K);

/* Config 4 with fused moments: t as qm_recycle_normal_to_t (the
 * same bits) and, in the same pass, the moment rows of qm_moment_rows below:
 * rows[4 c + k - 1] = sum of t^k over the fixed chunk c of QM_MOMENT_CHUNK
 * samples (k = 1..4), qm_moment_row_count(n) rows.  The rows are deterministic
 * and independent of the device count (chunks align with the shards of the
 * multi-GPU harness); their summation order inside a chunk differs from
 * qm_moment_rows (equal to rounding).  fp64, K = 10 or 16 and 16-byte aligned
 * arrays run one fused kernel; other cases run the map and qm_moment_rows. */
qm_status qm_recycle_normal_to_t_moments(const void *z, void *t, int64_t n, qm_precision p, double nu, int K,
                                         double zstar, double *rows, void *stream);

/* Recycle two-sided (Laplace) exponential samples into normal samples
 * (P:397-405): z = sign(v) Q(|v|) with the breakless rational
 * and no logarithm.  +-0 -> +-0, +-inf -> +-inf, NaN -> NaN. */
qm_status qm_recycle_exp_to_normal(const void *v, void *z, int64_t n, qm_precision p,
                                   qm_algorithm alg, void *stream);

/* Moment sums S_k = sum_i x_i^k, k = 1..4 (row a8; the north star's "moment
 * ... sums" that the multi-GPU harness all-reduces).  Deterministic for any
 * launch, device and DEVICE COUNT:
 *  - qm_moment_rows: the array is cut into fixed chunks of QM_MOMENT_CHUNK
 *    elements; rows[4r + k-1] = sum over chunk r of x^k, in a fixed order.
 *    rows has qm_moment_row_count(n) * 4 doubles (caller-owned, device).
 *  - qm_reduce_rows: out[c] = sum over r of rows[r * ncol + c] in a fixed tree
 *    (1 <= ncol <= 64).  A rank owning chunks [c0, c1) of a global stream
 *    writes rows [c0, c1) of a zeroed global matrix; an all-reduce(SUM) of the
 *    matrix is exact and qm_reduce_rows gives the same bits for 1 or 8 GPUs.
 *  - qm_moments = both, S_k in sums_dev[k-1] (kmax <= 4 written), rows_ws as
 *    for qm_moment_rows. */
#define QM_MOMENT_CHUNK 65536
int64_t   qm_moment_row_count(int64_t n);
qm_status qm_moment_rows(const void *x, int64_t n, qm_precision p, double *rows, void *stream);
qm_status qm_reduce_rows(const double *rows, int64_t nrows, int ncol, double *out, void *stream);
qm_status qm_moments(const void *x, int64_t n, qm_precision p, int kmax,
                     double *sums_dev, double *rows_ws, void *stream);

/* Monte-Carlo European-call sweep (BASELINE.json config 5) with normal
 * innovations from the EXPONENTIAL base: sample i of
 * the Philox stream (fp32 grid, qm_philox_uniform layout) gives v = -log u,
 * a sign from bit 8 of the Philox word, Z = sign * Q(v) (App C rational), and
 * S_T = S0 exp((r - sigma^2/2) T + sigma sqrt(T) Z).  For each of the
 * nstrikes <= 32 strikes K_j, row r (fixed chunk r of QM_MC_CHUNK samples)
 * receives rows[r*2*nstrikes + 2j] = sum (S_T - K_j)^+ and [.. + 2j+1] = sum of
 * its square.  rows: qm_mc_row_count(n) * 2 * nstrikes doubles (device).
 * Rows are all-reduced across GPUs exactly and added by qm_reduce_rows; the
 * price is exp(-rT) * sum / n.  Accumulation: fp32 over 64 samples per
 * thread, then fp64. */
#define QM_MC_CHUNK (1 << 20)
#define QM_MC_MAX_STRIKES 32
typedef struct {
    double S0, r, sigma, T;
    int nstrikes;
    double strikes[QM_MC_MAX_STRIKES];
} qm_mc_params;
int64_t   qm_mc_row_count(int64_t n);
qm_status qm_mc_european_call(int64_t n, uint64_t seed, uint64_t counter_offset, const qm_mc_params *params,
                              double *rows, void *stream);

/* Exponential-base recycling into hyperbolic and variance-gamma samples (row f1;
 * §4).  The base is the two-sided exponential of P:315-321 with the
 * target's masses p+-  and rates a-b (right), a+b (left);
 * the map Q(v) = F^-1(F0(v)) solves the Recycling ODE of P:330-345.
 *  - qm_exp_target_table builds the map for one parameter set into a
 *    caller-owned DEVICE buffer of QM_RODE_TABLE_DOUBLES doubles: host setup
 *    (masses by quadrature; the RODE integrated in long double backward from
 *    an anchor at base probability e^-800, where Q is fixed by its definition,
 *    down to v = 0 -- forward integration is exponentially ill-conditioned --
 *    and the first unit of rate*|v| redone forward from the exact centre
 *    conditions), then a synchronous copy (~1 MB; tens of ms of host work
 *    per parameter set; ~4 s for a non-integer VG lambda).  params: hyperbolic
 *    {alpha, beta, delta} (alpha > |beta|, delta > 0); VG {lambda, alpha, beta},
 *    alpha > |beta|, with lambda = 1 (the identity), integer 2..9
 *    (half-integer Bessel orders in closed form) or real 1.1 <= lambda <= 30
 *    (K of real order by Temme's series / Steed's continued fraction; the
 *    origin, where the density is not analytic for non-integer lambda, is
 *    approached on geometric meshes and the centre nodes are graded towards it,
 *    w_k = Wc (k/3584)^4 -- the "many steps near v = 0" of P:395).
 *    Bad parameters -> QM_EINVAL; lambda < 1 (out of scope),
 *    1 < lambda < 1.1 or lambda > 30 -> QM_EUNSUPPORTED.
 *  - qm_recycle_exp_to_hyperbolic / qm_recycle_exp_to_vg: x[i] = Q(v[i]) for
 *    base samples v (quintic Hermite on (Q, Q', Q'') at 24065 nodes per side:
 *    3585 on the centre rate*|v| <= 10 -- 7 octave levels [0, Wc/64], [Wc/64,
 *    Wc/32], ..., [Wc/2, Wc] of 512 uniform intervals (for a real lambda
 *    rate*|v| <= 2, graded as above) --, 16384 out to base probability e^-40,
 *    4096 out to e^-800; linear beyond).  +-0, +-inf,
 *    NaN pass through.
 *  - qm_exp_base_quantile: v[i] = Q0(u[i]) of P:322-329.
 *  - qm_exp_target_philox: fused Philox (qm_philox_uniform layout) -> Q0 -> Q.
 * Accuracy (the method's, against the exact map): < 2e-12 relative in fp64
 * (worst near v = 0), correctly rounded to within 2 ulp in fp32. */
#define QM_RODE_TABLE_DOUBLES (80 + 8 * (3584 + 16384 + 4096 + 1))
typedef enum { QM_TARGET_HYPERBOLIC = 1, QM_TARGET_VG = 2, QM_TARGET_STUDENT = 3 } qm_target;
qm_status qm_exp_target_table(qm_target kind, const double *params, double *table_dev);
qm_status qm_recycle_exp_to_hyperbolic(const void *v, void *x, int64_t n, qm_precision p,
                                       const double *table_dev, void *stream);
qm_status qm_recycle_exp_to_vg(const void *v, void *x, int64_t n, qm_precision p,
                               const double *table_dev, void *stream);
qm_status qm_exp_base_quantile(const void *u, void *v, int64_t n, qm_precision p,
                               const double *table_dev, void *stream);
qm_status qm_exp_target_philox(void *x, int64_t n, qm_precision p, const double *table_dev,
                               uint64_t seed, uint64_t counter_offset, void *stream);
/* Gaussian-base recycling by the "purely numerical method" of §3.6:
 * the Student Recycling ODE solved numerically and sampled by
 * interpolation -- the alternative to the series of qm_recycle_normal_to_t,
 * with no crossover and no restriction to a validated (nu, K).
 *  - qm_normal_target_table(QM_TARGET_STUDENT, {nu}, table_dev) builds the map
 *    t = F_nu^-1(Phi(z)) into a caller-owned DEVICE buffer of
 *    QM_RODE_TABLE_DOUBLES doubles (the layout of the exponential-base tables):
 *    host setup (~0.3 s) integrating the RODE in long double BACKWARD from an
 *    anchor at |z| = 38.5 (beyond the largest |z| a double uniform can give),
 *    where t is fixed by its definition -- forward from the centre conditions
 *    Q(0) = 0, Q'(0) = gamma the error grows like e^{z^2/2} --, in
 *    log t beyond |z| = 2; the nodes with |z| <= 2 are redone forward from the
 *    exact centre conditions.  1 <= nu <= 200; nu <= 0 or a wrong kind ->
 *    QM_EINVAL, 0 < nu < 1 or nu > 200 -> QM_EUNSUPPORTED.  Synchronous.
 *  - qm_recycle_normal_to_t_rode: t[i] = A(z[i]) for normal samples z (fp32 or
 *    fp64, any alignment, caller's stream): quintic Hermite on (Q, Q', Q'') at
 *    3585 nodes on |z| <= 4.5 (7 octave levels of 512 intervals, all in shared
 *    memory), 16384 on
 *    4.5..9, and on (log|Q|, (log|Q|)', (log|Q|)'') at 4096 on 9..38.5
 *    (exponentiated; log-linear beyond).  +-0, +-inf, NaN pass through; values
 *    beyond the double range -> +-inf.
 * Accuracy against the exact map: 4e-15 + 16 eps (1 + kappa(z)) relative, kappa =
 * |z t'(z)/t(z)| the map's condition number (<= 40 on |z| <= 6, so < 8e-14 there;
 * the paper's claim is 5e-8) -- the node coordinate and, in the tail, log|t|
 * carry roundings of an ulp or two that kappa amplifies. */
qm_status qm_normal_target_table(qm_target kind, const double *params, double *table_dev);
qm_status qm_recycle_normal_to_t_rode(const void *z, void *t, int64_t n, qm_precision p,
                                      const double *table_dev, void *stream);
/* the same table in HOST memory (diagnostics: header + nodes, see qm_rode_params.h) */
int qm_rode_table_host(int kind, const double *params, double *table);

/* End-to-end variant of qm_normal_quantile on HOST buffers: copies u in,
 * computes, copies z out in chunks on library-owned streams and device staging
 * buffers (allocated once per thread and reused).  Returns after z_host is
 * complete.  Host buffers may be pageable or pinned, but the copies overlap the
 * kernels only when they are PINNED (cudaHostAlloc / torch pin_memory): with
 * pageable memory each cudaMemcpyAsync is synchronous and the chunks run one
 * after another. */
qm_status qm_normal_quantile_host(const void *u_host, void *z_host, int64_t n,
                                  qm_precision p, qm_algorithm alg);

/* Diagnostics: the central-series coefficients c_0..c_K exactly as the
 * Student kernel receives them (host __float128 recurrence).
 * c_out has K+1 doubles.  Returns 0 on success. */
int qm_student_coefficients(double nu, int K, double *c_out);

#ifdef __cplusplus
}
#endif
#endif /* QM_H */
