// qm_rode_params.h -- layout of the exponential-base recycling tables (row f1),
// shared by the host builder (qm_rode_host.cpp) and the kernels (qm_rode.cuh).
//
// Per side s (0 = right, v > 0; 1 = left, v < 0) the map R(w) = Q(+-w), w = |v|,
// is tabulated on three segments j (node index ranges share their ends):
//   j = 0 centre  nodes 0..Nc            0 <= w <= Wc = QM_RODE_VRATE_CQ / rate_s (99.995 % of the
//                                        base samples) on 7 octave levels [0, Wc/64], [Wc/64, Wc/32],
//                                        ..., [Wc/2, Wc] of 512 uniform intervals each; for a
//                                        real-lambda VG table Wc = QM_RODE_VRATE_C / rate_s and node k
//                                        at Wc (k/Nc)^4 (R29); nodes with rate w <= 2 integrated
//                                        forward from the exact centre conditions
//   j = 1 fine    nodes Nc..Nc+N         Wc <= w <= V  = QM_RODE_VRATE  / rate_s   (base prob. e^-40)
//   j = 2 coarse  nodes Nc+N..NT         V <= w <= Vmax = QM_RODE_VRATE2 / rate_s  (e^-800, below the
//                                        smallest double: every finite Q0(u) is interpolated)
//
// table[0]  kind (1 hyperbolic, 2 VG, 3 Student)   table[1]  NT (nodes per side - 1)   table[2] nu (Student)
// table[3..5] alpha, beta, delta^2 (hyperbolic: the kernel's R'' from the RODE)
// table[8+s] p_s (base mass: s=0 right p+, s=1 left p-)    table[10+s] rate_s (a-b right, a+b left)
// table[12+s] Q(0) residual of the backward sweep           table[14+s] its slope residual
// table[16+s], table[18+s]: log p_s as hi + lo              table[20+s] 1/rate_s
// table[22+s] forward/backward mismatch of Q at the first backward node   table[28+s] Vmax_s
// table[30] 3     table[31] 1 if segment j = 2 holds log |R| (Student), else 0
// segment record (s, j) at table[32 + 8 (3 s + j)]: w0, h, 1/h, k0, n (intervals), w1, G, g
//   g = 0 uniform segment; g = 1 octave levels (j = 0; the 1/h slot holds 1/Wc): the
//   kernel reads the level from the exponent of x = w/Wc and the local coordinate
//   512 (m - 1) from its mantissa m (level 0: 2^15 x); g = 4 graded centre (j = 0):
//   w_k = Wc (k/n)^4, G = Wc/n^4, 1/h slot = 1/Wc; the kernel takes s = n (w/Wc)^(1/4)
//   and chain-rule derivatives
// nodes of side s at table[QM_RODE_HEADER + s*4*(QM_RODE_NT+1)]: (R_k, R'_k, R''_k, 0),
// k = 0..NT, R' = dR/dw (negative on the left side), R'' from the RODE itself
// (R'' = H(R) R'^2 - rate R'); quintic Hermite interpolation.
#pragma once

#define QM_RODE_HYPERBOLIC 1
#define QM_RODE_VG 2
#define QM_RODE_OCT_LEVELS 7        // centre octave levels (the innermost reaches down to 0)
#define QM_RODE_OCT_NODES 512       // uniform intervals per level
#define QM_RODE_CENTRE_NODES 3584   // = LEVELS * NODES; all fit in shared memory beside the TMA ring
#define QM_RODE_NODES 16384
#define QM_RODE_TAIL_NODES 4096
#define QM_RODE_NT (QM_RODE_CENTRE_NODES + QM_RODE_NODES + QM_RODE_TAIL_NODES)
#define QM_RODE_SUBSTEPS 16
#define QM_RODE_VRATE_C 2.0     // centre of a real-lambda VG table
#define QM_RODE_VRATE_CQ 10.0   // centre of the other exponential-base tables
#define QM_RODE_VRATE_FWD 2.0   // centre nodes with rate |v| <= 2 come from the forward sweep
#define QM_RODE_VRATE 40.0
#define QM_RODE_VRATE2 800.0
#define QM_RODE_HEADER 80
#define QM_RODE_SEG 32
#define QM_RODE_VG_MAXM 8                 // integer lambda <= QM_RODE_VG_MAXM + 1: closed-form K_{m+1/2}
#define QM_RODE_VG_LAMBDA_MIN_REAL 1.1    // non-integer lambda: K_nu of real order, lambda in [1.1, 30]
#define QM_RODE_VG_LAMBDA_MAX 30.0
// Gaussian base, Student t (§3.6): kind 3, params {nu}; segments
// centre [0, 4.5] (octave levels), fine [4.5, 9] (R values), coarse [9, 38.5] in log |R| (table[31] = 1;
// its nodes start at Nc + N + 1, M - 1 intervals), table[2] = nu
#define QM_RODE_STUDENT 3
#define QM_RODE_STUDENT_NU_MIN 1.0
#define QM_RODE_STUDENT_NU_MAX 200.0   // beyond, the anchor series cancels (2.7e-12 at nu = 500)
#define QM_RODE_STUDENT_WC 4.5L     // centre [0, 4.5] on octave levels (1 - 7e-6 of the samples)
#define QM_RODE_STUDENT_WF 2.0L     // centre nodes with |z| <= 2 from the forward sweep
#define QM_RODE_STUDENT_V 9.0L      // fine [4.5, 9] in t, coarse [9, 38.5] in log |t|
#define QM_RODE_STUDENT_VMAX 38.5L
#define QM_RODE_TABLE_LEN (QM_RODE_HEADER + 8 * (QM_RODE_NT + 1))

namespace qm {
// builds the table in host memory (QM_RODE_TABLE_LEN doubles = QM_RODE_TABLE_DOUBLES of qm.h);
// false on bad parameters
bool rode_table_build(int kind, const double *params, double *table);
// the Student table (kind QM_RODE_STUDENT) for 1 <= nu <= 200; false otherwise
bool rode_student_table_build(double nu, double *table);
}  // namespace qm
