// qm_rode_params.h -- layout of the exponential-base recycling tables (row f1),
// shared by the host builder (qm_rode_host.cpp) and the kernels (qm_rode.cuh).
//
// table[0]  kind (1 hyperbolic, 2 VG)        table[1]  N (intervals per side)
// table[2+s] h_s (node spacing in |v|)       table[4+s] 1/h_s
// table[6+s] V_s = QM_RODE_VRATE / rate_s    table[8+s] p_s (base mass: s=0 right p+, s=1 left p-)
// table[10+s] rate_s (a-b right, a+b left)   table[12+s] Q(0) residual   table[14+s] slope residual
// table[16+s], table[18+s]: log p_s as hi + lo            table[20+s] 1/rate_s
// nodes of side s at table[QM_RODE_HEADER + s*2*(N+1)]: (R_k, R'_k), k = 0..N,
// R(w) = Q(+-w) at w = k h_s, R' = dR/dw (negative values on the left side).
#pragma once

#define QM_RODE_HYPERBOLIC 1
#define QM_RODE_VG 2
#define QM_RODE_NODES 8192
#define QM_RODE_SUBSTEPS 16
#define QM_RODE_VRATE 40.0
#define QM_RODE_HEADER 24
#define QM_RODE_VG_MAXM 8
#define QM_RODE_TABLE_DOUBLES (QM_RODE_HEADER + 4 * (QM_RODE_NODES + 1))

namespace qm {
// builds the table in host memory (QM_RODE_TABLE_DOUBLES doubles); false on bad parameters
bool rode_table_build(int kind, const double *params, double *table);
}  // namespace qm
