// qm_student_params.h -- plain-data parameters of the normal -> Student-t kernel,
// shared by the device code (qm_student.cuh) and the host setup
// (qm_student_host.cpp).
#pragma once
#define QM_STUDENT_KMAX 24

namespace qm {

struct StudentParams {
    double c[QM_STUDENT_KMAX + 1];   // c_0..c_K of the central series
    int K;
    int kc;                          // number of compensated (error-free) final Horner steps
    double zstar;                    // crossover
    // double-double constants: in the far tail log w ~ -700, so 1/nu must carry
    // more than 53 bits for w^(-1/nu) to stay within an ulp
    double sqrt_nu, sqrt_nu_lo, inv_nu, inv_nu_lo, two_over_nu, two_over_nu_lo;
    double acoef;                    // (nu+1)/(2(nu+2))
    double logC_hi, logC_lo;         // log(C_nu / 2) as a double-double, C_nu = nu sqrt(pi) G(nu/2)/G((nu+1)/2)
};

// fills *out; false if the coefficients cannot be trusted (nu or K out of range)
bool student_params(double nu, int K, double zstar, StudentParams *out);

}  // namespace qm
