// spmm_epilogue.cuh — the SpMM epilogues shared by the CSR/ELL kernels
// (spmm.cu) and the binned vector kernel for irregular graphs (spmm_vec.cu).
#pragma once

#include "ops.cuh"

namespace spb {

// H accumulation of the product-form polynomial (preconditioners.cpp:184-185),
// in the reference's order: h_terms == 2 adds inv_cur*p_i then inv_next*p_{i+1};
// h_terms == 1 adds inv_next*p_{i+1} only; `first` starts from H = 0.
__device__ __forceinline__ double poly_h(const EpiArgs& ea, double hold, double xi, double pn) {
    double h = hold;
    if (ea.h_terms == 2) h = ea.first ? __dmul_rn(ea.inv_cur, xi) : __dadd_rn(h, __dmul_rn(ea.inv_cur, xi));
    return __dadd_rn(h, __dmul_rn(ea.inv_next, pn));
}

template <int EPI>
__device__ __forceinline__ void epilogue(const EpiArgs& ea, int64_t row, int c, double acc,
                                         double xi, double& sq) {
    if (EPI == EPI_STORE) {
        ea.Y.at(row, c) = acc;
    } else if (EPI == EPI_RESIDUAL) {
        // R = AX - BX * diag(theta)   (eigensolver.cpp:212-218): bx = d_i*x_i, r = ax - t*bx
        const double bx = ea.bdiag ? __dmul_rn(ea.bdiag[row], xi) : xi;
        const double r = __dsub_rn(acc, __dmul_rn(ea.theta[c], bx));
        ea.Y.at(row, c) = r;
        sq = fma(r, r, sq);
    } else {
        // prod_{i+1} = prod_i - inv_i * (A prod_i); H += inv_{i+1} * prod_{i+1}
        // (preconditioners.cpp:183-190, unrolled one step ahead)
        const double pn = __dsub_rn(xi, __dmul_rn(ea.inv_cur, acc));
        ea.Y.at(row, c) = pn;
        if (ea.h_terms) ea.H.at(row, c) = poly_h(ea, ea.first ? 0.0 : ea.H.at(row, c), xi, pn);
    }
}


} // namespace spb
