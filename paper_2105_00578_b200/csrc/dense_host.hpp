// dense_host.hpp — small dense linear algebra kept on the host (m <= 3*d, 25x25).
//
// These run on matrices of at most a few hundred entries per LOBPCG iteration
// (the projected Rayleigh-Ritz matrix, the Arnoldi Hessenberg). They follow the
// reference's algorithms operation for operation, because the solver trajectory
// (eigenvector rotations inside degenerate eigenspaces, Leja root order) depends
// on them, not only on their mathematical result:
//   sym_eig          cyclic Jacobi, ascending stable sort   (src/dense.cpp:29-84)
//   cholesky/solves                                         (src/dense.cpp:86-122)
//   harmonic_ritz    (Hk^T Hk + b^2 e e^T, Hk) pencil       (src/preconditioners.cpp:232-273)
//   leja_order       modified Leja ordering                 (src/preconditioners.cpp:278-307)
#pragma once

#include <cstdint>
#include <vector>

namespace spb {

// Column-major small matrix.
struct Mat {
    int rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
    double& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
    double operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
};

void sym_eig(const Mat& A, std::vector<double>& values, Mat& vectors);
bool cholesky_lower(Mat& A);
void solve_lower(const Mat& L, double* b);
void solve_lower_transposed(const Mat& L, double* b);
std::vector<double> harmonic_ritz_values(const Mat& Hk, double beta);
std::vector<double> leja_order(std::vector<double> roots);

} // namespace spb
