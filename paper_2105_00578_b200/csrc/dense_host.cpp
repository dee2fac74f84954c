// dense_host.cpp — see dense_host.hpp. Compiled with -ffp-contract=off so the
// arithmetic sequence (and hence every bit of the result) is the reference's.
#include "dense_host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>

namespace spb {

namespace {

double frobenius_offdiag(const Mat& M) {
    double acc = 0.0;
    for (int j = 0; j < M.cols; ++j)
        for (int i = 0; i < M.rows; ++i)
            if (i != j) acc += M(i, j) * M(i, j);
    return std::sqrt(acc);
}

// Apply the plane rotation (c, s) to columns p, q of M (M <- M G) or, with
// rows=true, to rows p, q (M <- G^T M).
void rotate(Mat& M, int p, int q, double c, double s, bool rows) {
    const int m = rows ? M.cols : M.rows;
    for (int k = 0; k < m; ++k) {
        double& xp = rows ? M(p, k) : M(k, p);
        double& xq = rows ? M(q, k) : M(k, q);
        const double vp = xp, vq = xq;
        xp = c * vp - s * vq;
        xq = s * vp + c * vq;
    }
}

} // namespace

// Cyclic-by-row Jacobi: sweeps over (p<q), rotation angle from
// tau = (a_qq - a_pp) / (2 a_pq), the smaller root t, c = 1/sqrt(1+t^2).
// Stops when the off-diagonal Frobenius norm <= 1e-15 * max|a| * m, at most 64
// sweeps; rotations with |a_pq| below stop/(m^2+1) are skipped.
void sym_eig(const Mat& A, std::vector<double>& values, Mat& vectors) {
    const int m = A.rows;
    if (A.cols != m) throw std::logic_error("sym_eig: matrix not square");
    Mat M = A;
    Mat V(m, m);
    for (int i = 0; i < m; ++i) V(i, i) = 1.0;

    double amax = 0.0;
    for (double x : M.a) amax = std::max(amax, std::abs(x));
    const double stop = amax == 0.0 ? 0.0 : 1e-15 * amax * static_cast<double>(m);
    const double skip = stop / (static_cast<double>(m) * m + 1.0);

    for (int sweep = 0; sweep < 64 && frobenius_offdiag(M) > stop; ++sweep) {
        for (int p = 0; p + 1 < m; ++p) {
            for (int q = p + 1; q < m; ++q) {
                const double apq = M(p, q);
                if (std::abs(apq) <= skip) continue;
                const double tau = (M(q, q) - M(p, p)) / (2.0 * apq);
                const double root = std::sqrt(1.0 + tau * tau);
                const double t = tau >= 0.0 ? 1.0 / (tau + root) : 1.0 / (tau - root);
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = t * c;
                rotate(M, p, q, c, s, false);
                rotate(M, p, q, c, s, true);
                rotate(V, p, q, c, s, false);
            }
        }
    }

    std::vector<int> idx(m);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return M(x, x) < M(y, y); });
    values.assign(m, 0.0);
    vectors = Mat(m, m);
    for (int j = 0; j < m; ++j) {
        values[j] = M(idx[j], idx[j]);
        for (int i = 0; i < m; ++i) vectors(i, j) = V(i, idx[j]);
    }
}

bool cholesky_lower(Mat& A) {
    const int n = A.rows;
    for (int j = 0; j < n; ++j) {
        double d = A(j, j);
        for (int k = 0; k < j; ++k) d -= A(j, k) * A(j, k);
        if (!(d > 0.0)) return false;
        const double l = std::sqrt(d);
        A(j, j) = l;
        for (int i = j + 1; i < n; ++i) {
            double s = A(i, j);
            for (int k = 0; k < j; ++k) s -= A(i, k) * A(j, k);
            A(i, j) = s / l;
        }
        for (int i = 0; i < j; ++i) A(i, j) = 0.0;
    }
    return true;
}

void solve_lower(const Mat& L, double* b) {
    for (int i = 0; i < L.rows; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L(i, k) * b[k];
        b[i] = s / L(i, i);
    }
}

void solve_lower_transposed(const Mat& L, double* b) {
    for (int i = L.rows - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < L.rows; ++k) s -= L(k, i) * b[k];
        b[i] = s / L(i, i);
    }
}

// Harmonic Ritz values: eigenvalues of (Hk^T Hk + beta^2 e_k e_k^T) y = theta Hk_sym y,
// reduced to W = L^{-1} C L^{-T} with L L^T = (Hk + Hk^T)/2 (+ a growing shift if
// that is not positive definite).
std::vector<double> harmonic_ritz_values(const Mat& Hk, double beta) {
    const int k = Hk.rows;
    Mat C(k, k);
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
            double s = 0.0;
            for (int l = 0; l < k; ++l) s += Hk(l, i) * Hk(l, j);
            C(i, j) = s;
        }
    C(k - 1, k - 1) += beta * beta;

    Mat T(k, k);
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) T(i, j) = 0.5 * (Hk(i, j) + Hk(j, i));
    double trace = 0.0;
    for (int i = 0; i < k; ++i) trace += T(i, i);

    Mat L = T;
    double shift = 0.0;
    while (!cholesky_lower(L)) {
        shift = shift == 0.0 ? 1e-14 * std::max(trace, 1.0) : shift * 100.0;
        L = T;
        for (int i = 0; i < k; ++i) L(i, i) += shift;
        if (shift > 1.0) throw std::runtime_error("harmonic Ritz reduction failed");
    }

    Mat W = C;
    for (int j = 0; j < k; ++j) solve_lower(L, &W.a[static_cast<size_t>(j) * k]);
    std::vector<double> row(k);
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < k; ++j) row[j] = W(i, j);
        solve_lower(L, row.data());
        for (int j = 0; j < k; ++j) W(i, j) = row[j];
    }
    std::vector<double> values;
    Mat vectors;
    sym_eig(W, values, vectors);
    return values;
}

// Largest magnitude first, then greedily the root maximising the sum of
// log-distances to the roots already placed (first index wins ties).
std::vector<double> leja_order(std::vector<double> roots) {
    const size_t k = roots.size();
    std::vector<double> out;
    if (k == 0) return out;
    out.reserve(k);
    std::vector<char> used(k, 0);
    size_t first = 0;
    for (size_t i = 1; i < k; ++i)
        if (std::abs(roots[i]) > std::abs(roots[first])) first = i;
    out.push_back(roots[first]);
    used[first] = 1;
    while (out.size() < k) {
        size_t best = k;
        double best_score = -std::numeric_limits<double>::infinity();
        for (size_t i = 0; i < k; ++i) {
            if (used[i]) continue;
            double score = 0.0;
            for (double r : out) score += std::log(std::max(std::abs(roots[i] - r), 1e-300));
            if (score > best_score) {
                best_score = score;
                best = i;
            }
        }
        out.push_back(roots[best]);
        used[best] = 1;
    }
    return out;
}

} // namespace spb
