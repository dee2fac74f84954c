// amg.hpp — aggregation AMG preconditioner on the device (preconditioners.cpp:384-728).
#pragma once

#include "context.hpp"

#include <functional>
#include <vector>

namespace spb {

// AmgConfig (include/specpart/preconditioners.hpp:56-70) and its two presets
// (preconditioners.cpp:24-40).
struct AmgCfg {
    bool smoothed = true;           // AggregationMode::Smoothed (false: Plain)
    double drop_tol = 0.0;
    int max_levels = 20;
    int cheby_degree = 3;
    int power_iters_setup = 10;
    double eig_ratio = 7.0;
    int64_t coarse_size_threshold = 500;
    bool coarse_direct = true;      // CoarseSolverKind::Direct (false: Chebyshev)
    int coarse_power_iters = 100;
    uint64_t seed = 0;
    static AmgCfg regular_defaults();
    static AmgCfg irregular_defaults();
};

// Explicit CSR operator on the device (square levels, P and P^T).
struct CsrDev {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int max_row = 0;
    DBuf<int64_t> offs;
    DBuf<int32_t> cols;
    DBuf<double> vals;
    DevOp op() const;
};

struct AmgLevelDev {
    CsrDev A;                 // explicit operator (level 0: the fine matrix)
    DBuf<double> diag, inv_diag;
    CsrDev P, Pt;             // prolongation from / restriction to the next coarser level
    double lambda_max = 0.0, low = 0.0, high = 0.0;  // ChebyshevData
    int degree = 0;
    // V-cycle work blocks (column-major, ld = rows)
    int64_t ld = 0;
    DBuf<double> z, dir, t, res, post, crhs;
};

class Amg {
public:
    using SpmmFn = std::function<void(const View& X, int m, const View& Y)>;
    // A0: explicit CSR of the fine operator (moved in) with its diagonal. fine_spmm
    // computes Y = A0 X with the solver's fast operator (ELL / band / binned) on
    // blocks allocated by fine_alloc (SpMM-input blocks of the solver layout) and
    // viewed with fine_view(ptr, cols) (the layout depends on the column count).
    Amg(sp_context* ctx, CsrDev&& A0, DBuf<double>&& diag0, const AmgCfg& cfg, SpmmFn fine_spmm,
        std::function<double*(int cols, DBuf<double>& store)> fine_alloc,
        std::function<View(double* p, int cols)> fine_view, int max_cols);
    // H = M^{-1} R (one V-cycle from zero), k columns of the solver's views.
    void apply(const View& R, int k, const View& H);
    int levels() const { return static_cast<int>(lv_.size()); }
    int64_t level_n(int l) const { return lv_[l].A.nrows; }
    int64_t level_nnz(int l) const { return lv_[l].A.nnz; }
    bool stagnated() const { return stagnated_; }
    bool coarse_direct() const { return direct_; }

private:
    void build();
    double power_lambda(int l, int iters, uint64_t seed);
    void spmm(int l, const View& X, int m, const View& Y);
    void chebyshev(int l, const View& rhs, int k, const View& Z);
    void vcycle(int l, const View& rhs, int k, const View& Z);
    void coarse_solve(const View& rhs, int k, const View& Z);

    sp_context* ctx_;
    cudaStream_t s_;
    AmgCfg cfg_;
    SpmmFn fine_spmm_;
    std::function<View(double*, int)> fine_view_;
    int max_cols_;
    std::vector<AmgLevelDev> lv_;
    bool stagnated_ = false, direct_ = true;
    DBuf<double> coarse_inv_;  // nc x nc column-major inverse of the shifted coarse matrix
    int64_t nc_ = 0;
    // level-0 blocks in the solver layout (SpMM inputs)
    DBuf<double> f_z_, f_dir_, f_t_, f_res_, f_post_;
    double *fz_ = nullptr, *fdir_ = nullptr, *ft_ = nullptr, *fres_ = nullptr, *fpost_ = nullptr;
    View fv(double* p, int k) const { return fine_view_(p, k); }
    DBuf<double> red_;  // reduction scratch
};

// Greedy aggregation of a strength graph (preconditioners.cpp:411-447): roots in
// ascending id, then leftovers join an adjacent aggregate, then singletons.
std::vector<int32_t> greedy_aggregate(int64_t n, const std::vector<int64_t>& offs, const std::vector<int32_t>& cols,
                                      int64_t& num_aggregates);

} // namespace spb
