// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// C wrapper over the UNMODIFIED reference library (/root/reference/proj/src/*.cpp),
// compiled by oracle/Makefile into oracle/_ref/libspecpart_ref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs load it,
// and only as the checker or the timed CPU baseline — never on the product path.
//
// Every ref_* function has the signature of the sp_* entry point of the same name
// in include/specpart_b200.h (minus the context), so tests can call both sides
// with identical arguments.
#include "specpart_b200.h"

#include "specpart/eigensolver.hpp"
#include "specpart/errors.hpp"
#include "specpart/generators.hpp"
#include "specpart/graph.hpp"
#include "specpart/kernels.hpp"
#include "specpart/laplacian.hpp"
#include "specpart/partitioner.hpp"
#include "specpart/pipeline.hpp"
#include "specpart/preconditioners.hpp"

#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <vector>

using namespace specpart;

namespace {

thread_local std::string g_err;

Graph to_graph(const sp_graph* g) {
    Graph out;
    const int64_t n = g->n;
    const int64_t nnz = g->row_offsets[n];
    out.adjacency.nrows = out.adjacency.ncols = n;
    out.adjacency.row_offsets.assign(g->row_offsets, g->row_offsets + n + 1);
    out.adjacency.col_indices.assign(g->col_indices, g->col_indices + nnz);
    if (g->values)
        out.adjacency.values.assign(g->values, g->values + nnz);
    else
        out.adjacency.values.assign(nnz, 1.0);
    if (g->vertex_weights)
        out.vertex_weights.assign(g->vertex_weights, g->vertex_weights + n);
    else
        out.vertex_weights.assign(n, 1.0);
    return out;
}

Dense to_dense(const double* colmajor, int64_t rows, int64_t cols) {
    Dense d(rows, cols);
    std::memcpy(d.data.data(), colmajor, sizeof(double) * rows * cols);
    return d;
}

template <class F> sp_status guarded(F&& f) {
    try {
        f();
        return SP_OK;
    } catch (const BreakdownError& e) {
        g_err = e.what();
        return SP_BREAKDOWN;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return SP_INFEASIBLE;
    } catch (const DegenerateDegreeError& e) {
        g_err = e.what();
        return SP_DEGENERATE;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return SP_DIMENSION;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SP_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SP_ERROR;
    }
}

LinearOperator build_kind(int32_t kind, const Graph& g) {
    switch (kind) {
    case SP_LAP_COMBINATORIAL: return build_combinatorial(g);
    case SP_LAP_NORMALIZED: return build_normalized(g);
    case SP_LAP_DEGREE: return build_degree(g);
    }
    throw std::invalid_argument("unknown operator kind");
}

ProblemKind problem_of(int32_t p) {
    switch (p) {
    case SP_PROBLEM_COMBINATORIAL: return ProblemKind::Combinatorial;
    case SP_PROBLEM_GENERALIZED: return ProblemKind::Generalized;
    case SP_PROBLEM_NORMALIZED: return ProblemKind::Normalized;
    }
    throw std::invalid_argument("problem must be explicit");
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

sp_status ref_partition(const sp_graph* g, const sp_config* c, int32_t* assignment_out,
                        sp_report* rep, const double* x0_colmajor) {
    return guarded([&] {
        Graph G = to_graph(g);
        RunConfig cfg;
        cfg.num_parts = c->num_parts;
        cfg.problem = static_cast<ProblemChoice>(c->problem);
        cfg.precond = static_cast<PrecondChoice>(c->precond);
        if (c->tol > 0.0) cfg.tol = c->tol;
        cfg.max_iters = c->max_iters;
        cfg.seed = c->seed;
        cfg.epsilon = c->epsilon;
        cfg.doubled_cut = c->doubled_cut != 0;
        cfg.init = static_cast<InitChoice>(c->init);
        cfg.record_trace = c->record_trace != 0;
        if (x0_colmajor)
            throw std::invalid_argument("ref_partition: use ref_lobpcg for explicit X0");
        RunResult r = partition_graph(G, cfg);
        std::memcpy(assignment_out, r.partition.assignment.data(), sizeof(int32_t) * G.n());
        if (!rep) return;
        const RunReport& R = r.report;
        double* pw = rep->part_weights;
        sp_trace_record* tr = rep->trace;
        const int32_t cap = rep->trace_capacity;
        std::memset(rep, 0, sizeof(*rep));
        rep->part_weights = pw;
        rep->trace = tr;
        rep->trace_capacity = cap;
        rep->n = R.n;
        rep->edges = R.edges;
        rep->graph_regular = R.graph_kind.kind == Regularity::Regular;
        rep->max_degree = R.graph_kind.max_degree;
        rep->avg_degree = R.graph_kind.avg_degree;
        rep->degree_ratio = R.graph_kind.ratio;
        rep->num_parts = R.num_parts;
        rep->problem = 1 + static_cast<int32_t>(R.resolved.problem);
        rep->precond = static_cast<int32_t>(R.resolved.precond);
        rep->tol = R.resolved.tol;
        rep->init = static_cast<int32_t>(R.resolved.init);
        rep->eigenvectors = R.resolved.eigenvectors;
        rep->seed = R.seed;
        rep->max_iters = R.max_iters;
        rep->doubled_cut = R.doubled_cut;
        rep->epsilon = R.epsilon;
        rep->iterations = R.iterations;
        for (size_t j = 0; j < R.theta.size() && j < SP_MAX_EIG; ++j) {
            rep->theta[j] = R.theta[j];
            rep->residual_norms[j] = R.residual_norms[j];
            rep->converged[j] = R.converged[j];
        }
        for (const std::string& w : R.warnings) {
            if (w.find("breakdown") != std::string::npos) rep->warnings |= SP_WARN_BREAKDOWN_RECOVERED;
            if (w.find("max_iters") != std::string::npos) rep->warnings |= SP_WARN_UNCONVERGED;
            if (w.find("imbalance") != std::string::npos) rep->warnings |= SP_WARN_IMBALANCE;
            if (w.find("amg coarsening stagnated") != std::string::npos) rep->warnings |= SP_WARN_AMG_STAGNATED;
        }
        rep->amg_levels = static_cast<int32_t>(std::min<size_t>(R.amg_levels.size(), SP_MAX_AMG_LEVELS));
        for (int32_t l = 0; l < rep->amg_levels; ++l) {
            rep->amg_n[l] = R.amg_levels[l].n;
            rep->amg_nnz[l] = R.amg_levels[l].nnz;
        }
        rep->laplacian_s = R.times.laplacian_s;
        rep->eigensolve_s = R.times.eigensolve_s;
        rep->partition_s = R.times.partition_s;
        rep->total_s = R.times.total_s;
        rep->cutsize = R.cutsize;
        rep->imbalance = R.imbalance;
        if (pw) std::memcpy(pw, R.part_weights.data(), sizeof(double) * R.part_weights.size());
        if (tr) {
            int32_t k = 0;
            for (const TraceRecord& t : R.trace) {
                if (k >= cap) break;
                tr[k].iter = t.iter;
                tr[k].ntheta = static_cast<int32_t>(t.theta.size());
                tr[k].min_residual = t.min_residual;
                tr[k].max_residual = t.max_residual;
                for (size_t j = 0; j < t.theta.size() && j < SP_MAX_EIG; ++j) tr[k].theta[j] = t.theta[j];
                ++k;
            }
            rep->trace_len = k;
        }
    });
}

sp_status ref_build_laplacian(int32_t kind, const sp_graph* g, int64_t* offsets_out,
                              int32_t* cols_out, double* vals_out, double* diag_out,
                              double* bound_out, int32_t* is_diagonal_out) {
    return guarded([&] {
        Graph G = to_graph(g);
        LinearOperator L = build_kind(kind, G);
        const SparseMatrix& m = L.matrix;
        if (offsets_out) std::memcpy(offsets_out, m.row_offsets.data(), sizeof(int64_t) * (m.nrows + 1));
        if (cols_out) std::memcpy(cols_out, m.col_indices.data(), sizeof(int32_t) * m.nnz());
        if (vals_out) std::memcpy(vals_out, m.values.data(), sizeof(double) * m.nnz());
        if (diag_out) std::memcpy(diag_out, L.diag.data(), sizeof(double) * m.nrows);
        if (bound_out) *bound_out = L.spectral_bound;
        if (is_diagonal_out) *is_diagonal_out = L.is_diagonal ? 1 : 0;
    });
}

sp_status ref_spmm(int32_t kind, const sp_graph* g, const double* X, int32_t m, double* Y) {
    return guarded([&] {
        Graph G = to_graph(g);
        LinearOperator L = build_kind(kind, G);
        Dense x = to_dense(X, G.n(), m);
        Dense y = apply_block(L, x);
        std::memcpy(Y, y.data.data(), sizeof(double) * G.n() * m);
    });
}

sp_status ref_spmm_csr(int64_t nrows, int64_t ncols, const int64_t* offsets, const int32_t* cols,
                       const double* vals, const double* X, int32_t m, double* Y) {
    return guarded([&] {
        SparseMatrix A;
        A.nrows = nrows;
        A.ncols = ncols;
        A.row_offsets.assign(offsets, offsets + nrows + 1);
        A.col_indices.assign(cols, cols + offsets[nrows]);
        if (vals) A.values.assign(vals, vals + offsets[nrows]);
        Dense x = to_dense(X, ncols, m);
        Dense y;
        kernels::spmv_block(A, x, y);
        std::memcpy(Y, y.data.data(), sizeof(double) * nrows * m);
    });
}

sp_status ref_gram(int64_t n, const double* U, int32_t mu, const double* V, int32_t mv,
                   const double* b, double* G) {
    return guarded([&] {
        Dense u = to_dense(U, n, mu);
        Dense v = to_dense(V, n, mv);
        if (b) {
            std::vector<double> d(b, b + n);
            Dense bv;
            kernels::diag_scale(d, v, bv);
            v = std::move(bv);
        }
        Dense g = kernels::gram(u, v);
        std::memcpy(G, g.data.data(), sizeof(double) * mu * mv);
    });
}

sp_status ref_mult(int64_t n, const double* X, int32_t k, const double* C, int32_t m, int32_t op, double* Y) {
    return guarded([&] {
        Dense x = to_dense(X, n, k);
        Dense c = to_dense(C, k, m);
        Dense y;
        if (op == 0) {
            kernels::mult(x, c, y);
        } else {
            y = to_dense(Y, n, m);
            kernels::mult_sub(y, x, c);
        }
        std::memcpy(Y, y.data.data(), sizeof(double) * n * m);
    });
}

sp_status ref_initial_guess(int32_t init, int64_t n, int32_t d, uint64_t seed, double* X_out) {
    return guarded([&] {
        Dense X = init == SP_INIT_PIECEWISE ? initial_guess_piecewise(n, d)
                                            : initial_guess_random(n, d, seed);
        std::memcpy(X_out, X.data.data(), sizeof(double) * n * d);
    });
}

sp_status ref_lobpcg(const sp_graph* g, int32_t problem, int32_t precond, uint64_t poly_seed,
                     int32_t poly_degree, const double* X0, int32_t nev, double tol,
                     int32_t max_iters, int32_t locking, double* theta_out, double* X_out,
                     double* residuals_out, uint8_t* converged_out, int32_t* iterations_out,
                     int32_t* retries_out) {
    return guarded([&] {
        Graph G = to_graph(g);
        EigenProblem p = build_problem(G, problem_of(problem));
        std::unique_ptr<Preconditioner> M;
        if (precond == SP_PRECOND_JACOBI) M = jacobi_build(p.A);
        if (precond == SP_PRECOND_POLYNOMIAL) {
            PolyConfig pc;
            pc.seed = poly_seed;
            if (poly_degree > 0) pc.degree = poly_degree;
            M = polynomial_build(p.A, pc);
        }
        if (precond == SP_PRECOND_AMG) {  // presets by classify (pipeline.cpp:107-112), seed from poly_seed
            AmgConfig ac = classify(G).kind == Regularity::Regular ? AmgConfig::regular_defaults()
                                                                   : AmgConfig::irregular_defaults();
            ac.seed = poly_seed;
            M = amg_build(p.A, ac);
        }
        SolverConfig sc;
        sc.nev = nev;
        sc.tol = tol;
        sc.max_iters = max_iters;
        sc.locking = locking != 0;
        Dense x0 = to_dense(X0, G.n(), nev);
        EigenResult r = lobpcg(p, M.get(), x0, sc);
        for (int j = 0; j < nev; ++j) {
            theta_out[j] = r.theta[j];
            if (residuals_out) residuals_out[j] = r.residual_norms[j];
            if (converged_out) converged_out[j] = r.converged[j];
        }
        if (X_out) std::memcpy(X_out, r.X.data.data(), sizeof(double) * G.n() * nev);
        if (iterations_out) *iterations_out = r.iterations;
        if (retries_out) *retries_out = r.breakdown_retries;
    });
}

sp_status ref_poly_apply(int32_t kind, const sp_graph* g, uint64_t seed, int32_t degree,
                         const double* R, int32_t m, double* H_out, double* roots_out,
                         int32_t* achieved_out) {
    (void)roots_out; // the reference keeps its roots private
    return guarded([&] {
        Graph G = to_graph(g);
        LinearOperator A = build_kind(kind, G);
        PolyConfig pc;
        pc.seed = seed;
        if (degree > 0) pc.degree = degree;
        auto M = polynomial_build(A, pc);
        Dense r = to_dense(R, G.n(), m);
        Dense h = M->apply(r);
        std::memcpy(H_out, h.data.data(), sizeof(double) * G.n() * m);
        if (achieved_out) *achieved_out = M->achieved_degree();
    });
}

// Same as ref_poly_apply on an explicit CSR operator (diagonal-operator KATs,
// preconditioner_test.cpp:38-118, acceptance.cpp:361-403).
sp_status ref_poly_apply_csr(int64_t n, const int64_t* offsets, const int32_t* cols,
                             const double* vals, uint64_t seed, int32_t degree, const double* R,
                             int32_t m, double* H_out, int32_t* achieved_out) {
    return guarded([&] {
        SparseMatrix A;
        A.nrows = A.ncols = n;
        A.row_offsets.assign(offsets, offsets + n + 1);
        A.col_indices.assign(cols, cols + offsets[n]);
        A.values.assign(vals, vals + offsets[n]);
        LinearOperator op = make_operator(std::move(A));
        PolyConfig pc;
        pc.seed = seed;
        if (degree > 0) pc.degree = degree;
        auto M = polynomial_build(op, pc);
        Dense r = to_dense(R, n, m);
        Dense h = M->apply(r);
        std::memcpy(H_out, h.data.data(), sizeof(double) * n * m);
        if (achieved_out) *achieved_out = M->achieved_degree();
    });
}

sp_status ref_precond_apply(int32_t kind, const sp_graph* g, int32_t precond, uint64_t seed, int32_t degree,
                            const double* R, int32_t m, double* H_out) {
    return guarded([&] {
        Graph G = to_graph(g);
        LinearOperator A = build_kind(kind, G);
        std::unique_ptr<Preconditioner> M;
        if (precond == SP_PRECOND_JACOBI) M = jacobi_build(A);
        else if (precond == SP_PRECOND_POLYNOMIAL) {
            PolyConfig pc;
            pc.seed = seed;
            if (degree > 0) pc.degree = degree;
            M = polynomial_build(A, pc);
        } else if (precond == SP_PRECOND_AMG) {
            AmgConfig ac = classify(G).kind == Regularity::Regular ? AmgConfig::regular_defaults()
                                                                   : AmgConfig::irregular_defaults();
            ac.seed = seed;
            M = amg_build(A, ac);
        }
        Dense r = to_dense(R, G.n(), m);
        Dense h = M ? M->apply(r) : r;
        std::memcpy(H_out, h.data.data(), sizeof(double) * G.n() * m);
    });
}

sp_status ref_mj_partition(int64_t n, int32_t dims, const double* coords, const double* weights,
                           int64_t num_parts, int32_t* assignment_out, double* part_weights_out,
                           double* imbalance_out) {
    return guarded([&] {
        Embedding e;
        e.coords = to_dense(coords, n, dims);
        e.d = dims + 1;
        std::vector<double> w = weights ? std::vector<double>(weights, weights + n)
                                        : std::vector<double>(n, 1.0);
        Partition p = mj_partition(e, w, num_parts);
        std::memcpy(assignment_out, p.assignment.data(), sizeof(int32_t) * n);
        if (part_weights_out)
            std::memcpy(part_weights_out, p.part_weights.data(), sizeof(double) * num_parts);
        if (imbalance_out) *imbalance_out = p.imbalance;
    });
}

sp_status ref_cut_imbalance(const sp_graph* g, const int32_t* assignment, int64_t num_parts,
                            int32_t doubled, double* cut_out, double* imbalance_out,
                            double* part_weights_out) {
    return guarded([&] {
        Graph G = to_graph(g);
        std::vector<int32_t> a(assignment, assignment + G.n());
        Partition p = make_partition(G, std::move(a), static_cast<int32_t>(num_parts), doubled != 0);
        if (cut_out) *cut_out = p.cutsize;
        if (imbalance_out) *imbalance_out = p.imbalance;
        if (part_weights_out)
            std::memcpy(part_weights_out, p.part_weights.data(), sizeof(double) * num_parts);
    });
}

sp_status ref_sym_eig(int32_t m, const double* A, double* values_out, double* vectors_out) {
    return guarded([&] {
        Dense a = to_dense(A, m, m);
        std::vector<double> vals;
        Dense vecs;
        sym_eig(a, vals, vecs);
        std::memcpy(values_out, vals.data(), sizeof(double) * m);
        std::memcpy(vectors_out, vecs.data.data(), sizeof(double) * m * m);
    });
}

// Graph generators of the reference (generators.cpp) — used to cross-check the
// repo's own generators byte for byte. Returns the CSR through caller buffers
// sized by a first call with NULL outputs (n and nnz written).
sp_status ref_generate(const char* spec, int64_t* n_out, int64_t* nnz_out, int64_t* offsets_out,
                       int32_t* cols_out) {
    return guarded([&] {
        Graph G = generate(GeneratorSpec::parse(spec));
        *n_out = G.n();
        *nnz_out = G.adjacency.nnz();
        if (offsets_out)
            std::memcpy(offsets_out, G.adjacency.row_offsets.data(), sizeof(int64_t) * (G.n() + 1));
        if (cols_out)
            std::memcpy(cols_out, G.adjacency.col_indices.data(), sizeof(int32_t) * G.adjacency.nnz());
    });
}

// symmetrize + largest_connected_component (graph.cpp:44-64, 118-171) on an
// arbitrary square pattern; writes the component CSR and the old-id map.
sp_status ref_symmetrize_lcc(int64_t n, const int64_t* offsets, const int32_t* cols,
                             int64_t* n_out, int64_t* nnz_out, int64_t* offsets_out,
                             int32_t* cols_out, int64_t* old_ids_out) {
    return guarded([&] {
        SparseMatrix A;
        A.nrows = A.ncols = n;
        A.row_offsets.assign(offsets, offsets + n + 1);
        A.col_indices.assign(cols, cols + offsets[n]);
        Graph whole = symmetrize(A);
        auto [sub, old] = largest_connected_component(whole);
        *n_out = sub.n();
        *nnz_out = sub.adjacency.nnz();
        if (offsets_out)
            std::memcpy(offsets_out, sub.adjacency.row_offsets.data(), sizeof(int64_t) * (sub.n() + 1));
        if (cols_out)
            std::memcpy(cols_out, sub.adjacency.col_indices.data(), sizeof(int32_t) * sub.adjacency.nnz());
        if (old_ids_out) std::memcpy(old_ids_out, old.data(), sizeof(int64_t) * old.size());
    });
}

} // extern "C"
