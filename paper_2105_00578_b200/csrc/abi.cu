// abi.cu — extern "C" entry points (include/specpart_b200.h) and the
// partition_graph pipeline (src/pipeline.cpp:47-167) on the device.
#include "specpart_b200.h"

#include "context.hpp"
#include "ingest.hpp"
#include "metrics.hpp"
#include "amg.hpp"
#include "mj.hpp"
#include "solver.hpp"

#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

namespace spb {

long long& launch_counter() {
    thread_local long long c = 0;
    return c;
}

int device_sm_count() {
    static int sms = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return 148;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
        return v > 0 ? v : 148;
    }();
    return sms;
}

namespace {

// rows with at least this many entries get a CTA each (spmm_long_kernel) in the
// solver; shorter rows stay in the order-exact group kernel
constexpr int64_t kLongRow = 512;

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

__global__ void rebase_kernel(int64_t n1, int64_t* offs, int64_t base) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n1;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        offs[i] -= base;
}

template <class T> void h2d(T* dst, const T* src, size_t count, cudaStream_t s) {
    if (count) SPB_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyHostToDevice, s));
}

// H2D of the local row block of the caller's host graph (no computation).
void copy_graph(sp_context* ctx, const sp_graph* hg, DevGraph& g) {
    if (!hg || hg->n < 0 || (hg->n > 0 && (!hg->row_offsets || !hg->col_indices)))
        throw_invalid("graph: null arrays");
    Comm& cm = ctx->comm;
    cudaStream_t s = ctx->stream;
    g.n_global = hg->n;
    g.nnz_global = hg->n > 0 ? hg->row_offsets[hg->n] : 0;
    cm.setup(hg->n);
    g.row0 = cm.active() ? cm.row0() : 0;
    g.n_local = cm.active() ? cm.nloc() : hg->n;
    const int64_t k0 = hg->n > 0 ? hg->row_offsets[g.row0] : 0;
    const int64_t k1 = hg->n > 0 ? hg->row_offsets[g.row0 + g.n_local] : 0;
    g.nnz_local = k1 - k0;
    g.offs.alloc(g.n_local + 1);
    g.cols.alloc(std::max<int64_t>(g.nnz_local, 1));
    if (hg->n > 0) {
        h2d(g.offs.p, hg->row_offsets + g.row0, g.n_local + 1, s);
        if (k0 != 0) {
            rebase_kernel<<<grid_for(g.n_local + 1, 256, 4), 256, 0, s>>>(g.n_local + 1, g.offs.p, k0);
            SPB_LAUNCH_CHECK();
        }
        h2d(g.cols.p, hg->col_indices + k0, g.nnz_local, s);
    }
    if (hg->values) {
        g.vals.alloc(std::max<int64_t>(g.nnz_local, 1));
        h2d(g.vals.p, hg->values + k0, g.nnz_local, s);
    } else {
        g.vals.release();
    }
    if (hg->vertex_weights) {
        // MJ and the part tallies need every vertex's weight
        g.vw_all.alloc(std::max<int64_t>(hg->n, 1));
        h2d(g.vw_all.p, hg->vertex_weights, hg->n, s);
    } else {
        g.vw_all.release();
    }
    g.prepared = false;
}

__global__ void weight_flags_kernel(int64_t n, const double* w, int* flags) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = w[i];
        if (v != 1.0) atomicOr(flags, 1);
        if (!(v > 0.0)) atomicOr(flags, 2);
    }
}

// Degrees, unit-cost / unit-weight detection, max degree; multi-GPU: global
// max degree and all-vertex degrees.
void prepare_graph(sp_context* ctx, DevGraph& g) {
    if (g.prepared) return;
    Comm& cm = ctx->comm;
    cudaStream_t s = ctx->stream;
    g.unit_weights = true;
    g.positive_weights = true;
    if (g.vw_all.p) {
        DBuf<int> f(1);
        SPB_CUDA(cudaMemsetAsync(f.p, 0, sizeof(int), s));
        weight_flags_kernel<<<grid_for(g.n_global, 256, 8), 256, 0, s>>>(g.n_global, g.vw_all.p, f.p);
        SPB_LAUNCH_CHECK();
        int hf = 0;
        SPB_CUDA(cudaMemcpyAsync(&hf, f.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        g.unit_weights = (hf & 1) == 0;
        g.positive_weights = (hf & 2) == 0;
        if (!g.unit_weights) {
            g.vw.alloc(std::max<int64_t>(g.n_local, 1));
            SPB_CUDA(cudaMemcpyAsync(g.vw.p, g.vw_all.p + g.row0, sizeof(double) * g.n_local,
                                     cudaMemcpyDeviceToDevice, s));
        }
    }
    graph_degrees(g, s);
    g.max_degree_global = g.max_degree_local;
    g.positive_degrees = g.positive_degrees_local;
    if (cm.active()) {
        DBuf<int64_t> t(cm.world), one(1);
        int64_t v = g.max_degree_local;
        h2d(one.p, &v, 1, s);
        SPB_NCCL(::spb::nccl().AllGather(one.p, t.p, 1, ncclInt64, cm.nccl, s));
        std::vector<int64_t> h(cm.world);
        SPB_CUDA(cudaMemcpyAsync(h.data(), t.p, sizeof(int64_t) * cm.world, cudaMemcpyDeviceToHost, s));
        int64_t flags[2] = {g.unit_values ? 0 : 1, g.positive_degrees_local ? 0 : 1};
        DBuf<int64_t> fl(2);
        h2d(fl.p, flags, 2, s);
        cm.sum_i64(fl.p, 2, s);
        SPB_CUDA(cudaMemcpyAsync(flags, fl.p, sizeof(flags), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        g.max_degree_global = *std::max_element(h.begin(), h.end());
        g.unit_values = flags[0] == 0;
        g.positive_degrees = flags[1] == 0;
        DBuf<double> padded(cm.n_pad);
        SPB_CUDA(cudaMemsetAsync(padded.p, 0, sizeof(double) * cm.n_pad, s));
        SPB_CUDA(cudaMemcpyAsync(padded.p, g.deg.p, sizeof(double) * g.n_local, cudaMemcpyDeviceToDevice, s));
        g.deg_all.alloc(static_cast<size_t>(cm.n_pad) * cm.world);
        cm.gather_f64(padded.p, g.deg_all.p, s);
    }
    g.prepared = true;
}

void upload_graph(sp_context* ctx, const sp_graph* hg, DevGraph& g) {
    copy_graph(ctx, hg, g);
    prepare_graph(ctx, g);
}

struct GraphKindInfo {
    bool regular = true;
    int64_t max_degree = 0;
    double avg = 0.0, ratio = 0.0;
};

// classify (graph.cpp:173-182)
GraphKindInfo classify(const DevGraph& g) {
    if (g.n_global == 0) throw_invalid("classify: empty graph");
    GraphKindInfo k;
    k.max_degree = g.max_degree_global;
    k.avg = static_cast<double>(g.nnz_global) / static_cast<double>(g.n_global);
    k.ratio = k.avg > 0.0 ? static_cast<double>(k.max_degree) / k.avg
                          : (k.max_degree > 0 ? std::numeric_limits<double>::infinity() : 0.0);
    k.regular = k.ratio <= 10.0;
    return k;
}

int eigenvector_count(int64_t K) {
    if (K < 2) throw_infeasible("eigenvector_count: K must be >= 2");
    return static_cast<int>(std::bit_width(static_cast<uint64_t>(K)));  // floor(log2 K) + 1
}

// select_defaults (pipeline.cpp:20-37): returns (problem, tol)
std::pair<int, double> select_defaults(bool regular, int precond) {
    switch (precond) {
    case SP_PRECOND_JACOBI:
    case SP_PRECOND_NONE:
        return regular ? std::pair{SP_PROBLEM_COMBINATORIAL, 1e-3} : std::pair{SP_PROBLEM_GENERALIZED, 1e-2};
    case SP_PRECOND_POLYNOMIAL:
        return regular ? std::pair{SP_PROBLEM_COMBINATORIAL, 1e-3} : std::pair{SP_PROBLEM_NORMALIZED, 1e-2};
    case SP_PRECOND_AMG:
        return regular ? std::pair{SP_PROBLEM_COMBINATORIAL, 1e-2} : std::pair{SP_PROBLEM_GENERALIZED, 1e-2};
    }
    throw_invalid("select_defaults: preconditioner must be resolved");
    return {};
}

// problem kind -> Laplacian kind of problem.A
int operator_kind(int problem) { return problem == SP_PROBLEM_NORMALIZED ? 1 : 0; }

sp_status map_exception(sp_context* ctx) {
    try {
        throw;
    } catch (const BreakdownErr& e) {
        if (ctx) ctx->err = e.what();
        return SP_BREAKDOWN;
    } catch (const SpError& e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return SP_ERROR;
    }
}

template <class F> sp_status guarded(sp_context* ctx, F&& f) {
    if (!ctx) return SP_INVALID;
    try {
        SPB_CUDA(cudaSetDevice(ctx->device));
        AllocStreamScope scope(ctx->stream);
        f();
        ctx->comm.sym_check(ctx->stream);  // a timed-out peer wait fails the call
        return SP_OK;
    } catch (...) {
        return map_exception(ctx);
    }
}

// row-major device block <-> column-major host array (local rows)
void upload_block(const double* host_colmajor, int64_t n_glob, int64_t row0, int64_t nloc, int m,
                  const View& dst, cudaStream_t s) {
    DBuf<double> tmp(static_cast<size_t>(std::max<int64_t>(nloc, 1)) * m);
    for (int c = 0; c < m; ++c)
        h2d(tmp.p + static_cast<size_t>(c) * nloc, host_colmajor + static_cast<size_t>(c) * n_glob + row0, nloc, s);
    copy_view(nloc, colmajor(tmp.p, nloc, m), dst, s);
    SPB_CUDA(cudaStreamSynchronize(s));
}

void download_block(const View& src, int64_t nloc, int m, double* host_colmajor, cudaStream_t s) {
    DBuf<double> tmp(static_cast<size_t>(std::max<int64_t>(nloc, 1)) * m);
    copy_view(nloc, src, colmajor(tmp.p, nloc, m), s);
    if (nloc * m) SPB_CUDA(cudaMemcpyAsync(host_colmajor, tmp.p, sizeof(double) * nloc * m, cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
}

// Gather a row-major local block (n_loc x m) to all ranks as a global
// row-major (n_global... padded) block.
View gather_block(sp_context* ctx, const View& local, int m, DBuf<double>& keep) {
    Comm& cm = ctx->comm;
    if (!cm.active()) return local;
    View g = cm.gather_rows(local, m, ctx->stream);
    keep.alloc(static_cast<size_t>(cm.n_pad) * cm.world * m);
    SPB_CUDA(cudaMemcpyAsync(keep.p, g.ptr, sizeof(double) * cm.n_pad * cm.world * m, cudaMemcpyDeviceToDevice, ctx->stream));
    return rowmajor(keep.p, m, m);
}

void validate_config(int64_t n, const sp_config* cfg) {
    const int64_t K = cfg->num_parts;
    if (K < 2) throw_infeasible("partition_graph: K must be >= 2");
    if (K > n)
        throw_infeasible("partition_graph: K exceeds vertex count (K=" + std::to_string(K) + ", n=" +
                         std::to_string(n) + ")");
    if (cfg->epsilon < 0.0) throw_infeasible("partition_graph: epsilon < 0");
}

// Gershgorin bound of an explicit CSR operator (laplacian.cpp:14-28): max_i (a_ii + sum_j!=i |a_ij|)
__global__ void explicit_bound_kernel(const DevOp op, unsigned long long* out) {
    double b = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double d = 0.0, off = 0.0;
        for (int64_t k = op.offs[i]; k < op.offs[i + 1]; ++k) {
            if (op.cols[k] == i) d += op.vals[k];
            else off += fabs(op.vals[k]);
        }
        b = fmax(b, d + off);
    }
    // the bound is >= 0 (it starts at 0.0): doubles >= 0 order like their bit patterns
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(b)));
}
// inverse_diagonal (preconditioners.cpp:44-49) of an explicit CSR operator
__global__ void explicit_inv_diag_kernel(const DevOp op, double* inv) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double d = 0.0;
        for (int64_t k = op.offs[i]; k < op.offs[i + 1]; ++k)
            if (op.cols[k] == i) d = op.vals[k];
        inv[i] = fabs(d) < 1e-300 ? 1.0 : 1.0 / d;
    }
}
double explicit_bound(const DevOp& op, cudaStream_t s) {
    DBuf<unsigned long long> d(1);
    SPB_CUDA(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), s));
    explicit_bound_kernel<<<grid_for(op.n, 256, 4), 256, 0, s>>>(op, d.p);
    SPB_LAUNCH_CHECK();
    unsigned long long h = 0;
    SPB_CUDA(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    double b;
    std::memcpy(&b, &h, sizeof(b));
    return b;
}

// amg_build on problem.A (the explicit CSR of the Laplacian, built here) into the solver
void setup_amg(sp_context* ctx, DevGraph& g, int lap_kind, bool regular, uint64_t seed, Solver& solver) {
    if (ctx->comm.active()) throw SpError(SP_ERROR, "amg_build: the AMG preconditioner runs on one GPU in this build");
    cudaStream_t s = ctx->stream;
    DevLaplacian Lx;
    build_laplacian(lap_kind, g, true, Lx, s);
    CsrDev A0;
    A0.nrows = A0.ncols = g.n_local;
    A0.nnz = g.nnz_local + g.n_local;
    A0.max_row = static_cast<int>(std::min<int64_t>(g.max_degree_global + 1, 1 << 30));
    A0.offs = std::move(Lx.offs_L);
    A0.cols = std::move(Lx.cols_L);
    A0.vals = std::move(Lx.vals_L);
    AmgCfg ac = regular ? AmgCfg::regular_defaults() : AmgCfg::irregular_defaults();
    ac.seed = seed;
    solver.build_amg(std::move(A0), std::move(Lx.diag), ac);
}

// partition_graph (pipeline.cpp:47-167) on a graph whose arrays are on the
// device. Writes all n part ids to asg (device) and fills the report.
void partition_core(sp_context* ctx, DevGraph& g, const sp_config* cfg, const double* x0, DBuf<int32_t>& asg,
                    sp_report* rep, Clock::time_point t_total) {
    cudaStream_t s = ctx->stream;
    const int64_t K = cfg->num_parts;
    const int64_t n = g.n_global;
    ctx->timers = Timers{};
    ctx->ev_used = 0;
    ctx->comm.bytes_moved = 0;
    const long long launches0 = launch_counter();
    ctx->prof.on = std::getenv("SPB_PROFILE") != nullptr;
    ctx->prof.start(s);
    sp_report R{};
    double* pw_out = rep ? rep->part_weights : nullptr;
    sp_trace_record* tr_out = rep ? rep->trace : nullptr;
    const int32_t tr_cap = rep ? rep->trace_capacity : 0;
    double* ev_out = rep ? rep->eigenvectors_out : nullptr;

    // Stage 1: degrees, classification, operators (the copy, if any, is already queued)
    const auto t_lap = Clock::now();
    prepare_graph(ctx, g);
    const GraphKindInfo kind = classify(g);
    R.n = n;
    R.edges = g.nnz_global / 2;
    R.graph_regular = kind.regular;
    R.max_degree = kind.max_degree;
    R.avg_degree = kind.avg;
    R.degree_ratio = kind.ratio;
    R.num_parts = K;
    R.seed = cfg->seed;
    R.max_iters = cfg->max_iters;
    R.epsilon = cfg->epsilon;
    R.doubled_cut = cfg->doubled_cut;
    // resolution order: classify -> precond -> (problem, tol) -> init (pipeline.cpp:66-82)
    R.precond = cfg->precond == SP_PRECOND_AUTO ? (kind.regular ? SP_PRECOND_AMG : SP_PRECOND_POLYNOMIAL)
                                                : cfg->precond;
    const auto [auto_problem, auto_tol] = select_defaults(kind.regular, R.precond);
    R.problem = cfg->problem == SP_PROBLEM_AUTO ? auto_problem : cfg->problem;
    R.tol = cfg->tol > 0.0 ? cfg->tol : auto_tol;
    R.init = cfg->init == SP_INIT_AUTO ? (kind.regular ? SP_INIT_RANDOM : SP_INIT_PIECEWISE) : cfg->init;
    R.eigenvectors = eigenvector_count(K);
    const int d = R.eigenvectors;
    if (d > n)
        throw_infeasible("partition_graph: needs d=" + std::to_string(d) + " eigenvectors but n=" +
                         std::to_string(n));
    if (d > 32) throw_dimension("partition_graph: d > 32 eigenvectors is not supported");

    // irregular graphs on one GPU: the solver runs on a degree-descending relabel of the
    // graph (relabel.cu; hub rows of every block stay L2-resident for the SpMM gathers)
    Relabel rl;
    DevGraph gr;
    if (!kind.regular && !ctx->comm.active() && ctx->relabel) {
        relabel_by_degree(g, gr, rl, s);
        prepare_graph(ctx, gr);
    }
    DevGraph& go = rl.on ? gr : g;  // the graph the operators are built on
    DevLaplacian A;
    build_laplacian(operator_kind(R.problem), go, false, A, s);
    A.op.bound = ctx->comm.max_f64(A.op.bound, s);  // Gershgorin bound of the whole operator
    if (!kind.regular) build_row_bins(A.op, kLongRow, A.bins, s);  // length bins + long-row list
    // multi-GPU: a structured mesh whose row blocks are whole z planes keeps the TMA
    // stencil kernel (halo planes after the own rows); recognised on global ids
    if (ctx->comm.active() && kind.regular && !no_mesh_kernel()) mesh_plan_slab(A.op, ctx->comm.n_global, s);
    localize_operator(ctx->comm, go, A, s);  // multi-GPU: halo numbering + exchange plan
    const double* bdiag = nullptr;
    if (R.problem == SP_PROBLEM_GENERALIZED) {
        // B = D must be positive (laplacian.cpp:169-173)
        if (!g.positive_degrees) throw_degenerate("generalized problem requires positive degrees");
        bdiag = go.deg.p;
    }
    SPB_CUDA(cudaStreamSynchronize(s));
    R.laplacian_s = since(t_lap);
    ctx->prof.mark(s, "laplacian");

    // Stage 2: preconditioner + eigensolve
    const auto t_eig = Clock::now();
    Solver solver(ctx, A.op, bdiag, d);
    solver.set_recurrence(ctx->recurrence);
    ctx->prof.mark(s, "solver_setup");  // operator analysis (ELL, slot patterns, mesh plan), blocks
    const int64_t nloc = g.n_local;
    DBuf<double> Xb, X0b;
    const View X = solver.block(solver.input_block(d, Xb), d);
    // the initial block in the reference's vertex order (then permuted into the relabel);
    // random draws run on the side stream, overlapping the preconditioner build
    if (rl.on) X0b.alloc(solver.block_elems(d));
    const View X0 = rl.on ? solver.block(X0b.p, d) : X;
    const bool side_rng = !x0 && R.init == SP_INIT_RANDOM;
    // however this scope ends, s waits for the side stream before the blocks are released
    struct AuxJoin {
        sp_context* c;
        bool on;
        ~AuxJoin() {
            if (on) cudaStreamWaitEvent(c->stream, c->aux_done, 0);
        }
    } aux_join{ctx, false};
    if (side_rng) {
        if (!ctx->aux) {
            SPB_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
            SPB_CUDA(cudaEventCreateWithFlags(&ctx->aux_ready, cudaEventDisableTiming));
            SPB_CUDA(cudaEventCreateWithFlags(&ctx->aux_done, cudaEventDisableTiming));
        }
        SPB_CUDA(cudaEventRecord(ctx->aux_ready, s));
        SPB_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->aux_ready, 0));
        initial_block_random(n, d, cfg->seed, g.row0, nloc, X0, ctx->aux);
        SPB_CUDA(cudaEventRecord(ctx->aux_done, ctx->aux));
        aux_join.on = true;
    }
    DBuf<double> inv;
    if (R.precond == SP_PRECOND_JACOBI) {
        inverse_diagonal(A, inv, s);
        solver.set_jacobi(inv.p);
    } else if (R.precond == SP_PRECOND_POLYNOMIAL) {
        solver.build_poly(cfg->seed ^ 0x706f6c79ULL, 25);
        R.poly_degree = static_cast<int32_t>(solver.roots().size());
    } else if (R.precond == SP_PRECOND_AMG) {
        // pipeline.cpp:107-118: regular / irregular presets, seed ^ "amg"
        setup_amg(ctx, go, operator_kind(R.problem), kind.regular, cfg->seed ^ 0x616d67ULL, solver);
        const Amg* amg = solver.amg();
        R.amg_levels = std::min(amg->levels(), SP_MAX_AMG_LEVELS);
        for (int l = 0; l < R.amg_levels; ++l) {
            R.amg_n[l] = amg->level_n(l);
            R.amg_nnz[l] = amg->level_nnz(l);
        }
        if (amg->stagnated()) R.warnings |= SP_WARN_AMG_STAGNATED;
    } else {
        solver.set_none();
    }
    ctx->prof.mark(s, "precond_build");
    if (x0) upload_block(x0, n, g.row0, nloc, d, X0, s);
    else if (side_rng) SPB_CUDA(cudaStreamWaitEvent(s, ctx->aux_done, 0));
    else initial_block_piecewise(n, d, g.row0, nloc, X0, s);
    ctx->prof.mark(s, "initial_block");
    if (rl.on) permute_rows_in(rl, nloc, d, X0, X, s);
    ctx->prof.mark(s, "initial_permute");
    SolveOpts so;
    so.nev = d;
    so.tol = R.tol;
    so.max_iters = cfg->max_iters;
    so.record_trace = cfg->record_trace != 0;
    SolveResult er = solver.lobpcg(X, so, X);
    SPB_CUDA(cudaStreamSynchronize(s));
    R.eigensolve_s = since(t_eig);
    R.iterations = er.iterations;
    R.breakdown_retries = er.retries;
    for (int j = 0; j < d; ++j) {
        R.theta[j] = er.theta[j];
        R.residual_norms[j] = er.residual_norms[j];
        R.converged[j] = er.converged[j];
    }
    if (er.retries > 0) R.warnings |= SP_WARN_BREAKDOWN_RECOVERED;
    if (!er.all_converged()) R.warnings |= SP_WARN_UNCONVERGED;

    // Stage 3: embed (drop column 0) + multi-jagged on the whole embedding
    const auto t_mj = Clock::now();
    DBuf<double> Xall;
    View Xsrc = X;
    if (rl.on) {  // back to the reference's vertex order (MJ ties break by vertex id)
        permute_rows_out(rl, nloc, d, X, X0, s);
        Xsrc = X0;
    }
    const View Xg = gather_block(ctx, Xsrc, d, Xall);
    asg.alloc(static_cast<size_t>(std::max<int64_t>(ctx->comm.active() ? ctx->comm.n_pad * ctx->comm.world : n, 1)));
    if (!g.positive_weights) throw_infeasible("mj_partition: weights must be positive");
    mj_partition_dev(n, d - 1, Xg.sub(1, d - 1), g.vw_all.p, g.unit_weights, K, asg.p, s);
    R.partition_s = since(t_mj);
    ctx->prof.mark(s, "mj");

    // metrics (make_partition, graph.cpp:209-230)
    PartitionMetrics pm = make_partition_dev(ctx, g, asg.p, K, cfg->doubled_cut != 0);
    R.cutsize = pm.cut;
    R.imbalance = pm.imbalance;
    if (R.imbalance > 1.0 + cfg->epsilon) R.warnings |= SP_WARN_IMBALANCE;
    SPB_CUDA(cudaStreamSynchronize(s));
    ctx->prof.mark(s, "metrics");
    if (ev_out) download_block(Xg, n, d, ev_out, s);  // EigenResult::X, on request (tests)
    ctx->prof.dump("partition_core");
    ctx->collect_spmm_times();
    R.total_s = since(t_total);
    R.spmm_launches = ctx->timers.spmm_launches;
    R.mesh_launches = ctx->timers.mesh_launches;
    R.spmm_bytes = ctx->timers.spmm_bytes;
    R.spmm_ms = ctx->timers.spmm_ms;
    R.poly_launches = ctx->timers.poly_launches;
    R.poly_bytes = ctx->timers.poly_bytes;
    R.poly_ms = ctx->timers.poly_ms;
    R.halo_launches = ctx->timers.halo_launches;
    R.halo_bytes = ctx->timers.halo_bytes;
    R.halo_ms = ctx->timers.halo_ms;
    R.spmm_eff_bytes = ctx->timers.spmm_eff_bytes;
    R.poly_eff_bytes = ctx->timers.poly_eff_bytes;
    R.kernel_launches = static_cast<int32_t>(launch_counter() - launches0 + ctx->timers.kernel_launches);
    R.n_gpus = ctx->comm.world;
    if (rep) {
        R.part_weights = pw_out;
        R.eigenvectors_out = ev_out;
        R.trace = tr_out;
        R.trace_capacity = tr_cap;
        if (pw_out) std::memcpy(pw_out, pm.part_weights.data(), sizeof(double) * K);
        if (tr_out) {
            int k = 0;
            for (const TraceRec& t : er.trace) {
                if (k >= tr_cap) break;
                tr_out[k].iter = t.iter;
                tr_out[k].ntheta = static_cast<int32_t>(t.theta.size());
                tr_out[k].min_residual = t.min_residual;
                tr_out[k].max_residual = t.max_residual;
                for (size_t j = 0; j < t.theta.size() && j < SP_MAX_EIG; ++j) tr_out[k].theta[j] = t.theta[j];
                ++k;
            }
            R.trace_len = k;
        }
        *rep = R;
    }
}

// The row block of an ingested whole graph that this rank owns (copy_graph's
// slicing, on device-resident arrays); one GPU takes the arrays over.
void adopt_ingested(sp_context* ctx, IngestResult& r, sp_device_graph& h) {
    Comm& cm = ctx->comm;
    cudaStream_t s = ctx->stream;
    DevGraph& g = h.g;
    g.n_global = r.n;
    g.nnz_global = r.nnz;
    g.unit_values = true;
    g.vals.release();
    g.vw_all.release();
    h.old_ids = std::move(r.old_ids);
    h.n_sym = r.n_sym;
    h.nnz_sym = r.nnz_sym;
    h.ingested = true;
    cm.setup(r.n);
    if (!cm.active()) {
        g.row0 = 0;
        g.n_local = r.n;
        g.nnz_local = r.nnz;
        g.offs = std::move(r.offs);
        g.cols = std::move(r.cols);
    } else {
        g.row0 = cm.row0();
        g.n_local = cm.nloc();
        int64_t k[2] = {0, 0};
        SPB_CUDA(cudaMemcpyAsync(&k[0], r.offs.p + g.row0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaMemcpyAsync(&k[1], r.offs.p + g.row0 + g.n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        g.nnz_local = k[1] - k[0];
        g.offs.alloc(g.n_local + 1);
        g.cols.alloc(std::max<int64_t>(g.nnz_local, 1));
        SPB_CUDA(cudaMemcpyAsync(g.offs.p, r.offs.p + g.row0, sizeof(int64_t) * (g.n_local + 1),
                                 cudaMemcpyDeviceToDevice, s));
        if (k[0] != 0) {
            rebase_kernel<<<grid_for(g.n_local + 1, 256, 4), 256, 0, s>>>(g.n_local + 1, g.offs.p, k[0]);
            SPB_LAUNCH_CHECK();
        }
        if (g.nnz_local)
            SPB_CUDA(cudaMemcpyAsync(g.cols.p, r.cols.p + k[0], sizeof(int32_t) * g.nnz_local,
                                     cudaMemcpyDeviceToDevice, s));
        h.full_offs = std::move(r.offs);
        h.full_cols = std::move(r.cols);
    }
    g.prepared = false;
}

void fill_info(sp_context* ctx, DevGraph& g, sp_graph_info* info) {
    prepare_graph(ctx, g);
    const GraphKindInfo k = classify(g);
    info->n = g.n_global;
    info->nnz = g.nnz_global;
    info->n_symmetrized = g.n_global;
    info->nnz_symmetrized = g.nnz_global;
    info->max_degree = k.max_degree;
    info->avg_degree = k.avg;
    info->degree_ratio = k.ratio;
    info->regular = k.regular ? 1 : 0;
    info->pad = 0;
}

} // namespace

} // namespace spb

using namespace spb;

extern "C" {

int sp_version(void) { return 1; }

sp_status sp_context_create(int device, sp_context** out) {
    if (!out) return SP_INVALID;
    *out = nullptr;
    auto* c = new sp_context();
    c->device = device;
    try {
        SPB_CUDA(cudaSetDevice(device));
        SPB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        cudaMemPool_t pool;
        SPB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        SPB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        // map the pool's memory up front (SPB_POOL_RESERVE_GB, default 96, at most
        // 60% of the free memory; the pool is per device and shared by every
        // context of the process): growing a
        // pool takes driver-global locks that other processes (e.g. an nvidia-smi
        // poller) can hold for a long time; a pre-mapped pool never grows mid-solve
        const char* rg = std::getenv("SPB_POOL_RESERVE_GB");
        const double gb = rg ? std::atof(rg) : 96.0;
        size_t fr = 0, tot = 0;
        SPB_CUDA(cudaMemGetInfo(&fr, &tot));
        const size_t want = std::min(static_cast<size_t>(gb * (1ull << 30)), fr / 10 * 6);
        if (want > 0) {
            void* p = nullptr;
            if (cudaMallocAsync(&p, want, c->stream) == cudaSuccess) {
                SPB_CUDA(cudaFreeAsync(p, c->stream));
                SPB_CUDA(cudaStreamSynchronize(c->stream));
            } else {
                cudaGetLastError();
            }
        }
        SPB_CUDA(cudaEventCreate(&c->ev0));
        SPB_CUDA(cudaEventCreate(&c->ev1));
    } catch (...) {
        const sp_status st = map_exception(c);
        delete c;
        return st;
    }
    *out = c;
    return SP_OK;
}

sp_status sp_nccl_unique_id(void* out128) {
    if (!out128) return SP_INVALID;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    try {
        ncclUniqueId id;
        if (nccl().GetUniqueId(&id) != ncclSuccess) return SP_NCCL;
        std::memcpy(out128, &id, sizeof(id));
    } catch (...) {
        return SP_NCCL;
    }
    return SP_OK;
}

sp_status sp_context_create_dist(int device, int rank, int world, const void* nccl_id128, sp_context** out) {
    sp_status st = sp_context_create(device, out);
    if (st != SP_OK) return st;
    if (world <= 1) return SP_OK;
    sp_context* c = *out;
    try {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id128, sizeof(id));
        SPB_NCCL(nccl().CommInitRank(&c->comm.nccl, world, id, rank));
        c->comm.rank = rank;
        c->comm.world = world;
    } catch (...) {
        st = map_exception(c);
        sp_context_destroy(c);
        *out = nullptr;
        return st;
    }
    return SP_OK;
}

void sp_context_destroy(sp_context* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    sym_release(c->comm);
    if (c->comm.nccl) nccl().CommDestroy(c->comm.nccl);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->aux) {
        cudaStreamSynchronize(c->aux);
        cudaEventDestroy(c->aux_ready);
        cudaEventDestroy(c->aux_done);
        cudaStreamDestroy(c->aux);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* sp_last_error(const sp_context* c) { return c ? c->err.c_str() : "null context"; }

sp_status sp_debug_guard_check(int64_t* violations, int64_t* buffers) {
    if (!violations || !buffers) return SP_INVALID;
    if (!spb::guard_on()) {
        *violations = *buffers = -1;
        return SP_OK;
    }
    try {
        long long checked = 0;
        *violations = spb::guard_check_all(&checked);
        *buffers = checked;
        return SP_OK;
    } catch (...) {
        return SP_CUDA;
    }
}

sp_status sp_context_set_timing(sp_context* c, int on) {
    if (!c) return SP_INVALID;
    c->time_spmm = on != 0;
    return SP_OK;
}

sp_status sp_context_set_recurrence(sp_context* ctx, int on) {
    if (!ctx) return SP_INVALID;
    ctx->recurrence = on != 0;
    return SP_OK;
}

sp_status sp_context_set_relabel(sp_context* ctx, int on) {
    if (!ctx) return SP_INVALID;
    ctx->relabel = on != 0;
    return SP_OK;
}

sp_status sp_partition(sp_context* ctx, const sp_graph* hg, const sp_config* cfg, int32_t* assignment_out,
                       sp_report* rep, const double* x0) {
    return guarded(ctx, [&] {
        if (!cfg || !assignment_out || !hg) throw_invalid("sp_partition: null argument");
        validate_config(hg->n, cfg);
        const auto t_total = Clock::now();
        DevGraph g;
        copy_graph(ctx, hg, g);
        if (ctx->prof.on) {
            SPB_CUDA(cudaStreamSynchronize(ctx->stream));
            std::fprintf(stderr, "[spb-profile] sp_partition copy_graph %.3f ms\n", since(t_total) * 1e3);
        }
        DBuf<int32_t> asg;
        partition_core(ctx, g, cfg, x0, asg, rep, t_total);
        const auto t_d2h = Clock::now();
        SPB_CUDA(cudaMemcpyAsync(assignment_out, asg.p, sizeof(int32_t) * hg->n, cudaMemcpyDeviceToHost, ctx->stream));
        SPB_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->prof.on) std::fprintf(stderr, "[spb-profile] sp_partition d2h %.3f ms\n", since(t_d2h) * 1e3);
        if (rep) rep->total_s = since(t_total);
    });
}

sp_status sp_graph_upload(sp_context* ctx, const sp_graph* hg, sp_device_graph** out) {
    return guarded(ctx, [&] {
        if (!out) throw_invalid("sp_graph_upload: null out");
        *out = nullptr;
        auto h = std::make_unique<sp_device_graph>();
        h->ctx = ctx;
        copy_graph(ctx, hg, h->g);
        SPB_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = h.release();
    });
}

void sp_graph_free(sp_device_graph* h) {
    if (!h) return;
    cudaSetDevice(h->ctx->device);
    cudaStreamSynchronize(h->ctx->stream);
    delete h;
}

sp_status sp_partition_resident(sp_context* ctx, sp_device_graph* h, const sp_config* cfg,
                                int32_t* assignment_out, sp_report* rep, const double* x0) {
    return guarded(ctx, [&] {
        if (!h || !cfg) throw_invalid("sp_partition_resident: null argument");
        validate_config(h->g.n_global, cfg);
        const auto t_total = Clock::now();
        h->g.prepared = false;  // degree scan etc. belong to the timed pipeline
        partition_core(ctx, h->g, cfg, x0, h->assignment, rep, t_total);
        if (assignment_out) {
            SPB_CUDA(cudaMemcpyAsync(assignment_out, h->assignment.p, sizeof(int32_t) * h->g.n_global,
                                     cudaMemcpyDeviceToHost, ctx->stream));
            SPB_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        if (rep) rep->total_s = since(t_total);
    });
}

sp_status sp_build_laplacian(sp_context* ctx, int32_t kind, const sp_graph* hg, int64_t* offsets_out,
                             int32_t* cols_out, double* vals_out, double* diag_out, double* bound_out,
                             int32_t* is_diagonal_out) {
    return guarded(ctx, [&] {
        if (kind < 0 || kind > 2) throw_invalid("sp_build_laplacian: unknown kind");
        if (hg->n == 0)
            throw_invalid(kind == 0 ? "build_combinatorial: empty graph"
                                    : kind == 1 ? "build_normalized: empty graph" : "build_degree: empty graph");
        if (ctx->comm.active()) throw_invalid("sp_build_laplacian: single-GPU entry point");
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        DevLaplacian L;
        build_laplacian(kind, g, true, L, s);
        const int64_t n = g.n_local;
        const int64_t nnz = kind == 2 ? n : g.nnz_local + n;
        if (offsets_out) SPB_CUDA(cudaMemcpyAsync(offsets_out, L.offs_L.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
        if (cols_out) SPB_CUDA(cudaMemcpyAsync(cols_out, L.cols_L.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, s));
        if (vals_out) SPB_CUDA(cudaMemcpyAsync(vals_out, L.vals_L.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
        if (diag_out) SPB_CUDA(cudaMemcpyAsync(diag_out, L.diag.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        if (bound_out) *bound_out = L.op.bound;
        if (is_diagonal_out) *is_diagonal_out = L.op.is_diagonal ? 1 : 0;
    });
}

sp_status sp_spmm(sp_context* ctx, int32_t kind, const sp_graph* hg, const double* X, int32_t m, double* Y) {
    return guarded(ctx, [&] {
        if (m < 1 || m > kMaxCols) throw_dimension("sp_spmm: 1 <= m <= 64");
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        DevLaplacian L;
        build_laplacian(kind, g, false, L, s);
        // multi-GPU: every rank passes the full X and receives the full Y; each
        // computes its row block after a halo exchange (the bit-exactness check
        // of the row-partitioned operator)
        localize_operator(ctx->comm, g, L, s);
        const int64_t nloc = g.n_local;
        Solver solver(ctx, L.op, nullptr, m);
        DBuf<double> xd, yd(solver.block_elems(m));
        const View Xv = solver.block(solver.input_block(m, xd), m);
        upload_block(X, hg->n, g.row0, nloc, m, Xv, s);
        solver.spmm_store(Xv, m, solver.block(yd.p, m));
        DBuf<double> keep;
        const View Yg = gather_block(ctx, solver.block(yd.p, m), m, keep);
        download_block(Yg, hg->n, m, Y, s);
    });
}

sp_status sp_spmm_solver(sp_context* ctx, int32_t kind, const sp_graph* hg, const double* X, int32_t m,
                         double* Y) {
    return guarded(ctx, [&] {
        if (m < 1 || m > kMaxCols) throw_dimension("sp_spmm_solver: 1 <= m <= 64");
        if (kind != 0 && kind != 1) throw_invalid("sp_spmm_solver: kind must be combinatorial or normalized");
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        const GraphKindInfo k = classify(g);
        DevLaplacian L;
        build_laplacian(kind, g, false, L, s);
        // the operator exactly as partition_core prepares it for the eigensolver
        if (!k.regular) build_row_bins(L.op, kLongRow, L.bins, s);
        localize_operator(ctx->comm, g, L, s);
        const int64_t nloc = g.n_local;
        Solver solver(ctx, L.op, nullptr, m);
        DBuf<double> xd, yd(solver.block_elems(m));
        const View Xv = solver.block(solver.input_block(m, xd), m);
        upload_block(X, hg->n, g.row0, nloc, m, Xv, s);
        solver.spmm_store(Xv, m, solver.block(yd.p, m));
        DBuf<double> keep;
        const View Yg = gather_block(ctx, solver.block(yd.p, m), m, keep);
        download_block(Yg, hg->n, m, Y, s);
    });
}

sp_status sp_spmm_csr(sp_context* ctx, int64_t nrows, int64_t ncols, const int64_t* offsets, const int32_t* cols,
                      const double* vals, const double* X, int32_t m, double* Y) {
    return guarded(ctx, [&] {
        if (m < 1 || m > kMaxCols) throw_dimension("sp_spmm_csr: 1 <= m <= 64");
        cudaStream_t s = ctx->stream;
        const int64_t nnz = offsets[nrows];
        DBuf<int64_t> o(nrows + 1);
        DBuf<int32_t> c(std::max<int64_t>(nnz, 1));
        DBuf<double> v(std::max<int64_t>(nnz, 1));
        h2d(o.p, offsets, nrows + 1, s);
        h2d(c.p, cols, nnz, s);
        if (vals) h2d(v.p, vals, nnz, s);
        else fill_view(nnz, rowmajor(v.p, 1, 1), 1.0, s);
        DevOp op;
        op.mode = OP_EXPLICIT;
        op.n = nrows;
        op.nnz = nnz;
        op.offs = o.p;
        op.cols = c.p;
        op.vals = v.p;
        op.long_threshold = int64_t(1) << 40;
        int64_t mr = 0;
        for (int64_t i = 0; i < nrows; ++i) mr = std::max(mr, offsets[i + 1] - offsets[i]);
        op.max_row = static_cast<int>(std::min<int64_t>(mr, 1 << 30));
        DBuf<double> xd(static_cast<size_t>(std::max<int64_t>(ncols, 1)) * m), yd(static_cast<size_t>(std::max<int64_t>(nrows, 1)) * m);
        upload_block(X, ncols, 0, ncols, m, rowmajor(xd.p, m, m), s);
        EpiArgs ea;
        ea.mode = EPI_STORE;
        ea.Y = rowmajor(yd.p, m, m);
        spmm_launch(op, rowmajor(xd.p, m, m), m, ea, s);
        download_block(rowmajor(yd.p, m, m), nrows, m, Y, s);
    });
}

sp_status sp_gram(sp_context* ctx, int64_t n, const double* U, int32_t mu, const double* V, int32_t mv,
                  const double* b, double* G) {
    return guarded(ctx, [&] {
        cudaStream_t s = ctx->stream;
        const size_t rows = static_cast<size_t>(std::max<int64_t>(n, 1));
        DBuf<double> ud(rows * mu), vd(rows * mv), bd, gd(static_cast<size_t>(mu + mv) * mv + 1),
            scratch(static_cast<size_t>(device_sm_count()) * 4 * (static_cast<size_t>(mu + mv) * mv + 1));
        upload_block(U, n, 0, n, mu, rowmajor(ud.p, mu, mu), s);
        upload_block(V, n, 0, n, mv, rowmajor(vd.p, mv, mv), s);
        if (b) {
            bd.alloc(rows);
            h2d(bd.p, b, n, s);
        }
        TsSpec sp;
        sp.n = n;
        sp.U0 = rowmajor(ud.p, mu, mu);
        sp.V = rowmajor(vd.p, mv, mv);
        sp.b = bd.p;
        sp.gram = true;
        sp.gram_left_u = true;
        sp.gram_left_self = false;
        SPB_CUDA(cudaMemsetAsync(scratch.p + scratch.n - 1, 0, sizeof(double), s));
        if (n > 0) ts_run(sp, gd.p, scratch.p, scratch.n, s);
        else SPB_CUDA(cudaMemsetAsync(gd.p, 0, sizeof(double) * mu * mv, s));
        SPB_CUDA(cudaMemcpyAsync(G, gd.p, sizeof(double) * mu * mv, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
    });
}

sp_status sp_block_combine(sp_context* ctx, int64_t n, const double* X, int32_t k, const double* C, int32_t m,
                           int32_t op, double* Y) {
    return guarded(ctx, [&] {
        if (n < 0 || k < 1 || m < 1 || k > 64 || m > 64) throw SpError(SP_DIMENSION, "sp_block_combine: bad sizes");
        if (op != 0 && op != 1) throw_invalid("sp_block_combine: op must be 0 (Y = X C) or 1 (Y -= X C)");
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        const size_t rows = static_cast<size_t>(n);
        DBuf<double> xd(rows * k), yd(rows * m), wd, cd(static_cast<size_t>(k) * m),
            scratch(static_cast<size_t>(device_sm_count()) * 8 * 64 + 64);
        upload_block(X, n, 0, n, k, rowmajor(xd.p, k, k), s);
        h2d(cd.p, C, static_cast<int64_t>(k) * m, s);
        SPB_CUDA(cudaMemsetAsync(scratch.p + scratch.n - 1, 0, sizeof(double), s));
        TsSpec sp;
        sp.n = n;
        sp.C = cd.p;
        sp.ldc = k;
        if (op == 0) {  // W = V C
            sp.V = rowmajor(xd.p, k, k);
            sp.W = rowmajor(yd.p, m, m);
            sp.transform = TS_COMBINE;
        } else {        // W = V - U C
            wd.alloc(rows * m);
            upload_block(Y, n, 0, n, m, rowmajor(yd.p, m, m), s);
            sp.U0 = rowmajor(xd.p, k, k);
            sp.V = rowmajor(yd.p, m, m);
            sp.W = rowmajor(wd.p, m, m);
            sp.transform = TS_UPDATE;
        }
        ts_run(sp, nullptr, scratch.p, scratch.n, s);
        download_block(sp.W, n, m, Y, s);
    });
}

sp_status sp_bench_blockop(sp_context* ctx, int64_t n, int32_t mu, int32_t mv, int32_t mw, int32_t transform,
                           int32_t gram, int32_t iters, double* ms_out) {
    return guarded(ctx, [&] {
        if (n < 1 || mv < 1 || mu < 0 || iters < 1) throw_invalid("sp_bench_blockop: bad sizes");
        if (transform == TS_UPDATE && mu < 1) throw_invalid("sp_bench_blockop: update needs mu >= 1");
        cudaStream_t s = ctx->stream;
        const int64_t ld = (n + 63) / 64 * 64;
        const int kw = transform == TS_UPDATE ? mv : (transform == TS_COMBINE ? mw : 0);
        DBuf<double> ub(static_cast<size_t>(ld) * std::max(mu, 1)), vb(static_cast<size_t>(ld) * mv),
            wb(static_cast<size_t>(ld) * std::max(kw, 1)), cb(static_cast<size_t>(std::max(mu, mv)) * std::max(kw, 1) + 1),
            gb(static_cast<size_t>(mu + mv + kw) * (mv + kw) + 64),
            scratch(static_cast<size_t>(device_sm_count()) * 8 * (static_cast<size_t>(mu + mv + kw) * (mv + kw) + 64));
        mt_uniform_block(7, ld, std::max(mu, 1), 0, ld, colmajor(ub.p, ld, std::max(mu, 1)), s);
        mt_uniform_block(8, ld, mv, 0, ld, colmajor(vb.p, ld, mv), s);
        mt_uniform_block(9, static_cast<int64_t>(cb.n), 1, 0, static_cast<int64_t>(cb.n), colmajor(cb.p, static_cast<int64_t>(cb.n), 1), s);
        TsSpec sp;
        sp.n = n;
        sp.U0 = mu > 0 ? colmajor(ub.p, ld, mu) : View{};
        sp.V = colmajor(vb.p, ld, mv);
        sp.transform = transform;
        if (transform != TS_NONE) {
            sp.W = colmajor(wb.p, ld, kw);
            sp.C = cb.p;
        }
        sp.gram = gram != 0;
        sp.gram_left_u = gram == 1 || gram == 2;
        sp.gram_left_self = gram == 1 || gram == 3;
        SPB_CUDA(cudaMemsetAsync(scratch.p + scratch.n - 1, 0, sizeof(double), s));
        ts_run(sp, gb.p, scratch.p, scratch.n, s);
        cudaEvent_t e0, e1;
        SPB_CUDA(cudaEventCreate(&e0));
        SPB_CUDA(cudaEventCreate(&e1));
        SPB_CUDA(cudaEventRecord(e0, s));
        for (int it = 0; it < iters; ++it) ts_run(sp, gb.p, scratch.p, scratch.n, s);
        SPB_CUDA(cudaEventRecord(e1, s));
        SPB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        SPB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_out = ms / iters;
    });
}

sp_status sp_initial_guess(sp_context* ctx, int32_t init, int64_t n, int32_t d, uint64_t seed, double* X_out) {
    return guarded(ctx, [&] {
        cudaStream_t s = ctx->stream;
        DBuf<double> xd(static_cast<size_t>(std::max<int64_t>(n, 1)) * std::max(d, 1));
        const View X = rowmajor(xd.p, d, d);
        if (init == SP_INIT_PIECEWISE) initial_block_piecewise(n, d, 0, n, X, s);
        else initial_block_random(n, d, seed, 0, n, X, s);
        download_block(X, n, d, X_out, s);
    });
}

sp_status sp_initial_guess_rows(sp_context* ctx, int32_t init, int64_t n, int32_t d, uint64_t seed, int64_t row0,
                               int64_t nloc, double* X_out) {
    return guarded(ctx, [&] {
        if (row0 < 0 || nloc < 0 || row0 + nloc > n) throw_dimension("sp_initial_guess_rows: slice outside [0, n)");
        cudaStream_t s = ctx->stream;
        DBuf<double> xd(static_cast<size_t>(std::max<int64_t>(nloc, 1)) * std::max(d, 1));
        const View X = rowmajor(xd.p, d, d);
        if (init == SP_INIT_PIECEWISE) initial_block_piecewise(n, d, row0, nloc, X, s);
        else initial_block_random(n, d, seed, row0, nloc, X, s);
        download_block(X, nloc, d, X_out, s);
    });
}

sp_status sp_lobpcg(sp_context* ctx, const sp_graph* hg, int32_t problem, int32_t precond, uint64_t poly_seed,
                    int32_t poly_degree, const double* X0, int32_t nev, double tol, int32_t max_iters,
                    int32_t locking, double* theta_out, double* X_out, double* residuals_out,
                    uint8_t* converged_out, int32_t* iterations_out, int32_t* retries_out) {
    return guarded(ctx, [&] {
        if (problem < SP_PROBLEM_COMBINATORIAL || problem > SP_PROBLEM_NORMALIZED)
            throw_invalid("sp_lobpcg: problem must be explicit");
        if (nev < 1) throw_infeasible("lobpcg: nev < 1");
        if (nev > 32) throw_dimension("sp_lobpcg: nev <= 32");
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        DevLaplacian A;
        build_laplacian(operator_kind(problem), g, false, A, s);
        A.op.bound = ctx->comm.max_f64(A.op.bound, s);
        localize_operator(ctx->comm, g, A, s);
        const double* bdiag = nullptr;
        if (problem == SP_PROBLEM_GENERALIZED) {
            if (!g.positive_degrees) throw_degenerate("generalized problem requires positive degrees");
            bdiag = g.deg.p;
        }
        Solver solver(ctx, A.op, bdiag, nev);
        solver.set_recurrence(ctx->recurrence);
        DBuf<double> inv;
        if (precond == SP_PRECOND_JACOBI) {
            inverse_diagonal(A, inv, s);
            solver.set_jacobi(inv.p);
        } else if (precond == SP_PRECOND_POLYNOMIAL) {
            solver.build_poly(poly_seed, poly_degree > 0 ? poly_degree : 25);
        } else if (precond == SP_PRECOND_AMG) {
            setup_amg(ctx, g, operator_kind(problem), classify(g).regular, poly_seed, solver);
        }
        const int64_t nloc = g.n_local;
        DBuf<double> Xb;
        const View X = solver.block(solver.input_block(nev, Xb), nev);
        upload_block(X0, hg->n, g.row0, nloc, nev, X, s);
        SolveOpts so;
        so.nev = nev;
        so.tol = tol;
        so.max_iters = max_iters;
        so.locking = locking != 0;
        SolveResult r = solver.lobpcg(X, so, X);
        for (int j = 0; j < nev; ++j) {
            theta_out[j] = r.theta[j];
            if (residuals_out) residuals_out[j] = r.residual_norms[j];
            if (converged_out) converged_out[j] = r.converged[j];
        }
        if (iterations_out) *iterations_out = r.iterations;
        if (retries_out) *retries_out = r.retries;
        if (X_out) {
            DBuf<double> Xall;
            const View Xg = gather_block(ctx, X, nev, Xall);
            download_block(Xg, hg->n, nev, X_out, s);
        }
    });
}

sp_status sp_poly_apply(sp_context* ctx, int32_t kind, const sp_graph* hg, uint64_t seed, int32_t degree,
                        const double* Rh, int32_t m, double* H_out, double* roots_out, int32_t* achieved_out) {
    return guarded(ctx, [&] {
        if (ctx->comm.active()) throw_invalid("sp_poly_apply: single-GPU entry point");
        if (m < 1 || m > 32) throw_dimension("sp_poly_apply: 1 <= m <= 32");
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        DevLaplacian A;
        build_laplacian(kind, g, false, A, s);
        Solver solver(ctx, A.op, nullptr, m);
        solver.build_poly(seed, degree > 0 ? degree : 25);
        const int64_t n = g.n_local;
        DBuf<double> rd, hd(solver.block_elems(m));
        const View Rv = solver.block(solver.input_block(m, rd), m);
        upload_block(Rh, n, 0, n, m, Rv, s);
        solver.apply_precond(Rv, m, solver.block(hd.p, m));
        download_block(solver.block(hd.p, m), n, m, H_out, s);
        const std::vector<double>& rt = solver.roots();
        if (roots_out) std::memcpy(roots_out, rt.data(), sizeof(double) * rt.size());
        if (achieved_out) *achieved_out = static_cast<int32_t>(rt.size());
    });
}

sp_status sp_precond_apply_csr(sp_context* ctx, int64_t n, const int64_t* offsets, const int32_t* cols,
                               const double* vals, int32_t precond, uint64_t seed, int32_t degree, const double* Rh,
                               int32_t m, double* H_out, double* roots_out, int32_t* achieved_out) {
    return guarded(ctx, [&] {
        if (ctx->comm.active()) throw_invalid("sp_precond_apply_csr: single-GPU entry point");
        if (m < 1 || m > 32) throw_dimension("sp_precond_apply_csr: 1 <= m <= 32");
        if (n < 1 || !offsets || !cols || !vals) throw_invalid("sp_precond_apply_csr: empty operator");
        cudaStream_t s = ctx->stream;
        const int64_t nnz = offsets[n];
        DBuf<int64_t> o(n + 1);
        DBuf<int32_t> c(std::max<int64_t>(nnz, 1));
        DBuf<double> v(std::max<int64_t>(nnz, 1));
        h2d(o.p, offsets, n + 1, s);
        h2d(c.p, cols, nnz, s);
        h2d(v.p, vals, nnz, s);
        DevOp op;
        op.mode = OP_EXPLICIT;
        op.n = n;
        op.nnz = nnz;
        op.offs = o.p;
        op.cols = c.p;
        op.vals = v.p;
        op.x_rows = n;
        op.long_threshold = int64_t(1) << 40;
        int64_t mr = 0;
        for (int64_t i = 0; i < n; ++i) mr = std::max(mr, offsets[i + 1] - offsets[i]);
        op.max_row = static_cast<int>(std::min<int64_t>(mr, 1 << 30));
        op.bound = explicit_bound(op, s);  // make_operator's Gershgorin bound (laplacian.cpp:14-28)
        Solver solver(ctx, op, nullptr, m);
        DBuf<double> inv(n);
        if (precond == SP_PRECOND_JACOBI) {
            explicit_inv_diag_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(op, inv.p);
            SPB_LAUNCH_CHECK();
            solver.set_jacobi(inv.p);
        } else if (precond == SP_PRECOND_POLYNOMIAL) {
            solver.build_poly(seed, degree > 0 ? degree : 25);
        } else if (precond == SP_PRECOND_NONE) {
            solver.set_none();
        } else {
            throw_invalid("sp_precond_apply_csr: jacobi, polynomial or none");
        }
        DBuf<double> rd, hd(solver.block_elems(m));
        const View Rv = solver.block(solver.input_block(m, rd), m);
        upload_block(Rh, n, 0, n, m, Rv, s);
        solver.apply_precond(Rv, m, solver.block(hd.p, m));
        download_block(solver.block(hd.p, m), n, m, H_out, s);
        const std::vector<double>& rt = solver.roots();
        if (roots_out) std::memcpy(roots_out, rt.data(), sizeof(double) * rt.size());
        if (achieved_out) *achieved_out = static_cast<int32_t>(rt.size());
    });
}

sp_status sp_precond_apply(sp_context* ctx, int32_t kind, const sp_graph* hg, int32_t precond, uint64_t seed,
                           int32_t degree, const double* Rh, int32_t m, double* H_out) {
    return guarded(ctx, [&] {
        if (ctx->comm.active()) throw_invalid("sp_precond_apply: single-GPU entry point");
        if (m < 1 || m > 32) throw_dimension("sp_precond_apply: 1 <= m <= 32");
        if (kind != 0 && kind != 1) throw_invalid("sp_precond_apply: kind must be combinatorial or normalized");
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        const GraphKindInfo k = classify(g);
        DevLaplacian A;
        build_laplacian(kind, g, false, A, s);
        if (!k.regular) build_row_bins(A.op, kLongRow, A.bins, s);
        Solver solver(ctx, A.op, nullptr, m);
        DBuf<double> inv;
        if (precond == SP_PRECOND_JACOBI) {
            inverse_diagonal(A, inv, s);
            solver.set_jacobi(inv.p);
        } else if (precond == SP_PRECOND_POLYNOMIAL) {
            solver.build_poly(seed, degree > 0 ? degree : 25);
        } else if (precond == SP_PRECOND_AMG) {
            setup_amg(ctx, g, kind, k.regular, seed, solver);
        } else if (precond == SP_PRECOND_NONE) {
            solver.set_none();
        } else {
            throw_invalid("sp_precond_apply: unknown preconditioner");
        }
        const int64_t n = g.n_local;
        DBuf<double> rd, hd(solver.block_elems(m));
        const View Rv = solver.block(solver.input_block(m, rd), m);
        upload_block(Rh, n, 0, n, m, Rv, s);
        solver.apply_precond(Rv, m, solver.block(hd.p, m));
        download_block(solver.block(hd.p, m), n, m, H_out, s);
    });
}

sp_status sp_mj_partition(sp_context* ctx, int64_t n, int32_t dims, const double* coords, const double* weights,
                          int64_t K, int32_t* assignment_out, double* part_weights_out, double* imbalance_out) {
    return guarded(ctx, [&] {
        if (K < 1) throw_infeasible("mj_partition: K < 1");
        if (n < K)
            throw_infeasible("mj_partition: fewer points than parts (n=" + std::to_string(n) + ", K=" +
                             std::to_string(K) + ")");
        bool unit = true;
        if (weights) {
            for (int64_t i = 0; i < n; ++i) {
                if (!(weights[i] > 0.0)) throw_infeasible("mj_partition: weights must be positive");
                unit &= weights[i] == 1.0;
            }
        }
        cudaStream_t s = ctx->stream;
        DBuf<double> cd(static_cast<size_t>(std::max<int64_t>(n, 1)) * std::max(dims, 1)), wd;
        upload_block(coords, n, 0, n, dims, rowmajor(cd.p, dims, dims), s);
        if (!unit) {
            wd.alloc(n);
            h2d(wd.p, weights, n, s);
        }
        DBuf<int32_t> asg(std::max<int64_t>(n, 1));
        mj_partition_dev(n, dims, rowmajor(cd.p, dims, dims), wd.p, unit, K, asg.p, s);
        SPB_CUDA(cudaMemcpyAsync(assignment_out, asg.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        // mj_partition's own tally (partitioner.cpp:161-168): vertex order per part
        std::vector<double> pw(K, 0.0);
        for (int64_t v = 0; v < n; ++v) pw[assignment_out[v]] += weights ? weights[v] : 1.0;
        if (part_weights_out) std::memcpy(part_weights_out, pw.data(), sizeof(double) * K);
        if (imbalance_out) *imbalance_out = imbalance_of(pw);
    });
}

sp_status sp_cut_imbalance(sp_context* ctx, const sp_graph* hg, const int32_t* assignment, int64_t K,
                           int32_t doubled, double* cut_out, double* imbalance_out, double* part_weights_out) {
    return guarded(ctx, [&] {
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        if (!g.unit_weights && !g.vw.p) throw_invalid("weights");
        DBuf<int32_t> a(std::max<int64_t>(ctx->comm.active() ? ctx->comm.n_pad * ctx->comm.world : hg->n, 1));
        h2d(a.p, assignment, hg->n, s);
        PartitionMetrics pm = make_partition_dev(ctx, g, a.p, K, doubled != 0);
        if (cut_out) *cut_out = pm.cut;
        if (imbalance_out) *imbalance_out = pm.imbalance;
        if (part_weights_out) std::memcpy(part_weights_out, pm.part_weights.data(), sizeof(double) * K);
    });
}

sp_status sp_cutsize(sp_context* ctx, const sp_graph* hg, const int32_t* assignment, int32_t doubled,
                     double* cut_out) {
    return guarded(ctx, [&] {
        cudaStream_t s = ctx->stream;
        DevGraph g;
        upload_graph(ctx, hg, g);
        DBuf<int32_t> a(std::max<int64_t>(ctx->comm.active() ? ctx->comm.n_pad * ctx->comm.world : hg->n, 1));
        h2d(a.p, assignment, hg->n, s);
        const double c = cutsize_dev(ctx, g, a.p, doubled != 0);
        if (cut_out) *cut_out = c;
    });
}

sp_status sp_ingest(sp_context* ctx, int64_t n, const int64_t* row_offsets, const int32_t* col_indices,
                    int32_t lcc, sp_device_graph** out) {
    return guarded(ctx, [&] {
        if (!out) throw_invalid("sp_ingest: null out");
        *out = nullptr;
        if (n < 0 || (n > 0 && (!row_offsets || !col_indices))) throw_invalid("sp_ingest: null arrays");
        cudaStream_t s = ctx->stream;
        const int64_t nnz = n > 0 ? row_offsets[n] : 0;
        if (n > 0 && row_offsets[0] != 0) throw_invalid("sp_ingest: row_offsets[0] != 0");
        DBuf<int64_t> offs(std::max<int64_t>(n + 1, 1));
        DBuf<int32_t> cols(std::max<int64_t>(nnz, 1));
        h2d(offs.p, row_offsets, n + 1, s);
        h2d(cols.p, col_indices, nnz, s);
        IngestResult r;
        ingest_graph(n, offs.p, cols.p, nnz, lcc != 0, r, s);
        offs.release();
        cols.release();
        auto h = std::make_unique<sp_device_graph>();
        h->ctx = ctx;
        adopt_ingested(ctx, r, *h);
        SPB_CUDA(cudaStreamSynchronize(s));
        *out = h.release();
    });
}

sp_status sp_device_graph_info(sp_context* ctx, sp_device_graph* h, sp_graph_info* info) {
    return guarded(ctx, [&] {
        if (!h || !info) throw_invalid("sp_device_graph_info: null argument");
        fill_info(ctx, h->g, info);
        if (h->ingested) {
            info->n_symmetrized = h->n_sym;
            info->nnz_symmetrized = h->nnz_sym;
        }
    });
}

sp_status sp_device_graph_download(sp_context* ctx, sp_device_graph* h, int64_t* offsets_out, int32_t* cols_out,
                                   int64_t* old_ids_out) {
    return guarded(ctx, [&] {
        if (!h) throw_invalid("sp_device_graph_download: null graph");
        cudaStream_t s = ctx->stream;
        const DevGraph& g = h->g;
        const bool whole = !ctx->comm.active();
        if (!whole && !h->ingested) throw_invalid("sp_device_graph_download: row-block graph");
        const int64_t* offs = whole ? g.offs.p : h->full_offs.p;
        const int32_t* cols = whole ? g.cols.p : h->full_cols.p;
        if (whole && g.row0 != 0) throw_invalid("sp_device_graph_download: row-block graph");
        if (offsets_out)
            SPB_CUDA(cudaMemcpyAsync(offsets_out, offs, sizeof(int64_t) * (g.n_global + 1), cudaMemcpyDeviceToHost, s));
        if (cols_out && g.nnz_global)
            SPB_CUDA(cudaMemcpyAsync(cols_out, cols, sizeof(int32_t) * g.nnz_global, cudaMemcpyDeviceToHost, s));
        if (old_ids_out) {
            if (!h->ingested) throw_invalid("sp_device_graph_download: old ids exist for ingested graphs only");
            SPB_CUDA(cudaMemcpyAsync(old_ids_out, h->old_ids.p, sizeof(int64_t) * g.n_global,
                                     cudaMemcpyDeviceToHost, s));
        }
        SPB_CUDA(cudaStreamSynchronize(s));
    });
}

sp_status sp_classify(sp_context* ctx, const sp_graph* hg, sp_graph_info* info) {
    return guarded(ctx, [&] {
        if (!info) throw_invalid("sp_classify: null info");
        if (!hg || hg->n == 0) throw_invalid("classify: empty graph");
        DevGraph g;
        copy_graph(ctx, hg, g);
        fill_info(ctx, g, info);
    });
}

} // extern "C"
