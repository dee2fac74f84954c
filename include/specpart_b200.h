/*
 * specpart_b200.h — C ABI of the B200-native spectral partitioning hot path.
 *
 * Drop-in boundary for the reference API
 *     RunResult specpart::partition_graph(const Graph&, const RunConfig&)
 *     (/root/reference/proj/include/specpart/pipeline.hpp:106, src/pipeline.cpp:47-167)
 * plus kernel-level entry points that mirror the reference's internal seams so
 * parity can be checked stage by stage:
 *     build_combinatorial / build_normalized / build_degree  (src/laplacian.cpp:53-144)
 *     kernels::spmv_block                                    (src/kernels.cpp:36-62)
 *     kernels::gram                                          (src/kernels.cpp:79-110)
 *     lobpcg                                                 (src/eigensolver.cpp:177-337)
 *     polynomial_build + GmresPolyPreconditioner::apply      (src/preconditioners.cpp:171-193, 315-382)
 *     mj_partition                                           (src/partitioner.cpp:140-170)
 *     make_partition / cutsize / imbalance                   (src/graph.cpp:184-230)
 *
 * Conventions: plain C types only. All array arguments are HOST pointers owned
 * by the caller and read (inputs) or written (outputs) during the call only.
 * Dense blocks cross the boundary column-major (the reference's Dense layout,
 * dense.hpp:10-39); the library keeps them row-major on the device.
 * Every entry point is blocking and returns an sp_status; the message of the
 * last failure on a context is available from sp_last_error().
 */
#ifndef SPECPART_B200_H
#define SPECPART_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: the reference's exception types (include/specpart/errors.hpp) --- */
typedef int32_t sp_status;
enum {
    SP_OK = 0,
    SP_ERROR = 1,        /* any other std::exception (CLI exit 1, tools/specpart.cpp:347) */
    SP_PARSE = 2,        /* ParseError            errors.hpp:10-19  (not produced by this path) */
    SP_BREAKDOWN = 3,    /* BreakdownError        errors.hpp:23-36 */
    SP_INFEASIBLE = 4,   /* InfeasibleError       errors.hpp:39-42 */
    SP_DEGENERATE = 5,   /* DegenerateDegreeError errors.hpp:45-48 */
    SP_DIMENSION = 6,    /* DimensionError        errors.hpp:51-54 */
    SP_INVALID = 7,      /* std::invalid_argument (graph.cpp:210-224, laplacian.cpp:54) */
    SP_CUDA = 8,         /* CUDA runtime failure (new) */
    SP_NCCL = 9          /* NCCL failure (new) */
};

/* ---- enums: numeric values follow the reference's enum order (pipeline.hpp:16-18,
 *      laplacian.hpp:40) so a C++ shim can static_cast between them. ---- */
enum { SP_PROBLEM_AUTO = 0, SP_PROBLEM_COMBINATORIAL = 1, SP_PROBLEM_GENERALIZED = 2,
       SP_PROBLEM_NORMALIZED = 3 };
enum { SP_PRECOND_AUTO = 0, SP_PRECOND_JACOBI = 1, SP_PRECOND_POLYNOMIAL = 2,
       SP_PRECOND_AMG = 3, SP_PRECOND_NONE = 4 };
enum { SP_INIT_AUTO = 0, SP_INIT_RANDOM = 1, SP_INIT_PIECEWISE = 2 };
/* operator kinds for sp_build_laplacian / sp_spmm (laplacian.hpp:24-33) */
enum { SP_LAP_COMBINATORIAL = 0, SP_LAP_NORMALIZED = 1, SP_LAP_DEGREE = 2 };

/* report warnings bitmask (pipeline.cpp:140-148, 161-163) */
enum { SP_WARN_BREAKDOWN_RECOVERED = 1, SP_WARN_UNCONVERGED = 2, SP_WARN_IMBALANCE = 4,
       SP_WARN_AMG_STAGNATED = 8 /* pipeline.cpp:116-117 */ };

#define SP_MAX_EIG 64
#define SP_MAX_AMG_LEVELS 20

/* Graph (graph.hpp:17-32): symmetric CSR adjacency without stored self-loops,
 * column indices strictly increasing per row. values == NULL means unit edge
 * costs, vertex_weights == NULL means unit vertex weights (the CLI's
 * symmetrize() output, graph.cpp:44-64). */
typedef struct sp_graph {
    int64_t n;
    const int64_t* row_offsets;   /* n+1 */
    const int32_t* col_indices;   /* row_offsets[n] */
    const double* values;         /* row_offsets[n] or NULL */
    const double* vertex_weights; /* n or NULL */
} sp_graph;

/* RunConfig (pipeline.hpp:20-31). tol <= 0 means "pick by graph kind" (nullopt). */
typedef struct sp_config {
    int64_t num_parts;
    int32_t problem;      /* SP_PROBLEM_* */
    int32_t precond;      /* SP_PRECOND_* */
    double tol;
    int32_t max_iters;
    int32_t init;         /* SP_INIT_* */
    uint64_t seed;
    double epsilon;
    int32_t doubled_cut;
    int32_t record_trace;
} sp_config;

/* TraceRecord (eigensolver.hpp:21-26) */
typedef struct sp_trace_record {
    int32_t iter;
    int32_t ntheta;
    double min_residual;
    double max_residual;
    double theta[SP_MAX_EIG];
} sp_trace_record;

/* RunReport (pipeline.hpp:53-86) with fixed-size arrays; caller-provided
 * buffers for the variable-length parts. */
typedef struct sp_report {
    /* graph */
    int64_t n;
    int64_t edges;
    int32_t graph_regular;     /* 1 = Regularity::Regular */
    int32_t pad0;
    int64_t max_degree;
    double avg_degree;
    double degree_ratio;
    /* resolved configuration (ResolvedConfig, pipeline.hpp:33-39) */
    int64_t num_parts;
    int32_t problem;           /* SP_PROBLEM_* (never AUTO) */
    int32_t precond;           /* SP_PRECOND_* (never AUTO) */
    double tol;
    int32_t init;              /* SP_INIT_* (never AUTO) */
    int32_t eigenvectors;      /* d */
    uint64_t seed;
    int32_t max_iters;
    int32_t doubled_cut;
    double epsilon;
    /* solver */
    int32_t iterations;
    int32_t breakdown_retries;
    double theta[SP_MAX_EIG];
    double residual_norms[SP_MAX_EIG];
    uint8_t converged[SP_MAX_EIG];
    int32_t poly_degree;       /* achieved GMRES-polynomial degree, 0 if not used */
    int32_t warnings;          /* SP_WARN_* bitmask */
    /* StageTimes (pipeline.hpp:41-46), seconds, same boundary as the reference */
    double laplacian_s;
    double eigensolve_s;
    double partition_s;
    double total_s;
    /* partition quality */
    double cutsize;
    double imbalance;
    /* device-side accounting (new): SpMM launches, algorithmic bytes, device ms */
    int64_t spmm_launches;
    double spmm_bytes;
    double spmm_ms;
    int32_t kernel_launches;
    int32_t n_gpus;
    /* the GMRES-polynomial step SpMM (the dominant kernel with precond=polynomial) */
    int64_t poly_launches;
    double poly_bytes;
    double poly_ms;
    /* multi-GPU halo exchanges before SpMMs (count, bytes sent, device ms incl. peer waits) */
    int64_t halo_launches;
    double halo_bytes;
    double halo_ms;
    /* spmm_bytes / poly_bytes count each operator in its own stored format (pattern ELL:
     * 1 B/row); these count the same launches as pattern CSR (4 B/nnz + offsets) */
    double spmm_eff_bytes;
    double poly_eff_bytes;
    /* caller-provided outputs (may be NULL) */
    double* part_weights;          /* num_parts */
    sp_trace_record* trace;        /* trace_capacity records */
    int32_t trace_capacity;
    int32_t trace_len;
    /* the eigenvectors the partition was computed from (EigenResult::X,
     * eigensolver.hpp:28-35): n x d column-major, B-orthonormal; column 0 is the
     * one embed() drops (partitioner.cpp:19-25). NULL = not wanted. */
    double* eigenvectors_out;
    /* RunReport::amg_levels (pipeline.hpp:48-51, 74): rows and stored entries per
     * level of the AMG hierarchy, 0 levels when AMG did not run */
    int32_t amg_levels;
    int32_t pad1;
    int64_t amg_n[SP_MAX_AMG_LEVELS];
    int64_t amg_nnz[SP_MAX_AMG_LEVELS];
    /* SpMM launches that ran the structured-mesh TMA stencil kernel (one GPU or z-slab) */
    int64_t mesh_launches;
} sp_report;

typedef struct sp_context sp_context;

/* ---- context ------------------------------------------------------------- */
/* One context per GPU. Owns device memory, streams and (for world > 1) the NCCL
 * communicator. One call in flight per context. */
sp_status sp_context_create(int device, sp_context** out);
/* Multi-GPU: one process per GPU, all ranks call this with the same 128-byte
 * unique id produced by sp_nccl_unique_id() on rank 0. */
sp_status sp_nccl_unique_id(void* out128);
sp_status sp_context_create_dist(int device, int rank, int world, const void* nccl_id128,
                                 sp_context** out);
void sp_context_destroy(sp_context* ctx);
const char* sp_last_error(const sp_context* ctx);
int sp_version(void);
/* Memory-safety check (debug): with SPECPART_B200_GUARD=1 in the environment of the
 * process, every device buffer carries guard bands that are verified when it is
 * released; this also verifies every live buffer now. *violations = bytes found
 * overwritten so far (0 = clean), *buffers = buffers checked so far; both -1 when the
 * process does not run in guard mode. */
sp_status sp_debug_guard_check(int64_t* violations, int64_t* buffers);
/* Record CUDA events around every SpMM launch (report.spmm_ms); off by default. */
sp_status sp_context_set_timing(sp_context* ctx, int on);
/* LOBPCG with the AX/AH/AP recurrence: one SpMM per iteration
 * on the new preconditioned block instead of the reference's A*S and A*X
 * (eigensolver.cpp:138-155, 210-222), with A*X recomputed exactly whenever the
 * recurrence reports convergence and every 10 iterations. Off by default (the
 * reference's algorithm); applies to sp_partition* and sp_lobpcg on this context. */
sp_status sp_context_set_recurrence(sp_context* ctx, int on);
/* Irregular graphs (classify) on one GPU: run the eigensolver on a degree-descending
 * relabel of the vertices (hub rows of every block stay L2-resident for the SpMM
 * gathers); the initial block and the eigenvectors are permuted in and out, so the
 * multi-jagged stage and the metrics see the caller's numbering. On by default. */
sp_status sp_context_set_relabel(sp_context* ctx, int on);

/* ---- end to end (pipeline.cpp:47-167) --------------------------------------
 * assignment_out: n int32 part ids in [0, K). x0_colmajor: optional n x d
 * initial block (d = floor(log2 K) + 1 = report->eigenvectors, n*d doubles)
 * replacing the init selection (the CLI's --init-file warm start,
 * tools/specpart.cpp:94-157); pass NULL for the reference behaviour.
 * With world > 1 every rank passes the same full graph; every rank receives
 * the full assignment. */
sp_status sp_partition(sp_context* ctx, const sp_graph* g, const sp_config* cfg,
                       int32_t* assignment_out, sp_report* report, const double* x0_colmajor);

/* ---- device-resident graphs ------------------------------------------------
 * sp_graph_upload copies the graph arrays into HBM (no computation);
 * sp_partition_resident then runs the whole pipeline of sp_partition on them
 * (degree scan and assembly included) and leaves the assignment in HBM,
 * optionally copying it to assignment_out (host, may be NULL). */
typedef struct sp_device_graph sp_device_graph;
sp_status sp_graph_upload(sp_context* ctx, const sp_graph* g, sp_device_graph** out);
/* Releases a device graph; call it before sp_context_destroy of the context that made it. */
void sp_graph_free(sp_device_graph* dg);
sp_status sp_partition_resident(sp_context* ctx, sp_device_graph* dg, const sp_config* cfg,
                                int32_t* assignment_out, sp_report* report, const double* x0_colmajor);

/* ---- ingestion (graph.cpp:44-182; what tools/specpart.cpp:89-104 runs before
 *      partition_graph) ------------------------------------------------------- */

/* GraphKind (graph.hpp:35-41) plus sizes. nnz counts stored entries (2 x edges). */
typedef struct sp_graph_info {
    int64_t n;
    int64_t nnz;
    int64_t n_symmetrized;    /* ingested graphs: before the component cut */
    int64_t nnz_symmetrized;
    int64_t max_degree;
    double avg_degree;
    double degree_ratio;
    int32_t regular;          /* 1 = Regularity::Regular (ratio <= 10) */
    int32_t pad;
} sp_graph_info;

/* symmetrize (graph.cpp:44-64: pattern of A + A^T, diagonal dropped, rows
 * sorted, unit costs and weights) of the square n x n pattern (values are
 * ignored, as in the reference) and, with lcc != 0, largest_connected_component
 * (graph.cpp:118-171: ties go to the component holding the smallest vertex id;
 * vertices keep their relative order). Runs on the device; the result stays in
 * HBM as a device graph ready for sp_partition_resident. Replaces
 *     Graph symmetrize(const SparseMatrix&)                          graph.hpp:53
 *     std::pair<Graph, std::vector<int64_t>> largest_connected_component(const Graph&)  graph.hpp:62
 * Errors: SP_INVALID for n == 0 or a column index outside [0, n). */
sp_status sp_ingest(sp_context* ctx, int64_t n, const int64_t* row_offsets, const int32_t* col_indices,
                    int32_t lcc, sp_device_graph** out);
/* Sizes and classify (graph.hpp:65, graph.cpp:173-182) of a device graph. */
sp_status sp_device_graph_info(sp_context* ctx, sp_device_graph* dg, sp_graph_info* info);
/* Copies a device graph to host buffers (n+1 offsets, nnz columns; any may be
 * NULL); old_ids_out (n int64, the LCC's old_ids) only for ingested graphs. */
sp_status sp_device_graph_download(sp_context* ctx, sp_device_graph* dg, int64_t* offsets_out,
                                   int32_t* cols_out, int64_t* old_ids_out);
/* classify (graph.cpp:173-182) of a host graph. Errors: SP_INVALID for n == 0. */
sp_status sp_classify(sp_context* ctx, const sp_graph* g, sp_graph_info* info);

/* ---- kernel-level entry points (parity seams) ------------------------------ */

/* Laplacian assembly (laplacian.cpp:53-144): writes the CSR of L (offsets n+1,
 * cols/vals nnz_L = nnz_A + n; for SP_LAP_DEGREE nnz = n), diag[n] and the
 * Gershgorin bound (min(bound, 2) for normalized). Bit-exact. */
sp_status sp_build_laplacian(sp_context* ctx, int32_t kind, const sp_graph* g,
                             int64_t* offsets_out, int32_t* cols_out, double* vals_out,
                             double* diag_out, double* bound_out, int32_t* is_diagonal_out);

/* Y = L * X with L assembled from g (kind as above). X, Y are n x m column-major. */
sp_status sp_spmm(sp_context* ctx, int32_t kind, const sp_graph* g, const double* X, int32_t m,
                  double* Y);

/* Y = L * X through the kernels the eigensolver runs on this graph (kind 0
 * combinatorial or 1 normalized): on irregular graphs (classify) the
 * row-length-binned kernels with chunked long rows, whose sums are
 * deterministic but not in storage order (compare within
 * |y - y_ref| <= c * eps * sum_k |a_ik x_k|); on meshes the same kernels as
 * sp_spmm (bit-exact). */
sp_status sp_spmm_solver(sp_context* ctx, int32_t kind, const sp_graph* g, const double* X, int32_t m,
                         double* Y);

/* Y = A * X for an explicit CSR operator (spmv_block, kernels.cpp:36-62). */
sp_status sp_spmm_csr(sp_context* ctx, int64_t nrows, int64_t ncols, const int64_t* offsets,
                      const int32_t* cols, const double* vals, const double* X, int32_t m,
                      double* Y);

/* G = U^T diag(b) V (kernels::gram, kernels.cpp:79-110; b == NULL means identity).
 * U: n x mu, V: n x mv column-major; G: mu x mv column-major. Deterministic. */
/* Diagnostics: times the tall-skinny block kernel (Gram / block update /
 * block combine, blockops.cu) on device-resident column-major blocks of n rows
 * filled with uniform(-1,1) data: mu columns of U, mv of V; transform 0 none,
 * 1 W = V - U C, 2 W = V C (C: mv x mw); gram 0 none, 1 [U V]^T V-or-W, 2
 * U^T V-or-W, 3 (V-or-W)^T (V-or-W). Writes the mean device ms per call over
 * iters calls (after one warm-up) to ms_out. */
sp_status sp_bench_blockop(sp_context* ctx, int64_t n, int32_t mu, int32_t mv, int32_t mw, int32_t transform,
                           int32_t gram, int32_t iters, double* ms_out);
sp_status sp_gram(sp_context* ctx, int64_t n, const double* U, int32_t mu, const double* V,
                  int32_t mv, const double* b, double* G);

/* kernels::mult / kernels::mult_sub (kernels.cpp:127-157, kernels.hpp:24-28): op 0 computes
 * Y = X C, op 1 computes Y -= X C, X n x k, C k x m, Y n x m, all column-major (Y is read for
 * op 1). The block product of LOBPCG's Rayleigh-Ritz combine and CGS projection: the TS
 * kernel's COMBINE / UPDATE transforms (fp64 DMMA, fixed summation order, so repeated calls
 * agree bit for bit; agreement with the reference's k-ordered loop is to rounding). k, m <= 64. */
sp_status sp_block_combine(sp_context* ctx, int64_t n, const double* X, int32_t k, const double* C,
                           int32_t m, int32_t op, double* Y);

/* Initial blocks (eigensolver.cpp:20-51), n x d column-major, bit-identical. */
sp_status sp_initial_guess(sp_context* ctx, int32_t init, int64_t n, int32_t d, uint64_t seed,
                           double* X_out);

/* Rows [row0, row0 + nloc) of the same n x d block (nloc x d column-major):
 * the slice a rank of a row-partitioned run generates for itself (the
 * mt19937_64 stream is jumped ahead to the slice, rng.cu). */
sp_status sp_initial_guess_rows(sp_context* ctx, int32_t init, int64_t n, int32_t d, uint64_t seed,
                                int64_t row0, int64_t nloc, double* X_out);

/* LOBPCG (eigensolver.cpp:177-337) on the problem built from g. precond is
 * SP_PRECOND_JACOBI, SP_PRECOND_POLYNOMIAL (poly_seed feeds PolyConfig.seed),
 * SP_PRECOND_AMG (poly_seed feeds AmgConfig.seed; regular/irregular preset by
 * classify(g)) or SP_PRECOND_NONE. X0 n x nev column-major. Outputs theta[nev], X n x nev,
 * residual norms, converged flags, iteration count, retries. */
sp_status sp_lobpcg(sp_context* ctx, const sp_graph* g, int32_t problem, int32_t precond,
                    uint64_t poly_seed, int32_t poly_degree, const double* X0, int32_t nev,
                    double tol, int32_t max_iters, int32_t locking, double* theta_out,
                    double* X_out, double* residuals_out, uint8_t* converged_out,
                    int32_t* iterations_out, int32_t* retries_out);

/* GMRES polynomial preconditioner (preconditioners.cpp:315-382) built on the
 * operator of kind `kind` from g, then applied to R (n x m column-major). Also
 * returns the Leja-ordered roots (capacity degree). */
sp_status sp_poly_apply(sp_context* ctx, int32_t kind, const sp_graph* g, uint64_t seed,
                        int32_t degree, const double* R, int32_t m, double* H_out,
                        double* roots_out, int32_t* achieved_out);

/* Jacobi (jacobi_build), the GMRES polynomial (polynomial_build: seed, degree;
 * roots_out/achieved_out as sp_poly_apply) or none, built on an explicit n x n
 * CSR operator (make_operator, laplacian.cpp:40-51, Gershgorin bound included)
 * and applied to R: the diagonal-operator KATs of preconditioner_test.cpp:38-118
 * and acceptance c12 (acceptance.cpp:361-403). */
sp_status sp_precond_apply_csr(sp_context* ctx, int64_t n, const int64_t* offsets, const int32_t* cols,
                               const double* vals, int32_t precond, uint64_t seed, int32_t degree, const double* R,
                               int32_t m, double* H_out, double* roots_out, int32_t* achieved_out);

/* H = M R for any preconditioner of the pipeline (Preconditioner::apply,
 * preconditioners.hpp:16-27) built on the operator of kind 0 (L_C) or 1 (L_N)
 * from g: SP_PRECOND_JACOBI, _POLYNOMIAL (seed, degree as PolyConfig), _AMG
 * (seed as AmgConfig.seed, preset by classify(g)), _NONE (H = R). */
sp_status sp_precond_apply(sp_context* ctx, int32_t kind, const sp_graph* g, int32_t precond, uint64_t seed,
                           int32_t degree, const double* R, int32_t m, double* H_out);

/* Multi-jagged partitioning (partitioner.cpp:140-170) of n points with `dims`
 * coordinates (n x dims column-major), positive weights (NULL = unit). */
sp_status sp_mj_partition(sp_context* ctx, int64_t n, int32_t dims, const double* coords,
                          const double* weights, int64_t num_parts, int32_t* assignment_out,
                          double* part_weights_out, double* imbalance_out);

/* cutsize (graph.cpp:184-196): cost of the edges whose endpoints have different
 * ids, each undirected edge once (twice with doubled); ids are not validated. */
sp_status sp_cutsize(sp_context* ctx, const sp_graph* g, const int32_t* assignment, int32_t doubled,
                     double* cut_out);

/* make_partition (graph.cpp:209-230): validates, tallies part weights, cut, imbalance. */
sp_status sp_cut_imbalance(sp_context* ctx, const sp_graph* g, const int32_t* assignment,
                           int64_t num_parts, int32_t doubled, double* cut_out,
                           double* imbalance_out, double* part_weights_out);

#ifdef __cplusplus
}
#endif

#endif /* SPECPART_B200_H */
