// ops.cuh — device operator representation and kernel launchers.
//
// The Laplacian operators of laplacian.cpp:53-144 are held on the device in one
// of four forms. All of them reproduce kernels::spmv_block (kernels.cpp:36-62)
// bit for bit: each output element is a sequential, FMA-free sum over the row of
// the explicit CSR of L, in storage order, with the diagonal term inserted at the
// position build_combinatorial/build_normalized place it (before the first
// column > i).
//   OP_EXPLICIT     : explicit CSR (int64 offsets, int32 cols, fp64 values).
//   OP_LAPLACE_UNIT : L_C of a unit-cost graph from the adjacency pattern alone:
//                     off-diagonals are -1 (exact), diagonal = degree. 4 B/nnz.
//   OP_NORMAL_UNIT  : L_N of a unit-cost graph from the pattern and
//                     isd = 1/sqrt(deg): off-diagonal (-isd_i)*isd_j (laplacian.cpp:114).
//   OP_DIAGONAL     : y = d .* x (build_degree / is_diagonal, kernels::diag_scale).
#pragma once

#include "common.cuh"

#include <climits>
#include "p2p.cuh"

namespace spb {

enum OpMode { OP_EXPLICIT = 0, OP_LAPLACE_UNIT = 1, OP_NORMAL_UNIT = 2, OP_DIAGONAL = 3 };

struct DevOp {
    int mode = OP_EXPLICIT;
    int64_t n = 0;              // local rows
    int64_t row0 = 0;           // global id of local row 0 (multi-GPU row block)
    int64_t nnz = 0;            // stored entries traversed by the kernel
    const int64_t* offs = nullptr;
    const int32_t* cols = nullptr;  // GLOBAL column ids (multi-GPU: index into the full vector)
    const double* vals = nullptr;
    const double* diag = nullptr;   // a_ii (degree for L_C, 1 for L_N, d for diagonal)
    const double* isd = nullptr;    // OP_NORMAL_UNIT: 1/sqrt(deg), indexed by global column
    // long-row bin (rows handled by the CTA-per-row kernel)
    const int32_t* long_rows = nullptr;
    int64_t n_long = 0;
    int64_t long_threshold = 1 << 30;
    int max_row = 1 << 30;      // max stored entries in a row (selects the tiled kernel when <= 32)
    // multi-GPU halo numbering: cols are local ids (own rows, then halo rows) and
    // dpos[i] is the storage slot of the diagonal (count of global cols < global i)
    const int32_t* dpos = nullptr;
    int64_t x_rows = 0;         // rows of the SpMM input block the columns address
    // irregular graphs in the solver (spmm_vec.cu): rows grouped by length into
    // bins 0..3 (<= 16, <= 64, <= 256, <= long threshold entries) and bin 4 (long rows)
    const int32_t* bin_rows = nullptr;
    int64_t bin_off[6] = {0, 0, 0, 0, 0, 0};
    // long rows in chunks (one CTA each) and their per-chunk column partials
    int64_t long_nchunks = 0;
    const int64_t* long_row_chunk0 = nullptr;  // n_long + 1
    const int32_t* long_chunk_row = nullptr;
    const int64_t* long_chunk_k0 = nullptr;
    double* long_part = nullptr;               // nchunks x 32
    // fixed-slot ELL of a mesh Laplacian (spmm_ell_kernel), built by the solver;
    // slot s of row i at ell[s*ell_ld + i]; padding slots hold ell_zero_row
    const int32_t* ell = nullptr;
    int ell_kl = 0, ell_ku = 0;
    int64_t ell_ld = 0;
    int64_t ell_zero_row = 0;
    // pattern-compressed form (structured meshes): row i's slots are
    // i + ell_pat_tab[pid*W + s] (kEllPad = zero row), its diagonal ell_pat_deg[pid],
    // pid = ell_pat[i]; at most 256 distinct row patterns
    const uint8_t* ell_pat = nullptr;
    const int32_t* ell_pat_tab = nullptr;
    const double* ell_pat_deg = nullptr;
    int ell_npat = 0;
    // structured mesh (spmm_mesh.cu): row (z*ny + y)*nx + x has exactly the in-bounds
    // points of its 5/7/27-point stencil (mesh_plan); 0 = not recognised
    int mesh_nx = 0, mesh_ny = 0, mesh_nz = 0;
    // multi-GPU z-slab of a structured mesh (mesh_plan_slab): the rank's rows are planes
    // [mesh_z0, mesh_z0 + mesh_nz) of mesh_nzg; its neighbours' boundary planes sit in the
    // halo rows of the input block at mesh_halo_lo / mesh_halo_hi (-1: no such neighbour)
    int mesh_z0 = 0, mesh_nzg = 0, mesh_box27 = 0;
    int64_t mesh_halo_lo = -1, mesh_halo_hi = -1;
    // two-plane halo of the two-step polynomial kernel: planes z0-2, z0-1 then z1, z1+1
    // (4 planes) from this row of the input block; -1: not set up (Solver)
    int64_t mesh_halo2 = -1;
    double bound = 0.0;
    bool is_diagonal = false;
};

// Epilogues fused into the SpMM.
enum EpiMode { EPI_STORE = 0, EPI_RESIDUAL = 1, EPI_POLY = 2 };

constexpr int kMaxCols = 64;

struct EpiArgs {
    int mode = EPI_STORE;
    View Y;                 // STORE: output; RESIDUAL: R; POLY: prod_{i+1}
    // RESIDUAL: R = A X - theta .* (B X); per-CTA partial sums of R^2 per column
    const double* bdiag = nullptr;
    double theta[kMaxCols];
    double* partial = nullptr;   // [grid_main + n_long] x m
    // POLY: prod_{i+1} = prod_i - inv_cur * A prod_i; H = (first ? inv_cur*prod_i : H) + inv_next*prod_{i+1}
    View H;
    double inv_cur = 0.0;
    double inv_next = 0.0;
    int first = 0;
    int h_terms = 1;         // 0: H untouched, 1: H += inv_next*p_{i+1}, 2: also inv_cur*p_i first
    // two steps in one pass (spmm_mesh_poly2_launch): p_{i+2} = p_{i+1} - inv_next * A p_{i+1};
    // H = (first ? inv_cur*p_i : H + inv_cur*p_i) + inv_next*p_{i+1} (+ inv_after*p_{i+2} when last)
    double inv_after = 0.0;
    int last = 0;
};

// Y-block SpMM with epilogue. X is the gathered block (rows = global columns of
// A; on one GPU the same n), m columns. Returns the number of partial rows
// written to ea.partial (for RESIDUAL), so the caller can reduce them.
// hf: multi-GPU halo exchange fused into the kernel (column-major short-row path only)
int spmm_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s,
                const HaloFuse* hf = nullptr);
// true when spmm_launch uses the column-major row-per-lane kernel for these arguments
bool spmm_col_path(const DevOp& op, const View& X, int m, const EpiArgs& ea);
// Builds the fixed-slot ELL of a LAPLACE_UNIT operator (spmm.cu); returns false
// (op unchanged) when the rows are too wide. Padding slots point at zero_row.
bool build_ell(DevOp& op, int64_t zero_row, DBuf<int32_t>& store, cudaStream_t s);
constexpr int32_t kEllPad = INT32_MIN;
// Pattern-compresses the ELL of a unit-cost Laplacian (ellpat.cu): succeeds when the
// rows have at most 256 distinct (column - row) slot vectors and every diagonal
// equals its row's neighbour count; the ELL stays as built otherwise.
struct EllPatStore {
    DBuf<uint8_t> pid;
    DBuf<int32_t> tab;
    DBuf<double> deg;
};
bool build_ell_patterns(DevOp& op, EllPatStore& st, cudaStream_t s);
// Structured-mesh SpMM (spmm_mesh.cu): mesh_plan recognises a naturally ordered
// 5/7/27-point box mesh behind a pattern-compressed ELL (false: op unchanged).
bool mesh_plan(DevOp& op, cudaStream_t s);
bool no_mesh_kernel();  // SPB_MESH=0: A/B diagnostics (ELL kernels on meshes)
// Multi-GPU: on the rank's rows before localization (global column ids), recognises a
// 3-D box mesh whose row block is whole z planes (sets the mesh_* fields, false: unchanged).
bool mesh_plan_slab(DevOp& op, int64_t n_global, cudaStream_t s);
bool spmm_mesh_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea);
// Two polynomial steps (i even, then i + 1) in one z-marching pass on a one-GPU 5/7-point
// mesh: p_{i+1} stays in shared memory (computed on the tile plus a one-point ring), only
// p_i is read and p_{i+2} written; same arithmetic, hence bit-identical to two steps.
bool spmm_mesh_poly2_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea);
int spmm_mesh_poly2_launch(const DevOp& op, const View& X, int m, const EpiArgs& ea, cudaStream_t s,
                           const HaloFuse* hf = nullptr);
// hf: the copy-engine halo of a z-slab (nopush): the producer waits for the peers'
// flags before it loads a halo plane
int spmm_mesh_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s,
                     const HaloFuse* hf = nullptr);
// Row-length bins for the vector SpMM (spmm_vec.cu); also sets the long-row list.
struct RowBins {
    DBuf<int32_t> rows;
    DBuf<int64_t> row_chunk0, chunk_k0;
    DBuf<int32_t> chunk_row;
    DBuf<double> part;
};
void build_row_bins(DevOp& op, int64_t long_thr, RowBins& st, cudaStream_t s);
bool spmm_vec_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea);
int spmm_vec_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s);
// Reduce partial[rows x m] over rows in fixed order into out[m] (device).
void reduce_partials(const double* partial, int rows, int m, double* out, cudaStream_t s);

// ---- tall-skinny block kernels (blockops.cu) ----
// Gram: G = [L0 | L1 | L2]^T diag(b) Rt, with optional pre-transforms:
//   UPDATE : W = V - [U0 | U1] * C   (C: (u0+u1) x k, column-major), Rt = W
//   COMBINE: W = V * C  (C: kv x kw column-major), W split across W/W2 views
struct TsSpec {
    int64_t n = 0;
    View U0, U1;            // basis ("against") views, cols may be 0
    View V;                 // input block
    View W, W2;             // outputs (W2 receives output columns >= W.cols for COMBINE)
    const double* C = nullptr;  // device, column-major
    int ldc = 0;                // leading dimension of C (0 = inner dimension)
    const double* b = nullptr;  // B diagonal (device) or null
    int transform = 0;      // 0 none, 1 update, 2 combine, 3 combine over [U | V]
    // gram request: left = [U0?][U1?][V or W?], right = V or W (post-transform)
    bool gram = false;
    bool gram_left_u = false;   // include U0, U1 on the left
    bool gram_left_self = true; // include the right block itself on the left
};
// TS_COMBINE_UV: W = [U0 | U1 | V] C (aligned column-major operands: the bulk kernel only)
enum { TS_NONE = 0, TS_UPDATE = 1, TS_COMBINE = 2, TS_COMBINE_UV = 3 };

// Runs the tile kernel; if spec.gram, writes the (P x Q) column-major Gram to
// gram_out (device) and returns P. Deterministic for a fixed n. The last element
// of scratch is a reduction counter: it must hold 0 (as unsigned) on the first
// call, and every call leaves it 0.
int ts_run(const TsSpec& spec, double* gram_out, double* scratch, size_t scratch_elems,
           cudaStream_t s);

// R = AX - theta .* (B X) (the SpMM RESIDUAL epilogue's arithmetic, eigensolver.cpp:212-218)
// from a tracked A X, with per-CTA partial sums of R^2 per column (fixed order); returns
// the number of partial rows (reduce with reduce_partials).
int residual_from_ax(int64_t n, const View& X, const View& AX, const double* bdiag, const double* theta_host,
                     int m, const View& R, double* partial, cudaStream_t s);

// Deterministic per-CTA column sums; returns the number of partial rows.
int colsum_partials(int64_t n, const View& v, double* scratch, cudaStream_t s);

// std::mt19937_64(seed) draws [0, n*d) as uniform(-1,1), column-major order;
// rows [row0, row0+nloc) written to out (rng.cu).
void mt_uniform_block(uint64_t seed, int64_t n, int d, int64_t row0, int64_t nloc, const View& out,
                      cudaStream_t s);

// Elementwise helpers
void scale_cols(View V, const double* colscale_dev, cudaStream_t s, int64_t n);  // V(:,j) *= s[j]
void diag_apply(int64_t n, const double* d, View in, View out, cudaStream_t s);    // out = d .* in
void copy_view(int64_t n, View in, View out, cudaStream_t s);
void gather_cols(int64_t n, View in, const int* cols_host, int k, View out, cudaStream_t s);
void fill_view(int64_t n, View v, double value, cudaStream_t s);
// out = inv_diag_guarded .* in (Jacobi, preconditioners.cpp:44-68)
void jacobi_apply(int64_t n, const double* inv_diag, View in, View out, cudaStream_t s);
void poly_first_only(int64_t n, double inv0, View R, View H, cudaStream_t s);  // H = inv0 * R

} // namespace spb
