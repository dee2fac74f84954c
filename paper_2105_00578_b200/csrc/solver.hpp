// solver.hpp — device LOBPCG with Jacobi / GMRES-polynomial preconditioning.
#pragma once

#include "context.hpp"
#include "amg.hpp"
#include "dense_host.hpp"

#include <memory>

#include <algorithm>
#include <vector>

namespace spb {

enum PrecKind { PREC_NONE = 0, PREC_JACOBI = 1, PREC_POLY = 2, PREC_AMG = 3 };

struct TraceRec {
    int iter = 0;
    double min_residual = 0.0, max_residual = 0.0;
    std::vector<double> theta;
};

struct SolveOpts {
    int nev = 1;
    double tol = 1e-4;
    int max_iters = 1000;
    bool locking = true;
    bool record_trace = false;
};

struct SolveResult {
    std::vector<double> theta;
    std::vector<double> residual_norms;
    std::vector<uint8_t> converged;
    int iterations = 0;
    int retries = 0;
    std::vector<TraceRec> trace;
    int slow_orth = 0;      // blocks that needed the exact column-wise path
    int cholqr_fixups = 0;  // second CholQR passes
    bool all_converged() const {
        for (uint8_t c : converged)
            if (!c) return false;
        return !converged.empty();
    }
};

class Solver {
public:
    // A: problem operator (local row block); bdiag: B = D diagonal (generalized) or null.
    Solver(sp_context* ctx, const DevOp& A, const double* bdiag, int max_cols);

    void set_jacobi(const double* inv_diag_dev) { prec_ = PREC_JACOBI; inv_diag_ = inv_diag_dev; }
    void set_none() { prec_ = PREC_NONE; }
    // AX/AH/AP recurrence: A is applied to the new H block only;
    // A*S, A*X and A*P follow the same small-matrix transforms as S, X and P, the
    // residual R = AX - BX diag(theta) needs no SpMM, and A*X is recomputed exactly
    // every kTrueResidualEvery iterations and whenever the recurrence says converged.
    // Off by default (the reference recomputes A*S and A*X every iteration,
    // eigensolver.cpp:138-155, 210-222).
    void set_recurrence(bool on) { recur_ = on; }
    // amg_build (preconditioners.cpp:722-728) on the explicit fine operator A0 (moved in)
    void build_amg(CsrDev&& A0, DBuf<double>&& diag0, const AmgCfg& cfg);
    const Amg* amg() const { return amg_.get(); }
    // polynomial_build (preconditioners.cpp:315-382): seeded Arnoldi -> harmonic
    // Ritz roots in Leja order. Throws on degree < 1.
    void build_poly(uint64_t seed, int degree);
    const std::vector<double>& roots() const { return roots_; }

    // H = M(R) on the local block (n_loc x k views).
    void apply_precond(const View& R, int k, const View& H);

    // lobpcg (eigensolver.cpp:177-337). X0/X: local n_loc x nev row-major views.
    SolveResult lobpcg(const View& X0, const SolveOpts& o, const View& X);

    // Y = A X (local rows, X local block) — exposed for the kernel-level ABI.
    void spmm_poly2(const View& X, int m, EpiArgs& ea);
    void spmm_store(const View& X, int m, const View& Y);

    // Block layout used by this solver: column-major (ld = padded rows) for
    // short-row operators (meshes: row-per-lane SpMM), row-major otherwise.
    bool colmajor_blocks() const { return colmajor_; }
    int64_t ld() const { return ld_; }
    // (padding row-major rows to 32-byte sectors was measured slower on cfg3: 287 vs 247 ms)
    View block(double* p, int cols) const { return colmajor_ ? colmajor(p, ld_, cols) : rowmajor(p, cols, cols); }
    // A block that can be an SpMM input (symmetric heap on multi-GPU P2P runs;
    // otherwise allocated into `fallback`). Collective in the multi-GPU case.
    double* input_block(int cols, DBuf<double>& fallback);
    size_t block_elems(int cols) const { return static_cast<size_t>(colmajor_ ? ld_ : rows_cap_) * cols; }

private:
    struct Orth {
        int kept = 0;
        std::vector<int> kept_idx;
    };
    // With AV (= A V), Aagainst and Adst (recurrence), every transform of V into dst is
    // applied to AV into Adst as well, so Adst = A dst on return.
    Orth b_orth(const View& V, int k, const View& against, int a, const View& dst, SolveResult& st,
                const View* AV = nullptr, const View* Aagainst = nullptr, const View* Adst = nullptr);
    void ts_mirror(const TsSpec& spec);  // a transform of a TsSpec without its Gram (recurrence side)
    void residuals_from(const View& X, const View& AX, const std::vector<double>& theta, SolveResult& r,
                        double thr);
    Orth b_orth_slow(const View& src, int k, const View& against, int a, const View& dst,
                     const std::vector<double>& orig, SolveResult& st);
    // gram helpers: run ts, all-reduce over ranks, copy to host (col-major)
    std::vector<double> gram_to_host(const TsSpec& spec, int& P, int& Q);
    void gram_dev(const TsSpec& spec, int& P, int& Q);  // result in gram_.p
    void spmm(const View& Xlocal, int m, EpiArgs& ea);
    void residuals(const View& X, const std::vector<double>& theta, SolveResult& r, double thr);
    void upload(const std::vector<double>& h, DBuf<double>& d);

    sp_context* ctx_;
    cudaStream_t s_;
    DevOp A_;
    const double* bdiag_;
    int64_t n_;       // local rows
    int max_cols_;
    bool colmajor_ = false;
    bool halo_ = false;     // multi-GPU: inputs get their halo rows before each SpMM
    bool sym_ = false;      // SpMM inputs live in the symmetric heap (P2P halo push)
    double *pR_ = nullptr, *pS_ = nullptr, *pW_ = nullptr, *pPA_ = nullptr, *pPB_ = nullptr;
    int64_t rows_cap_ = 1;  // own rows + halo rows
    // z-slab: copy plan of the two-plane halo of the two-step polynomial kernel
    std::vector<HaloPlan::CeSeg> ce2_;
    int64_t ld_ = 1;
    PrecKind prec_ = PREC_NONE;
    const double* inv_diag_ = nullptr;
    std::vector<double> roots_;
    std::unique_ptr<Amg> amg_;
    bool recur_ = false;
    double* pH_ = nullptr;      // H is an SpMM input (recurrence: A*H)
    DBuf<double> AX_, AP_, AH_;
    // column-major blocks: H and P side by side in one buffer ([H | P], P after H's
    // columns) so both are orthonormalized as one block (lobpcg); recurrence: [AH | AP]
    double* pHP_ = nullptr;
    DBuf<double> HP_, AHP_;

    DBuf<int32_t> ell_;  // fixed-slot ELL of A (meshes), see spmm_ell_kernel
    EllPatStore ellpat_; // its pattern-compressed form (ellpat.cu)
    DBuf<double> gram_, scratch_, cmat_, cmat2_, partial_, norms_;
    DBuf<double> R_, H_, P_, S_, AS_, prodA_, prodB_, work_;
};

// Host std::mt19937_64 initial blocks (eigensolver.cpp:20-51), local rows of the
// n x d column-major block written row-major to a device view.
void initial_block_random(int64_t n, int d, uint64_t seed, int64_t row0, int64_t nloc,
                          const View& X, cudaStream_t s);
void initial_block_piecewise(int64_t n, int d, int64_t row0, int64_t nloc, const View& X,
                             cudaStream_t s);
// Column sums of a local block (deterministic), result on device.
void colsum(int64_t n, const View& v, double* out_dev, double* scratch, cudaStream_t s);

} // namespace spb
