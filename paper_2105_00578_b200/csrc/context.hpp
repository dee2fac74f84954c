// context.hpp — the opaque sp_context: device, streams, NCCL communicator,
// reusable scratch, device event timers.
#pragma once

#include "graph_dev.cuh"

#include "nccl_dyn.hpp"
#include "p2p.cuh"

#include <string>
#include <utility>
#include <vector>

namespace spb {

#define SPB_NCCL(call)                                                                   \
    do {                                                                                 \
        ncclResult_t _r = (call);                                                        \
        if (_r != ncclSuccess)                                                           \
            throw ::spb::SpError(9, std::string("NCCL: ") + ::spb::nccl().GetErrorString(_r) + " at " + \
                                        __FILE__ + ":" + std::to_string(__LINE__));      \
    } while (0)

// Halo exchange plan of one row-partitioned operator (built by localize_operator).
// Local numbering: own rows [0, nloc), then the halo rows [nloc, nloc+nhalo) in
// ascending global id (hence grouped by owner rank). Every SpMM input block has
// room for the halo rows after its own rows.
struct HaloPlan {
    bool on = false;
    int64_t nhalo = 0;
    int64_t total_send = 0;
    std::vector<int64_t> send_cnt, send_off, recv_cnt, recv_off;  // rows, per peer
    DBuf<int32_t> send_idx;  // local row ids sent, grouped by destination rank
    DBuf<double> sendbuf, recvbuf;
    // P2P push: per send entry, destination rank and row in that rank's block
    DBuf<int32_t> dst_peer, dst_row;
    uint32_t send_mask = 0, recv_mask = 0;
    bool vec2 = false;     // send entries pair up for 16-byte pushes (slab halos)
    // copy-engine halo (slab partitions): per destination, one contiguous run of
    // own rows -> one contiguous run of the peer's halo rows
    struct CeSeg {
        int peer;
        int64_t src_row, dst_row, rows;
    };
    std::vector<CeSeg> ce;
    bool ce_ok = false;
    int64_t max_rows = 0;  // max over ranks of nloc_pad + nhalo (common block height)
    int64_t halo_base = 0; // first halo row: nloc rounded up to 32 rows (own and halo rows never share a cache line)
    int64_t rot_tiles = 0, n_int_tiles = 0;  // fused SpMM tile order (p2p.cuh HaloFuse)
};

// Symmetric peer memory (symm.cu): cudaMalloc'd segments mapped into every
// rank of the box through CUDA IPC, carved by a bump allocator that runs the
// same sequence on every rank, so an offset names the same block everywhere.
// SpMM input blocks live here; the halo rows of a peer's copy are written
// directly over NVLink, and small sums are gathered into per-rank slots.
constexpr int kSumMax = 16384;  // doubles per rank slot of a P2P sum
struct SymSeg {
    char* base = nullptr;
    size_t size = 0;
    std::vector<char*> peer;  // mapped base of every rank's segment (own = base)
};
struct SymHeap {
    bool tried = false;
    bool on = false;
    std::vector<SymSeg> segs;
    size_t seg_i = 0, off = 0;  // bump position
    SymSeg ctrl;                // flags + sum slots
    cudaStream_t side = nullptr;            // copy-engine halo stream
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    void* write_value64 = nullptr;          // cuStreamWriteValue64 (driver entry point)
    uint64_t halo_epoch = 0, sum_epoch = 0, bar_epoch = 0;
    DBuf<int> counter;          // last-CTA ticket of the push kernel
    DBuf<int> err;              // device error word (peer wait timed out)
    const void* last_halo_src = nullptr;
};
// control segment layout (bytes)
constexpr size_t kFlHalo = 0, kFlSum = 256, kFlBar = 512, kSumSlots = 4096;
constexpr size_t kCtrlBytes = kSumSlots + 2 * kMaxPeers * kSumMax * sizeof(double);

// 1-D row partition over the ranks of one box: rank k owns global
// rows [k*n_pad, min(n, (k+1)*n_pad)), so a row-gathered block indexed by global
// id is exactly the NCCL all-gather of the equal-size (padded) rank slices.
struct Comm {
    int rank = 0;
    int world = 1;
    ncclComm_t nccl = nullptr;
    int64_t n_global = 0;
    int64_t n_pad = 0;
    DBuf<double> stage;    // n_pad x m contiguous send slice
    DBuf<double> full;     // world*n_pad x m gathered block
    DBuf<double> small;    // world x count for deterministic small sums
    int64_t bytes_moved = 0;
    HaloPlan halo;
    SymHeap sym;

    bool active() const { return world > 1; }
    void setup(int64_t n) {
        n_global = n;
        n_pad = (n + world - 1) / world;
    }
    int64_t row0() const { return static_cast<int64_t>(rank) * n_pad; }
    int64_t nloc() const {
        const int64_t r0 = row0();
        return r0 >= n_global ? 0 : std::min<int64_t>(n_pad, n_global - r0);
    }

    // Gathers the local n_loc x m block `local` into a row-major (world*n_pad) x m
    // block indexed by global row id. One GPU: returns `local` untouched.
    View gather_rows(const View& local, int m, cudaStream_t s);
    // Fills the halo rows [nloc, nloc+nhalo) of the m-column block X from their
    // owners: pack -> grouped ncclSend/ncclRecv -> unpack (halo.cu).
    void halo_exchange(const View& X, int m, cudaStream_t s);
    // Symmetric heap (collective calls: every rank, same order, same sizes).
    bool sym_init(cudaStream_t s);   // maps the control segment; false = NCCL paths
    void sym_reset() { sym.seg_i = 0; sym.off = 0; sym.last_halo_src = nullptr; }
    double* sym_alloc(size_t elems, cudaStream_t s);
    // byte distance from a local symmetric address to the same object on `peer`
    int64_t sym_delta(const void* p, int peer) const;
    void sym_check(cudaStream_t s);  // throws if a peer wait timed out
    void barrier_p2p(cudaStream_t s);
    // In-place deterministic sum over ranks of `count` doubles on the device:
    // all-gather then a fixed rank-order sum (bit-identical on every rank).
    void sum_small(double* dev, int count, cudaStream_t s);
    // Sum of int64 counters (exact).
    void sum_i64(int64_t* dev, int count, cudaStream_t s);
    // Max over ranks of a host double (Gershgorin bounds of row blocks).
    double max_f64(double v, cudaStream_t s);
    // Gathers int32 per-row values (n_loc each) into a global array (world*n_pad).
    void gather_i32(const int32_t* local, int32_t* global, cudaStream_t s);
    void gather_f64(const double* local, double* global, cudaStream_t s);
};

// Phase profiler (SPB_PROFILE=1): stream-synchronizes at every mark and
// accumulates host wall time per phase name; printed to stderr per partition.
struct PhaseProf {
    bool on = false;
    std::vector<std::pair<std::string, double>> acc;
    double last = 0.0;
    static double now();
    void start(cudaStream_t s);
    void mark(cudaStream_t s, const char* name);
    void dump(const char* title);
};

struct Timers {
    double spmm_ms = 0.0;
    int64_t spmm_launches = 0;
    int64_t mesh_launches = 0;
    double spmm_bytes = 0.0;
    int64_t kernel_launches = 0;
    double poly_ms = 0.0;
    int64_t halo_launches = 0;
    double halo_bytes = 0.0;
    double halo_ms = 0.0;
    int64_t poly_launches = 0;
    double poly_bytes = 0.0;
    // the same launches in pattern-CSR-equivalent bytes (4 B/nnz + offsets), "effective"
    double spmm_eff_bytes = 0.0;
    double poly_eff_bytes = 0.0;
};

// symm.cu: P2P fast paths; return false when not applicable (caller uses NCCL)
bool halo_push(Comm& cm, const View& X, int m, cudaStream_t s);
// Fills hf for an SpMM with the exchange fused in; false = not applicable.
bool halo_fuse_prepare(Comm& cm, const View& X, int m, HaloFuse& hf, cudaStream_t s);
// Copy-engine variant: the boundary rows go out as 2-D peer copies on a side
// stream, each followed by a stream-ordered flag write; hf is set to wait only.
// After launching the SpMM the caller must call halo_ce_finish (the main stream
// may not overwrite X before the copies have read it).
// segs: another copy plan over the same peers (the two-plane halo of the two-step
// polynomial kernel, Solver); default the halo plan's own
bool halo_ce_start(Comm& cm, const View& X, int m, HaloFuse& hf, cudaStream_t s,
                   const std::vector<HaloPlan::CeSeg>* segs = nullptr);
void halo_ce_finish(Comm& cm, cudaStream_t s);
void halo_wait_flags(const HaloFuse& hf, cudaStream_t s);  // one warp waits for the peers' flags
bool sum_p2p(Comm& cm, double* dev, int count, cudaStream_t s);
void sym_release(Comm& cm);

struct DevGraph;
struct DevLaplacian;
// Rewrites L.op into the local halo numbering (cols -> local ids, row0 -> 0, isd
// -> own+halo entries, dpos = diagonal storage slots) and builds comm.halo.
// No-op on one GPU.
void localize_operator(Comm& cm, const DevGraph& g, DevLaplacian& L, cudaStream_t s);

} // namespace spb

struct sp_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    spb::Comm comm;
    std::string err;
    spb::Timers timers;
    bool time_spmm = false;   // record CUDA events around every SpMM (bench/diagnostics)
    bool recurrence = false;  // LOBPCG AX/AH/AP recurrence (Solver::set_recurrence)
    bool relabel = true;      // irregular graphs: degree-descending relabel (relabel.cu)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // side stream: the initial block's mt19937_64 draws run there while the
    // preconditioner is built (partition_core)
    cudaStream_t aux = nullptr;
    cudaEvent_t aux_ready = nullptr, aux_done = nullptr;
    // event pairs recorded around SpMM launches; resolved without extra syncs
    // once the pipeline has synchronized (collect_spmm_times)
    std::vector<cudaEvent_t> evpool;
    std::vector<char> ev_poly;  // per event pair: 0 SpMM, 1 polynomial-step SpMM, 2 halo exchange
    size_t ev_used = 0;
    spb::PhaseProf prof;

    std::pair<cudaEvent_t, cudaEvent_t> next_event_pair(int kind = 0) {
        while (evpool.size() < ev_used + 2) {
            cudaEvent_t e;
            SPB_CUDA(cudaEventCreate(&e));
            evpool.push_back(e);
        }
        if (ev_poly.size() < ev_used / 2 + 1) ev_poly.resize(ev_used / 2 + 1);
        ev_poly[ev_used / 2] = static_cast<char>(kind);
        auto p = std::make_pair(evpool[ev_used], evpool[ev_used + 1]);
        ev_used += 2;
        return p;
    }
    // after a stream sync: accumulate recorded pairs into timers.spmm_ms
    void collect_spmm_times() {
        for (size_t i = 0; i + 1 < ev_used; i += 2) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, evpool[i], evpool[i + 1]) == cudaSuccess) {
                if (ev_poly[i / 2] == 2) {
                    timers.halo_ms += ms;
                    continue;
                }
                timers.spmm_ms += ms;
                if (ev_poly[i / 2] == 1) timers.poly_ms += ms;
            }
        }
        ev_used = 0;
    }
};

// Device-resident graph handle (sp_graph_upload)
struct sp_device_graph {
    sp_context* ctx = nullptr;
    spb::DevGraph g;
    spb::DBuf<int32_t> assignment;  // last partition result (device)
    // sp_ingest only: original vertex id of every vertex (n_global); multi-GPU
    // also keeps the whole CSR (the DevGraph holds this rank's row block)
    spb::DBuf<int64_t> old_ids;
    spb::DBuf<int64_t> full_offs;
    spb::DBuf<int32_t> full_cols;
    int64_t n_sym = 0, nnz_sym = 0;
    bool ingested = false;
};
