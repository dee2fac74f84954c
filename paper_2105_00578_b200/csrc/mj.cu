// mj.cu — multi-jagged partitioning of the eigenvector embedding on the device.
//
// Restates mj_partition / mj_recurse / build_plan (src/partitioner.cpp:43-170).
// The recursion becomes a level-synchronous sweep: at every level all tree
// nodes of that depth are sorted at once by the composite key
// (node, coordinate, vertex id), so each node's points are in exactly the
// reference's std::sort order (coordinate ascending, ties by ascending id,
// -0.0 == +0.0). Child ranges are exact weighted quantiles: for unit weights
// their sizes follow in closed form from the reference's greedy loop; for other
// weights one thread per node replays that loop over the sorted weights, so
// fp sums happen in the reference's order. Leaves are numbered left to right,
// which is the reference's depth-first next_part order.
#include "mj.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cuda/std/tuple>

#include <algorithm>
#include <cmath>

namespace spb {

namespace {

struct MjKey {
    uint32_t id;
    uint32_t seg;
    uint64_t coord;
};

struct MjDecomposer {
    __host__ __device__ ::cuda::std::tuple<uint32_t&, uint64_t&, uint32_t&> operator()(MjKey& k) const {
        return {k.seg, k.coord, k.id};
    }
};

__device__ __forceinline__ uint64_t orderable(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 compares equal to +0.0 in the reference comparator
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// seg index of position p: largest r with starts[r] <= p
__device__ __forceinline__ int find_seg(const int64_t* starts, int nseg, int64_t p) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (starts[mid] <= p) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void make_keys_kernel(int64_t n, const uint32_t* ids, const int64_t* starts,
                                 const int* seg_dim, int nseg, View coords, MjKey* keys) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int sg = find_seg(starts, nseg, p);
        const uint32_t id = ids[p];
        const int dim = seg_dim[sg];
        MjKey k;
        k.id = id;
        k.seg = static_cast<uint32_t>(sg);
        k.coord = dim >= 0 ? orderable(coords.at(id, dim)) : 0ull;
        keys[p] = k;
    }
}

// equal (segment, coordinate) side by side after the sort on those bits: a tie the ids must break
__global__ void tie_kernel(int64_t n, const MjKey* keys, int* flag) {
    for (int64_t p = 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (keys[p].seg == keys[p - 1].seg && keys[p].coord == keys[p - 1].coord) *flag = 1;
}

__global__ void keys_to_ids_kernel(int64_t n, const MjKey* keys, uint32_t* ids) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ids[p] = keys[p].id;
}

// General weights: one thread per internal node replays mj_recurse's greedy
// loop (partitioner.cpp:100-132) over the node's weights in sorted order.
__global__ void weighted_cuts_kernel(int nnodes, const int64_t* nstart, const int64_t* nsize,
                                     const int* child_off, const int64_t* child_leaves,
                                     const int* nchild, const int64_t* nleaves,
                                     const uint32_t* ids, const double* w, int64_t* child_size) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nnodes) return;
    const int64_t start = nstart[t], size = nsize[t];
    double total = 0.0;
    for (int64_t p = 0; p < size; ++p) total += w[ids[start + p]];
    const int64_t L = nleaves[t];
    int64_t pos = 0, leaves_done = 0;
    double consumed = 0.0;
    const int nc = nchild[t];
    for (int s = 0; s < nc; ++s) {
        const int64_t cl = child_leaves[child_off[t] + s];
        leaves_done += cl;
        if (s + 1 == nc) {
            child_size[child_off[t] + s] = size - pos;
            pos = size;
            break;
        }
        const double target = total * static_cast<double>(leaves_done) / static_cast<double>(L);
        const int64_t leaves_after = L - leaves_done;
        const int64_t max_take = size - pos - leaves_after;
        const int64_t min_take = cl;
        int64_t taken = 0;
        while (pos < size && taken < max_take && (taken < min_take || consumed < target)) {
            consumed += w[ids[start + pos]];
            ++pos;
            ++taken;
        }
        child_size[child_off[t] + s] = taken;
    }
}

__global__ void assign_kernel(int64_t n, const uint32_t* ids, const int64_t* starts, int nseg,
                              int32_t* assignment) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        assignment[ids[p]] = find_seg(starts, nseg, p);
}

__global__ void iota_kernel(int64_t n, uint32_t* ids) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ids[p] = static_cast<uint32_t>(p);
}

int g1(int64_t n) { return grid_for(n, 256, 8); }

void build_plan(MjPlanNode& node, int64_t target, int dim, int remaining) {
    node.leaves = target;
    node.dim = -1;
    node.kids.clear();
    if (target <= 1 || remaining <= 0) return;
    const double root = std::pow(static_cast<double>(target), 1.0 / remaining);
    int64_t m = static_cast<int64_t>(std::ceil(root - 1e-12));
    m = std::min<int64_t>(target, std::max<int64_t>(m, 2));
    node.dim = dim;
    const int64_t base = target / m, rem = target % m;
    node.kids.resize(m);
    for (int64_t s = 0; s < m; ++s) build_plan(node.kids[s], base + (s < rem ? 1 : 0), dim + 1, remaining - 1);
}

// ---- unit weights: radix select instead of sorting ----
// Points never move: seg[v] is the tree node of vertex v at the current level. A node
// with m kids cuts its points, in (coordinate, id) order, at m - 1 ranks that follow in
// closed form from the sizes (partitioner.cpp:100-132 with unit weights), so the level
// only needs the m - 1 keys at those ranks (queries) and one labelling pass: a point's
// kid is the number of cut keys <= its own key. The keys are found by radix select over
// the 96-bit composite (orderable coordinate, id), 8 bits per pass: histogram passes over
// every point until each query's bucket holds at most kCandMax points, then those
// candidates are gathered and one CTA per query finishes the select in shared memory.
constexpr int kCandMax = 4096;

struct SelState {
    unsigned long long hi;   // processed bits of the coordinate key (left-aligned value prefix)
    unsigned int lo;         // processed bits of the id (after all 64 coordinate bits)
    long long rank;          // rank within the bucket still to resolve
    long long cnt;           // points in the current bucket (-1: the rank is past the node's points)
    int bits;                // bits of the composite key the prefix covers
    int pad;
};

__device__ __forceinline__ unsigned digit_of(uint64_t key, uint32_t id, int bits) {
    return bits < 64 ? static_cast<unsigned>((key >> (56 - bits)) & 255u)
                     : static_cast<unsigned>((id >> (24 - (bits - 64))) & 255u);
}
__device__ __forceinline__ bool prefix_match(uint64_t key, uint32_t id, int bits, const SelState& q) {
    if (bits == 0) return true;
    if (bits <= 64) return (key >> (64 - bits)) == q.hi;
    return key == q.hi && (id >> (32 - (bits - 64))) == q.lo;
}

// histogram of the next digit of every point matching a query's prefix (privatized in
// shared memory when the level's histograms fit, else straight to global memory)
template <bool SMEM>
__global__ void sel_hist_kernel(int64_t n, const int32_t* seg, View coords, const int* seg_q0, const int* seg_dim,
                                const SelState* qs, int nq, int bits, unsigned* hist) {
    extern __shared__ unsigned sh_dyn[];
    unsigned* sh = SMEM ? sh_dyn : hist;
    if (SMEM) {
        for (int i = threadIdx.x; i < nq * 256; i += blockDim.x) sh[i] = 0;
        __syncthreads();
    }
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int sgi = seg[v];
        const int q0 = seg_q0[sgi], q1 = seg_q0[sgi + 1];
        if (q0 == q1) continue;
        const uint64_t key = orderable(coords.at(v, seg_dim[sgi]));
        const uint32_t id = static_cast<uint32_t>(v);
        const unsigned d = digit_of(key, id, bits);
        for (int q = q0; q < q1; ++q)
            if (qs[q].cnt > kCandMax && prefix_match(key, id, bits, qs[q])) atomicAdd(&sh[q * 256 + d], 1u);
    }
    if (!SMEM) return;
    __syncthreads();
    for (int i = threadIdx.x; i < nq * 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// one block of 256 threads per query: pick the bucket holding the query's rank
__global__ void sel_pick_kernel(SelState* qs, int bits, unsigned* hist) {
    __shared__ unsigned long long cum[256];
    const int q = blockIdx.x, t = threadIdx.x;
    SelState st = qs[q];
    if (st.cnt <= kCandMax) return;  // small enough for the candidate stage
    const unsigned h = hist[q * 256 + t];
    cum[t] = h;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const unsigned long long v = t >= off ? cum[t - off] : 0ull;
        __syncthreads();
        cum[t] += v;
        __syncthreads();
    }
    const unsigned long long below = cum[t] - h;
    if (static_cast<unsigned long long>(st.rank) >= below && static_cast<unsigned long long>(st.rank) < cum[t]) {
        if (bits < 64) st.hi = (st.hi << 8) | t;
        else st.lo = (st.lo << 8) | t;
        st.rank -= static_cast<long long>(below);
        st.cnt = h;
        st.bits = bits + 8;
        qs[q] = st;
    }
    hist[q * 256 + t] = 0;  // ready for the next pass
}

struct Cand {
    uint64_t key;
    uint32_t id;
};

// candidates: the points in each query's final bucket (at most kCandMax per query)
__global__ void sel_collect_kernel(int64_t n, const int32_t* seg, View coords, const int* seg_q0, const int* seg_dim,
                                   const SelState* qs, unsigned* fill, Cand* cand) {
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int sgi = seg[v];
        const int q0 = seg_q0[sgi], q1 = seg_q0[sgi + 1];
        if (q0 == q1) continue;
        const uint64_t key = orderable(coords.at(v, seg_dim[sgi]));
        const uint32_t id = static_cast<uint32_t>(v);
        for (int q = q0; q < q1; ++q)
            if (qs[q].cnt >= 0 && prefix_match(key, id, qs[q].bits, qs[q])) {
                const unsigned slot = atomicAdd(&fill[q], 1u);
                if (slot < kCandMax) cand[static_cast<int64_t>(q) * kCandMax + slot] = Cand{key, id};
            }
    }
}

// one block per query: radix select of the remaining bits among the candidates -> cut key
__global__ void sel_finish_kernel(const SelState* qs, const unsigned* fill, const Cand* cand,
                                  unsigned long long* cut_key, unsigned* cut_id, int* cut_inf) {
    __shared__ unsigned hist[256];
    __shared__ unsigned long long cum[256];
    __shared__ unsigned long long s_hi;
    __shared__ unsigned s_lo;
    __shared__ long long s_rank;
    const int q = blockIdx.x, t = threadIdx.x;
    const SelState st = qs[q];
    if (st.cnt < 0) {  // rank past the node's points: no point reaches this cut
        if (t == 0) cut_inf[q] = 1;
        return;
    }
    const int c = static_cast<int>(min(fill[q], static_cast<unsigned>(kCandMax)));
    const Cand* cq = cand + static_cast<int64_t>(q) * kCandMax;
    if (t == 0) {
        s_hi = st.hi;
        s_lo = st.lo;
        s_rank = st.rank;
    }
    __syncthreads();
    for (int bits = st.bits; bits < 96; bits += 8) {
        hist[t] = 0;
        __syncthreads();
        SelState cur{s_hi, s_lo, 0, 0, bits, 0};
        for (int i = t; i < c; i += blockDim.x)
            if (prefix_match(cq[i].key, cq[i].id, bits, cur)) atomicAdd(&hist[digit_of(cq[i].key, cq[i].id, bits)], 1u);
        __syncthreads();
        cum[t] = hist[t];
        __syncthreads();
        for (int off = 1; off < 256; off <<= 1) {
            const unsigned long long v = t >= off ? cum[t - off] : 0ull;
            __syncthreads();
            cum[t] += v;
            __syncthreads();
        }
        const unsigned long long below = cum[t] - hist[t];
        const long long r = s_rank;
        __syncthreads();
        if (static_cast<unsigned long long>(r) >= below && static_cast<unsigned long long>(r) < cum[t]) {
            if (bits < 64) s_hi = (s_hi << 8) | t;
            else s_lo = (s_lo << 8) | t;
            s_rank = r - static_cast<long long>(below);
        }
        __syncthreads();
    }
    if (t == 0) {
        cut_key[q] = s_hi;
        cut_id[q] = s_lo;
        cut_inf[q] = 0;
    }
}

// kid = number of the node's cut keys <= the point's key; new node = first kid's index + kid
__global__ void sel_label_kernel(int64_t n, int32_t* seg, View coords, const int* seg_q0, const int* seg_dim,
                                 const int* seg_base, const unsigned long long* cut_key, const unsigned* cut_id,
                                 const int* cut_inf) {
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int sgi = seg[v];
        const int q0 = seg_q0[sgi], q1 = seg_q0[sgi + 1];
        int kid = 0;
        if (q0 != q1) {
            const uint64_t key = orderable(coords.at(v, seg_dim[sgi]));
            const uint32_t id = static_cast<uint32_t>(v);
            for (int q = q0; q < q1; ++q)
                if (!cut_inf[q] && (key > cut_key[q] || (key == cut_key[q] && id >= cut_id[q]))) ++kid;
        }
        seg[v] = seg_base[sgi] + kid;
    }
}

// child sizes of a unit-weight node (partitioner.cpp:100-132 in closed form)
std::vector<int64_t> unit_takes(const MjPlanNode& node, int64_t size) {
    const int64_t L = node.leaves;
    const double W = static_cast<double>(size);
    int64_t pos = 0, leaves_done = 0;
    const size_t nc = node.kids.size();
    std::vector<int64_t> takes(nc);
    for (size_t c = 0; c < nc; ++c) {
        const int64_t cl = node.kids[c].leaf_count();
        leaves_done += cl;
        int64_t take;
        if (c + 1 == nc) {
            take = size - pos;
        } else {
            const double target = W * static_cast<double>(leaves_done) / static_cast<double>(L);
            const int64_t max_take = size - pos - (L - leaves_done);
            const int64_t t_target = std::max<int64_t>(0, static_cast<int64_t>(std::ceil(target)) - pos);
            take = std::max(cl, t_target);
            take = std::min(take, max_take);
            take = std::min(take, size - pos);
            take = std::max<int64_t>(take, 0);
        }
        takes[c] = take;
        pos += take;
    }
    return takes;
}

void mj_select_unit(int64_t n, int dims, const View& coords, const MjPlanNode& plan, int32_t* assignment,
                    cudaStream_t s) {
    struct Node {
        const MjPlanNode* node;
        int64_t size;
    };
    std::vector<Node> nodes{{&plan, n}};
    SPB_CUDA(cudaMemsetAsync(assignment, 0, sizeof(int32_t) * n, s));  // seg: every point in the root
    DBuf<int> d_q0, d_dim, d_base, d_inf;
    DBuf<SelState> d_qs;
    DBuf<unsigned> d_hist, d_fill, d_cid;
    DBuf<unsigned long long> d_ckey;
    DBuf<Cand> d_cand;
    for (;;) {
        bool any_internal = false;
        for (const Node& nd : nodes) any_internal |= !nd.node->kids.empty();
        if (!any_internal) break;
        const int ns = static_cast<int>(nodes.size());
        std::vector<int> q0(ns + 1, 0), dim(ns, 0), base(ns, 0);
        std::vector<SelState> qs;
        std::vector<Node> next;
        for (int i = 0; i < ns; ++i) {
            const Node& nd = nodes[i];
            q0[i] = static_cast<int>(qs.size());
            base[i] = static_cast<int>(next.size());
            if (nd.node->kids.empty()) {
                next.push_back(nd);
                continue;
            }
            dim[i] = nd.node->dim % dims;
            const std::vector<int64_t> takes = unit_takes(*nd.node, nd.size);
            int64_t b = 0;
            for (size_t c = 0; c < takes.size(); ++c) {
                if (c > 0) {
                    // the cut at rank b: cnt = the node's size (the bucket before any digit)
                    SelState st{0ull, 0u, b, b < nd.size ? nd.size : -1, 0, 0};
                    qs.push_back(st);
                }
                b += takes[c];
                next.push_back({&nd.node->kids[c], takes[c]});
            }
        }
        q0[ns] = static_cast<int>(qs.size());
        const int nq = static_cast<int>(qs.size());
        d_q0.alloc(ns + 1);
        d_dim.alloc(ns);
        d_base.alloc(ns);
        d_qs.alloc(nq);
        d_hist.alloc(static_cast<size_t>(nq) * 256);
        d_fill.alloc(nq);
        d_ckey.alloc(nq);
        d_cid.alloc(nq);
        d_inf.alloc(nq);
        d_cand.alloc(static_cast<size_t>(nq) * kCandMax);
        SPB_CUDA(cudaMemcpyAsync(d_q0.p, q0.data(), sizeof(int) * (ns + 1), cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemcpyAsync(d_dim.p, dim.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemcpyAsync(d_base.p, base.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemcpyAsync(d_qs.p, qs.data(), sizeof(SelState) * nq, cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemsetAsync(d_hist.p, 0, sizeof(unsigned) * nq * 256, s));
        SPB_CUDA(cudaMemsetAsync(d_fill.p, 0, sizeof(unsigned) * nq, s));
        const size_t hsm = sizeof(unsigned) * nq * 256;
        // histogram passes until every bucket is small enough for the candidate stage
        long long worst = 0;
        for (const SelState& st : qs) worst = std::max(worst, st.cnt);
        for (int bits = 0; bits < 96 && worst > kCandMax; bits += 8) {
            if (bits >= 16) {  // from the third digit on, check first (one small read back)
                SPB_CUDA(cudaMemcpyAsync(qs.data(), d_qs.p, sizeof(SelState) * nq, cudaMemcpyDeviceToHost, s));
                SPB_CUDA(cudaStreamSynchronize(s));
                worst = 0;
                for (const SelState& st : qs) worst = std::max(worst, st.cnt);
                if (worst <= kCandMax) break;
            }
            if (hsm <= 96 * 1024) {
                static bool attr = false;
                if (!attr) {
                    SPB_CUDA(cudaFuncSetAttribute(sel_hist_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  96 * 1024));
                    attr = true;
                }
                sel_hist_kernel<true><<<grid_for(n, 256, 4), 256, hsm, s>>>(n, assignment, coords, d_q0.p, d_dim.p,
                                                                            d_qs.p, nq, bits, d_hist.p);
            } else {
                sel_hist_kernel<false><<<grid_for(n, 256, 8), 256, 0, s>>>(n, assignment, coords, d_q0.p, d_dim.p,
                                                                           d_qs.p, nq, bits, d_hist.p);
            }
            SPB_LAUNCH_CHECK();
            sel_pick_kernel<<<nq, 256, 0, s>>>(d_qs.p, bits, d_hist.p);
            SPB_LAUNCH_CHECK();
        }
        sel_collect_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, assignment, coords, d_q0.p, d_dim.p, d_qs.p,
                                                               d_fill.p, d_cand.p);
        SPB_LAUNCH_CHECK();
        sel_finish_kernel<<<nq, 256, 0, s>>>(d_qs.p, d_fill.p, d_cand.p, d_ckey.p, d_cid.p, d_inf.p);
        SPB_LAUNCH_CHECK();
        sel_label_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, assignment, coords, d_q0.p, d_dim.p, d_base.p, d_ckey.p,
                                                             d_cid.p, d_inf.p);
        SPB_LAUNCH_CHECK();
        nodes.swap(next);
    }
    SPB_CUDA(cudaStreamSynchronize(s));
}

} // namespace

int64_t MjPlanNode::leaf_count() const {
    if (kids.empty()) return 1;
    int64_t t = 0;
    for (const MjPlanNode& k : kids) t += k.leaf_count();
    return t;
}

MjPlanNode mj_plan(int64_t num_parts, int dims) {
    if (num_parts < 1) throw_infeasible("section_counts: K < 1");
    if (dims < 1) throw_infeasible("section_counts: dims < 1");
    MjPlanNode root;
    build_plan(root, num_parts, 0, dims);
    return root;
}

void mj_partition_dev(int64_t n, int dims, const View& coords, const double* weights_dev,
                      bool unit_weights, int64_t num_parts, int32_t* assignment_dev, cudaStream_t s) {
    if (num_parts < 1) throw_infeasible("mj_partition: K < 1");
    if (n < num_parts)
        throw_infeasible("mj_partition: fewer points than parts (n=" + std::to_string(n) +
                         ", K=" + std::to_string(num_parts) + ")");
    if (n >= (int64_t(1) << 32)) throw_dimension("mj_partition: n too large");
    const MjPlanNode plan = mj_plan(num_parts, dims);
    if (unit_weights) {
        mj_select_unit(n, dims, coords, plan, assignment_dev, s);
        return;
    }

    DBuf<uint32_t> ids(n);
    DBuf<MjKey> kin(n), kout(n);
    iota_kernel<<<g1(n), 256, 0, s>>>(n, ids.p);
    SPB_LAUNCH_CHECK();

    struct Range {
        int64_t start, size;
        const MjPlanNode* node;
    };
    std::vector<Range> ranges{{0, n, &plan}};
    DBuf<int64_t> d_starts;
    DBuf<int> d_dims;
    DBuf<char> temp;
    size_t temp_bytes = 0;
    DBuf<int> tie(1);
    int level = 0;

    auto upload_ranges = [&](const std::vector<Range>& rs, bool with_dims) {
        std::vector<int64_t> st(rs.size());
        std::vector<int> dm(rs.size());
        for (size_t i = 0; i < rs.size(); ++i) {
            st[i] = rs[i].start;
            dm[i] = (with_dims && !rs[i].node->kids.empty()) ? rs[i].node->dim % dims : -1;
        }
        d_starts.alloc(st.size());
        d_dims.alloc(dm.size());
        SPB_CUDA(cudaMemcpyAsync(d_starts.p, st.data(), sizeof(int64_t) * st.size(), cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemcpyAsync(d_dims.p, dm.data(), sizeof(int) * dm.size(), cudaMemcpyHostToDevice, s));
    };

    for (;;) {
        bool any_internal = false;
        for (const Range& r : ranges)
            if (!r.node->kids.empty()) any_internal = true;
        if (!any_internal) break;
        const int nseg = static_cast<int>(ranges.size());
        upload_ranges(ranges, true);
        make_keys_kernel<<<g1(n), 256, 0, s>>>(n, ids.p, d_starts.p, d_dims.p, nseg, coords, kin.p);
        SPB_LAUNCH_CHECK();
        int seg_bits = 1;
        while ((int64_t(1) << seg_bits) < nseg) ++seg_bits;
        // key bits: id 0-31, coordinate 32-95, segment from 96 (MjDecomposer). The stable
        // sort on (segment, coordinate) alone already gives the (coordinate, id) order when
        // no two points of a segment share a coordinate, or when the input is in id order
        // (the first level): only a tie needs the 4 extra digit passes of the ids
        const int end_bit = 64 + 32 + seg_bits;
        auto sort_from = [&](int begin_bit) {
            size_t need = 0;
            SPB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, need, kin.p, kout.p, n, MjDecomposer{}, begin_bit,
                                                    end_bit, s));
            if (need > temp_bytes) {
                temp.alloc(need);
                temp_bytes = need;
            }
            SPB_CUDA(cub::DeviceRadixSort::SortKeys(temp.p, need, kin.p, kout.p, n, MjDecomposer{}, begin_bit,
                                                    end_bit, s));
            launch_counter() += (end_bit - begin_bit + 7) / 8 + 2;  // CUB onesweep: histogram + one pass per digit
        };
        sort_from(32);
        if (level > 0) {
            SPB_CUDA(cudaMemsetAsync(tie.p, 0, sizeof(int), s));
            tie_kernel<<<g1(n), 256, 0, s>>>(n, kout.p, tie.p);
            SPB_LAUNCH_CHECK();
            int h = 0;
            SPB_CUDA(cudaMemcpyAsync(&h, tie.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            SPB_CUDA(cudaStreamSynchronize(s));
            if (h) sort_from(0);
        }
        ++level;
        keys_to_ids_kernel<<<g1(n), 256, 0, s>>>(n, kout.p, ids.p);
        SPB_LAUNCH_CHECK();

        // child ranges
        std::vector<Range> next;
        if (unit_weights) {
            for (const Range& r : ranges) {
                if (r.node->kids.empty()) {
                    next.push_back(r);
                    continue;
                }
                const int64_t size = r.size, L = r.node->leaves;
                const double W = static_cast<double>(size);
                int64_t pos = 0, leaves_done = 0;
                const size_t nc = r.node->kids.size();
                for (size_t c = 0; c < nc; ++c) {
                    const MjPlanNode& kid = r.node->kids[c];
                    const int64_t cl = kid.leaf_count();
                    leaves_done += cl;
                    int64_t take;
                    if (c + 1 == nc) {
                        take = size - pos;
                    } else {
                        const double target = W * static_cast<double>(leaves_done) / static_cast<double>(L);
                        const int64_t max_take = size - pos - (L - leaves_done);
                        const int64_t t_target = std::max<int64_t>(0, static_cast<int64_t>(std::ceil(target)) - pos);
                        take = std::max(cl, t_target);
                        take = std::min(take, max_take);
                        take = std::min(take, size - pos);
                        take = std::max<int64_t>(take, 0);
                    }
                    next.push_back({r.start + pos, take, &kid});
                    pos += take;
                }
            }
        } else {
            std::vector<int64_t> nst, nsz, nl, cleaves;
            std::vector<int> coff, nch;
            std::vector<const Range*> internal;
            for (const Range& r : ranges) {
                if (r.node->kids.empty()) continue;
                internal.push_back(&r);
                nst.push_back(r.start);
                nsz.push_back(r.size);
                nl.push_back(r.node->leaves);
                coff.push_back(static_cast<int>(cleaves.size()));
                nch.push_back(static_cast<int>(r.node->kids.size()));
                for (const MjPlanNode& k : r.node->kids) cleaves.push_back(k.leaf_count());
            }
            const int nn = static_cast<int>(internal.size());
            DBuf<int64_t> a(nn), b(nn), c(nn), d(cleaves.size()), out(cleaves.size());
            DBuf<int> e(nn), f(nn);
            SPB_CUDA(cudaMemcpyAsync(a.p, nst.data(), sizeof(int64_t) * nn, cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(b.p, nsz.data(), sizeof(int64_t) * nn, cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(c.p, nl.data(), sizeof(int64_t) * nn, cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(d.p, cleaves.data(), sizeof(int64_t) * cleaves.size(), cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(e.p, coff.data(), sizeof(int) * nn, cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(f.p, nch.data(), sizeof(int) * nn, cudaMemcpyHostToDevice, s));
            weighted_cuts_kernel<<<ceil_div(nn, 64), 64, 0, s>>>(nn, a.p, b.p, e.p, d.p, f.p, c.p, ids.p,
                                                                 weights_dev, out.p);
            SPB_LAUNCH_CHECK();
            std::vector<int64_t> sizes(cleaves.size());
            SPB_CUDA(cudaMemcpyAsync(sizes.data(), out.p, sizeof(int64_t) * sizes.size(), cudaMemcpyDeviceToHost, s));
            SPB_CUDA(cudaStreamSynchronize(s));
            size_t ii = 0;
            for (const Range& r : ranges) {
                if (r.node->kids.empty()) {
                    next.push_back(r);
                    continue;
                }
                int64_t pos = 0;
                for (size_t cidx = 0; cidx < r.node->kids.size(); ++cidx) {
                    const int64_t take = sizes[coff[ii] + cidx];
                    next.push_back({r.start + pos, take, &r.node->kids[cidx]});
                    pos += take;
                }
                ++ii;
            }
        }
        ranges.swap(next);
    }
    // every range is a leaf now; leaves in position order = DFS order
    upload_ranges(ranges, false);
    assign_kernel<<<g1(n), 256, 0, s>>>(n, ids.p, d_starts.p, static_cast<int>(ranges.size()), assignment_dev);
    SPB_LAUNCH_CHECK();
    SPB_CUDA(cudaStreamSynchronize(s));
}

} // namespace spb
