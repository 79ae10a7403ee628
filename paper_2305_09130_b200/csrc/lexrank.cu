// check_nontermination's traces (explore.cpp:207-233) on the GPU: every
// distinct terminal state of a configuration, in the order the reference's
// DFS meets them, each with the path the DFS followed to it.
//
// The DFS of explore_machine (explore.cpp:86-165) with a visited set visits
// every state along the lexicographically least path to it (paths compared as
// sequences of enabled() indices): a state reached along a larger path has
// already been met along the least one, whose prefix the DFS expands first.
// So the DFS tree is the tree of least paths, the discovery order is their
// lexicographic order, and a terminal's trace is its least path.  The state
// graphs are graded (every path to a state has the same length,
// tests/test_oracle.py), so least paths can be ranked level by level, in
// parallel:
//   * level d holds the states of depth d sorted by their least path; its
//     rank r is the state's position;
//   * expanding level d (one thread per state, the serial enabled() order of
//     machine.cuh) inserts every successor into a visited table and
//     min-combines (r << 16 | enabled index) into the successor's slot: the
//     least path of a successor extends the least path of its least-ranked
//     parent by its least edge from it;
//   * sorting level d+1 by that key (CUB radix sort) ranks it;
//   * a terminal's trace walks the parent ranks back to the root, and its DFS
//     position is the lexicographic order of its rank sequence.
// Limits follow the reference: states deeper than max_depth are not expanded
// (explore.cpp:124-127); a visited set that would exceed max_states makes the
// reference's traversal order-dependent (explore.cpp:28), which this engine
// reports as MCTB_LIMIT instead of guessing.
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "bfs.cuh"
#include "common.cuh"
#include "pack.cuh"
#include "traj.cuh"

namespace mctb {

namespace {

struct LrTable {
    unsigned long long* tag;   // 0 = empty, else hash | 1
    unsigned long long* best;  // min (parent rank << 16 | enabled index) over the in-edges
    uint32_t* keys;            // [slots * words] packed states (every word carries kGuard)
    uint64_t mask;
    int words;
};

struct LrLevel {
    uint32_t* list;          // slots of the next level, in discovery order
    unsigned long long* n;   // [0] next-level count, [1] transitions, [2] terminals,
                             // [3] error (1 table full, 2 deadlock, 3 apply), [4] depth cut
};

struct LrTerm {
    int64_t time;
    uint32_t depth, rank;
};

__device__ void lr_insert(const LrTable& t, const LrLevel& lv, const uint32_t* key, uint64_t h,
                          unsigned long long bestv) {
    const unsigned long long fp = h | 1ull;
    uint64_t i = h & t.mask;
    // the table holds 2x the states it is sized for: a probe sequence this long
    // means it is overfull (a level outgrew the bound) — report it instead of
    // scanning the whole table per insert
    for (uint64_t probe = 0; probe < 1024 && probe <= t.mask; ++probe, i = (i + 1) & t.mask) {
        unsigned long long tg = *(volatile unsigned long long*)&t.tag[i];
        if (tg == 0) {
            tg = atomicCAS(&t.tag[i], 0ull, fp);
            if (tg == 0) {
                uint32_t* k = t.keys + i * (uint64_t)t.words;
                for (int w = 0; w < t.words; ++w) k[w] = key[w];
                atomicMin(&t.best[i], bestv);
                const unsigned long long pos = atomicAdd(&lv.n[0], 1ull);
                lv.list[pos] = (uint32_t)i;
                return;
            }
        }
        if (tg != fp) continue;
        const volatile uint32_t* k = t.keys + i * (uint64_t)t.words;
        bool eq = true;
        for (int w = 0; w < t.words; ++w) {
            uint32_t v;
            while (!((v = k[w]) & kGuard)) {  // the claimer is still writing the key
            }
            eq &= v == key[w];
        }
        if (eq) {
            atomicMin(&t.best[i], bestv);
            return;
        }
    }
    atomicExch((unsigned long long*)&lv.n[3], 1ull);
}

// One thread per state of level d (rank r): enabled() in the reference's order,
// every successor into the table with key (r << 16 | index).
__global__ void __launch_bounds__(128) lr_expand_kernel(BfsDesc bd, const uint32_t* states,
                                                        uint32_t n, uint32_t depth,
                                                        uint32_t depth_cap, LrTable t, LrLevel lv,
                                                        LrTerm* terms, uint64_t term_cap) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const MachDesc& m = bd.m;
    MState s, x;
    unpack(bd, states + (uint64_t)r * t.words, s);
    Transition en[kMaxEnabled];
    const int ne = enabled(m, s, en);
    if (ne == 0) {
        if (!is_terminal(m, s)) {
            atomicExch((unsigned long long*)&lv.n[3], 2ull);
            return;
        }
        const unsigned long long k = atomicAdd(&lv.n[2], 1ull);
        if (k < term_cap) terms[k] = LrTerm{s.time, depth, r};
        return;
    }
    if (depth >= depth_cap) {  // explore.cpp:124-127: no transition past max_depth
        atomicExch((unsigned long long*)&lv.n[4], 1ull);
        return;
    }
    atomicAdd(&lv.n[1], (unsigned long long)ne);
    uint32_t key[kMaxWords];
    for (int e = 0; e < ne; ++e) {
        copy_state(m, x, s);
        if (!apply(m, x, en[e])) {
            atomicExch((unsigned long long*)&lv.n[3], 3ull);
            return;
        }
        pack(bd, 0, x, key);
        lr_insert(t, lv, key, hash_words(key, t.words),
                  ((unsigned long long)r << 16) | (unsigned long long)e);
    }
}

__global__ void lr_gather_kernel(const LrTable t, const uint32_t* list, uint32_t n,
                                 unsigned long long* sort_key, uint32_t* sort_val) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    sort_key[j] = t.best[list[j]];
    sort_val[j] = list[j];
}

// Level d+1 in rank order: packed states and their least in-edge.
__global__ void lr_place_kernel(const LrTable t, const unsigned long long* sorted_key,
                                const uint32_t* sorted_slot, uint32_t n, uint32_t* states,
                                unsigned long long* best) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t* k = t.keys + (uint64_t)sorted_slot[r] * t.words;
    for (int w = 0; w < t.words; ++w) states[(uint64_t)r * t.words + w] = k[w];
    best[r] = sorted_key[r];
}

// One thread per terminal: its rank at every level (the least path's nodes) and
// the enabled index taken at each.
__global__ void lr_chain_kernel(const LrTerm* terms, uint32_t n_terms, const uint64_t* off,
                                const uint64_t* level_base, const unsigned long long* best,
                                uint32_t* rank_out, uint32_t* edge_out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_terms) return;
    uint32_t cur = terms[j].rank;
    const uint64_t o = off[j];
    for (uint32_t l = terms[j].depth; l >= 1; --l) {
        const unsigned long long b = best[level_base[l] + cur];
        cur = (uint32_t)(b >> 16);
        rank_out[o + l - 1] = cur;
        edge_out[o + l - 1] = (uint32_t)(b & 0xffffull);
    }
}

// One thread per path step: the transition enabled()[edge] of the node's state.
__global__ void __launch_bounds__(128) lr_trans_kernel(BfsDesc bd, const uint32_t* states, int words,
                                                       const uint32_t* rank_of, const uint32_t* edge_of,
                                                       const uint32_t* level_of,
                                                       const uint64_t* level_base, uint64_t n,
                                                       int32_t* trace) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    MState s;
    unpack(bd, states + (level_base[level_of[i]] + rank_of[i]) * words, s);
    Transition en[kMaxEnabled];
    enabled(bd.m, s, en);
    const Transition t = en[edge_of[i]];
    trace[4 * i] = t.actor;
    trace[4 * i + 1] = t.peer;
    trace[4 * i + 2] = t.op;
    trace[4 * i + 3] = t.arg;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t st = nullptr;
    int alloc(size_t n, cudaStream_t s) {
        st = s;
        return cuda_check(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s), "lexrank alloc");
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

struct StreamGuard {
    cudaStream_t st = nullptr;
    ~StreamGuard() {
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
};

// One thread per state of a level: its least in-edge as a transition (the
// parent's enabled()[edge]), whether it is terminal and how many transitions it
// enables (the DFS applies them all unless it sits at the depth cap).
__global__ void __launch_bounds__(128) lr_info_kernel(BfsDesc bd, const uint32_t* parents,
                                                      const uint32_t* states, int words,
                                                      const unsigned long long* best, uint32_t n,
                                                      int32_t* meta) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    Transition en[kMaxEnabled];
    MState s;
    int32_t* o = meta + 7 * (uint64_t)r;
    if (parents) {
        const unsigned long long b = best[r];
        unpack(bd, parents + (b >> 16) * words, s);
        enabled(bd.m, s, en);
        const Transition t = en[b & 0xffffull];
        o[0] = t.actor;
        o[1] = t.peer;
        o[2] = t.op;
        o[3] = t.arg;
        o[6] = (int32_t)(b & 0xffffull);
    } else {
        o[0] = o[1] = o[2] = o[3] = o[6] = -1;
    }
    unpack(bd, states + (uint64_t)r * words, s);
    const int ne = enabled(bd.m, s, en);
    o[4] = ne;
    o[5] = ne == 0 && is_terminal(bd.m, s) ? 1 : 0;
}

// The level-synchronous ranking of one configuration, kept on the device: every
// state reachable within max_depth, level by level in least-path order.
struct LrRun {
    StreamGuard sg;  // destroyed last: the buffers free on its stream
    cudaStream_t st = nullptr;
    BfsDesc bd{};
    int words = 0;
    DevBuf<int32_t> ids;
    DevBuf<unsigned long long> tag, best_tab, lvl_best, sort_k[2], cnt;
    DevBuf<uint32_t> keys, lvl_states, list, sort_v[2];
    DevBuf<LrTerm> terms;
    DevBuf<char> sort_tmp;
    uint64_t term_cap = 0;
    std::vector<uint64_t> base{0, 1};  // level d occupies [base[d], base[d+1])
    unsigned long long hc[8] = {};
};

// Builds every level.  Returns MCTB_LIMIT when the exploration would exceed
// max_states states.
int lr_build(MachHost& h, int64_t max_depth, int64_t max_states, LrRun& run,
             uint64_t max_levels = UINT64_MAX) {
    MCTB_CUDA(cudaStreamCreateWithFlags(&run.sg.st, cudaStreamNonBlocking));
    cudaStream_t st = run.st = run.sg.st;
    int32_t* d_ids = nullptr;
    int rc = upload_desc(h, st, &d_ids);
    if (rc) return rc;
    run.ids.p = d_ids;
    run.ids.st = st;
    BfsDesc& bd = run.bd;
    bd.m = h.d;
    bd.l = bfs_layout(h.d, 1);
    const int words = run.words = bd.l.words;
    const uint64_t cap = (uint64_t)std::max<int64_t>(max_states, 1);
    uint64_t slots = 1024;
    while (slots < 2 * cap) slots <<= 1;
    // table + levels: sized for max_states states
    run.term_cap = cap;
    if ((rc = run.tag.alloc(slots, st)) || (rc = run.best_tab.alloc(slots, st)) ||
        (rc = run.keys.alloc(slots * words, st)) || (rc = run.lvl_states.alloc(cap * words, st)) ||
        (rc = run.lvl_best.alloc(cap, st)) || (rc = run.list.alloc(cap, st)) ||
        (rc = run.sort_k[0].alloc(cap, st)) || (rc = run.sort_k[1].alloc(cap, st)) ||
        (rc = run.sort_v[0].alloc(cap, st)) || (rc = run.sort_v[1].alloc(cap, st)) ||
        (rc = run.cnt.alloc(8, st)) || (rc = run.terms.alloc(run.term_cap, st)))
        return rc;
    MCTB_CUDA(cudaMemsetAsync(run.tag.p, 0, slots * 8, st));
    MCTB_CUDA(cudaMemsetAsync(run.best_tab.p, 0xff, slots * 8, st));
    MCTB_CUDA(cudaMemsetAsync(run.keys.p, 0, slots * words * 4, st));
    MCTB_CUDA(cudaMemsetAsync(run.cnt.p, 0, 8 * 8, st));
    LrTable t{run.tag.p, run.best_tab.p, run.keys.p, slots - 1, words};
    LrLevel lv{run.list.p, run.cnt.p};
    // level 0: the initial state, packed on the host (same pack() as the device)
    {
        MState s0;
        initial_state(h.d, s0);
        std::vector<uint32_t> k0(kMaxWords, 0);
        pack(bd, 0, s0, k0.data());
        MCTB_CUDA(cudaMemcpyAsync(run.lvl_states.p, k0.data(), words * 4, cudaMemcpyHostToDevice, st));
        const unsigned long long root = 0;
        MCTB_CUDA(cudaMemcpyAsync(run.lvl_best.p, &root, 8, cudaMemcpyHostToDevice, st));
    }
    std::vector<uint64_t>& base = run.base;
    const uint32_t depth_cap = (uint32_t)std::min<int64_t>(max_depth, 0x7fffffff);
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, run.sort_k[0].p, run.sort_k[1].p,
                                    run.sort_v[0].p, run.sort_v[1].p,
                                    (int)std::min<uint64_t>(cap, 0x7fffffff), 0, 64, st);
    if ((rc = run.sort_tmp.alloc(sort_bytes, st))) return rc;
    unsigned long long* hc = run.hc;
    for (uint32_t d = 0;; ++d) {
        const uint32_t n = (uint32_t)(base[d + 1] - base[d]);
        MCTB_CUDA(cudaMemsetAsync(run.cnt.p, 0, 8, st));  // next-level count only
        lr_expand_kernel<<<(n + 127) / 128, 128, 0, st>>>(
            bd, run.lvl_states.p + base[d] * words, n, d, depth_cap, t, lv, run.terms.p,
            run.term_cap);
        MCTB_CUDA(cudaGetLastError());
        MCTB_CUDA(cudaMemcpyAsync(hc, run.cnt.p, sizeof run.hc, cudaMemcpyDeviceToHost, st));
        MCTB_CUDA(cudaStreamSynchronize(st));
        if (hc[3]) {
            set_error(hc[3] == 1 ? "lexrank: visited table full"
                                 : "model bug: deadlock or inapplicable transition");
            return hc[3] == 1 ? MCTB_LIMIT : MCTB_MODEL_BUG;
        }
        const uint64_t n1 = hc[0];
        if (n1 == 0) break;
        if (base.size() > max_levels) {
            set_error("the state graph is deeper than the ranking's level bound");
            return MCTB_LIMIT;
        }
        if (base.back() + n1 > cap) {
            set_error("the exploration exceeds max_states, where the reference's visited set "
                      "truncates in traversal order");
            return MCTB_LIMIT;
        }
        // rank level d+1 by (parent rank, enabled index)
        lr_gather_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, st>>>(
            t, run.list.p, (uint32_t)n1, run.sort_k[0].p, run.sort_v[0].p);
        int end_bit = 16;
        while (end_bit < 64 && ((uint64_t)n >> (end_bit - 16)) != 0) ++end_bit;
        MCTB_CUDA(cub::DeviceRadixSort::SortPairs(run.sort_tmp.p, sort_bytes, run.sort_k[0].p,
                                                  run.sort_k[1].p, run.sort_v[0].p,
                                                  run.sort_v[1].p, (int)n1, 0, end_bit, st));
        lr_place_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, st>>>(
            t, run.sort_k[1].p, run.sort_v[1].p, (uint32_t)n1,
            run.lvl_states.p + base.back() * words, run.lvl_best.p + base.back());
        MCTB_CUDA(cudaGetLastError());
        base.push_back(base.back() + n1);
    }
    return MCTB_OK;
}

}  // namespace

// Every state of one configuration within max_depth, in the order the
// reference's DFS discovers them (explore.cpp:86-165: the preorder of the
// least-path tree, children by enabled() index), packed (bfs_layout(h.d, 1)).
// meta = int32[7] per state {in-transition actor, peer, op, arg, enabled count,
// terminal, in-edge index (the in-transition's position in the parent's enabled();
// -1 at the root)}; depth = the state's depth.  table_cap bounds the
// exploration (MCTB_LIMIT beyond it).
int lexrank_states(MachHost& h, int64_t max_depth, int64_t table_cap, int* words,
                   std::vector<uint32_t>* packed, std::vector<int32_t>* meta,
                   std::vector<uint32_t>* depth) {
    LrRun run;
    int rc = lr_build(h, max_depth, table_cap, run);
    if (rc) return rc;
    const cudaStream_t st = run.st;
    const uint64_t n = run.base.back();
    const int w = *words = run.words;
    DevBuf<int32_t> d_meta;
    if ((rc = d_meta.alloc(7 * n, st))) return rc;
    for (size_t d = 0; d + 1 < run.base.size(); ++d) {
        const uint64_t b = run.base[d], nl = run.base[d + 1] - b;
        lr_info_kernel<<<(unsigned)((nl + 127) / 128), 128, 0, st>>>(
            run.bd, d ? run.lvl_states.p + run.base[d - 1] * w : nullptr,
            run.lvl_states.p + b * w, w, run.lvl_best.p + b, (uint32_t)nl, d_meta.p + 7 * b);
    }
    MCTB_CUDA(cudaGetLastError());
    std::vector<uint32_t> lv(n * w);
    std::vector<int32_t> mt(7 * n);
    std::vector<unsigned long long> best(n);
    MCTB_CUDA(cudaMemcpyAsync(lv.data(), run.lvl_states.p, n * w * 4, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaMemcpyAsync(mt.data(), d_meta.p, n * 28, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaMemcpyAsync(best.data(), run.lvl_best.p, n * 8, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    // the children of a state are a contiguous run of the next level (sorted by
    // parent rank, then edge): [cb[g], ce[g]) in global indices
    const size_t L = run.base.size() - 1;
    std::vector<uint64_t> cb(n, 0), ce(n, 0);
    for (size_t d = 0; d + 1 < L; ++d) {
        const uint64_t b = run.base[d], nb = run.base[d + 1], ne = run.base[d + 2];
        uint64_t c = nb;
        for (uint64_t g = b; g < nb; ++g) {
            cb[g] = c;
            while (c < ne && (best[c] >> 16) == g - b) ++c;
            ce[g] = c;
        }
    }
    packed->resize(n * w);
    meta->resize(7 * n);
    depth->resize(n);
    std::vector<std::pair<uint64_t, size_t>> stack{{0, 0}};  // (global index, level)
    uint64_t out = 0;
    while (!stack.empty()) {
        const auto [g, d] = stack.back();
        stack.pop_back();
        std::memcpy(packed->data() + out * w, lv.data() + g * w, w * 4);
        std::memcpy(meta->data() + 7 * out, mt.data() + 7 * g, 28);
        (*depth)[out] = (uint32_t)d;
        ++out;
        for (uint64_t c = ce[g]; c > cb[g]; --c) stack.push_back({c - 1, d + 1});
    }
    return MCTB_OK;
}

__global__ void lr_ne_kernel(BfsDesc bd, const uint32_t* states, int words, uint64_t n,
                             uint16_t* ne) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    MState s;
    unpack(bd, states + r * words, s);
    Transition en[kMaxEnabled];
    ne[r] = (uint16_t)enabled(bd.m, s, en);
}

// The reference DFS's statistics when its visited set fills at `cap` states
// (explore.cpp:26-30, 124-138): the DFS then visits exactly the first cap
// states of its discovery order (a full set stops only new states), applies
// every transition of those below max_depth, and reaches their largest depth.
// The order is the preorder of the least-path tree (lexrank_states), so the
// whole graph within max_depth is ranked: graph_states is its size (known from a
// sweep, dfs_prefix_stats in bfs.cu).
int lexrank_prefix(MachHost& h, int64_t max_depth, uint64_t cap, uint64_t graph_states,
                   int64_t* applies, int64_t* max_depth_reached) {
    LrRun run;
    int rc = lr_build(h, max_depth, (int64_t)std::max<uint64_t>(graph_states, 1), run);
    if (rc) return rc;
    const cudaStream_t st = run.st;
    const uint64_t n = run.base.back();
    DevBuf<uint16_t> d_ne;
    if ((rc = d_ne.alloc(n, st))) return rc;
    lr_ne_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(run.bd, run.lvl_states.p, run.words,
                                                             n, d_ne.p);
    MCTB_CUDA(cudaGetLastError());
    std::vector<uint16_t> ne(n);
    std::vector<unsigned long long> best(n);
    MCTB_CUDA(cudaMemcpyAsync(ne.data(), d_ne.p, n * 2, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaMemcpyAsync(best.data(), run.lvl_best.p, n * 8, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    const size_t L = run.base.size() - 1;
    std::vector<uint64_t> cb(n, 0), ce(n, 0);
    for (size_t d = 0; d + 1 < L; ++d) {
        const uint64_t b = run.base[d], nb = run.base[d + 1], e = run.base[d + 2];
        uint64_t c = nb;
        for (uint64_t g = b; g < nb; ++g) {
            cb[g] = c;
            while (c < e && (best[c] >> 16) == g - b) ++c;
            ce[g] = c;
        }
    }
    int64_t a = 0, md = 0;
    uint64_t seen = 0;
    std::vector<std::pair<uint64_t, size_t>> stack{{0, 0}};
    while (!stack.empty() && seen < cap) {
        const auto [g, d] = stack.back();
        stack.pop_back();
        ++seen;
        if ((int64_t)d < max_depth) a += ne[g];
        md = std::max<int64_t>(md, (int64_t)d);
        for (uint64_t c = ce[g]; c > cb[g]; --c) stack.push_back({c - 1, d + 1});
    }
    *applies = a;
    *max_depth_reached = md;
    return MCTB_OK;
}

// All terminal states of one configuration in DFS order with their least paths.
// Returns MCTB_LIMIT when the exploration would exceed max_states (the
// reference's truncation then depends on its traversal order).
int lexrank_terminals(MachHost& h, int64_t max_depth, int64_t max_states,
                      std::vector<int64_t>* times, std::vector<int64_t>* lens,
                      std::vector<int32_t>* trace) {
    std::unique_ptr<LrRun> runp(new LrRun);
    int rc = lr_build(h, max_depth, max_states, *runp);
    // The visited set fills (explore.cpp:26-30): the DFS then meets only the
    // terminals among the first max_states states of its order.  The whole graph
    // is ranked (up to 2^22 states) and the terminals are cut at that prefix.
    uint64_t visit_cap = 0;
    constexpr int64_t kRankBound = 1ll << 22;
    if (rc == MCTB_LIMIT && runp->hc[3] == 0 && max_states < kRankBound) {
        runp.reset(new LrRun);
        rc = lr_build(h, max_depth, kRankBound, *runp);
        visit_cap = (uint64_t)max_states;
    }
    if (rc) {
        if (rc == MCTB_LIMIT && runp->hc[3] == 0)
            set_error("check_nontermination: the visited set fills up and the state graph "
                      "exceeds the 2^22 states the DFS order is ranked over");
        return rc;
    }
    LrRun& run = *runp;
    const cudaStream_t st = run.st;
    const BfsDesc& bd = run.bd;
    const int words = run.words;
    const std::vector<uint64_t>& base = run.base;
    const unsigned long long* hc = run.hc;
    const uint64_t n_terms = hc[2];
    if (n_terms > run.term_cap) {
        set_error("check_nontermination: more terminal states than max_states");
        return MCTB_LIMIT;
    }
    std::vector<LrTerm> ht(n_terms);
    MCTB_CUDA(cudaMemcpyAsync(ht.data(), run.terms.p, n_terms * sizeof(LrTerm), cudaMemcpyDeviceToHost,
                              st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    std::vector<uint64_t> off(n_terms + 1, 0);
    for (uint64_t j = 0; j < n_terms; ++j) off[j + 1] = off[j] + ht[j].depth;
    const uint64_t n_steps = off[n_terms];
    std::vector<uint32_t> level_of(n_steps);
    for (uint64_t j = 0; j < n_terms; ++j)
        for (uint32_t l = 0; l < ht[j].depth; ++l) level_of[off[j] + l] = l;
    DevBuf<uint64_t> d_off, d_base;
    DevBuf<uint32_t> d_rank, d_edge, d_level;
    DevBuf<LrTerm> d_terms_sorted;
    DevBuf<int32_t> d_trace;
    if ((rc = d_off.alloc(n_terms + 1, st)) || (rc = d_base.alloc(base.size(), st)) ||
        (rc = d_rank.alloc(n_steps, st)) || (rc = d_edge.alloc(n_steps, st)) ||
        (rc = d_level.alloc(n_steps, st)) || (rc = d_trace.alloc(4 * n_steps, st)))
        return rc;
    MCTB_CUDA(cudaMemcpyAsync(d_off.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMemcpyAsync(d_base.p, base.data(), base.size() * 8, cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMemcpyAsync(d_level.p, level_of.data(), n_steps * 4, cudaMemcpyHostToDevice, st));
    if (n_terms) {
        lr_chain_kernel<<<(unsigned)((n_terms + 127) / 128), 128, 0, st>>>(
            run.terms.p, (uint32_t)n_terms, d_off.p, d_base.p, run.lvl_best.p, d_rank.p, d_edge.p);
        if (n_steps)
            lr_trans_kernel<<<(unsigned)((n_steps + 127) / 128), 128, 0, st>>>(
                bd, run.lvl_states.p, words, d_rank.p, d_edge.p, d_level.p, d_base.p, n_steps,
                d_trace.p);
        MCTB_CUDA(cudaGetLastError());
    }
    std::vector<uint32_t> rank(n_steps);
    std::vector<int32_t> tr(4 * n_steps);
    MCTB_CUDA(cudaMemcpyAsync(rank.data(), d_rank.p, n_steps * 4, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaMemcpyAsync(tr.data(), d_trace.p, n_steps * 16, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    // DFS order = lexicographic order of the least paths = of the rank sequences
    // (rank at level 1, 2, ...; a terminal is never a prefix of another path)
    std::vector<uint64_t> order(n_terms);
    for (uint64_t j = 0; j < n_terms; ++j) order[j] = j;
    auto rank_at = [&](uint64_t j, uint32_t l) -> uint32_t {
        // the node at level l of terminal j's path (l <= depth; the terminal itself at depth)
        return l == ht[j].depth ? ht[j].rank : rank[off[j] + l];
    };
    std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
        const uint32_t da = ht[a].depth, db = ht[b].depth;
        for (uint32_t l = 1; l <= std::min(da, db); ++l) {
            const uint32_t ra = rank_at(a, l), rb = rank_at(b, l);
            if (ra != rb) return ra < rb;
        }
        return da < db;  // unreachable for distinct terminals
    });
    // under a full visited set: the terminals among the first visit_cap states of
    // the preorder of the least-path tree (the DFS's discovery order)
    std::vector<char> seen;
    if (visit_cap) {
        const uint64_t n = base.back();
        std::vector<unsigned long long> best(n);
        MCTB_CUDA(cudaMemcpyAsync(best.data(), run.lvl_best.p, n * 8, cudaMemcpyDeviceToHost, st));
        MCTB_CUDA(cudaStreamSynchronize(st));
        const size_t L = base.size() - 1;
        std::vector<uint64_t> cb(n, 0), ce(n, 0);
        for (size_t d = 0; d + 1 < L; ++d) {
            const uint64_t b = base[d], nb = base[d + 1], e = base[d + 2];
            uint64_t c = nb;
            for (uint64_t g = b; g < nb; ++g) {
                cb[g] = c;
                while (c < e && (best[c] >> 16) == g - b) ++c;
                ce[g] = c;
            }
        }
        seen.assign(n, 0);
        uint64_t visited = 0;
        std::vector<uint64_t> stack{0};
        while (!stack.empty() && visited < visit_cap) {
            const uint64_t g = stack.back();
            stack.pop_back();
            seen[g] = 1;
            ++visited;
            for (uint64_t c = ce[g]; c > cb[g]; --c) stack.push_back(c - 1);
        }
    }
    times->clear();
    lens->clear();
    trace->clear();
    for (uint64_t j : order) {
        if (visit_cap && !seen[base[ht[j].depth] + ht[j].rank]) continue;
        times->push_back(ht[j].time);
        lens->push_back(ht[j].depth);
        trace->insert(trace->end(), tr.begin() + 4 * off[j], tr.begin() + 4 * off[j + 1]);
    }
    return MCTB_OK;
}

int check_machine(const int* plat, int size, int kernel, int wg, int ts);

}  // namespace mctb

using namespace mctb;

extern "C" int mctb_nonterm_traces(const int* plat, int size, int kernel, const int64_t* input,
                                   int wg, int ts, int64_t max_depth, int64_t max_states,
                                   int64_t* n_traces, int64_t* rows, int64_t rows_cap,
                                   int32_t* trace, int64_t trace_cap, int64_t* trace_len) {
    if (max_depth < 1) {  // explore.cpp:91
        set_error("max_depth must be >= 1");
        return MCTB_CONFIG_ERROR;
    }
    int rc = check_machine(plat, size, kernel, wg, ts);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    MachHost h;
    if ((rc = build_desc(plat, size, kernel, input, wg, ts, &h))) return rc;
    std::vector<int64_t> times, lens;
    std::vector<int32_t> tr;
    if ((rc = lexrank_terminals(h, max_depth, max_states > 0 ? max_states : 5000000, &times, &lens,
                                &tr)))
        return rc;
    *n_traces = (int64_t)times.size();
    *trace_len = (int64_t)(tr.size() / 4);
    if (rows)
        for (size_t i = 0; i < times.size() && (int64_t)i < rows_cap; ++i) {
            rows[2 * i] = times[i];
            rows[2 * i + 1] = lens[i];
        }
    if (trace) std::memcpy(trace, tr.data(), std::min<int64_t>(trace_cap, *trace_len) * 16);
    if ((int64_t)times.size() > rows_cap || *trace_len > trace_cap) {
        set_error("check_nontermination: trace buffers too small");
        return MCTB_LIMIT;
    }
    return MCTB_OK;
}
