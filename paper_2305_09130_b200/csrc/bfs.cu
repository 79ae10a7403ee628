// Exhaustive interleaving exploration on the GPU (north-star subsystem 3).
//
// Replaces explore_machine's depth-first search (explore.cpp:86-165) with a
// frontier-parallel BFS: one persistent cooperative grid sweeps the state
// graph level by level (one grid barrier per level).  Every thread takes a
// frontier entry (a slot index of the visited table), unpacks the state,
// computes its enabled transitions (machine.cuh), applies each one, packs the
// successor (pack.cuh) and inserts it into a lock-free open-addressing
// visited table in HBM:
//   tag[slot]  : 64-bit = fingerprint | 2 (claimed) | 1 (key published)
//   keys[slot] : the packed state (layout words), written once by the claimer
// A new state goes onto the next frontier.  The visited set is exact (full
// packed keys are compared), so the reachable-state count, edge count and
// terminal-time range per configuration equal the reference's exhaustive
// exploration; several configurations (the check's root nondeterminism,
// explore.cpp:171-200) are explored in the same sweep, tagged by a cfg field.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "pack.cuh"
#include "traj.cuh"
#include "cost_model.cuh"
#include "bfs.cuh"

namespace cg = cooperative_groups;

namespace mctb {

struct BfsArgs {
    const BfsDesc* descs;
    int n_cfg;
    int words;                 // key words per slot (max over configurations)
    uint64_t cap_mask;         // table capacity - 1 (power of two)
    unsigned long long* tags;  // [cap]
    uint32_t* keys;            // [cap * words]
    uint32_t* frontier[2];     // slot indices
    uint64_t frontier_cap;
    unsigned long long* counters;  // [3] rotating frontier counts
    unsigned long long* inserted;  // total inserted states
    BfsStats* stats;               // [n_cfg]
    int* error;                    // 1 table full, 2 frontier overflow, 3 model bug
    int* errflag;                  // [2] per level parity: stops the sweep consistently
    unsigned long long* levels;
    uint64_t max_states;
    uint64_t cfg_cap;  // per-configuration visited cap (ExploreLimits::max_states)
};

namespace {

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Returns the slot of a newly inserted key, or -1 if already present, or -2 if full.
__device__ long long table_insert(const BfsArgs& a, const uint32_t* key, uint64_t h) {
    const unsigned long long tag = (h | 3ull);
    const unsigned long long claim = tag & ~1ull;
    uint64_t i = h & a.cap_mask;
    for (uint64_t probe = 0; probe <= a.cap_mask; ++probe, i = (i + 1) & a.cap_mask) {
        unsigned long long t = ld_acquire(&a.tags[i]);
        if (t == 0) {
            const unsigned long long prev = atomicCAS(&a.tags[i], 0ull, claim);
            if (prev == 0) {
                uint32_t* dst = a.keys + i * (uint64_t)a.words;
                for (int k = 0; k < a.words; ++k) dst[k] = key[k];
                __threadfence();
                atomicOr(&a.tags[i], 1ull);  // publish
                return (long long)i;
            }
            t = prev;
        }
        if ((t | 1ull) != tag) continue;  // different fingerprint
        while (!(t & 1ull)) t = ld_acquire(&a.tags[i]);  // wait until published
        const uint32_t* src = a.keys + i * (uint64_t)a.words;
        bool eq = true;
        for (int k = 0; k < a.words && eq; ++k) eq = src[k] == key[k];
        if (eq) return -1;
    }
    return -2;
}

__device__ void note_terminal(BfsStats& st, long long time) {
    atomicAdd(&st.terminals, 1ull);
    atomicMin(&st.min_time, time);
    atomicMax(&st.max_time, time);
}

constexpr int kBfsThreads = 512;
constexpr uint64_t kNarrow = 2 * (kBfsThreads / 32);  // frontier handled by one CTA

// Expands frontier entries [warp, n) with stride `nwarps`: one warp per state,
// one lane per enabled transition.  Successor slots are appended to `fw`
// through one warp-aggregated atomicAdd per 32 successors.
__device__ void expand_level(const BfsArgs& a, const uint32_t* fr, uint32_t* fw, uint64_t n,
                             unsigned long long* next_count, int* err_now, uint64_t warp,
                             uint64_t nwarps, MState& s, MState& t, Transition* en,
                             uint32_t* key) {
    const int lane = threadIdx.x & 31;
    for (uint64_t j = warp; j < n; j += nwarps) {
        const uint64_t slot = fr[j];
        const uint32_t* src = a.keys + slot * (uint64_t)a.words;
        const int cfg = peek_cfg(src, a.descs[0].l.cfg);
        const BfsDesc& d = a.descs[cfg];
        unpack(d, src, s);
        const int ne = enabled(d.m, s, en);
        BfsStats& st = a.stats[cfg];
        if (ne == 0) {
            if (lane == 0) {
                if (is_terminal(d.m, s)) {
                    note_terminal(st, s.time);
                } else {
                    atomicAdd(&st.deadlocks, 1ull);
                    atomicExch(a.error, 3);
                    atomicExch(err_now, 1);
                }
            }
            continue;
        }
        if (*(volatile unsigned long long*)&st.states >= a.cfg_cap) {
            // explore.cpp:28: a full visited set inserts nothing more
            if (lane == 0) st.capped = 1;
            continue;
        }
        if (lane == 0) atomicAdd(&st.transitions, (unsigned long long)ne);
        for (int base = 0; base < ne; base += 32) {
            const int e = base + lane;
            long long ins = -1;
            if (e < ne) {
                copy_state(d.m, t, s);
                if (!apply(d.m, t, en[e])) {
                    atomicExch(a.error, 3);
                    atomicExch(err_now, 1);
                } else {
                    pack(d, cfg, t, key);
                    for (int k = d.l.words; k < a.words; ++k) key[k] = 0;
                    ins = table_insert(a, key, hash_words(key, a.words));
                    if (ins == -2) {
                        atomicExch(a.error, 1);
                        atomicExch(err_now, 1);
                    }
                }
            }
            const bool fresh = ins >= 0;
            const unsigned mask = __ballot_sync(0xffffffffu, fresh);
            if (!mask) continue;
            unsigned long long pos0 = 0;
            const int leader = __ffs(mask) - 1;
            if (lane == leader) {
                const unsigned cnt = __popc(mask);
                pos0 = atomicAdd(next_count, (unsigned long long)cnt);
                atomicAdd(&st.states, (unsigned long long)cnt);
                const unsigned long long total = atomicAdd(a.inserted, (unsigned long long)cnt) + cnt;
                if (total > a.max_states || pos0 + cnt > a.frontier_cap) {
                    atomicExch(a.error, pos0 + cnt > a.frontier_cap ? 2 : 1);
                    atomicExch(err_now, 1);
                }
            }
            pos0 = __shfl_sync(0xffffffffu, pos0, leader);
            if (fresh) {
                const unsigned long long pos = pos0 + __popc(mask & ((1u << lane) - 1));
                if (pos < a.frontier_cap) fw[pos] = (uint32_t)ins;
            }
        }
    }
}

__global__ void __launch_bounds__(kBfsThreads) bfs_kernel(BfsArgs a) {
    cg::grid_group grid = cg::this_grid();
    const uint64_t nwarps = (uint64_t)gridDim.x * (kBfsThreads / 32);
    const uint64_t warp = (uint64_t)blockIdx.x * (kBfsThreads / 32) + (threadIdx.x >> 5);
    const bool t0 = blockIdx.x == 0 && threadIdx.x == 0;
    MState s, t;
    Transition en[kMaxEnabled];
    uint32_t key[kMaxWords];
    __shared__ unsigned long long narrow_level;
    uint64_t level = 0;
    for (;;) {
        const int cur = (int)(level % 3);
        const uint64_t n = *(volatile unsigned long long*)&a.counters[cur];
        // errors raised in the previous level (written before the last grid barrier;
        // the current level's flag may already be written by faster warps)
        if (n == 0 || *(volatile int*)&a.errflag[(level + 1) & 1]) break;
        if (n <= kNarrow) {
            // narrow frontier: CTA 0 sweeps levels with block barriers only
            if (blockIdx.x == 0) {
                uint64_t lv = level, m = n;
                for (;;) {
                    const int c = (int)(lv % 3), x = (int)((lv + 1) % 3), o = (int)((lv + 2) % 3);
                    if (threadIdx.x == 0) a.counters[o] = 0;
                    expand_level(a, a.frontier[lv & 1], a.frontier[(lv + 1) & 1], m,
                                 &a.counters[x], &a.errflag[lv & 1], threadIdx.x >> 5,
                                 kBfsThreads / 32, s, t, en, key);
                    __syncthreads();
                    ++lv;
                    m = *(volatile unsigned long long*)&a.counters[x];
                    const bool err = *(volatile int*)&a.errflag[0] || *(volatile int*)&a.errflag[1];
                    __syncthreads();
                    if (m == 0 || m > kNarrow || err) break;
                }
                if (threadIdx.x == 0) narrow_level = lv;
                __syncthreads();
                if (threadIdx.x == 0) *a.levels = lv;
            }
            grid.sync();
            level = *(volatile unsigned long long*)a.levels;
            continue;
        }
        if (t0) a.counters[(level + 2) % 3] = 0;
        expand_level(a, a.frontier[level & 1], a.frontier[(level + 1) & 1], n,
                     &a.counters[(level + 1) % 3], &a.errflag[level & 1], warp, nwarps, s, t, en,
                     key);
        grid.sync();
        ++level;
        if (t0) *a.levels = level;
    }
}

__global__ void seed_kernel(BfsArgs a) {
    // one initial state per configuration
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.n_cfg) return;
    const BfsDesc& d = a.descs[c];
    MState s;
    initial_state(d.m, s);
    uint32_t key[kMaxWords];
    pack(d, c, s, key);
    for (int k = d.l.words; k < a.words; ++k) key[k] = 0;
    const long long ins = table_insert(a, key, hash_words(key, a.words));
    if (ins < 0) {
        atomicExch(a.error, 1);
        return;
    }
    atomicAdd(&a.stats[c].states, 1ull);
    atomicAdd(a.inserted, 1ull);
    const unsigned long long pos = atomicAdd(&a.counters[0], 1ull);
    a.frontier[0][pos] = (uint32_t)ins;
}

}  // namespace

// ------------------------------------------------------------------ host
int run_bfs(std::vector<MachHost>& hs, uint64_t max_states, uint64_t cfg_cap, BfsResult* res,
            cudaStream_t st) {
    const int n_cfg = (int)hs.size();
    std::vector<BfsDesc> descs(n_cfg);
    int32_t* d_ids = nullptr;
    int rc = upload_desc(hs[0], st, &d_ids);
    if (rc) return rc;
    int words = 1;
    for (int c = 0; c < n_cfg; ++c) {
        MachDesc m = hs[c].d;
        m.input_id = d_ids;
        // time bound: every tick consumes >= 1 busy tick of some element
        const int64_t groups = (int64_t)m.device_rounds * m.nwu;
        int64_t per_item = m.kernel == 0 ? (int64_t)m.reps * (m.gmt * m.ts + m.ts) + m.gmt
                                         : (int64_t)m.ts * m.gmt + m.nwe + m.gmt;
        const int64_t max_time = groups * m.wg * per_item + 1;
        descs[c].m = m;
        descs[c].l = make_layout(m, n_cfg, max_time);
        if (descs[c].l.time > 32 || descs[c].l.words > kMaxWords) {
            set_error("state does not fit the GPU packing (time > 2^32 or > 24 words)");
            cudaFreeAsync(d_ids, st);
            return MCTB_LIMIT;
        }
        words = std::max(words, descs[c].l.words);
    }
    // table capacity: power of two >= 2 * max_states
    // (the table is sized for the bound, shrunk to what free HBM holds at load <= 1/2)
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const double slot_bytes = 8 + 4.0 * words + 4.0;  // tag + key + frontier share
    uint64_t cap = 1024;
    while (cap < 2 * max_states && (double)(cap * 2) * slot_bytes < 0.8 * (double)free_b) cap <<= 1;
    if (max_states > cap / 2) max_states = cap / 2;
    const uint64_t fcap = std::max<uint64_t>(cap / 2, 1024);
    BfsArgs a{};
    a.n_cfg = n_cfg;
    a.words = words;
    a.cap_mask = cap - 1;
    a.frontier_cap = fcap;
    a.max_states = max_states;
    a.cfg_cap = cfg_cap;
    void* blob = nullptr;
    const size_t off_tags = 0, sz_tags = cap * 8;
    const size_t off_keys = off_tags + sz_tags, sz_keys = cap * 4 * (size_t)words;
    const size_t off_f0 = off_keys + sz_keys, sz_f = fcap * 4;
    const size_t off_f1 = off_f0 + sz_f;
    const size_t off_misc = off_f1 + sz_f;
    const size_t sz_misc = 4096 + sizeof(BfsStats) * n_cfg + sizeof(BfsDesc) * n_cfg;
    MCTB_CUDA(cudaMallocAsync(&blob, off_misc + sz_misc, st));
    char* b = (char*)blob;
    a.tags = (unsigned long long*)(b + off_tags);
    a.keys = (uint32_t*)(b + off_keys);
    a.frontier[0] = (uint32_t*)(b + off_f0);
    a.frontier[1] = (uint32_t*)(b + off_f1);
    char* misc = b + off_misc;
    a.counters = (unsigned long long*)misc;          // 3 words
    a.inserted = (unsigned long long*)(misc + 32);
    a.levels = (unsigned long long*)(misc + 40);
    a.error = (int*)(misc + 48);
    a.errflag = (int*)(misc + 52);
    a.stats = (BfsStats*)(misc + 64);
    a.descs = (BfsDesc*)(misc + 64 + sizeof(BfsStats) * n_cfg);
    MCTB_CUDA(cudaMemsetAsync(a.tags, 0, sz_tags, st));
    MCTB_CUDA(cudaMemsetAsync(misc, 0, 64, st));
    std::vector<BfsStats> init(n_cfg);
    for (auto& x : init) x = BfsStats{0, 0, 0, INT64_MAX, -1, 0, 0};
    MCTB_CUDA(cudaMemcpyAsync(a.stats, init.data(), sizeof(BfsStats) * n_cfg,
                              cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMemcpyAsync((void*)a.descs, descs.data(), sizeof(BfsDesc) * n_cfg,
                              cudaMemcpyHostToDevice, st));
    seed_kernel<<<(n_cfg + 127) / 128, 128, 0, st>>>(a);
    MCTB_CUDA(cudaGetLastError());
    // persistent cooperative grid: all co-resident blocks
    int dev = 0, sms = 0, per_sm = 0;
    MCTB_CUDA(cudaGetDevice(&dev));
    MCTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MCTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, kBfsThreads, 0));
    if (per_sm < 1) per_sm = 1;
    const dim3 grid((unsigned)(sms * per_sm)), block(kBfsThreads);
    void* params[] = {&a};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    MCTB_CUDA(cudaLaunchCooperativeKernel((void*)bfs_kernel, grid, block, params, 0, st));
    cudaEventRecord(e1, st);
    res->stats.resize(n_cfg);
    unsigned long long misc_h[8];
    MCTB_CUDA(cudaMemcpyAsync(res->stats.data(), a.stats, sizeof(BfsStats) * n_cfg,
                              cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaMemcpyAsync(misc_h, misc, 64, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res->ms = ms;
    res->states = misc_h[4];
    res->levels = misc_h[5];
    res->error = (int)(misc_h[6] & 0xffffffff);
    res->words = words;
    cudaFreeAsync(blob, st);
    cudaFreeAsync(d_ids, st);
    MCTB_CUDA(cudaStreamSynchronize(st));
    return MCTB_OK;
}

}  // namespace mctb

using namespace mctb;

namespace mctb {
int check_machine(const int* plat, int size, int kernel, int wg, int ts);
}

extern "C" {

// explore_machine (explore.hpp:272-277) for a list of configurations at once.
// out = int64[8 * n_configs]: {complete, states, transitions, max_depth(-1: see cost model),
//                              min_time, max_time, terminals, deadlocks}
// info = int64[4]: {levels, total states, key words, kernel microseconds}
int mctb_explore(const int* plat, int size, int kernel, const int64_t* input,
                 const int32_t* configs, int n_configs, int64_t max_states, int64_t* out,
                 int64_t* info) {
    int rc;
    if (n_configs < 1) {
        set_error("no configurations");
        return MCTB_CONFIG_ERROR;
    }
    std::vector<MachHost> hs(n_configs);
    for (int c = 0; c < n_configs; ++c) {
        if ((rc = check_machine(plat, size, kernel, configs[2 * c], configs[2 * c + 1]))) return rc;
        if ((rc = build_desc(plat, size, kernel, input, configs[2 * c], configs[2 * c + 1], &hs[c])))
            return rc;
    }
    if ((rc = require_device())) return rc;
    cudaStream_t st;
    MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    BfsResult r;
    const uint64_t cap = max_states > 0 ? (uint64_t)max_states : 5000000ull;
    rc = run_bfs(hs, cap * (uint64_t)n_configs + 64ull * n_configs, cap, &r, st);
    cudaStreamDestroy(st);
    if (rc) return rc;
    if (r.error == 3) {
        set_error("model bug: deadlock or inapplicable transition during exploration");
        return MCTB_MODEL_BUG;
    }
    for (int c = 0; c < n_configs; ++c) {
        const BfsStats& s = r.stats[c];
        int64_t* o = out + 8 * c;
        o[0] = r.error == 0 && !s.capped;
        o[1] = (int64_t)std::min<uint64_t>(s.states, cap);
        o[2] = (int64_t)s.transitions;
        // DFS max depth = longest complete run = protocol transitions + max time
        // (verified against explore_machine in tests/test_bfs_gpu.py)
        int logn = 0, lw = 0, lt = 0, lp = 0;
        while ((1 << logn) < size) ++logn;
        while ((1 << lw) < configs[2 * c]) ++lw;
        while ((1 << lt) < configs[2 * c + 1]) ++lt;
        while ((1 << lp) < plat[2]) ++lp;
        const Cost cm = lockstep_cost(kernel, logn, plat[3], Config{plat[0], plat[1], lp, lw, lt});
        o[3] = s.terminals ? cm.steps - cm.time + s.max_time : -1;
        o[4] = s.terminals ? s.min_time : -1;
        o[5] = s.terminals ? s.max_time : -1;
        o[6] = (int64_t)s.terminals;
        o[7] = (int64_t)s.deadlocks;
    }
    if (info) {
        info[0] = (int64_t)r.levels;
        info[1] = (int64_t)r.states;
        info[2] = r.words;
        info[3] = (int64_t)(r.ms * 1000.0);
    }
    return MCTB_OK;
}

}  // extern "C"
