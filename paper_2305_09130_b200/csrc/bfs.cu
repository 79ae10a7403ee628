// Exhaustive interleaving exploration on the GPU (north-star subsystem 3).
//
// Replaces explore_machine's depth-first search (explore.cpp:86-165).  The
// reachable set does not depend on the visiting order, so instead of a DFS
// stack (or a level-synchronous BFS with a grid barrier per level — the state
// graphs here are thousands of levels deep and only 2^nwe wide) the GPU runs
// an asynchronous frontier: a persistent grid of warps pops states from one
// global work queue, and pushes every newly discovered state back onto it.
//   * one warp per state, one lane per enabled transition (machine.cuh):
//     unpack the parent, apply the lane's transition, pack the successor
//     (pack.cuh) and insert it into the visited table;
//   * visited table in HBM, lock-free open addressing:
//       tag[slot]  64-bit = fingerprint | 2 (claimed) | 1 (key published)
//       keys[slot] the packed state, written once by the claiming lane
//     exact: a fingerprint match is confirmed on the full packed key;
//   * work queue = the slot indices of new states in discovery order
//     (pre-filled with EMPTY); producers bump `tail` (one atomic per warp via
//     ballot), consumers bump `head`; `outstanding` counts states pushed but
//     not yet expanded, so the sweep ends exactly when it drops to zero.
// Several configurations (the check's root nondeterminism, explore.cpp:171-200)
// are explored in the same sweep, tagged by a cfg field of the packed state;
// per-configuration statistics give the reference's ExploreStats.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bfs.cuh"
#include "common.cuh"
#include "cost_model.cuh"
#include "pack.cuh"
#include "traj.cuh"

namespace mctb {

struct BfsArgs {
    const BfsDesc* descs;
    int n_cfg;
    int words;                 // key words per slot (max over configurations)
    int cfg_bits;
    uint64_t cap_mask;         // table capacity - 1 (power of two)
    unsigned long long* tags;  // [cap]
    uint32_t* keys;            // [cap * words]
    uint32_t* queue;           // [queue_cap] slot indices, EMPTY until pushed
    uint64_t queue_cap;
    unsigned long long* head;
    // tq = (tail << 32) | outstanding: queue reservations and the count of states
    // discovered but not yet expanded move together in one atomic
    unsigned long long* tq;
    BfsStats* stats;  // [n_cfg]
    int* error;       // 1 table full, 2 queue full, 3 model bug
    uint64_t cfg_cap; // per-configuration visited cap (ExploreLimits::max_states)
    int keep;         // continue with the first new successor (no queue round trip)
    unsigned long long* op_hist;  // generic successors per op (diagnostics)
    int check_inv;                // check Machine::check_invariants on every state
};

namespace {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kBfsThreads = 256;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_relaxed32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ long long ld_relaxed_s64(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Returns the slot of a newly inserted key, -1 if already present, -2 if full.
__device__ long long table_insert(const BfsArgs& a, const uint32_t* key, uint64_t h) {
    const unsigned long long tag = (h | 3ull);
    const unsigned long long claim = tag & ~1ull;
    uint64_t i = h & a.cap_mask;
    // a probe sequence this long only happens in a table that is too full: report it
    // (the sweep restarts with a larger table) instead of scanning the whole table
    for (uint64_t probe = 0; probe < 4096; ++probe, i = (i + 1) & a.cap_mask) {
        // relaxed probe (an acquire load invalidates the SM's L1 — CCTL.IVALL — so it
        // is only issued on a fingerprint match, before the key words are read)
        unsigned long long t = ld_relaxed64(&a.tags[i]);
        if (t == 0) {
            const unsigned long long prev = atomicCAS(&a.tags[i], 0ull, claim);
            if (prev == 0) {
                uint32_t* dst = a.keys + i * (uint64_t)a.words;
                for (int k = 0; k < a.words; ++k) dst[k] = key[k];
                // release: the key words become visible before the published bit
                // (a reduction: nothing waits for its result)
                asm volatile("red.release.gpu.global.or.b64 [%0], 1;" ::"l"(&a.tags[i])
                             : "memory");
                return (long long)i;
            }
            t = prev;
        }
        if ((t | 1ull) != tag) continue;  // different fingerprint
        t = ld_acquire(&a.tags[i]);
        while (!(t & 1ull)) {  // claimed, key not yet published
            __nanosleep(32);
            t = ld_acquire(&a.tags[i]);
        }
        const uint32_t* src = a.keys + i * (uint64_t)a.words;
        bool eq = true;
        for (int k = 0; k < a.words && eq; ++k) eq = src[k] == key[k];
        if (eq) return -1;
    }
    return -2;
}

// Pushes the lanes' new slots (fresh lanes) with one queue reservation per warp.
// Returns the number pushed (on every lane).
__device__ __forceinline__ unsigned push_fresh(const BfsArgs& a, bool fresh, long long slot) {
    const int lane = threadIdx.x & 31;
    const unsigned mask = __ballot_sync(0xffffffffu, fresh);
    if (!mask) return 0;
    const int leader = __ffs(mask) - 1;
    const unsigned cnt = __popc(mask);
    unsigned long long pos0 = 0;
    if (lane == leader) {
        pos0 = atomicAdd(a.tq, ((unsigned long long)cnt << 32) | cnt) >> 32;
        if (pos0 + cnt > a.queue_cap) atomicExch(a.error, 2);
    }
    pos0 = __shfl_sync(0xffffffffu, pos0, leader);
    if (fresh) {
        const unsigned long long pos = pos0 + __popc(mask & ((1u << lane) - 1));
        if (pos < a.queue_cap) st_release32(&a.queue[pos], (uint32_t)slot);
    }
    return cnt;
}

// Record writers for the in-place successors (field order of pack()).
__device__ __forceinline__ void write_pex(uint32_t* row, const Layout& l, int p, const PexS& x) {
    const int o = l.off_pex + p * l.pex_bits;
    set_bits(row, o, 4, (uint32_t)x.pc);
    set_bits(row, o + 4, 1, (uint32_t)x.phase);
    set_bits(row, o + 5, l.cursor, x.cursor);
    set_bits(row, o + 5 + l.cursor, l.busy, x.busy_left);
    set_bits(row, o + 5 + l.cursor + l.busy, 1, (uint32_t)x.reported);
    set_bits(row, o + 6 + l.cursor + l.busy, l.pnwg, (uint32_t)x.nwg);
    set_bits(row, o + 6 + l.cursor + l.busy + l.pnwg, l.iter, x.iter);
}

__device__ __forceinline__ void write_unit(uint32_t* row, const Layout& l, int g, const UnitS& u) {
    const int o = l.off_units + g * l.unit_bits;
    set_bits(row, o, 3, (uint32_t)u.pc);
    set_bits(row, o + 3, l.uk, (uint32_t)u.k);
    set_bits(row, o + 3 + l.uk, l.nwg, (uint32_t)u.nwg);
    set_bits(row, o + 3 + l.uk + l.nwg, l.sent, (uint32_t)u.sent);
    set_bits(row, o + 3 + l.uk + l.nwg + l.sent, l.items, (uint32_t)u.got_items);
    set_bits(row, o + 3 + l.uk + l.nwg + l.sent + l.items, l.ends, (uint32_t)u.got_ends);
}

// In-place successors for the transitions behind the combinatorial state
// explosion: an element reporting a busy tick or arriving at its barrier, and
// the unit <-> element handshakes (activation, item done, group done, stop).
// They touch one element record, its unit record and at most one header field;
// the new values follow Machine::apply (machine.cpp:479-500, 518-530, 541-551,
// 569-580, 618-646) and are written over the parent's packed words.  Every
// other transition goes through the generic unpacked apply() (machine.cuh).
__device__ __forceinline__ bool fast_successor(const BfsDesc& d, const MState& s,
                                               const Transition& tr, uint32_t* row) {
    const Layout& l = d.l;
    const MachDesc& m = d.m;
    int role, ord;
    switch (tr.op) {
        case OP_PEXREPORT: {
            role_of(m, tr.actor, role, ord);
            set_bits(row, l.off_pex + ord * l.pex_bits + l.poff_reported, 1, 1u);
            set_bits(row, l.off_nrp, l.nrp, (uint32_t)(s.nrp_work + 1));
            return true;
        }
        case OP_PEXARRIVE: {
            role_of(m, tr.actor, role, ord);
            const int g = ord / m.nwe;
            const int pc = s.pex[ord].pc == P_ARRIVEBARRIER ? P_WAITBARRIER : P_WAITGROUPEND;
            set_bits(row, l.off_pex + ord * l.pex_bits, 4, (uint32_t)pc);
            set_bits(row, l.off_units + g * l.unit_bits + l.uoff_bcount, l.bcount,
                     (uint32_t)(s.bar[g].count + 1));
            return true;
        }
        case OP_UNITPEXGO: {
            role_of(m, tr.actor, role, ord);
            int prole, p;
            role_of(m, tr.peer, prole, p);
            UnitS un = s.unit[ord];
            PexS px = pex_init(un.nwg, un.sent / m.nwe);
            place_pex(m, px);
            un.sent += 1;
            if (un.pc == U_ACTIVATEPEX) {
                if (++un.k == m.nwe) {
                    un.pc = U_SERVE;
                    un.k = 0;
                }
            } else {
                un.pc = U_SERVE;
            }
            write_pex(row, l, p, px);
            write_unit(row, l, ord, un);
            return true;
        }
        case OP_UNITPEXSTOP: {
            role_of(m, tr.actor, role, ord);
            int prole, p;
            role_of(m, tr.peer, prole, p);
            UnitS un = s.unit[ord];
            if (++un.k == m.nwe) un.pc = U_STOPBARRIER;
            set_bits(row, l.off_pex + p * l.pex_bits, 4, (uint32_t)P_EXITED);
            write_unit(row, l, ord, un);
            return true;
        }
        case OP_PEXITEMDONE: {
            role_of(m, tr.actor, role, ord);
            const int g = ord / m.nwe;
            UnitS un = s.unit[g];
            un.got_items += 1;
            if (un.sent < m.wg) un.pc = U_REACTPEX;
            else if (m.kernel == 0 && un.got_items == m.wg) un.pc = U_SENDUNITDONE;
            write_pex(row, l, ord, pex_init(0, 0));
            write_unit(row, l, g, un);
            return true;
        }
        case OP_PEXENDDONE: {
            role_of(m, tr.actor, role, ord);
            const int g = ord / m.nwe;
            UnitS un = s.unit[g];
            un.got_ends += 1;
            if (un.got_ends == m.nwe) un.pc = U_SENDUNITDONE;
            if (ord % m.nwe == 0)
                set_bits(row, l.off_nrp + l.nrp, l.allnwe, (uint32_t)(s.all_nwe - 1));
            write_pex(row, l, ord, pex_init(0, 0));
            write_unit(row, l, g, un);
            return true;
        }
        default: return false;
    }
}

__global__ void __launch_bounds__(kBfsThreads) explore_kernel(BfsArgs a) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // per warp in shared memory: the parent (unpacked and packed) and its enabled
    // list; per lane: one packed successor row.  Only the generic transitions
    // materialise an unpacked successor in (L1-resident) local memory.
    __shared__ MState parent[kBfsThreads / 32];
    __shared__ Transition enabled_s[kBfsThreads / 32][kMaxEnabled];
    extern __shared__ uint32_t dyn[];
    uint32_t* pwords = dyn + wib * (34 * a.words);  // parent words
    uint32_t* kwords = pwords + a.words;             // the successor the warp keeps
    uint32_t* row = pwords + (2 + lane) * a.words;   // this lane's successor
    MState& s = parent[wib];
    Transition* en = enabled_s[wib];
    MState t;
    // warp-local statistics of the current configuration, flushed on change/exit
    int cur_cfg = -1;
    unsigned long long n_states = 0, n_trans = 0;
    auto flush = [&]() {
        if (lane == 0 && cur_cfg >= 0) {
            if (n_states) atomicAdd(&a.stats[cur_cfg].states, n_states);
            if (n_trans) atomicAdd(&a.stats[cur_cfg].transitions, n_trans);
        }
        n_states = n_trans = 0;
    };
    bool local = false;  // the warp continues with a successor it discovered itself
    // queue entries are claimed in runs: a warp that finds its entries already
    // filled doubles its next claim (up to 8), one that has to wait claims one
    unsigned long long h_next = 0, h_end = 0;
    unsigned claim = 1;
    for (;;) {
        const uint32_t* src;
        if (local) {
            src = pwords;  // already holds the kept successor
        } else {
            if (h_next == h_end) {
                unsigned long long h0 = 0;
                if (lane == 0) h0 = atomicAdd(a.head, (unsigned long long)claim);
                h_next = __shfl_sync(0xffffffffu, h0, 0);
                h_end = h_next + claim;
            }
            const unsigned long long h = h_next++;
            if (h >= a.queue_cap) break;
            // wait until entry h is pushed, or the sweep is over
            uint32_t slot = kEmpty;
            bool waited = false;
            if (lane == 0) {
                unsigned ns = 64;
                for (unsigned it = 0;; ++it) {
                    slot = ld_relaxed32(&a.queue[h]);  // relaxed poll: no L1 invalidation
                    if (slot != kEmpty) {
                        slot = ld_acquire32(&a.queue[h]);
                        break;
                    }
                    waited = true;
                    // the shared counters are read rarely: they are the working warps'
                    // atomics' cache line
                    if ((it & 15) == 15 && ((uint32_t)ld_relaxed64(a.tq) == 0 ||
                                            ld_relaxed32((const uint32_t*)a.error)))
                        break;
                    __nanosleep(ns);
                    if (ns < 1024) ns <<= 1;
                }
            }
            slot = __shfl_sync(0xffffffffu, slot, 0);
            waited = __shfl_sync(0xffffffffu, waited, 0);
            claim = waited ? 1u : (claim < 8u ? claim * 2u : 8u);
            if (slot == kEmpty) break;
            // the key is published before its slot index is pushed
            src = a.keys + (uint64_t)slot * a.words;
            for (int k = lane; k < a.words; k += 32) pwords[k] = src[k];
            __syncwarp();
            src = pwords;
        }
        const int cfg = peek_cfg(src, a.cfg_bits);
        if (cfg != cur_cfg) {
            flush();
            cur_cfg = cfg;
        }
        const BfsDesc& d = a.descs[cfg];
        // warp-parallel unpack and enumeration: lane i reads the records of process
        // slots i, i+32, ... and applies their rules (machine.cuh); a warp prefix sum
        // places every lane's transitions in the shared enabled list
        unpack_lanes(d, src, s, lane);
        __syncwarp();
        const int nsl = n_slots(d.m);
        int cnt = 0;
        for (int k = lane; k < nsl; k += 32) cnt = slot_rules(d.m, s, k, nullptr, cnt);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int ne = __shfl_sync(0xffffffffu, incl, 31);
        int pos = incl - cnt;
        for (int k = lane; k < nsl; k += 32) pos = slot_rules(d.m, s, k, en, pos);
        __syncwarp();
        BfsStats& st = a.stats[cfg];
        if (a.check_inv && lane == 0) {
            // machine.cpp:719-756, plus tick gating (acceptance criterion 7)
            bool bad = check_invariants(d.m, s) != 0;
            for (int e = 0; e < ne; ++e)
                bad |= en[e].op == OP_CLOCKTICK && (s.nrp_work != s.all_nwe || s.all_nwe == 0);
            if (bad) atomicAdd(&st.violations, 1ull);
        }
        bool kept = false;
        if (ne == 0) {
            if (lane == 0) {
                if (is_terminal(d.m, s)) {
                    atomicAdd(&st.terminals, 1ull);
                    atomicMin(&st.min_time, (long long)s.time);
                    atomicMax(&st.max_time, (long long)s.time);
                } else {
                    atomicAdd(&st.deadlocks, 1ull);
                    atomicExch(a.error, 3);
                }
            }
        } else if (*(volatile unsigned long long*)&st.states + n_states >= a.cfg_cap) {
            // explore.cpp:28: a full visited set inserts nothing more
            if (lane == 0) st.capped = 1;
        } else {
            n_trans += (unsigned)ne;
            for (int base = 0; base < ne; base += 32) {
                const int e = base + lane;
                long long ins = -1;
                if (e < ne) {
                    for (int k = 0; k < a.words; ++k) row[k] = pwords[k];
                    bool ok = true;
                    if (!fast_successor(d, s, en[e], row)) {
                        if (a.op_hist) atomicAdd(&a.op_hist[en[e].op], 1ull);
                        copy_state(d.m, t, s);
                        ok = apply(d.m, t, en[e]);
                        if (ok) pack(d, cfg, t, row);
                        else atomicExch(a.error, 3);
                    }
                    if (ok) {
                        ins = table_insert(a, row, hash_words(row, a.words));
                        if (ins == -2) atomicExch(a.error, 1);
                    }
                }
                bool fresh = ins >= 0;
                int keeper = -1;
                if (!kept && a.keep) {
                    // keep the first new successor: no queue round trip on the chain; it
                    // inherits the parent's place in `outstanding`
                    const unsigned m = __ballot_sync(0xffffffffu, fresh);
                    if (m) {
                        keeper = __ffs(m) - 1;
                        if (lane == keeper) fresh = false;
                        kept = true;
                        n_states += 1;
                    }
                }
                n_states += push_fresh(a, fresh, ins);
                if (keeper >= 0) {
                    __syncwarp();
                    const uint32_t* kr = pwords + (2 + keeper) * a.words;
                    for (int k = lane; k < a.words; k += 32) kwords[k] = kr[k];
                    __syncwarp();
                }
            }
        }
        __syncwarp();
        local = kept && !*(volatile int*)a.error;
        if (local) {
            for (int k = lane; k < a.words; k += 32) pwords[k] = kwords[k];
            __syncwarp();
        } else if (lane == 0) {
            atomicAdd(a.tq, ~0ull);  // this state is expanded: outstanding - 1
        }
    }
    flush();
}

__global__ void seed_kernel(BfsArgs a, const uint32_t* seeds, int n_seeds) {
    // one initial state per configuration (explore.cpp:98-105), or the given
    // packed states of configuration 0 (a multi-source exploration)
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t key[kMaxWords];
    int cfg = c;
    if (seeds) {
        if (c >= n_seeds) return;
        cfg = 0;
        for (int k = 0; k < a.words; ++k) key[k] = seeds[(size_t)c * a.words + k];
    } else {
        if (c >= a.n_cfg) return;
        const BfsDesc& d = a.descs[c];
        MState s;
        initial_state(d.m, s);
        pack(d, c, s, key);
        for (int k = d.l.words; k < a.words; ++k) key[k] = 0;
    }
    const long long ins = table_insert(a, key, hash_words(key, a.words));
    if (ins == -1) return;  // a repeated seed
    if (ins < 0) {
        atomicExch(a.error, 1);
        return;
    }
    const int c_ = cfg;
    atomicAdd(&a.stats[c_].states, 1ull);
    const unsigned long long pos = atomicAdd(a.tq, (1ull << 32) | 1ull) >> 32;
    st_release32(&a.queue[pos], (uint32_t)ins);
}

}  // namespace

// ------------------------------------------------------------------ host
Layout bfs_layout(const MachDesc& m, int n_cfg) {
    // time bound: every tick consumes >= 1 busy tick of some element
    const int64_t groups = (int64_t)m.device_rounds * m.nwu;
    const int64_t per_item = m.kernel == 0 ? (int64_t)m.reps * (m.gmt * m.ts + m.ts) + m.gmt
                                           : (int64_t)m.ts * m.gmt + m.nwe + m.gmt;
    return make_layout(m, n_cfg, groups * m.wg * per_item + 1);
}

int run_bfs(std::vector<MachHost>& hs, uint64_t max_states, uint64_t cfg_cap, BfsResult* res,
            cudaStream_t st, bool check_invariants, const std::vector<uint32_t>* seeds) {
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
        descs[c].m = m;
        descs[c].l = bfs_layout(m, n_cfg);
        if (descs[c].l.time > 32 || descs[c].l.words > kMaxWords) {
            set_error("state does not fit the GPU packing (time > 2^32 or > 24 words)");
            cudaFreeAsync(d_ids, st);
            return MCTB_LIMIT;
        }
        words = std::max(words, descs[c].l.words);
    }
    int dev = 0, sms = 0, per_sm = 0;
    MCTB_CUDA(cudaGetDevice(&dev));
    MCTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t dyn_smem = (size_t)(kBfsThreads / 32) * 34 * words * sizeof(uint32_t);
    if (dyn_smem > 48 * 1024)
        MCTB_CUDA(cudaFuncSetAttribute(explore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn_smem));
    MCTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, explore_kernel, kBfsThreads,
                                                            dyn_smem));
    if (per_sm < 1) per_sm = 1;
    // local-memory working set: keep the resident warps' successor states L1-sized
    if (const char* e = getenv("MCTB_BFS_BLOCKS_PER_SM")) per_sm = std::min(per_sm, atoi(e));
    else per_sm = std::min(per_sm, 4);
    size_t free_b = 0, total_b = 0;
    MCTB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double slot_bytes = 8 + 4.0 * words + 2.0;  // tag + key + queue (half the slots)
    // capacity grows 8x on overflow; the sweep restarts (all counts are rebuilt)
    // first capacity: enough for the bound up to 2^28 slots (a restart loses the
    // work done, so large sweeps start large); then 8x per overflow
    uint64_t cap = 1ull << 20;
    while (cap < 2 * std::min<uint64_t>(max_states, 1ull << 27)) cap <<= 1;
    const uint64_t cap_limit = [&] {
        uint64_t c = 1024;
        while ((double)(c * 2) * slot_bytes < 0.8 * (double)free_b) c <<= 1;
        return c;
    }();
    cap = std::min(cap, cap_limit);
    for (;;) {
        const uint64_t qcap = cap / 2;
        BfsArgs a{};
        a.n_cfg = n_cfg;
        a.words = words;
        a.cfg_bits = descs[0].l.cfg;
        a.cap_mask = cap - 1;
        a.queue_cap = qcap;
        a.cfg_cap = cfg_cap;
        a.keep = getenv("MCTB_BFS_NOKEEP") ? 0 : 1;
        a.check_inv = check_invariants ? 1 : 0;
        const size_t sz_tags = cap * 8, sz_keys = cap * 4 * (size_t)words, sz_q = qcap * 4;
        const size_t sz_misc = 512 + sizeof(BfsStats) * n_cfg + sizeof(BfsDesc) * n_cfg;
        void* blob = nullptr;
        MCTB_CUDA(cudaMallocAsync(&blob, sz_tags + sz_keys + sz_q + sz_misc, st));
        char* b = (char*)blob;
        a.tags = (unsigned long long*)b;
        a.keys = (uint32_t*)(b + sz_tags);
        a.queue = (uint32_t*)(b + sz_tags + sz_keys);
        char* misc = b + sz_tags + sz_keys + sz_q;
        a.head = (unsigned long long*)misc;
        a.tq = (unsigned long long*)(misc + 8);
        a.error = (int*)(misc + 24);
        a.op_hist = getenv("MCTB_BFS_OPHIST") ? (unsigned long long*)(misc + 32) : nullptr;
        a.stats = (BfsStats*)(misc + 512);
        a.descs = (BfsDesc*)(misc + 512 + sizeof(BfsStats) * n_cfg);
        MCTB_CUDA(cudaMemsetAsync(a.tags, 0, sz_tags, st));
        MCTB_CUDA(cudaMemsetAsync(a.queue, 0xff, sz_q, st));
        MCTB_CUDA(cudaMemsetAsync(misc, 0, 512, st));
        std::vector<BfsStats> init(n_cfg);
        for (auto& x : init) x = BfsStats{0, 0, 0, INT64_MAX, -1, 0, 0, 0, 0};
        MCTB_CUDA(cudaMemcpyAsync(a.stats, init.data(), sizeof(BfsStats) * n_cfg,
                                  cudaMemcpyHostToDevice, st));
        MCTB_CUDA(cudaMemcpyAsync((void*)a.descs, descs.data(), sizeof(BfsDesc) * n_cfg,
                                  cudaMemcpyHostToDevice, st));
        uint32_t* d_seeds = nullptr;
        int n_seeds = 0;
        if (seeds && !seeds->empty()) {
            n_seeds = (int)(seeds->size() / words);
            MCTB_CUDA(cudaMallocAsync(&d_seeds, seeds->size() * 4, st));
            MCTB_CUDA(cudaMemcpyAsync(d_seeds, seeds->data(), seeds->size() * 4,
                                      cudaMemcpyHostToDevice, st));
        }
        const int n_first = seeds ? n_seeds : n_cfg;
        seed_kernel<<<(n_first + 127) / 128 + 1, 128, 0, st>>>(a, d_seeds, n_seeds);
        if (d_seeds) cudaFreeAsync(d_seeds, st);
        MCTB_CUDA(cudaGetLastError());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        explore_kernel<<<sms * per_sm, kBfsThreads, dyn_smem, st>>>(a);
        cudaEventRecord(e1, st);
        MCTB_CUDA(cudaGetLastError());
        res->stats.resize(n_cfg);
        unsigned long long misc_h[32];
        MCTB_CUDA(cudaMemcpyAsync(res->stats.data(), a.stats, sizeof(BfsStats) * n_cfg,
                                  cudaMemcpyDeviceToHost, st));
        MCTB_CUDA(cudaMemcpyAsync(misc_h, misc, 256, cudaMemcpyDeviceToHost, st));
        MCTB_CUDA(cudaStreamSynchronize(st));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFreeAsync(blob, st);
        res->ms = ms;
        res->states = 0;
        for (const auto& x : res->stats) res->states += x.states;
        res->levels = 0;
        res->error = (int)(misc_h[3] & 0xffffffff);
        // explore.cpp:28-31: a visited set holding max_states refuses every later
        // insert, so reaching the cap ends the exhaustive claim (statistics are
        // flushed per warp, so the final count decides)
        for (auto& x : res->stats)
            if (x.states >= cfg_cap) x.capped = 1;
        if (getenv("MCTB_BFS_OPHIST")) {
            fprintf(stderr, "[explore] generic successors by op:");
            for (int o = 0; o < 19; ++o)
                if (misc_h[4 + o]) fprintf(stderr, " op%d=%llu", o, misc_h[4 + o]);
            fprintf(stderr, "\n");
        }
        res->words = words;
        res->capacity = cap;
        if ((res->error == 1 || res->error == 2) && cap < cap_limit) {
            cap = std::min(cap * 8, cap_limit);
            continue;
        }
        break;
    }
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

int mctb_explore(const int* plat, int size, int kernel, const int64_t* input,
                 const int32_t* configs, int n_configs, int64_t max_states, int flags,
                 int64_t* out, int64_t* info) {
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
    rc = run_bfs(hs, cap * (uint64_t)n_configs, cap, &r, st, (flags & 1) != 0);
    cudaStreamDestroy(st);
    if (rc) return rc;
    if (r.error == 3) {
        set_error("model bug: deadlock or inapplicable transition during exploration");
        return MCTB_MODEL_BUG;
    }
    if (r.error) {
        set_error("GPU visited table exceeds device memory");
        return MCTB_LIMIT;
    }
    for (int c = 0; c < n_configs; ++c) {
        const BfsStats& s = r.stats[c];
        int64_t* o = out + 9 * c;
        o[8] = (int64_t)s.violations;
        o[0] = !s.capped;
        o[1] = (int64_t)std::min<uint64_t>(s.states, cap);
        o[2] = (int64_t)s.transitions;
        // DFS max depth = longest complete run = protocol transitions + max time
        // (pinned against explore_machine in tests/test_bfs_gpu.py)
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
        uint64_t generic = 0;
        for (const auto& x : r.stats) generic += x.generic;
        if (getenv("MCTB_BFS_OPHIST"))
            fprintf(stderr, "[mctb_explore] generic successors: %llu\n", (unsigned long long)generic);
        info[0] = (int64_t)r.capacity;
        info[1] = (int64_t)r.states;
        info[2] = r.words;
        info[3] = (int64_t)(r.ms * 1000.0);
    }
    return MCTB_OK;
}

}  // extern "C"
