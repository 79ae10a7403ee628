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
//   * visited table in HBM, lock-free open addressing over 64- or 128-byte
//     slots: {key words, guard-filled padding, 64-bit tag}.  A probe is one
//     line read (tag and key in the same round trip); an empty tag is claimed
//     with a CAS and the claimer writes the key after it.  Key words carry a
//     guard bit (pack.cuh), so a reader that races the writer sees a word
//     without it and reads again — no release/acquire pair on the table;
//     exact: a tag match is confirmed on the full packed key;
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
#include <memory>
#include <mutex>
#include <vector>

#include "bfs.cuh"
#include "common.cuh"
#include "cost_model.cuh"
#include "bfs_rules.cuh"
#include "pack.cuh"
#include "traj.cuh"

namespace mctb {

constexpr int kMaxParts = 8;

// One hash partition of the visited set: its table, work queue and counters.
// A state belongs to partition owner(h) = (hi32(h) * P) >> 32; the partitions
// of a sweep live on one device (a single-GPU partitioned run) or one per GPU
// (peer memory over NVLink, bfs_mp.cu).
struct BfsPart {
    uint32_t* table;           // [cap * SW]: slot = {key, padding, tag}
    uint32_t* queue;           // [queue_cap] slot indices, EMPTY until pushed
    unsigned long long* head;
    // tq = (tail << 32) | outstanding: queue reservations and the count of states
    // discovered but not yet expanded move together in one atomic
    unsigned long long* tq;
    int* error;                // 1 table full, 2 queue full, 3 model bug, >= 5 watchdog
    uint32_t* depth;           // [cap] depth | guard of each slot's state (depth cap only)
};

struct BfsArgs {
    const BfsDesc* descs;
    int n_cfg;
    int words;                 // key words per slot (max over configurations)
    int cfg_bits;
    uint64_t cap_mask;         // table capacity - 1 (power of two), every partition
    uint64_t queue_cap;
    BfsPart part[kMaxParts];
    int n_parts;               // P
    int part0, n_here;         // partitions this launch expands: [part0, part0 + n_here)
    const uint2* ftab;     // [n_cfg * kMaxFields] field tables (bfs_rules.cuh)
    const int* nfields;    // [n_cfg]
    BfsStats* stats;  // [n_cfg]
    uint64_t cfg_cap; // per-configuration visited cap (ExploreLimits::max_states)
    int keep;         // continue with the first new successor (no queue round trip)
    unsigned long long* op_hist;  // generic successors per op (diagnostics)
    int check_inv;                // check Machine::check_invariants on every state
    unsigned flush_states;        // publish a warp's state count once it holds this many
    uint32_t depth_cap;           // ExploreLimits::max_depth (0: no state reaches it)
    int canon;                    // insert a report's successor from its canonical parent only
};

namespace {

#ifndef MCTB_BFS_MAX_SLEEP
#define MCTB_BFS_MAX_SLEEP 1024  // ns: longest back-off of an idle warp's queue poll
#endif

// Diagnostics build (-DMCTB_BFS_PHASES, with MCTB_BFS_OPHIST set): cycles per
// phase of an expansion, for queue-popped and chained (kept) states separately.
#ifdef MCTB_BFS_PHASES
#define MCTB_PH(k)                                                                   \
    do {                                                                             \
        if (a.op_hist) {                                                             \
            const long long ph_now = clock64();                                      \
            if (lane == 0)                                                           \
                atomicAdd(&ph_s[(ph_chain ? 8 : 0) + (k)],                           \
                          (unsigned long long)(ph_now - ph_t));                      \
            ph_t = ph_now;                                                           \
        }                                                                            \
    } while (0)
#else
#define MCTB_PH(k) \
    do {           \
    } while (0)
#endif

#ifndef MCTB_BFS_MINB
#define MCTB_BFS_MINB 4  // resident blocks per SM the register allocation targets
#endif

constexpr uint32_t kEmpty = 0xffffffffu;
#ifndef MCTB_BFS_THREADS
#define MCTB_BFS_THREADS 256
#endif
constexpr int kBfsThreads = MCTB_BFS_THREADS;

// Memory operations on the shared structures (tables, queues, counters).
// SYS = the partitions span GPUs (peer memory): system scope; else GPU scope.
template <bool SYS>
__device__ __forceinline__ uint32_t ld_relaxed32(const uint32_t* p) {
    uint32_t v;
    if (SYS) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <bool SYS>
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    if (SYS) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <bool SYS>
__device__ __forceinline__ void ld_relaxed_v4(const uint32_t* p, uint32_t* v) {
    if (SYS)
        asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "l"(p)
                     : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "l"(p)
                     : "memory");
}

template <bool SYS>
__device__ __forceinline__ void st_relaxed32(uint32_t* p, uint32_t v) {
    if (SYS) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool SYS>
__device__ __forceinline__ unsigned long long atom_add(unsigned long long* p, unsigned long long v) {
    return SYS ? atomicAdd_system(p, v) : atomicAdd(p, v);
}

template <bool SYS>
__device__ __forceinline__ unsigned long long atom_cas(unsigned long long* p, unsigned long long c,
                                                       unsigned long long v) {
    return SYS ? atomicCAS_system(p, c, v) : atomicCAS(p, c, v);
}

template <bool SYS>
__device__ __forceinline__ void set_error(int* p, int code) {
    if (SYS) atomicExch_system(p, code);
    else atomicExch(p, code);
}

// One slot line (SW words: key + padding + tag), 16 bytes per load.
template <int SW, bool SYS>
__device__ __forceinline__ void ld_line(const uint32_t* p, uint32_t (&v)[SW]) {
#pragma unroll
    for (int c = 0; c < SW / 4; ++c) ld_relaxed_v4<SYS>(p + 4 * c, v + 4 * c);
}

// Partition of a state: the high half of its hash (the slot uses the low bits).
__device__ __forceinline__ int owner_of(uint64_t h, int n_parts) {
    return n_parts == 1 ? 0 : (int)(((h >> 32) * (uint64_t)n_parts) >> 32);
}

// The SW-2 key/padding words of a slot (the tag is not touched).
template <int SW>
__device__ __forceinline__ void st_key(uint32_t* p, const uint32_t* row) {
#pragma unroll
    for (int c = 0; c < (SW - 2) / 4; ++c)
        *reinterpret_cast<uint4*>(p + 4 * c) = *reinterpret_cast<const uint4*>(row + 4 * c);
    *reinterpret_cast<uint2*>(p + SW - 4) = *reinterpret_cast<const uint2*>(row + SW - 4);
}

template <int SW>
__device__ __forceinline__ void copy_key(uint32_t* dst, const uint32_t* src) {
#pragma unroll
    for (int c = 0; c < (SW - 2) / 4; ++c)
        *reinterpret_cast<uint4*>(dst + 4 * c) = *reinterpret_cast<const uint4*>(src + 4 * c);
    *reinterpret_cast<uint2*>(dst + SW - 4) = *reinterpret_cast<const uint2*>(src + SW - 4);
}

// Inserts into partition `pt`.  Returns the slot of a newly inserted key, -1
// if already present, -2 if the table is full, -3 on a stall (watchdog).
// `row` holds the key padded with guard words to SW-2 words.
template <int SW, bool SYS>
__device__ long long table_insert(const BfsArgs& a, const BfsPart& pt, const uint32_t* row,
                                  uint64_t h) {
    const unsigned long long fp = h | 1ull;  // nonzero: 0 marks an empty slot
    uint64_t i = h & a.cap_mask;
    // a probe sequence this long only happens in a table that is too full (at load
    // <= 1/2 linear probing's longest sequence over 1e8 keys is a few dozen): report
    // it early — the sweep restarts with a larger table — instead of crawling
    // through an overloaded one
    for (uint64_t probe = 0; probe < 256; ++probe, i = (i + 1) & a.cap_mask) {
        uint32_t* sl = pt.table + i * SW;
        uint32_t v[SW];
        unsigned long long t;
        // one line read: tag and key arrive together (claiming with a CAS issued
        // alongside every read was measured 2.4x slower on wide spaces)
        ld_line<SW, SYS>(sl, v);
        t = (unsigned long long)v[SW - 2] | ((unsigned long long)v[SW - 1] << 32);
        if (t == 0) {
            t = atom_cas<SYS>(reinterpret_cast<unsigned long long*>(sl + SW - 2), 0ull, fp);
            if (t == 0) {
                st_key<SW>(sl, row);
                return (long long)i;
            }
            // claimed meanwhile: its key is read below if the fingerprint matches
#pragma unroll
            for (int k = 0; k < SW - 2; ++k) v[k] = 0;
        }
        if (t != fp) continue;  // different fingerprint
        for (unsigned ns = 32, spins = 0;; ++spins) {
            bool eq = true, torn = false;
#pragma unroll
            for (int k = 0; k < SW - 2; ++k) {
                eq &= v[k] == row[k];
                torn |= !(v[k] & kGuard);
            }
            if (!torn) {
                if (eq) return -1;
                break;
            }
            // the claimer is still writing the key
            if (spins > (1u << 21)) {  // watchdog: a key that never completes
                set_error<SYS>(pt.error, 5);
                return -3;
            }
            __nanosleep(ns);
            if (ns < 512) ns <<= 1;
            ld_line<SW, SYS>(sl, v);
        }
    }
    return -2;
}

// Pushes the lanes' new slots (fresh lanes) onto their owners' queues with one
// reservation per owner per warp.  Returns the number pushed (on every lane).
template <bool SYS>
__device__ __forceinline__ unsigned push_fresh(const BfsArgs& a, bool fresh, long long slot, int owner) {
    const int lane = threadIdx.x & 31;
    unsigned mask = __ballot_sync(0xffffffffu, fresh);
    const unsigned total = __popc(mask);
    while (mask) {
        const int leader = __ffs(mask) - 1;
        const int o = __shfl_sync(0xffffffffu, owner, leader);
        const unsigned grp = __ballot_sync(0xffffffffu, fresh && owner == o);
        const BfsPart& pt = a.part[o];
        const unsigned cnt = __popc(grp);
        unsigned long long pos0 = 0;
        if (lane == leader) {
            pos0 = atom_add<SYS>(pt.tq, ((unsigned long long)cnt << 32) | cnt) >> 32;
            if (pos0 + cnt > a.queue_cap) set_error<SYS>(pt.error, 2);
        }
        pos0 = __shfl_sync(0xffffffffu, pos0, leader);
        if (grp & (1u << lane)) {
            const unsigned long long pos = pos0 + __popc(grp & ((1u << lane) - 1));
            // relaxed: the consumer re-reads the slot until every guard bit is set
            if (pos < a.queue_cap) st_relaxed32<SYS>(&pt.queue[pos], (uint32_t)slot);
        }
        mask &= ~grp;
    }
    return total;
}

// Any partition's error flag (read by idle and every-64th-state checks).
template <bool SYS>
__device__ __forceinline__ int any_error(const BfsArgs& a) {
    int e = 0;
    for (int p = 0; p < a.n_parts; ++p) e |= (int)ld_relaxed32<SYS>((const uint32_t*)a.part[p].error);
    return e;
}

// Global quiescence over the partitions: every pushed state has been expanded.
// One partition: outstanding == 0.  Several: pass 1 reads each partition's
// expanded count (tail - outstanding), pass 2 its tail; both are monotone, so
// equal sums mean that no state was outstanding at the end of pass 1 — and
// only an outstanding state can push another.
template <bool SYS>
__device__ __forceinline__ bool quiescent(const BfsArgs& a) {
    if (a.n_parts == 1) return (uint32_t)ld_relaxed64<SYS>(a.part[0].tq) == 0;
    unsigned long long done = 0, tail = 0;
    for (int p = 0; p < a.n_parts; ++p) {
        const unsigned long long t = ld_relaxed64<SYS>(a.part[p].tq);
        done += (t >> 32) - (t & 0xffffffffull);
    }
    for (int p = 0; p < a.n_parts; ++p) tail += ld_relaxed64<SYS>(a.part[p].tq) >> 32;
    return done == tail;
}

// 64-bit warp sum (every lane gets it)
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Canonical successors (explore_kernel's comment): false for a report by an
// element below the parent's highest reported one, for a barrier arrival below
// the highest element already waiting at that barrier and for an activation
// below the highest element of the unit untouched since its own — their
// successors are inserted by their canonical parents.
struct CanonMasks {
    // bits 0-7: highest reported element + 1 (0: none); bits 8-23: bit 8 + g set
    // when unit g activates a batch (U_ACTIVATEPEX, not a re-arm) — one register
    unsigned rep_batch;
    unsigned waiting;   // bit p: element p waits at its barrier
    unsigned pristine;  // bit p: element p untouched since its activation (abstract kernel)
};

// true unless a set bit of `mask` lies above element p within p's unit
__device__ __forceinline__ bool highest_in_unit(unsigned mask, int p, int lognwe) {
    const int end = ((p >> lognwe) + 1) << lognwe;
    const unsigned below_end = end >= 32 ? 0xffffffffu : (1u << end) - 1u;
    return (mask & below_end & ~((2u << p) - 1u)) == 0;
}

__device__ __forceinline__ bool canonical_successor(const Transition& tr, const CanonMasks& c,
                                                    int lognwe) {
    if (tr.op == OP_PEXREPORT) return (int)tr.actor + 1 >= (int)(c.rep_batch & 0xffu);
    if (tr.op == OP_PEXARRIVE) return highest_in_unit(c.waiting, tr.actor, lognwe);
    if (tr.op == OP_UNITPEXGO)
        return !((c.rep_batch >> (8 + tr.actor)) & 1u) ||
               highest_in_unit(c.pristine, tr.peer, lognwe);
    return true;
}

// The parent's masks; n_pex <= 32, one ballot each.  An activation of a batch
// (unit -> element go in U_ACTIVATEPEX, machine.cpp UNITPEXGO) commutes with what
// can follow it while its element has not moved (the other activations of the
// batch and the other elements' reports: no tick, barrier or item hand-back can
// pass an unmoved element), so the highest element still untouched since its
// activation marks the canonical last activation.  Untouched, for the abstract
// kernel: running its first busy(gmt*ts) at cursor 0, unreported.  A re-arm
// (U_REACTPEX, after a hand-back) is not pruned: the hand-backs that follow it
// need the unit it returns to serving.
__device__ __forceinline__ CanonMasks canon_masks(const MachDesc& m, const MState& s, int lane) {
    const PexS* px = lane < m.n_pex ? &s.pex[lane] : nullptr;
    CanonMasks c;
    const unsigned rb = __ballot_sync(0xffffffffu, px && px->reported);
    c.rep_batch = rb ? 32 - __clz(rb) : 0;
    c.waiting = __ballot_sync(0xffffffffu,
                              px && (px->pc == P_WAITBARRIER || px->pc == P_WAITGROUPEND));
    c.pristine = __ballot_sync(0xffffffffu, m.kernel == 0 && px && px->pc == P_RUN &&
                                                px->phase == 0 && px->cursor == 0 &&
                                                !px->reported &&
                                                px->busy_left == m.gmt * m.ts);
    c.rep_batch |= (__ballot_sync(0xffffffffu, lane < m.n_units && s.unit[lane].pc == U_ACTIVATEPEX)
                    & 0xffffu) << 8;
    return c;
}

template <int SW, bool SYS>
__global__ void __launch_bounds__(kBfsThreads, MCTB_BFS_MINB) explore_kernel(BfsArgs a) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // the partition this warp expands (round-robin over the launch's partitions)
    const int mp = a.part0 + (int)(((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % a.n_here);
    const BfsPart& me = a.part[mp];
    // per warp in shared memory: the parent (unpacked and packed) and its enabled
    // list; per lane: one packed successor row.  Only the generic transitions
    // materialise an unpacked successor in (L1-resident) local memory.
    __shared__ MState parent[kBfsThreads / 32];
    __shared__ Transition enabled_s[kBfsThreads / 32][kMaxEnabled];
    __shared__ uint64_t hk[32];  // hash coefficients K_i
    extern __shared__ uint32_t dyn[];
    if (threadIdx.x < 32) hk[threadIdx.x] = hash_coef(threadIdx.x);
#ifdef MCTB_BFS_PHASES
    __shared__ unsigned long long ph_s[16];
    if (threadIdx.x < 16) ph_s[threadIdx.x] = 0;
    long long ph_t = clock64();
    bool ph_chain = false;
#endif
    // unpack_fields writes the time's low word only
    if ((threadIdx.x & 31) == 0) parent[threadIdx.x >> 5].time = 0;
    __syncthreads();
    // rows are SW words apart (16-byte aligned); words [words, SW-2) are guard padding
    uint32_t* pwords = dyn + wib * (34 * SW);  // parent words
    uint32_t* kwords = pwords + SW;            // the successor the warp keeps
    uint32_t* row = pwords + (2 + lane) * SW;  // this lane's successor
    MState& s = parent[wib];
    Transition* en = enabled_s[wib];
    MState t;
    // warp-local statistics of the current configuration, flushed on change/exit
    int cur_cfg = -1;
    // (32-bit: flushed at least every 64 expansions; registers are the kernel's limit)
    unsigned n_states = 0, n_trans = 0;
    auto flush = [&]() {
        if (lane == 0 && cur_cfg >= 0) {
            if (n_states) atomicAdd(&a.stats[cur_cfg].states, (unsigned long long)n_states);
            if (n_trans) atomicAdd(&a.stats[cur_cfg].transitions, (unsigned long long)n_trans);
        }
        n_states = n_trans = 0;
    };
    bool local = false;  // the warp continues with a successor it discovered itself
    // the configuration's global state count and the error flag, re-read every
    // 64 expansions (not on every state's critical path): the visited cap and an
    // error stop the sweep a few states late, which only bounds extra work
    unsigned long long g_states = 0;
    int g_err = 0;
    unsigned since = 0;
    uint64_t H = 0;      // hash of the parent (known for a kept successor)
    // queue entries are claimed in runs: a warp that finds its entries already
    // filled doubles its next claim (up to 8), one that has to wait claims one
    // queue positions (< queue_cap <= 2^28, plus the idle warps' last claims)
    uint32_t h_next = 0, h_end = 0, h_run = 0;
    unsigned claim = 1;
    uint32_t peek = kEmpty;  // lane j: entry h_run + j of the current run, as first read
    uint32_t dep = 0;        // depth of the parent (tracked under a depth cap only)
#ifdef MCTB_BFS_DEBUG
    unsigned long long dbg_it = 0;
#endif
    for (;;) {
#ifdef MCTB_BFS_DEBUG
        if (++dbg_it == (1ull << 22)) {
            if (lane == 0)
                printf("[dbg] warp %d blk %d: %llu iterations, local %d cfg %d g_states %llu n_states %u "
                       "h_next %u h_end %u since %u dep %u err %d\n",
                       wib, blockIdx.x, dbg_it, (int)local, cur_cfg, g_states, n_states, h_next,
                       h_end, since, dep, g_err);
        }
#endif
#ifdef MCTB_BFS_PHASES
        ph_chain = local;
        if (a.op_hist && lane == 0) atomicAdd(&ph_s[(ph_chain ? 8 : 0) + 7], 1ull);
        ph_t = clock64();
#endif
        if (!local) {
            if (h_next == h_end) {
                unsigned long long h0 = 0;
                if (lane == 0) h0 = atomicAdd(me.head, (unsigned long long)claim);
                h_run = h_next = (uint32_t)__shfl_sync(0xffffffffu, h0, 0);
                h_end = h_next + claim;
                // read the whole run at once and start the filled entries' slot lines
                // on their way to L2; a later pop of a filled entry needs no poll
                peek = lane < (int)claim && h_run + lane < a.queue_cap
                           ? ld_relaxed32<SYS>(&me.queue[h_run + lane])
                           : kEmpty;
                if (peek != kEmpty)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(me.table + (uint64_t)peek * SW));
            }
            const uint32_t h = h_next++;
            if (h >= a.queue_cap) break;
            uint32_t slot = __shfl_sync(0xffffffffu, peek, (int)(h - h_run));
            bool waited = false;
            if (slot == kEmpty) {
                // wait until entry h is pushed, or the sweep is over
                if (lane == 0) {
                    unsigned ns = 64;
                    for (unsigned it = 0;; ++it) {
                        slot = ld_relaxed32<SYS>(&me.queue[h]);  // relaxed poll: no L1 invalidation
                        if (slot != kEmpty) break;
                        waited = true;
                        // the shared counters are read rarely: they are the working warps'
                        // atomics' cache line
                        if ((it & 15) == 15 && (quiescent<SYS>(a) || any_error<SYS>(a))) break;
                        if (it > (1u << 23)) {  // watchdog: outstanding states never arrive
                            set_error<SYS>(me.error, 7);
                            break;
                        }
                        __nanosleep(ns);
                        if (ns < MCTB_BFS_MAX_SLEEP) ns <<= 1;
                    }
                }
                slot = __shfl_sync(0xffffffffu, slot, 0);
                waited = __shfl_sync(0xffffffffu, waited, 0);
            }
            claim = waited ? 1u : (claim < 8u ? claim * 2u : 8u);
            if (slot == kEmpty) break;
            // one coalesced line read; a word without its guard bit is still being
            // written by the slot's claimer: read again
            const uint32_t* src = me.table + (uint64_t)slot * SW;
            uint32_t w;
            for (unsigned spins = 0;; ++spins) {
                w = lane < SW - 2 ? ld_relaxed32<SYS>(src + lane) : kGuard;
                if (__all_sync(0xffffffffu, w & kGuard)) break;
                if (spins > (1u << 22)) {  // watchdog: a pushed key that never completes
                    if (lane == 0) set_error<SYS>(me.error, 6);
                    break;
                }
                __nanosleep(64);
            }
            if (lane < SW - 2) pwords[lane] = w;
            H = warp_sum64(lane < a.words ? (uint64_t)w * hk[lane] : 0ull);
            if (a.depth_cap) {
                // written by the slot's claimer with its guard bit, like the key words
                uint32_t dv = 0;
                if (lane == 0)
                    for (unsigned spins = 0;; ++spins) {
                        dv = ld_relaxed32<SYS>(me.depth + slot);
                        if (dv & kGuard) break;
                        if (spins > (1u << 22)) {  // watchdog: a depth that never arrives
                            set_error<SYS>(me.error, 6);
                            break;
                        }
                        __nanosleep(64);
                    }
                dep = __shfl_sync(0xffffffffu, dv, 0) & ~kGuard;
            }
            __syncwarp();
        }
        MCTB_PH(0);  // pop: queue entry, slot line, parent hash
        const int cfg = peek_cfg(pwords, a.cfg_bits);
        if (cfg != cur_cfg) {
            flush();
            cur_cfg = cfg;
            since = 0;
        }
        if ((since++ & 63) == 0 || n_states >= a.flush_states) {
            // publish this warp's count first: the cap check below must see every
            // warp's insertions, or each warp would stop only at its own local cap
            // and max_states would bound neither work nor memory
            flush();
            __syncwarp();
            g_states = ld_relaxed64<false>(&a.stats[cfg].states);
            g_err = any_error<SYS>(a);
        }
        const BfsDesc& d = a.descs[cfg];
        const int lognwe = __ffs(d.m.nwe) - 1;
        // table-driven warp-parallel unpack, then one pass of the per-process rules
        // (bfs_rules.cuh) with a warp prefix sum placing every lane's transitions
        MCTB_PH(1);  // configuration bookkeeping
        unpack_fields(a.ftab + (size_t)cfg * kMaxFields, a.nfields[cfg], pwords, s, lane);
        __syncwarp();
        MCTB_PH(2);  // unpack
        const int nsl = n_slots(d.m);
        int ne = 0;
        for (int k0 = 0; k0 < nsl; k0 += 32) {
            Transition mine[2];
            const int cnt = k0 + lane < nsl ? bfs_slot_rules(d.m, s, k0 + lane, lognwe, mine) : 0;
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int pos = ne + incl - cnt;
            if (cnt > 0) en[pos] = mine[0];
            if (cnt > 1) en[pos + 1] = mine[1];
            ne += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        MCTB_PH(3);  // enumeration
        BfsStats& st = a.stats[cfg];
        if (a.check_inv && lane == 0) {
            // machine.cpp:719-756, plus tick gating (acceptance criterion 7)
            bool bad = check_invariants(d.m, s) != 0;
            for (int e = 0; e < ne; ++e)
                bad |= en[e].op == OP_CLOCKTICK && (s.nrp_work != s.all_nwe || s.all_nwe == 0);
            if (bad) atomicAdd(&st.violations, 1ull);
        }
        bool kept = false;
        uint64_t H_kept = 0;
        if (ne == 0) {
            if (lane == 0) {
                if (is_terminal(d.m, s)) {
                    atomicAdd(&st.terminals, 1ull);
                    atomicMin(&st.min_time, (long long)s.time);
                    atomicMax(&st.max_time, (long long)s.time);
                } else {
                    atomicAdd(&st.deadlocks, 1ull);
                    set_error<SYS>(me.error, 3);
                }
            }
        } else if (g_states + n_states >= a.cfg_cap) {
            // explore.cpp:28: a full visited set inserts nothing more
            if (lane == 0) st.capped = 1;
        } else if (a.depth_cap && dep >= a.depth_cap) {
            // explore.cpp:124-127: a transition past max_depth is not applied
            if (lane == 0) st.depth_cut = 1;
        } else {
            n_trans += (unsigned)ne;
            // Canonical report parents.  A report only sets its element's flag and
            // nrp_work, which no rule but the tick reads (machine.cpp:680-689), so
            // it commutes with every transition but the tick: a state whose
            // reported elements are R' is reached from the state without the
            // report of max(R') (reachable: that report can always be moved to
            // the end of a path).  Only that parent inserts it; a report by an
            // element below the parent's highest reported one is counted (it is a
            // transition) but its successor — present anyway — is neither built
            // nor probed.  In a lattice of b elements that skips all but
            // 2 / b of the report successors.  Barrier arrivals likewise
            // (machine.cpp arrive/release): an arrival only moves its element to
            // wait and counts it, which only the release (count = nwe, after every
            // arrival of the episode) and the other arrivals (count < nwe) read,
            // so within one barrier the arrival of the highest waiting element is
            // the canonical last one.  (n_pex <= 32: one ballot each.)
            CanonMasks cm{0u, 0u, 0u};
            if (a.canon) cm = canon_masks(d.m, s, lane);
            for (int base = 0; base < ne; base += 32) {
                const int e = base + lane;
                long long ins = -1;
                int owner = mp;
                uint64_t Hc = H;
                bool ok = false;
                if (e < ne && (!a.canon || canonical_successor(en[e], cm, lognwe))) {
                    copy_key<SW>(row, pwords);
                    ok = true;
                    if (!fast_successor(d, s, en[e], row, hk, Hc)) {
                        if (a.op_hist) atomicAdd(&a.op_hist[en[e].op], 1ull);
                        copy_state(d.m, t, s);
                        ok = apply(d.m, t, to_pid(d.m, en[e]));
                        if (ok) {
                            pack(d, cfg, t, row);
                            Hc = 0;
                            for (int k = 0; k < a.words; ++k) Hc += (uint64_t)row[k] * hk[k];
                        } else {
                            set_error<SYS>(me.error, 3);
                        }
                    }
                }
                // reconverge the per-op paths before the shared hash / insert code
                __syncwarp();
                MCTB_PH(4);  // successor rows
                if (ok) {
                    const uint64_t hh = fmix64(Hc);
                    if (a.n_parts > 1) owner = owner_of(hh, a.n_parts);
                    ins = table_insert<SW, SYS>(a, a.part[owner], row, hh);
                    if (a.op_hist) atomicAdd(&a.op_hist[24], 1ull);  // diagnostics: probes
                    if (ins == -2) set_error<SYS>(me.error, 1);
                    if (ins >= 0 && a.depth_cap)
                        st_relaxed32<SYS>(a.part[owner].depth + ins, (dep + 1) | kGuard);
                }
#ifdef MCTB_BFS_PHASES
                __syncwarp();
#endif
                MCTB_PH(5);  // hash, probe, claim
                bool fresh = ins >= 0;
                int keeper = -1;
                if (!kept && a.keep) {
                    // keep the first new successor, whichever partition owns its slot:
                    // no queue round trip on the chain (also none to another
                    // partition's queue); it inherits the parent's place in this
                    // partition's `outstanding`, which the chain's end releases
                    const unsigned m = __ballot_sync(0xffffffffu, fresh);
                    if (m) {
                        keeper = __ffs(m) - 1;
                        if (lane == keeper) fresh = false;
                        kept = true;
                        n_states += 1;
                        H_kept = __shfl_sync(0xffffffffu, Hc, keeper);
                    }
                }
                n_states += push_fresh<SYS>(a, fresh, ins, owner);
                if (keeper >= 0) {
                    __syncwarp();
                    const uint32_t* kr = pwords + (2 + keeper) * SW;
                    if (lane < SW - 2) kwords[lane] = kr[lane];
                    __syncwarp();
                }
            }
        }
        __syncwarp();
        MCTB_PH(6);  // keep / push / copy
        local = kept && !g_err;
        if (local) {
            if (lane < SW - 2) pwords[lane] = kwords[lane];
            H = H_kept;
            dep += 1;
            __syncwarp();
        } else if (lane == 0) {
            atom_add<SYS>(me.tq, ~0ull);  // this state is expanded: outstanding - 1
        }
    }
    flush();
#ifdef MCTB_BFS_PHASES
    __syncthreads();
    if (a.op_hist && threadIdx.x < 16) atomicAdd(&a.op_hist[28 + threadIdx.x], ph_s[threadIdx.x]);
#endif
}

template <int SW, bool SYS>
__global__ void seed_kernel(BfsArgs a, const uint32_t* seeds, int n_seeds,
                            const uint32_t* seed_dep) {
    // one initial state per configuration (explore.cpp:98-105), or the given
    // packed states of configuration 0 (a multi-source exploration), each into
    // its owner partition
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t key[SW];
    for (int k = 0; k < SW; ++k) key[k] = kGuard;
    int cfg = c;
    if (seeds) {
        if (c >= n_seeds) return;
        for (int k = 0; k < a.words; ++k) key[k] = seeds[(size_t)c * a.words + k];
        cfg = peek_cfg(key, a.cfg_bits);  // 0 for a single-configuration sweep
    } else {
        if (c >= a.n_cfg) return;
        const BfsDesc& d = a.descs[c];
        MState s;
        initial_state(d.m, s);
        pack(d, c, s, key);
    }
    const uint64_t h = fmix64(hash_full(key, a.words));
    const BfsPart& pt = a.part[owner_of(h, a.n_parts)];
    const long long ins = table_insert<SW, SYS>(a, pt, key, h);
    if (ins == -1) return;  // a repeated seed
    if (ins < 0) {
        set_error<SYS>(pt.error, 1);
        return;
    }
    atomicAdd(&a.stats[cfg].states, 1ull);
    if (a.depth_cap)
        st_relaxed32<SYS>(pt.depth + ins, (seeds && seed_dep ? seed_dep[c] : 0u) | kGuard);
    const unsigned long long pos = atom_add<SYS>(pt.tq, (1ull << 32) | 1ull) >> 32;
    if (pos >= a.queue_cap) {  // as push_fresh: the queue sits before the counters
        set_error<SYS>(pt.error, 2);
        return;
    }
    st_relaxed32<SYS>(&pt.queue[pos], (uint32_t)ins);
}

// ---------------------------------------------------------------------------
// Narrow state graphs: one CTA per configuration, level by level in shared
// memory.  The state graphs are graded (every path to a state has the same
// length: tests/test_oracle.py), so a state can only equal states
// of its own level: the visited set of a level-synchronous sweep is the next
// level alone.  A configuration whose levels stay within kLvlWidth states (the
// deep, narrow graphs of the tune sweeps: thousands to millions of levels of a
// few states) runs here with no HBM table, queue or atomics: per level, each
// warp expands its states exactly like explore_kernel (same unpack, rules and
// successor code) and inserts the successors into a shared-memory hash table of
// the next level.  A level that outgrows the table is handed to the global
// sweep (explore_kernel) as its seeds, with the level's statistics rolled back.
constexpr int kLvlThreads = 256;
constexpr int kLvlWidth = 256;  // widest level a CTA holds
constexpr int kLvlSlots = 512;  // hash slots per level (load <= 1/2)

struct LevelArgs {
    const BfsDesc* descs;
    const uint2* ftab;
    const int* nfields;
    BfsStats* stats;
    int words, cfg_bits, check_inv;
    uint64_t cfg_cap;
    uint32_t depth_cap;
    uint32_t* frontier;  // [n_cfg][kLvlWidth * words]: a handed-off level
    int64_t* fstat;      // [n_cfg][4]: {status (0 done, 1 handed off, 3 model bug), states, level}
    int skip;            // count pure tick cycles instead of exploring them
    unsigned max_width;  // a wider level goes to the global sweep (<= kLvlWidth)
    // so does a run of wide_run consecutive levels wider than wide: eight warps
    // take ceil(n / 8) expansions per level, where the global sweep's thousands
    // of warps take one; a short burst stays (the skips need the level pass)
    unsigned wide, wide_run;
    // and a window of `window` levels with no closed-form skip and at least
    // window_states states: several states per level wait for the slowest one
    // at every level barrier, where the global sweep's warps run ahead
    unsigned window, window_states;
    int canon;  // canonical successors only (explore_kernel)
};

// Inserts `row` (hash hh) into the level table; 1 new, 0 present, -1 full.
__device__ int level_insert(uint32_t* tags, uint32_t* keys, uint16_t* list, unsigned* n_list,
                            int words, const uint32_t* row, uint64_t hh, int* flags) {
    const uint32_t tg = (uint32_t)(hh >> 32) | 1u;
    uint32_t i = (uint32_t)hh & (kLvlSlots - 1);
    for (int probe = 0; probe < kLvlSlots; ++probe, i = (i + 1) & (kLvlSlots - 1)) {
        uint32_t t = *(volatile uint32_t*)&tags[i];
        if (t == 0) {
            t = atomicCAS(&tags[i], 0u, tg);
            if (t == 0) {
                uint32_t* k = keys + i * words;
                for (int w = 0; w < words; ++w) k[w] = row[w];  // every word carries kGuard
                const unsigned pos = atomicAdd(n_list, 1u);
                if (pos < (unsigned)kLvlWidth) list[pos] = (uint16_t)i;
                else atomicOr(flags, 4);
                return 1;
            }
        }
        if (t != tg) continue;
        const volatile uint32_t* k = keys + i * words;
        bool eq = true;
        for (int w = 0; w < words; ++w) {
            uint32_t v;
            while (!((v = k[w]) & kGuard)) {  // the claimer is still writing the key
            }
            eq &= v == row[w];
        }
        if (eq) return 0;
    }
    atomicOr(flags, 4);
    return -1;
}

#ifdef MCTB_BFS_PHASES
#define MCTB_LPH(k)                                          \
    do {                                                     \
        const long long lph_now = clock64();                 \
        if (threadIdx.x == 0) lph[k] += lph_now - lph_t;     \
        lph_t = lph_now;                                     \
    } while (0)
#else
#define MCTB_LPH(k) \
    do {            \
    } while (0)
#endif

template <int SW>
__global__ void __launch_bounds__(kLvlThreads, 1) level_kernel(LevelArgs a) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, cfg = blockIdx.x;
#ifdef MCTB_BFS_PHASES
    long long lph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long lph_t = clock64();
#endif
    const int words = a.words;
    __shared__ BfsDesc d;
    __shared__ MState parent[kLvlThreads / 32];
    __shared__ Transition enabled_s[kLvlThreads / 32][kMaxEnabled];
    __shared__ uint64_t hk[32];
    __shared__ uint32_t tags[2][kLvlSlots];
    __shared__ uint16_t list[2][kLvlWidth];
    __shared__ unsigned n_list[2];
    // the level's own statistics (committed when the level completes):
    // new states, transitions, terminals, deadlocks, invariant violations
    __shared__ unsigned long long lv[5];
    __shared__ long long lv_min, lv_max;
    __shared__ int lv_flags;  // 1 capped, 2 depth cut, 4 too wide, 8 model bug
    __shared__ uint32_t lv_jump;  // levels counted by a cycle skip beyond the next
    // the last rep-start state (abstract kernel), for the rep skip below
    __shared__ uint32_t rep_key[kMaxWords];
    __shared__ int rep_valid;
    __shared__ uint32_t rep_level;
    __shared__ unsigned long long rep_states, rep_trans, rep_events;
    __shared__ long long rep_time;
    __shared__ unsigned long long tot_states;
    extern __shared__ uint32_t dyn[];
    uint32_t* keys0 = dyn;
    uint32_t* keys1 = dyn + kLvlSlots * words;
    uint32_t* pwords = dyn + 2 * kLvlSlots * words + wib * (34 * SW);
    uint32_t* row = pwords + (2 + lane) * SW;
    if (threadIdx.x < 32) hk[threadIdx.x] = hash_coef(threadIdx.x);
    for (int i = threadIdx.x; i < (int)(sizeof(BfsDesc) / 4); i += kLvlThreads)
        reinterpret_cast<uint32_t*>(&d)[i] = reinterpret_cast<const uint32_t*>(a.descs + cfg)[i];
    for (int i = threadIdx.x; i < 2 * kLvlSlots; i += kLvlThreads) (&tags[0][0])[i] = 0;
    for (int i = threadIdx.x; i < 2 * kLvlSlots * words; i += kLvlThreads) dyn[i] = 0;
    if (lane == 0) parent[wib].time = 0;  // unpack_fields writes the time's low word only
    if (threadIdx.x == 0) {
        n_list[0] = n_list[1] = 0;
        lv_flags = 0;
        rep_valid = 0;
    }
    __syncthreads();
    MState& s = parent[wib];
    Transition* en = enabled_s[wib];
    MState t;
    const int lognwe = __ffs(d.m.nwe) - 1;
    const int nsl = n_slots(d.m);
    const uint2* ftab = a.ftab + (size_t)cfg * kMaxFields;
    const int nf = a.nfields[cfg];
    // level 0: the initial state (explore.cpp:98-105)
    if (wib == 0) {
        if (lane == 0) {
            MState s0;
            initial_state(d.m, s0);
            for (int k = 0; k < SW; ++k) row[k] = kGuard;
            pack(d, cfg, s0, row);
            uint64_t H0 = 0;
            for (int k = 0; k < words; ++k) H0 += (uint64_t)row[k] * hk[k];
            level_insert(tags[0], keys0, list[0], &n_list[0], words, row, fmix64(H0), &lv_flags);
            tot_states = 1;
        }
    }
    unsigned long long acc_trans = 0, acc_terms = 0, acc_dead = 0, acc_viol = 0;
    long long acc_min = INT64_MAX, acc_max = -1;
    int acc_flags = 0;
    int status = 0;
    unsigned handed = 0;
    unsigned wide_levels = 0;  // consecutive levels wider than a.wide
    unsigned win_levels = 0, win_states = 0;  // the current window (no skip in it yet)
    uint32_t level = 0;
    for (int cur = 0;; cur ^= 1, ++level) {
        const int nx = cur ^ 1;
        uint32_t* kc = cur ? keys1 : keys0;
        uint32_t* kn = cur ? keys0 : keys1;
        __syncthreads();
        MCTB_LPH(3);  // commit + loop top
        const unsigned n = n_list[cur];
        if (n == 0) break;
        // clear the next level's table: the slots of two levels ago
        const unsigned n_old = min(n_list[nx], (unsigned)kLvlWidth);
        for (unsigned i = threadIdx.x; i < n_old * words; i += kLvlThreads)
            kn[list[nx][i / words] * words + i % words] = 0;
        for (unsigned i = threadIdx.x; i < n_old; i += kLvlThreads) tags[nx][list[nx][i]] = 0;
        if (threadIdx.x == 0) {
            for (int k = 0; k < 5; ++k) lv[k] = 0;
            lv_min = INT64_MAX;
            lv_max = -1;
            lv_flags = 0;
            lv_jump = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) n_list[nx] = 0;
        __syncthreads();
        MCTB_LPH(0);  // clear + reset
        for (unsigned i = wib; i < n; i += kLvlThreads / 32) {
            if (*(volatile int*)&lv_flags & 12) break;  // the level is handed off anyway
            const uint32_t* src = kc + list[cur][i] * words;
            const uint32_t w = lane < words ? src[lane] : kGuard;
            if (lane < SW - 2) pwords[lane] = w;
            const uint64_t H = warp_sum64(lane < words ? (uint64_t)w * hk[lane] : 0ull);
            __syncwarp();
            unpack_fields(ftab, nf, pwords, s, lane);
            __syncwarp();
            MCTB_LPH(4);  // load + unpack
            int ne = 0;
            for (int k0 = 0; k0 < nsl; k0 += 32) {
                Transition mine[2];
                const int cnt = k0 + lane < nsl ? bfs_slot_rules(d.m, s, k0 + lane, lognwe, mine) : 0;
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const int pos = ne + incl - cnt;
                if (cnt > 0) en[pos] = mine[0];
                if (cnt > 1) en[pos + 1] = mine[1];
                ne += __shfl_sync(0xffffffffu, incl, 31);
            }
            __syncwarp();
            MCTB_LPH(5);  // enumeration
#ifdef MCTB_BFS_PHASES
            if (threadIdx.x == 0) lph[8] += 1;
#endif
            // Pure tick cycles.  When the level is this one state X, every launched
            // element is busy and unreported (nrp_work = 0, ne = all_nwe reports)
            // and nothing else is enabled, the next levels are fixed: the b = ne
            // reports in every order (the 2^b subsets, machine.cpp:680-689: a report
            // only sets its element's flag and nrp_work, which no rule but the tick
            // reads), then the tick (machine.cpp:531-546), which decrements every
            // element's busy_left and clears the flags.  While the least busy_left
            // stays >= 2 after it, the tick leads to X with time + 1 and every
            // busy_left - 1: the same structure again.  Graded graphs put nothing
            // else on those levels, so c such cycles are counted, not explored:
            // c * 2^b states and c * (b * 2^(b-1) + 1) transitions over c * (b + 1)
            // levels, ending at the state X' they reach (inserted for the next level).
            // Whole reps (abstract kernel).  An element's phase-0 program repeats
            // busy(gmt*ts), barrier, busy(ts), barrier for reps = size/ts reps
            // (kernel.cpp:33-43); the rules read its cursor only through instr_at(),
            // which is periodic with period 4 there, and no rule reads the time.  At
            // a rep start (the level is this one state; every launched element runs,
            // unreported, at a cursor = 0 mod 4 with a fresh busy(gmt*ts)) the state
            // is compared with the previous rep start X: if it equals X with the
            // time advanced and every running cursor + 4 (the packed words decide),
            // the levels between them form a period that the following reps repeat
            // exactly while their cursors stay in the rep range.  k periods are
            // counted: k times the period's states, transitions and levels.
            if (n == 1 && a.skip && !a.check_inv && d.m.kernel == 0) {
                long long k = 0;
                if (lane == 0) {
                    bool start = s.nrp_work == 0 && s.all_nwe > 0;
                    int running = 0;
                    for (int p = 0; p < d.m.n_pex && start; ++p) {
                        const PexS& px = s.pex[p];
                        if (px.pc == P_WAITGO || px.pc == P_EXITED) continue;
                        start = px.pc == P_RUN && px.phase == 0 && (px.cursor & 3) == 0 &&
                                (int)px.cursor <= 4 * d.m.reps - 4 &&
                                px.busy_left == d.m.gmt * d.m.ts && !px.reported;
                        ++running;
                    }
                    start = start && running == s.all_nwe;
                    if (start) {
                        const unsigned long long ev = acc_terms + acc_dead;
                        bool period = false;
                        if (rep_valid && ev == rep_events && !(acc_flags & 3)) {
                            copy_state(d.m, t, s);
                            t.time = rep_time;
                            for (int p = 0; p < d.m.n_pex; ++p)
                                if (t.pex[p].pc == P_RUN) t.pex[p].cursor -= 4;
                            for (int w = 0; w < SW; ++w) row[w] = kGuard;
                            pack(d, cfg, t, row);
                            period = true;
                            for (int w = 0; w < words; ++w) period &= row[w] == rep_key[w];
                        }
                        if (period) {
                            const long long P = level - rep_level;
                            const unsigned long long Sp = tot_states - rep_states;
                            const unsigned long long Tp = acc_trans - rep_trans;
                            const long long dt = s.time - rep_time;
                            k = 0x7fffffff;
                            for (int p = 0; p < d.m.n_pex; ++p)
                                if (s.pex[p].pc == P_RUN)
                                    k = min(k, (long long)(4 * d.m.reps - 4 - s.pex[p].cursor) / 4);
                            if (a.depth_cap) k = min(k, (long long)(a.depth_cap - level) / P);
                            const unsigned long long cap = a.cfg_cap, tot = tot_states;
                            const unsigned long long r = cap - (tot < cap ? tot : cap);
                            k = min(k, (long long)(r / Sp) - 1);
                            if (k > 0) {
                                s.time += k * dt;
                                for (int p = 0; p < d.m.n_pex; ++p)
                                    if (s.pex[p].pc == P_RUN) s.pex[p].cursor += (uint16_t)(4 * k);
                                for (int w = 0; w < SW; ++w) row[w] = kGuard;
                                pack(d, cfg, s, row);
                                uint64_t Hx = 0;
                                for (int w = 0; w < words; ++w) Hx += (uint64_t)row[w] * hk[w];
                                level_insert(tags[nx], kn, list[nx], &n_list[nx], words, row,
                                             fmix64(Hx), &lv_flags);
                                lv[0] += (unsigned long long)k * Sp;
                                lv[1] += (unsigned long long)k * Tp;
                                lv_jump = (uint32_t)(k * P - 1);
                                rep_valid = 0;
                            }
                        }
                        if (k <= 0) {
                            k = 0;
                            for (int w = 0; w < SW; ++w) row[w] = kGuard;
                            pack(d, cfg, s, row);
                            for (int w = 0; w < words; ++w) rep_key[w] = row[w];
                            rep_valid = 1;
                            rep_level = level;
                            rep_states = tot_states;
                            rep_trans = acc_trans;
                            rep_events = ev;
                            rep_time = s.time;
                        }
                    }
                }
                k = __shfl_sync(0xffffffffu, k, 0);
                if (k > 0) {
                    __syncwarp();
                    continue;
                }
                __syncwarp();
            }
            if (n == 1 && a.skip && !a.check_inv) {
                long long cyc = 0;
                if (lane == 0 && ne >= 1 && ne <= 16 && ne == s.all_nwe && s.nrp_work == 0 &&
                    (a.depth_cap == 0 || level < a.depth_cap)) {
                    int mb = 0x7fffffff;
                    bool pure = true;
                    for (int e = 0; e < ne; ++e) {
                        if (en[e].op != OP_PEXREPORT) {
                            pure = false;
                            break;
                        }
                        mb = min(mb, (int)s.pex[en[e].actor].busy_left);
                    }
                    if (pure && mb >= 2) {
                        cyc = mb - 1;
                        // every counted level below the depth cap (its states are
                        // all expanded), and room under the visited cap
                        if (a.depth_cap) cyc = min(cyc, (long long)(a.depth_cap - level) / (ne + 1));
                        const unsigned long long cap = a.cfg_cap, tot = tot_states;
                        const unsigned long long r = cap - (tot < cap ? tot : cap);
                        const long long room = r > (1ull << 62) ? (1ll << 62) : (long long)r;
                        cyc = min(cyc, room / (1ll << ne) - 1);
                    }
                }
                cyc = __shfl_sync(0xffffffffu, cyc, 0);
                if (cyc > 0) {
                    if (lane == 0) {
                        s.time += cyc;
                        for (int e = 0; e < ne; ++e) s.pex[en[e].actor].busy_left -= (uint16_t)cyc;
                        for (int k = 0; k < SW; ++k) row[k] = kGuard;
                        pack(d, cfg, s, row);
                        uint64_t Hx = 0;
                        for (int k = 0; k < words; ++k) Hx += (uint64_t)row[k] * hk[k];
                        level_insert(tags[nx], kn, list[nx], &n_list[nx], words, row, fmix64(Hx),
                                     &lv_flags);
                        lv[0] += (unsigned long long)cyc << ne;
                        lv[1] += (unsigned long long)cyc * (((unsigned long long)ne << (ne - 1)) + 1);
                        lv_jump = (uint32_t)(cyc * (ne + 1) - 1);
                    }
                    __syncwarp();
                    continue;
                }
            }
            if (a.check_inv && lane == 0) {
                bool bad = check_invariants(d.m, s) != 0;
                for (int e = 0; e < ne; ++e)
                    bad |= en[e].op == OP_CLOCKTICK && (s.nrp_work != s.all_nwe || s.all_nwe == 0);
                if (bad) atomicAdd(&lv[4], 1ull);
            }
            if (ne == 0) {
                if (lane == 0) {
                    if (is_terminal(d.m, s)) {
                        atomicAdd(&lv[2], 1ull);
                        atomicMin(&lv_min, (long long)s.time);
                        atomicMax(&lv_max, (long long)s.time);
                    } else {
                        atomicAdd(&lv[3], 1ull);
                        atomicOr(&lv_flags, 8);
                    }
                }
            } else if (tot_states + *(volatile unsigned long long*)&lv[0] >= a.cfg_cap) {
                if (lane == 0) atomicOr(&lv_flags, 1);  // explore.cpp:28
            } else if (a.depth_cap && level >= a.depth_cap) {
                if (lane == 0) atomicOr(&lv_flags, 2);  // explore.cpp:124-127
            } else {
                if (lane == 0) atomicAdd(&lv[1], (unsigned long long)ne);
                CanonMasks cm{0u, 0u, 0u};  // canonical successors only (explore_kernel)
                if (a.canon) cm = canon_masks(d.m, s, lane);
                for (int base = 0; base < ne; base += 32) {
                    const int e = base + lane;
                    uint64_t Hc = H;
                    bool ok = false;
                    if (e < ne && (!a.canon || canonical_successor(en[e], cm, lognwe))) {
                        copy_key<SW>(row, pwords);
                        ok = true;
                        if (!fast_successor(d, s, en[e], row, hk, Hc)) {
                            copy_state(d.m, t, s);
                            ok = apply(d.m, t, to_pid(d.m, en[e]));
                            if (ok) {
                                pack(d, cfg, t, row);
                                Hc = 0;
                                for (int k = 0; k < words; ++k) Hc += (uint64_t)row[k] * hk[k];
                            } else {
                                atomicOr(&lv_flags, 8);
                            }
                        }
                    }
                    __syncwarp();
                    MCTB_LPH(6);  // successor rows
                    int r = 0;
                    if (ok) r = level_insert(tags[nx], kn, list[nx], &n_list[nx], words, row,
                                             fmix64(Hc), &lv_flags);
                    const unsigned nn = __popc(__ballot_sync(0xffffffffu, r == 1));
                    if (lane == 0 && nn) atomicAdd(&lv[0], (unsigned long long)nn);
                    MCTB_LPH(7);  // insert
                }
            }
            __syncwarp();
        }
        MCTB_LPH(1);  // warp 0's other work
        __syncthreads();
        MCTB_LPH(2);  // waiting for the level's other warps
        if (lv_flags & 8) {
            status = 3;
            break;
        }
        wide_levels = n > a.wide ? wide_levels + 1 : 0;
        if (lv_jump) {
            win_levels = win_states = 0;
        } else {
            ++win_levels;
            win_states += n;
        }
        const bool slow_window = win_levels >= a.window && win_states >= a.window_states;
        if (win_levels >= a.window) win_levels = win_states = 0;
        if ((lv_flags & 4) || n_list[nx] > a.max_width || wide_levels >= a.wide_run ||
            slow_window) {
            // too wide: this level goes to the global sweep, unexpanded
            for (unsigned i = threadIdx.x; i < n * words; i += kLvlThreads)
                a.frontier[(size_t)cfg * kLvlWidth * words + i] = kc[list[cur][i / words] * words + i % words];
            status = 1;
            handed = n;
            break;
        }
        if (threadIdx.x == 0) tot_states += lv[0];
        level += lv_jump;
        acc_trans += lv[1];
        acc_terms += lv[2];
        acc_dead += lv[3];
        acc_viol += lv[4];
        acc_min = min(acc_min, lv_min);
        acc_max = max(acc_max, lv_max);
        acc_flags |= lv_flags;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BfsStats& st = a.stats[cfg];
        // the global sweep counts a handed-off level again as its seeds
        st.states = tot_states - handed;
        st.transitions = acc_trans;
        st.terminals = acc_terms;
        st.min_time = acc_min;
        st.max_time = acc_max;
        st.deadlocks = acc_dead;
        st.capped = (acc_flags & 1) ? 1 : 0;
        st.violations = acc_viol;
        st.depth_cut = (acc_flags & 2) ? 1 : 0;
        int64_t* fs = a.fstat + 4 * cfg;
        fs[0] = status;
        fs[1] = handed;
        fs[2] = level;
#ifdef MCTB_BFS_PHASES
        if (level > 100000) {
            printf("[level] cfg %d levels %u warp0 expansions %lld cycles per level: clear %.0f "
                   "other %.0f wait %.0f commit %.0f | per warp-0 expansion: unpack %.0f enum %.0f "
                   "rows %.0f insert %.0f\n",
                   cfg, level, lph[8], (double)lph[0] / level, (double)lph[1] / level,
                   (double)lph[2] / level, (double)lph[3] / level, (double)lph[4] / lph[8],
                   (double)lph[5] / lph[8], (double)lph[6] / lph[8], (double)lph[7] / lph[8]);
        }
#endif
    }
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

uint64_t depth_bound(const MachDesc& m, int64_t protocol_steps) {
    // every tick consumes >= 1 busy tick of some element (bfs_layout's time bound)
    const int64_t groups = (int64_t)m.device_rounds * m.nwu;
    const int64_t per_item = m.kernel == 0 ? (int64_t)m.reps * (m.gmt * m.ts + m.ts) + m.gmt
                                           : (int64_t)m.ts * m.gmt + m.nwe + m.gmt;
    return (uint64_t)protocol_steps + (uint64_t)(groups * m.wg * per_item + 1);
}

// Descriptors, packed layouts and field tables of a sweep (bfs_plan) — shared by
// the single-device run (run_bfs) and the multi-GPU partitions (mctb_explore_mp_*).
struct BfsPlan {
    int n_cfg = 0, words = 1, sw = 16;
    std::vector<BfsDesc> descs;
    std::vector<uint2> ftab;
    std::vector<int> nfields;
    int32_t* d_ids = nullptr;  // minimum-kernel value ids (device)
};

static int bfs_plan(std::vector<MachHost>& hs, cudaStream_t st, BfsPlan* pl) {
    pl->n_cfg = (int)hs.size();
    pl->descs.resize(pl->n_cfg);
    int rc = upload_desc(hs[0], st, &pl->d_ids);
    if (rc) return rc;
    for (int c = 0; c < pl->n_cfg; ++c) {
        MachDesc m = hs[c].d;
        m.input_id = pl->d_ids;
        pl->descs[c].m = m;
        pl->descs[c].l = bfs_layout(m, pl->n_cfg);
        if (pl->descs[c].l.time > 32 || pl->descs[c].l.words > kMaxWords) {
            set_error("state does not fit the GPU packing (time > 2^32 or > 24 words)");
            cudaFreeAsync(pl->d_ids, st);
            pl->d_ids = nullptr;
            return MCTB_LIMIT;
        }
        pl->words = std::max(pl->words, pl->descs[c].l.words);
    }
    // field tables of the table-driven unpack
    pl->ftab.assign((size_t)pl->n_cfg * kMaxFields, uint2{0, 0});
    pl->nfields.assign(pl->n_cfg, 0);
    for (int c = 0; c < pl->n_cfg; ++c)
        pl->nfields[c] = build_field_table(pl->descs[c].m, pl->descs[c].l,
                                           pl->ftab.data() + (size_t)c * kMaxFields);
    // slot stride: key words + guard padding + 8-byte tag in one 64- or 128-byte line
    pl->sw = pl->words <= 14 ? 16 : 32;
    return MCTB_OK;
}

using ExploreFn = void (*)(BfsArgs);
using SeedFn = void (*)(BfsArgs, const uint32_t*, int, const uint32_t*);

static ExploreFn explore_fn(int sw, bool sys) {
    if (sw == 16) return sys ? explore_kernel<16, true> : explore_kernel<16, false>;
    return sys ? explore_kernel<32, true> : explore_kernel<32, false>;
}
static SeedFn seed_fn(int sw, bool sys) {
    if (sw == 16) return sys ? seed_kernel<16, true> : seed_kernel<16, false>;
    return sys ? seed_kernel<32, true> : seed_kernel<32, false>;
}

// Persistent grid of the exploration kernel: blocks per SM and dynamic shared memory.
static int bfs_grid(ExploreFn kern, int sw, int* grid, size_t* dyn_smem) {
    int dev = 0, sms = 0, per_sm = 0;
    MCTB_CUDA(cudaGetDevice(&dev));
    MCTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    *dyn_smem = (size_t)(kBfsThreads / 32) * 34 * sw * sizeof(uint32_t);
    // static (parent states, enabled lists) + dynamic (rows) may exceed the 48 KB default
    MCTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)*dyn_smem));
    MCTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBfsThreads, *dyn_smem));
    if (per_sm < 1) per_sm = 1;
    // 4 blocks of 256 threads is the register-file limit at 64 registers; more
    // resident warps (a register-capped build) spill and run slower
    if (const char* e = getenv("MCTB_BFS_BLOCKS_PER_SM")) per_sm = std::min(per_sm, atoi(e));
    else per_sm = std::min(per_sm, 4);
    *grid = sms * per_sm;
    return MCTB_OK;
}

// Bytes of one partition (table + queue + counters [+ depths]) and the counters'
// offset.
static size_t part_bytes(uint64_t cap, int sw, size_t* misc_off, bool depth = false) {
    const size_t sz_table = cap * 4 * (size_t)sw, sz_q = (cap / 2) * 4;
    *misc_off = sz_table + sz_q;
    return sz_table + sz_q + 256 + (depth ? cap * 4 : 0);
}

static void part_at(char* base, uint64_t cap, int sw, BfsPart* p, bool depth = false) {
    size_t misc_off = 0;
    part_bytes(cap, sw, &misc_off, depth);
    p->table = (uint32_t*)base;
    p->queue = (uint32_t*)(base + cap * 4 * (size_t)sw);
    char* misc = base + misc_off;
    p->head = (unsigned long long*)misc;
    p->tq = (unsigned long long*)(misc + 8);
    p->error = (int*)(misc + 24);
    p->depth = depth ? (uint32_t*)(misc + 256) : nullptr;
}

static int part_clear(char* base, uint64_t cap, int sw, cudaStream_t st, bool depth = false) {
    size_t misc_off = 0;
    part_bytes(cap, sw, &misc_off, depth);
    MCTB_CUDA(cudaMemsetAsync(base, 0, cap * 4 * (size_t)sw, st));
    MCTB_CUDA(cudaMemsetAsync(base + cap * 4 * (size_t)sw, 0xff, (cap / 2) * 4, st));
    MCTB_CUDA(cudaMemsetAsync(base + misc_off, 0, 256 + (depth ? cap * 4 : 0), st));
    return MCTB_OK;
}

// The shared block of a launch: statistics, descriptors, field tables (+ the
// op histogram of diagnostics).  Returns its size.
static size_t shared_bytes(const BfsPlan& pl) {
    return 512 + (sizeof(BfsStats) + sizeof(BfsDesc)) * pl.n_cfg + pl.ftab.size() * 8 +
           pl.nfields.size() * 4;
}

static int shared_init(const BfsPlan& pl, char* blk, BfsArgs* a, cudaStream_t st) {
    a->op_hist = getenv("MCTB_BFS_OPHIST") ? (unsigned long long*)(blk + 32) : nullptr;
    a->stats = (BfsStats*)(blk + 512);
    a->descs = (BfsDesc*)(blk + 512 + sizeof(BfsStats) * pl.n_cfg);
    uint2* d_ftab = (uint2*)(blk + 512 + (sizeof(BfsStats) + sizeof(BfsDesc)) * pl.n_cfg);
    a->ftab = d_ftab;
    a->nfields = (const int*)(d_ftab + pl.ftab.size());
    MCTB_CUDA(cudaMemsetAsync(blk, 0, 512, st));
    MCTB_CUDA(cudaMemcpyAsync(d_ftab, pl.ftab.data(), pl.ftab.size() * 8, cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMemcpyAsync(d_ftab + pl.ftab.size(), pl.nfields.data(), pl.nfields.size() * 4,
                              cudaMemcpyHostToDevice, st));
    std::vector<BfsStats> init(pl.n_cfg);
    for (auto& x : init) x = BfsStats{0, 0, 0, INT64_MAX, -1, 0, 0, 0, 0, 0};
    MCTB_CUDA(cudaMemcpyAsync(a->stats, init.data(), sizeof(BfsStats) * pl.n_cfg,
                              cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMemcpyAsync((void*)a->descs, pl.descs.data(), sizeof(BfsDesc) * pl.n_cfg,
                              cudaMemcpyHostToDevice, st));
    a->n_cfg = pl.n_cfg;
    a->words = pl.words;
    a->cfg_bits = pl.descs[0].l.cfg;
    return MCTB_OK;
}

static int seed_launch(const BfsPlan& pl, const BfsArgs& a, bool sys, const std::vector<uint32_t>* seeds,
                       cudaStream_t st, const std::vector<uint32_t>* seed_depths = nullptr) {
    uint32_t* d_seeds = nullptr;
    uint32_t* d_dep = nullptr;
    int n_seeds = 0;
    if (seeds && !seeds->empty()) {
        n_seeds = (int)(seeds->size() / pl.words);
        MCTB_CUDA(cudaMallocAsync(&d_seeds, seeds->size() * 4, st));
        MCTB_CUDA(cudaMemcpyAsync(d_seeds, seeds->data(), seeds->size() * 4, cudaMemcpyHostToDevice, st));
        if (seed_depths && (int)seed_depths->size() == n_seeds) {
            MCTB_CUDA(cudaMallocAsync(&d_dep, n_seeds * 4, st));
            MCTB_CUDA(cudaMemcpyAsync(d_dep, seed_depths->data(), n_seeds * 4,
                                      cudaMemcpyHostToDevice, st));
        }
    }
    const int n_first = seeds ? n_seeds : pl.n_cfg;
    seed_fn(pl.sw, sys)<<<(n_first + 127) / 128 + 1, 128, 0, st>>>(a, d_seeds, n_seeds, d_dep);
    if (d_seeds) cudaFreeAsync(d_seeds, st);
    if (d_dep) cudaFreeAsync(d_dep, st);
    MCTB_CUDA(cudaGetLastError());
    return MCTB_OK;
}

// The visited tables live in one per-device buffer reused across sweeps:
// cudaMalloc maps even 32 GB in a few ms, while growing the stream-ordered pool
// cost ~80 ms per GB (B200), more than most sweeps take.  A sweep leases the
// cached buffer when it is large enough, else allocates its own; on return the
// larger of the two stays cached.
namespace {
struct TableCache {
    std::mutex mu;
    void* p[64] = {};
    size_t bytes[64] = {};
};
TableCache& table_cache() {
    static TableCache c;
    return c;
}
}  // namespace

static int table_lease(size_t bytes, void** out, size_t* got) {
    int dev = 0;
    MCTB_CUDA(cudaGetDevice(&dev));
    TableCache& c = table_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.p[dev] && c.bytes[dev] >= bytes) {
            *out = c.p[dev];
            *got = c.bytes[dev];
            c.p[dev] = nullptr;
            c.bytes[dev] = 0;
            return MCTB_OK;
        }
    }
    if (cudaMalloc(out, bytes) != cudaSuccess) {
        cudaGetLastError();
        // the cached (smaller) buffer may be what is missing: release it and retry
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.p[dev]) {
            cudaFree(c.p[dev]);
            c.p[dev] = nullptr;
            c.bytes[dev] = 0;
        }
        MCTB_CUDA(cudaMalloc(out, bytes));
    }
    *got = bytes;
    return MCTB_OK;
}

static void table_return(void* p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    TableCache& c = table_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.p[dev] || c.bytes[dev] < bytes) {
        if (c.p[dev]) cudaFree(c.p[dev]);
        c.p[dev] = p;
        c.bytes[dev] = bytes;
    } else {
        cudaFree(p);
    }
}

static size_t table_cached_bytes() {
    int dev = 0;
    cudaGetDevice(&dev);
    TableCache& c = table_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    return c.bytes[dev];
}

// A leased table buffer, returned when the attempt ends (after its stream drains).
struct TableLease {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;
    ~TableLease() {
        if (p) {
            cudaStreamSynchronize(st);
            table_return(p, bytes);
        }
    }
};

// Stream-ordered free at scope exit (every early error return included).
struct AsyncFree {
    void* p;
    cudaStream_t st;
    ~AsyncFree() {
        if (p) cudaFreeAsync(p, st);
    }
};

// The narrow-graph pass (level_kernel): one CTA per configuration.  Returns the
// statistics of the levels it completed and, for every configuration that
// outgrew it, the level handed to the global sweep (keys and depths).
struct LevelPass {
    std::vector<BfsStats> stats;
    std::vector<uint32_t> seeds, seed_depths;
    int handed = 0;   // configurations handed off
    int error = 0;    // 3: model bug (deadlock or inapplicable transition)
    double ms = 0;
};

static int level_pass(const BfsPlan& pl, uint64_t cfg_cap, uint32_t depth_cap, bool check_inv,
                      cudaStream_t st, LevelPass* out) {
    const int n_cfg = pl.n_cfg, words = pl.words;
    char* blk = nullptr;
    const size_t sb = (shared_bytes(pl) + 255) & ~(size_t)255;
    const size_t fb = (size_t)n_cfg * kLvlWidth * words * 4;
    MCTB_CUDA(cudaMallocAsync(&blk, sb + fb + (size_t)n_cfg * 32, st));
    const AsyncFree guard{blk, st};
    BfsArgs ba{};
    int rc = shared_init(pl, blk, &ba, st);
    if (rc) return rc;
    LevelArgs la{};
    la.descs = ba.descs;
    la.ftab = ba.ftab;
    la.nfields = ba.nfields;
    la.stats = ba.stats;
    la.words = words;
    la.cfg_bits = ba.cfg_bits;
    la.check_inv = check_inv ? 1 : 0;
    la.cfg_cap = cfg_cap;
    la.depth_cap = depth_cap;
    la.frontier = (uint32_t*)(blk + sb);
    la.fstat = (int64_t*)(blk + sb + fb);
    la.skip = getenv("MCTB_BFS_NOSKIP") ? 0 : 1;
    la.canon = getenv("MCTB_BFS_NOCANON") ? 0 : 1;
    la.max_width = kLvlWidth;
    la.wide = 24;
    la.wide_run = 32;
    if (const char* e = getenv("MCTB_BFS_LEVEL_WIDTH"))
        la.max_width = (unsigned)std::min(std::max(atoi(e), 1), kLvlWidth);
    if (const char* e = getenv("MCTB_BFS_LEVEL_WIDE")) la.wide = (unsigned)std::max(atoi(e), 1);
    if (const char* e = getenv("MCTB_BFS_LEVEL_RUN")) la.wide_run = (unsigned)std::max(atoi(e), 1);
    la.window = 1024;
    la.window_states = 2048;
    if (const char* e = getenv("MCTB_BFS_LEVEL_WINDOW")) la.window = (unsigned)std::max(atoi(e), 1);
    if (const char* e = getenv("MCTB_BFS_LEVEL_WSTATES"))
        la.window_states = (unsigned)std::max(atoi(e), 1);
    const size_t dyn = (2 * (size_t)kLvlSlots * words + (kLvlThreads / 32) * 34 * (size_t)pl.sw) * 4;
    auto kern = pl.sw == 16 ? level_kernel<16> : level_kernel<32>;
    MCTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    cudaEvent_t e0, e1;
    MCTB_CUDA(cudaEventCreate(&e0));
    MCTB_CUDA(cudaEventCreate(&e1));
    cudaEventRecord(e0, st);
    kern<<<n_cfg, kLvlThreads, dyn, st>>>(la);
    cudaEventRecord(e1, st);
    MCTB_CUDA(cudaGetLastError());
    out->stats.resize(n_cfg);
    std::vector<int64_t> fs(4 * (size_t)n_cfg);
    MCTB_CUDA(cudaMemcpyAsync(out->stats.data(), ba.stats, sizeof(BfsStats) * n_cfg,
                              cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaMemcpyAsync(fs.data(), la.fstat, fs.size() * 8, cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out->ms = ms;
    out->handed = 0;
    out->error = 0;
    for (int c = 0; c < n_cfg; ++c) {
        if (fs[4 * c] == 3) out->error = 3;
        if (fs[4 * c] != 1) continue;
        const size_t n = (size_t)fs[4 * c + 1];
        const size_t o = out->seeds.size();
        out->seeds.resize(o + n * words);
        MCTB_CUDA(cudaMemcpyAsync(out->seeds.data() + o, la.frontier + (size_t)c * kLvlWidth * words,
                                  n * words * 4, cudaMemcpyDeviceToHost, st));
        out->seed_depths.insert(out->seed_depths.end(), n, (uint32_t)fs[4 * c + 2]);
        ++out->handed;
    }
    MCTB_CUDA(cudaStreamSynchronize(st));
    return MCTB_OK;
}

int dfs_prefix_stats(MachHost& h, int64_t max_depth, uint64_t cap, int64_t run_len,
                     int64_t* applies, int64_t* max_depth_reached) {
    constexpr uint64_t kLimit = 1ull << 22;    // states ranked at most
    constexpr int64_t kMaxLevels = 16384;      // one host round trip per level
    if (cap >= kLimit || std::min(run_len, max_depth) >= kMaxLevels) {
        set_error("the capped state graph is beyond the ranking's bounds");
        return MCTB_LIMIT;
    }
    // the graph's size within max_depth, from the (fast) sweep capped at the bound:
    // ranking a graph that turns out too large would be wasted work
    std::vector<MachHost> one(1, h);
    BfsResult r;
    cudaStream_t st;
    MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int rc = run_bfs(one, kLimit + 64, kLimit, &r, st, false, nullptr, 1, false, 0,
                     (uint32_t)std::min<int64_t>(max_depth, 0x7fffffff));
    cudaStreamDestroy(st);
    if (rc) return rc;
    if (r.error == 3) {
        set_error("model bug: deadlock or inapplicable transition during exploration");
        return MCTB_MODEL_BUG;
    }
    if (r.error || r.stats[0].states >= kLimit) {
        set_error("the capped state graph exceeds the ranking's size bound");
        return MCTB_LIMIT;
    }
    return lexrank_prefix(h, max_depth, cap, r.stats[0].states, applies, max_depth_reached);
}

int run_bfs(std::vector<MachHost>& hs, uint64_t max_states, uint64_t cfg_cap, BfsResult* res,
            cudaStream_t st, bool check_invariants, const std::vector<uint32_t>* seeds, int n_parts,
            bool sys_scope, uint64_t first_cap, uint32_t depth_cap,
            const std::vector<uint32_t>* seed_depths) {
    const bool dep = depth_cap > 0;
    // Canonical-parent pruning needs every state's canonical parent in the sweep:
    // true from the initial states and from a complete level (the level pass's
    // hand-off), not from arbitrary seeds (the guided walk's abandoned siblings,
    // whose canonical parents can lie outside their reach).
    const bool canon = !seeds && !getenv("MCTB_BFS_NOCANON");
    if (n_parts < 1 || n_parts > kMaxParts) {
        set_error("partitions must be in [1, 8]");
        return MCTB_CONFIG_ERROR;
    }
    BfsPlan pl;
    int rc = bfs_plan(hs, st, &pl);
    if (rc) return rc;
    const AsyncFree ids_guard{pl.d_ids, st};
    const int n_cfg = pl.n_cfg, sw = pl.sw;
    const ExploreFn kern = explore_fn(sw, sys_scope);
    int grid = 0;
    size_t dyn_smem = 0;
    if ((rc = bfs_grid(kern, sw, &grid, &dyn_smem))) return rc;
    size_t free_b = 0, total_b = 0;
    MCTB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    free_b += table_cached_bytes();  // the cached table buffer is ours to reuse
    const double slot_bytes = 4.0 * sw + 2.0 + (dep ? 4.0 : 0.0);  // slot line + queue (+ depth)
    // capacity grows 16x on overflow; the sweep restarts (all counts are rebuilt)
    // first capacity: enough for the bound up to 2^29 slots (a restart loses the
    // work done, so large sweeps start large); then 16x per overflow.  Split over
    // the partitions (each holds ~1/P of the states).
    // load <= 1/4 at the bound: linear probing then averages ~1.2 probes per
    // successor (at 1/2 it was ~1.6: 14% slower on the 1.37e8-state space)
    uint64_t cap = 1ull << 20;
    while (cap < 4 * std::min<uint64_t>(max_states, 1ull << 27)) cap <<= 1;
    // callers whose bound is loose (the tune sweeps: the reference's per-machine
    // cap times the configurations) start small: a fresh multi-GB table costs
    // more to map than the sweep takes
    if (first_cap) cap = std::min(cap, first_cap);
    if (const char* e = getenv("MCTB_BFS_CAP_LOG2")) cap = 1ull << atoi(e);  // tests: force a restart
    const uint64_t cap_limit = [&] {
        uint64_t c = 1024;
        while ((double)(c * 2) * slot_bytes * n_parts < 0.8 * (double)free_b) c <<= 1;
        return c;
    }();
    if (n_parts > 1) {
        uint64_t c = 1ull << 16;
        while (c * n_parts < cap) c <<= 1;
        cap = c;
    }
    cap = std::min(cap, cap_limit);
    const bool trace = getenv("MCTB_BFS_TRACE") != nullptr;
    // narrow graphs first, level by level in shared memory (level_kernel); the
    // configurations that outgrow it continue in the global sweep from the level
    // they reached
    LevelPass lp;
    const bool use_level = !seeds && n_parts == 1 && !sys_scope && !getenv("MCTB_BFS_NOLEVEL");
    if (use_level) {
        if ((rc = level_pass(pl, cfg_cap, depth_cap, check_invariants, st, &lp))) return rc;
        if (trace)
            fprintf(stderr, "[bfs] level pass: %.3f ms, %d of %d configurations handed off\n",
                    lp.ms, lp.handed, n_cfg);
        if (lp.error || lp.handed == 0) {
            res->stats = lp.stats;
            res->states = 0;
            for (auto& x : res->stats) {
                if (x.states >= cfg_cap) x.capped = 1;
                res->states += x.states;
            }
            res->ms = lp.ms;
            res->levels = 0;
            res->error = lp.error;
            res->words = pl.words;
            res->capacity = 0;
            return MCTB_OK;
        }
        seeds = &lp.seeds;
        seed_depths = &lp.seed_depths;
    }
    for (;;) {
        BfsArgs a{};
        a.cap_mask = cap - 1;
        a.queue_cap = cap / 2;
        a.cfg_cap = cfg_cap;
        a.keep = getenv("MCTB_BFS_NOKEEP") ? 0 : 1;
        a.canon = canon ? 1 : 0;
        a.check_inv = check_invariants ? 1 : 0;
        // the visited cap must bound the sweep: every warp publishes its count at
        // least every 64 expansions, and sooner under a small cap, so the states
        // inserted past the cap stay below ~grid warps x 48 (cap <= table / 4)
        a.flush_states = (unsigned)std::min<uint64_t>(
            4096, std::max<uint64_t>(16, cfg_cap / (4ull * grid * (kBfsThreads / 32))));
        a.n_parts = n_parts;
        a.part0 = 0;
        a.n_here = n_parts;
        a.depth_cap = depth_cap;
        size_t misc_off = 0;
        const size_t pb = (part_bytes(cap, sw, &misc_off, dep) + 255) & ~(size_t)255;
        TableLease lease;  // returned to the cache when this attempt ends
        lease.st = st;
        if ((rc = table_lease(pb * n_parts + shared_bytes(pl), &lease.p, &lease.bytes))) return rc;
        char* b = (char*)lease.p;
        for (int p = 0; p < n_parts; ++p) {
            part_at(b + pb * p, cap, sw, &a.part[p], dep);
            if ((rc = part_clear(b + pb * p, cap, sw, st, dep))) return rc;
        }
        if ((rc = shared_init(pl, b + pb * n_parts, &a, st))) return rc;
        if (use_level)  // the narrow pass's counts; the global sweep adds its own
            MCTB_CUDA(cudaMemcpyAsync(a.stats, lp.stats.data(), sizeof(BfsStats) * n_cfg,
                                      cudaMemcpyHostToDevice, st));
        if ((rc = seed_launch(pl, a, sys_scope, seeds, st, seed_depths))) return rc;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        if (trace)
            fprintf(stderr, "[bfs] launch cfgs=%d words=%d sw=%d parts=%d cap=%llu grid=%d smem=%zu\n",
                    n_cfg, pl.words, sw, n_parts, (unsigned long long)cap, grid, dyn_smem);
        kern<<<grid, kBfsThreads, dyn_smem, st>>>(a);
        cudaEventRecord(e1, st);
        MCTB_CUDA(cudaGetLastError());
        res->stats.resize(n_cfg);
        std::vector<unsigned long long> misc_h(32 * n_parts);
        MCTB_CUDA(cudaMemcpyAsync(res->stats.data(), a.stats, sizeof(BfsStats) * n_cfg,
                                  cudaMemcpyDeviceToHost, st));
        for (int p = 0; p < n_parts; ++p)
            MCTB_CUDA(cudaMemcpyAsync(misc_h.data() + 32 * p, b + pb * p + misc_off, 256,
                                      cudaMemcpyDeviceToHost, st));
        unsigned long long hist[64] = {};
        if (a.op_hist)
            MCTB_CUDA(cudaMemcpyAsync(hist, b + pb * n_parts, 512, cudaMemcpyDeviceToHost, st));
        MCTB_CUDA(cudaStreamSynchronize(st));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        res->ms = ms + lp.ms;
        res->states = 0;
        for (const auto& x : res->stats) res->states += x.states;
        res->levels = 0;
        res->error = 0;
        for (int p = 0; p < n_parts; ++p)
            res->error = std::max(res->error, (int)(misc_h[32 * p + 3] & 0xffffffff));
        if (trace)
            for (int p = 0; p < n_parts; ++p)
                fprintf(stderr, "[bfs] part %d: %.3f ms error=%d head=%llu tail=%llu outstanding=%llu\n",
                        p, ms, (int)(misc_h[32 * p + 3] & 0xffffffff), misc_h[32 * p],
                        misc_h[32 * p + 1] >> 32, misc_h[32 * p + 1] & 0xffffffffull);
        if (res->error >= 5) {
            // a watchdog fired (bfs.cu spin loops): report instead of hanging
            char msg[256];
            snprintf(msg, sizeof msg,
                     "exploration stalled (watchdog %d: head %llu, tail %llu, outstanding %llu)",
                     res->error, misc_h[0], misc_h[1] >> 32, misc_h[1] & 0xffffffffull);
            fprintf(stderr, "[mctb] %s\n", msg);
            set_error(msg);
            return MCTB_MODEL_BUG;
        }
        // explore.cpp:28-31: a visited set holding max_states refuses every later
        // insert, so reaching the cap ends the exhaustive claim (statistics are
        // flushed per warp, so the final count decides)
        for (auto& x : res->stats)
            if (x.states >= cfg_cap) x.capped = 1;
        if (a.op_hist) {
            fprintf(stderr, "[explore] generic successors by op:");
            for (int o = 0; o < 19; ++o)
                if (hist[4 + o]) fprintf(stderr, " op%d=%llu", o, hist[4 + o]);
            fprintf(stderr, "\n[explore] table probes (successors built and inserted): %llu\n",
                    hist[4 + 24]);
#ifdef MCTB_BFS_PHASES
            static const char* names[7] = {"pop", "cfg", "unpack", "enum", "rows", "insert", "keep"};
            for (int c = 0; c < 2; ++c) {
                const unsigned long long* ph = hist + 32 + 8 * c;
                fprintf(stderr, "[explore] %s expansions %llu, cycles each:",
                        c ? "chained" : "popped", ph[7]);
                for (int k = 0; k < 7; ++k)
                    fprintf(stderr, " %s=%.0f", names[k], ph[7] ? (double)ph[k] / ph[7] : 0.0);
                fprintf(stderr, "\n");
            }
#endif
        }
        res->words = pl.words;
        res->capacity = cap * n_parts;
        if ((res->error == 1 || res->error == 2) && cap < cap_limit) {
            cap = std::min(cap * 16, cap_limit);
            continue;
        }
        break;
    }
    MCTB_CUDA(cudaStreamSynchronize(st));
    return MCTB_OK;
}

}  // namespace mctb

namespace mctb {

// One rank's share of a multi-GPU exploration (mctb_explore_mp_*): its hash
// partition (cudaMalloc'd so it can be exported over CUDA IPC), the peers'
// partitions mapped into this process, and the launch state.
struct MpCtx {
    int world = 1, rank = 0;
    std::vector<MachHost> hs;
    BfsPlan pl;
    uint64_t cap = 0, cfg_cap = 0;
    size_t pb = 0, misc_off = 0;
    char* local = nullptr;
    char* shared = nullptr;
    char* peer[kMaxParts] = {};
    BfsArgs a{};
    cudaStream_t st = nullptr;
    int grid = 0;
    size_t smem = 0;
    int n_cfg = 0, size = 0, kernel = 0, plat[4] = {};
    std::vector<int32_t> configs;

    ~MpCtx() {
        for (int r = 0; r < kMaxParts; ++r)
            if (peer[r]) cudaIpcCloseMemHandle(peer[r]);
        if (local) cudaFree(local);
        if (shared) cudaFree(shared);
        if (pl.d_ids) cudaFreeAsync(pl.d_ids, st);
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
};

}  // namespace mctb

using namespace mctb;

namespace mctb {
int check_machine(const int* plat, int size, int kernel, int wg, int ts);
}

extern "C" {

int mctb_explore(const int* plat, int size, int kernel, const int64_t* input,
                 const int32_t* configs, int n_configs, int64_t max_states, int64_t max_depth,
                 int flags, int64_t* out, int64_t* info) {
    int rc;
    if (n_configs < 1) {
        set_error("no configurations");
        return MCTB_CONFIG_ERROR;
    }
    if (max_depth < 1) {  // explore.cpp:91
        set_error("max_depth must be >= 1");
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
    // flags: bit 0 invariants; bits 8-11 hash partitions on this device (0 = 1);
    // bit 1 system-scope memory operations (the multi-GPU kernel variant)
    const int n_parts = std::max(1, (flags >> 8) & 15);
    // protocol transitions of every run (steps - time of the cost model): a terminal
    // state of time t sits at depth protocol + t
    std::vector<int64_t> proto(n_configs), cm_time(n_configs);
    uint32_t depth_cap = 0;
    for (int c = 0; c < n_configs; ++c) {
        int logn = 0, lw = 0, lt = 0, lp = 0;
        while ((1 << logn) < size) ++logn;
        while ((1 << lw) < configs[2 * c]) ++lw;
        while ((1 << lt) < configs[2 * c + 1]) ++lt;
        while ((1 << lp) < plat[2]) ++lp;
        const Cost cm = lockstep_cost(kernel, logn, plat[3], Config{plat[0], plat[1], lp, lw, lt});
        proto[c] = cm.steps - cm.time;
        cm_time[c] = cm.time;
        if (depth_bound(hs[c].d, proto[c]) > (uint64_t)max_depth)
            depth_cap = (uint32_t)std::min<int64_t>(max_depth, 0x7fffffff);
    }
    rc = run_bfs(hs, cap * (uint64_t)n_configs, cap, &r, st, (flags & 1) != 0, nullptr, n_parts,
                 (flags & 2) != 0, 0, depth_cap);
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
        o[0] = !s.capped && !s.depth_cut;
        o[1] = (int64_t)std::min<uint64_t>(s.states, cap);
        o[2] = (int64_t)s.transitions;
        // DFS max depth = longest complete run = protocol transitions + max time
        // (pinned against explore_machine in tests/test_bfs_gpu.py); under the depth
        // cap the deepest visited states sit at max_depth
        o[3] = s.depth_cut ? max_depth : s.terminals ? proto[c] + s.max_time : -1;
        if (s.capped) {
            // a full visited set: the DFS's own prefix decides both (lexrank.cu), for
            // graphs of fewer than 2^22 states
            int64_t a = 0, md = 0;
            rc = dfs_prefix_stats(hs[c], max_depth, cap, proto[c] + cm_time[c], &a, &md);
            if (rc == MCTB_OK) {
                o[2] = a;
                o[3] = md;
            } else if (rc != MCTB_LIMIT) {
                return rc;
            }
        }
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

// ---------------------------------------------------------------------------
// Multi-GPU exploration: one process per GPU, each owning one hash partition of
// the visited set.  A successor owned by another rank is probed, claimed and
// queued directly in that rank's table and queue over peer memory (NVLink P2P,
// system-scope atomics); the sweep ends at global quiescence (quiescent()).

int mctb_explore_mp_open(const int* plat, int size, int kernel, const int64_t* input,
                         const int32_t* configs, int n_configs, int64_t max_states, int world,
                         int rank, int flags, void** ctx, void* handle) {
    int rc;
    if (world < 1 || world > kMaxParts || rank < 0 || rank >= world) {
        set_error("world must be in [1, 8] and rank in [0, world)");
        return MCTB_CONFIG_ERROR;
    }
    if (n_configs < 1) {
        set_error("no configurations");
        return MCTB_CONFIG_ERROR;
    }
    std::unique_ptr<MpCtx> holder(new MpCtx);  // every early return frees it (~MpCtx)
    MpCtx* c = holder.get();
    c->world = world;
    c->rank = rank;
    c->n_cfg = n_configs;
    c->size = size;
    c->kernel = kernel;
    for (int i = 0; i < 4; ++i) c->plat[i] = plat[i];
    c->configs.assign(configs, configs + 2 * n_configs);
    c->hs.resize(n_configs);
    auto fail = [](int code) { return code; };
    for (int k = 0; k < n_configs; ++k) {
        if ((rc = check_machine(plat, size, kernel, configs[2 * k], configs[2 * k + 1]))) return fail(rc);
        if ((rc = build_desc(plat, size, kernel, input, configs[2 * k], configs[2 * k + 1], &c->hs[k])))
            return fail(rc);
    }
    if ((rc = require_device())) return fail(rc);
    MCTB_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    if ((rc = bfs_plan(c->hs, c->st, &c->pl))) return fail(rc);
    if ((rc = bfs_grid(explore_fn(c->pl.sw, true), c->pl.sw, &c->grid, &c->smem))) return fail(rc);
    c->cfg_cap = max_states > 0 ? (uint64_t)max_states : 5000000ull;
    // each partition holds ~1/world of the states, table load <= 1/2
    const uint64_t total = c->cfg_cap * (uint64_t)n_configs;
    uint64_t cap = 1ull << 16;
    while (cap * world < 2 * std::min<uint64_t>(total, 1ull << 28)) cap <<= 1;
    if (const char* e = getenv("MCTB_MP_CAP_LOG2")) cap = 1ull << atoi(e);
    c->cap = cap;
    c->pb = (part_bytes(cap, c->pl.sw, &c->misc_off) + 255) & ~(size_t)255;
    MCTB_CUDA(cudaMalloc(&c->local, c->pb));
    if ((rc = part_clear(c->local, cap, c->pl.sw, c->st))) return fail(rc);
    MCTB_CUDA(cudaMalloc(&c->shared, shared_bytes(c->pl)));
    BfsArgs& a = c->a;
    if ((rc = shared_init(c->pl, c->shared, &a, c->st))) return fail(rc);
    a.cap_mask = cap - 1;
    a.queue_cap = cap / 2;
    a.cfg_cap = c->cfg_cap;
    a.keep = 1;
    a.canon = getenv("MCTB_BFS_NOCANON") ? 0 : 1;
    a.check_inv = (flags & 1) ? 1 : 0;
    // as run_bfs: publish warp counts often enough for the visited cap to bind
    a.flush_states = (unsigned)std::min<uint64_t>(
        4096, std::max<uint64_t>(16, c->cfg_cap / (4ull * c->grid * (kBfsThreads / 32) * world)));
    a.n_parts = world;
    a.part0 = rank;
    a.n_here = 1;
    part_at(c->local, cap, c->pl.sw, &a.part[rank]);
    MCTB_CUDA(cudaStreamSynchronize(c->st));
    MCTB_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), c->local));
    *ctx = holder.release();
    return MCTB_OK;
}

int mctb_explore_mp_connect(void* ctx, const void* handles) {
    auto* c = static_cast<MpCtx*>(ctx);
    const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) continue;
        void* p = nullptr;
        MCTB_CUDA(cudaIpcOpenMemHandle(&p, h[r], cudaIpcMemLazyEnablePeerAccess));
        c->peer[r] = static_cast<char*>(p);
        part_at(c->peer[r], c->cap, c->pl.sw, &c->a.part[r]);
    }
    return MCTB_OK;
}

int mctb_explore_mp_seed(void* ctx) {
    auto* c = static_cast<MpCtx*>(ctx);
    int rc = seed_launch(c->pl, c->a, true, nullptr, c->st);
    if (rc) return rc;
    MCTB_CUDA(cudaStreamSynchronize(c->st));
    return MCTB_OK;
}

int mctb_explore_mp_run(void* ctx, int64_t* out, int64_t* info) {
    auto* c = static_cast<MpCtx*>(ctx);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c->st);
    explore_fn(c->pl.sw, true)<<<c->grid, kBfsThreads, c->smem, c->st>>>(c->a);
    cudaEventRecord(e1, c->st);
    MCTB_CUDA(cudaGetLastError());
    std::vector<BfsStats> stats(c->n_cfg);
    unsigned long long misc_h[32];
    MCTB_CUDA(cudaMemcpyAsync(stats.data(), c->a.stats, sizeof(BfsStats) * c->n_cfg,
                              cudaMemcpyDeviceToHost, c->st));
    MCTB_CUDA(cudaMemcpyAsync(misc_h, c->local + c->misc_off, 256, cudaMemcpyDeviceToHost, c->st));
    MCTB_CUDA(cudaStreamSynchronize(c->st));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const int err = (int)(misc_h[3] & 0xffffffff);
    int logn = 0, lp = 0;
    while ((1 << logn) < c->size) ++logn;
    while ((1 << lp) < c->plat[2]) ++lp;
    for (int k = 0; k < c->n_cfg; ++k) {
        const BfsStats& s = stats[k];
        int lw = 0, lt = 0;
        while ((1 << lw) < c->configs[2 * k]) ++lw;
        while ((1 << lt) < c->configs[2 * k + 1]) ++lt;
        const Cost cm = lockstep_cost(c->kernel, logn, c->plat[3],
                                      Config{c->plat[0], c->plat[1], lp, lw, lt});
        int64_t* o = out + 8 * k;
        // this rank's share: states it discovered, transitions and terminals of the
        // states it expanded; the caller sums (min/max for the times) over ranks
        o[0] = (int64_t)s.states;
        o[1] = (int64_t)s.transitions;
        o[2] = (int64_t)s.terminals;
        o[3] = s.terminals ? s.min_time : INT64_MAX;
        o[4] = s.terminals ? s.max_time : -1;
        o[5] = (int64_t)s.deadlocks;
        o[6] = (int64_t)s.violations;
        o[7] = cm.steps - cm.time;  // protocol transitions: max depth = this + max time
    }
    if (info) {
        info[0] = (int64_t)(c->cap * c->world);
        info[1] = c->pl.words;
        info[2] = (int64_t)(ms * 1000.0);
        info[3] = err;
    }
    if (err == 3) {
        set_error("model bug: deadlock or inapplicable transition during exploration");
        return MCTB_MODEL_BUG;
    }
    if (err >= 5) {
        set_error("exploration stalled (watchdog)");
        return MCTB_MODEL_BUG;
    }
    if (err) {
        set_error("a partition's visited table or queue is full (raise max_states)");
        return MCTB_LIMIT;
    }
    return MCTB_OK;
}

void mctb_explore_mp_close(void* ctx) {
    delete static_cast<MpCtx*>(ctx);  // ~MpCtx unmaps the peers and frees this rank's memory
}

}  // extern "C"
