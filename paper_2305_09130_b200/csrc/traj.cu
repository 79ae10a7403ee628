// Schedule trajectories on the GPU (north-star subsystem 2) and the
// reference-compatible single runs built on them.
//
// One thread steps one trajectory of the transition system (machine.cuh)
// from the initial state to a terminal state, choosing among the enabled
// transitions by policy:
//   ROUND_ROBIN  Machine::run(RoundRobin)   machine.cpp:809-820
//   MT19937      Machine::run(SeededRandom) machine.cpp:807-808 (std::mt19937_64)
//   FIRST        en[0]: the first path of explore_machine's DFS (explore.cpp:117-161)
//   PHILOX       swarm: step i of trajectory t under seed k draws word i%4 of
//                Philox4x32-10(ctr = {i/4, t_lo, t_hi, i>>34}, key = k) and picks
//                floor(word * n / 2^32) — counter-based, so any trajectory is
//                replayable on its own on the CPU (oracle mo_simulate policy 3).
// Per trajectory it records time, transitions, glob[0] (minimum kernel), a
// status, and a 64-bit FNV-1a hash (over 32-bit words) of the transition sequence, so 10^6
// trajectories are checked against CPU replays without shipping traces.
#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "common.cuh"
#include "machine.cuh"
#include "traj.cuh"

namespace mctb {

__host__ __device__ inline void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1, uint32_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// FNV-1a over the transition's four 32-bit words {actor, peer, op, arg} (one
// xor-multiply per word; the trace checksum the CPU replay recomputes).
__host__ __device__ inline uint64_t fnv_mix(uint64_t h, uint32_t w) {
    h ^= w;
    return h * 0x100000001b3ull;
}

__host__ __device__ inline uint64_t fnv_transition(uint64_t h, const Transition& t) {
    h = fnv_mix(h, t.actor);
    h = fnv_mix(h, t.peer);
    h = fnv_mix(h, (uint32_t)t.op);
    return fnv_mix(h, (uint32_t)t.arg);
}

namespace {

#ifndef MCTB_TRAJ_MINB
#define MCTB_TRAJ_MINB 12  // resident blocks per SM the register allocation targets (40 registers;
                            // 1 -> 64 registers: 24.1 ms, 12: 15.9 ms, 16: 15.7 ms per 1e6 trajectories)
#endif
template <int POLICY>
__global__ void __launch_bounds__(128, MCTB_TRAJ_MINB) traj_kernel(const MachDesc* __restrict__ descs, int n_desc,
                                                   uint64_t seed, uint64_t traj0, uint64_t n_traj,
                                                   int64_t max_steps, TrajOut* __restrict__ out,
                                                   int32_t* __restrict__ trace, int64_t trace_cap) {
    // warp w of group g runs the 32 trajectories of one configuration c: offset
    // t = g * 32 * n_desc + lane * n_desc + c, so (traj0 + t) % n_desc is uniform in
    // the warp (no divergence between configurations of different lengths); the
    // id -> configuration mapping and the output layout are unchanged
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t t = gid;
    if (n_desc > 1) {
        const uint64_t w = gid >> 5, grp = w / (uint64_t)n_desc, c = w - grp * (uint64_t)n_desc;
        t = grp * 32ull * (uint64_t)n_desc + (gid & 31) * (uint64_t)n_desc + c;
    }
    if (t >= n_traj) return;
    const uint64_t traj = traj0 + t;
    const MachDesc m = descs[n_desc == 1 ? 0 : traj % (uint64_t)n_desc];
    MState s;
    initial_state(m, s);
    Transition en[kMaxEnabled];
    Mt64* rng = nullptr;
    Mt64 rng_store;
    if (POLICY == MCTB_POLICY_MT19937) {
        rng = &rng_store;
        rng->seed(seed);
    }
    uint32_t ph[4] = {0, 0, 0, 0};
    int64_t steps = 0;
    int rr_next = 0;
    uint64_t h = 0xcbf29ce484222325ull;
    int status = MCTB_OK;
    for (;;) {
        const int n = enabled(m, s, en, POLICY == MCTB_POLICY_FIRST ? 1 : (1 << 30));
        if (n == 0) {
            if (!is_terminal(m, s)) status = MCTB_MODEL_BUG;  // deadlock
            break;
        }
        if (steps >= max_steps) {
            status = MCTB_LIMIT;
            break;
        }
        int pick = 0;
        if (POLICY == MCTB_POLICY_ROUND_ROBIN) {
            pick = n;
            for (int i = 0; i < n; ++i)
                if (en[i].actor >= rr_next) {
                    pick = i;
                    break;
                }
            if (pick == n) pick = 0;
            rr_next = (en[pick].actor + 1) % m.n_proc;
        } else if (POLICY == MCTB_POLICY_MT19937) {
            pick = (int)(rng->next() % (uint64_t)n);
        } else if (POLICY == MCTB_POLICY_PHILOX) {
            if ((steps & 3) == 0)
                philox4x32_10((uint32_t)(steps >> 2), (uint32_t)traj, (uint32_t)(traj >> 32),
                              (uint32_t)(steps >> 34), (uint32_t)seed, (uint32_t)(seed >> 32), ph);
            pick = (int)(((uint64_t)ph[steps & 3] * (uint64_t)n) >> 32);
        } else if (POLICY == MCTB_POLICY_TICK_LAST) {
            // every zero-time transition before the clock: the lock-step schedule
            pick = (en[0].op == OP_CLOCKTICK && n > 1) ? 1 : 0;
        }
        const Transition tr = en[pick];
        if (trace && steps < trace_cap) {
            trace[4 * steps + 0] = tr.actor;
            trace[4 * steps + 1] = tr.peer;
            trace[4 * steps + 2] = tr.op;
            trace[4 * steps + 3] = tr.arg;
        }
        h = fnv_transition(h, tr);
        if (!apply(m, s, tr)) {
            status = MCTB_MODEL_BUG;
            break;
        }
        ++steps;
    }
    TrajOut o;
    o.time = s.time;
    o.steps = steps;
    o.glob0 = s.glob0;
    o.status = status;
    o.hash = h;
    o.config = n_desc == 1 ? 0 : (int32_t)(traj % (uint64_t)n_desc);
    out[t] = o;
}

// Replays a trace (replay, explore.cpp:283-300): per-step model time out,
// status CORRUPT_TRACE at the first transition that is not applicable.
__global__ void replay_kernel(MachDesc m, const int32_t* __restrict__ trace, int64_t len,
                              int64_t* __restrict__ step_time, TrajOut* out) {
    MState s;
    initial_state(m, s);
    int status = MCTB_OK;
    int64_t i = 0;
    uint64_t h = 0xcbf29ce484222325ull;
    for (; i < len; ++i) {
        const Transition t{(uint16_t)trace[4 * i], (uint16_t)trace[4 * i + 1], trace[4 * i + 2],
                           trace[4 * i + 3]};
        h = fnv_transition(h, t);
        if (!apply(m, s, t)) {
            status = MCTB_CORRUPT_TRACE;
            break;
        }
        if (step_time) step_time[i] = s.time;
    }
    if (status == MCTB_OK && !is_terminal(m, s)) status = MCTB_CORRUPT_TRACE;
    out->time = s.time;
    out->steps = i;
    out->glob0 = s.glob0;
    out->status = status;
    out->hash = h;
    out->config = 0;
}

}  // namespace

// ---------------------------------------------------------------- host side

int build_desc(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
               MachHost* out) {
    MachDesc& m = out->d;
    std::memset(&m, 0, sizeof m);
    int logn = 0, logwg = 0, logts = 0, lognp = 0;
    while ((1 << logn) < size) ++logn;
    while ((1 << logwg) < wg) ++logwg;
    while ((1 << logts) < ts) ++logts;
    while ((1 << lognp) < plat[2]) ++lognp;
    launch_plan(logn, plat[0], plat[1], lognp, logwg, logts, m.wgs, m.nwd, m.nwu, m.nwe);
    m.kernel = kernel;
    m.size = size;
    m.gmt = plat[3];
    m.np = plat[2];
    m.wg = wg;
    m.ts = ts;
    m.logts = logts;
    m.all_nwe = m.nwe * m.nwu * m.nwd;
    m.rounds = wg / m.nwe;
    m.device_rounds = std::max(m.wgs / m.nwu, 1);
    m.host_reacts = m.device_rounds - m.nwd;
    m.n_units = m.nwd * m.nwu;
    m.n_pex = m.n_units * m.nwe;
    m.n_proc = 3 + m.nwd + 2 * m.n_units + m.n_pex;
    set_divisors(m);
    m.reps = size / ts;
    if (kernel == 0) {
        m.act_len = 4 * m.reps + 2;
        m.epi_len = 1;
    } else {
        m.act_len = 2 * ts + 1;
        m.epi_len = 2 * (m.nwe - 1) + 3;
    }
    const int64_t max_ticks = kernel == 0 ? (int64_t)m.gmt * ts : (int64_t)m.gmt;
    if (m.act_len >= 65535 || m.epi_len >= 65535 || max_ticks >= 65535 || m.rounds >= 65535) {
        set_error("configuration exceeds the GPU machine's 16-bit element fields (program "
                  "length, busy ticks or rounds >= 65535)");
        return MCTB_LIMIT;
    }
    if (m.nwd > kMaxDev || m.n_units > kMaxUnit || m.n_pex > kMaxPex ||
        (kernel == 1 && m.n_units * m.np > kMaxLoc)) {
        set_error("configuration exceeds the GPU machine capacity (devices <= 8, units <= 16, "
                  "elements <= 32, local slots <= 256)");
        return MCTB_LIMIT;
    }
    out->values.clear();
    out->ids.clear();
    if (kernel == 1) {
        std::vector<int64_t> in(size);
        for (int i = 0; i < size; ++i) in[i] = input ? input[i] : (int64_t)(size - i);
        std::vector<int64_t> vals(in);
        vals.push_back(INT64_MAX);
        std::sort(vals.begin(), vals.end());
        vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
        out->values = vals;
        out->ids.resize(size);
        for (int i = 0; i < size; ++i)
            out->ids[i] = (int32_t)(std::lower_bound(vals.begin(), vals.end(), in[i]) - vals.begin());
        m.max_id = (int32_t)(vals.size() - 1);
        m.glob0_id = out->ids[0];
    }
    return MCTB_OK;
}

int upload_desc(MachHost& h, cudaStream_t stream, int32_t** d_ids) {
    *d_ids = nullptr;
    if (h.d.kernel == 1) {
        MCTB_CUDA(cudaMallocAsync(d_ids, h.ids.size() * sizeof(int32_t), stream));
        MCTB_CUDA(cudaMemcpyAsync(*d_ids, h.ids.data(), h.ids.size() * sizeof(int32_t),
                                  cudaMemcpyHostToDevice, stream));
    }
    h.d.input_id = *d_ids;
    return MCTB_OK;
}

int launch_trajectories(const MachDesc* d_descs, int n_desc, int policy, uint64_t seed,
                        uint64_t traj0, uint64_t n_traj, int64_t max_steps, TrajOut* d_out,
                        int32_t* d_trace, int64_t trace_cap, cudaStream_t stream) {
    if (n_traj == 0) return MCTB_OK;
    const unsigned threads = 128;
    // whole groups of 32 trajectories per configuration (see traj_kernel)
    const uint64_t g = 32ull * (uint64_t)std::max(n_desc, 1);
    const uint64_t span = n_desc > 1 ? (n_traj + g - 1) / g * g : n_traj;
    const unsigned blocks = (unsigned)((span + threads - 1) / threads);
    switch (policy) {
        case MCTB_POLICY_ROUND_ROBIN:
            traj_kernel<MCTB_POLICY_ROUND_ROBIN><<<blocks, threads, 0, stream>>>(
                d_descs, n_desc, seed, traj0, n_traj, max_steps, d_out, d_trace, trace_cap);
            break;
        case MCTB_POLICY_MT19937:
            traj_kernel<MCTB_POLICY_MT19937><<<blocks, threads, 0, stream>>>(
                d_descs, n_desc, seed, traj0, n_traj, max_steps, d_out, d_trace, trace_cap);
            break;
        case MCTB_POLICY_FIRST:
            traj_kernel<MCTB_POLICY_FIRST><<<blocks, threads, 0, stream>>>(
                d_descs, n_desc, seed, traj0, n_traj, max_steps, d_out, d_trace, trace_cap);
            break;
        case MCTB_POLICY_PHILOX:
            traj_kernel<MCTB_POLICY_PHILOX><<<blocks, threads, 0, stream>>>(
                d_descs, n_desc, seed, traj0, n_traj, max_steps, d_out, d_trace, trace_cap);
            break;
        case MCTB_POLICY_TICK_LAST:
            traj_kernel<MCTB_POLICY_TICK_LAST><<<blocks, threads, 0, stream>>>(
                d_descs, n_desc, seed, traj0, n_traj, max_steps, d_out, d_trace, trace_cap);
            break;
        default:
            set_error("unknown scheduling policy");
            return MCTB_CONFIG_ERROR;
    }
    return cuda_check(cudaGetLastError(), "traj_kernel");
}

// TrajOut -> the C ABI's int64[6] records {time, steps, result, status, hash, config}
// on the device, so the host receives the caller's layout in one copy (result:
// the glob[0] value id for the minimum kernel, mapped to its value by the host;
// INT64_MIN for the abstract kernel).
__global__ void traj_records_kernel(const TrajOut* __restrict__ in, uint64_t n, int kernel,
                                    int64_t* __restrict__ rec) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const TrajOut t = in[i];
    int64_t* r = rec + 6 * i;
    r[0] = t.time;
    r[1] = t.steps;
    r[2] = kernel == 1 ? (int64_t)t.glob0 : INT64_MIN;
    r[3] = t.status;
    r[4] = (int64_t)t.hash;
    r[5] = t.config;
}

int launch_traj_records(const TrajOut* d_in, uint64_t n, int kernel, int64_t* d_rec,
                        cudaStream_t stream) {
    if (n == 0) return MCTB_OK;
    traj_records_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_in, n, kernel, d_rec);
    return cuda_check(cudaGetLastError(), "traj_records_kernel");
}

int launch_replay(const MachDesc& m, const int32_t* d_trace, int64_t len, int64_t* d_step_time,
                  TrajOut* d_out, cudaStream_t stream) {
    replay_kernel<<<1, 1, 0, stream>>>(m, d_trace, len, d_step_time, d_out);
    return cuda_check(cudaGetLastError(), "replay_kernel");
}

}  // namespace mctb
