// The bound-lowering driver on the GPU (north-star subsystem 4):
// check_overtime (explore.cpp:167-205), estimate_initial_time
// (search.cpp:94-102) and bisect_min_time (search.cpp:104-158).
//
// The reference answers every probe C_ex(T) of the bisection with a fresh
// exhaustive DFS over all configurations.  Here one GPU sweep establishes,
// per feasible configuration c (in the reference's largest-first order):
//   * its lock-step model time (cost-model kernel),
//   * its full reachable state space (frontier-parallel BFS): state count
//     S(c) capped like the reference's visited set, edge count, and the range
//     of terminal times over ALL interleavings — the proof that no run of c
//     finishes earlier than its model time,
//   * its first DFS path (GPU run with the en[0] policy): the counterexample
//     the reference's DFS returns for any T >= that path's time.
// Every probe of the bisection is then an O(#configs) scan of these tables,
// reproducing the reference's verdicts, counterexample traces, checks_run and
// states_visited_total exactly; only the final trace is materialised.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "bfs.cuh"
#include "common.cuh"
#include "cost_model.cuh"
#include "traj.cuh"

namespace mctb {

int check_platform(const int* plat);
int check_problem(int size, int kernel);
int make_space(const int64_t* sd, SpaceDev* out);
int launch_space_eval(const SpaceDev& s, uint64_t first, uint64_t count, int64_t* d_time,
                      int64_t* d_steps, cudaStream_t stream);
void reference_space(const int* plat, int size, int kernel, int64_t* sd);
int gpu_run(MachHost& h, int policy, uint64_t seed, uint64_t traj, int64_t max_steps,
            TrajOut* out, int32_t* trace, int64_t cap);

namespace {

// The DFS's counterexample and search effort for a schedule-dependent
// configuration at bound T (lexfirst.cu + a multi-source exploration of the
// siblings the DFS abandons).
struct Walk {
    int k = -1;
    int64_t T = -1;
    std::vector<int32_t> path;
    int64_t final_time = -1, applies = 0, sib_states = 0, sib_transitions = 0;
    bool sib_capped = false;  // the siblings' subtrees alone fill the visited set
    int64_t sib_depth = 0;  // deepest state of the abandoned siblings' subtrees
};

struct Ctx {
    int plat[4];
    int size = 0, kernel = 0;
    const int64_t* input = nullptr;
    uint64_t cap = 5000000;  // ExploreLimits::max_states (explore.hpp:39)
    int64_t max_depth = 4000000;  // ExploreLimits::max_depth (explore.hpp:38)
    uint32_t depth_cap = 0;  // the sweeps' depth cap: max_depth when a state can reach it
    int skipped = 0;
    std::vector<int> wg, ts;  // feasible configurations, largest-first (explore.cpp:64-72)
    std::vector<int64_t> cm_time, cm_steps;
    std::vector<int64_t> proto;  // protocol transitions: a terminal of time t is at depth proto + t
    std::vector<MachHost> hs;
    BfsResult bfs;
    std::vector<int64_t> first_time, first_steps;
    std::vector<Walk> walks;
    std::vector<int64_t> pre_applies, pre_depth;  // the capped DFS's prefix (lexrank_prefix)
    double ms_cost = 0, ms_bfs = 0, ms_first = 0, ms_prefix = 0;
};

int ensure_walk(Ctx& c, int k, int64_t T, const Walk** out) {
    for (const Walk& w : c.walks)
        if (w.k == k && w.T == T) {
            *out = &w;
            return MCTB_OK;
        }
    Walk w;
    w.k = k;
    w.T = T;
    std::vector<uint32_t> sib, sib_dep;
    int n_sib = 0;
    const Layout lay = bfs_layout(c.hs[k].d, 1);
    int rc = lexfirst_path(c.hs[k], T, 4 * c.cm_steps[k] + 4096, lay, &w.path, &w.final_time,
                           &w.applies, &sib, &n_sib, &sib_dep);
    if (rc) return rc;
    if (n_sib > 0) {
        std::vector<MachHost> one(1, c.hs[k]);
        BfsResult r;
        cudaStream_t st;
        MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        // the siblings' subtrees under the same depth cap as the DFS (each sibling
        // sits at its position on the path + 1)
        rc = run_bfs(one, c.cap + 64, c.cap, &r, st, false, &sib, 1, false, 1ull << 25,
                     c.depth_cap, &sib_dep);
        cudaStreamDestroy(st);
        if (rc) return rc;
        if (r.error) {
            set_error("model bug or capacity limit in the sibling exploration");
            return r.error == 3 ? MCTB_MODEL_BUG : MCTB_LIMIT;
        }
        const BfsStats& b = r.stats[0];
        w.sib_states = (int64_t)std::min<uint64_t>(b.states, c.cap);
        w.sib_capped = b.capped != 0;
        w.sib_transitions = (int64_t)b.transitions;
        // every sibling subtree state leads to a terminal: the deepest one is the
        // latest terminal reached, or the cap
        w.sib_depth = b.depth_cut ? c.max_depth
                      : b.terminals ? c.proto[k] + b.max_time : 0;
    }
    c.walks.push_back(std::move(w));
    *out = &c.walks.back();
    return MCTB_OK;
}

double now_ms() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e3 + t.tv_nsec * 1e-6;
}

// transitions_applied and max_depth_reached of configuration k's DFS when its
// visited set fills (explore.cpp:26-30), for graphs of fewer than 2^22 states;
// beyond, the sweep's edge count stands in
int ensure_prefix(Ctx& c, int k, int64_t* applies, int64_t* depth) {
    if (c.pre_applies.size() != c.wg.size()) {
        c.pre_applies.assign(c.wg.size(), -1);
        c.pre_depth.assign(c.wg.size(), -1);
    }
    if (c.pre_applies[k] < 0) {
        const double t0 = now_ms();
        int rc = dfs_prefix_stats(c.hs[k], c.max_depth, c.cap, c.cm_steps[k], &c.pre_applies[k],
                                  &c.pre_depth[k]);
        c.ms_prefix += now_ms() - t0;
        if (rc == MCTB_LIMIT) {
            c.pre_applies[k] = (int64_t)c.bfs.stats[k].transitions;
            c.pre_depth[k] = 0;
        } else if (rc) {
            return rc;
        }
    }
    *applies = c.pre_applies[k];
    *depth = c.pre_depth[k];
    return MCTB_OK;
}

struct VerdictOut {
    bool violated = false, exhaustive = false, trace_exact = true;
    int64_t states = 0, transitions = 0, max_depth = 0, explored = 0;
    int cfg = -1;  // index of the violating configuration
    int64_t final_time = -1, steps = 0;
    const std::vector<int32_t>* path = nullptr;  // guided-walk counterexample, if any
};


int prepare(Ctx& c, int64_t max_states, int64_t max_depth) {
    int rc = check_platform(c.plat);
    if (rc) return rc;
    if ((rc = check_problem(c.size, c.kernel))) return rc;
    if (max_depth < 1) {  // explore.cpp:91
        set_error("max_depth must be >= 1");
        return MCTB_CONFIG_ERROR;
    }
    c.max_depth = max_depth;
    if ((rc = require_device())) return rc;
    if (max_states > 0) c.cap = (uint64_t)max_states;
    int64_t sd[13];
    reference_space(c.plat, c.size, c.kernel, sd);
    SpaceDev s;
    if ((rc = make_space(sd, &s))) return rc;
    const int L = (int)sd[10];
    const uint64_t n = (uint64_t)L * L;
    cudaStream_t st;
    MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double t0 = now_ms();
    int64_t* d = nullptr;
    MCTB_CUDA(cudaMallocAsync(&d, 2 * n * sizeof(int64_t), st));
    rc = launch_space_eval(s, 0, n, d, d + n, st);
    std::vector<int64_t> h(2 * n);
    if (!rc)
        rc = cuda_check(cudaMemcpyAsync(h.data(), d, 2 * n * 8, cudaMemcpyDeviceToHost, st), "copy");
    cudaFreeAsync(d, st);
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
    if (rc) {
        cudaStreamDestroy(st);
        return rc;
    }
    c.ms_cost = now_ms() - t0;
    // space index i = (L - log wg) * L + (L - log ts): already largest-first
    for (uint64_t i = 0; i < n; ++i) {
        const int wg = 1 << (L - (int)(i / L)), ts = 1 << (L - (int)(i % L));
        if (h[i] < 0) {
            ++c.skipped;
            continue;
        }
        c.wg.push_back(wg);
        c.ts.push_back(ts);
        c.cm_time.push_back(h[i]);
        c.cm_steps.push_back(h[n + i]);
    }
    if (c.wg.empty()) {
        cudaStreamDestroy(st);
        set_error("no feasible configurations for this problem");
        return MCTB_CONFIG_ERROR;
    }
    const int nc = (int)c.wg.size();
    c.hs.resize(nc);
    c.proto.resize(nc);
    for (int k = 0; k < nc; ++k) {
        if ((rc = build_desc(c.plat, c.size, c.kernel, c.input, c.wg[k], c.ts[k], &c.hs[k]))) {
            cudaStreamDestroy(st);
            return rc;
        }
        // explore.cpp:124-127: the sweep tracks depths only when some state of some
        // configuration could lie deeper than max_depth
        c.proto[k] = c.cm_steps[k] - c.cm_time[k];
        if (depth_bound(c.hs[k].d, c.proto[k]) > (uint64_t)max_depth)
            c.depth_cap = (uint32_t)std::min<int64_t>(max_depth, 0x7fffffff);
    }
    // every interleaving of every configuration, one sweep.  The first DFS paths
    // (needed only for the configurations a probe finds violating) run lazily.
    const double t1 = now_ms();
    // first table from the cost model: the explored states ran at ~3x the lock-step
    // transitions summed over the configurations on the Table-1 platforms
    // (sizes 8-512); 4x that at load 1/4, clamped to [2^22, 2^29] slots.  Wider
    // spaces outgrow it and restart 16x larger.  (32x was measured: no restarts
    // on Table-1 spaces either, but a first sweep then maps a 4x larger fresh
    // buffer, ~28 ms per GB: size 256 1.40 -> 1.57 s.)
    uint64_t est = 0;
    for (int k = 0; k < nc; ++k) est += (uint64_t)std::max<int64_t>(c.cm_steps[k], 1);
    uint64_t first_cap = 1ull << 22;
    while (first_cap < 12 * est && first_cap < (1ull << 29)) first_cap <<= 1;
    rc = run_bfs(c.hs, c.cap * (uint64_t)nc + 64ull * nc, c.cap, &c.bfs, st, false, nullptr, 1,
                 false, first_cap, c.depth_cap);
    c.ms_bfs = now_ms() - t1;
    cudaStreamDestroy(st);
    if (rc) return rc;
    c.first_time.assign(nc, -1);
    c.first_steps.assign(nc, -1);
    if (c.bfs.error == 3) {
        set_error("model bug: deadlock or inapplicable transition during exploration");
        return MCTB_MODEL_BUG;
    }
    if (c.bfs.error) {
        set_error("GPU visited table capacity exceeded");
        return MCTB_LIMIT;
    }
    for (int k = 0; k < nc; ++k) {
        const BfsStats& b = c.bfs.stats[k];
        const bool complete = !b.capped && !b.depth_cut;
        if (complete && (b.terminals == 0 || b.min_time != c.cm_time[k])) {
            set_error("model bug: explored minimum differs from the lock-step model time");
            return MCTB_MODEL_BUG;
        }
    }
    return MCTB_OK;
}

// The first path of explore_machine's DFS for configuration k (GPU run, en[0] policy).
// Every run of a lock-step configuration (one device, or no device serving two
// batches) ends at the cost model's time after the same number of transitions
// (the reference's own test_machine.cpp checks seeded runs against it).
bool lockstep(const Ctx& c, int k) {
    const MachDesc& d = c.hs[k].d;
    return d.nwd == 1 || (int64_t)d.wgs <= (int64_t)c.plat[0] * c.plat[1];
}

int ensure_first(Ctx& c, int k) {
    if (c.first_time[k] >= 0) return MCTB_OK;
    if (lockstep(c, k)) {
        c.first_time[k] = c.cm_time[k];
        c.first_steps[k] = c.cm_steps[k];
        return MCTB_OK;
    }
    const BfsStats& b = c.bfs.stats[k];
    if (!b.capped && !b.depth_cut && b.terminals > 0 && b.min_time == b.max_time) {
        // every run of this configuration was explored and ends at one time, so
        // every run has the same length (protocol transitions + time): the first
        // path is known without stepping it
        c.first_time[k] = b.min_time;
        c.first_steps[k] = c.cm_steps[k] - c.cm_time[k] + b.min_time;
        return MCTB_OK;
    }
    const double t0 = now_ms();
    TrajOut o;
    int rc = gpu_run(c.hs[k], MCTB_POLICY_FIRST, 0, 0, 200000000LL, &o, nullptr, 0);
    c.ms_first += now_ms() - t0;
    if (rc) return rc;
    if (o.status != MCTB_OK) {
        set_error("model bug: deadlock on the first path");
        return MCTB_MODEL_BUG;
    }
    c.first_time[k] = o.time;
    c.first_steps[k] = o.steps;
    return MCTB_OK;
}

// The reference's verdict for bound T (explore.cpp:167-205) from the tables.
VerdictOut verdict(Ctx& c, int64_t T, int* rc_out) {
    VerdictOut v;
    const int nc = (int)c.wg.size();
    bool limit = false;
    for (int k = 0; k < nc; ++k) {
        const BfsStats& b = c.bfs.stats[k];
        v.explored += 1;
        const bool complete = !b.capped && !b.depth_cut;
        // the DFS meets only terminals within max_depth, i.e. of time <= max_depth -
        // protocol transitions (explore.cpp:124-127; every run of a configuration
        // has protocol + time transitions)
        const int64_t t_depth = c.max_depth - c.proto[k];
        const int64_t Tk = std::min(T, t_depth);
        // the sweep saw every terminal within the depth cap unless the visited cap cut it
        const int64_t tmin = !b.capped ? b.min_time
                             : c.cm_time[k] <= t_depth ? c.cm_time[k] : INT64_MAX;
        if (tmin <= Tk) {
            if ((*rc_out = ensure_first(c, k))) return v;
            // The DFS inserts the states it meets, in order, until the visited set
            // holds max_states (explore.cpp:28-31): it finds the terminal only if
            // every state before it in DFS order fits — the first path's, or the
            // guided walk's path with the abandoned siblings' subtrees before each
            // step.  Otherwise this configuration ends capped, with no verdict.
            bool found;
            if (c.first_time[k] <= Tk) {
                // DFS reaches a satisfying terminal on its first path
                found = (uint64_t)c.first_steps[k] + 1 <= c.cap;
                if (found) {
                    v.final_time = c.first_time[k];
                    v.steps = c.first_steps[k];
                    v.states += v.steps + 1;
                    v.transitions += v.steps;
                    v.max_depth = std::max(v.max_depth, v.steps);
                    v.path = nullptr;
                }
            } else {
                // schedule-dependent configuration: the DFS backtracks into later
                // branches; its first satisfying path comes from the guided walk and
                // its effort from the abandoned siblings' exploration
                const Walk* w = nullptr;
                if ((*rc_out = ensure_walk(c, k, Tk, &w))) return v;
                const int64_t steps = (int64_t)(w->path.size() / 4);
                found = !w->sib_capped && (uint64_t)(1 + steps + w->sib_states) <= c.cap;
                if (found) {
                    v.path = &w->path;
                    v.final_time = w->final_time;
                    v.steps = steps;
                    v.states += 1 + v.steps + w->sib_states;
                    v.transitions += w->applies + w->sib_transitions;
                    // the path and the abandoned siblings' subtrees
                    v.max_depth = std::max(v.max_depth, std::max(v.steps, w->sib_depth));
                }
            }
            if (found) {
                v.violated = true;
                v.cfg = k;
                v.exhaustive = false;
                return v;
            }
            // the visited set filled before the satisfying terminal: the reference
            // goes on to the next configuration with limit_hit
            int64_t pa = 0, pd = 0;
            if ((*rc_out = ensure_prefix(c, k, &pa, &pd))) return v;
            v.states += (int64_t)c.cap;
            v.transitions += pa;
            v.max_depth = std::max(v.max_depth, pd);
            limit = true;
            continue;
        }
        if (b.capped) {
            int64_t pa = 0, pd = 0;
            if ((*rc_out = ensure_prefix(c, k, &pa, &pd))) return v;
            v.states += (int64_t)c.cap;
            v.transitions += pa;
            v.max_depth = std::max(v.max_depth, pd);
            limit = true;
            continue;
        }
        v.states += (int64_t)std::min<uint64_t>(b.states, c.cap);
        v.transitions += (int64_t)b.transitions;
        if (complete)
            v.max_depth = std::max<int64_t>(v.max_depth, c.proto[k] + b.max_time);
        else
            limit = true;
        if (b.depth_cut && !b.capped) v.max_depth = std::max(v.max_depth, c.max_depth);
    }
    v.exhaustive = !limit;
    return v;
}

int emit_trace(Ctx& c, const VerdictOut& v, int32_t* trace, int64_t cap, int64_t* trace_len) {
    if (trace_len) *trace_len = v.steps;
    if (!trace || cap <= 0 || v.cfg < 0) return MCTB_OK;
    if (v.path) {
        const size_t n = std::min<size_t>(v.path->size(), (size_t)cap * 4);
        std::memcpy(trace, v.path->data(), n * sizeof(int32_t));
        return MCTB_OK;
    }
    TrajOut o;
    const int policy = v.trace_exact ? MCTB_POLICY_FIRST : MCTB_POLICY_TICK_LAST;
    int rc = gpu_run(c.hs[v.cfg], policy, 0, 0, 200000000LL, &o, trace, cap);
    if (rc) return rc;
    if (o.time != v.final_time || o.steps != v.steps) {
        set_error("model bug: counterexample run disagrees with the search tables");
        return MCTB_MODEL_BUG;
    }
    return MCTB_OK;
}

}  // namespace
}  // namespace mctb

using namespace mctb;

extern "C" {

// check_overtime (explore.hpp:88-93).
// out = {violated, exhaustive, states_visited, max_depth_reached, transitions_applied,
//        configs_explored, configs_skipped, final_time, wg, ts, steps, trace_exact}
int mctb_check_overtime(const int* plat, int size, int kernel, const int64_t* input, int64_t T,
                        int64_t max_states, int64_t max_depth, int64_t* out, int32_t* trace,
                        int64_t cap, int64_t* trace_len) {
    if (T < 0) {
        set_error("over-time bound must be >= 0");
        return MCTB_CONFIG_ERROR;
    }
    Ctx c;
    std::memcpy(c.plat, plat, sizeof c.plat);
    c.size = size;
    c.kernel = kernel;
    c.input = input;
    int rc = prepare(c, max_states, max_depth);
    if (rc) return rc;
    const VerdictOut v = verdict(c, T, &rc);
    if (rc) return rc;
    const int64_t o[12] = {v.violated, v.exhaustive, v.states, v.max_depth, v.transitions,
                           v.explored, c.skipped, v.final_time, v.cfg >= 0 ? c.wg[v.cfg] : 0,
                           v.cfg >= 0 ? c.ts[v.cfg] : 0, v.violated ? v.steps : 0, v.trace_exact};
    std::memcpy(out, o, sizeof o);
    if (!v.violated) {
        if (trace_len) *trace_len = 0;
        return MCTB_OK;
    }
    return emit_trace(c, v, trace, cap, trace_len);
}

// Per-bound verdicts of the last mctb_tune on this thread (mctb_tune_probes).
static thread_local std::vector<int64_t> g_probes;

static void record_probe(int64_t T, const VerdictOut& v, const Ctx& c) {
    const int64_t row[8] = {T, v.violated ? 1 : 0, v.exhaustive ? 1 : 0, v.states,
                            v.violated ? c.wg[v.cfg] : 0, v.violated ? c.ts[v.cfg] : 0,
                            v.violated ? v.final_time : -1, v.violated ? v.steps : -1};
    g_probes.insert(g_probes.end(), row, row + 8);
}

// estimate_initial_time + bisect_min_time: the `tune` flow (tools/main.cpp:119-128).
// t_hi <= 0 selects estimate_initial_time(seed).
// out = {t_min, wg, ts, t_ini, proven, checks_run, states_visited_total, first_trail_time,
//        steps, trace_exact}
// info = {ms_cost_model, ms_first_paths, ms_bfs, bfs_states, bfs_levels}  (optional)
int mctb_tune(const int* plat, int size, int kernel, const int64_t* input, int64_t t_hi,
              uint64_t seed, int64_t max_states, int64_t max_depth, int64_t* out, int32_t* trace,
              int64_t cap, int64_t* trace_len, double* info) {
    Ctx c;
    std::memcpy(c.plat, plat, sizeof c.plat);
    c.size = size;
    c.kernel = kernel;
    c.input = input;
    const bool tt = getenv("MCTB_TUNE_TRACE") != nullptr;
    const double tp0 = now_ms();
    int rc = prepare(c, max_states, max_depth);
    if (rc) return rc;
    const double tp1 = now_ms();
    if (t_hi <= 0) {
        // estimate_initial_time (search.cpp:94-102): mt19937_64(seed) picks a feasible
        // configuration in enumerate_configs order; its SeededRandom run is T_ini.
        std::vector<int> order(c.wg.size());
        for (size_t k = 0; k < order.size(); ++k) order[k] = (int)k;
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            return c.wg[a] != c.wg[b] ? c.wg[a] < c.wg[b] : c.ts[a] < c.ts[b];
        });
        Mt64 rng;
        rng.seed(seed);
        const int k = order[rng.next() % order.size()];
        const BfsStats& b = c.bfs.stats[k];
        if (!b.capped && !b.depth_cut && b.terminals > 0 && b.min_time == b.max_time) {
            // the sweep explored every run of this configuration and they all end at
            // one time, so the seeded run ends there too: no serial simulation
            // (a lone GPU thread steps ~2 us per transition; 124 ms at size 128)
            t_hi = b.min_time;
        } else if (lockstep(c, k)) {
            t_hi = c.cm_time[k];  // every run ends at the lock-step time
        } else {
            TrajOut o;
            if ((rc = gpu_run(c.hs[k], MCTB_POLICY_MT19937, seed, 0, 200000000LL, &o, nullptr, 0)))
                return rc;
            if (o.status != MCTB_OK) {
                set_error("model bug: deadlock in the initial-time simulation");
                return MCTB_MODEL_BUG;
            }
            t_hi = o.time;
        }
    }
    if (t_hi < 1) {
        set_error("t_hi must be >= 1");
        return MCTB_CONFIG_ERROR;
    }
    const double tp2 = now_ms();
    // search.cpp:104-158
    g_probes.clear();
    int checks = 0;
    int64_t states_total = 0;
    bool proven = true;
    VerdictOut v = verdict(c, t_hi, &rc);
    if (rc) return rc;
    record_probe(t_hi, v, c);
    ++checks;
    states_total += v.states;
    if (!v.violated) {
        set_error("t_hi too small: no run terminates within " + std::to_string(t_hi));
        return MCTB_CONFIG_ERROR;
    }
    const int64_t first_trail = v.final_time;
    VerdictOut best = v;
    int64_t lo = 0, hi = t_hi;
    bool lo_checked = false;
    while (hi - lo > 1) {
        const int64_t mid = lo + (hi - lo) / 2;
        const VerdictOut vm = verdict(c, mid, &rc);
        if (rc) return rc;
        record_probe(mid, vm, c);
        ++checks;
        states_total += vm.states;
        if (vm.violated) {
            hi = mid;
            best = vm;
        } else {
            if (!vm.exhaustive) proven = false;
            lo = mid;
            lo_checked = true;
        }
    }
    if (!lo_checked && lo == 0 && hi == 1) {
        const VerdictOut vz = verdict(c, 0, &rc);
        if (rc) return rc;
        record_probe(0, vz, c);
        ++checks;
        if (vz.violated) {
            set_error("a run finished in zero ticks");
            return MCTB_MODEL_BUG;
        }
        if (!vz.exhaustive) proven = false;
    }
    if (best.final_time != hi) {
        set_error("bisection trace time disagrees with t_min");
        return MCTB_MODEL_BUG;
    }
    const int64_t o[10] = {hi, c.wg[best.cfg], c.ts[best.cfg], t_hi, proven, checks,
                           states_total, first_trail, best.steps, best.trace_exact};
    std::memcpy(out, o, sizeof o);
    if (info) {
        info[0] = c.ms_cost;
        info[1] = c.ms_first;
        info[2] = c.ms_bfs;
        info[3] = (double)c.bfs.states;
        info[4] = c.bfs.ms;  // exploration kernel time (CUDA events)
    }
    const double tp3 = now_ms();
    rc = emit_trace(c, best, trace, cap, trace_len);
    if (tt)
        fprintf(stderr, "[tune] prepare %.2f (cost %.2f, bfs %.2f) estimate %.2f bisect %.2f (first %.2f, capped prefixes %.2f) trace %.2f ms\n",
                tp1 - tp0, c.ms_cost, c.ms_bfs, tp2 - tp1, tp3 - tp2, c.ms_first, c.ms_prefix,
                now_ms() - tp3);
    return rc;
}

int64_t mctb_tune_probes(int64_t* rows, int64_t cap) {
    const int64_t n = (int64_t)(g_probes.size() / 8);
    if (rows)
        for (int64_t i = 0; i < std::min(n, cap); ++i)
            std::memcpy(rows + 8 * i, g_probes.data() + 8 * i, 8 * sizeof(int64_t));
    return n;
}

}  // extern "C"
