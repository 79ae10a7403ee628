// Swarm search on the GPU (north-star subsystem 2): swarm_min_time
// (search.cpp:160-210) re-designed around counter-based trajectories.
//
// The reference runs `workers` threads of randomised bitstate DFS per round
// under a wall-clock budget.  Here a round is one launch of n trajectories
// (Philox4x32-10 schedules, one GPU thread each) spread over every feasible
// configuration; trajectory ids continue across rounds, so every trajectory
// of the search is replayable on its own (oracle mo_simulate, policy PHILOX).
// The stop rule is the reference's: round 0 collects terminating runs; each
// further round keeps only runs strictly below the best time so far and the
// search stops when a round finds none (or no smaller time).  Ties prefer the
// largest wg, then the largest ts (pick_preferred, search.cpp:67-78).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "traj.cuh"

namespace mctb {

int check_platform(const int* plat);
int check_problem(int size, int kernel);
int gpu_run(MachHost& h, int policy, uint64_t seed, uint64_t traj, int64_t max_steps,
            TrajOut* out, int32_t* trace, int64_t cap);

}  // namespace mctb

using namespace mctb;

extern "C" {

// out = {t_min, wg, ts, t_ini, rounds(checks_run), transitions_total, first_trail_time,
//        steps, best_trajectory_id, trajectories_run}
// trails (optional) = int64[4 * trails_cap]: {time, wg, ts, steps} of every trajectory of the
// first round (the trail table of `tune-swarm`), *n_trails its count.
int mctb_swarm(const int* plat, int size, int kernel, const int64_t* input, int64_t per_round,
               int max_rounds, uint64_t seed, int64_t max_steps, int64_t* out, int32_t* trace,
               int64_t cap, int64_t* trace_len, int64_t* trails, int64_t trails_cap,
               int64_t* n_trails) {
    int rc = check_platform(plat);
    if (rc) return rc;
    if ((rc = check_problem(size, kernel))) return rc;
    if (per_round < 1) {
        set_error("swarm needs at least one worker");
        return MCTB_CONFIG_ERROR;
    }
    if ((rc = require_device())) return rc;
    if (max_steps <= 0) max_steps = 4000000;  // ExploreLimits::max_depth (explore.hpp:37)
    // feasible configurations, enumerate_configs order (model.cpp:96-98)
    int n = 0;
    while ((1 << n) < size) ++n;
    std::vector<MachHost> hs;
    for (int i = 1; i <= n - 1; ++i)
        for (int j = 1; j <= n - 1; ++j) {
            const int wg = 1 << i, ts = 1 << j;
            if (kernel == 1 && (long long)wg * ts > size) continue;
            hs.emplace_back();
            if ((rc = build_desc(plat, size, kernel, input, wg, ts, &hs.back()))) return rc;
        }
    if (hs.empty()) {
        set_error("no feasible configurations for this problem");
        return MCTB_CONFIG_ERROR;
    }
    const int nc = (int)hs.size();
    cudaStream_t st;
    MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int32_t* d_ids = nullptr;
    if ((rc = upload_desc(hs[0], st, &d_ids))) return rc;
    std::vector<MachDesc> descs(nc);
    for (int k = 0; k < nc; ++k) {
        hs[k].d.input_id = d_ids;
        descs[k] = hs[k].d;
    }
    MachDesc* d_desc = nullptr;
    TrajOut* d_out = nullptr;
    MCTB_CUDA(cudaMallocAsync(&d_desc, nc * sizeof(MachDesc), st));
    MCTB_CUDA(cudaMallocAsync(&d_out, per_round * sizeof(TrajOut), st));
    MCTB_CUDA(cudaMemcpyAsync(d_desc, descs.data(), nc * sizeof(MachDesc), cudaMemcpyHostToDevice, st));
    std::vector<TrajOut> h(per_round);
    int64_t best_time = -1, first_trail = -1, transitions = 0, trajectories = 0, t_ini = -1;
    int best_cfg = -1, rounds = 0;
    uint64_t best_traj = 0, traj0 = 0;
    int64_t best_steps = 0;
    if (n_trails) *n_trails = 0;
    for (int round = 0; round < std::max(1, max_rounds); ++round) {
        rc = launch_trajectories(d_desc, nc, MCTB_POLICY_PHILOX, seed, traj0, per_round, max_steps,
                                 d_out, nullptr, 0, st);
        if (!rc)
            rc = cuda_check(cudaMemcpyAsync(h.data(), d_out, per_round * sizeof(TrajOut),
                                            cudaMemcpyDeviceToHost, st), "copy");
        if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "sync");
        if (rc) break;
        ++rounds;
        trajectories += per_round;
        const int64_t target = round == 0 ? INT64_MAX : best_time - 1;
        int64_t round_best = -1;
        int round_cfg = -1;
        uint64_t round_traj = 0;
        int64_t round_steps = 0;
        for (int64_t i = 0; i < per_round; ++i) {
            const TrajOut& o = h[i];
            transitions += o.steps;
            if (o.status != MCTB_OK) continue;  // depth limit (explore.cpp:124-127)
            if (round == 0 && n_trails && trails && *n_trails < trails_cap) {
                int64_t* r = trails + 4 * (*n_trails);
                r[0] = o.time;
                r[1] = hs[o.config].d.wg;
                r[2] = hs[o.config].d.ts;
                r[3] = o.steps;
                ++*n_trails;
            }
            if (round == 0 && first_trail < 0) first_trail = o.time;
            if (o.time > target) continue;
            const int wg = hs[o.config].d.wg, ts = hs[o.config].d.ts;
            const bool better =
                round_best < 0 || o.time < round_best ||
                (o.time == round_best && (wg > hs[round_cfg].d.wg ||
                                          (wg == hs[round_cfg].d.wg && ts > hs[round_cfg].d.ts)));
            if (better) {
                round_best = o.time;
                round_cfg = o.config;
                round_traj = traj0 + (uint64_t)i;
                round_steps = o.steps;
            }
        }
        traj0 += (uint64_t)per_round;
        if (round == 0) {
            if (round_best < 0) {
                rc = MCTB_CONFIG_ERROR;
                set_error("model never terminated within the swarm limits");
                break;
            }
        } else if (round_best < 0 || round_best >= best_time) {
            break;  // nothing below the best time: the reference's stop rule
        }
        best_time = round_best;
        if (round == 0) t_ini = round_best;
        best_cfg = round_cfg;
        best_traj = round_traj;
        best_steps = round_steps;
        if (best_time <= 1) break;
    }
    cudaFreeAsync(d_desc, st);
    cudaFreeAsync(d_out, st);
    cudaFreeAsync(d_ids, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (rc) return rc;
    const int64_t o[10] = {best_time, hs[best_cfg].d.wg, hs[best_cfg].d.ts, t_ini, rounds,
                           transitions, first_trail, best_steps, (int64_t)best_traj, trajectories};
    std::memcpy(out, o, sizeof o);
    if (trace_len) *trace_len = best_steps;
    if (trace && cap > 0) {
        TrajOut r;
        if ((rc = gpu_run(hs[best_cfg], MCTB_POLICY_PHILOX, seed, best_traj, max_steps, &r, trace,
                          cap)))
            return rc;
        if (r.time != best_time || r.steps != best_steps) {
            set_error("model bug: swarm trajectory does not reproduce");
            return MCTB_MODEL_BUG;
        }
    }
    return MCTB_OK;
}

}  // extern "C"
