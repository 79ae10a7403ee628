// Lock-step cost model of the mctune transition system.
//
// The reference computes a configuration's model time by running or
// exhaustively exploring the transition system (machine.cpp:788-825,
// explore.cpp:86-165).  Every interleaving of one configuration advances the
// clock only when all obligated elements reported (machine.cpp:209-210), so
// elements of every unit and device move in lock step and a workgroup batch
// takes a fixed number of ticks D:
//   abstract : D = rounds * A,  A = (size/ts)*(gmt*ts + ts) + gmt   (kernel.cpp:33-43)
//   minimum  : D = rounds * ts * gmt + (nwe - 1) + gmt             (kernel.cpp:67-80)
// with rounds = wg / nwe (machine.cpp:70).  The host serves device_rounds =
// max(wgs / nwu, 1) batches (machine.cpp:71-73) over nwd devices that are
// re-armed at zero model time, giving
//   time = ceil(device_rounds / nwd) * D,
// the minimum over all interleavings (what check_overtime/bisect_min_time
// decide) and the Machine::run(RoundRobin) time (what exhaustive_sweep
// reports).  The transition count adds the fixed per-process protocol
// handshakes to `time` ticks.  Pinned against the reference over every
// configuration of sizes 4..64 on 96 platforms in tests/test_cost_model.py.
#pragma once

#include <stdint.h>

namespace mctb {

struct SpaceDev {
    int32_t kernel, logn, gmt;
    int32_t nd_lo, nd_hi, nu_lo, nu_hi;
    int32_t lognp_lo, lognp_hi, logwg_lo, logwg_hi, logts_lo, logts_hi;
    // radices (digit counts) of the mixed-radix index, least significant first
    uint32_t n_nd, n_nu, n_np, n_ts, n_wg;
};

struct Config {
    int32_t nd, nu, lognp, logwg, logts;
};

struct Cost {
    int64_t time, steps;
    int32_t wgs, nwd, nwu, nwe;
    bool feasible;
};

// derive_launch, model.cpp:72-88 (powers of two as logs)
__host__ __device__ inline void launch_plan(int logn, int nd, int nu, int lognp, int logwg,
                                            int logts, int& wgs, int& nwd, int& nwu, int& nwe) {
    const int s = logwg + logts;
    wgs = s < logn ? (1 << (logn - s)) : 1;  // size/(wg*ts), clamped to >= 1
    const int q = wgs / nu;
    nwd = ((long long)wgs <= (long long)nu * nd) ? q : nd;
    if (q == 0) nwd = 1;
    nwu = wgs <= nu ? wgs : nu;
    nwe = 1 << (logwg < lognp ? logwg : lognp);
}

__host__ __device__ inline Cost lockstep_cost(int kernel, int logn, int gmt, const Config& c) {
    Cost r;
    launch_plan(logn, c.nd, c.nu, c.lognp, c.logwg, c.logts, r.wgs, r.nwd, r.nwu, r.nwe);
    const int64_t size = 1ll << logn, wg = 1ll << c.logwg, ts = 1ll << c.logts;
    r.feasible = !(kernel == 1 && c.logwg + c.logts > logn);  // kernel.cpp:84-87
    if (!r.feasible) {
        r.time = r.steps = -1;
        return r;
    }
    const int64_t rounds = wg / r.nwe;
    int64_t dr = r.wgs / r.nwu;
    if (dr < 1) dr = 1;
    const int64_t reacts = dr - r.nwd;
    const int64_t waves = (dr + r.nwd - 1) / r.nwd;
    const int64_t groups = dr * r.nwu;
    const int64_t items = groups * wg;
    const int64_t reps = size / ts;
    int64_t D, busy, arrivals, releases, item_done, end_done, effects;
    if (kernel == 0) {
        const int64_t A = reps * (gmt * ts + ts) + gmt;
        D = rounds * A;
        busy = items * A;
        arrivals = items * 2 * reps;
        releases = groups * rounds * 2 * reps;
        item_done = items;
        end_done = 0;
        effects = 0;
    } else {
        const int64_t epi = (r.nwe - 1) + gmt;
        D = rounds * ts * gmt + epi;
        busy = items * ts * gmt + groups * epi;
        arrivals = groups * r.nwe;
        releases = groups;
        item_done = groups * (rounds - 1) * r.nwe;
        end_done = groups * r.nwe;
        effects = items * ts + groups * r.nwe;
    }
    r.time = waves * D;
    const int64_t host = 2 * r.nwd + reacts + 1;                         // go, react, stop, fin
    const int64_t clock = r.time + 1;                                    // ticks + halt
    const int64_t dev = dr * (r.nwu + 1) + (int64_t)r.nwd * r.nwu;       // unit go, done, stop
    const int64_t unit = groups * (wg + 1) + (int64_t)r.nwd * r.nwu * (r.nwe + 1);
    r.steps = host + clock + dev + unit + busy + arrivals + releases + item_done + end_done +
              effects;
    return r;
}

// Mixed-radix decode (index order documented in include/mctune_b200.h).
__host__ __device__ inline Config decode(const SpaceDev& sd, uint64_t index) {
    Config c;
    const uint64_t a = index / sd.n_nd;
    c.nd = sd.nd_lo + (int)(index - a * sd.n_nd);
    const uint64_t b = a / sd.n_nu;
    c.nu = sd.nu_lo + (int)(a - b * sd.n_nu);
    const uint64_t d = b / sd.n_np;
    c.lognp = sd.lognp_lo + (int)(b - d * sd.n_np);
    const uint64_t e = d / sd.n_ts;
    c.logts = sd.logts_hi - (int)(d - e * sd.n_ts);
    c.logwg = sd.logwg_hi - (int)e;
    return c;
}

}  // namespace mctb
