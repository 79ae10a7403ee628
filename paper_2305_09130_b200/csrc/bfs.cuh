// Host-side interface of the GPU interleaving exploration (bfs.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "traj.cuh"

namespace mctb {

struct BfsStats {
    unsigned long long states, transitions, terminals;
    long long min_time, max_time;
    unsigned long long deadlocks;
    unsigned long long capped;   // the per-configuration state cap was reached
    unsigned long long generic;  // successors built by the generic unpacked apply()
    unsigned long long violations;  // states breaking Machine::check_invariants
};

struct BfsResult {
    std::vector<BfsStats> stats;
    uint64_t levels = 0, states = 0, capacity = 0;
    int error = 0;
    double ms = 0;
    int words = 0;
};

// Explores every configuration in `hs` in one sweep.  max_states bounds the
// whole table; cfg_cap is the per-configuration visited cap of the reference
// (ExploreLimits::max_states, explore.hpp:227-233).
int run_bfs(std::vector<MachHost>& hs, uint64_t max_states, uint64_t cfg_cap, BfsResult* res,
            cudaStream_t st, bool check_invariants = false);

}  // namespace mctb
