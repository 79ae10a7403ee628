// Host-side interface of the GPU interleaving exploration (bfs.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "pack.cuh"
#include "traj.cuh"

namespace mctb {

struct BfsStats {
    unsigned long long states, transitions, terminals;
    long long min_time, max_time;
    unsigned long long deadlocks;
    unsigned long long capped;   // the per-configuration state cap was reached
    unsigned long long generic;  // successors built by the generic unpacked apply()
    unsigned long long violations;  // states breaking Machine::check_invariants
    unsigned long long depth_cut;   // a non-terminal state at the depth cap (explore.cpp:124-127)
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
// (ExploreLimits::max_states, explore.hpp:36-42).
// seeds (optional): packed states of configuration 0 (layout bfs_layout(hs[0].d, 1))
// to start from instead of the initial states — a multi-source exploration.
// first_cap (0 = sized for max_states) bounds the first table; it grows 16x
// (restarting the sweep) on overflow.
// n_parts > 1 splits the visited set into hash partitions on this device (the
// multi-GPU exchange path, exercised on one GPU); sys_scope selects the
// system-scope memory operations of the multi-GPU kernel.
// depth_cap > 0 applies ExploreLimits::max_depth (explore.cpp:124-127): a state at
// depth >= depth_cap is visited but not expanded (depth_cut is set when it has
// enabled transitions).  The state graphs are graded — every path from the
// initial state to a state has the same length (tests/test_oracle.py) — so the
// depth-limited DFS visits exactly the states of depth <= max_depth and the cap
// is order-independent.  seed_depths gives the depth of each seed (0 when NULL).
int run_bfs(std::vector<MachHost>& hs, uint64_t max_states, uint64_t cfg_cap, BfsResult* res,
            cudaStream_t st, bool check_invariants = false,
            const std::vector<uint32_t>* seeds = nullptr, int n_parts = 1,
            bool sys_scope = false, uint64_t first_cap = 0, uint32_t depth_cap = 0,
            const std::vector<uint32_t>* seed_depths = nullptr);

// Upper bound on the depth of any state of a configuration (protocol transitions
// + the largest model time the packing admits): a sweep whose configurations
// stay below max_depth needs no depth tracking.
uint64_t depth_bound(const MachDesc& m, int64_t protocol_steps);

// The packed layout the exploration uses for a configuration among n_cfg.
Layout bfs_layout(const MachDesc& m, int n_cfg);

// The reference DFS's transitions_applied and max_depth_reached when its visited
// set fills at cap states: lexrank_prefix (lexrank.cu) ranks the graph of
// graph_states states; dfs_prefix_stats (bfs.cu) first sizes the graph with a
// sweep and returns MCTB_LIMIT (nothing ranked) when it holds 2^22 states or
// more, spans 16,384 levels or more (run_len: the lock-step run's transitions),
// or the cap is itself 2^22 or more.
int lexrank_prefix(MachHost& h, int64_t max_depth, uint64_t cap, uint64_t graph_states,
                   int64_t* applies, int64_t* max_depth_reached);
int dfs_prefix_stats(MachHost& h, int64_t max_depth, uint64_t cap, int64_t run_len,
                     int64_t* applies, int64_t* max_depth_reached);

// The reference DFS's counterexample for bound T (lexfirst.cu).
// sibling_depths (optional): the depth of each abandoned sibling (its position on
// the path + 1).
int lexfirst_path(MachHost& h, int64_t T, int64_t max_len, const Layout& layout,
                  std::vector<int32_t>* path, int64_t* final_time, int64_t* sibling_applies,
                  std::vector<uint32_t>* siblings, int* n_siblings,
                  std::vector<uint32_t>* sibling_depths = nullptr);

}  // namespace mctb
