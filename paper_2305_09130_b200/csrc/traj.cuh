// Host-side interface of the trajectory kernels (traj.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "cost_model.cuh"
#include "machine.cuh"

namespace mctb {

struct TrajOut {
    int64_t time, steps;
    int32_t glob0, status;
    uint64_t hash;  // FNV-1a 64 over the transitions' int32 words {actor, peer, op, arg}
    int32_t config, pad;
};

// A machine description plus the host copy of the minimum kernel's value table.
struct MachHost {
    MachDesc d;
    std::vector<int64_t> values;  // sorted distinct input values + INT64_MAX
    std::vector<int32_t> ids;     // value id of input[i]
    int64_t value(int32_t id) const { return values.empty() ? 0 : values[(size_t)id]; }
};

int build_desc(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
               MachHost* out);
int upload_desc(MachHost& h, cudaStream_t stream, int32_t** d_ids);
int launch_trajectories(const MachDesc* d_descs, int n_desc, int policy, uint64_t seed,
                        uint64_t traj0, uint64_t n_traj, int64_t max_steps, TrajOut* d_out,
                        int32_t* d_trace, int64_t trace_cap, cudaStream_t stream);
int launch_replay(const MachDesc& m, const int32_t* d_trace, int64_t len, int64_t* d_step_time,
                  TrajOut* d_out, cudaStream_t stream);

}  // namespace mctb
