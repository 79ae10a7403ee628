// Host-side interface of the trajectory kernels (traj.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "cost_model.cuh"
#include "machine.cuh"

namespace mctb {

// std::mt19937_64 (only for the reference's SeededRandom policy)
struct Mt64 {
    uint64_t mt[312];
    int idx;
    __host__ __device__ void seed(uint64_t s) {
        mt[0] = s;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
        idx = 312;
    }
    __host__ __device__ uint64_t next() {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ull) | (mt[(i + 1) % 312] & 0x7FFFFFFFull);
                uint64_t xa = x >> 1;
                if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        return y;
    }
};


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
int launch_traj_records(const TrajOut* d_in, uint64_t n, int kernel, int64_t* d_rec,
                        cudaStream_t stream);
int launch_replay(const MachDesc& m, const int32_t* d_trace, int64_t len, int64_t* d_step_time,
                  TrajOut* d_out, cudaStream_t stream);

}  // namespace mctb
