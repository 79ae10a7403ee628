// C ABI of mctune_b200 (include/mctune_b200.h): argument validation with the
// reference's error classes, host<->device staging, and the host-side parts
// of the reference drivers (row sorting, bisection bookkeeping).  All model
// time is computed on the GPU.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "cost_model.cuh"

namespace mctb {

int make_space(const int64_t* sd, SpaceDev* out);
uint64_t space_count(const SpaceDev& s);
int launch_space_argmin(const SpaceDev& s, uint64_t first, uint64_t count, uint64_t* d_key,
                        cudaStream_t stream);
int launch_space_eval(const SpaceDev& s, uint64_t first, uint64_t count, int64_t* d_time,
                      int64_t* d_steps, cudaStream_t stream);
int launch_space_point(const SpaceDev& s, const uint64_t* d_key, int64_t* d_out,
                       cudaStream_t stream);
int launch_fill_key(uint64_t* d_key, cudaStream_t stream);
int launch_space_exact(const SpaceDev& s, uint64_t first, uint64_t count, uint64_t* d_time,
                       uint64_t* d_index, cudaStream_t stream);

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& what) { g_error = what; }

int cuda_check(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return MCTB_OK;
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return MCTB_CUDA_ERROR;
}

int require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_error("no CUDA device: mctune_b200 has no CPU path");
        return MCTB_NO_DEVICE;
    }
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) {
        set_error("mctune_b200 is built for sm_100a (B200) only");
        return MCTB_NO_DEVICE;
    }
    // keep freed stream-ordered allocations (visited tables, queues) in the pool
    // instead of returning them to the driver at every synchronisation
    static bool pool_set[64] = {};
    if (!pool_set[dev & 63]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
        pool_set[dev & 63] = true;
    }
    return MCTB_OK;
}

// Per-device scratch: a few pinned/device words reused by the host-buffer calls.
struct Scratch {
    uint64_t* d_key = nullptr;
    uint64_t* d_exact = nullptr;  // {time, index} of the exact resolution
    int64_t* d_out = nullptr;
    uint64_t* h_key = nullptr;
    int64_t* h_out = nullptr;
    cudaStream_t stream = nullptr;
};

int scratch(Scratch** out) {
    static std::mutex mu;
    static Scratch per_dev[64];
    int dev = 0;
    MCTB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    Scratch& s = per_dev[dev & 63];
    if (!s.d_key) {
        // [key, out[0..15]] contiguous on both sides: one copy brings the result back
        MCTB_CUDA(cudaMalloc(&s.d_key, 17 * sizeof(uint64_t)));
        s.d_out = reinterpret_cast<int64_t*>(s.d_key + 1);
        MCTB_CUDA(cudaMalloc(&s.d_exact, 2 * sizeof(uint64_t)));
        MCTB_CUDA(cudaMallocHost(&s.h_key, 17 * sizeof(uint64_t)));
        s.h_out = reinterpret_cast<int64_t*>(s.h_key + 1);
        MCTB_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    }
    *out = &s;
    return MCTB_OK;
}

bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }
int log2i(long long v) {
    int n = 0;
    while ((1ll << n) < v) ++n;
    return n;
}

// PlatformConfig::validate (model.cpp:12-17)
int check_platform(const int* plat) {
    if (plat[0] < 1 || plat[1] < 1 || plat[2] < 1 || plat[3] < 1) {
        set_error("platform constants nd, nu, np, gmt must all be >= 1");
        return MCTB_CONFIG_ERROR;
    }
    if (!is_pow2(plat[2])) {
        set_error("np must be a power of two, got " + std::to_string(plat[2]));
        return MCTB_CONFIG_ERROR;
    }
    return MCTB_OK;
}

// ProblemSpec::validate (model.cpp:51-60)
int check_problem(int size, int kernel) {
    if (size < 4 || !is_pow2(size)) {
        set_error("size must be a power of two >= 4, got " + std::to_string(size));
        return MCTB_CONFIG_ERROR;
    }
    if (kernel != 0 && kernel != 1) {
        set_error("unknown kernel kind (expected abstract or minimum)");
        return MCTB_CONFIG_ERROR;
    }
    return MCTB_OK;
}

// The reference's own tuning space for one (platform, problem):
// enumerate_configs (model.cpp:90-100) as a space descriptor.
void reference_space(const int* plat, int size, int kernel, int64_t* sd) {
    const int n = log2i(size);
    const int64_t v[13] = {kernel, size, plat[3], plat[0], plat[0], plat[1], plat[1],
                           log2i(plat[2]), log2i(plat[2]), 1, n - 1, 1, n - 1};
    std::memcpy(sd, v, sizeof v);
}

}  // namespace mctb

using namespace mctb;

extern "C" {

const char* mctb_last_error(void) { return g_error.c_str(); }

int mctb_version(void) { return 1; }

int mctb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int count = 0;
    for (int d = 0; d < n; ++d) {
        int major = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
        count += major == 10;
    }
    return count;
}

int mctb_derive_launch(const int* plat, int size, int wg, int ts, int* out) {
    int rc = check_platform(plat);
    if (rc) return rc;
    if (size < 4 || !is_pow2(size)) {
        set_error("size must be a power of two >= 4");
        return MCTB_CONFIG_ERROR;
    }
    const int hi = size / 2;
    if (!is_pow2(wg) || wg < 2 || wg > hi) {
        set_error("wg must be a power of two in [2, size/2], got " + std::to_string(wg));
        return MCTB_CONFIG_ERROR;
    }
    if (!is_pow2(ts) || ts < 2 || ts > hi) {
        set_error("ts must be a power of two in [2, size/2], got " + std::to_string(ts));
        return MCTB_CONFIG_ERROR;
    }
    launch_plan(log2i(size), plat[0], plat[1], log2i(plat[2]), log2i(wg), log2i(ts), out[0],
                out[1], out[2], out[3]);
    out[4] = out[3] * out[2] * out[1];
    return MCTB_OK;
}

uint64_t mctb_space_count(const int64_t* sd) {
    SpaceDev s;
    if (make_space(sd, &s)) return 0;
    return space_count(s);
}

int mctb_space_argmin_async(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* d_key,
                            void* stream) {
    SpaceDev s;
    int rc = make_space(sd, &s);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    return launch_space_argmin(s, first, count, d_key, static_cast<cudaStream_t>(stream));
}

int mctb_space_argmin(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* key,
                      int64_t* out) {
    SpaceDev s;
    int rc = make_space(sd, &s);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    Scratch* sc;
    if ((rc = scratch(&sc))) return rc;
    if ((rc = launch_fill_key(sc->d_key, sc->stream))) return rc;
    if ((rc = launch_space_argmin(s, first, count, sc->d_key, sc->stream))) return rc;
    if ((rc = launch_space_point(s, sc->d_key, sc->d_out, sc->stream))) return rc;
    MCTB_CUDA(cudaMemcpyAsync(sc->h_key, sc->d_key, 9 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                              sc->stream));
    MCTB_CUDA(cudaStreamSynchronize(sc->stream));
    *key = *sc->h_key;
    std::memcpy(out, sc->h_out, 8 * sizeof(int64_t));
    if (*key != kKeyNone && (*key >> MCTB_KEY_INDEX_BITS) == kKeySat) {
        // saturated time field: every configuration of the range has time >= 2^30 - 1
        // (or is infeasible), so the key's index is not the winner — resolve exactly
        if ((rc = launch_space_exact(s, first, count, sc->d_exact, sc->d_exact + 1, sc->stream)))
            return rc;
        uint64_t ex[2];
        MCTB_CUDA(cudaMemcpyAsync(ex, sc->d_exact, sizeof ex, cudaMemcpyDeviceToHost, sc->stream));
        MCTB_CUDA(cudaStreamSynchronize(sc->stream));
        if (ex[0] == UINT64_MAX) {
            *key = kKeyNone;
        } else {
            *key = ((uint64_t)kKeySat << MCTB_KEY_INDEX_BITS) | ex[1];
            MCTB_CUDA(cudaMemcpyAsync(sc->d_key, key, sizeof(uint64_t), cudaMemcpyHostToDevice,
                                      sc->stream));
            if ((rc = launch_space_point(s, sc->d_key, sc->d_out, sc->stream))) return rc;
            MCTB_CUDA(cudaMemcpyAsync(sc->h_out, sc->d_out, 8 * sizeof(int64_t),
                                      cudaMemcpyDeviceToHost, sc->stream));
            MCTB_CUDA(cudaStreamSynchronize(sc->stream));
            std::memcpy(out, sc->h_out, 8 * sizeof(int64_t));
        }
    }
    if (*key == kKeyNone || out[0] < 0) {
        set_error("tuning space range holds no configuration");
        return MCTB_CONFIG_ERROR;
    }
    return MCTB_OK;
}

int mctb_space_exact_async(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* d_time,
                           uint64_t* d_index, void* stream) {
    SpaceDev s;
    int rc = make_space(sd, &s);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    return launch_space_exact(s, first, count, d_time, d_index, static_cast<cudaStream_t>(stream));
}

int mctb_space_eval_async(const int64_t* sd, uint64_t first, uint64_t count, int64_t* d_time,
                          int64_t* d_steps, void* stream) {
    SpaceDev s;
    int rc = make_space(sd, &s);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    return launch_space_eval(s, first, count, d_time, d_steps, static_cast<cudaStream_t>(stream));
}

// exhaustive_sweep (search.cpp:212-244): every enumerated configuration,
// infeasible ones flagged, stable-sorted by (ok first, time, transitions).
int mctb_sweep(const int* plat, int size, int kernel, const int64_t* input, int64_t* rows,
               int64_t cap, int64_t* n_rows) {
    (void)input;  // model time and transition count do not depend on the data
    int rc = check_platform(plat);
    if (rc) return rc;
    if ((rc = check_problem(size, kernel))) return rc;
    if ((rc = require_device())) return rc;
    int64_t sd[13];
    reference_space(plat, size, kernel, sd);
    SpaceDev s;
    if ((rc = make_space(sd, &s))) return rc;
    const uint64_t n = space_count(s);
    Scratch* sc;
    if ((rc = scratch(&sc))) return rc;
    int64_t* d = nullptr;
    MCTB_CUDA(cudaMallocAsync(&d, 2 * n * sizeof(int64_t), sc->stream));
    rc = launch_space_eval(s, 0, n, d, d + n, sc->stream);
    std::vector<int64_t> h(2 * n);
    if (!rc)
        rc = cuda_check(cudaMemcpyAsync(h.data(), d, 2 * n * sizeof(int64_t),
                                        cudaMemcpyDeviceToHost, sc->stream),
                        "sweep copy");
    cudaFreeAsync(d, sc->stream);
    if (!rc) rc = cuda_check(cudaStreamSynchronize(sc->stream), "sweep sync");
    if (rc) return rc;
    struct Row {
        int64_t wg, ts, time, transitions, ok, note;
    };
    std::vector<Row> out;
    out.reserve(n);
    // enumerate_configs order: wg ascending, then ts ascending (model.cpp:96-98);
    // space index order is wg descending, ts descending.
    const int L = log2i(size) - 1;
    for (int i = 1; i <= L; ++i)
        for (int j = 1; j <= L; ++j) {
            const uint64_t idx = (uint64_t)(L - i) * L + (uint64_t)(L - j);
            Row r{1ll << i, 1ll << j, h[idx], h[n + idx], 1, 0};
            if (r.time < 0) {
                r.ok = 0;
                r.note = 1;
                r.time = r.transitions = 0;
            }
            out.push_back(r);
        }
    std::stable_sort(out.begin(), out.end(), [](const Row& a, const Row& b) {
        if (a.ok != b.ok) return a.ok > b.ok;
        if (!a.ok) return false;
        if (a.time != b.time) return a.time < b.time;
        return a.transitions < b.transitions;
    });
    *n_rows = (int64_t)out.size();
    for (size_t i = 0; i < out.size() && (int64_t)i < cap; ++i) {
        const Row& r = out[i];
        const int64_t v[6] = {r.wg, r.ts, r.time, r.transitions, r.ok, r.note};
        std::memcpy(rows + 6 * i, v, sizeof v);
    }
    return MCTB_OK;
}

}  // extern "C"
