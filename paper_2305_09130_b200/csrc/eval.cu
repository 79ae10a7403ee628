// Exhaustive evaluation of a tuning space on B200 (north-star subsystem 1).
//
// One thread evaluates a contiguous run of configuration indices with the
// lock-step cost model (cost_model.cuh) in integer model time, keeps the
// lexicographic minimum of (saturated time, index), reduces it across the
// warp with shuffles and across the CTA in shared memory, and min-combines
// one packed 64-bit key per CTA with atomicMin:
//     key = (min(time, 2^30 - 1) << 33) | index.
// The index order puts the reference's preferred configuration (largest wg,
// then largest ts — explore.cpp:64-72, search.cpp:67-78) first, so the
// minimum key breaks ties exactly as bisect_min_time does.
//
// Nothing here reads memory on the hot path: the kernel is bound by integer
// issue (one u32 division and ~30 IADD3/IMAD/ISETP per configuration), so the
// grid is a multiple of the 148 SMs and each thread amortises its index decode
// over thousands of configurations (nd is the fastest digit; per-(wg, ts, np,
// nu) quantities are hoisted out of the nd loop).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "cost_model.cuh"

namespace mctb {

namespace {

constexpr int kThreads = 256;
#ifndef MCTB_ARGMIN_MINB
#define MCTB_ARGMIN_MINB 1  // resident CTAs per SM the register allocation targets
#endif

// a << sh, saturating at INT64_MAX (a >= 0)
__device__ __forceinline__ int64_t shl_sat(int64_t a, int sh) {
    return (sh >= 62 || (a >> (62 - sh)) != 0) ? INT64_MAX : (a << sh);
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

__device__ __forceinline__ void cta_min_commit(uint64_t key, unsigned long long* out) {
    __shared__ uint64_t warp_best[kThreads / 32];
    key = warp_min_u64(key);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_best[warp] = key;
    __syncthreads();
    if (warp == 0) {
        key = lane < kThreads / 32 ? warp_best[lane] : kKeyNone;
        key = warp_min_u64(key);
        if (lane == 0 && key != kKeyNone) atomicMin(out, (unsigned long long)key);
    }
}

// a * b + c with a multiplier unknown to ptxas: stays an IMAD (FMA pipe)
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

template <int KERNEL>
__global__ void __launch_bounds__(kThreads, MCTB_ARGMIN_MINB) space_argmin_kernel(SpaceDev sd, uint64_t first,
                                                                uint64_t count,
                                                                uint64_t per_thread,
                                                                unsigned long long* out_key) {
    const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    uint64_t pos = tid * per_thread;
    const uint64_t end = min(pos + per_thread, count);
    uint32_t best_tf = kKeySat + 1;  // "nothing yet": above every real (saturated) time
    uint64_t best_idx = 0;
    if (pos < end) {
        const Config c0 = decode(sd, first + pos);
        uint32_t nd_d = (uint32_t)(c0.nd - sd.nd_lo);
        int nu = c0.nu, lognp = c0.lognp, logwg = c0.logwg, logts = c0.logts;
        const int64_t size = 1ll << sd.logn;
        const int64_t gmt = sd.gmt;
        const int64_t A = size * (gmt + 1) + gmt;  // abstract: (size/ts)(gmt ts + ts) + gmt
        while (pos < end) {
            // ---- quantities fixed along the nd digit
            const int s = logwg + logts;
            const uint32_t wgs = s < sd.logn ? (1u << (sd.logn - s)) : 1u;
            const uint32_t q = wgs / (uint32_t)nu;
            const uint32_t nwu = wgs <= (uint32_t)nu ? wgs : (uint32_t)nu;
            const int lognwe = logwg < lognp ? logwg : lognp;
            const uint32_t dr = max(wgs / nwu, 1u);
            const uint32_t nd_thr = (wgs + (uint32_t)nu - 1) / (uint32_t)nu;  // wgs <= nu*nd
            int64_t D;
            bool feasible = true;
            if (KERNEL == 0) {
                D = shl_sat(A, logwg - lognwe);
            } else {
                feasible = s <= sd.logn;
                D = shl_sat(gmt, logts + logwg - lognwe);
                if (D != INT64_MAX) D += (1ll << lognwe) - 1 + gmt;
            }
            const uint32_t run = (uint32_t)min((uint64_t)(sd.n_nd - nd_d), end - pos);
            if (!feasible || D >= (int64_t)kKeySat) {
                if (best_tf > kKeySat) {  // only reachable before any real time
                    best_tf = kKeySat;
                    best_idx = first + pos;
                }
            } else {
                const uint32_t D32 = (uint32_t)D;
                uint32_t nd = (uint32_t)sd.nd_lo + nd_d;
                const uint64_t base = first + pos;
                // waves = ceil(dr / nwd) with nwd = nd below nd_thr (one working device per
                // workgroup batch) and nwd = q above it.  Below nd_thr the quotient is
                // strength-reduced along the nd digit: dr = Q*nd + R, and nd -> nd+1 gives
                // R -= Q with at most one correction (Q -= 1, R += nd+1) once Q <= nd+1,
                // predicated, so the hot loop has no branch and no XU (I2F/MUFU/F2I) work.
                const uint32_t w_hi = q == 0 ? dr : (dr + q - 1) / q;
                const uint32_t thr = q == 0 ? 0u : nd_thr;  // nd >= thr: waves = w_hi
                // waves * D32 < kKeySat  <=>  waves <= wmax (32-bit saturating product)
                const uint32_t wmax = (kKeySat - 1) / D32;
                uint32_t best_k = 0xffffffffu;
                uint32_t k = 0;
                // one correction per step needs Q = (dr - 1) / nd <= nd + 1, implied by
                // dr <= nd (nd + 2): below that (small nd) divide exactly
                for (; k < run && nd < 65536u && dr > nd * (nd + 2); ++k, ++nd) {
                    const uint32_t waves = nd >= thr ? w_hi : (dr + nd - 1) / nd;
                    const uint32_t tf = waves <= wmax ? waves * D32 : kKeySat;
                    if (tf < best_tf) {
                        best_tf = tf;
                        best_k = k;
                    }
                }
                // ceil(dr / nd) = floor((dr - 1) / nd) + 1 (dr >= 1): the recurrence runs
                // on dm = dr - 1, so waves is one add (no R != 0 test)
                const uint32_t dm = dr - 1;
                uint32_t Q = dm / nd;
                int32_t R = (int32_t)(dm - Q * nd);
                // for nd < thr, nd <= q, so ceil(dr/nd) >= ceil(dr/q) = w_hi; for nd >= thr
                // ceil(dr/nd) <= w_hi: waves = max(Q + 1, w_hi) in both ranges.  waves is
                // non-increasing along nd, so the saturated configurations (waves > wmax)
                // form a prefix of the run: the main loop needs no saturation test
                for (; k < run; ++k) {
                    if (max(Q + 1, w_hi) <= wmax) break;
                    if (kKeySat < best_tf) {
                        best_tf = kKeySat;
                        best_k = k;
                    }
                    ++nd;
                    R -= (int32_t)Q;
                    if (R < 0) {
                        Q -= 1;
                        R += (int32_t)nd;
                    }
                }
                // Every configuration's waves is evaluated and compared.  Within the run
                // the batch duration D32 is fixed and waves is non-increasing, so the
                // run's least (time, index) is its last waves at the first index that
                // reached it: compare each waves with its predecessor (one ISETP and a
                // predicated move; no product, no running min) and form the time once
                // at the end of the run.
                // (waves - 1 = max(Q, w_hi - 1) is compared: the same order, one VIMNMX)
                if (k < run) {
                    const uint32_t w_hm1 = w_hi - 1;  // w_hi >= 1
                    uint32_t prev = 0xffffffffu, run_k = k;
#pragma unroll 16
                    for (; k < run; ++k) {
                        const uint32_t w = max(Q, w_hm1);
                        run_k = w < prev ? k : run_k;
                        prev = w;
                        // nd -> nd + 1: dm = Q (nd+1) + (R - Q), at most one correction,
                        // applied as c * nd with c = (R < 0) in {0, 1}: one IMAD (FMA
                        // pipe) in place of a mask and an add on the saturated ALU pipe
                        ++nd;
                        R -= (int32_t)Q;
                        const uint32_t c = (uint32_t)R >> 31;
                        Q -= c;
                        R = (int32_t)mad_u32(c, nd, (uint32_t)R);
                    }
                    // strict: an equal time from the prefix loops keeps its smaller index
                    const uint32_t tf = (prev + 1) * D32;
                    if (tf < best_tf) {
                        best_tf = tf;
                        best_k = run_k;
                    }
                }
                if (best_k != 0xffffffffu) best_idx = base + best_k;
            }
            pos += run;
            // ---- odometer: advance nu, np, ts, wg digits
            nd_d = 0;
            if (++nu > sd.nu_hi) {
                nu = sd.nu_lo;
                if (++lognp > sd.lognp_hi) {
                    lognp = sd.lognp_lo;
                    if (--logts < sd.logts_lo) {
                        logts = sd.logts_hi;
                        --logwg;
                    }
                }
            }
        }
    }
    const uint64_t key =
        best_tf > kKeySat ? kKeyNone : (((uint64_t)best_tf << MCTB_KEY_INDEX_BITS) | best_idx);
    cta_min_commit(key, out_key);
}

__global__ void space_eval_kernel(SpaceDev sd, int kernel, uint64_t first, uint64_t count,
                                  int64_t* __restrict__ time, int64_t* __restrict__ steps) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const Cost c = lockstep_cost(kernel, sd.logn, sd.gmt, decode(sd, first + i));
    time[i] = c.time;
    steps[i] = c.steps;
}

// Exact evaluation of the winning index: out = {time, steps, nd, nu, np, gmt, wg, ts}
__global__ void space_point_kernel(SpaceDev sd, int kernel, const unsigned long long* key,
                                   int64_t* out) {
    const uint64_t k = *key;
    if (k == kKeyNone) {
        out[0] = -2;
        return;
    }
    const Config c = decode(sd, k & kKeyIndexMask);
    const Cost r = lockstep_cost(kernel, sd.logn, sd.gmt, c);
    out[0] = r.time;
    out[1] = r.steps;
    out[2] = c.nd;
    out[3] = c.nu;
    out[4] = 1ll << c.lognp;
    out[5] = sd.gmt;
    out[6] = 1ll << c.logwg;
    out[7] = 1ll << c.logts;
}

__global__ void fill_u64_kernel(unsigned long long* p, unsigned long long v) { *p = v; }

// ---- exact resolution of a saturated key ("Exactness").
// The packed key saturates its time field at 2^30 - 1, so when every
// configuration of the range has time >= 2^30 - 1 the key's index is only the
// first saturated (or infeasible) index.  These two plain passes are the exact
// argmin by construction: the least full 64-bit time of the feasible
// configurations (make_space bounds every time and transition count below
// 2^62), then the least index with that time (the reference's tie rule,
// search.cpp:67-78).  Not on the hot path: they run only for saturated keys.
__device__ __forceinline__ unsigned long long warp_min_ull(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

__global__ void space_min_time_kernel(SpaceDev sd, uint64_t first, uint64_t count,
                                      unsigned long long* out_time) {
    unsigned long long best = ULLONG_MAX;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const Cost c = lockstep_cost(sd.kernel, sd.logn, sd.gmt, decode(sd, first + i));
        if (c.feasible && (unsigned long long)c.time < best) best = (unsigned long long)c.time;
    }
    best = warp_min_ull(best);
    if ((threadIdx.x & 31) == 0 && best != ULLONG_MAX) atomicMin(out_time, best);
}

__global__ void space_first_at_kernel(SpaceDev sd, uint64_t first, uint64_t count,
                                      const unsigned long long* time,
                                      unsigned long long* out_index) {
    const unsigned long long t = *time;
    unsigned long long best = ULLONG_MAX;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const Cost c = lockstep_cost(sd.kernel, sd.logn, sd.gmt, decode(sd, first + i));
        if (c.feasible && (unsigned long long)c.time == t) {
            best = first + i;  // grid-stride order: a thread's first hit is its least index
            break;
        }
    }
    best = warp_min_ull(best);
    if ((threadIdx.x & 31) == 0 && best != ULLONG_MAX) atomicMin(out_index, best);
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

}  // namespace

// Validates the descriptor and fills the device view.  The ranges must keep
// every configuration inside validate_params (model.cpp:62-70).
int make_space(const int64_t* sd, SpaceDev* out) {
    const int64_t kernel = sd[0], size = sd[1];
    if (kernel != 0 && kernel != 1) {
        set_error("kernel must be 0 (abstract) or 1 (minimum)");
        return MCTB_CONFIG_ERROR;
    }
    if (size < 4 || (size & (size - 1)) || size > (1ll << 30)) {
        set_error("size must be a power of two in [4, 2^30]");
        return MCTB_CONFIG_ERROR;
    }
    int logn = 0;
    while ((1ll << logn) < size) ++logn;
    if (sd[2] < 1 || sd[2] > (1 << 20)) {
        set_error("gmt must be in [1, 2^20]");
        return MCTB_CONFIG_ERROR;
    }
    if (sd[3] < 1 || sd[4] < sd[3] || sd[4] > (1 << 24) || sd[5] < 1 || sd[6] < sd[5] ||
        sd[6] > (1 << 24)) {
        set_error("nd and nu ranges must satisfy 1 <= lo <= hi <= 2^24");
        return MCTB_CONFIG_ERROR;
    }
    if (sd[7] < 0 || sd[8] < sd[7] || sd[8] > 24) {
        set_error("log2 np range must satisfy 0 <= lo <= hi <= 24");
        return MCTB_CONFIG_ERROR;
    }
    if (sd[9] < 1 || sd[10] < sd[9] || sd[10] > logn - 1 || sd[11] < 1 || sd[12] < sd[11] ||
        sd[12] > logn - 1) {
        set_error("log2 wg and log2 ts ranges must lie in [1, log2(size) - 1]");
        return MCTB_CONFIG_ERROR;
    }
    // every model time and transition count of the space must fit int64 (the
    // reference's Tick, model.hpp): the abstract kernel's largest time is below
    // (size/2)(size(gmt+1) + gmt) and its transition count below 3 size^2 (gmt+1)
    // (cost_model.cuh), so 4 size^2 (gmt+1) <= 2^62 bounds both.  The minimum
    // kernel's are below 16 size (gmt+1) <= 2^55 for every admitted size and gmt.
    if (kernel == 0) {
        int lg = 0;
        while ((1ll << lg) < sd[2] + 1) ++lg;
        if (2 * logn + lg + 2 > 62) {
            set_error("size^2 * (gmt + 1) must be below 2^60 (model times fit int64)");
            return MCTB_CONFIG_ERROR;
        }
    }
    SpaceDev s;
    s.kernel = (int32_t)kernel;
    s.logn = logn;
    s.gmt = (int32_t)sd[2];
    s.nd_lo = (int32_t)sd[3];
    s.nd_hi = (int32_t)sd[4];
    s.nu_lo = (int32_t)sd[5];
    s.nu_hi = (int32_t)sd[6];
    s.lognp_lo = (int32_t)sd[7];
    s.lognp_hi = (int32_t)sd[8];
    s.logwg_lo = (int32_t)sd[9];
    s.logwg_hi = (int32_t)sd[10];
    s.logts_lo = (int32_t)sd[11];
    s.logts_hi = (int32_t)sd[12];
    s.n_nd = (uint32_t)(s.nd_hi - s.nd_lo + 1);
    s.n_nu = (uint32_t)(s.nu_hi - s.nu_lo + 1);
    s.n_np = (uint32_t)(s.lognp_hi - s.lognp_lo + 1);
    s.n_ts = (uint32_t)(s.logts_hi - s.logts_lo + 1);
    s.n_wg = (uint32_t)(s.logwg_hi - s.logwg_lo + 1);
    const double total = (double)s.n_nd * s.n_nu * s.n_np * s.n_ts * s.n_wg;
    if (total >= (double)(1ull << MCTB_KEY_INDEX_BITS)) {
        set_error("tuning space exceeds 2^33 configurations");
        return MCTB_CONFIG_ERROR;
    }
    *out = s;
    return MCTB_OK;
}

uint64_t space_count(const SpaceDev& s) {
    return (uint64_t)s.n_nd * s.n_nu * s.n_np * s.n_ts * s.n_wg;
}

int launch_space_argmin(const SpaceDev& s, uint64_t first, uint64_t count, uint64_t* d_key,
                        cudaStream_t stream) {
    if (first + count > space_count(s)) {
        set_error("index range outside the tuning space");
        return MCTB_CONFIG_ERROR;
    }
    if (count == 0) return MCTB_OK;
    // 64 CTAs of 256 threads per SM (8 waves of the 8 resident CTAs), each thread a
    // contiguous run of >= 16 indices.  Threads' costs differ (exact division for
    // small nd, odometer carries), so one resident wave of long runs left half the
    // warps idle at the tail; the hardware CTA scheduler balances the finer grid.
    // configs[4] per step (1e9): 8 CTAs/SM 0.50 ms, 16 0.44, 32 0.40, 64 0.385,
    // 128 0.40, 256 0.45
    static const int kCtasPerSm = [] {
        const char* e = getenv("MCTB_ARGMIN_CTAS_PER_SM");  // experiments only
        return e ? std::max(1, atoi(e)) : 64;
    }();
    const uint64_t max_threads = (uint64_t)sm_count() * kCtasPerSm * kThreads;
    // a multiple of the 16x-unrolled loop: whole runs need no remainder iterations
    uint64_t per_thread = ((count + max_threads - 1) / max_threads + 15) & ~15ull;
    if (per_thread < 16) per_thread = 16;
    const uint64_t threads = (count + per_thread - 1) / per_thread;
    const unsigned blocks = (unsigned)((threads + kThreads - 1) / kThreads);
    auto* key = reinterpret_cast<unsigned long long*>(d_key);
    if (s.kernel == 0)
        space_argmin_kernel<0><<<blocks, kThreads, 0, stream>>>(s, first, count, per_thread, key);
    else
        space_argmin_kernel<1><<<blocks, kThreads, 0, stream>>>(s, first, count, per_thread, key);
    return cuda_check(cudaGetLastError(), "space_argmin_kernel");
}

int launch_space_eval(const SpaceDev& s, uint64_t first, uint64_t count, int64_t* d_time,
                      int64_t* d_steps, cudaStream_t stream) {
    if (first + count > space_count(s)) {
        set_error("index range outside the tuning space");
        return MCTB_CONFIG_ERROR;
    }
    if (count == 0) return MCTB_OK;
    const unsigned blocks = (unsigned)((count + 255) / 256);
    space_eval_kernel<<<blocks, 256, 0, stream>>>(s, s.kernel, first, count, d_time, d_steps);
    return cuda_check(cudaGetLastError(), "space_eval_kernel");
}

int launch_space_point(const SpaceDev& s, const uint64_t* d_key, int64_t* d_out,
                       cudaStream_t stream) {
    space_point_kernel<<<1, 1, 0, stream>>>(s, s.kernel,
                                           reinterpret_cast<const unsigned long long*>(d_key),
                                           d_out);
    return cuda_check(cudaGetLastError(), "space_point_kernel");
}

int launch_space_exact(const SpaceDev& s, uint64_t first, uint64_t count, uint64_t* d_time,
                       uint64_t* d_index, cudaStream_t stream) {
    if (first + count > space_count(s)) {
        set_error("index range outside the tuning space");
        return MCTB_CONFIG_ERROR;
    }
    auto* t = reinterpret_cast<unsigned long long*>(d_time);
    auto* x = reinterpret_cast<unsigned long long*>(d_index);
    fill_u64_kernel<<<1, 1, 0, stream>>>(t, ULLONG_MAX);
    fill_u64_kernel<<<1, 1, 0, stream>>>(x, ULLONG_MAX);
    if (count == 0) return cuda_check(cudaGetLastError(), "fill_u64_kernel");
    const uint64_t want = (count + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count() * 16;
    const unsigned blocks = (unsigned)(want < cap ? want : cap);
    space_min_time_kernel<<<blocks, 256, 0, stream>>>(s, first, count, t);
    space_first_at_kernel<<<blocks, 256, 0, stream>>>(s, first, count, t, x);
    return cuda_check(cudaGetLastError(), "space_exact_kernels");
}

int launch_fill_key(uint64_t* d_key, cudaStream_t stream) {
    fill_u64_kernel<<<1, 1, 0, stream>>>(reinterpret_cast<unsigned long long*>(d_key), kKeyNone);
    return cuda_check(cudaGetLastError(), "fill_u64_kernel");
}

}  // namespace mctb
