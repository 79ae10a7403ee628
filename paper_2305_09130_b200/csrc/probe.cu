// Issue-rate probes: the measured denominator of the cost-model kernel's
// roofline (bench.py "roofline").  The cost-model kernel is bound by
// instruction issue on the integer pipes (ncu: issue active ~90%, ALU pipe
// ~83%), so its ceiling is the rate at which an SM can issue integer
// instructions.  Each probe runs 8 independent dependency chains per thread at
// full occupancy (64 warps per SM), so latency is hidden and only issue
// throughput remains:
//   variant 0: IMAD (fma pipe) alternating with LOP3 (alu pipe)
//   variant 1: IADD3 only
//   variant 2: IADD3 + LOP3 + IMAD + SHF, the cost-model loop's mix
//   variant 3: FFMA only (the chip's fp32 issue rate: the SMSP issue ceiling)
// Every probe operation is one PTX instruction that ptxas maps to one SASS
// instruction, so operations/s = thread instructions/s, the unit of the
// kernel's ncu count.  mctb_int32_peak reports the best integer variant
// (thread instructions per second over the chip); mctb_issue_probe one variant.
#include "common.cuh"

namespace mctb {
namespace {

template <int V>
__global__ void __launch_bounds__(256) issue_probe_kernel(uint32_t iters, uint32_t seed,
                                                          uint32_t* sink) {
    uint32_t a[8];
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = seed ^ (threadIdx.x * (2 * k + 1));
        f[k] = (float)a[k] * 1e-9f;
    }
    const uint32_t c = seed >> 3;
    const float fm = 0.999f, fc = 1e-7f;
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                // each chain takes its neighbour as an operand: nothing folds at
                // compile time, and the 8 chains stay independent within a step
                const uint32_t b = a[(k + 1) & 7];
                if (V == 0) {
                    if (k & 1)
                        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
                    else
                        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
                } else if (V == 1) {
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
                } else if (V == 2) {
                    if ((k & 3) == 0)
                        asm volatile("add.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
                    else if ((k & 3) == 1)
                        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
                    else if ((k & 3) == 2)
                        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
                    else
                        asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(b));
                } else {
                    asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[k]) : "f"(fm), "f"(fc));
                }
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r ^= a[k] ^ __float_as_uint(f[k]);
    if (r == 0x9e3779b9u) *sink = r;  // keeps the chains alive
}

using ProbeFn = void (*)(uint32_t, uint32_t, uint32_t*);

int run_probe(int variant, double* ops_per_sec, double* ms) {
    int rc = require_device();
    if (rc) return rc;
    static const ProbeFn fns[4] = {issue_probe_kernel<0>, issue_probe_kernel<1>,
                                   issue_probe_kernel<2>, issue_probe_kernel<3>};
    if (variant < 0 || variant > 3) {
        set_error("probe variant must be 0..3");
        return MCTB_CONFIG_ERROR;
    }
    int dev = 0, sms = 0;
    MCTB_CUDA(cudaGetDevice(&dev));
    MCTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    uint32_t* sink = nullptr;
    MCTB_CUDA(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1;
    MCTB_CUDA(cudaEventCreate(&e0));
    MCTB_CUDA(cudaEventCreate(&e1));
    const unsigned blocks = (unsigned)sms * 8, threads = 256;
    const uint32_t iters = 1024;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        fns[variant]<<<blocks, threads>>>(iters, 0x1234567u + rep, sink);
        cudaEventRecord(e1);
        MCTB_CUDA(cudaEventSynchronize(e1));
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        if (rep > 0 && t < best) best = t;  // first launch is warm-up
    }
    MCTB_CUDA(cudaGetLastError());
    // 256 probe instructions per iteration (one SASS instruction each, checked with
    // cuobjdump) plus ~3 of loop control (~1%, not counted: a slight underestimate)
    const double ops = (double)blocks * threads * iters * 32.0 * 8.0;
    *ops_per_sec = ops / (best * 1e-3);
    *ms = best;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return MCTB_OK;
}

}  // namespace
}  // namespace mctb

extern "C" int mctb_issue_probe(int variant, double* ops_per_sec, double* ms) {
    return mctb::run_probe(variant, ops_per_sec, ms);
}

extern "C" int mctb_int32_peak(double* ops_per_sec, double* ms) {
    double best = 0, best_ms = 0;
    for (int v = 0; v < 3; ++v) {
        double o = 0, t = 0;
        const int rc = mctb::run_probe(v, &o, &t);
        if (rc) return rc;
        if (o > best) {
            best = o;
            best_ms = t;
        }
    }
    *ops_per_sec = best;
    *ms = best_ms;
    return MCTB_OK;
}
