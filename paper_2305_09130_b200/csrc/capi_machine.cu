// C ABI over the GPU transition system: single runs (Machine::run), batched
// trajectories (swarm), replay and trace rendering.
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "traj.cuh"

namespace mctb {

int check_platform(const int* plat);
int check_problem(int size, int kernel);
bool is_pow2(long long v);

// Machine::Machine preconditions (machine.cpp:60-69): validate_params
// (model.cpp:62-70) and, for the minimum kernel, the feasibility check of
// build_minimum_kernel (kernel.cpp:56-62).
int check_machine(const int* plat, int size, int kernel, int wg, int ts) {
    int rc = check_platform(plat);
    if (rc) return rc;
    if ((rc = check_problem(size, kernel))) return rc;
    const int hi = size / 2;
    if (!is_pow2(wg) || wg < 2 || wg > hi) {
        set_error("wg must be a power of two in [2, size/2], got " + std::to_string(wg));
        return MCTB_CONFIG_ERROR;
    }
    if (!is_pow2(ts) || ts < 2 || ts > hi) {
        set_error("ts must be a power of two in [2, size/2], got " + std::to_string(ts));
        return MCTB_CONFIG_ERROR;
    }
    if (kernel == 1) {
        int logn = 0;
        while ((1 << logn) < size) ++logn;
        const long long wgs = std::max((long long)size / ((long long)wg * ts), 1ll);
        if (wgs * wg * ts > size) {
            set_error("infeasible (wg, ts): workgroups would index past the input (" +
                      std::to_string(wgs * wg * ts) + " > " + std::to_string(size) + ")");
            return MCTB_CONFIG_ERROR;
        }
    }
    return MCTB_OK;
}

// The cost-and-effect programs the machine runs (kernel.cpp build_abstract_kernel /
// build_minimum_kernel), materialised from the instruction view the GPU kernels
// compute arithmetically (machine.cuh instr_at): out = int32[3 * cap] rows {kind
// (0 busy, 1 barrier, 2 effect, 3 end), ticks, operand} — the per-activation
// sequence, then the epilogue; operand = the effect's source offset (phase 0:
// glob[shift + operand] into loc[me]; epilogue: loc[me + operand] into loc[me],
// or -1: loc[me] into glob[0]).
int kernel_program(const int* plat, int size, int kernel, int wg, int ts, int32_t* out,
                   int cap, int* n_act, int* n_epi) {
    int rc = check_machine(plat, size, kernel, wg, ts);
    if (rc) return rc;
    MachHost h;
    if ((rc = build_desc(plat, size, kernel, nullptr, wg, ts, &h))) return rc;
    int n = 0;
    for (int phase = 0; phase < 2; ++phase) {
        int len = 0;
        if (phase == 1 && !has_epilogue(h.d)) {
            *n_epi = 0;
            break;
        }
        for (int c = 0;; ++c) {
            const Instr in = instr_at(h.d, phase, c);
            const int kind = in.kind == IK_BUSY ? 0 : in.kind == IK_BARRIER ? 1
                             : in.kind == IK_EFFECT ? 2 : 3;
            if (n < cap) {
                out[3 * n] = kind;
                out[3 * n + 1] = in.kind == IK_BUSY ? (int32_t)in.ticks : 0;
                out[3 * n + 2] = in.kind == IK_EFFECT ? in.src : 0;
            }
            ++n;
            ++len;
            if (kind == 3) break;
        }
        (phase == 0 ? *n_act : *n_epi) = len;
    }
    if (n > cap) {
        set_error("kernel program buffer too small");
        return MCTB_LIMIT;
    }
    return MCTB_OK;
}

namespace {

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

const char* kRoles[] = {"main", "host", "clock", "device", "unit", "barrier", "pex"};

}  // namespace

// Machine::process_name (machine.cpp:103-113)
std::string pname(const MachDesc& m, int pid) {
    int role, ord;
    role_of(m, pid, role, ord);
    if (role <= 2) return kRoles[role];
    return std::string(kRoles[role]) + std::to_string(ord);
}

namespace {

// Machine::label (machine.cpp:758-786)
std::string label(const MachDesc& m, const Transition& t) {
    const std::string peer = t.peer == kNoPeer || t.peer >= m.n_proc ? "" : pname(m, t.peer);
    switch (t.op) {
        case OP_CLOCKTICK: return "tick";
        case OP_CLOCKHALT: return "halt";
        case OP_HOSTGO: return "go -> " + peer;
        case OP_HOSTREACTGO: return "go(react) -> " + peer;
        case OP_HOSTSTOP: return "stop -> " + peer;
        case OP_HOSTSETFIN: return "fin";
        case OP_DEVICEUNITGO: return "go(wg" + std::to_string(t.arg) + ") -> " + peer;
        case OP_DEVICEDONE: return "done -> host";
        case OP_DEVICEUNITSTOP: return "stop -> " + peer;
        case OP_UNITPEXGO: return "go(round" + std::to_string(t.arg) + ") -> " + peer;
        case OP_UNITDONE: return "done(wg" + std::to_string(t.arg) + ") -> " + peer;
        case OP_UNITPEXSTOP: return "stop -> " + peer;
        case OP_UNITBARRIERSTOP: return "stop -> " + peer;
        case OP_PEXREPORT: return "report";
        case OP_PEXEFFECT: return "effect[" + std::to_string(t.arg) + "]";
        case OP_PEXARRIVE: return "barrier-arrive -> " + peer;
        case OP_PEXITEMDONE: return "item-done -> " + peer;
        case OP_PEXENDDONE: return "group-done -> " + peer;
        case OP_BARRIERRELEASE: return "barrier-release";
    }
    return "?";
}

thread_local double g_traj_kernel_ms = 0.0;  // last mctb_trajectories kernel time

int stream_of(cudaStream_t* s) {
    static thread_local cudaStream_t st = nullptr;
    if (!st) MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *s = st;
    return MCTB_OK;
}

}  // namespace

// Replays `trace` on the GPU; fills per-step times (optional) and the outcome.
int gpu_replay(MachHost& h, const int32_t* trace, int64_t len, std::vector<int64_t>* step_time,
               TrajOut* out) {
    cudaStream_t st;
    int rc = stream_of(&st);
    if (rc) return rc;
    int32_t* d_ids = nullptr;
    if ((rc = upload_desc(h, st, &d_ids))) return rc;
    DevBuf ids{d_ids, st}, tr{nullptr, st}, times{nullptr, st}, o{nullptr, st};
    MCTB_CUDA(cudaMallocAsync(&tr.p, std::max<int64_t>(len, 1) * 16, st));
    MCTB_CUDA(cudaMallocAsync(&o.p, sizeof(TrajOut), st));
    if (step_time) MCTB_CUDA(cudaMallocAsync(&times.p, std::max<int64_t>(len, 1) * 8, st));
    if (len) MCTB_CUDA(cudaMemcpyAsync(tr.p, trace, len * 16, cudaMemcpyHostToDevice, st));
    if ((rc = launch_replay(h.d, (int32_t*)tr.p, len, (int64_t*)times.p, (TrajOut*)o.p, st)))
        return rc;
    if (step_time) {
        step_time->resize(len);
        if (len)
            MCTB_CUDA(cudaMemcpyAsync(step_time->data(), times.p, len * 8, cudaMemcpyDeviceToHost, st));
    }
    MCTB_CUDA(cudaMemcpyAsync(out, o.p, sizeof(TrajOut), cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    return MCTB_OK;
}

// One run on the GPU with trace capture (trace may be null).
int gpu_run(MachHost& h, int policy, uint64_t seed, uint64_t traj, int64_t max_steps,
            TrajOut* out, int32_t* trace, int64_t cap) {
    cudaStream_t st;
    int rc = stream_of(&st);
    if (rc) return rc;
    int32_t* d_ids = nullptr;
    if ((rc = upload_desc(h, st, &d_ids))) return rc;
    DevBuf ids{d_ids, st}, desc{nullptr, st}, o{nullptr, st}, tr{nullptr, st};
    MCTB_CUDA(cudaMallocAsync(&desc.p, sizeof(MachDesc), st));
    MCTB_CUDA(cudaMemcpyAsync(desc.p, &h.d, sizeof(MachDesc), cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMallocAsync(&o.p, sizeof(TrajOut), st));
    if (trace && cap > 0) MCTB_CUDA(cudaMallocAsync(&tr.p, cap * 16, st));
    if ((rc = launch_trajectories((MachDesc*)desc.p, 1, policy, seed, traj, 1, max_steps,
                                  (TrajOut*)o.p, (int32_t*)tr.p, trace ? cap : 0, st)))
        return rc;
    MCTB_CUDA(cudaMemcpyAsync(out, o.p, sizeof(TrajOut), cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    if (trace && cap > 0) {
        const int64_t n = std::min<int64_t>(out->steps, cap);
        if (n) MCTB_CUDA(cudaMemcpyAsync(trace, tr.p, n * 16, cudaMemcpyDeviceToHost, st));
        MCTB_CUDA(cudaStreamSynchronize(st));
    }
    return MCTB_OK;
}

std::string render_trace(const MachHost& h, const int32_t* trace, int64_t len,
                         const std::vector<int64_t>& times, int64_t final_time, int32_t glob0) {
    std::string os;
    os.reserve((size_t)len * 40 + 64);
    for (int64_t i = 0; i < len; ++i) {
        const Transition t{(uint16_t)trace[4 * i], (uint16_t)trace[4 * i + 1], trace[4 * i + 2],
                           trace[4 * i + 3]};
        int role, ord;
        role_of(h.d, t.actor, role, ord);
        os += std::to_string(i) + ' ' + std::to_string(t.actor) + ' ' + kRoles[role] + ' ' +
              label(h.d, t) + " time=" + std::to_string(times[i]) + '\n';
    }
    os += "FINAL time=" + std::to_string(final_time) + " wg=" + std::to_string(h.d.wg) +
          " ts=" + std::to_string(h.d.ts);
    if (h.d.kernel == 1) os += " result=" + std::to_string(h.value(glob0));
    os += '\n';
    return os;
}

}  // namespace mctb

using namespace mctb;

extern "C" {

int mctb_simulate(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                  int policy, uint64_t seed, uint64_t traj, int64_t* out, int32_t* trace,
                  int64_t cap, int64_t* trace_len) {
    int rc = check_machine(plat, size, kernel, wg, ts);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    MachHost h;
    if ((rc = build_desc(plat, size, kernel, input, wg, ts, &h))) return rc;
    TrajOut o;
    if ((rc = gpu_run(h, policy, seed, traj, 200000000LL, &o, trace, trace ? cap : 0))) return rc;
    if (trace_len) *trace_len = o.steps;
    if (o.status == MCTB_MODEL_BUG) {
        set_error("machine (wg=" + std::to_string(wg) + ", ts=" + std::to_string(ts) +
                  "): deadlock: non-terminal state with no enabled transition at time " +
                  std::to_string(o.time));
        return MCTB_MODEL_BUG;
    }
    if (o.status == MCTB_LIMIT) {
        set_error("machine: run exceeded the step limit");
        return MCTB_MODEL_BUG;
    }
    out[0] = o.time;
    out[1] = o.steps;
    out[2] = kernel == 1 ? h.value(o.glob0) : INT64_MIN;
    out[3] = h.d.n_proc;
    return MCTB_OK;
}

int mctb_trajectories(const int* plat, int size, int kernel, const int64_t* input,
                      const int32_t* configs, int n_configs, int policy, uint64_t seed,
                      uint64_t traj0, uint64_t n_traj, int64_t max_steps, int64_t* out) {
    int rc;
    if (n_configs < 1) {
        set_error("no configurations");
        return MCTB_CONFIG_ERROR;
    }
    std::vector<MachHost> hs(n_configs);
    for (int c = 0; c < n_configs; ++c) {
        if ((rc = check_machine(plat, size, kernel, configs[2 * c], configs[2 * c + 1]))) return rc;
        if ((rc = build_desc(plat, size, kernel, input, configs[2 * c], configs[2 * c + 1], &hs[c])))
            return rc;
    }
    if ((rc = require_device())) return rc;
    cudaStream_t st;
    if ((rc = stream_of(&st))) return rc;
    int32_t* d_ids = nullptr;
    if ((rc = upload_desc(hs[0], st, &d_ids))) return rc;
    DevBuf ids{d_ids, st}, desc{nullptr, st}, o{nullptr, st};
    std::vector<MachDesc> descs(n_configs);
    for (int c = 0; c < n_configs; ++c) {
        hs[c].d.input_id = d_ids;
        descs[c] = hs[c].d;
    }
    MCTB_CUDA(cudaMallocAsync(&desc.p, n_configs * sizeof(MachDesc), st));
    MCTB_CUDA(cudaMemcpyAsync(desc.p, descs.data(), n_configs * sizeof(MachDesc),
                              cudaMemcpyHostToDevice, st));
    MCTB_CUDA(cudaMallocAsync(&o.p, std::max<uint64_t>(n_traj, 1) * sizeof(TrajOut), st));
    DevBuf rec{nullptr, st};
    MCTB_CUDA(cudaMallocAsync(&rec.p, std::max<uint64_t>(n_traj, 1) * 6 * sizeof(int64_t), st));
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    if (!ev[0]) {
        MCTB_CUDA(cudaEventCreate(&ev[0]));
        MCTB_CUDA(cudaEventCreate(&ev[1]));
    }
    MCTB_CUDA(cudaEventRecord(ev[0], st));
    if ((rc = launch_trajectories((MachDesc*)desc.p, n_configs, policy, seed, traj0, n_traj,
                                  max_steps, (TrajOut*)o.p, nullptr, 0, st)))
        return rc;
    MCTB_CUDA(cudaEventRecord(ev[1], st));
    // the records are formatted on the device and land in the caller's buffer
    // with one copy (no host staging or per-record host loop)
    if ((rc = launch_traj_records((TrajOut*)o.p, n_traj, kernel, (int64_t*)rec.p, st))) return rc;
    MCTB_CUDA(cudaMemcpyAsync(out, rec.p, n_traj * 6 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MCTB_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    MCTB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    g_traj_kernel_ms = ms;
    if (kernel == 1)
        for (uint64_t i = 0; i < n_traj; ++i) {
            int64_t* r = out + 6 * i;
            r[2] = hs[r[5]].value((int32_t)r[2]);
        }
    return MCTB_OK;
}

double mctb_trajectories_kernel_ms(void) { return g_traj_kernel_ms; }

int mctb_replay(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                const int32_t* trace, int64_t len, int64_t final_time, int64_t* out) {
    int rc = check_machine(plat, size, kernel, wg, ts);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    MachHost h;
    if ((rc = build_desc(plat, size, kernel, input, wg, ts, &h))) return rc;
    TrajOut o;
    if ((rc = gpu_replay(h, trace, len, nullptr, &o))) return rc;
    if (o.status != MCTB_OK) {
        set_error(o.steps < len ? "replay diverged at step " + std::to_string(o.steps)
                                : std::string("replayed trace does not end terminal"));
        return MCTB_CORRUPT_TRACE;
    }
    if (o.time != final_time) {
        set_error("replayed final time " + std::to_string(o.time) + " != recorded " +
                  std::to_string(final_time));
        return MCTB_CORRUPT_TRACE;
    }
    out[0] = o.time;
    out[1] = kernel == 1 ? h.value(o.glob0) : INT64_MIN;
    return MCTB_OK;
}

int64_t mctb_trace_text(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, const int32_t* trace, int64_t len, char* buf, int64_t cap) {
    if (check_machine(plat, size, kernel, wg, ts) || require_device()) return -1;
    MachHost h;
    if (build_desc(plat, size, kernel, input, wg, ts, &h)) return -1;
    TrajOut o;
    std::vector<int64_t> times;
    if (gpu_replay(h, trace, len, &times, &o)) return -1;
    if (o.steps < len) {
        set_error("trace does not replay");
        return -1;
    }
    const std::string s = render_trace(h, trace, len, times, o.time, o.glob0);
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, (int64_t)s.size());
        std::memcpy(buf, s.data(), (size_t)n);
        buf[n] = 0;
    }
    return (int64_t)s.size();
}

// the programs of build_abstract_kernel / build_minimum_kernel (kernel.hpp:92-118)
int mctb_kernel_program(const int* plat, int size, int kernel, int wg, int ts, int32_t* out,
                        int cap, int* n_act, int* n_epi) {
    return kernel_program(plat, size, kernel, wg, ts, out, cap, n_act, n_epi);
}

}  // extern "C"
