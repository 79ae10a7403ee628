// Machine introspection on the GPU: the reference's Machine methods on one
// explicit state (machine.hpp:151-233: initial_state, enabled, apply,
// is_terminal, check_invariants, serialize / fingerprint, process_name) for the
// C++ drop-in's `Machine` class.  Every rule and transition runs in a one-thread
// kernel over the device's MState (machine.cuh); the host only converts between
// that and a flat int64 state vector with values instead of value ids:
//   {time, nrp_work, all_nwe, fin, next_wg, host_pc, host_k, clock,
//    nwd, {pc, k, batch_base} x nwd,
//    n_units, {pc, k, nwg, sent, got_items, got_ends} x n_units,
//    n_units, {pc, count} x n_units,
//    n_pex, {pc, phase, cursor, busy_left, reported, nwg, iter} x n_pex,
//    n_glob, glob values (minimum kernel: size; abstract: 0),
//    n_loc, loc values (minimum kernel: n_units * np; abstract: 0)}
// — the fields of the reference's MachineState (machine.hpp:112-130).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "bfs.cuh"
#include "common.cuh"
#include "pack.cuh"
#include "traj.cuh"

namespace mctb {

int check_machine(const int* plat, int size, int kernel, int wg, int ts);
std::string pname(const MachDesc& m, int pid);
int lexrank_states(MachHost& h, int64_t max_depth, int64_t table_cap, int* words,
                   std::vector<uint32_t>* packed, std::vector<int32_t>* meta,
                   std::vector<uint32_t>* depth);

namespace {

__global__ void machine_op_kernel(BfsDesc bd, int op, MState* s, Transition* tr, int* out,
                                  uint32_t* words) {
    const MachDesc& m = bd.m;
    switch (op) {
        case 0: initial_state(m, *s); break;
        case 1: out[0] = enabled(m, *s, tr); break;
        case 2: out[0] = apply(m, *s, tr[0]) ? 1 : 0; break;
        case 4: {  // replay: apply out[0] transitions from the initial state
            const int n = out[0];
            initial_state(m, *s);
            int i = 0;
            while (i < n && apply(m, *s, tr[i])) ++i;
            out[0] = i;
            out[1] = is_terminal(m, *s) ? 1 : 0;
            break;
        }
        default: {
            out[0] = is_terminal(m, *s) ? 1 : 0;
            out[1] = check_invariants(m, *s);
            uint32_t key[kMaxWords];
            pack(bd, 0, *s, key);
            for (int k = 0; k < bd.l.words; ++k) words[k] = key[k];
            out[2] = bd.l.words;
        }
    }
}

int64_t value_of(const MachHost& h, int32_t id) { return h.values[(size_t)id]; }

int id_of(const MachHost& h, int64_t v, int32_t* id) {
    const auto it = std::lower_bound(h.values.begin(), h.values.end(), v);
    if (it == h.values.end() || *it != v) {
        set_error("state value " + std::to_string(v) + " is not one of the input's values");
        return MCTB_CONFIG_ERROR;
    }
    *id = (int32_t)(it - h.values.begin());
    return MCTB_OK;
}

void to_flat(const MachHost& h, const MState& s, std::vector<int64_t>& f) {
    const MachDesc& m = h.d;
    f.assign({s.time, s.nrp_work, s.all_nwe, s.fin, s.next_wg, s.host_pc, s.host_k, s.clock});
    f.push_back(m.nwd);
    for (int d = 0; d < m.nwd; ++d) f.insert(f.end(), {s.dev[d].pc, s.dev[d].k, s.dev[d].batch_base});
    f.push_back(m.n_units);
    for (int g = 0; g < m.n_units; ++g) {
        const UnitS& u = s.unit[g];
        f.insert(f.end(), {u.pc, u.k, u.nwg, u.sent, u.got_items, u.got_ends});
    }
    f.push_back(m.n_units);
    for (int g = 0; g < m.n_units; ++g) f.insert(f.end(), {s.bar[g].pc, s.bar[g].count});
    f.push_back(m.n_pex);
    for (int p = 0; p < m.n_pex; ++p) {
        const PexS& x = s.pex[p];
        f.insert(f.end(), {x.pc, x.phase, x.cursor, x.busy_left, x.reported, x.nwg, x.iter});
    }
    if (m.kernel == 1) {
        // glob[1..size) never changes (kernel.cpp:66-80): the input
        f.push_back(m.size);
        f.push_back(value_of(h, s.glob0));
        for (int i = 1; i < m.size; ++i) f.push_back(value_of(h, h.ids[(size_t)i]));
        f.push_back((int64_t)m.n_units * m.np);
        for (int i = 0; i < m.n_units * m.np; ++i) f.push_back(value_of(h, s.loc[i]));
    } else {
        f.push_back(0);
        f.push_back(0);
    }
}

int from_flat(const MachHost& h, const int64_t* f, int64_t n, MState& s) {
    const MachDesc& m = h.d;
    std::memset(&s, 0, sizeof s);
    int64_t i = 0;
    auto get = [&](int64_t& v) {
        if (i >= n) return false;
        v = f[i++];
        return true;
    };
    auto bad = [&]() {
        set_error("state vector does not match this machine's shape");
        return MCTB_CONFIG_ERROR;
    };
    int64_t v[8];
    for (int k = 0; k < 8; ++k)
        if (!get(v[k])) return bad();
    s.time = v[0];
    s.nrp_work = (int32_t)v[1];
    s.all_nwe = (int32_t)v[2];
    s.fin = (int32_t)v[3];
    s.next_wg = (int32_t)v[4];
    s.host_pc = (int32_t)v[5];
    s.host_k = (int32_t)v[6];
    s.clock = (int32_t)v[7];
    int64_t c;
    if (!get(c) || c != m.nwd) return bad();
    for (int d = 0; d < m.nwd; ++d) {
        int64_t a, b, e;
        if (!get(a) || !get(b) || !get(e)) return bad();
        s.dev[d] = DevS{(int32_t)a, (int32_t)b, (int32_t)e};
    }
    if (!get(c) || c != m.n_units) return bad();
    for (int g = 0; g < m.n_units; ++g) {
        int64_t u[6];
        for (int k = 0; k < 6; ++k)
            if (!get(u[k])) return bad();
        s.unit[g] = UnitS{(int32_t)u[0], (int32_t)u[1], (int32_t)u[2], (int32_t)u[3], (int32_t)u[4],
                          (int32_t)u[5]};
    }
    if (!get(c) || c != m.n_units) return bad();
    for (int g = 0; g < m.n_units; ++g) {
        int64_t a, b;
        if (!get(a) || !get(b)) return bad();
        s.bar[g] = BarS{(int32_t)a, (int32_t)b};
    }
    if (!get(c) || c != m.n_pex) return bad();
    for (int p = 0; p < m.n_pex; ++p) {
        int64_t x[7];
        for (int k = 0; k < 7; ++k)
            if (!get(x[k])) return bad();
        PexS& px = s.pex[p];
        px.pc = (int16_t)x[0];
        px.phase = (int16_t)x[1];
        px.cursor = (uint16_t)x[2];
        px.busy_left = (uint16_t)x[3];
        px.reported = (int16_t)x[4];
        px.nwg = (int32_t)x[5];
        px.iter = (uint16_t)x[6];
    }
    int64_t ng, nl;
    if (!get(ng)) return bad();
    if (m.kernel == 1) {
        if (ng != m.size || i + ng > n) return bad();
        int rc = id_of(h, f[i], &s.glob0);
        if (rc) return rc;
        for (int64_t k = 1; k < ng; ++k)
            if (f[i + k] != value_of(h, h.ids[(size_t)k])) {
                set_error("glob[1..size) is the input and never changes (kernel.cpp:66-80)");
                return MCTB_CONFIG_ERROR;
            }
        i += ng;
        if (!get(nl) || nl != (int64_t)m.n_units * m.np || i + nl > n) return bad();
        for (int64_t k = 0; k < nl; ++k)
            if ((rc = id_of(h, f[i + k], &s.loc[k]))) return rc;
        i += nl;
    } else {
        if (ng != 0 || !get(nl) || nl != 0) return bad();
    }
    return i == n ? MCTB_OK : bad();
}

// One machine (the last one asked for on this thread, kept) and its device view.
// Its few device buffers (one state, one enabled list) live as long as the
// thread; they are not freed at exit, when the CUDA runtime may already be gone.
struct Ctx {
    int key[6] = {-1, -1, -1, -1, -1, -1};
    std::vector<int64_t> input;
    MachHost h;
    BfsDesc bd{};
    int32_t* d_ids = nullptr;
    MState* d_state = nullptr;
    Transition* d_tr = nullptr;
    int* d_out = nullptr;
    uint32_t* d_words = nullptr;
    cudaStream_t st = nullptr;
};

int ctx_for(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
            Ctx** out) {
    static thread_local Ctx c;
    const int key[6] = {plat[0], plat[1], plat[2], plat[3], size, kernel * 1000000 + 0};
    std::vector<int64_t> in;
    if (kernel == 1 && input) in.assign(input, input + size);
    if (!(std::memcmp(key, c.key, sizeof key) == 0 && c.h.d.wg == wg && c.h.d.ts == ts &&
          in == c.input && c.d_state)) {
        int rc = check_machine(plat, size, kernel, wg, ts);
        if (rc) return rc;
        if ((rc = require_device())) return rc;
        if (!c.st) MCTB_CUDA(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
        if ((rc = build_desc(plat, size, kernel, input, wg, ts, &c.h))) return rc;
        if (c.d_ids) cudaFreeAsync(c.d_ids, c.st);
        c.d_ids = nullptr;
        if ((rc = upload_desc(c.h, c.st, &c.d_ids))) return rc;
        c.bd.m = c.h.d;
        c.bd.l = bfs_layout(c.h.d, 1);
        if (!c.d_state) {
            MCTB_CUDA(cudaMalloc(&c.d_state, sizeof(MState)));
            MCTB_CUDA(cudaMalloc(&c.d_tr, kMaxEnabled * sizeof(Transition)));
            MCTB_CUDA(cudaMalloc(&c.d_out, 4 * sizeof(int)));
            MCTB_CUDA(cudaMalloc(&c.d_words, kMaxWords * sizeof(uint32_t)));
        }
        std::memcpy(c.key, key, sizeof key);
        c.input = in;
    }
    *out = &c;
    return MCTB_OK;
}

int run_op(Ctx& c, int op, const MState* in, MState* s_out, Transition* tr, int n_tr, int* out,
           uint32_t* words) {
    if (in) MCTB_CUDA(cudaMemcpyAsync(c.d_state, in, sizeof(MState), cudaMemcpyHostToDevice, c.st));
    if (n_tr) MCTB_CUDA(cudaMemcpyAsync(c.d_tr, tr, n_tr * sizeof(Transition), cudaMemcpyHostToDevice, c.st));
    machine_op_kernel<<<1, 1, 0, c.st>>>(c.bd, op, c.d_state, c.d_tr, c.d_out, c.d_words);
    MCTB_CUDA(cudaGetLastError());
    MCTB_CUDA(cudaMemcpyAsync(out, c.d_out, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.st));
    if (s_out) MCTB_CUDA(cudaMemcpyAsync(s_out, c.d_state, sizeof(MState), cudaMemcpyDeviceToHost, c.st));
    if (op == 1 && tr)
        MCTB_CUDA(cudaMemcpyAsync(tr, c.d_tr, kMaxEnabled * sizeof(Transition),
                                  cudaMemcpyDeviceToHost, c.st));
    if (words)
        MCTB_CUDA(cudaMemcpyAsync(words, c.d_words, kMaxWords * 4, cudaMemcpyDeviceToHost, c.st));
    MCTB_CUDA(cudaStreamSynchronize(c.st));
    return MCTB_OK;
}

int emit_flat(const MachHost& h, const MState& s, int64_t* flat, int64_t cap, int64_t* n) {
    std::vector<int64_t> f;
    to_flat(h, s, f);
    *n = (int64_t)f.size();
    if (flat) std::memcpy(flat, f.data(), std::min<int64_t>(cap, *n) * 8);
    if (*n > cap) {
        set_error("state vector buffer too small");
        return MCTB_LIMIT;
    }
    return MCTB_OK;
}

}  // namespace
}  // namespace mctb

using namespace mctb;

extern "C" {

// Machine::initial_state (machine.cpp:116-162)
int mctb_machine_initial(const int* plat, int size, int kernel, const int64_t* input, int wg,
                         int ts, int64_t* flat, int64_t cap, int64_t* n) {
    Ctx* c;
    int rc = ctx_for(plat, size, kernel, input, wg, ts, &c);
    if (rc) return rc;
    MState s;
    int out[4];
    if ((rc = run_op(*c, 0, nullptr, &s, nullptr, 0, out, nullptr))) return rc;
    return emit_flat(c->h, s, flat, cap, n);
}

// Machine::enabled (machine.cpp:174-336): int32[4 * cap] {actor, peer, op, arg}
int mctb_machine_enabled(const int* plat, int size, int kernel, const int64_t* input, int wg,
                         int ts, const int64_t* flat, int64_t n, int32_t* trans, int64_t cap,
                         int64_t* n_trans) {
    Ctx* c;
    int rc = ctx_for(plat, size, kernel, input, wg, ts, &c);
    if (rc) return rc;
    MState s;
    if ((rc = from_flat(c->h, flat, n, s))) return rc;
    std::vector<Transition> tr(kMaxEnabled);
    int out[4];
    if ((rc = run_op(*c, 1, &s, nullptr, tr.data(), 0, out, nullptr))) return rc;
    *n_trans = out[0];
    for (int k = 0; k < out[0] && k < cap; ++k) {
        trans[4 * k] = tr[k].actor;
        trans[4 * k + 1] = tr[k].peer;
        trans[4 * k + 2] = tr[k].op;
        trans[4 * k + 3] = tr[k].arg;
    }
    return MCTB_OK;
}

// Machine::apply (machine.cpp:361-649): MCTB_MODEL_BUG when t is not enabled
int mctb_machine_apply(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                       const int64_t* flat, int64_t n, const int32_t* t, int64_t* out_flat,
                       int64_t cap, int64_t* n_out) {
    Ctx* c;
    int rc = ctx_for(plat, size, kernel, input, wg, ts, &c);
    if (rc) return rc;
    MState s;
    if ((rc = from_flat(c->h, flat, n, s))) return rc;
    Transition tr{(uint16_t)t[0], (uint16_t)t[1], t[2], t[3]};
    int out[4];
    if ((rc = run_op(*c, 2, &s, &s, &tr, 1, out, nullptr))) return rc;
    if (!out[0]) {
        set_error("transition not enabled: actor " + std::to_string(t[0]) + " (" +
                  (t[0] < c->h.d.n_proc ? pname(c->h.d, t[0]) : std::string("?")) + ") op " +
                  std::to_string(t[2]));
        return MCTB_MODEL_BUG;
    }
    return emit_flat(c->h, s, out_flat, cap, n_out);
}

// is_terminal / check_invariants (machine.cpp:708-756) and the canonical packed
// words of the state (the engine's serialization: pack.cuh, every field of
// Machine::serialize, machine.cpp:669-706).  out = {terminal, invariant code (0 ok),
// words}; words = uint32[cap].
int mctb_machine_query(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                       const int64_t* flat, int64_t n, int64_t* out, uint32_t* words,
                       int64_t cap) {
    Ctx* c;
    int rc = ctx_for(plat, size, kernel, input, wg, ts, &c);
    if (rc) return rc;
    MState s;
    if ((rc = from_flat(c->h, flat, n, s))) return rc;
    int o[4];
    std::vector<uint32_t> w(kMaxWords);
    if ((rc = run_op(*c, 3, &s, nullptr, nullptr, 0, o, w.data()))) return rc;
    out[0] = o[0];
    out[1] = o[1];
    out[2] = o[2];
    if (words) std::memcpy(words, w.data(), std::min<int64_t>(cap, o[2]) * 4);
    return MCTB_OK;
}

// Machine::process_name (machine.cpp:103-113): returns the length, copies <= cap-1 + NUL
int64_t mctb_machine_process_name(const int* plat, int size, int kernel, int wg, int ts, int pid,
                                  char* buf, int64_t cap) {
    if (check_machine(plat, size, kernel, wg, ts)) return -1;
    MachHost h;
    if (build_desc(plat, size, kernel, nullptr, wg, ts, &h)) return -1;
    if (pid < 0 || pid >= h.d.n_proc) {
        set_error("pid out of range");
        return -1;
    }
    const std::string s = pname(h.d, pid);
    if (buf && cap > 0) {
        const size_t k = std::min<size_t>(s.size(), (size_t)cap - 1);
        std::memcpy(buf, s.data(), k);
        buf[k] = 0;
    }
    return (int64_t)s.size();
}

// replay (explore.cpp:283-300): the trace from the initial state, in one GPU
// thread; MCTB_CORRUPT_TRACE on a divergence, a non-terminal end or a final time
// other than final_time; the terminal state goes to out_flat.
int mctb_machine_replay(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, const int32_t* trace, int64_t len, int64_t final_time,
                        int64_t* out_flat, int64_t cap, int64_t* n_out) {
    Ctx* c;
    int rc = ctx_for(plat, size, kernel, input, wg, ts, &c);
    if (rc) return rc;
    if (len < 0 || len > 0x7fffffff) {
        set_error("bad trace length");
        return MCTB_CONFIG_ERROR;
    }
    std::vector<Transition> tr((size_t)std::max<int64_t>(len, 1));
    for (int64_t i = 0; i < len; ++i)
        tr[(size_t)i] = Transition{(uint16_t)trace[4 * i], (uint16_t)trace[4 * i + 1],
                                   trace[4 * i + 2], trace[4 * i + 3]};
    Transition* d_tr = nullptr;
    MCTB_CUDA(cudaMallocAsync(&d_tr, tr.size() * sizeof(Transition), c->st));
    int o[4] = {(int)len, 0, 0, 0};
    MState s;
    cudaMemcpyAsync(d_tr, tr.data(), tr.size() * sizeof(Transition), cudaMemcpyHostToDevice, c->st);
    cudaMemcpyAsync(c->d_out, o, sizeof o, cudaMemcpyHostToDevice, c->st);
    machine_op_kernel<<<1, 1, 0, c->st>>>(c->bd, 4, c->d_state, d_tr, c->d_out, c->d_words);
    cudaMemcpyAsync(o, c->d_out, sizeof o, cudaMemcpyDeviceToHost, c->st);
    cudaMemcpyAsync(&s, c->d_state, sizeof(MState), cudaMemcpyDeviceToHost, c->st);
    cudaFreeAsync(d_tr, c->st);
    MCTB_CUDA(cudaStreamSynchronize(c->st));
    MCTB_CUDA(cudaGetLastError());
    if (o[0] < len) {
        set_error("replay diverged at step " + std::to_string(o[0]));
        return MCTB_CORRUPT_TRACE;
    }
    if (!o[1]) {
        set_error("replayed trace does not end terminal");
        return MCTB_CORRUPT_TRACE;
    }
    if (s.time != final_time) {
        set_error("replayed final time " + std::to_string(s.time) + " != recorded " +
                  std::to_string(final_time));
        return MCTB_CORRUPT_TRACE;
    }
    return emit_flat(c->h, s, out_flat, cap, n_out);
}

// explore_machine's visit order (explore.cpp:86-165) for the per-state hooks:
// every state within max_depth in the order the reference's DFS discovers it
// (lexrank.cu), truncated to the first max_states (the visited set's capacity,
// explore.cpp:26-30: once full, no further state is visited).  flat = the
// states' vectors (stride info[2]); meta = int32[8] per state {in-transition
// actor, peer, op, arg (-1 at the root), depth, terminal, enabled count, in-edge
// index}.  info = {states in the full exploration, states returned, stride}.
// MCTB_LIMIT (info filled) when a buffer is too small.
int mctb_machine_states(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, int64_t max_depth, int64_t max_states, int64_t* flat,
                        int64_t flat_cap, int32_t* meta, int64_t meta_cap, int64_t* info) {
    if (max_depth < 1) {
        set_error("max_depth must be >= 1");
        return MCTB_CONFIG_ERROR;
    }
    if (max_states < 1) {
        set_error("max_states must be >= 1");
        return MCTB_CONFIG_ERROR;
    }
    int rc = check_machine(plat, size, kernel, wg, ts);
    if (rc) return rc;
    if ((rc = require_device())) return rc;
    MachHost h;
    if ((rc = build_desc(plat, size, kernel, input, wg, ts, &h))) return rc;
    int words = 0;
    std::vector<uint32_t> packed, depth;
    std::vector<int32_t> mt;
    // the order needs the whole graph: the table grows until it fits
    for (int64_t cap = 1 << 16;; cap *= 16) {
        rc = lexrank_states(h, max_depth, cap, &words, &packed, &mt, &depth);
        if (rc != MCTB_LIMIT || cap >= (int64_t)1 << 24) break;
    }
    if (rc) return rc;
    const int64_t total = (int64_t)depth.size();
    const int64_t n = std::min(total, max_states);
    BfsDesc bd;
    bd.m = h.d;
    bd.l = bfs_layout(h.d, 1);
    std::vector<int64_t> f;
    MState s;
    int64_t stride = 0;
    for (int64_t i = 0; i < n; ++i) {
        std::memset(&s, 0, sizeof s);
        unpack(bd, packed.data() + (size_t)i * words, s);
        to_flat(h, s, f);
        stride = (int64_t)f.size();
        if (flat && (i + 1) * stride <= flat_cap)
            std::memcpy(flat + i * stride, f.data(), (size_t)stride * 8);
        if (meta && i < meta_cap) {
            const int32_t* m = mt.data() + 7 * i;
            int32_t* o = meta + 8 * i;
            o[0] = m[0];
            o[1] = m[1];
            o[2] = m[2];
            o[3] = m[3];
            o[4] = (int32_t)depth[(size_t)i];
            o[5] = m[5];
            o[6] = m[4];
            o[7] = m[6];
        }
    }
    info[0] = total;
    info[1] = n;
    info[2] = stride;
    if (n * stride > flat_cap || n > meta_cap) {
        set_error("state buffers too small");
        return MCTB_LIMIT;
    }
    return MCTB_OK;
}

}  // extern "C"
