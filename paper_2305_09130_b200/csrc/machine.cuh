// Device-side transition system of the mctune model (machine.cpp re-designed
// for the GPU).  One configuration = one MachDesc; a state is an unpacked
// register/local-memory record (MState) that the trajectory kernels step and
// the BFS kernels pack into a few 32-bit words.
//
// Differences in representation from the reference (semantics are identical,
// pinned bit-exactly by tests/test_machine_gpu.py against the oracle and the
// reference's golden traces):
//  * the kernel program (kernel.cpp:26-82) is not materialised: the
//    instruction at a cursor is computed arithmetically (instr_at below);
//  * minimum-kernel memory holds order-preserving value ids (index into the
//    sorted distinct input values, +1 slot for the MAX sentinel), so
//    min-combines (machine.cpp:562-564) compare ids;  glob[1..size) never
//    changes (no effect writes there, kernel.cpp:66-80), only glob[0] is state.
#pragma once

#include <stdint.h>

namespace mctb {

// Op ordinals, machine.hpp:48-68
enum : int {
    OP_CLOCKTICK, OP_CLOCKHALT, OP_HOSTGO, OP_HOSTREACTGO, OP_HOSTSTOP, OP_HOSTSETFIN,
    OP_DEVICEUNITGO, OP_DEVICEDONE, OP_DEVICEUNITSTOP, OP_UNITPEXGO, OP_UNITDONE,
    OP_UNITPEXSTOP, OP_UNITBARRIERSTOP, OP_PEXREPORT, OP_PEXEFFECT, OP_PEXARRIVE,
    OP_PEXITEMDONE, OP_PEXENDDONE, OP_BARRIERRELEASE
};
// control locations, machine.hpp:22-46
enum : int { H_SENDGO, H_WAITDONEREACT, H_REACTGO, H_WAITDONESTOP, H_SENDSTOP, H_SETFIN, H_EXITED };
enum : int { D_WAITGO, D_SENDUNITGO, D_WAITUNITDONE, D_SENDDONE, D_STOPUNITS, D_EXITED };
enum : int { U_WAITGO, U_ACTIVATEPEX, U_SERVE, U_REACTPEX, U_SENDUNITDONE, U_STOPPEXES,
             U_STOPBARRIER, U_EXITED };
enum : int { B_COUNTING, B_EXITED };
enum : int { P_WAITGO, P_RUN, P_ARRIVEBARRIER, P_WAITBARRIER, P_ARRIVEGROUPEND, P_WAITGROUPEND,
             P_SENDITEMDONE, P_SENDENDDONE, P_EXITED };
enum : int { IK_BUSY, IK_BARRIER, IK_EFFECT, IK_END };

constexpr int kMaxDev = 8;
constexpr int kMaxUnit = 16;
constexpr int kMaxPex = 32;
constexpr int kMaxLoc = 256;
constexpr int kMaxEnabled = 2 + kMaxDev + kMaxUnit * 2 + kMaxPex + 4;
constexpr uint16_t kNoPeer = 0xffff;

struct MachDesc {
    int32_t kernel, size, gmt, np, wg, ts, logts;
    int32_t wgs, nwd, nwu, nwe, all_nwe;
    int32_t rounds, device_rounds, host_reacts;
    int32_t n_units, n_pex, n_proc;
    int32_t reps;        // size / ts (abstract)
    int32_t act_len;     // per-activation instruction count
    int32_t epi_len;     // epilogue instruction count
    int32_t max_id;      // value id of the MAX sentinel (minimum kernel)
    int32_t glob0_id;    // initial value id of glob[0]
    // division-free hierarchy arithmetic (set_divisors): nwe is a power of two;
    // the others divide by multiply-high with ceil(2^32 / d) (0 when d == 1)
    int32_t lognwe;
    uint32_t mag_nwu, mag_perdev, mag_ue;  // nwu, 1 + nwu (2 + nwe), 2 + nwe
    const int32_t* input_id;  // device: value id of input[i] (minimum kernel)
};

// x / d for 0 <= x, x * d < 2^32, given mag = ceil(2^32 / d) (0 for d == 1).
__host__ __device__ inline int udiv_mag(int x, int d, uint32_t mag) {
#ifdef __CUDA_ARCH__
    (void)d;
    return mag ? (int)__umulhi((uint32_t)x, mag) : x;
#else
    (void)mag;
    return x / d;
#endif
}

__host__ inline uint32_t div_magic(uint32_t d) {
    return d <= 1 ? 0u : (uint32_t)(((1ull << 32) + d - 1) / d);
}

__host__ inline void set_divisors(MachDesc& m) {
    int l = 0;
    while ((1 << l) < m.nwe) ++l;
    m.lognwe = l;
    m.mag_nwu = div_magic((uint32_t)m.nwu);
    m.mag_perdev = div_magic((uint32_t)(1 + m.nwu * (2 + m.nwe)));
    m.mag_ue = div_magic((uint32_t)(2 + m.nwe));
}

__host__ __device__ inline int div_nwe(const MachDesc& m, int x) { return x >> m.lognwe; }
__host__ __device__ inline int mod_nwe(const MachDesc& m, int x) { return x & (m.nwe - 1); }
__host__ __device__ inline int div_nwu(const MachDesc& m, int x) {
    return udiv_mag(x, m.nwu, m.mag_nwu);
}

struct Transition {
    uint16_t actor, peer;
    int32_t op, arg;
};

struct DevS { int32_t pc, k, batch_base; };
struct UnitS { int32_t pc, k, nwg, sent, got_items, got_ends; };
struct BarS { int32_t pc, count; };
// Per-element record, 16 bytes: the element fields are the bulk of a state and
// the exploration keeps one state per lane, so they are narrow (build_desc
// rejects configurations whose cursor, busy ticks or rounds exceed 16 bits).
struct PexS {
    int16_t pc, phase;
    uint16_t cursor, busy_left;
    int16_t reported;
    uint16_t iter;
    int32_t nwg;
};
__host__ __device__ inline PexS pex_init(int32_t nwg, int iter) {
    PexS p;
    p.pc = 0;
    p.phase = 0;
    p.cursor = 0;
    p.busy_left = 0;
    p.reported = 0;
    p.iter = (uint16_t)iter;
    p.nwg = nwg;
    return p;
}

struct MState {
    int64_t time;
    int32_t nrp_work, all_nwe, fin, next_wg, host_pc, host_k, clock;
    int32_t glob0;
    DevS dev[kMaxDev];
    UnitS unit[kMaxUnit];
    BarS bar[kMaxUnit];
    PexS pex[kMaxPex];
    int32_t loc[kMaxLoc];  // value ids, n_units * np slots (minimum kernel)
};

// ------------------------------------------------------------ hierarchy
__host__ __device__ inline int device_pid(const MachDesc& m, int d) {
    return 3 + d * (1 + m.nwu * (2 + m.nwe));
}
__host__ __device__ inline int unit_pid(const MachDesc& m, int g) {
    const int d = div_nwu(m, g), u = g - d * m.nwu;
    return device_pid(m, d) + 1 + u * (2 + m.nwe);
}
__host__ __device__ inline int barrier_pid(const MachDesc& m, int g) { return unit_pid(m, g) + 1; }
__host__ __device__ inline int pex_pid(const MachDesc& m, int p) {
    const int g = div_nwe(m, p);
    return unit_pid(m, g) + 2 + (p - g * m.nwe);
}

// pid -> (role, ordinal); role: 0 main, 1 host, 2 clock, 3 device, 4 unit, 5 barrier, 6 pex
__host__ __device__ inline void role_of(const MachDesc& m, int pid, int& role, int& ord) {
    if (pid < 3) {
        role = pid;
        ord = -1;
        return;
    }
    const int per_dev = 1 + m.nwu * (2 + m.nwe);
    const int d = udiv_mag(pid - 3, per_dev, m.mag_perdev);
    int r = (pid - 3) - d * per_dev;
    if (r == 0) {
        role = 3;
        ord = d;
        return;
    }
    r -= 1;
    const int u = udiv_mag(r, 2 + m.nwe, m.mag_ue);
    const int q = r - u * (2 + m.nwe);
    const int g = d * m.nwu + u;
    if (q == 0) {
        role = 4;
        ord = g;
    } else if (q == 1) {
        role = 5;
        ord = g;
    } else {
        role = 6;
        ord = g * m.nwe + (q - 2);
    }
}

// ------------------------------------------------------------ program
// build_abstract_kernel (kernel.cpp:26-46): reps x [busy(gmt*ts) G, barrier,
// busy(ts) L, barrier], busy(gmt) G, end.  Epilogue: [end].
// build_minimum_kernel (kernel.cpp:48-82): ts x [effect(loc[me] <- glob[shift+i]),
// busy(gmt)], end.  Epilogue: (nwe-1) x [effect(loc[me] <- loc[me+i]), busy(1)],
// effect(glob[0] <- loc[me]), busy(gmt), end.
struct Instr {
    int kind;
    int32_t ticks;
    int src;  // effect source: activation -> global offset i; epilogue reduce -> slot offset;
              // -1 = publish (glob[0] <- loc[me])
};

__host__ __device__ inline Instr instr_at(const MachDesc& m, int phase, int c) {
    Instr in{IK_END, 0, 0};
    if (m.kernel == 0) {
        if (phase == 0) {
            if (c < 4 * m.reps) {
                const int r = c & 3;
                if (r == 0) in = Instr{IK_BUSY, m.gmt * m.ts, 0};
                else if (r == 2) in = Instr{IK_BUSY, m.ts, 0};
                else in = Instr{IK_BARRIER, 0, 0};
            } else if (c == 4 * m.reps) {
                in = Instr{IK_BUSY, m.gmt, 0};
            }
        }
        return in;
    }
    if (phase == 0) {
        if (c < 2 * m.ts) in = (c & 1) ? Instr{IK_BUSY, m.gmt, 0} : Instr{IK_EFFECT, 0, c >> 1};
        return in;
    }
    const int red = 2 * (m.nwe - 1);
    if (c < red) in = (c & 1) ? Instr{IK_BUSY, 1, 0} : Instr{IK_EFFECT, 0, (c >> 1) + 1};
    else if (c == red) in = Instr{IK_EFFECT, 0, -1};
    else if (c == red + 1) in = Instr{IK_BUSY, m.gmt, 0};
    return in;
}

// has_epilogue (kernel.hpp:84): only the minimum kernel's
__host__ __device__ inline bool has_epilogue(const MachDesc& m) { return m.kernel == 1; }

// ------------------------------------------------------------ state
__host__ __device__ inline void initial_state(const MachDesc& m, MState& s) {
    s.time = 0;
    s.nrp_work = 0;
    s.all_nwe = m.all_nwe;
    s.fin = 0;
    s.next_wg = 0;
    s.host_pc = H_SENDGO;
    s.host_k = 0;
    s.clock = 0;
    s.glob0 = m.glob0_id;
    for (int d = 0; d < m.nwd; ++d) s.dev[d] = DevS{0, 0, 0};
    for (int g = 0; g < m.n_units; ++g) {
        s.unit[g] = UnitS{0, 0, 0, 0, 0, 0};
        s.bar[g] = BarS{0, 0};
    }
    for (int p = 0; p < m.n_pex; ++p) s.pex[p] = pex_init(0, 0);
    if (m.kernel == 1)
        for (int i = 0; i < m.n_units * m.np; ++i) s.loc[i] = m.max_id;
}

// Copies the live part of a state (the arrays are sized for the capacity).
__host__ __device__ inline void copy_state(const MachDesc& m, MState& d, const MState& s) {
    d.time = s.time;
    d.nrp_work = s.nrp_work;
    d.all_nwe = s.all_nwe;
    d.fin = s.fin;
    d.next_wg = s.next_wg;
    d.host_pc = s.host_pc;
    d.host_k = s.host_k;
    d.clock = s.clock;
    d.glob0 = s.glob0;
    for (int i = 0; i < m.nwd; ++i) d.dev[i] = s.dev[i];
    for (int g = 0; g < m.n_units; ++g) {
        d.unit[g] = s.unit[g];
        d.bar[g] = s.bar[g];
    }
    for (int p = 0; p < m.n_pex; ++p) d.pex[p] = s.pex[p];
    if (m.kernel == 1)
        for (int i = 0; i < m.n_units * m.np; ++i) d.loc[i] = s.loc[i];
}

// Machine::place_pex, machine.cpp:136-162
__host__ __device__ inline void place_pex(const MachDesc& m, PexS& px) {
    const Instr in = instr_at(m, px.phase, px.cursor);
    switch (in.kind) {
        case IK_BUSY:
            px.pc = P_RUN;
            px.busy_left = (uint16_t)in.ticks;
            px.reported = 0;
            break;
        case IK_EFFECT:
            px.pc = P_RUN;
            px.busy_left = 0;
            break;
        case IK_BARRIER: px.pc = P_ARRIVEBARRIER; break;
        default:
            if (px.phase == 1) px.pc = P_SENDENDDONE;
            else if (m.kernel == 1 && px.iter == m.rounds - 1) px.pc = P_ARRIVEGROUPEND;
            else px.pc = P_SENDITEMDONE;
    }
}

// Machine::is_terminal, machine.cpp:651-662
// Machine::check_invariants, machine.cpp:719-756: 0 when every structural
// invariant holds, else the number of the violated one (1 nrp_work range,
// 2 all_nwe range, 3 barrier count vs waiting elements, 4 over-counted barrier,
// 5 elements waiting at different barrier instances, 6 unit serving after fin,
// 7 element working after fin).
__host__ __device__ inline int check_invariants(const MachDesc& m, const MState& s) {
    if (s.nrp_work < 0 || s.nrp_work > s.all_nwe) return 1;
    if (s.all_nwe < 0 || s.all_nwe > m.all_nwe) return 2;
    for (int g = 0; g < m.n_units; ++g) {
        int waiting = 0, cursor = -1, phase = 0;
        bool mixed = false;
        for (int e = 0; e < m.nwe; ++e) {
            const PexS& px = s.pex[g * m.nwe + e];
            if (px.pc == P_WAITBARRIER || px.pc == P_WAITGROUPEND) {
                if (waiting == 0) {
                    cursor = px.cursor;
                    phase = px.phase;
                } else if (px.cursor != cursor || px.phase != phase) {
                    mixed = true;
                }
                ++waiting;
            }
        }
        if (s.bar[g].pc == B_COUNTING && s.bar[g].count != waiting) return 3;
        if (s.bar[g].count > m.nwe) return 4;
        if (mixed) return 5;
    }
    if (s.fin) {
        for (int g = 0; g < m.n_units; ++g) {
            const int pc = s.unit[g].pc;
            if (pc != U_WAITGO && pc != U_STOPPEXES && pc != U_STOPBARRIER && pc != U_EXITED)
                return 6;
        }
        for (int p = 0; p < m.n_pex; ++p)
            if (s.pex[p].pc != P_WAITGO && s.pex[p].pc != P_EXITED) return 7;
    }
    return 0;
}

__host__ __device__ inline bool is_terminal(const MachDesc& m, const MState& s) {
    if (!s.fin || s.clock != 1 || s.host_pc != H_EXITED) return false;
    for (int d = 0; d < m.nwd; ++d)
        if (s.dev[d].pc != D_EXITED) return false;
    for (int g = 0; g < m.n_units; ++g)
        if (s.unit[g].pc != U_EXITED || s.bar[g].pc != B_EXITED) return false;
    for (int p = 0; p < m.n_pex; ++p)
        if (s.pex[p].pc != P_EXITED) return false;
    return true;
}

// Machine::enabled, machine.cpp:174-336, split per process: each rule appends
// the transitions whose ACTOR is that process (to out + n, when out != null)
// and returns the new count.  The serial enumeration below visits the
// processes in ascending pid — the reference's stable sort by actor — and the
// exploration visits them warp-parallel (bfs.cu).
#define MCTB_PUSH(A, P, O, G)                                                   \
    do {                                                                        \
        if (out) out[n] = Transition{(uint16_t)(A), (uint16_t)(P), (O), (G)};   \
        ++n;                                                                    \
    } while (0)

__host__ __device__ inline int host_rules(const MachDesc& m, const MState& s, Transition* out,
                                          int n) {
    switch (s.host_pc) {
        case H_SENDGO:
        case H_REACTGO:
        case H_SENDSTOP: {
            const int op = s.host_pc == H_SENDGO ? OP_HOSTGO
                           : s.host_pc == H_REACTGO ? OP_HOSTREACTGO
                                                    : OP_HOSTSTOP;
            for (int d = 0; d < m.nwd; ++d)
                if (s.dev[d].pc == D_WAITGO) MCTB_PUSH(1, device_pid(m, d), op, s.host_k);
            break;
        }
        case H_SETFIN: MCTB_PUSH(1, kNoPeer, OP_HOSTSETFIN, 0); break;
        default: break;
    }
    return n;
}

__host__ __device__ inline int clock_rules(const MachDesc&, const MState& s, Transition* out,
                                           int n) {
    if (s.clock == 0) {
        if (s.fin) MCTB_PUSH(2, kNoPeer, OP_CLOCKHALT, 0);
        if (s.all_nwe != 0 && s.nrp_work == s.all_nwe) MCTB_PUSH(2, kNoPeer, OP_CLOCKTICK, 0);
    }
    return n;
}

__host__ __device__ inline int device_rules(const MachDesc& m, const MState& s, int d,
                                            Transition* out, int n) {
    const DevS& dv = s.dev[d];
    const int dpid = device_pid(m, d);
    if (dv.pc == D_SENDUNITGO || dv.pc == D_STOPUNITS) {
        const int op = dv.pc == D_SENDUNITGO ? OP_DEVICEUNITGO : OP_DEVICEUNITSTOP;
        const int arg = dv.pc == D_SENDUNITGO ? dv.batch_base + dv.k : 0;
        for (int u = 0; u < m.nwu; ++u)
            if (s.unit[d * m.nwu + u].pc == U_WAITGO) MCTB_PUSH(dpid, unit_pid(m, d * m.nwu + u), op, arg);
    } else if (dv.pc == D_SENDDONE) {
        if (s.host_pc == H_WAITDONEREACT || s.host_pc == H_WAITDONESTOP)
            MCTB_PUSH(dpid, 1, OP_DEVICEDONE, 0);
    }
    return n;
}

// (the _at forms take the process ids the serial enumeration already has)
__host__ __device__ inline int unit_rules_at(const MachDesc& m, const MState& s, int g, int upid,
                                             int d, Transition* out, int n) {
    const UnitS& un = s.unit[g];
    switch (un.pc) {
        case U_ACTIVATEPEX:
        case U_REACTPEX:
        case U_STOPPEXES: {
            const int op = un.pc == U_STOPPEXES ? OP_UNITPEXSTOP : OP_UNITPEXGO;
            const int arg = un.pc == U_STOPPEXES ? 0 : div_nwe(m, un.sent);
            for (int e = 0; e < m.nwe; ++e)
                if (s.pex[g * m.nwe + e].pc == P_WAITGO) MCTB_PUSH(upid, upid + 2 + e, op, arg);
            break;
        }
        case U_SENDUNITDONE:
            if (s.dev[d].pc == D_WAITUNITDONE) MCTB_PUSH(upid, device_pid(m, d), OP_UNITDONE, un.nwg);
            break;
        case U_STOPBARRIER:
            if (s.bar[g].pc == B_COUNTING && s.bar[g].count == 0)
                MCTB_PUSH(upid, upid + 1, OP_UNITBARRIERSTOP, 0);
            break;
        default: break;
    }
    return n;
}

__host__ __device__ inline int unit_rules(const MachDesc& m, const MState& s, int g,
                                          Transition* out, int n) {
    return unit_rules_at(m, s, g, unit_pid(m, g), div_nwu(m, g), out, n);
}

__host__ __device__ inline int barrier_rules_at(const MachDesc& m, const MState& s, int g,
                                                int bpid, Transition* out, int n) {
    const BarS& b = s.bar[g];
    if (b.pc == B_COUNTING && b.count == m.nwe) MCTB_PUSH(bpid, kNoPeer, OP_BARRIERRELEASE, 0);
    return n;
}

__host__ __device__ inline int barrier_rules(const MachDesc& m, const MState& s, int g,
                                             Transition* out, int n) {
    return barrier_rules_at(m, s, g, barrier_pid(m, g), out, n);
}

// element p = g * nwe + e of unit g (process ids upid, upid + 2 + e)
__host__ __device__ inline int pex_rules_at(const MachDesc& m, const MState& s, int p, int g,
                                            int upid, int ppid, Transition* out, int n) {
    const PexS& px = s.pex[p];
    switch (px.pc) {
        case P_RUN: {
            const Instr in = instr_at(m, px.phase, px.cursor);
            if (in.kind == IK_BUSY) {
                if (px.busy_left > 0 && !px.reported) MCTB_PUSH(ppid, kNoPeer, OP_PEXREPORT, 0);
            } else if (in.kind == IK_EFFECT) {
                MCTB_PUSH(ppid, kNoPeer, OP_PEXEFFECT, px.cursor);
            }
            break;
        }
        case P_ARRIVEBARRIER:
        case P_ARRIVEGROUPEND:
            if (s.bar[g].pc == B_COUNTING && s.bar[g].count < m.nwe)
                MCTB_PUSH(ppid, upid + 1, OP_PEXARRIVE, 0);
            break;
        case P_SENDITEMDONE:
            if (s.unit[g].pc == U_SERVE) MCTB_PUSH(ppid, upid, OP_PEXITEMDONE, px.iter);
            break;
        case P_SENDENDDONE:
            if (s.unit[g].pc == U_SERVE) MCTB_PUSH(ppid, upid, OP_PEXENDDONE, 0);
            break;
        default: break;
    }
    return n;
}

__host__ __device__ inline int pex_rules(const MachDesc& m, const MState& s, int p,
                                         Transition* out, int n) {
    const int g = div_nwe(m, p);
    const int upid = unit_pid(m, g);
    return pex_rules_at(m, s, p, g, upid, upid + 2 + (p - g * m.nwe), out, n);
}
#undef MCTB_PUSH

// Process slot k of the warp-parallel enumeration: host, clock, devices,
// units, barriers, elements (any order gives the same successor set).
__host__ __device__ inline int slot_rules(const MachDesc& m, const MState& s, int k,
                                          Transition* out, int n) {
    if (k == 0) return host_rules(m, s, out, n);
    if (k == 1) return clock_rules(m, s, out, n);
    k -= 2;
    if (k < m.nwd) return device_rules(m, s, k, out, n);
    k -= m.nwd;
    if (k < m.n_units) return unit_rules(m, s, k, out, n);
    k -= m.n_units;
    if (k < m.n_units) return barrier_rules(m, s, k, out, n);
    k -= m.n_units;
    return pex_rules(m, s, k, out, n);
}

__host__ __device__ inline int n_slots(const MachDesc& m) {
    return 2 + m.nwd + 2 * m.n_units + m.n_pex;
}

// Every enabled transition in ascending actor pid (max_out stops early: the
// first path needs en[0] only).
__host__ __device__ inline int enabled(const MachDesc& m, const MState& s, Transition* out,
                                      int max_out = 1 << 30) {
    int n = host_rules(m, s, out, 0);
    if (n >= max_out) return n;
    n = clock_rules(m, s, out, n);
    if (n >= max_out) return n;
    // process ids advance with the enumeration (device_pid / unit_pid without divisions)
    int g = 0, p = 0, pid = 3;
    for (int d = 0; d < m.nwd; ++d) {
        n = device_rules(m, s, d, out, n);
        if (n >= max_out) return n;
        ++pid;
        for (int u = 0; u < m.nwu; ++u, ++g) {
            const int upid = pid;
            n = unit_rules_at(m, s, g, upid, d, out, n);
            n = barrier_rules_at(m, s, g, upid + 1, out, n);
            if (n >= max_out) return n;
            for (int e = 0; e < m.nwe; ++e, ++p) {
                n = pex_rules_at(m, s, p, g, upid, upid + 2 + e, out, n);
                if (n >= max_out) return n;
            }
            pid += 2 + m.nwe;
        }
    }
    return n;
}

// Machine::apply, machine.cpp:361-649, in place.  Returns false when the
// transition is not enabled (replay divergence) or a model bug is hit.
__host__ __device__ inline bool apply(const MachDesc& m, MState& s, const Transition& t) {
    int role, ord;
    if (t.actor >= m.n_proc) return false;
    role_of(m, t.actor, role, ord);
    int prole = -1, pord = -1;
    if (t.peer != kNoPeer) {
        if (t.peer >= m.n_proc) return false;
        role_of(m, t.peer, prole, pord);
    }
    switch (t.op) {
        case OP_CLOCKTICK: {
            if (role != 2 || s.clock != 0 || s.all_nwe == 0 || s.nrp_work != s.all_nwe) return false;
            s.nrp_work = 0;
            s.time += 1;
            for (int p = 0; p < m.n_pex; ++p) {
                PexS& px = s.pex[p];
                if (!px.reported) continue;
                if (px.pc != P_RUN || px.busy_left <= 0) return false;
                px.reported = 0;
                if (--px.busy_left == 0) {
                    px.cursor += 1;
                    place_pex(m, px);
                }
            }
            return true;
        }
        case OP_CLOCKHALT:
            if (role != 2 || s.clock != 0 || !s.fin) return false;
            s.clock = 1;
            return true;
        case OP_HOSTGO:
        case OP_HOSTREACTGO: {
            const bool react = t.op == OP_HOSTREACTGO;
            if (role != 1 || s.host_pc != (react ? H_REACTGO : H_SENDGO) || prole != 3) return false;
            DevS& dv = s.dev[pord];
            if (dv.pc != D_WAITGO) return false;
            if (s.next_wg + m.nwu > m.wgs) return false;  // workgroup dispatch overflow
            if (react) s.all_nwe += m.nwe * m.nwu;
            dv.batch_base = s.next_wg;
            s.next_wg += m.nwu;
            dv.pc = D_SENDUNITGO;
            dv.k = 0;
            s.host_k += 1;
            if (react) {
                if (s.host_k < m.host_reacts) {
                    s.host_pc = H_WAITDONEREACT;
                } else {
                    s.host_pc = H_WAITDONESTOP;
                    s.host_k = 0;
                }
            } else if (s.host_k == m.nwd) {
                s.host_pc = m.host_reacts > 0 ? H_WAITDONEREACT : H_WAITDONESTOP;
                s.host_k = 0;
            }
            return true;
        }
        case OP_HOSTSTOP: {
            if (role != 1 || s.host_pc != H_SENDSTOP || prole != 3) return false;
            DevS& dv = s.dev[pord];
            if (dv.pc != D_WAITGO) return false;
            dv.pc = D_STOPUNITS;
            dv.k = 0;
            s.host_k += 1;
            s.host_pc = s.host_k == m.nwd ? H_SETFIN : H_WAITDONESTOP;
            return true;
        }
        case OP_HOSTSETFIN:
            if (role != 1 || s.host_pc != H_SETFIN) return false;
            s.fin = 1;
            s.host_pc = H_EXITED;
            return true;
        case OP_DEVICEUNITGO: {
            if (role != 3 || prole != 4) return false;
            DevS& dv = s.dev[ord];
            if (dv.pc != D_SENDUNITGO || div_nwu(m, pord) != ord) return false;
            UnitS& un = s.unit[pord];
            const int nwg = dv.batch_base + dv.k;
            if (un.pc != U_WAITGO || t.arg != nwg) return false;
            un = UnitS{U_ACTIVATEPEX, 0, nwg, 0, 0, 0};
            if (++dv.k == m.nwu) {
                dv.pc = D_WAITUNITDONE;
                dv.k = 0;
            }
            return true;
        }
        case OP_DEVICEDONE: {
            if (role != 3) return false;
            DevS& dv = s.dev[ord];
            if (dv.pc != D_SENDDONE) return false;
            if (s.host_pc != H_WAITDONEREACT && s.host_pc != H_WAITDONESTOP) return false;
            s.host_pc = s.host_pc == H_WAITDONEREACT ? H_REACTGO : H_SENDSTOP;
            dv = DevS{0, 0, 0};
            return true;
        }
        case OP_DEVICEUNITSTOP: {
            if (role != 3 || prole != 4) return false;
            DevS& dv = s.dev[ord];
            if (dv.pc != D_STOPUNITS || div_nwu(m, pord) != ord) return false;
            UnitS& un = s.unit[pord];
            if (un.pc != U_WAITGO) return false;
            un.pc = U_STOPPEXES;
            un.k = 0;
            if (++dv.k == m.nwu) dv.pc = D_EXITED;
            return true;
        }
        case OP_UNITPEXGO: {
            if (role != 4 || prole != 6) return false;
            UnitS& un = s.unit[ord];
            if (un.pc != U_ACTIVATEPEX && un.pc != U_REACTPEX) return false;
            if (div_nwe(m, pord) != ord) return false;
            PexS& px = s.pex[pord];
            const int iter = div_nwe(m, un.sent);
            if (px.pc != P_WAITGO || t.arg != iter) return false;
            px = pex_init(un.nwg, iter);  // start_activation, machine.cpp:164-172
            place_pex(m, px);
            un.sent += 1;
            if (un.pc == U_ACTIVATEPEX) {
                if (++un.k == m.nwe) {
                    un.pc = U_SERVE;
                    un.k = 0;
                }
            } else {
                un.pc = U_SERVE;
            }
            return true;
        }
        case OP_UNITDONE: {
            if (role != 4) return false;
            UnitS& un = s.unit[ord];
            if (un.pc != U_SENDUNITDONE) return false;
            DevS& dv = s.dev[div_nwu(m, ord)];
            if (dv.pc != D_WAITUNITDONE) return false;
            if (m.kernel == 0) s.all_nwe -= m.nwe;
            un = UnitS{0, 0, 0, 0, 0, 0};
            if (++dv.k == m.nwu) {
                dv.pc = D_SENDDONE;
                dv.k = 0;
            }
            return true;
        }
        case OP_UNITPEXSTOP: {
            if (role != 4 || prole != 6) return false;
            UnitS& un = s.unit[ord];
            if (un.pc != U_STOPPEXES || div_nwe(m, pord) != ord) return false;
            PexS& px = s.pex[pord];
            if (px.pc != P_WAITGO) return false;
            px.pc = P_EXITED;
            if (++un.k == m.nwe) un.pc = U_STOPBARRIER;
            return true;
        }
        case OP_UNITBARRIERSTOP: {
            if (role != 4) return false;
            UnitS& un = s.unit[ord];
            BarS& b = s.bar[ord];
            if (un.pc != U_STOPBARRIER || b.pc != B_COUNTING || b.count != 0) return false;
            b.pc = B_EXITED;
            un.pc = U_EXITED;
            return true;
        }
        case OP_PEXREPORT: {
            if (role != 6) return false;
            PexS& px = s.pex[ord];
            if (px.pc != P_RUN) return false;
            const Instr in = instr_at(m, px.phase, px.cursor);
            if (in.kind != IK_BUSY || px.busy_left <= 0 || px.reported) return false;
            px.reported = 1;
            s.nrp_work += 1;
            return true;
        }
        case OP_PEXEFFECT: {
            if (role != 6) return false;
            PexS& px = s.pex[ord];
            if (px.pc != P_RUN) return false;
            const Instr in = instr_at(m, px.phase, px.cursor);
            if (in.kind != IK_EFFECT || t.arg != px.cursor) return false;
            const int g = div_nwe(m, ord), me = ord - g * m.nwe;
            const int slot = g * m.np + me;  // myloc, machine.hpp:208
            int32_t v;
            int32_t* dst;
            if (px.phase == 0) {
                // glob[shift + i] -> loc[myloc]; global_item_id, kernel.hpp:93-95
                const int gid = m.wg > m.np ? px.nwg * m.wg + me + px.iter * m.np
                                            : px.nwg * m.wg + me;
                const int idx = gid * m.ts + in.src;
                if (idx < 0 || idx >= m.size) return false;  // memory read out of range
                v = idx == 0 ? s.glob0 : m.input_id[idx];
                dst = &s.loc[slot];
            } else if (in.src > 0) {
                if (slot + in.src >= m.n_units * m.np) return false;
                v = s.loc[slot + in.src];
                dst = &s.loc[slot];
            } else {
                v = s.loc[slot];
                dst = &s.glob0;
            }
            if (v < *dst) *dst = v;
            px.cursor += 1;
            place_pex(m, px);
            return true;
        }
        case OP_PEXARRIVE: {
            if (role != 6) return false;
            PexS& px = s.pex[ord];
            if (px.pc != P_ARRIVEBARRIER && px.pc != P_ARRIVEGROUPEND) return false;
            BarS& b = s.bar[div_nwe(m, ord)];
            if (b.pc != B_COUNTING || b.count >= m.nwe) return false;
            b.count += 1;
            px.pc = px.pc == P_ARRIVEBARRIER ? P_WAITBARRIER : P_WAITGROUPEND;
            return true;
        }
        case OP_BARRIERRELEASE: {
            if (role != 5) return false;
            BarS& b = s.bar[ord];
            if (b.pc != B_COUNTING || b.count != m.nwe) return false;
            int wk = 0, wg_ = 0;
            for (int e = 0; e < m.nwe; ++e) {
                const int pc = s.pex[ord * m.nwe + e].pc;
                wk += pc == P_WAITBARRIER;
                wg_ += pc == P_WAITGROUPEND;
            }
            if (wk != m.nwe && wg_ != m.nwe) return false;
            b.count = 0;
            if (wk == m.nwe) {
                for (int e = 0; e < m.nwe; ++e) {
                    PexS& px = s.pex[ord * m.nwe + e];
                    px.cursor += 1;
                    place_pex(m, px);
                }
            } else {
                s.all_nwe -= m.nwe - 1;
                for (int e = 0; e < m.nwe; ++e) {
                    PexS& px = s.pex[ord * m.nwe + e];
                    if (e == 0 && has_epilogue(m)) {
                        px.phase = 1;
                        px.cursor = 0;
                        place_pex(m, px);
                    } else {
                        px.pc = P_SENDENDDONE;
                    }
                }
            }
            return true;
        }
        case OP_PEXITEMDONE: {
            if (role != 6) return false;
            PexS& px = s.pex[ord];
            if (px.pc != P_SENDITEMDONE) return false;
            UnitS& un = s.unit[div_nwe(m, ord)];
            if (un.pc != U_SERVE) return false;
            un.got_items += 1;
            px = pex_init(0, 0);
            if (un.sent < m.wg) un.pc = U_REACTPEX;
            else if (m.kernel == 0 && un.got_items == m.wg) un.pc = U_SENDUNITDONE;
            return true;
        }
        case OP_PEXENDDONE: {
            if (role != 6) return false;
            PexS& px = s.pex[ord];
            if (px.pc != P_SENDENDDONE) return false;
            UnitS& un = s.unit[div_nwe(m, ord)];
            if (un.pc != U_SERVE) return false;
            un.got_ends += 1;
            if (mod_nwe(m, ord) == 0) s.all_nwe -= 1;
            px = pex_init(0, 0);
            if (un.got_ends == m.nwe) un.pc = U_SENDUNITDONE;
            return true;
        }
        default: return false;
    }
}

}  // namespace mctb
