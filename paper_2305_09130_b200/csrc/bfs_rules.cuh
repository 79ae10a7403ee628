// Exploration-side views of the transition system (bfs.cu): a table-driven
// warp-parallel unpack, a per-process enumeration of the enabled set in which
// every lane emits at most two transitions, and the linear state hash that
// in-place successors update word by word.
//
// The enumeration yields exactly the set of Machine::enabled
// (machine.cpp:174-336, machine.cuh host/clock/device/unit/barrier/pex_rules)
// but in a different order: a handshake is emitted by the process it is
// offered TO (host -> device, device -> unit, unit -> element), so no lane loops
// over its peers.  The exploration's counts do not depend on the order
// (states, transitions, terminal times are set properties); the paths that do
// (first DFS path, lexfirst walk, trajectories) keep using enabled().
//
// Transitions in the exploration's enabled list name processes by ORDINAL
// within their role (to_pid() gives the pid form that apply() takes):
//   clock ops (0, -)        host ops (0, device d)     DEVICEDONE (d, 0)
//   DEVICEUNIT* (d, unit g) UNITDONE (g, d)            UNITBARRIERSTOP (g, g)
//   BARRIERRELEASE (g, -)   UNITPEX* (g, element p)    PEXREPORT/EFFECT (p, -)
//   PEXARRIVE (p, g)        PEXITEMDONE/ENDDONE (p, g)
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "machine.cuh"
#include "pack.cuh"

namespace mctb {

// one entry per packed field: {word i (5 bits) | shift sh (5) | 31 - sh (5) |
// byte offset in MState (13, from bit 16) | store size (bit 29: 0 = 16-bit,
// 1 = 32-bit), value mask}
constexpr int kMaxFields = 10 + 3 * kMaxDev + 8 * kMaxUnit + 7 * kMaxPex + kMaxLoc;

__host__ __device__ inline uint2 field_entry(int off, int width, size_t dst, int sz) {
    const int i = off / kWordBits, sh = off % kWordBits;
    uint2 e;
    e.x = (uint32_t)i | ((uint32_t)sh << 5) | ((uint32_t)(kWordBits - sh) << 10) |
          ((uint32_t)dst << 16) | ((uint32_t)sz << 29);
    e.y = (uint32_t)((1ull << width) - 1);
    return e;
}

// The field table of a layout, in pack() order (pack.cuh).  Returns the count.
__host__ inline int build_field_table(const MachDesc& m, const Layout& l, uint2* out) {
    int n = 0, off = l.cfg;
    auto add = [&](int width, size_t dst, int sz) {
        out[n++] = field_entry(off, width, dst, sz);
        off += width;
    };
    add(l.time, offsetof(MState, time), 1);  // low word; l.time <= 32 (run_bfs)
    add(l.nrp, offsetof(MState, nrp_work), 1);
    add(l.allnwe, offsetof(MState, all_nwe), 1);
    add(1, offsetof(MState, fin), 1);
    add(l.nextwg, offsetof(MState, next_wg), 1);
    add(3, offsetof(MState, host_pc), 1);
    add(l.hostk, offsetof(MState, host_k), 1);
    add(1, offsetof(MState, clock), 1);
    add(l.glob0, offsetof(MState, glob0), 1);
    for (int i = 0; i < m.nwd; ++i) {
        const size_t b = offsetof(MState, dev) + i * sizeof(DevS);
        add(3, b + offsetof(DevS, pc), 1);
        add(l.dk, b + offsetof(DevS, k), 1);
        add(l.bb, b + offsetof(DevS, batch_base), 1);
    }
    for (int g = 0; g < m.n_units; ++g) {
        const size_t b = offsetof(MState, unit) + g * sizeof(UnitS);
        const size_t bb = offsetof(MState, bar) + g * sizeof(BarS);
        add(3, b + offsetof(UnitS, pc), 1);
        add(l.uk, b + offsetof(UnitS, k), 1);
        add(l.nwg, b + offsetof(UnitS, nwg), 1);
        add(l.sent, b + offsetof(UnitS, sent), 1);
        add(l.items, b + offsetof(UnitS, got_items), 1);
        add(l.ends, b + offsetof(UnitS, got_ends), 1);
        add(1, bb + offsetof(BarS, pc), 1);
        add(l.bcount, bb + offsetof(BarS, count), 1);
    }
    for (int p = 0; p < m.n_pex; ++p) {
        const size_t b = offsetof(MState, pex) + p * sizeof(PexS);
        add(4, b + offsetof(PexS, pc), 0);
        add(1, b + offsetof(PexS, phase), 0);
        add(l.cursor, b + offsetof(PexS, cursor), 0);
        add(l.busy, b + offsetof(PexS, busy_left), 0);
        add(1, b + offsetof(PexS, reported), 0);
        add(l.pnwg, b + offsetof(PexS, nwg), 1);
        add(l.iter, b + offsetof(PexS, iter), 0);
    }
    if (m.kernel == 1)
        for (int i = 0; i < m.n_units * m.np; ++i) add(l.loc, offsetof(MState, loc) + 4 * i, 1);
    return n;
}

// Warp-parallel unpack: lane f extracts fields f, f+32, ... into the shared
// MState (the caller syncs the warp).  `in` holds >= words+1 readable words.
// The time field is written as the low word of MState::time: the caller keeps
// the high word zero.  A field's bits are the data bits [sh, 31) of word i
// followed by the low bits of word i+1 (pack.cuh: 31 data bits per word).
__host__ __device__ inline void unpack_fields(const uint2* __restrict__ ftab, int nf,
                                              const uint32_t* in, MState& s, int lane,
                                              int lanes = 32) {
    char* base = reinterpret_cast<char*>(&s);
    for (int f = lane; f < nf; f += lanes) {
#ifdef __CUDA_ARCH__
        const uint2 e = __ldg(ftab + f);
#else
        const uint2 e = ftab[f];
#endif
        const int i = e.x & 31, sh = (e.x >> 5) & 31, rsh = (e.x >> 10) & 31;
        const uint32_t v = (((in[i] & kData) >> sh) | (in[i + 1] << rsh)) & e.y;
        const uint32_t dst = (e.x >> 16) & 0x1fff;
        if (e.x & (1u << 29)) *reinterpret_cast<uint32_t*>(base + dst) = v;
        else *reinterpret_cast<uint16_t*>(base + dst) = (uint16_t)v;
    }
}

// Process slot k (host, clock, devices, units, barriers, elements): its own
// transitions plus the handshake offered to it.  Writes <= 2 to o.
__host__ __device__ inline int bfs_slot_rules(const MachDesc& m, const MState& s, int k,
                                              int lognwe, Transition* o) {
    int n = 0;
    if (k == 0) {
        if (s.host_pc == H_SETFIN) o[n++] = Transition{0, kNoPeer, OP_HOSTSETFIN, 0};
        return n;
    }
    if (k == 1) {
        if (s.clock == 0) {
            if (s.fin) o[n++] = Transition{0, kNoPeer, OP_CLOCKHALT, 0};
            if (s.all_nwe != 0 && s.nrp_work == s.all_nwe)
                o[n++] = Transition{0, kNoPeer, OP_CLOCKTICK, 0};
        }
        return n;
    }
    k -= 2;
    if (k < m.nwd) {
        const int d = k;
        const DevS& dv = s.dev[d];
        // host_rules: offered by the host to every waiting device
        if (dv.pc == D_WAITGO &&
            (s.host_pc == H_SENDGO || s.host_pc == H_REACTGO || s.host_pc == H_SENDSTOP)) {
            const int op = s.host_pc == H_SENDGO ? OP_HOSTGO
                           : s.host_pc == H_REACTGO ? OP_HOSTREACTGO
                                                    : OP_HOSTSTOP;
            o[n++] = Transition{0, (uint16_t)d, op, s.host_k};
        }
        if (dv.pc == D_SENDDONE && (s.host_pc == H_WAITDONEREACT || s.host_pc == H_WAITDONESTOP))
            o[n++] = Transition{(uint16_t)d, 0, OP_DEVICEDONE, 0};
        return n;
    }
    k -= m.nwd;
    if (k < m.n_units) {
        const int g = k, d = m.nwd == 1 ? 0 : div_nwu(m, g);
        const UnitS& un = s.unit[g];
        const DevS& dv = s.dev[d];
        // device_rules: offered by the unit's device
        if (un.pc == U_WAITGO && (dv.pc == D_SENDUNITGO || dv.pc == D_STOPUNITS)) {
            const bool go = dv.pc == D_SENDUNITGO;
            o[n++] = Transition{(uint16_t)d, (uint16_t)g, go ? OP_DEVICEUNITGO : OP_DEVICEUNITSTOP,
                                go ? dv.batch_base + dv.k : 0};
        }
        if (un.pc == U_SENDUNITDONE) {
            if (dv.pc == D_WAITUNITDONE)
                o[n++] = Transition{(uint16_t)g, (uint16_t)d, OP_UNITDONE, un.nwg};
        } else if (un.pc == U_STOPBARRIER) {
            if (s.bar[g].pc == B_COUNTING && s.bar[g].count == 0)
                o[n++] = Transition{(uint16_t)g, (uint16_t)g, OP_UNITBARRIERSTOP, 0};
        }
        return n;
    }
    k -= m.n_units;
    if (k < m.n_units) {
        const BarS& b = s.bar[k];
        if (b.pc == B_COUNTING && b.count == m.nwe)
            o[n++] = Transition{(uint16_t)k, kNoPeer, OP_BARRIERRELEASE, 0};
        return n;
    }
    k -= m.n_units;
    const int p = k, g = p >> lognwe;  // nwe = min(wg, np) is a power of two
    const PexS& px = s.pex[p];
    const UnitS& un = s.unit[g];
    // unit_rules: offered by the element's unit
    if (px.pc == P_WAITGO &&
        (un.pc == U_ACTIVATEPEX || un.pc == U_REACTPEX || un.pc == U_STOPPEXES)) {
        const bool stop = un.pc == U_STOPPEXES;
        o[n++] = Transition{(uint16_t)g, (uint16_t)p, stop ? OP_UNITPEXSTOP : OP_UNITPEXGO,
                            stop ? 0 : un.sent >> lognwe};
    }
    // pex_rules
    switch (px.pc) {
        case P_RUN: {
            const Instr in = instr_at(m, px.phase, px.cursor);
            if (in.kind == IK_BUSY) {
                if (px.busy_left > 0 && !px.reported)
                    o[n++] = Transition{(uint16_t)p, kNoPeer, OP_PEXREPORT, 0};
            } else if (in.kind == IK_EFFECT) {
                o[n++] = Transition{(uint16_t)p, kNoPeer, OP_PEXEFFECT, px.cursor};
            }
            break;
        }
        case P_ARRIVEBARRIER:
        case P_ARRIVEGROUPEND:
            if (s.bar[g].pc == B_COUNTING && s.bar[g].count < m.nwe)
                o[n++] = Transition{(uint16_t)p, (uint16_t)g, OP_PEXARRIVE, 0};
            break;
        case P_SENDITEMDONE:
            if (un.pc == U_SERVE) o[n++] = Transition{(uint16_t)p, (uint16_t)g, OP_PEXITEMDONE, px.iter};
            break;
        case P_SENDENDDONE:
            if (un.pc == U_SERVE) o[n++] = Transition{(uint16_t)p, (uint16_t)g, OP_PEXENDDONE, 0};
            break;
        default: break;
    }
    return n;
}

// Ordinal form -> the pid form of machine.hpp:76-84 (what apply() takes).
__host__ __device__ inline Transition to_pid(const MachDesc& m, const Transition& t) {
    Transition r{0, kNoPeer, t.op, t.arg};
    const int a = t.actor, p = t.peer;
    switch (t.op) {
        case OP_CLOCKTICK:
        case OP_CLOCKHALT: r.actor = 2; break;
        case OP_HOSTGO:
        case OP_HOSTREACTGO:
        case OP_HOSTSTOP:
            r.actor = 1;
            r.peer = (uint16_t)device_pid(m, p);
            break;
        case OP_HOSTSETFIN: r.actor = 1; break;
        case OP_DEVICEDONE:
            r.actor = (uint16_t)device_pid(m, a);
            r.peer = 1;
            break;
        case OP_DEVICEUNITGO:
        case OP_DEVICEUNITSTOP:
            r.actor = (uint16_t)device_pid(m, a);
            r.peer = (uint16_t)unit_pid(m, p);
            break;
        case OP_UNITDONE:
            r.actor = (uint16_t)unit_pid(m, a);
            r.peer = (uint16_t)device_pid(m, p);
            break;
        case OP_UNITBARRIERSTOP:
            r.actor = (uint16_t)unit_pid(m, a);
            r.peer = (uint16_t)barrier_pid(m, p);
            break;
        case OP_UNITPEXGO:
        case OP_UNITPEXSTOP:
            r.actor = (uint16_t)unit_pid(m, a);
            r.peer = (uint16_t)pex_pid(m, p);
            break;
        case OP_BARRIERRELEASE: r.actor = (uint16_t)barrier_pid(m, a); break;
        case OP_PEXREPORT:
        case OP_PEXEFFECT: r.actor = (uint16_t)pex_pid(m, a); break;
        case OP_PEXARRIVE:
            r.actor = (uint16_t)pex_pid(m, a);
            r.peer = (uint16_t)barrier_pid(m, p);
            break;
        case OP_PEXITEMDONE:
        case OP_PEXENDDONE:
            r.actor = (uint16_t)pex_pid(m, a);
            r.peer = (uint16_t)unit_pid(m, p);
            break;
        default: break;
    }
    return r;
}

// ------------------------------------------------------------------ hashing
// H(key) = sum_i w_i * K_i (mod 2^64) over the key words, K_i odd and random;
// an in-place successor updates H by (new - old) * K_i for each word it
// rewrites.  The table slot and fingerprint come from fmix64(H).  (Equal H for
// different keys only costs a probe: the table compares full keys.)
__host__ __device__ inline uint64_t fmix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

__host__ __device__ inline uint64_t hash_coef(int i) {
    return fmix64(0x9E3779B97F4A7C15ull * (uint64_t)(i + 1)) | 1ull;
}

__host__ __device__ inline uint64_t hash_full(const uint32_t* w, int n) {
    uint64_t h = 0;
    for (int i = 0; i < n; ++i) h += (uint64_t)w[i] * hash_coef(i);
    return h;
}

// set_bits (pack.cuh) of a field up to 62 bits wide (at most three words) that
// also updates the linear hash H (coefficients k).
__host__ __device__ inline void set_bits_h(uint32_t* w, int off, int width, uint64_t v,
                                           const uint64_t* k, uint64_t& H) {
    int i = div31(off), b = off - i * kWordBits;
    while (width > 0) {
        const int take = kWordBits - b < width ? kWordBits - b : width;
        const uint32_t mask = ((1u << take) - 1u) << b;
        const uint32_t o = w[i];
        const uint32_t n = (o & ~mask) | (((uint32_t)v << b) & mask);
        w[i] = n;
        H += ((uint64_t)n - (uint64_t)o) * k[i];
        v >>= take;
        width -= take;
        b = 0;
        ++i;
    }
}

// ------------------------------------------------------------------ in-place successors
// Record writers for the in-place successors (field order of pack()): the
// record is composed in a register and written with one multi-word set (every
// rewritten word also updates the state hash H); records wider than 62 bits
// are written field by field.
__host__ __device__ inline void write_pex(uint32_t* row, const Layout& l, int p, const PexS& x,
                                          const uint64_t* hk, uint64_t& H) {
    const int o = l.off_pex + p * l.pex_bits;
    const int s1 = 5 + l.cursor, s2 = s1 + l.busy, s3 = s2 + 1, s4 = s3 + l.pnwg;
    if (l.pex_bits <= 62) {
        const uint64_t v = (uint64_t)x.pc | ((uint64_t)x.phase << 4) | ((uint64_t)x.cursor << 5) |
                           ((uint64_t)x.busy_left << s1) | ((uint64_t)x.reported << s2) |
                           ((uint64_t)(uint32_t)x.nwg << s3) | ((uint64_t)x.iter << s4);
        set_bits_h(row, o, l.pex_bits, v, hk, H);
        return;
    }
    set_bits_h(row, o, 4, (uint32_t)x.pc, hk, H);
    set_bits_h(row, o + 4, 1, (uint32_t)x.phase, hk, H);
    set_bits_h(row, o + 5, l.cursor, x.cursor, hk, H);
    set_bits_h(row, o + s1, l.busy, x.busy_left, hk, H);
    set_bits_h(row, o + s2, 1, (uint32_t)x.reported, hk, H);
    set_bits_h(row, o + s3, l.pnwg, (uint32_t)x.nwg, hk, H);
    set_bits_h(row, o + s4, l.iter, x.iter, hk, H);
}

// The unit's own fields (not its barrier's, which follow them in the record).
__host__ __device__ inline void write_unit(uint32_t* row, const Layout& l, int g, const UnitS& u,
                                           const uint64_t* hk, uint64_t& H) {
    const int o = l.off_units + g * l.unit_bits;
    const int s1 = 3 + l.uk, s2 = s1 + l.nwg, s3 = s2 + l.sent, s4 = s3 + l.items;
    const int width = s4 + l.ends;
    if (width <= 62) {
        const uint64_t v = (uint64_t)(uint32_t)u.pc | ((uint64_t)(uint32_t)u.k << 3) |
                           ((uint64_t)(uint32_t)u.nwg << s1) | ((uint64_t)(uint32_t)u.sent << s2) |
                           ((uint64_t)(uint32_t)u.got_items << s3) |
                           ((uint64_t)(uint32_t)u.got_ends << s4);
        set_bits_h(row, o, width, v, hk, H);
        return;
    }
    set_bits_h(row, o, 3, (uint32_t)u.pc, hk, H);
    set_bits_h(row, o + 3, l.uk, (uint32_t)u.k, hk, H);
    set_bits_h(row, o + s1, l.nwg, (uint32_t)u.nwg, hk, H);
    set_bits_h(row, o + s2, l.sent, (uint32_t)u.sent, hk, H);
    set_bits_h(row, o + s3, l.items, (uint32_t)u.got_items, hk, H);
    set_bits_h(row, o + s4, l.ends, (uint32_t)u.got_ends, hk, H);
}

// In-place successors for the transitions behind the combinatorial state
// explosion: an element reporting a busy tick or arriving at its barrier, the
// unit <-> element handshakes (activation, item done, group done, stop), the
// clock tick and the barrier release (one record per element concerned: the
// chain steps of deep graphs).
// They touch one element record, its unit record and at most one header field;
// the new values follow Machine::apply (machine.cpp:479-500, 518-530, 541-551,
// 569-580, 618-646) and are written over the parent's packed words.  `tr` is in
// the ordinal form of bfs_rules.cuh.  Every other transition goes through the
// generic unpacked apply() (machine.cuh).
__host__ __device__ inline bool fast_successor(const BfsDesc& d, const MState& s,
                                               const Transition& tr, uint32_t* row,
                                               const uint64_t* hk, uint64_t& H) {
    const Layout& l = d.l;
    const MachDesc& m = d.m;
    switch (tr.op) {
        case OP_CLOCKTICK: {
            // machine.cpp ClockTick (machine.cuh apply): time + 1, nrp_work = 0, and
            // every reported element un-reports and burns one busy tick, advancing
            // its cursor when the tick was its last (the enumeration only offers
            // the tick when nrp_work == all_nwe, i.e. every busy element reported)
            set_bits_h(row, l.cfg, l.time, (uint32_t)(s.time + 1), hk, H);
            set_bits_h(row, l.off_nrp, l.nrp, 0u, hk, H);
            for (int p = 0; p < m.n_pex; ++p) {
                if (!s.pex[p].reported) continue;
                PexS px = s.pex[p];
                px.reported = 0;
                if (--px.busy_left == 0) {
                    px.cursor += 1;
                    place_pex(m, px);
                }
                write_pex(row, l, p, px, hk, H);
            }
            return true;
        }
        case OP_BARRIERRELEASE: {
            // machine.cpp BarrierRelease (machine.cuh apply): the count resets; a
            // barrier releases its elements to their next instruction, a group end
            // sends them to SENDENDDONE (element 0 of the minimum kernel starts the
            // epilogue) and retires nwe - 1 of the working elements
            const int g = tr.actor, p0 = g * m.nwe;
            int wk = 0, wge = 0;
            for (int e = 0; e < m.nwe; ++e) {
                wk += s.pex[p0 + e].pc == P_WAITBARRIER;
                wge += s.pex[p0 + e].pc == P_WAITGROUPEND;
            }
            if (wk != m.nwe && wge != m.nwe) return false;  // apply() reports the bug
            set_bits_h(row, l.off_units + g * l.unit_bits + l.uoff_bcount, l.bcount, 0u, hk, H);
            if (wge == m.nwe)
                set_bits_h(row, l.off_nrp + l.nrp, l.allnwe, (uint32_t)(s.all_nwe - (m.nwe - 1)),
                           hk, H);
            for (int e = 0; e < m.nwe; ++e) {
                PexS px = s.pex[p0 + e];
                if (wk == m.nwe) {
                    px.cursor += 1;
                    place_pex(m, px);
                } else if (e == 0 && has_epilogue(m)) {
                    px.phase = 1;
                    px.cursor = 0;
                    place_pex(m, px);
                } else {
                    px.pc = P_SENDENDDONE;
                }
                write_pex(row, l, p0 + e, px, hk, H);
            }
            return true;
        }
        case OP_PEXEFFECT: {
            // machine.cpp PexEffect (machine.cuh apply), minimum kernel: min-combine a
            // global item, a neighbour's slot, or (publish) the element's slot into
            // glob[0]; then the next instruction
            const int p = tr.actor, g = p >> m.lognwe, me = p - g * m.nwe;
            const int slot = g * m.np + me;  // myloc, machine.hpp:208
            PexS px = s.pex[p];
            const Instr in = instr_at(m, px.phase, px.cursor);
            int32_t v, cur;
            int off, width;
            const int off_glob0 = l.cfg + l.time + l.nrp + l.allnwe + 1 + l.nextwg + 3 + l.hostk + 1;
            if (px.phase == 0) {
                const int gid = m.wg > m.np ? px.nwg * m.wg + me + px.iter * m.np : px.nwg * m.wg + me;
                const int idx = gid * m.ts + in.src;
                if (idx < 0 || idx >= m.size) return false;  // apply() reports the bug
                v = idx == 0 ? s.glob0 : m.input_id[idx];
                cur = s.loc[slot];
                off = l.off_loc + slot * l.loc;
                width = l.loc;
            } else if (in.src > 0) {
                if (slot + in.src >= m.n_units * m.np) return false;
                v = s.loc[slot + in.src];
                cur = s.loc[slot];
                off = l.off_loc + slot * l.loc;
                width = l.loc;
            } else {
                v = s.loc[slot];
                cur = s.glob0;
                off = off_glob0;
                width = l.glob0;
            }
            if (v < cur) set_bits_h(row, off, width, (uint32_t)v, hk, H);
            px.cursor += 1;
            place_pex(m, px);
            write_pex(row, l, p, px, hk, H);
            return true;
        }
        case OP_PEXREPORT: {
            const int off = l.off_pex + tr.actor * l.pex_bits + l.poff_reported;
            const int i = div31(off);
            const uint32_t bit = 1u << (off - i * kWordBits);  // reported was 0
            row[i] |= bit;
            H += (uint64_t)bit * hk[i];
            set_bits_h(row, l.off_nrp, l.nrp, (uint32_t)(s.nrp_work + 1), hk, H);
            return true;
        }
        case OP_PEXARRIVE: {
            const int p = tr.actor, g = tr.peer;
            const int pc = s.pex[p].pc == P_ARRIVEBARRIER ? P_WAITBARRIER : P_WAITGROUPEND;
            set_bits_h(row, l.off_pex + p * l.pex_bits, 4, (uint32_t)pc, hk, H);
            set_bits_h(row, l.off_units + g * l.unit_bits + l.uoff_bcount, l.bcount,
                       (uint32_t)(s.bar[g].count + 1), hk, H);
            return true;
        }
        case OP_UNITPEXGO: {
            const int g = tr.actor, p = tr.peer;
            UnitS un = s.unit[g];
            PexS px = pex_init(un.nwg, tr.arg);  // arg = sent / nwe
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
            write_pex(row, l, p, px, hk, H);
            write_unit(row, l, g, un, hk, H);
            return true;
        }
        case OP_UNITPEXSTOP: {
            const int g = tr.actor, p = tr.peer;
            UnitS un = s.unit[g];
            if (++un.k == m.nwe) un.pc = U_STOPBARRIER;
            set_bits_h(row, l.off_pex + p * l.pex_bits, 4, (uint32_t)P_EXITED, hk, H);
            write_unit(row, l, g, un, hk, H);
            return true;
        }
        case OP_PEXITEMDONE: {
            const int p = tr.actor, g = tr.peer;
            UnitS un = s.unit[g];
            un.got_items += 1;
            if (un.sent < m.wg) un.pc = U_REACTPEX;
            else if (m.kernel == 0 && un.got_items == m.wg) un.pc = U_SENDUNITDONE;
            write_pex(row, l, p, pex_init(0, 0), hk, H);
            write_unit(row, l, g, un, hk, H);
            return true;
        }
        case OP_PEXENDDONE: {
            const int p = tr.actor, g = tr.peer;
            UnitS un = s.unit[g];
            un.got_ends += 1;
            if (un.got_ends == m.nwe) un.pc = U_SENDUNITDONE;
            if ((p & (m.nwe - 1)) == 0)
                set_bits_h(row, l.off_nrp + l.nrp, l.allnwe, (uint32_t)(s.all_nwe - 1), hk, H);
            write_pex(row, l, p, pex_init(0, 0), hk, H);
            write_unit(row, l, g, un, hk, H);
            return true;
        }
        default: return false;
    }
}

}  // namespace mctb
