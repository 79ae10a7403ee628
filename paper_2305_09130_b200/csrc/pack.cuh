// Bit-packed state encoding for the interleaving exploration (bfs.cu).
//
// The reference keys its exact visited set on the canonical byte
// serialization of every state field (machine.cpp:669-706, explore.cpp:21-44).
// We key ours on an injective bit packing of the same fields: each field gets
// the width of its reachable range for this configuration (computed on the
// host from the launch plan), so a state of a desk-scale configuration fits in
// a handful of 32-bit words and one hash-table probe moves one 64-byte line.
// Two states of one configuration are equal iff their packings are equal,
// which is what makes the GPU state counts equal the reference's.
//
// Every packed word carries 31 data bits and a guard bit (bit 31) that is
// always set.  The visited table starts zeroed, so a reader that races the
// writer of a slot sees a word without its guard bit and reads again: the key
// words need no release/acquire ordering against the slot's tag (bfs.cu).
#pragma once

#include <stdint.h>

#include "machine.cuh"

namespace mctb {

constexpr int kMaxWords = 24;
constexpr int kWordBits = 31;            // data bits per packed word
constexpr uint32_t kGuard = 0x80000000u;  // set in every written key word
constexpr uint32_t kData = 0x7fffffffu;

// floor(x / 31) for 0 <= x < 1.5e8 (bit offsets), without a division
__host__ __device__ inline int div31(int x) {
    return (int)(((uint64_t)(uint32_t)x * 0x8421085ull) >> 32);
}

struct Layout {
    // widths in bits
    uint8_t time, nrp, allnwe, nextwg, hostk, glob0;  // header (+ fin, clock, host_pc fixed)
    uint8_t dk, bb;                                   // device
    uint8_t uk, nwg, sent, items, ends;               // unit
    uint8_t bcount;                                   // barrier
    uint8_t cursor, busy, iter, pnwg;                 // pex
    uint8_t loc;                                      // minimum-kernel local slots
    uint8_t cfg;                                      // configuration id (multi-config search)
    int32_t words;                                    // packed size in 32-bit words
    int32_t bits;
    // bit offsets for in-place successor writes (explore fast paths)
    int32_t off_nrp, off_units, unit_bits, uoff_bcount, off_pex, pex_bits, poff_reported;
    int32_t off_dev, dev_bits, off_loc;
};

struct BfsDesc {
    MachDesc m;
    Layout l;
};

__host__ __device__ inline int bits_for(int64_t max_value) {
    int b = 0;
    while (b < 63 && (max_value >> b) != 0) ++b;
    return b;
}

// Field bounds (all inclusive maxima of reachable values).
__host__ inline Layout make_layout(const MachDesc& m, int n_cfg, int64_t max_time) {
    Layout l{};
    l.cfg = (uint8_t)bits_for(n_cfg > 0 ? n_cfg - 1 : 0);
    l.time = (uint8_t)bits_for(max_time);
    l.nrp = (uint8_t)bits_for(m.all_nwe);
    l.allnwe = (uint8_t)bits_for(m.all_nwe);
    l.nextwg = (uint8_t)bits_for(m.wgs);
    l.hostk = (uint8_t)bits_for(m.nwd > m.host_reacts ? m.nwd : m.host_reacts);
    l.glob0 = (uint8_t)(m.kernel == 1 ? bits_for(m.max_id) : 0);
    l.dk = (uint8_t)bits_for(m.nwu);
    l.bb = (uint8_t)bits_for(m.wgs);
    l.uk = (uint8_t)bits_for(m.nwe);
    l.nwg = (uint8_t)bits_for(m.wgs);
    l.sent = (uint8_t)bits_for(m.wg);
    l.items = (uint8_t)bits_for(m.wg);
    l.ends = (uint8_t)bits_for(m.nwe);
    l.bcount = (uint8_t)bits_for(m.nwe);
    const int64_t cur = m.act_len > m.epi_len ? m.act_len : m.epi_len;
    l.cursor = (uint8_t)bits_for(cur);
    int64_t busy = m.kernel == 0 ? (int64_t)m.gmt * m.ts : (m.gmt > 1 ? m.gmt : 1);
    if (m.kernel == 0 && m.ts > busy) busy = m.ts;
    l.busy = (uint8_t)bits_for(busy);
    l.iter = (uint8_t)bits_for(m.rounds);
    l.pnwg = l.nwg;
    l.loc = (uint8_t)(m.kernel == 1 ? bits_for(m.max_id) : 0);
    int bits = l.cfg + l.time + l.nrp + l.allnwe + 1 + l.nextwg + 3 + l.hostk + 1 + l.glob0;
    bits += m.nwd * (3 + l.dk + l.bb);
    bits += m.n_units * (3 + l.uk + l.nwg + l.sent + l.items + l.ends);
    bits += m.n_units * (1 + l.bcount);
    bits += m.n_pex * (4 + 1 + l.cursor + l.busy + 1 + l.pnwg + l.iter);
    if (m.kernel == 1) bits += m.n_units * m.np * l.loc;
    l.bits = bits;
    l.off_nrp = l.cfg + l.time;
    l.off_units = l.cfg + l.time + l.nrp + l.allnwe + 1 + l.nextwg + 3 + l.hostk + 1 + l.glob0 +
                  m.nwd * (3 + l.dk + l.bb);
    l.uoff_bcount = 3 + l.uk + l.nwg + l.sent + l.items + l.ends + 1;
    l.unit_bits = l.uoff_bcount + l.bcount;
    l.off_pex = l.off_units + m.n_units * l.unit_bits;
    l.pex_bits = 4 + 1 + l.cursor + l.busy + 1 + l.pnwg + l.iter;
    l.poff_reported = 4 + 1 + l.cursor + l.busy;
    l.dev_bits = 3 + l.dk + l.bb;
    l.off_dev = l.off_units - m.nwd * l.dev_bits;
    l.off_loc = l.off_pex + m.n_pex * l.pex_bits;
    l.words = (bits + kWordBits - 1) / kWordBits;
    return l;
}

struct BitWriter {
    uint32_t* w;
    uint64_t acc = 0;
    int n = 0, idx = 0;
    __host__ __device__ explicit BitWriter(uint32_t* out) : w(out) {}
    __host__ __device__ inline void put(uint32_t v, int bits) {
        if (!bits) return;
        acc |= (uint64_t)(v & (uint32_t)((1ull << bits) - 1)) << n;
        n += bits;
        while (n >= kWordBits) {
            w[idx++] = ((uint32_t)acc & kData) | kGuard;
            acc >>= kWordBits;
            n -= kWordBits;
        }
    }
    // pads with guard-only words up to `words`
    __host__ __device__ inline void flush(int words) {
        if (n > 0) w[idx++] = ((uint32_t)acc & kData) | kGuard;
        while (idx < words) w[idx++] = kGuard;
    }
};

struct BitReader {
    const uint32_t* w;
    uint64_t acc = 0;
    int n = 0, idx = 0;
    __host__ __device__ explicit BitReader(const uint32_t* in) : w(in) {}
    // positioned at bit `off`
    __host__ __device__ BitReader(const uint32_t* in, int off) : w(in) {
        idx = div31(off);
        const int sh = off - idx * kWordBits;
        if (sh) {
            acc = (uint64_t)(w[idx++] & kData) >> sh;
            n = kWordBits - sh;
        }
    }
    __host__ __device__ inline uint32_t get(int bits) {
        if (!bits) return 0;
        while (n < bits) {
            acc |= (uint64_t)(w[idx++] & kData) << n;
            n += kWordBits;
        }
        const uint32_t v = (uint32_t)(acc & ((1ull << bits) - 1));
        acc >>= bits;
        n -= bits;
        return v;
    }
};

__host__ __device__ inline void pack(const BfsDesc& d, int cfg, const MState& s, uint32_t* out) {
    const MachDesc& m = d.m;
    const Layout& l = d.l;
    BitWriter w(out);
    w.put((uint32_t)cfg, l.cfg);
    w.put((uint32_t)s.time, l.time);
    w.put((uint32_t)s.nrp_work, l.nrp);
    w.put((uint32_t)s.all_nwe, l.allnwe);
    w.put((uint32_t)s.fin, 1);
    w.put((uint32_t)s.next_wg, l.nextwg);
    w.put((uint32_t)s.host_pc, 3);
    w.put((uint32_t)s.host_k, l.hostk);
    w.put((uint32_t)s.clock, 1);
    w.put((uint32_t)s.glob0, l.glob0);
    for (int i = 0; i < m.nwd; ++i) {
        w.put((uint32_t)s.dev[i].pc, 3);
        w.put((uint32_t)s.dev[i].k, l.dk);
        w.put((uint32_t)s.dev[i].batch_base, l.bb);
    }
    for (int g = 0; g < m.n_units; ++g) {
        const UnitS& u = s.unit[g];
        w.put((uint32_t)u.pc, 3);
        w.put((uint32_t)u.k, l.uk);
        w.put((uint32_t)u.nwg, l.nwg);
        w.put((uint32_t)u.sent, l.sent);
        w.put((uint32_t)u.got_items, l.items);
        w.put((uint32_t)u.got_ends, l.ends);
        w.put((uint32_t)s.bar[g].pc, 1);
        w.put((uint32_t)s.bar[g].count, l.bcount);
    }
    for (int p = 0; p < m.n_pex; ++p) {
        const PexS& x = s.pex[p];
        w.put((uint32_t)x.pc, 4);
        w.put((uint32_t)x.phase, 1);
        w.put((uint32_t)x.cursor, l.cursor);
        w.put((uint32_t)x.busy_left, l.busy);
        w.put((uint32_t)x.reported, 1);
        w.put((uint32_t)x.nwg, l.pnwg);
        w.put((uint32_t)x.iter, l.iter);
    }
    if (m.kernel == 1)
        for (int i = 0; i < m.n_units * m.np; ++i) w.put((uint32_t)s.loc[i], l.loc);
    w.flush(l.words);
}

// cfg id first (so a reader can select the layout), then the fields in pack order.
__host__ __device__ inline int peek_cfg(const uint32_t* in, int cfg_bits) {
    return cfg_bits ? (int)(in[0] & ((1u << cfg_bits) - 1)) : 0;  // cfg_bits < 31
}

__host__ __device__ inline void unpack(const BfsDesc& d, const uint32_t* in, MState& s) {
    const MachDesc& m = d.m;
    const Layout& l = d.l;
    BitReader r(in);
    r.get(l.cfg);
    s.time = r.get(l.time);
    s.nrp_work = (int32_t)r.get(l.nrp);
    s.all_nwe = (int32_t)r.get(l.allnwe);
    s.fin = (int32_t)r.get(1);
    s.next_wg = (int32_t)r.get(l.nextwg);
    s.host_pc = (int32_t)r.get(3);
    s.host_k = (int32_t)r.get(l.hostk);
    s.clock = (int32_t)r.get(1);
    s.glob0 = (int32_t)r.get(l.glob0);
    for (int i = 0; i < m.nwd; ++i) {
        s.dev[i].pc = (int32_t)r.get(3);
        s.dev[i].k = (int32_t)r.get(l.dk);
        s.dev[i].batch_base = (int32_t)r.get(l.bb);
    }
    for (int g = 0; g < m.n_units; ++g) {
        UnitS& u = s.unit[g];
        u.pc = (int32_t)r.get(3);
        u.k = (int32_t)r.get(l.uk);
        u.nwg = (int32_t)r.get(l.nwg);
        u.sent = (int32_t)r.get(l.sent);
        u.got_items = (int32_t)r.get(l.items);
        u.got_ends = (int32_t)r.get(l.ends);
        s.bar[g].pc = (int32_t)r.get(1);
        s.bar[g].count = (int32_t)r.get(l.bcount);
    }
    for (int p = 0; p < m.n_pex; ++p) {
        PexS& x = s.pex[p];
        x.pc = (int32_t)r.get(4);
        x.phase = (int32_t)r.get(1);
        x.cursor = (int32_t)r.get(l.cursor);
        x.busy_left = (int32_t)r.get(l.busy);
        x.reported = (int32_t)r.get(1);
        x.nwg = (int32_t)r.get(l.pnwg);
        x.iter = (int32_t)r.get(l.iter);
    }
    if (m.kernel == 1)
        for (int i = 0; i < m.n_units * m.np; ++i) s.loc[i] = (int32_t)r.get(l.loc);
}

// Overwrites `width` (<= 32) bits at data-bit offset `off` of a packed state
// (the BitWriter order); a field spans at most two words.
__host__ __device__ inline void set_bits(uint32_t* w, int off, int width, uint32_t v) {
    if (!width) return;
    const int i = div31(off), sh = off - i * kWordBits;
    const uint64_t mask = ((1ull << width) - 1) << sh;
    const bool two = sh + width > kWordBits;
    uint64_t cur = (uint64_t)(w[i] & kData) | (two ? (uint64_t)(w[i + 1] & kData) << kWordBits : 0ull);
    cur = (cur & ~mask) | (((uint64_t)v << sh) & mask);
    w[i] = ((uint32_t)cur & kData) | kGuard;
    if (two) w[i + 1] = ((uint32_t)(cur >> kWordBits) & kData) | kGuard;
}

// Warp-parallel unpack (exploration): lane 0 reads the header, lane i the
// records of device/unit/element i (+32k); the caller syncs the warp after.
__device__ inline void unpack_lanes(const BfsDesc& d, const uint32_t* in, MState& s, int lane) {
    const MachDesc& m = d.m;
    const Layout& l = d.l;
    if (lane == 0) {
        BitReader r(in);
        r.get(l.cfg);
        s.time = r.get(l.time);
        s.nrp_work = (int32_t)r.get(l.nrp);
        s.all_nwe = (int32_t)r.get(l.allnwe);
        s.fin = (int32_t)r.get(1);
        s.next_wg = (int32_t)r.get(l.nextwg);
        s.host_pc = (int32_t)r.get(3);
        s.host_k = (int32_t)r.get(l.hostk);
        s.clock = (int32_t)r.get(1);
        s.glob0 = (int32_t)r.get(l.glob0);
    }
    for (int i = lane; i < m.nwd; i += 32) {
        BitReader r(in, l.off_dev + i * l.dev_bits);
        s.dev[i].pc = (int32_t)r.get(3);
        s.dev[i].k = (int32_t)r.get(l.dk);
        s.dev[i].batch_base = (int32_t)r.get(l.bb);
    }
    for (int g = lane; g < m.n_units; g += 32) {
        BitReader r(in, l.off_units + g * l.unit_bits);
        UnitS& u = s.unit[g];
        u.pc = (int32_t)r.get(3);
        u.k = (int32_t)r.get(l.uk);
        u.nwg = (int32_t)r.get(l.nwg);
        u.sent = (int32_t)r.get(l.sent);
        u.got_items = (int32_t)r.get(l.items);
        u.got_ends = (int32_t)r.get(l.ends);
        s.bar[g].pc = (int32_t)r.get(1);
        s.bar[g].count = (int32_t)r.get(l.bcount);
    }
    for (int p = lane; p < m.n_pex; p += 32) {
        BitReader r(in, l.off_pex + p * l.pex_bits);
        PexS& x = s.pex[p];
        x.pc = (int16_t)r.get(4);
        x.phase = (int16_t)r.get(1);
        x.cursor = (uint16_t)r.get(l.cursor);
        x.busy_left = (uint16_t)r.get(l.busy);
        x.reported = (int16_t)r.get(1);
        x.nwg = (int32_t)r.get(l.pnwg);
        x.iter = (uint16_t)r.get(l.iter);
    }
    if (m.kernel == 1)
        for (int i = lane; i < m.n_units * m.np; i += 32) {
            BitReader r(in, l.off_loc + i * l.loc);
            s.loc[i] = (int32_t)r.get(l.loc);
        }
}

// 64-bit hash of a packed state (splitmix64-style mixing of the words).
__host__ __device__ inline uint64_t hash_words(const uint32_t* w, int n) {
    uint64_t h = 0x9E3779B97F4A7C15ull * (uint64_t)(n + 1);
    for (int i = 0; i < n; ++i) {
        h ^= w[i];
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
    }
    h ^= h >> 32;
    h *= 0x94D049BB133111EBull;
    h ^= h >> 31;
    return h;
}

}  // namespace mctb
