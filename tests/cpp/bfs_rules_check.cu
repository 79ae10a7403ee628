// Host-side invariants of the exploration's fast paths (csrc/bfs_rules.cuh)
// against the serial semantics they replace (machine.cuh enabled()/apply(),
// pack.cuh pack()), on random walks through many configurations.  Test
// infrastructure: runs on the CPU, no device needed.
//  (1) the per-process enumeration (bfs_slot_rules, ordinal form) yields exactly
//      the multiset of transitions enabled() yields (machine.cpp:174-336);
//  (2) the table-driven unpack (unpack_fields) inverts pack();
//  (3) every in-place successor (fast_successor) equals pack(apply(...)), and its
//      incrementally updated hash equals the full hash of the packed words.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <tuple>
#include <vector>

#include "bfs.cuh"
#include "bfs_rules.cuh"
#include "traj.cuh"

using namespace mctb;

namespace {
struct Case {
    int plat[4];
    int size, kernel, wg, ts;
};

auto key(const Transition& t) { return std::make_tuple(t.actor, t.peer, t.op, t.arg); }
}  // namespace

int main() {
    std::vector<Case> cases;
    const int plats[][4] = {{1, 1, 4, 4}, {1, 1, 8, 2}, {2, 1, 2, 4}, {1, 2, 4, 3}, {2, 3, 2, 1},
                            {1, 1, 16, 4}, {3, 2, 4, 2}};
    for (const auto& p : plats)
        for (int size : {8, 16, 32, 64})
            for (int kernel : {0, 1})
                for (int wg = 2; wg <= size / 2; wg *= 2)
                    for (int ts = 2; ts <= size / 2; ts *= 4)
                        cases.push_back(Case{{p[0], p[1], p[2], p[3]}, size, kernel, wg, ts});
    uint64_t hk[32];
    for (int i = 0; i < 32; ++i) hk[i] = hash_coef(i);
    long long checks = 0, fails = 0, states = 0, fast = 0;
    int configs = 0;
    std::mt19937_64 rng(2305);
    auto fail = [&](const char* what, const Case& c) {
        if (++fails <= 20)
            std::fprintf(stderr, "FAIL %s: plat (%d,%d,%d,%d) size %d kernel %d (wg %d, ts %d)\n",
                         what, c.plat[0], c.plat[1], c.plat[2], c.plat[3], c.size, c.kernel, c.wg,
                         c.ts);
    };
    for (const Case& c : cases) {
        MachHost h;
        if (build_desc(c.plat, c.size, c.kernel, nullptr, c.wg, c.ts, &h) != 0) continue;
        MachDesc m = h.d;
        m.input_id = h.ids.data();
        BfsDesc d;
        d.m = m;
        d.l = bfs_layout(m, 1);
        if (d.l.words > kMaxWords || d.l.time > 32) continue;
        ++configs;
        std::vector<uint2> ftab(kMaxFields);
        const int nf = build_field_table(m, d.l, ftab.data());
        const int W = d.l.words, lognwe = m.lognwe;
        for (int walk = 0; walk < 6; ++walk) {
            MState s;
            initial_state(m, s);
            for (int step = 0; step < 4000; ++step, ++states) {
                Transition en[kMaxEnabled];
                const int n = enabled(m, s, en);
                // (1) the enumeration as a multiset
                std::vector<Transition> ord, pid;
                for (int k = 0; k < n_slots(m); ++k) {
                    Transition o[2];
                    const int cnt = bfs_slot_rules(m, s, k, lognwe, o);
                    for (int j = 0; j < cnt; ++j) {
                        ord.push_back(o[j]);
                        pid.push_back(to_pid(m, o[j]));
                    }
                }
                std::vector<Transition> ref(en, en + n);
                auto lt = [](const Transition& a, const Transition& b) { return key(a) < key(b); };
                std::sort(pid.begin(), pid.end(), lt);
                std::sort(ref.begin(), ref.end(), lt);
                ++checks;
                if (pid.size() != ref.size() ||
                    !std::equal(pid.begin(), pid.end(), ref.begin(),
                                [](const Transition& a, const Transition& b) {
                                    return key(a) == key(b);
                                }))
                    fail("enumeration differs from enabled()", c);
                // (2) unpack_fields inverts pack
                uint32_t row[32], row2[32];
                for (int i = 0; i < 32; ++i) row[i] = row2[i] = kGuard;
                pack(d, 0, s, row);
                MState u;
                std::memset(&u, 0, sizeof u);
                unpack_fields(ftab.data(), nf, row, u, 0, 1);
                pack(d, 0, u, row2);
                ++checks;
                if (std::memcmp(row, row2, 4 * W) != 0) fail("unpack_fields(pack(s)) != s", c);
                // (3) in-place successors
                const uint64_t H0 = hash_full(row, W);
                for (const Transition& o : ord) {
                    uint32_t r1[32];
                    std::memcpy(r1, row, sizeof r1);
                    uint64_t H = H0;
                    if (!fast_successor(d, s, o, r1, hk, H)) continue;
                    ++fast;
                    MState t;
                    copy_state(m, t, s);
                    const bool ok = apply(m, t, to_pid(m, o));
                    uint32_t r2[32];
                    for (int i = 0; i < 32; ++i) r2[i] = kGuard;
                    pack(d, 0, t, r2);
                    ++checks;
                    if (!ok || std::memcmp(r1, r2, 4 * W) != 0)
                        fail("fast successor != pack(apply)", c);
                    ++checks;
                    if (H != hash_full(r1, W)) fail("incremental hash != full hash", c);
                }
                if (n == 0) break;
                apply(m, s, en[rng() % (uint64_t)n]);
            }
        }
    }
    std::printf("bfs_rules_check: %d configurations, %lld states, %lld in-place successors, "
                "%lld checks, %lld failed\n", configs, states, fast, checks, fails);
    return fails ? 1 : 0;
}
