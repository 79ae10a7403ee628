"""Randomised GPU-against-reference checks (the reference core oracle/_ref, built
here and shipped with the snapshot): explore_machine, check_overtime and
check_nontermination on random small platforms, problems and ExploreLimits
(depth and visited caps included), every compared field equal."""
import hashlib
import random
import struct

import pytest

pytestmark = pytest.mark.gpu


def sha(trace):
    return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()


def problem(m, size, kernel, inp=None):
    return m.ProblemSpec.abstract(size) if kernel == 0 else m.ProblemSpec.minimum(size, inp)


def _case(rng):
    plat = (rng.randint(1, 3), rng.randint(1, 2), 1 << rng.randint(0, 2), rng.randint(1, 4))
    size = rng.choice((4, 8, 8, 16))
    kernel = rng.randint(0, 1)
    inp = [rng.randint(-99, 99) for _ in range(size)] if kernel and rng.random() < 0.5 else None
    return plat, size, kernel, inp


@pytest.mark.parametrize("seed", range(16))
def test_random_explorations(engine, ref, seed):
    m = engine
    rng = random.Random(1000 + seed)
    for _ in range(10):
        plat, size, kernel, inp = _case(rng)
        cfgs = [c for c in m.enumerate_configs(size) if kernel == 0 or c.wg * c.ts <= size]
        c = rng.choice(cfgs)
        depth = rng.choice((0, 0, rng.randint(1, 300)))
        states = rng.choice((0, 0, rng.randint(1, 5000)))
        x = ref.explore(plat, size, kernel, c.wg, c.ts, inp, max_depth=depth, max_states=states)
        g = m.explore_machine(m.PlatformConfig(*plat), problem(m, size, kernel, inp), c,
                              max_states=states or 5_000_000, max_depth=depth or 4_000_000)
        key = (plat, size, kernel, c, depth, states)
        assert (g.complete, g.states_visited, g.transitions_applied, g.max_depth_reached) == (
            bool(x["complete"]), x["states"], x["transitions"], x["max_depth"]), key
        if x["states"] < (states or 5_000_000):  # the cap did not bind: every terminal met
            assert g.terminals == x["n_terminal"], key


@pytest.mark.parametrize("seed", range(16))
def test_random_checks(engine, ref, seed):
    m = engine
    rng = random.Random(2000 + seed)
    for _ in range(6):
        plat, size, kernel, inp = _case(rng)
        t = m.tune(m.PlatformConfig(*plat), problem(m, size, kernel, inp))
        T = rng.choice((t.t_min, t.t_min - 1, t.t_min + rng.randint(0, 50), t.t_ini))
        depth = rng.choice((0, 0, rng.randint(20, 400)))
        states = rng.choice((0, 0, rng.randint(50, 5000)))
        r = ref.check_overtime(plat, size, kernel, T, inp, max_depth=depth, max_states=states)
        v = m.check_overtime(m.PlatformConfig(*plat), problem(m, size, kernel, inp), T,
                             max_states=states or 5_000_000, max_depth=depth or 4_000_000)
        key = (plat, size, kernel, T, depth, states)
        assert (v.violated, v.exhaustive, v.stats.states_visited) == (
            bool(r["violated"]), bool(r["exhaustive"]), r["states"]), key
        assert (v.stats.transitions_applied, v.stats.max_depth_reached) == (
            r["transitions"], r["max_depth"]), key
        if v.violated:
            assert (v.trace.final_time, v.trace.params.wg, v.trace.params.ts, v.trace.steps) == (
                r["final_time"], r["wg"], r["ts"], r["steps"]), key
            assert sha(v.trace.transitions) == sha(r["trace"]), key


@pytest.mark.parametrize("seed", range(8))
def test_random_nontermination(engine, ref, seed):
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_golden_nonterm import ref_nonterm
    m = engine
    rng = random.Random(3000 + seed)
    for _ in range(3):
        plat, size, kernel, _ = _case(rng)
        depth = rng.choice((0, 0, rng.randint(20, 300)))
        states = rng.choice((0, 0, rng.randint(100, 20_000)))
        r = ref_nonterm(ref, plat, size, kernel, max_depth=depth, max_states=states,
                        rows_cap=4096)
        traces, stats = m.check_nontermination(m.PlatformConfig(*plat), problem(m, size, kernel),
                                               max_depth=depth or 4_000_000,
                                               max_states=states or 5_000_000)
        key = (plat, size, kernel, depth, states)
        assert len(traces) == r["n"], key
        for t, g in zip(traces, r["traces"]):
            assert (t.params.wg, t.params.ts, t.final_time, t.steps) == (
                g["wg"], g["ts"], g["final_time"], g["steps"]), key
            assert sha(t.transitions) == g["sha"], key
        assert sum(s.states_visited for s in stats) == r["states"], key
        assert sum(s.transitions_applied for s in stats) == r["transitions"], key


@pytest.mark.parametrize("seed", range(8))
def test_random_tunes(engine, ref, seed):
    m = engine
    rng = random.Random(4000 + seed)
    for _ in range(3):
        plat, size, kernel, inp = _case(rng)
        depth = rng.choice((0, 0, rng.randint(60, 400)))
        states = rng.choice((0, 0, rng.randint(200, 5000)))
        s = rng.randint(1, 9)
        try:
            r = ref.tune(plat, size, kernel, seed=s, inp=inp, max_depth=depth, max_states=states)
        except Exception:
            with pytest.raises(m.MctuneError):
                m.tune(m.PlatformConfig(*plat), problem(m, size, kernel, inp), seed=s,
                       max_states=states or 5_000_000, max_depth=depth or 4_000_000)
            continue
        g = m.tune(m.PlatformConfig(*plat), problem(m, size, kernel, inp), seed=s,
                   max_states=states or 5_000_000, max_depth=depth or 4_000_000)
        key = (plat, size, kernel, s, depth, states)
        assert (g.t_min, g.params.wg, g.params.ts, g.t_ini, g.proven) == (
            r["t_min"], r["wg"], r["ts"], r["t_ini"], bool(r["proven"])), key
        assert (g.stats.checks_run, g.stats.states_visited_total, g.first_trail_time) == (
            r["checks_run"], r["states_visited_total"], r["first_trail_time"]), key
        assert g.trace.steps == r["steps"] and sha(g.trace.transitions) == sha(r["trace"]), key


@pytest.mark.parametrize("seed", range(4))
def test_random_sweeps_and_runs(engine, ref, seed):
    """exhaustive_sweep rows and Machine::run (RoundRobin / SeededRandom, with the
    trace) on random platforms, sizes up to 64 and random inputs."""
    m = engine
    rng = random.Random(5000 + seed)
    for _ in range(4):
        plat = (rng.randint(1, 6), rng.randint(1, 5), 1 << rng.randint(0, 4), rng.randint(1, 6))
        size = rng.choice((8, 16, 32, 64))
        kernel = rng.randint(0, 1)
        inp = [rng.randint(-999, 999) for _ in range(size)] if kernel else None
        prob = problem(m, size, kernel, inp)
        got = [(r.wg, r.ts, r.time, r.transitions, int(r.ok)) for r in
               m.exhaustive_sweep(m.PlatformConfig(*plat), prob)]
        want = [tuple(r[:5]) for r in ref.sweep(plat, size, kernel, inp)]
        assert got == want, (plat, size, kernel)
        cfgs = [c for c in m.enumerate_configs(size) if kernel == 0 or c.wg * c.ts <= size]
        for _ in range(3):
            c = rng.choice(cfgs)
            policy, s = rng.choice((0, 1)), rng.randint(0, 1 << 40)
            tr = []
            g = m.Machine(m.PlatformConfig(*plat), prob, c).run(policy, s, trace_out=tr)
            r = ref.simulate(plat, size, kernel, c.wg, c.ts, policy, s, inp, trace=True)
            assert (g.time, g.steps, g.result) == (r["time"], r["steps"], r["result"]), (plat, c)
            assert sha(tr) == sha(r["trace"]), (plat, c)


def _fnv_flat(vals):
    h = 0xcbf29ce484222325
    for v in vals:
        for b in range(8):
            h ^= (v >> (8 * b)) & 0xff
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.mark.parametrize("seed", range(6))
def test_random_explore_order_matches_reference(engine, ref, seed):
    """ExploreHooks parity: the states explore_machine visits, in the order its DFS
    discovers them (on_state), against the reference's own explore_machine
    (ref_explore_order), state by state — with depth and visited caps (a full
    visited set keeps the first max_states of that order)."""
    import ctypes as C
    from paper_2305_09130_b200._lib import lib
    m = engine
    rng = random.Random(6000 + seed)
    for _ in range(4):
        plat, size, kernel, inp = _case(rng)
        size = min(size, 8)
        inp = inp[:size] if inp else None
        cfgs = [c for c in m.enumerate_configs(size) if kernel == 0 or c.wg * c.ts <= size]
        c = rng.choice(cfgs)
        depth = rng.choice((0, 0, rng.randint(5, 200)))
        states = rng.choice((0, 0, rng.randint(10, 3000)))
        want, n_want = ref.explore_order(plat, size, kernel, c.wg, c.ts, inp, max_depth=depth,
                                         max_states=states)
        prob = problem(m, size, kernel, inp)
        cap = max(n_want, 1)
        flat = (C.c_int64 * (cap * 1024))()
        meta = (C.c_int32 * (8 * cap))()
        info = (C.c_int64 * 3)()
        rc = lib.mctb_machine_states(m.PlatformConfig(*plat).as_array(), size, kernel,
                                     prob.input_array(), c.wg, c.ts, depth or 4_000_000,
                                     states or 5_000_000, flat, cap * 1024, meta, cap, info)
        assert rc == 0, (plat, size, kernel, c)
        n, stride = info[1], info[2]
        got = [_fnv_flat(flat[i * stride:(i + 1) * stride]) for i in range(n)]
        key = (plat, size, kernel, c, depth, states)
        assert n == n_want, key
        assert got == want, key
