"""The CPU oracle against the reference's own outputs (golden vectors made by
tests/golden/make_golden.py from /root/reference through oracle/_ref)."""
import hashlib
import struct

import pytest


def sha(trace):
    return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()


def test_known_answer_vectors(oracle):
    # Philox4x32-10 known-answer vectors (Random123 kat_vectors)
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert oracle.philox([0xffffffff] * 4, [0xffffffff] * 2) == [
        0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert oracle.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                         [0xa4093822, 0x299f31d0]) == [0xd16cfe09, 0x94fdcceb, 0x5001e420,
                                                       0x24126ea1]
    # std::mt19937_64 default seed: the 10000th output is fixed by the C++ standard
    assert oracle.mt19937_64(5489, 10000)[-1] == 9981545732273789042


def test_launch_plans(oracle, gold):
    for plat, size, wg, ts, want in gold("launch.json"):
        assert oracle.derive_launch(plat, size, wg, ts) == want, (plat, size, wg, ts)


def test_round_robin_runs_reproduce_sweeps(oracle, gold):
    for case in gold("sweeps.json"):
        plat, size, kernel = case["plat"], case["size"], case["kernel"]
        for wg, ts, time, transitions, ok, note in case["rows"]:
            if not ok:
                assert note == 1 and kernel == 1 and wg * ts > size
                continue
            r = oracle.simulate(plat, size, kernel, wg, ts, policy=0)
            assert (r["time"], r["steps"]) == (time, transitions), (plat, size, kernel, wg, ts)


def test_seeded_runs_bit_exact(oracle, gold):
    for c in gold("simulate.json"):
        r = oracle.simulate(c["plat"], c["size"], c["kernel"], c["wg"], c["ts"], c["policy"],
                            c["seed"], c["input"], trace=True)
        key = (c["plat"], c["size"], c["kernel"], c["wg"], c["ts"], c["policy"])
        assert (r["time"], r["steps"], r["result"]) == (c["time"], c["steps"], c["result"]), key
        assert sha(r["trace"]) == c["trace_sha"], key


def test_exploration_counts(oracle, gold):
    for c in gold("explore.json"):
        r = oracle.explore(c["plat"], c["size"], c["kernel"], c["wg"], c["ts"])
        for k in ("complete", "states", "transitions", "max_depth", "min_time", "max_time",
                  "n_terminal", "n_distinct"):
            assert r[k] == c[k], (k, c)


def test_check_overtime(oracle, gold):
    for c in gold("check.json"):
        r = oracle.check_overtime(c["plat"], c["size"], c["kernel"], c["T"])
        for k in ("violated", "exhaustive", "states", "max_depth", "transitions",
                  "configs_explored", "configs_skipped", "final_time", "wg", "ts", "steps"):
            assert r[k] == c[k], (k, c["plat"], c["size"], c["T"])
        assert sha(r["trace"]) == c["trace_sha"]


def test_fingerprints_and_text(oracle, gold):
    for c in gold("fingerprints.json"):
        fp = oracle.fingerprints(c["plat"], c["size"], c["kernel"], c["wg"], c["ts"],
                                 [tuple(t) for t in c["trace"]])
        assert [str(v) for v in fp] == c["fingerprints"]
    for c in gold("tune.json"):
        if "trace" in c:
            text = oracle.trace_text(c["plat"], c["size"], c["kernel"], c["wg"], c["ts"],
                                     [tuple(t) for t in c["trace"]])
            assert text == c["text"]


def test_replay_rejects_tampering(oracle, gold):
    c = next(c for c in gold("tune.json") if c["size"] == 8 and c["kernel"] == 0)
    tr = [tuple(t) for t in c["trace"]]
    assert oracle.replay(c["plat"], 8, 0, c["wg"], c["ts"], tr, c["t_min"])[0] == 44
    from checkers import CheckerError
    with pytest.raises(CheckerError) as e:
        oracle.replay(c["plat"], 8, 0, c["wg"], c["ts"], tr[:-1], c["t_min"])
    assert e.value.rc == 3
    with pytest.raises(CheckerError):
        oracle.replay(c["plat"], 8, 0, c["wg"], c["ts"], tr, c["t_min"] + 1)
    with pytest.raises(CheckerError):
        oracle.replay(c["plat"], 8, 0, c["wg"], c["ts"], [(2, 0xffff, 0, 0)] + tr[1:], c["t_min"])


def test_oracle_against_reference_directly(oracle, ref):
    """Random schedules on random platforms, traces compared transition by transition."""
    import random
    rng = random.Random(7)
    for _ in range(150):
        plat = (rng.randint(1, 3), rng.randint(1, 3), 1 << rng.randint(0, 3), rng.randint(1, 5))
        size = 1 << rng.randint(2, 5)
        n = size.bit_length() - 1
        wg, ts = 1 << rng.randint(1, n - 1), 1 << rng.randint(1, n - 1)
        kernel = rng.randint(0, 1)
        if kernel == 1 and wg * ts > size:
            continue
        inp = [rng.randint(-99, 99) for _ in range(size)] if kernel else None
        seed = rng.randrange(1 << 63)
        a = ref.simulate(plat, size, kernel, wg, ts, 1, seed, inp, trace=True)
        b = oracle.simulate(plat, size, kernel, wg, ts, 1, seed, inp, trace=True)
        assert a == b


GRADED = [((1, 1, 4, 4), 8, 0, 4, 4), ((2, 1, 2, 4), 8, 0, 2, 2), ((1, 1, 4, 4), 8, 1, 4, 2),
          ((3, 1, 1, 1), 16, 0, 2, 2), ((2, 1, 4, 2), 16, 1, 2, 2), ((3, 1, 1, 4), 16, 1, 2, 2),
          ((2, 2, 2, 2), 16, 0, 2, 4)]


@pytest.mark.parametrize("case", GRADED)
def test_state_graphs_are_graded(oracle, case):
    """Every path from the initial state to a state has the same length (each
    transition advances one process's fixed amount of protocol, and every run of
    a configuration has protocol + time transitions).  The GPU's depth cap relies
    on it: the depth-limited DFS (explore.cpp:124-127) then visits exactly the
    states of depth <= max_depth, whatever its order."""
    plat, size, kernel, wg, ts = case
    init = oracle.successors(plat, size, kernel, wg, ts)
    depth = {s: 0 for _, s in init}
    frontier = [s for _, s in init]
    d = 0
    while frontier:
        nxt = []
        for s in frontier:
            for _, t in oracle.successors(plat, size, kernel, wg, ts, s):
                if t in depth:
                    assert depth[t] == d + 1, (case, d)
                else:
                    depth[t] = d + 1
                    nxt.append(t)
        frontier = nxt
        d += 1
    # the deepest state is the end of the longest run: protocol transitions + max time
    t, steps, _ = oracle.cost_model(plat, size, kernel, wg, ts)
    r = oracle.explore(plat, size, kernel, wg, ts)
    assert d - 1 == r["max_depth"] == steps - t + r["max_time"]


def test_depth_cap_against_reference(oracle, gold):
    """The oracle's depth-limited DFS against the reference's (tests/golden/depth.json)."""
    g = gold("depth.json")
    for c in g["explores"]:
        r = oracle.explore(c["plat"], c["size"], c["kernel"], c["wg"], c["ts"],
                           max_depth=c["depth_cap"])
        for k in ("complete", "states", "transitions", "max_depth", "min_time", "max_time",
                  "n_terminal"):
            assert r[k] == c[k], (k, c)
    for c in g["checks"]:
        if c["plat"] == [2, 1, 2, 4] and not c["violated"]:
            continue  # 4e5-state sweeps: the GPU tests cover them
        r = oracle.check_overtime(c["plat"], c["size"], c["kernel"], c["T"],
                                  max_depth=c["depth_cap"])
        for k in ("violated", "exhaustive", "states", "max_depth", "transitions",
                  "configs_explored", "configs_skipped", "final_time", "wg", "ts", "steps"):
            assert r[k] == c[k], (k, c["plat"], c["size"], c["T"], c["depth_cap"])
        assert sha(r["trace"]) == c["trace_sha"]
