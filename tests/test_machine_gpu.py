"""The GPU transition system against the reference (golden traces) and the oracle."""
import hashlib
import random
import struct

import pytest

pytestmark = pytest.mark.gpu


def sha(trace):
    return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()


def problem(m, size, kernel, inp=None):
    return m.ProblemSpec.abstract(size) if kernel == 0 else m.ProblemSpec.minimum(size, inp)


def test_runs_bit_exact_with_reference_traces(engine, gold):
    """Machine::run RoundRobin and SeededRandom(mt19937_64): same transitions,
    time, transition count and result as the reference."""
    m = engine
    for c in gold("simulate.json"):
        mach = m.Machine(m.PlatformConfig(*c["plat"]),
                         problem(m, c["size"], c["kernel"], c["input"]),
                         m.TuningParams(c["wg"], c["ts"]))
        tr = []
        r = mach.run(c["policy"], c["seed"], trace_out=tr)
        key = (c["plat"], c["size"], c["kernel"], c["wg"], c["ts"], c["policy"])
        assert (r.time, r.steps, r.result) == (c["time"], c["steps"], c["result"]), key
        assert len(tr) == c["trace_len"] and sha(tr) == c["trace_sha"], key


def test_first_path_is_the_reference_counterexample(engine, gold):
    """The en[0] schedule is the first DFS path, i.e. the reference's
    counterexample of check_overtime whenever that path is fast enough."""
    m = engine
    seen = 0
    for c in gold("check.json"):
        if not c["violated"]:
            continue
        mach = m.Machine(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]),
                         m.TuningParams(c["wg"], c["ts"]))
        tr = []
        r = mach.run(m.FIRST, trace_out=tr)
        if r.time <= c["T"]:
            seen += 1
            assert sha(tr) == c["trace_sha"] and len(tr) == c["steps"]
    assert seen >= 8


def test_trace_text_and_replay_match_reference(engine, gold):
    m = engine
    for c in gold("tune.json"):
        if "trace" not in c:
            continue
        plat, prob = m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"])
        t = m.Trace([tuple(x) for x in c["trace"]], c["t_min"], m.TuningParams(c["wg"], c["ts"]),
                    len(c["trace"]))
        assert m.trace_to_text(plat, prob, t) == c["text"]
        assert m.replay(plat, prob, t)[0] == c["t_min"]


def test_replay_rejects_tampered_traces(engine, gold):
    m = engine
    c = next(c for c in gold("tune.json") if c["size"] == 8 and c["kernel"] == 0)
    plat, prob = m.PlatformConfig(*c["plat"]), m.ProblemSpec.abstract(8)
    tr = [tuple(x) for x in c["trace"]]
    good = m.Trace(tr, 44, m.TuningParams(4, 4), len(tr))
    assert m.replay(plat, prob, good) == (44, None)
    for bad in (m.Trace(tr[:-1], 44, good.params), m.Trace(tr, 45, good.params),
                m.Trace([(2, 0xffff, 0, 0)] + tr[1:], 44, good.params)):
        with pytest.raises(m.CorruptTrace):
            m.replay(plat, prob, bad)


@pytest.mark.parametrize("seed", range(6))
def test_philox_trajectories_replay_on_cpu(engine, oracle, seed):
    """Swarm trajectories: every GPU trajectory equals its CPU replay (same
    time, transitions, result and FNV-1a hash of the whole transition list)."""
    m = engine
    rng = random.Random(seed)
    plat = (rng.randint(1, 3), rng.randint(1, 2), 1 << rng.randint(0, 3), rng.randint(1, 4))
    size = 1 << rng.randint(3, 5)
    kernel = rng.randint(0, 1)
    cfgs = [c for c in m.enumerate_configs(size) if kernel == 0 or c.wg * c.ts <= size]
    inp = [rng.randint(-500, 500) for _ in range(size)] if kernel else None
    n = 600
    traj0 = rng.randrange(1 << 40)
    g = m.trajectories(m.PlatformConfig(*plat), problem(m, size, kernel, inp), cfgs, m.PHILOX,
                       seed + 11, traj0, n)
    o = oracle.trajectories(plat, size, kernel, [(c.wg, c.ts) for c in cfgs], 3, seed + 11,
                            traj0, n, inp)
    assert g.status == [0] * n
    assert g.time == o[0] and g.steps == o[1] and g.result == o[2]
    assert g.hash == o[4] and g.config == o[5]


def test_minimum_kernel_functional_correctness(engine):
    """Acceptance criterion 5: 100 random arrays, random valid configs and
    platforms, random schedules -> glob[0] = min(input), also on replay."""
    m = engine
    rng = random.Random(2024)
    for trial in range(100):
        size = 1 << rng.randint(2, 6)
        inp = [rng.randrange(100000) - 50000 for _ in range(size)]
        plat = m.PlatformConfig(1, rng.randint(1, 2), 1 << rng.randint(1, 3), rng.randint(1, 4))
        cfg = rng.choice([c for c in m.enumerate_configs(size) if c.wg * c.ts <= size])
        prob = m.ProblemSpec.minimum(size, inp)
        tr = []
        r = m.Machine(plat, prob, cfg).run(m.PHILOX, rng.randrange(1 << 60), trace_out=tr)
        assert r.result == min(inp), trial
        assert m.replay(plat, prob, m.Trace(tr, r.time, cfg, len(tr))) == (r.time, min(inp))
