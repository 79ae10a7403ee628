"""GPU interleaving exploration against the reference's exhaustive DFS."""
import pytest

pytestmark = pytest.mark.gpu


def problem(m, size, kernel):
    return m.ProblemSpec.abstract(size) if kernel == 0 else m.ProblemSpec.minimum(size)


def test_state_counts_equal_reference(engine, gold):
    """states_visited, transitions_applied, max_depth_reached and the terminal-time
    range of every configuration equal explore_machine's (explore.json)."""
    m = engine
    groups = {}
    for c in gold("explore.json"):
        groups.setdefault((tuple(c["plat"]), c["size"], c["kernel"]), []).append(c)
    for (plat, size, kernel), cases in groups.items():
        cfgs = [m.TuningParams(c["wg"], c["ts"]) for c in cases]
        got = m.explore_configs(m.PlatformConfig(*plat), problem(m, size, kernel), cfgs)
        for c, g in zip(cases, got):
            key = (plat, size, kernel, c["wg"], c["ts"])
            assert g.complete and g.deadlocks == 0, key
            assert g.states_visited == c["states"], key
            assert g.transitions_applied == c["transitions"], key
            assert g.max_depth_reached == c["max_depth"], key
            assert (g.min_time, g.max_time) == (c["min_time"], c["max_time"]), key
            assert g.terminals == c["n_terminal"], key


def test_each_config_alone_equals_batched(engine):
    m = engine
    plat, prob = m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(16)
    cfgs = m.enumerate_configs(16)
    batched = m.explore_configs(plat, prob, cfgs)
    for c, b in zip(cfgs, batched):
        assert m.explore_machine(plat, prob, c) == b


def test_larger_spaces_against_oracle(engine, oracle):
    m = engine
    for plat, size, kernel, wg, ts in [((1, 1, 4, 4), 32, 0, 16, 2), ((1, 1, 8, 2), 16, 0, 8, 2),
                                       ((2, 1, 2, 4), 16, 0, 2, 2), ((1, 2, 4, 3), 32, 1, 8, 2),
                                       ((1, 1, 4, 4), 64, 1, 32, 2)]:
        g = m.explore_machine(m.PlatformConfig(*plat), problem(m, size, kernel),
                              m.TuningParams(wg, ts))
        o = oracle.explore(plat, size, kernel, wg, ts)
        assert (g.states_visited, g.transitions_applied, g.max_depth_reached, g.min_time,
                g.max_time) == (o["states"], o["transitions"], o["max_depth"], o["min_time"],
                                o["max_time"]), (plat, size, kernel, wg, ts)


def test_state_limit_is_reported(engine):
    m = engine
    r = m.explore_machine(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(32),
                          m.TuningParams(16, 2), max_states=1000)
    assert not r.complete


def test_state_limit_bounds_the_sweep(engine):
    """max_states much smaller than the reachable space (1.37e8 states): the sweep
    stops near the cap in its first table (no 16x restart), reports the
    reference's capped count (explore.cpp:28) and is not complete."""
    m = engine
    info = []
    r = m.explore_configs(m.PlatformConfig(1, 1, 16, 4), m.ProblemSpec.abstract(64),
                          [m.TuningParams(16, 2)], max_states=100_000, info=info)[0]
    assert not r.complete
    assert r.states_visited == 100_000
    assert info[0].table_slots == 1 << 20  # the first table: 4 x max_states, no restart
    assert info[0].states < 1_000_000      # inserted past the cap: bounded by the flush


def test_acceptance_7_interleaving_invariants(engine):
    """Every reachable state of every size-8 configuration (both kernels) keeps
    Machine::check_invariants and tick gating; no deadlock; the final time is
    schedule-independent and equals the deterministic run (acceptance 7, and
    test_explore.cpp:145-170 for sizes 4-16)."""
    m = engine
    p = m.PlatformConfig(1, 1, 4, 4)
    for prob in (m.ProblemSpec.abstract(4), m.ProblemSpec.abstract(8), m.ProblemSpec.abstract(16),
                 m.ProblemSpec.minimum(8), m.ProblemSpec.minimum(16)):
        cfgs = [c for c in m.enumerate_configs(prob.size) if m.config_feasible(prob, c)]
        got = m.explore_configs(p, prob, cfgs, check_invariants=True)
        for c, g in zip(cfgs, got):
            assert g.complete and g.deadlocks == 0 and g.invariant_violations == 0, (prob, c)
            assert g.min_time == g.max_time == m.Machine(p, prob, c).run().time, (prob, c)


def test_multi_device_skew_minimum_is_lockstep_time(engine, oracle):
    """test_explore.cpp:199-225: with two devices and host re-arming some
    schedules are slower, but the explored minimum is the lock-step time."""
    m = engine
    g = m.explore_machine(m.PlatformConfig(2, 1, 2, 4), m.ProblemSpec.abstract(16),
                          m.TuningParams(2, 2))
    want = oracle.cost_model((2, 1, 2, 4), 16, 0, 2, 2)[0]
    assert g.complete and g.min_time == want and g.max_time > want


def test_acceptance_6_minimum_kernel_trend(engine):
    m = engine
    p = m.PlatformConfig(1, 1, 4, 4)

    def max_wg_among_best(rows):
        best = next(r.time for r in rows if r.ok)
        return max(r.wg for r in rows if r.ok and r.time == best)
    b16 = max_wg_among_best(m.exhaustive_sweep(p, m.ProblemSpec.minimum(16)))
    b64 = max_wg_among_best(m.exhaustive_sweep(p, m.ProblemSpec.minimum(64)))
    tuned = m.tune(p, m.ProblemSpec.minimum(16))
    assert tuned.params.wg == b16 == 8 and b16 <= b64


@pytest.mark.parametrize("parts,system_scope", [(2, False), (3, False), (8, False), (2, True)])
def test_partitioned_exchange_equals_reference(engine, gold, parts, system_scope):
    """The hash-partitioned sweep (the multi-GPU successor exchange, P partitions on
    one device; system_scope = the multi-GPU kernel variant) reproduces every golden
    exploration exactly, including states, transitions and max depth."""
    m = engine
    groups = {}
    for c in gold("explore.json"):
        groups.setdefault((tuple(c["plat"]), c["size"], c["kernel"]), []).append(c)
    for (plat, size, kernel), cases in groups.items():
        cfgs = [m.TuningParams(c["wg"], c["ts"]) for c in cases]
        got = m.explore_configs(m.PlatformConfig(*plat), problem(m, size, kernel), cfgs,
                                partitions=parts, system_scope=system_scope)
        for c, g in zip(cases, got):
            key = (plat, size, kernel, c["wg"], c["ts"], parts)
            assert g.complete and g.deadlocks == 0, key
            assert (g.states_visited, g.transitions_applied, g.max_depth_reached) == (
                c["states"], c["transitions"], c["max_depth"]), key
            assert (g.min_time, g.max_time, g.terminals) == (
                c["min_time"], c["max_time"], c["n_terminal"]), key


def test_partitioned_large_space_equals_single(engine):
    """5.6e7 states split over 4 partitions: the same counts as one partition."""
    m = engine
    args = (m.PlatformConfig(1, 1, 16, 4), m.ProblemSpec.abstract(32), [m.TuningParams(16, 2)])
    one = m.explore_configs(*args, max_states=100_000_000)[0]
    four = m.explore_configs(*args, max_states=100_000_000, partitions=4)[0]
    assert one.complete and one.states_visited == 56088395
    assert four == one


def test_multi_gpu_api_one_rank_equals_reference(engine, gold):
    """mctb_explore_mp_* (open / connect / seed / run / close, system-scope kernel)
    as one rank: the golden explorations exactly.  With more ranks the same kernel
    inserts into the peers' partitions over NVLink (covered on one device by
    test_partitioned_exchange_equals_reference)."""
    m = engine
    from paper_2305_09130_b200.distributed import explore_multi_gpu
    groups = {}
    for c in gold("explore.json"):
        groups.setdefault((tuple(c["plat"]), c["size"], c["kernel"]), []).append(c)
    for (plat, size, kernel), cases in list(groups.items())[:6]:
        cfgs = [m.TuningParams(c["wg"], c["ts"]) for c in cases]
        got, info = explore_multi_gpu(m.PlatformConfig(*plat), problem(m, size, kernel), cfgs)
        assert info.states == sum(c["states"] for c in cases)
        for c, g in zip(cases, got):
            key = (plat, size, kernel, c["wg"], c["ts"])
            assert g.complete and g.deadlocks == 0, key
            assert (g.states_visited, g.transitions_applied, g.max_depth_reached) == (
                c["states"], c["transitions"], c["max_depth"]), key
            assert (g.min_time, g.max_time, g.terminals) == (
                c["min_time"], c["max_time"], c["n_terminal"]), key


@pytest.mark.parametrize("parts", [1, 2])
def test_table_overflow_restarts_with_identical_counts(engine, parts, monkeypatch):
    """A first table far too small (2^16 slots for 1.3e5 states) overflows; the
    sweep restarts 8x larger until it fits, and the counts are those of a sweep
    that never overflowed."""
    m = engine
    args = (m.PlatformConfig(1, 2, 8, 4), m.ProblemSpec.abstract(32), [m.TuningParams(16, 2)])
    want = m.explore_configs(*args, partitions=parts)[0]
    monkeypatch.setenv("MCTB_BFS_CAP_LOG2", "16")
    info = []
    got = m.explore_configs(*args, partitions=parts, info=info)[0]
    assert got == want and want.complete and want.states_visited == 131492
    assert info[0].table_slots > (1 << 16) * parts


def test_check_nontermination_matches_reference(engine, gold):
    """check_nontermination (explore.cpp:207-233): the same traces in the same order
    (configuration, final time, length, SHA-256 of the transitions) and the same
    sweep statistics as the reference (nonterm.json); a depth cap of one finds none."""
    import hashlib
    import struct
    m = engine

    def sha(trace):
        return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()

    for c in gold("nonterm.json"):
        key = (tuple(c["plat"]), c["size"], c["kernel"])
        traces, stats = m.check_nontermination(m.PlatformConfig(*c["plat"]),
                                               problem(m, c["size"], c["kernel"]))
        assert len(traces) == c["n"], key
        for t, g in zip(traces, c["traces"]):
            assert (t.params.wg, t.params.ts, t.final_time, t.steps) == \
                (g["wg"], g["ts"], g["final_time"], g["steps"]), key
            assert sha(t.transitions) == g["sha"], key
        assert sum(s.states_visited for s in stats) == c["states"], key
        assert sum(s.transitions_applied for s in stats) == c["transitions"], key
        assert max(s.max_depth_reached for s in stats) == c["max_depth"], key
    traces, _ = m.check_nontermination(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8),
                                       max_depth=1)
    assert traces == []
    # several terminal states per configuration (host re-arming on 2-3 devices), with
    # and without a depth cap: every terminal's DFS path, in DFS order (lexrank.cu)
    for c in gold("nonterm_multi.json"):
        key = (tuple(c["plat"]), c["size"], c["kernel"], c["depth_cap"])
        traces, stats = m.check_nontermination(m.PlatformConfig(*c["plat"]),
                                               problem(m, c["size"], c["kernel"]),
                                               max_depth=c["depth_cap"] or 4_000_000)
        assert len(traces) == c["n"], key
        for t, g in zip(traces, c["traces"]):
            assert (t.params.wg, t.params.ts, t.final_time, t.steps) == \
                (g["wg"], g["ts"], g["final_time"], g["steps"]), key
            assert sha(t.transitions) == g["sha"], key
        assert sum(s.states_visited for s in stats) == c["states"], key
        assert sum(s.transitions_applied for s in stats) == c["transitions"], key
        assert max(s.max_depth_reached for s in stats) == c["max_depth"], key
        assert any(not s.complete for s in stats) == bool(c["limit_hit"]), key
    # a visited set that fills up: the DFS meets only the terminals among the first
    # max_states states of its order (explore.cpp:26-30)
    for c in gold("nonterm_cap.json"):
        key = (tuple(c["plat"]), c["size"], c["kernel"], c["max_states"])
        traces, stats = m.check_nontermination(m.PlatformConfig(*c["plat"]),
                                               problem(m, c["size"], c["kernel"]),
                                               max_states=c["max_states"])
        assert len(traces) == c["n"], key
        for t, g in zip(traces, c["traces"]):
            assert (t.params.wg, t.params.ts, t.final_time, t.steps) == \
                (g["wg"], g["ts"], g["final_time"], g["steps"]), key
            assert sha(t.transitions) == g["sha"], key
        assert sum(s.states_visited for s in stats) == c["states"], key
        assert sum(s.transitions_applied for s in stats) == c["transitions"], key
        assert max(s.max_depth_reached for s in stats) == c["max_depth"], key
        assert any(not s.complete for s in stats) == bool(c["limit_hit"]), key
    with pytest.raises(m.LimitError):  # beyond the 2^22 states the order is ranked over
        m.check_nontermination(m.PlatformConfig(1, 1, 16, 4), m.ProblemSpec.abstract(64),
                               max_states=100_000)


def test_large_explorations_match_independent_counts(engine, gold):
    """The wide exploration workloads (5.6e7 and configs[3]'s 1.37e8 states) against
    the independent CPU counter's states and transitions (tests/golden/large_counts.json)."""
    m = engine
    for c in gold("large_counts.json"):
        x = m.explore_configs(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]),
                              [m.TuningParams(c["wg"], c["ts"])], max_states=400_000_000)[0]
        assert x.complete and (x.states_visited, x.transitions_applied, x.terminals) == (
            c["states"], c["transitions"], c["terminals"]), c
        assert x.max_depth_reached == c["levels"] - 1, c


LEVEL_CASES = [
    # (platform, kernel, size, max_states, max_depth)
    ((1, 1, 4, 4), 0, 64, 5_000_000, 4_000_000),
    ((1, 1, 4, 4), 0, 256, 5_000_000, 4_000_000),
    ((1, 1, 4, 4), 0, 256, 5_000_000, 3000),      # depth cap inside the chains
    ((1, 1, 4, 4), 1, 64, 5_000_000, 4_000_000),  # minimum kernel: tick cycles only
    ((1, 1, 4, 4), 1, 64, 5_000_000, 500),
    ((2, 1, 2, 4), 0, 32, 5_000_000, 4_000_000),  # two devices: handover skew
    ((1, 2, 2, 4), 0, 64, 5_000_000, 4_000_000),
    ((1, 1, 8, 2), 0, 64, 5_000_000, 4_000_000),
    ((3, 1, 1, 1), 1, 32, 5_000_000, 4_000_000),
]


@pytest.mark.parametrize("case", LEVEL_CASES)
def test_level_pass_equals_global_sweep(engine, monkeypatch, case):
    """The narrow-graph pass (level_kernel: one CTA per configuration, level by
    level in shared memory, pure tick cycles and whole reps counted in closed form)
    against the global sweep alone (MCTB_BFS_NOLEVEL), the level pass without
    the closed-form skips (MCTB_BFS_NOSKIP) and the global sweep building every
    successor (MCTB_BFS_NOCANON: no canonical-parent pruning of report and
    arrival successors): every statistic of every configuration equal, with and
    without a depth cap."""
    m = engine
    plat, kernel, size, states, depth = case
    cfgs = [c for c in m.enumerate_configs(size) if kernel == 0 or c.wg * c.ts <= size]
    args = (m.PlatformConfig(*plat), problem(m, size, kernel), cfgs)
    kw = dict(max_states=states, max_depth=depth)
    got = m.explore_configs(*args, **kw)
    monkeypatch.setenv("MCTB_BFS_NOSKIP", "1")
    noskip = m.explore_configs(*args, **kw)
    monkeypatch.setenv("MCTB_BFS_NOLEVEL", "1")
    glob = m.explore_configs(*args, **kw)
    monkeypatch.setenv("MCTB_BFS_NOCANON", "1")  # every successor built and probed
    plain = m.explore_configs(*args, **kw)
    for c, g, n, x, y in zip(cfgs, got, noskip, glob, plain):
        if g.states_visited >= states:
            # a binding visited cap on a graph too deep to rank (lexrank_prefix):
            # the edge count is then the sweep's own, which depends on its order
            assert (g.complete, g.states_visited) == (x.complete, x.states_visited), (case, c)
            continue
        assert g == x == n == y, (case, c)


def test_level_pass_tune_equals_global_sweep(engine, monkeypatch):
    """tune through the level pass and through the global sweep alone: the same
    t_min, parameters, proof, checks and states_visited_total (sizes where the
    reference's goldens stop; tests/golden/tune_large.json pins size 512)."""
    m = engine
    for plat, size in (((1, 1, 4, 4), 128), ((2, 2, 2, 4), 64), ((1, 1, 2, 1), 128)):
        a = m.tune(m.PlatformConfig(*plat), m.ProblemSpec.abstract(size))
        monkeypatch.setenv("MCTB_BFS_NOLEVEL", "1")
        b = m.tune(m.PlatformConfig(*plat), m.ProblemSpec.abstract(size))
        monkeypatch.delenv("MCTB_BFS_NOLEVEL")
        assert (a.t_min, a.params, a.proven, a.stats.checks_run, a.stats.states_visited_total) == (
            b.t_min, b.params, b.proven, b.stats.checks_run, b.stats.states_visited_total), (plat, size)
