"""The GPU bound-lowering driver against the reference's own tune / check results."""
import hashlib
import struct

import pytest

pytestmark = pytest.mark.gpu


def sha(trace):
    return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()


def problem(m, size, kernel):
    return m.ProblemSpec.abstract(size) if kernel == 0 else m.ProblemSpec.minimum(size)


def test_tune_bit_exact_with_reference(engine, gold):
    """T_min, (wg, ts), T_ini, proven, checks_run, states_visited_total,
    first-trail time and the counterexample trace itself."""
    m = engine
    for c in gold("tune.json"):
        r = m.tune(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]), seed=c["seed"])
        key = (c["plat"], c["size"], c["kernel"], c["seed"])
        assert (r.t_min, r.params.wg, r.params.ts) == (c["t_min"], c["wg"], c["ts"]), key
        assert r.t_ini == c["t_ini"] and r.first_trail_time == c["first_trail_time"], key
        assert r.proven == bool(c["proven"]), key
        assert r.stats.checks_run == c["checks_run"], key
        assert r.stats.states_visited_total == c["states_visited_total"], key
        assert r.trace_exact and r.trace.steps == c["steps"] == c["trace_len"], key
        assert sha(r.trace.transitions) == c["trace_sha"], key


def test_check_overtime_bit_exact_with_reference(engine, gold):
    m = engine
    for c in gold("check.json"):
        v = m.check_overtime(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]),
                             c["T"])
        key = (c["plat"], c["size"], c["kernel"], c["T"])
        assert (v.violated, v.exhaustive) == (bool(c["violated"]), bool(c["exhaustive"])), key
        assert v.stats.states_visited == c["states"], key
        assert v.stats.transitions_applied == c["transitions"], key
        assert v.stats.max_depth_reached == c["max_depth"], key
        assert (v.stats.configs_explored, v.stats.configs_skipped) == (
            c["configs_explored"], c["configs_skipped"]), key
        if v.violated:
            assert (v.trace.final_time, v.trace.params.wg, v.trace.params.ts, v.trace.steps) == (
                c["final_time"], c["wg"], c["ts"], c["steps"]), key
            assert sha(v.trace.transitions) == c["trace_sha"], key


def test_paper_table1_row1_and_boundary(engine):
    """Acceptance 1-2: size 8 -> T_min 44 at (4, 4); check(T_min) violated,
    check(T_min - 1) holds exhaustively; verdicts monotone on a 10-point grid."""
    m = engine
    p, prob = m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8)
    r = m.tune(p, prob)
    assert (r.t_min, r.params.wg, r.params.ts, r.proven) == (44, 4, 4, True)
    assert m.check_overtime(p, prob, 44).violated
    below = m.check_overtime(p, prob, 43)
    assert not below.violated and below.exhaustive
    for T in range(40, 50):
        assert m.check_overtime(p, prob, T).violated == (T >= 44)
    assert m.extract_params(p, prob, r.trace) == (4, 4, 44)


def test_bisect_errors(engine):
    m = engine
    p, prob = m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8)
    with pytest.raises(m.ConfigError):
        m.bisect_min_time(p, prob, 43)
    r = m.bisect_min_time(p, prob, 100)
    assert r.t_min == 44 and r.stats.checks_run <= 9


def test_swarm_matches_bisection_at_desk_scale(engine, oracle):
    """Acceptance 4: the swarm optimum equals bisection's (never below it), its
    trace replays, and the best trajectory replays on the CPU from its id."""
    m = engine
    p = m.PlatformConfig(1, 1, 4, 4)
    for prob in (m.ProblemSpec.abstract(8), m.ProblemSpec.abstract(16), m.ProblemSpec.minimum(16)):
        b = m.tune(p, prob)
        s = m.swarm_min_time(p, prob, workers=4, seed=9)
        assert s.t_min == b.t_min and not s.proven
        assert (s.params.wg, s.params.ts) == (b.params.wg, b.params.ts)
        assert m.replay(p, prob, s.trace)[0] == s.t_min
        o = oracle.simulate((1, 1, 4, 4), prob.size, prob.kernel, s.params.wg, s.params.ts,
                            policy=3, seed=9, traj=s.best_trajectory, trace=True)
        assert o["time"] == s.t_min and [tuple(t) for t in o["trace"]] == s.trace.transitions
    a = m.swarm_min_time(p, m.ProblemSpec.abstract(8), workers=1, seed=11)
    b2 = m.swarm_min_time(p, m.ProblemSpec.abstract(8), workers=1, seed=11)
    assert a.trace.transitions == b2.trace.transitions
    with pytest.raises(m.ConfigError):
        m.swarm_min_time(p, m.ProblemSpec.abstract(8), workers=0)


def test_rank_trails_contract(engine):
    m = engine
    mk = lambda t, wg, ts, st: m.Trace([], t, m.TuningParams(wg, ts), st)  # noqa: E731
    r = m.rank_trails([mk(50, 2, 2, 10), mk(44, 4, 4, 1700), mk(44, 2, 4, 1650)])
    assert [(x.time, x.transitions) for x in r] == [(44, 1650), (44, 1700), (50, 10)]
    assert m.rank_trails([]) == []


def _tune_matches(m, c):
    r = m.tune(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]), seed=c["seed"])
    key = (c["plat"], c["size"], c["kernel"], c["seed"])
    assert (r.t_min, r.params.wg, r.params.ts) == (c["t_min"], c["wg"], c["ts"]), key
    assert (r.t_ini, r.first_trail_time, r.proven) == (
        c["t_ini"], c["first_trail_time"], bool(c["proven"])), key
    assert (r.stats.checks_run, r.stats.states_visited_total) == (
        c["checks_run"], c["states_visited_total"]), key
    assert r.trace.steps == c["steps"] and sha(r.trace.transitions) == c["trace_sha"], key


def test_tune_bit_exact_on_multi_device_platforms(engine, gold):
    """96 platforms with nd in {2,3}, nu in {1,2}: host re-arming makes some
    schedules slower than the lock-step time."""
    for c in gold("tune_multidevice.json"):
        _tune_matches(engine, c)


def test_schedule_dependent_counterexamples(engine, gold):
    """Bounds where the violating configuration's first DFS path is too slow:
    the reference's DFS backtracks; the GPU reproduces its counterexample
    (guided walk) and its search effort (sibling exploration)."""
    m = engine
    g = gold("skew.json")
    for c in g["checks"]:
        v = m.check_overtime(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]),
                             c["T"])
        key = (c["plat"], c["size"], c["T"])
        assert v.violated and v.trace_exact, key
        assert (v.trace.final_time, v.trace.params.wg, v.trace.params.ts, v.trace.steps) == (
            c["final_time"], c["wg"], c["ts"], c["steps"]), key
        assert sha(v.trace.transitions) == c["trace_sha"], key
        assert (v.stats.states_visited, v.stats.transitions_applied) == (
            c["states"], c["transitions"]), key
        # the deepest state the DFS met: the path or the abandoned siblings' subtrees
        assert v.stats.max_depth_reached == c["max_depth"], key
    for c in g["tunes"]:
        _tune_matches(m, c)


def test_tune_probes_are_the_per_bound_checks(engine, gold):
    """Every bound the bisection probes is reported with the verdict and the
    counterexample check_overtime(T) returns on its own (the reference's per-bound
    counterexamples), and they add up to checks_run / states_visited_total."""
    m = engine
    for c in gold("tune.json")[:8]:
        plat = m.PlatformConfig(*c["plat"])
        prob = (m.ProblemSpec.abstract(c["size"]) if c["kernel"] == 0
                else m.ProblemSpec.minimum(c["size"]))
        r = m.tune(plat, prob, seed=1)
        assert len(r.probes) == r.stats.checks_run
        assert sum(p.states_visited for p in r.probes) == r.stats.states_visited_total
        assert r.probes[0].T == r.t_ini and r.probes[0].final_time == r.first_trail_time
        for p in r.probes:
            v = m.check_overtime(plat, prob, p.T)
            assert (p.violated, p.exhaustive, p.states_visited) == (
                v.violated, v.exhaustive, v.stats.states_visited), (c, p.T)
            if v.violated:
                assert (p.wg, p.ts, p.final_time, p.steps) == (
                    v.trace.params.wg, v.trace.params.ts, v.trace.final_time, v.trace.steps)


def test_depth_cap_matches_reference(engine, gold):
    """ExploreLimits::max_depth (explore.cpp:124-127) against the reference: the
    DFS applies no transition past the cap, so some configurations' runs are cut
    (limit_hit, not exhaustive) and their terminals are unreachable — explore,
    check_overtime (single-device and schedule-dependent spaces, violated and
    not) and tune, whose optimum moves when the cap hides the best runs."""
    m = engine
    g = gold("depth.json")
    for c in g["explores"]:
        r = m.explore_machine(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]),
                              m.TuningParams(c["wg"], c["ts"]), max_depth=c["depth_cap"])
        key = (c["plat"], c["size"], c["wg"], c["ts"], c["depth_cap"])
        assert (r.complete, r.states_visited, r.transitions_applied, r.max_depth_reached) == (
            bool(c["complete"]), c["states"], c["transitions"], c["max_depth"]), key
        assert (r.terminals, r.min_time, r.max_time) == (c["n_terminal"], c["min_time"],
                                                         c["max_time"]), key
    for c in g["checks"]:
        plat, prob = m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"])
        key = (c["plat"], c["size"], c["kernel"], c["T"], c["depth_cap"])
        v = m.check_overtime(plat, prob, c["T"], max_depth=c["depth_cap"])
        assert (v.violated, v.exhaustive) == (bool(c["violated"]), bool(c["exhaustive"])), key
        assert (v.stats.states_visited, v.stats.transitions_applied, v.stats.max_depth_reached) == (
            c["states"], c["transitions"], c["max_depth"]), key
        assert (v.stats.configs_explored, v.stats.configs_skipped) == (
            c["configs_explored"], c["configs_skipped"]), key
        if v.violated:
            assert (v.trace.final_time, v.trace.params.wg, v.trace.params.ts, v.trace.steps) == (
                c["final_time"], c["wg"], c["ts"], c["steps"]), key
            assert sha(v.trace.transitions) == c["trace_sha"], key
    for c in g["tunes"]:
        plat, prob = m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"])
        if "error" in c:
            with pytest.raises(m.ConfigError):
                m.tune(plat, prob, seed=c["seed"], max_depth=c["depth_cap"])
            continue
        r = m.tune(plat, prob, seed=c["seed"], max_depth=c["depth_cap"])
        key = (c["plat"], c["size"], c["kernel"], c["depth_cap"])
        assert (r.t_min, r.params.wg, r.params.ts, r.t_ini, r.proven) == (
            c["t_min"], c["wg"], c["ts"], c["t_ini"], bool(c["proven"])), key
        assert (r.stats.checks_run, r.stats.states_visited_total, r.first_trail_time) == (
            c["checks_run"], c["states_visited_total"], c["first_trail_time"]), key
        assert r.trace.steps == c["steps"] and sha(r.trace.transitions) == c["trace_sha"], key
    with pytest.raises(m.ConfigError):
        m.check_overtime(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8), 44, max_depth=0)


def test_tune_at_large_sizes_matches_reference(engine, gold):
    """configs[1]: `tune` on the paper's platform at size 512 (and 1024 when its
    reference run is recorded) against the reference's own run (~66 min on one
    core at 512): every result field and the counterexample trace."""
    m = engine
    for c in gold("tune_large.json"):
        r = m.tune(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]), seed=c["seed"])
        key = c["size"]
        assert (r.t_min, r.params.wg, r.params.ts, r.t_ini, r.proven) == (
            c["t_min"], c["wg"], c["ts"], c["t_ini"], bool(c["proven"])), key
        assert (r.stats.checks_run, r.stats.states_visited_total, r.first_trail_time) == (
            c["checks_run"], c["states_visited_total"], c["first_trail_time"]), key
        assert r.trace.steps == c["steps"] and sha(r.trace.transitions) == c["trace_sha"], key


def test_visited_cap_matches_reference(engine, gold):
    """A small max_states (explore.cpp:28-31): a configuration whose satisfying
    terminal lies beyond the visited set's capacity in the DFS's order (its first
    path, or the guided walk's path behind the abandoned siblings' subtrees) ends
    capped with no verdict and the check moves on, as the reference does.  The
    verdicts, states_visited, counterexamples and tune results match, and so do
    transitions_applied and max_depth_reached, which under a binding cap depend on
    the DFS order (derived from the least-path ranking, lexrank_prefix)."""
    m = engine
    g = gold("cap.json")
    for c in g["checks"]:
        key = (c["plat"], c["size"], c["T"], c["max_states"])
        v = m.check_overtime(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]),
                             c["T"], max_states=c["max_states"])
        assert (v.violated, v.exhaustive, v.stats.states_visited) == (
            bool(c["violated"]), bool(c["exhaustive"]), c["states"]), key
        assert (v.stats.transitions_applied, v.stats.max_depth_reached) == (
            c["transitions"], c["max_depth"]), key
        if v.violated:
            assert (v.trace.final_time, v.trace.params.wg, v.trace.params.ts, v.trace.steps) == (
                c["final_time"], c["wg"], c["ts"], c["steps"]), key
            assert sha(v.trace.transitions) == c["trace_sha"], key
    for c in g["tunes"]:
        key = (c["plat"], c["size"], c["max_states"])
        r = m.tune(m.PlatformConfig(*c["plat"]), problem(m, c["size"], c["kernel"]), seed=1,
                   max_states=c["max_states"])
        assert (r.t_min, r.params.wg, r.params.ts, r.t_ini, r.proven) == (
            c["t_min"], c["wg"], c["ts"], c["t_ini"], bool(c["proven"])), key
        assert (r.stats.checks_run, r.stats.states_visited_total) == (
            c["checks_run"], c["states_visited_total"]), key
        assert r.trace.steps == c["steps"] and sha(r.trace.transitions) == c["trace_sha"], key


def test_guided_walk_sweeps_equal_without_pruning(engine, monkeypatch):
    """The guided walk's sibling sweep starts from arbitrary states, where the
    canonical-parent pruning of explore_kernel would lose states whose canonical
    parent lies outside the siblings' reach: it runs unpruned.  Verdicts and
    statistics over a range of bounds on schedule-dependent spaces equal those of
    the engine with pruning switched off everywhere (MCTB_BFS_NOCANON)."""
    m = engine
    cases = [((2, 1, 2, 4), m.ProblemSpec.abstract(16)), ((3, 1, 1, 1), m.ProblemSpec.minimum(16)),
             ((2, 1, 2, 4), m.ProblemSpec.abstract(32)), ((3, 1, 1, 4), m.ProblemSpec.minimum(16))]
    for plat, prob in cases:
        t = m.tune(m.PlatformConfig(*plat), prob)
        for T in range(t.t_min - 2, t.t_ini + 1, max(1, (t.t_ini - t.t_min) // 12)):
            monkeypatch.delenv("MCTB_BFS_NOCANON", raising=False)
            a = m.check_overtime(m.PlatformConfig(*plat), prob, T)
            monkeypatch.setenv("MCTB_BFS_NOCANON", "1")
            b = m.check_overtime(m.PlatformConfig(*plat), prob, T)
            key = (plat, prob.size, T)
            assert (a.violated, a.exhaustive, a.stats.states_visited) == (
                b.violated, b.exhaustive, b.stats.states_visited), key
            if a.exhaustive:
                # (otherwise a configuration capped on a graph beyond the ranking's
                # bound may contribute its sweep's own, order-dependent edge count)
                assert (a.stats.transitions_applied, a.stats.max_depth_reached) == (
                    b.stats.transitions_applied, b.stats.max_depth_reached), key
            if a.violated:
                assert (a.trace.final_time, a.trace.steps, a.trace.transitions) == (
                    b.trace.final_time, b.trace.steps, b.trace.transitions), key
