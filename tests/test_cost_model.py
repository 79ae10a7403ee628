"""The lock-step cost model against the reference.

The GPU cost-model kernel evaluates this closed form; here its CPU statement
(oracle mo_cost_model) is pinned against (a) the reference's Machine::run
(RoundRobin) times and transition counts — the exhaustive_sweep rows — and
(b) the minimum terminal time over ALL interleavings found by the reference's
exhaustive explore_machine, which is what check_overtime / bisect_min_time
decide."""
import itertools
import random

import pytest


def test_cost_model_reproduces_reference_sweeps(oracle, gold):
    for case in gold("sweeps.json"):
        plat, size, kernel = case["plat"], case["size"], case["kernel"]
        for wg, ts, time, transitions, ok, note in case["rows"]:
            t, steps, feasible = oracle.cost_model(plat, size, kernel, wg, ts)
            assert feasible == ok
            if ok:
                assert (t, steps) == (time, transitions), (plat, size, kernel, wg, ts)


def test_cost_model_is_min_over_interleavings(oracle, gold):
    for c in gold("explore.json"):
        t, _, _ = oracle.cost_model(c["plat"], c["size"], c["kernel"], c["wg"], c["ts"])
        assert c["complete"] == 1 and t == c["min_time"], c


def test_tune_optimum_is_cost_model_argmin(oracle, gold):
    """bisect_min_time's (t_min, wg, ts) = argmin of the cost model with the
    reference's tie rule (largest wg, then largest ts)."""
    for c in gold("tune.json"):
        size, kernel = c["size"], c["kernel"]
        n = size.bit_length() - 1
        best = None
        for i in range(n - 1, 0, -1):
            for j in range(n - 1, 0, -1):
                wg, ts = 1 << i, 1 << j
                t, _, ok = oracle.cost_model(c["plat"], size, kernel, wg, ts)
                if ok and (best is None or t < best[0]):
                    best = (t, wg, ts)
        assert best == (c["t_min"], c["wg"], c["ts"]), c["plat"]


@pytest.mark.slow
def test_cost_model_against_reference_exploration_grid(oracle, ref):
    rng = random.Random(11)
    plats = list(itertools.product((1, 2, 3, 4), (1, 2, 3, 5), (1, 2, 4), (1, 2, 5)))
    rng.shuffle(plats)
    for k, plat in enumerate(plats[:16]):
        for size in ((4, 8, 16) if k < 4 else (4, 8)):
            n = size.bit_length() - 1
            for i in range(1, n):
                for j in range(1, n):
                    wg, ts = 1 << i, 1 << j
                    for kernel in (0, 1):
                        if kernel == 1 and wg * ts > size:
                            continue
                        x = ref.explore(plat, size, kernel, wg, ts)
                        t, _, _ = oracle.cost_model(plat, size, kernel, wg, ts)
                        assert x["complete"] and x["min_time"] == t, (plat, size, kernel, wg, ts)


@pytest.mark.slow
def test_cost_model_against_reference_runs_at_bench_scale(oracle, ref):
    """Size 1024 (Table 1's largest) and the bench space's size 16384: the closed
    form's (time, transitions) against the reference's Machine::run (RoundRobin)
    on random configurations with nd / nu / np drawn from the bench ranges, both
    kernels, multi-device plans included (runs of up to ~3e5 transitions)."""
    rng = random.Random(2024)
    checked = multi = 0
    while checked < 72:
        size = rng.choice((1024, 1024, 16384))
        kernel = rng.randint(0, 1)
        n = size.bit_length() - 1
        wg, ts = 1 << rng.randint(1, n - 1), 1 << rng.randint(1, n - 1)
        if rng.random() < 0.3:  # the bench ranges
            plat = (rng.randint(1, 4096), rng.randint(1, 2048), 1 << rng.randint(0, 5), 4)
        else:  # few units per device: several devices share the workgroups
            plat = (rng.randint(2, 64), rng.randint(1, 8), 1 << rng.randint(0, 5), 4)
        t, steps, ok = oracle.cost_model(plat, size, kernel, wg, ts)
        if not ok or steps > 300_000:
            continue
        plan = oracle.derive_launch(plat, size, wg, ts)  # wgs, nwd, nwu, nwe, all_nwe
        if plan[4] + 2 * plan[1] * plan[2] + plan[1] > 6000:
            continue  # keep the reference's O(processes) steps cheap
        r = ref.simulate(plat, size, kernel, wg, ts, policy=0)
        assert (r["time"], r["steps"]) == (t, steps), (plat, size, kernel, wg, ts)
        checked += 1
        multi += plan[1] > 1
    assert multi >= 10
