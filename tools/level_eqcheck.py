"""Randomised equality check of the narrow-graph level pass (with canonical-parent
pruning) against the global sweep alone building every successor
(MCTB_BFS_NOLEVEL + MCTB_BFS_NOCANON): random platforms, sizes 8-64, both kernels, random depth
caps; every statistic of every configuration compared (states and completeness only
where the 2e6 visited cap binds).  Usage: python tools/level_eqcheck.py SEED SECONDS"""
import os, random, sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
t_end = time.time() + float(sys.argv[2] if len(sys.argv) > 2 else 240)
n = bad = 0
while time.time() < t_end:
    plat = (rng.randint(1, 3), rng.randint(1, 2), 1 << rng.randint(0, 3), rng.randint(1, 4))
    size = rng.choice((8, 16, 32, 64))
    kernel = rng.randint(0, 1)
    inp = [rng.randint(-50, 50) for _ in range(size)] if kernel and rng.random() < 0.5 else None
    prob = m.ProblemSpec.abstract(size) if kernel == 0 else m.ProblemSpec.minimum(size, inp)
    cfgs = [c for c in m.enumerate_configs(size) if kernel == 0 or c.wg * c.ts <= size]
    depth = rng.choice((4_000_000, 4_000_000, rng.randint(20, 3000)))
    states = 2_000_000
    os.environ.pop("MCTB_BFS_NOLEVEL", None)
    t0 = time.time()
    try:
        a = m.explore_configs(m.PlatformConfig(*plat), prob, cfgs, max_states=states, max_depth=depth)
    except m.LimitError:
        continue
    t1 = time.time()
    os.environ["MCTB_BFS_NOLEVEL"] = "1"
    os.environ["MCTB_BFS_NOCANON"] = "1"
    b = m.explore_configs(m.PlatformConfig(*plat), prob, cfgs, max_states=states, max_depth=depth)
    os.environ.pop("MCTB_BFS_NOCANON", None)
    t2 = time.time()
    print("case", plat, size, kernel, depth, "level %.2f s global %.2f s" % (t1 - t0, t2 - t1), flush=True)
    for c, x, y in zip(cfgs, a, b):
        n += 1
        if x.states_visited >= states:
            ok = (x.complete, x.states_visited) == (y.complete, y.states_visited)
        else:
            ok = x == y
        if not ok:
            bad += 1
            print("MISMATCH", plat, size, kernel, c, depth, x, y, flush=True)
print("checked", n, "configurations, mismatches", bad)
