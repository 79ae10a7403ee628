"""GPU cost-model kernel + argmin against the oracle and the reference's outputs."""
import random

import pytest

pytestmark = pytest.mark.gpu


def test_reference_space_argmin_matches_tune(engine, gold):
    m = engine
    for c in gold("tune.json"):
        plat = m.PlatformConfig(*c["plat"])
        prob = (m.ProblemSpec.abstract(c["size"]) if c["kernel"] == 0
                else m.ProblemSpec.minimum(c["size"]))
        r = m.space_argmin(m.Space.reference(plat, prob))
        assert (r.time, r.params.wg, r.params.ts) == (c["t_min"], c["wg"], c["ts"])


def test_sweep_matches_reference(engine, gold):
    m = engine
    for case in gold("sweeps.json"):
        plat = m.PlatformConfig(*case["plat"])
        prob = (m.ProblemSpec.abstract(case["size"]) if case["kernel"] == 0
                else m.ProblemSpec.minimum(case["size"]))
        rows = m.exhaustive_sweep(plat, prob)
        got = [(r.wg, r.ts, r.time, r.transitions, int(r.ok), {"": 0, "infeasible": 1}[r.note])
               for r in rows]
        assert got == [tuple(r) for r in case["rows"]]


@pytest.mark.parametrize("seed", range(12))
def test_generalised_space_argmin_matches_oracle(engine, oracle, seed):
    m = engine
    rng = random.Random(seed)
    logn = rng.randint(2, 24)
    kernel = rng.randint(0, 1)
    nd_lo = rng.randint(1, 40)
    nu_lo = rng.randint(1, 40)
    sp = m.Space(kernel, 1 << logn, rng.randint(1, 9), (nd_lo, nd_lo + rng.randint(0, 60)),
                 (nu_lo, nu_lo + rng.randint(0, 30)), (0, rng.randint(0, 6)))
    count = sp.count
    first = rng.randint(0, count - 1) if rng.random() < 0.5 else 0
    n = min(count - first, 400000)
    r = m.space_argmin(sp, first, n)
    key, t, idx = oracle.space_argmin(list(sp.desc()), first, n)
    # the oracle's (t, idx) is the exact least (time, index); its key is the packed one
    assert r.index == idx and r.time == t
    if (key >> m.KEY_INDEX_BITS) < m.KEY_SAT:
        assert r.key == key
    else:
        assert r.key == (m.KEY_SAT << m.KEY_INDEX_BITS) | idx
    plat, params = sp.decode(idx)
    t2, steps, ok = oracle.cost_model((plat.nd, plat.nu, plat.np, plat.gmt), sp.size, kernel,
                                      params.wg, params.ts)
    assert (r.time, r.steps) == (t2, steps)
    assert (r.platform, r.params) == (plat, params)


def test_eval_table_matches_oracle(engine, oracle):
    import torch
    m = engine
    sp = m.Space(1, 1 << 10, 3, (1, 7), (1, 5), (0, 4))
    n = sp.count
    t = torch.empty(n, dtype=torch.int64, device="cuda")
    s = torch.empty(n, dtype=torch.int64, device="cuda")
    from paper_2305_09130_b200.space import space_eval_async
    space_eval_async(sp, 0, n, t.data_ptr(), s.data_ptr(), torch.cuda.current_stream().cuda_stream)
    t, s = t.cpu().tolist(), s.cpu().tolist()
    for i in range(n):
        plat, params = sp.decode(i)
        want = oracle.cost_model((plat.nd, plat.nu, plat.np, plat.gmt), sp.size, 1, params.wg,
                                 params.ts)
        if want[2]:
            assert (t[i], s[i]) == (want[0], want[1])
        else:
            assert t[i] == -1


@pytest.mark.parametrize("space_id", range(5))
def test_argmin_windows_match_oracle(engine, oracle, space_id):
    """Many short windows [first, first+count) of large spaces, each against the
    oracle's argmin: every window exercises one thread's run logic (the exact
    small-nd prefix, the saturated prefix, the branch-free recurrence and the
    index tie-break) instead of only the global winner."""
    m = engine
    spaces = [
        m.Space(1, 1 << 14, 4, (1, 166830), (1, 2048), (0, 5), (1, 2), (1, 2)),  # bench space
        m.Space(1, 1 << 24, 4, (1, 2670000), (1, 128), (0, 5), (4, 5), (1, 2)),  # rich space
        m.Space(0, 1 << 10, 4, (1, 160000), (1, 64), (0, 9), (1, 9), (1, 9)),  # round-1 bench
        m.Space(1, 1 << 20, 7, (1, 5000), (1, 13), (0, 4), (1, 19), (1, 19)),  # saturating
        m.Space(0, 1 << 6, 2, (3, 700), (2, 9), (0, 3)),
    ]
    sp = spaces[space_id]
    import torch
    from paper_2305_09130_b200.space import space_argmin_async
    stream = torch.cuda.current_stream().cuda_stream
    rng = random.Random(100 + space_id)
    for _ in range(120):
        count = rng.choice([1, 2, 3, 17, 200, 1000, 5000])
        first = rng.randint(0, sp.count - count)
        if rng.random() < 0.3:  # windows starting at small nd
            first -= first % (sp.desc()[4] - sp.desc()[3] + 1)
        # the packed key itself (device-resident call): windows of only infeasible
        # configurations have a key too (saturated time, first index)
        d_key = torch.full((1,), (1 << 63) - 1, dtype=torch.int64, device="cuda")
        space_argmin_async(sp, first, count, d_key.data_ptr(), stream)
        key, t, idx = oracle.space_argmin(list(sp.desc()), first, count)
        assert int(d_key.item()) == key, (space_id, first, count)


def _brute_force(sp, first, count):
    """Exact argmin from the per-configuration time table (no packed key): the least
    time of the feasible configurations, then the least index with that time."""
    import torch
    from paper_2305_09130_b200.space import space_eval_async
    t = torch.empty(count, dtype=torch.int64, device="cuda")
    s = torch.empty(count, dtype=torch.int64, device="cuda")
    space_eval_async(sp, first, count, t.data_ptr(), s.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
    t = torch.where(t < 0, torch.full_like(t, (1 << 63) - 1), t)
    tmin = int(t.min().item())
    idx = int(torch.nonzero(t == tmin)[0].item())
    return tmin, first + idx, int(s[idx].item())


SATURATING = [
    # the round-1 counterexample: every time >= 2^30 - 1, winner index 8706
    ((0, 1 << 24, 100, (1, 3), (1, 2), (0, 2)), 0, None, (1694498916, 8706)),
    # minimum kernel, every feasible time saturated, infeasible indices first
    ((1, 1 << 26, 1 << 14, (1, 2), (1, 2), (0, 1), (13, 25), (12, 25)), 0, None, None),
    # mixed: saturated and unsaturated configurations, windows in both regions
    ((0, 1 << 20, 1000, (1, 4000), (1, 3), (0, 2), (1, 19), (1, 19)), 0, 3_000_000, None),
    ((0, 1 << 20, 1000, (1, 4000), (1, 3), (0, 2), (1, 19), (1, 19)), 17, 500_000, None),
    ((1, 1 << 22, 3, (1, 200), (1, 7), (0, 5), (1, 21), (1, 21)), 0, None, None),
]


@pytest.mark.parametrize("case", range(len(SATURATING)))
def test_space_argmin_exact_against_brute_force(engine, oracle, case):
    """mctb_space_argmin against a brute-force exact-time argmin (not the packed key),
    including spaces whose least time saturates the key's 30-bit time field."""
    m = engine
    args, first, count, want = SATURATING[case]
    sp = m.Space(*args)
    if count is None:
        count = sp.count - first
    t, idx, steps = _brute_force(sp, first, count)
    r = m.space_argmin(sp, first, count)
    assert (r.time, r.index, r.steps) == (t, idx, steps)
    plat, params = sp.decode(idx)
    assert (r.platform, r.params) == (plat, params)
    if want is not None:
        assert (r.time, r.index) == want
    if count <= 400_000:
        _, ot, oi = oracle.space_argmin(list(sp.desc()), first, count)
        assert (ot, oi) == (t, idx)


def test_space_exact_async_matches_brute_force(engine):
    import torch
    from paper_2305_09130_b200.space import space_exact_async
    m = engine
    sp = m.Space(0, 1 << 24, 100, (1, 3), (1, 2), (0, 2))
    d = torch.empty(2, dtype=torch.int64, device="cuda")
    space_exact_async(sp, 0, sp.count, d.data_ptr(), d.data_ptr() + 8,
                      torch.cuda.current_stream().cuda_stream)
    assert d.tolist() == [1694498916, 8706]
    # a range with no feasible configuration: time = 2^64 - 1 (int64 -1)
    sp2 = m.Space(1, 1 << 8, 2, (1, 1), (1, 1), (0, 0), (7, 7), (7, 7))
    space_exact_async(sp2, 0, 1, d.data_ptr(), d.data_ptr() + 8,
                      torch.cuda.current_stream().cuda_stream)
    assert d.tolist() == [-1, -1]
    with pytest.raises(m.ConfigError):
        m.space_argmin(sp2)
