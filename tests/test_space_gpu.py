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
    assert r.key == key
    assert r.index == idx
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


@pytest.mark.parametrize("space_id", range(3))
def test_argmin_windows_match_oracle(engine, oracle, space_id):
    """Many short windows [first, first+count) of large spaces, each against the
    oracle's argmin: every window exercises one thread's run logic (the exact
    small-nd prefix, the saturated prefix, the branch-free recurrence and the
    index tie-break) instead of only the global winner."""
    m = engine
    spaces = [
        m.Space(0, 1 << 10, 4, (1, 160000), (1, 64), (0, 9), (1, 9), (1, 9)),  # bench space
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
