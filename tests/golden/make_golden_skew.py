"""Golden check_overtime verdicts of the reference where the violating
configuration is schedule-dependent (its first DFS path is slower than the bound,
so the DFS backtracks into later branches).  Found with the oracle's cost model
and first-path runs; recorded from the reference itself (oracle/_ref).
Re-run with: python tests/golden/make_golden_skew.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import Ref, build_ref  # noqa: E402
from make_golden import trace_sha  # noqa: E402

CASES = [((3, 1, 1, 1), 32, 1, T) for T in (15, 16, 19, 22, 24)] + \
        [((3, 1, 1, 4), 32, 1, T) for T in (60, 61, 80, 99)]
TUNES = [((3, 1, 1, 1), 32, 1, s) for s in (1, 2, 3)] + [((3, 1, 1, 4), 32, 1, s) for s in (1, 5)]


def main():
    assert build_ref()
    ref = Ref()
    checks, tunes = [], []
    for plat, size, kernel, T in CASES:
        r = ref.check_overtime(plat, size, kernel, T)
        tr = r.pop("trace")
        checks.append({"plat": plat, "size": size, "kernel": kernel, "T": T, **r,
                       "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    for plat, size, kernel, seed in TUNES:
        r = ref.tune(plat, size, kernel, seed=seed)
        tr = r.pop("trace")
        tunes.append({"plat": plat, "size": size, "kernel": kernel, "seed": seed, **r,
                      "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    with open(os.path.join(HERE, "skew.json"), "w") as f:
        json.dump({"checks": checks, "tunes": tunes}, f, separators=(",", ":"))
        f.write("\n")
    for c in checks:
        print(c["plat"], c["T"], c["violated"], c["states"], c["transitions"], c["wg"], c["ts"],
              c["final_time"], c["steps"])
    for t in tunes:
        print(t["plat"], t["seed"], t["t_min"], t["states_visited_total"], t["checks_run"])


if __name__ == "__main__":
    main()
