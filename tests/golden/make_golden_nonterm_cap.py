"""Golden check_nontermination results of the reference (explore.cpp:207-233)
under a small ExploreLimits::max_states: once a configuration's visited set fills
(explore.cpp:26-30) its DFS meets only the terminal states among the first
max_states states of its order.  Multi-terminal spaces (host re-arming on 2-3
devices) and single-terminal ones.  Recorded from the reference itself
(oracle/_ref); every trace as (wg, ts, final_time, steps, SHA-256).
Re-run with: python tests/golden/make_golden_nonterm_cap.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from checkers import Ref, build_ref  # noqa: E402
from make_golden_nonterm import ref_nonterm  # noqa: E402

CASES = [((3, 1, 1, 1), 32, 1, cap) for cap in (2_000, 30_000, 100_000)] + \
        [((2, 1, 2, 4), 16, 0, cap) for cap in (500, 5_000, 50_000)] + \
        [((3, 1, 1, 4), 16, 1, 3_000), ((1, 1, 4, 4), 16, 0, 300), ((1, 1, 4, 4), 32, 1, 1_000)]


def main():
    assert build_ref()
    ref = Ref()
    cases = []
    for plat, size, kernel, cap in CASES:
        r = ref_nonterm(ref, plat, size, kernel, max_states=cap, rows_cap=4096)
        cases.append({"plat": plat, "size": size, "kernel": kernel, "max_states": cap, **r})
        print(plat, size, kernel, cap, r["n"], r["states"], r["limit_hit"], flush=True)
    with open(os.path.join(HERE, "nonterm_cap.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
        f.write("\n")


if __name__ == "__main__":
    main()
