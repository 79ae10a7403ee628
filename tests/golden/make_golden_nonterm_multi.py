"""Golden check_nontermination results of the reference (explore.cpp:207-233) on
spaces whose configurations end in several distinct terminal states (multi-device
platforms with host re-arming: schedules finish at different times, or in
different states at the same time), with and without a depth cap.  Recorded from
the reference itself (oracle/_ref); every trace as (wg, ts, final_time, steps,
SHA-256).  Re-run with: python tests/golden/make_golden_nonterm_multi.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from checkers import Ref, build_ref  # noqa: E402
from make_golden_nonterm import ref_nonterm  # noqa: E402

CASES = [((2, 1, 2, 4), 8, 0, 0), ((3, 1, 1, 1), 16, 1, 0), ((3, 1, 1, 1), 16, 0, 0),
         ((3, 1, 1, 4), 16, 1, 0), ((2, 1, 2, 4), 16, 0, 0), ((3, 1, 1, 1), 32, 1, 0),
         ((3, 1, 1, 1), 16, 1, 70), ((2, 1, 2, 4), 16, 0, 1000), ((3, 1, 1, 4), 16, 1, 160)]


def main():
    assert build_ref()
    ref = Ref()
    cases = []
    for plat, size, kernel, depth in CASES:
        r = ref_nonterm(ref, plat, size, kernel, max_depth=depth, rows_cap=4096)
        cases.append({"plat": plat, "size": size, "kernel": kernel, "depth_cap": depth, **r})
        print(plat, size, kernel, depth, r["n"], r["states"], r["limit_hit"], flush=True)
    with open(os.path.join(HERE, "nonterm_multi.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
        f.write("\n")


if __name__ == "__main__":
    main()
