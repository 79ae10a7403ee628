"""Golden check_overtime / tune results of the reference under a small
ExploreLimits::max_states (explore.cpp:28-31): the visited set fills before the
DFS meets a satisfying terminal in some configurations (their first path, or the
guided walk's path behind the abandoned siblings' subtrees), which then end with
limit_hit and no verdict.  Recorded from the reference itself (oracle/_ref).
Re-run with: python tests/golden/make_golden_cap.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import CheckerError, Ref, build_ref  # noqa: E402
from make_golden import trace_sha  # noqa: E402

CHECKS = [((3, 1, 1, 1), 16, 1, T, cap) for T in (9, 10, 12, 17) for cap in (200, 1000, 3000, 8000)] + \
         [((1, 1, 4, 4), 16, 0, T, cap) for T in (84, 200) for cap in (100, 300, 600, 2000)] + \
         [((2, 1, 2, 4), 8, 0, T, cap) for T in (44, 60, 88) for cap in (50, 150, 400, 1200)]
TUNES = [((3, 1, 1, 1), 16, 1, cap) for cap in (1000, 3000)] + [((1, 1, 4, 4), 16, 0, cap) for cap in (300, 2000)]


def main():
    assert build_ref()
    ref = Ref()
    checks, tunes = [], []
    for plat, size, kernel, T, cap in CHECKS:
        r = ref.check_overtime(plat, size, kernel, T, max_states=cap)
        tr = r.pop("trace")
        checks.append({"plat": plat, "size": size, "kernel": kernel, "T": T, "max_states": cap, **r,
                       "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    for plat, size, kernel, cap in TUNES:
        try:
            r = ref.tune(plat, size, kernel, seed=1, max_states=cap)
        except CheckerError as e:
            tunes.append({"plat": plat, "size": size, "kernel": kernel, "max_states": cap,
                          "error": e.rc})
            continue
        tr = r.pop("trace")
        tunes.append({"plat": plat, "size": size, "kernel": kernel, "max_states": cap, **r,
                      "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    with open(os.path.join(HERE, "cap.json"), "w") as f:
        json.dump({"checks": checks, "tunes": tunes}, f, separators=(",", ":"))
        f.write("\n")
    for c in checks:
        print(c["plat"], c["size"], c["T"], c["max_states"], c["violated"], c["exhaustive"],
              c["states"], c["wg"], c["ts"], c["steps"])
    for t in tunes:
        print("tune", t["plat"], t["max_states"], t.get("t_min"), t.get("error"))


if __name__ == "__main__":
    main()
