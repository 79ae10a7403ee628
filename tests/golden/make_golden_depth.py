"""Golden outputs of the reference under ExploreLimits::max_depth (explore.cpp:124-127):
explore_machine, check_overtime and tune with depth caps that cut some
configurations' runs and not others (single-device platforms and the
schedule-dependent 3-device ones).  Recorded from the reference itself
(oracle/_ref).  Re-run with: python tests/golden/make_golden_depth.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import CheckerError, Oracle, Ref, build_ref  # noqa: E402
from make_golden import configs, trace_sha  # noqa: E402

EXPLORES = [((1, 1, 4, 4), 8, 0, 4, 4, (1, 2, 50, 130, 260, 261, 262, 1000)),
            ((3, 1, 1, 1), 16, 0, 2, 2, (100, 400, 650, 697, 698, 699)),
            ((2, 1, 4, 2), 16, 1, 2, 2, (10, 100, 144, 145, 146)),
            ((2, 2, 2, 3), 16, 0, 2, 2, (300, 700, 843))]
SPACES = [((1, 1, 4, 4), 16, 0), ((1, 1, 4, 4), 32, 1), ((1, 1, 4, 4), 16, 1),
          ((3, 1, 1, 1), 16, 1), ((3, 1, 1, 4), 16, 1), ((2, 1, 2, 4), 16, 0)]


def depths(orc, plat, size, kernel):
    """Terminal depth (protocol transitions + lock-step time) of every feasible configuration."""
    out = []
    for wg, ts in configs(size):
        t, steps, ok = orc.cost_model(plat, size, kernel, wg, ts)
        if ok:
            out.append(steps)
    return sorted(set(out))


def main():
    assert build_ref()
    ref, orc = Ref(), Oracle()
    explores, checks, tunes = [], [], []
    for plat, size, kernel, wg, ts, ks in EXPLORES:
        for k in ks:
            r = ref.explore(plat, size, kernel, wg, ts, max_depth=k)
            explores.append({"plat": plat, "size": size, "kernel": kernel, "wg": wg, "ts": ts,
                             "depth_cap": k, **r})
    for plat, size, kernel in SPACES:
        ds = depths(orc, plat, size, kernel)
        # caps between consecutive configurations' lock-step run lengths, and on them
        ks = sorted({ds[0] - 1, ds[0], ds[len(ds) // 3], (ds[len(ds) // 3] + ds[len(ds) // 3 + 1]) // 2,
                     ds[len(ds) // 2], ds[-1] - 1, ds[-1] + 5})
        t = ref.tune(plat, size, kernel, seed=1)
        for k in ks:
            for T in (t["t_min"], t["t_min"] - 1, t["t_ini"], 10 * t["t_ini"]):
                try:
                    r = ref.check_overtime(plat, size, kernel, T, max_depth=k)
                except CheckerError as e:
                    checks.append({"plat": plat, "size": size, "kernel": kernel, "T": T,
                                   "depth_cap": k, "error": e.rc})
                    continue
                tr = r.pop("trace")
                checks.append({"plat": plat, "size": size, "kernel": kernel, "T": T,
                               "depth_cap": k, **r, "trace_len": len(tr),
                               "trace_sha": trace_sha(tr)})
            try:
                r = ref.tune(plat, size, kernel, seed=1, max_depth=k)
            except CheckerError as e:
                tunes.append({"plat": plat, "size": size, "kernel": kernel, "seed": 1,
                              "depth_cap": k, "error": e.rc})
                continue
            tr = r.pop("trace")
            tunes.append({"plat": plat, "size": size, "kernel": kernel, "seed": 1, "depth_cap": k,
                          **r, "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    with open(os.path.join(HERE, "depth.json"), "w") as f:
        json.dump({"explores": explores, "checks": checks, "tunes": tunes}, f,
                  separators=(",", ":"))
        f.write("\n")
    print(len(explores), "explores", len(checks), "checks", len(tunes), "tunes")
    for c in checks:
        if "error" in c:
            print("check error", c["plat"], c["size"], c["T"], c["depth_cap"], c["error"])
        else:
            print(c["plat"], c["size"], c["T"], c["depth_cap"], c["violated"], c["exhaustive"],
                  c["states"], c["max_depth"], c["wg"], c["ts"], c["steps"])
    for t in tunes:
        print("tune", t["plat"], t["size"], t["depth_cap"], t.get("t_min"), t.get("error"))


if __name__ == "__main__":
    main()
