"""Golden `tune` results of the reference on multi-device / multi-unit platforms
(nd in {2,3}, nu in {1,2}, np in {1,2,4}, gmt in {1,4}, sizes 8 and 16, both
kernels) — the configurations where host re-arming makes some schedules slower
than the lock-step time.  Generated from the reference itself (oracle/_ref);
re-run with: python tests/golden/make_golden_multidevice.py"""
import itertools
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import Ref, build_ref  # noqa: E402
from make_golden import trace_sha  # noqa: E402


def main():
    assert build_ref()
    ref = Ref()
    out = []
    for plat in itertools.product((2, 3), (1, 2), (1, 2, 4), (1, 4)):
        for size in (8, 16):
            for kernel in (0, 1):
                r = ref.tune(plat, size, kernel, seed=1)
                tr = r.pop("trace")
                out.append({"plat": plat, "size": size, "kernel": kernel, "seed": 1, **r,
                            "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    with open(os.path.join(HERE, "tune_multidevice.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
        f.write("\n")
    print(len(out), "cases")


if __name__ == "__main__":
    main()
