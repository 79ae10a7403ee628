"""Reachable-state and transition counts of exploration workloads too large for
the reference's DFS (its visited set of serialized states needs more than this
host's 62 GB at 1.4e8 states), from the independent CPU counter
oracle/count_states.c (a level-synchronous BFS over the oracle's successor
function with 128-bit fingerprints; the oracle is pinned against the reference
in tests/test_oracle.py).  Re-run with: python tests/golden/make_golden_counts.py
(size 32: ~8 min, size 64: ~20 min on 6 threads)."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CASES = [((1, 1, 16, 4), 32, 0, 16, 2, 27), ((1, 1, 16, 4), 64, 0, 16, 2, 28)]


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "count_states"], check=True)
    exe = os.path.join(ROOT, "oracle", "_build", "count_states")
    out = []
    for plat, size, kernel, wg, ts, lg in CASES:
        r = subprocess.run([exe, *map(str, plat), str(size), str(kernel), str(wg), str(ts), str(lg),
                            str(os.cpu_count() or 4)], capture_output=True, text=True, check=True)
        d = json.loads(r.stdout)
        d.update(plat=list(plat), size=size, kernel=kernel, wg=wg, ts=ts)
        out.append(d)
        print(d, flush=True)
    with open(os.path.join(HERE, "large_counts.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    sys.exit(main())
