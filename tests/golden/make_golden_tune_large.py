"""Golden `tune` results of the reference (estimate_initial_time + bisect_min_time,
search.cpp:94-158, the `tune` command flow of tools/main.cpp:119-128) at the
paper's large sizes on its use-case platform (1,1,4,4), abstract kernel, seed 1,
default ExploreLimits — configs[1] of BASELINE.json.  Recorded from the reference
itself (oracle/_ref) on one host core: size 512 takes ~66 min, size 1024 hours.
Re-run with: python tests/golden/make_golden_tune_large.py 512 [1024]
(appends / replaces entries in tune_large.json)."""
import hashlib
import json
import os
import struct
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import Ref, build_ref  # noqa: E402


def main():
    assert build_ref()
    ref = Ref()
    path = os.path.join(HERE, "tune_large.json")
    cases = json.load(open(path)) if os.path.exists(path) else []
    for size in (int(a) for a in sys.argv[1:]):
        t0 = time.time()
        r = ref.tune((1, 1, 4, 4), size, 0, seed=1)
        tr = r.pop("trace")
        r["trace_sha"] = hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in tr)).hexdigest()
        r["reference_seconds"] = time.time() - t0
        r.update(plat=[1, 1, 4, 4], size=size, kernel=0, seed=1)
        cases = [c for c in cases if c["size"] != size] + [r]
        print(json.dumps(r), flush=True)
    with open(path, "w") as f:
        json.dump(sorted(cases, key=lambda c: c["size"]), f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
