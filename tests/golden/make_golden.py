"""Generates the golden vectors in tests/golden/*.json FROM THE REFERENCE ITSELF.

Runs the unmodified reference core (/root/reference/proj/src, compiled into
oracle/_ref/libmctune_ref.so by oracle/Makefile) and records its outputs.
The GPU box has no /root/reference: the committed JSON files are what the
tests read there.  Re-run with:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import itertools
import json
import os
import random
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import Ref, build_ref  # noqa: E402


def trace_sha(trace) -> str:
    return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()


def configs(size):
    n = size.bit_length() - 1
    return [(1 << i, 1 << j) for i in range(1, n) for j in range(1, n)]


PLATFORMS = [(1, 1, 4, 4), (1, 1, 2, 1), (1, 2, 2, 4), (2, 2, 2, 4), (1, 1, 8, 2), (1, 1, 1, 2),
             (2, 1, 2, 4), (3, 1, 2, 3), (1, 3, 4, 4), (3, 2, 1, 1), (2, 3, 4, 2), (4, 1, 2, 4)]


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
        f.write("\n")
    print(name, os.path.getsize(os.path.join(HERE, name)), "bytes")


def main():
    assert build_ref(), "the reference must be buildable here (/root/reference)"
    ref = Ref()
    rng = random.Random(20230915)

    launch = []
    for nd, nu, np_ in itertools.product((1, 2, 3), (1, 2, 3, 4), (1, 2, 4, 8)):
        for size in (4, 16, 1024):
            for wg, ts in configs(size):
                launch.append([[nd, nu, np_, 4], size, wg, ts,
                               ref.derive_launch((nd, nu, np_, 4), size, wg, ts)])
    dump("launch.json", launch)

    sweeps = []
    for plat in PLATFORMS:
        for size in (4, 8, 16, 32, 64):
            for kernel in (0, 1):
                sweeps.append({"plat": plat, "size": size, "kernel": kernel,
                               "rows": ref.sweep(plat, size, kernel)})
    dump("sweeps.json", sweeps)

    explore = []
    for plat in PLATFORMS[:8]:
        for size in (4, 8, 16):
            for kernel in (0, 1):
                for wg, ts in configs(size):
                    if kernel == 1 and wg * ts > size:
                        continue
                    r = ref.explore(plat, size, kernel, wg, ts)
                    explore.append({"plat": plat, "size": size, "kernel": kernel, "wg": wg,
                                    "ts": ts, **r})
    dump("explore.json", explore)

    tunes = []
    cases = [((1, 1, 4, 4), s, 0, seed) for s in (4, 8, 16, 32) for seed in (1, 7)]
    cases += [((1, 1, 4, 4), s, 1, seed) for s in (8, 16, 32) for seed in (1, 3)]
    cases += [((2, 1, 2, 4), 16, 0, 1), ((1, 2, 2, 4), 16, 0, 1), ((2, 2, 2, 4), 16, 0, 2),
              ((1, 1, 8, 2), 16, 1, 5), ((1, 1, 2, 1), 32, 0, 9), ((3, 1, 2, 3), 16, 0, 4)]
    for plat, size, kernel, seed in cases:
        r = ref.tune(plat, size, kernel, seed=seed)
        tr = r.pop("trace")
        entry = {"plat": plat, "size": size, "kernel": kernel, "seed": seed, **r,
                 "trace_len": len(tr), "trace_sha": trace_sha(tr)}
        if len(tr) <= 400:
            entry["trace"] = tr
            entry["text"] = ref.trace_text(plat, size, kernel, r["wg"], r["ts"], tr)
        tunes.append(entry)
    dump("tune.json", tunes)

    checks = []
    for T in range(40, 50):
        checks.append(((1, 1, 4, 4), 8, 0, T))
    checks += [((1, 1, 4, 4), 16, 1, T) for T in (20, 22, 23, 24, 100)]
    checks += [((2, 1, 2, 4), 16, 0, T) for T in (150, 167, 168, 500)]
    checks += [((1, 1, 4, 4), 8, 0, 10 ** 9)]
    check_out = []
    for plat, size, kernel, T in checks:
        r = ref.check_overtime(plat, size, kernel, T)
        tr = r.pop("trace")
        check_out.append({"plat": plat, "size": size, "kernel": kernel, "T": T, **r,
                          "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    dump("check.json", check_out)

    sims = []
    for plat in PLATFORMS:
        for size in (8, 16, 32):
            for kernel in (0, 1):
                for wg, ts in configs(size):
                    if kernel == 1 and wg * ts > size:
                        continue
                    if rng.random() > 0.35:
                        continue
                    inp = None
                    if kernel == 1 and rng.random() < 0.5:
                        inp = [rng.randrange(-10 ** 6, 10 ** 6) for _ in range(size)]
                    seed = rng.randrange(1 << 62)
                    for policy, s in ((0, 0), (1, seed)):
                        r = ref.simulate(plat, size, kernel, wg, ts, policy, s, inp, trace=True)
                        tr = r.pop("trace")
                        sims.append({"plat": plat, "size": size, "kernel": kernel, "wg": wg,
                                     "ts": ts, "policy": policy, "seed": s, "input": inp, **r,
                                     "trace_len": len(tr), "trace_sha": trace_sha(tr)})
    dump("simulate.json", sims)

    fps = []
    for plat, size, kernel, wg, ts, seed in [((1, 1, 4, 4), 8, 0, 4, 4, 3),
                                             ((2, 2, 2, 4), 16, 1, 2, 2, 77),
                                             ((3, 1, 2, 3), 16, 0, 2, 4, 5)]:
        tr = ref.simulate(plat, size, kernel, wg, ts, 1, seed, trace=True)["trace"]
        fp = ref.fingerprints(plat, size, kernel, wg, ts, tr)
        fps.append({"plat": plat, "size": size, "kernel": kernel, "wg": wg, "ts": ts,
                    "seed": seed, "trace": tr, "fingerprints": [str(v) for v in fp]})
    dump("fingerprints.json", fps)

if __name__ == "__main__":
    main()
