"""Time-to-optimum of the `tune` flow (estimate_initial_time + bisect_min_time):
the GPU engine against the reference's own C++ core (oracle/_ref) on the
same host, same inputs, results compared field by field.

Usage: python bench_tune.py [--sizes 8,16,32,64] [--ref-timeout 300]
Prints one JSON line per case.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def sha(trace):
    return hashlib.sha256(b"".join(struct.pack("<4i", *t) for t in trace)).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8,16,32,64")
    ap.add_argument("--platforms", default="1,1,4,4")
    ap.add_argument("--kernels", default="0,1")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    import paper_2305_09130_b200 as m
    import checkers
    ref = None
    if not args.no_ref and os.path.exists(checkers.REF_SO):
        ref = checkers.Ref()
    plats = [tuple(int(x) for x in p.split(",")) for p in args.platforms.split(";")]
    # warm-up (context creation, module load)
    m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8))
    cases = [(plat, kernel, size) for plat in plats
             for kernel in (int(k) for k in args.kernels.split(","))
             for size in (int(s) for s in args.sizes.split(","))]
    # every GPU case first, back to back (a GPU left idle through a long host-only
    # reference run starts the next call down-clocked), then the reference runs
    lines, results = [], []
    for plat, kernel, size in cases:
        prob = m.ProblemSpec.abstract(size) if kernel == 0 else m.ProblemSpec.minimum(size)
        t0 = time.perf_counter()
        m.tune(m.PlatformConfig(*plat), prob, seed=1)
        cold_s = time.perf_counter() - t0  # first call: maps a larger visited table
        t0 = time.perf_counter()
        r = m.tune(m.PlatformConfig(*plat), prob, seed=1)
        gpu_s = time.perf_counter() - t0
        results.append(r)
        lines.append({"case": {"platform": plat, "size": size,
                               "kernel": ["abstract", "minimum"][kernel], "seed": 1},
                      "gpu": {"seconds": gpu_s, "cold_seconds": cold_s, "t_min": r.t_min,
                              "wg": r.params.wg, "ts": r.params.ts, "proven": r.proven,
                              "checks_run": r.stats.checks_run,
                              "states_visited_total": r.stats.states_visited_total,
                              "explored_states": r.timings_ms["explored_states"],
                              "timings_ms": r.timings_ms, "trace_steps": r.trace.steps}})
    for (plat, kernel, size), r, line in zip(cases, results, lines):
        if ref is not None:
            t0 = time.perf_counter()
            rr = ref.tune(plat, size, kernel, seed=1)
            ref_s = time.perf_counter() - t0
            same = ((rr["t_min"], rr["wg"], rr["ts"], rr["t_ini"], bool(rr["proven"]),
                     rr["checks_run"], rr["states_visited_total"],
                     rr["first_trail_time"], rr["steps"])
                    == (r.t_min, r.params.wg, r.params.ts, r.t_ini, r.proven,
                        r.stats.checks_run, r.stats.states_visited_total,
                        r.first_trail_time, r.trace.steps)
                    and sha(rr["trace"]) == sha(r.trace.transitions))
            line["reference"] = {"seconds": ref_s, "cores": 1, "t_min": rr["t_min"],
                                 "wg": rr["wg"], "ts": rr["ts"],
                                 "states_visited_total": rr["states_visited_total"]}
            line["identical"] = same
            line["speedup"] = ref_s / line["gpu"]["seconds"]
        print(json.dumps(line), flush=True)

if __name__ == "__main__":
    main()
