"""Probe: repeated minimum-kernel tune calls (MCTB_TUNE_TRACE=1 prints the phases)."""
import sys
import time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(128))
for size in (8, 16, 8, 16, 32, 8):
    for rep in range(2):
        t0 = time.perf_counter()
        r = m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.minimum(size), seed=1)
        el = time.perf_counter() - t0
        print(size, rep, round(el * 1e3, 1), {k: round(v, 1) for k, v in r.timings_ms.items()}, flush=True)
