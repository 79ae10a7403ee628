"""Probe: tune wall time vs its exploration kernel time across a size sequence
(MCTB_BFS_TRACE=1 prints every exploration attempt)."""
import sys
import time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8))
for size in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,32,32,64,128,128").split(",")]:
    t0 = time.perf_counter()
    r = m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(size), seed=1)
    el = time.perf_counter() - t0
    print(size, round(el * 1e3, 1), {k: round(v, 1) for k, v in r.timings_ms.items()}, flush=True)
