"""Probe: tune time at sizes 128-512 and the configs[3] sweep rate (for build-parameter A/B)."""
import sys
import time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(512))
for size in (128, 256, 512):
    best = 1e9
    for _ in range(2):
        t0 = time.perf_counter()
        m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(size), seed=1)
        best = min(best, time.perf_counter() - t0)
    print('tune', size, round(best * 1e3, 1), flush=True)
info = []
m.explore_configs(m.PlatformConfig(1, 1, 16, 4), m.ProblemSpec.abstract(64), [m.TuningParams(16, 2)], max_states=400_000_000)
x = m.explore_configs(m.PlatformConfig(1, 1, 16, 4), m.ProblemSpec.abstract(64), [m.TuningParams(16, 2)], max_states=400_000_000, info=info)[0]
print('explore Mstates/s', round(x.states_visited / (info[0].kernel_us * 1e-6) / 1e6, 1), flush=True)
