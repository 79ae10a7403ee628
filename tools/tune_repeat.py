import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
p = m.PlatformConfig(1, 1, 4, 4)
for rep in range(3):
    for prob in (m.ProblemSpec.abstract(8), m.ProblemSpec.minimum(8), m.ProblemSpec.minimum(16), m.ProblemSpec.abstract(64)):
        t0 = time.perf_counter(); r = m.tune(p, prob); el = time.perf_counter() - t0
        print(rep, prob.size, prob.kernel, r.t_min, '%.1f ms' % (el * 1e3), {k: round(v, 2) for k, v in r.timings_ms.items()}, flush=True)
