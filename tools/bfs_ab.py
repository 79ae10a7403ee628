"""A/B of the exploration kernels on configs[3] (1.37e8 states) and a tune sweep."""
import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
p16 = m.PlatformConfig(1, 1, 16, 4)
for rep in range(3):
    info = []
    x = m.explore_configs(p16, m.ProblemSpec.abstract(64), [m.TuningParams(16, 2)],
                          max_states=400_000_000, info=info)[0]
    print("configs[3]", x.states_visited, x.transitions_applied, x.complete,
          "kernel_ms %.1f" % (info[0].kernel_us / 1e3),
          "Mstates/s %.1f" % (x.states_visited / (info[0].kernel_us * 1e-6) / 1e6), flush=True)
for size in (128, 256):
    for rep in range(2):
        t0 = time.perf_counter()
        r = m.tune(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(size))
        print("tune", size, r.t_min, r.params, r.stats.states_visited_total,
              "%.3f s" % (time.perf_counter() - t0), flush=True)
