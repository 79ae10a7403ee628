"""Probe: the deep chain of the tune sweeps — explore_machine of (2,2) on (1,1,4,4)
abstract at a size, alone, and the whole tune at that size."""
import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = m.PlatformConfig(1, 1, 4, 4)
prob = m.ProblemSpec.abstract(size)
for rep in range(2):
    info = []
    x = m.explore_configs(p, prob, [m.TuningParams(2, 2)], info=info)[0]
    print("chain", size, x.states_visited, x.max_depth_reached, x.complete,
          "kernel_ms %.1f" % (info[0].kernel_us / 1e3),
          "us/level %.2f" % (info[0].kernel_us / max(1, x.max_depth_reached)), flush=True)
for rep in range(2):
    t0 = time.perf_counter()
    r = m.tune(p, prob)
    print("tune", size, r.t_min, "%.3f s" % (time.perf_counter() - t0), flush=True)
