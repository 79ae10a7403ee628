"""Probe: state-space sizes and sweep rates of candidate exploration workloads."""
import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
cases = [((1,1,16,4), 32, (16,2)), ((1,1,16,4), 32, (16,4)), ((1,1,16,4), 64, (16,2)),
         ((1,1,16,4), 64, (16,4)), ((1,2,8,4), 32, (16,2)), ((1,1,8,4), 64, (16,2)), ((1,1,16,2), 32, (16,2)), ((2,1,8,4), 32, (8,2)),
         ((1,1,12,4), 32, (16,2))]
for plat, size, c in cases:
    info = []
    t0 = time.time()
    try:
        r = m.explore_configs(m.PlatformConfig(*plat), m.ProblemSpec.abstract(size), [m.TuningParams(*c)],
                              max_states=400_000_000, info=info)
    except Exception as e:
        print(plat, size, c, 'ERR', e, flush=True); continue
    print(plat, size, c, 'states', r[0].states_visited, 'complete', r[0].complete, 'words', info[0].key_words,
          'kernel_ms', info[0].kernel_us / 1e3, 'Mstates/s', round(r[0].states_visited / (info[0].kernel_us * 1e-6) / 1e6, 1),
          'wall', round(time.time() - t0, 2), flush=True)
