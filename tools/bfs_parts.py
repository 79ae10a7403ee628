"""Probe: the partitioned exploration (P hash partitions on one GPU) against P = 1."""
import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
for plat, size, c in [((1,1,16,4), 32, (16,2)), ((1,1,8,4), 64, (16,2)), ((2,1,8,4), 32, (8,2))]:
    base = None
    for P, sysm in [(1, False), (2, False), (4, False), (8, False), (1, True), (2, True)]:
        info = []
        r = m.explore_configs(m.PlatformConfig(*plat), m.ProblemSpec.abstract(size), [m.TuningParams(*c)],
                              max_states=400_000_000, info=info, partitions=P, system_scope=sysm)[0]
        key = (r.states_visited, r.transitions_applied, r.min_time, r.max_time, r.terminals, r.complete)
        base = base or key
        print(plat, size, c, 'P', P, 'sys', sysm, key, 'same' if key == base else 'DIFF',
              'Mstates/s', round(r.states_visited / (info[0].kernel_us * 1e-6) / 1e6, 1), flush=True)
