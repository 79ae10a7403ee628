import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
cases = [((1,1,4,4), 64, 0, [(32,2)]), ((1,1,8,4), 32, 0, [(8,2)]), ((1,1,16,4), 32, 0, [(16,2)]),
         ((1,1,4,4), 64, 0, None), ((1,1,8,2), 64, 0, [(8,2),(8,4)])]
for plat, size, kernel, cfgs in cases:
    cfgs = [m.TuningParams(*c) for c in cfgs] if cfgs else m.enumerate_configs(size)
    info = []
    t0 = time.time()
    try:
        r = m.explore_configs(m.PlatformConfig(*plat), m.ProblemSpec.abstract(size), cfgs, max_states=400_000_000, info=info)
    except Exception as e:
        print(plat, size, 'ERR', e); continue
    el = time.time() - t0
    st = sum(x.states_visited for x in r)
    print(plat, size, len(cfgs), 'states', st, 'complete', all(x.complete for x in r), 'slots', info[0].table_slots,
          'words', info[0].key_words, 'kernel_ms', info[0].kernel_us/1e3, 'wall', round(el,3),
          'Mstates/s', round(st/(info[0].kernel_us*1e-6)/1e6, 1), flush=True)
