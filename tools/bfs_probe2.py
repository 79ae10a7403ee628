import sys, time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
plat, size, cfgs = (1,1,16,4), 32, [(16,2)]
if len(sys.argv) > 1:
    plat = tuple(int(x) for x in sys.argv[1].split(','))
    size = int(sys.argv[2]); cfgs = [tuple(int(x) for x in sys.argv[3].split(','))]
info = []
t0 = time.time()
r = m.explore_configs(m.PlatformConfig(*plat), m.ProblemSpec.abstract(size), [m.TuningParams(*c) for c in cfgs], max_states=400_000_000, info=info)
print(plat, size, cfgs, r[0].states_visited, r[0].complete, info[0], 'wall', time.time()-t0, flush=True)
