"""Probe: wall time of single serial runs (mctb_simulate) per policy, with trace capture."""
import sys
import time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
from paper_2305_09130_b200 import machine as mm
size = int(sys.argv[1]) if len(sys.argv) > 1 else 128
plat = m.PlatformConfig(1, 1, 4, 4)
mach = mm.Machine(plat, m.ProblemSpec.abstract(size), m.TuningParams(4, 32))
mach.run(mm.ROUND_ROBIN)
for name in ("ROUND_ROBIN", "MT19937", "FIRST"):
    pol = getattr(mm, name)
    for tr in (None, []):
        t0 = time.perf_counter()
        r = mach.run(pol, seed=1, trace_out=tr)
        el = time.perf_counter() - t0
        print(name, 'trace' if tr is not None else 'notrace', 'steps', r.steps, 'ms', round(el * 1e3, 2),
              'us/step', round(el * 1e6 / max(r.steps, 1), 2), flush=True)
