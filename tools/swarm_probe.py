"""Probe: the swarm trajectory kernel (1e6 Philox trajectories, size 16, all configs)."""
import ctypes as C
import sys
import time
sys.path.insert(0, '.')
import paper_2305_09130_b200 as m
from paper_2305_09130_b200._lib import i32arr, lib
size = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ntr = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
plat = m.PlatformConfig(1, 1, 4, 4)
cfgs = m.enumerate_configs(size)
carr = i32arr([v for c in cfgs for v in (c.wg, c.ts)])
outb = (C.c_int64 * (6 * ntr))()
for rep in range(2):
    t0 = time.perf_counter()
    rc = lib.mctb_trajectories(plat.as_array(), size, 0, None, carr, len(cfgs), 3, C.c_uint64(1),
                               C.c_uint64(0), C.c_uint64(ntr), C.c_int64(200_000_000), outb)
    el = time.perf_counter() - t0
    steps = sum(outb[1::6][:ntr])
    kms = lib.mctb_trajectories_kernel_ms()
    print('rc', rc, 'kernel_ms', kms, 'kernel traj/s', ntr / (kms * 1e-3), 'traj/s', ntr / el, 'transitions/s', steps / el, 'steps/traj', steps / ntr, flush=True)
