"""Probe: space_argmin over [0, 1e9) of bench.SPACE or bench.RICH_SPACE (for ncu)."""
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
import paper_2305_09130_b200 as m
from paper_2305_09130_b200.space import space_argmin_async
sp = m.Space(**(bench.RICH_SPACE if len(sys.argv) > 1 and sys.argv[1] == "rich" else bench.SPACE))
key = torch.empty(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for rep in range(4):
    key.fill_((1 << 63) - 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    space_argmin_async(sp, 0, 10 ** 9, key.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    print(rep, "%.4f ms" % e0.elapsed_time(e1), key.item() >> 33, key.item() & ((1 << 33) - 1), flush=True)
