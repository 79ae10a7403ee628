import sys; sys.path.insert(0,'.')
import torch, bench
import paper_2305_09130_b200 as m
from paper_2305_09130_b200.space import space_exact_async
for name, sp in (("headline", bench.SPACE), ("sat", dict(kernel=0, size=1<<24, gmt=100, nd=(1,3000), nu=(1,64), log2np=(0,5), log2wg=(1,23), log2ts=(1,23)))):
    s = m.Space(**sp); n = min(s.count, 10**9)
    d = torch.empty(2, dtype=torch.int64, device="cuda"); st = torch.cuda.current_stream()
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); space_exact_async(s, 0, n, d.data_ptr(), d.data_ptr()+8, st.cuda_stream); e1.record(st)
        torch.cuda.synchronize(); print(name, n, "%.2f ms" % e0.elapsed_time(e1), d.tolist())
    import time; t0=time.perf_counter(); r = m.space_argmin(s, 0, n); print(name, "space_argmin %.2f ms" % ((time.perf_counter()-t0)*1e3), r.time, r.index)
