"""Benchmark of the B200 search engine (one JSON line on rank 0).

Workload (BASELINE.json configs[4], the configuration the metric is quoted on
at 1-8 GPUs): exhaustive evaluation of a synthetic tuning space of the
paper's OpenCL use-case model (minimum kernel, size 16384, gmt 4), generalised
from the reference's (wg, ts) space to
  wg = 2^1..2^2 x ts = 2^1..2^2 x np (work-items per unit) = 2^0..2^5
  x nu = 1..2048 x nd = 1..166830            (8.20e9 configurations)
A step finds the minimal-model-time configuration of the job's shard: every
rank evaluates its own 10^9 configurations (weak scaling) with the cost-model
kernel, and the packed (time << 33 | index) key is min-reduced over ranks with
one NCCL all-reduce.  `value` = configurations evaluated per second by the
whole job; `e2e` is the same through the host-buffer C-ABI call
mctb_space_argmin (descriptor in, winner out, copies + sync in the region).

Why this space.  Every configuration of it is one the reference can evaluate
(Machine::run numbers processes with 16-bit pids, machine.hpp:76-84, and steps
in O(processes) per transition): the largest has 20,482 processes, and the
reference takes ~1-7 s per configuration on one core.  Within that domain the
launch plan (wgs, nwd, nwu, nwe) varies along nd only while nd * nu < wgs
<= size / 4, so a 10^9-configuration shard holds at most a few 10^4 distinct
plans (21,786 here; 10 in round 1's space).  The kernel's throughput does not
depend on that (it evaluates every configuration with the same branch-free
loop): `secondary.rich_space` times the same kernel on a 2^24-size space whose
rank-0 shard holds 2.13e6 distinct plans (beyond the reference's domain).

--impl reference runs the reference's own CPU path for a configuration's
model time (Machine::run, the exhaustive_sweep evaluator, machine.cpp:788-825)
on random configurations of the same shards, with one worker process per
host core, measured in steady state (configurations completed per second).
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import random
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PER_RANK = 10 ** 9
SPACE = dict(kernel=1, size=1 << 14, gmt=4, nd=(1, 166830), nu=(1, 2048), log2np=(0, 5),
             log2wg=(1, 2), log2ts=(1, 2))
# the same kernel on a space beyond the reference's domain, rich in launch plans
RICH_SPACE = dict(kernel=1, size=1 << 24, gmt=4, nd=(1, 2670000), nu=(1, 128), log2np=(0, 5),
                  log2wg=(4, 5), log2ts=(1, 2))
# distinct (wgs, nwd, nwu, nwe) launch plans, and configurations with nd * nu < wgs
# (the nd digit changes the plan), in each space's rank-0 shard [0, 10^9):
# distinct_plans() below, pinned by tests/test_bench_contract.py
PLANS_SHARD0 = {"distinct_plans": 21786, "nondegenerate_configs": 21753}
RICH_PLANS_SHARD0 = {"distinct_plans": 2126710, "nondegenerate_configs": 2126687}
METRIC = "tuning configs explored/sec (exhaustive argmin of model time)"
UNIT = "configs/s"
WORKLOAD = ("synthetic 8.20e9-configuration tuning space of the paper's OpenCL use-case model "
            "(minimum kernel, size 16384, gmt 4; wg x ts x np x nu x nd), 1e9 configurations per "
            "GPU, allreduce-min of the packed argmin key")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample-secs", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def bench_config(world):
    """The `config` of both arms (identical by construction)."""
    return {"workload": WORKLOAD, "space": SPACE, "per_rank_configs": PER_RANK,
            "shard0": PLANS_SHARD0, "parallelism": f"shard{world}",
            "l2": "256 MB flush between timed steps; the kernel reads no DRAM"}


# ------------------------------------------------------------ space helpers
def decode(index, s=SPACE):
    """Index -> ((nd, nu, np, gmt), (wg, ts)) in the documented order (no GPU needed)."""
    n_nd = s["nd"][1] - s["nd"][0] + 1
    n_nu = s["nu"][1] - s["nu"][0] + 1
    n_np = s["log2np"][1] - s["log2np"][0] + 1
    n_ts = s["log2ts"][1] - s["log2ts"][0] + 1
    index, nd = divmod(index, n_nd)
    index, nu = divmod(index, n_nu)
    index, lnp = divmod(index, n_np)
    wg_d, ts_d = divmod(index, n_ts)
    return ((s["nd"][0] + nd, s["nu"][0] + nu, 1 << (s["log2np"][0] + lnp), s["gmt"]),
            (1 << (s["log2wg"][1] - wg_d), 1 << (s["log2ts"][1] - ts_d)))


def distinct_plans(s, first, count):
    """Distinct launch plans (wgs, nwd, nwu, nwe) of derive_launch (model.cpp:72-88) over
    [first, first+count), and the configurations whose nd digit changes the plan
    (nd * nu < wgs): walks the (wg, ts, np, nu) blocks, nd analytically."""
    logn = s["size"].bit_length() - 1
    n_nd = s["nd"][1] - s["nd"][0] + 1
    n_nu = s["nu"][1] - s["nu"][0] + 1
    n_np = s["log2np"][1] - s["log2np"][0] + 1
    n_ts = s["log2ts"][1] - s["log2ts"][0] + 1
    plans, nondeg = set(), 0
    end = first + count
    for b in range(first // n_nd, (end - 1) // n_nd + 1):
        x = b
        nu = s["nu"][0] + x % n_nu
        x //= n_nu
        lnp = s["log2np"][0] + x % n_np
        x //= n_np
        lts, lwg = s["log2ts"][1] - x % n_ts, s["log2wg"][1] - x // n_ts
        lo = max(first, b * n_nd) - b * n_nd
        hi = min(end, (b + 1) * n_nd) - b * n_nd
        nd_lo, nd_hi = s["nd"][0] + lo, s["nd"][0] + hi - 1
        sh = lwg + lts
        wgs = 1 << (logn - sh) if sh < logn else 1
        nwu, nwe, q = min(wgs, nu), 1 << min(lwg, lnp), wgs // nu
        lim = (wgs - 1) // nu  # nd <= lim  <=>  nd * nu < wgs: nwd = nd
        if nd_lo <= min(nd_hi, lim):
            nondeg += min(nd_hi, lim) - nd_lo + 1
            plans.update((wgs, nd, nwu, nwe) for nd in range(nd_lo, min(nd_hi, lim) + 1))
        if nd_hi > lim:
            plans.add((wgs, q if q else 1, nwu, nwe))
    return {"distinct_plans": len(plans), "nondegenerate_configs": nondeg}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- reference
def _checker():
    """The reference core (oracle/_ref, Machine::run) or, where it is not built, the
    oracle port; and its kind for the JSON line."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import checkers
    try:
        if os.path.exists(checkers.REF_SO):
            return checkers.Ref(), "reference"
    except OSError:
        pass
    return checkers.Oracle(), "port"


def _ref_worker(wid, seed, hi, q):
    """One host core: Machine::run (RoundRobin) on random configurations of [0, hi),
    each result (end time, index, time, transitions) onto q, until killed."""
    chk, _ = _checker()
    rng = random.Random(seed * 1000 + wid)
    while True:
        idx = rng.randrange(hi)
        plat, params = decode(idx)
        r = chk.simulate(plat, SPACE["size"], SPACE["kernel"], params[0], params[1], 0, 0)
        q.put((time.perf_counter(), idx, r["time"], r["steps"]))


class ReferencePool:
    """The reference's evaluator on every host core, in steady state: worker processes
    evaluate random configurations back to back; a measurement window counts the
    configurations completed inside it (no in-flight work is counted, none is cut)."""

    def __init__(self, hi, seed=1, workers=None):
        self.workers = workers or os.cpu_count() or 1
        # spawn, not fork: the GPU arm has CUDA and torch's threads running
        ctx = mp.get_context("spawn")
        self.q = ctx.Queue()
        self.procs = [ctx.Process(target=_ref_worker, args=(w, seed, hi, self.q), daemon=True)
                      for w in range(self.workers)]
        for p in self.procs:
            p.start()
        self.done = []
        _, self.kind = _checker()

    def _drain(self):
        while True:
            try:
                self.done.append(self.q.get_nowait())
            except Exception:
                return

    def window(self, secs):
        """Configurations completed in the next `secs` seconds: (count, seconds, results)."""
        self._drain()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < secs:
            time.sleep(0.05)
            self._drain()
        t1 = time.perf_counter()
        time.sleep(0.1)
        self._drain()
        got = [d for d in self.done if t0 <= d[0] < t1]
        return len(got), t1 - t0, got

    def close(self):
        for p in self.procs:
            p.kill()
        for p in self.procs:
            p.join(timeout=5)


def closed_form_cpu(secs, first, count):
    """The oracle's C closed form (the same cost model, no simulation) on every host
    core over consecutive chunks of [first, first+count): configurations/s."""
    from concurrent.futures import ThreadPoolExecutor
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import checkers
    orc = checkers.Oracle()
    threads = os.cpu_count() or 1
    chunk = 2_000_000
    sd = space_desc(SPACE)
    deadline = time.perf_counter() + secs
    counts = [0] * threads

    def work(w):
        k = 0
        while time.perf_counter() < deadline:
            lo = first + ((w + k * threads) * chunk) % max(1, count - chunk)
            orc.space_argmin(sd, lo, chunk)
            counts[w] += chunk
            k += 1
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    el = time.perf_counter() - t0
    return {"value": sum(counts) / el, "unit": UNIT, "cores": threads,
            "sample": f"{sum(counts)} configurations of the rank-0 shard in {el:.1f} s "
                      "(oracle/mctune_oracle.c mo_space_argmin: the lock-step closed form in C, "
                      "one thread per core)"}


def space_desc(s):
    n = s["size"].bit_length() - 1
    return [s["kernel"], s["size"], s["gmt"], s["nd"][0], s["nd"][1], s["nu"][0], s["nu"][1],
            s["log2np"][0], s["log2np"][1], s["log2wg"][0], s["log2wg"][1], s["log2ts"][0],
            s["log2ts"][1]] if n else []


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    pool = ReferencePool(world * PER_RANK)
    per_step, n_tot, el_tot = [], 0, 0.0
    try:
        secs = max(4.0, min(args.cpu_sample_secs, 120.0 / max(1, args.steps)))
        pool.window(max(2.0, secs))  # fill the pipeline: every core busy
        for k in range(args.warmup + args.steps):
            n, el, _ = pool.window(secs if k >= args.warmup else 1.0)
            if k >= args.warmup:
                per_step.append(n / el)
                n_tot += n
                el_tot += el
    finally:
        pool.close()
    value = n_tot / el_tot if el_tot else 0.0
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el_tot / max(1, len(per_step)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference", "config": bench_config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": pool.workers,
                             "kind": pool.kind,
                             "sample": f"{n_tot} random configurations of the job's shards "
                                       f"evaluated by Machine::run (RoundRobin) in {el_tot:.1f} s "
                                       "of steady state, one worker process per core"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ b200
def _argmin_rate(m, space_dict, first, count, steps, warmup, stream, flush):
    """Device-timed argmin of [first, first+count) of a space: (ms per launch list, key)."""
    import torch
    from paper_2305_09130_b200.space import space_argmin_async
    space = m.Space(**space_dict)
    desc = space.desc()
    key = torch.empty(1, dtype=torch.int64, device="cuda")
    none_key = torch.tensor([(1 << 63) - 1], dtype=torch.int64, device="cuda")
    for _ in range(warmup):
        key.copy_(none_key)
        space_argmin_async(space, first, count, key.data_ptr(), stream.cuda_stream, desc)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        flush.fill_(k)
        key.copy_(none_key)
        ev[k][0].record(stream)
        space_argmin_async(space, first, count, key.data_ptr(), stream.cuda_stream, desc)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev], int(key.item())


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2305_09130_b200 as m
    from paper_2305_09130_b200._lib import lib
    from paper_2305_09130_b200.space import space_argmin_async, space_exact_async
    import ctypes as C

    space = m.Space(**SPACE)
    total = space.count
    assert world * PER_RANK <= total, "space too small for this many ranks"
    first = rank * PER_RANK
    desc = space.desc()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    key = torch.empty(1, dtype=torch.int64, device="cuda")
    none_key = torch.tensor([(1 << 63) - 1], dtype=torch.int64, device="cuda")  # >= every key
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")  # 256 MB > L2
    launches_per_step = 1  # argmin kernel (the key reset is a torch copy)

    def step():
        key.copy_(none_key)
        space_argmin_async(space, first, PER_RANK, key.data_ptr(), sptr, desc)
        if world > 1:
            dist.all_reduce(key, op=dist.ReduceOp.MIN)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(k)  # L2 flush between timed steps (outside the events)
        e0, e1, e2 = ev[k]
        e0.record(stream)
        key.copy_(none_key)
        space_argmin_async(space, first, PER_RANK, key.data_ptr(), sptr, desc)
        e1.record(stream)
        if world > 1:
            dist.all_reduce(key, op=dist.ReduceOp.MIN)
        e2.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    kern_ms = [a.elapsed_time(b) for a, b, c in ev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = tot.item()
    best_key = key.item()
    value = world * PER_RANK * args.steps / (total_ms * 1e-3)
    sat = (best_key >> m.KEY_INDEX_BITS) >= m.KEY_SAT
    assert not sat, "the benchmark space's winner must not saturate the key"

    # winner, exact (GPU point evaluation through the host API on rank 0's view)
    idx = best_key & ((1 << m.KEY_INDEX_BITS) - 1)
    win = m.space_argmin(space, idx, 1)

    # ---- end to end through the host-buffer C ABI (descriptor in, winner out)
    hkey = C.c_uint64()
    hout = (C.c_int64 * 8)()
    e2e_dev = torch.empty(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        lib.mctb_space_argmin(desc, first, PER_RANK, C.byref(hkey), hout)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_times = []
    for k in range(args.steps):
        flush.fill_(k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.mctb_space_argmin(desc, first, PER_RANK, C.byref(hkey), hout)
        if world > 1:
            e2e_dev.fill_(hkey.value)  # H2D of the local key, NCCL min, D2H of the winner
            dist.all_reduce(e2e_dev, op=dist.ReduceOp.MIN)
            _ = e2e_dev.item()
        e2e_times.append(time.perf_counter() - t0)
        assert rc == 0
    e2e_tot = torch.tensor([sum(e2e_times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_value = world * PER_RANK * args.steps / e2e_tot.item()

    # ---- roofline of the cost-model kernel: integer instruction issue against the
    # measured issue rate of integer instructions on this GPU (mctb_int32_peak)
    probe_ops, probe_ms = C.c_double(), C.c_double()
    lib.mctb_int32_peak(C.byref(probe_ops), C.byref(probe_ms))
    kern_avg_s = statistics.mean(kern_ms) * 1e-3
    achieved = PER_RANK * INT_OPS_PER_CONFIG / kern_avg_s
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    clk_mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    nominal = sms * 128 * clk_mhz * 1e6

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": bench_config(world),
            "time_to_optimum_ms": total_ms / args.steps,
            "result": {"t_min": win.time, "index": idx, "platform": win.platform.__dict__,
                       "params": win.params.__dict__, "steps": win.steps},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 13 * 8,
                    "d2h_bytes_per_step": 8 + 8 * 8},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "int32 issue", "achieved": achieved / 1e12,
                         "peak": probe_ops.value / 1e12, "unit": "T inst/s",
                         "frac": achieved / probe_ops.value, "traffic": None,
                         "kernel": "space_argmin_kernel<1>", "kernel_ms": statistics.mean(kern_ms),
                         "inst_per_config": INT_OPS_PER_CONFIG,
                         "inst_source": INT_OPS_SOURCE,
                         "peak_source": "measured: mctb_int32_peak (best of the integer issue "
                                        "probes, csrc/probe.cu) on this GPU in this run",
                         "nominal_issue_peak": nominal / 1e12,
                         "frac_of_nominal": achieved / nominal,
                         "alu_pipe_frac_ncu": ALU_PIPE_FRAC_NCU,
                         "traffic_note": "the kernel reads no DRAM (ncu: a few KB per launch)"},
            "clocks": clk,
        }
        if world == 1 and not args.no_secondary:
            line["secondary"] = secondary_metrics(m, with_reference=not args.no_cpu_baseline,
                                                  sm_clock_mhz=clk_mhz, flush=flush,
                                                  probe_peak=probe_ops.value)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg(m, args.cpu_sample_secs, world)
            line["cpu_closed_form"] = closed_form_cpu(min(5.0, args.cpu_sample_secs), first,
                                                      PER_RANK)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline_leg(m, secs, world):
    """The reference's Machine::run on random configurations of the shard, every host
    core, steady state; each result checked against the GPU's per-configuration
    table (mctb_space_eval_async) for the same index."""
    import torch
    from paper_2305_09130_b200.space import space_eval_async
    pool = ReferencePool(world * PER_RANK, seed=7)
    try:
        pool.window(2.0)
        n, el, got = pool.window(secs)
    finally:
        pool.close()
    space = m.Space(**SPACE)
    t = torch.empty(1, dtype=torch.int64, device="cuda")
    s = torch.empty(1, dtype=torch.int64, device="cuda")
    mism = 0
    checked = sorted({(g[1], g[2], g[3]) for g in pool.done})
    for idx, rt, rs in checked:
        space_eval_async(space, idx, 1, t.data_ptr(), s.data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
        if (int(t.item()), int(s.item())) != (rt, rs):
            mism += 1
    return {"value": n / el, "unit": UNIT, "cores": pool.workers, "kind": pool.kind,
            "sample": f"{n} random configurations of the shard evaluated by the reference's "
                      f"Machine::run (RoundRobin) in {el:.1f} s of steady state, one worker "
                      "process per core",
            "checked_against_gpu": len(checked), "mismatches": mism}


def hbm_peak_gbps():
    """The measured copy bandwidth of this pool (MEASURED_PEAKS.json), else the
    profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def secondary_metrics(m, with_reference=True, sm_clock_mhz=1965.0, flush=None, probe_peak=None):
    """The other north-star paths, one measurement each (reported, not the headline):
    the cost-model kernel on a plan-rich space, time-to-optimum of `tune` (BASELINE
    configs[0..1] scale), the interleaving exploration (configs[3]) and the swarm
    trajectories (configs[2])."""
    import hashlib
    import struct
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import checkers
    ref = checkers.Ref() if with_reference and os.path.exists(checkers.REF_SO) else None
    out = {}
    # (0) the same cost-model kernel on a space with 2.1e6 distinct launch plans in its
    # rank-0 shard, its winner re-derived by the plain exact two-pass kernels
    from paper_2305_09130_b200.space import space_exact_async
    stream = torch.cuda.current_stream()
    ms, rkey = _argmin_rate(m, RICH_SPACE, 0, PER_RANK, 8, 3, stream, flush)
    rich = m.Space(**RICH_SPACE)
    d = torch.empty(2, dtype=torch.int64, device="cuda")
    space_exact_async(rich, 0, PER_RANK, d.data_ptr(), d.data_ptr() + 8, stream.cuda_stream)
    ex_t, ex_i = d.tolist()
    kern_s = statistics.mean(ms) * 1e-3
    out["rich_space"] = {
        "workload": "space_argmin over [0, 1e9) of a 2^24-size minimum-kernel space (beyond the "
                    "reference's 16-bit process ids)", "space": RICH_SPACE, "shard0": RICH_PLANS_SHARD0,
        "configs_per_s": PER_RANK / kern_s, "kernel_ms": statistics.mean(ms),
        "winner": {"key": rkey, "time": rkey >> m.KEY_INDEX_BITS,
                   "index": rkey & ((1 << m.KEY_INDEX_BITS) - 1)},
        "exact_check": {"time": ex_t, "index": ex_i,
                        "equal": (ex_t, ex_i) == (rkey >> m.KEY_INDEX_BITS,
                                                  rkey & ((1 << m.KEY_INDEX_BITS) - 1))},
        "roofline": {"achieved": PER_RANK * RICH_INST_PER_CONFIG / kern_s / 1e12,
                     "peak": (probe_peak or 0) / 1e12, "unit": "T inst/s",
                     "frac": PER_RANK * RICH_INST_PER_CONFIG / kern_s / probe_peak
                     if probe_peak else None,
                     "inst_per_config": RICH_INST_PER_CONFIG, "inst_source": INT_OPS_SOURCE}}
    # (1) tune: paper use case, abstract kernel, size 64 on (1,1,4,4)
    plat, prob = m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(64)
    m.tune(plat, prob)  # warm
    t0 = time.perf_counter()
    r = m.tune(plat, prob, seed=1)
    gpu_s = time.perf_counter() - t0
    tune = {"workload": "tune (estimate_initial_time + bisect_min_time), abstract kernel, size 64, "
                        "platform (1,1,4,4), seed 1",
            "gpu_seconds": gpu_s, "t_min": r.t_min, "wg": r.params.wg, "ts": r.params.ts,
            "proven": r.proven, "states_visited_total": r.stats.states_visited_total,
            "explored_states": r.timings_ms["explored_states"]}
    if ref is not None:
        t0 = time.perf_counter()
        rr = ref.tune((1, 1, 4, 4), 64, 0, seed=1)
        tune["reference_seconds"] = time.perf_counter() - t0
        tune["reference_cores"] = 1
        sha = lambda tr: hashlib.sha256(b"".join(struct.pack("<4i", *x) for x in tr)).hexdigest()  # noqa: E731
        tune["identical"] = ((rr["t_min"], rr["wg"], rr["ts"], rr["t_ini"], bool(rr["proven"]),
                              rr["checks_run"], rr["states_visited_total"], rr["steps"])
                             == (r.t_min, r.params.wg, r.params.ts, r.t_ini, r.proven,
                                 r.stats.checks_run, r.stats.states_visited_total, r.trace.steps)
                             and sha(rr["trace"]) == sha(r.trace.transitions))
    out["tune"] = tune
    # (1b) tune at the paper's largest sizes (BASELINE configs[1]), the result checked
    # against the reference's own run recorded in tests/golden/tune_large.json
    with open(os.path.join(ROOT, "tests", "golden", "tune_large.json")) as f:
        gold = {g["size"]: g for g in json.load(f)}
    large = []
    for size in (512, 1024):
        pl = m.ProblemSpec.abstract(size)
        m.tune(plat, pl)  # warm
        t0 = time.perf_counter()
        r = m.tune(plat, pl, seed=1)
        row = {"size": size, "gpu_seconds": time.perf_counter() - t0, "t_min": r.t_min,
               "wg": r.params.wg, "ts": r.params.ts, "proven": r.proven,
               "checks_run": r.stats.checks_run,
               "states_visited_total": r.stats.states_visited_total}
        g = gold.get(size)
        if g is not None:
            row["reference_seconds_recorded"] = g["reference_seconds"]
            row["reference_cores"] = 1
            row["identical_to_reference"] = (
                (r.t_min, r.params.wg, r.params.ts, r.t_ini, r.proven, r.stats.checks_run,
                 r.stats.states_visited_total, r.trace.steps)
                == (g["t_min"], g["wg"], g["ts"], g["t_ini"], bool(g["proven"]), g["checks_run"],
                    g["states_visited_total"], g["steps"]))
        large.append(row)
    out["tune_large"] = {
        "workload": "tune, abstract kernel, platform (1,1,4,4), seed 1, sizes 512 and 1024 "
                    "(Table 1's largest); reference_seconds_recorded: the reference's tune "
                    "on one core of the build container (tests/golden/make_golden_tune_large.py)",
        "runs": large}
    # (2) exploration of one configuration's full interleaving space (configs[3]:
    # ~10^8 states with the visited-state hash table in HBM)
    plat16 = m.PlatformConfig(1, 1, 16, 4)
    # the global sweep alone (explore_kernel with its HBM table): the level pass's
    # closed-form counts would otherwise cover part of the space
    os.environ["MCTB_BFS_NOLEVEL"] = "1"
    # one warm-up sweep of the same workload: the first call in a process maps the
    # table's HBM into the stream-ordered pool (reported as cold_api_seconds)
    t0 = time.perf_counter()
    m.explore_configs(plat16, m.ProblemSpec.abstract(EXPLORE_SIZE),
                      [m.TuningParams(*EXPLORE_PARAMS)], max_states=400_000_000)
    cold = time.perf_counter() - t0
    info = []
    t0 = time.perf_counter()
    x = m.explore_configs(plat16, m.ProblemSpec.abstract(EXPLORE_SIZE),
                          [m.TuningParams(*EXPLORE_PARAMS)], max_states=400_000_000, info=info)[0]
    wall = time.perf_counter() - t0
    words = info[0].key_words
    line_bytes = 64 if words <= 14 else 128
    kern_s = info[0].kernel_us * 1e-6
    rate = x.states_visited / kern_s
    # algorithmic bytes per state: its slot line written once and read once at
    # expansion, one slot line read per probed successor (the canonical ones,
    # EXPLORE_PROBES_PER_STATE of the outdegree's ~9.7), 8 B of queue
    bps = line_bytes * (2 + EXPLORE_PROBES_PER_STATE) + 8
    hbm_peak, hbm_src = hbm_peak_gbps()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk = sm_clock_mhz
    issue_peak = sms * 4 * clk * 1e6  # warp instructions/s (one issue per SMSP per cycle)
    ex = {"workload": f"explore_machine, abstract kernel, size {EXPLORE_SIZE}, platform (1,1,16,4), "
                      f"(wg,ts)={EXPLORE_PARAMS}: every interleaving",
          "states": x.states_visited, "transitions": x.transitions_applied,
          "complete": x.complete, "states_pinned": x.states_visited == EXPLORE_STATES,
          "kernel_ms": kern_s * 1e3, "api_seconds": wall,
          "cold_api_seconds": cold,
          "states_per_s": rate, "states_per_s_api": x.states_visited / wall,
          "key_words": words, "slot_bytes": line_bytes, "table_slots": info[0].table_slots,
          "path": "global sweep only (MCTB_BFS_NOLEVEL): every state expanded by explore_kernel",
          "roofline": {
              "bound": "instruction issue and dependent L2/HBM round trips per state "
                       "(probe, claim, queue); not HBM bandwidth",
              "probes_per_state": EXPLORE_PROBES_PER_STATE,
              "hbm": {"achieved": bps * rate / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": bps * rate / 1e9 / hbm_peak, "peak_source": hbm_src,
                      "algorithmic_bytes_per_state": bps,
                      "traffic_bytes_per_state": EXPLORE_DRAM_BYTES_PER_STATE,
                      "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum / states "
                                        "(profiles/)"},
              "issue": {"achieved": EXPLORE_INST_PER_STATE * rate / 1e9,
                        "peak": issue_peak / 1e9, "unit": "G warp-inst/s",
                        "frac": EXPLORE_INST_PER_STATE * rate / issue_peak,
                        "warp_inst_per_state": EXPLORE_INST_PER_STATE,
                        "peak_source": f"{sms} SMs x 4 SMSPs x 1 issue/cycle x {clk:.0f} MHz"}}}
    # the same sweep through the multi-GPU exchange path, its 8 hash partitions on
    # this one device (system-scope variant): the exchange's cost, counts equal
    info8 = []
    x8 = m.explore_configs(plat16, m.ProblemSpec.abstract(EXPLORE_SIZE),
                           [m.TuningParams(*EXPLORE_PARAMS)], max_states=400_000_000, info=info8,
                           partitions=8, system_scope=True)[0]
    ex["partitioned_8"] = {"states_per_s": x8.states_visited / (info8[0].kernel_us * 1e-6),
                           "same_counts": (x8.states_visited, x8.transitions_applied)
                           == (x.states_visited, x.transitions_applied),
                           "how": "8 hash partitions on one GPU, system-scope memory operations "
                                  "(the multi-GPU kernel variant)"}
    if ref is not None:
        t0 = time.perf_counter()
        rx = ref.explore((1, 1, 8, 4), 32, 0, 8, 2)
        el = time.perf_counter() - t0
        ex["reference_states_per_s"] = rx["states"] / el
        ex["reference_sample"] = ("explore_machine (1,1,8,4) size 32 (8,2): "
                                  f"{rx['states']} states in {el:.2f} s, 1 core")
    os.environ.pop("MCTB_BFS_NOLEVEL", None)
    out["explore"] = ex
    # (3) swarm trajectories: 10^6 Philox schedules over every configuration, size 16
    import ctypes as C
    from paper_2305_09130_b200._lib import i32arr, lib
    plat = m.PlatformConfig(1, 1, 4, 4)
    cfgs = m.enumerate_configs(16)
    ntr = 1_000_000
    carr = i32arr([v for c in cfgs for v in (c.wg, c.ts)])
    outb = (C.c_int64 * (6 * ntr))()
    lib.mctb_trajectories(plat.as_array(), 16, 0, None, carr, len(cfgs), 3, C.c_uint64(1),
                          C.c_uint64(0), C.c_uint64(4096), C.c_int64(200_000_000), outb)
    t0 = time.perf_counter()
    rc = lib.mctb_trajectories(plat.as_array(), 16, 0, None, carr, len(cfgs), 3, C.c_uint64(1),
                               C.c_uint64(0), C.c_uint64(ntr), C.c_int64(200_000_000), outb)
    el = time.perf_counter() - t0
    assert rc == 0
    kern_ms = lib.mctb_trajectories_kernel_ms()
    steps = sum(outb[1::6][:ntr])
    rate_k = ntr / (kern_ms * 1e-3)
    out["swarm"] = {"workload": "1e6 Philox4x32-10 schedule trajectories, abstract kernel, size 16, "
                                "(1,1,4,4), all 9 configurations, through mctb_trajectories "
                                "(host buffers: per-trajectory time, transitions, result, status, "
                                "trace hash copied back)",
                    "seconds": el, "trajectories_per_s": ntr / el,
                    "kernel_ms": kern_ms, "trajectories_per_s_kernel": rate_k,
                    "transitions_per_s": steps / el, "min_time": min(outb[0::6][:ntr]),
                    "roofline": {"bound": "issue (serial per-trajectory enabled() scan)",
                                 "achieved": SWARM_INST_PER_TRAJ * rate_k / 1e12,
                                 "peak": (probe_peak or 0) / 1e12, "unit": "T inst/s",
                                 "frac": SWARM_INST_PER_TRAJ * rate_k / probe_peak
                                 if probe_peak else None,
                                 "inst_per_trajectory": SWARM_INST_PER_TRAJ,
                                 "inst_source": SWARM_INST_SOURCE}}
    # every trajectory is reproducible on the CPU from its id: replay a random sample of
    # 10^4 (40 blocks of 250) with the oracle port and compare all six outputs
    orc = checkers.Oracle()
    rng = random.Random(12345)
    cfg = [(c.wg, c.ts) for c in cfgs]
    mism, checked = 0, 0
    for b in rng.sample(range(ntr // 250), 40):
        cols = orc.trajectories((1, 1, 4, 4), 16, 0, cfg, 3, 1, b * 250, 250)
        for i in range(250):
            g = outb[6 * (b * 250 + i):6 * (b * 250 + i) + 6]
            want = (cols[0][i], cols[1][i], cols[2][i], cols[3][i], cols[4][i], cols[5][i])
            got = (g[0], g[1], None if g[2] == -(1 << 63) else g[2], g[3],
                   g[4] & ((1 << 64) - 1), g[5])
            mism += got != want
            checked += 1
    out["swarm"]["cpu_replay"] = {"checked": checked, "mismatches": mism,
                                  "how": "oracle port mo_trajectories (Philox4x32-10 by "
                                         "trajectory id), time/transitions/result/status/"
                                         "trace FNV-1a hash/config"}
    if with_reference:
        # the same trajectories replayed by the CPU port (oracle, all host cores)
        from concurrent.futures import ThreadPoolExecutor
        threads = os.cpu_count() or 1
        per = 2000

        def work(w):
            orc.trajectories((1, 1, 4, 4), 16, 0, cfg, 3, 1, w * per, per)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex_:
            list(ex_.map(work, range(threads)))
        cel = time.perf_counter() - t0
        out["swarm"]["cpu_port_trajectories_per_s"] = threads * per / cel
        out["swarm"]["cpu_port_cores"] = threads
    return out


# Thread-level instructions executed per configuration by space_argmin_kernel<1>
# on the headline workload (and on the rich space): ncu smsp__inst_executed.sum x 32
# / 1e9 configurations.  Re-measured after every kernel change.
INT_OPS_PER_CONFIG = 9.69  # 3.029e8 warp inst / 1e9 (profiles/r02_argmin_v9_ncu.txt)
RICH_INST_PER_CONFIG = 9.38  # 2.931e8 warp inst / 1e9 (profiles/r02_argmin_v9_rich_ncu.csv)
INT_OPS_SOURCE = "ncu smsp__inst_executed.sum x 32 / configurations (profiles/r02_argmin_*)"
# the binding pipe of that kernel in the same capture:
# sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active
ALU_PIPE_FRAC_NCU = 0.787
# thread instructions per trajectory of traj_kernel on the swarm workload (ncu)
SWARM_INST_PER_TRAJ = 372337.0  # 1.1636e10 warp inst / 1e6 trajectories
SWARM_INST_SOURCE = "ncu smsp__inst_executed.sum x 32 / trajectories (profiles/r02_swarm_traj_ncu.csv)"

# configs[3]: the exploration workload (1.37e8 states) and its ncu figures per
# state (smsp__inst_executed.sum / states; DRAM read + write bytes / states),
# re-measured after every change of explore_kernel (profiles/).
EXPLORE_SIZE = 64
EXPLORE_PARAMS = (16, 2)
EXPLORE_STATES = 137_145_999  # pinned by the independent CPU count (tests/golden/large_counts.json)
EXPLORE_INST_PER_STATE = 938.1  # profiles/r02_explore_canon_ncu.txt
EXPLORE_DRAM_BYTES_PER_STATE = 325.0
# table probes per state (MCTB_BFS_OPHIST diagnostics): canonical-parent pruning
# builds and probes 225,402,137 of the 1,326,882,267 successors
EXPLORE_PROBES_PER_STATE = 1.644


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
