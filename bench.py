"""Benchmark of the B200 search engine (one JSON line on rank 0).

Workload (BASELINE.json configs[4], the configuration the metric is quoted on
at 1-8 GPUs): exhaustive evaluation of a synthetic tuning space of the
paper's OpenCL use-case model (abstract kernel, size 1024 — the largest
Table-1 size — gmt 4), generalised from the reference's (wg, ts) space to
  wg = 2^1..2^9 x ts = 2^1..2^9 x np (work-items per unit) = 2^0..2^9
  x nu = 1..64 x nd = 1..160000            (8.29e9 configurations)
A step finds the minimal-model-time configuration of the job's shard: every
rank evaluates its own 10^9 configurations (weak scaling) with the cost-model
kernel, and the packed (time << 33 | index) key is min-reduced over ranks with
one NCCL all-reduce.  `value` = configurations evaluated per second by the
whole job; `e2e` is the same through the host-buffer C-ABI call
mctb_space_argmin (descriptor in, winner out, copies + sync in the region).

--impl reference runs the reference's own CPU path for a configuration's
model time (Machine::run, the exhaustive_sweep evaluator, machine.cpp:788-825)
on a bounded random sample of the same space with all host cores.
"""
from __future__ import annotations

import argparse
import json
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
SPACE = dict(kernel=0, size=1024, gmt=4, nd=(1, 160000), nu=(1, 64), log2np=(0, 9),
             log2wg=(1, 9), log2ts=(1, 9))
METRIC = "tuning configs explored/sec (exhaustive argmin of model time)"
UNIT = "configs/s"
WORKLOAD = ("synthetic 8.29e9-configuration tuning space of the paper's abstract OpenCL "
            "use-case model (size 1024, gmt 4; wg x ts x np x nu x nd), 1e9 configurations per "
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
def reference_sample(secs, seed=1, max_index=PER_RANK, threads=None):
    """The reference's CPU evaluator (Machine::run RoundRobin via oracle/_ref, or the
    oracle port when the reference is not built on this machine) on random
    configurations of the benchmark space, all host cores, for ~secs seconds."""
    from concurrent.futures import ThreadPoolExecutor

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import checkers
    kind = "reference"
    try:
        chk = checkers.Ref() if os.path.exists(checkers.REF_SO) else None
    except OSError:
        chk = None
    if chk is None:
        chk, kind = checkers.Oracle(), "port"
    threads = threads or os.cpu_count() or 1
    deadline = time.perf_counter() + secs
    counts = [0] * threads
    steps = [0] * threads

    def worker(w):
        rng = random.Random(seed * 1000 + w)
        while time.perf_counter() < deadline:
            idx = rng.randrange(max_index)
            plat, params = decode(idx)
            r = chk.simulate(plat, SPACE["size"], SPACE["kernel"], params[0], params[1], 0, 0)
            counts[w] += 1  # in-flight work finishing after the deadline is counted and
            steps[w] += r["steps"]  # its time is inside `el` as well

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(worker, range(threads)))
    el = time.perf_counter() - t0
    return sum(counts) / el, kind, threads, sum(counts), sum(steps), el


def decode(index):
    """Index -> ((nd, nu, np, gmt), (wg, ts)) in the documented order (no GPU needed)."""
    s = SPACE
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


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    per_step = []
    for k in range(args.warmup + args.steps):
        secs = 1.0 if k < args.warmup else max(2.0, min(args.cpu_sample_secs,
                                                          120.0 / max(1, args.steps)))
        v, kind, thr, n, st, el = reference_sample(secs, seed=k + 1)
        if k >= args.warmup:
            per_step.append((v, n, st, el))
    value = statistics.mean(p[0] for p in per_step)
    n_tot = sum(p[1] for p in per_step)
    el_tot = sum(p[3] for p in per_step)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el_tot / max(1, len(per_step)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "space": SPACE, "per_rank_configs": PER_RANK},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": kind,
                             "sample": f"{n_tot} random configurations of the space evaluated by "
                                       f"Machine::run (RoundRobin) in {el_tot:.1f} s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ b200
def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2305_09130_b200 as m
    from paper_2305_09130_b200._lib import lib
    from paper_2305_09130_b200.space import space_argmin_async
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

    # ---- roofline of the cost-model kernel: integer issue (thread instructions per
    # second) against the chip's issue peak, 148 SMs x 4 SMSPs x 32 lanes x SM clock
    probe_ops, _ = C.c_double(), C.c_double()
    lib.mctb_int32_peak(C.byref(probe_ops), C.byref(_))
    kern_avg_s = statistics.mean(kern_ms) * 1e-3
    ops_per_cfg = INT_OPS_PER_CONFIG
    achieved = PER_RANK * ops_per_cfg / kern_avg_s
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    clk_mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    peak_issue = sms * 128 * clk_mhz * 1e6

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "space": SPACE, "per_rank_configs": PER_RANK,
                       "time_to_optimum_ms": total_ms / args.steps,
                       "l2": "256 MB flush between timed steps; kernel reads no DRAM",
                       "parallelism": f"shard{world}"},
            "result": {"t_min": win.time, "index": idx, "platform": win.platform.__dict__,
                       "params": win.params.__dict__, "steps": win.steps},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 13 * 8,
                    "d2h_bytes_per_step": 8 + 8 * 8},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "int32", "achieved": achieved / 1e12,
                         "peak": peak_issue / 1e12, "unit": "Tops/s",
                         "frac": achieved / peak_issue, "traffic": None,
                         "kernel": "space_argmin_kernel<0>", "kernel_ms": statistics.mean(kern_ms),
                         "ops_per_config": ops_per_cfg,
                         "alu_pipe_frac_ncu": ALU_PIPE_FRAC_NCU,
                         "peak_source": "nominal INT32 issue rate at the sampled SM clock "
                                        f"({sms} SMs x 128 lanes x {clk_mhz:.0f} MHz); not in "
                                        "MEASURED_PEAKS.json",
                         "probe_peak": probe_ops.value / 1e12},
            "clocks": clk,
        }
        if world == 1 and not args.no_secondary:
            line["secondary"] = secondary_metrics(m, with_reference=not args.no_cpu_baseline,
                                                  sm_clock_mhz=clk_mhz)
        if world == 1 and not args.no_cpu_baseline:
            v, kind, thr, n, st, el = reference_sample(args.cpu_sample_secs)
            line["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": thr, "kind": kind,
                "sample": f"{n} random configurations of the space ({st} transitions) evaluated "
                          f"by the reference's Machine::run (RoundRobin) in {el:.1f} s"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def hbm_peak_gbps():
    """The measured copy bandwidth of this pool (MEASURED_PEAKS.json), else the
    profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def secondary_metrics(m, with_reference=True, sm_clock_mhz=1965.0):
    """The other north-star paths, one measurement each (reported, not the headline):
    time-to-optimum of `tune` (BASELINE configs[0..1] scale), the interleaving
    exploration (configs[3]) and the swarm trajectories (configs[2])."""
    import hashlib
    import struct
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import checkers
    ref = checkers.Ref() if with_reference and os.path.exists(checkers.REF_SO) else None
    out = {}
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
    # (2) exploration of one configuration's full interleaving space (configs[3]:
    # ~10^8 states with the visited-state hash table in HBM)
    import torch
    plat16 = m.PlatformConfig(1, 1, 16, 4)
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
    outdeg = x.transitions_applied / max(1, x.states_visited)
    # algorithmic bytes per state: its slot line written once and read once at
    # expansion, one slot line read per generated successor (the probe), 8 B of queue
    bps = line_bytes * (2 + outdeg) + 8
    hbm_peak, hbm_src = hbm_peak_gbps()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk = sm_clock_mhz
    issue_peak = sms * 4 * clk * 1e6  # warp instructions/s (one issue per SMSP per cycle)
    ex = {"workload": f"explore_machine, abstract kernel, size {EXPLORE_SIZE}, platform (1,1,16,4), "
                      f"(wg,ts)={EXPLORE_PARAMS}: every interleaving",
          "states": x.states_visited, "transitions": x.transitions_applied,
          "complete": x.complete, "kernel_ms": kern_s * 1e3, "api_seconds": wall,
          "cold_api_seconds": cold,
          "states_per_s": rate, "states_per_s_api": x.states_visited / wall,
          "key_words": words, "slot_bytes": line_bytes, "table_slots": info[0].table_slots,
          "roofline": {
              "bound": "latency: dependent L2/HBM round trips per state (probe, claim, queue)",
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
    if ref is not None:
        t0 = time.perf_counter()
        rx = ref.explore((1, 1, 8, 4), 32, 0, 8, 2)
        el = time.perf_counter() - t0
        ex["reference_states_per_s"] = rx["states"] / el
        ex["reference_sample"] = ("explore_machine (1,1,8,4) size 32 (8,2): "
                                  f"{rx['states']} states in {el:.2f} s, 1 core")
    out["explore"] = ex
    # (3) swarm trajectories: 10^6 Philox schedules over every configuration, size 16
    import ctypes as C
    from paper_2305_09130_b200._lib import i32arr, lib
    plat = m.PlatformConfig(1, 1, 4, 4)
    prob = m.ProblemSpec.abstract(16)
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
    out["swarm"] = {"workload": "1e6 Philox4x32-10 schedule trajectories, abstract kernel, size 16, "
                                "(1,1,4,4), all 9 configurations, through mctb_trajectories "
                                "(host buffers: per-trajectory time, transitions, result, status, "
                                "trace hash copied back)",
                    "seconds": el, "trajectories_per_s": ntr / el,
                    "kernel_ms": kern_ms, "trajectories_per_s_kernel": ntr / (kern_ms * 1e-3),
                    "transitions_per_s": steps / el, "min_time": min(outb[0::6][:ntr])}
    if with_reference:
        # the same trajectories replayed by the CPU port (oracle, all host cores)
        from concurrent.futures import ThreadPoolExecutor
        orc = checkers.Oracle()
        threads = os.cpu_count() or 1
        per = 2000
        cfg = [(c.wg, c.ts) for c in cfgs]

        def work(w):
            orc.trajectories((1, 1, 4, 4), 16, 0, cfg, 3, 1, w * per, per)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(threads)))
        cel = time.perf_counter() - t0
        out["swarm"]["cpu_port_trajectories_per_s"] = threads * per / cel
        out["swarm"]["cpu_port_cores"] = threads
    return out


# Thread-level instructions executed per configuration by space_argmin_kernel<0>
# on this workload: ncu smsp__inst_executed.sum x 32 / 1e9 configurations
# (profiles/r01_argmin_v8_ncu.txt).  Re-measured after every kernel change.
INT_OPS_PER_CONFIG = 11.80
# the binding pipe of that kernel in the same capture:
# sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active
ALU_PIPE_FRAC_NCU = 0.814

# configs[3]: the exploration workload (1.37e8 states) and its ncu figures per
# state (smsp__inst_executed.sum / states; DRAM read + write bytes / states),
# re-measured after every change of explore_kernel (profiles/).
EXPLORE_SIZE = 64
EXPLORE_PARAMS = (16, 2)
EXPLORE_INST_PER_STATE = 1071.9  # profiles/r01_explore_v8_ncu.txt
EXPLORE_DRAM_BYTES_PER_STATE = 1038.8


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
