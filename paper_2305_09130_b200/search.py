"""Auto-tuning drivers (reference: include/mctune/search.hpp, explore.hpp).

Same names, arguments and results as the reference's drivers; the model time
of every configuration, the explorations and the counterexample traces are
computed on the GPU through the C ABI (include/mctune_b200.h).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List

from ._lib import check, lib
from .model import PlatformConfig, ProblemSpec


@dataclass(frozen=True)
class SweepRow:
    """(search.hpp:36-44)"""
    size: int
    wg: int
    ts: int
    time: int
    transitions: int
    ok: bool
    note: str


_NOTES = {0: "", 1: "infeasible", 2: "deadlock"}


def exhaustive_sweep(platform: PlatformConfig, problem: ProblemSpec) -> List[SweepRow]:
    """Every enumerated configuration, sorted by (time, transitions), flagged rows last
    (search.hpp:73-77, search.cpp:212-244)."""
    n = (problem.size.bit_length() - 2) ** 2 if problem.size >= 4 else 0
    rows = (C.c_int64 * (6 * max(n, 1)))()
    got = C.c_int64()
    check(lib.mctb_sweep(platform.as_array(), problem.size, problem.kernel, problem.input_array(),
                         rows, n, C.byref(got)))
    out = []
    for i in range(got.value):
        wg, ts, t, tr, ok, note = rows[6 * i:6 * i + 6]
        out.append(SweepRow(problem.size, wg, ts, t, tr, bool(ok), _NOTES[note]))
    return out


# --------------------------------------------------------------------------
# Verdicts and the bound-lowering driver (explore.hpp:65-70, search.hpp:16-34)

from .machine import Trace  # noqa: E402
from .model import TuningParams  # noqa: E402

_TRACE_CAP = 1 << 22
_TRACE_BUF = None


def _trace_buffer():
    """One reusable host buffer for counterexample traces (allocated once)."""
    global _TRACE_BUF
    if _TRACE_BUF is None:
        _TRACE_BUF = (C.c_int32 * (4 * _TRACE_CAP))()
    return _TRACE_BUF


@dataclass
class ExploreStatsSummary:
    states_visited: int = 0
    transitions_applied: int = 0
    max_depth_reached: int = 0
    configs_explored: int = 0
    configs_skipped: int = 0


@dataclass
class Verdict:
    violated: bool
    exhaustive: bool
    trace: "Trace | None"
    stats: ExploreStatsSummary
    trace_exact: bool = True


@dataclass
class TuneStats:
    checks_run: int = 0
    states_visited_total: int = 0
    wall_seconds: float = 0.0


@dataclass
class TuneProbe:
    """One bound of the bisection: check_overtime(T)'s verdict (explore.hpp:88-93)
    and, when violated, its counterexample's configuration, time and length."""
    T: int
    violated: bool
    exhaustive: bool
    states_visited: int
    wg: int
    ts: int
    final_time: int
    steps: int


@dataclass
class TuneResult:
    """(search.hpp:22-34)"""
    t_min: int
    params: TuningParams
    trace: Trace
    t_ini: int
    stats: TuneStats
    method: str
    proven: bool
    first_trail_time: int
    trace_exact: bool = True
    timings_ms: dict = None
    probes: list = None  # TuneProbe per bisection bound (bisect/tune only)

    def first_trail_optimality(self) -> float:
        if self.first_trail_time <= 0:
            return 1.0
        return self.t_min / self.first_trail_time


def _trace_from(buf, n, final_time, wg, ts):
    tr = [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]
    return Trace(tr, final_time, TuningParams(wg, ts), n)


def check_overtime(platform: PlatformConfig, problem: ProblemSpec, T: int,
                   max_states: int = 5_000_000, max_depth: int = 4_000_000) -> Verdict:
    """Exhaustive check of "every terminating run takes more than T ticks" over all
    configurations and interleavings (explore.hpp:88-93), within ExploreLimits'
    max_states and max_depth (explore.cpp:124-135)."""
    out = (C.c_int64 * 12)()
    buf = _trace_buffer()
    n = C.c_int64()
    check(lib.mctb_check_overtime(platform.as_array(), problem.size, problem.kernel,
                                  problem.input_array(), T, max_states, max_depth, out, buf,
                                  _TRACE_CAP,
                                  C.byref(n)))
    st = ExploreStatsSummary(out[2], out[4], out[3], out[5], out[6])
    trace = _trace_from(buf, n.value, out[7], out[8], out[9]) if out[0] else None
    return Verdict(bool(out[0]), bool(out[1]), trace, st, bool(out[11]))


def tune(platform: PlatformConfig, problem: ProblemSpec, seed: int = 1, t_hi: int = 0,
         max_states: int = 5_000_000, max_depth: int = 4_000_000) -> TuneResult:
    """The `tune` command flow: estimate_initial_time(seed) then bisect_min_time
    (tools/main.cpp:119-128)."""
    import time as _time
    t0 = _time.perf_counter()
    out = (C.c_int64 * 10)()
    buf = _trace_buffer()
    n = C.c_int64()
    info = (C.c_double * 5)()
    check(lib.mctb_tune(platform.as_array(), problem.size, problem.kernel, problem.input_array(),
                        t_hi, C.c_uint64(seed), max_states, max_depth, out, buf, _TRACE_CAP,
                        C.byref(n),
                        info))
    wall = _time.perf_counter() - t0
    trace = _trace_from(buf, n.value, out[0], out[1], out[2])
    res = TuneResult(out[0], TuningParams(out[1], out[2]), trace, out[3],
                     TuneStats(out[5], out[6], wall), "bisect", bool(out[4]), out[7],
                     bool(out[9]), {"cost_model": info[0], "first_paths": info[1],
                                    "exploration": info[2], "explored_states": info[3],
                                    "exploration_kernel": info[4]})
    # the bound-lowering probes, in order: one check_overtime(T) verdict each
    k = lib.mctb_tune_probes(None, 0)
    rows = (C.c_int64 * (8 * max(k, 1)))()
    lib.mctb_tune_probes(rows, k)
    res.probes = [TuneProbe(*rows[8 * i:8 * i + 8]) for i in range(k)]
    return res


def bisect_min_time(platform: PlatformConfig, problem: ProblemSpec, t_hi: int,
                    max_states: int = 5_000_000, max_depth: int = 4_000_000) -> TuneResult:
    """Counterexample-guided binary search for the minimal time (search.hpp:58-63)."""
    if t_hi < 1:
        from ._lib import ConfigError
        raise ConfigError("t_hi must be >= 1")
    return tune(platform, problem, 0, t_hi, max_states, max_depth)


def extract_params(platform: PlatformConfig, problem: ProblemSpec, trace: Trace):
    """Reads (wg, ts, time) out of a counterexample after replay validation (search.hpp:85-87)."""
    from .machine import replay
    replay(platform, problem, trace)
    return trace.params.wg, trace.params.ts, trace.final_time


@dataclass
class RankedTrail:
    time: int
    wg: int
    ts: int
    transitions: int


def rank_trails(traces) -> list:
    """Stable sort of trail summaries by (time, transitions) (search.hpp:89-90)."""
    out = [RankedTrail(t.final_time, t.params.wg, t.params.ts, t.steps) for t in traces]
    return sorted(out, key=lambda r: (r.time, r.transitions))


def swarm_min_time(platform: PlatformConfig, problem: ProblemSpec, workers: int = 4,
                   seed: int = 1, trajectories_per_worker: int = 4096, max_rounds: int = 64,
                   max_depth: int = 4_000_000, trails_out: list | None = None) -> TuneResult:
    """Randomized search for the minimal time (search.hpp:65-71): rounds of
    counter-based Philox trajectories on the GPU with the reference's stop rule.
    Heuristic: never a proof (proven = False)."""
    import time as _time
    t0 = _time.perf_counter()
    per_round = max(1, workers) * trajectories_per_worker
    if workers < 1:
        from ._lib import ConfigError
        raise ConfigError("swarm needs at least one worker")
    out = (C.c_int64 * 10)()
    buf = _trace_buffer()
    n = C.c_int64()
    tcap = per_round if trails_out is not None else 0
    trails = (C.c_int64 * (4 * max(tcap, 1)))()
    nt = C.c_int64()
    check(lib.mctb_swarm(platform.as_array(), problem.size, problem.kernel, problem.input_array(),
                         per_round, max_rounds, C.c_uint64(seed), max_depth, out, buf, _TRACE_CAP,
                         C.byref(n), trails, tcap, C.byref(nt)))
    if trails_out is not None:
        for i in range(nt.value):
            tm, wg, ts, st = trails[4 * i:4 * i + 4]
            trails_out.append(Trace([], tm, TuningParams(wg, ts), st))
    trace = _trace_from(buf, n.value, out[0], out[1], out[2])
    res = TuneResult(out[0], TuningParams(out[1], out[2]), trace, out[3],
                     TuneStats(out[4] - 1, out[5], _time.perf_counter() - t0), "swarm", False,
                     out[6])
    res.best_trajectory = out[8]
    res.trajectories = out[9]
    return res
