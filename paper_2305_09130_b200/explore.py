"""Exhaustive interleaving exploration on the GPU (reference: include/mctune/explore.hpp).

`explore_configs` runs the frontier-parallel BFS over the full state spaces of
one or more configurations of a (platform, problem) in one sweep and returns
the reference's ExploreStats fields per configuration, plus the range of
terminal model times (a proof of the minimal time over all interleavings).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence

from ._lib import check, i32arr, lib
from .model import PlatformConfig, ProblemSpec, TuningParams


@dataclass
class ExploreStats:
    """(explore.hpp:44-56) + terminal-time range."""
    complete: bool
    states_visited: int
    transitions_applied: int
    max_depth_reached: int
    min_time: int
    max_time: int
    terminals: int
    deadlocks: int
    invariant_violations: int = 0


@dataclass
class SweepInfo:
    table_slots: int
    states: int
    key_words: int
    kernel_us: int


def explore_configs(platform: PlatformConfig, problem: ProblemSpec,
                    configs: Sequence[TuningParams], max_states: int = 5_000_000,
                    info: list | None = None, check_invariants: bool = False,
                    partitions: int = 1, system_scope: bool = False,
                    max_depth: int = 4_000_000) -> List[ExploreStats]:
    """partitions > 1 splits the visited set into hash partitions on this device:
    the successor exchange of the multi-GPU sweep, run on one GPU (same kernel,
    same results); system_scope selects the multi-GPU kernel variant."""
    if not 1 <= partitions <= 8:
        from ._lib import ConfigError
        raise ConfigError("partitions must be in [1, 8]")
    cfg = i32arr([v for c in configs for v in (c.wg, c.ts)])
    out = (C.c_int64 * (9 * len(configs)))()
    inf = (C.c_int64 * 4)()
    check(lib.mctb_explore(platform.as_array(), problem.size, problem.kernel,
                           problem.input_array(), cfg, len(configs), max_states, max_depth,
                           (1 if check_invariants else 0) | (2 if system_scope else 0)
                           | (partitions << 8 if partitions > 1 else 0), out, inf))
    if info is not None:
        info.append(SweepInfo(*inf))
    return [ExploreStats(bool(out[9 * i]), *out[9 * i + 1:9 * i + 9]) for i in range(len(configs))]


def explore_machine(platform: PlatformConfig, problem: ProblemSpec, params: TuningParams,
                    max_states: int = 5_000_000, max_depth: int = 4_000_000) -> ExploreStats:
    """Every interleaving of one machine (explore.hpp:81-86) within ExploreLimits'
    max_states / max_depth (explore.cpp:124-135)."""
    return explore_configs(platform, problem, [params], max_states, max_depth=max_depth)[0]


def nonterm_traces(platform: PlatformConfig, problem: ProblemSpec, params: TuningParams,
                   max_depth: int = 4_000_000, max_states: int = 5_000_000,
                   n_hint: int = 0, len_hint: int = 0):
    """Every distinct terminal state of one configuration in the reference DFS's order,
    each with the path that DFS follows to it (mctb_nonterm_traces, lexrank.cu).
    Returns [(final_time, transitions)]."""
    from ._lib import LimitError
    rows_cap, trace_cap = max(n_hint, 16), max(len_hint, 4096)
    for _ in range(2):
        rows = (C.c_int64 * (2 * rows_cap))()
        buf = (C.c_int32 * (4 * trace_cap))()
        n, tl = C.c_int64(), C.c_int64()
        rc = lib.mctb_nonterm_traces(platform.as_array(), problem.size, problem.kernel,
                                     problem.input_array(), params.wg, params.ts, max_depth,
                                     max_states, C.byref(n), rows, rows_cap, buf, trace_cap,
                                     C.byref(tl))
        if rc == 4 and (n.value > rows_cap or tl.value > trace_cap):
            rows_cap, trace_cap = max(rows_cap, n.value), max(trace_cap, tl.value)
            continue
        check(rc)
        out, pos = [], 0
        for i in range(n.value):
            t, steps = rows[2 * i], rows[2 * i + 1]
            out.append((t, [tuple(buf[4 * k:4 * k + 4]) for k in range(pos, pos + steps)]))
            pos += steps
        return out
    raise LimitError("check_nontermination: trace buffers")


def check_nontermination(platform: PlatformConfig, problem: ProblemSpec, max_depth: int = 4_000_000,
                         max_states: int = 5_000_000):
    """Terminating traces, one per distinct terminal state, for every feasible
    configuration largest-first (explore.hpp:95-100, explore.cpp:207-233).  One GPU
    sweep gives the statistics and each configuration's terminal count; a
    configuration with one terminal state contributes its FIRST-policy run (where
    the reference's DFS first meets it); one with several gets every terminal with
    its DFS path in DFS order from the level-synchronous least-path ranking
    (nonterm_traces), and one whose visited set fills up gets the terminals among
    the first max_states states of that order (explore.cpp:26-30; graphs up to
    2^22 states, LimitError beyond).  Returns (traces, stats of the sweep per
    configuration)."""
    from ._lib import ConfigError, ModelBug
    from .machine import FIRST, Machine, Trace
    from .model import config_feasible, enumerate_configs
    if max_depth < 1:
        raise ConfigError("max_depth must be >= 1")
    configs = sorted((c for c in enumerate_configs(problem.size) if config_feasible(problem, c)),
                     key=lambda c: (-c.wg, -c.ts))
    if not configs:
        return [], []
    stats = explore_configs(platform, problem, configs, max_states, max_depth=max_depth)
    traces = []
    for c, st in zip(configs, stats):
        if st.deadlocks:
            raise ModelBug("deadlock reached during exploration")
        # a full visited set: the DFS meets only the terminals among the first
        # max_states states of its order (nonterm_traces cuts them there)
        capped = st.states_visited >= max_states
        if st.terminals == 0 and not capped:
            continue
        if st.terminals == 1 and st.complete:
            tr = []
            r = Machine(platform, problem, c).run(FIRST, trace_out=tr)
            traces.append(Trace(tr, r.time, c, len(tr)))
            continue
        for t, tr in nonterm_traces(platform, problem, c, max_depth,
                                    min(max_states, st.states_visited + 1), st.terminals,
                                    st.terminals * (st.max_depth_reached + 1)):
            traces.append(Trace(tr, t, c, len(tr)))
    return traces, stats
