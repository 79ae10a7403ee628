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


def check_nontermination(platform: PlatformConfig, problem: ProblemSpec, max_depth: int = 4_000_000,
                         max_states: int = 5_000_000):
    """Terminating traces, one per distinct terminal state, for every feasible
    configuration largest-first (explore.hpp:95-100, explore.cpp:207-233).  One GPU
    sweep; a single-terminal configuration contributes the FIRST-policy run (where
    the reference's DFS first meets its terminal state); several terminal states
    raise LimitError.  Returns (traces, stats of the sweep per configuration)."""
    from ._lib import ConfigError, LimitError, ModelBug
    from .machine import FIRST, Machine, Trace
    from .model import config_feasible, enumerate_configs
    if max_depth < 1:
        raise ConfigError("max_depth must be >= 1")
    configs = sorted((c for c in enumerate_configs(problem.size) if config_feasible(problem, c)),
                     key=lambda c: (-c.wg, -c.ts))
    if not configs:
        return [], []
    stats = explore_configs(platform, problem, configs, max_states)
    traces = []
    for c, st in zip(configs, stats):
        if st.deadlocks:
            raise ModelBug("deadlock reached during exploration")
        if st.terminals == 0:
            continue
        if st.terminals > 1:
            raise LimitError(f"check_nontermination: configuration ({c.wg}, {c.ts}) has "
                             f"{st.terminals} terminal states; only single-terminal spaces are served")
        tr = []
        r = Machine(platform, problem, c).run(FIRST, trace_out=tr)
        if len(tr) > max_depth:
            continue
        traces.append(Trace(tr, r.time, c, len(tr)))
    return traces, stats
