"""The transition system on the GPU (reference: include/mctune/machine.hpp,
explore.hpp replay, report.hpp trace_to_text).

`Machine(platform, problem, params).run(policy, seed)` mirrors
mctune::Machine::run; traces use the reference's Transition fields
(actor, peer, op, arg) with op = the ordinal of mctune::Op.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from ._lib import check, i32arr, lib
from .model import PlatformConfig, ProblemSpec, TuningParams

ROUND_ROBIN, MT19937, FIRST, PHILOX = 0, 1, 2, 3
SEEDED_RANDOM = MT19937  # SchedPolicy::SeededRandom

OPS = ["ClockTick", "ClockHalt", "HostGo", "HostReactGo", "HostStop", "HostSetFin",
       "DeviceUnitGo", "DeviceDone", "DeviceUnitStop", "UnitPexGo", "UnitDone", "UnitPexStop",
       "UnitBarrierStop", "PexReport", "PexEffect", "PexArrive", "PexItemDone", "PexEndDone",
       "BarrierRelease"]

Transition = Tuple[int, int, int, int]  # (actor, peer, op, arg)


@dataclass
class RunOutcome:
    """(machine.hpp:145-149)"""
    time: int = 0
    result: Optional[int] = None
    steps: int = 0


@dataclass
class Trace:
    """(explore.hpp:58-63)"""
    transitions: List[Transition] = field(default_factory=list)
    final_time: int = 0
    params: TuningParams = TuningParams()
    steps: int = 0


def _trace_buf(trace: Sequence[Transition]):
    flat = [v for t in trace for v in t]
    return (C.c_int32 * max(1, len(flat)))(*flat), len(trace)


class Machine:
    """One (platform, problem, params) choice (machine.hpp:151-233)."""

    def __init__(self, platform: PlatformConfig, problem: ProblemSpec, params: TuningParams):
        platform.validate()
        problem.validate()
        self.platform, self.problem, self.params = platform, problem, params

    def _args(self):
        return (self.platform.as_array(), self.problem.size, self.problem.kernel,
                self.problem.input_array(), self.params.wg, self.params.ts)

    def run(self, policy: int = ROUND_ROBIN, seed: int = 0, trace_out: Optional[list] = None,
            traj: int = 0, trace_cap: int = 1 << 22) -> RunOutcome:
        out = (C.c_int64 * 4)()
        n = C.c_int64()
        buf = (C.c_int32 * (4 * trace_cap))() if trace_out is not None else None
        check(lib.mctb_simulate(*self._args(), policy, C.c_uint64(seed), C.c_uint64(traj), out,
                                buf, trace_cap if buf is not None else 0, C.byref(n)))
        if trace_out is not None:
            m = min(n.value, trace_cap)
            trace_out.extend(tuple(buf[4 * i:4 * i + 4]) for i in range(m))
        self.process_count = out[3]
        return RunOutcome(out[0], None if out[2] == -(1 << 63) else out[2], out[1])


def replay(platform: PlatformConfig, problem: ProblemSpec, trace: Trace) -> Tuple[int, Optional[int]]:
    """Re-applies a trace on the GPU (explore.hpp:111-113); returns (final time, result).
    Raises CorruptTrace on divergence, non-terminal end or time mismatch."""
    buf, n = _trace_buf(trace.transitions)
    out = (C.c_int64 * 2)()
    check(lib.mctb_replay(platform.as_array(), problem.size, problem.kernel,
                          problem.input_array(), trace.params.wg, trace.params.ts, buf, n,
                          trace.final_time, out))
    return out[0], (None if out[1] == -(1 << 63) else out[1])


def trace_to_text(platform: PlatformConfig, problem: ProblemSpec, trace: Trace) -> str:
    """report.hpp:33-38: one line per transition, then the FINAL line."""
    buf, n = _trace_buf(trace.transitions)
    need = lib.mctb_trace_text(platform.as_array(), problem.size, problem.kernel,
                               problem.input_array(), trace.params.wg, trace.params.ts, buf, n,
                               None, 0)
    if need < 0:
        check(3)
    out = C.create_string_buffer(need + 1)
    lib.mctb_trace_text(platform.as_array(), problem.size, problem.kernel, problem.input_array(),
                        trace.params.wg, trace.params.ts, buf, n, out, need + 1)
    return out.value.decode()


@dataclass
class TrajectoryBatch:
    time: List[int]
    steps: List[int]
    result: List[Optional[int]]
    status: List[int]
    hash: List[int]
    config: List[int]


def trajectories(platform: PlatformConfig, problem: ProblemSpec, configs: Sequence[TuningParams],
                 policy: int = PHILOX, seed: int = 1, traj0: int = 0, n: int = 1024,
                 max_steps: int = 200_000_000) -> TrajectoryBatch:
    """n schedule trajectories on the GPU; trajectory t runs configs[t % len(configs)]."""
    cfg = i32arr([v for c in configs for v in (c.wg, c.ts)])
    out = (C.c_int64 * (6 * max(n, 1)))()
    check(lib.mctb_trajectories(platform.as_array(), problem.size, problem.kernel,
                                problem.input_array(), cfg, len(configs), policy,
                                C.c_uint64(seed), C.c_uint64(traj0), C.c_uint64(n),
                                C.c_int64(max_steps), out))
    cols = [out[k::6][:n] for k in range(6)]
    res = [None if v == -(1 << 63) else v for v in cols[2]]
    return TrajectoryBatch(list(cols[0]), list(cols[1]), res, list(cols[3]),
                           [v & ((1 << 64) - 1) for v in cols[4]], list(cols[5]))
