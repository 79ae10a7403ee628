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
    """(search.hpp:44-52)"""
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
    (search.hpp:381-385, search.cpp:214-246)."""
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
