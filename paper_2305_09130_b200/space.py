"""Exhaustive evaluation of tuning spaces on the GPU (north-star subsystem 1).

A Space generalises the reference's enumerate_configs (model.cpp:90-100):
besides wg and ts it ranges over the platform shape (nd devices, nu units,
np = 2^k processing elements = work-items a unit runs at once).  The
reference's own space for one platform is Space.reference(platform, problem).
Index order (least = preferred on ties): wg descending, ts descending, then
np, nu, nd ascending — explore.cpp:64-72's preference, extended.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

from ._lib import ConfigError, check, i64arr, lib
from .model import PlatformConfig, ProblemSpec, TuningParams, log2_exact

KEY_TIME_BITS = 30
KEY_INDEX_BITS = 33
KEY_SAT = (1 << KEY_TIME_BITS) - 1
KEY_NONE = 1 << 63


@dataclass(frozen=True)
class Space:
    kernel: int
    size: int
    gmt: int
    nd: Tuple[int, int] = (1, 1)
    nu: Tuple[int, int] = (1, 1)
    log2np: Tuple[int, int] = (2, 2)
    log2wg: Optional[Tuple[int, int]] = None  # default [1, n-1]
    log2ts: Optional[Tuple[int, int]] = None

    @staticmethod
    def reference(platform: PlatformConfig, problem: ProblemSpec) -> "Space":
        platform.validate()
        problem.validate()
        lnp = log2_exact(platform.np)
        return Space(problem.kernel, problem.size, platform.gmt, (platform.nd, platform.nd),
                     (platform.nu, platform.nu), (lnp, lnp))

    def desc(self):
        n = log2_exact(self.size) if self.size >= 1 and self.size & (self.size - 1) == 0 else 0
        wg = self.log2wg or (1, n - 1)
        ts = self.log2ts or (1, n - 1)
        return i64arr([self.kernel, self.size, self.gmt, self.nd[0], self.nd[1], self.nu[0],
                       self.nu[1], self.log2np[0], self.log2np[1], wg[0], wg[1], ts[0], ts[1]])

    @property
    def count(self) -> int:
        n = lib.mctb_space_count(self.desc())
        if n == 0:
            raise ConfigError(lib.mctb_last_error().decode())
        return int(n)

    def decode(self, index: int) -> Tuple[PlatformConfig, TuningParams]:
        """Index -> (platform, params); pure index arithmetic of the documented order."""
        d = list(self.desc())
        n_nd, n_nu = d[4] - d[3] + 1, d[6] - d[5] + 1
        n_np, n_ts = d[8] - d[7] + 1, d[12] - d[11] + 1
        index, nd = divmod(index, n_nd)
        index, nu = divmod(index, n_nu)
        index, lnp = divmod(index, n_np)
        wg_d, ts_d = divmod(index, n_ts)
        return (PlatformConfig(d[3] + nd, d[5] + nu, 1 << (d[7] + lnp), self.gmt),
                TuningParams(1 << (d[10] - wg_d), 1 << (d[12] - ts_d)))


@dataclass(frozen=True)
class SpaceResult:
    key: int
    index: int
    time: int
    steps: int
    platform: PlatformConfig
    params: TuningParams


def space_argmin(space: Space, first: int = 0, count: Optional[int] = None) -> SpaceResult:
    """Minimal-time configuration of [first, first+count) (host buffers in, host result out).
    Exact for every space: when the packed key's time field saturates, the C ABI
    resolves the winner with the exact two-pass evaluation (include/mctune_b200.h)."""
    if count is None:
        count = space.count - first
    key = C.c_uint64()
    out = (C.c_int64 * 8)()
    check(lib.mctb_space_argmin(space.desc(), first, count, C.byref(key), out))
    return SpaceResult(key.value, key.value & ((1 << KEY_INDEX_BITS) - 1), out[0], out[1],
                       PlatformConfig(out[2], out[3], out[4], out[5]), TuningParams(out[6], out[7]))


def space_argmin_async(space: Space, first: int, count: int, d_key_ptr: int, stream: int = 0,
                       desc=None) -> None:
    """Device-resident argmin into a uint64 device word (no sync, no allocation)."""
    check(lib.mctb_space_argmin_async(desc if desc is not None else space.desc(), first, count,
                                      C.c_void_p(d_key_ptr), C.c_void_p(stream)))


def space_exact_async(space: Space, first: int, count: int, d_time_ptr: int, d_index_ptr: int,
                      stream: int = 0, desc=None) -> None:
    """Exact argmin of [first, first+count) without the packed key (two plain passes):
    uint64 device words *time = least model time of the feasible configurations
    (2^64-1: none), *index = least index with that time.  Resolves a key whose time
    field saturated (key >> KEY_INDEX_BITS == KEY_SAT)."""
    check(lib.mctb_space_exact_async(desc if desc is not None else space.desc(), first, count,
                                     C.c_void_p(d_time_ptr), C.c_void_p(d_index_ptr),
                                     C.c_void_p(stream)))


def space_eval_async(space: Space, first: int, count: int, d_time_ptr: int, d_steps_ptr: int,
                     stream: int = 0) -> None:
    """Per-configuration (time, transitions) table into device int64 arrays."""
    check(lib.mctb_space_eval_async(space.desc(), first, count, C.c_void_p(d_time_ptr),
                                    C.c_void_p(d_steps_ptr), C.c_void_p(stream)))
