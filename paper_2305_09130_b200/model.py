"""Model-core types of the tuner (reference: include/mctune/model.hpp).

Same names, fields, validation rules and error classes as the reference's
PlatformConfig / ProblemSpec / TuningParams / LaunchPlan, so code written
against mctune reads the same here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from ._lib import ConfigError, check, i32arr, lib


def is_pow2(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


def log2_exact(v: int) -> int:
    """model.cpp:5-10"""
    if not is_pow2(v):
        raise ConfigError(f"not a power of two: {v}")
    return v.bit_length() - 1


@dataclass(frozen=True)
class PlatformConfig:
    """Abstract platform constants (model.hpp:33-40)."""
    nd: int = 1
    nu: int = 1
    np: int = 4
    gmt: int = 4

    def validate(self) -> None:  # model.cpp:12-17
        if self.nd < 1 or self.nu < 1 or self.np < 1 or self.gmt < 1:
            raise ConfigError("platform constants nd, nu, np, gmt must all be >= 1")
        if not is_pow2(self.np):
            raise ConfigError(f"np must be a power of two, got {self.np}")

    def as_array(self):
        return i32arr([self.nd, self.nu, self.np, self.gmt])


ABSTRACT, MINIMUM = 0, 1


def kernel_kind_from_string(s: str) -> int:
    """model.cpp:23-27"""
    if s == "abstract":
        return ABSTRACT
    if s == "minimum":
        return MINIMUM
    raise ConfigError(f"unknown kernel kind '{s}' (expected abstract or minimum)")


@dataclass(frozen=True)
class ProblemSpec:
    """Problem instance (model.hpp:48-58)."""
    size: int = 8
    kernel: int = ABSTRACT
    input: tuple = field(default_factory=tuple)

    @staticmethod
    def abstract(size: int) -> "ProblemSpec":
        p = ProblemSpec(size, ABSTRACT, ())
        p.validate()
        return p

    @staticmethod
    def minimum(size: int, input: Optional[Sequence[int]] = None) -> "ProblemSpec":
        """Empty input selects glob[i] = size - i (model.cpp:37-49)."""
        vals = tuple(int(v) for v in input) if input else tuple(size - i for i in range(size))
        p = ProblemSpec(size, MINIMUM, vals)
        p.validate()
        return p

    def validate(self) -> None:  # model.cpp:51-60
        if self.size < 4 or not is_pow2(self.size):
            raise ConfigError(f"size must be a power of two >= 4, got {self.size}")
        if self.kernel == MINIMUM:
            if len(self.input) != self.size:
                raise ConfigError("minimum kernel needs an input array of length size")
        elif self.input:
            raise ConfigError("abstract kernel takes no input array")

    def input_array(self):
        if self.kernel != MINIMUM:
            return None
        return (C.c_int64 * self.size)(*self.input)


@dataclass(frozen=True)
class TuningParams:
    """(model.hpp:61-66)"""
    wg: int = 0
    ts: int = 0


@dataclass(frozen=True)
class LaunchPlan:
    """(model.hpp:69-77)"""
    wgs: int = 0
    nwd: int = 0
    nwu: int = 0
    nwe: int = 0
    all_nwe: int = 0


def validate_params(size: int, params: TuningParams) -> None:
    """model.cpp:62-70"""
    hi = size // 2
    if not is_pow2(params.wg) or params.wg < 2 or params.wg > hi:
        raise ConfigError(f"wg must be a power of two in [2, size/2], got {params.wg}")
    if not is_pow2(params.ts) or params.ts < 2 or params.ts > hi:
        raise ConfigError(f"ts must be a power of two in [2, size/2], got {params.ts}")


def derive_launch(platform: PlatformConfig, size: int, params: TuningParams) -> LaunchPlan:
    """Listing-3 launch arithmetic (model.cpp:72-88), through the C ABI."""
    out = (C.c_int32 * 5)()
    check(lib.mctb_derive_launch(platform.as_array(), size, params.wg, params.ts, out))
    return LaunchPlan(*out)


def enumerate_configs(size: int) -> List[TuningParams]:
    """All (wg, ts) = (2^i, 2^j), i, j in [1, n-1], (wg, ts) ascending (model.cpp:90-100)."""
    if size < 4 or not is_pow2(size):
        raise ConfigError(f"size must be a power of two >= 4, got {size}")
    n = log2_exact(size)
    return [TuningParams(1 << i, 1 << j) for i in range(1, n) for j in range(1, n)]


def config_feasible(problem: ProblemSpec, params: TuningParams) -> bool:
    """kernel.cpp:84-87"""
    if problem.kernel == ABSTRACT:
        return True
    return params.wg * params.ts <= problem.size
