"""Loader for the in-tree CUDA library (libmctune_b200.so) and its C ABI.

There is no CPU implementation behind this package: if the library is missing
the import fails, and every compute call fails with NoDeviceError when no
sm_100 GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MCTB_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("MCTB_LIB") or os.path.join(HERE, "libmctune_b200.so")


class MctuneError(RuntimeError):
    """Base class of the engine's errors."""


class ConfigError(MctuneError):
    """Invalid user input (reference: mctune::ConfigError, model.hpp:15-17)."""


class ModelBug(MctuneError):
    """Internal contract violation (reference: mctune::ModelBug, model.hpp:21)."""


class CorruptTrace(MctuneError):
    """A trace failed to replay (reference: mctune::CorruptTrace, explore.hpp:14)."""


class LimitError(MctuneError):
    """A capacity limit of the GPU engine was hit."""


class NoDeviceError(MctuneError):
    """No sm_100 (B200) device: the engine has no CPU path."""


class CudaError(MctuneError):
    """A CUDA runtime call failed."""


_ERRORS = {1: ModelBug, 2: ConfigError, 3: CorruptTrace, 4: LimitError, 5: NoDeviceError,
           6: CudaError}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -m paper_2305_09130_b200.build` "
        "(nvcc, sm_100a).  There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

lib.mctb_last_error.restype = C.c_char_p
lib.mctb_version.restype = C.c_int
lib.mctb_device_count.restype = C.c_int
lib.mctb_derive_launch.argtypes = [i32p, C.c_int, C.c_int, C.c_int, i32p]
lib.mctb_space_count.argtypes = [i64p]
lib.mctb_space_count.restype = C.c_uint64
lib.mctb_space_argmin_async.argtypes = [i64p, C.c_uint64, C.c_uint64, vp, vp]
lib.mctb_space_argmin.argtypes = [i64p, C.c_uint64, C.c_uint64, u64p, i64p]
lib.mctb_space_eval_async.argtypes = [i64p, C.c_uint64, C.c_uint64, vp, vp, vp]
lib.mctb_space_exact_async.argtypes = [i64p, C.c_uint64, C.c_uint64, vp, vp, vp]
lib.mctb_int32_peak.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
lib.mctb_issue_probe.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
lib.mctb_sweep.argtypes = [i32p, C.c_int, C.c_int, i64p, i64p, C.c_int64, i64p]
lib.mctb_simulate.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int, C.c_int, C.c_int,
                              C.c_uint64, C.c_uint64, i64p, i32p, C.c_int64, i64p]
lib.mctb_trajectories.argtypes = [i32p, C.c_int, C.c_int, i64p, i32p, C.c_int, C.c_int,
                                  C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, i64p]
lib.mctb_trajectories_kernel_ms.argtypes = []
lib.mctb_trajectories_kernel_ms.restype = C.c_double
lib.mctb_replay.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int, C.c_int, i32p, C.c_int64,
                            C.c_int64, i64p]
lib.mctb_trace_text.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int, C.c_int, i32p, C.c_int64,
                                C.c_char_p, C.c_int64]
lib.mctb_trace_text.restype = C.c_int64

EXPORTED = [
    "mctb_last_error", "mctb_version", "mctb_device_count", "mctb_derive_launch",
    "mctb_space_count", "mctb_space_argmin_async", "mctb_space_argmin",
    "mctb_space_eval_async", "mctb_space_exact_async", "mctb_sweep", "mctb_int32_peak", "mctb_issue_probe", "mctb_simulate",
    "mctb_trajectories", "mctb_trajectories_kernel_ms", "mctb_replay", "mctb_trace_text",
]


def check(rc: int) -> None:
    if rc != 0:
        msg = lib.mctb_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, MctuneError)(msg)


def i32arr(vals):
    return (C.c_int32 * len(vals))(*vals)


def i64arr(vals):
    return (C.c_int64 * len(vals))(*vals)


def device_count() -> int:
    return lib.mctb_device_count()

lib.mctb_explore.argtypes = [i32p, C.c_int, C.c_int, i64p, i32p, C.c_int, C.c_int64, C.c_int64,
                             C.c_int, i64p, i64p]
EXPORTED.append("mctb_explore")
lib.mctb_check_overtime.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int64, C.c_int64, C.c_int64,
                                    i64p,
                                    i32p, C.c_int64, i64p]
lib.mctb_tune.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int64, C.c_uint64, C.c_int64, C.c_int64,
                          i64p,
                          i32p, C.c_int64, i64p, C.POINTER(C.c_double)]
EXPORTED += ["mctb_check_overtime", "mctb_tune"]
lib.mctb_swarm.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int64, C.c_int, C.c_uint64,
                           C.c_int64, i64p, i32p, C.c_int64, i64p, i64p, C.c_int64, i64p]
EXPORTED.append("mctb_swarm")
lib.mctb_explore_mp_open.argtypes = [i32p, C.c_int, C.c_int, i64p, i32p, C.c_int, C.c_int64,
                                     C.c_int, C.c_int, C.c_int, C.POINTER(vp), C.c_char_p]
lib.mctb_explore_mp_connect.argtypes = [vp, C.c_char_p]
lib.mctb_explore_mp_seed.argtypes = [vp]
lib.mctb_explore_mp_run.argtypes = [vp, i64p, i64p]
lib.mctb_explore_mp_close.argtypes = [vp]
lib.mctb_explore_mp_close.restype = None
EXPORTED += ["mctb_explore_mp_open", "mctb_explore_mp_connect", "mctb_explore_mp_seed",
             "mctb_explore_mp_run", "mctb_explore_mp_close"]
lib.mctb_tune_probes.argtypes = [i64p, C.c_int64]
lib.mctb_tune_probes.restype = C.c_int64
EXPORTED.append("mctb_tune_probes")
lib.mctb_nonterm_traces.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int, C.c_int, C.c_int64,
                                    C.c_int64, i64p, i64p, C.c_int64, i32p, C.c_int64, i64p]
EXPORTED.append("mctb_nonterm_traces")
lib.mctb_kernel_program.argtypes = [i32p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, C.c_int,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]
EXPORTED.append("mctb_kernel_program")
EXPORTED += ["mctb_machine_initial", "mctb_machine_enabled", "mctb_machine_apply",
             "mctb_machine_query", "mctb_machine_process_name", "mctb_machine_replay",
             "mctb_machine_states"]
# explore_machine's visit order (the C++ drop-in's ExploreHooks; the parity tests)
lib.mctb_machine_states.argtypes = [i32p, C.c_int, C.c_int, i64p, C.c_int, C.c_int, C.c_int64,
                                    C.c_int64, i64p, C.c_int64, i32p, C.c_int64, i64p]
