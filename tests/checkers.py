"""ctypes bindings of the CHECKERS (test infrastructure only).

* Oracle : oracle/_build/libmctune_oracle.so — plain-C restatement of the reference.
* Ref    : oracle/_ref/libmctune_ref.so     — the reference's own C++ core + shim
           (built only where /root/reference exists; optional on the GPU box).
Both expose the same Python methods so tests can run one against the other.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libmctune_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libmctune_ref.so")
REFERENCE_SRC = "/root/reference/proj/src"

TRACE_CAP = 1 << 21


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


def build_ref() -> bool:
    if not os.path.isdir(REFERENCE_SRC):
        return os.path.exists(REF_SO)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    return True


def _plat(p):
    return (C.c_int * 4)(*p)


def _inp(size, kernel, inp):
    if kernel != 1 or inp is None:
        return None
    return (C.c_int64 * size)(*inp)


def _tr(trace):
    flat = [v for t in trace for v in t]
    return (C.c_int32 * max(len(flat), 1))(*flat), len(trace)


def _untr(buf, n):
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]


class CheckerError(RuntimeError):
    def __init__(self, rc, msg):
        super().__init__(f"rc={rc}: {msg}")
        self.rc = rc


class _Base:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        self.err = getattr(self.lib, self.prefix + "last_error")
        self.err.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            raise CheckerError(rc, self.err().decode(errors="replace"))

    def simulate(self, plat, size, kernel, wg, ts, policy=0, seed=0, inp=None, traj=0,
                 trace=False):
        raise NotImplementedError


class Oracle(_Base):
    prefix = "mo_"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        super().__init__(path)
        L = self.lib
        L.mo_trace_text.restype = C.c_int64

    def derive_launch(self, plat, size, wg, ts):
        out = (C.c_int * 5)()
        self._chk(self.lib.mo_derive_launch(_plat(plat), size, wg, ts, out))
        return list(out)

    def cost_model(self, plat, size, kernel, wg, ts):
        out = (C.c_int64 * 3)()
        self._chk(self.lib.mo_cost_model(_plat(plat), size, kernel, wg, ts, out))
        return list(out)

    def simulate(self, plat, size, kernel, wg, ts, policy=0, seed=0, inp=None, traj=0,
                 trace=False, cap=TRACE_CAP):
        out = (C.c_int64 * 4)()
        buf = (C.c_int32 * (4 * cap))() if trace else None
        n = C.c_int64()
        self._chk(self.lib.mo_simulate(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                       policy, C.c_uint64(seed), C.c_uint64(traj), out, buf,
                                       C.c_int64(cap), C.byref(n)))
        res = {"time": out[0], "steps": out[1], "result": None if out[2] == -(1 << 63) else out[2],
               "processes": out[3]}
        if trace:
            res["trace"] = _untr(buf, min(n.value, cap))
        return res

    def explore(self, plat, size, kernel, wg, ts, inp=None, max_depth=0, max_states=0):
        out = (C.c_int64 * 8)()
        self._chk(self.lib.mo_explore(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                      C.c_int64(max_depth), C.c_int64(max_states), out))
        return dict(zip(["complete", "states", "transitions", "max_depth", "min_time",
                         "max_time", "n_terminal", "n_distinct"], out))

    def check_overtime(self, plat, size, kernel, T, inp=None, max_depth=0, max_states=0):
        out = (C.c_int64 * 11)()
        buf = (C.c_int32 * (4 * TRACE_CAP))()
        n = C.c_int64()
        self._chk(self.lib.mo_check_overtime(_plat(plat), size, kernel, _inp(size, kernel, inp),
                                             C.c_int64(T), C.c_int64(max_depth),
                                             C.c_int64(max_states), out, buf,
                                             C.c_int64(TRACE_CAP), C.byref(n)))
        r = dict(zip(["violated", "exhaustive", "states", "max_depth", "transitions",
                      "configs_explored", "configs_skipped", "final_time", "wg", "ts", "steps"],
                     out))
        r["trace"] = _untr(buf, n.value)
        return r

    def replay(self, plat, size, kernel, wg, ts, trace, final_time, inp=None):
        t, n = _tr(trace)
        out = (C.c_int64 * 2)()
        self._chk(self.lib.mo_replay(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                     t, C.c_int64(n), C.c_int64(final_time), out))
        return out[0], (None if out[1] == -(1 << 63) else out[1])

    def trace_text(self, plat, size, kernel, wg, ts, trace, inp=None):
        t, n = _tr(trace)
        need = self.lib.mo_trace_text(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                      t, C.c_int64(n), None, C.c_int64(0))
        buf = C.create_string_buffer(need + 1)
        self.lib.mo_trace_text(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts, t,
                               C.c_int64(n), buf, C.c_int64(need + 1))
        return buf.value.decode()

    def fingerprints(self, plat, size, kernel, wg, ts, trace, inp=None):
        t, n = _tr(trace)
        out = (C.c_uint64 * (n + 1))()
        self._chk(self.lib.mo_run_fingerprints(_plat(plat), size, kernel, _inp(size, kernel, inp),
                                               wg, ts, t, C.c_int64(n), out))
        return list(out)

    def successors(self, plat, size, kernel, wg, ts, ser=None, cap=256):
        """[(fingerprint, serialized state)] of the initial state (ser None) or of a
        serialized state's successors, in the reference's enabled() order."""
        self.lib.mo_successors.restype = C.c_int64
        rec = C.c_int64()
        if getattr(self, "_succ_cap", 0) < cap:
            self._succ_buf = C.create_string_buffer(cap * 4096)
            self._succ_fps = (C.c_uint64 * cap)()
            self._succ_cap = cap
        buf, fps = self._succ_buf, self._succ_fps
        n = self.lib.mo_successors(_plat(plat), size, kernel, None, wg, ts, ser, buf, cap, fps,
                                   C.byref(rec))
        if n < 0:
            raise CheckerError(int(n), self.err().decode(errors="replace"))
        L = rec.value
        return [(fps[i], bytes(buf.raw[i * L:(i + 1) * L])) for i in range(n)]

    def space_argmin(self, sd, first, count):
        key, idx = C.c_uint64(), C.c_uint64()
        t = C.c_int64()
        self._chk(self.lib.mo_space_argmin((C.c_int64 * 13)(*sd), C.c_uint64(first),
                                           C.c_uint64(count), C.byref(key), C.byref(t),
                                           C.byref(idx)))
        return key.value, t.value, idx.value

    def trajectories(self, plat, size, kernel, configs, policy, seed, traj0, n, inp=None):
        cfg = (C.c_int32 * (2 * len(configs)))(*[v for c in configs for v in c])
        out = (C.c_int64 * (6 * n))()
        self._chk(self.lib.mo_trajectories(_plat(plat), size, kernel, _inp(size, kernel, inp), cfg,
                                           len(configs), policy, C.c_uint64(seed),
                                           C.c_uint64(traj0), C.c_uint64(n), out))
        cols = [list(out[k::6]) for k in range(6)]
        cols[4] = [v & ((1 << 64) - 1) for v in cols[4]]
        cols[2] = [None if v == -(1 << 63) else v for v in cols[2]]
        return cols

    def philox(self, ctr, key):
        out = (C.c_uint32 * 4)()
        self.lib.mo_philox4x32_10((C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), out)
        return list(out)

    def mt19937_64(self, seed, n):
        out = (C.c_uint64 * n)()
        self.lib.mo_mt19937_64(C.c_uint64(seed), n, out)
        return list(out)


class Ref(_Base):
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self.lib.ref_trace_text.restype = C.c_longlong

    def derive_launch(self, plat, size, wg, ts):
        out = (C.c_int * 5)()
        self._chk(self.lib.ref_derive_launch(_plat(plat), size, wg, ts, out))
        return list(out)

    def simulate(self, plat, size, kernel, wg, ts, policy=0, seed=0, inp=None, traj=0,
                 trace=False, cap=TRACE_CAP):
        assert policy in (0, 1)
        out = (C.c_int64 * 4)()
        buf = (C.c_int32 * (4 * cap))() if trace else None
        n = C.c_longlong()
        self._chk(self.lib.ref_simulate(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                        policy, C.c_uint64(seed), out, buf, C.c_longlong(cap),
                                        C.byref(n) if trace else None))
        res = {"time": out[0], "steps": out[1], "result": None if out[2] == -(1 << 63) else out[2],
               "processes": out[3]}
        if trace:
            res["trace"] = _untr(buf, min(n.value, cap))
        return res

    def explore(self, plat, size, kernel, wg, ts, inp=None, max_depth=0, max_states=0,
                invariants=False):
        out = (C.c_int64 * 8)()
        self._chk(self.lib.ref_explore(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                       C.c_longlong(max_depth), C.c_longlong(max_states), 0,
                                       int(invariants), out))
        return dict(zip(["complete", "states", "transitions", "max_depth", "min_time",
                         "max_time", "n_terminal", "n_distinct"], out))

    def explore_order(self, plat, size, kernel, wg, ts, inp=None, max_depth=0, max_states=0,
                      cap=1 << 20):
        """FNV-1a 64 of every state explore_machine visits, in on_state order
        (ref_explore_order: the fields in the engine's flat-vector order)."""
        hashes = (C.c_uint64 * cap)()
        n = C.c_longlong()
        self._chk(self.lib.ref_explore_order(_plat(plat), size, kernel, _inp(size, kernel, inp),
                                             wg, ts, C.c_longlong(max_depth),
                                             C.c_longlong(max_states), hashes, C.c_longlong(cap),
                                             C.byref(n)))
        return list(hashes[:min(n.value, cap)]), n.value

    def check_overtime(self, plat, size, kernel, T, inp=None, max_depth=0, max_states=0):
        out = (C.c_int64 * 11)()
        buf = (C.c_int32 * (4 * TRACE_CAP))()
        n = C.c_longlong()
        self._chk(self.lib.ref_check_overtime(_plat(plat), size, kernel, _inp(size, kernel, inp),
                                              C.c_int64(T), C.c_longlong(max_depth),
                                              C.c_longlong(max_states), 0, out, buf,
                                              C.c_longlong(TRACE_CAP), C.byref(n)))
        r = dict(zip(["violated", "exhaustive", "states", "max_depth", "transitions",
                      "configs_explored", "configs_skipped", "final_time", "wg", "ts", "steps"],
                     out))
        r["trace"] = _untr(buf, n.value)
        return r

    def tune(self, plat, size, kernel, seed=1, t_hi=0, inp=None, max_depth=0, max_states=0):
        out = (C.c_int64 * 9)()
        buf = (C.c_int32 * (4 * TRACE_CAP))()
        n = C.c_longlong()
        self._chk(self.lib.ref_tune(_plat(plat), size, kernel, _inp(size, kernel, inp),
                                    C.c_int64(t_hi), C.c_uint64(seed), C.c_longlong(max_depth),
                                    C.c_longlong(max_states), out, buf, C.c_longlong(TRACE_CAP),
                                    C.byref(n)))
        r = dict(zip(["t_min", "wg", "ts", "t_ini", "proven", "checks_run", "states_visited_total",
                      "first_trail_time", "steps"], out))
        r["trace"] = _untr(buf, n.value)
        return r

    def sweep(self, plat, size, kernel, inp=None):
        n_max = 64 * 64
        rows = (C.c_int64 * (6 * n_max))()
        n = C.c_longlong()
        self._chk(self.lib.ref_sweep(_plat(plat), size, kernel, _inp(size, kernel, inp), rows,
                                     C.c_longlong(n_max), C.byref(n)))
        return [tuple(rows[6 * i:6 * i + 6]) for i in range(n.value)]

    def replay(self, plat, size, kernel, wg, ts, trace, final_time, inp=None):
        t, n = _tr(trace)
        out = (C.c_int64 * 2)()
        self._chk(self.lib.ref_replay(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                      t, C.c_longlong(n), C.c_int64(final_time), out))
        return out[0], (None if out[1] == -(1 << 63) else out[1])

    def trace_text(self, plat, size, kernel, wg, ts, trace, inp=None):
        t, n = _tr(trace)
        need = self.lib.ref_trace_text(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts,
                                       t, C.c_longlong(n), None, C.c_longlong(0))
        buf = C.create_string_buffer(need + 1)
        self.lib.ref_trace_text(_plat(plat), size, kernel, _inp(size, kernel, inp), wg, ts, t,
                                C.c_longlong(n), buf, C.c_longlong(need + 1))
        return buf.value.decode()

    def fingerprints(self, plat, size, kernel, wg, ts, trace, inp=None):
        t, n = _tr(trace)
        out = (C.c_uint64 * (n + 1))()
        self._chk(self.lib.ref_run_fingerprints(_plat(plat), size, kernel,
                                                _inp(size, kernel, inp), wg, ts, t,
                                                C.c_longlong(n), out))
        return list(out)

    def swarm(self, plat, size, kernel, workers, budget, seed, inp=None, max_depth=0):
        out = (C.c_int64 * 8)()
        self._chk(self.lib.ref_swarm(_plat(plat), size, kernel, _inp(size, kernel, inp), workers,
                                     C.c_double(budget), C.c_longlong(max_depth),
                                     C.c_uint64(seed), out))
        return dict(zip(["t_min", "wg", "ts", "t_ini", "checks_run", "states_visited_total",
                         "first_trail_time", "steps"], out))


def load_ref():
    """The reference checker, or None when it cannot be built here."""
    try:
        if not build_ref():
            return None
        return Ref()
    except Exception:
        return None
