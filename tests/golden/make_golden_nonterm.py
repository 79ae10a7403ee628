"""Golden check_nontermination results of the reference (explore.cpp:207-233),
recorded from the reference itself (oracle/_ref): per (platform, size, kernel)
the traces in the reference's order — (wg, ts, final_time, steps, SHA-256 of the
transitions) — and the sweep statistics.  Only single-terminal spaces (every
configuration's schedules end in one state) are recorded: those the GPU engine
serves.  Re-run with: python tests/golden/make_golden_nonterm.py"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import Ref, TRACE_CAP, _inp, _plat, _untr, build_ref  # noqa: E402
from make_golden import trace_sha  # noqa: E402

CASES = [((1, 1, 4, 4), s, k) for s in (8, 16, 32) for k in (0, 1)] + \
        [((1, 2, 4, 4), 16, 0), ((1, 1, 8, 2), 16, 1), ((2, 1, 4, 4), 8, 0), ((1, 2, 2, 3), 16, 0)]


def ref_nonterm(ref, plat, size, kernel, max_depth=0, max_states=0, rows_cap=256):
    out = (C.c_int64 * 5)()
    rows = (C.c_int64 * (4 * rows_cap))()
    buf = (C.c_int32 * (4 * TRACE_CAP))()
    n = C.c_longlong()
    ref._chk(ref.lib.ref_check_nontermination(_plat(plat), size, kernel, _inp(size, kernel, None),
                                              C.c_longlong(max_depth), C.c_longlong(max_states),
                                              out, rows, C.c_longlong(rows_cap), buf,
                                              C.c_longlong(TRACE_CAP), C.byref(n)))
    trs, pos, allt = [], 0, _untr(buf, n.value)
    for i in range(min(out[0], rows_cap)):
        wg, ts, t, steps = rows[4 * i:4 * i + 4]
        trs.append({"wg": wg, "ts": ts, "final_time": t, "steps": steps,
                    "sha": trace_sha(allt[pos:pos + steps])})
        pos += steps
    return {"n": out[0], "states": out[1], "transitions": out[2], "max_depth": out[3],
            "limit_hit": out[4], "traces": trs}


def main():
    assert build_ref()
    ref = Ref()
    cases = []
    for plat, size, kernel in CASES:
        r = ref_nonterm(ref, plat, size, kernel)
        cases.append({"plat": plat, "size": size, "kernel": kernel, **r})
        print(plat, size, kernel, r["n"], [(t["wg"], t["ts"], t["final_time"]) for t in r["traces"]])
    with open(os.path.join(HERE, "nonterm.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
        f.write("\n")


if __name__ == "__main__":
    main()
