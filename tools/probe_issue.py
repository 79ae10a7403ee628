"""Probe: the issue-rate probes of csrc/probe.cu (thread instructions/s per variant)."""
import ctypes as C
import sys
sys.path.insert(0, '.')
from paper_2305_09130_b200._lib import lib
names = ["IMAD+LOP3", "IADD3", "IADD3+LOP3+IMAD+SHF", "FFMA"]
for v in range(4):
    o, t = C.c_double(), C.c_double()
    rc = lib.mctb_issue_probe(v, C.byref(o), C.byref(t))
    print(v, names[v], rc, "%.2f T inst/s" % (o.value / 1e12), "%.3f ms" % t.value, flush=True)
o, t = C.c_double(), C.c_double()
lib.mctb_int32_peak(C.byref(o), C.byref(t))
print("int32_peak %.2f T inst/s" % (o.value / 1e12))
