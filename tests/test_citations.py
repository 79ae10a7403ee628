"""Every `file.cpp:N[-M]` / `file.hpp:N[-M]` citation of the reference in this
repository points inside that reference file (CPU; skipped where /root/reference
is absent, e.g. on the GPU box)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
PAT = re.compile(r"\b([a-z_]+\.(?:hpp|cpp)):(\d+)(?:-(\d+))?\b")


@pytest.mark.skipif(not os.path.isdir(REF), reason="needs /root/reference")
def test_reference_citations_are_in_range():
    lengths = {}
    for d, _, fs in os.walk(REF):
        for f in fs:
            if f.endswith((".hpp", ".cpp")):
                n = sum(1 for _ in open(os.path.join(d, f), errors="replace"))
                lengths[f] = max(lengths.get(f, 0), n)
    bad = []
    for d, dirs, fs in os.walk(ROOT):
        dirs[:] = [x for x in dirs if x not in (".git", "gpurun_out", "_build", "_ref", "variants")]
        for f in fs:
            if not f.endswith((".md", ".h", ".hpp", ".cu", ".cuh", ".py", ".c", ".cpp")):
                continue
            if f in ("doctest.h", "PAPERS.md", "SNIPPETS.md"):
                continue
            p = os.path.join(d, f)
            for i, line in enumerate(open(p, errors="replace"), 1):
                for m in PAT.finditer(line):
                    name, a, b = m.group(1), int(m.group(2)), int(m.group(3) or m.group(2))
                    if name in lengths and not (1 <= a <= b <= lengths[name]):
                        bad.append(f"{os.path.relpath(p, ROOT)}:{i} {m.group(0)}")
    assert not bad, bad[:20]
