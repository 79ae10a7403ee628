"""The C++ host API (include/mctune_b200.hpp, the drop-in headers
include/compat/mctune/*.hpp): it compiles and links against the C-ABI library
here (CPU), and on a B200 its own tests and the reference's own test_model.cpp /
test_search.cpp (compiled where they lie under /root/reference, tests/cpp/Makefile
`ref`) pass against the GPU engine."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _lib():
    import paper_2305_09130_b200._lib as L  # builds/loads the in-tree library
    return L


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cpp_api_compiles_and_links(tmp_path):
    _lib()
    exe = tmp_path / "test_api"
    r = subprocess.run(["g++", "-std=c++20", "-O0", "-Wall", "-Werror",
                        "-I", os.path.join(ROOT, "include"),
                        "-I", os.path.join(ROOT, "include", "compat"), "-I", CPP,
                        os.path.join(CPP, "test_api.cpp"), "-o", str(exe),
                        "-L", os.path.join(ROOT, "paper_2305_09130_b200"), "-lmctune_b200"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cpp_api_without_a_device_raises_no_device(tmp_path):
    """No CPU path behind the C++ API either: every compute call throws NoDevice."""
    _lib()
    src = tmp_path / "nodev.cpp"
    src.write_text('#include "mctune_b200.hpp"\n#include <cstdio>\n'
                   "int main() { if (mctune_b200::device_count() > 0) return 3;\n"
                   "  try { mctune_b200::bisect_min_time({1,1,4,4}, mctune_b200::ProblemSpec::abstract(8),"
                   " 100, {}); } catch (const mctune_b200::NoDevice&) { return 0; } return 1; }\n")
    exe = tmp_path / "nodev"
    lib_dir = os.path.join(ROOT, "paper_2305_09130_b200")
    r = subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                        str(exe), "-L", lib_dir, "-lmctune_b200", f"-Wl,-rpath,{lib_dir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    if _lib().device_count() > 0:
        pytest.skip("a device is present")
    assert subprocess.run([str(exe)]).returncode == 0


@pytest.mark.gpu
def test_cpp_api_on_the_gpu():
    _lib()
    r = subprocess.run(["make", "-s", "-C", CPP, "all"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([os.path.join(CPP, "_build", "test_api")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_model_and_search_tests_pass_on_the_gpu_engine():
    exe = os.path.join(CPP, "_build", "ref_tests")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/_build/ref_tests is built by __graft_entry__.build() where "
                    "/root/reference exists")
    _lib()
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "36 test cases, 0 failed" in r.stdout  # test_model, _kernel, _search, _machine, _explore


@pytest.mark.skipif(not os.path.exists("/usr/local/cuda/bin/nvcc"), reason="no nvcc")
def test_exploration_fast_paths_match_serial_semantics():
    """tests/cpp/bfs_rules_check.cu, on the CPU: on random walks through 433
    configurations, the exploration's per-process enumeration equals enabled(),
    the table-driven unpack inverts pack(), and every in-place successor equals
    pack(apply(...)) with its incremental hash equal to the full hash."""
    _lib()
    r = subprocess.run(["make", "-s", "-C", CPP, "_build/bfs_rules_check"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([os.path.join(CPP, "_build", "bfs_rules_check")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert " 0 failed" in r.stdout
