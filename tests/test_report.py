"""Data formats either side of the path (report.hpp) — host formatting of GPU results."""
import json
import os
import shutil
import subprocess

import pytest


def test_csv_and_json_shapes(tmp_path):
    import paper_2305_09130_b200 as m
    from paper_2305_09130_b200 import report
    rows = [m.SweepRow(16, 8, 2, 23, 148, True, ""), m.SweepRow(16, 4, 8, 0, 0, False, "infeasible")]
    csv = report.sweep_to_csv(rows)
    assert csv == "size,wg,ts,time,transitions\n16,8,2,23,148\n16,4,8,,\n"
    j = json.loads(report.sweep_to_json(rows))
    assert j[1] == {"size": 16, "wg": 4, "ts": 8, "note": "infeasible"}
    trails = m.rank_trails([m.Trace([], 50, m.TuningParams(2, 2), 10),
                            m.Trace([], 44, m.TuningParams(4, 4), 1700)])
    assert report.trails_to_csv(8, trails) == "size,wg,ts,time,transitions\n8,4,4,44,1700\n8,2,2,50,10\n"


def test_config_and_input_files(tmp_path):
    from paper_2305_09130_b200 import report, ConfigError
    (tmp_path / "data.txt").write_text("\n".join(str(v) for v in [5, 3, 9, 7]) + "\n")
    (tmp_path / "c.json").write_text(json.dumps({
        "platform": {"nd": 1, "nu": 2, "np": 4, "gmt": 3},
        "problem": {"size": 4, "kernel": "minimum", "input_path": "data.txt"}}))
    cfg = report.load_config_file(str(tmp_path / "c.json"))
    assert (cfg.platform.nu, cfg.platform.gmt) == (2, 3)
    assert cfg.problem.input == (5, 3, 9, 7)
    with pytest.raises(ConfigError):
        report.read_input_file(str(tmp_path / "data.txt"), 5)
    (tmp_path / "bad.json").write_text("{")
    with pytest.raises(ConfigError):
        report.load_config_file(str(tmp_path / "bad.json"))


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cpp_report_mirror_matches_python_mirror(tmp_path):
    """include/mctune_b200_report.hpp (the C++ drop-in for report.hpp) writes the
    same bytes as report.py for the same inputs, and reads the same config file."""
    from types import SimpleNamespace as NS

    import paper_2305_09130_b200 as m
    from paper_2305_09130_b200 import report
    import paper_2305_09130_b200._lib as L
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "report_check"
    lib_dir = os.path.dirname(L.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++20", "-O0", "-Wall", "-Werror",
                        "-I", os.path.join(root, "include"),
                        "-I", os.path.join(root, "include", "compat"),
                        os.path.join(root, "tests", "cpp", "report_check.cpp"), "-o", str(exe),
                        "-L", lib_dir, "-lmctune_b200", f"-Wl,-rpath,{lib_dir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    (tmp_path / "data.txt").write_text("5\n3\n9\n7\n")
    (tmp_path / "c.json").write_text(json.dumps({
        "platform": {"nd": 1, "nu": 2, "np": 4, "gmt": 3},
        "problem": {"size": 4, "kernel": "minimum", "input_path": "data.txt"}}))
    (tmp_path / "bad.json").write_text("{")
    out = subprocess.run([str(exe), str(tmp_path / "c.json"), str(tmp_path / "bad.json")],
                         capture_output=True, text=True, check=True).stdout.split("@@\n")
    rows = [m.SweepRow(16, 8, 2, 23, 148, True, ""), m.SweepRow(16, 4, 8, 0, 0, False, "infeasible")]
    trails = [NS(time=44, wg=4, ts=4, transitions=1700), NS(time=50, wg=2, ts=2, transitions=10)]
    v = NS(violated=True, exhaustive=False,
           stats=NS(states_visited=15884, max_depth_reached=261, wall_seconds=0.0123456789),
           trace=NS(final_time=44, params=m.TuningParams(4, 4)))
    h = NS(violated=False, exhaustive=True,
           stats=NS(states_visited=0, max_depth_reached=0, wall_seconds=0.0), trace=None)
    t = NS(method="bisect", t_min=44, params=m.TuningParams(4, 4), t_ini=60, proven=True,
           first_trail_time=48, first_trail_optimality=lambda: 44 / 48,
           stats=NS(checks_run=8, states_visited_total=15884, wall_seconds=1.0),
           trace=NS(steps=261))
    expect = [report.sweep_to_csv(rows), report.sweep_to_json(rows), report.sweep_to_json([]),
              report.trails_to_csv(8, trails), report.verdict_to_json(v, 44, "out/trace.txt"),
              report.verdict_to_json(h, 43, ""), report.tune_result_to_json(t, "t.txt"),
              report.tune_result_to_csv(8, t)]
    for k, e in enumerate(expect):
        assert out[k] == e, (k, out[k], e)
    assert out[8] == "1 2 4 3 4 minimum 5 3 9 7\n"
    assert out[9] == "ConfigError\n"
