"""Data formats either side of the path (report.hpp) — host formatting of GPU results."""
import json
import os

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
