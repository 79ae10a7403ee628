"""Data formats either side of the tuning path (reference: include/mctune/report.hpp,
src/report.cpp): config files, input arrays, CSV/JSON tables and summaries.

Pure formatting / parsing on the host; every number in them comes from the GPU.
JSON objects are written like nlohmann::json::dump(2) (keys sorted, 2-space indent).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Optional

from ._lib import ConfigError
from .model import PlatformConfig, ProblemSpec, kernel_kind_from_string

CSV_HEADER = "size,wg,ts,time,transitions\n"


@dataclass
class RunConfig:
    """(report.hpp:12-20)"""
    platform: PlatformConfig = field(default_factory=PlatformConfig)
    problem: ProblemSpec = field(default_factory=lambda: ProblemSpec.abstract(8))
    max_depth: int = 4_000_000
    max_states: int = 5_000_000
    workers: int = 4
    seed: int = 1
    output_dir: str = "out"


def read_input_file(path: str, expected: int) -> List[int]:
    """One decimal integer per line, exactly `expected` values (report.cpp:55-72)."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise ConfigError(f"cannot open input file: {path}")
    values = []
    for line in lines:
        if not line:
            continue
        try:
            values.append(int(line.strip()))
        except ValueError:
            raise ConfigError(f"bad integer '{line}' in {path}")
    if len(values) != expected:
        raise ConfigError(f"input file {path} holds {len(values)} values, expected {expected}")
    return values


def load_config_file(path: str) -> RunConfig:
    """{"platform": {nd, nu, np, gmt}, "problem": {size, kernel, input_path}} (report.cpp:13-53)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise ConfigError(f"cannot open config file: {path}")
    except json.JSONDecodeError as e:
        raise ConfigError(f"bad config JSON in {path}: {e}")
    cfg = RunConfig()
    p = j.get("platform", {})
    cfg.platform = PlatformConfig(p.get("nd", 1), p.get("nu", 1), p.get("np", 4), p.get("gmt", 4))
    if "problem" in j:
        q = j["problem"]
        size = q.get("size", 8)
        kind = kernel_kind_from_string(q.get("kernel", "abstract"))
        if kind == 1:
            inp = None
            if "input_path" in q:
                inp = read_input_file(os.path.join(os.path.dirname(path), q["input_path"]), size)
            cfg.problem = ProblemSpec.minimum(size, inp)
        else:
            cfg.problem = ProblemSpec.abstract(size)
    cfg.platform.validate()
    return cfg


def write_text_file(path: str, content: str) -> None:
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    with open(path, "w") as f:
        f.write(content)


def _dump(obj) -> str:
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def sweep_to_csv(rows) -> str:
    """report.cpp:99-111 (flagged rows keep their place with empty value fields)"""
    out = [CSV_HEADER]
    for r in rows:
        vals = f"{r.time},{r.transitions}" if r.ok else ","
        out.append(f"{r.size},{r.wg},{r.ts},{vals}\n")
    return "".join(out)


def sweep_to_json(rows) -> str:
    """report.cpp:113-129"""
    arr = []
    for r in rows:
        row = {"size": r.size, "wg": r.wg, "ts": r.ts}
        if r.ok:
            row.update(time=r.time, transitions=r.transitions)
        else:
            row["note"] = r.note
        arr.append(row)
    return _dump(arr)


def trails_to_csv(size: int, trails) -> str:
    """report.cpp:131-138"""
    return CSV_HEADER + "".join(f"{size},{t.wg},{t.ts},{t.time},{t.transitions}\n" for t in trails)


def verdict_to_json(v, T: int, trace_path: str = "") -> str:
    """report.cpp:140-155"""
    j = {"verdict": "violated" if v.violated else "holds", "exhaustive": v.exhaustive, "T": T,
         "states_visited": v.stats.states_visited,
         "max_depth_reached": v.stats.max_depth_reached,
         "wall_seconds": float(getattr(v.stats, "wall_seconds", 0.0))}
    if v.violated and v.trace is not None:
        j.update(final_time=v.trace.final_time, wg=v.trace.params.wg, ts=v.trace.params.ts)
    if trace_path:
        j["trace_path"] = trace_path
    return _dump(j)


def tune_result_to_json(r, trace_path: str = "") -> str:
    """report.cpp:157-172"""
    j = {"method": r.method, "t_min": r.t_min, "wg": r.params.wg, "ts": r.params.ts,
         "t_ini": r.t_ini, "proven": r.proven, "first_trail_time": r.first_trail_time,
         "first_trail_optimality": r.first_trail_optimality(),
         "stats": {"checks_run": r.stats.checks_run,
                   "states_visited_total": r.stats.states_visited_total,
                   "wall_seconds": r.stats.wall_seconds}}
    if trace_path:
        j["trace_path"] = trace_path
    return _dump(j)


def tune_result_to_csv(size: int, r) -> str:
    """report.cpp:174-180"""
    return CSV_HEADER + f"{size},{r.params.wg},{r.params.ts},{r.t_min},{r.trace.steps}\n"
