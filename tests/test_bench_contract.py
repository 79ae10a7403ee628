"""bench.py's reference arm (CPU only): one JSON line with the contract's keys on
rank 0, nothing on the other ranks (the driver launches it under torchrun too)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmctune_ref.so"))
                    and not os.path.exists(os.path.join(ROOT, "oracle", "_build",
                                                        "libmctune_oracle.so")),
                    reason="checkers not built")
def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--cpu-sample-secs", "6"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    import bench
    assert d["config"] == json.loads(json.dumps(bench.bench_config(1)))  # same as the GPU arm's
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
    env["RANK"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       env=env, timeout=120, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_shard0_plan_counts_are_pinned():
    """The distinct launch plans of the timed shards quoted in the bench line."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.distinct_plans(bench.SPACE, 0, bench.PER_RANK) == bench.PLANS_SHARD0
    assert bench.distinct_plans(bench.RICH_SPACE, 0, bench.PER_RANK) == bench.RICH_PLANS_SHARD0
    # every configuration of the headline space is within the reference's 16-bit pid range:
    # processes = 2 + nwd + 2 nwd nwu + nwd nwu nwe <= 2 + wgs (3 + nwe)
    s = bench.SPACE
    logn = s["size"].bit_length() - 1
    worst = max(2 + (1 << (logn - lw - lt)) * (3 + (1 << min(lw, lp)))
                for lw in range(s["log2wg"][0], s["log2wg"][1] + 1)
                for lt in range(s["log2ts"][0], s["log2ts"][1] + 1)
                for lp in range(s["log2np"][0], s["log2np"][1] + 1))
    assert worst < 65535
