"""bench.py contract checks that run without a GPU: the reference arm's JSON line, and the
algorithmic-byte bookkeeping the roofline is computed from."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=REPO, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["grid"] == [1080, 1920]


def test_reference_arm_other_ranks_exit_quietly():
    env = {**os.environ, "RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2"],
                       cwd=REPO, capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_algorithmic_bytes_match_survey_table():
    sys.path.insert(0, REPO)
    import bench
    ab = bench.algorithmic_bytes(1, 4141202)
    # lap 497.7 MB (10 it), bilateral 745.4 (5 it), tri 289.9 MB
    assert abs(ab["laplacian_per_launch"] * 10 / 1e6 - 497.7) < 0.5
    assert abs(ab["triangulate_per_launch"] / 1e6 - 289.9) < 0.5
    assert abs(ab["frame_total"] / 1e6 - 1756.7) < 1.0


def test_algorithmic_bytes_other_configs():
    sys.path.insert(0, REPO)
    import bench
    # 140.0 MB / frame (lap 22.1, FC 18.4, bil 44.1, tri 41.1, gather 14.3)
    ab = bench.algorithmic_bytes(1, 575884, bench.WORKLOADS["C2"])
    assert abs(ab["frame_total"] / 1e6 - 140.0) < 0.5
    assert abs(ab["triangulate_per_launch"] / 1e6 - 41.1) < 0.1
    # C3: no bilateral -> triangulation carries the l_max flags (T) and the normals (12T)
    ab = bench.algorithmic_bytes(1, 91991, bench.WORKLOADS["C3"])
    assert ab["bilateral_stage"] == 0
    assert abs(ab["triangulate_per_launch"] / 1e6 - (7.26 + 0.09 + 1.10)) < 0.02
    assert bench.WORKLOADS["C5"].total == 512
