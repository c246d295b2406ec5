"""bench.py contract pieces that run without a GPU: the reference arm (the fp64 oracle on the
host, BASELINE configs[0]) prints one JSON line with the keys the driver reads, and the
multi-GPU layout label both arms print."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                        "c0_sbm2k", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT, env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["steps"] == 2 and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c0_sbm2k" and d["config"]["parallelism"] == "single GPU"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_grid_label_matches_decomposition():
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    from scinputs import configs
    w = configs.WORKLOADS["c3_sbm1m"]
    args = argparse.Namespace(col_groups=0)
    assert bench.grid_label(args, w, 1) == "single GPU"
    assert bench.grid_label(args, w, 8).startswith("2 column groups x 4 row blocks")
    assert bench.grid_label(argparse.Namespace(col_groups=1), w, 4) == "row-partitioned x4"
