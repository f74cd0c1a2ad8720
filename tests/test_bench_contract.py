"""bench.py's reference arm on CPU (no GPU needed): one JSON line with the contract's keys,
timed on the oracle port, for a small workload (GPT-2 shape, batch 1)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "gpt2_fp16",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "tok/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["steps_requested"] == 2
    assert d["config"]["workload"] == "gpt2_fp16"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_launch_plan():
    """`bench.py --gpus N` starts its own ranks when no launcher did; under torchrun it checks
    WORLD_SIZE against --gpus; the reference arm never spawns."""
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.launch_plan(1, "ours", {}, []) == ("run", None)
    assert bench.launch_plan(4, "reference", {}, []) == ("run", None)
    assert bench.launch_plan(2, "ours", {"WORLD_SIZE": "2"}, []) == ("run", None)
    mode, cmd = bench.launch_plan(8, "ours", {}, ["--gpus", "8", "--steps", "5"])
    assert mode == "spawn"
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "5"][-3:]
    import pytest
    with pytest.raises(SystemExit):
        bench.launch_plan(4, "ours", {"WORLD_SIZE": "2"}, [])
