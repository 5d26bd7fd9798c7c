"""bench.py --gpus N launches N ranks itself when no torchrun environment is
present (the driver's 1/2/4/8-GPU runs must really run N ranks),
and refuses a torchrun world that disagrees with --gpus. CPU only: the
--launch-check mode exercises the same self-launch and rank plumbing over
gloo and reports every rank's world and plan."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    return env


@pytest.mark.parametrize("config,n", [("cfg2", 2), ("cfg5", 2), ("cfg2", 3)])
def test_bench_self_launches_n_ranks(config, n):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n),
                          "--config", config, "--launch-check"], cwd=ROOT, env=_env(),
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout  # one JSON line, from rank 0 only
    out = json.loads(lines[0])
    assert out["n_gpus"] == n and out["gpus_arg"] == n
    assert sorted(r[0] for r in out["ranks"]) == list(range(n))
    assert all(r[1] == n for r in out["ranks"])
    want = f"field split n_pf={n}" if config == "cfg5" else f"circulant n_pv={n}"
    assert out["parallelism"] == want
    assert "self-launch" in res.stderr


def test_bench_rejects_world_size_mismatch():
    env = _env()
    env.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4",
                          "--launch-check"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=120)
    assert res.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 4" in res.stderr
