"""Multi-GPU NCCL parity inside the suite (it ran only by hand).

When the box shows >= 2 CUDA devices, tools/mgpu_check.py runs under
torchrun (one process per GPU, NCCL over NVLink) at world size 2 and, with
>= 4 devices, 4: every golden case whose grid has that many ranks (the
reference's checksums, including the benchmarked configurations' shapes:
cfg3 circulant, cfg4 tetrahedral, cfg5 field split with its ordered fold),
extra grids against the single-GPU run (field splits n_pf = 2 and = world,
replicas, flattened circulant tasks), host-value delivery and the
per-rank output files. Skipped on a single-GPU box."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import cuda_available

ROOT = Path(__file__).resolve().parent.parent


def _devices() -> int:
    if not cuda_available():
        return 0
    import torch

    return torch.cuda.device_count()


pytestmark = [pytest.mark.gpu]


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_parity_under_torchrun(world):
    if _devices() < world:
        pytest.skip(f"needs {world} GPUs, {_devices()} visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           str(ROOT / "tools" / "mgpu_check.py")]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    rows = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    bad = [r for r in rows if not r.get("ok")]
    assert res.returncode == 0 and rows and not bad, (bad, res.stderr[-4000:])
    # the config-shaped golden cases of this world size all ran
    assert any(r.get("n_f") == 50000 for r in rows)
    assert any(r.get("n_f") == 2_000_000 for r in rows)
