"""torch.distributed plumbing for transport="nccl".

The data path of a multi-GPU run is libpsim's own (csrc/runtime.cu:
psim_run2 / psim_run3 drive every NCCL send / recv, the ordered field
reduce-scatter and the totals gather on their own communicator; runtime.py
binds them). torch.distributed only brings the processes up (the torchrun
environment), passes rank 0's 128-byte NCCL id once, and carries the
collective output writer's record routing (output.py).
``transport="nccl"`` requires world_size == grid.n_p; rank r takes the
reference's coordinates coords_of_rank(r) (field-fastest, core.py:83-97).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .domain import ConfigError, n_ranks


def ensure_initialized(grid) -> tuple[int, int]:
    """Initialise the default NCCL group from the torchrun environment if needed."""
    if not dist.is_initialized():
        if "RANK" not in os.environ:
            raise ConfigError("transport='nccl' needs a torch.distributed launch (torchrun)")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    if world != n_ranks(grid):
        raise ConfigError(f"transport='nccl' needs world_size == grid.n_p "
                          f"({world} != {n_ranks(grid)})")
    return world, rank
