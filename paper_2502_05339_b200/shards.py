"""Row-sharded multi-GPU plumbing.

One process per GPU (torchrun / torch.multiprocessing), `torch.distributed`
for the collectives: NCCL on GPUs, gloo for the CPU harness and for the
1-GPU multi-rank tests (their device tensors are staged through host memory
by `Shard`). The snapshot matrix, the sketch, the POD basis and the mode
tables are contiguous row blocks; every reduction over rows is one
all-reduce of a small block (Gram l x l, projection l x m, table Gram,
pair statistics) — see DESIGN.md §6 for the list and sizes.

Determinism: the reference promises bitwise-repeatable fits per seed
(tests/test_linalg.py:61-68 there). Within a rank every libfdmd reduction has
a fixed order; across ranks NCCL's algorithm and protocol are pinned (Ring /
Simple, whose summation order depends only on the world size), so a sharded
fit repeats bit for bit on the same world size.
"""

from __future__ import annotations

import os
from typing import Optional, Tuple

import numpy as np
import torch

from .device import Shard

# NCCL reduction order fixed (Ring / Simple): set before the first communicator
NCCL_PINS = {"NCCL_ALGO": "Ring", "NCCL_PROTO": "Simple"}


def pin_nccl():
    for k, v in NCCL_PINS.items():
        os.environ.setdefault(k, v)


def init_process_group(backend: Optional[str] = None) -> Tuple[int, int, int]:
    """Join the job described by RANK / WORLD_SIZE / LOCAL_RANK / MASTER_*
    (torchrun); NCCL when CUDA is present (one GPU per local rank), gloo
    otherwise. Returns (rank, world, local_rank)."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        pin_nccl()
        if torch.cuda.device_count() <= local:
            raise RuntimeError(f"local rank {local} has no GPU ({torch.cuda.device_count()} visible)")
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    return rank, world, local


def row_bounds(n: int, world: int) -> np.ndarray:
    """Contiguous, balanced row blocks: rank i owns [b[i], b[i+1])."""
    return np.linspace(0, n, world + 1).astype(np.int64)


def row_shard(n: int, group=None) -> Optional[Shard]:
    """This rank's Shard of an n-row matrix (None when not distributed)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b = row_bounds(n, world)
    return Shard(int(b[rank]), int(b[rank + 1] - b[rank]), n, group or dist.group.WORLD, world)
