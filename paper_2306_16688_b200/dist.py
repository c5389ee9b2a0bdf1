"""Process-group plumbing for multi-GPU runs (one process per GPU).  torch.distributed is
used only to bootstrap: rank 0's NCCL unique id is broadcast to every rank, after which the
library's own NCCL communicator carries the a2/a6 exchanges."""
from __future__ import annotations

import os

import torch


def env_ranks():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def broadcast_unique_id(make_id=None, device=None) -> bytes:
    """Rank 0 makes a 128-byte NCCL unique id (srl_nccl_unique_id by default); every rank of the
    default process group returns the same bytes.  Works over gloo (CPU) and nccl (device)."""
    import torch.distributed as dist
    if make_id is None:
        from .srl import nccl_unique_id as make_id
    buf = torch.zeros(128, dtype=torch.uint8, device=device or "cpu")
    if dist.get_rank() == 0:
        raw = make_id()
        assert len(raw) == 128
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())
