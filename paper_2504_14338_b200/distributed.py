"""Multi-rank plumbing for one-process-per-GPU runs (torchrun).

torch.distributed carries only control traffic here: rank 0's NCCL unique id
(so every rank's C-ABI context joins one NCCL communicator) and the
max-over-ranks timing. The snapshot pass's own collectives (the MAX of the
scales and the K×K Gram reduction) run inside libdopinf_b200 over NCCL.
"""
from __future__ import annotations

import os


def env_ranks():
    """(rank, world_size, local_rank) from the torchrun environment (1 rank if absent)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init_control_plane(backend: str = "gloo"):
    """Join the torchrun group (MASTER_ADDR/PORT from the environment)."""
    import torch.distributed as dist

    rank, world, _ = env_ranks()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world


def share_unique_id(rank: int, fake: bytes | None = None) -> bytes:
    """Rank 0 creates the NCCL unique id (C ABI) and broadcasts its bytes."""
    import torch.distributed as dist

    from . import api

    payload = [None]
    if rank == 0:
        payload[0] = fake if fake is not None else api.DeviceContext.unique_id()
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast_object_list(payload, src=0)
    return payload[0]


def max_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return value
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
