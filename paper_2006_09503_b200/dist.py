"""Multi-process plumbing for data-parallel replicas (torch.distributed is only
plumbing here: rendezvous, the NCCL unique-id exchange and max-over-ranks
timing).  The data-path collective itself is the engine's NCCL all-reduce at
the AllReduce op (include/p2bw.h: p2bw_engine_join_replicas)."""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

UNIQUE_ID_BYTES = 128


def share_unique_ids(n_ids: int, make_id: Callable[[], bytes]) -> bytes:
    """Rank 0 creates `n_ids` ids (one NCCL communicator per pipeline stage);
    every rank receives the same concatenated bytes."""
    rank = dist.get_rank()
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(n_ids * UNIQUE_ID_BYTES, dtype=torch.uint8, device=dev)
    if rank == 0:
        raw = b"".join(make_id() for _ in range(n_ids))
        if len(raw) != n_ids * UNIQUE_ID_BYTES:
            raise ValueError("unique ids must be 128 bytes each")
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, src=0)
    return bytes(buf.cpu().numpy().tobytes())


def max_over_ranks(value: float) -> float:
    """Time of the slowest rank (the contract's whole-job time)."""
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id from libp2bw.so (same libnccl as the engine)."""
    import ctypes as C

    from . import _lib
    buf = (C.c_ubyte * UNIQUE_ID_BYTES)()
    _lib.check(_lib.lib().p2bw_nccl_unique_id(buf, UNIQUE_ID_BYTES))
    return bytes(buf)


def join_replicas(engine, depth: int) -> None:
    """Make this process's pipeline one of `world` data-parallel replicas."""
    import ctypes as C

    from . import _lib
    ids = share_unique_ids(depth, nccl_unique_id)
    arr = (C.c_ubyte * len(ids)).from_buffer_copy(ids)
    _lib.check(_lib.lib().p2bw_engine_join_replicas(engine.h, arr, dist.get_world_size(), dist.get_rank()))
