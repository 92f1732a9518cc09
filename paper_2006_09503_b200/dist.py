"""Multi-process plumbing for pipelines and data-parallel replicas.

torch.distributed is only plumbing here: rendezvous, the exchange of NCCL
unique ids and of CUDA-IPC blobs, and max-over-ranks timing.  The data path is
the engine's: stage hand-offs over CUDA IPC (p2bw_engine_connect_stage) and the
replicas' gradient reduction -- on one node a fused reduce-scatter + optimizer +
all-gather kernel over CUDA-IPC peer memory (p2bw_engine_join_replicas_ipc),
across nodes the NCCL all-reduce at the AllReduce op (p2bw_engine_join_replicas).

Rank layout (profile.cpp:99-101): gpu = stage * width + replica."""
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


def grid(world: int, rank: int, depth: int) -> tuple[int, int, int]:
    """(stage, replica, width) of `rank` when `world` processes run a depth-`depth`
    pipeline, one stage per process: gpu = stage * width + replica."""
    if depth < 1 or world % depth:
        raise ValueError(f"{world} processes cannot form pipelines of depth {depth}")
    width = world // depth
    return rank // width, rank % width, width


def _engine_join(engine, ids: bytes, width: int, replica: int) -> None:
    import ctypes as C

    from . import _lib
    arr = (C.c_ubyte * len(ids)).from_buffer_copy(ids)
    _lib.check(_lib.lib().p2bw_engine_join_replicas(engine.h, arr, width, replica))


def one_node() -> bool:
    """Every rank runs on this host (CUDA IPC reaches all of them)."""
    import socket
    names: list = [None] * dist.get_world_size()
    dist.all_gather_object(names, socket.gethostname())
    return len(set(names)) == 1


def join_replicas(engine, depth: int, pipelined: bool = False, make_id: Callable[[], bytes] | None = None,
                  join: Callable | None = None, transport: str = "auto") -> str:
    """Join this process's stages to their data-parallel replica groups.

    pipelined=False: every process runs a whole pipeline (width = world).
    pipelined=True: one stage per process laid out by :func:`grid`.
    transport: "ipc" -- peer-memory groups (one node; the AllReduce fused into the
    update kernel); "nccl" -- every replica of every stage receives the same `depth`
    unique ids (one NCCL communicator per stage, rank = replica index; make_id / join
    default to the engine's p2bw_nccl_unique_id / p2bw_engine_join_replicas);
    "auto" -- ipc when every rank is on this host.  Returns the transport used."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if pipelined:
        _, replica, width = grid(world, rank, depth)
    else:
        replica, width = rank, world
    if transport == "auto":
        transport = "ipc" if (make_id is None and join is None and one_node()) else "nccl"
    if transport == "ipc":
        join_replicas_ipc(engine, depth, pipelined)
        return "ipc"
    ids = share_unique_ids(depth, make_id or nccl_unique_id)
    (join or _engine_join)(engine, ids, width, replica)
    return "nccl"


def join_replicas_ipc(engine, depth: int, pipelined: bool = False) -> None:
    """Peer-memory replica groups: each process exports its local stages
    (p2bw_engine_export_replica); every stage joins with the blobs of its replicas in
    replica order.  Collective over the default group."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if pipelined:
        _, replica, width = grid(world, rank, depth)
    else:
        replica, width = rank, world
    mine = {s: engine.export_replica(s) for s in range(depth) if engine.is_local(s)}
    gathered: list = [None] * world
    dist.all_gather_object(gathered, (replica, mine))
    for s in mine:
        group = {rep: blobs[s] for rep, blobs in gathered if s in blobs}
        if sorted(group) != list(range(width)):
            raise RuntimeError(f"stage {s}: replicas {sorted(group)} found, expected {width}")
        engine.join_replicas_ipc(s, [group[q] for q in range(width)], replica)
    dist.barrier()


def connect_pipeline(engine, depth: int) -> None:
    """Exchange CUDA-IPC stage blobs and connect each local stage's remote
    neighbours (same replica, stage +- 1).  Collective over the default group."""
    world, rank = dist.get_world_size(), dist.get_rank()
    _, replica, width = grid(world, rank, depth)
    mine = {s: engine.export_stage(s) for s in range(depth) if engine.is_local(s)}
    gathered: list = [None] * world
    dist.all_gather_object(gathered, (replica, mine))
    for rep, blobs in gathered:
        if rep != replica:
            continue
        for s, blob in blobs.items():
            if engine.is_local(s):
                continue
            if (s > 0 and engine.is_local(s - 1)) or (s + 1 < depth and engine.is_local(s + 1)):
                engine.connect_stage(blob)
    dist.barrier()
