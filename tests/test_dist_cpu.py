"""N > 1 plumbing on CPU with gloo, world_size 2 (no GPU needed): the NCCL
unique-id exchange every replica uses to join its stage communicator, and the
max-over-ranks step time.  Also the data-parallel equivalence the AllReduce op
relies on: w replicas with b columns each, gradients averaged,
equal one pipeline with b*w columns -- checked on the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pipesim_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_09503_b200 import dist as D
    ids = D.share_unique_ids(3, lambda: bytes(range(rank * 7, rank * 7 + 128)))
    t = D.max_over_ranks(1.5 + rank)
    q.put((rank, ids, t))
    dist.destroy_process_group()


def test_unique_ids_and_max_over_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = {r: i for r, i, _ in out}
    assert ids[0] == ids[1] == bytes(range(0, 128)) * 3  # rank 0's ids everywhere
    assert all(t == 2.5 for _, _, t in out)


def _replica_gradient_average(model, W, t, m, w):
    """Each replica r sees columns [r*b/w, (r+1)*b/w) of every microbatch; the
    AllReduce sums their per-replica gradients, the update divides by m*w."""
    b = model.dataset[0][0].shape[1]
    cols = b // w
    total = [np.zeros_like(x) for x in W]
    for r in range(w):
        sub = O.ToyModel(model.dim, model.weights,
                         [(x[:, r * cols:(r + 1) * cols], y[:, r * cols:(r + 1) * cols]) for x, y in model.dataset])
        g, _ = O._batch_gradient(sub, W, t, m)  # mean over m microbatches of this replica
        total = [a + gi for a, gi in zip(total, g)]
    return [a / w for a in total]


@pytest.mark.parametrize("w", [2, 4])
def test_data_parallel_average_equals_wide_microbatch(w):
    model = O.ToyModel.make(6, 3, 8, 4, 5)
    W = model.weights
    g_dp = _replica_gradient_average(model, W, 1, 4, w)
    g_one, _ = O._batch_gradient(model, W, 1, 4)
    for a, b in zip(g_dp, g_one):
        assert np.allclose(a, b, rtol=1e-12, atol=1e-14)


def test_pipeline_rank_grid():
    """gpu = stage * width + replica (profile.cpp:99-101)."""
    from paper_2006_09503_b200.dist import grid
    assert [grid(8, r, 4) for r in range(8)] == [(s, w, 2) for s in range(4) for w in range(2)]
    assert [grid(4, r, 4)[0] for r in range(4)] == [0, 1, 2, 3]
    assert grid(8, 5, 1) == (0, 5, 8)
    with pytest.raises(ValueError):
        grid(6, 0, 4)


class _FakeEngine:
    """Stands in for the engine's stage-blob and replica-join entry points (no GPU):
    records what connect_pipeline / join_replicas hand it."""

    def __init__(self, depth, local):
        self.depth, self.local = depth, local
        self.connected, self.joined = [], None

    def is_local(self, s):
        return s == self.local

    def export_stage(self, s):
        assert s == self.local
        return bytes([s]) * 128

    def connect_stage(self, blob):
        self.connected.append(blob[0])


def _pipeline_worker(rank, world, port, depth, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_09503_b200 import dist as D
    stage, replica, width = D.grid(world, rank, depth)
    eng = _FakeEngine(depth, stage)
    D.connect_pipeline(eng, depth)
    ids_seen = []
    D.join_replicas(eng, depth, pipelined=True, make_id=lambda: os.urandom(128),
                    join=lambda e, ids, w, r: ids_seen.append((ids, w, r)))
    q.put((rank, stage, replica, sorted(eng.connected), ids_seen[0][0], ids_seen[0][1], ids_seen[0][2]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,depth", [(2, 2), (4, 2), (4, 4)])
def test_connect_pipeline_and_replica_groups_gloo(world, depth):
    """connect_pipeline's blob exchange (semantics.cpp:299 / :333 hand-offs across
    processes) and join_replicas' id sharing under world-size 2 / 4: each process
    connects exactly its stage's neighbours of the SAME replica, and every replica of a
    stage gets the same communicator id at rank = replica (gpu = stage * width + replica)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, world, port, depth, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    width = world // depth
    ids = {o[4] for o in out}
    assert len(ids) == 1 and len(next(iter(ids))) == 128 * depth  # one id per stage, shared by all
    for rank, stage, replica, connected, _, w, r in out:
        assert (stage, replica) == (rank // width, rank % width)
        assert connected == [s for s in (stage - 1, stage + 1) if 0 <= s < depth]
        assert (w, r) == (width, replica)


def _allreduce_worker(rank, world, port, q):
    """The AllReduce op's arithmetic across w replicas on gloo: each replica's gradient
    of its column shard, summed by the collective and divided by count * w at the
    update (engine.cpp issue_update), equals the wide-microbatch gradient."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    model = O.ToyModel.make(6, 3, 8, 4, 5)
    cols = 8 // world
    sub = O.ToyModel(model.dim, model.weights,
                     [(x[:, rank * cols:(rank + 1) * cols], y[:, rank * cols:(rank + 1) * cols]) for x, y in model.dataset])
    g, _ = O._batch_gradient(sub, model.weights, 1, 4)  # mean over the m microbatches
    flat = torch.from_numpy(np.concatenate([x.flatten() for x in g]))
    dist.all_reduce(flat)
    q.put((rank, (flat / world).numpy()))
    dist.destroy_process_group()


def test_allreduce_average_equals_wide_microbatch_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_allreduce_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    model = O.ToyModel.make(6, 3, 8, 4, 5)
    g_one, _ = O._batch_gradient(model, model.weights, 1, 4)
    want = np.concatenate([x.flatten() for x in g_one])
    assert np.array_equal(out[0], out[1])
    assert np.allclose(out[0], want, rtol=1e-12, atol=1e-14)


class _FakeReplicaEngine:
    """Stands in for export_replica / join_replicas_ipc (no GPU)."""

    def __init__(self, depth, local_stages, tag):
        self.depth, self.local_stages, self.tag = depth, local_stages, tag
        self.joined = {}

    def is_local(self, s):
        return s in self.local_stages

    def export_replica(self, s):
        return bytes([s, self.tag]) * 512

    def join_replicas_ipc(self, s, blobs, rank):
        self.joined[s] = ([b[1] for b in blobs], rank)


def _ipc_group_worker(rank, world, port, depth, pipelined, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_09503_b200 import dist as D
    local = [D.grid(world, rank, depth)[0]] if pipelined else list(range(depth))
    eng = _FakeReplicaEngine(depth, local, tag=rank)
    used = D.join_replicas(eng, depth, pipelined=pipelined, transport="ipc")
    q.put((rank, used, eng.joined))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,depth,pipelined", [(2, 1, False), (4, 2, False), (4, 2, True), (4, 1, True)])
def test_ipc_replica_groups_gloo(world, depth, pipelined):
    """join_replicas(transport="ipc"): every local stage joins with the blobs of exactly
    its replicas, in replica order, at rank = its replica index (pipelined: gpu = stage *
    width + replica; data parallel: every process holds every stage, replica = rank)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_group_worker, args=(r, world, port, depth, pipelined, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2006_09503_b200.dist import grid
    for rank, used, joined in out:
        assert used == "ipc"
        if pipelined:
            stage, replica, width = grid(world, rank, depth)
            assert joined == {stage: ([stage * width + q for q in range(width)], replica)}
        else:
            assert joined == {s: (list(range(world)), rank) for s in range(depth)}
