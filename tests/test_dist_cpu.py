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
