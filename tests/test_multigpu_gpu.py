"""Multi-GPU paths; every test here needs >= 2 visible GPUs and is skipped otherwise
(the development box has one: these run on the 8-GPU node).

  - stages on distinct devices of one process: the producing kernel writes the next
    stage's receive-ring slot in PEER memory (the fp64 chain's SIMT stores, the bf16
    chain's TMA tensor stores from the GEMM epilogue) -- the reference's in-process
    hand-offs out_act / grad_to_prev (semantics.cpp:289-291, 299, 321-322, 333);
  - data-parallel replicas, one process per GPU: the AllReduce op's ncclAllReduce
    over a w = 2 communicator per stage (schedule.cpp:80-84, costmodel.cpp:23-27)
    against the wide-microbatch construction."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import pipesim_oracle as O
from paper_2006_09503_b200 import pipesim as P
from paper_2006_09503_b200 import synthetic as S
from tests import _golden as G

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count()


needs2 = pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")


def _flat(traj):
    return np.stack([np.stack([w.flatten(order="F") for w in ws]) for ws in traj])


@needs2
@pytest.mark.parametrize("idx", [i for i, (m, _) in enumerate(G.toy()) if m["depth"] >= 2])
def test_stages_on_distinct_devices_fp64_bit_identical(idx):
    """Peer stores into the neighbour's ring: the same goldens as one device."""
    meta, ref = G.toy()[idx]
    model = O.ToyModel.make(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"])
    toy = P.ToyModel(model.dim, model.weights, model.dataset)
    cfg = P.TrainerConfig(meta["lr"], meta["beta"], meta["m"], meta["T"])
    devs = [s % _gpus() for s in range(meta["depth"])]
    res = P.pipelined_execute(toy, cfg, P.PipelinePolicy(meta["policy"]), meta["depth"], devices=devs)
    assert O.max_rel_diff(_flat(res.trajectory), ref) == 0.0


@needs2
@pytest.mark.parametrize("depth", [2, 4, 8])
def test_stages_on_distinct_devices_bf16_bit_identical_to_one_device(depth):
    """The production path with the GEMM epilogue TMA-storing each stage's output into
    the next device's receive ring (and the dgrad into the previous one's gradient
    ring): bit-identical to every stage on one device (same kernels, same order)."""
    cfg = P.TrainerConfig(1e-3, 0.9, max(4, depth), 3)
    toy = P.ToyModel(256, *S.toy_model(256, 8, 128, cfg.microbatches_per_batch * 3, 5))
    one = P.pipelined_execute(toy, cfg, P.PipelinePolicy.TwoBW, depth, precision="bf16", with_losses=True)
    many = P.pipelined_execute(toy, cfg, P.PipelinePolicy.TwoBW, depth, precision="bf16", with_losses=True,
                               devices=[s % _gpus() for s in range(depth)])
    assert np.array_equal(_flat(one.trajectory), _flat(many.trajectory))
    assert np.array_equal(one.losses, many.losses)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@needs2
@pytest.mark.parametrize("precision,depth", [("fp64", 1), ("fp64", 2), ("bf16", 1)])
def test_nccl_replicas_equal_wide_microbatch(tmp_path, precision, depth):
    """w = 2 replicas (one process per GPU) on column shards, the AllReduce op summing
    their coalesced gradients over NCCL: every replica ends with the weights of one
    pipeline fed all b columns (fp64: to rounding, 1e-12; bf16: 2e-2 of Delta W)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_replica_worker.py"), "--out", str(tmp_path), "--depth", str(depth),
           "--precision", precision, "--transport", "nccl"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = [np.load(tmp_path / f"rank{i}.npz")["weights"] for i in range(2)]
    assert np.array_equal(got[0], got[1])  # the replicas stay identical
    dim, L, b, m, T, seed = (8, 4, 8, 4, 5, 31) if precision == "fp64" else (128, 4, 128, 4, 4, 31)
    model = O.ToyModel.make(dim, L, b, m * T, seed)
    traj, _, _ = O.pipelined_execute(model, 0.05, 0.9, m, T, O.TWOBW, depth)
    want = np.concatenate([w.flatten(order="F") for w in traj[-1]])
    w0 = np.concatenate([w.flatten(order="F") for w in model.weights])
    if precision == "fp64":
        assert O.max_rel_diff(got[0], want) < 1e-12
    else:
        assert np.linalg.norm((got[0] - w0) - (want - w0)) / np.linalg.norm(want - w0) < 2e-2
