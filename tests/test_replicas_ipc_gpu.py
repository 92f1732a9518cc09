"""Data-parallel replicas over CUDA-IPC peer memory (p2bw_engine_join_replicas_ipc):
the AllReduce op (schedule.cpp:80-84) fused into WeightUpdate -- each replica sums its
shard of every replica's coalesced gradient, applies the optimizer and stores the new
version of the shard into every replica.  CUDA IPC works between processes on one
device, so these run w = 2 and w = 4 replicas as 2-4 processes sharing cuda:0 -- the
same code path as one process per GPU minus the NVLink hop.

Parity: w replicas on column / sequence shards must train exactly as ONE pipeline fed
the whole microbatch (costmodel.cpp:23-27 prices the exchange):
  - fp64 linear chain against the oracle's pipelined_execute (semantics.cpp:238-375)
    on the wide ToyModel, to rounding (the replica sum is one more add);
  - bf16 linear chain and transformer against the same wide run within bf16
    tolerance;
  - every replica ends bit-identical (each shard has one writer)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import pipesim_oracle as O
from paper_2006_09503_b200 import pipesim as P
from paper_2006_09503_b200 import synthetic as S
from tests import _replica_worker as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(tmp_path, nproc, *args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_replica_worker.py"), "--out", str(tmp_path), "--transport", "ipc", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [np.load(tmp_path / f"rank{i}.npz") for i in range(nproc)]


@pytest.mark.parametrize("precision,depth,width", [("fp64", 1, 2), ("fp64", 2, 2), ("fp64", 1, 4), ("bf16", 1, 2),
                                                   ("bf16", 2, 2)])
def test_ipc_replicas_equal_wide_microbatch(tmp_path, precision, depth, width):
    got = [g["weights"] for g in _launch(tmp_path, width, "--depth", str(depth), "--precision", precision)]
    for g in got[1:]:
        assert np.array_equal(got[0], g)  # the replicas stay bit-identical
    dim, L, b, m, T, seed = (8, 4, 8, 4, 5, 31) if precision == "fp64" else (128, 4, 128, 4, 4, 31)
    model = O.ToyModel.make(dim, L, b, m * T, seed)
    traj, _, _ = O.pipelined_execute(model, 0.05, 0.9, m, T, O.TWOBW, depth)
    want = np.concatenate([w.flatten(order="F") for w in traj[-1]])
    w0 = np.concatenate([w.flatten(order="F") for w in model.weights])
    if precision == "fp64":
        # per element: (g_0 + g_1) / (count w) against the wide column sum / count
        assert O.max_rel_diff(got[0], want) < 1e-12
    else:
        assert np.linalg.norm((got[0] - w0) - (want - w0)) / np.linalg.norm(want - w0) < 2e-2


@pytest.mark.parametrize("precision", ["fp64", "bf16"])
def test_ipc_pipeline_of_replica_groups(tmp_path, precision):
    """Depth 2 x width 2 as four processes, one stage each (gpu = stage * width + replica):
    CUDA-IPC stage hand-offs inside each replica's pipeline AND a peer-memory replica group
    per stage -- the layout `bench.py --depth 2` uses under torchrun.  Each stage's two
    replicas end bit-identical and the whole equals one pipeline fed the wide microbatch."""
    res = _launch(tmp_path, 4, "--depth", "2", "--precision", precision, "--pipelined")
    by_stage = {}
    for r in res:
        by_stage.setdefault(int(r["stages"][0]), []).append(r["weights"])
    for s, ws in by_stage.items():
        assert np.array_equal(ws[0], ws[1]), s
    got = np.concatenate([by_stage[0][0], by_stage[1][0]])
    dim, L, b, m, T, seed = (8, 4, 8, 4, 5, 31) if precision == "fp64" else (128, 4, 128, 4, 4, 31)
    model = O.ToyModel.make(dim, L, b, m * T, seed)
    traj, _, _ = O.pipelined_execute(model, 0.05, 0.9, m, T, O.TWOBW, 2)
    want = np.concatenate([w.flatten(order="F") for w in traj[-1]])
    w0 = np.concatenate([w.flatten(order="F") for w in model.weights])
    if precision == "fp64":
        assert O.max_rel_diff(got, want) < 1e-12
    else:
        assert np.linalg.norm((got - w0) - (want - w0)) / np.linalg.norm(want - w0) < 2e-2


def _transformer_run(depth, optimizer, shard=None):
    """One engine in this process on the wide batch (shard=None) or on replica `shard`'s
    half of it alone (no reduction: the control)."""
    sp = W.TRANSFORMER_WIDE
    spec = S.TransformerSpec(**{k: sp[k] for k in ("layers", "hidden", "heads", "seq", "vocab", "batch", "causal")})
    m, T = sp["m"], sp["T"]
    ids, tg = S.token_batch(spec, m * T, 11)
    b = spec.batch
    if shard is not None:
        b //= 2
        ids = np.ascontiguousarray(ids.reshape(m * T, spec.batch, -1)[:, shard * b:(shard + 1) * b].reshape(m * T, -1))
        tg = np.ascontiguousarray(tg.reshape(m * T, spec.batch, -1)[:, shard * b:(shard + 1) * b].reshape(m * T, -1))
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                   microbatch_size=b, layers=spec.layers, hidden=spec.hidden, heads=spec.heads,
                   seq_len=spec.seq, vocab=spec.vocab, causal=1, learning_rate=sp["lr"], momentum=0.9, seed=7,
                   optimizer=optimizer)
    eng.init_weights()
    w0 = np.concatenate([eng.read_master(s) for s in range(depth)])
    eng.set_data(ids, tg, 1, m * T)
    eng.run_schedule(T)
    eng.sync()
    w = np.concatenate([eng.read_master(s) for s in range(depth)])
    losses = eng.losses(1, m * T)
    eng.close()
    return w0, w, losses


@pytest.mark.parametrize("depth,optimizer", [(1, "sgd"), (2, "sgd"), (1, "adam")])
def test_ipc_transformer_replicas_equal_wide_microbatch(tmp_path, depth, optimizer):
    """Two transformer replicas (2 sequences each) against one pipeline fed all 4: the
    same weight trajectory within bf16 tolerance (the two runs' GEMMs have different
    shapes and round differently) and the wide run's loss = the mean of the replicas'
    losses.  Adam's step lr m / sqrt(v) is ~lr for any gradient, rounding noise included,
    so its tolerance is looser; the control (replica 0's half alone, no reduction) must be
    several times further off, which is what proves the gradients were combined."""
    res = _launch(tmp_path, 2, "--depth", str(depth), "--precision", "transformer", "--optimizer", optimizer)
    got = [r["weights"] for r in res]
    assert np.array_equal(got[0], got[1])
    w0, want, wide_losses = _transformer_run(depth, optimizer)
    _, alone, _ = _transformer_run(depth, optimizer, shard=0)

    def rel(w):
        return float(np.linalg.norm((w - w0) - (want - w0)) / np.linalg.norm(want - w0))

    tol = 2e-2 if optimizer == "sgd" else 5e-2
    assert rel(got[0]) < tol, rel(got[0])
    assert rel(got[0]) < 0.25 * rel(alone), (rel(got[0]), rel(alone))
    mean_losses = 0.5 * (res[0]["losses"] + res[1]["losses"])
    assert np.allclose(mean_losses, wide_losses, rtol=1e-2), (mean_losses, wide_losses)
