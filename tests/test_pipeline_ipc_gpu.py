"""Cross-process pipelines: one process per stage, hand-offs over CUDA IPC.

The reference interprets every stage in one loop (semantics.cpp:270-361); the
B200 engine can split the stages over processes (one per GPU), each process
interpreting its own program and handing out_act (:299) / grad_to_prev (:333) to
its neighbours through their exported receive blocks.  Results must be
BIT-IDENTICAL to the single-process engine: the same kernels run on the same
data in the same per-stage order, only the transport differs.  On the one-GPU
test box all ranks share the GPU (CUDA IPC within a device), which exercises the
same export / open / copy / flag protocol as the NVLink case."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import pipesim_oracle as O
from oracle import transformer_oracle as TO
from paper_2006_09503_b200 import pipesim as P

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(nproc: int, model: str, out: str, runs: int):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_pipeline_worker.py"), "--model", model, "--out", out, "--runs", str(runs)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(out, f"rank{i}.npz"))) for i in range(nproc)]


def _single_process_linear(depth: int, runs: int):
    dim, L, b, m, T, seed = 8, 4, 4, 4, 5, 77
    toy = O.ToyModel.make(dim, L, b, m * T * runs, seed)
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                   microbatch_size=b, layers=L, dim=dim, learning_rate=0.05, momentum=0.9)
    per = L // depth
    for s in range(depth):
        eng.load_stage_weights(s, np.concatenate([w.flatten(order="F") for w in toy.weights[s * per:(s + 1) * per]]))
    xs = np.stack([x.flatten(order="F") for x, _ in toy.dataset])
    ys = np.stack([y.flatten(order="F") for _, y in toy.dataset])
    losses = []
    for r in range(runs):
        rows = slice(r * m * T, (r + 1) * m * T)
        eng.set_data(xs[rows], ys[rows], 1, m * T)
        eng.run_schedule(T)
        eng.sync()
        losses.append(eng.losses(1, m * T))
    ws = [eng.read_version(s, T * runs) for s in range(depth)]
    eng.close()
    return ws, losses


def _single_process_transformer(depth: int, runs: int):
    spec = TO.Spec(layers=2 * depth, hidden=128, heads=2, seq=128, vocab=500, batch=2, causal=True, head_rows=0)
    m, T, seed = max(2, depth), 3, 99
    xs, ys = TO.synthetic_batch(spec, m * T * runs, seed + 1)
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                   microbatch_size=spec.batch, layers=spec.layers, hidden=spec.hidden, heads=spec.heads,
                   seq_len=spec.seq, vocab=spec.vocab, causal=1, head_rows=0, learning_rate=0.5, momentum=0.9,
                   seed=seed)
    eng.init_weights()
    losses = []
    for r in range(runs):
        rows = slice(r * m * T, (r + 1) * m * T)
        eng.set_data(xs[rows], ys[rows], 1, m * T)
        eng.run_schedule(T)
        eng.sync()
        losses.append(eng.losses(1, m * T))
    ws = [eng.read_master(s) for s in range(depth)]
    eng.close()
    return ws, losses


@pytest.mark.parametrize("nproc,runs", [(2, 1), (2, 2), (4, 1)])
def test_linear_pipeline_across_processes_is_bit_identical(tmp_path, nproc, runs):
    got = _launch(nproc, "linear", str(tmp_path), runs)
    ref_w, ref_l = _single_process_linear(nproc, runs)
    for g in got:
        s = int(g["stage"])
        assert np.array_equal(g["weights"], ref_w[s]), f"stage {s} weights differ"
    last = [g for g in got if int(g["stage"]) == nproc - 1][0]
    for r in range(runs):
        assert np.array_equal(last[f"losses{r}"], ref_l[r])


@pytest.mark.parametrize("nproc", [2, 3])
def test_transformer_pipeline_across_processes_is_bit_identical(tmp_path, nproc):
    got = _launch(nproc, "transformer", str(tmp_path), 2)
    ref_w, ref_l = _single_process_transformer(nproc, 2)
    for g in got:
        s = int(g["stage"])
        assert np.array_equal(g["weights"], ref_w[s]), f"stage {s} weights differ"
    last = [g for g in got if int(g["stage"]) == nproc - 1][0]
    for r in range(2):
        assert np.array_equal(last[f"losses{r}"], ref_l[r])


def test_unconnected_remote_stage_is_an_error():
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy.TwoBW, depth=2, microbatches=2,
                   microbatch_size=2, layers=2, dim=4, learning_rate=0.1, local_stages=(0, 1))
    try:
        assert eng.is_local(0) and not eng.is_local(1)
        with pytest.raises(P.PipesimError, match="another process"):
            eng.run_schedule(1)
        with pytest.raises(P.PipesimError, match="another process"):
            eng.read_version(1, 0)
    finally:
        eng.close()


def test_nccl_runtime_loads_on_the_gpu_box():
    """The data-parallel path dlopens libnccl.so.2 (torch's copy) at run time: the
    unique id that rank 0 shares with the replicas must come out of it."""
    from paper_2006_09503_b200 import dist as D
    a, b = D.nccl_unique_id(), D.nccl_unique_id()
    assert len(a) == D.UNIQUE_ID_BYTES and a != b


@pytest.mark.parametrize("depth", [1, 2])
def test_data_parallel_nccl_path_single_replica(depth):
    """The data-parallel path end to end on one GPU: a width-1 NCCL communicator per
    stage (ncclCommInitRank from the dlopened runtime, the AllReduce op's
    ncclAllReduce on the update stream, the 1/width scale) must leave 2BW training
    bit-identical to the engine without replicas -- the 8-GPU run differs only in
    the communicator's size."""
    import torch.distributed as dist

    from paper_2006_09503_b200 import dist as D

    spec = TO.Spec(layers=2, hidden=128, heads=2, seq=128, vocab=500, batch=2, causal=True)
    m, T = 2, 4
    ids, tg = TO.synthetic_batch(spec, m * T, 5)

    def run(join):
        eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                       microbatch_size=spec.batch, layers=spec.layers, hidden=spec.hidden, heads=spec.heads,
                       seq_len=spec.seq, vocab=spec.vocab, causal=1, learning_rate=0.3, momentum=0.9, seed=11)
        try:
            eng.init_weights()
            if join:
                D.join_replicas(eng, depth)
            eng.set_data(ids, tg, 1, m * T)
            eng.run_schedule(T)
            eng.sync()
            return eng.losses(1, m * T), [eng.read_master(s) for s in range(depth)]
        finally:
            eng.close()

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    os.environ["P2BW_NCCL_SINGLE_RANK"] = "1"  # build the communicator even for one replica
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        l_dp, w_dp = run(True)
    finally:
        dist.destroy_process_group()
        del os.environ["P2BW_NCCL_SINGLE_RANK"]
    l_ref, w_ref = run(False)
    assert np.array_equal(l_dp, l_ref)
    for a, b in zip(w_dp, w_ref):
        assert np.array_equal(a, b)
