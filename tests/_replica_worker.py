"""One data-parallel replica (launched by tests/test_multigpu_gpu.py under
torch.distributed.run, one process per GPU -- or several per GPU for the
peer-memory transport, which CUDA IPC allows between processes on one device).  Every rank trains the whole linear
chain (depth --depth, width = world) on its column shard of every microbatch --
columns [r*b/w, (r+1)*b/w) of ToyModel::make(dim, L, b, ...) -- joins its stages'
replica group (--transport ipc: the AllReduce fused into the update kernel over
CUDA-IPC peer memory; nccl: NCCL communicators), and writes its final weights to
<out>/rank<r>.npz.  The AllReduce op sums the replicas' coalesced gradients and
WeightUpdate divides by count * w
(engine.cpp issue_update; costmodel.cpp:23-27 prices it), so every replica must end
with the weights of ONE pipeline fed the full b columns.

Test infrastructure: imports the oracle only to build the ToyModel."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pipesim_oracle as O  # noqa: E402
from paper_2006_09503_b200 import dist as D  # noqa: E402
from paper_2006_09503_b200 import pipesim as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--precision", choices=["fp64", "bf16", "transformer"], default="fp64")
    ap.add_argument("--transport", choices=["ipc", "nccl"], default="nccl")
    ap.add_argument("--optimizer", choices=["sgd", "adam"], default="sgd")
    ap.add_argument("--pipelined", action="store_true",
                    help="one stage per process (gpu = stage * width + replica), CUDA-IPC hand-offs")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    if a.precision == "transformer":
        return transformer(a, rank, world)
    dim, L, b, m, T, seed = (8, 4, 8, 4, 5, 31) if a.precision == "fp64" else (128, 4, 128, 4, 4, 31)
    toy = O.ToyModel.make(dim, L, b, m * T, seed)
    if a.pipelined:
        stage, replica, width = D.grid(world, rank, a.depth)
        mine = [stage]
    else:
        replica, width = rank, world
        mine = list(range(a.depth))
    cols = b // width
    kind = P.MODEL_LINEAR_F64 if a.precision == "fp64" else P.MODEL_LINEAR_BF16
    eng = P.Engine(model_kind=kind, policy=P.PipelinePolicy.TwoBW, depth=a.depth, microbatches=m,
                   microbatch_size=cols, layers=L, dim=dim, learning_rate=0.05, momentum=0.9,
                   local_stages=(mine[0], 1) if a.pipelined else None)
    per = L // a.depth
    for s in mine:
        eng.load_stage_weights(s, np.concatenate([w.flatten(order="F") for w in toy.weights[s * per:(s + 1) * per]]))
    if a.pipelined:
        D.connect_pipeline(eng, a.depth)
    assert D.join_replicas(eng, a.depth, pipelined=a.pipelined, transport=a.transport) == a.transport
    xs = np.stack([x[:, replica * cols:(replica + 1) * cols].flatten(order="F") for x, _ in toy.dataset])
    ys = np.stack([y[:, replica * cols:(replica + 1) * cols].flatten(order="F") for _, y in toy.dataset])
    eng.set_data(xs, ys, 1, m * T)
    eng.run_schedule(T, snapshots=True)
    eng.sync()
    w = np.concatenate([eng.snapshot(s, T) for s in mine])
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), weights=w, stages=np.array(mine))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


def transformer(a, rank, world):
    """Transformer replicas: replica r trains on sequences [r b, (r + 1) b) of every wide
    microbatch of b * world sequences (TRANSFORMER_WIDE below); writes each stage's fp32
    master."""
    from paper_2006_09503_b200 import synthetic as S
    sp = TRANSFORMER_WIDE
    b = sp["batch"] // world
    spec = S.TransformerSpec(**{k: sp[k] for k in ("layers", "hidden", "heads", "seq", "vocab", "batch", "causal")})
    m, T = sp["m"], sp["T"]
    ids, tg = S.token_batch(spec, m * T, 11)
    seq = spec.seq
    ids = ids.reshape(m * T, sp["batch"], seq)[:, rank * b:(rank + 1) * b].reshape(m * T, b * seq)
    tg = tg.reshape(m * T, sp["batch"], -1)[:, rank * b:(rank + 1) * b].reshape(m * T, -1)
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=a.depth, microbatches=m,
                   microbatch_size=b, layers=spec.layers, hidden=spec.hidden, heads=spec.heads, seq_len=seq,
                   vocab=spec.vocab, causal=1, learning_rate=sp["lr"], momentum=0.9, seed=7, optimizer=a.optimizer)
    eng.init_weights()
    assert D.join_replicas(eng, a.depth, transport=a.transport) == a.transport
    eng.set_data(np.ascontiguousarray(ids), np.ascontiguousarray(tg), 1, m * T)
    eng.run_schedule(T)
    eng.sync()
    w = np.concatenate([eng.read_master(s) for s in range(a.depth)])
    losses = eng.losses(1, m * T)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), weights=w, losses=losses)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


# the wide run both sides of the transformer replica test use (batch = sequences per
# wide microbatch, split over the replicas)
TRANSFORMER_WIDE = dict(layers=2, hidden=128, heads=2, seq=128, vocab=320, batch=4, causal=True, m=2, T=3, lr=0.5)


if __name__ == "__main__":
    main()
