"""One data-parallel replica (launched by tests/test_multigpu_gpu.py under
torch.distributed.run, one process per GPU).  Every rank trains the whole linear
chain (depth --depth, width = world) on its column shard of every microbatch --
columns [r*b/w, (r+1)*b/w) of ToyModel::make(dim, L, b, ...) -- joins its stages'
NCCL communicators, and writes its final weights to <out>/rank<r>.npz.  The AllReduce
op sums the replicas' coalesced gradients and WeightUpdate divides by count * w
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
    ap.add_argument("--precision", choices=["fp64", "bf16"], default="fp64")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dim, L, b, m, T, seed = (8, 4, 8, 4, 5, 31) if a.precision == "fp64" else (128, 4, 128, 4, 4, 31)
    toy = O.ToyModel.make(dim, L, b, m * T, seed)
    cols = b // world
    kind = P.MODEL_LINEAR_F64 if a.precision == "fp64" else P.MODEL_LINEAR_BF16
    eng = P.Engine(model_kind=kind, policy=P.PipelinePolicy.TwoBW, depth=a.depth, microbatches=m,
                   microbatch_size=cols, layers=L, dim=dim, learning_rate=0.05, momentum=0.9)
    per = L // a.depth
    for s in range(a.depth):
        eng.load_stage_weights(s, np.concatenate([w.flatten(order="F") for w in toy.weights[s * per:(s + 1) * per]]))
    D.join_replicas(eng, a.depth)
    xs = np.stack([x[:, rank * cols:(rank + 1) * cols].flatten(order="F") for x, _ in toy.dataset])
    ys = np.stack([y[:, rank * cols:(rank + 1) * cols].flatten(order="F") for _, y in toy.dataset])
    eng.set_data(xs, ys, 1, m * T)
    eng.run_schedule(T, snapshots=True)
    eng.sync()
    w = np.concatenate([eng.snapshot(s, T) for s in range(a.depth)])
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), weights=w)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
