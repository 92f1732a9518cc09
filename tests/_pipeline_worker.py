"""One rank of a cross-process pipeline (launched by tests/test_pipeline_ipc_gpu.py
under torch.distributed.run).  Every rank runs ONE stage of a depth-`world`
pipeline (width 1) on the same GPU; the stages hand activations and gradients to
each other through CUDA IPC (p2bw_engine_export_stage / connect_stage).  Each rank
writes its stage's final weights (and the last stage its losses) to
<out>/rank<r>.npz for the parent test to compare against the single-process run.

Test infrastructure: imports the oracle only to build the linear ToyModel."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pipesim_oracle as O  # noqa: E402
from oracle import transformer_oracle as TO  # noqa: E402
from paper_2006_09503_b200 import dist as D  # noqa: E402
from paper_2006_09503_b200 import pipesim as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["linear", "transformer"], required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--runs", type=int, default=1)
    a = ap.parse_args()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    depth = world
    stage, _, _ = D.grid(world, rank, depth)
    out = {}
    if a.model == "linear":
        dim, L, b, m, T, seed = 8, 4, 4, 4, 5, 77
        toy = O.ToyModel.make(dim, L, b, m * T * a.runs, seed)
        eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                       microbatch_size=b, layers=L, dim=dim, learning_rate=0.05, momentum=0.9,
                       local_stages=(stage, 1))
        per = L // depth
        eng.load_stage_weights(stage, np.concatenate(
            [w.flatten(order="F") for w in toy.weights[stage * per:(stage + 1) * per]]))
        xs = np.stack([x.flatten(order="F") for x, _ in toy.dataset])
        ys = np.stack([y.flatten(order="F") for _, y in toy.dataset])
        dtype = np.float64
    else:
        spec = TO.Spec(layers=2 * depth, hidden=128, heads=2, seq=128, vocab=500, batch=2, causal=True, head_rows=0)
        m, T, seed = max(2, depth), 3, 99
        xs, ys = TO.synthetic_batch(spec, m * T * a.runs, seed + 1)
        eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                       microbatch_size=spec.batch, layers=spec.layers, hidden=spec.hidden, heads=spec.heads,
                       seq_len=spec.seq, vocab=spec.vocab, causal=1, head_rows=0, learning_rate=0.5, momentum=0.9,
                       seed=seed, local_stages=(stage, 1))
        eng.init_weights()
        dtype = np.float32
    # a process owns only its stage
    assert eng.is_local(stage) and all(not eng.is_local(s) for s in range(depth) if s != stage)
    D.connect_pipeline(eng, depth)
    # several runs exercise the flag sequence numbers carried across begin()
    for r in range(a.runs):
        rows = slice(r * m * T, (r + 1) * m * T)  # [microbatch, elements]
        eng.set_data(xs[rows], ys[rows], 1, m * T)
        eng.run_schedule(T)
        eng.sync()
        if stage == depth - 1:
            out[f"losses{r}"] = eng.losses(1, m * T)
    out["weights"] = eng.read_master(stage) if a.model == "transformer" else eng.read_version(stage, T * a.runs, dtype)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), stage=stage, **out)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
