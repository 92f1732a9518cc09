"""Do persistent GEMM CTAs start late inside the training step?  (diagnostic)

Runs a few GPT-2.2B-width layers through the engine with p2bw_debug_gemm_timing on and
prints, for the last GEMM launch of the step (a weight-gradient / dgrad of layer 0,
concurrent with the other stream), the spread of CTA entry and exit times (%globaltimer,
ns): a wide entry spread means some CTAs waited for SMs held by the concurrent kernel,
and with static round-robin tiles the kernel then ends late.
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200 import pipesim as P  # noqa: E402
from paper_2006_09503_b200 import synthetic as S  # noqa: E402
from paper_2006_09503_b200._lib import call  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
spec = S.TransformerSpec(layers=layers, hidden=1920, heads=30, seq=512, vocab=51200, batch=16, causal=True,
                         head_rows=0)
m = 4
eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=1, microbatches=m,
               microbatch_size=16, layers=layers, hidden=1920, heads=30, seq_len=512, vocab=51200, causal=1,
               learning_rate=1e-4, momentum=0.9, seed=1)
eng.init_weights()
ids, tg = S.token_batch(spec, m * 8, 3)
eng.set_data(ids, tg, 1, m * 8)
eng.run_schedule(2)
eng.sync()
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
for trial in range(3):
    buf.zero_()
    call("p2bw_debug_gemm_timing", C.c_void_p(buf.data_ptr()))
    eng.run_schedule(1)
    eng.sync()
    call("p2bw_debug_gemm_timing", C.c_void_p(0))
    t = buf.view(148, 8).cpu().numpy().astype(np.float64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    entry = (t[:, 0] - t0) / 1e3
    done = (t[:, 7] - t0) / 1e3
    print(f"trial {trial}: {used.sum()} CTAs; entry spread us: p50 {np.median(entry):.1f} p90 "
          f"{np.percentile(entry, 90):.1f} max {entry.max():.1f}; exit us: min {done.min():.1f} p50 "
          f"{np.median(done):.1f} max {done.max():.1f}")
eng.close()
