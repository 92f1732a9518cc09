"""Is the stage executor host-bound? (diagnostic)  BERT-base as bench.py; per batch,
the host time spent inside issue(t) against the device time per batch."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200 import pipesim as P  # noqa: E402

b, m, s, V = 16, 4, 512, 30522
eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=1, microbatches=m,
               microbatch_size=b, layers=12, hidden=768, heads=12, seq_len=s, vocab=V, causal=0, head_rows=77,
               learning_rate=1e-3, momentum=0.9, seed=1)
eng.init_weights()
rng = np.random.default_rng(0)
ids = rng.integers(0, V, size=(2 * m, b * s), dtype=np.int32)
tg = rng.integers(0, V, size=(2 * m, b * 77), dtype=np.int32)
eng.set_data(ids[:m], tg[:m], 1, m)
eng.set_data(ids[m:], tg[m:], m + 1, m)
eng.sync()
n = 14
for rep in range(2):
    eng.begin(n)
    host = []
    t_all = time.perf_counter()
    for t in range(1, n + 1):
        t0 = time.perf_counter()
        eng.issue(t)
        host.append(time.perf_counter() - t0)
    t_issue = time.perf_counter() - t_all
    eng.finish()
    eng.sync()
    t_wall = time.perf_counter() - t_all
    dev = eng.update_elapsed_ms(0, 3, n - 1) / (n - 4)
    print(f"rep {rep}: host issue per batch median {1e3 * float(np.median(host)):.2f} ms "
          f"(min {1e3 * min(host):.2f}, max {1e3 * max(host):.2f}); all issues {1e3 * t_issue:.1f} ms; "
          f"wall {1e3 * t_wall:.1f} ms; device per batch {dev:.2f} ms")
