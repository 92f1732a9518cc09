"""2BW against GPipe and PipeDream-Flush on the 24-layer
GPT (h 1024, 16 heads, s 512, V 51200, causal LM head on every position), depth
d in {2, 4, 8} and m in {4, 8, 16, 32} microbatches of b sequences.

One B200 runs all d stages (one stage stream each, the stages sharing the SMs), so
the measured samples/s is what one GPU shows of each schedule: a flush drains the
stage streams and leaves less independent work to overlap.  For every point it
records the steady samples/s (device events between weight updates at every stage,
max over stages, as bench.py), and from a second, traced pass the measured
SimReport document's bubble fraction / steady batch time (simulate()'s formulas on
measured op times, simulator.cpp:298-329) beside the closed-form pipeline bubble
of the schedule, (d - 1) / (m + d - 1) for GPipe / Flush and 0 for 2BW's steady state.

  python scripts/policy_sweep.py [out.json] [--quick]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2006_09503_b200 import pipesim as P  # noqa: E402

B, L, H, HEADS, S, V = 4, 24, 1024, 16, 512, 51200
WARM, STEPS = 2, 4


def run_point(policy, d, m):
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=policy, depth=d, microbatches=m, microbatch_size=B,
                   layers=L, hidden=H, heads=HEADS, seq_len=S, vocab=V, causal=1, learning_rate=1e-4,
                   momentum=0.9, seed=7)
    try:
        eng.init_weights()
        rng = np.random.default_rng(d * 100 + m)
        ids = rng.integers(0, V, size=(2 * m, B * S), dtype=np.int32)
        tgs = np.roll(ids, -1, axis=1)
        eng.set_data(ids[:m], tgs[:m], 1, m)  # the token ring holds two batches; later batches reuse it
        eng.set_data(ids[m:], tgs[m:], m + 1, m)
        eng.sync()
        n = WARM + STEPS

        def one_pass():
            eng.begin(n)
            for t in range(1, n + 1):
                eng.issue(t)
            eng.finish()
            eng.sync()

        one_pass()  # warm-up (kernel attributes, tensor maps, clocks)
        t0 = time.time()
        one_pass()
        wall = time.time() - t0
        ms = max(eng.update_elapsed_ms(s, WARM, WARM + STEPS) for s in range(d))
        sps = STEPS * m * B / (ms / 1e3)
        eng.set_trace(True)
        one_pass()
        rep = eng.trace_report()
        bubble_cf = 0.0 if policy == P.PipelinePolicy.TwoBW else (d - 1) / (m + d - 1)
        return {"policy": P.to_string(policy), "d": d, "m": m, "b": B, "samples_per_s": round(sps, 1),
                "steady_batch_ms": round(ms / STEPS, 3), "wall_s": round(wall, 3),
                "traced_throughput": round(rep["throughput"], 1),
                "traced_bubble_fraction": round(rep["bubble_fraction"], 4),
                "closed_form_bubble": round(bubble_cf, 4),
                "max_versions": max(x["versions"] for mem in rep["memory"] for x in mem)}
    finally:
        eng.close()


def main():
    out = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else None
    quick = "--quick" in sys.argv
    depths = (2, 4) if quick else (2, 4, 8)
    ms_ = (4, 8) if quick else (4, 8, 16, 32)
    pols = (P.PipelinePolicy.TwoBW, P.PipelinePolicy.GPipe, P.PipelinePolicy.PipeDreamFlush)
    rows = []
    for d in depths:
        for m in ms_:
            if m < d:
                continue
            for pol in pols:
                r = run_point(pol, d, m)
                rows.append(r)
                print(json.dumps(r), flush=True)
    doc = {"workload": f"gpt-24 (L {L}, h {H}, {HEADS} heads, s {S}, V {V}), b {B}, 1 B200 running all d stages",
           "rows": rows}
    if out:
        with open(out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
