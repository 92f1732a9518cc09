"""Activation recomputation (planner r flag planner.cpp:21-22,
Recompute op timing simulator.cpp:242-247): a Forward keeps only the stage input,
each Backward re-runs the stage forward first.  The numerics must not change."""
import numpy as np
import pytest

from oracle import pipesim_oracle as O
from paper_2006_09503_b200 import pipesim as P

pytestmark = pytest.mark.gpu


def _linear_run(policy, depth, m, T, recompute):
    model = O.ToyModel.make(8, 4, 4, m * T, 17)
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=policy, depth=depth, microbatches=m, microbatch_size=4,
                   layers=4, dim=8, learning_rate=0.05, momentum=0.9, recompute=recompute)
    per = 4 // depth
    for s in range(depth):
        eng.load_stage_weights(s, np.concatenate([w.flatten(order="F") for w in model.weights[s * per:(s + 1) * per]]))
    xs = np.stack([x.flatten(order="F") for x, _ in model.dataset])
    ys = np.stack([y.flatten(order="F") for _, y in model.dataset])
    eng.set_data(xs, ys, 1, m * T)
    eng.run_schedule(T)
    eng.sync()
    latest = T * (m if policy == P.PipelinePolicy.PipeDream1F1B else 1)
    out = np.concatenate([eng.read_version(s, latest) for s in range(depth)])
    losses = eng.losses(1, m * T)
    eng.close()
    return out, losses


@pytest.mark.parametrize("policy,depth,m", [(P.PipelinePolicy.TwoBW, 2, 2), (P.PipelinePolicy.TwoBW, 4, 4),
                                            (P.PipelinePolicy.PipeDream1F1B, 2, 2),
                                            (P.PipelinePolicy.GPipe, 2, 4)])
def test_linear_recompute_bit_identical(policy, depth, m):
    w0, l0 = _linear_run(policy, depth, m, 4, False)
    w1, l1 = _linear_run(policy, depth, m, 4, True)
    assert np.array_equal(w0, w1)
    assert np.array_equal(l0, l1)


def _tr_run(recompute, trace=False):
    m, T = 4, 4
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=2, microbatches=m,
                   microbatch_size=2, layers=4, hidden=128, heads=2, seq_len=128, vocab=512, causal=1,
                   learning_rate=0.05, momentum=0.9, seed=5, recompute=recompute)
    eng.init_weights()
    ids = np.random.default_rng(1).integers(0, 512, size=(m * T, 2 * 128), dtype=np.int32)
    eng.set_data(ids, np.roll(ids, -1, axis=1), 1, m * T)
    eng.set_trace(trace)
    eng.run_schedule(T)
    eng.sync()
    losses = eng.losses(1, m * T)
    rep = eng.trace_report() if trace else None
    w = eng.read_master(1)
    eng.close()
    return losses, w, rep


def test_transformer_recompute_matches_stashing():
    l0, w0, _ = _tr_run(False)
    l1, w1, rep = _tr_run(True, trace=True)
    # same kernels on the same inputs; only fp32 split-K reduction order may differ
    assert np.max(np.abs(l0 - l1) / np.abs(l0)) < 1e-3
    assert np.max(np.abs(w0 - w1)) < 1e-3 * np.max(np.abs(w0))
    # every backward is preceded by its recompute on the same stage
    for s in (0, 1):
        ops = [(e["op"], e["mb"]) for e in rep["timeline"] if e["worker"] == s and e["op"] in ("recompute", "backward")]
        assert ops and all(a[0] == "recompute" and b == ("backward", a[1]) for a, b in zip(ops[::2], ops[1::2]))
