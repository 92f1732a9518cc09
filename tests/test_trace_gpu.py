"""Measured timeline -> the reference's SimReport document.

The engine brackets every issued op with CUDA events; trace_report() renders the
run in report_to_json's layout (simulator.cpp:356-390) with throughput, steady
batch time and bubble fraction computed by simulate()'s own formulas
(simulator.cpp:298-329) from the measured times."""
import numpy as np
import pytest

from paper_2006_09503_b200 import pipesim as P

pytestmark = pytest.mark.gpu


def _transformer_engine(policy, depth, m):
    return P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=policy, depth=depth, microbatches=m,
                    microbatch_size=2, layers=4, hidden=128, heads=2, seq_len=128, vocab=512, causal=1,
                    learning_rate=0.01, momentum=0.9, seed=3)


@pytest.mark.parametrize("policy,depth,m", [(P.PipelinePolicy.TwoBW, 2, 2), (P.PipelinePolicy.TwoBW, 4, 4),
                                            (P.PipelinePolicy.GPipe, 2, 4), (P.PipelinePolicy.PipeDreamFlush, 2, 2)])
def test_trace_report_matches_programs(policy, depth, m):
    T = 5
    eng = _transformer_engine(policy, depth, m)
    eng.init_weights()
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 512, size=(m * T, 2 * 128), dtype=np.int32)
    eng.set_data(ids, ids, 1, m * T)
    eng.set_trace(True)
    eng.run_schedule(T)
    rep = eng.trace_report()
    eng.close()
    progs = P.generate_schedule(policy, depth, m, T)
    assert rep["policy"] == P.to_string(policy)
    assert rep["config"]["depth"] == depth and rep["config"]["microbatch_size"] == 2
    assert rep["num_batches"] == T and rep["measured"]
    assert rep["steady_batch_time"] > 0 and rep["throughput"] == pytest.approx(2 * m / rep["steady_batch_time"])
    assert 0.0 <= rep["bubble_fraction"] < 1.0
    for s, prog in enumerate(progs):
        mine = [e for e in rep["timeline"] if e["worker"] == s]
        # every program op once (a Forward may overlap the previous Backward on its own
        # stream, so the start-sorted timeline need not follow program order)
        assert sorted((e["op"], e["mb"]) for e in mine) == sorted((P._OP_TEXT[o.kind], o.microbatch) for o in prog.ops)
        assert all(e["start"] <= e["end"] for e in mine)
        fwd_end = {e["mb"]: e["end"] for e in mine if e["op"] == "forward"}
        for e in mine:
            if e["op"] == "backward":
                # a backward follows its forward (events a few us apart on two streams)
                assert e["start"] >= fwd_end[e["mb"]] - 2e-5
        mem = rep["memory"][s]
        assert len(mem) == len(prog.ops)
        assert max(x["versions"] for x in mem) <= (2 if policy == P.PipelinePolicy.TwoBW else 1)
