"""The B200 stage executor on the reference's parity model (fp64 linear chain):
trajectories must be BIT-IDENTICAL to the reference's pipelined_execute
(golden vectors from the reference, tests/golden/toy_trajectories.*), for
GPipe / Flush / 2BW / 1F1B at depths 1-8 with every stage on its own stream.
Reference: semantics.cpp:238-375; semantics_test.cpp:199-231."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import pipesim_oracle as O
from paper_2006_09503_b200 import pipesim as P
from tests import _golden as G

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def _toy(meta):
    m = O.ToyModel.make(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"])
    return P.ToyModel(m.dim, m.weights, m.dataset)


def _flat(traj):
    return np.stack([np.stack([w.flatten(order="F") for w in ws]) for ws in traj])


@pytest.mark.parametrize("idx", range(len(G.toy())))
def test_engine_trajectory_bit_identical_to_reference(idx):
    meta, ref = G.toy()[idx]
    cfg = P.TrainerConfig(meta["lr"], meta["beta"], meta["m"], meta["T"])
    res = P.pipelined_execute(_toy(meta), cfg, P.PipelinePolicy(meta["policy"]), meta["depth"])
    got = _flat(res.trajectory)
    assert got.shape == ref.shape
    assert O.max_rel_diff(got, ref) == 0.0
    assert res.max_versions_held == meta["max_versions_held"]
    assert res.version_consistent


def test_2bw_holds_exactly_two_versions_and_is_not_vanilla():
    meta, ref = G.toy()[0]
    model = O.ToyModel.make(8, 4, 4, 4 * 6, 5)
    toy = P.ToyModel(model.dim, model.weights, model.dataset)
    cfg = P.TrainerConfig(0.05, 0.9, 4, 6)
    twobw = P.pipelined_execute(toy, cfg, P.PipelinePolicy.TwoBW, 4)
    vanilla = P.pipelined_execute(toy, cfg, P.PipelinePolicy.GPipe, 4)
    assert twobw.max_versions_held == 2
    assert O.max_rel_diff(_flat(twobw.trajectory), _flat(vanilla.trajectory)) > 1e-6
    delayed, _ = O.reference_loop(model, 0.05, 0.9, 4, 6, True)
    assert O.max_rel_diff(_flat(twobw.trajectory), O.flat_trajectory(delayed)) == 0.0


def test_engine_rejects_discarded_version_and_bad_shapes():
    model = O.ToyModel.make(4, 2, 2, 8, 3)
    toy = P.ToyModel(model.dim, model.weights, model.dataset)
    with pytest.raises(P.PipesimError, match="not divisible"):
        P.pipelined_execute(toy, P.TrainerConfig(0.1, 0.0, 2, 2), P.PipelinePolicy.GPipe, 3)
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy.TwoBW, depth=1, microbatches=1,
                   microbatch_size=2, layers=2, dim=4, learning_rate=0.1)
    eng.load_stage_weights(0, np.concatenate([w.flatten(order="F") for w in model.weights]))
    xs = np.concatenate([x.flatten(order="F") for x, _ in model.dataset])
    ys = np.concatenate([y.flatten(order="F") for _, y in model.dataset])
    eng.set_data(xs, ys, 1, 8)
    ops = [P.ScheduledOp(P.OpKind.Forward, 1, 0), P.ScheduledOp(P.OpKind.Backward, 1, 0),
           P.ScheduledOp(P.OpKind.WeightUpdate), P.ScheduledOp(P.OpKind.Forward, 2, 0),
           P.ScheduledOp(P.OpKind.Backward, 2, 0), P.ScheduledOp(P.OpKind.WeightUpdate),
           P.ScheduledOp(P.OpKind.Forward, 3, 0)]  # version 0 was discarded by the 2nd update
    with pytest.raises(P.PipesimError, match="needs discarded weight version 0"):
        eng.run([P.StageProgram(0, ops)])
    eng.close()


def test_engine_detects_deadlock():
    model = O.ToyModel.make(4, 2, 2, 4, 3)
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy.GPipe, depth=2, microbatches=1,
                   microbatch_size=2, layers=2, dim=4, learning_rate=0.1)
    for s in range(2):
        eng.load_stage_weights(s, model.weights[s].flatten(order="F"))
    xs = np.concatenate([x.flatten(order="F") for x, _ in model.dataset])
    ys = np.concatenate([y.flatten(order="F") for _, y in model.dataset])
    eng.set_data(xs, ys, 1, 4)
    # stage 0 waits for a backward of microbatch 1 that stage 1 never runs
    s0 = [P.ScheduledOp(P.OpKind.Forward, 1, 0), P.ScheduledOp(P.OpKind.Backward, 1, 0)]
    s1 = [P.ScheduledOp(P.OpKind.Forward, 1, 0), P.ScheduledOp(P.OpKind.Forward, 2, 0)]
    with pytest.raises(P.PipesimError, match="deadlock"):
        eng.run([P.StageProgram(0, s0), P.StageProgram(1, s1)])
    eng.close()


@pytest.mark.skipif(not (BIN / "dropin_gpu_tests").exists(), reason="drop-in harness not built")
def test_reference_semantics_and_acceptance_suites_on_gpu_engine():
    r = subprocess.run([str(BIN / "dropin_gpu_tests")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "failed: 0 | assertions:" in r.stdout


@pytest.mark.parametrize("idx", range(len(G.loops())))
def test_engine_reference_loops_bit_identical_at_any_m(idx):
    """reference_vanilla / reference_2bw (semantics.cpp:188-194) on the engine: with
    reference_loop's per-microbatch 1/m scaling (:145) they match the reference's loop
    goldens bit for bit at m = 3..6, where pipelined_execute's sum / count (:338-340)
    differs from them in the last bits."""
    meta, ref = G.loops()[idx]
    model = O.ToyModel.make(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"])
    toy = P.ToyModel(model.dim, model.weights, model.dataset)
    cfg = P.TrainerConfig(meta["lr"], meta["beta"], meta["m"], meta["T"])
    fn = P.reference_2bw if meta["delayed"] else P.reference_vanilla
    assert O.max_rel_diff(_flat(fn(toy, cfg)), ref) == 0.0
    pol = P.PipelinePolicy.TwoBW if meta["delayed"] else P.PipelinePolicy.GPipe
    piped = _flat(P.pipelined_execute(toy, cfg, pol, 1).trajectory)
    gap = O.max_rel_diff(piped, ref)
    assert (gap == 0.0) if meta["m"] in (1, 2, 4, 8) else (0.0 < gap < 1e-12)


def test_load_stage_weights_after_a_run_replaces_the_live_version():
    """A reload between runs lands in the latest version's buffer: the next
    run starts from the loaded weights whichever slot 2BW left them in."""
    model = O.ToyModel.make(8, 2, 4, 12, 5)
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy.TwoBW, depth=1, microbatches=2,
                   microbatch_size=4, layers=2, dim=8, learning_rate=0.05, momentum=0.0)
    w0 = np.concatenate([w.flatten(order="F") for w in model.weights])
    xs = np.concatenate([x.flatten(order="F") for x, _ in model.dataset])
    ys = np.concatenate([y.flatten(order="F") for _, y in model.dataset])
    eng.load_stage_weights(0, w0)
    eng.set_data(xs, ys, 1, 12)
    eng.run_schedule(3)  # 3 updates: version 3 lives in slot 1
    eng.sync()
    eng.load_stage_weights(0, w0)
    got = eng.read_version(0, 3)
    eng.close()
    assert np.array_equal(got, w0)


def test_set_data_in_pieces_keeps_earlier_microbatches():
    """Ranged set_data: growing the dataset keeps what was uploaded before."""
    meta, ref = G.toy()[0]
    model = O.ToyModel.make(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"])
    n = meta["m"] * meta["T"]
    eng = P.Engine(model_kind=P.MODEL_LINEAR_F64, policy=P.PipelinePolicy(meta["policy"]), depth=meta["depth"],
                   microbatches=meta["m"], microbatch_size=meta["b"], layers=meta["layers"], dim=meta["dim"],
                   learning_rate=meta["lr"], momentum=meta["beta"])
    per = meta["layers"] // meta["depth"]
    for s in range(meta["depth"]):
        eng.load_stage_weights(s, np.concatenate([w.flatten(order="F") for w in model.weights[s * per:(s + 1) * per]]))
    for k in range(1, n + 1):  # one microbatch per call
        x, y = model.dataset[k - 1]
        eng.set_data(x.flatten(order="F"), y.flatten(order="F"), k, 1)
    eng.run_schedule(meta["T"], snapshots=True)
    eng.sync()
    last = np.concatenate([eng.snapshot(s, meta["T"]).reshape(per, -1) for s in range(meta["depth"])])
    eng.close()
    assert O.max_rel_diff(last, ref[-1]) == 0.0
