"""The PRODUCTION path pinned to the reference itself.

P2BW_MODEL_LINEAR_BF16 runs the reference's ToyModel (semantics.hpp:31-43) through the
kernels and streams the transformer bench uses: the tcgen05 GEMM for the forward (W as
an MN-major operand), the dgrad (K-major) and the wgrad (fp32 epilogue: store on the
batch's first microbatch, TMA reduce-add afterwards, on the weight-gradient side
stream), k_sgd writing the next bf16 version into the alternate buffer on the update
stream, double-buffered gradients, the forward stream.  Its trajectories are compared
with the reference's pipelined_execute (semantics.cpp:238-375) -- golden vectors from
oracle/_ref/ref_tool at the configs' widths (dim 256 / 768 / 1024, 4-12 layers,
128-512 columns, d 1-8, m 3-8, 2BW and 1F1B; tests/golden/make_golden.py BF16_GRID).

Tolerance (bf16): every microbatch's activations and the weights the GEMMs read are
bf16 (8-bit significand, unit roundoff 2^-9), the master / momentum / gradient fp32.
A float emulation of exactly that rounding (same configs) puts the relative Frobenius
error of Delta W(t) = W(t) - W(0) at 0.3-0.7%; DELTA_TOL = 2e-2 leaves ~3x headroom.
The 2BW trajectory differs from vanilla SGD by 9-31% at the last snapshot of every
configuration, so the test also asserts a margin: a semantics error (wrong version,
missing delay, wrong normalisation) moves the result by far more than the tolerance."""
import numpy as np
import pytest

from paper_2006_09503_b200 import pipesim as P
from paper_2006_09503_b200 import synthetic as S
from tests import _golden as G

pytestmark = pytest.mark.gpu

DELTA_TOL = 2e-2   # relative Frobenius error of Delta W(t), sampled entries
MARGIN = 3.0       # the 2BW-vs-vanilla gap must exceed MARGIN * DELTA_TOL at the last snapshot

CASES = {m["name"]: (m, g) for m, g in G.linear_bf16()}


def _run(meta):
    ws, data = S.toy_model(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"],
                           exact=meta["dim"] <= 256)
    toy = P.ToyModel(meta["dim"], ws, data)
    cfg = P.TrainerConfig(meta["lr"], meta["beta"], meta["m"], meta["T"])
    return P.pipelined_execute(toy, cfg, P.PipelinePolicy(meta["policy"]), meta["depth"], precision="bf16",
                               with_losses=True)


@pytest.mark.parametrize("name", sorted(CASES))
def test_bf16_trajectory_tracks_reference_pipelined_execute(name):
    meta, g = CASES[name]
    res = _run(meta)
    L, T = meta["layers"], meta["T"]
    idx = g["idx"]
    w0 = [w.flatten(order="F") for w in res.trajectory[0]]
    errs = []
    for t in range(1, T + 1):
        d_eng = np.stack([(res.trajectory[t][l].flatten(order="F") - w0[l])[idx[l]] for l in range(L)])
        d_ref = g["d_ref"][t].astype(np.float64)
        errs.append(np.linalg.norm(d_eng - d_ref) / np.linalg.norm(d_ref))
    gap = g["norm_gap"][T] / g["norm_ref"][T]  # exact, from the full reference matrices
    print(f"{name}: rel err of Delta W per snapshot {np.round(errs, 5).tolist()}, 2BW vs vanilla {gap:.4f}")
    assert max(errs) < DELTA_TOL, errs
    assert gap > MARGIN * DELTA_TOL, gap
    # the engine's own distance to vanilla SGD shows the 2BW delay, not vanilla's update
    d_van = g["d_van"].astype(np.float64)  # the last snapshot
    d_eng = np.stack([(res.trajectory[T][l].flatten(order="F") - w0[l])[idx[l]] for l in range(L)])
    assert np.linalg.norm(d_eng - d_van) / np.linalg.norm(g["d_ref"][T]) > MARGIN * DELTA_TOL
    assert res.version_consistent
    assert res.max_versions_held == meta["max_versions_held"]
    assert np.all(np.isfinite(res.losses))


def test_bf16_losses_track_the_fp64_engine():
    """Per-microbatch losses of the bf16 path against the bit-exact fp64 engine on the
    same small chain (both fed by ToyModel::make): loss is formed in fp32 from the fp32
    network output, so the bf16 activations set the error (LOSS_RTOL 1e-2)."""
    ws, data = S.toy_model(64, 4, 64, 8, 3)
    toy = P.ToyModel(64, ws, data)
    cfg = P.TrainerConfig(0.05, 0.9, 4, 2)
    a = P.pipelined_execute(toy, cfg, P.PipelinePolicy.TwoBW, 2, precision="bf16", with_losses=True)
    b = P.pipelined_execute(toy, cfg, P.PipelinePolicy.TwoBW, 2, with_losses=True)
    assert np.max(np.abs(a.losses - b.losses) / np.abs(b.losses)) < 1e-2
    assert a.max_versions_held == b.max_versions_held == 2


def test_bf16_streamed_batches_match_one_upload():
    """The bf16 stage's data ring (capacity max(count, 2m)): feeding batch after batch
    through begin / set_data / issue gives the same weights as one upload of every batch."""
    ws, data = S.toy_model(64, 2, 32, 12, 9)
    m, T = 2, 6
    flat_w = np.concatenate([w.flatten(order="F") for w in ws])
    xs = np.stack([x.flatten(order="F") for x, _ in data])
    ys = np.stack([y.flatten(order="F") for _, y in data])

    def engine():
        e = P.Engine(model_kind=P.MODEL_LINEAR_BF16, policy=P.PipelinePolicy.TwoBW, depth=1, microbatches=m,
                     microbatch_size=32, layers=2, dim=64, learning_rate=0.05, momentum=0.9)
        e.load_stage_weights(0, flat_w)
        return e

    a = engine()
    a.set_data(xs, ys, 1, m * T)
    a.run_schedule(T)
    a.sync()
    wa = a.read_master(0, np.float64)
    a.close()
    b = engine()
    b.set_data(xs[:2 * m], ys[:2 * m], 1, 2 * m)  # ring of 2m microbatches
    b.begin(T)
    for t in range(1, T + 1):
        if t >= 2 and t + 1 <= T:
            b.set_data(xs[t * m:(t + 1) * m], ys[t * m:(t + 1) * m], t * m + 1, m)
        b.issue(t)
    b.finish()
    b.sync()
    wb = b.read_master(0, np.float64)
    b.close()
    assert np.array_equal(wa, wb)


def test_device_toy_model_matches_toymodel_make():
    """init_weights / make_toy_data generate ToyModel::make on the device (the bench's
    same-config workload): the weights equal the reference's rounded to fp32, and a run
    on the device-made data tracks a run on the host-made dataset (y = A x differs by the
    bf16 GEMM's rounding only)."""
    dim, L, b, m, T, seed = 128, 4, 64, 2, 3, 2024
    ws, data = S.toy_model(dim, L, b, m * T, seed)
    kw = dict(model_kind=P.MODEL_LINEAR_BF16, policy=P.PipelinePolicy.TwoBW, depth=2, microbatches=m,
              microbatch_size=b, layers=L, dim=dim, learning_rate=0.05, momentum=0.9, seed=seed)
    a = P.Engine(**kw)
    a.init_weights()
    for s in range(2):
        want = np.concatenate([w.flatten(order="F") for w in ws[2 * s:2 * s + 2]]).astype(np.float32)
        assert np.array_equal(a.read_master(s, np.float64).astype(np.float32), want)
    a.make_toy_data(1, m * T)
    a.run_schedule(T)
    a.sync()
    got = [a.read_master(s, np.float64) for s in range(2)]
    la = a.losses(1, m * T)
    a.close()
    bb = P.Engine(**kw)
    for s in range(2):
        bb.load_stage_weights(s, np.concatenate([w.flatten(order="F") for w in ws[2 * s:2 * s + 2]]))
    bb.set_data(np.stack([x.flatten(order="F") for x, _ in data]), np.stack([y.flatten(order="F") for _, y in data]),
                1, m * T)
    bb.run_schedule(T)
    bb.sync()
    want = [bb.read_master(s, np.float64) for s in range(2)]
    lb = bb.losses(1, m * T)
    bb.close()
    w0 = np.concatenate([w.flatten(order="F") for w in ws])
    dg, dw = np.concatenate(got) - w0, np.concatenate(want) - w0
    assert np.linalg.norm(dg - dw) / np.linalg.norm(dw) < 2e-2
    assert np.max(np.abs(la - lb) / lb) < 2e-2


def test_graph_run_equals_eager_runs_linear_bf16():
    """CUDA-graph mode on the bf16 linear chain (production GEMMs, k_sgd, side stream),
    after an eager run: 2 launches of a 4-batch 2BW run equal 2 eager runs bit for bit
    (no run-order-dependent reductions on this path)."""
    outs = []
    for mode in ("eager", "graph"):
        eng = P.Engine(model_kind=P.MODEL_LINEAR_BF16, policy=P.PipelinePolicy.TwoBW, depth=2, microbatches=2,
                       microbatch_size=128, layers=4, dim=128, learning_rate=1e-3, momentum=0.9, seed=9)
        eng.init_weights()
        eng.make_toy_data(1, 4)
        eng.run_schedule(4)
        if mode == "eager":
            eng.run_schedule(4)
            eng.run_schedule(4)
        else:
            eng.run_schedule_graph(4, 2)
        eng.sync()
        outs.append(np.concatenate([eng.read_version(s, 12) for s in range(2)]))  # 3 runs x 4 updates
        eng.close()
    assert np.array_equal(outs[0], outs[1])
