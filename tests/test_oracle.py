"""Pins the CPU oracle (oracle/pipesim_oracle.py) to the reference: golden
vectors produced by the reference itself (tests/golden/) and, where the
reference has been compiled here (oracle/_ref/ref_tool), live comparisons.
Reference known-answer tests restated: schedule_test.cpp:31-76,
planner_test.cpp:10-29, semantics_test.cpp:199-231."""
import hashlib
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import pipesim_oracle as O
from tests import _golden as G

TOOL = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "ref_tool"


def test_version_formula_known_answers():
    # schedule_test.cpp:31-40
    assert [O.weight_version_2bw(k, 4) for k in (9, 1, 8, 13, 4, 5)] == [1, 0, 0, 2, 0, 0]
    for bad in ((0, 4), (1, 0)):
        with pytest.raises(O.OracleError):
            O.weight_version_2bw(*bad)
    for key, v in G.schedules()["versions"].items():
        k, m = map(int, key.split("/"))
        assert O.weight_version_2bw(k, m) == v


def _trace(ops):
    sym = {O.FORWARD: "F", O.BACKWARD: "B"}
    out = []
    for kind, mb, _ in ops:
        out.append(f"{sym[kind]}{mb}" if kind in sym else {O.FLUSHB: "|", O.ALLREDUCE: "AR", O.UPDATE: "U"}[kind])
    return " ".join(out)


def test_golden_program_shapes():
    # schedule_test.cpp:50-76
    p = O.generate_schedule(O.GPIPE, 2, 4, 1)
    assert _trace(p[0]) == _trace(p[1]) == "F1 F2 F3 F4 B1 B2 B3 B4 | AR U"
    p = O.generate_schedule(O.FLUSH, 2, 4, 1)
    assert _trace(p[0]) == "F1 F2 B1 F3 B2 F4 B3 B4 | AR U"
    assert _trace(p[1]) == "F1 B1 F2 B2 F3 B3 F4 B4 | AR U"
    p = O.generate_schedule(O.TWOBW, 1, 1, 3)
    assert _trace(p[0]) == "F1 B1 AR U F2 B2 AR U F3 B3 AR U"
    assert [v for k, _, v in p[0] if k == O.FORWARD] == [0, 0, 1]
    assert _trace(O.generate_schedule(O.NONE, 2, 2, 1)[0]) == "F1 B1 F2 B2 AR U"
    with pytest.raises(O.OracleError, match="m >= d"):
        O.generate_schedule(O.TWOBW, 4, 2, 1)


def test_schedules_match_reference_golden_text():
    g = G.schedules()
    for key, text in g["schedules"].items():
        p, d, m, T = map(int, key.split("/"))
        if text.startswith("ERROR"):
            with pytest.raises(O.OracleError):
                O.generate_schedule(p, d, m, T)
            continue
        assert O.serialize_programs(O.generate_schedule(p, d, m, T)) == text, key
    for key, digest in g["sweep_sha256"].items():
        p, d, m, T = map(int, key.split("/"))
        text = O.serialize_programs(O.generate_schedule(p, d, m, T))
        assert hashlib.sha256(text.encode()).hexdigest() == digest, key


def test_plans_match_reference_golden():
    g = G.plans()
    for key, ref in g["plans"].items():
        mname, cname, B = key.split("/")
        blocks = O.load_model_profile(g["models"][mname])
        cluster = O.load_cluster_spec(json.dumps(g["clusters"][cname]))
        got = O.plan(blocks, cluster, int(B))
        assert got["best"] == ref["best"], key
        assert got["predicted_throughput"] == ref["predicted_throughput"], key  # bit-exact
        assert got["predicted_memory_bytes"] == ref["predicted_memory_bytes"], key
        assert got["pairs_examined"] == ref["pairs_examined"], key
        assert got["grad_accum_for_cluster"] == ref["grad_accum_for_cluster"], key
        assert [(r["width"], r["depth"], r["microbatch_size"], r["recompute"], r["throughput"])
                for r in got["ranked"]] == \
               [(r["width"], r["depth"], r["microbatch_size"], r["recompute"], r["throughput"])
                for r in ref["ranked"]], key


def test_planner_known_answers():
    # planner_test.cpp:10-29
    mj = O.uniform_profile_json("u4", 4, 1e-3, 2e-3, 1e8, 1e6, 2.5e5, [1, 2, 4])
    one = O.Cluster(1, 1, 1e12, 1e11, 32e9)
    r = O.plan(O.load_model_profile(mj), one, 64)
    assert (r["best"]["width"], r["best"]["depth"], r["pairs_examined"]) == (1, 1, 1)
    m8 = O.load_model_profile(O.uniform_profile_json("u8", 8, 1e-3, 2e-3, 1e8, 1e6, 2.5e5, [1, 2, 4]))
    r = O.plan(m8, O.Cluster(8, 8, 1e12, 1e11, 32e9), 128)
    assert r["pairs_examined"] == sum(8 // w for w in range(1, 9))


def test_toy_trajectories_bit_identical_to_reference():
    for meta, ref in G.toy():
        model = O.ToyModel.make(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"])
        traj, consistent, maxv = O.pipelined_execute(model, meta["lr"], meta["beta"], meta["m"], meta["T"],
                                                     meta["policy"], meta["depth"])
        got = O.flat_trajectory(traj)
        assert got.shape == ref.shape
        assert O.max_rel_diff(got, ref) == 0.0, meta
        assert maxv == meta["max_versions_held"], meta


def test_2bw_equals_delayed_loop_and_differs_from_vanilla():
    # semantics_test.cpp:199-231 (1e-10 there; bit-exact here for power-of-two m)
    model = O.ToyModel.make(4, 2, 2, 4 * 10, 12345)
    traj, _, maxv = O.pipelined_execute(model, 0.05, 0.9, 4, 10, O.TWOBW, 2)
    delayed, _ = O.reference_loop(model, 0.05, 0.9, 4, 10, True)
    vanilla, _ = O.reference_loop(model, 0.05, 0.9, 4, 10, False)
    assert O.max_rel_diff(O.flat_trajectory(traj), O.flat_trajectory(delayed)) < 1e-10
    assert O.max_rel_diff(O.flat_trajectory(traj), O.flat_trajectory(vanilla)) > 1e-6
    assert maxv == 2


@pytest.mark.skipif(not TOOL.exists(), reason="reference not compiled here (oracle/_ref/ref_tool)")
@pytest.mark.parametrize("policy,d,m,T", [(4, 3, 7, 3), (3, 5, 6, 2), (2, 4, 4, 2), (1, 6, 6, 1)])
def test_oracle_matches_live_reference_schedules(policy, d, m, T):
    ref = subprocess.run([str(TOOL), "schedule", str(policy), str(d), str(m), str(T)],
                         capture_output=True, text=True).stdout
    assert O.serialize_programs(O.generate_schedule(policy, d, m, T)) == ref


@pytest.mark.skipif(not TOOL.exists(), reason="reference not compiled here (oracle/_ref/ref_tool)")
def test_oracle_matches_live_reference_toy(tmp_path):
    dim, L, b, seed, lr, beta, m, T, pol, d = 6, 6, 3, 31337, 0.03, 0.5, 6, 4, 4, 3
    out = tmp_path / "t.bin"
    subprocess.run([str(TOOL), "toy", *map(str, (dim, L, b, seed, lr, beta, m, T, pol, d)), str(out)],
                   check=True, capture_output=True)
    ref = np.fromfile(out, dtype=np.float64).reshape(T + 1, L, dim * dim)
    model = O.ToyModel.make(dim, L, b, m * T, seed)
    traj, _, _ = O.pipelined_execute(model, lr, beta, m, T, pol, d)
    assert O.max_rel_diff(O.flat_trajectory(traj), ref) == 0.0


@pytest.mark.parametrize("idx", range(8))
def test_oracle_reference_loop_bit_identical_at_any_m(idx):
    """reference_loop (semantics.cpp:167-184) restated: bit-identical to the reference at
    m = 3..6.  pipelined_execute sums the microbatch gradients and divides by the count at
    the update (:338-340) while reference_loop scales each by 1/m (:145): the two agree to
    the last bit only for power-of-two m, and otherwise within a few ulps."""
    meta, ref = G.loops()[idx]
    model = O.ToyModel.make(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"])
    traj, _ = O.reference_loop(model, meta["lr"], meta["beta"], meta["m"], meta["T"], bool(meta["delayed"]))
    assert O.max_rel_diff(O.flat_trajectory(traj), ref) == 0.0
    pol = O.TWOBW if meta["delayed"] else O.GPIPE
    piped, _, _ = O.pipelined_execute(model, meta["lr"], meta["beta"], meta["m"], meta["T"], pol, 1)
    gap = O.max_rel_diff(O.flat_trajectory(piped), ref)
    if meta["m"] & (meta["m"] - 1) == 0:
        assert gap == 0.0
    else:
        assert 0.0 < gap < 1e-12, gap


def test_package_splitmix64_matches_reference_toy_model():
    """paper_2006_09503_b200.synthetic.toy_model is ToyModel::make bit for bit (the
    oracle's scalar splitmix64 restatement, itself pinned by the trajectories above)."""
    from paper_2006_09503_b200 import synthetic as S
    for dim, L, b, nmb, seed in ((4, 2, 2, 3, 12345), (16, 3, 8, 2, 7), (32, 1, 5, 4, 2 ** 63 + 5)):
        m = O.ToyModel.make(dim, L, b, nmb, seed)
        ws, data = S.toy_model(dim, L, b, nmb, seed)
        assert all(np.array_equal(a, c) for a, c in zip(m.weights, ws))
        assert all(np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1]) for a, c in zip(m.dataset, data))
