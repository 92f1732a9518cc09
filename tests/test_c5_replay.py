"""scripts/c5_replay.py restates the simulator's dependency rules (simulator.cpp:195-290);
on uniform stages with free transfers its bubble must be the closed form
(d - 1) / (m + d - 1) for GPipe / Flush and 0 for 2BW's steady state."""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "scripts"))
sys.path.insert(0, str(ROOT))

import c5_replay as R  # noqa: E402
from paper_2006_09503_b200 import pipesim as P  # noqa: E402


def _uniform(n):
    blk = {"fwd_ms": {"4": 1.0}, "bwd_ms": {"4": 2.0}, "weight_bytes": 1e6, "act_total_bytes": {"4": 1e6},
           "act_input_bytes": {"4": 0.0}, "act_boundary_bytes": {"4": 0.0}}
    return json.dumps({"model": "uniform", "blocks": [blk] * n})


@pytest.mark.parametrize("d,m", [(2, 4), (4, 4), (4, 8), (8, 16)])
def test_replay_matches_closed_form(d, m):
    stages = P.partition_equal(_uniform(8), d)
    fb = (1.0 + 2.0) * (8 // d) * 1e-3  # seconds per microbatch per stage
    for pol in (P.PipelinePolicy.GPipe, P.PipelinePolicy.PipeDreamFlush):
        r = R.replay(P.generate_schedule(pol, d, m, R.T_BATCHES), stages, pol, 4, 1e30)
        assert r["bubble_fraction"] == pytest.approx((d - 1) / (m + d - 1), abs=1e-9)
        assert r["steady_batch_ms"] == pytest.approx((m + d - 1) * fb * 1e3, rel=1e-9)
    r = R.replay(P.generate_schedule(P.PipelinePolicy.TwoBW, d, m, R.T_BATCHES), stages, P.PipelinePolicy.TwoBW,
                 4, 1e30)
    assert r["bubble_fraction"] == pytest.approx(0.0, abs=1e-9)
    assert r["throughput"] == pytest.approx(4 / fb, rel=1e-9)


def _c5_rows():
    gold = json.loads((ROOT / "tests" / "golden" / "c5_simulate.json").read_text())
    prof = (ROOT / "tests" / "golden" / gold["profile"]).read_text()
    return prof, gold["num_batches"], gold["rows"]


def test_replay_equals_reference_simulate_on_b200_profile():
    """The config-5 replay against the reference's own simulate_policy (golden rows from
    oracle/_ref/ref_tool simulate, simulator.cpp:140-339) on the B200-measured GPT-24
    profile: every policy, d 2/4/8, m 4-32, NVLink-priced and free transfers."""
    prof, T, rows = _c5_rows()
    assert T == R.T_BATCHES
    for row in rows:
        stages = P.partition_equal(prof, row["d"])
        pol = P.PipelinePolicy(row["policy"])
        bps = R.NVLINK_BPS if row["link"] == "nvlink" else 1e18
        r = R.replay(P.generate_schedule(pol, row["d"], row["m"], T), stages, pol, row["b"], bps)
        assert r["throughput"] == pytest.approx(row["throughput"], rel=1e-9), row
        assert r["steady_batch_ms"] == pytest.approx(row["steady_batch_time"] * 1e3, rel=1e-9), row
        assert r["bubble_fraction"] == pytest.approx(row["bubble_fraction"], rel=1e-9, abs=1e-12), row


def test_breakdown_columns_sum_to_the_step():
    """schedule bubble + stage imbalance + exposed transfer explain the simulated step:
    steady = m * mean(F + B) * (1 + imbalance loss) ... decomposed additively in time."""
    prof, T, rows = _c5_rows()
    for row in [r for r in rows if r["link"] == "nvlink"]:
        b = R.breakdown(prof, P.PipelinePolicy(row["policy"]), row["d"], row["m"], row["b"], T)
        parts = b["ideal_ms"] + b["imbalance_ms"] + b["schedule_bubble_ms"] + b["exposed_transfer_ms"]
        assert parts == pytest.approx(b["steady_batch_ms"], rel=1e-9)
        assert b["exposed_transfer_ms"] >= -1e-9 and b["imbalance_ms"] >= -1e-9
