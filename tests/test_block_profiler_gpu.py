"""B200 block profiler -> the reference's profile document -> plan().

The profile is produced by timing the stage executor's own Forward / Backward
kernels (p2bw_profile_blocks) and must load through the reference's profile reader
(load_model_profile, profile.cpp:162-193) as used by partition_equal and plan()."""
import json

import pytest

from paper_2006_09503_b200 import pipesim as P

pytestmark = pytest.mark.gpu

CLUSTER_8xB200 = json.dumps({"total_workers": 8, "gpus_per_server": 8, "bandwidth_high_gbps": 900.0,
                             "bandwidth_low_gbps": 50.0, "memory_capacity_gb": 180.0})


@pytest.fixture(scope="module")
def profile():
    return P.profile_blocks(layers=4, hidden=256, heads=4, seq_len=128, vocab=1000, causal=1,
                            microbatch_sizes=(1, 2, 4), warmup=1, iters=3, name="small-gpt")


def test_profile_document_shape(profile):
    doc = json.loads(profile)
    assert doc["model"] == "small-gpt"
    blocks = doc["blocks"]
    assert len(blocks) == 4
    for blk in blocks:
        for key in ("fwd_ms", "bwd_ms", "act_total_bytes", "act_input_bytes", "act_boundary_bytes"):
            assert sorted(blk[key], key=int) == ["1", "2", "4"]
        assert all(v > 0 for v in blk["fwd_ms"].values()) and all(v > 0 for v in blk["bwd_ms"].values())
        assert blk["act_input_bytes"]["2"] == 2 * blk["act_input_bytes"]["1"]
    # interior blocks are the same measurement; the ends carry embedding / LM head
    assert blocks[1]["fwd_ms"] == blocks[2]["fwd_ms"]
    assert blocks[0]["weight_bytes"] > blocks[1]["weight_bytes"] < blocks[3]["weight_bytes"]


def test_profile_feeds_partition_and_plan(profile):
    stages = P.partition_equal(profile, 2)
    assert len(stages) == 2
    result = P.plan(profile, CLUSTER_8xB200, 64, P.PipelinePolicy.TwoBW)
    cfg = result["best"]
    assert cfg["width"] * cfg["depth"] <= 8
    assert cfg["microbatch_size"] in (1, 2, 4)
    assert result["predicted_throughput"] > 0
    assert result["ranked"] and all(r["feasible"] for r in result["ranked"])


def test_profile_rejects_bad_sizes():
    with pytest.raises(Exception, match="microbatch sizes"):
        P.profile_blocks(layers=2, hidden=128, heads=2, seq_len=128, vocab=100, microbatch_sizes=(0,))
