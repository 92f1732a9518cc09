"""libp2bw.so host path (schedule, planner, partition) through the C-ABI,
checked bit-exactly against the reference's golden vectors and the oracle.
No GPU needed: these entry points are host C++ (the reference's own behaviour,
schedule.cpp / planner.cpp / profile.cpp)."""
import ctypes as C
import hashlib
import json
import re
import subprocess
from pathlib import Path

import pytest

from oracle import pipesim_oracle as O
from paper_2006_09503_b200 import _lib
from paper_2006_09503_b200 import pipesim as P
from tests import _golden as G

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "p2bw.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+char\s*\*|int|void|long\s+long)\s+(p2bw_\w+)\s*\(", header,
                              re.M))
    assert declared, "no declarations parsed"
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines()}
    assert declared <= exported, sorted(declared - exported)
    assert set(_lib.declared_symbols()) == declared  # the ctypes table covers the header exactly
    lib = _lib.lib()
    for name in declared:
        getattr(lib, name)


def test_version_formula_and_errors():
    for key, v in G.schedules()["versions"].items():
        k, m = map(int, key.split("/"))
        assert P.weight_version_2bw(k, m) == v
    with pytest.raises(P.PipesimError, match="microbatch index must be >= 1"):
        P.weight_version_2bw(0, 4)
    with pytest.raises(P.PipesimError, match="m >= d"):
        P.generate_schedule(P.PipelinePolicy.TwoBW, 4, 2, 1)
    assert P.required_versions(P.PipelinePolicy.TwoBW, 8, 8) == 2
    assert P.required_versions(P.PipelinePolicy.PipeDream1F1B, 4, 1) == 4


def test_schedules_bit_identical_to_reference():
    g = G.schedules()
    for key, text in g["schedules"].items():
        p, d, m, T = map(int, key.split("/"))
        if text.startswith("ERROR"):
            with pytest.raises(P.PipesimError):
                P.schedule_text(p, d, m, T)
            continue
        assert P.schedule_text(p, d, m, T) == text, key
    for key, digest in g["sweep_sha256"].items():
        p, d, m, T = map(int, key.split("/"))
        assert hashlib.sha256(P.schedule_text(p, d, m, T).encode()).hexdigest() == digest, key


def test_program_round_trip_and_parse_errors():
    text = P.schedule_text(P.PipelinePolicy.TwoBW, 4, 8, 2)
    progs = P.parse_programs(text)
    assert P.serialize_programs(progs) == text
    assert progs == P.generate_schedule(P.PipelinePolicy.TwoBW, 4, 8, 2)
    with pytest.raises(P.PipesimError, match="teleport"):
        P.parse_programs("stage=0 op=teleport")
    with pytest.raises(P.PipesimError, match="missing stage"):
        P.parse_programs("op=forward mb=1 ver=0")
    for pol in P.PipelinePolicy:
        assert P.parse_policy(P.to_string(pol)) == pol
    with pytest.raises(P.PipesimError, match="bogus"):
        P.parse_policy("bogus")


def test_plans_bit_identical_to_reference():
    g = G.plans()
    for key, ref in g["plans"].items():
        mname, cname, B = key.split("/")
        got = P.plan(g["models"][mname], json.dumps(g["clusters"][cname]), int(B))
        assert got == ref, key  # every field, parsed values


def test_plan_errors_keep_reference_wording():
    fat = O.uniform_profile_json("fat", 4, 1e-3, 2e-3, 1e8, 3e9, 1e9, [1])
    tiny = json.dumps(dict(total_workers=4, gpus_per_server=4, bandwidth_high_gbps=1000,
                           bandwidth_low_gbps=100, memory_capacity_gb=1e-3))
    with pytest.raises(P.PipesimError, match="no feasible"):
        P.plan(fat, tiny, 64)
    with pytest.raises(P.PipesimError, match="max safe batch size"):
        P.plan(fat, tiny, 0)
    assert "best configuration: w=" in P.plan_text(
        fat, json.dumps(dict(total_workers=4, gpus_per_server=4, bandwidth_high_gbps=1000,
                             bandwidth_low_gbps=100, memory_capacity_gb=8)), 64)


def test_partition_equal_matches_oracle_exactly():
    mj = G.plans()["models"]["gpt_like48"]
    blocks = O.load_model_profile(mj)
    for d in (1, 2, 3, 4, 6, 8, 12, 16, 24, 48):
        got = P.partition_equal(mj, d)
        ref = O.partition_equal(blocks, d)
        assert len(got) == d
        for g, r in zip(got, ref):
            assert {int(k): v for k, v in g["fwd_time"].items()} == r.fwd
            assert {int(k): v for k, v in g["bwd_time"].items()} == r.bwd
            assert g["weight_bytes"] == r.weight_bytes
            assert {int(k): v for k, v in g["act_output_bytes"].items()} == r.act_output
    with pytest.raises(P.PipesimError, match="does not divide"):
        P.partition_equal(mj, 5)


def _profile_doc(times, b=4):
    import json as _json
    return _json.dumps({"model": "t", "blocks": [
        {"fwd_ms": {str(b): t}, "bwd_ms": {str(b): 2 * t}, "weight_bytes": 1, "act_total_bytes": {str(b): 1},
         "act_input_bytes": {str(b): 1}, "act_boundary_bytes": {str(b): 1}} for t in times]})


def _brute_best(times, d):
    import itertools
    n = len(times)
    best = None
    for cuts in itertools.combinations(range(1, n), d - 1):
        b = [0, *cuts, n]
        worst = max(sum(times[lo:hi]) for lo, hi in zip(b[:-1], b[1:]))
        best = worst if best is None else min(best, worst)
    return best


@pytest.mark.parametrize("times,d", [([1.0] * 8, 4), ([1.0] * 7 + [2.5], 4), ([1.3] + [1.0] * 22 + [2.5], 8),
                                     ([0.5, 3.0, 1.0, 1.0, 0.2, 2.0, 1.0], 3), ([1.0] * 5, 5)])
def test_partition_balanced_is_optimal(times, d):
    """B200 extension beside partition_equal (profile.cpp:104-131): the split minimises the
    slowest stage (checked by brute force), and uniform blocks give the equal split."""
    bounds = P.partition_balanced(_profile_doc(times), d, 4)
    assert bounds[0] == 0 and bounds[-1] == len(times) and len(bounds) == d + 1
    assert all(hi > lo for lo, hi in zip(bounds[:-1], bounds[1:]))
    worst = max(3 * sum(times[lo:hi]) for lo, hi in zip(bounds[:-1], bounds[1:]))
    assert abs(worst - 3 * _brute_best(times, d)) < 1e-9
    if len(set(times)) == 1 and len(times) % d == 0:
        assert bounds == [i * len(times) // d for i in range(d + 1)]
    with pytest.raises(Exception, match="exceeds block count"):
        P.partition_balanced(_profile_doc(times), len(times) + 1, 4)


def test_bench_flop_profile_balances_the_lm_head():
    """bench.py's pipeline leg: the GPT-2.2B blocks costed by algorithmic FLOPs put the
    51200-way LM head (~2 layers) on the last block, so the balanced split at depth 8 gives
    the last stage fewer layers and a slowest stage below the equal split's."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", Path(__file__).resolve().parents[1] / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    c = bench.CONFIGS["gpt-2.2b"]
    doc = bench.flop_profile(c)
    bounds = P.partition_balanced(doc, 8, c["b"])
    layers = P.stage_layers_from_bounds(bounds)
    assert sum(layers) == 48 and layers[-1] < 6
    t = [b["fwd_ms"][str(c["b"])] + b["bwd_ms"][str(c["b"])] for b in json.loads(doc)["blocks"]]
    worst = max(sum(t[lo:hi]) for lo, hi in zip(bounds[:-1], bounds[1:]))
    assert worst < sum(t[42:48]) * 0.9
