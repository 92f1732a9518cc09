"""Depth-d 2BW pipelines of a B200-profiled model, replayed with the reference
simulator's rules (scripts/c5_replay.py, pinned to the reference's simulate_policy by
tests/test_c5_replay.py): equal vs balanced stage splits, and the steady batch time split
into ideal / imbalance / schedule bubble / exposed NVLink transfer (the north star's
"pipeline bubble plus exposed NVLink transfer under 10% of step time at depth 8").

  python scripts/pipeline_replay.py profiles/r1_profile_gpt2.2b_b200.json 16 [out.json]
"""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import c5_replay as R  # noqa: E402
from paper_2006_09503_b200 import pipesim as P  # noqa: E402


def main():
    prof = open(sys.argv[1]).read()
    b = int(sys.argv[2])
    rows = []
    for d in (2, 4, 8):
        bal = P.partition_balanced(prof, d, b)
        for m in (d, 2 * d, 4 * d):
            for name, bounds in (("equal", None), ("balanced", bal)):
                bd = R.breakdown(prof, P.PipelinePolicy.TwoBW, d, m, b=b, bounds=bounds)
                st = bd["steady_batch_ms"]
                row = {"partition": name, "stage_layers": None if bounds is None else P.stage_layers_from_bounds(bounds),
                       "d": d, "m": m, "b": b, "samples_per_s": round(bd["throughput"], 1),
                       "steady_batch_ms": round(st, 3),
                       "frac_imbalance": round(bd["imbalance_ms"] / st, 4),
                       "frac_schedule_bubble": round(bd["schedule_bubble_ms"] / st, 4),
                       "frac_exposed_transfer": round(bd["exposed_transfer_ms"] / st, 4),
                       "bubble_plus_exposed": round((bd["schedule_bubble_ms"] + bd["exposed_transfer_ms"]) / st, 4),
                       "not_ideal": round(1.0 - bd["ideal_ms"] / st, 4)}
                rows.append(row)
                print(json.dumps(row))
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as f:
            json.dump({"profile": sys.argv[1], "b": b, "policy": "2bw", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
