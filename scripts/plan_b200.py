"""Config 4 planner loop on B200: profile the GPT-style 2.2B
decoder's blocks with the stage executor's kernels on this GPU, then run the
reference planner (plan(), planner.cpp:45-99) for an 8 x B200 NVSwitch server.

    python scripts/plan_b200.py [out_dir]     (needs a GPU)

Writes <out>/profile_gpt2.2b_b200.json (the reference profile document) and
<out>/plan_gpt2.2b_8xb200.json / .txt (plan_to_json / plan_to_text)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_09503_b200 import pipesim as P  # noqa: E402

out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
out.mkdir(parents=True, exist_ok=True)
# BASELINE configs[3]: GPT-style 2.2B decoder (h 1920 = 30 heads of 64, 48 layers, seq 512, V 51200)
t0 = time.time()
prof = P.profile_blocks(layers=48, hidden=1920, heads=30, seq_len=512, vocab=51200, causal=1,
                        microbatch_sizes=(1, 2, 4, 8, 16), warmup=2, iters=5, name="gpt-2.2b")
t1 = time.time()
cluster = json.dumps({"total_workers": 8, "gpus_per_server": 8, "bandwidth_high_gbps": 900.0,
                      "bandwidth_low_gbps": 50.0, "memory_capacity_gb": 180.0})
(out / "profile_gpt2.2b_b200.json").write_text(prof)
for pol in (P.PipelinePolicy.TwoBW, P.PipelinePolicy.PipeDreamFlush):
    tag = P.to_string(pol)
    (out / f"plan_gpt2.2b_8xb200_{tag}.json").write_text(json.dumps(P.plan(prof, cluster, 512, pol), indent=1))
    (out / f"plan_gpt2.2b_8xb200_{tag}.txt").write_text(P.plan_text(prof, cluster, 512, pol))
print(json.dumps({"profile_s": round(t1 - t0, 1), "plan_2bw": P.plan(prof, cluster, 512)["best"]}))

# validate_plan-style closure (planner.cpp:101-120) on what one GPU can measure:
# BERT-base blocks profiled here, planned for a 1-GPU "cluster", against the measured
# bench throughput of the same configuration.
prof_b = P.profile_blocks(layers=12, hidden=768, heads=12, seq_len=512, vocab=30522, causal=0, head_rows=77,
                          microbatch_sizes=(4, 8, 16), warmup=2, iters=5, name="bert-base")
one = json.dumps({"total_workers": 1, "gpus_per_server": 1, "bandwidth_high_gbps": 900.0,
                  "bandwidth_low_gbps": 50.0, "memory_capacity_gb": 180.0})
plan1 = P.plan(prof_b, one, 64)
(out / "profile_bert-base_b200.json").write_text(prof_b)
(out / "plan_bert-base_1xb200.json").write_text(json.dumps(plan1, indent=1))
print(json.dumps({"bert_base_1gpu_predicted_samples_per_s": plan1["predicted_throughput"],
                  "bert_base_1gpu_best": plan1["best"]}))
