mkdir -p gpurun_out/r2f
for h in 768 1024 1920; do timeout 300 python scripts/mem_kernels_probe.py $h; done > gpurun_out/r2f/mem.jsonl 2> gpurun_out/r2f/mem.err; cat gpurun_out/r2f/mem.jsonl; tail -3 gpurun_out/r2f/mem.err
timeout 300 python scripts/attn_bench.py bert-base gpt-2.2b >> gpurun_out/r2f/attn.jsonl 2>&1; cat gpurun_out/r2f/attn.jsonl
