mkdir -p gpurun_out/r2e
timeout 600 python scripts/attn_bench.py > gpurun_out/r2e/attn.jsonl 2> gpurun_out/r2e/attn.err; cat gpurun_out/r2e/attn.jsonl; tail -3 gpurun_out/r2e/attn.err
timeout 600 python scripts/gemm_bench.py gpt-2.2b > gpurun_out/r2e/gemm.jsonl 2> gpurun_out/r2e/gemm.err; cat gpurun_out/r2e/gemm.jsonl; tail -3 gpurun_out/r2e/gemm.err
