mkdir -p gpurun_out/r2h
timeout 600 python -m pytest tests/test_transformer_kernels_gpu.py -q -x -p no:cacheprovider -k attention > gpurun_out/r2h/pytest_attn.txt 2>&1; tail -15 gpurun_out/r2h/pytest_attn.txt
timeout 300 python scripts/attn_bench.py > gpurun_out/r2h/attn.jsonl 2>&1; cat gpurun_out/r2h/attn.jsonl
