mkdir -p gpurun_out/r2b
timeout 600 python scripts/diag/bf16_m3.py m3_d2 m5_d4 c1_d2 > gpurun_out/r2b/diag.txt 2>&1; tail -40 gpurun_out/r2b/diag.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r2b/pytest_gpu.txt 2>&1; tail -15 gpurun_out/r2b/pytest_gpu.txt
