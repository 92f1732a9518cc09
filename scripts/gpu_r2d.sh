mkdir -p gpurun_out/r2d
timeout 300 python scripts/diag/bf16_env.py c1_d2 m3_d2 m5_d4 > gpurun_out/r2d/env.txt 2>&1; cat gpurun_out/r2d/env.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r2d/pytest_gpu.txt 2>&1; tail -15 gpurun_out/r2d/pytest_gpu.txt
