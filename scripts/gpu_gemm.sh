# GEMM tile validation + sweep (launched through gpurun)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
timeout 900 python scripts/gemm_sweep.py 8192 768 > gpurun_out/sweep_192.json 2>&1
timeout 600 python scripts/gemm_sweep.py 4096 1024 > gpurun_out/sweep_192_h1024.json 2>&1
