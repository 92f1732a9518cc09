set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
P2BW_GEMM_TILE=256,2 timeout 150 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -15
P2BW_GEMM_TILE=128,2 timeout 150 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -8
timeout 400 python scripts/gemm_sweep.py 8192 768 > gpurun_out/sweep2.json 2>&1
cat gpurun_out/sweep2.json
