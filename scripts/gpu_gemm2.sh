set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -5
SWEEP_CFGS="auto 256,2 256,4 192,1 192,4 128,4" timeout 900 python scripts/gemm_sweep.py 8192 768 > gpurun_out/sweep_c4.json 2>&1
SWEEP_CFGS="auto 256,2 256,4 192,4 128,4" timeout 600 python scripts/gemm_sweep.py 4096 1024 > gpurun_out/sweep_c4_h1024.json 2>&1
timeout 300 python -m pytest tests/test_transformer_kernels_gpu.py -x -q -k attention 2>&1 | tail -3
python scripts/attn_bwd_timing.py 0 2>&1 | head -3
