set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
SWEEP_CFGS="auto 256,2 192,1" timeout 900 python scripts/gemm_sweep.py 8192 768 > gpurun_out/sweep_model.json 2>&1
SWEEP_CFGS="auto 256,2 192,1" timeout 900 python scripts/gemm_sweep.py 4096 1024 > gpurun_out/sweep_model_h1024.json 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -c 300 gpurun_out/bench7.json; tail -3 gpurun_out/bench7.err
