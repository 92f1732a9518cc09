# GEMM half-width last N tile (P2BW_GEMM_HALF_N): GEMM tests, stand-alone GPT-2.2B GEMMs, in-step A/B.
mkdir -p gpurun_out/hn
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/hn/pytest_gemm.txt 2>&1; tail -2 gpurun_out/hn/pytest_gemm.txt
for v in 0 1; do P2BW_GEMM_HALF_N=$v timeout 300 python scripts/gemm_bench.py gpt-2.2b > gpurun_out/hn/gemm_bench_$v.txt 2>&1; echo "half_n=$v"; tail -15 gpurun_out/hn/gemm_bench_$v.txt; done
for i in 1 2; do for v in 0 1; do
  P2BW_GEMM_HALF_N=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-same-config --no-graph > gpurun_out/hn/bench_${v}_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hn/bench_${v}_$i.json'));b=d['kernel_breakdown'];print('half_n=$v', d['value'], d['clocks']['sm_mhz'], 'fwd', b['gemm_fwd']['tflops'], 'dgrad', b['gemm_dgrad']['tflops'], 'wgrad', b['gemm_wgrad']['tflops'])"
done; done
timeout 900 python -m pytest tests/test_transformer_engine_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/hn/pytest_engine.txt 2>&1; tail -2 gpurun_out/hn/pytest_engine.txt
