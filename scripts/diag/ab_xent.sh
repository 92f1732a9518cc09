# Softmax cross-entropy with two rows per SM (P2BW_XENT_2CTA): tests, in-step A/B with the kernel's own timing.
mkdir -p gpurun_out/xe
timeout 600 python -m pytest tests/test_transformer_kernels_gpu.py -q -m gpu -p no:cacheprovider -k xent > gpurun_out/xe/pytest.txt 2>&1; tail -1 gpurun_out/xe/pytest.txt
for i in 1 2 3; do for v in 0 1; do
  P2BW_XENT_2CTA=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-same-config --no-graph > gpurun_out/xe/bench_${v}_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/xe/bench_${v}_$i.json'));b=d['kernel_breakdown']['softmax_xent'];print('xent_2cta=$v', d['value'], d['clocks']['sm_mhz'], 'xent share', b['share'], 'GB/s', b['gbs'])"
done; done
