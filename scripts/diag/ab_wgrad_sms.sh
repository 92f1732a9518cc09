# In-step A/B: weight-gradient GEMMs held to fewer SMs (P2BW_GEMM_WGRAD_SMS), alternating runs.
mkdir -p gpurun_out/ws
for i in 1 2; do for v in 0 120 96 74; do
  P2BW_GEMM_WGRAD_SMS=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-same-config --no-graph > gpurun_out/ws/bench_${v}_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ws/bench_${v}_$i.json'));print('wgrad_sms=$v', d['value'], d['clocks']['sm_mhz'])"
done; done
