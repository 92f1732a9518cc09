# In-step A/B of the double-buffered attention dQ accumulator (P2BW_ATTN_DQ_DBUF), alternating runs.
mkdir -p gpurun_out/dq
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "engine or attention or transformer" > gpurun_out/dq/pytest.txt 2>&1; tail -2 gpurun_out/dq/pytest.txt
P2BW_ATTN_DQ_DBUF=0 timeout 900 python -m pytest tests/test_transformer_engine_gpu.py -q -m gpu -p no:cacheprovider -k "bench_width or head_dim" > gpurun_out/dq/pytest_off.txt 2>&1; tail -1 gpurun_out/dq/pytest_off.txt
for i in 1 2; do for v in 0 1; do
  P2BW_ATTN_DQ_DBUF=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-same-config --no-graph > gpurun_out/dq/bench_${v}_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/dq/bench_${v}_$i.json'));b=d['kernel_breakdown'];print('dbuf=$v', d['value'], d['clocks']['sm_mhz'], 'attn_bwd', b['attention_bwd'])"
done; done
