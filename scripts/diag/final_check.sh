mkdir -p gpurun_out/f2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/f2/pytest_gpu.txt 2>&1; tail -2 gpurun_out/f2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2/smoke.txt 2>&1; tail -1 gpurun_out/f2/smoke.txt
for i in 1 2 3; do for v in 0 1; do
  P2BW_GEMM_HALF_N=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-same-config --no-graph > gpurun_out/f2/ab_${v}_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/f2/ab_${v}_$i.json'));print('half_n=$v', d['value'], d['clocks']['sm_mhz'])"
done; done
timeout 900 python bench.py > gpurun_out/f2/bench.json 2> gpurun_out/f2/bench.err; python -c "import json;d=json.load(open('gpurun_out/f2/bench.json'));print('default line', d['value'], d['e2e']['value'], d['mfu'], d['roofline']['frac'], d['clocks']['sm_mhz'], d.get('cuda_graph',{}).get('value'))"
