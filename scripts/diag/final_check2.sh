# Last validation of the round: GPU suite, smoke, default bench line, ncu launch list of one batch.
mkdir -p gpurun_out/f3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/f3/pytest_gpu.txt 2>&1; tail -2 gpurun_out/f3/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.txt 2>&1; tail -1 gpurun_out/f3/smoke.txt
timeout 900 python bench.py > gpurun_out/f3/bench.json 2> gpurun_out/f3/bench.err; python -c "import json;d=json.load(open('gpurun_out/f3/bench.json'));print('default line', d['value'], d['e2e']['value'], d['mfu'], d['roofline']['frac'], d['clocks'], d.get('cuda_graph',{}).get('value'))"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --launch-skip 700 -c 5100 --kill yes --csv --log-file gpurun_out/f3/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-same-config > gpurun_out/f3/ncu_launch.log 2>&1; tail -1 gpurun_out/f3/ncu_launch.log
timeout 600 python bench.py --impl reference > gpurun_out/f3/bench_reference.json 2>/dev/null; tail -c 200 gpurun_out/f3/bench_reference.json
