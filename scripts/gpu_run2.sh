# Round-1 evidence run (launched through gpurun): tests, bench, launch list, ncu captures, GEMM sweep.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 400 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; cat gpurun_out/bench3.json | head -c 1500
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --launch-skip 2000 -c 1800 --csv --log-file gpurun_out/launches_r1c.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel --launch-skip 300 -c 1 \
  -f -o gpurun_out/gemm_full_r1c python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attn_bwd_tc --launch-skip 20 -c 1 \
  -f -o gpurun_out/attn_bwd_full_r1c python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
timeout 600 python scripts/gemm_sweep.py 8192 768 > gpurun_out/sweep3.json 2>&1
