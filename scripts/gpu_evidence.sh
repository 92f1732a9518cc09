# Round-1 evidence (launched through gpurun): GPU tests, bench line, ncu launch list of the
# same bench command, ncu --set full of the top kernels.  Outputs in gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev/pytest_gpu.txt 2>&1; tail -2 gpurun_out/ev/pytest_gpu.txt
timeout 400 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; tail -c 400 gpurun_out/ev/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --launch-skip 2000 -c 1400 --csv --log-file gpurun_out/ev/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1; tail -1 gpurun_out/ev/ncu_launch.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel --launch-skip 300 -c 3 \
  -f -o gpurun_out/ev/gemm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_gemm.log 2>&1; tail -1 gpurun_out/ev/ncu_gemm.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_attn_bwd_tc|k_attn_fwd_tc" --launch-skip 20 -c 2 \
  -f -o gpurun_out/ev/attn_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_attn.log 2>&1; tail -1 gpurun_out/ev/ncu_attn.log
timeout 600 python scripts/plan_b200.py gpurun_out/ev/plan > gpurun_out/ev/plan.log 2>&1; tail -1 gpurun_out/ev/plan.log
