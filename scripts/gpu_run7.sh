set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_transformer_kernels_gpu.py tests/test_transformer_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -3 gpurun_out/bench8.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --launch-skip 2000 -c 1400 --csv --log-file gpurun_out/launches_r1d.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_d.log 2>&1; tail -1 gpurun_out/ncu_launch_d.log
