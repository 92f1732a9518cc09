set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_transformer_kernels_gpu.py -x -q -k attention 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 400 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -c 1500 gpurun_out/bench5.json; tail -5 gpurun_out/bench5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attn_bwd_tc --launch-skip 20 -c 1 \
  -f -o gpurun_out/attn_bwd_v3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn3.log 2>&1; tail -2 gpurun_out/ncu_attn3.log
timeout 900 python scripts/plan_b200.py gpurun_out/plan > gpurun_out/plan.log 2>&1; tail -3 gpurun_out/plan.log
