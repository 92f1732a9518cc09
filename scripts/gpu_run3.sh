# attention-bwd rewrite + profiler + trace validation, bench, attention ncu
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_transformer_kernels_gpu.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 400 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -c 3000 gpurun_out/bench4.json; tail -5 gpurun_out/bench4.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attn_bwd_tc --launch-skip 20 -c 1 \
  -f -o gpurun_out/attn_bwd_v2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn2.log 2>&1; tail -2 gpurun_out/ncu_attn2.log
timeout 600 python scripts/plan_b200.py gpurun_out/plan > gpurun_out/plan.log 2>&1; tail -3 gpurun_out/plan.log
