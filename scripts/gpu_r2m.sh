T='tests/test_transformer_engine_gpu.py::test_bench_width_layers_match_delayed_oracle'
for env in "X=1" "P2BW_PDL=0" "P2BW_SERIAL_STAGE=1" "CUDA_LAUNCH_BLOCKING=1"; do
  echo "== $env"; env $env timeout 300 python -m pytest "$T" -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|max loss" | head -5
done
