mkdir -p gpurun_out/r2c
for env in "X=1" "P2BW_PDL=0" "P2BW_SERIAL_STAGE=1" "CUDA_LAUNCH_BLOCKING=1"; do
  echo "== $env"; env $env timeout 300 python scripts/diag/bf16_env.py c1_d2 m3_d2 2>&1 | tail -8
done > gpurun_out/r2c/env.txt 2>&1
cat gpurun_out/r2c/env.txt
