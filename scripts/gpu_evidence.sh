# Evidence for profiles/ (launched through gpurun): GPU tests, the default bench line
# (GPT-2.2B), the ncu launch list of the same bench command in steady state, ncu --set
# full of the top kernels, smoke().  Outputs in gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/ev/pytest_gpu.txt 2>&1; tail -3 gpurun_out/ev/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.txt 2>&1; tail -1 gpurun_out/ev/smoke.txt
timeout 900 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; tail -c 400 gpurun_out/ev/bench.json
# one batch of the bench's resident pass (~5000 launches after weight initialisation)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --launch-skip 700 -c 5100 --kill yes --csv --log-file gpurun_out/ev/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-same-config > gpurun_out/ev/ncu_launch.log 2>&1; tail -1 gpurun_out/ev/ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel --launch-skip 2000 -c 3 \
  -f -o gpurun_out/ev/gemm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-same-config > gpurun_out/ev/ncu_gemm.log 2>&1; tail -1 gpurun_out/ev/ncu_gemm.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attn_bwd_tc|k_attn_fwd_tc|k_ln_bwd|k_ln_fwd_wide" --launch-skip 200 -c 4 \
  -f -o gpurun_out/ev/other_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-same-config > gpurun_out/ev/ncu_other.log 2>&1; tail -1 gpurun_out/ev/ncu_other.log
# the other configurations' bench lines
for c in bert-base bert-large gpt-24 small gpt-2.2b-h128; do
  timeout 600 python bench.py --config $c > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err; tail -c 200 gpurun_out/ev/bench_$c.json
done
# the reference arm and the multi-rank plumbing (4 ranks sharing the one GPU: not a scaling number)
timeout 600 python bench.py --impl reference > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err; tail -c 300 gpurun_out/ev/bench_reference.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 4 --config bert-base --steps 5 --warmup 3 > gpurun_out/ev/bench_bert-base_4ranks_shared.json 2> gpurun_out/ev/bench_4ranks.err; tail -c 300 gpurun_out/ev/bench_bert-base_4ranks_shared.json
