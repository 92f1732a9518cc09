mkdir -p gpurun_out/r2g
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_attn_fwd_tc|k_attn_bwd_tc" -s 4 -c 2 -f -o gpurun_out/r2g/attn_gpt python scripts/attn_bench.py gpt-2.2b > gpurun_out/r2g/ncu_gpt.log 2>&1; tail -2 gpurun_out/r2g/ncu_gpt.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ln_fwd|k_ln_bwd|k_colstats" -s 5 -c 3 -f -o gpurun_out/r2g/mem1920 python scripts/mem_kernels_probe.py 1920 > gpurun_out/r2g/ncu_mem.log 2>&1; tail -2 gpurun_out/r2g/ncu_mem.log
ls -la gpurun_out/r2g
