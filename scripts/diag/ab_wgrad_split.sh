# In-step A/B of the weight-gradient split-K cap (P2BW_GEMM_MAX_SPLIT), alternating runs on one box.
mkdir -p gpurun_out/sp
for cap in "" 1 2; do P2BW_GEMM_MAX_SPLIT=$cap python - <<'PY'
import ctypes as C, os
lib = C.CDLL('paper_2006_09503_b200/libp2bw.so'); out = (C.c_int * 4)()
h = 1920
for name, m, n in [('fc1', 4 * h, h), ('fc2', h, 4 * h), ('qkv', 3 * h, h), ('proj', h, h)]:
    lib.p2bw_debug_gemm_plan(m, n, 8192, 1, 1, 1, 0, out)
    print('cap', os.environ.get('P2BW_GEMM_MAX_SPLIT'), name, 'wgrad plan {BN, cl, splits, tail}', list(out))
PY
done
for i in 1 2; do for cap in "" 1 2; do
  P2BW_GEMM_MAX_SPLIT=$cap timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-same-config --no-graph > gpurun_out/sp/bench_${cap:-d}_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sp/bench_${cap:-d}_$i.json'));b=d['kernel_breakdown'];print('cap=${cap:-default}', d['value'], d['clocks']['sm_mhz'], 'wgrad', b['gemm_wgrad'])"
done; done
