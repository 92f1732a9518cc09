# P2BW_GEMM_TILE sweep of scripts/gemm_bench.py (diagnostic): $1 = shape set ("" = BERT-base, T 16384; gpt-2.2b)
cd $GRAFT_REPO_ROOT
for t in auto 256,2 256,1 192,2 192,1; do
  if [ "$t" = auto ]; then unset P2BW_GEMM_TILE; else export P2BW_GEMM_TILE=$t; fi
  echo "== $t"
  timeout 200 python scripts/gemm_bench.py $1 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['name'], d['m'], d['n'], d['k'], d['tflops'])
"
done
