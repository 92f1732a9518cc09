# Marginal cost of each kernel class inside the overlapped step: bench.py with one class
# issued twice (P2BW_DEBUG_DUP bit), 2 reps each.
one() { P2BW_DEBUG_DUP="$1" timeout 400 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for b in 0 1 2 4 8 16 32; do one $b; done
done
