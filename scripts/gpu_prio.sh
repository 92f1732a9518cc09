# Stream-priority experiment: bench.py under several P2BW_STREAM_PRIO settings.
one() { P2BW_STREAM_PRIO="$1" timeout 150 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"; }
for r in 1 2; do
  one "side=-2,main=-1"
  one "side=-3,main=-2,fwd=-1"
  one "side=-2,main=-2"
  one "side=-1,main=-2"
  one "side=-2,main=-1,update=-3"
done
