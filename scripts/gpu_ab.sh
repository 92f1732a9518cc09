# A/B of two builds of libp2bw.so on one box (abtest/old.so vs abtest/new.so), alternating.
L=paper_2006_09503_b200/libp2bw.so
one() { cp abtest/$1.so $L; timeout 150 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; }
for r in $(seq ${REPS:-3}); do one old; one new; done
cp abtest/new.so $L
