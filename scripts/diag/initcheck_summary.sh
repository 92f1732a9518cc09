# initcheck on smoke() with a large print limit, aggregated by (kernel, source line): which
# kernels read global memory that compute-sanitizer never saw written (TMA bulk-tensor
# stores and tcgen05 traffic are invisible to it).
mkdir -p gpurun_out/sanitize
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 20000 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize/initcheck_full.txt 2>&1
python3 - <<'PY'
import re, collections
c = collections.Counter()
lines = open("gpurun_out/sanitize/initcheck_full.txt").read().splitlines()
for i, l in enumerate(lines):
    m = re.search(r"at (?:void )?p2bw::(?:<unnamed>::)?(\w+)[^)]*\)\+0x[0-9a-f]+ in (\S+)", l)
    if m and "Uninitialized" in lines[i - 1]:
        c[(m.group(1), m.group(2))] += 1
for (k, src), n in c.most_common():
    print(f"{n:6d}  {k}  {src}")
print([l for l in lines if "ERROR SUMMARY" in l])
PY
