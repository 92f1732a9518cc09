"""Summarise ncu output for profiles/ (committed evidence).

  python scripts/summarize_ncu.py launches <launches.csv>     -> per-kernel share table (markdown)
  python scripts/summarize_ncu.py full <report.ncu-rep>       -> key SOL / DRAM / tensor metrics per launch

The launch list comes from `ncu --metrics gpu__time_duration.sum --clock-control none`
(cold-cache, serialised: compare shares, not absolutes)."""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("p2bw::", "").replace("(anonymous namespace)::", "")
    return name.replace("<unnamed>::", "").strip()


def launches(path: str) -> str:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])  # launches, us, DRAM bytes
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        name = r.get("Metric Name")
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        k = short(r["Kernel Name"])
        if name == "gpu__time_duration.sum":
            us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
            tot[k][0] += 1
            tot[k][1] += us
        elif name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot[k][2] += v * scale.get(unit, 1.0)
    total = sum(v[1] for v in tot.values()) or 1.0
    have_dram = any(v[2] for v in tot.values())
    out = ["| kernel | launches | total us | share | avg us |" + (" DRAM MB / launch |" if have_dram else ""),
           "|---|---|---|---|---|" + ("---|" if have_dram else "")]
    for k, (n, us, by) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / total:.1f}% | {us / n:.2f} |" +
                   (f" {by / n / 1e6:.1f} |" if have_dram else ""))
    nl = sum(v[0] for v in tot.values())
    out.append(f"\n{nl} launches, {total:.1f} us of kernel time in the window.")
    if have_dram:
        g = [v for k, v in tot.items() if "gemm_tc_kernel" in k]
        n, by = sum(v[0] for v in g), sum(v[2] for v in g)
        if n:
            out.append(f"gemm_tc_kernel: {n} launches, mean DRAM read + write {by / n:.0f} bytes per launch.")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = [hdr.index(m) for m in METRICS if m in hdr]
    kn = hdr.index("Kernel Name")
    head = "| kernel | " + " | ".join(f"{hdr[i].split('.')[0]} ({units[i]})" for i in idx) + " |"
    out = [head, "|" + "---|" * (len(idx) + 1)]
    for r in rows[2:]:
        out.append(f"| `{short(r[kn])[:60]}` | " + " | ".join(r[i] for i in idx) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
