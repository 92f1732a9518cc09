"""SASS instruction histogram of libp2bw.so per kernel: the tcgen05 / TMA / TMEM
mnemonics (B200_PROFILING.md) that prove which kernels run on the tensor cores.

    python scripts/sass_histogram.py > profiles/r2_sass_histogram.md
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2006_09503_b200" / "libp2bw.so"
KEYS = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF", "LDTM", "STTM",
        "UBLKCP", "UBLKRED", "SYNCS", "HMMA", "DMUL", "DADD", "MUFU.EX2"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    per = defaultdict(Counter)
    total = Counter()
    fn = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if not m or fn is None:
            continue
        op = m.group(1)
        per[fn]["instructions"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                if k == "UTCHMMA" and ".2CTA" in op:
                    continue
                per[fn][k] += 1
                total[k] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True, text=True).stdout.split("\n")
    names = dict(zip(per, demangle))
    # one row per kernel (template instantiations summed)
    groups = defaultdict(Counter)
    inst = Counter()
    for fn, c in per.items():
        base = names[fn].replace("(anonymous namespace)::", "")
        base = re.sub(r"<.*", "", re.sub(r"\(.*", "", base)).replace("void ", "").strip()
        groups[base].update(c)
        inst[base] += 1
    cols = ["instructions"] + [k for k in KEYS if total[k]]
    print(f"# SASS histogram of {LIB.name} (cuobjdump -sass, sm_100a)\n")
    print("Per kernel, template instantiations summed.  UTCHMMA = tcgen05.mma (.2CTA = cta_group::2),")
    print("UTMALDG / UTMASTG / UTMAREDG = TMA tensor load / store / reduce, LDTM / STTM = tcgen05.ld / st,")
    print("UBLKCP = bulk copy, DMUL / DADD = fp64 (the linear-chain parity kernels).\n")
    print("| kernel | instantiations | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for base, c in sorted(groups.items(), key=lambda kv: -kv[1]["instructions"]):
        print(f"| `{base}` | {inst[base]} | " + " | ".join(str(c[k]) for k in cols) + " |")
    print(f"| **total** | {sum(inst.values())} | " + " | ".join(
        str(sum(c["instructions"] for c in per.values())) if k == "instructions" else str(total[k]) for k in cols) + " |")


if __name__ == "__main__":
    sys.exit(main())
