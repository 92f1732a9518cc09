"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/ref_tool, built from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
The outputs are committed; GPU-box tests read them without /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import pipesim_oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"


def tool(*args) -> str:
    r = subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True)
    return r.stdout


def schedule_text(policy, d, m, T):
    return tool("schedule", policy, d, m, T)


SMALL_SCHEDULES = [(p, d, m, T) for p in range(5) for (d, m, T) in
                   [(1, 1, 3), (2, 4, 1), (2, 4, 3), (4, 4, 3), (4, 8, 2), (8, 8, 2), (3, 5, 2)]]
SWEEP_SCHEDULES = [(p, d, m, 2) for p in (1, 3, 4) for d in (2, 4, 8) for m in (4, 8, 16, 32) if m >= d or p != 4]

CLUSTERS = {
    "fixture_8x8": dict(total_workers=8, gpus_per_server=8, bandwidth_high_gbps=1000,
                        bandwidth_low_gbps=100, memory_capacity_gb=32),
    "fixture_16x8": dict(total_workers=16, gpus_per_server=8, bandwidth_high_gbps=1000,
                         bandwidth_low_gbps=100, memory_capacity_gb=32),
    "fixture_4x4_8gb": dict(total_workers=4, gpus_per_server=4, bandwidth_high_gbps=1000,
                            bandwidth_low_gbps=100, memory_capacity_gb=8),
    # one 8x B200 NVSwitch node: 900 GB/s per direction NVLink, 180 GB HBM3e
    "b200_8": dict(total_workers=8, gpus_per_server=8, bandwidth_high_gbps=900,
                   bandwidth_low_gbps=50, memory_capacity_gb=180),
}
MODELS = {
    "uniform8": O.uniform_profile_json("uniform8", 8, 1e-3, 2e-3, 1e8, 1e6, 2.5e5, [1, 2, 4]),
    "uniform24": O.uniform_profile_json("uniform24", 24, 1e-3, 2e-3, 1e8, 1e6, 2.5e5, [1, 2, 4, 8]),
    "fat4": O.uniform_profile_json("fat", 4, 1e-3, 2e-3, 1e8, 3e9, 1e9, [1]),
    "gpt_like48": O.uniform_profile_json("gpt48", 48, 2.1e-4, 4.2e-4, 8.85e7, 4.0e8, 2.0e6,
                                         [1, 2, 4, 8, 16]),
}
PLANS = [("uniform8", "fixture_8x8", 128), ("uniform8", "fixture_16x8", 128),
         ("uniform24", "fixture_8x8", 512), ("fat4", "fixture_4x4_8gb", 64),
         ("gpt_like48", "b200_8", 2048), ("uniform24", "b200_8", 256)]

TOY_GRID = [dict(dim=4, layers=d, b=2, seed=12345, lr=0.05, beta=beta, m=m, T=10, policy=p, depth=d)
            for d in (1, 2, 4) for m in (d, 2 * d) for beta in (0.0, 0.9) for p in (1, 3, 4)]
TOY_EXTRA = [dict(dim=16, layers=4, b=8, seed=424242, lr=0.05, beta=0.9, m=4, T=6, policy=4, depth=2),
             dict(dim=32, layers=8, b=16, seed=7, lr=0.02, beta=0.9, m=8, T=4, policy=4, depth=8),
             dict(dim=8, layers=4, b=4, seed=99, lr=0.05, beta=0.9, m=4, T=5, policy=2, depth=4)]


# reference_loop (semantics.cpp:167-184) at power-of-two and other m: its per-microbatch
# 1/m scaling (:145) differs from pipelined_execute's sum / count (:338-340) in the last bits
# when m is not a power of two.
LOOP_GRID = [dict(dim=8, layers=4, b=4, seed=31, lr=0.05, beta=0.9, m=m, T=5, delayed=dl)
             for m in (3, 4, 5, 6) for dl in (0, 1)]

# The production (bf16 tcgen05) path against the reference at the configs' widths:
# reference pipelined_execute trajectories (2BW unless stated) plus the vanilla-SGD
# trajectory (reference_vanilla) for the margin.  Stored as sampled entries of
# Delta W(t) = W(t) - W(0) (the full matrices are too large to commit) and the exact
# Frobenius norms of Delta W(t) and of Delta W(t) - Delta W_vanilla(t).
BF16_GRID = [
    dict(name="c1_d2", dim=256, layers=4, b=128, seed=7, lr=0.05, beta=0.9, m=4, T=6, policy=4, depth=2),
    dict(name="m3_d2", dim=256, layers=8, b=256, seed=11, lr=1e-3, beta=0.9, m=3, T=5, policy=4, depth=2),
    dict(name="m5_d4", dim=256, layers=8, b=256, seed=13, lr=1e-3, beta=0.9, m=5, T=4, policy=4, depth=4),
    dict(name="m8_d8", dim=256, layers=8, b=128, seed=17, lr=1e-3, beta=0.9, m=8, T=4, policy=4, depth=8),
    dict(name="1f1b_d4", dim=256, layers=4, b=128, seed=19, lr=0.05, beta=0.9, m=4, T=4, policy=2, depth=4),
    dict(name="c2_d4", dim=768, layers=12, b=512, seed=23, lr=1e-7, beta=0.9, m=4, T=4, policy=4, depth=4),
    dict(name="c2_m6_d1", dim=768, layers=12, b=512, seed=29, lr=1e-7, beta=0.9, m=6, T=4, policy=4, depth=1),
    dict(name="c3_d8", dim=1024, layers=8, b=256, seed=37, lr=1.5e-6, beta=0.9, m=8, T=4, policy=4, depth=8),
]
BF16_SAMPLES = 1024  # entries of Delta W per layer (relative norms: ~2% sampling error)


def _ref_run(args, shape):
    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / "traj.bin"
        out = tool(*args, path)
        return np.fromfile(path, dtype=np.float64).reshape(shape), out


def _bf16_case(c):
    L, n2 = c["layers"], c["dim"] ** 2
    common = (c["dim"], L, c["b"], c["seed"], repr(c["lr"]), repr(c["beta"]), c["m"], c["T"])
    traj, info = _ref_run(("toy", *common, c["policy"], c["depth"]), (c["T"] + 1, L, n2))
    van, _ = _ref_run(("loop", *common, 0), (c["T"] + 1, L, n2))
    rng = np.random.default_rng(c["seed"])
    idx = np.stack([np.sort(rng.choice(n2, BF16_SAMPLES, replace=False)) for _ in range(L)]).astype(np.int32)
    d_ref = traj - traj[0]
    d_van = van - van[0]
    pick = lambda a: np.stack([a[:, l, idx[l]] for l in range(L)], axis=1)  # [T+1, L, S]
    return dict(idx=idx, d_ref=pick(d_ref).astype(np.float32), d_van=pick(d_van)[-1].astype(np.float32),
                norm_ref=np.sqrt((d_ref ** 2).sum(axis=(1, 2))),
                norm_gap=np.sqrt(((d_ref - d_van) ** 2).sum(axis=(1, 2)))), json.loads(info)


def bf16_goldens():
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(_bf16_case, BF16_GRID))
    arrays, meta = {}, []
    for c, (arr, info) in zip(BF16_GRID, results):
        for k, v in arr.items():
            arrays[f"{c['name']}.{k}"] = v
        meta.append(dict(c, **info))
    np.savez_compressed(OUT / "linear_bf16.npz", **arrays)
    json.dump(meta, open(OUT / "linear_bf16.json", "w"), indent=1)


def loop_goldens():
    arrays, meta = {}, []
    for idx, c in enumerate(LOOP_GRID):
        traj, _ = _ref_run(("loop", c["dim"], c["layers"], c["b"], c["seed"], repr(c["lr"]), repr(c["beta"]),
                            c["m"], c["T"], c["delayed"]), (c["T"] + 1, c["layers"], c["dim"] ** 2))
        arrays[f"traj_{idx}"] = traj
        meta.append(c)
    np.savez_compressed(OUT / "loop_trajectories.npz", **arrays)
    json.dump(meta, open(OUT / "loop_trajectories.json", "w"), indent=1)


# Config 5: the reference's own simulate_policy (simulator.cpp:140-339) on
# the B200-measured GPT-24 block profile (p2bw_profile_blocks, b 4), one 8 x B200 NVSwitch
# node (900 GB/s per direction), 2BW / GPipe / PipeDream-Flush at d 2 / 4 / 8, m 4-32 (m a
# multiple of d: ParallelConfig's m = d * grad_accum), T = 8 batches -- and the same with
# free transfers (bandwidth 1e9 GB/s), so the exposed-transfer column is the reference's too.
C5_T = 8


def simulate_goldens():
    prof = OUT / "c5_profile_gpt-24_b200.json"
    rows = []
    with tempfile.TemporaryDirectory() as tmp:
        for tag, gbps in (("nvlink", 900), ("free", 1e9)):
            cp = Path(tmp) / f"c_{tag}.json"
            cp.write_text(json.dumps(dict(CLUSTERS["b200_8"], bandwidth_high_gbps=gbps, bandwidth_low_gbps=min(gbps, 50))))
            for d in (2, 4, 8):
                for m in (4, 8, 16, 32):
                    if m % d:
                        continue
                    for pol in (4, 1, 3):
                        r = json.loads(tool("simulate", prof, cp, pol, 1, d, 4, m // d, 0, C5_T))
                        rows.append(dict(link=tag, policy=pol, d=d, m=m, b=4, **r))
    json.dump({"profile": prof.name, "cluster": "b200_8", "num_batches": C5_T, "rows": rows},
              open(OUT / "c5_simulate.json", "w"), indent=1)


def main():
    if "--simulate" in sys.argv:
        return simulate_goldens()
    if "--bf16" in sys.argv:
        return bf16_goldens()
    if "--loop" in sys.argv:
        return loop_goldens()
    sched = {f"{p}/{d}/{m}/{T}": schedule_text(p, d, m, T) for p, d, m, T in SMALL_SCHEDULES}
    sweep = {f"{p}/{d}/{m}/{T}": hashlib.sha256(schedule_text(p, d, m, T).encode()).hexdigest()
             for p, d, m, T in SWEEP_SCHEDULES}
    versions = {f"{k}/{m}": int(tool("version", k, m)) for k in range(1, 40) for m in (1, 2, 4, 8)}
    json.dump({"schedules": sched, "sweep_sha256": sweep, "versions": versions},
              open(OUT / "schedules.json", "w"), indent=1, sort_keys=True)

    plans = {}
    with tempfile.TemporaryDirectory() as tmp:
        for mname, cname, B in PLANS:
            mp, cp = Path(tmp) / "m.json", Path(tmp) / "c.json"
            mp.write_text(MODELS[mname])
            cp.write_text(json.dumps(CLUSTERS[cname]))
            out = tool("plan", mp, cp, B, 4)
            plans[f"{mname}/{cname}/{B}"] = (json.loads(out) if not out.startswith("ERROR")
                                             else {"error": out.strip()})
        json.dump({"models": MODELS, "clusters": CLUSTERS, "plans": plans},
                  open(OUT / "plans.json", "w"), indent=1, sort_keys=True)

        arrays, meta = {}, []
        for idx, c in enumerate(TOY_GRID + TOY_EXTRA):
            path = Path(tmp) / "traj.bin"
            info = json.loads(tool("toy", c["dim"], c["layers"], c["b"], c["seed"], repr(c["lr"]),
                                   repr(c["beta"]), c["m"], c["T"], c["policy"], c["depth"], path))
            traj = np.fromfile(path, dtype=np.float64).reshape(c["T"] + 1, c["layers"], c["dim"] ** 2)
            arrays[f"traj_{idx}"] = traj
            meta.append(dict(c, **info))
    np.savez_compressed(OUT / "toy_trajectories.npz", **arrays)
    json.dump(meta, open(OUT / "toy_trajectories.json", "w"), indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
