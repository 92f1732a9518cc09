"""Diagnose the bf16 linear-chain case m3_d2: per-layer error vs the fp64 engine."""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2006_09503_b200 import pipesim as P
from paper_2006_09503_b200 import synthetic as S
from tests import _golden as G
cases = {m["name"]: (m, g) for m, g in G.linear_bf16()}
for name in sys.argv[1:]:
    meta, g = cases[name]
    ws, data = S.toy_model(meta["dim"], meta["layers"], meta["b"], meta["m"] * meta["T"], meta["seed"], exact=False)
    toy = P.ToyModel(meta["dim"], ws, data)
    for m_over in [meta["m"]]:
        cfg = P.TrainerConfig(meta["lr"], meta["beta"], meta["m"], meta["T"])
        for depth in sorted({1, meta["depth"]}):
            a = P.pipelined_execute(toy, cfg, P.PipelinePolicy(meta["policy"]), depth, precision="bf16", with_losses=True)
            b = P.pipelined_execute(toy, cfg, P.PipelinePolicy(meta["policy"]), depth, precision="fp64", with_losses=True)
            print(name, "depth", depth, "loss rel", np.max(np.abs(a.losses - b.losses) / np.abs(b.losses)))
            for t in range(1, meta["T"] + 1):
                errs = []
                for l in range(meta["layers"]):
                    da = a.trajectory[t][l] - ws[l]; db = b.trajectory[t][l] - ws[l]
                    errs.append(np.linalg.norm(da - db) / np.linalg.norm(db))
                print("  t", t, "per-layer rel err", np.round(errs, 4).tolist())
