"""bf16 linear chain at depth d vs the fp64 engine: max per-layer rel err of Delta W at t=1..T."""
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
    cfg = P.TrainerConfig(meta["lr"], meta["beta"], meta["m"], meta["T"])
    b = P.pipelined_execute(toy, cfg, P.PipelinePolicy(meta["policy"]), meta["depth"], precision="fp64")
    for rep in range(3):
        a = P.pipelined_execute(toy, cfg, P.PipelinePolicy(meta["policy"]), meta["depth"], precision="bf16")
        e = max(np.linalg.norm((a.trajectory[t][l] - ws[l]) - (b.trajectory[t][l] - ws[l])) /
                np.linalg.norm(b.trajectory[t][l] - ws[l]) for t in range(1, meta["T"] + 1) for l in range(meta["layers"]))
        print(name, "rep", rep, "max rel err", round(e, 5), flush=True)
