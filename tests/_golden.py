"""Loaders for the committed golden fixtures (made by tests/golden/make_golden.py
from the reference itself)."""
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(None)
def schedules():
    return json.loads((GOLDEN / "schedules.json").read_text())


@lru_cache(None)
def plans():
    return json.loads((GOLDEN / "plans.json").read_text())


@lru_cache(None)
def toy():
    meta = json.loads((GOLDEN / "toy_trajectories.json").read_text())
    arrs = np.load(GOLDEN / "toy_trajectories.npz")
    return [(m, arrs[f"traj_{i}"]) for i, m in enumerate(meta)]


@lru_cache(None)
def loops():
    """reference_loop trajectories (ref_tool loop) at m = 3..6, vanilla and delayed."""
    meta = json.loads((GOLDEN / "loop_trajectories.json").read_text())
    arrs = np.load(GOLDEN / "loop_trajectories.npz")
    return [(m, arrs[f"traj_{i}"]) for i, m in enumerate(meta)]


@lru_cache(None)
def linear_bf16():
    """Reference pipelined_execute at the configs' widths, sampled (make_golden.py BF16_GRID)."""
    meta = json.loads((GOLDEN / "linear_bf16.json").read_text())
    arrs = np.load(GOLDEN / "linear_bf16.npz")
    return [(m, {k.split(".", 1)[1]: arrs[k] for k in arrs.files if k.startswith(m["name"] + ".")}) for m in meta]
