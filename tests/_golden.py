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
