"""CPU restatement of the reference's pipelined-training path -- TEST INFRASTRUCTURE.

This module is the parity oracle.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm may import it, and only as the checker;
the product (paper_2006_09503_b200, libp2bw.so) never routes through it.

It restates, function by function, the reference pipesim library
(/root/reference/proj/core/src, cited file:line) in plain Python + numpy:
  schedule    weight_version_2bw, required_versions, generate_schedule,
              serialize_programs                        (schedule.cpp)
  profile     partition_equal, load_model_profile / load_cluster_spec  (profile.cpp)
  costmodel   bandwidth tiers, throughput, memory        (costmodel.cpp)
  planner     search_microbatch, plan                    (planner.cpp)
  semantics   ToyModel.make (splitmix64), reference loops, pipelined_execute
              interpreter                                (semantics.cpp)
Floating-point expressions keep the reference's operation order; numpy
element-wise ops round like scalar C++ (no FMA), so trajectories and plans are
bit-identical to the reference.  It is pinned against the reference itself
(oracle/_ref/libpipesim_ref.so, built by oracle/Makefile) and against the
golden vectors in tests/golden/ (see tests/test_oracle.py).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

# ---- schedule (schedule.hpp:10-46) -------------------------------------------------

NONE, GPIPE, ONEF1B, FLUSH, TWOBW = range(5)
POLICY_NAMES = ["none", "gpipe", "1f1b", "flush", "2bw"]
(FORWARD, BACKWARD, RECOMPUTE, UPDATE, FLUSHB, ACT_SEND, ACT_RECV, GRAD_SEND, GRAD_RECV,
 ALLREDUCE) = range(10)
OP_NAMES = ["forward", "backward", "recompute", "update", "flush", "act_send", "act_recv",
            "grad_send", "grad_recv", "allreduce"]
LATEST = -1


class OracleError(Exception):
    """pipesim::Error (error.hpp:9-12)."""


def weight_version_2bw(k: int, m: int) -> int:
    """schedule.cpp:58-62"""
    if k < 1:
        raise OracleError("microbatch index must be >= 1")
    if m < 1:
        raise OracleError("microbatches per batch must be >= 1")
    return max((k - 1) // m - 1, 0)


def required_versions(policy: int, d: int, m: int) -> int:
    """schedule.cpp:64-78"""
    if policy == TWOBW:
        return 2
    if policy == ONEF1B:
        return d
    return 1


def _emit_update(ops, flush):
    """schedule.cpp:80-84"""
    if flush:
        ops.append((FLUSHB, 0, 0))
    ops.append((ALLREDUCE, 0, 0))
    ops.append((UPDATE, 0, 0))


def _batched(policy, m, T):
    """schedule.cpp:88-105"""
    ops = []
    for t in range(1, T + 1):
        base, ver = (t - 1) * m, t - 1
        if policy == GPIPE:
            ops += [(FORWARD, base + j, ver) for j in range(1, m + 1)]
            ops += [(BACKWARD, base + j, ver) for j in range(1, m + 1)]
        else:
            for j in range(1, m + 1):
                ops += [(FORWARD, base + j, ver), (BACKWARD, base + j, ver)]
        _emit_update(ops, policy == GPIPE)
    return ops


def _flush(stage, d, m, T):
    """schedule.cpp:109-123"""
    ops = []
    warm = min(d - stage, m)
    for t in range(1, T + 1):
        base, ver = (t - 1) * m, t - 1
        ops += [(FORWARD, base + j, ver) for j in range(1, warm + 1)]
        for j in range(1, m + 1):
            ops.append((BACKWARD, base + j, ver))
            if j + warm <= m:
                ops.append((FORWARD, base + j + warm, ver))
        _emit_update(ops, True)
    return ops


def _continuous(policy, stage, d, m, T):
    """schedule.cpp:126-144"""
    total = m * T
    warm = min(d - stage, total)
    ver = (lambda k: weight_version_2bw(k, m)) if policy == TWOBW else (lambda k: LATEST)
    ops = [(FORWARD, j, ver(j)) for j in range(1, warm + 1)]
    for k in range(1, total + 1):
        ops.append((BACKWARD, k, ver(k)))
        if policy == ONEF1B or k % m == 0:
            _emit_update(ops, False)
        if k + warm <= total:
            ops.append((FORWARD, k + warm, ver(k + warm)))
    return ops


def generate_schedule(policy: int, d: int, m: int, T: int) -> list[list[tuple[int, int, int]]]:
    """schedule.cpp:148-175 -> one list of (kind, microbatch, version) per stage."""
    if d < 1:
        raise OracleError("depth must be >= 1")
    if m < 1:
        raise OracleError("microbatches per batch must be >= 1")
    if T < 1:
        raise OracleError("num_batches must be >= 1")
    if policy == TWOBW and m < d:
        raise OracleError(f"2bw requires m >= d (m={m}, d={d})")
    out = []
    for s in range(d):
        if policy in (GPIPE, NONE):
            out.append(_batched(policy, m, T))
        elif policy == FLUSH:
            out.append(_flush(s, d, m, T))
        else:
            out.append(_continuous(policy, s, d, m, T))
    return out


def serialize_programs(programs) -> str:
    """schedule.cpp:177-195"""
    lines = []
    for s, ops in enumerate(programs):
        for kind, mb, ver in ops:
            line = f"stage={s} op={OP_NAMES[kind]}"
            if kind in (FORWARD, BACKWARD, RECOMPUTE):
                line += f" mb={mb} ver={'latest' if ver == LATEST else ver}"
            lines.append(line + "\n")
    return "".join(lines)


# ---- profile (profile.hpp:13-93, profile.cpp) --------------------------------------

@dataclass
class Block:
    fwd: dict
    bwd: dict
    weight_bytes: float
    act_total: dict
    act_input: dict
    act_boundary: dict


@dataclass
class Cluster:
    total_workers: int
    gpus_per_server: int
    bandwidth_high: float
    bandwidth_low: float
    memory_capacity: float


@dataclass
class Stage:
    fwd: dict = field(default_factory=dict)
    bwd: dict = field(default_factory=dict)
    weight_bytes: float = 0.0
    act_total: dict = field(default_factory=dict)
    act_input: dict = field(default_factory=dict)
    act_output: dict = field(default_factory=dict)


def _table(j, scale):
    return {int(k): float(v) * scale for k, v in j.items()}


def load_model_profile(text: str) -> list[Block]:
    """profile.cpp:162-193 (ms -> s)."""
    doc = json.loads(text)
    return [Block(_table(b["fwd_ms"], 1e-3), _table(b["bwd_ms"], 1e-3), float(b["weight_bytes"]),
                  _table(b["act_total_bytes"], 1.0), _table(b["act_input_bytes"], 1.0),
                  _table(b["act_boundary_bytes"], 1.0)) for b in doc["blocks"]]


def load_cluster_spec(text: str) -> Cluster:
    """profile.cpp:212-230 (*_gbps are GB/s)."""
    d = json.loads(text)
    return Cluster(int(d["total_workers"]), int(d["gpus_per_server"]),
                   float(d["bandwidth_high_gbps"]) * 1e9, float(d["bandwidth_low_gbps"]) * 1e9,
                   float(d["memory_capacity_gb"]) * 1e9)


def uniform_profile_json(name, n, fwd_b1, bwd_b1, weight, act_total_b1, act_input_b1, sizes) -> str:
    """make_uniform_profile (profile.cpp:261-282) rendered as a profile document."""
    blk = {"fwd_ms": {str(b): fwd_b1 * b * 1e3 for b in sizes},
           "bwd_ms": {str(b): bwd_b1 * b * 1e3 for b in sizes},
           "weight_bytes": weight,
           "act_total_bytes": {str(b): act_total_b1 * b for b in sizes},
           "act_input_bytes": {str(b): act_input_b1 * b for b in sizes},
           "act_boundary_bytes": {str(b): 2.0 * act_input_b1 * b for b in sizes}}
    return json.dumps({"model": name, "blocks": [blk] * n})


def partition_equal(blocks: list[Block], d: int) -> list[Stage]:
    """profile.cpp:104-131 (block-by-block summation order)."""
    n = len(blocks)
    if d < 1:
        raise OracleError("depth must be >= 1")
    if n % d:
        raise OracleError(f"depth {d} does not divide block count {n}")
    per = n // d
    out = []
    for s in range(d):
        st = Stage()
        first, last = blocks[s * per], blocks[(s + 1) * per - 1]
        st.act_input = dict(first.act_input)
        st.act_output = {b: v - last.act_input[b] for b, v in last.act_boundary.items()}
        for blk in blocks[s * per:(s + 1) * per]:
            st.weight_bytes += blk.weight_bytes
            for b, v in blk.fwd.items():
                st.fwd[b] = st.fwd.get(b, 0.0) + v
            for b, v in blk.bwd.items():
                st.bwd[b] = st.bwd.get(b, 0.0) + v
            for b, v in blk.act_total.items():
                st.act_total[b] = st.act_total.get(b, 0.0) + v
        out.append(st)
    return out


# ---- costmodel (costmodel.cpp) ---------------------------------------------------------

def bwdth_width(w, c: Cluster):
    """costmodel.cpp:7-10"""
    return c.bandwidth_high if w <= c.gpus_per_server else c.bandwidth_low


def bwdth_depth(d, w, c: Cluster):
    """costmodel.cpp:12-16"""
    return c.bandwidth_high if w * d <= c.gpus_per_server else c.bandwidth_low


def comm_interstage(boundary, c, d, w):
    """costmodel.cpp:18-21"""
    return 0.0 if d <= 1 else 2.0 * boundary / bwdth_depth(d, w, c)


def allreduce_seconds(weight_bytes, w, c):
    """costmodel.cpp:23-27"""
    if w <= 1:
        return 0.0
    return 2.0 * (w - 1) / w * weight_bytes / bwdth_width(w, c)


def _comm_into(stages, c, w, i, b):
    """costmodel.cpp:33-47"""
    d = len(stages)
    if d == 1:
        return 0.0
    t = 0.0
    if i > 0:
        t += comm_interstage(stages[i - 1].act_output[b], c, d, w)
    if i < d - 1:
        t += comm_interstage(stages[i].act_output[b], c, d, w)
    return t


def throughput_nopipeline(stages, c, w, b, m):
    """costmodel.cpp:55-64"""
    t = 0.0
    for i, st in enumerate(stages):
        ar = allreduce_seconds(st.weight_bytes, w, c)
        t += max(st.fwd[b] + st.bwd[b] + _comm_into(stages, c, w, i, b), ar / m)
    return float(b) * w / t


def throughput_pipelined(stages, c, w, b, m, recompute, c_extra=4.0 / 3.0):
    """costmodel.cpp:66-78"""
    cext = c_extra if recompute else 1.0
    t = 0.0
    for i, st in enumerate(stages):
        ar = allreduce_seconds(st.weight_bytes, w, c)
        t = max(t, max(cext * (st.fwd[b] + st.bwd[b]) + _comm_into(stages, c, w, i, b), ar / m))
    return float(b) * w / t


def memory_footprint(stages, policy, b, m, recompute):
    """costmodel.cpp:80-107"""
    d = len(stages)
    worst = None
    for s, st in enumerate(stages):
        versions = max(d - s, 1) if policy == ONEF1B else required_versions(policy, d, m)
        stashes = 1 if policy == NONE else (m if policy == GPIPE else min(d - s, m))
        unit = st.act_input[b] if recompute else st.act_total[b] + st.act_input[b]
        transient = st.act_total[b] if recompute else 0.0
        v = versions * st.weight_bytes + stashes * unit + transient
        worst = v if worst is None else max(worst, v)
    return worst


# ---- planner (planner.cpp:13-99) -------------------------------------------------------

def search_microbatch(stages, c: Cluster, w, d, max_batch, policy=TWOBW):
    """planner.cpp:13-43 -> dict or None"""
    best = None
    for b in sorted(stages[0].fwd):
        g = max_batch // (w * d * b)
        if g < 1:
            continue
        for r in (False, True):
            if d == 1 and r:
                continue
            m = d * g
            mem = memory_footprint(stages, policy, b, m, r)
            if mem > c.memory_capacity:
                continue
            tput = (throughput_nopipeline(stages, c, w, b, m) if d == 1
                    else throughput_pipelined(stages, c, w, b, m, r))
            if best is None or tput > best["throughput"] or (
                    tput == best["throughput"] and b > best["microbatch_size"]):
                best = {"width": w, "depth": d, "microbatch_size": b, "recompute": r,
                        "grad_accum": g, "throughput": tput, "memory_bytes": mem}
    return best


def plan(blocks: list[Block], c: Cluster, max_batch: int, policy=TWOBW) -> dict:
    """planner.cpp:45-99"""
    if max_batch < 1:
        raise OracleError("max safe batch size must be >= 1")
    n = c.total_workers
    ranked, rejected, pairs = [], [], 0
    cache = {}
    for w in range(1, n + 1):
        d = 1
        while d * w <= n:
            pairs += 1
            if len(blocks) % d:
                rejected.append({"width": w, "depth": d,
                                 "reject_reason": "depth does not divide block count"})
            else:
                if d not in cache:
                    cache[d] = partition_equal(blocks, d)
                hit = search_microbatch(cache[d], c, w, d, max_batch, policy)
                if hit is None:
                    rejected.append({"width": w, "depth": d, "reject_reason":
                                     "no (b, r) fits the memory capacity and batch cap"})
                else:
                    ranked.append(hit)
            d += 1
    if not ranked:
        raise OracleError("no feasible configuration for this cluster:")
    # stable sort: throughput desc, depth asc, width asc
    ranked.sort(key=lambda s: (-s["throughput"], s["depth"], s["width"]))
    best = ranked[0]
    g_cluster = max(max_batch // (n * best["microbatch_size"]), 1)
    return {"best": {k: best[k] for k in ("width", "depth", "microbatch_size", "recompute",
                                          "grad_accum")},
            "predicted_throughput": best["throughput"], "predicted_memory_bytes": best["memory_bytes"],
            "grad_accum_for_cluster": g_cluster, "pairs_examined": pairs,
            "ranked": ranked, "rejected": rejected}


# ---- semantics (semantics.cpp) -----------------------------------------------------------

_M64 = (1 << 64) - 1


class SplitMix64:
    """semantics.cpp:64-75"""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def next(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0) - 0.5

    def mat(self, rows: int, cols: int) -> np.ndarray:
        """random_mat (semantics.cpp:77-81): column-major fill order."""
        vals = np.array([self.next() for _ in range(rows * cols)], dtype=np.float64)
        return vals.reshape((cols, rows)).T.copy()


def matmul(a, b):
    """semantics.cpp:9-19: c(i,j) += a(i,k) b(k,j), k ascending."""
    c = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        c += np.outer(a[:, k], b[k, :])
    return c


def matmul_tn(a, b):
    """semantics.cpp:21-32: c(i,j) = sum_k a(k,i) b(k,j)."""
    c = np.zeros((a.shape[1], b.shape[1]))
    for k in range(a.shape[0]):
        c += np.outer(a[k, :], b[k, :])
    return c


def matmul_nt(a, b):
    """semantics.cpp:34-44: c(i,j) += a(i,k) b(j,k)."""
    c = np.zeros((a.shape[0], b.shape[0]))
    for k in range(a.shape[1]):
        c += np.outer(a[:, k], b[:, k])
    return c


@dataclass
class ToyModel:
    dim: int
    weights: list
    dataset: list  # [(x, y)]

    @staticmethod
    def make(dim, layers, b, nmb, seed) -> "ToyModel":
        """semantics.cpp:85-109"""
        if min(dim, layers, b, nmb) < 1:
            raise OracleError("toy model dimensions must be >= 1")
        g = SplitMix64(seed)
        ws = []
        for _ in range(layers):
            w = g.mat(dim, dim) * 0.2
            w[np.diag_indices(dim)] += 1.0
            ws.append(w)
        a = g.mat(dim, dim) * 0.3
        a[np.diag_indices(dim)] += 1.0
        data = []
        for _ in range(nmb):
            x = g.mat(dim, b)
            data.append((x, matmul(a, x)))
        return ToyModel(dim, ws, data)


def _apply_update(weights, vel, grad, lr, beta):
    """semantics.cpp:153-165"""
    for l in range(len(weights)):
        vel[l] = beta * vel[l] + (1.0 - beta) * grad[l]
        weights[l] = weights[l] + (-lr) * vel[l]


def _batch_gradient(model, weights, t, m):
    """semantics.cpp:122-151 -> (grad, loss)"""
    L = len(weights)
    b = model.dataset[0][0].shape[1]
    grad = [np.zeros_like(w) for w in weights]
    loss = 0.0
    for j in range(m):
        x, y = model.dataset[(t - 1) * m + j]
        inputs, cur = [], x
        for l in range(L):
            inputs.append(cur)
            cur = matmul(weights[l], cur)
        diff = cur - y
        g = diff / b
        loss += float(np.sum((diff * diff / (2.0 * b)).flatten(order="F")))
        for l in range(L - 1, -1, -1):
            grad[l] = grad[l] + (1.0 / m) * matmul_nt(g, inputs[l])
            if l > 0:
                g = matmul_tn(weights[l], g)
    return grad, loss / m


def reference_loop(model, lr, beta, m, T, delayed):
    """semantics.cpp:167-184 -> (trajectory, losses)"""
    traj = [[w.copy() for w in model.weights]]
    weights = [w.copy() for w in model.weights]
    vel = [np.zeros_like(w) for w in weights]
    losses = []
    for t in range(1, T + 1):
        ev = max(t - 2, 0) if delayed else t - 1
        grad, loss = _batch_gradient(model, traj[ev], t, m)
        losses.append(loss)
        _apply_update(weights, vel, grad, lr, beta)
        traj.append([w.copy() for w in weights])
    return traj, losses


def pipelined_execute(model: ToyModel, lr, beta, m, T, policy, depth):
    """semantics.cpp:238-375 (round-robin interpreter) -> (trajectory, consistent, max_versions)"""
    L = len(model.weights)
    if L % depth:
        raise OracleError(f"block count {L} not divisible by depth {depth}")
    if len(model.dataset) < m * T:
        raise OracleError("toy dataset has too few microbatches for the requested run")
    per = L // depth
    b = model.dataset[0][0].shape[1]
    programs = generate_schedule(policy, depth, m, T)
    st = [{"versions": {0: [w.copy() for w in model.weights[s * per:(s + 1) * per]]},
           "vel": None, "gsum": None, "count": 0, "upd": 0, "ptr": 0, "stash": {},
           "out": {}, "gprev": {}, "snap": {}} for s in range(depth)]
    consistent, max_v = True, 1
    total = sum(len(p) for p in programs)
    done = 0
    while done < total:
        progress = False
        for s in range(depth):
            S, ops = st[s], programs[s]
            while S["ptr"] < len(ops):
                kind, k, ver = ops[S["ptr"]]
                if kind == FORWARD:
                    if s > 0 and k not in st[s - 1]["out"]:
                        break
                    v = S["upd"] if ver == LATEST else ver
                    if v not in S["versions"]:
                        raise OracleError(f"stage {s} forward of microbatch {k} needs discarded "
                                          f"weight version {v}")
                    W = S["versions"][v]
                    cur = model.dataset[k - 1][0] if s == 0 else st[s - 1]["out"].pop(k)
                    ins = []
                    for l in range(per):
                        ins.append(cur)
                        cur = matmul(W[l], cur)
                    S["stash"][k] = (v, ins)
                    S["out"][k] = cur
                elif kind == BACKWARD:
                    if s < depth - 1 and k not in st[s + 1]["gprev"]:
                        break
                    if k not in S["stash"]:
                        raise OracleError(f"backward before forward for microbatch {k}")
                    v, ins = S["stash"].pop(k)
                    W = S["versions"][v]
                    if s == depth - 1:
                        g = (S["out"].pop(k) - model.dataset[k - 1][1]) / b
                    else:
                        g = st[s + 1]["gprev"].pop(k)
                    if S["gsum"] is None:
                        S["gsum"] = [np.zeros_like(w) for w in W]
                    for l in range(per - 1, -1, -1):
                        S["gsum"][l] = S["gsum"][l] + 1.0 * matmul_nt(g, ins[l])
                        if l > 0 or s > 0:
                            g = matmul_tn(W[l], g)
                    S["count"] += 1
                    if s > 0:
                        S["gprev"][k] = g
                elif kind == UPDATE:
                    if S["count"] == 0:
                        raise OracleError("weight update with no gradients")
                    grad = [gm / S["count"] for gm in S["gsum"]]
                    W = [w.copy() for w in S["versions"][S["upd"]]]
                    if S["vel"] is None:
                        S["vel"] = [np.zeros_like(w) for w in W]
                    _apply_update(W, S["vel"], grad, lr, beta)
                    S["upd"] += 1
                    S["versions"][S["upd"]] = W
                    S["snap"][S["upd"]] = [w.copy() for w in W]
                    _prune(S, policy)
                    S["gsum"], S["count"] = None, 0
                    max_v = max(max_v, len(S["versions"]))
                S["ptr"] += 1
                done += 1
                progress = True
        if not progress:
            raise OracleError("dependency deadlock in toy-model replay")
    upb = m if policy == ONEF1B else 1
    traj = [[w.copy() for w in model.weights]]
    for t in range(1, T + 1):
        traj.append([w for s in range(depth) for w in st[s]["snap"][t * upb]])
    return traj, consistent, max_v


def _prune(S, policy):
    """semantics.cpp:213-234"""
    latest = S["upd"]
    if policy == TWOBW:
        S["versions"].pop(latest - 2, None)
    elif policy == ONEF1B:
        ref = {v for v, _ in S["stash"].values()}
        for v in list(S["versions"]):
            if v != latest and v not in ref:
                del S["versions"][v]
    else:
        for v in list(S["versions"]):
            if v != latest:
                del S["versions"][v]


def flat_trajectory(traj) -> np.ndarray:
    """(T+1) x layers x dim*dim, each matrix column-major like Mat::data."""
    return np.stack([np.stack([w.flatten(order="F") for w in ws]) for ws in traj])


def max_rel_diff(a: np.ndarray, b: np.ndarray) -> float:
    """semantics.cpp:51-59 over whole arrays."""
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return float(np.max(np.abs(a - b) / denom)) if a.size else 0.0
