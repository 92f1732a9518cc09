"""CPU oracle for the transformer stages -- TEST INFRASTRUCTURE (never shipped).

The reference has no layer arithmetic (parity for LN / attention /
GELU / CE is unpinned), so this oracle fixes the math the B200 engine
implements and checks it with torch CPU autograd in float64:

  pre-LN GPT-2 / BERT block, LayerNorm eps 1e-5, tanh-GELU, softmax attention
  with head dim hidden / heads (64 or 128) and scale 1/sqrt(head dim) (causal mask
  for GPT), token + position
  embedding on stage 0, LNf + untied LM head + mean cross-entropy over the
  head rows (every position, or `head_rows` evenly spaced positions per
  sequence) on the last stage.

Training semantics are the reference's (semantics.cpp): the 2BW pipeline is
equivalent to delay-1 momentum SGD with dampening -- batch t's gradient is taken
at W^(max(t-2,0)) and applied to W^(t-1) (reference_loop, semantics.cpp:167-184;
update :153-165).  `train()` restates that loop for the transformer loss.

Parameters use the engine's flat per-stage layout (model_transformer.cu
layout_params): 64-element aligned tensors, vocab padded to a multiple of 128,
and the same deterministic initialiser (init_uniform in tkernels.cu).
"""
from __future__ import annotations

import math

import numpy as np
import torch

_M64 = (1 << 64) - 1


# The configuration type and the synthetic data are the package's (the bench feeds the
# same batches); the oracle only restates the arithmetic.
from paper_2006_09503_b200.synthetic import TransformerSpec as Spec  # noqa: E402
from paper_2006_09503_b200.synthetic import head_positions  # noqa: E402,F401
from paper_2006_09503_b200.synthetic import token_batch as synthetic_batch  # noqa: E402,F401


def _a64(n):
    return (n + 63) // 64 * 64


def stage_layout(spec: Spec, lo: int, hi: int, depth_first: bool, depth_last: bool):
    """Offsets of every tensor in one stage's flat vector (layout_params)."""
    h = spec.hidden
    off = 0
    out = {}

    def take(name, shape):
        nonlocal off
        n = int(np.prod(shape))
        out[name] = (off, shape)
        off += _a64(n)

    if depth_first:
        take("tok", (spec.vp, h))
        take("pos", (spec.seq, h))
    for l in range(lo, hi):
        take(f"{l}.ln1g", (h,))
        take(f"{l}.ln1b", (h,))
        take(f"{l}.wqkv", (3 * h, h))
        take(f"{l}.bqkv", (3 * h,))
        take(f"{l}.wo", (h, h))
        take(f"{l}.bo", (h,))
        take(f"{l}.ln2g", (h,))
        take(f"{l}.ln2b", (h,))
        take(f"{l}.w1", (4 * h, h))
        take(f"{l}.b1", (4 * h,))
        take(f"{l}.w2", (h, 4 * h))
        take(f"{l}.b2", (h,))
    if depth_last:
        take("lnfg", (h,))
        take("lnfb", (h,))
        take("head", (spec.vp, h))
    return out, off


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def init_uniform(n: int, seed: int, uid: int, hw: float) -> np.ndarray:
    """tkernels.cu k_init_uniform: (u - 0.5) * 2 hw, u from mix64(key + i * C)."""
    key = (seed * 0x9E3779B97F4A7C15 + uid * 0xBF58476D1CE4E5B9) & _M64
    with np.errstate(over="ignore"):
        i = np.arange(n, dtype=np.uint64)
        r = _mix64(np.uint64(key) + i * np.uint64(0xD1B54A32D192ED03))
    u = (r >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return ((u - 0.5) * 2.0 * hw).astype(np.float32)


def init_params(spec: Spec, seed: int) -> dict[str, np.ndarray]:
    """Model-wide tensors by name (independent of the stage partition)."""
    h, hw = spec.hidden, np.float32(0.02 * math.sqrt(3.0))
    p = {}
    tok = np.zeros((spec.vp, h), np.float32)
    tok[:spec.vocab] = init_uniform(spec.vocab * h, seed, 1 << 40, hw).reshape(spec.vocab, h)
    p["tok"] = tok
    p["pos"] = init_uniform(spec.seq * h, seed, (1 << 40) + 1, hw).reshape(spec.seq, h)
    for l in range(spec.layers):
        uid = l * 16
        p[f"{l}.ln1g"] = np.ones(h, np.float32)
        p[f"{l}.ln1b"] = np.zeros(h, np.float32)
        p[f"{l}.wqkv"] = init_uniform(3 * h * h, seed, uid + 1, hw).reshape(3 * h, h)
        p[f"{l}.bqkv"] = np.zeros(3 * h, np.float32)
        p[f"{l}.wo"] = init_uniform(h * h, seed, uid + 2, hw).reshape(h, h)
        p[f"{l}.bo"] = np.zeros(h, np.float32)
        p[f"{l}.ln2g"] = np.ones(h, np.float32)
        p[f"{l}.ln2b"] = np.zeros(h, np.float32)
        p[f"{l}.w1"] = init_uniform(4 * h * h, seed, uid + 3, hw).reshape(4 * h, h)
        p[f"{l}.b1"] = np.zeros(4 * h, np.float32)
        p[f"{l}.w2"] = init_uniform(4 * h * h, seed, uid + 4, hw).reshape(h, 4 * h)
        p[f"{l}.b2"] = np.zeros(h, np.float32)
    p["lnfg"] = np.ones(h, np.float32)
    p["lnfb"] = np.zeros(h, np.float32)
    head = np.zeros((spec.vp, h), np.float32)
    head[:spec.vocab] = init_uniform(spec.vocab * h, seed, 1 << 41, hw).reshape(spec.vocab, h)
    p["head"] = head
    return p


def flatten_stage(params: dict, spec: Spec, depth: int, s: int) -> np.ndarray:
    per = spec.layers // depth
    lay, n = stage_layout(spec, s * per, (s + 1) * per, s == 0, s == depth - 1)
    flat = np.zeros(n, np.float32)
    for name, (off, shape) in lay.items():
        flat[off:off + int(np.prod(shape))] = params[name].reshape(-1)
    return flat


def unflatten_stage(flat: np.ndarray, spec: Spec, depth: int, s: int) -> dict:
    per = spec.layers // depth
    lay, _ = stage_layout(spec, s * per, (s + 1) * per, s == 0, s == depth - 1)
    return {name: flat[off:off + int(np.prod(shape))].reshape(shape) for name, (off, shape) in lay.items()}


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def loss_fn(P: dict, ids: torch.Tensor, targets: torch.Tensor, spec: Spec) -> torch.Tensor:
    """Mean cross-entropy of one microbatch (torch, differentiable w.r.t. P)."""
    b, s, h, nh = spec.batch, spec.seq, spec.hidden, spec.heads
    T = b * s
    x = P["tok"][ids] + P["pos"][torch.arange(T) % s]
    for l in range(spec.layers):
        xn = torch.nn.functional.layer_norm(x, (h,), P[f"{l}.ln1g"], P[f"{l}.ln1b"], 1e-5)
        qkv = xn @ P[f"{l}.wqkv"].T + P[f"{l}.bqkv"]
        q, k, v = qkv.split(h, dim=1)
        hd = h // nh
        q = q.reshape(b, s, nh, hd).transpose(1, 2)
        k = k.reshape(b, s, nh, hd).transpose(1, 2)
        v = v.reshape(b, s, nh, hd).transpose(1, 2)
        sc = (q @ k.transpose(-1, -2)) * hd ** -0.5
        if spec.causal:
            mask = torch.triu(torch.ones(s, s, dtype=torch.bool), 1)
            sc = sc.masked_fill(mask, float("-inf"))
        o = (torch.softmax(sc, -1) @ v).transpose(1, 2).reshape(T, h)
        x1 = o @ P[f"{l}.wo"].T + P[f"{l}.bo"] + x
        xn2 = torch.nn.functional.layer_norm(x1, (h,), P[f"{l}.ln2g"], P[f"{l}.ln2b"], 1e-5)
        a = _gelu(xn2 @ P[f"{l}.w1"].T + P[f"{l}.b1"])
        x = a @ P[f"{l}.w2"].T + P[f"{l}.b2"] + x1
    rows = torch.as_tensor(head_positions(spec))
    xf = torch.nn.functional.layer_norm(x[rows], (h,), P["lnfg"], P["lnfb"], 1e-5)
    logits = (xf @ P["head"].T)[:, :spec.vocab]
    return torch.nn.functional.cross_entropy(logits, targets)


def train(params: dict, spec: Spec, ids: np.ndarray, targets: np.ndarray, lr: float, beta: float,
          m: int, T: int, delayed: bool = True, dtype=torch.float64, optimizer: str = "sgd",
          beta2: float = 0.999, eps: float = 1e-8):
    """reference_loop (semantics.cpp:167-184) on the transformer loss.

    optimizer "sgd": the reference's momentum SGD with dampening (semantics.cpp:153-165);
    "adam": Adam with bias correction (beta1 = beta) -- the paper's optimizer
    (PAPER.md:605-607), not in the reference: unpinned, restated here.

    ids: [m*T, b*seq] int, targets: [m*T, R] int.  Returns (trajectory of param
    dicts W^(0..T), per-microbatch losses measured at the weights each batch's
    gradient was taken at)."""
    W = {k: torch.tensor(v, dtype=dtype) for k, v in params.items()}
    traj = [{k: v.clone() for k, v in W.items()}]
    vel = {k: torch.zeros_like(v) for k, v in W.items()}
    vel2 = {k: torch.zeros_like(v) for k, v in W.items()}
    losses = []
    for t in range(1, T + 1):
        ev = traj[max(t - 2, 0) if delayed else t - 1]
        grads = {k: torch.zeros_like(v) for k, v in W.items()}
        for j in range(m):
            kk = (t - 1) * m + j
            P = {k: v.clone().requires_grad_(True) for k, v in ev.items()}
            loss = loss_fn(P, torch.as_tensor(ids[kk], dtype=torch.long),
                           torch.as_tensor(targets[kk], dtype=torch.long), spec)
            loss.backward()
            losses.append(float(loss.detach()))
            for k in grads:
                if P[k].grad is not None:
                    grads[k] += P[k].grad
        for k in W:
            g = grads[k] / m
            vel[k] = beta * vel[k] + (1.0 - beta) * g
            if optimizer == "adam":
                vel2[k] = beta2 * vel2[k] + (1.0 - beta2) * g * g
                mh = vel[k] / (1.0 - beta ** t)
                vh = vel2[k] / (1.0 - beta2 ** t)
                W[k] = W[k] - lr * mh / (torch.sqrt(vh) + eps)
            else:
                W[k] = W[k] + (-lr) * vel[k]
        traj.append({k: v.clone() for k, v in W.items()})
    return traj, np.array(losses)
