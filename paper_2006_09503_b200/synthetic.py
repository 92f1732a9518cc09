"""Synthetic workloads of the bench and tests, from the reference's splitmix64.

splitmix64 is the generator of the reference's ToyModel (semantics.cpp:64-75):
state += 0x9e3779b97f4a7c15, then two xor-shift-multiply rounds; a double in
[-0.5, 0.5) is (z >> 11) * 2^-53 - 0.5.  Draw i (1-based) of a stream seeded
with s is therefore mix(s + i * gamma), which vectorises.

  splitmix64_u01(seed, n, skip)   draws skip+1 .. skip+n as doubles in [0, 1)
  toy_model(dim, L, b, nmb, seed) ToyModel::make (semantics.cpp:85-109), bit-exact
  TransformerSpec, token_batch    the transformer configs' token ids and targets
                                  (ids uniform over [0, V) from
                                  splitmix64(seed))
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix64_bits(seed: int, n: int, skip: int = 0) -> np.ndarray:
    """Raw 64-bit draws skip+1 .. skip+n of splitmix64(seed) (semantics.cpp:66-72)."""
    with np.errstate(over="ignore"):
        i = np.arange(skip + 1, skip + n + 1, dtype=np.uint64)
        return _mix(np.uint64(seed & ((1 << 64) - 1)) + i * _GAMMA)


def splitmix64_u01(seed: int, n: int, skip: int = 0) -> np.ndarray:
    return (splitmix64_bits(seed, n, skip) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _colmajor(u: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """random_mat's fill order (semantics.cpp:77-81): Mat::data is column-major."""
    return u.reshape(cols, rows).T


def _matmul_ref_order(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """matmul (semantics.cpp:9-19): c(i, j) += a(i, k) b(k, j) with k ascending, one
    rounded multiply and one rounded add per term (no FMA on the reference's x86-64
    build), so y = A x matches the reference bit for bit."""
    c = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        c += np.outer(a[:, k], b[k, :])
    return c


def toy_model(dim: int, layers: int, b: int, nmb: int, seed: int, exact: bool = True):
    """ToyModel::make (semantics.cpp:85-109) -> (weights [L x (dim, dim)], dataset
    [(x, y)]): W_l = I + 0.2 U, hidden map A = I + 0.3 U, x = U (dim x b), y = A x,
    drawn in that order from one splitmix64 stream.  exact=False forms y = A x with a
    BLAS product (last-bit differences in y only; for the bf16-tolerance runs)."""
    if min(dim, layers, b, nmb) < 1:
        raise ValueError("toy model dimensions must be >= 1")
    u = splitmix64_u01(seed, (layers + 1) * dim * dim + nmb * dim * b) - 0.5
    p = 0
    ws = []
    for _ in range(layers):
        w = _colmajor(u[p:p + dim * dim], dim, dim) * 0.2
        p += dim * dim
        w[np.diag_indices(dim)] += 1.0
        ws.append(np.ascontiguousarray(w))
    a = _colmajor(u[p:p + dim * dim], dim, dim) * 0.3
    p += dim * dim
    a[np.diag_indices(dim)] += 1.0
    data = []
    for _ in range(nmb):
        x = np.ascontiguousarray(_colmajor(u[p:p + dim * b], dim, b))
        p += dim * b
        data.append((x, _matmul_ref_order(a, x) if exact else a @ x))
    return ws, data


@dataclass
class TransformerSpec:
    """One transformer configuration (model_transformer.cu) and its batch shape."""
    layers: int
    hidden: int
    heads: int
    seq: int
    vocab: int
    batch: int            # sequences per microbatch (b)
    causal: bool = True
    head_rows: int = 0    # LM-head rows per sequence (0: every position)

    @property
    def vp(self):
        return (self.vocab + 127) // 128 * 128

    @property
    def rows_per_seq(self):
        return self.head_rows if self.head_rows > 0 else self.seq


def head_positions(spec: TransformerSpec) -> np.ndarray:
    """Rows the LM head reads (model_transformer.cu alloc_all): every position, or
    `head_rows` evenly spaced positions per sequence (the same for every sequence)."""
    r = spec.rows_per_seq
    per_seq = np.array([(j * spec.seq) // r for j in range(r)], dtype=np.int64)
    return np.concatenate([bb * spec.seq + per_seq for bb in range(spec.batch)])


def token_batch(spec: TransformerSpec, count: int, seed: int):
    """`count` microbatches of token ids [count, b*seq] and targets [count, rows].

    Ids are uniform over [0, V) from splitmix64(seed): id = floor(u * V).
      GPT (causal): targets are the next token at every head row (the last position of a
      sequence predicts the sequence's first token: a fixed-length synthetic stream).
      BERT (encoder, masked LM): the head rows are the masked positions -- the target is
      the original token and the input there is replaced by the [MASK] id V - 1.
      Simplifications against BERT pre-training, stated in the bench line: the masked
      positions are the same evenly spaced 15% of every sequence (not re-drawn per
      sequence), always [MASK] (no 80/10/10 split), and the LM head is untied."""
    T = spec.batch * spec.seq
    u = splitmix64_u01(seed, count * T)
    ids = np.minimum((u * spec.vocab).astype(np.int64), spec.vocab - 1).astype(np.int32).reshape(count, T)
    rows = head_positions(spec)
    if spec.causal:
        nxt = np.roll(ids.reshape(count, spec.batch, spec.seq), -1, axis=2).reshape(count, T)
        tg = nxt[:, rows]
    else:
        tg = ids[:, rows].copy()
        ids[:, rows] = spec.vocab - 1
    return np.ascontiguousarray(ids), np.ascontiguousarray(tg.astype(np.int32))
