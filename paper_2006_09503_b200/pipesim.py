"""Python mirror of the reference pipesim API for the pipelined training path,
bound to libp2bw.so's C-ABI (include/p2bw.h).

Same names and argument meaning as the reference C++ API
(/root/reference/proj/core/include/pipesim/*.hpp); errors raise
``PipesimError`` carrying the reference's pipesim::Error message text.

  weight_version_2bw, required_versions, generate_schedule,
  serialize_programs, parse_programs, parse_policy    schedule.hpp:18-64
  plan, plan_text, partition_equal                     planner.hpp:40-41, profile.hpp:76
  ToyModel, TrainerConfig, pipelined_execute,
  reference_vanilla, reference_2bw                     semantics.hpp:31-74 (run on the GPU)
  Engine                                               the stage executor itself
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib
from ._lib import P2bwError as PipesimError  # noqa: F401


class PipelinePolicy(IntEnum):
    """schedule.hpp:10-16"""
    NoPipelining = 0
    GPipe = 1
    PipeDream1F1B = 2
    PipeDreamFlush = 3
    TwoBW = 4


class OpKind(IntEnum):
    """schedule.hpp:21-32"""
    Forward = 0
    Backward = 1
    Recompute = 2
    WeightUpdate = 3
    FlushBarrier = 4
    ActivationSend = 5
    ActivationRecv = 6
    GradSend = 7
    GradRecv = 8
    AllReduce = 9


kLatestVersion = -1


@dataclass(frozen=True)
class ScheduledOp:
    """schedule.hpp:40-46"""
    kind: OpKind
    microbatch: int = 0
    weight_version: int = 0


@dataclass
class StageProgram:
    """schedule.hpp:48-51"""
    stage: int
    ops: list[ScheduledOp] = field(default_factory=list)


def _call(name, *args):
    _lib.check(getattr(_lib.lib(), name)(*args))


def _take_string(ptr: C.c_char_p) -> str:
    try:
        return C.cast(ptr, C.c_char_p).value.decode()
    finally:
        _lib.lib().p2bw_free(ptr)


def weight_version_2bw(k: int, m: int) -> int:
    out = C.c_int()
    _call("p2bw_weight_version_2bw", k, m, C.byref(out))
    return out.value


def required_versions(policy: PipelinePolicy, d: int, m: int) -> int:
    out = C.c_int()
    _call("p2bw_required_versions", int(policy), d, m, C.byref(out))
    return out.value


def to_string(policy: PipelinePolicy) -> str:
    name = C.c_char_p()
    _call("p2bw_policy_name", int(policy), C.byref(name))
    return name.value.decode()


def parse_policy(name: str) -> PipelinePolicy:
    out = C.c_int()
    _call("p2bw_policy_parse", name.encode(), C.byref(out))
    return PipelinePolicy(out.value)


class _Schedule:
    """Owns a p2bw_schedule handle."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            _lib.lib().p2bw_schedule_destroy(self.h)
            self.h = None

    def programs(self) -> list[StageProgram]:
        n = C.c_int()
        _call("p2bw_schedule_num_stages", self.h, C.byref(n))
        out = []
        for s in range(n.value):
            ops = C.POINTER(_lib.Op)()
            cnt = C.c_size_t()
            _call("p2bw_schedule_ops", self.h, s, C.byref(ops), C.byref(cnt))
            out.append(StageProgram(s, [ScheduledOp(OpKind(ops[i].kind), ops[i].microbatch,
                                                    ops[i].weight_version) for i in range(cnt.value)]))
        return out

    def text(self) -> str:
        p = C.c_void_p()
        _call("p2bw_schedule_serialize", self.h, C.byref(p))
        return _take_string(p)


def _generate(policy, d, m, num_batches) -> _Schedule:
    h = C.c_void_p()
    _call("p2bw_schedule_generate", int(policy), d, m, num_batches, C.byref(h))
    return _Schedule(h)


def generate_schedule(policy: PipelinePolicy, d: int, m: int, num_batches: int) -> list[StageProgram]:
    return _generate(policy, d, m, num_batches).programs()


def schedule_text(policy: PipelinePolicy, d: int, m: int, num_batches: int) -> str:
    """serialize_programs(generate_schedule(...)) in one call."""
    return _generate(policy, d, m, num_batches).text()


def parse_programs(text: str) -> list[StageProgram]:
    h = C.c_void_p()
    _call("p2bw_schedule_parse", text.encode(), C.byref(h))
    return _Schedule(h).programs()


def serialize_programs(programs: list[StageProgram]) -> str:
    """Text form (schedule.cpp:177-195), rendered by the library from a parsed copy."""
    lines = []
    for p in programs:
        for op in p.ops:
            line = f"stage={p.stage} op={_OP_TEXT[op.kind]}"
            if op.kind in (OpKind.Forward, OpKind.Backward, OpKind.Recompute):
                ver = "latest" if op.weight_version == kLatestVersion else str(op.weight_version)
                line += f" mb={op.microbatch} ver={ver}"
            lines.append(line + "\n")
    text = "".join(lines)
    h = C.c_void_p()
    _call("p2bw_schedule_parse", text.encode(), C.byref(h))
    return _Schedule(h).text()


_OP_TEXT = {OpKind.Forward: "forward", OpKind.Backward: "backward", OpKind.Recompute: "recompute",
            OpKind.WeightUpdate: "update", OpKind.FlushBarrier: "flush",
            OpKind.ActivationSend: "act_send", OpKind.ActivationRecv: "act_recv",
            OpKind.GradSend: "grad_send", OpKind.GradRecv: "grad_recv", OpKind.AllReduce: "allreduce"}


def plan(model_json: str, cluster_json: str, max_batch: int,
         policy: PipelinePolicy = PipelinePolicy.TwoBW) -> dict:
    """plan() rendered through plan_to_json (planner.cpp:160-186), parsed."""
    p = C.c_void_p()
    _call("p2bw_plan", model_json.encode(), cluster_json.encode(), C.c_longlong(max_batch),
          int(policy), 0, C.byref(p))
    return json.loads(_take_string(p))


def plan_text(model_json: str, cluster_json: str, max_batch: int,
              policy: PipelinePolicy = PipelinePolicy.TwoBW) -> str:
    p = C.c_void_p()
    _call("p2bw_plan", model_json.encode(), cluster_json.encode(), C.c_longlong(max_batch),
          int(policy), 1, C.byref(p))
    return _take_string(p)


def partition_equal(model_json: str, d: int) -> list[dict]:
    p = C.c_void_p()
    _call("p2bw_partition_equal", model_json.encode(), d, C.byref(p))
    return json.loads(_take_string(p))


def partition_balanced(model_json: str, d: int, b: int) -> list[int]:
    """B200 extension: the d + 1 block boundaries of the contiguous split whose slowest
    stage (fwd + bwd at microbatch size b) is fastest (pipesim::partition_balanced)."""
    p = C.c_void_p()
    _call("p2bw_partition_balanced", model_json.encode(), d, b, C.byref(p))
    return json.loads(_take_string(p))


def stage_layers_from_bounds(bounds: list[int]) -> list[int]:
    return [hi - lo for lo, hi in zip(bounds[:-1], bounds[1:])]


# ---- the stage executor ---------------------------------------------------------------

class Desc(C.Structure):
    _fields_ = [("model_kind", C.c_int), ("policy", C.c_int), ("depth", C.c_int), ("width", C.c_int),
                ("microbatches", C.c_int), ("microbatch_size", C.c_int), ("layers", C.c_int),
                ("dim", C.c_int), ("hidden", C.c_int), ("heads", C.c_int), ("seq_len", C.c_int),
                ("vocab", C.c_int), ("causal", C.c_int), ("head_rows", C.c_int),
                ("learning_rate", C.c_double), ("momentum", C.c_double), ("seed", C.c_ulonglong),
                ("devices", C.POINTER(C.c_int)), ("first_local_stage", C.c_int), ("local_stages", C.c_int),
                ("recompute", C.c_int), ("optimizer", C.c_int), ("beta2", C.c_double), ("eps", C.c_double),
                ("loop_scaling", C.c_int), ("stage_layers", C.POINTER(C.c_int))]


STAGE_BLOB_BYTES = 128  # P2BW_STAGE_BLOB_BYTES
REPLICA_BLOB_BYTES = 1024  # P2BW_REPLICA_BLOB_BYTES


def profile_blocks(*, layers: int, hidden: int, heads: int, seq_len: int, vocab: int, causal: int = 0,
                   head_rows: int = 0, microbatch_sizes=(1, 2, 4, 8), warmup: int = 2, iters: int = 5,
                   name: str = "p2bw-transformer", seed: int = 1) -> str:
    """B200 block profiler (p2bw_profile_blocks): the transformer's per-block fwd / bwd
    times, weight and activation bytes measured on the current GPU, as the reference's
    profile document (profile.cpp:162-193) -- the input of plan() / partition_equal()."""
    d = Desc(MODEL_TRANSFORMER, int(PipelinePolicy.TwoBW), 1, 1, 1, 1, layers, 0, hidden, heads, seq_len,
             vocab, causal, head_rows, 0.0, 0.0, seed, None, 0, 0, 0, OPT_MOMENTUM_SGD, 0.999, 1e-8, 0)
    sizes = (C.c_int * len(microbatch_sizes))(*microbatch_sizes)
    p = C.c_void_p()
    _call("p2bw_profile_blocks", C.byref(d), sizes, len(microbatch_sizes), warmup, iters, name.encode(),
          C.byref(p))
    return _take_string(p)


class Counters(C.Structure):
    _fields_ = [("version_consistent", C.c_int), ("max_versions_held", C.c_int),
                ("ops_executed", C.c_longlong), ("last_run_ms", C.c_double)]


MODEL_LINEAR_F64 = 0
MODEL_TRANSFORMER = 1
MODEL_LINEAR_BF16 = 2  # the ToyModel on the production bf16 / tcgen05 path
OPT_MOMENTUM_SGD = 0  # P2BW_OPT_*
OPT_ADAM = 1


class Engine:
    """The B200 stage executor (one CUDA stream per stage).

    ``local_stages=None`` runs every stage of the pipeline in this process;
    ``local_stages=(first, count)`` runs only those, the others living in other
    processes that are connected through :meth:`export_stage` / :meth:`connect_stage`
    (see :func:`paper_2006_09503_b200.dist.connect_pipeline`)."""

    def __init__(self, *, model_kind: int, policy: PipelinePolicy, depth: int, microbatches: int,
                 microbatch_size: int, layers: int, dim: int = 0, hidden: int = 0, heads: int = 0,
                 seq_len: int = 0, vocab: int = 0, causal: int = 0, head_rows: int = 0,
                 learning_rate: float = 0.0, momentum: float = 0.0, seed: int = 0,
                 devices: list[int] | None = None, local_stages: tuple[int, int] | None = None,
                 recompute: bool = False, optimizer: str = "sgd", beta2: float = 0.999, eps: float = 1e-8,
                 loop_scaling: bool = False, stage_layers: list[int] | None = None):
        self._devs = (C.c_int * depth)(*devices) if devices else None
        self._split = (C.c_int * depth)(*stage_layers) if stage_layers else None
        first, count = local_stages if local_stages is not None else (0, 0)
        d = Desc(model_kind, int(policy), depth, 1, microbatches, microbatch_size, layers, dim, hidden,
                 heads, seq_len, vocab, causal, head_rows, learning_rate, momentum, seed,
                 C.cast(self._devs, C.POINTER(C.c_int)) if self._devs else None, first, count, int(recompute),
                 {"sgd": OPT_MOMENTUM_SGD, "adam": OPT_ADAM}[optimizer], beta2, eps, int(loop_scaling),
                 C.cast(self._split, C.POINTER(C.c_int)) if self._split else None)
        self.h = C.c_void_p()
        _call("p2bw_engine_create", C.byref(d), C.byref(self.h))
        self.depth = depth

    def close(self):
        if getattr(self, "h", None):
            if _lib is not None:  # None during interpreter shutdown: the process teardown frees it
                _lib.lib().p2bw_engine_destroy(self.h)
            self.h = None

    __del__ = close

    def stage_weight_bytes(self, s: int) -> int:
        n = C.c_size_t()
        _call("p2bw_engine_stage_weight_bytes", self.h, s, C.byref(n))
        return n.value

    def load_stage_weights(self, s: int, host: np.ndarray):
        host = np.ascontiguousarray(host)
        _call("p2bw_engine_load_stage_weights", self.h, s, host.ctypes.data_as(C.c_void_p),
              C.c_size_t(host.nbytes))

    def init_weights(self):
        _call("p2bw_engine_init_weights", self.h)

    def set_data(self, inputs: np.ndarray | None, targets: np.ndarray | None, first_mb: int, count: int):
        ip = np.ascontiguousarray(inputs) if inputs is not None else None
        tp = np.ascontiguousarray(targets) if targets is not None else None
        _call("p2bw_engine_set_data", self.h, ip.ctypes.data_as(C.c_void_p) if ip is not None else None,
              tp.ctypes.data_as(C.c_void_p) if tp is not None else None, first_mb, count)

    def make_toy_data(self, first_mb: int, count: int):
        """Device-side ToyModel::make dataset for microbatches [first_mb, first_mb+count)
        (bf16 linear chain; seed from the engine's description)."""
        _call("p2bw_engine_make_toy_data", self.h, first_mb, count)

    def run_schedule(self, num_batches: int, snapshots: bool = False):
        _call("p2bw_engine_run_schedule", self.h, num_batches, int(snapshots))

    def run_schedule_graph(self, num_batches: int, launches: int = 1) -> float:
        """CUDA-graph run (p2bw_engine_run_schedule_graph): device ms per launch."""
        ms = C.c_double()
        _call("p2bw_engine_run_schedule_graph", self.h, num_batches, launches, C.byref(ms))
        return ms.value

    def run(self, programs: list[StageProgram], snapshots: bool = False):
        arrs = [(_lib.Op * max(len(p.ops), 1))(*[_lib.Op(int(o.kind), o.microbatch, o.weight_version)
                                                 for o in p.ops]) for p in programs]
        ptrs = (C.POINTER(_lib.Op) * len(arrs))(*[C.cast(a, C.POINTER(_lib.Op)) for a in arrs])
        ns = (C.c_size_t * len(arrs))(*[len(p.ops) for p in programs])
        _call("p2bw_engine_run", self.h, ptrs, ns, int(snapshots))

    def begin(self, num_batches: int):
        _call("p2bw_engine_begin", self.h, num_batches)

    def issue(self, upto_batch: int):
        _call("p2bw_engine_issue", self.h, upto_batch)

    def finish(self):
        _call("p2bw_engine_finish", self.h)

    def update_elapsed_ms(self, stage: int, u0: int, u1: int) -> float:
        out = C.c_double()
        _call("p2bw_engine_update_elapsed_ms", self.h, stage, u0, u1, C.byref(out))
        return out.value

    def sync(self):
        _call("p2bw_engine_sync", self.h)

    def set_trace(self, on: bool = True):
        """Bracket every issued op with CUDA events (takes effect at the next begin / run)."""
        _call("p2bw_engine_set_trace", self.h, int(on))

    def trace_report(self) -> dict:
        """The last traced run as the reference's SimReport document (measured times)."""
        p = C.c_void_p()
        _call("p2bw_engine_trace_report", self.h, C.byref(p))
        return json.loads(_take_string(p))

    def is_local(self, stage: int) -> bool:
        out = C.c_int()
        _call("p2bw_engine_is_local", self.h, stage, C.byref(out))
        return bool(out.value)

    def export_stage(self, stage: int) -> bytes:
        buf = (C.c_char * STAGE_BLOB_BYTES)()
        _call("p2bw_engine_export_stage", self.h, stage, buf, C.c_size_t(STAGE_BLOB_BYTES))
        return bytes(buf)

    def export_replica(self, stage: int) -> bytes:
        """CUDA-IPC description of this replica's stage for a peer-memory replica group."""
        buf = (C.c_char * REPLICA_BLOB_BYTES)()
        _call("p2bw_engine_export_replica", self.h, stage, buf, C.c_size_t(REPLICA_BLOB_BYTES))
        return bytes(buf)

    def join_replicas_ipc(self, stage: int, blobs: list[bytes], rank: int):
        """Stage `stage` joins the group of its len(blobs) replicas (blobs in replica order):
        the AllReduce is then fused into WeightUpdate over peer memory (no NCCL)."""
        if any(len(b) != REPLICA_BLOB_BYTES for b in blobs):
            raise ValueError("replica blobs must be %d bytes" % REPLICA_BLOB_BYTES)
        buf = (C.c_char * (REPLICA_BLOB_BYTES * len(blobs))).from_buffer_copy(b"".join(blobs))
        _call("p2bw_engine_join_replicas_ipc", self.h, stage, buf, len(blobs), rank)

    def connect_stage(self, blob: bytes):
        if len(blob) != STAGE_BLOB_BYTES:
            raise ValueError("stage blob must be %d bytes" % STAGE_BLOB_BYTES)
        buf = (C.c_char * STAGE_BLOB_BYTES).from_buffer_copy(blob)
        _call("p2bw_engine_connect_stage", self.h, buf, C.c_size_t(STAGE_BLOB_BYTES))

    def counters(self) -> Counters:
        c = Counters()
        _call("p2bw_engine_counters", self.h, C.byref(c))
        return c

    def snapshot(self, s: int, update_index: int, dtype=np.float64) -> np.ndarray:
        n = self.stage_weight_bytes(s)
        out = np.empty(n // np.dtype(dtype).itemsize, dtype=dtype)
        _call("p2bw_engine_read_snapshot", self.h, s, update_index, out.ctypes.data_as(C.c_void_p),
              C.c_size_t(n))
        return out

    def read_version(self, s: int, version: int, dtype=np.float64) -> np.ndarray:
        n = self.stage_weight_bytes(s)
        out = np.empty(n // np.dtype(dtype).itemsize, dtype=dtype)
        _call("p2bw_engine_read_version", self.h, s, version, out.ctypes.data_as(C.c_void_p),
              C.c_size_t(n))
        return out

    def read_master(self, s: int, dtype=np.float32) -> np.ndarray:
        """fp32 master weights in the model's public layout (transformer: fp32 flat vector;
        linear chains: fp64 column-major matrices, pass dtype=np.float64)."""
        n = self.stage_weight_bytes(s)
        out = np.empty(n // np.dtype(dtype).itemsize, dtype=dtype)
        _call("p2bw_engine_read_master", self.h, s, out.ctypes.data_as(C.c_void_p), C.c_size_t(n))
        return out

    def losses(self, first_mb: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        _call("p2bw_engine_losses", self.h, first_mb, count, out.ctypes.data_as(C.c_void_p))
        return out


# ---- semantics.hpp mirror: the linear-chain ToyModel on the GPU ---------------------

@dataclass
class TrainerConfig:
    """semantics.hpp:45-52"""
    learning_rate: float = 0.0
    momentum: float = 0.0
    microbatches_per_batch: int = 1
    num_batches: int = 1


@dataclass
class ToyModel:
    """semantics.hpp:31-43; matrices are numpy arrays indexed (row, col)."""
    dim: int
    init_weights: list
    dataset: list  # [(x, y)]

    @property
    def num_layers(self):
        return len(self.init_weights)

    @property
    def microbatch_samples(self):
        return self.dataset[0][0].shape[1]


@dataclass
class PipelinedResult:
    """semantics.hpp:65-69"""
    trajectory: list
    version_consistent: bool
    max_versions_held: int
    losses: np.ndarray | None = None


def pipelined_execute(model: ToyModel, cfg: TrainerConfig, policy: PipelinePolicy, depth: int,
                      devices: list[int] | None = None, with_losses: bool = False,
                      precision: str = "fp64", loop_scaling: bool = False) -> PipelinedResult:
    """semantics.hpp:73-74, executed by the B200 stage executor.

    precision "fp64": the fp64 linear stages, bit-identical to the reference;
    "bf16": the production path (bf16 tcgen05 GEMMs, fp32 master / momentum / gradient,
    the fused optimizer, the transformer's streams) -- trajectories are the fp32 master
    weights after every update, within a bf16 tolerance of the reference.
    loop_scaling (fp64 only): reference_loop's per-microbatch 1/m gradient scaling
    (semantics.cpp:145) instead of pipelined_execute's sum / count (:338-340)."""
    L = model.num_layers
    if L % depth:
        raise PipesimError(f"block count {L} not divisible by depth {depth}")
    m, T = cfg.microbatches_per_batch, cfg.num_batches
    if len(model.dataset) < m * T:
        raise PipesimError("toy dataset has too few microbatches for the requested run")
    per = L // depth
    kind = {"fp64": MODEL_LINEAR_F64, "bf16": MODEL_LINEAR_BF16}[precision]
    eng = Engine(model_kind=kind, policy=policy, depth=depth, microbatches=m,
                 microbatch_size=model.microbatch_samples, layers=L, dim=model.dim,
                 learning_rate=cfg.learning_rate, momentum=cfg.momentum, devices=devices,
                 loop_scaling=loop_scaling)
    try:
        for s in range(depth):
            eng.load_stage_weights(s, np.concatenate(
                [w.flatten(order="F") for w in model.init_weights[s * per:(s + 1) * per]]))
        xs = np.concatenate([x.flatten(order="F") for x, _ in model.dataset[:m * T]])
        ys = np.concatenate([y.flatten(order="F") for _, y in model.dataset[:m * T]])
        eng.set_data(xs, ys, 1, m * T)
        eng.run_schedule(T, snapshots=True)
        eng.sync()
        c = eng.counters()
        upb = m if policy == PipelinePolicy.PipeDream1F1B else 1
        dim = model.dim
        traj = [[w.copy() for w in model.init_weights]]
        for t in range(1, T + 1):
            ws = []
            for s in range(depth):
                flat = eng.snapshot(s, t * upb)
                ws += [flat[i * dim * dim:(i + 1) * dim * dim].reshape((dim, dim), order="F")
                       for i in range(per)]
            traj.append(ws)
        losses = eng.losses(1, m * T) if with_losses else None
        return PipelinedResult(traj, bool(c.version_consistent), c.max_versions_held, losses)
    finally:
        eng.close()


def reference_vanilla(model: ToyModel, cfg: TrainerConfig):
    """Vanilla SGD == one-stage GPipe on the engine with reference_loop's 1/m scaling
    (semantics.cpp:145, 188-190): bit-identical to the reference for every m."""
    return pipelined_execute(model, cfg, PipelinePolicy.GPipe, 1, loop_scaling=True).trajectory


def reference_2bw(model: ToyModel, cfg: TrainerConfig):
    """Delay-1 SGD == one-stage 2BW on the engine with reference_loop's 1/m scaling
    (semantics.cpp:145, 192-194)."""
    return pipelined_execute(model, cfg, PipelinePolicy.TwoBW, 1, loop_scaling=True).trajectory
