#!/usr/bin/env python3
"""2BW training throughput (samples/s) on B200s -- the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

One "step" is one 2BW batch (m microbatches of b sequences, every stage's
weight update included) of the workload named by --config with synthetic token
data.  Default: configs[3], the GPT-style 2.2B decoder (48 layers, hidden 1920,
seq 512, V 51200) at the reference planner's per-GPU choice for 8 x B200 (w 8,
d 1, b 16, m 4) -- the largest configuration one GPU runs (the other configs are
--config choices and parity-test shapes).  Under torchrun (N > 1) every rank drives one GPU; rank 0 prints
ONE JSON line.  By default N GPUs run N data-parallel replicas of the whole
pipeline (width N); --depth D > 1 under torchrun runs one pipeline stage per
process (gpu = stage * width + replica, width = N / D) with CUDA-IPC stage
hand-offs; on one GPU --depth D runs D stages on one device.

Timing: W warm-up batches, then K batches timed on the device with the
engine's CUDA events at each stage's weight updates (steady state, as
simulator.cpp:298-309 defines it), barrier + synchronize on both sides, max
over ranks and stages.  `value` counts every replica's sequences with the
token batches already resident in HBM.  `e2e` is a second timed pass through
the C-ABI in which each step's token ids / targets are copied host->device
from pinned memory and its losses device->host inside the timed region.  `roofline` comes from a second, profiled pass of the same workload
(per-launch CUDA events around every stage kernel).  `cpu_baseline` times the
reference's own pipelined_execute (oracle/_ref/ref_tool, built from
/root/reference) on the linear-chain analog of the config on this host, and
`same_config` times that same linear chain on the GPU through the production
path (P2BW_MODEL_LINEAR_BF16: the tcgen05 GEMMs, fused optimizer and streams the
transformer uses), so one ratio in the line compares like with like.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import shutil
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MEASURED = ROOT / "MEASURED_PEAKS.json"
REF_TOOL = ROOT / "oracle" / "_ref" / "ref_tool"

# BASELINE.json configs; dims the reference leaves open are recorded here.
CONFIGS = {
    # configs[0]: the CPU reference's default-sized run, as a transformer
    "small": dict(layers=4, hidden=256, heads=4, seq=128, vocab=8192, causal=True, head_rows=0,
                  b=4, m=4, depth=2),
    # configs[1]: BERT-base-sized encoder; MLM head on 15% (77 of 512) positions
    "bert-base": dict(layers=12, hidden=768, heads=12, seq=512, vocab=30522, causal=False, head_rows=77,
                      b=16, m=4, depth=1),
    # configs[2]: BERT-large, depth 8 x m 8 on 8 GPUs (per-GPU work: 3 layers)
    "bert-large": dict(layers=24, hidden=1024, heads=16, seq=512, vocab=30522, causal=False, head_rows=77,
                       b=8, m=8, depth=1),
    # configs[3]: GPT-style 2.2B decoder (h 1920, 48 layers, 30 x 64 heads, V 51200) at the
    # planner's per-GPU choice on 8 x B200 (w 8, d 1, b 16, m 4:
    # profiles/r1_plan_gpt2.2b_8xb200_2bw.txt, planner.cpp:45-99)
    "gpt-2.2b": dict(layers=48, hidden=1920, heads=30, seq=512, vocab=51200, causal=True, head_rows=0,
                     b=16, m=4, depth=1),
    # configs[3] at SURVEY a14's recommended head layout: 15 heads of 128 (the D = 128
    # tcgen05 attention); same GEMMs and FLOPs
    "gpt-2.2b-h128": dict(layers=48, hidden=1920, heads=15, seq=512, vocab=51200, causal=True, head_rows=0,
                          b=16, m=4, depth=1),
    # configs[4]: 24-layer GPT (h 1024, V 51200, causal LM head on every position)
    "gpt-24": dict(layers=24, hidden=1024, heads=16, seq=512, vocab=51200, causal=True, head_rows=0,
                   b=8, m=4, depth=1),
}


def flops_per_sample(c) -> float:
    """L*3*(24 s h^2 + 4 s^2 h) + 6 s h V_head (head tokens only)."""
    L, h, s = c["layers"], c["hidden"], c["seq"]
    attn = 4 * s * s * h * (0.5 if c["causal"] else 1.0)
    head_tokens = c["head_rows"] or s
    return L * 3 * (24 * s * h * h + attn) + 6 * head_tokens * h * c["vocab"]


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_rank{gpu}.csv"
        if shutil.which("nvidia-smi") is None:
            return
        self.path.parent.mkdir(exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.f = open(self.path, "w")
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                      "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        rows = [r.split(",") for r in self.path.read_text().strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


def peaks():
    if MEASURED.exists():
        d = json.loads(MEASURED.read_text())
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# ---- CPU baseline: the reference's own trainer on the linear-chain analog --------------

REF_GFLOPS_EST = 2.5  # the reference's fp64 loops on one core (SURVEY §6 probe: 2.0-3.0)


def cpu_layers(c, target_s: float = 8.0) -> int:
    """Layers of the linear-chain analog one CPU sample runs: all of them when that takes
    <= target_s on one core, else fewer (the time is linear in the layer count; the
    result is scaled to the full depth)."""
    per_layer = 6.0 * c["hidden"] ** 2 * c["seq"] / (REF_GFLOPS_EST * 1e9)
    return max(1, min(c["layers"], int(target_s / per_layer)))


def cpu_sample(c, procs: int = 1, microbatches: int = 1) -> dict:
    """The reference's own 2BW trainer on the config's linear-chain analog: ToyModel::make(
    dim=h, layers=L', cols=seq) -- one sequence (seq columns) per microbatch -- 2BW, d 1,
    timed by oracle/_ref/ref_tool (the reference compiled from its own sources), L' <= L
    layers (cpu_layers) with the time scaled by L / L'."""
    dim, L, cols = c["hidden"], c["layers"], c["seq"]
    Ls = cpu_layers(c)
    if REF_TOOL.exists():
        cmd = [str(REF_TOOL), "time", str(dim), str(Ls), str(cols), str(microbatches), "1", "1", "1"]
        t0 = time.time()
        ps = [subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True) for _ in range(procs)]
        outs = [json.loads(p.communicate()[0]) for p in ps]
        wall = time.time() - t0
        sec = max(o["seconds"] for o in outs)
        kind = "reference"
    else:  # the oracle port (numpy restatement of semantics.cpp), single process
        from oracle import pipesim_oracle as O
        model = O.ToyModel.make(dim, Ls, cols, microbatches, 1)
        t0 = time.time()
        O.pipelined_execute(model, 0.01, 0.9, microbatches, 1, O.TWOBW, 1)
        sec = wall = time.time() - t0
        procs, kind = 1, "port"
    full = sec * L / Ls
    samples = procs * microbatches  # one sequence (seq columns) per microbatch
    return {"value": samples / full, "unit": "samples/s", "cores": procs, "kind": kind,
            "sample": f"pipelined_execute(ToyModel dim={dim} layers={Ls} cols={cols}, 2BW d=1, "
                      f"m={microbatches} T=1) x {procs} process(es), fp64, {sec:.2f} s"
                      + (f", scaled x{L}/{Ls} to the config's {L} layers" if Ls < L else ""),
            "seconds": full, "wall_s": wall}


def run_reference(args, c):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    procs = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(c, procs=procs, microbatches=1)
        if i >= args.warmup:
            times.append(r["seconds"])
    sec = max(times) if times else 0.0
    total = sum(times)
    value = args.steps * procs / total if total else 0.0
    line = {"metric": "2BW training samples/sec", "value": value, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (splitmix64 ToyModel, reference generator)", "impl": "reference",
            "config": {"workload": f"{args.config}: linear-chain analog (reference has no transformer)",
                       "dim": c["hidden"], "layers": c["layers"], "cols_per_microbatch": c["seq"],
                       "policy": "2bw", "depth": 1},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": procs, "kind": r["kind"],
                             "sample": r["sample"]},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- same-config leg: the reference's own workload on the production GPU path ----------

# The linear-chain ToyModel the reference trains (semantics.cpp:85-109) at BERT-base's
# width: dim 768, 12 layers, one 512-column sequence per sample.  (Deeper / wider analogs
# leave the bf16 range: ToyModel's I + 0.2 U grows activations ~sqrt(1 + dim / 300) per
# layer, 2.7x at dim 1920 -- 1e20 after 48 layers -- so the gradients overflow.)
SAME = dict(hidden=768, layers=12, seq=512, b=16, m=4)


def linear_same_config(steps: int, warm: int, cpu: bool) -> dict:
    """2BW samples/s of the SAME workload on both sides: the reference's pipelined_execute
    on the host cores (ref_tool, one process per core, fp64) and the engine's bf16
    production path (P2BW_MODEL_LINEAR_BF16: tcgen05 GEMMs, fused optimizer, the
    transformer's streams) with ToyModel::make's data generated on the device."""
    from paper_2006_09503_b200 import _lib
    from paper_2006_09503_b200 import pipesim as P
    c = SAME
    cols = c["seq"] * c["b"]
    eng = P.Engine(model_kind=P.MODEL_LINEAR_BF16, policy=P.PipelinePolicy.TwoBW, depth=1, microbatches=c["m"],
                   microbatch_size=cols, layers=c["layers"], dim=c["hidden"], learning_rate=1e-7, momentum=0.9,
                   seed=12345)
    eng.init_weights()
    eng.make_toy_data(1, 2 * c["m"])  # the data ring (2 batches), resident
    eng.sync()
    total = warm + steps + 1
    l0 = _lib.lib().p2bw_launch_count()
    eng.begin(total)
    for t in range(1, total + 1):
        eng.issue(t)
    eng.finish()
    eng.sync()
    launches = _lib.lib().p2bw_launch_count() - l0
    ms = eng.update_elapsed_ms(0, warm, warm + steps)
    losses = eng.losses(1, 2 * c["m"])
    eng.close()
    gpu = c["b"] * c["m"] * steps / (ms / 1e3)
    flops = 3 * 2 * c["hidden"] ** 2 * c["seq"] * c["layers"]  # per sample: fwd + dgrad + wgrad
    out = {"workload": f"ToyModel linear chain (semantics.cpp:85-109): dim {c['hidden']}, {c['layers']} layers, "
                       f"{c['seq']} columns per sample, 2BW d=1, m={c['m']}",
           "gpu": {"value": round(gpu, 1), "unit": "samples/s", "dtype": "bf16 (fp32 master)",
                   "microbatch": f"{c['b']} samples = {cols} columns", "ms_per_step": round(ms / steps, 3),
                   "tflops": round(gpu * flops / 1e12, 1), "gpu_launches_per_step": round(launches / total, 1),
                   "losses_finite": bool(np.all(np.isfinite(losses)))},
           "parity": "tests/test_linear_bf16_gpu.py: trajectories vs the reference's pipelined_execute"}
    if cpu:
        procs = os.cpu_count() or 1
        r = cpu_sample(dict(c, vocab=0, heads=0), procs=procs, microbatches=1)
        out["cpu_reference"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        out["gpu_over_cpu"] = round(gpu / r["value"], 1)
    return out


# ---- our engine ---------------------------------------------------------------------

def run_ours(args, c):
    import torch
    from paper_2006_09503_b200 import _lib
    from paper_2006_09503_b200 import pipesim as P
    from paper_2006_09503_b200 import synthetic as S

    rank, world, local = dist_env()
    ngpu = torch.cuda.device_count()
    shared = world > ngpu  # more ranks than GPUs: ranks share devices (a plumbing check, not a scaling number)
    local = local % ngpu
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if shared:  # NCCL refuses two ranks on one device; the engine's data path does not use it
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2006_09503_b200 import dist as D

    depth = args.depth or (c["depth"] if world == 1 else 1)
    pipelined = world > 1 and depth > 1  # one stage per process, CUDA-IPC hand-offs
    if pipelined:
        stage, _, width = D.grid(world, rank, depth)
        local_stages = (stage, 1)
    else:
        width, local_stages = world, None
    spec = S.TransformerSpec(layers=c["layers"], hidden=c["hidden"], heads=c["heads"], seq=c["seq"], vocab=c["vocab"],
                   batch=c["b"], causal=c["causal"], head_rows=c["head_rows"])
    m, steps, warm = c["m"], args.steps, args.warmup
    total_batches = warm + steps + 1
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                   microbatch_size=c["b"], layers=c["layers"], hidden=c["hidden"], heads=c["heads"],
                   seq_len=c["seq"], vocab=c["vocab"], causal=int(c["causal"]), head_rows=c["head_rows"],
                   learning_rate=1e-3, momentum=0.9, seed=1234,  # replicas start identical
                   local_stages=local_stages, recompute=args.recompute, optimizer=args.optimizer)
    eng.init_weights()
    my_stages = [s for s in range(depth) if eng.is_local(s)]
    has_loss = eng.is_local(depth - 1)
    if pipelined:
        D.connect_pipeline(eng, depth)
    transport = None
    if width > 1:  # one node: fused all-reduce + update over CUDA-IPC peer memory; else NCCL
        transport = D.join_replicas(eng, depth, pipelined=pipelined)

    # synthetic token batches in pinned host memory (one batch = m microbatches)
    T, R = c["b"] * c["seq"], c["b"] * (c["head_rows"] or c["seq"])
    pool = 4
    replica = D.grid(world, rank, depth)[1] if pipelined else rank
    ids_np, tg_np = S.token_batch(spec, m * pool, 99 + replica)
    ids = torch.from_numpy(ids_np).pin_memory()
    tgs = torch.from_numpy(tg_np).pin_memory()
    loss_host = torch.zeros(total_batches * m, dtype=torch.float32).pin_memory()
    h2d_bytes = m * (T + R) * 4
    d2h_bytes = m * 4

    def set_batch(t):  # batch t (1-based) -> microbatches (t-1)m+1 .. tm
        j = (t - 1) % pool
        _lib.check(_lib.lib().p2bw_engine_set_data(
            eng.h, C.c_void_p(ids[j * m].data_ptr()), C.c_void_p(tgs[j * m].data_ptr()), (t - 1) * m + 1, m))

    def fetch_loss(t):
        if has_loss:
            _lib.check(_lib.lib().p2bw_engine_losses_async(eng.h, (t - 1) * m + 1, m,
                                                           C.c_void_p(loss_host[(t - 1) * m].data_ptr())))

    def one_pass(n_batches, io=True, profile=False):
        """io=True: per-step H2D of the batch and D2H of its losses (the e2e pass);
        io=False: the token ring already holds the batches (resident inputs)."""
        eng.begin(n_batches)
        if io:
            set_batch(1)
        for t in range(1, n_batches + 1):
            if io and t + 1 <= n_batches:
                set_batch(t + 1)
            if profile and t == warm + 1:
                _lib.lib().p2bw_profile_enable(1)
            if profile and t == warm + 1 + steps:
                _lib.lib().p2bw_profile_enable(0)
            eng.issue(t)
            if io:
                fetch_loss(t)
        eng.finish()

    def steady_ms():
        """K steady-state batches: update events of every local stage, max over ranks."""
        ms = max(eng.update_elapsed_ms(s, warm, warm + steps) for s in my_stages)
        if world > 1:
            ms = D.max_over_ranks(ms)
        return ms

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # token ring filled once (2 batches = the ring's capacity); the resident pass reuses it
    set_batch(1)
    set_batch(2)
    eng.sync()

    # ---- timed pass 1: inputs resident in HBM -> value ----
    barrier()
    clocks = Clocks(local)
    launches0 = _lib.lib().p2bw_launch_count()
    one_pass(total_batches, io=False)
    eng.sync()
    launches = _lib.lib().p2bw_launch_count() - launches0
    clk = clocks.stop()
    ms = steady_ms()
    barrier()

    # ---- timed pass 2: end to end through the C-ABI with host buffers -> e2e ----
    wall0 = time.time()
    one_pass(total_batches, io=True)
    eng.sync()
    wall = time.time() - wall0
    ms_e2e = steady_ms()
    barrier()
    losses = loss_host.numpy()[: total_batches * m]

    samples = width * c["b"] * m * steps
    value = samples / (ms / 1e3)
    value_e2e = samples / (ms_e2e / 1e3)
    fps = flops_per_sample(c)
    peak, peak_sus, hbm, peak_kind = peaks()

    # ---- profiled pass (same workload, every rank runs it, rank 0 records) ----
    classes = []
    one_pass(total_batches, io=False, profile=(rank == 0))
    eng.sync()
    if rank == 0:
        arr = (KernelClass * 64)()
        n = C.c_int()
        _lib.check(_lib.lib().p2bw_profile_collect(arr, 64, C.byref(n)))
        classes = [dict(name=arr[i].name.decode(), launches=arr[i].launches, ms=arr[i].ms, flops=arr[i].flops,
                        bytes=arr[i].bytes) for i in range(min(n.value, 64))]
    barrier()
    graph = None
    if world == 1 and not args.no_graph:
        # CUDA-graph form of the same training (p2bw_engine_run_schedule_graph): whole runs
        # of nb batches captured once and launched 3 times -- the host's op interpretation
        # and kernel launches are out of the picture.  Each run starts with its pipeline fill
        # (d > 1), so it is quoted beside `value`, not as it.
        try:
            nb = 2 if depth == 1 else 8
            gms = eng.run_schedule_graph(nb, 3)
            graph = {"value": round(c["b"] * m * nb / (gms / 1e3), 2), "unit": "samples/s",
                     "batches_per_launch": nb, "launches": 3, "ms_per_batch": round(gms / nb, 3),
                     "note": "whole runs (fill / drain included at d > 1) captured into one CUDA graph across "
                             "the stage, forward, update and weight-gradient streams, device-timed per launch"}
        except Exception as e:  # noqa: BLE001 -- an extra measurement
            graph = {"error": f"{type(e).__name__}: {e}"[:300]}
    eng.close()

    pipe = None
    if world > 1 and not pipelined and not args.no_pipeline_leg:
        try:
            pipe = pipeline_leg(args, c, world, rank, local)
        except Exception as e:  # noqa: BLE001 -- the data-parallel line stands on its own
            pipe = {"error": f"{type(e).__name__}: {e}"[:300]}

    if rank != 0:
        return 0
    tot_ms = sum(k["ms"] for k in classes) or 1.0
    gk = [k for k in classes if k["name"].startswith("gemm")]
    gemm = {"name": "gemm", **{f: sum(k[f] for k in gk) for f in ("launches", "ms", "flops", "bytes")}} if gk else None
    roofline = None
    if gemm and gemm["ms"] > 0:
        achieved = gemm["flops"] / (gemm["ms"] / 1e3) / 1e12
        traffic = None
        prof_json = ROOT / "profiles" / "ncu_gemm_dram_bytes.json"
        if prof_json.exists():
            traffic = json.loads(prof_json.read_text()).get(args.config)
        roofline = {"bound": "tensor", "kernel": "gemm_tc_kernel (tcgen05, all GEMM launches of a step)",
                    # the GEMMs run inside a long step (the sw_power_cap regime), so the
                    # denominator is the sustained bf16 figure; the burst one is kept beside it
                    "achieved": round(achieved, 1), "peak": peak_sus, "unit": "TFLOP/s",
                    "frac": round(achieved / peak_sus, 4),
                    "peak_kind": f"{peak_kind} sustained bf16 (MEASURED_PEAKS.json: back-to-back 8192^3 for 4 s)",
                    "peak_burst": peak, "frac_of_burst": round(achieved / peak, 4),
                    "traffic": traffic,
                    "flops_per_launch": gemm["flops"] / max(gemm["launches"], 1),
                    "avg_launch_us": 1e3 * gemm["ms"] / max(gemm["launches"], 1),
                    "share_of_kernel_time": round(gemm["ms"] / tot_ms, 4),
                    "measured_over": f"{steps} profiled steps after the timed pass (per-launch CUDA events; "
                                     "weight gradients serialised on the stage stream so each launch is timed alone)"}
    breakdown = {k["name"]: {"share": round(k["ms"] / tot_ms, 4), "launches": k["launches"],
                             "tflops": round(k["flops"] / (k["ms"] / 1e3) / 1e12, 1) if k["flops"] else None,
                             "gbs": round(k["bytes"] / (k["ms"] / 1e3) / 1e9, 1) if k["bytes"] else None}
                 for k in classes}
    mfu = value * fps / (world * peak * 1e12)
    par = f"2bw d={depth} w={width}"
    if pipelined:
        par += " (one stage per process, CUDA-IPC stage hand-offs over NVLink)"
    if width > 1:
        par += (" (AllReduce fused into WeightUpdate: reduce-scatter + optimizer + all-gather of the new version "
                "over CUDA-IPC peer memory, one kernel per replica)" if transport == "ipc" else
                " (NCCL all-reduce of the coalesced gradient at each AllReduce op)")

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = cpu_sample(c, procs=1, microbatches=1)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
    same = None
    if world == 1 and not args.no_same_config:
        same = linear_same_config(steps, warm, cpu=not args.no_cpu_baseline)

    line = {
        "metric": "2BW training samples/sec", "value": round(value, 2), "unit": "samples/s", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": round(ms / steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens: ids uniform over [0, V) from splitmix64 (SURVEY 8(d)); random-init weights",
        "config": {"workload": args.config, "layers": c["layers"], "hidden": c["hidden"], "heads": c["heads"],
                   "seq_len": c["seq"], "vocab": c["vocab"], "causal": c["causal"],
                   "head_rows_per_seq": c["head_rows"] or c["seq"], "microbatch_size": c["b"],
                   "microbatches_m": m, "global_batch": width * c["b"] * m,
                   "parallelism": par, "inputs": "value: token batches resident in HBM; e2e: per-step host copies",
                   "policy": "2bw", "recompute": bool(args.recompute), "optimizer": args.optimizer,
                   "head": ("causal LM: next-token targets at every position, untied LM head" if c["causal"] else
                            f"masked LM, simplified: {c['head_rows']} evenly spaced positions per sequence (the same "
                            "in every sequence) replaced by [MASK] (id V-1) with the original ids as targets; no "
                            "80/10/10 split, untied LM head"),
                   "reproducibility": "not bit-reproducible run to run: the token-embedding gradient uses vector "
                                      "atomics and attention dQ a TMA reduce-add (fp32 summation order only)",
                   "l2": "working set (activations >> 126 MB L2) exceeds L2 every step"},
        "e2e": {"value": round(value_e2e, 2), "unit": "samples/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes, "wall_s": round(wall, 3),
                "note": "second timed pass: per-step pinned H2D of ids/targets and D2H of losses "
                        "through the C-ABI (p2bw_engine_set_data / p2bw_engine_losses_async), "
                        "device-timed between weight-update events like `value`"},
        "gpu_launches": int(launches * steps / total_batches),
        "gpu_launches_per_step": round(launches / total_batches, 1),
        "mfu": round(mfu, 4), "flops_per_sample": fps,
        "roofline": roofline, "kernel_breakdown": breakdown,
        "kernel_ms_per_step": round(tot_ms / steps, 3) if classes else None,
        "cpu_baseline": cpu, "same_config": same, "clocks": clk,
        "loss_first_last": [float(losses[0]), float(losses[-1])] if has_loss else None,
    }
    if shared:
        line["shared_gpus"] = f"{world} ranks on {ngpu} GPU(s): a plumbing check, not a scaling measurement"
    if pipe is not None:
        line["pipeline"] = pipe
    if graph is not None:
        line["cuda_graph"] = graph
    print(json.dumps(line), flush=True)
    return 0


def flop_profile(c) -> str:
    """The config's blocks as a reference profile document (profile.cpp:162-193) with
    times proportional to their algorithmic FLOPs: block 0 also carries
    the embedding, the last block the LM head and its loss -- what partition_balanced
    needs to move layers off the last stage (the head of the GPT configs costs ~2 layers)."""
    L, h, s, V = c["layers"], c["hidden"], c["seq"], c["vocab"]
    layer = 3 * (24 * s * h * h + 4 * s * s * h * (0.5 if c["causal"] else 1.0))
    head = 6 * (c["head_rows"] or s) * h * V
    unit = 1e12  # "ms" per FLOP scale; only ratios matter
    blocks = []
    for i in range(L):
        f = layer + (head if i == L - 1 else 0.0)
        blocks.append({"fwd_ms": {str(c["b"]): f / 3 / unit}, "bwd_ms": {str(c["b"]): 2 * f / 3 / unit},
                       "weight_bytes": 1.0, "act_total_bytes": {str(c["b"]): 1.0},
                       "act_input_bytes": {str(c["b"]): 1.0}, "act_boundary_bytes": {str(c["b"]): 2.0}})
    return json.dumps({"model": "flops", "blocks": blocks})


def pipeline_leg(args, c, world: int, rank: int, local: int) -> dict:
    """N > 1, data-parallel default run: the same workload ALSO as one pipeline of depth N
    (one stage per process, width 1; CUDA-IPC stage hand-offs over NVLink) -- the
    configs' stated pipelines (C2 d 4, C3 d 8) next to the planner's data-parallel choice.
    Reports samples/s (update events, max over ranks), the per-stage bubble fraction of a
    traced run (stage idle time inside the steady window: schedule bubble + exposed
    hand-offs, simulator.cpp:311-329 on measured times), the bytes each boundary moves per
    microbatch and a device-to-device copy of that size between two of this node's GPUs."""
    from paper_2006_09503_b200 import dist as D
    from paper_2006_09503_b200 import pipesim as P

    depth = world
    if c["layers"] < depth:
        return {"skipped": f"{c['layers']} layers cannot fill {depth} stages"}
    m = max(c["m"], depth)  # 2BW needs m >= d (schedule.cpp:153-156)
    stage, _, _ = D.grid(world, rank, depth)
    out = {"workload": f"{args.config} as one 2BW pipeline: depth {depth}, width 1, m {m}, b {c['b']}",
           "unit": "samples/s", "boundary_bytes_per_microbatch_per_direction": c["b"] * c["seq"] * c["hidden"] * 2,
           "handoff": "producer kernel -> local staging slot -> copy stream into the neighbour's ring (CUDA IPC) "
                      "-> sequence flag (cuStreamWaitValue32 on the consumer's stream)"}
    split = P.stage_layers_from_bounds(P.partition_balanced(flop_profile(c), depth, c["b"]))
    runs = ([("equal", None)] if c["layers"] % depth == 0 else []) + [("balanced", split)]
    for name, layers in runs:
        r = _pipeline_run(args, c, depth, m, stage, layers)
        out[name] = dict(r, stage_layers=layers or [c["layers"] // depth] * depth)
    out["value"] = max(out[name]["value"] for name, _ in runs)
    out["d2d_copy_of_one_boundary"] = _link_probe(rank, out["boundary_bytes_per_microbatch_per_direction"])
    return out


def _pipeline_run(args, c, depth, m, stage, layers) -> dict:
    import torch
    from paper_2006_09503_b200 import dist as D
    from paper_2006_09503_b200 import pipesim as P
    from paper_2006_09503_b200 import synthetic as S
    spec = S.TransformerSpec(layers=c["layers"], hidden=c["hidden"], heads=c["heads"], seq=c["seq"], vocab=c["vocab"],
                             batch=c["b"], causal=c["causal"], head_rows=c["head_rows"])
    eng = P.Engine(model_kind=P.MODEL_TRANSFORMER, policy=P.PipelinePolicy.TwoBW, depth=depth, microbatches=m,
                   microbatch_size=c["b"], layers=c["layers"], hidden=c["hidden"], heads=c["heads"],
                   seq_len=c["seq"], vocab=c["vocab"], causal=int(c["causal"]), head_rows=c["head_rows"],
                   learning_rate=1e-3, momentum=0.9, seed=1234, local_stages=(stage, 1), stage_layers=layers)
    try:
        eng.init_weights()
        D.connect_pipeline(eng, depth)
        ids, tg = S.token_batch(spec, 2 * m, 99)
        eng.set_data(ids, tg, 1, 2 * m)  # the ring (2 batches) stays resident
        steps, warm = args.steps, args.warmup
        total = warm + steps + 1
        torch.distributed.barrier()
        torch.cuda.synchronize()
        eng.begin(total)
        eng.issue(total)
        eng.finish()
        eng.sync()
        ms = D.max_over_ranks(eng.update_elapsed_ms(stage, warm, warm + steps))
        value = c["b"] * m * steps / (ms / 1e3)
        # one traced run: per-stage busy / idle inside the steady window
        eng.set_trace(True)
        eng.begin(4)
        eng.issue(4)
        eng.finish()
        eng.sync()
        rep = eng.trace_report()
        bubble = D.max_over_ranks(float(rep.get("bubble_fraction", 0.0)))
        torch.distributed.barrier()
    finally:
        eng.close()
    return {"value": round(value, 2), "ms_per_step": round(ms / steps, 3),
            "stage_bubble_fraction_max": round(bubble, 4)}


def _link_probe(rank: int, boundary: int):
    """Device-to-device copy of one boundary tensor between two of this node's GPUs."""
    import torch
    link = None
    if rank == 0 and torch.cuda.device_count() > 1:  # one hand-off's bytes between two GPUs
        a = torch.empty(boundary // 2, dtype=torch.bfloat16, device="cuda:0")
        b = torch.empty_like(a, device="cuda:1")
        for _ in range(3):
            b.copy_(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        link = {"bytes": boundary, "us": round(us, 2), "gbs": round(boundary / us / 1e3, 1),
                "peak_gbs_per_direction": 900.0}
    return link


class KernelClass(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_longlong), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="gpt-2.2b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-same-config", action="store_true",
                    help="skip the same-workload leg (reference linear chain on CPU and on the bf16 GPU path)")
    ap.add_argument("--optimizer", default="sgd", choices=["sgd", "adam"],
                    help="WeightUpdate optimizer: the reference's momentum SGD (default) or Adam")
    ap.add_argument("--recompute", action="store_true",
                    help="activation recomputation (the planner's r flag): stash stage inputs only")
    ap.add_argument("--no-graph", action="store_true",
                    help="skip the CUDA-graph measurement of the same training (N = 1)")
    ap.add_argument("--no-pipeline-leg", action="store_true",
                    help="N > 1: skip the depth-N pipeline measured beside the data-parallel line")
    ap.add_argument("--depth", type=int, default=0,
                    help="pipeline depth (default: the config's on 1 GPU, 1 = data parallel on N GPUs)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, c)
    return run_ours(args, c)


if __name__ == "__main__":
    sys.exit(main())
