"""Config 5: 2BW against GPipe and PipeDream-Flush on d B200s,
predicted from B200-measured blocks.

The stage op times come from p2bw_profile_blocks (the engine's own Forward /
Backward kernels, one block at a time, on a B200; run with --profile on a GPU box,
or pass a saved profile).  partition_equal() splits the 24-layer GPT into d stages
and the programs of generate_schedule() are replayed with the reference
simulator's dependency rules (simulator.cpp:195-290, restated below):

  * a stage runs its program in order, one compute op at a time;
  * Forward(s, k) starts after Forward(s-1, k) + the activation transfer, and after
    the update that produced its weight version (1F1B: the latest);
  * Backward(s, k) starts after Backward(s+1, k) + the gradient transfer;
  * AllReduce is zero at width 1; WeightUpdate / FlushBarrier take no compute time.

Throughput and bubble use simulate()'s steady-state window (simulator.cpp:298-329).
Beside them: the closed-form pipeline bubble, the stage imbalance (slowest stage's
per-microbatch F + B over the mean) and the exposed time (steady batch time minus
the slowest stage's m (F + B): flush bubble + transfers on the critical path).

With --balanced, 2BW is replayed twice per (d, m): on partition_equal's split and on
partition_balanced's (the B200 extension: the contiguous split whose slowest stage is
fastest -- the last stage also carries the 51200-way LM head), to show what the
imbalance term becomes.

  python scripts/c5_replay.py --profile out_profile.json      # on a GPU box
  python scripts/c5_replay.py profile.json [out.json]         # anywhere
  python scripts/c5_replay.py --balanced profile.json [out.json]
"""
import json
import sys

sys.path.insert(0, ".")
from paper_2006_09503_b200 import pipesim as P  # noqa: E402

B = 4
NVLINK_BPS = 900e9  # per direction, NVSwitch
T_BATCHES = 8


def replay(programs, stages, policy, b, xfer_bps):
    d = len(programs)
    key = str(b)
    fwd = [st["fwd_time"][key] for st in stages]
    bwd = [st["bwd_time"][key] for st in stages]
    xfer = [st["act_output_bytes"][key] / xfer_bps if s < d - 1 else 0.0 for s, st in enumerate(stages)]
    fwd_end = [dict() for _ in range(d)]
    bwd_end = [dict() for _ in range(d)]
    free = [0.0] * d
    updates = [[] for _ in range(d)]
    busy = [[] for _ in range(d)]
    ptr = [0] * d
    total = sum(len(p.ops) for p in programs)
    done = 0
    while done < total:
        progress = False
        for s in range(d):
            ops = programs[s].ops
            while ptr[s] < len(ops):
                op = ops[ptr[s]]
                k = op.microbatch
                if op.kind == P.OpKind.Forward:
                    if s > 0 and k not in fwd_end[s - 1]:
                        break
                    v = op.weight_version if op.weight_version >= 0 else len(updates[s])
                    if v > len(updates[s]):
                        break
                    t0 = free[s]
                    if s > 0:
                        t0 = max(t0, fwd_end[s - 1][k] + xfer[s - 1])
                    if v >= 1:
                        t0 = max(t0, updates[s][v - 1])
                    t1 = t0 + fwd[s]
                    fwd_end[s][k] = t1
                    free[s] = t1
                    busy[s].append((t0, t1))
                elif op.kind == P.OpKind.Backward:
                    if s < d - 1 and k not in bwd_end[s + 1]:
                        break
                    t0 = free[s]
                    if s < d - 1:
                        t0 = max(t0, bwd_end[s + 1][k] + xfer[s])
                    t1 = t0 + bwd[s]
                    bwd_end[s][k] = t1
                    free[s] = t1
                    busy[s].append((t0, t1))
                elif op.kind == P.OpKind.WeightUpdate:
                    updates[s].append(free[s])
                # AllReduce (width 1) and FlushBarrier: no time
                ptr[s] += 1
                done += 1
                progress = True
        if not progress:
            raise RuntimeError("dependency deadlock")
    m = max(op.microbatch for op in programs[0].ops) // T_BATCHES
    upb = m if policy == P.PipelinePolicy.PipeDream1F1B else 1

    def upd(s, t):
        return updates[s][t * upb - 1]

    steady = (upd(d - 1, T_BATCHES - 1) - upd(d - 1, 1)) / (T_BATCHES - 2)
    win = bz = 0.0
    for s in range(d):
        w0, w1 = upd(s, 1), upd(s, T_BATCHES - 1)
        win += w1 - w0
        bz += sum(max(0.0, min(e, w1) - max(a, w0)) for a, e in busy[s])
    stage_mb = [f + g for f, g in zip(fwd, bwd)]
    compute_bound = m * max(stage_mb)
    return {"throughput": m * b / steady, "steady_batch_ms": steady * 1e3,
            "bubble_fraction": 1.0 - bz / win if win > 0 else 0.0,
            "imbalance": max(stage_mb) / (sum(stage_mb) / d),
            "exposed_fraction": max(0.0, steady - compute_bound) / steady}


def stages_from_bounds(prof: str, bounds: list) -> list:
    """partition_equal's stage records (seconds, bytes) for an arbitrary contiguous split."""
    blocks = json.loads(prof)["blocks"]
    out = []
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        st = {"fwd_time": {}, "bwd_time": {}, "act_output_bytes": {}}
        tail = blocks[hi - 1]
        for key in tail["fwd_ms"]:
            st["fwd_time"][key] = sum(blocks[i]["fwd_ms"][key] for i in range(lo, hi)) * 1e-3
            st["bwd_time"][key] = sum(blocks[i]["bwd_ms"][key] for i in range(lo, hi)) * 1e-3
            st["act_output_bytes"][key] = tail["act_boundary_bytes"][key] - tail["act_input_bytes"][key]
        out.append(st)
    return out


def breakdown(prof: str, policy, d: int, m: int, b: int = B, T: int = T_BATCHES, bounds=None) -> dict:
    """Steady batch time split into additive parts (all from the simulator's rules):
      ideal            m * mean_s(F_s + B_s)       -- perfectly balanced, no bubble, free links
      imbalance        m * max_s(F_s + B_s) - ideal -- the slowest stage sets the pace
      schedule bubble  steady(free links) - m * max_s(F_s + B_s)   -- fill / drain / flush
      exposed transfer steady(NVLink) - steady(free links)          -- hand-offs on the critical path"""
    stages = P.partition_equal(prof, d) if bounds is None else stages_from_bounds(prof, bounds)
    progs = P.generate_schedule(policy, d, m, T)
    link = replay(progs, stages, policy, b, NVLINK_BPS)
    free = replay(progs, stages, policy, b, 1e18)
    key = str(b)
    stage_mb = [st["fwd_time"][key] + st["bwd_time"][key] for st in stages]
    ideal = m * sum(stage_mb) / d * 1e3
    slow = m * max(stage_mb) * 1e3
    return {"steady_batch_ms": link["steady_batch_ms"], "ideal_ms": ideal, "imbalance_ms": slow - ideal,
            "schedule_bubble_ms": free["steady_batch_ms"] - slow,
            "exposed_transfer_ms": link["steady_batch_ms"] - free["steady_batch_ms"],
            "throughput": link["throughput"], "bubble_fraction": link["bubble_fraction"]}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--profile" in sys.argv:
        prof = P.profile_blocks(layers=24, hidden=1024, heads=16, seq_len=512, vocab=51200, causal=1, head_rows=0,
                                microbatch_sizes=(B,), warmup=2, iters=5, name="gpt-24")
        with open(args[0], "w") as f:
            f.write(prof)
        return
    prof = open(args[0]).read()
    if "--balanced" in sys.argv:
        rows = []
        pol = P.PipelinePolicy.TwoBW
        for d in (2, 4, 8):
            bal = P.partition_balanced(prof, d, B)
            for m in (d, 2 * d):
                for name, bounds in (("equal", None), ("balanced", bal)):
                    bd = breakdown(prof, pol, d, m, bounds=bounds)
                    st = bd["steady_batch_ms"]
                    row = {"partition": name, "stage_layers": None if bounds is None else P.stage_layers_from_bounds(bounds),
                           "d": d, "m": m, "b": B, "samples_per_s": round(bd["throughput"], 1),
                           "steady_batch_ms": round(st, 3), "bubble_fraction": round(bd["bubble_fraction"], 4),
                           "frac_imbalance": round(bd["imbalance_ms"] / st, 4),
                           "frac_schedule_bubble": round(bd["schedule_bubble_ms"] / st, 4),
                           "frac_exposed_transfer": round(bd["exposed_transfer_ms"] / st, 4)}
                    rows.append(row)
                    print(json.dumps(row))
        if len(args) > 1:
            with open(args[1], "w") as f:
                json.dump({"workload": "gpt-24, b 4, 2BW on d B200s: partition_equal vs partition_balanced "
                                       "(B200-measured blocks, simulator rules)", "rows": rows}, f, indent=1)
        return
    pols = (P.PipelinePolicy.TwoBW, P.PipelinePolicy.GPipe, P.PipelinePolicy.PipeDreamFlush)
    rows = []
    for d in (2, 4, 8):
        stages = P.partition_equal(prof, d)
        for m in (4, 8, 16, 32):
            if m < d:
                continue
            for pol in pols:
                r = replay(P.generate_schedule(pol, d, m, T_BATCHES), stages, pol, B, NVLINK_BPS)
                bd = breakdown(prof, pol, d, m)
                closed = 0.0 if pol == P.PipelinePolicy.TwoBW else (d - 1) / (m + d - 1)
                st = bd["steady_batch_ms"]
                row = {"policy": P.to_string(pol), "d": d, "m": m, "b": B,
                       "samples_per_s": round(r["throughput"], 1),
                       "steady_batch_ms": round(r["steady_batch_ms"], 3),
                       "bubble_fraction": round(r["bubble_fraction"], 4), "closed_form_bubble": round(closed, 4),
                       "imbalance": round(r["imbalance"], 4), "exposed_fraction": round(r["exposed_fraction"], 4),
                       # additive split of the steady batch time (fractions of it)
                       "frac_imbalance": round(bd["imbalance_ms"] / st, 4),
                       "frac_schedule_bubble": round(bd["schedule_bubble_ms"] / st, 4),
                       "frac_exposed_transfer": round(bd["exposed_transfer_ms"] / st, 4)}
                rows.append(row)
                print(json.dumps(row))
    if len(args) > 1:
        with open(args[1], "w") as f:
            json.dump({"workload": "gpt-24 (L 24, h 1024, 16 heads, s 512, V 51200), b 4, d B200s over NVLink "
                                   "(900 GB/s per direction), B200-measured blocks, simulator rules",
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
