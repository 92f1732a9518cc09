"""Attention fwd / bwd: ours (p2bw_kernel_attention_*) against torch SDPA (cuDNN / flash
backends, library code: the bar, not the product) on the configs' shapes.  CUDA events,
warm, per-launch average.  Diagnostic only; prints one JSON line per shape."""
import ctypes as C
import json
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

SHAPES = [("gpt-2.2b", 16, 512, 30, 1, 64), ("bert-base", 16, 512, 12, 0, 64), ("bert-large", 8, 512, 16, 0, 64),
          ("gpt-24", 8, 512, 16, 1, 64), ("gpt-2.2b-h128", 16, 512, 15, 1, 128), ("bert-base-h128", 16, 512, 6, 0, 128)]
if len(sys.argv) > 1:
    SHAPES = [s for s in SHAPES if s[0] in sys.argv[1:]]


def keep_async_pool():
    """The C-ABI backward allocates its scratch per call with cudaMallocAsync; keep the
    default pool's memory mapped between calls so the timing is the kernels'."""
    try:
        from cuda.bindings import driver as dr
        from cuda.bindings import runtime as rt
        err, pool = rt.cudaDeviceGetDefaultMemPool(torch.cuda.current_device())
        rt.cudaMemPoolSetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold,
                                   dr.cuuint64_t(2**64 - 1))
    except Exception as e:  # noqa: BLE001
        print(f"# mempool threshold not set: {e}", file=sys.stderr)


keep_async_pool()


def timeit(fn, iters=20, reps=5):
    """Best of `reps` averages (the C-ABI backward allocates its scratch per call with
    cudaMallocAsync, whose pool occasionally re-maps memory inside a window)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters * 1e3)  # us
    return best


for name, b, s, nh, causal, hd in SHAPES:
    h = nh * hd
    qkv = (torch.randn(b * s, 3 * h, device="cuda") * 0.5).to(torch.bfloat16)
    o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b * nh * s, device="cuda")
    do = torch.randn(b * s, h, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(b * nh * s, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    fwd = lambda: call("p2bw_kernel_attention_fwd_hd", P(qkv), P(o), P(lse), b, s, nh, hd, causal, st)  # noqa: E731
    bwd = lambda: call("p2bw_kernel_attention_bwd_hd", P(qkv), P(o), P(do), P(lse), P(dqkv), P(delta), b, s,  # noqa: E731
                       nh, hd, causal, st)
    fl = 4.0 * b * nh * hd * s * s * (0.5 if causal else 1.0)
    t_f = timeit(fwd)
    t_b = timeit(bwd)
    q, k, v = [t.view(b, s, nh, hd).transpose(1, 2) for t in qkv.split(h, dim=1)]
    q, k, v = [t.contiguous().requires_grad_() for t in (q, k, v)]
    res = {"shape": name, "b": b, "s": s, "heads": nh, "head_dim": hd, "causal": causal,
           "ours_fwd_us": round(t_f, 1), "ours_fwd_tflops": round(fl / t_f / 1e6, 1),
           "ours_bwd_us": round(t_b, 1), "ours_bwd_tflops": round(2 * fl / t_b / 1e6, 1)}
    for be_name, be in [("cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION),
                        ("flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION)]:
        try:
            with torch.nn.attention.sdpa_kernel(be):
                out = F.scaled_dot_product_attention(q, k, v, is_causal=bool(causal))
                g = torch.randn_like(out)
                tf = timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=bool(causal)))
                tfb = timeit(lambda: torch.autograd.grad(F.scaled_dot_product_attention(q, k, v, is_causal=bool(causal)),
                                                         (q, k, v), g)) - tf
            res[f"{be_name}_fwd_tflops"] = round(fl / tf / 1e6, 1)
            res[f"{be_name}_bwd_tflops"] = round(2 * fl / tfb / 1e6, 1)
        except Exception as e:  # noqa: BLE001
            res[f"{be_name}"] = str(e)[:80]
    print(json.dumps(res), flush=True)
