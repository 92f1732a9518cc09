"""Phase timeline of one tcgen05 GEMM launch (diagnostic): p2bw_debug_gemm_timing's
per-CTA %globaltimer marks, as medians / maxima over CTAs relative to the earliest
CTA entry.  Shapes: the stage GEMMs at several token counts."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import GemmEpilogue, call  # noqa: E402

NAMES = ["entry", "setup", "last load", "1st stage", "last MMA", "1st acc", "epi done", "exit"]
cases = [("qkv", 2048, 2304, 768), ("qkv", 8192, 2304, 768), ("proj", 8192, 768, 768), ("fc2", 8192, 768, 3072)]
for name, T, n, k in cases:
    a = torch.randn(T * k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n * k, device="cuda").to(torch.bfloat16)
    d = torch.empty(T * n, device="cuda", dtype=torch.bfloat16)
    epi = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    run = lambda: call("p2bw_kernel_gemm_bf16", C.c_void_p(a.data_ptr()), k, 0, C.c_void_p(b.data_ptr()), k, 0,  # noqa
                       T, n, k, C.byref(epi), s)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    dbg = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    call("p2bw_debug_gemm_timing", C.c_void_p(dbg.data_ptr()))
    run()  # previous launch of the same kernel just before: warm
    run()
    torch.cuda.synchronize()
    call("p2bw_debug_gemm_timing", None)
    m = dbg.view(148, 8).cpu().double()
    m = m[m[:, 0] > 0]
    t0 = m[:, 0].min()
    rel = (m - t0) / 1e3
    print(f"{name} T={T} n={n} k={k}: {us:.1f} us/launch (events), {m.shape[0]} CTAs")
    for j, nm in enumerate(NAMES):
        col = rel[:, j]
        col = col[m[:, j] > 0]
        if col.numel():
            print(f"   {nm:10s} min {col.min().item():7.2f}  med {col.median().item():7.2f}  max {col.max().item():7.2f} us")
