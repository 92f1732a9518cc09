"""Per-launch GEMM time vs token count (CUDA events, back-to-back launches): the
intercept of time(T) is the fixed per-launch cost (prologue, pipeline fill, last
tile's epilogue).  Diagnostic only."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import GemmEpilogue, call  # noqa: E402

shapes = [("qkv_fwd", 2304, 768, 0), ("fc1_fwd", 3072, 768, 0), ("fc2_fwd", 768, 3072, 0), ("proj_fwd", 768, 768, 0),
          ("fc2_dgrad", 3072, 768, 1)]
for name, n, k, bm in shapes:
    pts = []
    for T in (2048, 4096, 8192, 16384, 32768):
        a = torch.randn(T * k, device="cuda").to(torch.bfloat16)
        b = torch.randn(n * k, device="cuda").to(torch.bfloat16)
        d = torch.empty(T * n, device="cuda", dtype=torch.bfloat16)
        epi = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0)
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ldb = k if bm == 0 else n
        run = lambda: call("p2bw_kernel_gemm_bf16", C.c_void_p(a.data_ptr()), k, 0, C.c_void_p(b.data_ptr()), ldb, bm,
                           T, n, k, C.byref(epi), s)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 30
        e0.record()
        for _ in range(it):
            run()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / it * 1e3
        pts.append((T, round(us, 2), round(2 * T * n * k / us / 1e6, 1)))
    # least squares on the three largest points
    xs = [p[0] for p in pts[2:]]
    ys = [p[1] for p in pts[2:]]
    mx, my = sum(xs) / 3, sum(ys) / 3
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    print(json.dumps({"name": name, "points(T,us,TF)": pts, "intercept_us": round(my - slope * mx, 2),
                      "marginal_tflops": round(2 * n * k / slope / 1e6, 1)}), flush=True)
