"""Times p2bw_kernel_gemm_bf16 on the stage GEMM shapes (CUDA events, warm, L2 >> inputs
rotated) and prints TFLOP/s per shape/layout. Diagnostic only."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import GemmEpilogue, call  # noqa: E402

shapes = [
    ("qkv_fwd", 16384, 2304, 768, 0, 0, 0),
    ("proj_fwd", 16384, 768, 768, 0, 0, 0),
    ("fc1_fwd", 16384, 3072, 768, 0, 0, 0),
    ("fc2_fwd", 16384, 768, 3072, 0, 0, 0),
    ("fc1_dgrad", 16384, 768, 3072, 0, 1, 0),
    ("fc2_dgrad", 16384, 3072, 768, 0, 1, 0),
    ("fc1_wgrad", 3072, 768, 16384, 1, 1, 1),
    ("fc2_wgrad", 768, 3072, 16384, 1, 1, 1),
    ("sq8192", 8192, 8192, 8192, 0, 0, 0),
]
if "gpt-2.2b" in sys.argv[1:]:  # T = 8192 tokens (b 16 x s 512), h 1920, V 51200 (padded)
    T, H, V = 8192, 1920, 51200
    shapes = [
        ("qkv_fwd", T, 3 * H, H, 0, 0, 0), ("proj_fwd", T, H, H, 0, 0, 0), ("fc1_fwd", T, 4 * H, H, 0, 0, 0),
        ("fc2_fwd", T, H, 4 * H, 0, 0, 0), ("head_fwd", T, V, H, 0, 0, 0),
        ("qkv_dgrad", T, H, 3 * H, 0, 1, 0), ("proj_dgrad", T, H, H, 0, 1, 0), ("fc1_dgrad", T, H, 4 * H, 0, 1, 0),
        ("fc2_dgrad", T, 4 * H, H, 0, 1, 0), ("head_dgrad", T, H, V, 0, 1, 0),
        ("qkv_wgrad", 3 * H, H, T, 1, 1, 1), ("proj_wgrad", H, H, T, 1, 1, 1), ("fc1_wgrad", 4 * H, H, T, 1, 1, 1),
        ("fc2_wgrad", H, 4 * H, T, 1, 1, 1), ("head_wgrad", V, H, T, 1, 1, 1),
    ]
res = []
for name, m, n, k, am, bm, f32 in shapes:
    a = torch.randn(m * k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n * k, device="cuda").to(torch.bfloat16)
    d = torch.empty(m * n, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    lda = k if am == 0 else m
    ldb = k if bm == 0 else n
    epi = GemmEpilogue(kind=1 if f32 else 0, d=d.data_ptr(), ldd=n, alpha=1.0, beta=1.0 if f32 else 0.0)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    def run():
        call("p2bw_kernel_gemm_bf16", C.c_void_p(a.data_ptr()), lda, am, C.c_void_p(b.data_ptr()), ldb, bm,
             m, n, k, C.byref(epi), s)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    iters = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2 * m * n * k / ms / 1e9
    # torch (cuBLAS) for comparison
    A = a.view(m, k) if am == 0 else a.view(k, m).t()
    B = b.view(n, k) if bm == 0 else b.view(k, n).t()
    for _ in range(3):
        torch.matmul(A, B.t())
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        torch.matmul(A, B.t())
    e1.record()
    torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1) / iters
    res.append({"name": name, "m": m, "n": n, "k": k, "ms": round(ms, 4), "tflops": round(tf, 1),
                "cublas_tflops": round(2 * m * n * k / ms_t / 1e9, 1)})
    print(json.dumps(res[-1]), flush=True)
