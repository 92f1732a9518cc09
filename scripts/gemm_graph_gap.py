"""Per-launch GEMM time with and without host launch overhead (diagnostic): the same
20 back-to-back launches timed from a Python loop and replayed from a CUDA graph."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import GemmEpilogue, call  # noqa: E402

for name, T, n, k in [("qkv", 2048, 2304, 768), ("qkv", 8192, 2304, 768), ("proj", 8192, 768, 768),
                      ("fc2", 8192, 768, 3072)]:
    a = torch.randn(T * k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n * k, device="cuda").to(torch.bfloat16)
    d = torch.empty(T * n, device="cuda", dtype=torch.bfloat16)
    epi = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0)

    def run():
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        call("p2bw_kernel_gemm_bf16", C.c_void_p(a.data_ptr()), k, 0, C.c_void_p(b.data_ptr()), k, 0, T, n, k,
             C.byref(epi), s)

    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    loop_us = e0.elapsed_time(e1) / 20 * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) / 100 * 1e3
    print(f"{name} T={T}: python loop {loop_us:.1f} us/launch, CUDA graph {graph_us:.1f} us/launch, "
          f"{2 * T * n * k / graph_us / 1e6:.0f} TF/s (graph)")
