"""Attention forward time vs batch (CUDA-graph timed): shows the wave quantisation of
768 CTAs on 148 SMs x 4 CTAs (diagnostic)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

s, nh = 512, 12
h = nh * 64
for b in (4, 8, 12, 16, 20, 24, 32):
    qkv = torch.randn(b * s, 3 * h, device="cuda").to(torch.bfloat16)
    o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b * nh * s, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    run = lambda: call("p2bw_kernel_attention_fwd", P(qkv), P(o), P(lse), b, s, nh, 0,  # noqa: E731
                       C.c_void_p(torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    ctas = b * nh * (s // 128)
    print(f"b={b:2d}: {ctas:4d} CTAs ({ctas / 592:.2f} waves of 4/SM): {us:6.1f} us, "
          f"{4 * s * s * h * b / us / 1e6:.0f} TF/s")
