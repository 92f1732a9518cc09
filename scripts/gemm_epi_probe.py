"""Stage GEMMs with their real epilogues (bias / GELU + pre-activation / residual /
dGELU) vs a plain store, isolated (diagnostic)."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import GemmEpilogue, call  # noqa: E402

T, h = 8192, 768
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rnd(*shape):
    return (torch.randn(*shape, device="cuda") * 0.1).to(torch.bfloat16)


out = {}
for name, n, k, epi in [("qkv", 3 * h, h, "bias"), ("proj", h, h, "bias_res"), ("fc1", 4 * h, h, "gelu"),
                        ("fc2", h, 4 * h, "bias_res"), ("fc2_dgrad", 4 * h, h, "dgelu")]:
    a, w = rnd(T, k), rnd(n, k)
    d = torch.empty(T, n, device="cuda", dtype=torch.bfloat16)
    bias, res, pre, u = rnd(n), rnd(T, n), torch.empty_like(d), rnd(T, n)
    res_row = {}
    for mode in ("plain", epi):
        e = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, alpha=1.0)
        bm = 0
        if mode == "bias":
            e.bias = bias.data_ptr()
        elif mode == "bias_res":
            e.bias, e.residual, e.ldr = bias.data_ptr(), res.data_ptr(), n
        elif mode == "gelu":
            e.bias, e.gelu, e.preact = bias.data_ptr(), 1, pre.data_ptr()
        elif mode == "dgelu":
            e.kind, e.aux, bm = 2, u.data_ptr(), 1
        wt = w if bm == 0 else w.t().contiguous()
        ldb = k if bm == 0 else n
        ms = bench(lambda: call("p2bw_kernel_gemm_bf16", P(a), k, 0, P(wt), ldb, bm, T, n, k, C.byref(e), s))
        res_row[mode] = round(2 * T * n * k / ms / 1e9, 1)
    out[name] = res_row
print(json.dumps(out))
