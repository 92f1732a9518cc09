"""Phase timing of the tcgen05 attention forward (diagnostic): clock64 marks per CTA."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

b, s, nh, causal = 16, 512, 12, 0
h = nh * 64
qkv = torch.randn(b * s, 3 * h, device="cuda").to(torch.bfloat16)
o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b * nh * s, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ctas = b * nh * (s // 128)
dbg = torch.zeros(ctas * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    call("p2bw_kernel_attention_fwd", C.c_void_p(qkv.data_ptr()), C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()),
         b, s, nh, causal, st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    call("p2bw_kernel_attention_fwd", C.c_void_p(qkv.data_ptr()), C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()),
         b, s, nh, causal, st)
e1.record()
torch.cuda.synchronize()
print(f"attention fwd: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per launch ({ctas} CTAs)")
call("p2bw_debug_attention_timing", C.c_void_p(dbg.data_ptr()))
call("p2bw_kernel_attention_fwd", C.c_void_p(qkv.data_ptr()), C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()),
     b, s, nh, causal, st)
torch.cuda.synchronize()
call("p2bw_debug_attention_timing", None)
d = dbg.view(ctas, 16).cpu().double()
names = ["start->S ready", "pass1 (max)", "max exchange", "pass2 (exp, P)", "sum exchange", "wait O", "epilogue"]
for i, n in enumerate(names):
    dt = d[:, i + 1] - d[:, i]
    print(f"{n:16s} mean {dt.mean():9.0f} cycles  p50 {dt.median():9.0f}  max {dt.max():9.0f}")
tot = d[:, 7] - d[:, 0]
print(f"total per CTA   mean {tot.mean():9.0f} cycles")
gt = d[:, 9] - d[:, 8]
print(f"CTA wall (globaltimer) mean {gt.mean() / 1e3:.2f} us; kernel span {(d[:, 9].max() - d[:, 8].min()) / 1e3:.1f} us")
