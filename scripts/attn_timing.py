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
# (the key-blocked forward has no phase marks; the launch time above is the measurement)
