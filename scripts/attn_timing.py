"""Phase timing of the tcgen05 attention forward (diagnostic): clock64 marks of the
first 4 key blocks of every CTA (attention_tc.cu g_attn_dbg)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

b, s, nh, causal = 16, 512, 12, int(sys.argv[1]) if len(sys.argv) > 1 else 0
h = nh * 64
qkv = torch.randn(b * s, 3 * h, device="cuda").to(torch.bfloat16)
o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b * nh * s, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
fwd = lambda: call("p2bw_kernel_attention_fwd", P(qkv), P(o), P(lse), b, s, nh, causal, st)  # noqa: E731
for _ in range(3):
    fwd()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    fwd()
e1.record()
torch.cuda.synchronize()
ctas = b * nh * (s // 128)
print(f"attention fwd: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per launch ({ctas} CTAs)")
dbg = torch.zeros(ctas * 16, dtype=torch.int64, device="cuda")
call("p2bw_debug_attention_timing", P(dbg))
fwd()
torch.cuda.synchronize()
call("p2bw_debug_attention_timing", None)
d = dbg.view(ctas, 4, 4).cpu().double()
t0 = d[:, 0, 0:1]
print("per key block j (median cycles from S_0 seen): S seen | pass 1 done | P stored | PV issued")
for j in range(4):
    print(f"j={j}: " + " ".join(f"{(d[:, j, k:k + 1] - t0).median().item():8.0f}" for k in range(4)))
