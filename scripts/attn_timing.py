"""Phase timing of the persistent tcgen05 attention forward (diagnostic): clock64 marks of
the first 8 key blocks of each slot of every CTA (attention_tc.cu g_attn_dbg).
    python scripts/attn_timing.py [causal] [heads]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

causal = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nh = int(sys.argv[2]) if len(sys.argv) > 2 else 30
b, s = 16, 512
h = nh * 64
qkv = (torch.randn(b * s, 3 * h, device="cuda") * 0.5).to(torch.bfloat16)
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
print(f"attention fwd: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per launch")
dbg = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
call("p2bw_debug_attention_timing", P(dbg))
fwd()
torch.cuda.synchronize()
call("p2bw_debug_attention_timing", None)
d = dbg.view(148, 8, 8).cpu().double()  # [cta][series][e]
t0 = d[:, 0, 0:1]  # slot 0 only
names = ["S issued", "S seen", "max exch", "P arrived", "-", "-", "-", "PV issued"]
print("median cycles from the first S issue, per block e of the slot's stream")
print("      " + " ".join(f"{n:>12s}" for n in names))
for e in range(8):
    print(f"e={e}: " + " ".join(f"{(d[:, k, e:e + 1] - t0).median().item():12.0f}" for k in range(8)))
