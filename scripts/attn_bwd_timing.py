"""Phase timing of the tcgen05 attention backward (diagnostic): clock64 marks of the
first 8 query tiles of every CTA (see attention_tc_bwd.cu g_attn_bwd_dbg)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

causal = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nh = int(sys.argv[2]) if len(sys.argv) > 2 else 12
b, s = 16, 512
h = nh * 64
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (torch.randn(b * s, 3 * h, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
dout = torch.randn(b * s, h, device="cuda", generator=g).to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
lse = torch.empty(b * nh * s, device="cuda")
delta = torch.empty(b * nh * s, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
call("p2bw_kernel_attention_fwd", P(qkv), P(o), P(lse), b, s, nh, causal, st)
bwd = lambda: call("p2bw_kernel_attention_bwd", P(qkv), P(o), P(dout), P(lse), P(dqkv), P(delta), b, s, nh,  # noqa
                   causal, st)
for _ in range(3):
    bwd()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    bwd()
e1.record()
torch.cuda.synchronize()
print(f"attention bwd (delta + main + dq convert): {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per call")
dbg = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
call("p2bw_debug_attention_timing", P(dbg))
bwd()
torch.cuda.synchronize()
call("p2bw_debug_attention_timing", None)
d = dbg.view(148, 8, 8).cpu().double()  # [cta][slot][g]
names = ["elem S/dP seen", "elem computed", "elem mm2(g-1) seen", "elem pds", "mma S/dP issued", "mma mm2 issued",
         "flush mm2 seen", "flush dq free"]
t0 = d[:, 4, 0:1]  # first S/dP issue
for gi in range(8):
    row = " ".join(f"{(d[:, k, gi:gi + 1] - t0).median().item():8.0f}" for k in range(8))
    print(f"g={gi}: {row}")
print("columns:", " | ".join(names))
