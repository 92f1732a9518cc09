"""Sweeps the GEMM tile configurations (BN x cluster) on the stage GEMM shapes of a
config (diagnostic, to calibrate gemm.cu:choose_tile).  Each config runs in a
subprocess because the choice is read from P2BW_GEMM_TILE per call."""
import json
import os
import subprocess
import sys

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
h = int(sys.argv[2]) if len(sys.argv) > 2 else 768
shapes = [  # name, m, n, k, a_major, b_major, f32 out
    ("qkv_fwd", T, 3 * h, h, 0, 0, 0), ("proj_fwd", T, h, h, 0, 0, 0), ("fc1_fwd", T, 4 * h, h, 0, 0, 0),
    ("fc2_fwd", T, h, 4 * h, 0, 0, 0), ("fc1_dgrad", T, h, 4 * h, 0, 1, 0), ("fc2_dgrad", T, 4 * h, h, 0, 1, 0),
    ("qkv_dgrad", T, h, 3 * h, 0, 1, 0), ("proj_dgrad", T, h, h, 0, 1, 0),
    ("qkv_wgrad", 3 * h, h, T, 1, 1, 1), ("proj_wgrad", h, h, T, 1, 1, 1), ("fc1_wgrad", 4 * h, h, T, 1, 1, 1),
    ("fc2_wgrad", h, 4 * h, T, 1, 1, 1),
]
CHILD = r'''
import ctypes as C, json, os, sys, torch
sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import GemmEpilogue, call
name, m, n, k, am, bm, f32 = json.loads(sys.argv[1])
a = torch.randn(m * k, device="cuda").to(torch.bfloat16); b = torch.randn(n * k, device="cuda").to(torch.bfloat16)
d = torch.zeros(m * n, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
epi = GemmEpilogue(kind=1 if f32 else 0, d=d.data_ptr(), ldd=n, alpha=1.0, beta=1.0 if f32 else 0.0)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
if os.environ.get("SWEEP_CUBLAS"):  # library baseline: torch.mm (cuBLAS) on the same shape
    a2, b2 = a.view(m, k), b.view(n, k)
    o2 = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    run = lambda: torch.mm(a2, b2.t(), out=o2)
else:
  run = lambda: call("p2bw_kernel_gemm_bf16", C.c_void_p(a.data_ptr()), k if am == 0 else m, am,
                   C.c_void_p(b.data_ptr()), k if bm == 0 else n, bm, m, n, k, C.byref(epi), s)
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"name": name, "tflops": round(2 * m * n * k / ms / 1e9, 1)}))
'''
rows = {}
for cfg in os.environ.get("SWEEP_CFGS", "auto 128,1 128,2 192,1 192,2 256,1 256,2 cublas").split():
    env = dict(os.environ)
    if cfg == "cublas":
        env["SWEEP_CUBLAS"] = "1"
    elif cfg != "auto":
        env["P2BW_GEMM_TILE"] = cfg
    for sh in shapes:
        out = subprocess.run([sys.executable, "-c", CHILD, json.dumps(sh)], capture_output=True, text=True, env=env)
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            r = {"name": sh[0], "tflops": None}
        rows.setdefault(sh[0], {})[cfg] = r["tflops"]
print(json.dumps({"T": T, "h": h, "tflops": rows}, indent=1))
