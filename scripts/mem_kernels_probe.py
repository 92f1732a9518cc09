"""Memory-bound stage kernels in isolation (diagnostic): LayerNorm forward / backward
and the bias column sum at the BERT-base microbatch shape, effective GB/s."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_09503_b200._lib import call  # noqa: E402

T = 8192
h = int(sys.argv[1]) if len(sys.argv) > 1 else 768
P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731


class _S:  # the current stream at call time (graph capture runs on a side stream)
    @property
    def _as_parameter_(self):
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)


s = _S()


def bench(fn, reps=20):
    """Device time per call: reps calls captured in a CUDA graph (no host launch cost)."""
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3  # us


x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
g = torch.ones(h, device="cuda").to(torch.bfloat16)
bb = torch.zeros(h, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
mean = torch.empty(T, device="cuda")
rstd = torch.empty(T, device="cuda")
dy = torch.randn(T, h, device="cuda").to(torch.bfloat16)
dres = torch.randn(T, h, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(x)
dg = torch.empty(h, device="cuda")
db = torch.empty(h, device="cuda")
ds = torch.empty(h, device="cuda")
u = torch.randn(T, 4 * h, device="cuda").to(torch.bfloat16)
bias = torch.empty(4 * h, device="cuda")
out = {}
t = bench(lambda: call("p2bw_kernel_layernorm_fwd", P(x), P(g), P(bb), P(y), P(mean), P(rstd), T, h, s))
out["ln_fwd_us"], out["ln_fwd_gbs"] = round(t, 2), round(4 * T * h / t / 1e3, 1)
t = bench(lambda: call("p2bw_kernel_layernorm_bwd", P(dy), P(x), P(mean), P(rstd), P(g), P(dres), P(dx), P(dg), P(db),
                       P(ds), 1, T, h, s))
out["ln_bwd_us"], out["ln_bwd_gbs"] = round(t, 2), round(8 * T * h / t / 1e3, 1)
t = bench(lambda: call("p2bw_kernel_colsum", P(u), T, 4 * h, 4 * h, P(bias), 1, s))
out["colsum_us"], out["colsum_gbs"] = round(t, 2), round(2 * T * 4 * h / t / 1e3, 1)
R, V, VP = 16 * 77, 30522, 30592  # BERT-base MLM head rows of one microbatch
logits = torch.randn(R, VP, device="cuda").to(torch.bfloat16)
tg = torch.randint(0, V, (R,), device="cuda", dtype=torch.int32)
rl = torch.empty(R, device="cuda")
t = bench(lambda: call("p2bw_kernel_softmax_xent", P(logits), P(tg), R, V, VP, C.c_float(1.0), P(rl), s))
out["xent_us"], out["xent_gbs"] = round(t, 2), round(4 * R * VP / t / 1e3, 1)
out["h"] = h
print(json.dumps(out))
