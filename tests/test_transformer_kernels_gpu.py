"""Transformer-stage kernels against torch fp32 references of the same op on
the GPU (the reference has no layer math): attention fwd/bwd
(head dim 64, causal and bidirectional), LayerNorm fwd/bwd, fused softmax-CE.
Tolerances are bf16-storage level and stated per test."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_2006_09503_b200._lib import call  # noqa: E402

pytestmark = pytest.mark.gpu


def ptr(t):
    return C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ref_attention(qkv, b, s, nh, causal, hd=64):
    h = nh * hd
    q, k, v = qkv.float().view(b, s, 3, nh, hd).permute(2, 0, 3, 1, 4)
    sc = q @ k.transpose(-1, -2) * hd ** -0.5
    if causal:
        sc = sc.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool, device=qkv.device), 1), float("-inf"))
    p = torch.softmax(sc, -1)
    o = (p @ v).transpose(1, 2).reshape(b * s, h)
    lse = torch.logsumexp(sc, -1).reshape(-1)
    return o, lse


@pytest.mark.parametrize("b,s,nh,causal", [(2, 128, 2, True), (2, 128, 2, False), (1, 512, 4, True),
                                           (3, 512, 2, False), (2, 1024, 3, True), (1, 2048, 2, False),
                                           # more work items than SMs: the persistent backward's
                                           # cross-item pipeline (K/V ring, dK/dV hand-off)
                                           (16, 512, 12, False), (8, 384, 12, True),
                                           # one unit (the second slot idle), an odd unit count,
                                           # and the GPT-2.2B step's shape (30 heads, causal)
                                           (1, 128, 1, True), (1, 384, 1, False), (16, 512, 30, True),
                                           # odd (sequence, head) counts: the forward pairs two heads per
                                           # causal unit, so one unit runs a single tile; odd tile counts
                                           (3, 256, 3, True), (5, 384, 1, True), (3, 384, 3, False)])
def test_attention_fwd_bwd_vs_torch(b, s, nh, causal):
    """One tcgen05 implementation per pass, for every seq % 128 == 0 (no CUDA-core path)."""
    h = nh * 64
    g = torch.Generator(device="cuda").manual_seed(b * 1000 + s + nh)
    qkv = (torch.randn(b * s, 3 * h, device="cuda", generator=g) * 0.8).to(torch.bfloat16)
    o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b * nh * s, device="cuda", dtype=torch.float32)
    call("p2bw_kernel_attention_fwd", ptr(qkv), ptr(o), ptr(lse), b, s, nh, int(causal), stream())
    ref_in = qkv.float().requires_grad_(True)
    ro, rl = ref_attention(ref_in, b, s, nh, causal)
    torch.cuda.synchronize()
    assert (o.float() - ro).abs().max().item() < 2e-2          # bf16 output rounding
    assert (lse - rl.detach()).abs().max().item() < 1e-2
    dout = torch.randn(b * s, h, device="cuda", generator=g).to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(b * nh * s, device="cuda", dtype=torch.float32)
    call("p2bw_kernel_attention_bwd", ptr(qkv), ptr(o), ptr(dout), ptr(lse), ptr(dqkv), ptr(delta), b, s, nh,
         int(causal), stream())
    ro.backward(dout.float())
    torch.cuda.synchronize()
    ref = ref_in.grad
    err = (dqkv.float() - ref).abs().max().item()
    assert err < 3e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("b,s,nh,causal", [(2, 128, 2, True), (2, 128, 1, False), (1, 512, 4, True),
                                           (3, 384, 2, False), (2, 1024, 3, True),
                                           # more items than SMs (single-buffered K / V and Q / dO
                                           # hand-offs across items), and GPT-2.2B at 15 x 128 heads
                                           (16, 512, 8, False), (16, 512, 15, True), (5, 384, 1, True)])
def test_attention_head_dim_128_vs_torch(b, s, nh, causal):
    """Head dim 128 (SURVEY a14's 15 x 128-head GPT layout): the key-quarter forward at
    D = 128 and the D = 128 backward (P^T through SMEM, dQ in the S^T columns)."""
    hd, h = 128, nh * 128
    g = torch.Generator(device="cuda").manual_seed(b * 1000 + s + nh + 77)
    qkv = (torch.randn(b * s, 3 * h, device="cuda", generator=g) * 0.6).to(torch.bfloat16)
    o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b * nh * s, device="cuda", dtype=torch.float32)
    call("p2bw_kernel_attention_fwd_hd", ptr(qkv), ptr(o), ptr(lse), b, s, nh, hd, int(causal), stream())
    ref_in = qkv.float().requires_grad_(True)
    ro, rl = ref_attention(ref_in, b, s, nh, causal, hd)
    torch.cuda.synchronize()
    assert (o.float() - ro).abs().max().item() < 2e-2
    assert (lse - rl.detach()).abs().max().item() < 1e-2
    dout = torch.randn(b * s, h, device="cuda", generator=g).to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(b * nh * s, device="cuda", dtype=torch.float32)
    call("p2bw_kernel_attention_bwd_hd", ptr(qkv), ptr(o), ptr(dout), ptr(lse), ptr(dqkv), ptr(delta), b, s, nh,
         hd, int(causal), stream())
    ro.backward(dout.float())
    torch.cuda.synchronize()
    ref = ref_in.grad
    for part, name in enumerate("qkv"):
        d = dqkv.view(b * s, 3, h)[:, part].float()
        r = ref.view(b * s, 3, h)[:, part]
        err = (d - r).abs().max().item()
        assert err < 3e-2 * max(1.0, r.abs().max().item()), (name, err)


def test_attention_rejects_bad_head_dim():
    qkv = torch.zeros(128, 3 * 96, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(128, 96, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(128, device="cuda", dtype=torch.float32)
    with pytest.raises(Exception, match="head dim"):
        call("p2bw_kernel_attention_fwd_hd", ptr(qkv), ptr(o), ptr(lse), 1, 128, 1, 96, 1, stream())


def test_attention_rejects_untiled_sequence_length():
    qkv = torch.zeros(2 * 96, 3 * 128, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(2 * 96, 128, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(2 * 2 * 96, device="cuda", dtype=torch.float32)
    with pytest.raises(Exception, match="multiple of 128"):
        call("p2bw_kernel_attention_fwd", ptr(qkv), ptr(o), ptr(lse), 2, 96, 2, 1, stream())


@pytest.mark.parametrize("rows,h", [(300, 256), (1024, 768), (64, 1024), (33, 1920), (4099, 1920), (2500, 1280),
                                    (20000, 768), (5000, 2048), (9001, 256)])  # ring wrap-around
@pytest.mark.parametrize("with_dsum", [False, True])
def test_layernorm_fwd_bwd_vs_torch(rows, h, with_dsum):
    g = torch.Generator(device="cuda").manual_seed(rows + h)
    x = (torch.randn(rows, h, device="cuda", generator=g) * 2 + 0.5).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(h, device="cuda", generator=g)).to(torch.bfloat16)
    bb = (0.1 * torch.randn(h, device="cuda", generator=g)).to(torch.bfloat16)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    call("p2bw_kernel_layernorm_fwd", ptr(x), ptr(w), ptr(bb), ptr(y), ptr(mean), ptr(rstd), rows, h, stream())
    xr = x.float().requires_grad_(True)
    wr = w.float().requires_grad_(True)
    br = bb.float().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (h,), wr, br, 1e-5)
    torch.cuda.synchronize()
    assert (y.float() - yr).abs().max().item() < 3e-2
    dy = torch.randn(rows, h, device="cuda", generator=g).to(torch.bfloat16)
    dres = torch.randn(rows, h, device="cuda", generator=g).to(torch.bfloat16)
    dx = torch.empty_like(x)
    dg = torch.full((h,), 5.0, device="cuda")
    db = torch.full((h,), 5.0, device="cuda")
    ds = torch.full((h,), 5.0, device="cuda")
    call("p2bw_kernel_layernorm_bwd", ptr(dy), ptr(x), ptr(mean), ptr(rstd), ptr(w), ptr(dres), ptr(dx), ptr(dg),
         ptr(db), ptr(ds) if with_dsum else None, 0, rows, h, stream())  # accumulate onto 5.0
    yr.backward(dy.float())
    torch.cuda.synchronize()
    ref_dx = xr.grad + dres.float()
    assert (dx.float() - ref_dx).abs().max().item() < 3e-2 * max(1.0, ref_dx.abs().max().item())
    assert (dg - 5.0 - wr.grad).abs().max().item() < 1e-2 * max(1.0, wr.grad.abs().max().item())
    assert (db - 5.0 - br.grad).abs().max().item() < 1e-2 * max(1.0, br.grad.abs().max().item())
    if with_dsum:  # fused bias gradient: column sums of the bf16 dx the kernel stored
        ref_ds = dx.float().sum(0)
        assert (ds - 5.0 - ref_ds).abs().max().item() < 1e-3 * max(1.0, ref_ds.abs().max().item())
    else:
        assert torch.all(ds == 5.0)


@pytest.mark.parametrize("rows,vocab", [(64, 1000), (16, 51200), (130, 30522), (3, 7), (8, 70001)])  # 70001: two-pass path
def test_softmax_xent_vs_torch(rows, vocab):
    vp = (vocab + 127) // 128 * 128
    g = torch.Generator(device="cuda").manual_seed(rows + vocab)
    logits = (torch.randn(rows, vp, device="cuda", generator=g) * 3).to(torch.bfloat16)
    tgt = torch.randint(0, vocab, (rows,), device="cuda", generator=g, dtype=torch.int32)
    lr = logits.float()[:, :vocab].requires_grad_(True)
    loss = torch.nn.functional.cross_entropy(lr, tgt.long(), reduction="none")
    row_loss = torch.empty(rows, device="cuda")
    call("p2bw_kernel_softmax_xent", ptr(logits), ptr(tgt), rows, vocab, vp, C.c_float(1.0 / rows), ptr(row_loss),
         stream())
    loss.mean().backward()
    torch.cuda.synchronize()
    assert (row_loss - loss.detach()).abs().max().item() < 1e-3 * max(1.0, loss.abs().max().item())
    assert (logits.float()[:, :vocab] - lr.grad).abs().max().item() < 2e-3 / rows + 1e-5
    if vp > vocab:
        assert logits.float()[:, vocab:].abs().max().item() == 0.0


@pytest.mark.parametrize("rows,n,ld", [(128, 128, 128), (128, 384, 384), (8192, 768, 768), (8192, 3072, 3072),
                                       (300, 2304, 2304), (77, 512, 640)])
@pytest.mark.parametrize("overwrite", [0, 1])
def test_colsum_bias_grad_vs_torch(rows, n, ld, overwrite):
    g = torch.Generator(device="cuda").manual_seed(rows + n + overwrite)
    x = torch.randn(rows, ld, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((n,), 3.0, device="cuda")
    call("p2bw_kernel_colsum", ptr(x), rows, n, ld, ptr(out), overwrite, stream())
    torch.cuda.synchronize()
    ref = x.float()[:, :n].sum(0) + (0.0 if overwrite else 3.0)
    assert (out - ref).abs().max().item() < 1e-3 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("nvl", ["1", "2"])
@pytest.mark.parametrize("rows,h", [(4099, 1920), (700, 1024), (2500, 1280), (5000, 2048), (300, 512), (1000, 768)])
def test_layernorm_bwd_vectors_per_lane(rows, h, nvl, monkeypatch):
    """Both LayerNorm-backward layouts (one or two 16-byte vectors per lane; P2BW_LN_BWD_NVL
    forces one, the default picks two for h >= 1024) against torch."""
    monkeypatch.setenv("P2BW_LN_BWD_NVL", nvl)
    test_layernorm_fwd_bwd_vs_torch(rows, h, True)
    test_layernorm_fwd_bwd_vs_torch(rows, h, False)


@pytest.mark.parametrize("rows,h", [(128, 128), (4096, 768)])
def test_layernorm_bwd_small_hidden(rows, h):
    test_layernorm_fwd_bwd_vs_torch(rows, h, True)


def test_layernorm_bwd_in_place():
    """The last stage runs LNf backward with dx aliasing dy (model_transformer.cu)."""
    rows, h = 256, 768
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(rows, h, device="cuda", generator=g).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(h, device="cuda", generator=g)).to(torch.bfloat16)
    bb = torch.zeros(h, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    call("p2bw_kernel_layernorm_fwd", ptr(x), ptr(w), ptr(bb), ptr(y), ptr(mean), ptr(rstd), rows, h, stream())
    dy = torch.randn(rows, h, device="cuda", generator=g).to(torch.bfloat16)
    buf = dy.clone()
    dg = torch.empty(h, device="cuda")
    db = torch.empty(h, device="cuda")
    ds = torch.empty(h, device="cuda")
    call("p2bw_kernel_layernorm_bwd", ptr(buf), ptr(x), ptr(mean), ptr(rstd), ptr(w), None, ptr(buf), ptr(dg),
         ptr(db), ptr(ds), 1, rows, h, stream())
    xr = x.float().requires_grad_(True)
    wr = w.float().requires_grad_(True)
    br = bb.float().requires_grad_(True)
    torch.nn.functional.layer_norm(xr, (h,), wr, br, 1e-5).backward(dy.float())
    torch.cuda.synchronize()
    assert (buf.float() - xr.grad).abs().max().item() < 3e-2 * max(1.0, xr.grad.abs().max().item())
    assert (dg - wr.grad).abs().max().item() < 1e-2 * max(1.0, wr.grad.abs().max().item())
    assert (db - br.grad).abs().max().item() < 1e-2 * max(1.0, br.grad.abs().max().item())
    assert (ds - buf.float().sum(0)).abs().max().item() < 1e-3 * max(1.0, buf.float().sum(0).abs().max().item())


@pytest.mark.parametrize("causal", [True, False])
def test_attention_fwd_bit_stable_under_concurrent_load(causal):
    """The persistent forward's warps of different TMEM lane quarters run unsynchronised
    (only the four key-quarter warps of a row meet at the max exchange); under a
    concurrent kernel on another stream they drift apart.  The kernel has no atomics, so
    every repeat must reproduce the quiet run bit for bit (a barrier-phase race -- an
    arrival for block g + 1 counted towards block g -- shows up here as garbage)."""
    b, s, nh = 16, 512, 12
    h = nh * 64
    g = torch.Generator(device="cuda").manual_seed(11)
    qkv = (torch.randn(b * s, 3 * h, device="cuda", generator=g) * 0.8).to(torch.bfloat16)
    o0 = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    l0 = torch.empty(b * nh * s, device="cuda", dtype=torch.float32)
    call("p2bw_kernel_attention_fwd", ptr(qkv), ptr(o0), ptr(l0), b, s, nh, int(causal), stream())
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    x = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    for _ in range(10):
        o = torch.empty_like(o0)
        lse = torch.empty_like(l0)
        with torch.cuda.stream(side):
            for _ in range(3):
                y = x @ x  # noqa: F841 -- contention only
        call("p2bw_kernel_attention_fwd", ptr(qkv), ptr(o), ptr(lse), b, s, nh, int(causal), stream())
        torch.cuda.synchronize()
        assert torch.equal(o, o0) and torch.equal(lse, l0)
