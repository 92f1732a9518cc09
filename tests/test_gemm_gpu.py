"""Parity of the tcgen05 GEMM (p2bw_kernel_gemm_bf16) against a torch fp32
reference of the same contraction, for every operand-major combination the
stage executor uses (forward K/K, dgrad K/MN, wgrad MN/MN) and every epilogue.
Reference ops replaced: matmul / matmul_tn / matmul_nt, semantics.cpp:9-44."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_2006_09503_b200._lib import GemmEpilogue, call  # noqa: E402

pytestmark = pytest.mark.gpu


def _operand(rows, k, major, gen):
    """Logical [rows x k] matrix stored K-major (rows x k) or MN-major (k x rows)."""
    logical = torch.randn(rows, k, generator=gen, device="cuda").to(torch.bfloat16)
    if major == 0:
        store = logical.contiguous()
        return logical, store, store.stride(0)
    store = logical.t().contiguous()
    return logical, store, store.stride(0)


def _gemm(a, lda, am, b, ldb, bm, m, n, k, epi):
    call("p2bw_kernel_gemm_bf16", C.c_void_p(a.data_ptr()), lda, am, C.c_void_p(b.data_ptr()), ldb,
         bm, m, n, k, C.byref(epi), C.c_void_p(torch.cuda.current_stream().cuda_stream))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("m,n,k", [(256, 256, 128), (384, 768, 320), (200, 96, 64), (1024, 2304, 768)])
def test_gemm_f32_store_matches_torch(am, bm, m, n, k):
    gen = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k + am * 2 + bm)
    A, a, lda = _operand(m, k, am, gen)
    B, b, ldb = _operand(n, k, bm, gen)
    d = torch.full((m, n), 7.0, device="cuda", dtype=torch.float32)
    epi = GemmEpilogue(kind=1, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0)
    _gemm(a, lda, am, b, ldb, bm, m, n, k, epi)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    err = (d - ref).abs().max().item()
    assert err <= 1e-3 * (1 + ref.abs().max().item()), err


@pytest.mark.parametrize("am,bm", [(0, 0), (1, 1)])
def test_gemm_f32_accumulate(am, bm):
    m, n, k = 512, 512, 256
    gen = torch.Generator(device="cuda").manual_seed(5)
    A, a, lda = _operand(m, k, am, gen)
    B, b, ldb = _operand(n, k, bm, gen)
    d0 = torch.randn(m, n, device="cuda", generator=gen)
    d = d0.clone()
    epi = GemmEpilogue(kind=1, d=d.data_ptr(), ldd=n, alpha=0.5, beta=1.0)
    _gemm(a, lda, am, b, ldb, bm, m, n, k, epi)
    torch.cuda.synchronize()
    ref = d0 + 0.5 * (A.float() @ B.float().t())
    assert (d - ref).abs().max().item() < 2e-3 * ref.abs().max().item()


def test_gemm_bf16_bias_gelu_residual():
    m, n, k = 640, 1024, 384
    gen = torch.Generator(device="cuda").manual_seed(11)
    A, a, lda = _operand(m, k, 0, gen)
    B, b, ldb = _operand(n, k, 0, gen)
    bias = torch.randn(n, device="cuda", generator=gen).to(torch.bfloat16)
    res = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    pre = torch.empty_like(out)
    epi = GemmEpilogue(kind=0, d=out.data_ptr(), ldd=n, bias=bias.data_ptr(), residual=res.data_ptr(),
                       ldr=n, preact=pre.data_ptr(), gelu=1, alpha=1.0)
    _gemm(a, lda, 0, b, ldb, 0, m, n, k, epi)
    torch.cuda.synchronize()
    u = A.float() @ B.float().t() + bias.float()
    assert (pre.float() - u).abs().max().item() < 0.05 * u.abs().max().item()
    ref = gelu_tanh(pre.float()) + res.float()
    assert (out.float() - ref).abs().max().item() < 0.02 * ref.abs().max().item()


def test_gemm_dgelu_epilogue():
    m, n, k = 256, 512, 256
    gen = torch.Generator(device="cuda").manual_seed(13)
    A, a, lda = _operand(m, k, 0, gen)
    B, b, ldb = _operand(n, k, 1, gen)
    u = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    epi = GemmEpilogue(kind=2, d=out.data_ptr(), ldd=n, aux=u.data_ptr(), alpha=1.0)
    _gemm(a, lda, 0, b, ldb, 1, m, n, k, epi)
    torch.cuda.synchronize()
    uf = u.float().requires_grad_(True)
    g = torch.autograd.grad(gelu_tanh(uf).sum(), uf)[0]
    ref = (A.float() @ B.float().t()) * g
    assert (out.float() - ref).abs().max().item() < 0.02 * ref.abs().max().item()


@pytest.mark.parametrize("beta", [0.0, 1.0])
@pytest.mark.parametrize("m,n,k", [(768, 768, 8192), (2304, 768, 4096), (256, 512, 2048)])
def test_gemm_wgrad_split_k(m, n, k, beta):
    """Small-output, long-K wgrad GEMMs take the split-K path (TMA reduce-add per K slice)."""
    gen = torch.Generator(device="cuda").manual_seed(m + n + k)
    A, a, lda = _operand(m, k, 1, gen)
    B, b, ldb = _operand(n, k, 1, gen)
    d0 = torch.randn(m, n, device="cuda", generator=gen)
    d = d0.clone()
    epi = GemmEpilogue(kind=1, d=d.data_ptr(), ldd=n, alpha=1.0, beta=beta)
    _gemm(a, lda, 1, b, ldb, 1, m, n, k, epi)
    torch.cuda.synchronize()
    ref = beta * d0 + A.float() @ B.float().t()
    assert (d - ref).abs().max().item() < 2e-3 * ref.abs().max().item()


@pytest.mark.parametrize("tile", ["128,1", "128,2", "192,1", "192,2", "256,1", "256,2", "128,4", "192,4", "256,4"])
@pytest.mark.parametrize("am,bm,kind", [(0, 0, 0), (0, 1, 0), (1, 1, 1), (0, 1, 2)])
@pytest.mark.parametrize("n", [768, 640, 608])  # 640 / 608: a last N tile of <= BN / 2 columns
def test_gemm_every_tile(monkeypatch, tile, am, bm, kind, n):
    """Every (BN, cluster) tile the shape-based chooser may pick, on a ragged shape,
    for the forward (bf16 + bias), dgrad (bf16 / dGELU) and wgrad (fp32) layouts.
    Pair tiles whose B half is not whole 64-column atoms fall back to one CTA.  The
    4-CTA clusters (two pairs sharing A through TMA multicast) leave the second pair
    of the last N group past N when the tile count along N is odd.  A last N tile with
    at most BN / 2 valid columns runs its MMAs at N = BN / 2 (KParams::half_n)."""
    monkeypatch.setenv("P2BW_GEMM_TILE", tile)
    m, k = 1000, 704
    gen = torch.Generator(device="cuda").manual_seed(17 + am + 2 * bm + 4 * kind + n)
    A, a, lda = _operand(m, k, am, gen)
    B, b, ldb = _operand(n, k, bm, gen)
    ref = A.float() @ B.float().t()
    if kind == 1:
        d = torch.zeros(m, n, device="cuda")
        epi = GemmEpilogue(kind=1, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0)
    elif kind == 2:
        u = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
        d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        epi = GemmEpilogue(kind=2, d=d.data_ptr(), ldd=n, aux=u.data_ptr(), alpha=1.0)
        uf = u.float().requires_grad_(True)
        ref = ref * torch.autograd.grad(gelu_tanh(uf).sum(), uf)[0]
    else:
        bias = torch.randn(n, device="cuda", generator=gen).to(torch.bfloat16)
        d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        epi = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, bias=bias.data_ptr(), alpha=1.0)
        ref = ref + bias.float()
    _gemm(a, lda, am, b, ldb, bm, m, n, k, epi)
    torch.cuda.synchronize()
    tol = 1e-3 if kind == 1 else 0.02
    assert (d.float() - ref).abs().max().item() <= tol * ref.abs().max().item()


@pytest.mark.parametrize("tile", ["256,4", "192,4"])
@pytest.mark.parametrize("m,n,k", [(8192, 768, 3072), (4096, 2304, 768), (2304, 768, 8192)])
def test_gemm_multicast_cluster_large(monkeypatch, tile, m, n, k):
    """4-CTA clusters on stage-sized shapes (many K blocks, several waves)."""
    monkeypatch.setenv("P2BW_GEMM_TILE", tile)
    gen = torch.Generator(device="cuda").manual_seed(m + n + k)
    A, a, lda = _operand(m, k, 0, gen)
    B, b, ldb = _operand(n, k, 0, gen)
    d = torch.zeros(m, n, device="cuda")
    epi = GemmEpilogue(kind=1, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0)
    _gemm(a, lda, 0, b, ldb, 0, m, n, k, epi)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    assert (d - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()


@pytest.mark.parametrize("m,n,k,bm", [(1232, 768, 30592, 1), (300, 256, 8192, 0)])
def test_gemm_bf16_split_k_workspace(m, n, k, bm):
    """A plain bf16 store with few output tiles and a long K (the LM-head dgrad) runs
    split-K into the fp32 workspace and is cast: same result as the direct store."""
    gen = torch.Generator(device="cuda").manual_seed(m + k)
    A, a, lda = _operand(m, k, 0, gen)
    B, b, ldb = _operand(n, k, bm, gen)
    ws = torch.full((m * n,), 3.0, device="cuda")
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    epi = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, alpha=0.5, workspace=ws.data_ptr(), workspace_floats=m * n)
    _gemm(a, lda, 0, b, ldb, bm, m, n, k, epi)
    d2 = torch.empty_like(d)
    epi2 = GemmEpilogue(kind=0, d=d2.data_ptr(), ldd=n, alpha=0.5)
    _gemm(a, lda, 0, b, ldb, bm, m, n, k, epi2)
    torch.cuda.synchronize()
    ref = 0.5 * (A.float() @ B.float().t())
    scale = ref.abs().max().item()
    assert (d.float() - ref).abs().max().item() <= 0.01 * scale
    assert (d2.float() - ref).abs().max().item() <= 0.01 * scale


@pytest.mark.parametrize("accumulate", [0, 1])
@pytest.mark.parametrize("m,n,k", [(3072, 768, 8192), (2304, 768, 8192), (200, 256, 1000)])
def test_gemm_wgrad_fused_bias_grad(m, n, k, accumulate):
    """The wgrad GEMM also sums its A operand's rows (the bias gradient of the layer
    whose output gradient A is) from the SMEM tiles: bias (=|+=) A.sum(K)."""
    gen = torch.Generator(device="cuda").manual_seed(m + n + k + accumulate)
    A, a, lda = _operand(m, k, 1, gen)
    B, b, ldb = _operand(n, k, 1, gen)
    d = torch.zeros(m, n, device="cuda")
    bias0 = torch.randn(m, device="cuda", generator=gen)
    bias = bias0.clone()
    scratch = torch.zeros((k // 512 + 1) * m, device="cuda")
    epi = GemmEpilogue(kind=1, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0, bias_grad=bias.data_ptr(),
                       bias_grad_accumulate=accumulate, bias_scratch=scratch.data_ptr(),
                       bias_scratch_floats=scratch.numel())
    _gemm(a, lda, 1, b, ldb, 1, m, n, k, epi)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    assert (d - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()
    bref = A.float().sum(1) + (bias0 if accumulate else 0)
    assert (bias - bref).abs().max().item() <= 1e-3 * (1 + bref.abs().max().item())


@pytest.mark.parametrize("accumulate", [0, 1])
@pytest.mark.parametrize("m,n,k", [(8192, 768, 3072), (8192, 768, 2304), (300, 256, 1000), (1000, 224, 64)])
def test_gemm_dgrad_fused_bias_grad(m, n, k, accumulate):
    """The dgrad GEMM (A K-major = the layer's output gradient, B MN-major = the weight)
    also sums A over its rows from the SMEM tiles: bias (=|+=) A.sum(M) -- the bias
    gradient the model used to compute in a separate column-sum pass."""
    gen = torch.Generator(device="cuda").manual_seed(m + n + k + accumulate + 7)
    A, a, lda = _operand(m, k, 0, gen)
    B, b, ldb = _operand(n, k, 1, gen)
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    bias0 = torch.randn(k, device="cuda", generator=gen)
    bias = bias0.clone()
    scratch = torch.full((2 * ((m + 127) // 128) * k,), float("nan"), device="cuda")
    epi = GemmEpilogue(kind=0, d=d.data_ptr(), ldd=n, alpha=1.0, beta=0.0, bias_grad=bias.data_ptr(),
                       bias_grad_accumulate=accumulate, bias_scratch=scratch.data_ptr(),
                       bias_scratch_floats=scratch.numel())
    _gemm(a, lda, 0, b, ldb, 1, m, n, k, epi)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    assert (d.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    bref = A.float().sum(0) + (bias0 if accumulate else 0)
    assert (bias - bref).abs().max().item() <= 1e-3 * (1 + bref.abs().max().item())


def _plan(m, n, k, am, bm, kind, bias_grad=0):
    out = (C.c_int * 4)()
    call("p2bw_debug_gemm_plan", m, n, k, am, bm, kind, bias_grad, out)
    return list(out)


# GPT-2.2B (h 1920, 8192-token microbatches) stage shapes whose last wave is ragged:
# attention projection / fc2 forward (bias + residual), the fc1 / QKV dgrads with the
# fused bias gradient, a plain store, and a single-CTA-tile shape.
TAIL_CASES = [
    ("fwd_res", 8192, 1920, 7680, 0, 0, 0),
    ("fwd_res", 8192, 1920, 3840, 0, 0, 0),
    ("plain", 8192, 1920, 5760, 0, 1, 0),
    ("dgrad_bias", 8192, 1920, 7680, 0, 1, 0),
    ("dgelu", 1000, 1024, 4096, 0, 1, 2),
]


@pytest.mark.parametrize("case,m,n,k,am,bm,kind", TAIL_CASES)
def test_gemm_tail_split(case, m, n, k, am, bm, kind):
    """Ragged-last-wave shapes take the tail split (the last wave's tiles run as K parts
    on otherwise idle SMs; contributors hand fp32 partials to a finisher through L2):
    the result matches torch, and repeated launches -- whose arrival counters the
    finishers re-arm -- are bit-identical."""
    plan = _plan(m, n, k, am, bm, kind, 1 if case == "dgrad_bias" else 0)
    assert plan[3] >= 2, plan  # the case exercises the tail split
    gen = torch.Generator(device="cuda").manual_seed(m + n + k + kind)
    A, a, lda = _operand(m, k, am, gen)
    B, b, ldb = _operand(n, k, bm, gen)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    ref = A.float() @ B.float().t()
    kw = {}
    if case == "fwd_res":
        bias = torch.randn(n, device="cuda", generator=gen).to(torch.bfloat16)
        res = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
        kw = dict(bias=bias.data_ptr(), residual=res.data_ptr(), ldr=n)
        ref = ref + bias.float() + res.float()
    elif case == "dgrad_bias":
        bgrad = torch.zeros(k, device="cuda")
        scratch = torch.empty(2 * ((m + 127) // 128) * k, device="cuda")
        kw = dict(bias_grad=bgrad.data_ptr(), bias_scratch=scratch.data_ptr(), bias_scratch_floats=scratch.numel())
    elif case == "dgelu":
        u = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
        kw = dict(aux=u.data_ptr())
        uf = u.float().requires_grad_(True)
        ref = ref * torch.autograd.grad(gelu_tanh(uf).sum(), uf)[0]
    epi = GemmEpilogue(kind=kind, d=out.data_ptr(), ldd=n, alpha=1.0, **kw)
    outs = []
    for _ in range(3):
        out.fill_(float("nan"))
        _gemm(a, lda, am, b, ldb, bm, m, n, k, epi)
        torch.cuda.synchronize()
        outs.append(out.clone())
    err = (outs[0].float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item(), (case, plan, err)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    if case == "dgrad_bias":
        bref = A.float().sum(0)
        assert (bgrad - bref).abs().max().item() <= 1e-3 * (1 + bref.abs().max().item())


def test_gemm_tail_split_concurrent_streams():
    """Two tail-split GEMMs on two streams at once (each stream has its own partial
    workspace and counters) finish and agree with their serial results."""
    m, n, k = 8192, 1920, 3840
    assert _plan(m, n, k, 0, 0, 0)[3] >= 2
    gen = torch.Generator(device="cuda").manual_seed(99)
    ops = [(_operand(m, k, 0, gen), _operand(n, k, 0, gen)) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    serial, outs = [], [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    for i, ((_, a, lda), (_, b, ldb)) in enumerate(ops):
        _gemm(a, lda, 0, b, ldb, 0, m, n, k, GemmEpilogue(kind=0, d=outs[i].data_ptr(), ldd=n, alpha=1.0))
        torch.cuda.synchronize()
        serial.append(outs[i].clone())
    torch.cuda.synchronize()
    for rep in range(4):
        for i, ((_, a, lda), (_, b, ldb)) in enumerate(ops):
            with torch.cuda.stream(streams[i]):
                _gemm(a, lda, 0, b, ldb, 0, m, n, k, GemmEpilogue(kind=0, d=outs[i].data_ptr(), ldd=n, alpha=1.0))
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(outs[i], serial[i]), (rep, i)
