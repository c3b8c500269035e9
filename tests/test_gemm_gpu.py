"""GPU: tcgen05 GEMM (gemm_sm100.cu) against a plain PyTorch fp32 reference of the same op.
Tolerance: bf16 inputs, fp32 accumulation -> compare to fp32 matmul of the bf16 inputs with
rel 2e-3 of the row scale (accumulation-order differences only); bf16 outputs add one bf16
rounding (rel 8e-3)."""
import ctypes

import pytest
import torch

import paper_2510_26475_b200 as rb

pytestmark = pytest.mark.gpu


def _run(A, B, out, bias=None, epi=0, scale=1.0, block_n=0, splits=1):
    dev = rb.default_device()
    torch.cuda.synchronize()
    rb._check(rb.lib().rs_gemm_bf16(dev.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                    ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_void_p(bias.data_ptr()) if bias is not None else None,
                                    A.shape[0], B.shape[0], A.shape[1], epi, scale, block_n, splits))
    dev.sync()


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 0), (1344, 2560, 2048, 0), (200, 1000, 256, 128),
                                      (7, 96, 136, 128), (1, 151936 // 64, 2048, 0), (513, 2048, 11008, 256)])
def test_gemm_bf16_bias(M, N, K, bn):
    torch.manual_seed(M + N + K)
    A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    bias = (torch.randn(N, device="cuda") * 0.1).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _run(A, B, out, bias, 0, 1.0, bn)
    ref = A.float() @ B.float().t() + bias.float()
    err = (out.float() - ref).abs().max().item()
    assert err <= 8e-3 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K", [(300, 1024, 256), (1344, 4096, 2048)])
def test_gemm_f32_scaled(M, N, K):
    torch.manual_seed(1)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    _run(A, B, out, None, 1, 3.0)
    ref = (A.float() @ B.float().t()) * 3.0
    assert (out - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()


def test_gemm_residual_add():
    torch.manual_seed(2)
    M, N, K = 777, 2048, 2048
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    R = torch.randn(M, N, device="cuda")
    out = R.clone()
    _run(A, B, out, None, 2)
    ref = R + A.float() @ B.float().t()
    assert (out - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()


@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_tile_width_does_not_change_results(epi):
    """Every supported BLOCK_N gives bitwise-identical outputs (same K order per element), so
    the M-dependent automatic tile choice keeps rows invariant to the batch they sit in."""
    torch.manual_seed(5)
    M, N, K = 700, 2560, 2048
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    bias = (torch.randn(N, device="cuda") * 0.1).bfloat16()
    outs = []
    for bn in (256, 224, 192, 160, 128):
        if epi == 0:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        else:
            out = torch.ones(M, N, device="cuda", dtype=torch.float32)
        _run(A, B, out, bias if epi == 0 else None, epi, 1.0, bn)
        outs.append(out)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("splits", [2, 3, 5])
def test_gemm_residual_split_k_deterministic_and_row_invariant(splits):
    """Split-K partials are added in split order: repeated runs are bitwise identical and a
    row's result does not depend on M (the same rows inside a larger batch)."""
    torch.manual_seed(4)
    M, N, K = 1344, 2048, 11008
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.01).bfloat16()
    R = torch.randn(M, N, device="cuda")
    outs = []
    for _ in range(2):
        out = R.clone()
        _run(A, B, out, None, 2, splits=splits)
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    ref = R + A.float() @ B.float().t()
    assert (outs[0] - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()
    small = R[:64].clone()
    _run(A[:64].contiguous(), B, small, None, 2, splits=splits)
    assert torch.equal(small, outs[0][:64])


def test_gemm_swiglu():
    torch.manual_seed(3)
    M, F, K = 333, 512, 256  # N = 2F interleaved per 256-row block: [128 gate, 128 up]
    A = torch.randn(M, K, device="cuda").bfloat16()
    G = (torch.randn(F, K, device="cuda") * 0.05).bfloat16()
    U = (torch.randn(F, K, device="cuda") * 0.05).bfloat16()
    B = torch.cat([torch.cat([G[b * 128:(b + 1) * 128], U[b * 128:(b + 1) * 128]]) for b in range(F // 128)])
    out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    _run(A, B.contiguous(), out, None, 3)
    g, u = A.float() @ G.float().t(), A.float() @ U.float().t()
    ref = torch.nn.functional.silu(g) * u
    assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("M,N,K,tau", [(256, 151936, 2048, 1.0), (37, 4104, 256, 0.7), (130, 1024, 128, 1.3)])
def test_lm_head_fused_stats_bitwise(M, N, K, tau):
    """LM-head epilogue softmax partials == the stand-alone row-stats kernel, BITWISE (same
    tile order, tilestat.cuh), and == a torch fp64 restatement within 1e-12 relative."""
    torch.manual_seed(N)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    B[5] = 0  # a constant column (ties inside one tile)
    nt = (N + 255) // 256
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    fused = torch.full((M, nt, 2), float("nan"), device="cuda", dtype=torch.float64)
    sep = torch.full_like(fused, float("nan"))
    dev = rb.default_device()
    torch.cuda.synchronize()
    rb._check(rb.lib().rs_lm_head_bf16(dev.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(fused.data_ptr()),
                                       M, N, K, 2.0, tau))
    rb._check(rb.lib().rs_row_stats(dev.handle, ctypes.c_void_p(out.data_ptr()), M, N, tau,
                                    ctypes.c_void_p(sep.data_ptr())))
    dev.sync()
    ref = (A.float() @ B.float().t()) * 2.0
    assert (out - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()
    assert torch.equal(fused, sep)
    y = out.double()[:, : N - 1]
    y = y / torch.full_like(y, tau)  # true division (a python-scalar divisor may become a reciprocal multiply)
    pad = nt * 256 - (N - 1)
    y = torch.nn.functional.pad(y, (0, pad), value=float("-inf")).view(M, nt, 256)
    m = y.max(-1).values
    s = torch.exp(y - m[..., None]).sum(-1)
    assert torch.equal(fused[..., 0], m)
    assert torch.allclose(fused[..., 1], s, rtol=1e-12, atol=0)


@pytest.fixture
def gemm_path():
    yield
    rb.set_tuning("gemm2", 0)


@pytest.mark.parametrize("T,F,K", [(1344, 2560, 2048), (37, 512, 256), (300, 2048, 11008), (1344, 151936, 2048)])
@pytest.mark.parametrize("epi", [0, 1, 2, 4])
def test_gemm_sm_pair_matches_torch(gemm_path, T, F, K, epi):
    """Weight GEMMs on SM pairs (cta_group::2, weights as the 256-row M operand) vs torch fp32,
    for every epilogue the forward uses (bias/bf16, scaled fp32, residual add, pairwise SwiGLU)."""
    if epi == 4 and F > 30000:
        pytest.skip("LM-head shape only for the plain epilogues")
    rb.set_tuning("gemm2", 0)
    torch.manual_seed(T + F)
    A = (torch.randn(T, K, device="cuda") * 0.5).bfloat16()
    B = (torch.randn(F, K, device="cuda") * 0.03).bfloat16()
    bias = (torch.randn(F, device="cuda") * 0.1).bfloat16()
    ref = A.float() @ B.float().t()
    if epi == 0:
        out = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
        _run(A, B, out, bias, 0)
        want = ref + bias.float()
        tol = 8e-3
    elif epi == 1:
        out = torch.empty(T, F, device="cuda", dtype=torch.float32)
        _run(A, B, out, None, 1, 2.0)
        want, tol = ref * 2.0, 2e-3
    elif epi == 2:
        base = torch.randn(T, F, device="cuda")
        out = base.clone()
        _run(A, B, out, None, 2)
        want, tol = base + ref, 2e-3
    else:
        out = torch.empty(T, F // 2, device="cuda", dtype=torch.bfloat16)
        _run(A, B, out, None, 4)
        g, u = ref[:, 0::2], ref[:, 1::2]
        want, tol = torch.nn.functional.silu(g) * u, 1e-2
    err = (out.float() - want).abs().max().item()
    assert err <= tol * want.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("epi", [0, 2, 4])
def test_gemm_sm_pair_token_tile_invariance(gemm_path, epi):
    """A token's outputs are bitwise independent of the token tile (64 .. 256) it lands in --
    the K order per output is fixed, which keeps the forward row-invariant."""
    rb.set_tuning("gemm2", 0)
    torch.manual_seed(5)
    T, F, K = 517, 1024, 2048
    A = torch.randn(T, K, device="cuda").bfloat16()
    B = (torch.randn(F, K, device="cuda") * 0.03).bfloat16()
    bias = (torch.randn(F, device="cuda") * 0.1).bfloat16()
    outs = []
    base = torch.randn(T, F, device="cuda")
    for bt in (64, 96, 128, 160, 192, 224, 256):
        if epi == 0:
            out = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
            _run(A, B, out, bias, 0, 1.0, bt)
        elif epi == 2:
            out = base.clone()
            _run(A, B, out, None, 2, 1.0, bt)
        else:
            out = torch.empty(T, F // 2, device="cuda", dtype=torch.bfloat16)
            _run(A, B, out, None, 4, 1.0, bt)
        outs.append(out)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    # and a row computed alone equals the same row inside the batch
    one = torch.empty(1, F, device="cuda", dtype=torch.bfloat16) if epi != 2 else base[7:8].clone()
    if epi == 4:
        one = torch.empty(1, F // 2, device="cuda", dtype=torch.bfloat16)
    _run(A[7:8].contiguous(), B, one, bias if epi == 0 else None, epi)
    assert torch.equal(one[0], outs[0][7])


def test_gemm_split_k_on_sm_pairs(gemm_path):
    rb.set_tuning("gemm2", 0)
    torch.manual_seed(3)
    T, F, K = 600, 2048, 11008
    A = (torch.randn(T, K, device="cuda") * 0.5).bfloat16()
    B = (torch.randn(F, K, device="cuda") * 0.02).bfloat16()
    base = torch.randn(T, F, device="cuda")
    o1, o3, o3b = base.clone(), base.clone(), base.clone()
    _run(A, B, o1, None, 2, 1.0, 0, 1)
    _run(A, B, o3, None, 2, 1.0, 0, 3)
    _run(A, B, o3b, None, 2, 1.0, 0, 3)
    assert torch.equal(o3, o3b)  # deterministic split order
    ref = base + A.float() @ B.float().t()
    assert (o3 - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()
    assert (o1 - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()



@pytest.fixture
def epi3_default():
    yield
    rb.set_tuning("epi3", 0)


@pytest.mark.parametrize("T,F,K,epi", [(1344, 2048, 2048, 2), (1344, 2048, 11008, 2), (1344, 2560, 2048, 0),
                                       (300, 2048, 2048, 4), (256, 2048, 4096, 1)])
def test_gemm_third_epilogue_group_bitwise(gemm_path, epi3_default, T, F, K, epi):
    """Single-wave launches hand a third of the accumulator chunks to the control warps
    (tuning key "epi3"); the outputs are bitwise those of the two-group epilogue."""
    rb.set_tuning("gemm2", 0)
    torch.manual_seed(T + F + K)
    A = (torch.randn(T, K, device="cuda") * 0.5).bfloat16()
    B = (torch.randn(F, K, device="cuda") * 0.03).bfloat16()
    bias = (torch.randn(F, device="cuda") * 0.1).bfloat16()
    base = torch.randn(T, F, device="cuda")
    outs = []
    for v in (0, -1):
        rb.set_tuning("epi3", v)
        if epi == 0:
            out = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
            _run(A, B, out, bias, 0)
        elif epi == 1:
            out = torch.empty(T, F, device="cuda", dtype=torch.float32)
            _run(A, B, out, None, 1, 0.5)
        elif epi == 2:
            out = base.clone()
            _run(A, B, out, None, 2)
        else:
            out = torch.empty(T, F // 2, device="cuda", dtype=torch.bfloat16)
            _run(A, B, out, None, 4)
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    ref = A.float() @ B.float().t()
    want = {0: ref + bias.float(), 1: ref * 0.5, 2: base + ref}.get(epi)
    if want is not None:
        assert (outs[0].float() - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-3
