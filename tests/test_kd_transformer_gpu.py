"""GPU: K5 for EAGLE drafters -- reward-weighted KL distillation loss and the gradient of EVERY
drafter tensor (kd_update, learner.cpp:98-160, with the target rows recomputed by the target;
the reference's gradient covers the whole model, learner.cpp:62-82 / :146-151).

Against a plain PyTorch fp32 restatement on the same synthetic weights (tests/torch_ref.py):
  loss = sum_i w_i sum_t KL(p~_t || q_t)      (learner.cpp:33-60)
  dW   = logit_scale * sum dZ_t^T h_t,  dZ = w (q - p~) / tau   (learner.cpp:62-82)
Tolerances: the forwards run bf16 activations with fp32 accumulation (logits within 3e-2 of
their scale, test_transformer_gpu.py) and dZ enters the tensor-core GEMM as bf16 -- loss within
2e-2 relative, gradient within 3e-2 of its max magnitude. The update itself is checked exactly:
new w == bf16(w - lr * grad) for every tensor and version + 1; the gradient is bitwise
reproducible. The whole-drafter gradient (LM head, final norm, MLP, post-attention norm, O,
causal attention, RoPE, QKV + bias, input norms, fc) is checked tensor by tensor against torch
autograd through the same forward (test_whole_drafter_grad_matches_autograd)."""
import random

import pytest
import torch

import paper_2510_26475_b200 as rb
from torch_ref import DrafterRef, TargetRef

pytestmark = pytest.mark.gpu

SHAPE = rb.TransformerShape.tiny(vocab=1024, max_ctx=256)


@pytest.fixture(scope="module")
def models():
    tgt = rb.TransformerModel(SHAPE, seed=31)
    drf = rb.EagleDrafter(tgt, seed=32, version=5)
    return tgt, drf


def samples(n=5, seed=1):
    rng = random.Random(seed)
    out = []
    for i in range(n):
        p = [rng.randrange(SHAPE.vocab - 1) for _ in range(3 + i)]
        r = [rng.randrange(SHAPE.vocab) for _ in range(4 + 3 * i)]
        out.append(rb.RolloutSample(p, r, [], eos_bias=[-1.0, 0.0, 0.5, -2.0, 1.0][i % 5], reward=rng.random()))
    return out


def torch_kd(tgt, drf, ss, ws, tau=1.0):
    tref = TargetRef(tgt)
    dref = DrafterRef(drf, tref)
    V, d = SHAPE.vocab, SHAPE.d_model
    loss = 0.0
    dW = torch.zeros(V, d, dtype=torch.float64, device="cuda")
    for s, w in zip(ss, ws):
        toks = s.prompt + s.response
        P = len(s.prompt)
        zt, feats = tref.forward(toks)
        T = len(toks)
        prev = torch.zeros(T, 3 * d, device="cuda")
        prev[1:] = feats[:-1].reshape(T - 1, 3 * d)
        f = prev @ dref.fc.t()
        zq, x = dref._layer_logits(toks, f)
        hn = tref.rms(x, dref.final)
        rows = slice(P - 1, T - 1)
        a, b = zt[rows].double().clone(), zq[rows].double().clone()
        a[:, -1] += s.eos_bias
        b[:, -1] += s.eos_bias
        lp, lq = torch.log_softmax(a / tau, -1), torch.log_softmax(b / tau, -1)
        p, q = lp.exp(), lq.exp()
        loss += w * float((p * (lp - lq)).sum())
        dz = w * (q - p) / tau * SHAPE.logit_scale
        dW += dz.t() @ hn[rows].double()
    return loss, dW


def test_kd_loss_and_lm_grad_match_torch(models):
    tgt, drf = models
    ss = samples()
    ws = [0.5, 1.0, 2.0, 0.0, 1.5]
    loss, gb = rb.kd_grad_transformer(drf, ss, ws)
    rl, rg = torch_kd(tgt, drf, ss, ws)
    assert loss == pytest.approx(rl, rel=2e-2)
    g = gb.to_torch(*drf.grad_layout("lm_w")).view(SHAPE.vocab, SHAPE.d_model)
    err = (g.double() - rg).abs().max().item()
    assert err <= 3e-2 * rg.abs().max().item(), (err, rg.abs().max().item())
    # bitwise reproducible (every tensor), and accumulation adds
    loss2, g2 = rb.kd_grad_transformer(drf, ss, ws)
    assert loss2 == loss and torch.equal(gb.to_torch(), g2.to_torch())
    _, g3 = rb.kd_grad_transformer(drf, ss, ws, grad=g2.clone(), zero_grad=False)
    assert torch.allclose(g3.to_torch(), 2 * gb.to_torch(), rtol=1e-6, atol=1e-7)


def test_kd_non_unit_temperature_matches_torch():
    """tau != 1 takes K5's general path (the unit-temperature kernel skips the divisions)."""
    shape = rb.TransformerShape.tiny(vocab=1024, max_ctx=256, temperature=0.7)
    tgt = rb.TransformerModel(shape, seed=31)
    drf = rb.EagleDrafter(tgt, seed=32, version=5)
    ss = samples(4, seed=5)
    ws = [1.0, 0.5, 2.0, 1.5]
    loss, gb = rb.kd_grad_transformer(drf, ss, ws)
    rl, rg = torch_kd(tgt, drf, ss, ws, tau=0.7)
    assert loss == pytest.approx(rl, rel=2e-2)
    g = gb.to_torch(*drf.grad_layout("lm_w")).view(shape.vocab, shape.d_model)
    err = (g.double() - rg).abs().max().item()
    assert err <= 3e-2 * rg.abs().max().item(), (err, rg.abs().max().item())
    # and differs from the unit-temperature gradient of the same weights
    _, g1 = rb.kd_grad_transformer(rb.EagleDrafter(rb.TransformerModel(SHAPE, seed=31), seed=32, version=5), ss, ws)
    assert not torch.equal(g1.to_torch(), gb.to_torch())


def test_kd_weights_are_linear(models):
    _, drf = models
    ss = samples(3, seed=7)
    l1, g1 = rb.kd_grad_transformer(drf, ss, [1.0, 1.0, 1.0])
    l2, g2 = rb.kd_grad_transformer(drf, ss, [2.0, 2.0, 2.0])
    assert l2 == pytest.approx(2 * l1, rel=1e-12)
    a, b = g1.to_torch(), g2.to_torch()
    assert (b - 2 * a).norm().item() <= 2e-2 * (2 * a).norm().item()
    l0, g0 = rb.kd_grad_transformer(drf, ss, [0.0, 0.0, 0.0])
    assert l0 == 0.0 and not g0.to_torch().any()


def test_kd_update_snapshot_and_sgd(models):
    tgt, drf = models
    ss = samples(6, seed=3)
    pol = rb.KDPolicy(interval=2, mode=0, clip_lo=0.0, clip_hi=4.0, lr=0.5)
    rng_a, rng_b = rb.SelectionRng(123), rb.SelectionRng(123)
    from paper_2510_26475_b200.distributed import kd_select
    sel = kd_select(len(ss), pol.interval, rng_b)
    br = [ss[i].reward for i in sel]
    ws = [rb.kd_weight(ss[i].reward, br, pol) for i in sel]
    res = rb.kd_update(drf, ss, pol, rng_a, 0.02)
    assert res.updated and res.samples_used == len(sel) == 3
    assert res.drafter.version == drf.version + 1
    assert res.sim_time == pytest.approx(0.02 * sum(len(ss[i].response) for i in sel))
    loss, g = rb.kd_grad_transformer(drf, [ss[i] for i in sel], ws)
    assert res.loss == loss
    for name in rb.EagleDrafter.GRAD_TENSORS:  # every tensor moves: w - lr * grad
        old = drf.to_torch(name).float()
        new = res.drafter.to_torch(name)
        gt = g.to_torch(*drf.grad_layout(name))
        want = old - 0.5 * gt
        assert torch.equal(new, want.to(new.dtype)), name
        if name in ("lm_w", "fc_w", "o_w", "down_w"):
            assert not torch.equal(new, old.to(new.dtype)), name
    # the updated drafter generates through the engine
    eng = rb.BatchEngine(tgt, lambda: res.drafter, None, rb.TimingModel(),
                         [rb.RequestState(0, [1, 2, 3], 0.0, 6, rb.DecodeRng.from_seed(1, 0))],
                         rb.SDConfig.tree(1, 2, 2), "sample", record_full_logprobs=False)
    while not eng.all_done():
        eng.step()
    assert len(eng.requests()[0].generated) == 6


def test_kd_update_errors_and_empty(models):
    _, drf = models
    with pytest.raises(rb.LogicError):
        rb.kd_update(drf, samples(2), rb.KDPolicy(mode=2), rb.SelectionRng(1), 0.0)
    res = rb.kd_update(drf, [], rb.KDPolicy(), rb.SelectionRng(1), 0.0)
    assert not res.updated and res.drafter.version == drf.version


def test_distributed_step_single_rank(models):
    """The prompt-sharded step with one rank == kd_update (same selection, weights, SGD)."""
    from paper_2510_26475_b200.distributed import kd_step_distributed_transformer
    tgt, drf = models
    ss = samples(4, seed=11)
    pol = rb.KDPolicy(interval=1, mode=0, lr=0.25)
    st = kd_step_distributed_transformer(drf, [s.reward for s in ss], [len(s.response) for s in ss], ss,
                                         list(range(len(ss))), pol, rb.SelectionRng(9), 0.01)
    ref = rb.kd_update(drf, ss, pol, rb.SelectionRng(9), 0.01)
    assert st.loss == pytest.approx(ref.loss, rel=1e-12)
    assert torch.equal(st.drafter.to_torch("lm_w"), ref.drafter.to_torch("lm_w"))


def _engine_rollouts(tgt, drf, n=4, seed=3, max_len=9):
    rng = random.Random(seed)
    reqs = [rb.RequestState(i, [rng.randrange(SHAPE.vocab - 1) for _ in range(4 + 3 * i)], -2.0 + 0.5 * i,
                            max_len + i, rb.DecodeRng.from_seed(17, i)) for i in range(n)]
    return rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 2, 3), "sample",
                          record_full_logprobs=False)


@pytest.mark.parametrize("kd_rows", [0, 7])
def test_engine_kd_grad_matches_recompute(models, kd_rows):
    """rs_engine_kd_grad (resident KV cache + features, response positions only through the
    target) == kd_grad_transformer (teacher-forced recompute of prompt + response): identical
    per-row losses (so an identical total), the same gradient -- bitwise when both use one group,
    to fp32 grouping otherwise (kd_rows=7 forces several groups and drafter chunks)."""
    tgt, drf = models
    other = rb.EagleDrafter(tgt, seed=77, version=9)  # KD drafter != the engine's drafter
    eng = _engine_rollouts(tgt, drf)
    while not eng.all_done():
        eng.step()
    reqs = eng.requests()
    ids = [0, 2, 3, 1]
    ws = [0.5, 1.5, 1.0, 2.0]
    ss = [rb.RolloutSample(list(reqs[i].prompt), list(reqs[i].generated), [], reqs[i].eos_bias) for i in ids]
    rb.set_tuning("kd_rows", kd_rows)
    try:
        loss_e, g_e = eng.kd_grad(other, ids, ws)
    finally:
        rb.set_tuning("kd_rows", 0)
    loss_r, g_r = rb.kd_grad_transformer(other, ss, ws)
    assert loss_e == loss_r
    a, b = g_e.to_torch(), g_r.to_torch()
    if kd_rows == 0:
        assert torch.equal(a, b)
    else:
        for name in rb.EagleDrafter.GRAD_TENSORS:
            o, n = other.grad_layout(name)
            x, y = a[o:o + n], b[o:o + n]
            assert (x - y).abs().max().item() <= 1e-4 * y.abs().max().item(), name


def test_engine_kd_grad_leaves_engine_state(models):
    """A KD pass in the middle of a rollout does not perturb the rollout (private drafter cache;
    target keys rewritten bit-identically)."""
    tgt, drf = models
    a, b = _engine_rollouts(tgt, drf, max_len=14), _engine_rollouts(tgt, drf, max_len=14)
    for _ in range(2):
        a.step()
        b.step()
    a.kd_grad(rb.EagleDrafter(tgt, seed=78), [0, 1, 2, 3], [1.0] * 4)
    while not a.all_done():
        a.step()
    while not b.all_done():
        b.step()
    assert [r.generated for r in a.requests()] == [r.generated for r in b.requests()]


def _bf_st(x):
    """bf16 rounding in the forward, identity in the backward (the CUDA path keeps fp32 grads)."""
    return x + (x.to(torch.bfloat16).float() - x).detach()


def torch_kd_full(tgt, drf, ss, ws):
    """Autograd through the drafter forward of tests/torch_ref.py (same bf16 rounding points),
    loss = sum_i w_i sum_t KL(p~_t || q_t) over the response positions; returns the loss and the
    gradient of every drafter tensor in the library's layout (gate / up interleaved pairwise)."""
    tref = TargetRef(tgt)
    s = drf.shape
    d, H, KV, hd = s.d_model, s.n_heads, s.n_kv_heads, s.head_dim
    q = (H + 2 * KV) * hd
    W = {n: drf.to_torch(n).float().clone().requires_grad_(True) for n in rb.EagleDrafter.GRAD_TENSORS}
    fc, ne, nh = W["fc_w"].view(d, 3 * d), W["norm_emb"], W["norm_hid"]
    qkv_w, qkv_b = W["qkv_w"].view(q, 2 * d), W["qkv_b"]
    o_w, ln2 = W["o_w"].view(d, H * hd), W["ln2"]
    gu = W["gu_w"].view(2 * s.d_ff, d)
    g_w, u_w = gu[0::2], gu[1::2]
    down, fin, lm = W["down_w"].view(d, s.d_ff), W["final_norm"], W["lm_w"].view(s.vocab, d)

    def rms(x, w):
        return _bf_st(x * torch.rsqrt((x * x).mean(-1, keepdim=True) + s.rms_eps) * w)

    def rope(x, pos):
        half = hd // 2
        inv = torch.tensor([s.rope_theta ** (-2.0 * i / hd) for i in range(half)], dtype=torch.float64, device="cuda")
        ang = pos.double()[:, None] * inv[None]
        c, sn = torch.cos(ang).float()[:, None], torch.sin(ang).float()[:, None]
        x1, x2 = x[..., :half], x[..., half:]
        return _bf_st(torch.cat([x1 * c - x2 * sn, x2 * c + x1 * sn], -1))

    loss = 0.0
    for smp, w in zip(ss, ws):
        toks = smp.prompt + smp.response
        P, T = len(smp.prompt), len(smp.prompt) + len(smp.response)
        with torch.no_grad():
            zt, feats = tref.forward(toks)
        rows = T - 1  # positions 0..T-2
        prev = torch.zeros(rows, 3 * d, device="cuda")
        prev[1:] = feats[:rows - 1].reshape(rows - 1, 3 * d)
        f = prev @ fc.t()
        tok = torch.tensor(toks[:rows], device="cuda")
        pos = torch.arange(rows, device="cuda")
        e = tref.emb[tok]
        h = torch.cat([rms(e, ne), rms(f, nh)], -1)
        qkv = _bf_st(h @ qkv_w.t() + qkv_b)
        qq = rope(qkv[:, :H * hd].view(rows, H, hd), pos)
        kk = rope(qkv[:, H * hd:(H + KV) * hd].view(rows, KV, hd), pos)
        vv = qkv[:, (H + KV) * hd:].view(rows, KV, hd)
        G = H // KV
        kr, vr = kk.repeat_interleave(G, 1), vv.repeat_interleave(G, 1)
        sc = torch.einsum("thd,shd->hts", qq, kr) / hd ** 0.5
        mask = torch.triu(torch.ones(rows, rows, dtype=torch.bool, device="cuda"), 1)
        pr = torch.softmax(sc.masked_fill(mask, float("-inf")), -1)
        ao = _bf_st(torch.einsum("hts,shd->thd", pr, vr)).reshape(rows, H * hd)
        x = f + ao @ o_w.t()
        h2 = rms(x, ln2)
        x = x + _bf_st(torch.nn.functional.silu(h2 @ g_w.t()) * (h2 @ u_w.t())) @ down.t()
        zq = (rms(x, fin) @ lm.t()) * s.logit_scale
        kd = slice(P - 1, rows)
        a = zt[kd].double().clone()
        b = zq[kd].double()
        a[:, -1] += smp.eos_bias
        b = torch.cat([b[:, :-1], b[:, -1:] + smp.eos_bias], 1)
        lp, lq = torch.log_softmax(a, -1), torch.log_softmax(b, -1)
        loss = loss + w * (lp.exp() * (lp - lq)).sum()
    loss.backward()
    return float(loss), {n: W[n].grad.detach().reshape(-1) for n in W}


def test_whole_drafter_grad_matches_autograd(models):
    """Every drafter tensor's gradient vs torch autograd (relative Frobenius error; the backward
    GEMMs take bf16 operands, fp32 accumulation)."""
    tgt, drf = models
    ss = samples(3, seed=5)
    ws = [0.7, 1.3, 1.0]
    loss, g = rb.kd_grad_transformer(drf, ss, ws)
    rl, ref = torch_kd_full(tgt, drf, ss, ws)
    assert loss == pytest.approx(rl, rel=2e-2)
    gt = g.to_torch()
    errs = {}
    for name in rb.EagleDrafter.GRAD_TENSORS:
        o, n = drf.grad_layout(name)
        x, y = gt[o:o + n].double(), ref[name].double()
        errs[name] = ((x - y).norm() / y.norm().clamp_min(1e-30)).item()
    print("whole-drafter grad rel. errors:", {k: round(v, 4) for k, v in errs.items()})
    assert all(v < 5e-2 for v in errs.values()), errs


def test_whole_drafter_grad_gqa8_matches_autograd():
    """The attention backward stacks a GQA group's query heads; G = 8 as at Qwen2.5-3B (one KV head
    of eight query heads, hd = 128) against torch autograd."""
    shape = rb.TransformerShape(1024, 1024, 2, 8, 1, 128, 512, 256)
    tgt = rb.TransformerModel(shape, seed=41)
    drf = rb.EagleDrafter(tgt, seed=42, version=1)
    rng = random.Random(9)
    ss = [rb.RolloutSample([rng.randrange(shape.vocab - 1) for _ in range(20 + 7 * i)],
                           [rng.randrange(shape.vocab) for _ in range(9 + 5 * i)], [], eos_bias=0.25 * i,
                           reward=rng.random()) for i in range(3)]
    ws = [0.7, 1.3, 1.0]
    loss, g = rb.kd_grad_transformer(drf, ss, ws)
    rl, ref = torch_kd_full(tgt, drf, ss, ws)
    assert loss == pytest.approx(rl, rel=2e-2)
    gt = g.to_torch()
    errs = {}
    for name in rb.EagleDrafter.GRAD_TENSORS:
        o, n = drf.grad_layout(name)
        x, y = gt[o:o + n].double(), ref[name].double()
        errs[name] = ((x - y).norm() / y.norm().clamp_min(1e-30)).item()
    assert all(v < 5e-2 for v in errs.values()), errs
