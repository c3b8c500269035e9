"""GPU: K5 for EAGLE drafters -- reward-weighted KL distillation loss and the drafter LM-head
gradient (kd_update, learner.cpp:98-160, with the target rows recomputed by the target).

Against a plain PyTorch fp32 restatement on the same synthetic weights (tests/torch_ref.py):
  loss = sum_i w_i sum_t KL(p~_t || q_t)      (learner.cpp:33-60)
  dW   = logit_scale * sum dZ_t^T h_t,  dZ = w (q - p~) / tau   (learner.cpp:62-82)
Tolerances: the forwards run bf16 activations with fp32 accumulation (logits within 3e-2 of
their scale, test_transformer_gpu.py) and dZ enters the tensor-core GEMM as bf16 -- loss within
2e-2 relative, gradient within 3e-2 of its max magnitude. The update itself is checked exactly:
new lm_w == bf16(lm_w - lr * grad) and version + 1; the gradient is bitwise reproducible."""
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


def torch_kd(tgt, drf, ss, ws):
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
        lp, lq = torch.log_softmax(a, -1), torch.log_softmax(b, -1)
        p, q = lp.exp(), lq.exp()
        loss += w * float((p * (lp - lq)).sum())
        dz = w * (q - p) * SHAPE.logit_scale
        dW += dz.t() @ hn[rows].double()
    return loss, dW


def test_kd_loss_and_lm_grad_match_torch(models):
    tgt, drf = models
    ss = samples()
    ws = [0.5, 1.0, 2.0, 0.0, 1.5]
    loss, g = rb.kd_grad_transformer(drf, ss, ws)
    rl, rg = torch_kd(tgt, drf, ss, ws)
    assert loss == pytest.approx(rl, rel=2e-2)
    err = (g.double() - rg).abs().max().item()
    assert err <= 3e-2 * rg.abs().max().item(), (err, rg.abs().max().item())
    # bitwise reproducible, and accumulation adds
    loss2, g2 = rb.kd_grad_transformer(drf, ss, ws)
    assert loss2 == loss and torch.equal(g, g2)
    _, g3 = rb.kd_grad_transformer(drf, ss, ws, grad=g2.clone(), zero_grad=False)
    assert torch.allclose(g3, 2 * g, rtol=1e-6, atol=1e-7)


def test_kd_weights_are_linear(models):
    _, drf = models
    ss = samples(3, seed=7)
    l1, g1 = rb.kd_grad_transformer(drf, ss, [1.0, 1.0, 1.0])
    l2, g2 = rb.kd_grad_transformer(drf, ss, [2.0, 2.0, 2.0])
    assert l2 == pytest.approx(2 * l1, rel=1e-12)
    assert torch.allclose(g2, 2 * g1, rtol=1e-2, atol=1e-6)
    l0, g0 = rb.kd_grad_transformer(drf, ss, [0.0, 0.0, 0.0])
    assert l0 == 0.0 and not g0.any()


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
    V, d = SHAPE.vocab, SHAPE.d_model
    old = drf.to_torch("lm_w").view(V, d).float()
    new = res.drafter.to_torch("lm_w").view(V, d)
    assert torch.equal(new, (old - 0.5 * g).bfloat16())
    assert torch.equal(res.drafter.to_torch("fc_w"), drf.to_torch("fc_w"))
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
    if kd_rows == 0:
        assert torch.equal(g_e, g_r)
    else:
        assert (g_e - g_r).abs().max().item() <= 1e-5 * g_r.abs().max().item()


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
