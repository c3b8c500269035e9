"""GPU: the single-sequence API -- spec_step_tree / spec_step_chain / generate / mean_accept_len
(specdec.hpp:98-131) -- on the device engine against the compiled reference
(tests/test_specdec.cpp's cases: cycle-by-cycle continuation of one DecodeRng&, chain == tree(1,1,k)
token for token, drafter == target accepts every drafted token, max_len / EOS edges).

Tokens, accept lengths, bonus tokens, round costs and draft-record counts are exact; logprobs
within 1e-12 (test_specdec.cpp:99-116)."""
import random

import pytest

import paper_2510_26475_b200 as rb
from helpers import model_of

pytestmark = pytest.mark.gpu


def _models(seed, V, to=1, do=0, scale=1.0):
    rng = random.Random(seed)
    t = {"vocab": V, "order": to, "logits": [rng.gauss(0, scale) for _ in range(V ** to * V)]}
    d = {"vocab": V, "order": do, "logits": [rng.gauss(0, scale) for _ in range(V ** do * V)]}
    return t, d


def _cfg(c):
    return rb.SDConfig(c["s"], c["t"], c["n"], True)


def _same_steps(got, exp, full=True):
    assert [s.token for s in got] == [e["token"] for e in exp]
    assert [s.drafted for s in got] == [e["drafted"] for e in exp]
    for s, e in zip(got, exp):
        assert s.logp == pytest.approx(e["logp"], abs=1e-12)
        if e["drafted"]:
            assert s.logq == pytest.approx(e["logq"], abs=1e-12)
        if full and "target_logprobs" in e:
            assert max(abs(a - b) if a != b else 0.0 for a, b in zip(s.target_logprobs, e["target_logprobs"])) < 1e-12


CASES = [(1, 8, {"s": 1, "t": 1, "n": 3}, 0.0), (2, 8, {"s": 2, "t": 2, "n": 2}, 0.5), (3, 20, {"s": 1, "t": 4, "n": 5}, -1.0),
         (4, 50, {"s": 3, "t": 3, "n": 2}, 1.5), (5, 8, {"s": 1, "t": 2, "n": 4}, 3.0)]


@pytest.mark.parametrize("seed,V,c,bias", CASES)
def test_spec_step_tree_cycles_match_reference(reference, seed, V, c, bias):
    t, d = _models(seed, V)
    ctx = [1, 2]
    exp = reference("spec_step_tree", target=t, drafter=d, ctx=ctx, cfg=dict(c, enabled=True), seed=77, stream=seed,
                    cycles=4, advance_ctx=True, record_logprobs=True, eos_bias=bias)["outcomes"]
    T, D = model_of(t), model_of(d)
    rng = rb.DecodeRng.from_seed(77, seed)
    cur = list(ctx)
    for e in exp:
        o = rb.spec_step_tree(T, D, cur, _cfg(c), rng, bias)
        assert o.accepted_tokens == e["accepted_tokens"]
        assert o.accept_len == e["accept_len"] and o.bonus_token == e["bonus_token"] and o.ended == e["ended"]
        assert [[r.drafter_forwards, r.drafter_tokens_each, r.target_tokens] for r in o.rounds] == e["rounds"]
        assert o.draft_records == e["draft_records"]
        _same_steps(o.steps, e["steps"])
        cur += o.accepted_tokens


def test_chain_equals_tree_t1_token_for_token():
    """test_specdec.cpp:118-131: tree(1,1,k) reproduces spec_step_chain(k)."""
    t, d = _models(11, 8)
    T, D = model_of(t), model_of(d)
    for stream in range(12):
        ra, rb_ = rb.DecodeRng.from_seed(5, stream), rb.DecodeRng.from_seed(5, stream)
        ca, cb = [3], [3]
        for _ in range(3):
            a = rb.spec_step_chain(T, D, ca, 3, ra)
            b = rb.spec_step_tree(T, D, cb, rb.SDConfig.tree(1, 1, 3), rb_)
            assert a.accepted_tokens == b.accepted_tokens and a.accept_len == b.accept_len
            ca += a.accepted_tokens
            cb += b.accepted_tokens


def test_drafter_equal_target_accepts_every_token():
    """test_specdec.cpp:76-85: drafter == target -> accept_len = k, k + 1 tokens (no EOS)."""
    t, _ = _models(12, 8)
    T = model_of(t)
    rng = rb.DecodeRng.from_seed(1, 0)
    o = rb.spec_step_tree(T, T, [0, 1], rb.SDConfig.chain(4), rng, -30.0)
    assert o.accept_len == 4 and len(o.accepted_tokens) == 5 and o.bonus_token == o.accepted_tokens[-1]


@pytest.mark.parametrize("cfg,max_len,bias,stop", [({"s": 1, "t": 2, "n": 3}, 12, 0.0, True),
                                                   ({"s": 2, "t": 1, "n": 2}, 1, 0.0, True),
                                                   ({"s": 1, "t": 4, "n": 5}, 2, 0.0, True),
                                                   ({"s": 1, "t": 3, "n": 2}, 30, 2.5, True),
                                                   ({"s": 1, "t": 2, "n": 3}, 25, 2.5, False),
                                                   (None, 9, 0.5, True)])
def test_generate_matches_reference(reference, cfg, max_len, bias, stop):
    t, d = _models(21, 8)
    c = dict(cfg, enabled=True) if cfg else {"enabled": False}
    exp = reference("generate", target=t, drafter=d, prompt=[1, 2], cfg=c, max_len=max_len, seed=9, stream=4,
                    eos_bias=bias, stop_at_eos=stop)
    sd = rb.SDConfig(c.get("s", 1), c.get("t", 1), c.get("n", 1), c["enabled"])
    g = rb.generate(model_of(t), model_of(d), [1, 2], sd, max_len, rb.DecodeRng.from_seed(9, 4), bias, stop)
    assert g.tokens == exp["tokens"] and g.accept_lens == exp["accept_lens"] and g.ended_eos == exp["ended_eos"]
    assert [list(e) for e in g.ledger] == exp["ledger"]
    _same_steps(g.steps, exp["steps"], full=False)
    if g.accept_lens:
        assert rb.mean_accept_len(g.accept_lens) == exp["mean_accept_len"]
    with pytest.raises(rb.InvalidArgument, match="no verification cycles"):
        rb.mean_accept_len([])


def test_kd_loss_and_gradient_match_reference(reference):
    """kd_loss / kd_loss_gradient (learner.hpp:32-37) on the device vs the reference (1e-10 / 1e-12,
    test_learner.cpp:93-110)."""
    from conftest import load_golden
    g = load_golden("kd_update.json")
    buf = g["buffer"][:6]
    ws = [0.5, 1.0, 2.0, 0.0, 1.5, 3.0]
    exp = reference("kd_grad", drafter=g["drafter"], samples=buf, weights=ws)
    drafter = model_of(g["drafter"])
    samples = [rb.RolloutSample(s["prompt"], s["response"],
                                [rb.StepRecord(st["token"], st["logp"], st["drafted"], st["logq"], st["target_logprobs"])
                                 for st in s["steps"]], s["eos_bias"], s["reward"]) for s in buf]
    for smp, w, e in zip(samples, ws, exp["losses"]):
        assert rb.kd_loss(drafter, smp, w) == pytest.approx(e, rel=1e-10, abs=1e-12)
    grad = rb.kd_loss_gradient(drafter, list(zip(samples, ws)))
    assert max(abs(a - b) for a, b in zip(grad, exp["grad"])) < 1e-12
