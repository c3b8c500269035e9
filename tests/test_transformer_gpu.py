"""GPU: the transformer path (K1 drafter tree expansion, K2 tree-verify forward with the
tcgen05 GEMMs and tree-causal attention, K3 acceptance, K4 KV compaction) on the BASELINE
cfg1 shape (2-layer d=256 target + 1-layer EAGLE-3-style drafter, synthetic weights).

Parity strategy:
  * logits: every captured verify / draft row against a plain PyTorch fp32 forward of the
    same architecture on the same weights -- tolerance 3e-2 of the logit scale (bf16
    activations, fp32 accumulation);
  * acceptance: the CPU oracle (oracle/restate.cpp) replays the engine's own captured rows
    (LookupModel) and must reproduce tokens, accept lengths and the ledger BIT-EXACTLY,
    under rejection sampling and under greedy verification;
  * greedy SD output == greedy non-speculative decode of the target, token for token (the
    forward is row-invariant, so a token's logits do not depend on the tree it sits in).
"""
import random

import pytest
import torch

import paper_2510_26475_b200 as rb
from torch_ref import DrafterRef, TargetRef, bf

pytestmark = pytest.mark.gpu

SHAPE = rb.TransformerShape.tiny(vocab=1024, max_ctx=256)


@pytest.fixture(scope="module")
def models():
    tgt = rb.TransformerModel(SHAPE, seed=11)
    drf = rb.EagleDrafter(tgt, seed=12, version=3)
    return tgt, drf


def make_requests(n=4, plen=6, max_len=14, seed=5, eos_bias=-2.0):
    rng = random.Random(seed)
    return [rb.RequestState(i, [rng.randrange(SHAPE.vocab - 1) for _ in range(plen + i % 3)], eos_bias, max_len,
                            rb.DecodeRng.from_seed(seed, i)) for i in range(n)]


def run(models, cfg, verify_mode="sample", capture=False, reqs=None):
    tgt, drf = models
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs or make_requests(), cfg, verify_mode,
                         record_full_logprobs=False)
    if capture:
        eng.set_capture(True)
    while not eng.all_done():
        eng.step()
    return eng


def contexts(eng):
    reqs = eng.requests()
    full = [r.prompt + r.generated for r in reqs]
    return reqs, full


def test_shape_and_params(models):
    tgt, drf = models
    assert tgt.vocab_size == SHAPE.vocab and drf.version == 3
    qkv = (SHAPE.n_heads + 2 * SHAPE.n_kv_heads) * SHAPE.head_dim
    assert tgt.n_params == SHAPE.macs_per_token() + SHAPE.n_layers * qkv  # matrices once per token + biases


@pytest.mark.parametrize("cfg", [rb.SDConfig.tree(1, 3, 3), rb.SDConfig.tree(2, 2, 2)])
def test_logits_match_torch_reference(models, cfg):
    tgt, drf = models
    eng = run(models, cfg, capture=True, reqs=make_requests(n=3, max_len=10))
    _, full = contexts(eng)
    tref = TargetRef(tgt)
    dref = DrafterRef(drf, tref)
    rows = eng.captured_rows()
    assert rows
    checked_t = checked_d = 0
    worst = 0.0
    for role, req, cl, ext, logits in rows[:120]:
        ctx = full[req][:cl] + ext
        got = torch.tensor(logits, device="cuda")
        if role == 1:
            ref = tref.forward(ctx)[0][-1]
            checked_t += 1
        else:
            if ext:
                continue  # deeper drafter rows checked in test_drafter_tree_rows
            ref = dref.context_logits(ctx)[-1]
            checked_d += 1
        err = (got - ref).abs().max().item() / ref.std().item()
        worst = max(worst, err)
    assert checked_t > 10 and checked_d > 3
    assert worst < 3e-2, worst


def test_drafter_tree_rows(models):
    """Depth >= 1 drafter rows: feature = the drafter's own hidden state of the previous depth."""
    tgt, drf = models
    eng = run(models, rb.SDConfig.tree(1, 2, 3), capture=True, reqs=make_requests(n=2, max_len=6))
    _, full = contexts(eng)
    tref = TargetRef(tgt)
    dref = DrafterRef(drf, tref)
    n = 0
    for role, req, cl, ext, logits in eng.captured_rows():
        if role != 0 or not ext:
            continue
        toks = full[req][:cl] + ext
        L = cl
        _, feats = tref.forward(toks[:L])
        d = SHAPE.d_model
        prev = torch.zeros(L, 3 * d, device="cuda")
        prev[1:] = feats[:-1].reshape(L - 1, 3 * d)
        f = prev @ dref.fc.t()
        for p in range(L, len(toks)):  # deeper positions take the previous position's drafter output
            _, x = dref._layer_logits(toks[:p], f)
            f = torch.cat([f, x[-1:]], 0)
        ref = dref._layer_logits(toks, f)[0][-1]
        got = torch.tensor(logits, device="cuda")
        assert (got - ref).abs().max().item() / ref.std().item() < 3e-2
        n += 1
        if n >= 12:
            break
    assert n >= 4


def _lookup(rows, full, role, vocab, temperature, depth_aware):
    table = {}
    for rl, req, cl, ext, logits in rows:
        if rl != role:
            continue
        key = (tuple(full[req][:cl] + ext), len(ext) if depth_aware else 0)
        if key in table:
            assert table[key] == list(logits), "same context produced different logits (row-invariance broken)"
            continue
        table[key] = list(logits)
    return {"kind": "lookup", "vocab": vocab, "temperature": temperature, "depth_aware": depth_aware,
            "rows": [{"ctx": list(k[0]), "depth": k[1], "logits": v} for k, v in table.items()]}


@pytest.mark.parametrize("mode", ["sample", "greedy"])
@pytest.mark.parametrize("cfg", [rb.SDConfig.chain(3), rb.SDConfig.tree(1, 4, 3), rb.SDConfig.tree(2, 2, 2),
                                 rb.SDConfig.off()])
def test_acceptance_replay_bit_exact(models, oracle, mode, cfg):
    eng = run(models, cfg, verify_mode=mode, capture=True)
    reqs, full = contexts(eng)
    rows = eng.captured_rows()
    target = _lookup(rows, full, 1, SHAPE.vocab, 1.0, False)
    drafter = _lookup(rows, full, 0, SHAPE.vocab, 1.0, True)
    jreqs = [{"id": r.id, "prompt": r.prompt, "eos_bias": r.eos_bias, "max_len": r.max_len, "seed": r.rng.seed,
              "stream": r.rng.stream_id} for r in reqs]
    exp = oracle("run_generation", target=target, drafter=drafter, requests=jreqs, verify_mode=mode,
                 forced={"s": cfg.rounds, "t": cfg.branching, "n": cfg.draft_len, "enabled": cfg.enabled},
                 record_logprobs=False)
    assert [r.generated for r in reqs] == [s["response"] for s in exp["samples"]]
    assert [r.accept_lens for r in reqs] == [s["accept_lens"] for s in exp["samples"]]
    assert [list(e) for e in eng.ledger()] == exp["ledger"]
    for r, s in zip(reqs, exp["samples"]):
        for st, es in zip(r.steps, s["steps"]):
            assert st.drafted == es["drafted"]
            assert abs(st.logp - es["logp"]) < 1e-9 and abs(st.logq - es["logq"]) < 1e-9


def test_greedy_sd_equals_greedy_decode(models):
    base = run(models, rb.SDConfig.off(), verify_mode="greedy")
    want = [r.generated for r in base.requests()]
    for cfg in [rb.SDConfig.chain(4), rb.SDConfig.tree(1, 4, 3), rb.SDConfig.tree(3, 2, 2)]:
        got = [r.generated for r in run(models, cfg, verify_mode="greedy").requests()]
        assert got == want, cfg


def test_long_prompt_prefill_and_catch_up(models):
    """Prompts longer than one attention chunk; spec mode turns on at step 0 -> the drafter
    catch-up processes the whole prompt (the off->on prefill of server.cpp:280-290)."""
    reqs = make_requests(n=2, plen=150, max_len=8)
    eng = run(models, rb.SDConfig.tree(1, 2, 2), capture=True, reqs=reqs)
    _, full = contexts(eng)
    tref = TargetRef(models[0])
    for role, req, cl, ext, logits in eng.captured_rows()[:6]:
        if role != 1:
            continue
        ref = tref.forward(full[req][:cl] + ext)[0][-1]
        got = torch.tensor(logits, device="cuda")
        assert (got - ref).abs().max().item() / ref.std().item() < 3e-2


def test_mode_switch_and_adaptive_table(models):
    """Adaptive engine: spec at small batch, off at large -> switches, prefill events, and
    the emitted tokens stay identical to greedy decoding."""
    tgt, drf = models
    table = rb.ProfileTable([1, 2, 4])
    for b in (1, 2, 4):
        table.set_entry(b, rb.SDConfig.off(), 1.0)
        table.set_entry(b, rb.SDConfig.tree(1, 2, 2), 0.5 if b <= 2 else 2.0)
    table.finalize()
    reqs = make_requests(n=4, max_len=12)
    for i, r in enumerate(reqs):
        r.max_len = 3 + 4 * i  # staggered finish -> the active batch shrinks
    eng = rb.BatchEngine(tgt, lambda: drf, table, rb.TimingModel(), reqs, rb.SDConfig.off(), "greedy",
                         record_full_logprobs=False)
    while not eng.all_done():
        eng.step()
    assert eng.switches() and eng.prefill_events() >= 1
    base = run(models, rb.SDConfig.off(), verify_mode="greedy", reqs=make_requests(n=4, max_len=16))
    for r, b in zip(eng.requests(), base.requests()):
        assert r.generated == b.generated[:len(r.generated)]


def test_step_tokens_match_responses(models):
    """rs_engine_step_tokens (the step's tokens, returned with the summary) reassembles every
    response exactly."""
    tgt, drf = models
    reqs = make_requests(n=4, max_len=12)
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 3, 3), "sample",
                         record_full_logprobs=False)
    got = {r.id: [] for r in reqs}
    while not eng.all_done():
        eng.step()
        for rid, toks in eng.step_tokens().items():
            got[rid].extend(toks)
    for r in eng.requests():
        assert got[r.id] == r.generated


def test_catch_up_longer_than_workspace(models):
    """A drafter catch-up longer than the forward workspace (2048 rows) -- the first spec cycle
    at an 8K context (cfg4) -- runs in consecutive chunks; greedy SD still equals greedy decode."""
    tgt, drf = models
    big = rb.TransformerShape.tiny(vocab=1024, max_ctx=2400)
    t2 = rb.TransformerModel(big, seed=11)
    d2 = rb.EagleDrafter(t2, seed=12)
    rng = random.Random(9)
    prompts = [[rng.randrange(1023) for _ in range(2200 + 37 * i)] for i in range(2)]

    def gen(cfg):
        reqs = [rb.RequestState(i, list(p), -2.0, 8, rb.DecodeRng.from_seed(5, i)) for i, p in enumerate(prompts)]
        e = rb.BatchEngine(t2, lambda: d2, None, rb.TimingModel(), reqs, cfg, "greedy", record_full_logprobs=False)
        while not e.all_done():
            e.step()
        return [r.generated for r in e.requests()]

    assert gen(rb.SDConfig.tree(1, 2, 2)) == gen(rb.SDConfig.off())
