"""GPU parity at the BENCHMARKED head geometry (VERDICT r1 "next" item 1).

The bench runs Qwen2.5-3B (d=2048, 16 query / 2 KV heads -> G=8, hd=128, d_ff=11008,
V=151936); cfg3/cfg4 name 7B (G=7, V=152064) and 14B (G=5). These tests use exactly those
d / head / d_ff / vocabulary geometries, with the layer count reduced to 4 (the EAGLE
feature layers are then 1, 2, 3) and contexts at the bench's 1664-token start, so the
attention row mapping (row = token*G + head, dead rows at G=7), the LM-head tiles over
151936 columns and the acceptance passes at V ~ 152K all run as in the bench:

  (a) greedy SD == greedy decode, token for token, for tree(1,4,5) and chain(3)
      (specdec.cpp:197-267 with the greedy rule of DESIGN.md §5; the forward is row
      invariant, so a token's logits do not depend on the tree it sits in);
  (b) verify and draft logit rows vs the plain PyTorch fp32 forward on the same weights,
      max|d|/std < 3e-2 (bf16 activations, fp32 accumulation);
  (c) the CPU oracle (oracle/restate.cpp, pinned to the compiled reference) replays the
      engine's own captured rows -- handed over as fp32 through the binary entry
      oracle_lookup_add_f32 -- and must reproduce tokens, accept lengths and the ledger
      BIT-EXACTLY under rejection sampling (model.cpp:23-68, specdec.cpp:25-52, :197-267,
      server.cpp:266-349) and under greedy verification.

With synthetic weights the greedy drafter almost never matches the target argmax, so (a)
mostly exercises the root rows inside a tree; the sampled replay (c) and the deeper-row
checks (b) cover accepted chains.
"""
import random

import numpy as np
import pytest
import torch

import paper_2510_26475_b200 as rb
from torch_ref import DrafterRef, TargetRef

pytestmark = pytest.mark.gpu

CTX = 1664  # bench.py --ctx default: 128-token prompt + 1536 generated
GEOM = {  # public Qwen2.5 config.json geometry, 4 layers
    "3b": dict(vocab=151936, d_model=2048, n_heads=16, n_kv_heads=2, d_ff=11008),
    "7b": dict(vocab=152064, d_model=3584, n_heads=28, n_kv_heads=4, d_ff=18944),
    "14b": dict(vocab=152064, d_model=5120, n_heads=40, n_kv_heads=8, d_ff=13824),
}
LAYERS = 4


def shape_of(name, max_len=16):
    g = GEOM[name]
    return rb.TransformerShape(g["vocab"], g["d_model"], LAYERS, g["n_heads"], g["n_kv_heads"], 128, g["d_ff"],
                               max_ctx=CTX + 8 + max_len + 64)


@pytest.fixture(scope="module", params=["3b", "7b", "14b"])
def models(request):
    shape = shape_of(request.param)
    tgt = rb.TransformerModel(shape, seed=20251026)
    drf = rb.EagleDrafter(tgt, seed=4242, version=1)
    yield request.param, tgt, drf
    del tgt, drf
    torch.cuda.empty_cache()


def make_requests(shape, n, max_len, seed=5, eos_bias=-20.0):
    rng = random.Random(seed)
    return [rb.RequestState(i, [rng.randrange(shape.vocab - 1) for _ in range(CTX + i % 3)], eos_bias, max_len,
                            rb.DecodeRng.from_seed(seed, i)) for i in range(n)]


def run(tgt, drf, reqs, cfg, mode, capture=False):
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, cfg, mode, record_full_logprobs=False)
    if capture:
        eng.set_capture(True)
    while not eng.all_done():
        eng.step()
    return eng


def batch_of(name):
    return 8 if name == "3b" else 4


@pytest.mark.parametrize("cfg", [rb.SDConfig.tree(1, 4, 5), rb.SDConfig.chain(3)], ids=["tree145", "chain3"])
def test_greedy_sd_equals_greedy_decode(models, cfg):
    name, tgt, drf = models
    reqs = lambda: make_requests(tgt.shape, batch_of(name), 12)  # noqa: E731
    want = [r.generated for r in run(tgt, drf, reqs(), rb.SDConfig.off(), "greedy").requests()]
    got = [r.generated for r in run(tgt, drf, reqs(), cfg, "greedy").requests()]
    assert all(len(w) == 12 for w in want)
    assert got == want


def _ref_row(tref, dref, role, toks, cl, ext):
    d = tref.s.d_model
    if role == 1:
        return tref.forward(toks, last_only=True)[0][-1]
    if not ext:
        return dref.context_logits(toks, last_only=True)[-1]
    # deeper drafter rows: feature = the drafter's own hidden state one depth up
    _, feats = tref.forward(toks[:cl], last_only=True)
    prev = torch.zeros(cl, 3 * d, device="cuda")
    prev[1:] = feats[:-1].reshape(cl - 1, 3 * d)
    f = tref.mm(prev, dref.fc)
    for p in range(cl, len(toks)):
        _, x = dref._layer_logits(toks[:p], f, last_only=True)
        f = torch.cat([f, x[-1:]], 0)
    return dref._layer_logits(toks, f, last_only=True)[0][-1]


def _err(a, ref):
    dz = a - ref
    sd = ref.std().item()
    return dz.abs().max().item() / sd, dz.pow(2).mean().sqrt().item() / sd


def test_logits_match_torch_reference(models):
    """Target verify rows (root and in-tree), depth-0 and deeper drafter rows vs fp32 torch.

    Tolerance, self-calibrated: the fp32 reference and the same reference with bf16-operand
    matmuls (fp32 accumulation; a second valid bf16 implementation) differ by the flips of the
    bf16 rounding points, which grow with d and depth (rms ~1e-2 of the logit std at 4 layers,
    d = 2048..5120; the max over V ~ 152K columns sits ~5 rms out). The CUDA rows must stay
    within 2x that floor (rms and max), and below absolute bars of 2e-2 rms / 1e-1 max."""
    name, tgt, drf = models
    eng = run(tgt, drf, make_requests(tgt.shape, 2, 6), rb.SDConfig.tree(1, 4, 5), "sample", capture=True)
    reqs = eng.requests()
    full = [r.prompt + r.generated for r in reqs]
    meta = eng.captured_meta()
    t32, tbf = TargetRef(tgt), TargetRef(tgt, bf16_mm=True)
    d32, dbf = DrafterRef(drf, t32), DrafterRef(drf, tbf)
    picked = {"t_root": [], "t_tree": [], "d_root": [], "d_deep": []}
    for i, (role, req, cl, ext) in enumerate(meta):
        k = ("t_" if role == 1 else "d_") + (("tree" if role == 1 else "deep") if ext else "root")
        if len(picked[k]) < 4:
            picked[k].append(i)
    assert all(len(v) >= 2 for v in picked.values()), {k: len(v) for k, v in picked.items()}
    got_e, floor_e = [0.0, 0.0], [0.0, 0.0]
    for kind, idx in picked.items():
        for i in idx:
            role, req, cl, ext = meta[i]
            got = torch.from_numpy(eng.captured_logits_f32(i, 1)[0]).cuda()
            toks = full[req][:cl] + ext
            ref = _ref_row(t32, d32, role, toks, cl, ext)
            alt = _ref_row(tbf, dbf, role, toks, cl, ext)
            g, f = _err(got, ref), _err(alt, ref)
            got_e = [max(got_e[0], g[0]), max(got_e[1], g[1])]
            floor_e = [max(floor_e[0], f[0]), max(floor_e[1], f[1])]
    print(name, "cuda vs fp32 (max, rms)/std:", [round(x, 4) for x in got_e],
          "bf16-matmul torch vs fp32:", [round(x, 4) for x in floor_e])
    assert got_e[0] < max(2 * floor_e[0], 2e-2) and got_e[0] < 1e-1, (got_e, floor_e)
    assert got_e[1] < max(2 * floor_e[1], 4e-3) and got_e[1] < 2e-2, (got_e, floor_e)


def _replay(oracle, eng, vocab, mode, cfg):
    reqs = eng.requests()
    full = [r.prompt + r.generated for r in reqs]
    meta = eng.captured_meta()
    tl = oracle.lookup(vocab, 1.0, depth_aware=False)
    dl = oracle.lookup(vocab, 1.0, depth_aware=True)
    chunk = 64
    for first in range(0, len(meta), chunk):
        rows = eng.captured_logits_f32(first, min(chunk, len(meta) - first))
        for j, row in enumerate(rows):
            role, req, cl, ext = meta[first + j]
            ctx = full[req][:cl] + ext
            (tl if role == 1 else dl).add(ctx, len(ext) if role == 0 else 0, row)
    jreqs = [{"id": r.id, "prompt": r.prompt, "eos_bias": r.eos_bias, "max_len": r.max_len, "seed": r.rng.seed,
              "stream": r.rng.stream_id} for r in reqs]
    exp = oracle("run_generation", target=tl.json(), drafter=dl.json(), requests=jreqs, verify_mode=mode,
                 forced={"s": cfg.rounds, "t": cfg.branching, "n": cfg.draft_len, "enabled": cfg.enabled},
                 record_logprobs=False)
    assert [r.generated for r in reqs] == [s["response"] for s in exp["samples"]]
    assert [r.accept_lens for r in reqs] == [s["accept_lens"] for s in exp["samples"]]
    assert [list(e) for e in eng.ledger()] == exp["ledger"]
    for r, s in zip(reqs, exp["samples"]):
        for st, es in zip(r.steps, s["steps"]):
            assert st.drafted == es["drafted"]
            assert abs(st.logp - es["logp"]) < 1e-9 and abs(st.logq - es["logq"]) < 1e-9
    return reqs, tl, dl


@pytest.mark.parametrize("mode", ["sample", "greedy"])
@pytest.mark.parametrize("cfg", [rb.SDConfig.tree(1, 4, 5), rb.SDConfig.chain(3)], ids=["tree145", "chain3"])
def test_acceptance_replay_bit_exact(models, oracle, mode, cfg):
    name, tgt, drf = models
    if name != "3b" and (mode, cfg.branching) != ("sample", 4):
        pytest.skip("7B / 14B geometry: the bench's sampled tree(1,4,5) only")
    eng = run(tgt, drf, make_requests(tgt.shape, 4, 10, seed=17), cfg, mode, capture=True)
    reqs, tl, dl = _replay(oracle, eng, tgt.shape.vocab, mode, cfg)
    assert tl.added > 20 and dl.added > 10
    if mode == "sample":  # rejection sampling at T=1 accepts drafted tokens now and then
        assert sum(sum(r.accept_lens) for r in reqs) > 0


def test_mean_accept_len_definition(models):
    """accept_len counts drafted tokens only (specdec.hpp:67); the bonus /
    replacement token is extra. n_eff = min(n, remaining - 1) (specdec.cpp:170), so every
    drafting cycle emits exactly accept_len + 1 tokens; a cycle at remaining == 1 drafts
    nothing, emits one token and records no accept_len (server.cpp:319-321)."""
    name, tgt, drf = models
    if name != "3b":
        pytest.skip("geometry-independent")
    eng = run(tgt, drf, make_requests(tgt.shape, 4, 13, seed=23), rb.SDConfig.tree(1, 4, 5), "sample")
    for r in eng.requests():
        assert len(r.generated) == 13
        assert 13 - sum(a + 1 for a in r.accept_lens) in (0, 1)
        assert all(0 <= a <= 5 for a in r.accept_lens)
    al = [a for r in eng.requests() for a in r.accept_lens]
    assert rb.mean_accept_len(al) == pytest.approx(sum(al) / len(al))


def test_north_star_batch256_greedy_sd_equals_greedy_decode():
    """BASELINE north star: the 3B-geometry SD step at BATCH 256 (the bench's north-star leg) still
    decodes exactly like greedy decoding, request for request -- attention items, GEMM token
    tiles and acceptance clusters are all at their batch-256 sizes."""
    shape = shape_of("3b", max_len=6)
    tgt = rb.TransformerModel(shape, seed=20251026)
    drf = rb.EagleDrafter(tgt, seed=4242, version=1)
    reqs = lambda: make_requests(shape, 256, 6, seed=31)  # noqa: E731
    want = [r.generated for r in run(tgt, drf, reqs(), rb.SDConfig.off(), "greedy").requests()]
    got = [r.generated for r in run(tgt, drf, reqs(), rb.SDConfig.tree(1, 4, 5), "greedy").requests()]
    assert all(len(w) == 6 for w in want) and got == want
    del tgt, drf
    torch.cuda.empty_cache()


def test_bench_config_batch64_replay_bit_exact(oracle):
    """The bench's own configuration -- 3B geometry, batch 64, tree(1,4,5), rejection sampling at
    T = 1 -- replayed by the CPU oracle on the engine's captured rows: tokens, accept lengths,
    ledger and log-probabilities bit-exact for every one of the 64 requests."""
    shape = shape_of("3b", max_len=4)
    tgt = rb.TransformerModel(shape, seed=20251026)
    drf = rb.EagleDrafter(tgt, seed=4242, version=1)
    cfg = rb.SDConfig.tree(1, 4, 5)
    eng = run(tgt, drf, make_requests(shape, 64, 4, seed=37), cfg, "sample", capture=True)
    reqs, tl, dl = _replay(oracle, eng, shape.vocab, "sample", cfg)
    assert len(reqs) == 64 and tl.added > 64 * 5
    del eng, tgt, drf
    torch.cuda.empty_cache()


def test_cfg4_long_context_14b_8k(oracle):
    """BASELINE cfg4's long-context regime: Qwen2.5-14B head geometry (G = 5, V = 152064, 4 layers)
    at 8K contexts -- ~260 key passes per attention item, the drafter's first catch-up longer than
    its 2048-row workspace (chunked) -- with greedy SD == greedy decode and the oracle's bit-exact
    replay of rejection sampling at T = 1 on the engine's own rows."""
    g = GEOM["14b"]
    ctx = 8192
    shape = rb.TransformerShape(g["vocab"], g["d_model"], LAYERS, g["n_heads"], g["n_kv_heads"], 128, g["d_ff"],
                                max_ctx=ctx + 8 + 6 + 64)
    tgt = rb.TransformerModel(shape, seed=20251026)
    drf = rb.EagleDrafter(tgt, seed=4242, version=1)
    rng = random.Random(41)

    def reqs(max_len, seed):
        return [rb.RequestState(i, [rng.randrange(shape.vocab - 1) for _ in range(ctx + i)], -20.0, max_len,
                                rb.DecodeRng.from_seed(seed, i)) for i in range(2)]

    base = reqs(6, 43)
    clone = lambda: [rb.RequestState(r.id, list(r.prompt), r.eos_bias, r.max_len, rb.DecodeRng.from_seed(43, r.id))  # noqa: E731
                     for r in base]
    want = [r.generated for r in run(tgt, drf, clone(), rb.SDConfig.off(), "greedy").requests()]
    got = [r.generated for r in run(tgt, drf, clone(), rb.SDConfig.tree(1, 4, 5), "greedy").requests()]
    assert all(len(w) == 6 for w in want) and got == want
    cfg = rb.SDConfig.tree(1, 4, 5)
    eng = run(tgt, drf, clone(), cfg, "sample", capture=True)
    _replay(oracle, eng, shape.vocab, "sample", cfg)
    del eng, tgt, drf
    torch.cuda.empty_cache()


def test_cfg3_dynamic_tuning_7b_replay_bit_exact(oracle):
    """BASELINE cfg3's dynamic SD-config tuning at the 7B head geometry (G = 7, V = 152064): a
    ProfileTable whose best configuration changes as requests finish (server.cpp:21-54,
    :266-349), so the engine switches trees between cycles. Greedy decoding is reproduced token
    for token, and the oracle's run_generation -- given the same table -- replays rejection
    sampling on the engine's own rows bit-exactly, switch events and ledger included."""
    shape = shape_of("7b", max_len=14)
    tgt = rb.TransformerModel(shape, seed=20251026)
    drf = rb.EagleDrafter(tgt, seed=4242, version=1)
    buckets = [1, 2, 4, 8]
    best = {1: rb.SDConfig.chain(3), 2: rb.SDConfig.tree(1, 2, 3), 4: rb.SDConfig.tree(1, 4, 5),
            8: rb.SDConfig.tree(1, 2, 2)}
    grid = [rb.SDConfig.chain(3), rb.SDConfig.tree(1, 2, 3), rb.SDConfig.tree(1, 4, 5), rb.SDConfig.tree(1, 2, 2)]

    def table():
        t = rb.ProfileTable(buckets)
        for b in buckets:
            t.set_entry(b, rb.SDConfig.off(), 10.0)
            for c in grid:
                t.set_entry(b, c, 1.0 if c == best[b] else 5.0)
        t.finalize()
        return t

    rng = random.Random(53)
    prompts = [[rng.randrange(shape.vocab - 1) for _ in range(CTX + i)] for i in range(8)]
    lens = [3, 5, 7, 9, 11, 12, 13, 14]  # requests finish one by one: the active batch crosses the buckets

    def reqs():
        return [rb.RequestState(i, list(prompts[i]), -20.0, lens[i], rb.DecodeRng.from_seed(61, i)) for i in range(8)]

    def run_t(mode, capture=False):
        eng = rb.BatchEngine(tgt, lambda: drf, table(), rb.TimingModel(), reqs(), rb.SDConfig.off(), mode,
                             record_full_logprobs=False)
        if capture:
            eng.set_capture(True)
        while not eng.all_done():
            eng.step()
        return eng

    want = [r.generated for r in run(tgt, drf, reqs(), rb.SDConfig.off(), "greedy").requests()]
    g = run_t("greedy")
    assert [r.generated for r in g.requests()] == want
    eng = run_t("sample", capture=True)
    sw = eng.switches()
    assert len({s.to.key() for s in sw}) >= 2, [(s.cycle, s.active_batch, s.to.key()) for s in sw]
    done = eng.requests()
    full = [r.prompt + r.generated for r in done]
    meta = eng.captured_meta()
    tl = oracle.lookup(shape.vocab, 1.0, depth_aware=False)
    dl = oracle.lookup(shape.vocab, 1.0, depth_aware=True)
    for first in range(0, len(meta), 64):
        rows = eng.captured_logits_f32(first, min(64, len(meta) - first))
        for j, row in enumerate(rows):
            role, req, cl, ext = meta[first + j]
            (tl if role == 1 else dl).add(full[req][:cl] + ext, len(ext) if role == 0 else 0, row)
    entries = [{"bucket": b, "s": c.rounds, "t": c.branching, "n": c.draft_len, "enabled": c.enabled,
                "time_per_token": 10.0 if not c.enabled else (1.0 if c == best[b] else 5.0)}
               for b in buckets for c in [rb.SDConfig.off()] + grid]
    exp = oracle("run_generation", target=tl.json(), drafter=dl.json(), table={"buckets": buckets, "entries": entries},
                 requests=[{"id": r.id, "prompt": r.prompt, "eos_bias": r.eos_bias, "max_len": r.max_len, "seed": 61,
                            "stream": r.id} for r in done], verify_mode="sample", record_logprobs=False)
    assert [r.generated for r in done] == [s["response"] for s in exp["samples"]]
    assert [r.accept_lens for r in done] == [s["accept_lens"] for s in exp["samples"]]
    assert [list(e) for e in eng.ledger()] == exp["ledger"]
    assert [(s.cycle, s.active_batch, s.to.key()) for s in sw] == \
        [(e["cycle"], e["active_batch"], rb.SDConfig(e["to"]["s"], e["to"]["t"], e["to"]["n"], e["to"]["enabled"]).key())
         for e in exp["switches"]]
    del eng, g, tgt, drf
    torch.cuda.empty_cache()
