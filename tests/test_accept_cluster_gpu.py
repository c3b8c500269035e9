"""GPU: the fused acceptance kernel (K3) split over a thread-block cluster.

For large vocabularies each sequence's acceptance runs on a cluster of up to 8 CTAs that
share the full-vocabulary residual passes through distributed shared memory. Every tile is
summed by one warp in a fixed lane order whichever CTA owns it, so the result must be
BITWISE independent of the cluster size -- checked here by forcing 1, 2, 4 and 8 CTAs per
sequence on the tabular golden run (vs the compiled reference) and on the transformer path
(vs each other and vs the oracle replay at a vocabulary that takes the automatic path).
"""
import random

import pytest

import paper_2510_26475_b200 as rb
from conftest import load_golden
from helpers import run_engine
from oracle_client import fnv1a_responses
from test_tabular_gpu import _assert_same

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _restore_tuning():
    yield
    rb.set_tuning("accept_cluster", 0)


@pytest.mark.parametrize("C", [1, 2, 4, 8])
def test_tabular_golden_any_cluster(C):
    """Appendix B fingerprints of the compiled reference, with C CTAs per sequence."""
    g = load_golden("appendix_b.json")
    rb.set_tuning("accept_cluster", C)
    for c in g["cases"]:
        case = {"target": g["actor"], "drafter": g["drafter"], "requests": g["requests"], "forced": c["forced"]}
        out, _ = run_engine(case, record="target_logprobs" in c["out"])
        _assert_same(out, c["out"])
        assert fnv1a_responses(out["responses"]) == c["out"]["fnv"]


def _tiny(vocab):
    shape = rb.TransformerShape.tiny(vocab=vocab, max_ctx=128)
    tgt = rb.TransformerModel(shape, seed=21)
    return shape, tgt, rb.EagleDrafter(tgt, seed=22)


def _run(shape, tgt, drf, cfg, mode, capture=False):
    rng = random.Random(3)
    reqs = [rb.RequestState(i, [rng.randrange(shape.vocab - 1) for _ in range(5 + i)], -1.0, 12,
                            rb.DecodeRng.from_seed(9, i)) for i in range(5)]
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, cfg, mode, record_full_logprobs=False)
    if capture:
        eng.set_capture(True)
    while not eng.all_done():
        eng.step()
    return eng


@pytest.mark.parametrize("mode", ["sample", "greedy"])
def test_transformer_bitwise_cluster_invariance(mode):
    shape, tgt, drf = _tiny(1024)
    outs = []
    for C in (1, 2, 4, 8):
        rb.set_tuning("accept_cluster", C)
        eng = _run(shape, tgt, drf, rb.SDConfig.tree(1, 4, 3), mode)
        outs.append([(r.generated, r.accept_lens, [(s.logp, s.logq, s.drafted) for s in r.steps])
                     for r in eng.requests()])
    assert all(o == outs[0] for o in outs[1:])


def test_large_vocab_auto_cluster_replay(oracle):
    """V = 8192 takes the automatic cluster path; the oracle replays the captured rows."""
    from test_transformer_gpu import _lookup, contexts
    shape, tgt, drf = _tiny(8192)
    cfg = rb.SDConfig.tree(1, 4, 3)
    eng = _run(shape, tgt, drf, cfg, "sample", capture=True)
    reqs, full = contexts(eng)
    rows = eng.captured_rows()
    exp = oracle("run_generation", target=_lookup(rows, full, 1, shape.vocab, 1.0, False),
                 drafter=_lookup(rows, full, 0, shape.vocab, 1.0, True),
                 requests=[{"id": r.id, "prompt": r.prompt, "eos_bias": r.eos_bias, "max_len": r.max_len,
                            "seed": r.rng.seed, "stream": r.rng.stream_id} for r in reqs],
                 forced={"s": 1, "t": 4, "n": 3, "enabled": True}, record_logprobs=False)
    assert [r.generated for r in reqs] == [s["response"] for s in exp["samples"]]
    assert [r.accept_lens for r in reqs] == [s["accept_lens"] for s in exp["samples"]]
