"""CPU: pin the oracle restatement (oracle/restate.cpp) against the compiled reference and
the golden fixtures. TEST INFRASTRUCTURE checks -- no product code involved."""
import random

import pytest

from conftest import load_golden
from oracle_client import CheckerError, fnv1a_responses

APPENDIX_B = {  # SURVEY.md Appendix B (measured on the compiled reference)
    "off": (377, 24, 0, 0, 816.0, "7e7c402007eee680", [4, 6, 7]),
    "s1_t1_n3": (368, 16, 192, 188, 1062.8, "554c6eb730479aa0", [4, 4, 7]),
    "s2_t1_n2": (395, 16, 209, 202, 1572.8, "3f98505b73ee8b80", [4, 7]),
    "s1_t4_n5": (346, 13, 196, 168, 4009.0, "c96c42d1e22b7021", [4, 7]),
}


def key(c):
    return "off" if not c["enabled"] else f"s{c['s']}_t{c['t']}_n{c['n']}"


def test_appendix_b_fingerprints_restatement(oracle):
    g = load_golden("appendix_b.json")
    assert g["actor"]["logits"][:4] == [0.48635725206852604, 0.04020821067022811, 0.06832073026090159,
                                        0.4822737645126581]
    assert g["drafter"]["version"] == 4
    for c in g["cases"]:
        out = oracle("run_generation", target=g["actor"], drafter=g["drafter"], requests=g["requests"],
                     forced=c["forced"], record_logprobs=False)
        resp = [s["response"] for s in out["samples"]]
        tok, cyc, al, ndr, sim, fnv, r0 = APPENDIX_B[key(c["forced"])]
        assert sum(map(len, resp)) == tok
        assert out["cycles"] == cyc
        assert sum(out["accept_lens"]) == al and len(out["accept_lens"]) == ndr
        assert out["total_time"] == pytest.approx(sim, rel=1e-12)
        assert fnv1a_responses(resp) == fnv == c["out"]["fnv"]
        assert resp[0] == r0


def test_restatement_matches_reference_fixtures(oracle):
    for item in load_golden("tabular_engine.json"):
        case, exp = item["case"], item["out"]
        out = oracle("run_generation", record_logprobs=True, **case)
        assert [s["response"] for s in out["samples"]] == exp["responses"]
        assert out["accept_lens"] == exp["accept_lens"]
        assert out["cycles"] == exp["cycles"]
        assert out["ledger"] == exp["ledger"]
        assert out["active_trace"] == exp["active_trace"]
        for s, es in zip(out["samples"], exp["steps"]):
            for st, (lp, dr, lq) in zip(s["steps"], es):
                assert st["drafted"] == dr
                assert st["logp"] == pytest.approx(lp, abs=1e-12)
                assert st["logq"] == pytest.approx(lq, abs=1e-12)


def test_restatement_adaptive_matches_reference(oracle):
    g = load_golden("appendix_b.json")
    out = oracle("run_generation", target=g["actor"], drafter=g["drafter"], requests=g["requests"], table=g["table"],
                 record_logprobs=False)
    assert fnv1a_responses([s["response"] for s in out["samples"]]) == g["adaptive"]["fnv"]
    assert out["switches"] == g["adaptive"]["switches"]
    assert out["prefill_events"] == g["adaptive"]["prefill_events"]


@pytest.mark.parametrize("seed", range(6))
def test_restatement_vs_live_reference_spec_step_tree(oracle, reference, seed):
    rng = random.Random(seed)
    V = rng.choice([3, 5, 8])
    to, do = rng.choice([(2, 1), (1, 0), (0, 0)])
    tgt = {"vocab": V, "order": to, "temperature": 1.0, "logits": [rng.gauss(0, 1) for _ in range(V ** to * V)]}
    drf = {"vocab": V, "order": do, "temperature": 1.0, "logits": [rng.gauss(0, 1) for _ in range(V ** do * V)]}
    for c in [{"s": 1, "t": 3, "n": 2}, {"s": 2, "t": 2, "n": 3}, {"s": 3, "t": 1, "n": 1}]:
        c["enabled"] = True
        kw = dict(target=tgt, drafter=drf, ctx=[1], cfg=c, seed=seed, stream=7, eos_bias=0.3, cycles=40,
                  advance_ctx=True, max_emit=rng.choice([1, 2, 5, 100]), record_logprobs=True)
        a = oracle("spec_step_tree", **kw)["outcomes"]
        b = reference("spec_step_tree", **kw)["outcomes"]
        for x, y in zip(a, b):
            assert x["accepted_tokens"] == y["accepted_tokens"]
            assert x["accept_len"] == y["accept_len"] and x["bonus_token"] == y["bonus_token"]
            assert x["rounds"] == y["rounds"] and x["ended"] == y["ended"]


def test_restatement_kd_update_matches_reference(oracle):
    g = load_golden("kd_update.json")
    for c in g["cases"]:
        out = oracle("kd_update", drafter=g["drafter"], buffer=g["buffer"], policy=c["policy"],
                     selection_seed=c["selection_seed"], cost_per_token=0.02)
        e = c["out"]
        assert out["samples_used"] == e["samples_used"]
        assert out["loss"] == pytest.approx(e["loss"], rel=1e-12)
        assert out["weight_mean"] == e["weight_mean"] and out["weight_max"] == e["weight_max"]
        assert max(abs(a - b) for a, b in zip(out["logits"], e["logits"])) < 1e-12
    # SURVEY App. B KD fingerprint
    c0 = g["cases"][0]["out"]
    assert c0["loss"] == pytest.approx(454.08181997182356, rel=1e-12)
    assert c0["samples_used"] == 32 and c0["weight_mean"] == 0.375 and c0["weight_max"] == 4.0
    assert sum(x * x for x in c0["logits"]) == pytest.approx(314.25454535470607, rel=1e-12)


def test_restatement_greedy_mode_is_plain_greedy_decode(oracle):
    """Greedy verification must reproduce greedy decoding of the target, token for token."""
    rng = random.Random(5)
    V = 7
    tgt = {"vocab": V, "order": 2, "logits": [rng.gauss(0, 2) for _ in range(V ** 3)]}
    drf = {"vocab": V, "order": 1, "logits": [rng.gauss(0, 2) for _ in range(V ** 2)]}
    reqs = [{"id": i, "prompt": [i % (V - 1)], "eos_bias": -1.0, "max_len": 25, "seed": 1, "stream": i}
            for i in range(6)]
    base = oracle("run_generation", target=tgt, drafter=drf, requests=reqs, verify_mode="greedy",
                  forced={"enabled": False}, record_logprobs=False)
    for c in [{"s": 1, "t": 1, "n": 3}, {"s": 2, "t": 3, "n": 2}, {"s": 1, "t": 4, "n": 5}]:
        c["enabled"] = True
        sd = oracle("run_generation", target=tgt, drafter=drf, requests=reqs, verify_mode="greedy", forced=c,
                    record_logprobs=False)
        assert [s["response"] for s in sd["samples"]] == [s["response"] for s in base["samples"]]


def test_errors_match_reference(oracle, reference):
    for lib in (oracle, reference):
        with pytest.raises(CheckerError) as e:
            lib("profile_table", buckets=[1], entries=[{"bucket": 1, "s": 1, "t": 1, "n": 2, "enabled": True,
                                                         "time_per_token": 1.0}])
        assert "missing non-spec baseline" in e.value.what
