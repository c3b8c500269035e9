"""GPU: the dynamic SD-config tuner fed by MEASURED step latency (the B200 replacement of the
reference's simulated profile(), server.cpp:182-239): per batch bucket and SD config, a wave of
exactly `bucket` requests runs timed engine steps; ProfileTable::finalize picks the argmin
time/token (ties -> fewer drafted, then non-spec, server.cpp:21-54) and the engine re-solves
every cycle from the live batch (server.cpp:279)."""
import random

import pytest

import paper_2510_26475_b200 as rb

pytestmark = pytest.mark.gpu

SHAPE = rb.TransformerShape.tiny(vocab=1024, max_ctx=256)
CFGS = [rb.SDConfig.chain(2), rb.SDConfig.tree(1, 2, 2), rb.SDConfig.tree(1, 4, 3)]


@pytest.fixture(scope="module")
def models():
    tgt = rb.TransformerModel(SHAPE, seed=41)
    return tgt, rb.EagleDrafter(tgt, seed=42)


@pytest.fixture(scope="module")
def table(models):
    tgt, drf = models
    return rb.profile_measured(tgt, drf, [1, 2, 4], CFGS, prompt_len=16, warmup=1, cycles=3)


def _reference_best(ents):
    """ProfileTable::finalize (server.cpp:21-54): a scan in insertion order; strictly lower
    time wins, ties go to fewer drafted tokens (off counts 0), then to non-spec."""
    best = None
    for cfg, tpt in ents:
        if best is None or tpt < best[1]:
            best = (cfg, tpt)
        elif tpt == best[1]:
            cur = cfg.drafted_per_cycle() if cfg.enabled else 0
            old = best[0].drafted_per_cycle() if best[0].enabled else 0
            if cur < old or (cur == old and not cfg.enabled and best[0].enabled):
                best = (cfg, tpt)
    return best[0]


def test_measured_table_is_complete(table, oracle):
    keys = {c.key() for c in CFGS} | {rb.SDConfig.off().key()}
    j = table.to_json()
    exp = oracle("profile_table", buckets=j["buckets"], entries=j["entries"], solve=[1, 2, 3, 4, 9])
    for b in (1, 2, 4):
        ents = table._entries[b]
        assert {c.key() for c, _ in ents} == keys
        assert all(0 < t < 1e3 for _, t in ents)  # ms per emitted token
        best = table.best_for_bucket(b)
        assert best.key() == _reference_best(ents).key()  # measured argmin, reference tie-break
        want = next(e["cfg"] for e in exp["best"] if e["bucket"] == b)
        assert (best.rounds, best.branching, best.draft_len, best.enabled) == \
            ((want["s"], want["t"], want["n"], True) if want["enabled"] else (best.rounds, best.branching,
                                                                              best.draft_len, False))
    for s in exp["solve"]:  # bucket_for clamps above the largest bucket (server.cpp:56-66)
        assert table.bucket_for(s["batch"]) == s["bucket"]
    j = table.to_json()
    t2 = rb.ProfileTable.from_json(j)
    for b in (1, 2, 4):
        assert t2.best_for_bucket(b).key() == table.best_for_bucket(b).key()


def test_adaptive_engine_follows_the_measured_table(models, table):
    tgt, drf = models
    rng = random.Random(2)
    reqs = [rb.RequestState(i, [rng.randrange(SHAPE.vocab - 1) for _ in range(8)], -3.0, 4 + 5 * i,
                            rb.DecodeRng.from_seed(3, i)) for i in range(4)]
    eng = rb.BatchEngine(tgt, lambda: drf, table, rb.TimingModel(), reqs, rb.SDConfig.off(), "sample",
                         record_full_logprobs=False)
    modes = []
    while not eng.all_done():
        info = eng.step()
        modes.append((info.active_batch, rb.SDConfig._from_c(info.mode).key()))
    for batch, key in modes:
        assert key == table.solve(batch).key()
