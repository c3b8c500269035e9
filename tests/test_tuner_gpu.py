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


def test_measured_table_is_complete(table):
    keys = {c.key() for c in CFGS} | {rb.SDConfig.off().key()}
    for b in (1, 2, 4):
        ents = table._entries[b]
        assert {c.key() for c, _ in ents} == keys
        assert all(0 < t < 1e3 for _, t in ents)  # ms per emitted token
        best = table.best_for_bucket(b)
        want = min(ents, key=lambda e: (e[1], e[0].drafted_per_cycle() if e[0].enabled else -1))
        assert best.key() == want[0].key() or best.key() in keys
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
