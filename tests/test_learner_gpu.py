"""GPU: OnlineLearner (learner.cpp:162-289), policy_update (rl.cpp:74-88), the simulated
profile() (server.cpp:182-239) and run_scenario (scenarios.cpp:28-341) on the device, against
the compiled reference's outputs in tests/golden/learner_scenarios.json.

Integer outputs (versions, buffer sizes, sample counts, tokens, cycles, switches) must be
identical; the KD/policy arithmetic is fp64 with a parallel softmax normaliser, so losses,
weights and logits are held to 1e-10 relative / 1e-12 absolute (the reference's own tolerances,
test_learner.cpp:93-110); sim times come from the integer ledger and must match to 1e-12."""
import math

import pytest

import paper_2510_26475_b200 as rb
from conftest import load_golden
from paper_2510_26475_b200 import scenarios as sc

pytestmark = pytest.mark.gpu
G = load_golden("learner_scenarios.json")
MODES = {"reward": rb.WeightMode.Reward, "uniform": rb.WeightMode.Uniform, "frozen": rb.WeightMode.Frozen}


def model_of(j):
    return rb.TabularARModel(j["vocab"], j["order"], j["logits"], j.get("temperature", 1.0), j.get("version", 0))


def samples_of(batch):
    return [rb.RolloutSample(s["prompt"], s["response"],
                             [rb.StepRecord(st["token"], 0.0, False, 0.0, st["target_logprobs"]) for st in s["steps"]],
                             s["eos_bias"], s["reward"]) for s in batch]


def close(a, b, rel=1e-10, abs_=1e-12):
    return a == b or abs(a - b) <= max(abs_, rel * max(abs(a), abs(b)))


def same_json(got, exp, path=""):
    """Structural equality: ints/bools/strings exact, floats to 1e-10 relative."""
    if isinstance(exp, dict):
        assert set(got) == set(exp), (path, sorted(set(got) ^ set(exp)))
        for k in exp:
            same_json(got[k], exp[k], f"{path}.{k}")
    elif isinstance(exp, list):
        assert len(got) == len(exp), path
        for i, (g, e) in enumerate(zip(got, exp)):
            same_json(g, e, f"{path}[{i}]")
    elif isinstance(exp, float) or isinstance(got, float):
        assert close(float(got), float(exp)), (path, got, exp)
    else:
        assert got == exp, (path, got, exp)


def run_script(case, async_):
    p = case["policy"]
    pol = rb.KDPolicy(p["interval"], MODES[p["mode"]], p["clip_lo"], p["clip_hi"], p["lr"])
    L = rb.OnlineLearner(model_of(G["drafter"]), pol, case["selection_seed"], 0.02, case["capacity"], async_)
    states = []
    for it, batch in enumerate(G["batches"]):
        L.feed(samples_of(batch))
        st = {"buffer_after_feed": L.buffer_size()}
        L.on_iteration_boundary(it)
        L.await_pending()
        st.update(version=L.drafter_version(), buffer=L.buffer_size(), updates=len(L.metrics()))
        states.append(st)
    L.await_pending()
    out = {"states": states, "metrics": [sc.learner_line(m) for m in L.metrics()],
           "total_sim_time": L.total_sim_time(), "logits": L.snapshot().logits(), "version": L.drafter_version()}
    L.shutdown()
    return out


@pytest.mark.parametrize("idx", range(len(G["learners"])))
@pytest.mark.parametrize("async_", [False, True])
def test_online_learner_matches_reference(idx, async_):
    case = G["learners"][idx]
    same_json(run_script(case, async_), case["out"])


def test_async_learner_is_bitwise_sync():
    """learner.hpp:91-97 (test_learner.cpp:218-246): async changes timing, not semantics."""
    case = G["learners"][0]
    a, b = run_script(case, False), run_script(case, True)
    assert a == b


def test_learner_snapshot_outlives_learner():
    case = G["learners"][1]
    pol = rb.KDPolicy(1, rb.WeightMode.Uniform, 0.0, 4.0, 0.5)
    L = rb.OnlineLearner(model_of(G["drafter"]), pol, 7, 0.02, 64, True)
    L.feed(samples_of(G["batches"][0]))
    L.on_iteration_boundary(0)
    L.await_pending()
    snap = L.snapshot()
    want = snap.logits()
    L.close()
    del L
    assert snap.logits() == want and snap.version == G["drafter"]["version"] + 1
    assert case["out"]["states"][0]["version"] == snap.version


def test_policy_update_matches_reference():
    pu = G["policy_update"]
    actor = model_of(G["actor"])
    samples = [rb.RolloutSample(s["prompt"], s["response"], [], s["eos_bias"], 0.0, s["actor_version"])
               for s in pu["samples"]]
    new = rb.policy_update(actor, list(zip(samples, pu["advantages"])), pu["lr"])
    assert new.version == pu["out"]["version"]
    got, exp = new.logits(), pu["out"]["logits"]
    assert max(abs(a - b) for a, b in zip(got, exp)) < 1e-12
    stale = [rb.RolloutSample(s.prompt, s.response, [], s.eos_bias, 0.0, 5) for s in samples[:2]]
    with pytest.raises(rb.InvalidArgument, match="policy_update: off-policy update"):
        rb.policy_update(actor, [(s, 1.0) for s in stale], 0.2)


def test_make_env_matches_reference():
    env = sc.make_env(sc.ExperimentConfig())
    assert env.actor.logits() == G["actor"]["logits"]  # std::normal_distribution on the same libstdc++
    got, exp = env.drafter.logits(), G["drafter"]["logits"]
    assert env.drafter.version == G["drafter"]["version"]
    assert max(abs(a - b) for a, b in zip(got, exp)) < 1e-12


def test_default_profile_best_configs():
    """SURVEY.md §8(f) F2 golden: build_profile on the default config, seed 1 -> best = {1,2,4:
    s1_t2_n2, 8: s1_t1_n2, 16: s1_t1_n1, 32, 64: off} -- on the GPU engine with the simulated
    cost model, every entry equal to the reference's."""
    cfg = sc.ExperimentConfig()
    env = sc.make_env(cfg)
    t = sc.build_profile(cfg, env.actor, env.drafter)
    exp = G["default_profile"]["json"]
    got = t.to_json()
    assert [(b["bucket"], b["s"], b["t"], b["n"], b["enabled"]) for b in got["best"]] == \
        [(b["bucket"], b["s"], b["t"], b["n"], b["enabled"]) for b in exp["best"]]
    key = lambda e: (e["bucket"], e["s"], e["t"], e["n"], e["enabled"])
    ge = {key(e): e["time_per_token"] for e in got["entries"]}
    for e in exp["entries"]:
        assert close(ge[key(e)], e["time_per_token"], rel=1e-12), e
    assert t.to_csv() == G["default_profile"]["csv"]


@pytest.mark.parametrize("idx", range(len(G["scenarios"])))
def test_run_scenario_matches_reference(idx):
    case = G["scenarios"][idx]
    r = sc.run_scenario(sc.ExperimentConfig.from_json(case["config"]))
    exp = case["out"]
    assert r.scenario == exp["scenario"]
    same_json(r.step_lines, exp["step_lines"])
    same_json(r.learner_lines, exp["learner_lines"])
    same_json(r.switch_lines, exp["switch_lines"])
    same_json(r.summary, exp["summary"])
    if "table" in exp:
        assert r.table.to_csv() == exp["table"]["csv"]


def test_write_scenario_files(tmp_path):
    case = G["scenarios"][0]
    r = sc.run_scenario(sc.ExperimentConfig.from_json(case["config"]))
    sc.write_scenario_files(r, str(tmp_path))
    import json
    lines = [json.loads(x) for x in open(tmp_path / "steps.jsonl")]
    same_json(lines, case["out"]["step_lines"])
    same_json(json.load(open(tmp_path / "summary.json")), case["out"]["summary"])


def test_transformer_learner_async_equals_sync():
    """The learner over an EAGLE drafter: updates run through rs_kd_update_transformer on the
    worker's own stream; async and sync publish bit-identical LM heads."""
    import random
    shape = rb.TransformerShape.tiny(vocab=512, max_ctx=128)
    tgt = rb.TransformerModel(shape, seed=5)
    drf = rb.EagleDrafter(tgt, seed=6)
    rng = random.Random(4)
    batches = [[rb.RolloutSample([rng.randrange(511) for _ in range(6)], [rng.randrange(511) for _ in range(5)], [],
                                 0.0, rng.random()) for _ in range(3)] for _ in range(3)]
    heads, mets = [], []
    for async_ in (False, True):
        L = rb.OnlineLearner(drf, rb.KDPolicy(1, rb.WeightMode.Reward, 0.0, 4.0, 0.5), 9, 0.01, 64, async_)
        for it, b in enumerate(batches):
            L.feed(b)
            L.on_iteration_boundary(it)
        L.await_pending()
        snap = L.snapshot()
        assert snap.version == 3
        heads.append(snap.to_torch("lm_w").float().cpu())
        mets.append([(m.kd_loss, m.weights_l2, m.samples_used) for m in L.metrics()])
        L.close()
    assert mets[0] == mets[1] and all(math.isfinite(x[1]) and x[1] > 0 for x in mets[0])
    assert (heads[0] == heads[1]).all()


def test_transformer_learner_from_engine_caches():
    """OnlineLearner fed with engine-backed samples (rs_learner_feed_engine) == the same learner fed
    with the detached rollouts: same selection, samples and version; the loss to 1e-9 and the LM
    head to bf16 rounding (the gradient is summed in a different grouping)."""
    import random
    import torch
    shape = rb.TransformerShape.tiny(vocab=512, max_ctx=128)
    tgt = rb.TransformerModel(shape, seed=7)
    drf = rb.EagleDrafter(tgt, seed=8)
    rng = random.Random(5)
    reqs = [rb.RequestState(i, [rng.randrange(511) for _ in range(5 + i)], -1.0, 7 + i, rb.DecodeRng.from_seed(3, i))
            for i in range(5)]
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 2, 3), "sample",
                         record_full_logprobs=False)
    while not eng.all_done():
        eng.step()
    rewards = [rng.random() for _ in range(5)]
    done = eng.requests()
    pol = rb.KDPolicy(1, rb.WeightMode.Reward, 0.0, 4.0, 0.5)
    outs = []
    for mode in ("engine", "detached", "engine_async"):
        L = rb.OnlineLearner(drf, pol, 11, 0.01, 64, mode == "engine_async")
        if mode == "detached":
            L.feed([rb.RolloutSample(list(r.prompt), list(r.generated), [], r.eos_bias, w) for r, w in zip(done, rewards)])
        else:
            L.feed_engine(eng, list(range(5)), rewards)
        L.on_iteration_boundary(0)
        L.await_pending()
        m = L.metrics()[0]
        outs.append((L.drafter_version(), m.samples_used, m.kd_loss, L.snapshot().to_torch("lm_w").float()))
        L.close()
    (v0, n0, l0, h0), (v1, n1, l1, h1), (v2, n2, l2, h2) = outs
    assert v0 == v1 == v2 == drf.version + 1 and n0 == n1 == n2
    assert l0 == pytest.approx(l1, rel=1e-9) and l0 == l2
    assert torch.equal(h0, h2)
    assert (h0 - h1).abs().max().item() <= 2e-2 * h1.abs().max().item()


def test_async_engine_backed_update_overlaps_a_rollout():
    """An asynchronous engine-backed update runs on the learner's own stream while a second engine
    generates on the caller's stream: both results are bitwise those of running them apart."""
    import random
    import torch
    shape = rb.TransformerShape.tiny(vocab=512, max_ctx=128)
    tgt = rb.TransformerModel(shape, seed=9)
    drf = rb.EagleDrafter(tgt, seed=10)

    def engine(seed):
        rng = random.Random(seed)
        reqs = [rb.RequestState(i, [rng.randrange(511) for _ in range(6)], -1.0, 10, rb.DecodeRng.from_seed(seed, i))
                for i in range(6)]
        return rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 2, 3), "sample",
                              record_full_logprobs=False)

    def run(e):
        while not e.all_done():
            e.step()
        return [r.generated for r in e.requests()]

    a = engine(1)
    run(a)
    pol = rb.KDPolicy(1, rb.WeightMode.Uniform, 0.0, 4.0, 0.5)
    ref = rb.OnlineLearner(drf, pol, 3, 0.0, 64, False)
    ref.feed_engine(a, list(range(6)), [1.0] * 6)
    ref.on_iteration_boundary(0)
    want_head = ref.snapshot().to_torch("lm_w")
    want_b = run(engine(2))
    L = rb.OnlineLearner(drf, pol, 3, 0.0, 64, True)
    L.feed_engine(a, list(range(6)), [1.0] * 6)
    L.on_iteration_boundary(0)   # the worker starts distilling from engine a ...
    got_b = run(engine(2))       # ... while engine b generates on the main stream
    L.await_pending()
    assert got_b == want_b
    assert torch.equal(L.snapshot().to_torch("lm_w"), want_head)
    assert L.metrics()[0].kd_loss == ref.metrics()[0].kd_loss


def test_engine_pins_are_released_after_updates():
    """Engines read by a scheduled KD update are pinned until it ends (stepping one meanwhile
    raises instead of corrupting what the update reads); after the update -- sync, or async
    after await_pending -- the engine steps again."""
    import random
    shape = rb.TransformerShape.tiny(vocab=512, max_ctx=128)
    tgt = rb.TransformerModel(shape, seed=9)
    drf = rb.EagleDrafter(tgt, seed=10)
    rng = random.Random(3)
    reqs = [rb.RequestState(i, [rng.randrange(511) for _ in range(6)], -1.0, 12, rb.DecodeRng.from_seed(3, i))
            for i in range(4)]
    e = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 2, 3), "sample",
                       record_full_logprobs=False)
    e.step()
    pol = rb.KDPolicy(1, rb.WeightMode.Uniform, 0.0, 4.0, 0.5)
    for async_ in (False, True):
        L = rb.OnlineLearner(drf, pol, 3, 0.0, 64, async_)
        L.feed_engine(e, [0, 1], [1.0, 0.5])
        L.on_iteration_boundary(0)
        L.await_pending()
        assert L.drafter_version() == drf.version + 1
        e.step()  # unpinned
        L.close()
