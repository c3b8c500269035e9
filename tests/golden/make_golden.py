"""Generates tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref/librespec_ref.so,
built from /root/reference/proj/core by oracle/Makefile). TEST INFRASTRUCTURE ONLY.

    make -C oracle && python tests/golden/make_golden.py

The fixtures let the GPU box (which has no /root/reference) check the CUDA engine against
the reference's own outputs. Every case records its inputs and the reference outputs.
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_client import Reference, fnv1a_responses  # noqa: E402

R = Reference()


def cfg(s, t, n):
    return {"s": s, "t": t, "n": n, "enabled": True}


OFF = {"s": 1, "t": 1, "n": 1, "enabled": False}


def run(case, record=True):
    out = R("run_generation", record_logprobs=record, **case)
    res = {"cycles": out["cycles"], "total_time": out["total_time"], "active_trace": out["active_trace"],
           "switches": out["switches"], "ledger": out["ledger"], "prefill_events": out["prefill_events"],
           "accept_lens": out["accept_lens"],
           "responses": [s["response"] for s in out["samples"]],
           "per_request_accept_lens": [s["accept_lens"] for s in out["samples"]],
           "steps": [[[st["logp"], st["drafted"], st["logq"]] for st in s["steps"]] for s in out["samples"]],
           "fnv": fnv1a_responses([s["response"] for s in out["samples"]])}
    if record:
        res["target_logprobs"] = [[st["target_logprobs"] for st in s["steps"]] for s in out["samples"]]
    return res


def random_table(rng, V, order, scale):
    return [rng.gauss(0.0, scale) for _ in range(V ** order * V)]


def main():
    # 1. SURVEY.md Appendix B: default env, step-0 requests, forced configs.
    env = R("make_env", seed=1, with_profile=True)
    reqs = R("make_step_requests", seed=1, step=0)["requests"]
    fp = {"actor": env["actor"], "drafter": env["drafter"], "requests": reqs, "table": env["table"], "cases": []}
    for c in [OFF, cfg(1, 1, 3), cfg(2, 1, 2), cfg(1, 4, 5)]:
        case = {"target": env["actor"], "drafter": env["drafter"], "requests": reqs, "forced": c}
        fp["cases"].append({"forced": c, "out": run(case, record=(c == cfg(1, 1, 3)))})
    # adaptive (table) run on the same requests
    case = {"target": env["actor"], "drafter": env["drafter"], "requests": reqs, "table": env["table"]}
    fp["adaptive"] = run(case, record=False)
    with open(os.path.join(HERE, "appendix_b.json"), "w") as f:
        json.dump(fp, f)

    # 2. Random tabular engines: vocab, orders, configs, EOS hazards, max_len edge cases.
    rng = random.Random(20251026)
    cases = []
    configs = [cfg(1, 1, 1), cfg(1, 1, 4), cfg(2, 1, 2), cfg(1, 2, 3), cfg(1, 3, 2), cfg(2, 2, 2), cfg(3, 2, 1),
               cfg(1, 4, 5), cfg(4, 1, 1), cfg(2, 3, 3)]
    for k in range(24):
        V = rng.choice([3, 4, 5, 8, 16])
        t_order, d_order = rng.choice([(2, 1), (1, 1), (1, 0), (2, 2), (0, 0)])
        tau = rng.choice([1.0, 1.0, 0.7, 1.5])
        target = {"kind": "tabular", "vocab": V, "order": t_order, "temperature": tau, "version": 0,
                  "logits": random_table(rng, V, t_order, rng.choice([0.5, 1.0, 2.0]))}
        drafter = {"kind": "tabular", "vocab": V, "order": d_order, "temperature": tau, "version": k,
                   "logits": random_table(rng, V, d_order, rng.choice([0.5, 1.0, 2.0]))}
        nreq = rng.choice([1, 3, 8, 13])
        requests = []
        for i in range(nreq):
            plen = rng.choice([0, 1, 2, 3])
            requests.append({"id": i, "prompt": [rng.randrange(V - 1) for _ in range(plen)],
                             "eos_bias": rng.choice([-3.0, -1.0, 0.0, 1.0, 2.5]),
                             "max_len": rng.choice([1, 2, 3, 7, 16, 30]), "seed": rng.randrange(2 ** 63),
                             "stream": rng.randrange(2 ** 40)})
        forced = OFF if k % 6 == 0 else configs[k % len(configs)]
        case = {"target": target, "drafter": drafter, "requests": requests, "forced": forced}
        out = run(case, record=V <= 8)
        cases.append({"case": case, "out": out})
    with open(os.path.join(HERE, "tabular_engine.json"), "w") as f:
        json.dump(cases, f)

    # 3. KD update on the step-0 SD-off rollouts with rewards (SURVEY App. B KD fingerprint).
    base = R("run_generation", target=env["actor"], drafter=None, requests=reqs, forced=OFF, record_logprobs=True)
    rewards = R("reward", responses=[s["response"] for s in base["samples"]])["rewards"]
    buf = []
    for s, r in zip(base["samples"], rewards):
        buf.append({"prompt": s["prompt"], "response": s["response"], "steps": s["steps"], "eos_bias": s["eos_bias"],
                    "reward": r})
    kd_cases = []
    for pol, seed in [({"interval": 1, "mode": "reward", "clip_lo": 0.0, "clip_hi": 4.0, "lr": 0.5}, 123),
                      ({"interval": 3, "mode": "uniform", "clip_lo": 0.0, "clip_hi": 4.0, "lr": 0.1}, 7),
                      ({"interval": 2, "mode": "reward", "clip_lo": 0.5, "clip_hi": 2.0, "lr": 0.05}, 99)]:
        out = R("kd_update", drafter=env["drafter"], buffer=buf, policy=pol, selection_seed=seed, cost_per_token=0.02)
        kd_cases.append({"policy": pol, "selection_seed": seed, "out": out})
    with open(os.path.join(HERE, "kd_update.json"), "w") as f:
        json.dump({"drafter": env["drafter"], "buffer": buf, "cases": kd_cases}, f)
    learner_and_scenarios(env)
    for name in ["appendix_b.json", "tabular_engine.json", "kd_update.json", "learner_scenarios.json"]:
        print(name, os.path.getsize(os.path.join(HERE, name)))


# Small profiling grid for the scenario fixtures (the full default grid is checked separately
# through build_profile's best-config list).
SMALL_PROFILE = {"batch_sizes": [1, 2, 4, 8, 16, 32], "profile_cycles": 16, "profile_requests": 32}


def learner_and_scenarios(env):
    """OnlineLearner scripts (learner.cpp:162-289), policy_update (rl.cpp:74-88), the default
    build_profile, and run_scenario for every scenario (scenarios.cpp:28-341) at small sizes."""
    out = {"drafter": env["drafter"], "actor": env["actor"]}
    # rollout batches with rewards: SD-off generations of steps 0..5, 8 samples each
    batches = []
    for step in range(6):
        reqs = R("make_step_requests", seed=1, step=step)["requests"][step * 4: step * 4 + 8]
        gen = R("run_generation", target=env["actor"], drafter=None, requests=reqs, forced=OFF, record_logprobs=True)
        rewards = R("reward", responses=[s["response"] for s in gen["samples"]])["rewards"]
        batches.append([{"prompt": s["prompt"], "response": s["response"],
                         "steps": [{"token": t, "target_logprobs": st["target_logprobs"]}
                                   for t, st in zip(s["response"], s["steps"])],
                         "eos_bias": s["eos_bias"], "reward": r} for s, r in zip(gen["samples"], rewards)])
    out["batches"] = batches
    learners = []
    for name, pol, cap, seed in [
            ("interval2_reward_evict", {"interval": 2, "mode": "reward", "clip_lo": 0.0, "clip_hi": 4.0, "lr": 0.3}, 12, 31),
            ("interval1_uniform", {"interval": 1, "mode": "uniform", "clip_lo": 0.0, "clip_hi": 4.0, "lr": 0.5}, 4096, 7),
            ("interval3_clip", {"interval": 3, "mode": "reward", "clip_lo": 0.5, "clip_hi": 2.0, "lr": 0.2}, 4096, 5),
            ("frozen", {"interval": 1, "mode": "frozen", "clip_lo": 0.0, "clip_hi": 4.0, "lr": 0.5}, 64, 7)]:
        script = [{"feed": b, "boundary": it, "await": True} for it, b in enumerate(batches)]
        res = {}
        for mode in (False, True):
            res["async" if mode else "sync"] = R("online_learner", drafter=env["drafter"], policy=pol, selection_seed=seed,
                                                   cost_per_token=0.02, capacity=cap, script=script, **{"async": mode})
        assert res["sync"] == res["async"], name  # learner.hpp:91-97: async changes timing, not semantics
        learners.append({"name": name, "policy": pol, "capacity": cap, "selection_seed": seed, "out": res["sync"]})
    out["learners"] = learners
    # policy_update on one group-structured batch (step-0 requests, all 32)
    reqs = R("make_step_requests", seed=1, step=0)["requests"]
    gen = R("run_generation", target=env["actor"], drafter=None, requests=reqs, forced=OFF, record_logprobs=False)
    rewards = R("reward", responses=[s["response"] for s in gen["samples"]])["rewards"]
    adv = []
    for g in range(0, len(rewards), 8):
        adv += R("group_advantages", rewards=rewards[g:g + 8])["advantages"]
    samples = [{"prompt": s["prompt"], "response": s["response"], "eos_bias": s["eos_bias"], "actor_version": 0}
               for s in gen["samples"]]
    out["policy_update"] = {"samples": samples, "rewards": rewards, "advantages": adv, "lr": 0.2,
                            "out": R("policy_update", actor=env["actor"], samples=samples, advantages=adv, lr=0.2)}
    out["default_profile"] = R("build_profile", config={})
    out["config_default"] = R("config_roundtrip", config={})
    scen = []
    for name, over in [("baseline", {"steps": 6}), ("naive-spec", {"steps": 6}), ("frozen", {"steps": 5}),
                       ("uniform-kd", {"steps": 6, "async_learner": False}), ("respec", dict(SMALL_PROFILE, steps=6)),
                       ("async-ablation", {"steps": 6}), ("skew-demo", dict(SMALL_PROFILE)),
                       ("respec", dict(SMALL_PROFILE, steps=4, kd_interval=2, async_learner=False, seed=3))]:
        c = dict(over, scenario=name)
        scen.append({"config": c, "out": R("run_scenario", config=c)})
    out["scenarios"] = scen
    with open(os.path.join(HERE, "learner_scenarios.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
