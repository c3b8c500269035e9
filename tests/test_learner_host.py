"""CPU: host pieces of the learner / GRPO / scenario layer against the compiled reference's
fixtures (tests/golden/learner_scenarios.json): reward, group_advantages (pure host C-ABI),
ExperimentConfig JSON round trip, mix64, and a world-size-free check that every scenario name
dispatches."""
import pytest

import paper_2510_26475_b200 as rb
from conftest import load_golden
from paper_2510_26475_b200 import scenarios as sc

G = load_golden("learner_scenarios.json")


def test_reward_and_group_advantages_match_reference():
    pu = G["policy_update"]
    got = [rb.reward(s["response"]) for s in pu["samples"]]
    assert got == pu["rewards"]
    adv = []
    for g in range(0, len(got), 8):
        adv += rb.group_advantages(got[g:g + 8])
    assert adv == pu["advantages"]  # same formula, same summation order: bit-identical
    with pytest.raises(rb.InvalidArgument, match="group size must be >= 2"):
        rb.group_advantages([1.0])
    assert rb.reward([1]) == 0.0 and rb.reward([1, 2, 1, 2]) == pytest.approx(2 / 3)


def test_experiment_config_round_trip():
    d = sc.ExperimentConfig()
    assert d.to_json() == G["config_default"]
    c = sc.ExperimentConfig.from_json({"scenario": "respec", "steps": 7, "kd_weight_mode": "uniform",
                                       "timing": {"target": {"unit_cost": 3.0}}, "fixed_cfg": {"enabled": True,
                                                                                              "rounds": 1}})
    assert c.steps == 7 and c.kd.mode == rb.WeightMode.Uniform and c.timing.target.unit_cost == 3.0
    assert c.timing.target.saturation_tokens == 32 and c.fixed_cfg == rb.SDConfig.tree(1, 1, 1)
    with pytest.raises(rb.InvalidArgument, match="unknown weight mode"):
        sc.ExperimentConfig.from_json({"kd_weight_mode": "bogus"})
    assert len(d.config_grid()) == 18


def test_mix64_and_scenario_names():
    # splitmix64 of 1 (rng.hpp:15-26); the default env seeds its actor with mix64(seed)
    assert sc.mix64(1) == 0x910A2DEC89025CC1
    assert sc.scenario_names() == ["baseline", "naive-spec", "respec", "frozen", "uniform-kd", "async-ablation",
                                   "skew-demo"]
    with pytest.raises(rb.InvalidArgument, match="unknown scenario"):
        sc.run_scenario(sc.ExperimentConfig(scenario="nope"))


def test_replay_buffer_eviction():
    b = rb.ReplayBuffer(2)
    for i in range(3):
        b.push(rb.RolloutSample([i], [], []))
    assert b.size() == 2 and [s.prompt for s in b.take_all()] == [[1], [2]] and b.size() == 0


def test_round_costs_from_single_sequence_ledger():
    """spec_step_tree's RoundCost list is read back from the one-request engine's forward events
    (charge_batched_cycle over one outcome, server.cpp:154-178)."""
    ledger = [(0, 2, 2), (0, 2, 2), (1, 7, 7), (0, 2, 2), (1, 5, 5), (1, 1, 1)]
    rounds = rb._rounds_of(ledger)
    assert [(r.drafter_forwards, r.drafter_tokens_each, r.target_tokens) for r in rounds] == \
        [(2, 2, 7), (1, 2, 5), (0, 0, 1)]
    assert rb.mean_accept_len([1, 0, 3, 3]) == 1.75
