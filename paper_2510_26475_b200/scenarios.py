"""Experiment scenarios (scenarios.hpp / scenarios.cpp, config.cpp of the reference) on the GPU path.

ExperimentConfig mirrors the reference's JSON config (config.cpp:93-174); make_env,
build_profile and run_scenario follow scenarios.cpp:28-341 with every generation, KD update,
policy step and profiling wave running through the device engine (BatchEngine / OnlineLearner /
policy_update / profile). Output is the reference's ScenarioResult: a summary object plus the
steps / learner / switches JSONL streams and the profile table (write_scenario_files writes the
same files, byte for byte the same layout: sorted keys, 2-space summary).
"""
import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

from . import (KDPolicy, OnlineLearner, ProfileOptions, RequestState, RewardSpec, RoleTiming, SDConfig, SDTrainMode,
               SelectionRng, TabularARModel, Task, TimingModel, TrainOptions, WeightMode, DecodeRng, InvalidArgument,
               _check, _f64arr, kd_update, lib, make_step_requests, profile, run_generation, train_loop)
import ctypes

_M64 = (1 << 64) - 1
WARMUP_STREAM_BASE = 1 << 20  # scenarios.cpp:19
SKEW_STREAM_BASE = 2 << 20    # scenarios.cpp:20
_MODE_NAMES = {WeightMode.Reward: "reward", WeightMode.Uniform: "uniform", WeightMode.Frozen: "frozen"}


def mix64(x: int) -> int:
    """mix64 = one splitmix64 step (rng.hpp:15-26)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _sd_to_json(c: SDConfig) -> dict:
    return {"enabled": c.enabled, "rounds": c.rounds, "branching": c.branching, "draft_len": c.draft_len}


def _sd_from_json(j: dict) -> SDConfig:
    return SDConfig(j.get("rounds", 1), j.get("branching", 1), j.get("draft_len", 1), j.get("enabled", False))


def weight_mode_from_string(s: str) -> int:
    for k, v in _MODE_NAMES.items():
        if v == s:
            return k
    raise InvalidArgument(f"config: unknown weight mode '{s}'")


@dataclass
class ExperimentConfig:
    """ExperimentConfig (config.hpp:15-61) with the reference defaults."""
    seed: int = 1
    scenario: str = "baseline"
    out_dir: str = "out"
    vocab_size: int = 8
    target_order: int = 2
    drafter_order: int = 1
    temperature: float = 1.0
    actor_init_scale: float = 0.5
    reward_spec: RewardSpec = field(default_factory=lambda: RewardSpec(1, 2))
    prompts: List[List[int]] = field(default_factory=lambda: [[0, 1], [2, 3], [4, 5], [0, 2]])
    eos_biases: List[float] = field(default_factory=lambda: [1.0, 0.0, -1.0, -2.5])
    group_size: int = 8
    max_len: int = 24
    steps: int = 200
    policy_lr: float = 0.2
    kd: KDPolicy = field(default_factory=lambda: KDPolicy(1, WeightMode.Reward, 0.0, 4.0, 0.5))
    warmup_rounds: int = 4
    kd_step_cost: float = 0.02
    async_learner: bool = True
    buffer_capacity: int = 4096
    timing: TimingModel = field(default_factory=TimingModel)
    grid_rounds: List[int] = field(default_factory=lambda: [1, 2, 4])
    grid_branching: List[int] = field(default_factory=lambda: [1, 2])
    grid_draft_len: List[int] = field(default_factory=lambda: [1, 2, 4])
    batch_sizes: List[int] = field(default_factory=lambda: [1, 2, 4, 8, 16, 32, 64])
    profile_cycles: int = 64
    profile_requests: int = 64
    fixed_cfg: SDConfig = field(default_factory=lambda: SDConfig.tree(2, 1, 2))
    skew_requests: int = 32
    skew_max_len: int = 48

    def make_task(self) -> Task:  # config.cpp:7-21
        if len(self.prompts) != len(self.eos_biases):
            raise InvalidArgument("config: prompts/eos_biases length mismatch")
        return Task([list(p) for p in self.prompts], list(self.eos_biases), self.reward_spec, self.group_size,
                    self.max_len)

    def config_grid(self) -> List[SDConfig]:  # config.cpp:23-33
        return [SDConfig.tree(s, t, n) for s in self.grid_rounds for t in self.grid_branching
                for n in self.grid_draft_len]

    def to_json(self) -> dict:  # config.cpp:93-129
        def role(r):
            return {"unit_cost": r.unit_cost, "saturation_tokens": r.saturation_tokens,
                    "latency_floor": r.latency_floor}
        return {"seed": self.seed, "scenario": self.scenario, "out_dir": self.out_dir, "vocab_size": self.vocab_size,
                "target_order": self.target_order, "drafter_order": self.drafter_order,
                "temperature": self.temperature, "actor_init_scale": self.actor_init_scale,
                "golden_a": self.reward_spec.golden_a, "golden_b": self.reward_spec.golden_b,
                "prompts": self.prompts, "eos_biases": self.eos_biases, "group_size": self.group_size,
                "max_len": self.max_len, "steps": self.steps, "policy_lr": self.policy_lr,
                "kd_interval": self.kd.interval, "kd_weight_mode": _MODE_NAMES[self.kd.mode],
                "kd_clip_lo": self.kd.clip_lo, "kd_clip_hi": self.kd.clip_hi, "kd_lr": self.kd.lr,
                "warmup_rounds": self.warmup_rounds, "kd_step_cost": self.kd_step_cost,
                "async_learner": self.async_learner, "buffer_capacity": self.buffer_capacity,
                "timing": {"target": role(self.timing.target), "drafter": role(self.timing.drafter)},
                "grid_rounds": self.grid_rounds, "grid_branching": self.grid_branching,
                "grid_draft_len": self.grid_draft_len, "batch_sizes": self.batch_sizes,
                "profile_cycles": self.profile_cycles, "profile_requests": self.profile_requests,
                "fixed_cfg": _sd_to_json(self.fixed_cfg), "skew_requests": self.skew_requests,
                "skew_max_len": self.skew_max_len}

    @staticmethod
    def from_json(j: dict) -> "ExperimentConfig":  # config.cpp:131-172: missing keys keep defaults
        d = ExperimentConfig()
        c = ExperimentConfig()
        for k in ("seed", "scenario", "out_dir", "vocab_size", "target_order", "drafter_order", "temperature",
                  "actor_init_scale", "prompts", "eos_biases", "group_size", "max_len", "steps", "policy_lr",
                  "warmup_rounds", "kd_step_cost", "async_learner", "buffer_capacity", "grid_rounds",
                  "grid_branching", "grid_draft_len", "batch_sizes", "profile_cycles", "profile_requests",
                  "skew_requests", "skew_max_len"):
            setattr(c, k, j.get(k, getattr(d, k)))
        c.reward_spec = RewardSpec(j.get("golden_a", d.reward_spec.golden_a), j.get("golden_b", d.reward_spec.golden_b))
        c.kd = KDPolicy(j.get("kd_interval", d.kd.interval),
                        weight_mode_from_string(j.get("kd_weight_mode", _MODE_NAMES[d.kd.mode])),
                        j.get("kd_clip_lo", d.kd.clip_lo), j.get("kd_clip_hi", d.kd.clip_hi), j.get("kd_lr", d.kd.lr))
        if "timing" in j:
            def role(rj, dr):
                return RoleTiming(rj.get("unit_cost", dr.unit_cost), rj.get("saturation_tokens", dr.saturation_tokens),
                                  rj.get("latency_floor", dr.latency_floor))
            t = j["timing"]
            c.timing = TimingModel(role(t["target"], d.timing.target) if "target" in t else d.timing.target,
                                   role(t["drafter"], d.timing.drafter) if "drafter" in t else d.timing.drafter)
        if "fixed_cfg" in j:
            c.fixed_cfg = _sd_from_json(j["fixed_cfg"])
        return c


@dataclass
class Env:
    actor: TabularARModel
    drafter: TabularARModel
    task: Task


def make_env(cfg: ExperimentConfig) -> Env:
    """make_env (scenarios.cpp:28-51): random actor, zero drafter warmed by uniform KD on
    SD-off rollout batches (all on the device)."""
    actor = TabularARModel.random(cfg.vocab_size, cfg.target_order, cfg.temperature, cfg.actor_init_scale,
                                  mix64(cfg.seed))
    drafter = TabularARModel.zeros(cfg.vocab_size, cfg.drafter_order, cfg.temperature)
    task = cfg.make_task()
    warm = KDPolicy(1, WeightMode.Uniform, 0.0, 4.0, cfg.kd.lr)
    sel = SelectionRng(mix64(cfg.seed ^ 0x77A95D1E))
    for w in range(cfg.warmup_rounds):
        reqs = make_step_requests(task, cfg.seed, WARMUP_STREAM_BASE + w)
        run = run_generation(reqs, actor, None, None, cfg.timing, SDConfig.off(), actor.version)
        res = kd_update(drafter, run.samples, warm, sel, 0.0)
        if res.updated:
            drafter = res.drafter
    return Env(actor, drafter, task)


def build_profile(cfg: ExperimentConfig, actor, drafter):
    """build_profile (scenarios.cpp:53-62)."""
    opts = ProfileOptions(list(cfg.batch_sizes), cfg.profile_cycles, cfg.profile_requests, cfg.seed)
    return profile(actor, drafter, cfg.config_grid(), cfg.make_task().prompts, cfg.timing, opts)


SCENARIO_NAMES = ["baseline", "naive-spec", "respec", "frozen", "uniform-kd", "async-ablation", "skew-demo"]


def scenario_names() -> List[str]:
    return list(SCENARIO_NAMES)


def is_valid_scenario(name: str) -> bool:
    return name in SCENARIO_NAMES


@dataclass
class ScenarioResult:
    """ScenarioResult (scenarios.hpp:31-38)."""
    scenario: str
    summary: dict = field(default_factory=dict)
    step_lines: List[dict] = field(default_factory=list)
    learner_lines: List[dict] = field(default_factory=list)
    switch_lines: List[dict] = field(default_factory=list)
    table: Optional[object] = None


@dataclass
class TrainRun:
    result: object
    learner: list
    final_drafter: Optional[TabularARModel]


def run_training(cfg: ExperimentConfig, env: Env, sd: int, table, kd_mode: int, interval: int,
                 async_: bool) -> TrainRun:
    """run_training (scenarios.cpp:84-112)."""
    learner = None
    if sd != SDTrainMode.Off:
        pol = KDPolicy(interval, kd_mode, cfg.kd.clip_lo, cfg.kd.clip_hi, cfg.kd.lr)
        learner = OnlineLearner(env.drafter, pol, mix64(cfg.seed ^ 0x1234ABCD), cfg.kd_step_cost,
                                cfg.buffer_capacity, async_)
    opts = TrainOptions(cfg.steps, sd, cfg.fixed_cfg, table, cfg.policy_lr, cfg.seed, not async_)
    res = train_loop(env.actor, learner, env.task, cfg.timing, opts)
    run = TrainRun(res, [], None)
    if learner is not None:
        run.learner = learner.metrics()
        run.final_drafter = learner.snapshot()
        learner.shutdown()
        learner.close()
    return run


def step_line(m) -> dict:  # scenarios.cpp:114-123
    return {"step": m.step, "mean_reward": m.mean_reward, "mean_accept_len": m.mean_accept_len,
            "sim_time": m.sim_time, "actor_version": m.actor_version, "drafter_version": m.drafter_version,
            "cycles": m.cycles, "switches": m.switches}


def learner_line(m) -> dict:  # scenarios.cpp:125-134
    return {"update": m.update_idx, "drafter_version": m.drafter_version, "kd_loss": m.kd_loss,
            "samples": m.samples_used, "weight_mean": m.weight_mean, "weight_min": m.weight_min,
            "weight_max": m.weight_max, "weights_l2": m.weights_l2}


def _mean(xs) -> float:
    s = 0.0
    for x in xs:
        s += x
    return s / len(xs)


def train_summary(run: TrainRun) -> dict:  # scenarios.cpp:136-153
    ms = run.result.metrics
    tail = min(5, len(ms))
    last = [m.mean_reward for m in ms[len(ms) - tail:]]
    return {"steps": len(ms), "first_mean_reward": ms[0].mean_reward, "last_mean_reward": ms[-1].mean_reward,
            "final_mean_reward": _mean(last), "reward_improvement": _mean(last) - ms[0].mean_reward,
            "accept_len_first": ms[0].mean_accept_len, "accept_len_last": ms[-1].mean_accept_len,
            "total_sim_time": run.result.total_sim_time, "learner_updates": len(run.learner)}


def append_step_lines(out: ScenarioResult, run: TrainRun, interval: Optional[int] = None) -> None:
    for m in run.result.metrics:
        j = step_line(m)
        if interval is not None:
            j["interval"] = interval
        out.step_lines.append(j)
    for m in run.learner:
        j = learner_line(m)
        if interval is not None:
            j["interval"] = interval
        out.learner_lines.append(j)


def make_skew_requests(cfg: ExperimentConfig, task: Task) -> List[RequestState]:
    """make_skew_requests (scenarios.cpp:175-189)."""
    biases = (ctypes.c_double * max(1, cfg.skew_requests))()
    _check(lib().rs_skew_eos_biases(mix64(cfg.seed ^ 0x5EEDCAFE), cfg.skew_requests, biases))
    return [RequestState(i, list(task.prompts[i % len(task.prompts)]), biases[i], cfg.skew_max_len,
                         DecodeRng.from_seed(cfg.seed, SKEW_STREAM_BASE + i)) for i in range(cfg.skew_requests)]


def skew_run_time(cfg: ExperimentConfig, env: Env, table, forced: SDConfig, keep: Optional[list] = None) -> float:
    """skew_run_time (scenarios.cpp:191-202)."""
    snap = env.drafter
    run = run_generation(make_skew_requests(cfg, env.task), env.actor, lambda: snap, table, cfg.timing, forced,
                         env.actor.version, record_full_logprobs=False)
    if keep is not None:
        keep.append(run)
    return run.total_time


def scenario_skew_demo(cfg: ExperimentConfig) -> ScenarioResult:  # scenarios.cpp:204-268
    env = make_env(cfg)
    table = build_profile(cfg, env.actor, env.drafter)
    keep = []
    adaptive_time = skew_run_time(cfg, env, table, SDConfig.off(), keep)
    run = keep[0]
    nonincreasing = all(run.active_trace[i] <= run.active_trace[i - 1] for i in range(1, len(run.active_trace)))
    buckets = {table.bucket_for(a) for a in run.active_trace}
    lengths = [len(s.response) for s in run.samples]
    early = sum(1 for n in lengths if n <= cfg.skew_max_len // 3)
    late = sum(1 for n in lengths if n > 2 * cfg.skew_max_len // 3)
    best_fixed, worst_fixed, fixed_times = math.inf, 0.0, {}
    for fixed in cfg.config_grid():
        t = skew_run_time(cfg, env, None, fixed)
        fixed_times[fixed.key()] = t
        best_fixed = min(best_fixed, t)
        worst_fixed = max(worst_fixed, t)
    out = ScenarioResult(cfg.scenario, table=table)
    out.switch_lines = [{"cycle": sw.cycle, "active_batch": sw.active_batch, "from": sw.from_.key(),
                         "to": sw.to.key()} for sw in run.switches]
    out.summary = {"adaptive_time": adaptive_time, "best_fixed_time": best_fixed, "worst_fixed_time": worst_fixed,
                   "fixed_times": fixed_times, "num_switches": len(run.switches), "buckets_visited": len(buckets),
                   "active_trace_nonincreasing": nonincreasing, "active_trace": list(run.active_trace),
                   "response_lengths": lengths, "frac_finished_first_third": early / len(run.samples),
                   "frac_survived_two_thirds": late / len(run.samples)}
    return out


def scenario_async_ablation(cfg: ExperimentConfig) -> ScenarioResult:  # scenarios.cpp:270-294
    env = make_env(cfg)
    out = ScenarioResult(cfg.scenario)
    per = []
    for interval in (1, 3, 5):
        run = run_training(cfg, env, SDTrainMode.Fixed, None, WeightMode.Reward, interval, cfg.async_learner)
        append_step_lines(out, run, interval)
        ms = run.result.metrics
        tail = min(10, len(ms))
        per.append({"interval": interval, "final_accept_len": _mean([m.mean_accept_len for m in ms[len(ms) - tail:]]),
                    "accept_len_last_step": ms[-1].mean_accept_len, "total_sim_time": run.result.total_sim_time,
                    "learner_updates": len(run.learner)})
    out.summary = {"per_interval": per}
    return out


def scenario_train(cfg: ExperimentConfig) -> ScenarioResult:  # scenarios.cpp:296-326
    env = make_env(cfg)
    out = ScenarioResult(cfg.scenario)
    sd, kd_mode, table = SDTrainMode.Fixed, WeightMode.Reward, None
    if cfg.scenario == "baseline":
        sd = SDTrainMode.Off
    elif cfg.scenario in ("naive-spec", "frozen"):
        kd_mode = WeightMode.Frozen
    elif cfg.scenario == "uniform-kd":
        kd_mode = WeightMode.Uniform
    elif cfg.scenario == "respec":
        sd = SDTrainMode.Adaptive
        table = build_profile(cfg, env.actor, env.drafter)
        out.table = table
    else:
        raise InvalidArgument(f"unknown scenario '{cfg.scenario}'")
    run = run_training(cfg, env, sd, table, kd_mode, cfg.kd.interval, cfg.async_learner)
    append_step_lines(out, run)
    out.summary = train_summary(run)
    out.summary["scenario"] = cfg.scenario
    return out


def run_scenario(cfg: ExperimentConfig) -> ScenarioResult:
    """run_scenario (scenarios.cpp:330-341)."""
    if not is_valid_scenario(cfg.scenario):
        raise InvalidArgument(f"unknown scenario '{cfg.scenario}'")
    if cfg.scenario == "skew-demo":
        return scenario_skew_demo(cfg)
    if cfg.scenario == "async-ablation":
        return scenario_async_ablation(cfg)
    out = scenario_train(cfg)
    out.scenario = cfg.scenario
    return out


def _dump(j, indent=None) -> str:
    return json.dumps(j, sort_keys=True, indent=indent, separators=(",", ":") if indent is None else None)


def write_scenario_files(result: ScenarioResult, out_dir: str) -> None:
    """write_scenario_files (scenarios.cpp:359-381): steps/learner/switches JSONL, summary.json
    and, when the scenario profiled, profile.csv + profile.json."""
    os.makedirs(out_dir, exist_ok=True)
    for name, lines in (("steps.jsonl", result.step_lines), ("learner.jsonl", result.learner_lines),
                        ("switches.jsonl", result.switch_lines)):
        with open(os.path.join(out_dir, name), "w") as f:
            for j in lines:
                f.write(_dump(j) + "\n")
    with open(os.path.join(out_dir, "summary.json"), "w") as f:
        f.write(_dump(result.summary, 2) + "\n")
    if result.table is not None:
        with open(os.path.join(out_dir, "profile.csv"), "w") as f:
            f.write(result.table.to_csv())
        with open(os.path.join(out_dir, "profile.json"), "w") as f:
            f.write(_dump(result.table.to_json(), 2) + "\n")
