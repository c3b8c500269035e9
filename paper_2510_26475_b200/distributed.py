"""Multi-GPU plumbing for the rollout path.

Generation shards BY PROMPT: every rank runs its own BatchEngine on its own requests and no
collective touches the decode path (a request's tokens depend only on its own RNG streams and
the models -- verified on the compiled reference for fixed configs). The one exchange is the
KD update of the drafter: the ceil(N/I) selection runs replicated on every rank from the same
selection stream over GLOBAL buffer indices (learner.cpp:107-121), each rank computes the
reward-weighted gradient of its locally held selected samples on its GPU (K5), and the
gradients are summed with torch.distributed (NCCL over NVLink on the GPUs, gloo in the CPU
tests). The sum equals the reference's gradient up to fp64 summation order
(learner.cpp:68-80 sums over samples)."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

from . import (KDPolicy, RolloutSample, SelectionRng, TabularARModel, _KDSample, _check, _f64arr, _i32arr,
               kd_grad_transformer, kd_weight, lib)


def shard_requests(requests: Sequence, rank: int, world: int, group_size: int = 1) -> List:
    """Requests of rank `rank`: GRPO groups (group_size consecutive requests, rl.cpp:97-109)
    stay together so group advantages stay local; groups are dealt round-robin so the length
    skew of different prompts spreads evenly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_requests: bad rank / world")
    if group_size < 1 or len(requests) % group_size:
        raise ValueError("shard_requests: request count must be a multiple of group_size")
    groups = [list(requests[i:i + group_size]) for i in range(0, len(requests), group_size)]
    return [r for g in groups[rank::world] for r in g]


def kd_select(n: int, interval: int, selection_rng: SelectionRng) -> List[int]:
    """The kd_update selection (learner.cpp:107-121); advances selection_rng in place."""
    idx = (ctypes.c_int32 * max(1, n))()
    take = ctypes.c_int32()
    _check(lib().rs_kd_select(n, interval, selection_rng.state, idx, ctypes.byref(take)))
    return list(idx[:take.value])


def _samples(buffer: Sequence[RolloutSample]):
    keep = []
    arr = (_KDSample * max(1, len(buffer)))()
    for i, s in enumerate(buffer):
        p, r = _i32arr(s.prompt), _i32arr(s.response)
        lp = _f64arr([x for st in s.steps for x in st.target_logprobs])
        keep += [p, r, lp]
        arr[i] = _KDSample(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), len(s.prompt),
                           ctypes.cast(r, ctypes.POINTER(ctypes.c_int32)), len(s.response),
                           ctypes.cast(lp, ctypes.POINTER(ctypes.c_double)), s.eos_bias, s.reward)
    return arr, keep


def kd_grad_tabular(drafter: TabularARModel, samples: Sequence[RolloutSample],
                    weights: Sequence[float]) -> Tuple[List[float], float]:
    """K5 on the GPU: sum_i w_i (q - p~)/tau per visited row, and sum_i w_i KL_i."""
    arr, keep = _samples(samples)
    n = drafter.vocab_size ** (drafter.order + 1)
    g = (ctypes.c_double * n)()
    loss = ctypes.c_double()
    _check(lib().rs_kd_grad_tabular(drafter.device.handle, drafter.handle, arr, len(samples), _f64arr(weights), g,
                                    ctypes.byref(loss)))
    return list(g), loss.value


def apply_delta(drafter: TabularARModel, grad: Sequence[float], scale: float) -> TabularARModel:
    """with_logits_delta(grad * scale) (model.cpp:161-170): a new model, version + 1."""
    h = ctypes.c_void_p()
    _check(lib().rs_tabular_apply_delta(drafter.device.handle, drafter.handle, _f64arr(grad), scale,
                                        ctypes.byref(h)))
    return TabularARModel._wrap(h, drafter.order, drafter.temperature, drafter.device)


@dataclass
class DistributedKDResult:
    grad: List[float]
    loss: float
    selected: List[int]
    weights: List[float]
    samples_used: int
    sim_time: float


def kd_step_distributed(global_rewards: Sequence[float], global_lengths: Sequence[int],
                        local_samples: Sequence[RolloutSample], local_global_idx: Sequence[int], policy: KDPolicy,
                        selection_rng: SelectionRng, sim_cost_per_token: float,
                        grad_fn: Callable[[Sequence[RolloutSample], Sequence[float]], Tuple[List[float], float]],
                        all_reduce: Optional[Callable[[List[float]], List[float]]] = None) -> DistributedKDResult:
    """One prompt-sharded KD step (kd_update, learner.cpp:98-160, minus the weight update):
    replicated selection and weights, local K5 gradient of the selected samples this rank
    holds, then the cross-rank sum. `all_reduce(vec) -> vec` sums a float vector over ranks
    (torch.distributed in practice; None = single rank)."""
    if policy.mode == 2:
        from . import LogicError
        raise LogicError("kd_update: frozen drafter takes no updates")
    sel = kd_select(len(global_rewards), policy.interval, selection_rng)
    batch_rewards = [global_rewards[i] for i in sel]
    weights = {i: kd_weight(global_rewards[i], batch_rewards, policy) for i in sel}
    order = {g: k for k, g in enumerate(sel)}  # reference order of the selected samples
    mine = sorted([(order[g], s, weights[g]) for s, g in zip(local_samples, local_global_idx) if g in weights])
    grad, loss = grad_fn([s for _, s, _ in mine], [w for _, _, w in mine])
    vec = list(grad) + [loss]
    if all_reduce is not None:
        vec = all_reduce(vec)
    tokens = sum(global_lengths[i] for i in sel)
    return DistributedKDResult(vec[:-1], vec[-1], sel, [weights[i] for i in sel], len(sel),
                               sim_cost_per_token * tokens)


def torch_all_reduce(group=None, device: str = "cpu") -> Callable[[List[float]], List[float]]:
    """Sum over ranks with torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""
    import torch
    import torch.distributed as dist

    def fn(vec):
        t = torch.tensor(vec, dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().tolist()

    return fn


@dataclass
class TransformerKDStep:
    drafter: object          # the new EagleDrafter snapshot (version + 1), identical on every rank
    loss: float              # sum over ALL ranks' selected samples of w_i KL_i
    selected: List[int]
    weights: List[float]
    samples_used: int
    sim_time: float


def kd_step_distributed_transformer(drafter, global_rewards: Sequence[float], global_lengths: Sequence[int],
                                    local_samples: Sequence[RolloutSample], local_global_idx: Sequence[int],
                                    policy: KDPolicy, selection_rng: SelectionRng, sim_cost_per_token: float,
                                    group=None, reduce: bool = True, engine=None,
                                    local_req_ids: Optional[Sequence[int]] = None) -> TransformerKDStep:
    """Prompt-sharded kd_update for an EAGLE drafter: replicated selection + reward weights over
    GLOBAL buffer indices (learner.cpp:107-140), this rank's K5 + LM-head gradient on its GPU,
    ONE all-reduce of the fp32 [V, d] gradient (and the loss) with torch.distributed -- NCCL over
    NVLink on a B200 box, the only collective of the whole rollout path -- then the same SGD
    step (-lr) on every rank, so every rank publishes the same snapshot.

    With `engine` (this rank's BatchEngine that generated the local rollouts; local_req_ids[k] =
    its request index of local_samples[k]) the gradient comes from the engine's resident KV cache
    and features (BatchEngine.kd_grad) instead of a teacher-forced recompute of the prompts."""
    import torch
    if policy.mode == 2:
        from . import LogicError
        raise LogicError("kd_update: frozen drafter takes no updates")
    sel = kd_select(len(global_rewards), policy.interval, selection_rng)
    batch_rewards = [global_rewards[i] for i in sel]
    weights = {i: kd_weight(global_rewards[i], batch_rewards, policy) for i in sel}
    order = {g: k for k, g in enumerate(sel)}
    rids = list(local_req_ids) if local_req_ids is not None else list(range(len(local_samples)))
    mine = sorted([(order[g], s, weights[g], q) for s, g, q in zip(local_samples, local_global_idx, rids)
                   if g in weights], key=lambda t: t[0])
    if engine is not None:
        loss, grad = engine.kd_grad(drafter, [q for *_, q in mine], [w for _, _, w, _ in mine])
    else:
        loss, grad = kd_grad_transformer(drafter, [s for _, s, _, _ in mine], [w for _, _, w, _ in mine])
    if reduce:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
            lt = torch.tensor([loss], dtype=torch.float64, device=grad.device)
            dist.all_reduce(lt, op=dist.ReduceOp.SUM, group=group)
            loss = float(lt.item())
    new = drafter.apply_grad(grad, -policy.lr)
    tokens = sum(global_lengths[i] for i in sel)
    return TransformerKDStep(new, loss, sel, [weights[i] for i in sel], len(sel), sim_cost_per_token * tokens)
