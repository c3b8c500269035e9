"""Multi-GPU plumbing for the rollout path -- no PyTorch.

Generation shards BY PROMPT: every rank runs its own BatchEngine on its own requests and no
collective touches the decode path (a request's tokens depend only on its own RNG streams and
the models -- verified on the compiled reference for fixed configs). The one exchange is the
KD update of the drafter: the ceil(N/I) selection runs replicated on every rank from the same
selection stream over GLOBAL buffer indices (learner.cpp:107-121), each rank computes the
reward-weighted gradient of its locally held selected samples on its GPU (K5 + the drafter
backward), and the gradients are summed by the library's NCCL communicator (`Comm`, rs_comm_*:
NCCL over NVLink / NVSwitch, in place on the library-owned gradient buffer). The sum equals the
reference's gradient up to summation order (learner.cpp:68-80 sums over samples).

Ranks find each other through the launcher's environment (RANK / WORLD_SIZE / LOCAL_RANK /
MASTER_ADDR / MASTER_PORT, as torchrun sets them): rank 0 creates the NCCL unique id and hands
it to the others over a TCP socket (Comm.from_env). Host-side reductions in tests go through a
caller-supplied hook (`all_reduce=`), e.g. gloo on CPU."""
from __future__ import annotations

import ctypes
import os
import socket
import time
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

from . import (Device, DeviceBuffer, KDPolicy, RolloutSample, SelectionRng, TabularARModel, _KDSample, _check,
               _f64arr, _i32arr, default_device, kd_grad_transformer, kd_weight, lib)

RS_COMM_ID_BYTES = 128
_DT = {"f32": 0, "f64": 1, "i64": 2}
_OP = {"sum": 0, "max": 1}


def dist_env() -> Tuple[int, int, int]:
    """(rank, world size, local rank) from the launcher's environment (1 rank when unset)."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _rendezvous(rank: int, world: int, payload: Optional[bytes], addr: str, port: int, timeout: float) -> bytes:
    """Rank 0 serves `payload` to ranks 1..world-1 over TCP; they return it."""
    if rank == 0:
        srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        srv.bind((addr, port))
        srv.listen(world)
        srv.settimeout(timeout)
        try:
            for _ in range(world - 1):
                c, _ = srv.accept()
                with c:
                    c.sendall(payload)
        finally:
            srv.close()
        return payload
    deadline = time.time() + timeout
    while True:
        try:
            with socket.create_connection((addr, port), timeout=5) as c:
                buf = b""
                while len(buf) < RS_COMM_ID_BYTES:
                    chunk = c.recv(RS_COMM_ID_BYTES - len(buf))
                    if not chunk:
                        raise ConnectionError("rendezvous: short read")
                    buf += chunk
                return buf
        except OSError:
            if time.time() > deadline:
                raise TimeoutError(f"rendezvous with rank 0 at {addr}:{port} timed out")
            time.sleep(0.2)


class Comm:
    """One rank of the library's NCCL communicator (rs_comm_create): the drafter-gradient
    all-reduce of the prompt-sharded KD update, plus small host reductions (losses, token
    counts, max-over-ranks device times)."""

    def __init__(self, nranks: int, rank: int, uid: bytes, device: Optional[Device] = None):
        self.device = device or default_device()
        self.size, self.rank = nranks, rank
        idbuf = (ctypes.c_uint8 * RS_COMM_ID_BYTES).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(lib().rs_comm_create(self.device.handle, nranks, rank, idbuf, ctypes.byref(h)))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * RS_COMM_ID_BYTES)()
        _check(lib().rs_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl_version() -> int:
        v = ctypes.c_int32()
        _check(lib().rs_nccl_version(ctypes.byref(v)))
        return v.value

    @staticmethod
    def from_env(device: Optional[Device] = None, timeout: float = 300.0) -> "Comm":
        """All ranks of a torchrun-style launch: rank 0's unique id reaches the others over
        MASTER_ADDR : (RS_COMM_PORT or MASTER_PORT + 17)."""
        rank, world, _ = dist_env()
        addr = os.environ.get("MASTER_ADDR", "127.0.0.1")
        port = int(os.environ.get("RS_COMM_PORT", int(os.environ.get("MASTER_PORT", 29500)) + 17))
        uid = Comm.unique_id() if rank == 0 else None
        if world > 1:
            uid = _rendezvous(rank, world, uid, addr, port, timeout)
        return Comm(world, rank, uid, device)

    def allreduce_(self, buf, count: Optional[int] = None, dtype: str = "f32", op: str = "sum"):
        """In place on a device buffer (DeviceBuffer / pointer), on the device's stream."""
        ptr = buf.data_ptr() if hasattr(buf, "data_ptr") else int(buf)
        if count is None:
            count = buf.nbytes // (8 if dtype in ("f64", "i64") else 4)
        _check(lib().rs_comm_allreduce(self.handle, self.device.handle, ctypes.c_void_p(ptr), count, _DT[dtype],
                                       _OP[op]))
        return buf

    def allreduce_host(self, vals: Sequence[float], op: str = "sum") -> List[float]:
        arr = (ctypes.c_double * max(1, len(vals)))(*vals)
        _check(lib().rs_comm_allreduce_host(self.handle, self.device.handle, arr, len(vals), _OP[op]))
        return list(arr[:len(vals)])

    def barrier(self) -> None:
        self.allreduce_host([0.0])

    def host_all_reduce(self) -> Callable[[List[float]], List[float]]:
        """The `all_reduce=` hook of kd_step_distributed (sum of a host vector, in slices)."""
        def fn(vec):
            out = []
            for i in range(0, len(vec), 64):
                out += self.allreduce_host(vec[i:i + 64])
            return out
        return fn

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().rs_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


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
    (Comm.host_all_reduce() on GPUs, gloo in the CPU tests; None = single rank)."""
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
                                    comm: Optional[Comm] = None, engine=None,
                                    local_req_ids: Optional[Sequence[int]] = None, grad: Optional[DeviceBuffer] = None
                                    ) -> TransformerKDStep:
    """Prompt-sharded kd_update for an EAGLE drafter: replicated selection + reward weights over
    GLOBAL buffer indices (learner.cpp:107-140), this rank's K5 + whole-drafter gradient on its
    GPU, ONE in-place all-reduce of the fp32 gradient buffer (every drafter tensor) plus the loss
    through the library's NCCL communicator -- the only collective of the whole rollout path --
    then the same SGD step (-lr) on every rank, so every rank publishes the same snapshot.

    With `engine` (this rank's BatchEngine that generated the local rollouts; local_req_ids[k] =
    its request index of local_samples[k]) the gradient comes from the engine's resident KV cache
    and features (BatchEngine.kd_grad) instead of a teacher-forced recompute of the prompts."""
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
        loss, grad = engine.kd_grad(drafter, [q for *_, q in mine], [w for _, _, w, _ in mine], grad=grad)
    else:
        loss, grad = kd_grad_transformer(drafter, [s for _, s, _, _ in mine], [w for _, _, w, _ in mine], grad=grad)
    if comm is not None and comm.size > 1:
        comm.allreduce_(grad)
        loss = comm.allreduce_host([loss])[0]
    new = drafter.apply_grad(grad, -policy.lr)
    tokens = sum(global_lengths[i] for i in sel)
    return TransformerKDStep(new, loss, sel, [weights[i] for i in sel], len(sel), sim_cost_per_token * tokens)
