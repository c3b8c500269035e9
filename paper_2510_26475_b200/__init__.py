"""paper_2510_26475_b200 -- B200-native ReSpec rollout hot path.

Python mirror of the reference's C++ API for the batched speculative-decode step
(/root/reference/proj/core: specdec.hpp, server.hpp, learner.hpp), bound with ctypes to
the C-ABI library librespec_b200.so (include/respec_b200.h). Every compute call runs in
the CUDA library; there is no CPU fallback -- if the library is missing the import of
`lib()` raises.

Names, argument meaning and error behaviour follow the reference:
  SDConfig, TabularARModel, ProfileTable, RequestState, DecodeRng, BatchEngine,
  run_generation, GenerationRun, RolloutSample, StepRecord, KDPolicy, WeightMode,
  kd_weight, kd_update.
Exceptions: std::invalid_argument -> InvalidArgument (ValueError), std::runtime_error ->
EngineError (RuntimeError), std::logic_error -> LogicError.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librespec_b200.so")


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class EngineError(RuntimeError):
    """std::runtime_error in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference."""


class CudaError(RuntimeError):
    pass


RS_OK, RS_EINVAL, RS_ESTATE, RS_ELOGIC, RS_ECUDA, RS_ENOMEM = range(6)
RS_VERIFY_SAMPLE, RS_VERIFY_GREEDY = 0, 1
RS_DTYPE_BF16, RS_DTYPE_F32 = 0, 1


# ---- C structs ------------------------------------------------------------------------------
class _SDConfig(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int32), ("branching", ctypes.c_int32), ("draft_len", ctypes.c_int32),
                ("enabled", ctypes.c_int32)]


class _RoleTiming(ctypes.Structure):
    _fields_ = [("unit_cost", ctypes.c_double), ("saturation_tokens", ctypes.c_int32),
                ("latency_floor", ctypes.c_double)]


class _TimingModel(ctypes.Structure):
    _fields_ = [("target", _RoleTiming), ("drafter", _RoleTiming)]


class _Request(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("prompt", ctypes.POINTER(ctypes.c_int32)), ("prompt_len", ctypes.c_int32),
                ("eos_bias", ctypes.c_double), ("max_len", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("stream_id", ctypes.c_uint64)]


class _SwitchEvent(ctypes.Structure):
    _fields_ = [("cycle", ctypes.c_int32), ("active_batch", ctypes.c_int32), ("from_", _SDConfig), ("to", _SDConfig)]


class _ForwardEvent(ctypes.Structure):
    _fields_ = [("role", ctypes.c_int32), ("positions", ctypes.c_int32), ("batch_tokens", ctypes.c_int32)]


class _StepInfo(ctypes.Structure):
    _fields_ = [("active_batch", ctypes.c_int32), ("mode", _SDConfig), ("drafter_version", ctypes.c_int32),
                ("emitted_tokens", ctypes.c_int32), ("drafted_cycles", ctypes.c_int32),
                ("accepted_drafted", ctypes.c_int32), ("redraft_passes", ctypes.c_int32), ("step_ms", ctypes.c_float),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64)]


class _TransformerShape(ctypes.Structure):
    _fields_ = [("vocab", ctypes.c_int32), ("d_model", ctypes.c_int32), ("n_layers", ctypes.c_int32),
                ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("d_ff", ctypes.c_int32), ("max_ctx", ctypes.c_int32), ("rope_theta", ctypes.c_float),
                ("rms_eps", ctypes.c_float), ("init_std", ctypes.c_float), ("logit_scale", ctypes.c_float),
                ("temperature", ctypes.c_double)]


class _KDPolicy(ctypes.Structure):
    _fields_ = [("interval", ctypes.c_int32), ("mode", ctypes.c_int32), ("clip_lo", ctypes.c_double),
                ("clip_hi", ctypes.c_double), ("lr", ctypes.c_double)]


class _KDSample(ctypes.Structure):
    _fields_ = [("prompt", ctypes.POINTER(ctypes.c_int32)), ("prompt_len", ctypes.c_int32),
                ("response", ctypes.POINTER(ctypes.c_int32)), ("response_len", ctypes.c_int32),
                ("target_logprobs", ctypes.POINTER(ctypes.c_double)), ("eos_bias", ctypes.c_double),
                ("reward", ctypes.c_double)]


class _KDResult(ctypes.Structure):
    _fields_ = [("updated", ctypes.c_int32), ("samples_used", ctypes.c_int32), ("loss", ctypes.c_double),
                ("weight_mean", ctypes.c_double), ("weight_min", ctypes.c_double), ("weight_max", ctypes.c_double),
                ("sim_time", ctypes.c_double)]


class _LearnerMetric(ctypes.Structure):
    _fields_ = [("update_idx", ctypes.c_int32), ("drafter_version", ctypes.c_int32), ("kd_loss", ctypes.c_double),
                ("samples_used", ctypes.c_int32), ("weight_mean", ctypes.c_double), ("weight_min", ctypes.c_double),
                ("weight_max", ctypes.c_double), ("weights_l2", ctypes.c_double)]


# Every symbol include/respec_b200.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = [
    "rs_model_tensor_shape", "rs_model_load_tensor", "rs_model_store_tensor",
    "rs_last_error", "rs_version", "rs_launch_count", "rs_launch_count_reset",
    "rs_ctx_create", "rs_ctx_destroy", "rs_ctx_sync", "rs_ctx_set_stream",
    "rs_tabular_create", "rs_tabular_logits", "rs_transformer_create", "rs_drafter_create",
    "rs_model_version", "rs_model_vocab", "rs_model_destroy",
    "rs_table_create", "rs_table_set_entry", "rs_table_finalize", "rs_table_bucket_for", "rs_table_solve",
    "rs_table_best_for_bucket", "rs_table_entry", "rs_table_to_csv", "rs_table_destroy",
    "rs_engine_create", "rs_engine_set_drafter", "rs_engine_step", "rs_engine_all_done", "rs_engine_active_batch",
    "rs_engine_cycles", "rs_engine_prefill_events", "rs_engine_ledger_time", "rs_engine_ledger",
    "rs_engine_switches", "rs_engine_active_trace", "rs_engine_drafter_versions", "rs_engine_response",
    "rs_engine_steps", "rs_engine_step_logprobs", "rs_engine_accept_lens", "rs_engine_destroy",
    "rs_engine_set_capture", "rs_engine_capture_count", "rs_engine_capture_read", "rs_engine_capture_read_f32",
    "rs_kd_weight", "rs_kd_update_tabular", "rs_mt19937_64_seed", "rs_gemm_bf16",
    "rs_model_tensor", "rs_memcpy_d2d", "rs_model_params", "rs_prof_enable", "rs_prof_reset", "rs_prof_json", "rs_set_tuning", "rs_lm_head_bf16", "rs_row_stats", "rs_kd_grad_transformer", "rs_drafter_apply_grad",
    "rs_kd_update_transformer", "rs_engine_step_tokens", "rs_profile_measured",
    "rs_kd_select", "rs_kd_grad_tabular", "rs_tabular_apply_delta", "rs_model_retain",
    "rs_learner_create", "rs_learner_destroy", "rs_learner_feed", "rs_learner_on_iteration_boundary",
    "rs_learner_await_pending", "rs_learner_shutdown", "rs_learner_snapshot", "rs_learner_drafter_version",
    "rs_learner_total_sim_time", "rs_learner_buffer_size", "rs_learner_metrics",
    "rs_reward", "rs_group_advantages", "rs_policy_update_tabular",
    "rs_engine_set_stop_at_eos", "rs_profile_simulated", "rs_tabular_random", "rs_skew_eos_biases",
    "rs_engine_kd_grad", "rs_engine_rng_export", "rs_engine_rng_import", "rs_learner_feed_engine",
    "rs_drafter_grad_layout", "rs_nccl_version", "rs_comm_unique_id", "rs_comm_create", "rs_comm_destroy",
    "rs_comm_size", "rs_comm_allreduce", "rs_comm_allreduce_host", "rs_device_alloc", "rs_device_free",
    "rs_memset_async", "rs_memcpy_h2d", "rs_memcpy_d2h",
]

_lib = None


def lib():
    """Load librespec_b200.so (built in-tree by __graft_entry__.build()). Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        i32, i64, u64, dbl, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        sig = {
            "rs_last_error": ([], ctypes.c_char_p),
            "rs_version": ([], ctypes.c_int),
            "rs_launch_count": ([], i64),
            "rs_launch_count_reset": ([], None),
            "rs_ctx_create": ([ctypes.c_int, P(vp)], ctypes.c_int),
            "rs_ctx_destroy": ([vp], ctypes.c_int),
            "rs_ctx_sync": ([vp], ctypes.c_int),
            "rs_ctx_set_stream": ([vp, vp], ctypes.c_int),
            "rs_tabular_create": ([vp, i32, i32, dbl, P(dbl), i32, P(vp)], ctypes.c_int),
            "rs_tabular_logits": ([vp, P(dbl), i64], ctypes.c_int),
            "rs_transformer_create": ([vp, P(_TransformerShape), u64, P(vp)], ctypes.c_int),
            "rs_drafter_create": ([vp, vp, u64, i32, P(vp)], ctypes.c_int),
            "rs_model_version": ([vp, P(i32)], ctypes.c_int),
            "rs_model_vocab": ([vp, P(i32)], ctypes.c_int),
            "rs_model_destroy": ([vp], ctypes.c_int),
            "rs_table_create": ([P(i32), i32, P(vp)], ctypes.c_int),
            "rs_table_set_entry": ([vp, i32, _SDConfig, dbl], ctypes.c_int),
            "rs_table_finalize": ([vp], ctypes.c_int),
            "rs_table_bucket_for": ([vp, i32, P(i32)], ctypes.c_int),
            "rs_table_solve": ([vp, i32, P(_SDConfig)], ctypes.c_int),
            "rs_table_best_for_bucket": ([vp, i32, P(_SDConfig)], ctypes.c_int),
            "rs_table_entry": ([vp, i32, _SDConfig, P(dbl)], ctypes.c_int),
            "rs_table_to_csv": ([vp, ctypes.c_char_p, i64, P(i64)], ctypes.c_int),
            "rs_table_destroy": ([vp], ctypes.c_int),
            "rs_engine_create": ([vp, vp, vp, vp, P(_TimingModel), P(_Request), i32, _SDConfig, i32, i32, P(vp)],
                                 ctypes.c_int),
            "rs_engine_set_drafter": ([vp, vp], ctypes.c_int),
            "rs_engine_step": ([vp, P(_StepInfo)], ctypes.c_int),
            "rs_engine_all_done": ([vp, P(i32)], ctypes.c_int),
            "rs_engine_active_batch": ([vp, P(i32)], ctypes.c_int),
            "rs_engine_cycles": ([vp, P(i32)], ctypes.c_int),
            "rs_engine_prefill_events": ([vp, P(i32)], ctypes.c_int),
            "rs_engine_ledger_time": ([vp, P(dbl)], ctypes.c_int),
            "rs_engine_ledger": ([vp, P(_ForwardEvent), i32, P(i32)], ctypes.c_int),
            "rs_engine_switches": ([vp, P(_SwitchEvent), i32, P(i32)], ctypes.c_int),
            "rs_engine_active_trace": ([vp, P(i32), i32, P(i32)], ctypes.c_int),
            "rs_engine_drafter_versions": ([vp, P(i32), i32, P(i32)], ctypes.c_int),
            "rs_engine_response": ([vp, i32, P(i32), i32, P(i32)], ctypes.c_int),
            "rs_engine_steps": ([vp, i32, P(dbl), P(ctypes.c_uint8), P(dbl), i32, P(i32)], ctypes.c_int),
            "rs_engine_step_logprobs": ([vp, i32, P(dbl), i64, P(i32)], ctypes.c_int),
            "rs_engine_accept_lens": ([vp, i32, P(i32), i32, P(i32)], ctypes.c_int),
            "rs_engine_destroy": ([vp], ctypes.c_int),
            "rs_engine_set_capture": ([vp, i32], ctypes.c_int),
            "rs_engine_capture_count": ([vp, P(i64), P(i32), P(i32)], ctypes.c_int),
            "rs_engine_capture_read": ([vp, i64, i64, P(i32), P(i32), P(i32), P(i32), P(dbl)], ctypes.c_int),
            "rs_engine_capture_read_f32": ([vp, i64, i64, ctypes.c_void_p], ctypes.c_int),
            "rs_kd_weight": ([dbl, P(dbl), i32, _KDPolicy, P(ctypes.c_int)], dbl),
            "rs_kd_update_tabular": ([vp, vp, P(_KDSample), i32, _KDPolicy, P(u64), dbl, P(vp), P(_KDResult)],
                                     ctypes.c_int),
            "rs_mt19937_64_seed": ([u64, P(u64)], ctypes.c_int),
            "rs_gemm_bf16": ([vp, vp, vp, vp, vp, i32, i32, i32, i32, ctypes.c_float, i32, i32], ctypes.c_int),
            "rs_model_tensor": ([vp, ctypes.c_char_p, i32, P(vp), P(i64)], ctypes.c_int),
            "rs_memcpy_d2d": ([vp, vp, vp, i64], ctypes.c_int),
            "rs_model_params": ([vp, P(i64)], ctypes.c_int),
            "rs_prof_enable": ([i32], None),
            "rs_prof_reset": ([], None),
            "rs_set_tuning": ([ctypes.c_char_p, i64], ctypes.c_int),
            "rs_lm_head_bf16": ([vp, vp, vp, vp, vp, i32, i32, i32, ctypes.c_float, dbl], ctypes.c_int),
            "rs_row_stats": ([vp, vp, i32, i32, dbl, vp], ctypes.c_int),
            "rs_kd_grad_transformer": ([vp, vp, vp, P(_KDSample), i32, P(dbl), vp, i32, P(dbl)], ctypes.c_int),
            "rs_drafter_apply_grad": ([vp, vp, vp, dbl, P(vp)], ctypes.c_int),
            "rs_engine_step_tokens": ([vp, P(i32), P(i32), P(i32), i32, P(i32)], ctypes.c_int),
            "rs_profile_measured": ([vp, vp, vp, P(i32), i32, P(_SDConfig), i32, i32, i32, i32, u64, P(dbl)],
                                    ctypes.c_int),
            "rs_kd_update_transformer": ([vp, vp, vp, P(_KDSample), i32, _KDPolicy, P(u64), dbl, P(vp),
                                          P(_KDResult)], ctypes.c_int),
            "rs_prof_json": ([ctypes.c_char_p, i64, P(i64)], ctypes.c_int),
            "rs_kd_select": ([i32, i32, P(u64), P(i32), P(i32)], ctypes.c_int),
            "rs_kd_grad_tabular": ([vp, vp, P(_KDSample), i32, P(dbl), P(dbl), P(dbl)], ctypes.c_int),
            "rs_tabular_apply_delta": ([vp, vp, P(dbl), dbl, P(vp)], ctypes.c_int),
            "rs_model_retain": ([vp], ctypes.c_int),
            "rs_learner_create": ([vp, vp, _KDPolicy, u64, dbl, i64, i32, P(vp)], ctypes.c_int),
            "rs_learner_destroy": ([vp], ctypes.c_int),
            "rs_learner_feed": ([vp, P(_KDSample), i32], ctypes.c_int),
            "rs_learner_on_iteration_boundary": ([vp, i32], ctypes.c_int),
            "rs_learner_await_pending": ([vp], ctypes.c_int),
            "rs_learner_shutdown": ([vp], ctypes.c_int),
            "rs_learner_snapshot": ([vp, P(vp)], ctypes.c_int),
            "rs_learner_drafter_version": ([vp, P(i32)], ctypes.c_int),
            "rs_learner_total_sim_time": ([vp, P(dbl)], ctypes.c_int),
            "rs_learner_buffer_size": ([vp, P(i64)], ctypes.c_int),
            "rs_learner_metrics": ([vp, P(_LearnerMetric), i32, P(i32)], ctypes.c_int),
            "rs_reward": ([P(i32), i32, i32, i32, P(dbl)], ctypes.c_int),
            "rs_group_advantages": ([P(dbl), i32, P(dbl)], ctypes.c_int),
            "rs_policy_update_tabular": ([vp, vp, P(_KDSample), P(dbl), P(i32), i32, dbl, P(vp)], ctypes.c_int),
            "rs_engine_set_stop_at_eos": ([vp, i32], ctypes.c_int),
            "rs_profile_simulated": ([vp, vp, vp, P(_SDConfig), i32, P(i32), P(i32), i32, P(_TimingModel), P(i32),
                                      i32, i32, i32, u64, P(dbl)], ctypes.c_int),
            "rs_tabular_random": ([vp, i32, i32, dbl, dbl, u64, P(vp)], ctypes.c_int),
            "rs_skew_eos_biases": ([u64, i32, P(dbl)], ctypes.c_int),
            "rs_engine_kd_grad": ([vp, vp, P(i32), i32, P(dbl), vp, i32, P(dbl)], ctypes.c_int),
            "rs_engine_rng_export": ([vp, i32, P(u64), i64, P(i64)], ctypes.c_int),
            "rs_engine_rng_import": ([vp, i32, P(u64), i64], ctypes.c_int),
            "rs_learner_feed_engine": ([vp, vp, P(i32), P(dbl), i32], ctypes.c_int),
            "rs_drafter_grad_layout": ([vp, ctypes.c_char_p, P(i64), P(i64)], ctypes.c_int),
            "rs_nccl_version": ([P(i32)], ctypes.c_int),
            "rs_comm_unique_id": ([P(ctypes.c_uint8)], ctypes.c_int),
            "rs_comm_create": ([vp, i32, i32, P(ctypes.c_uint8), P(vp)], ctypes.c_int),
            "rs_comm_destroy": ([vp], ctypes.c_int),
            "rs_comm_size": ([vp, P(i32), P(i32)], ctypes.c_int),
            "rs_comm_allreduce": ([vp, vp, vp, i64, i32, i32], ctypes.c_int),
            "rs_comm_allreduce_host": ([vp, vp, P(dbl), i32, i32], ctypes.c_int),
            "rs_device_alloc": ([vp, i64, P(vp)], ctypes.c_int),
            "rs_device_free": ([vp, vp], ctypes.c_int),
            "rs_memset_async": ([vp, vp, i32, i64], ctypes.c_int),
            "rs_memcpy_h2d": ([vp, vp, vp, i64], ctypes.c_int),
            "rs_memcpy_d2h": ([vp, vp, vp, i64], ctypes.c_int),
            "rs_model_tensor_shape": ([vp, ctypes.c_char_p, i32, P(i64), P(i64)], ctypes.c_int),
            "rs_model_load_tensor": ([vp, vp, ctypes.c_char_p, i32, vp, i32, i64], ctypes.c_int),
            "rs_model_store_tensor": ([vp, vp, ctypes.c_char_p, i32, vp, i32, i64], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(status):
    if status == RS_OK:
        return
    msg = lib().rs_last_error().decode()
    raise {RS_EINVAL: InvalidArgument, RS_ESTATE: EngineError, RS_ELOGIC: LogicError,
           RS_ECUDA: CudaError, RS_ENOMEM: MemoryError}.get(status, RuntimeError)(msg)


def _i32arr(xs):
    xs = list(xs)
    return (ctypes.c_int32 * max(1, len(xs)))(*xs)


def _f64arr(xs):
    xs = list(xs)
    return (ctypes.c_double * max(1, len(xs)))(*xs)


# ---- device context ---------------------------------------------------------------------------
class Device:
    """One GPU + stream (rs_ctx). One per host thread."""

    def __init__(self, index: int = 0):
        h = ctypes.c_void_p()
        _check(lib().rs_ctx_create(index, ctypes.byref(h)))
        self.handle = h
        self.index = index

    def sync(self):
        _check(lib().rs_ctx_sync(self.handle))

    def set_stream(self, cuda_stream_ptr: int):
        _check(lib().rs_ctx_set_stream(self.handle, ctypes.c_void_p(cuda_stream_ptr)))

    def close(self):
        if self.handle:
            lib().rs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_device: Optional[Device] = None


def default_device() -> Device:
    global _default_device
    if _default_device is None:
        _default_device = Device(0)
    return _default_device


class DeviceBuffer:
    """Library-owned device memory (rs_device_alloc): the drafter gradient of the KD update and
    its all-reduce need no tensor framework. fp32 elements unless stated."""

    def __init__(self, nbytes: int, device: Optional["Device"] = None, zero: bool = True):
        self.device = device or default_device()
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        _check(lib().rs_device_alloc(self.device.handle, self.nbytes, ctypes.byref(p)))
        self.ptr = p.value or 0
        if zero:
            self.zero()

    @staticmethod
    def floats(n: int, device: Optional["Device"] = None) -> "DeviceBuffer":
        return DeviceBuffer(4 * int(n), device)

    def data_ptr(self) -> int:
        return self.ptr

    @property
    def numel(self) -> int:
        return self.nbytes // 4

    def zero(self) -> "DeviceBuffer":
        _check(lib().rs_memset_async(self.device.handle, ctypes.c_void_p(self.ptr), 0, self.nbytes))
        return self

    def clone(self) -> "DeviceBuffer":
        out = DeviceBuffer(self.nbytes, self.device, zero=False)
        _check(lib().rs_memcpy_d2d(self.device.handle, ctypes.c_void_p(out.ptr), ctypes.c_void_p(self.ptr),
                                   self.nbytes))
        return out

    def to_numpy(self, offset: int = 0, count: Optional[int] = None):
        """fp32 elements [offset, offset + count) copied to the host."""
        import numpy as np
        count = self.numel - offset if count is None else count
        out = np.empty(count, dtype=np.float32)
        _check(lib().rs_memcpy_d2h(self.device.handle, ctypes.c_void_p(out.ctypes.data),
                                   ctypes.c_void_p(self.ptr + 4 * offset), 4 * count))
        return out

    def to_torch(self, offset: int = 0, count: Optional[int] = None):
        """A torch CUDA copy (tests only)."""
        import torch
        count = self.numel - offset if count is None else count
        t = torch.empty(count, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        _check(lib().rs_memcpy_d2d(self.device.handle, ctypes.c_void_p(t.data_ptr()),
                                   ctypes.c_void_p(self.ptr + 4 * offset), 4 * count))
        return t

    def __del__(self):
        try:
            if self.ptr:
                lib().rs_device_free(self.device.handle, ctypes.c_void_p(self.ptr))
                self.ptr = 0
        except Exception:
            pass


def device_profile(enable: Optional[bool] = None, reset: bool = False):
    """Per-kernel-class device timings (see rs_prof_json); returns the current totals."""
    import json
    if reset:
        lib().rs_prof_reset()
    if enable is not None:
        lib().rs_prof_enable(1 if enable else 0)
    n = ctypes.c_int64()
    _check(lib().rs_prof_json(None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(lib().rs_prof_json(buf, n.value + 1, ctypes.byref(n)))
    return json.loads(buf.value.decode())


def set_tuning(key: str, value: int) -> None:
    """Process-wide kernel knobs (rs_set_tuning); 0 restores the automatic choice."""
    _check(lib().rs_set_tuning(key.encode(), int(value)))


def launch_count() -> int:
    return int(lib().rs_launch_count())


def reset_launch_count():
    lib().rs_launch_count_reset()


# ---- SDConfig (specdec.hpp:17-37) ---------------------------------------------------------------
@dataclass(frozen=True)
class SDConfig:
    rounds: int = 1
    branching: int = 1
    draft_len: int = 1
    enabled: bool = False

    @staticmethod
    def off() -> "SDConfig":
        return SDConfig()

    @staticmethod
    def chain(k: int) -> "SDConfig":
        return SDConfig(1, 1, k, True)

    @staticmethod
    def tree(s: int, t: int, n: int) -> "SDConfig":
        return SDConfig(s, t, n, True)

    def drafted_per_cycle(self) -> int:
        return self.rounds * self.branching * self.draft_len

    def key(self) -> str:
        return "off" if not self.enabled else f"s{self.rounds}_t{self.branching}_n{self.draft_len}"

    def __eq__(self, o):
        if not isinstance(o, SDConfig):
            return NotImplemented
        if not self.enabled and not o.enabled:
            return True
        return (self.enabled == o.enabled and self.rounds == o.rounds and self.branching == o.branching
                and self.draft_len == o.draft_len)

    def __hash__(self):
        return hash(self.key())

    def _c(self) -> _SDConfig:
        return _SDConfig(self.rounds, self.branching, self.draft_len, 1 if self.enabled else 0)

    @staticmethod
    def _from_c(c: _SDConfig) -> "SDConfig":
        return SDConfig(c.rounds, c.branching, c.draft_len, bool(c.enabled))


# ---- TimingModel (costsim.hpp:34-53) ---------------------------------------------------------------
@dataclass
class RoleTiming:
    unit_cost: float = 1.0
    saturation_tokens: int = 32
    latency_floor: float = 0.0


@dataclass
class TimingModel:
    target: RoleTiming = field(default_factory=lambda: RoleTiming(1.0, 32, 2.0))
    drafter: RoleTiming = field(default_factory=lambda: RoleTiming(0.1, 32, 0.4))

    def _c(self):
        return _TimingModel(_RoleTiming(self.target.unit_cost, self.target.saturation_tokens, self.target.latency_floor),
                            _RoleTiming(self.drafter.unit_cost, self.drafter.saturation_tokens,
                                        self.drafter.latency_floor))


# ---- models ------------------------------------------------------------------------------------------
class Model:
    handle = None

    @property
    def version(self) -> int:
        v = ctypes.c_int32()
        _check(lib().rs_model_version(self.handle, ctypes.byref(v)))
        return v.value

    @property
    def vocab_size(self) -> int:
        v = ctypes.c_int32()
        _check(lib().rs_model_vocab(self.handle, ctypes.byref(v)))
        return v.value

    def eos(self) -> int:  # Vocabulary::eos, model.hpp:20
        return self.vocab_size - 1

    def __del__(self):
        try:
            if self.handle:
                lib().rs_model_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class TabularARModel(Model):
    """TabularARModel (model.hpp:105-147) held in HBM in fp64 (parity mode)."""

    def __init__(self, vocab: int, order: int, logits: Sequence[float], temperature: float = 1.0, version: int = 0,
                 device: Optional[Device] = None):
        self.device = device or default_device()
        rows = vocab ** order if order >= 0 and vocab >= 2 else 0
        logits = list(logits)
        if vocab >= 2 and order >= 0 and temperature > 0 and len(logits) != rows * vocab:
            raise InvalidArgument("TabularARModel: logits table has wrong shape")
        self.order = order
        self.temperature = temperature
        h = ctypes.c_void_p()
        _check(lib().rs_tabular_create(self.device.handle, vocab, order, temperature, _f64arr(logits), version,
                                       ctypes.byref(h)))
        self.handle = h

    @staticmethod
    def random(vocab: int, order: int, temperature: float, scale: float, seed: int,
               device: Optional[Device] = None) -> "TabularARModel":
        """TabularARModel::random (model.cpp:102-111) with rng = std::mt19937_64(seed)."""
        device = device or default_device()
        h = ctypes.c_void_p()
        _check(lib().rs_tabular_random(device.handle, vocab, order, temperature, scale, seed & (2 ** 64 - 1),
                                       ctypes.byref(h)))
        return TabularARModel._wrap(h, order, temperature, device)

    @staticmethod
    def zeros(vocab: int, order: int, temperature: float = 1.0, device: Optional[Device] = None) -> "TabularARModel":
        """TabularARModel::zeros (model.cpp:97-100)."""
        return TabularARModel(vocab, order, [0.0] * (vocab ** order * vocab), temperature, 0, device)

    @staticmethod
    def from_json(j: dict, device: Optional[Device] = None) -> "TabularARModel":  # model.cpp:183-191
        return TabularARModel(j["vocab_size"] if "vocab_size" in j else j["vocab"], j["order"], j["logits"],
                              j.get("temperature", 1.0), j.get("version", 0), device)

    @staticmethod
    def _wrap(handle, order, temperature, device):
        m = TabularARModel.__new__(TabularARModel)
        m.handle, m.order, m.temperature, m.device = handle, order, temperature, device
        return m

    def logits(self) -> List[float]:
        n = self.vocab_size ** (self.order + 1)
        buf = (ctypes.c_double * n)()
        _check(lib().rs_tabular_logits(self.handle, buf, n))
        return list(buf)

    def to_json(self) -> dict:
        return {"vocab_size": self.vocab_size, "order": self.order, "temperature": self.temperature,
                "logits": self.logits()}


@dataclass
class TransformerShape:
    """Qwen2-style decoder shape. Presets follow the public Qwen2.5 config.json values."""
    vocab: int
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int = 128
    d_ff: int = 0
    max_ctx: int = 4096
    rope_theta: float = 1e6
    rms_eps: float = 1e-6
    init_std: float = 0.02
    logit_scale: float = 1.0
    temperature: float = 1.0

    @staticmethod
    def tiny(vocab=1024, max_ctx=512, **kw):
        """BASELINE cfg1: 2-layer d=256 target (CPU-runnable size)."""
        return TransformerShape(vocab, 256, 2, 4, 2, 128, 512, max_ctx, **kw)

    @staticmethod
    def qwen2_5_3b(max_ctx=4096, **kw):
        return TransformerShape(151936, 2048, 36, 16, 2, 128, 11008, max_ctx, **kw)

    @staticmethod
    def qwen2_5_7b(max_ctx=4096, **kw):
        return TransformerShape(152064, 3584, 28, 28, 4, 128, 18944, max_ctx, **kw)

    @staticmethod
    def qwen2_5_14b(max_ctx=4096, **kw):
        return TransformerShape(152064, 5120, 48, 40, 8, 128, 13824, max_ctx, **kw)

    def _c(self):
        return _TransformerShape(self.vocab, self.d_model, self.n_layers, self.n_heads, self.n_kv_heads, self.head_dim,
                                 self.d_ff, self.max_ctx, self.rope_theta, self.rms_eps, self.init_std,
                                 self.logit_scale, self.temperature)

    def macs_per_token(self) -> int:
        """Dense MACs per token (QKV+O+MLP over all layers + LM head), SURVEY.md §8."""
        q = (self.n_heads + 2 * self.n_kv_heads) * self.head_dim
        per_layer = self.d_model * q + self.n_heads * self.head_dim * self.d_model + 3 * self.d_model * self.d_ff
        return self.n_layers * per_layer + self.d_model * self.vocab

    def kv_bytes_per_token(self) -> int:
        return self.n_layers * 2 * self.n_kv_heads * self.head_dim * 2


class _NeuralModel(Model):
    def tensor(self, name: str, layer: int = -1):
        """(device pointer, bytes) of a named weight tensor."""
        p, b = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().rs_model_tensor(self.handle, name.encode(), layer, ctypes.byref(p), ctypes.byref(b)))
        return p.value, b.value

    def to_torch(self, name: str, layer: int = -1, dtype=None, shape=None):
        """Copy a weight tensor into a new torch CUDA tensor (tests / export only)."""
        import torch
        ptr, nbytes = self.tensor(name, layer)
        dtype = dtype or (torch.float32 if name in ("ln1", "ln2", "final_norm", "norm_emb", "norm_hid", "rope")
                          else torch.bfloat16)
        t = torch.empty(nbytes // torch.tensor([], dtype=dtype).element_size(), dtype=dtype, device="cuda")
        torch.cuda.synchronize()
        _check(lib().rs_memcpy_d2d(self.device.handle, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(ptr), nbytes))
        return t.view(*shape) if shape else t

    @property
    def n_params(self) -> int:
        v = ctypes.c_int64()
        _check(lib().rs_model_params(self.handle, ctypes.byref(v)))
        return v.value

    # ---- checkpoints (Hugging Face names; the transformer counterpart of to_json / from_json,
    # model.cpp:176-191). Host arrays are numpy float32 (converted to bf16 with round-to-nearest-
    # even for bf16 weights), numpy uint16 (bf16 bit patterns) or torch tensors.
    # subclasses name their tensors: checkpoint_names() and _split(full) -> (name, layer)
    def tensor_shape(self, name: str, layer: int = -1):
        r, c = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().rs_model_tensor_shape(self.handle, name.encode(), layer, ctypes.byref(r), ctypes.byref(c)))
        return (r.value, c.value) if r.value > 1 else (c.value,)

    def load_tensor(self, name: str, layer: int, array) -> None:
        import numpy as np
        if hasattr(array, "detach"):  # torch tensor
            import torch
            t = array.detach().contiguous().cpu()
            array = t.view(torch.int16).numpy().view(np.uint16) if t.dtype == torch.bfloat16 else t.float().numpy()
        a = np.ascontiguousarray(array)
        if a.dtype == np.uint16:
            dt = RS_DTYPE_BF16
        else:
            a = np.ascontiguousarray(a, dtype=np.float32)
            dt = RS_DTYPE_F32
        _check(lib().rs_model_load_tensor(self.device.handle, self.handle, name.encode(), layer,
                                          a.ctypes.data_as(ctypes.c_void_p), dt, a.size))

    def store_tensor(self, name: str, layer: int = -1, bf16_bits: bool = False):
        """The tensor as numpy float32 (exact for bf16 weights) or, bf16_bits, uint16 bit patterns."""
        import numpy as np
        shape = self.tensor_shape(name, layer)
        a = np.empty(shape, dtype=np.uint16 if bf16_bits else np.float32)
        _check(lib().rs_model_store_tensor(self.device.handle, self.handle, name.encode(), layer,
                                           a.ctypes.data_as(ctypes.c_void_p),
                                           RS_DTYPE_BF16 if bf16_bits else RS_DTYPE_F32, a.size))
        return a

    def state_dict(self, bf16_bits: bool = False) -> dict:
        return {full: self.store_tensor(*self._split(full), bf16_bits=bf16_bits) for full in self.checkpoint_names()}

    def load_state_dict(self, sd: dict, strict: bool = True) -> None:
        names = set(self.checkpoint_names())
        if strict:
            missing, extra = names - set(sd), set(sd) - names - set(self._optional)
            if missing or extra:
                raise InvalidArgument(f"load_state_dict: missing {sorted(missing)[:4]}, unexpected {sorted(extra)[:4]}")
        for full, arr in sd.items():
            if full in names:
                self.load_tensor(*self._split(full), arr)

    def save(self, path: str) -> None:
        """numpy .npz of the checkpoint: bf16 weights as uint16 bit patterns, norm gains fp32."""
        import numpy as np
        out = {}
        for full in self.checkpoint_names():
            name, layer = self._split(full)
            out[full] = self.store_tensor(name, layer, bf16_bits=not name.endswith("norm.weight"))
        np.savez(path, **out)

    def load(self, path: str) -> None:
        import numpy as np
        with np.load(path) as z:
            self.load_state_dict({k: z[k] for k in z.files})

    _optional = ()

    _LAYER_TENSORS = ("self_attn.q_proj.weight", "self_attn.k_proj.weight", "self_attn.v_proj.weight",
                      "self_attn.q_proj.bias", "self_attn.k_proj.bias", "self_attn.v_proj.bias",
                      "self_attn.o_proj.weight", "mlp.gate_proj.weight", "mlp.up_proj.weight",
                      "mlp.down_proj.weight", "post_attention_layernorm.weight")


class TransformerModel(_NeuralModel):
    """Qwen2-shaped target with synthetic N(0, init_std) bf16 weights generated on the device."""

    def __init__(self, shape: TransformerShape, seed: int = 0, device: Optional[Device] = None):
        self.device = device or default_device()
        self.shape = shape
        h = ctypes.c_void_p()
        sc = shape._c()
        _check(lib().rs_transformer_create(self.device.handle, ctypes.byref(sc), seed & (2 ** 64 - 1),
                                           ctypes.byref(h)))
        self.handle = h

    # Qwen2 checkpoint names (model.safetensors of Qwen2.5-*); the LM head is tied to the embedding
    _optional = ("lm_head.weight",)

    def checkpoint_names(self) -> List[str]:
        names = ["model.embed_tokens.weight", "model.norm.weight"]
        for i in range(self.shape.n_layers):
            names.append(f"model.layers.{i}.input_layernorm.weight")
            names += [f"model.layers.{i}.{t}" for t in self._LAYER_TENSORS]
        return names

    def _split(self, full: str):
        parts = full.split(".")
        if parts[0] == "model" and parts[1] == "layers":
            return ".".join(parts[-2:]), int(parts[2])
        return ".".join(parts[-2:]), -1

    @staticmethod
    def from_pretrained(shape: TransformerShape, state_dict: dict, device: Optional[Device] = None):
        """A target with the given checkpoint tensors (HF Qwen2 names)."""
        m = TransformerModel(shape, seed=0, device=device)
        m.load_state_dict(state_dict)
        return m


class EagleDrafter(_NeuralModel):
    """EAGLE-3-style drafter bound to `target` (consumes its low/mid/high hidden states)."""

    def __init__(self, target: TransformerModel, seed: int = 1, version: int = 0):
        self.device = target.device
        self.target = target
        self.shape = target.shape
        h = ctypes.c_void_p()
        _check(lib().rs_drafter_create(self.device.handle, target.handle, seed & (2 ** 64 - 1), version,
                                       ctypes.byref(h)))
        self.handle = h

    # EAGLE-3 checkpoint names (one decoder layer "midlayer" over [norm(emb), hidden_norm(f)])
    def checkpoint_names(self) -> List[str]:
        return (["fc.weight", "midlayer.input_layernorm.weight", "midlayer.hidden_norm.weight", "norm.weight",
                 "lm_head.weight"] + [f"midlayer.{t}" for t in self._LAYER_TENSORS])

    def _split(self, full: str):
        return ".".join(full.split(".")[-2:]), 0

    @staticmethod
    def _wrap(handle, target: TransformerModel) -> "EagleDrafter":
        m = EagleDrafter.__new__(EagleDrafter)
        m.handle, m.target, m.shape, m.device = handle, target, target.shape, target.device
        return m

    GRAD_TENSORS = ("lm_w", "fc_w", "norm_emb", "norm_hid", "qkv_w", "qkv_b", "o_w", "ln2", "gu_w", "down_w",
                    "final_norm")

    def grad_layout(self, name: Optional[str] = None):
        """(offset, count) of one tensor in the fp32 drafter gradient (name None: (0, total))."""
        o, n = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().rs_drafter_grad_layout(self.handle, name.encode() if name else None, ctypes.byref(o),
                                            ctypes.byref(n)))
        return o.value, n.value

    def new_grad(self) -> DeviceBuffer:
        """A zeroed fp32 gradient buffer covering every drafter tensor."""
        return DeviceBuffer.floats(self.grad_layout()[1], self.device)

    def apply_grad(self, grad, scale: float) -> "EagleDrafter":
        """New snapshot (version + 1): every tensor w + scale * grad (the fp32 layout of
        grad_layout; a DeviceBuffer, a tensor with data_ptr, or a raw pointer)."""
        h = ctypes.c_void_p()
        ptr = grad.data_ptr() if hasattr(grad, "data_ptr") else grad
        _check(lib().rs_drafter_apply_grad(self.device.handle, self.handle, ctypes.c_void_p(ptr), scale,
                                           ctypes.byref(h)))
        return EagleDrafter._wrap(h, self.target)


def profile_measured(target, drafter, buckets: Sequence[int], configs: Sequence["SDConfig"], prompt_len: int = 128,
                     warmup: int = 2, cycles: int = 8, seed: int = 1) -> "ProfileTable":
    """profile() (server.cpp:182-239) from MEASURED device latency per emitted token: one wave
    of exactly `bucket` requests per (bucket, config), `cycles` timed engine steps after
    `warmup`. The non-spec entry is always measured (finalize requires it)."""
    cfgs = [SDConfig.off()] + [c for c in configs if c.enabled]
    arr = (_SDConfig * len(cfgs))(*[c._c() for c in cfgs])
    out = (ctypes.c_double * (len(buckets) * len(cfgs)))()
    dev = target.device
    _check(lib().rs_profile_measured(dev.handle, target.handle, drafter.handle if drafter else None,
                                     _i32arr(buckets), len(buckets), arr, len(cfgs), prompt_len, warmup, cycles,
                                     seed & (2 ** 64 - 1), out))
    table = ProfileTable(buckets)
    for ib, b in enumerate(buckets):
        for ic, c in enumerate(cfgs):
            table.set_entry(b, c, out[ib * len(cfgs) + ic])
    table.finalize()
    return table


# ---- ProfileTable (server.hpp:21-49) ------------------------------------------------------------------
@dataclass
class ProfileOptions:
    """ProfileOptions (server.hpp:51-56)."""
    batch_sizes: List[int] = field(default_factory=lambda: [1, 2, 4, 8, 16, 32, 64])
    cycles_per_request: int = 64
    num_requests: int = 64
    seed: int = 1


def profile(target: Model, drafter: Optional[Model], config_grid: Sequence["SDConfig"],
            eval_prompts: Sequence[Sequence[int]], tm: "TimingModel", opts: ProfileOptions = None) -> "ProfileTable":
    """profile() (server.cpp:182-239): the offline Solver under the SIMULATED timing model, run on
    the GPU engine (fixed-width waves, stop_at_eos = false, one ledger per bucket x config).
    For measured B200 latency use profile_measured()."""
    opts = opts or ProfileOptions()
    if not eval_prompts:
        raise InvalidArgument("profile: no eval prompts")
    grid = [c for c in config_grid]
    garr = (_SDConfig * max(1, len(grid)))(*[c._c() for c in grid])
    flat = [t for p in eval_prompts for t in p]
    off = [0]
    for p in eval_prompts:
        off.append(off[-1] + len(p))
    nc = len(grid) + 1
    out = (ctypes.c_double * max(1, len(opts.batch_sizes) * nc))()
    tmc = tm._c()
    _check(lib().rs_profile_simulated(target.device.handle, target.handle, drafter.handle if drafter else None, garr,
                                      len(grid), _i32arr(flat), _i32arr(off), len(eval_prompts), ctypes.byref(tmc),
                                      _i32arr(opts.batch_sizes), len(opts.batch_sizes), opts.cycles_per_request,
                                      opts.num_requests, opts.seed & (2 ** 64 - 1), out))
    table = ProfileTable(opts.batch_sizes)
    cfgs = [SDConfig.off()] + grid
    for ib, b in enumerate(opts.batch_sizes):
        for ic, c in enumerate(cfgs):
            table.set_entry(b, c, out[ib * nc + ic])
    table.finalize()
    return table



class ProfileTable:
    def __init__(self, buckets: Sequence[int]):
        h = ctypes.c_void_p()
        _check(lib().rs_table_create(_i32arr(buckets), len(buckets), ctypes.byref(h)))
        self.handle = h
        self._buckets = sorted(buckets)
        self._entries = {}

    def set_entry(self, bucket: int, cfg: SDConfig, time_per_token: float):
        _check(lib().rs_table_set_entry(self.handle, bucket, cfg._c(), time_per_token))
        self._entries.setdefault(bucket, []).append((cfg, time_per_token))

    def finalize(self):
        _check(lib().rs_table_finalize(self.handle))

    def bucket_for(self, active_batch: int) -> int:
        v = ctypes.c_int32()
        _check(lib().rs_table_bucket_for(self.handle, active_batch, ctypes.byref(v)))
        return v.value

    def solve(self, active_batch: int) -> SDConfig:
        c = _SDConfig()
        _check(lib().rs_table_solve(self.handle, active_batch, ctypes.byref(c)))
        return SDConfig._from_c(c)

    def best_for_bucket(self, bucket: int) -> SDConfig:
        c = _SDConfig()
        _check(lib().rs_table_best_for_bucket(self.handle, bucket, ctypes.byref(c)))
        return SDConfig._from_c(c)

    def entry(self, bucket: int, cfg: SDConfig) -> float:
        v = ctypes.c_double()
        _check(lib().rs_table_entry(self.handle, bucket, cfg._c(), ctypes.byref(v)))
        return v.value

    def baseline(self, bucket: int) -> float:
        return self.entry(bucket, SDConfig.off())

    def buckets(self) -> List[int]:
        return list(self._buckets)

    def entries_for(self, bucket: int):
        if bucket not in self._entries:
            raise InvalidArgument("ProfileTable: unknown bucket")
        return list(self._entries[bucket])

    def to_csv(self) -> str:
        n = ctypes.c_int64()
        _check(lib().rs_table_to_csv(self.handle, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(lib().rs_table_to_csv(self.handle, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def to_json(self) -> dict:  # server.cpp:98-118 schema
        entries = [{"bucket": b, "s": c.rounds, "t": c.branching, "n": c.draft_len, "enabled": c.enabled,
                    "time_per_token": t} for b in self._buckets for (c, t) in self._entries.get(b, [])]
        best = [{"bucket": b, "s": c.rounds, "t": c.branching, "n": c.draft_len, "enabled": c.enabled}
                for b in self._buckets for c in [self.best_for_bucket(b)]]
        return {"buckets": self._buckets, "entries": entries, "best": best}

    @staticmethod
    def from_json(j: dict) -> "ProfileTable":  # server.cpp:120-130
        t = ProfileTable(j["buckets"])
        for e in j["entries"]:
            t.set_entry(e["bucket"], SDConfig(e["s"], e["t"], e["n"], e["enabled"]), e["time_per_token"])
        t.finalize()
        return t

    def __del__(self):
        try:
            if self.handle:
                lib().rs_table_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


# ---- requests / records ------------------------------------------------------------------------------------
@dataclass
class DecodeRng:
    """DecodeRng::from_seed(seed, stream_id) (rng.hpp:37-43); the streams live on the device.
    `state` is the advanced stream image after spec_step_tree / generate consumed draws from it
    (None = freshly seeded); an engine created with this rng continues where it stopped."""
    seed: int = 0
    stream_id: int = 0
    state: Optional[object] = field(default=None, compare=False, repr=False)

    @staticmethod
    def from_seed(seed: int, stream_id: int = 0) -> "DecodeRng":
        return DecodeRng(seed, stream_id)


@dataclass
class StepRecord:
    token: int
    logp: float
    drafted: bool
    logq: float
    target_logprobs: Optional[List[float]] = None


@dataclass
class RequestState:
    """RequestState (server.hpp:69-83)."""
    id: int = 0
    prompt: List[int] = field(default_factory=list)
    eos_bias: float = 0.0
    max_len: int = 1
    rng: DecodeRng = field(default_factory=DecodeRng)
    generated: List[int] = field(default_factory=list)
    steps: List[StepRecord] = field(default_factory=list)
    accept_lens: List[int] = field(default_factory=list)
    done: bool = False

    def full_ctx(self) -> List[int]:
        return list(self.prompt) + list(self.generated)

    def remaining(self) -> int:
        return self.max_len - len(self.generated)


@dataclass
class RolloutSample:
    """RolloutSample (rollout.hpp:12-20)."""
    prompt: List[int]
    response: List[int]
    steps: List[StepRecord]
    eos_bias: float = 0.0
    reward: float = 0.0
    actor_version: int = 0
    drafter_version: int = 0


@dataclass
class SwitchEvent:
    cycle: int
    active_batch: int
    from_: SDConfig
    to: SDConfig


@dataclass
class GenerationRun:
    """GenerationRun (server.hpp:134-142)."""
    samples: List[RolloutSample]
    total_time: float
    accept_lens: List[int]
    switches: List[SwitchEvent]
    active_trace: List[int]
    ledger: List[tuple]
    cycles: int
    prefill_events: int = 0
    wall_ms: float = 0.0  # measured device time over all steps


DrafterSnapshotFn = Callable[[], Optional[Model]]


class BatchEngine:
    """BatchEngine (server.hpp:98-132) on the GPU: cycle-synchronous spec/non-spec state machine.

    table=None selects fixed mode with `forced`. `drafter` is a DrafterSnapshotFn read once per
    cycle, or None. verify_mode is "sample" (the reference's lossless rejection sampling) or
    "greedy" (not in the reference)."""

    def __init__(self, target: Model, drafter: Optional[DrafterSnapshotFn], table: Optional[ProfileTable],
                 tm: Optional[TimingModel], requests: Sequence[RequestState], forced: SDConfig = SDConfig.off(),
                 verify_mode: str = "sample", record_full_logprobs: bool = True, device: Optional[Device] = None):
        self.device = device or getattr(target, "device", None) or default_device()
        self._target = target
        self._drafter_fn = drafter
        self._table = table
        self._reqs = [r for r in requests]
        self._record_full = record_full_logprobs
        self._vmode = {"sample": RS_VERIFY_SAMPLE, "greedy": RS_VERIFY_GREEDY}[verify_mode]
        self._keep = []
        arr = (_Request * max(1, len(self._reqs)))()
        for i, r in enumerate(self._reqs):
            p = _i32arr(r.prompt)
            self._keep.append(p)
            arr[i] = _Request(r.id, ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), len(r.prompt), r.eos_bias,
                              r.max_len, r.rng.seed & (2 ** 64 - 1), r.rng.stream_id & (2 ** 64 - 1))
        snap = drafter() if drafter is not None else None
        self._snap = snap
        tmc = (tm or TimingModel())._c()
        h = ctypes.c_void_p()
        _check(lib().rs_engine_create(self.device.handle, target.handle, snap.handle if snap else None,
                                      table.handle if table else None, ctypes.byref(tmc), arr, len(self._reqs),
                                      forced._c(), self._vmode, 1 if record_full_logprobs else 0, ctypes.byref(h)))
        self.handle = h
        self.last_info = None
        for i, r in enumerate(self._reqs):  # continue advanced DecodeRng streams
            if r.rng.state is not None:
                _check(lib().rs_engine_rng_import(self.handle, i, r.rng.state, len(r.rng.state)))

    def set_stop_at_eos(self, stop: bool) -> None:
        """stop_at_eos = False (before the first step): EOS is an ordinary token (server.cpp:215)."""
        _check(lib().rs_engine_set_stop_at_eos(self.handle, 1 if stop else 0))

    def rng_state(self, req: int):
        """The request's advanced DecodeRng stream image (rs_engine_rng_export)."""
        n = ctypes.c_int64()
        _check(lib().rs_engine_rng_export(self.handle, req, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_uint64 * n.value)()
        _check(lib().rs_engine_rng_export(self.handle, req, buf, n.value, ctypes.byref(n)))
        return buf

    def step(self):
        """One engine cycle (server.cpp:266-349); raises EngineError on an empty batch."""
        snap = self._drafter_fn() if self._drafter_fn is not None else None
        self._snap = snap
        _check(lib().rs_engine_set_drafter(self.handle, snap.handle if snap else None))
        info = _StepInfo()
        _check(lib().rs_engine_step(self.handle, ctypes.byref(info)))
        self.last_info = info
        return info

    def _i(self, fn):
        v = ctypes.c_int32()
        _check(fn(self.handle, ctypes.byref(v)))
        return v.value

    def all_done(self) -> bool:
        return bool(self._i(lib().rs_engine_all_done))

    def active_batch(self) -> int:
        return self._i(lib().rs_engine_active_batch)

    def cycles(self) -> int:
        return self._i(lib().rs_engine_cycles)

    def prefill_events(self) -> int:
        return self._i(lib().rs_engine_prefill_events)

    def ledger_time(self) -> float:
        v = ctypes.c_double()
        _check(lib().rs_engine_ledger_time(self.handle, ctypes.byref(v)))
        return v.value

    def _arr(self, fn, ctype):
        n = ctypes.c_int32()
        _check(fn(self.handle, None, 0, ctypes.byref(n)))
        buf = (ctype * max(1, n.value))()
        _check(fn(self.handle, buf, n.value, ctypes.byref(n)))
        return list(buf)[: n.value]

    def ledger(self):
        return [(e.role, e.positions, e.batch_tokens) for e in self._arr(lib().rs_engine_ledger, _ForwardEvent)]

    def switches(self) -> List[SwitchEvent]:
        return [SwitchEvent(s.cycle, s.active_batch, SDConfig._from_c(s.from_), SDConfig._from_c(s.to))
                for s in self._arr(lib().rs_engine_switches, _SwitchEvent)]

    def active_trace(self) -> List[int]:
        return self._arr(lib().rs_engine_active_trace, ctypes.c_int32)

    def drafter_version_at_cycle(self, cycle: int) -> int:
        v = self._arr(lib().rs_engine_drafter_versions, ctypes.c_int32)
        if cycle < 0 or cycle >= len(v):
            raise IndexError("drafter_version_at_cycle: out of range")
        return v[cycle]

    def _response(self, i):
        n = ctypes.c_int32()
        _check(lib().rs_engine_response(self.handle, i, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_int32 * max(1, n.value))()
        _check(lib().rs_engine_response(self.handle, i, buf, n.value, ctypes.byref(n)))
        return list(buf)[: n.value]

    def _steps(self, i, V):
        n = len(self._response(i))
        lp = (ctypes.c_double * max(1, n))()
        lq = (ctypes.c_double * max(1, n))()
        dr = (ctypes.c_uint8 * max(1, n))()
        m = ctypes.c_int32()
        _check(lib().rs_engine_steps(self.handle, i, lp, dr, lq, n, ctypes.byref(m)))
        full = None
        if self._record_full and n:
            fb = (ctypes.c_double * (n * V))()
            _check(lib().rs_engine_step_logprobs(self.handle, i, fb, n * V, ctypes.byref(m)))
            full = [list(fb[k * V:(k + 1) * V]) for k in range(n)]
        toks = self._response(i)
        return [StepRecord(toks[k], lp[k], bool(dr[k]), lq[k], full[k] if full else None) for k in range(n)]

    def step_tokens(self) -> dict:
        """{request index: tokens emitted by the last step()} -- host data that arrived with the
        step summary (no extra device round trip)."""
        cap = 512
        n = len(self._reqs)
        req, cnt = (ctypes.c_int32 * n)(), (ctypes.c_int32 * n)()
        toks = (ctypes.c_int32 * (n * cap))()
        na = ctypes.c_int32()
        _check(lib().rs_engine_step_tokens(self.handle, req, cnt, toks, cap, ctypes.byref(na)))
        return {req[a]: list(toks[a * cap: a * cap + min(cnt[a], cap)]) for a in range(na.value)}

    def kd_grad(self, drafter: "EagleDrafter", req_ids: Sequence[int], weights: Sequence[float], grad=None,
                zero_grad: bool = True):
        """Per-rank K5 + whole-drafter gradient over these requests' generated tokens, from the
        engine's resident target KV cache and features (rs_engine_kd_grad): (loss, DeviceBuffer
        in the drafter's grad_layout). Same result as kd_grad_transformer on the same rollouts
        without the teacher-forced recompute of the prompts."""
        if grad is None:
            grad = drafter.new_grad()
        loss = ctypes.c_double()
        self.device.sync()
        _check(lib().rs_engine_kd_grad(self.handle, drafter.handle, _i32arr(req_ids), len(req_ids), _f64arr(weights),
                                       ctypes.c_void_p(grad.data_ptr()), 1 if zero_grad else 0, ctypes.byref(loss)))
        return loss.value, grad

    def requests(self) -> List[RequestState]:
        V = self._target.vocab_size
        out = []
        for i, r in enumerate(self._reqs):
            al = self._arr(lambda h, b, c, n, i=i: lib().rs_engine_accept_lens(h, i, b, c, n), ctypes.c_int32)
            gen = self._response(i)
            out.append(RequestState(r.id, list(r.prompt), r.eos_bias, r.max_len, r.rng, gen, self._steps(i, V), al,
                                    len(gen) >= r.max_len or (len(gen) > 0 and gen[-1] == V - 1)))
        return out

    # debug: logits capture for replay against the CPU oracle
    def set_capture(self, on: bool):
        _check(lib().rs_engine_set_capture(self.handle, 1 if on else 0))

    def captured_rows(self):
        """[(role, request, ctx_len, ext_tokens, logits)] for every row produced since capture was
        enabled; role 1 = target (p rows), 0 = drafter (q rows). The row's context is the
        request's first ctx_len tokens followed by ext_tokens."""
        n, V, W = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().rs_engine_capture_count(self.handle, ctypes.byref(n), ctypes.byref(V), ctypes.byref(W)))
        k, V, W = n.value, V.value, W.value
        if k == 0:
            return []
        role, req, cl = (ctypes.c_int32 * k)(), (ctypes.c_int32 * k)(), (ctypes.c_int32 * k)()
        ext = (ctypes.c_int32 * (k * W))()
        lg = (ctypes.c_double * (k * V))()
        _check(lib().rs_engine_capture_read(self.handle, 0, k, role, req, cl, ext, lg))
        out = []
        for i in range(k):
            e = [x for x in ext[i * W:(i + 1) * W] if x >= 0]
            out.append((role[i], req[i], cl[i], e, lg[i * V:(i + 1) * V]))
        return out

    def captured_meta(self):
        """Metadata of the captured rows without the logits: [(role, request, ctx_len, ext)]."""
        n, V, W = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().rs_engine_capture_count(self.handle, ctypes.byref(n), ctypes.byref(V), ctypes.byref(W)))
        k, W = n.value, W.value
        if k == 0:
            return []
        role, req, cl = (ctypes.c_int32 * k)(), (ctypes.c_int32 * k)(), (ctypes.c_int32 * k)()
        ext = (ctypes.c_int32 * (k * W))()
        _check(lib().rs_engine_capture_read(self.handle, 0, k, role, req, cl, ext, None))
        return [(role[i], req[i], cl[i], [x for x in ext[i * W:(i + 1) * W] if x >= 0]) for i in range(k)]

    def captured_logits_f32(self, first: int, count: int):
        """numpy float32 [count, V] of captured transformer rows first..first+count."""
        import numpy as np
        out = np.empty((count, self._target.vocab_size), dtype=np.float32)
        _check(lib().rs_engine_capture_read_f32(self.handle, first, count, ctypes.c_void_p(out.ctypes.data)))
        return out

    def __del__(self):
        try:
            if self.handle:
                lib().rs_engine_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def run_generation(requests: Sequence[RequestState], target: Model, drafter: Optional[DrafterSnapshotFn],
                   table: Optional[ProfileTable], tm: TimingModel, forced: SDConfig = SDConfig.off(),
                   actor_version: int = 0, verify_mode: str = "sample", record_full_logprobs: bool = True,
                   device: Optional[Device] = None) -> GenerationRun:
    """run_generation (server.cpp:351-376): step until every request completes."""
    eng = BatchEngine(target, drafter, table, tm, requests, forced, verify_mode, record_full_logprobs, device)
    wall = 0.0
    while not eng.all_done():
        wall += eng.step().step_ms
    reqs = eng.requests()
    samples = [RolloutSample(r.prompt, r.generated, r.steps, r.eos_bias, 0.0, actor_version) for r in reqs]
    al = [a for r in reqs for a in r.accept_lens]
    return GenerationRun(samples, eng.ledger_time(), al, eng.switches(), eng.active_trace(), eng.ledger(),
                         eng.cycles(), eng.prefill_events(), wall)


# ---- single-sequence API (specdec.hpp:58-131) -------------------------------------------------------------------
@dataclass
class RoundCost:
    """RoundCost (specdec.hpp:58-63)."""
    drafter_forwards: int = 0
    drafter_tokens_each: int = 0
    target_tokens: int = 0


@dataclass
class VerifyOutcome:
    """VerifyOutcome (specdec.hpp:65-75). draft_records holds the number of drafted positions
    (one DraftPosRecord each in the reference)."""
    accepted_tokens: List[int]
    accept_len: int
    bonus_token: int
    steps: List[StepRecord]
    rounds: List[RoundCost]
    ended: bool
    draft_records: int = 0


def _rounds_of(ledger) -> List[RoundCost]:
    """Per-round costs of a single-sequence cycle from its forward events (charge_batched_cycle
    over one outcome, server.cpp:154-178): `drafter_forwards` drafter passes of t tokens, then one
    target pass of t*n_eff + 1 tokens."""
    out, fw, each = [], 0, 0
    for role, _, tokens in ledger:
        if role == 0:
            fw += 1
            each = tokens
        else:
            out.append(RoundCost(fw, each, tokens))
            fw, each = 0, 0
    return out


def spec_step_tree(target: Model, drafter: Model, ctx: Sequence[int], cfg: SDConfig, rng: DecodeRng,
                   eos_bias: float = 0.0, stop_at_eos: bool = True, max_emit: int = 2 ** 31 - 1,
                   record_full_logprobs: bool = True) -> VerifyOutcome:
    """spec_step_tree (specdec.cpp:146-269): ONE verification cycle of one sequence on the GPU
    engine. `rng` is advanced in place (DecodeRng& in the reference), so consecutive calls
    continue the same draft / accept streams."""
    if not cfg.enabled:
        raise InvalidArgument("spec_step_tree: SD config must be enabled")
    cap = cfg.rounds * cfg.draft_len + 1  # the most one cycle can emit
    req = RequestState(0, list(ctx), eos_bias, max(1, min(max_emit, cap)), rng)
    eng = BatchEngine(target, lambda: drafter, None, TimingModel(), [req], cfg, "sample", record_full_logprobs,
                      getattr(target, "device", None))
    eng.set_stop_at_eos(stop_at_eos)
    eng.step()
    r = eng.requests()[0]
    rng.state = eng.rng_state(0)
    steps = r.steps
    eos = target.vocab_size - 1
    ended = bool(stop_at_eos and r.generated and r.generated[-1] == eos)
    bonus = steps[-1].token if steps and not steps[-1].drafted else -1
    rounds = _rounds_of(eng.ledger())
    return VerifyOutcome(list(r.generated), r.accept_lens[0] if r.accept_lens else 0, bonus, steps, rounds, ended,
                         sum(x.target_tokens - 1 for x in rounds))


def spec_step_chain(target: Model, drafter: Model, ctx: Sequence[int], k: int, rng: DecodeRng,
                    eos_bias: float = 0.0, stop_at_eos: bool = True) -> VerifyOutcome:
    """spec_step_chain (specdec.cpp:78-144) == spec_step_tree with tree(1, 1, k) (specdec.hpp:108-113)."""
    return spec_step_tree(target, drafter, ctx, SDConfig.chain(k), rng, eos_bias, stop_at_eos)


@dataclass
class GenerateResult:
    """GenerateResult (specdec.hpp:117-123)."""
    tokens: List[int]
    steps: List[StepRecord]
    accept_lens: List[int]
    ledger: List[tuple]
    ended_eos: bool = False


def _naive_step(target: Model, ctx: Sequence[int], rng: DecodeRng, eos_bias: float) -> StepRecord:
    """One target sample on the DRAFT stream (specdec.cpp:281-291 / server.cpp:328-347)."""
    eng = BatchEngine(target, None, None, TimingModel(), [RequestState(0, list(ctx), eos_bias, 1, rng)],
                      SDConfig.off(), "sample", True, getattr(target, "device", None))
    eng.set_stop_at_eos(True)
    eng.step()
    rng.state = eng.rng_state(0)
    return eng.requests()[0].steps[0]


def generate(target: Model, drafter: Optional[Model], prompt: Sequence[int], cfg: SDConfig, max_len: int,
             rng: DecodeRng, eos_bias: float = 0.0, stop_at_eos: bool = True) -> GenerateResult:
    """generate (specdec.cpp:271-316): one sequence to EOS or max_len -- naive target steps on the
    DRAFT stream when the config is off or one token is left (specdec.cpp:293-297), otherwise a
    spec_step_tree cycle capped at the remaining budget -- every cycle on the GPU engine."""
    if max_len < 1:
        raise InvalidArgument("generate: max_len must be >= 1")
    eos = target.vocab_size - 1
    res = GenerateResult([], [], [], [], False)
    ctx = list(prompt)
    while len(res.tokens) < max_len and not res.ended_eos:
        remaining = max_len - len(res.tokens)
        if not cfg.enabled or remaining == 1:
            st = _naive_step(target, ctx, rng, eos_bias)
            res.steps.append(st)
            res.tokens.append(st.token)
            res.ledger.append((1, 1, 1))
            ctx.append(st.token)
            if stop_at_eos and st.token == eos:
                res.ended_eos = True
            continue
        out = spec_step_tree(target, drafter, ctx, cfg, rng, eos_bias, stop_at_eos, remaining)
        for rc in out.rounds:
            res.ledger += [(0, rc.drafter_tokens_each, rc.drafter_tokens_each)] * rc.drafter_forwards
            res.ledger.append((1, rc.target_tokens, rc.target_tokens))
        res.accept_lens.append(out.accept_len)
        res.tokens += out.accepted_tokens
        ctx += out.accepted_tokens
        res.steps += out.steps
        res.ended_eos = out.ended
    return res


def mean_accept_len(accept_lens: Sequence[int]) -> float:
    """mean_accept_len (specdec.cpp:318-327)."""
    if not accept_lens:
        raise InvalidArgument("mean_accept_len: no verification cycles recorded")
    s = 0.0
    for a in accept_lens:
        s += a
    return s / len(accept_lens)


# ---- KD learner (learner.hpp:15-69) --------------------------------------------------------------------------
class WeightMode:
    Reward, Uniform, Frozen = 0, 1, 2


@dataclass
class KDPolicy:
    interval: int = 1
    mode: int = WeightMode.Reward
    clip_lo: float = 0.0
    clip_hi: float = 4.0
    lr: float = 0.1

    def _c(self):
        return _KDPolicy(self.interval, self.mode, self.clip_lo, self.clip_hi, self.lr)


def kd_weight(r: float, batch_rewards: Sequence[float], policy: KDPolicy) -> float:
    st = ctypes.c_int()
    w = lib().rs_kd_weight(r, _f64arr(batch_rewards), len(batch_rewards), policy._c(), ctypes.byref(st))
    _check(st.value)
    return w


class SelectionRng:
    """std::mt19937_64 selection stream for kd_update, state kept host-side (learner.cpp:116-121)."""

    def __init__(self, seed: int):
        self.state = (ctypes.c_uint64 * 313)()
        _check(lib().rs_mt19937_64_seed(seed & (2 ** 64 - 1), self.state))


@dataclass
class KDUpdateResult:
    drafter: TabularARModel
    updated: bool
    loss: float
    samples_used: int
    weight_mean: float
    weight_min: float
    weight_max: float
    sim_time: float


def _kd_samples(buffer: Sequence[RolloutSample], with_logprobs):
    """ctypes rs_kd_sample array (+ the arrays it points into). with_logprobs: True (required),
    False (omitted) or "auto" (passed when every step carries its target_logprobs row)."""
    keep = []
    arr = (_KDSample * max(1, len(buffer)))()
    for i, s in enumerate(buffer):
        p, r = _i32arr(s.prompt), _i32arr(s.response)
        lp = None
        want = with_logprobs
        if want == "auto":
            want = len(s.steps) == len(s.response) and all(st.target_logprobs is not None for st in s.steps)
        if want:
            if len(s.steps) != len(s.response):
                raise InvalidArgument("kd_loss: steps/response length mismatch")
            lp = _f64arr([x for st in s.steps for x in st.target_logprobs])
        keep += [p, r, lp]
        arr[i] = _KDSample(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), len(s.prompt),
                           ctypes.cast(r, ctypes.POINTER(ctypes.c_int32)), len(s.response),
                           ctypes.cast(lp, ctypes.POINTER(ctypes.c_double)) if lp is not None else None,
                           s.eos_bias, s.reward)
    return arr, keep


def kd_grad_transformer(drafter: "EagleDrafter", samples: Sequence[RolloutSample], weights: Sequence[float],
                        grad=None, zero_grad: bool = True):
    """Per-rank K5 + backward for a transformer drafter: (sum_i w_i KL_i, gradient of every
    drafter tensor as a DeviceBuffer in drafter.grad_layout()). The gradient is what the
    prompt-sharded learner all-reduces."""
    if grad is None:
        grad = drafter.new_grad()
    arr, keep = _kd_samples(samples, False)
    loss = ctypes.c_double()
    drafter.device.sync()
    _check(lib().rs_kd_grad_transformer(drafter.device.handle, drafter.target.handle, drafter.handle, arr,
                                        len(samples), _f64arr(weights), ctypes.c_void_p(grad.data_ptr()),
                                        1 if zero_grad else 0, ctypes.byref(loss)))
    return loss.value, grad


def kd_loss(drafter, sample: RolloutSample, w: float) -> float:
    """kd_loss (learner.cpp:33-60): w * sum_t KL(p~_t || q_theta(.|ctx_t)) for one sample, on the device
    (tabular: from the sample's target_logprobs; EAGLE drafter: p~ recomputed by its target)."""
    if isinstance(drafter, EagleDrafter):
        loss, _ = kd_grad_transformer(drafter, [sample], [w])
        return loss
    from .distributed import kd_grad_tabular
    return kd_grad_tabular(drafter, [sample], [w])[1]


def kd_loss_gradient(drafter, weighted: Sequence[tuple]):
    """kd_loss_gradient (learner.cpp:62-82): the drafter-logit gradient of sum_i w_i L_KD(sample_i),
    weighted = [(RolloutSample, w)]. Tabular: the full logit-table gradient (list of V^(order+1)
    floats, reference order); EAGLE drafter: the gradient of every drafter tensor (DeviceBuffer,
    drafter.grad_layout())."""
    samples, ws = [x for x, _ in weighted], [w for _, w in weighted]
    if isinstance(drafter, EagleDrafter):
        return kd_grad_transformer(drafter, samples, ws)[1]
    from .distributed import kd_grad_tabular
    return kd_grad_tabular(drafter, samples, ws)[0]


def kd_update(drafter, buffer: Sequence[RolloutSample], policy: KDPolicy, selection_rng: SelectionRng,
              sim_cost_per_token: float) -> KDUpdateResult:
    """kd_update (learner.cpp:98-160): loss + analytic gradient + SGD step on the device.
    Tabular drafters follow the reference bit-for-bit; EAGLE drafters train their LM head with
    p~ recomputed by the target (rs_kd_update_transformer)."""
    if isinstance(drafter, EagleDrafter):
        arr, keep = _kd_samples(buffer, False)
        h = ctypes.c_void_p()
        res = _KDResult()
        _check(lib().rs_kd_update_transformer(drafter.device.handle, drafter.target.handle, drafter.handle, arr,
                                              len(buffer), policy._c(), selection_rng.state, sim_cost_per_token,
                                              ctypes.byref(h), ctypes.byref(res)))
        return KDUpdateResult(EagleDrafter._wrap(h, drafter.target), bool(res.updated), res.loss, res.samples_used,
                              res.weight_mean, res.weight_min, res.weight_max, res.sim_time)
    V = drafter.vocab_size
    keep = []
    arr = (_KDSample * max(1, len(buffer)))()
    for i, s in enumerate(buffer):
        p, r = _i32arr(s.prompt), _i32arr(s.response)
        if len(s.steps) != len(s.response):
            raise InvalidArgument("kd_loss: steps/response length mismatch")
        flat = [x for st in s.steps for x in st.target_logprobs]
        lp = _f64arr(flat)
        keep += [p, r, lp]
        arr[i] = _KDSample(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), len(s.prompt),
                           ctypes.cast(r, ctypes.POINTER(ctypes.c_int32)), len(s.response),
                           ctypes.cast(lp, ctypes.POINTER(ctypes.c_double)), s.eos_bias, s.reward)
    h = ctypes.c_void_p()
    res = _KDResult()
    _check(lib().rs_kd_update_tabular(drafter.device.handle, drafter.handle, arr, len(buffer), policy._c(),
                                      selection_rng.state, sim_cost_per_token, ctypes.byref(h), ctypes.byref(res)))
    new = TabularARModel._wrap(h, drafter.order, drafter.temperature, drafter.device)
    return KDUpdateResult(new, bool(res.updated), res.loss, res.samples_used, res.weight_mean, res.weight_min,
                          res.weight_max, res.sim_time)


# ---- online learner (learner.hpp:39-139) -------------------------------------------------------------------
class ReplayBuffer:
    """ReplayBuffer (learner.hpp:39-51): FIFO of RolloutSamples, the oldest dropped when full."""

    def __init__(self, capacity: int = 4096):
        self._capacity = capacity
        self._entries: List[RolloutSample] = []

    def push(self, sample: RolloutSample) -> None:  # learner.cpp:84-89
        if self._capacity <= 0:
            return
        if len(self._entries) == self._capacity:
            self._entries.pop(0)
        self._entries.append(sample)

    def take_all(self) -> List[RolloutSample]:  # learner.cpp:91-96
        out, self._entries = self._entries, []
        return out

    def size(self) -> int:
        return len(self._entries)

    def capacity(self) -> int:
        return self._capacity


@dataclass
class LearnerMetrics:
    """LearnerMetrics (learner.hpp:75-84)."""
    update_idx: int
    drafter_version: int
    kd_loss: float
    samples_used: int
    weight_mean: float
    weight_min: float
    weight_max: float
    weights_l2: float


class OnlineLearner:
    """OnlineLearner (learner.hpp:87-139) over the device kd_update (rs_learner_*).

    feed() copies samples into the native replay buffer; on_iteration_boundary(it) fires an
    update when (it + 1) % interval == 0 and consumes the whole buffer. With async_=True the
    update runs on a native worker thread with its own CUDA stream, overlapping the caller's
    rollouts; await_pending() is the rendezvous. Async and synchronous learners publish identical
    snapshot sequences (learner.hpp:91-97). Works for tabular and EAGLE drafters."""

    def __init__(self, drafter: Model, policy: KDPolicy, selection_seed: int, sim_cost_per_token: float,
                 buffer_capacity: int = 4096, async_: bool = False):
        self._proto = drafter
        self._policy = policy
        self._engines = []
        self.device = drafter.device
        h = ctypes.c_void_p()
        _check(lib().rs_learner_create(self.device.handle, drafter.handle, policy._c(),
                                       selection_seed & (2 ** 64 - 1), sim_cost_per_token, buffer_capacity,
                                       1 if async_ else 0, ctypes.byref(h)))
        self.handle = h

    def feed(self, samples: Sequence[RolloutSample]) -> None:
        samples = list(samples)
        if not samples:
            return
        arr, keep = _kd_samples(samples, "auto")
        _check(lib().rs_learner_feed(self.handle, arr, len(samples)))

    def feed_engine(self, engine: "BatchEngine", req_ids: Sequence[int], rewards: Sequence[float]) -> None:
        """Samples backed by a live transformer engine (rs_learner_feed_engine): updates read its
        resident KV cache and features instead of recomputing the prompts. The engine is kept
        alive here until no update can still read it; do not step it while one is pending."""
        req_ids = list(req_ids)
        if not req_ids:
            return
        self._engines.append(engine)
        _check(lib().rs_learner_feed_engine(self.handle, engine.handle, _i32arr(req_ids), _f64arr(rewards),
                                            len(req_ids)))

    def on_iteration_boundary(self, iteration: int) -> None:
        _check(lib().rs_learner_on_iteration_boundary(self.handle, iteration))

    def await_pending(self) -> None:
        _check(lib().rs_learner_await_pending(self.handle))
        if self.buffer_size() == 0:
            self._engines = []  # no buffered or pending update reads them any more

    def shutdown(self) -> None:
        _check(lib().rs_learner_shutdown(self.handle))

    def snapshot(self) -> Model:
        h = ctypes.c_void_p()
        _check(lib().rs_learner_snapshot(self.handle, ctypes.byref(h)))
        d = self._proto
        if isinstance(d, EagleDrafter):
            return EagleDrafter._wrap(h, d.target)
        return TabularARModel._wrap(h, d.order, d.temperature, d.device)

    def drafter_version(self) -> int:
        v = ctypes.c_int32()
        _check(lib().rs_learner_drafter_version(self.handle, ctypes.byref(v)))
        return v.value

    def total_sim_time(self) -> float:
        v = ctypes.c_double()
        _check(lib().rs_learner_total_sim_time(self.handle, ctypes.byref(v)))
        return v.value

    def buffer_size(self) -> int:
        v = ctypes.c_int64()
        _check(lib().rs_learner_buffer_size(self.handle, ctypes.byref(v)))
        return v.value

    def metrics(self) -> List[LearnerMetrics]:
        n = ctypes.c_int32()
        _check(lib().rs_learner_metrics(self.handle, None, 0, ctypes.byref(n)))
        buf = (_LearnerMetric * max(1, n.value))()
        _check(lib().rs_learner_metrics(self.handle, buf, n.value, ctypes.byref(n)))
        return [LearnerMetrics(m.update_idx, m.drafter_version, m.kd_loss, m.samples_used, m.weight_mean,
                               m.weight_min, m.weight_max, m.weights_l2) for m in buf[:n.value]]

    def policy(self) -> KDPolicy:
        return self._policy

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().rs_learner_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- GRPO stage + training loop (rl.hpp, trainer.cpp) ------------------------------------------------------
@dataclass
class RewardSpec:
    golden_a: int = 1
    golden_b: int = 2


def reward(y: Sequence[int], spec: RewardSpec = RewardSpec()) -> float:
    """reward (rl.cpp:8-19)."""
    out = ctypes.c_double()
    _check(lib().rs_reward(_i32arr(y), len(y), spec.golden_a, spec.golden_b, ctypes.byref(out)))
    return out.value


def group_advantages(rewards: Sequence[float]) -> List[float]:
    """group_advantages (rl.cpp:21-40)."""
    out = (ctypes.c_double * max(1, len(rewards)))()
    _check(lib().rs_group_advantages(_f64arr(rewards), len(rewards), out))
    return list(out[:len(rewards)])


def policy_update(actor: TabularARModel, weighted: Sequence[tuple], lr: float) -> TabularARModel:
    """policy_update (rl.cpp:74-88) on the device: weighted = [(RolloutSample, advantage)]."""
    samples = [s for s, _ in weighted]
    arr, keep = _kd_samples(samples, False)
    h = ctypes.c_void_p()
    _check(lib().rs_policy_update_tabular(actor.device.handle, actor.handle, arr, _f64arr([a for _, a in weighted]),
                                          _i32arr([s.actor_version for s in samples]), len(samples), lr,
                                          ctypes.byref(h)))
    return TabularARModel._wrap(h, actor.order, actor.temperature, actor.device)


@dataclass
class Task:
    """Task (rl.hpp:23-29)."""
    prompts: List[List[int]]
    eos_biases: List[float]
    reward_spec: RewardSpec = field(default_factory=RewardSpec)
    group_size: int = 8
    max_len: int = 24


def make_step_requests(task: Task, seed: int, step: int) -> List[RequestState]:
    """make_step_requests (rl.cpp:92-111): G requests per prompt, stream (step << 24) | idx."""
    if len(task.prompts) != len(task.eos_biases):
        raise InvalidArgument("make_step_requests: prompts/eos_biases length mismatch")
    out, idx = [], 0
    for p, prompt in enumerate(task.prompts):
        for _ in range(task.group_size):
            out.append(RequestState(idx, list(prompt), task.eos_biases[p], task.max_len,
                                    DecodeRng.from_seed(seed, (step << 24) | idx)))
            idx += 1
    return out


class SDTrainMode:
    Off, Fixed, Adaptive = 0, 1, 2


@dataclass
class TrainOptions:
    """TrainOptions (rl.hpp:54-64)."""
    steps: int = 200
    sd: int = SDTrainMode.Off
    fixed_cfg: SDConfig = field(default_factory=SDConfig.off)
    table: Optional[ProfileTable] = None
    policy_lr: float = 0.2
    seed: int = 1
    count_learner_time: bool = False


@dataclass
class StepMetrics:
    """StepMetrics (rl.hpp:66-75)."""
    step: int = 0
    mean_reward: float = 0.0
    mean_accept_len: float = 0.0
    sim_time: float = 0.0
    actor_version: int = 0
    drafter_version: int = -1
    cycles: int = 0
    switches: int = 0
    wall_ms: float = 0.0  # measured device time of the step's rollout


@dataclass
class TrainResult:
    metrics: List[StepMetrics]
    actor: TabularARModel
    total_sim_time: float = 0.0


def train_loop(actor: TabularARModel, learner: Optional[OnlineLearner], task: Task, tm: TimingModel,
               opts: TrainOptions) -> TrainResult:
    """train_loop (trainer.cpp:9-90): per step, rendezvous with the learner and read its snapshot
    once, generate one group per prompt with the GPU BatchEngine, score, take one policy step on
    the device, then hand the rollouts to the learner at the iteration boundary (async learners
    overlap their update with the next step's rollout)."""
    if opts.sd == SDTrainMode.Adaptive and opts.table is None:
        raise InvalidArgument("train_loop: adaptive mode needs a profile table")
    if opts.sd != SDTrainMode.Off and learner is None:
        raise InvalidArgument("train_loop: spec decoding needs a drafter learner")
    result = TrainResult([], actor, 0.0)
    for step in range(opts.steps):
        drafter = None
        if learner is not None:
            learner.await_pending()
            drafter = learner.snapshot()
        drafter_fn = (lambda d=drafter: d) if opts.sd != SDTrainMode.Off else None
        forced = opts.fixed_cfg if opts.sd == SDTrainMode.Fixed else SDConfig.off()
        table = opts.table if opts.sd == SDTrainMode.Adaptive else None
        run = run_generation(make_step_requests(task, opts.seed, step), result.actor, drafter_fn, table, tm, forced,
                             result.actor.version, record_full_logprobs=learner is not None)
        G = task.group_size
        weighted, reward_sum = [], 0.0
        for p in range(len(task.prompts)):
            rewards = []
            for g in range(G):
                smp = run.samples[p * G + g]
                smp.reward = reward(smp.response, task.reward_spec)
                smp.drafter_version = drafter.version if drafter is not None else -1
                rewards.append(smp.reward)
                reward_sum += smp.reward
            adv = group_advantages(rewards)
            weighted += [(run.samples[p * G + g], adv[g]) for g in range(G)]
        next_actor = policy_update(result.actor, weighted, opts.policy_lr)
        m = StepMetrics(step, reward_sum / len(run.samples),
                        (sum(run.accept_lens) / len(run.accept_lens)) if run.accept_lens else 0.0, run.total_time,
                        result.actor.version, drafter.version if drafter is not None else -1, run.cycles,
                        len(run.switches), run.wall_ms)
        if learner is not None:
            before = learner.total_sim_time()
            learner.feed(run.samples)
            learner.on_iteration_boundary(step)
            if opts.count_learner_time:
                learner.await_pending()
                m.sim_time += learner.total_sim_time() - before
        result.total_sim_time += m.sim_time
        result.metrics.append(m)
        result.actor = next_actor
    if learner is not None:
        learner.await_pending()
    return result
