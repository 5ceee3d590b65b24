"""ctypes binding of include/april_b200.h (the drop-in C-ABI).

This is the exact binding a maintainer of the reference would add: plain
ctypes structs mirroring the header, one function per entry point, status
codes mapped to the reference's exception types (src/april_sim/errors.py:4-9).
Loading fails loudly when the library is missing — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, ContractViolation

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libapril_b200.so")

OK, ERR_CONFIG, ERR_CONTRACT, ERR_CUDA, ERR_OUT_OF_KV, ERR_NCCL = range(6)
STOP_TRACE, STOP_POLICY = 0, 1
MODEL_NONE, MODEL_CONTEXT_FREE, MODEL_TRANSFORMER = 0, 1, 2
REASONS = ("stop_token", "target_length", "max_length")
RUN_TRIGGER, RUN_EVENT, RUN_MAX_ITERS, RUN_DRAINED = 0, 1, 2, 3


class EngineError(RuntimeError):
    """CUDA / NCCL failure inside the engine."""


class OutOfKV(RuntimeError):
    """The KV page pool is exhausted."""


class ModelConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_q_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
                ("qkv_bias", C.c_int32), ("qk_norm", C.c_int32), ("tied_embeddings", C.c_int32),
                ("rope_theta", C.c_float), ("norm_eps", C.c_float)]


class EngineConfigC(C.Structure):
    _fields_ = [("max_slots", C.c_int32), ("l_max", C.c_int32), ("max_handles", C.c_int32),
                ("max_groups", C.c_int32), ("stop_mode", C.c_int32), ("model_kind", C.c_int32),
                ("n_symbols", C.c_int32), ("page_size", C.c_int32), ("kv_pages", C.c_int64),
                ("max_prompt", C.c_int32), ("temperature", C.c_float), ("top_p", C.c_float),
                ("greedy", C.c_int32), ("n_eos", C.c_int32), ("eos_ids", C.c_int32 * 8),
                ("record_payload", C.c_int32), ("weight_seed", C.c_uint64), ("weight_std", C.c_float),
                ("nondeterministic_gemm", C.c_int32), ("kv_resume", C.c_int32),
                ("gemm_autotune", C.c_int32), ("reserved", C.c_int32 * 4)]


class SampleDesc(C.Structure):
    _fields_ = [("handle", C.c_int32), ("group_slot", C.c_int32), ("gen_len", C.c_int32), ("stop_at", C.c_int32),
                ("key0", C.c_uint64), ("key1", C.c_uint64)]


class RunArgs(C.Structure):
    _fields_ = [("max_iters", C.c_int64), ("stop_on_event", C.c_int32), ("use_trigger", C.c_int32),
                ("trigger_mode", C.c_int32), ("n_target", C.c_int32), ("group_size", C.c_int32),
                ("reserved", C.c_int32), ("completed_groups", C.c_int64), ("completed_samples", C.c_int64)]


class Event(C.Structure):
    _fields_ = [("handle", C.c_int32), ("tokens", C.c_int32), ("iteration", C.c_int64), ("reason", C.c_int32),
                ("group_complete", C.c_int32), ("clock", C.c_double)]


class Admit(C.Structure):
    _fields_ = [("handle", C.c_int32), ("slot", C.c_int32), ("iteration", C.c_int64)]


class RunResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("stop_reason", C.c_int32), ("n_events", C.c_int32),
                ("n_admits", C.c_int32), ("reserved", C.c_int32), ("completed_groups", C.c_int64),
                ("completed_samples", C.c_int64), ("iteration_index", C.c_int64),
                ("cumulative_tokens", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("iteration_index", C.c_int64), ("cumulative_tokens", C.c_int64), ("active", C.c_int32),
                ("queued", C.c_int32), ("clock", C.c_double), ("kv_pages_total", C.c_int64),
                ("kv_pages_free", C.c_int64), ("prefill_tokens", C.c_int64), ("kernel_launches", C.c_int64),
                ("reprefill_tokens", C.c_int64), ("reprefill_seconds", C.c_double)]


class DpPeer(C.Structure):
    _fields_ = [("ptr", C.c_uint64), ("kind", C.c_int32), ("reserved", C.c_int32), ("ipc", C.c_uint8 * 64)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double), ("bytes", C.c_double),
                ("flops", C.c_double)]


P = C.c_void_p
I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)

# name -> argtypes; restype is always int (status)
_SIGS = {
    "ab_engine_create": [C.POINTER(EngineConfigC), C.POINTER(ModelConfig), C.c_int, C.POINTER(P)],
    "ab_engine_destroy": [P],
    "ab_engine_weight_count": [P, C.POINTER(C.c_int)],
    "ab_engine_weight_info": [P, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "ab_engine_get_weight": [P, C.c_int, P, C.c_size_t],
    "ab_engine_set_weight": [P, C.c_int, P, C.c_size_t],
    "ab_engine_release_memory": [P],
    "ab_engine_resume_memory": [P],
    "ab_engine_begin_step": [P, C.c_int64, F64P],
    "ab_engine_open_group": [P, C.c_int32, I32P, C.c_int32],
    "ab_engine_release_group": [P, C.c_int32],
    "ab_engine_submit": [P, C.POINTER(SampleDesc), C.c_int],
    "ab_engine_set_group_done": [P, I32P, C.c_int],
    "ab_engine_run": [P, C.POINTER(RunArgs), C.POINTER(RunResult), C.POINTER(Event), C.c_int,
                      C.POINTER(Admit), C.c_int],
    "ab_engine_abort": [P, I32P, I32P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "ab_engine_active": [P, I32P, I32P, C.c_int, C.POINTER(C.c_int)],
    "ab_engine_read_payload": [P, I32P, I32P, I32P, C.c_int, I32P, F64P],
    "ab_engine_sequence_logprobs": [P, I32P, C.c_int, F64P, I32P],
    "ab_engine_score": [P, I32P, C.POINTER(C.c_int64), I32P, C.c_int, F64P],
    "ab_engine_release": [P, I32P, C.c_int],
    "ab_engine_stats": [P, C.POINTER(Stats)],
    "ab_engine_profile": [P, C.c_int, C.c_int],
    "ab_engine_kernel_stats": [P, C.POINTER(KernelStat), C.c_int, C.POINTER(C.c_int)],
    "ab_engine_synchronize": [P],
    "ab_engine_set_iteration": [P, C.c_int64],
    "ab_engine_set_counters": [P, C.c_int64, C.c_int64],
    "ab_engine_dp_export": [P, C.c_int, C.POINTER(C.c_uint64), P],
    "ab_engine_dp_attach": [P, C.c_int, C.c_int, C.POINTER(DpPeer), C.c_int64],
    "ab_engine_dp_detach": [P],
    "ab_group_advantages": [F64P, C.c_int, C.c_int, C.c_int, C.c_double, F64P, I32P, C.c_int],
    "ab_clipped_ratio_terms": [F64P, F64P, I64P, C.c_int, F64P, C.c_double, C.c_double, C.c_int, F64P, I32P,
                               F64P, C.c_int],
    "ab_debug_gemm": [P, P, P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int],
    "ab_debug_gemm_time": [P, P, P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                           C.POINTER(C.c_float)],
    "ab_debug_gemm_sched": [C.c_int] * 8,
    "ab_debug_gemm_clusters": [C.c_int, C.POINTER(C.c_int)],
    "ab_debug_gemm_trace": [C.c_int, P],
    "ab_debug_trace_mark": [C.c_int],
    "ab_debug_decode_attn": [P, P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, I32P, C.c_int,
                             C.c_int, P, C.POINTER(C.c_int)],
    "ab_debug_sample_rows": [P, C.c_int, C.c_int, C.c_float, C.c_int, C.c_float, P, P, P],
}
EXPORTS = sorted(_SIGS) + ["ab_last_error", "ab_version"]

_lib = None


def lib():
    """Load the C-ABI library (raises if the CUDA build is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2509_18521_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.ab_last_error.restype = C.c_char_p
        L.ab_last_error.argtypes = []
        L.ab_version.restype = C.c_int
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().ab_last_error().decode(errors="replace")
    if status == ERR_CONFIG:
        raise ConfigError(msg)
    if status == ERR_CONTRACT:
        raise ContractViolation(msg)
    if status == ERR_OUT_OF_KV:
        raise OutOfKV(msg)
    raise EngineError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
