"""ctypes prototypes for the C-ABI in include/double_b200.h (libdouble_b200.so, built in-tree).

There is no fallback: importing this module without the built library raises, and every compute
entry point fails with DBL_CUDA_ERROR when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DBL_LIB") or os.path.join(PKG, "libdouble_b200.so")  # DBL_LIB: A/B timing of two builds

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
F32P = C.POINTER(C.c_float)
U16P = C.POINTER(C.c_uint16)
VP = C.c_void_p

OK, INVALID_ARGUMENT, RUNTIME_ERROR, LOGIC_ERROR, CUDA_ERROR, NCCL_ERROR = range(6)


class TransformerConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("ffn", C.c_int), ("n_heads", C.c_int),
                ("n_kv_heads", C.c_int), ("head_dim", C.c_int), ("vocab", C.c_int),
                ("tied_embeddings", C.c_int), ("qk_norm", C.c_int), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float), ("init_std", C.c_float), ("max_seq", C.c_int),
                ("seed", C.c_uint64), ("tp_rank", C.c_int), ("tp_size", C.c_int),
                ("layer_std_scale", C.c_float), ("scale_from_layer", C.c_int)]


class PipelineOptions(C.Structure):
    _fields_ = [("gamma", C.c_int), ("depth", C.c_int), ("draft_retrieval", C.c_int),
                ("target_retrieval", C.c_int), ("concurrent", C.c_int), ("t_target", C.c_double),
                ("t_draft", C.c_double), ("t_lookup", C.c_double), ("t_sync", C.c_double),
                ("use_graphs", C.c_int), ("temperature", C.c_double), ("rng_seed", C.c_uint64)]


class RunMetrics(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("rounds", C.c_int64), ("clock", C.c_double),
                ("m", C.c_double), ("amt", C.c_double), ("speedup", C.c_double),
                ("hit_rate", C.c_double), ("lookups", C.c_int64), ("device_ms", C.c_double),
                ("prefill_ms", C.c_double), ("target_fwd_ms", C.c_double),
                ("target_fwd_count", C.c_int64), ("target_rows", C.c_int64),
                ("kernel_launches", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RetrievalResult(C.Structure):
    _fields_ = [("matched_len", C.c_int), ("n_emitted", C.c_int), ("source", C.c_int), ("n_probs", C.c_int)]


MAX_SEGS = 64


class RoundTrace(C.Structure):
    _fields_ = [("round", C.c_int64), ("mode", C.c_int), ("pending", C.c_int), ("draft_len", C.c_int),
                ("n_draft_matched", C.c_int), ("draft_matched", C.c_int32 * MAX_SEGS), ("target_matched", C.c_int),
                ("target_source", C.c_int), ("accepted_pending", C.c_int), ("pending_reject", C.c_int),
                ("rejected", C.c_int), ("committed_count", C.c_int), ("kind", C.c_int), ("clock_delta", C.c_double)]


class PipelineStateC(C.Structure):
    _fields_ = [("committed", I32P), ("n_committed", C.c_int64), ("committed_cap", C.c_int64),
                ("speculative", I32P), ("n_speculative", C.c_int64), ("speculative_cap", C.c_int64),
                ("n_spec_probs", C.c_int64), ("spec_probs", F64P), ("spec_probs_cap", C.c_int64),
                ("mode", C.c_int), ("prev_tokens", C.c_int), ("round", C.c_int64), ("clock", C.c_double),
                ("last_committed_len", C.c_int64)]


# name -> argtypes (all return int status unless listed in _RESTYPE)
PROTOTYPES = {
    "dbl_last_error": [],
    "dbl_version": [],
    "dbl_device_ok": [],
    "dbl_store_create": [C.c_int, C.c_int, C.c_int, C.POINTER(VP)],
    "dbl_store_destroy": [VP],
    "dbl_store_set_rejected_enabled": [VP, C.c_int],
    "dbl_store_set_layer_order": [VP, C.c_int, C.c_int],
    "dbl_store_insert": [VP, C.c_int, I32P, C.c_int, C.c_int64],
    "dbl_store_record": [VP, C.c_int, I32P, C.c_int],
    "dbl_store_flush_session": [VP],
    "dbl_store_clear_layer": [VP, C.c_int],
    "dbl_store_get_step": [VP, I64P],
    "dbl_store_set_step": [VP, C.c_int64],
    "dbl_store_layer_info": [VP, C.c_int, I64P, I64P, I64P],
    "dbl_store_layer_read": [VP, C.c_int, I32P, C.c_int64, I32P, I64P, C.c_int64],
    "dbl_store_lookup": [VP, I32P, C.c_int, C.c_int, I32P, C.c_int, C.POINTER(C.c_int),
                         C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "dbl_store_lookup_batch": [VP, C.c_int, I64P, I32P, I32P, C.c_int, I32P, I32P, I32P, I32P],
    "dbl_store_stats": [VP, I64P],
    "dbl_store_build_index": [VP, C.c_int],
    "dbl_store_index_entries": [VP, C.c_int, I64P],
    "dbl_store_profile_lookup": [VP, I32P, C.c_int, C.c_int, C.c_int, F64P],
    "dbl_table_create": [C.c_int, C.c_int, C.c_int64, I32P, F64P, F64P, C.c_int, C.POINTER(VP)],
    "dbl_transformer_create": [C.POINTER(TransformerConfig), C.c_int, VP, C.POINTER(VP)],
    "dbl_tp_transformer_create": [C.POINTER(TransformerConfig), I32P, C.c_int, C.POINTER(VP)],
    "dbl_model_destroy": [VP],
    "dbl_model_vocab": [VP, C.POINTER(C.c_int)],
    "dbl_model_weight_bytes": [VP, I64P],
    "dbl_forward_argmax": [VP, I32P, C.c_int, I32P, C.c_int, I32P],
    "dbl_forward_logits": [VP, I32P, C.c_int, I32P, C.c_int, F32P],
    "dbl_forward_dists": [VP, I32P, C.c_int, I32P, C.c_int, F64P],
    "dbl_transformer_get_weight": [VP, C.c_char_p, C.c_int, U16P, C.c_int64],
    "dbl_run": [VP, VP, VP, I32P, C.c_int, C.c_int, C.POINTER(PipelineOptions), I32P, C.c_int,
                C.POINTER(C.c_int), C.POINTER(RunMetrics), C.c_char_p, C.c_int64, I64P],
    "dbl_set_exact_sampling": [C.c_int],
    "dbl_run_ar": [VP, I32P, C.c_int, C.c_int, C.c_double, I32P, C.c_int, C.POINTER(C.c_int),
                   C.POINTER(RunMetrics), C.c_char_p, C.c_int64, I64P],
    "dbl_run_ar_sampled": [VP, I32P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64, I32P, C.c_int,
                           C.POINTER(C.c_int), C.POINTER(RunMetrics), C.c_char_p, C.c_int64, I64P],
    "dbl_tp_ipc_export": [VP, VP, C.c_int64],
    "dbl_tp_ipc_import": [VP, VP, C.c_int],
    "dbl_run_batch": [VP, VP, C.c_int, C.POINTER(VP), I64P, I32P, C.c_int, C.POINTER(PipelineOptions), I32P, I32P,
                      C.POINTER(RunMetrics), C.c_char_p, C.c_int64, I64P],
    "dbl_run_ar_batch": [VP, C.c_int, I64P, I32P, C.c_int, I32P, I32P, F64P, I64P],
    "dbl_run_serial_sd": [VP, VP, VP, I32P, C.c_int, C.c_int, C.POINTER(PipelineOptions), C.c_int,
                          I32P, C.c_int, C.POINTER(C.c_int), C.POINTER(RunMetrics), C.c_char_p,
                          C.c_int64, I64P],
    "dbl_last_run_log": [I32P, C.c_int64, I64P],
    "dbl_last_run_jsonl": [C.c_char_p, C.c_int64, I64P],
    "dbl_profile_forward": [VP, C.c_int, C.c_int, C.c_int, F64P],
    "dbl_debug_gemm_trace": [C.POINTER(C.c_uint64), C.c_int64, I32P, I64P, C.POINTER(C.c_int)],
    "dbl_debug_fwd_trace": [C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "dbl_debug_gemm_bench": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, F64P],
    "dbl_rng_create": [C.c_uint64, C.c_int, C.POINTER(VP)],
    "dbl_rng_derive": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(VP)],
    "dbl_rng_uniform": [VP, F64P, C.c_int],
    "dbl_rng_destroy": [VP],
    "dbl_accept_prob": [F64P, C.c_int, F64P, C.c_int, C.c_int32, F64P],
    "dbl_residual_sample": [F64P, C.c_int, F64P, C.c_int, VP, I32P],
    "dbl_residual_sample_point_mass": [F64P, C.c_int, C.c_int32, VP, I32P],
    "dbl_verify_against_target": [I32P, C.c_int, F64P, I64P, C.c_int, F64P, I64P, C.c_int, C.c_double, VP,
                                  C.POINTER(C.c_int)],
    "dbl_guided_output": [I32P, C.c_int, F64P, I64P, C.c_int, I32P, C.c_int, F64P, I64P, C.c_int, C.c_int,
                          C.c_double, VP, I32P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                          C.POINTER(C.c_int)],
    "dbl_tempered": [F64P, C.c_int, C.c_double, C.c_int, F64P],
    "dbl_argmax_token": [F64P, C.c_int, C.c_int, I32P],
    "dbl_argmax_rows": [F64P, I64P, C.c_int, C.c_int, I32P],
    "dbl_sample": [F64P, C.c_int, C.c_double, VP, C.c_int, I32P],
    "dbl_accept_with_model": [F64P, I64P, C.c_int, I32P, C.c_int, C.c_double, VP, C.c_int, I32P, C.c_int, F64P,
                              C.c_int64, C.POINTER(RetrievalResult)],
    "dbl_retrieval_forward": [VP, VP, I32P, C.c_int, C.c_int, C.c_double, VP, C.c_int, I32P, C.c_int, F64P,
                              C.c_int64, C.POINTER(RetrievalResult)],
    "dbl_iterative_draft": [VP, VP, I32P, C.c_int, C.c_int, C.c_int, C.c_double, VP, C.c_int,
                            C.POINTER(RetrievalResult), I32P, C.c_int, C.POINTER(C.c_int), F64P, C.c_int64],
    "dbl_measure_amt": [I32P, C.c_int, F64P],
    "dbl_rollback": [C.POINTER(PipelineStateC), C.c_int64],
    "dbl_session_create": [VP, VP, C.POINTER(VP)],
    "dbl_session_destroy": [VP],
    "dbl_run_round": [VP, VP, C.POINTER(PipelineOptions), C.POINTER(PipelineStateC), C.POINTER(RoundTrace)],
    "dbl_compute_metrics": [C.POINTER(RoundTrace), C.c_int, C.c_double, C.POINTER(RunMetrics)],
    "dbl_traces_to_jsonl": [C.POINTER(RoundTrace), C.c_int, C.c_char_p, C.c_int64, I64P],
    "dbl_write_traces": [C.POINTER(RoundTrace), C.c_int, C.c_char_p],
    "dbl_last_run_traces": [C.POINTER(RoundTrace), C.c_int64, I64P],
    "dbl_store_clone": [VP, C.POINTER(VP)],
    "dbl_build_prior": [VP, I64P, I32P, C.c_int, C.c_int, C.c_int],
    "dbl_debug_gemm": [C.c_int, U16P, C.c_int, C.c_int, U16P, C.c_int, C.c_int, C.c_int, F32P,
                       I32P],
}
_RESTYPE = {"dbl_last_error": C.c_char_p}

_lib = None


def lib() -> C.CDLL:
    """Load libdouble_b200.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing — run `python -m paper_2601_05524_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in PROTOTYPES.items():
            if os.environ.get("DBL_LIB") and not hasattr(L, name):
                continue  # A/B timing against an older build: entry points it predates are absent
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


class DoubleError(RuntimeError):
    status = RUNTIME_ERROR


class InvalidArgument(DoubleError, ValueError):  # std::invalid_argument
    status = INVALID_ARGUMENT


class LogicError(DoubleError):  # std::logic_error
    status = LOGIC_ERROR


class CudaError(DoubleError):
    status = CUDA_ERROR


_EXC = {INVALID_ARGUMENT: InvalidArgument, RUNTIME_ERROR: DoubleError, LOGIC_ERROR: LogicError,
        CUDA_ERROR: CudaError, NCCL_ERROR: DoubleError}


def check(status: int):
    if status != OK:
        msg = lib().dbl_last_error().decode(errors="replace")
        raise _EXC.get(status, DoubleError)(msg)
