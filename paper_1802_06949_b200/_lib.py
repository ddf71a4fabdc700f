"""ctypes binding of libcollsim_b200.so (include/collsim_b200.h).

The library is built in-tree by ``paper_1802_06949_b200.build``.  There is no
fallback: if the shared object is missing or fails to load, importing the
package raises -- the product path never runs on the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libcollsim_b200.so"

CS_F64, CS_F32, CS_BF16 = 0, 1, 2
CS_OP_COMPUTE, CS_OP_COPY, CS_OP_COLLECTIVE, CS_OP_OTHER = 0, 1, 2, 3
CS_DISPATCH_INLINE, CS_DISPATCH_POOL, CS_DISPATCH_HOST = 0, 1, 2
CS_KV_FUNNEL, CS_KV_DEPCHA, CS_KV_CONCOM, CS_KV_NAIVE = 0, 1, 2, 3
CS_MAX_RANKS = 16

STATUS_NAMES = {
    0: "OK", -1: "ConfigError", -2: "UsageError", -3: "MismatchError",
    -4: "DeadlockTimeout", -5: "EngineError", -6: "CudaError", -7: "NcclError", -8: "InternalError",
}


class CopyEntry(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("n", C.c_uint64)]


class UpdateEntry(C.Structure):
    _fields_ = [("w", C.c_void_p), ("g", C.c_void_p), ("mom", C.c_void_p), ("n", C.c_uint64)]


class P2PUpdateC(C.Structure):
    _fields_ = [("entries", C.c_void_p), ("n_entries", C.c_int), ("w_dtype", C.c_int), ("lr", C.c_double),
                ("rescale", C.c_double), ("momentum", C.c_double), ("shard_only", C.c_int)]


class KvConfigC(C.Structure):
    _fields_ = [("mode", C.c_int), ("outstanding", C.c_int), ("num_keys", C.c_int),
                ("comm_dtype", C.c_int), ("bucket_bytes", C.c_uint64), ("issue_order", C.c_int),
                ("comm_priority", C.c_int), ("p2p", C.c_int), ("zero", C.c_int)]


class SlotC(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int), ("numel", C.c_uint64), ("tag", C.c_uint64)]


class SgdC(C.Structure):
    _fields_ = [("lr", C.c_double), ("rescale", C.c_double), ("momentum", C.c_double)]


HOST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
STREAM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)

_P = C.c_void_p
_I = C.c_int
_U64 = C.c_uint64
_PI = C.POINTER(C.c_int)
_PU64 = C.POINTER(C.c_uint64)

# name -> argtypes (restype is int unless listed in _RESTYPE)
SIGNATURES = {
    "cs_last_error": [],
    "cs_status_name": [_I],
    "cs_version": [],
    "cs_device_count": [_PI],
    "cs_pack": [C.POINTER(CopyEntry), _I, _I, _I, _P],
    "cs_sum_buffers": [C.POINTER(_P), _I, C.POINTER(_P), _I, _U64, _I, _P],
    "cs_sgd_update": [C.POINTER(UpdateEntry), _I, _I, _I, C.c_double, C.c_double, C.c_double, _P],
    "cs_synth_backward": [_P, _P, _U64, _I, _U64, _I, _P],
    "cs_checksum": [_P, _U64, _I, _P, _P],
    "cs_trace_create": [C.POINTER(_P)],
    "cs_trace_destroy": [_P],
    "cs_trace_count": [_P, _PU64],
    "cs_trace_write_jsonl": [_P, C.c_char_p],
    "cs_trace_gauges": [_P, _PI, _PI],
    "cs_engine_create": [_I, _I, _I, _P, C.POINTER(_P)],
    "cs_engine_destroy": [_P],
    "cs_engine_new_variable": [_P, _PU64],
    "cs_engine_push_host": [_P, HOST_FN, _P, _PU64, _I, _PU64, _I, _I, _I, _PU64],
    "cs_engine_push_stream": [_P, STREAM_FN, _P, _PU64, _I, _PU64, _I, _I, _I, _I, _I, _PU64],
    "cs_engine_wait_for": [_P, _U64],
    "cs_engine_wait_all": [_P],
    "cs_engine_import_event": [_P, _P, _PU64, _I, _I, _I, _PU64],
    "cs_engine_stream_wait": [_P, _PU64, _I, _P],
    "cs_engine_shutdown": [_P],
    "cs_engine_new_lane": [_P, _I, _PI],
    "cs_engine_lane_stream": [_P, _I, C.POINTER(_P)],
    "cs_engine_stats": [_P, _PU64, _PU64],
    "cs_engine_num_threads": [_P, _PI],
    "cs_engine_set_watchdog": [_P, C.c_int64],
    "cs_transport_create_local": [_I, _I, _P, C.POINTER(_P)],
    "cs_transport_create_local_peer": [_I, _I, _P, C.POINTER(_P)],
    "cs_transport_create_nccl": [C.c_char_p, _I, _I, _I, _I, _P, C.POINTER(_P)],
    "cs_transport_create_ledger_only": [C.c_char_p, _I, _I, _I, _P, C.POINTER(_P)],
    "cs_transport_destroy": [_P],
    "cs_transport_num_ranks": [_P, _PI],
    "cs_transport_num_communicators": [_P, _PI],
    "cs_transport_new_communicator": [_P, _PI],
    "cs_transport_set_inject_latency": [_P, C.c_int64],
    "cs_transport_abort": [_P],
    "cs_allreduce_sum": [_P, _I, _I, _P, _U64, _I, _I, _P],
    "cs_broadcast": [_P, _I, _I, _I, _P, _U64, _I, _I, _P],
    "cs_barrier": [_P, _I, _I, _I, _P],
    "cs_transport_p2p_capable": [_P, _PI],
    "cs_transport_share_buffer": [_P, _P, C.POINTER(_P)],
    "cs_transport_share_buffer_rank": [_P, _I, _P, C.POINTER(_P)],
    "cs_transport_device_failure": [_P, C.c_char_p, _I],
    "cs_transport_p2p_stamps": [_P, _I, C.POINTER(C.c_uint64), _I, C.POINTER(_I)],
    "cs_allreduce_p2p": [_P, _I, _I, C.POINTER(_P), _U64, _I, _I, C.c_void_p, _P],
    "cs_transport_nvls_capable": [_P, _PI],
    "cs_transport_alloc_nvls": [_P, _U64, C.POINTER(_P), C.POINTER(_P)],
    "cs_allreduce_nvls": [_P, _I, _I, _P, _P, _U64, _I, _I, C.c_void_p, _P],
    "cs_create_communicators": [_P, _I, _PI],
    "cs_kv_create": [_P, _P, _I, C.POINTER(KvConfigC), _PI, _I, C.POINTER(_P)],
    "cs_kv_destroy": [_P],
    "cs_kv_init": [_P, _I, SlotC],
    "cs_kv_push": [_P, _PI, C.POINTER(SlotC), _I],
    "cs_kv_pull": [_P, _PI, C.POINTER(SlotC), _I],
    "cs_kv_pull_update": [_P, _PI, C.POINTER(SlotC), _I, C.POINTER(SgdC)],
    "cs_kv_barrier": [_P],
    "cs_kv_outstanding_in_flight": [_P, _PI],
    "cs_kv_comm_buf": [_P, _I, _P, _PU64, _PI],
    "cs_kv_key_map": [_P, _I, _PI, _PU64],
    "cs_kv_bucket_view": [_P, _I, C.POINTER(_P)],
    "cs_kv_arena": [_P, C.POINTER(_P), _PU64],
    "cs_kv_register_grads": [_P, _P, C.c_uint64],
    "cs_kv_num_buckets": [_P, _PI],
    "cs_kv_bucket_lane": [_P, _I, _PI],
    "cs_synth_create": [_P, _P, _I, _I, C.c_void_p, _PU64, _I, _PI, _I, C.POINTER(_P)],
    "cs_synth_create_profiled": [_P, _P, _I, _I, C.c_void_p, _PU64, C.POINTER(C.c_double), _I, _PI, _I,
                                 C.POINTER(_P)],
    "cs_synth_destroy": [_P],
    "cs_synth_init": [_P],
    "cs_synth_step": [_P, _I],
    "cs_synth_run": [_P, _I, _I, C.POINTER(C.c_double)],
    "cs_synth_run_e2e": [_P, _I, _I, C.POINTER(C.c_double)],
    "cs_synth_checksum": [_P, C.POINTER(C.c_double)],
    "cs_synth_read_weights": [_P, _P, _U64],
    "cs_synth_info": [_P, _PU64, _PU64, _PI],
    "cs_synth_last_host_ms": [_P, C.POINTER(C.c_double)],
    "cs_launch_count": [_PU64],
    "cs_profile_enable": [_I],
    "cs_profile_collect": [_I, _PU64, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "cs_profile_reset": [],
    "cs_host_profile": [C.c_char_p, _I, _I],
}


class SynthConfigC(C.Structure):
    _fields_ = [("mode", C.c_int), ("w_dtype", C.c_int), ("g_dtype", C.c_int), ("comm_dtype", C.c_int),
                ("bucket_bytes", C.c_uint64), ("issue_order", C.c_int), ("outstanding", C.c_int),
                ("lr", C.c_double), ("rescale", C.c_double), ("momentum", C.c_double),
                ("backward_ns", C.c_uint64), ("backward_ctas", C.c_int), ("fused_update", C.c_int),
                ("comm_priority", C.c_int), ("host_source", C.c_int), ("p2p", C.c_int),
                ("grad_views", C.c_int), ("zero", C.c_int), ("order_seed", C.c_int),
                ("direct_grads", C.c_int)]


CS_STEP_BACKWARD, CS_STEP_COMM, CS_STEP_LOCAL_UPDATE, CS_STEP_CHECKSUM = 1, 2, 4, 8
KERNEL_KINDS = {"pack": 0, "sum": 1, "sgd": 2, "synth": 3, "checksum": 4, "pack_sgd": 5}
_RESTYPE = {"cs_last_error": C.c_char_p, "cs_status_name": C.c_char_p}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1802_06949_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    return lib


lib = _load()


class CsError(RuntimeError):
    """Raised for a non-zero status; ``kind`` is the reference Error kind name
    (R/core/include/collsim/error.hpp:19-28)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, "InternalError")
        super().__init__(f"{self.kind}: {message}")


class ConfigError(CsError):
    pass


class UsageError(CsError):
    pass


class MismatchError(CsError):
    pass


class DeadlockTimeout(CsError):
    pass


class EngineError(CsError):
    pass


class CudaError(CsError):
    pass


class NcclError(CsError):
    pass


_ERRORS = {-1: ConfigError, -2: UsageError, -3: MismatchError, -4: DeadlockTimeout,
           -5: EngineError, -6: CudaError, -7: NcclError}


def check(status: int) -> None:
    if status != 0:
        msg = lib.cs_last_error().decode(errors="replace")
        raise _ERRORS.get(status, CsError)(status, msg)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
