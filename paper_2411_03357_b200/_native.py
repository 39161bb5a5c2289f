"""ctypes binding of libspgcm.so (include/spgcm.h) and libsppipe.so.

The shared libraries are built in-tree by `__graft_entry__.build()` into
`paper_2411_03357_b200/lib/`.  There is no fallback: if the library or a CUDA
device is missing, every crypto entry point raises `NativeUnavailable`.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
SPGCM_PATH = os.environ.get("SPGCM_LIB") or os.path.join(LIB_DIR, "libspgcm.so")  # env: A/B builds
SPPIPE_PATH = os.environ.get("SPPIPE_LIB") or os.path.join(LIB_DIR, "libsppipe.so")  # env: A/B builds

SP_OK, SP_EINVAL, SP_EAUTH, SP_ECUDA, SP_ENODEV = 0, 1, 2, 3, 4

# Every symbol include/spgcm.h declares (checked by tests/test_abi.py).
SPGCM_SYMBOLS = (
    "sp_ctx_create", "sp_ctx_destroy", "sp_seal", "sp_open", "sp_seal_batch", "sp_open_batch",
    "sp_crypt_batch", "sp_seal_host", "sp_open_host", "sp_seal_host_batch", "sp_open_host_batch",
    "sp_last_error", "sp_version", "sp_launch_count", "sp_ctx_round_keys", "sp_ctx_hash_key",
    "sp_ctx_set_max_sms", "sp_ctx_max_sms", "sp_crypt_levels", "sp_ctx_set_small_sms",
)


class NativeUnavailable(RuntimeError):
    """libspgcm could not be loaded or has no usable sm_100a device."""


class SpDesc(ctypes.Structure):
    _fields_ = [
        ("dir", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("iv", ctypes.c_uint64),
        ("len", ctypes.c_uint64),
        ("src", ctypes.c_void_p),
        ("dst", ctypes.c_void_p),
        ("tag", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib = None


def load_spgcm() -> ctypes.CDLL:
    """Load libspgcm.so (no GPU needed just to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SPGCM_PATH):
            raise NativeUnavailable(
                f"{SPGCM_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(SPGCM_PATH)
        vp, u8p = ctypes.c_void_p, ctypes.c_void_p
        lib.sp_ctx_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        lib.sp_ctx_create.restype = ctypes.c_int
        lib.sp_ctx_destroy.argtypes = [vp]
        lib.sp_ctx_destroy.restype = None
        lib.sp_seal.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, vp, vp, vp]
        lib.sp_open.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, vp, vp, vp, vp]
        for name in ("sp_seal_batch", "sp_open_batch", "sp_crypt_batch"):
            getattr(lib, name).argtypes = [vp, ctypes.POINTER(SpDesc), ctypes.c_int, vp]
        lib.sp_crypt_levels.argtypes = [vp, ctypes.POINTER(SpDesc), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                        ctypes.c_int, vp]
        for name in ("sp_seal_host_batch", "sp_open_host_batch"):
            getattr(lib, name).argtypes = [vp, ctypes.POINTER(SpDesc), ctypes.c_int]
        lib.sp_seal_host.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, vp, u8p]
        lib.sp_open_host.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, u8p, vp]
        lib.sp_last_error.restype = ctypes.c_char_p
        lib.sp_version.restype = ctypes.c_char_p
        lib.sp_launch_count.restype = ctypes.c_uint64
        lib.sp_ctx_round_keys.argtypes = [vp, vp]
        lib.sp_ctx_hash_key.argtypes = [vp, vp]
        lib.sp_ctx_set_max_sms.argtypes = [vp, ctypes.c_int]
        lib.sp_ctx_set_small_sms.argtypes = [vp, ctypes.c_int]
        lib.sp_ctx_max_sms.argtypes = [vp]
        _lib = lib
        return lib


def last_error() -> str:
    return load_spgcm().sp_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load_spgcm().sp_launch_count())


# ---- libsppipe (include/sppipe.h) ------------------------------------------------------
SP_EENGINE, SP_EOVERLAP, SP_ESTATE, SP_EUNKNOWN_BLOCK, SP_EBOUNDS, SP_EGUARD, SP_EAMBIGUOUS, SP_EIVREUSE, \
    SP_EKEY = range(10, 19)

SPPIPE_SYMBOLS = (
    "sp_pred_create", "sp_pred_destroy", "sp_pred_classify", "sp_pred_observe_out", "sp_pred_observe_in",
    "sp_pred_observe_sync", "sp_pred_recognize", "sp_pred_cycle_entry", "sp_pred_predict_batches",
    "sp_pred_outstanding", "sp_pred_in_batch_count", "sp_pred_decision_count", "sp_pred_decision",
    "sp_pred_predict_batches_in", "sp_pred_script", "sp_pred_event_count", "sp_pred_event", "sp_pred_in_batch",
    "sp_pipe_create", "sp_pipe_destroy", "sp_pipe_register_block", "sp_pipe_seed_device", "sp_pipe_submit_h2d",
    "sp_pipe_submit_d2h", "sp_pipe_small_io", "sp_pipe_sync", "sp_pipe_speculate", "sp_pipe_relinquish",
    "sp_pipe_drain_decrypts", "sp_pipe_finish", "sp_pipe_audit", "sp_pipe_finish_observable", "sp_pipe_flush", "sp_pipe_app_write", "sp_pipe_app_read", "sp_pipe_replay", "sp_pipe_plain_replay",
    "sp_pipe_handle_done", "sp_pipe_test_corrupt", "sp_test_xfer", "sp_pipe_report", "sp_pipe_counter_name", "sp_pipe_send_iv",
    "sp_pipe_recv_iv",
    "sp_pipe_action_count", "sp_pipe_actions", "sp_pipe_sent_count", "sp_pipe_sent_log",
    "sp_pipe_record_count", "sp_pipe_record_first", "sp_pipe_record", "sp_pipe_pending", "sp_pipe_pending_at_iv", "sp_pipe_delivered_count",
    "sp_pipe_delivered", "sp_pipe_compute", "sp_pipe_compute_stats", "sp_pipe_issuer_stats", "sp_pipe_stats", "sp_pipe_pool_stats", "sp_pipe_last_error",
    "sp_val_create", "sp_val_destroy", "sp_val_label", "sp_val_validate", "sp_val_commit", "sp_val_invalidate",
    "sp_val_write_fault", "sp_val_pending_at_iv", "sp_val_has_pending_range", "sp_val_invalidate_pending_below", "sp_val_pending",
    "sp_val_record_count", "sp_val_record", "sp_val_counters",
)


class SpPredConfig(ctypes.Structure):
    _fields_ = [
        ("small_io_threshold", ctypes.c_uint64),
        ("swap_min", ctypes.c_uint64),
        ("chunk_bytes", ctypes.c_uint64),
        ("warmup_matches", ctypes.c_int64),
        ("history_cap", ctypes.c_int64),
        ("layer_param_bytes", ctypes.c_uint64),
        ("kv_block_bytes", ctypes.c_uint64),
    ]


class SpPrediction(ctypes.Structure):
    _fields_ = [("block", ctypes.c_int64), ("predicted_iv", ctypes.c_uint64), ("leeway", ctypes.c_uint64),
                ("batch", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class SpDecision(ctypes.Structure):
    _fields_ = [("event", ctypes.c_int32), ("pattern", ctypes.c_int32), ("confidence", ctypes.c_int64),
                ("after_batches", ctypes.c_int64)]


class SpPipeConfig(ctypes.Structure):
    _fields_ = [
        ("window", ctypes.c_uint32), ("leeway", ctypes.c_uint32), ("depth", ctypes.c_uint32),
        ("workers", ctypes.c_uint32), ("chunk_bytes", ctypes.c_uint64), ("nop_bytes", ctypes.c_uint32),
        ("ring_slots", ctypes.c_uint32), ("speculate", ctypes.c_uint8), ("defer_swap_decrypt", ctypes.c_uint8),
        ("record_stream", ctypes.c_uint8), ("strict_auth", ctypes.c_uint8), ("reference_compat", ctypes.c_uint8),
        ("dry", ctypes.c_uint8), ("hw_guards", ctypes.c_uint8), ("window_aware", ctypes.c_uint8),
        ("initial_h2d_iv", ctypes.c_uint64),
        ("initial_d2h_iv", ctypes.c_uint64), ("batch_bytes", ctypes.c_uint64), ("reserve_bytes", ctypes.c_uint64),
        ("record_history", ctypes.c_uint64), ("crypto_sms", ctypes.c_uint32), ("reserved2", ctypes.c_uint32),
    ]


class SpAction(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("flags", ctypes.c_int32), ("iv", ctypes.c_int64),
                ("nbytes", ctypes.c_uint64), ("record_id", ctypes.c_int64), ("task_id", ctypes.c_int64),
                ("count", ctypes.c_int64), ("seq", ctypes.c_int64)]


class SpSent(ctypes.Structure):
    _fields_ = [("iv", ctypes.c_uint64), ("size", ctypes.c_uint64), ("nop", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class SpRecord(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int64), ("base", ctypes.c_uint64), ("len", ctypes.c_uint64), ("iv", ctypes.c_uint64),
                ("span", ctypes.c_uint64), ("block_id", ctypes.c_int64), ("state", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class SpDelivery(ctypes.Structure):
    _fields_ = [("seq", ctypes.c_uint64), ("addr", ctypes.c_uint64), ("size", ctypes.c_uint64)]


class SpEvent(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("cls", ctypes.c_int32), ("block", ctypes.c_int64),
                ("base", ctypes.c_uint64), ("len", ctypes.c_uint64), ("payload", ctypes.c_uint64)]


_pipe_lib = None


def load_sppipe() -> ctypes.CDLL:
    """Load libsppipe.so (links libspgcm.so from the same directory)."""
    global _pipe_lib
    with _lock:
        if _pipe_lib is not None:
            return _pipe_lib
        if not os.path.exists(SPPIPE_PATH):
            raise NativeUnavailable(
                f"{SPPIPE_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(SPPIPE_PATH)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        P = ctypes.POINTER
        sig = {
            "sp_pred_create": [P(SpPredConfig), P(vp)],
            "sp_pred_classify": [vp, u64, P(i32)],
            "sp_pred_observe_out": [vp, i64],
            "sp_pred_observe_in": [vp, P(i64), i32],
            "sp_pred_observe_sync": [vp],
            "sp_pred_recognize": [vp, P(i32), P(i64), P(i64), P(i64)],
            "sp_pred_cycle_entry": [vp, i64, P(i64), i32, P(i32)],
            "sp_pred_predict_batches": [vp, u64, u64, i32, P(SpPrediction), i32, P(i32)],
            "sp_pred_outstanding": [vp, P(i64), i64, P(i64)],
            "sp_pred_decision": [vp, i64, P(SpDecision)],
            "sp_pred_predict_batches_in": [vp, u64, u64, i32, P(i64), i64, P(SpPrediction), i32, P(i32)],
            "sp_pred_script": [vp, P(SpPrediction), i32, P(i64), i64],
            "sp_pred_event": [vp, i64, P(i32), P(i64)],
            "sp_pred_in_batch": [vp, i64, P(i64), i32, P(i32)],
            "sp_pipe_pending": [vp, P(i64), i64, P(i64)],
            "sp_val_create": [u64, P(vp)],
            "sp_val_label": [vp, u64, u64, u64, u64, i64, P(i64)],
            "sp_val_validate": [vp, u64, u64, u64, P(i32), P(i64)],
            "sp_val_commit": [vp, i64], "sp_val_invalidate": [vp, i64], "sp_val_write_fault": [vp, i64],
            "sp_val_invalidate_pending_below": [vp, u64, P(i64)],
            "sp_val_pending": [vp, P(i64), i64, P(i64)],
            "sp_val_record": [vp, i64, P(SpRecord)],
            "sp_val_counters": [vp, P(i64)],
            "sp_pipe_create": [P(SpPipeConfig), ctypes.c_char_p, vp, P(vp)],
            "sp_pipe_register_block": [vp, i64, u64, u64, i32, vp],
            "sp_pipe_seed_device": [vp, i64, vp, u64, i32],
            "sp_pipe_submit_h2d": [vp, u64, u64, i32, i64, P(u64), P(i32)],
            "sp_pipe_submit_d2h": [vp, u64, u64, i32, i64, P(u64)],
            "sp_pipe_small_io": [vp, i32, vp, u64],
            "sp_pipe_sync": [vp], "sp_pipe_speculate": [vp], "sp_pipe_relinquish": [vp, P(i64)],
            "sp_pipe_drain_decrypts": [vp], "sp_pipe_finish": [vp], "sp_pipe_audit": [vp], "sp_pipe_finish_observable": [vp],
            "sp_pipe_flush": [vp, i32],
            "sp_pipe_app_write": [vp, i64, u64, vp, u64, P(i64)],
            "sp_pipe_app_read": [vp, i64, u64, u64, vp],
            "sp_pipe_replay": [vp, P(SpEvent), u64, vp, P(u64)],
            "sp_pipe_plain_replay": [vp, P(SpEvent), u64, vp],
            "sp_pipe_handle_done": [vp, u64, P(i32)],
            "sp_pipe_test_corrupt": [vp, i32, u64, u64, ctypes.c_uint8],
            "sp_test_xfer": [i32, P(vp), P(vp), P(u64)],
            "sp_pipe_report": [vp, P(i64), i32, P(i32)],
            "sp_pipe_actions": [vp, i64, P(SpAction), i64, P(i64)],
            "sp_pipe_sent_log": [vp, i32, i64, P(SpSent), i64, P(i64)],
            "sp_pipe_delivered": [vp, i32, i64, P(SpDelivery), vp],
            "sp_pipe_record": [vp, i64, P(SpRecord)],
            "sp_pipe_stats": [vp, P(u64), P(u64), P(u64)],
            "sp_pipe_compute": [vp, u64],
            "sp_pipe_compute_stats": [vp, P(u64), P(u64), P(u64)],
            "sp_pipe_issuer_stats": [vp, P(u64), P(u64), P(u64)],
            "sp_pipe_pool_stats": [vp, P(u64), P(u64), P(u64)],
        }
        for name, args in sig.items():
            if not hasattr(lib, name):  # older A/B builds (SPPIPE_LIB); tests/test_native_engine.py checks the ABI
                continue
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        for name in ("sp_pred_destroy", "sp_pipe_destroy", "sp_val_destroy"):
            getattr(lib, name).argtypes = [vp]
            getattr(lib, name).restype = None
        for name in ("sp_pred_in_batch_count", "sp_pred_decision_count", "sp_pred_event_count", "sp_val_record_count"):
            getattr(lib, name).argtypes = [vp]
            getattr(lib, name).restype = i64
        for name in ("sp_pipe_action_count",):
            getattr(lib, name).argtypes = [vp]
            getattr(lib, name).restype = i64
        lib.sp_pipe_pending_at_iv.argtypes = [vp, u64]
        lib.sp_pipe_pending_at_iv.restype = i64
        lib.sp_val_pending_at_iv.argtypes = [vp, u64]
        lib.sp_val_pending_at_iv.restype = i64
        lib.sp_val_has_pending_range.argtypes = [vp, u64, u64]
        lib.sp_val_has_pending_range.restype = i32
        lib.sp_pipe_sent_count.argtypes = [vp, i32]
        lib.sp_pipe_sent_count.restype = i64
        for name in ("sp_pipe_record_count", "sp_pipe_record_first"):
            getattr(lib, name).argtypes = [vp]
            getattr(lib, name).restype = i64
        lib.sp_pipe_delivered_count.argtypes = [vp, i32]
        lib.sp_pipe_delivered_count.restype = i64
        for name in ("sp_pipe_send_iv", "sp_pipe_recv_iv"):
            getattr(lib, name).argtypes = [vp, i32]
            getattr(lib, name).restype = u64
        lib.sp_pipe_counter_name.argtypes = [i32]
        lib.sp_pipe_counter_name.restype = ctypes.c_char_p
        lib.sp_pipe_last_error.restype = ctypes.c_char_p
        _pipe_lib = lib
        return lib


def pipe_error() -> str:
    return load_sppipe().sp_pipe_last_error().decode(errors="replace")
