"""ctypes declaration of libdaso.so (include/daso.h).  Argument marshalling only.

The library must exist (built by ``python -m paper_2104_05588_b200.build`` or
``__graft_entry__.build()``); there is no fallback of any kind — a missing or
unloadable library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdaso.so")

# status codes (daso.h)
OK, ERR_CONFIG, ERR_RANGE, ERR_PROTOCOL, ERR_ARGUMENT, ERR_CUDA, ERR_NCCL, ERR_NONFINITE = range(8)
WARMUP, CYCLING, COOLDOWN = 0, 1, 2
WIRE_BF16, WIRE_FP32 = 0, 1
MODE_FAITHFUL, MODE_SHARDED, MODE_FUSED = 0, 1, 2
STEP_GRADS_REDUCED = 1
EXCH_NCCL, EXCH_CE = 0, 1


class SchedConfig(C.Structure):
    _fields_ = [("B_init", C.c_int32), ("S_init", C.c_int32), ("warmup_epochs", C.c_int32),
                ("cooldown_epochs", C.c_int32), ("total_epochs", C.c_int32),
                ("steps_per_epoch", C.c_int32), ("gpus_per_node", C.c_int32)]


RECORD_FIELDS = ["step", "epoch", "phase", "B", "S", "batch_in_cycle", "plateau_action", "send",
                 "blocking", "send_group", "n_syncs", "merge", "merge_S", "merge_group", "merge_sent",
                 "pending", "due"]


class Record(C.Structure):
    _fields_ = [(f, C.c_int64) for f in RECORD_FIELDS]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f in RECORD_FIELDS}


class Config(C.Structure):
    _fields_ = [("rank", C.c_int32), ("warmup_epochs", C.c_int32), ("cooldown_epochs", C.c_int32),
                ("total_epochs", C.c_int32), ("steps_per_epoch", C.c_int32), ("momentum", C.c_float),
                ("weight_decay", C.c_float), ("wire", C.c_int32), ("mode", C.c_int32),
                ("check_finite", C.c_int32), ("nccl_max_ctas", C.c_int32), ("exchange", C.c_int32)]


TRACE_FIELDS = [("steps", C.c_int64), ("kernel_launches", C.c_int64), ("kernel_ms", C.c_double),
                ("kernel_bytes", C.c_double), ("local_ops", C.c_int64), ("local_ms", C.c_double),
                ("local_bytes", C.c_double), ("node_ops", C.c_int64), ("node_ms", C.c_double),
                ("node_bytes", C.c_double), ("wait_ops", C.c_int64), ("wait_ms", C.c_double),
                ("exch_ops", C.c_int64), ("exch_ms", C.c_double), ("exch_bytes", C.c_double),
                ("kernel_nvl_bytes", C.c_double)]


class Trace(C.Structure):
    _fields_ = TRACE_FIELDS

    def as_dict(self) -> dict:
        return {f: (float(getattr(self, f)) if t is C.c_double else int(getattr(self, f))) for f, t in TRACE_FIELDS}


class DasoError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str = ""):
        self.status = status
        super().__init__(f"{where}: status {status} ({_status_string(status)}){': ' + msg if msg else ''}")


_lib = None
_SIG = {
    "daso_status_string": (C.c_char_p, [C.c_int]),
    "daso_version": (C.c_char_p, []),
    "daso_padded_numel": (C.c_size_t, [C.c_size_t, C.c_int]),
    "daso_sched_create": (C.c_int, [C.POINTER(SchedConfig), C.POINTER(C.c_void_p)]),
    "daso_sched_next": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Record)]),
    "daso_sched_destroy": (C.c_int, [C.c_void_p]),
    "daso_get_unique_id": (C.c_int, [C.c_void_p]),
    "daso_plateau_create": (C.c_int, [C.c_int, C.c_double, C.POINTER(C.c_void_p)]),
    "daso_plateau_update": (C.c_int, [C.c_void_p, C.c_double, C.POINTER(C.c_int)]),
    "daso_plateau_destroy": (C.c_int, [C.c_void_p]),
    "daso_lr_at": (C.c_int, [C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                             C.POINTER(C.c_double)]),
    "daso_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Config),
                            C.c_void_p]),
    "daso_bind": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "daso_alloc_bind": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_void_p)]),
    "daso_local_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "daso_local_update": (C.c_int, [C.c_void_p, C.c_float, C.c_void_p]),
    "daso_global_send": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "daso_global_merge": (C.c_int, [C.c_void_p, C.c_void_p]),
    "daso_step": (C.c_int, [C.c_void_p, C.c_float, C.c_int, C.c_void_p, C.POINTER(Record)]),
    "daso_step_ex": (C.c_int, [C.c_void_p, C.c_float, C.c_int, C.c_int, C.c_void_p, C.POINTER(Record)]),
    "daso_local_sync_bucket": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p]),
    "daso_step_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_float, C.c_int, C.c_void_p, C.POINTER(Record),
                                 C.POINTER(C.c_uint32)]),
    "daso_query": (C.c_int, [C.c_void_p, C.POINTER(Record)]),
    "daso_trace_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "daso_trace_read": (C.c_int, [C.c_void_p, C.POINTER(Trace), C.c_int]),
    "daso_check_finite": (C.c_int, [C.c_void_p, C.c_void_p]),
    "daso_finalize": (C.c_int, [C.c_void_p]),
    "daso_last_error": (C.c_char_p, [C.c_void_p]),
    "daso_topology": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]),
    "daso_k_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_float, C.c_float, C.c_float,
                                C.c_float, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "daso_k_update_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_float, C.c_float,
                                      C.c_float, C.c_float, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                      C.c_int, C.c_void_p, C.c_void_p]),
    "daso_k_merge": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                               C.c_int, C.c_void_p, C.c_void_p]),
    "daso_k_average": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                 C.c_void_p]),
    "daso_k_pack": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_int, C.c_void_p]),
    "daso_flat_layout": (C.c_int, [C.POINTER(C.c_size_t), C.c_int, C.c_size_t, C.POINTER(C.c_size_t),
                                   C.POINTER(C.c_size_t)]),
    "daso_k_gather": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.c_int,
                                C.c_void_p, C.c_void_p]),
    "daso_k_scatter": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                 C.c_int, C.c_void_p]),
    "daso_k_checksum": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "daso_kernel_impl": (C.c_int, [C.c_int]),
    "daso_set_exchange": (C.c_int, [C.c_void_p, C.c_int]),
    "daso_exchange_alone": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    "daso_vcluster_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Config),
                                       C.c_size_t]),
    "daso_vcluster_buffers": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_void_p)]),
    "daso_vcluster_rank": (C.c_void_p, [C.c_void_p, C.c_int]),
    "daso_vcluster_step": (C.c_int, [C.c_void_p, C.c_float, C.c_int, C.c_void_p, C.POINTER(Record)]),
    "daso_vcluster_destroy": (C.c_int, [C.c_void_p]),
    "daso_vcluster_last_error": (C.c_char_p, [C.c_void_p]),
}
EXPORTED = sorted(_SIG)


def lib() -> C.CDLL:
    """Load libdaso.so (once).  Raises if it is missing: no fallback path exists."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2104_05588_b200.build` "
                              "(there is no CPU / PyTorch fallback)")
        try:
            import torch  # noqa: F401  (load torch's libnccl.so.2 / CUDA first: one NCCL per process)
        except Exception:
            pass
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIG.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _status_string(s: int) -> str:
    try:
        return lib().daso_status_string(s).decode()
    except Exception:
        return "?"


def check(status: int, where: str, ctx=None) -> None:
    if status != OK:
        msg = ""
        if ctx is not None:
            m = lib().daso_last_error(ctx)
            msg = m.decode() if m else ""
        raise DasoError(status, where, msg)
