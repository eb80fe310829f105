"""ctypes binding of the C ABI in include/burst_b200.h (libburst_b200.so, in-tree).

There is no fallback: if the library is missing or cannot be loaded every
entry point raises CudaError, so a GPU run can never silently take another
path.  `paper_2403_09347_b200.build` (or `__graft_entry__.build()`) produces it.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CODE_TO_ERROR, CudaError

LIB_PATH = os.environ.get("BURST_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                        "libburst_b200.so")

DTYPE_BF16 = 0
DTYPE_F32 = 1

_c_i32, _c_i64, _c_f32, _c_p, _c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                       ctypes.c_void_p, ctypes.c_size_t)


class PosMap(ctypes.Structure):
    """burst_posmap: global position of local row i (two monotone segments)."""
    _fields_ = [("pos0", _c_i64), ("pos1", _c_i64), ("seg_len", _c_i64)]


class Hop(ctypes.Structure):
    """burst_hop: one (pinned query block x visiting key block) rectangle."""
    _fields_ = [("batch", _c_i32), ("heads", _c_i32), ("head_dim", _c_i32), ("dtype", _c_i32),
                ("n_q", _c_i64), ("n_k", _c_i64),
                ("q_begin", _c_i64), ("q_len", _c_i64), ("k_begin", _c_i64), ("k_len", _c_i64),
                ("softmax_scale", _c_f32), ("causal", _c_i32),
                ("q_map", PosMap), ("k_map", PosMap),
                ("grid_skip", _c_p), ("grid_nqb", _c_i32), ("grid_nkb", _c_i32),
                ("grid_qcell", _c_i64), ("grid_kcell", _c_i64), ("flags", _c_p),
                ("dq_order", _c_p), ("key_order", _c_p)]


class IpcOp(ctypes.Structure):
    """burst_ipc_op: one send or receive of an IPC-ring exchange (with its region tag)."""
    _fields_ = [("buf", _c_p), ("bytes", _c_sz), ("peer", _c_i32), ("is_send", _c_i32),
                ("tag", _c_i32), ("pad_", _c_i32)]


class P2POp(ctypes.Structure):
    """burst_p2p: one send or receive of a grouped ring exchange."""
    _fields_ = [("buf", _c_p), ("bytes", _c_sz), ("peer", _c_i32), ("is_send", _c_i32)]


_SIGS = {
    "burst_version": ([], _c_i32),
    "burst_last_error": ([], ctypes.c_char_p),
    "burst_workspace_floats": ([_c_i32, _c_i32, _c_i32, _c_i64], _c_sz),
    "burst_lao_fwd": ([ctypes.POINTER(Hop), _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                       _c_i32, _c_i32, _c_p], _c_i32),
    "burst_fwd_finalize": ([_c_i32, _c_i32, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                            _c_p, _c_p], _c_i32),
    "burst_bwd_preprocess": ([_c_i32, _c_i32, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p,
                              _c_p, _c_p], _c_i32),
    "burst_lao_bwd": ([ctypes.POINTER(Hop), _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                       _c_i32, _c_p], _c_i32),
    "burst_bwd_finalize": ([_c_i32, _c_i32, _c_i32, _c_i32, _c_i64, _c_p,
                            ctypes.POINTER(_c_p), ctypes.POINTER(_c_p), _c_i32, _c_p, _c_p, _c_p,
                            _c_p, _c_p], _c_i32),
    "burst_tl_sum": ([_c_i32, _c_i32, _c_i32, _c_i32, _c_i64, ctypes.POINTER(_c_p), _c_i32, _c_p,
                      _c_p, _c_p], _c_i32),
    "burst_tl_accumulate": ([_c_i32, _c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p], _c_i32),
    "burst_read_flags": ([_c_p, ctypes.POINTER(_c_i32)], _c_i32),
    "burst_ipc_handle_bytes": ([], _c_sz),
    "burst_ipc_alloc": ([_c_sz, ctypes.POINTER(_c_p)], _c_i32),
    "burst_ipc_free": ([_c_p], _c_i32),
    "burst_ipc_mem_handle": ([_c_p, _c_p], _c_i32),
    "burst_ipc_open_mem": ([_c_p, ctypes.POINTER(_c_p)], _c_i32),
    "burst_ipc_close_mem": ([_c_p], _c_i32),
    "burst_ipc_event_create": ([ctypes.POINTER(_c_p), _c_p], _c_i32),
    "burst_ipc_event_open": ([_c_p, ctypes.POINTER(_c_p)], _c_i32),
    "burst_signal_u32": ([_c_p, _c_p, _c_p, ctypes.c_uint32], _c_i32),
    "burst_wait_u32": ([_c_p, _c_p, ctypes.c_uint32], _c_i32),
    "burst_ipc_ring_create": ([_c_i32, _c_i32, _c_p, _c_p, ctypes.POINTER(_c_p)], _c_i32),
    "burst_ipc_ring_set_peer": ([_c_p, _c_i32, _c_p, _c_p], _c_i32),
    "burst_ipc_ring_set_mailbox": ([_c_p, _c_p, _c_sz, ctypes.POINTER(ctypes.c_uint64)], _c_i32),
    "burst_ipc_ring_exchange": ([_c_p, _c_p, _c_i32, _c_p], _c_i32),
    "burst_ipc_ring_destroy": ([_c_p], _c_i32),
    "burst_event_record": ([_c_p, _c_p], _c_i32),
    "burst_stream_wait_event": ([_c_p, _c_p], _c_i32),
    "burst_event_destroy": ([_c_p], _c_i32),
    "burst_copy_async": ([_c_p, _c_p, _c_sz, _c_p], _c_i32),
    "burst_ring_unique_id": ([_c_p], _c_i32),
    "burst_ring_create": ([_c_p, _c_i32, _c_i32, _c_i32, ctypes.c_double, ctypes.POINTER(_c_p)],
                          _c_i32),
    "burst_ring_poll": ([_c_p, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)],
                        _c_i32),
    "burst_ring_wait": ([_c_p], _c_i32),
    "burst_ring_exchange": ([_c_p, _c_p, _c_p, _c_sz, _c_i32, _c_i32, _c_p], _c_i32),
    "burst_ring_sendrecv": ([_c_p, ctypes.POINTER(P2POp), _c_i32, _c_p], _c_i32),
    "burst_ring_destroy": ([_c_p], _c_i32),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load libburst_b200.so (raises CudaError when absent: no fallback path)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise CudaError(f"{path} is missing: build it with `python -m "
                            "paper_2403_09347_b200.build` (no CPU fallback exists)")
        try:
            lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
        except OSError as e:
            raise CudaError(f"cannot load {path}: {e}") from e
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Raise the reference-taxonomy exception for a non-zero BURST_E_* code."""
    if rc != 0:
        msg = load().burst_last_error().decode(errors="replace")
        raise CODE_TO_ERROR.get(rc, CudaError)(msg or f"burst error {rc}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
