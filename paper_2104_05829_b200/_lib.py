"""ctypes binding of libnekb200.so (include/nekb200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2104_05829_b200/csrc``).  There is no fallback: if the shared object is
missing, every operator raises ``NativeLibraryError``.
"""

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnekb200.so")

NK_OK, NK_ERR_INVALID, NK_ERR_CUDA, NK_ERR_UNSUPPORTED = 0, 1, 2, 3
OP_CODES = {"+": 0, "*": 1, "min": 2, "max": 3}


class NativeLibraryError(RuntimeError):
    """libnekb200.so missing or a CUDA error inside it."""


class ContractError(ValueError):
    """Invalid arguments (SPEC's 'contract error')."""


class UnsupportedOrderError(ValueError):
    pass


class CGState(ctypes.Structure):
    _fields_ = [
        ("rz", ctypes.c_double), ("pAp", ctypes.c_double), ("rz_new", ctypes.c_double),
        ("rr", ctypes.c_double), ("zap", ctypes.c_double), ("bb", ctypes.c_double),
        ("thresh2", ctypes.c_double), ("alpha", ctypes.c_double),
        ("iter", ctypes.c_int32), ("done", ctypes.c_int32), ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32), ("max_iter", ctypes.c_int32),
        ("flexible", ctypes.c_int32), ("ticket", ctypes.c_uint32 * 4),
        ("gen", ctypes.c_uint32), ("pad_", ctypes.c_uint32),
    ]


CG_STATE_BYTES = ctypes.sizeof(CGState)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_D = ctypes.c_double

_SIGS = {
    "nk_version": ([], _I32),
    "nk_last_error": ([], ctypes.c_char_p),
    "nk_order_range": ([_P, _P], _I32),
    "nk_device_info": ([_P, _P, _P, _P], _I32),
    "nk_l2_flush": ([_P, _I64, _P], _I32),
    "nk_bw_probe": ([_I64, _I32, _P, _P, _P, _I32, _P], _I32),
    "nk_box_coords": ([_I32, _I64, _P, _P, _P, _P, _I32, _D, _P, _P, _P], _I32),
    "nk_geom_factors": ([_I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_box_ids": ([_I32, _I64, _P, _P, _P, _P, _P], _I32),
    "nk_box_mask": ([_I32, _I64, _P, _P, _P, _P, _P], _I32),
    "nk_bk5": ([_I32, _I64, _P, _P, _P, _P, _D, _P, _D, _I32, _I64, _P, _P, _I64, _P, _P,
                _I64, _I64, _P], _I32),
    "nk_bk5_blocks": ([_I32, _I64, _I32], _I64),
    "nk_bk5_pcg": ([_I32, _I64, _P, _P, _P, _P, _D, _P, _D, _P, _P, _I64, _P, _P, _P, _P, _P,
                    _I64, _I64, _P, _P], _I32),
    "nk_bk5_pcg_blocks": ([_I32, _I64], _I64),
    "nk_bk5_pcg_gs": ([_I32, _I64, _P, _P, _P, _P, _D, _P, _D, _P, _P, _P, _P, _P, _P, _I64,
                       _P, _I32, _P, _P, _P, _P], _I32),
    "nk_bk5_pcg_gs_fused": ([_I32], _I32),
    "nk_cg_update_gs_cls": ([_I64, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_update_gs_cls_fused": ([_I64], _I32),
    "nk_bk5_set_variant": ([_I32], _I32),
    "nk_bk5_tune": ([_I32, _I32], _I32),
    "nk_set_knob": ([_I32, _I32], _I32),
    "nk_bk5_set_gate": ([_P], _I32),
    "nk_stream_write_u64": ([_P, ctypes.c_uint64, _P], _I32),
    "nk_l2_set_aside_max": ([], _I64),
    "nk_local_diag": ([_I32, _I64, _P, _P, _D, _P, _D, _P, _P], _I32),
    "nk_gs_op": ([_I64, _P, _P, _P, _I32, _I32, _I64, _P, _P], _I32),
    "nk_gs_op_classes": ([_I32, _P, _P, _P, _P, _I32, _I32, _I64, _P, _P], _I32),
    "nk_gs_op_f32": ([_I64, _P, _P, _P, _I32, _I32, _I64, _P, _P], _I32),
    "nk_gs_op_classes_f32": ([_I32, _P, _P, _P, _P, _I32, _I32, _I64, _P, _P], _I32),
    "nk_gs_plan_build": ([_P, _I64, _P, _P, _P, _P], _I32),
    "nk_gather": ([_I64, _P, _P, _P, _P, _P], _I32),
    "nk_gs_create": ([_P, _P, _I64, _I64, _P], _I32),
    "nk_gs_apply": ([_P, _P, _I32, _I32, _I64, _P, _P], _I32),
    "nk_gs_destroy": ([_P], _I32),
    "nk_halo_combine": ([_I64, _P, _P, _P, _P, _P, _P, _I32, _P, _P], _I32),
    "nk_ipc_handle_size": ([], _I32),
    "nk_ipc_alloc": ([_I64, _P, _P], _I32),
    "nk_ipc_free": ([_P], _I32),
    "nk_ipc_open": ([_P, _P], _I32),
    "nk_ipc_close": ([_P], _I32),
    "nk_halo_push": ([_I32, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P], _I32),
    "nk_halo_combine_wait": ([_I64, _P, _P, _P, _I64, _I64, _P, _P, _P, _I32, _P, _I32, _P, _P,
                              _P], _I32),
    "nk_board_allreduce": ([_I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_partials_len": ([_I64], _I64),
    "nk_cg_init": ([_I64, _P, _P, _P, _P, _P, _P, _P, _P, _D, _I32, _I32, _P], _I32),
    "nk_cg_init_finalize": ([_P, _P, _P], _I32),
    "nk_cg_update": ([_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_update_gs": ([_I64, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_pupdate": ([_I64, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_xpstep": ([_I64, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_wdot": ([_I64, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_gate": ([_P, _P, _P], _I32),
    "nk_interp3": ([_I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _I32, _P, _P], _I32),
    "nk_cheb_step": ([_I64, _P, _P, _P, _P, _P, _P, _D, _D, _I32, _P, _P], _I32),
    "nk_dense_matvec": ([_I64, _P, _P, _P, _P, _P], _I32),
    "nk_dense_matvec32": ([_I64, _I64, _P, _P, _P, _P, _P], _I32),
    "nk_multi_wdot_partials_len": ([], _I64),
    "nk_multi_wdot": ([_I64, _I32, _P, _I64, _P, _P, _P, _P, _P], _I32),
    "nk_multi_axpy": ([_I64, _I32, _P, _D, _P, _I64, _P, _P, _P], _I32),
    "nk_vscale": ([_I64, _P, _P, _P, _P], _I32),
    "nk_pointwise": ([_I64, _P, _P, _P, _D, _P, _P], _I32),
    "nk_bk5_batch": ([_I32, _I64, _P, _P, _P, _P, _D, _P, _D, _I32, _I64, _P, _P, _I64, _P, _P,
                      _I64, _I64, _I64, _P], _I32),
    "nk_bk5_batch_variant": ([_I32], _I32),
    "nk_bk5_batch_blocks": ([_I32, _I64], _I64),
    "nk_cg_update_gs_batch": ([_I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_update_gs_seg": ([_I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "nk_cg_xpstep_batch": ([_I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _I64, _P], _I32),
    "nk_fdm": ([_I32, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _D, _P, _I32, _P, _P], _I32),
    "nk_fdm32": ([_I32, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _D, _P, _I32, _P, _P], _I32),
    "nk_gather_diff": ([_I64, _P, _P, _P, _P, _P, _P], _I32),
    "nk_schwarz_post": ([_I32, _I64, _P, _I32, _P, _P, _P, _P, _D, _D, _I32, _P, _P], _I32),
}

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library (loads on first use; raises if not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (there is no CPU fallback)")
            import torch  # noqa: F401  (load torch's CUDA runtime / NCCL first)
            L = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc, what=""):
    if rc == NK_OK:
        return
    msg = lib().nk_last_error().decode(errors="replace")
    if rc == NK_ERR_INVALID:
        raise ContractError(f"contract error in {what}: {msg}")
    if rc == NK_ERR_UNSUPPORTED:
        raise UnsupportedOrderError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what}: {msg}")


def ptr(t):
    """Device/host pointer of a tensor or ndarray (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
