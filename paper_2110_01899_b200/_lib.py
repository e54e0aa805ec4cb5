"""ctypes binding of include/rf.h — argument marshalling only.

Every step of the path runs in librf_b200.so (sm_100a kernels).  PyTorch is used only to own device
memory and streams.  There is no fallback: if the shared library is missing or the device is not
sm_100 the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RF_B200_LIB") or os.path.join(_HERE, "librf_b200.so")   # env: A/B experiments only

RF_OK, RF_E_INVALID, RF_E_UNSUPPORTED, RF_E_NONFINITE, RF_E_CUDA, RF_E_NCCL, RF_E_WORKSPACE = range(7)
STATUS_NAMES = {0: "RF_OK", 1: "RF_E_INVALID", 2: "RF_E_UNSUPPORTED", 3: "RF_E_NONFINITE", 4: "RF_E_CUDA",
                5: "RF_E_NCCL", 6: "RF_E_WORKSPACE"}
ACT = {"tanh": 0, "erf": 1, "sigmoid_half": 2, "relu": 3, "abs": 4, "sign": 5, "step": 6, "cos": 7, "sin": 8,
       "ident": 9, "quad": 10, "bump": 11}
DT = {"f64": 0, "f32": 1, "bf16": 2}
PREC = {"fp64": 0, "fp32": 1, "3xtf32": 2, "tf32": 3, "bf16": 4}
OUT = {"upper": 0, "full": 1, "upper_centered": 2, "full_centered": 3, "packed_tri": 4}

# exported symbols declared in include/rf.h
SYMBOLS = ("rf_last_error", "rf_version", "rf_device_supported", "rf_moments", "rf_tau_workspace_size",
           "rf_estimate_tau", "rf_gram_workspace_size", "rf_gram", "rf_phi_workspace_size",
           "rf_phi_closed_form", "rf_phi_row_split", "rf_last_launch_count", "rf_profile_enable",
           "rf_profile_read", "rf_debug_gemm_workspace_size", "rf_debug_gemm_nt", "rf_pack_plan",
           "rf_pack_tile_map", "rf_gram_packed", "rf_stream_wait_chunk", "rf_trf_thresholds",
           "rf_trf_thresholds_for", "rf_ter_features", "rf_gram_ter_workspace_size", "rf_gram_ter",
           "rf_ktilde_workspace_size", "rf_ktilde", "rf_phi_eq2", "rf_gram_packed_p2p", "rf_pack_reduce",
           "rf_ipc_handle", "rf_ipc_open", "rf_ipc_close", "rf_packed_tri_elems", "rf_ridge_workspace_size",
           "rf_ridge", "rf_round_bf16")

RF_PACK_TILE = 256
RF_PACK_MAX_CHUNKS = 64


class rf_moments_t(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_double), ("kd", (ctypes.c_double * 3) * 5), ("e_sigma_sq", ctypes.c_double),
                ("d0", ctypes.c_double), ("d1", ctypes.c_double), ("d2", ctypes.c_double),
                ("nodes", ctypes.c_int32), ("method", ctypes.c_int32), ("quad_err_est", ctypes.c_double)]


class rf_pack_plan_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("world", ctypes.c_int32), ("nchunks", ctypes.c_int32),
                ("prec", ctypes.c_int32), ("tiles_per_pair", ctypes.c_int32), ("pair_tiles", ctypes.c_int64),
                ("send_elems", ctypes.c_int64), ("recv_elems", ctypes.c_int64),
                ("chunk_tile0", ctypes.c_int64 * (RF_PACK_MAX_CHUNKS + 1)),
                ("chunk_slots", ctypes.c_int64 * RF_PACK_MAX_CHUNKS),
                ("chunk_send_off", ctypes.c_int64 * (RF_PACK_MAX_CHUNKS + 1)),
                ("chunk_recv_off", ctypes.c_int64 * (RF_PACK_MAX_CHUNKS + 1))]


class RFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    i64, i32, dbl, vp, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t
    lib.rf_last_error.restype = ctypes.c_char_p
    lib.rf_version.restype = ctypes.c_char_p
    lib.rf_device_supported.argtypes = [ctypes.c_int]
    lib.rf_device_supported.restype = ctypes.c_int
    lib.rf_moments.argtypes = [ctypes.c_int, dbl, i32, ctypes.POINTER(rf_moments_t)]
    lib.rf_tau_workspace_size.argtypes = [i64, ctypes.POINTER(sz)]
    lib.rf_estimate_tau.argtypes = [vp, ctypes.c_int, i64, i64, i64, ctypes.POINTER(dbl), vp, sz, vp]
    lib.rf_gram_workspace_size.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_gram.argtypes = [vp, i64, vp, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, i64,
                            vp, sz, vp]
    lib.rf_packed_tri_elems.argtypes = [i64, ctypes.POINTER(i64)]
    lib.rf_ridge_workspace_size.argtypes = [i64, ctypes.POINTER(sz)]
    lib.rf_ridge.argtypes = [vp, i64, i64, i64, ctypes.POINTER(dbl), i32, vp, i64, i32, vp, vp, vp, sz, vp]
    lib.rf_phi_workspace_size.argtypes = [i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_phi_closed_form.argtypes = [vp, i64, i64, i64, ctypes.c_int, dbl, ctypes.POINTER(rf_moments_t),
                                       ctypes.c_int, ctypes.c_int, i64, i64, vp, i64, vp, sz, vp]
    lib.rf_phi_eq2.argtypes = [vp, i64, i64, i64, ctypes.c_int, dbl, ctypes.POINTER(rf_moments_t),
                               ctypes.c_int, ctypes.c_int, i64, i64, vp, i64, vp, sz, vp]
    lib.rf_phi_row_split.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.rf_last_launch_count.restype = i32
    lib.rf_profile_enable.argtypes = [ctypes.c_int]
    lib.rf_debug_gemm_workspace_size.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_debug_gemm_nt.argtypes = [vp, i64, vp, i64, i64, i64, i64, ctypes.c_int, i32, vp, i64, vp, sz, vp]
    lib.rf_profile_read.argtypes = [i32, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
    PP = ctypes.POINTER(rf_pack_plan_t)
    lib.rf_pack_plan.argtypes = [i64, i32, i32, ctypes.c_int, PP]
    lib.rf_pack_tile_map.argtypes = [PP, i32, ctypes.POINTER(i32)]
    lib.rf_gram_packed.argtypes = [vp, i64, vp, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int, PP, i32, vp, vp,
                                   ctypes.c_uint32, vp, sz, vp]
    lib.rf_stream_wait_chunk.argtypes = [PP, vp, i32, ctypes.c_uint32, vp]
    lib.rf_trf_thresholds.argtypes = [dbl, dbl, dbl, i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
    lib.rf_trf_thresholds_for.argtypes = [ctypes.c_int, dbl, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
    lib.rf_ter_features.argtypes = [vp, i64, vp, i64, i64, i64, i64, dbl, dbl, dbl, vp, i64, vp]
    lib.rf_gram_ter_workspace_size.argtypes = [i64, i64, i64, ctypes.POINTER(sz)]
    lib.rf_gram_ter.argtypes = [vp, i64, vp, i64, i64, i64, i64, i64, dbl, dbl, dbl, ctypes.c_int, vp, i64, vp, sz, vp]
    lib.rf_ktilde_workspace_size.argtypes = [i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_ktilde.argtypes = [vp, i64, i64, i64, vp, i64, i32, ctypes.POINTER(dbl), dbl, dbl, dbl, ctypes.c_int,
                              ctypes.c_int, vp, i64, vp, sz, vp]
    lib.rf_gram_packed_p2p.argtypes = [vp, i64, vp, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int, PP, i32,
                                       ctypes.POINTER(vp), i32, vp, sz, vp]
    lib.rf_pack_reduce.argtypes = [PP, vp, vp, vp]
    lib.rf_round_bf16.argtypes = [vp, i64, i64, i64, vp, i64, vp]
    lib.rf_ipc_handle.argtypes = [vp, ctypes.c_char_p]
    lib.rf_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    lib.rf_ipc_close.argtypes = [vp]
    for name in ("rf_gram_packed_p2p", "rf_pack_reduce", "rf_ipc_handle", "rf_ipc_open", "rf_ipc_close", "rf_phi_eq2", "rf_ktilde_workspace_size", "rf_ktilde", "rf_trf_thresholds", "rf_trf_thresholds_for", "rf_ter_features", "rf_gram_ter_workspace_size",
                 "rf_gram_ter", "rf_pack_plan", "rf_pack_tile_map", "rf_gram_packed", "rf_stream_wait_chunk",
                 "rf_moments", "rf_tau_workspace_size", "rf_estimate_tau", "rf_gram_workspace_size", "rf_gram",
                 "rf_phi_workspace_size", "rf_phi_closed_form", "rf_phi_row_split", "rf_profile_enable",
                 "rf_profile_read", "rf_debug_gemm_workspace_size", "rf_debug_gemm_nt"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != RF_OK:
        raise RFError(status, load().rf_last_error().decode())
