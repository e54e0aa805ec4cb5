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
OUT = {"upper": 0, "full": 1, "upper_centered": 2, "full_centered": 3, "packed_tri": 4, "packed_tiles": 5}

# exported symbols declared in include/rf.h
SYMBOLS = ("rf_last_error", "rf_version", "rf_device_supported", "rf_moments", "rf_tau_workspace_size",
           "rf_estimate_tau", "rf_gram_workspace_size", "rf_gram", "rf_phi_workspace_size",
           "rf_phi_closed_form", "rf_phi_row_split", "rf_last_launch_count", "rf_profile_enable",
           "rf_profile_read", "rf_debug_gemm_workspace_size", "rf_debug_gemm_nt", "rf_trf_thresholds",
           "rf_trf_thresholds_for", "rf_ter_features", "rf_gram_ter_workspace_size", "rf_gram_ter",
           "rf_ktilde_workspace_size", "rf_ktilde", "rf_phi_eq2", "rf_packed_tri_elems", "rf_ridge_workspace_size",
           "rf_ridge", "rf_round_bf16", "rf_ctx_create", "rf_ctx_destroy", "rf_ctx_set_option", "rf_ctx_get_option",
           "rf_tile_map", "rf_nccl_get_unique_id", "rf_ctx_init_nccl", "rf_ctx_attach_nccl", "rf_ctx_attach_peers",
           "rf_ctx_peer_handle", "rf_ctx_open_peers", "rf_ctx_peer_base", "rf_ctx_connect_peers", "rf_ctx_collective",
           "rf_workspace_size", "rf_act_leaky_relu", "rf_act_quadratic", "rf_profile_timeline")

RF_PACK_TILE = 256
RF_MAX_PEERS = 16
OPT = {"k3_hybrid": 0, "k4_hybrid": 1, "k4_cl8": 2, "k4_split_r100": 3, "k3_split_r100": 4, "lock_w": 5, "lock_ks": 6,
       "k5_wide": 7, "eq1_general": 8, "kchunk": 9, "max_sms": 10, "comm_sms": 11, "verbose": 12, "g5_phases": 13, "k4_dynamic": 14, "k5_ares": 15, "k5_dynamic": 16, "g5_pipe": 17}


class rf_moments_t(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_double), ("kd", (ctypes.c_double * 3) * 5), ("e_sigma_sq", ctypes.c_double),
                ("d0", ctypes.c_double), ("d1", ctypes.c_double), ("d2", ctypes.c_double),
                ("nodes", ctypes.c_int32), ("method", ctypes.c_int32), ("quad_err_est", ctypes.c_double)]


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
    u8p = ctypes.c_char_p
    lib.rf_moments.argtypes = [ctypes.c_int, dbl, i32, ctypes.POINTER(rf_moments_t)]
    lib.rf_tau_workspace_size.argtypes = [i64, ctypes.POINTER(sz)]
    lib.rf_estimate_tau.argtypes = [vp, vp, ctypes.c_int, i64, i64, i64, ctypes.POINTER(dbl), vp, sz, vp]
    lib.rf_gram_workspace_size.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_gram.argtypes = [vp, vp, i64, vp, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, i64,
                            vp, sz, vp]
    lib.rf_packed_tri_elems.argtypes = [i64, ctypes.POINTER(i64)]
    lib.rf_ridge_workspace_size.argtypes = [i64, ctypes.POINTER(sz)]
    lib.rf_ridge.argtypes = [vp, vp, i64, i64, i64, ctypes.POINTER(dbl), i32, vp, i64, i32, vp, vp, vp, sz, vp]
    lib.rf_phi_workspace_size.argtypes = [i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_phi_closed_form.argtypes = [vp, vp, i64, i64, i64, ctypes.c_int, dbl, ctypes.POINTER(rf_moments_t),
                                       ctypes.c_int, ctypes.c_int, i64, i64, vp, i64, vp, sz, vp]
    lib.rf_phi_eq2.argtypes = lib.rf_phi_closed_form.argtypes
    lib.rf_phi_row_split.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.rf_last_launch_count.restype = i32
    lib.rf_profile_enable.argtypes = [ctypes.c_int]
    lib.rf_debug_gemm_workspace_size.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_debug_gemm_nt.argtypes = [vp, vp, i64, vp, i64, i64, i64, i64, ctypes.c_int, i32, vp, i64, vp, sz, vp]
    lib.rf_profile_read.argtypes = [i32, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
    lib.rf_profile_timeline.argtypes = [i32, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float),
                                        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
    lib.rf_trf_thresholds.argtypes = [dbl, dbl, dbl, i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
    lib.rf_trf_thresholds_for.argtypes = [ctypes.c_int, dbl, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
    lib.rf_ter_features.argtypes = [vp, vp, i64, vp, i64, i64, i64, i64, dbl, dbl, dbl, vp, i64, vp]
    lib.rf_gram_ter_workspace_size.argtypes = [i64, i64, i64, ctypes.POINTER(sz)]
    lib.rf_gram_ter.argtypes = [vp, vp, i64, vp, i64, i64, i64, i64, i64, dbl, dbl, dbl, ctypes.c_int, vp, i64, vp, sz,
                                vp]
    lib.rf_ktilde_workspace_size.argtypes = [i64, i64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_ktilde.argtypes = [vp, vp, i64, i64, i64, vp, i64, i32, ctypes.POINTER(dbl), dbl, dbl, dbl, ctypes.c_int,
                              ctypes.c_int, vp, i64, vp, sz, vp]
    lib.rf_round_bf16.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp]
    lib.rf_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    lib.rf_ctx_destroy.argtypes = [vp]
    lib.rf_ctx_destroy.restype = None
    lib.rf_ctx_set_option.argtypes = [vp, ctypes.c_int, i64]
    lib.rf_ctx_get_option.argtypes = [vp, ctypes.c_int, ctypes.POINTER(i64)]
    lib.rf_tile_map.argtypes = [i64, i32, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.rf_nccl_get_unique_id.argtypes = [u8p]
    lib.rf_ctx_init_nccl.argtypes = [vp, u8p, i32, i32]
    lib.rf_ctx_attach_nccl.argtypes = [vp, vp, i32, i32]
    lib.rf_ctx_attach_peers.argtypes = [vp, i32, i32, i64]
    lib.rf_ctx_peer_handle.argtypes = [vp, u8p]
    lib.rf_ctx_open_peers.argtypes = [vp, u8p]
    lib.rf_ctx_peer_base.argtypes = [vp, ctypes.POINTER(vp)]
    lib.rf_ctx_connect_peers.argtypes = [vp, ctypes.POINTER(vp)]
    lib.rf_ctx_collective.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.rf_workspace_size.argtypes = [vp, i32, i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(sz)]
    lib.rf_act_leaky_relu.argtypes = [dbl, dbl, ctypes.POINTER(ctypes.c_int)]
    lib.rf_act_quadratic.argtypes = [dbl, dbl, dbl, ctypes.POINTER(ctypes.c_int)]
    for name in SYMBOLS:
        if name not in ("rf_last_error", "rf_version", "rf_device_supported", "rf_ctx_destroy", "rf_last_launch_count"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != RF_OK:
        raise RFError(status, load().rf_last_error().decode())
