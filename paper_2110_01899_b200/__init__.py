"""B200-native random-features Gram G and closed-form kernel Φ (arXiv 2110.01899).

Python face of the C ABI in include/rf.h (same names).  The functions below only marshal arguments: they allocate
outputs/workspace with torch when the caller does not pass them (on the stream the work is enqueued on, so the
caching allocator orders reuse after it), pass raw device pointers and the stream, and raise on any non-OK status.
All arithmetic runs in librf_b200.so.  Every compute call takes `ctx` (a Context, or None = the thread's default
context of the current device).
"""
from __future__ import annotations

import contextlib
import ctypes
from typing import Dict, Optional, Sequence, Tuple

from . import _lib
from ._lib import ACT, OPT, OUT, PREC, RF_MAX_PEERS, RF_PACK_TILE, RFError, load, rf_moments_t  # noqa: F401

__all__ = ["Context", "rf_moments", "rf_estimate_tau", "rf_gram", "rf_phi_closed_form", "rf_phi_row_split",
           "rf_gram_workspace_size", "rf_phi_workspace_size", "rf_workspace_size", "rf_version", "rf_device_supported",
           "rf_last_launch_count", "rf_tile_map", "rf_trf_thresholds", "rf_trf_thresholds_for", "rf_ter_features",
           "rf_gram_ter", "rf_gram_ter_workspace_size", "rf_ktilde", "rf_ktilde_workspace_size", "rf_packed_tri_elems",
           "rf_ridge", "rf_ridge_workspace_size", "rf_round_bf16", "rf_nccl_get_unique_id", "rf_act_leaky_relu",
           "rf_act_quadratic", "RFError", "PREC", "ACT",
           "OPT"]


def _torch():
    import torch
    return torch


def _dtype_for(prec: str):
    torch = _torch()
    return {"fp64": torch.float64, "fp32": torch.float32, "3xtf32": torch.float32, "tf32": torch.float32,
            "bf16": torch.bfloat16}[prec]


def _out_dtype(prec: str):
    torch = _torch()
    return torch.float64 if prec == "fp64" else torch.float32


def _stream_ptr(stream) -> ctypes.c_void_p:
    torch = _torch()
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _on(stream):
    """Allocate on the stream the call enqueues on (include/rf.h: all GPU work goes to `stream`)."""
    return _torch().cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _cp(ctx) -> Optional[ctypes.c_void_p]:
    return None if ctx is None else ctx._handle()


def _check_tensor(name, t, dtype):
    if not t.is_cuda:
        raise RFError(_lib.RF_E_INVALID, f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise RFError(_lib.RF_E_INVALID, f"{name} has dtype {t.dtype}, precision mode needs {dtype}")
    if t.dim() != 2 or (t.stride(1) != 1 and t.shape[1] > 1):
        raise RFError(_lib.RF_E_INVALID, f"{name} must be 2-D with unit column stride")


# ------------------------------------------------------------------------------------------ context
class Context:
    """rf_ctx (include/rf.h): a device, tuning options, and (optionally) a G5 collective.

        ctx = Context(device=0)
        ctx.set_option("k4_hybrid", 0)
        ctx.attach_peers(rank, world, n_max); ctx.open_peers(handles)        # or ctx.init_nccl(id, rank, world)
        rf_gram(X, W_local, out="packed_tiles", G=recv, ctx=ctx, m_total=m)  # collective
    """

    def __init__(self, device: int = 0):
        p = ctypes.c_void_p()
        _lib.check(load().rf_ctx_create(int(device), ctypes.byref(p)))
        self._p = p
        self.device = int(device)

    def _handle(self) -> ctypes.c_void_p:
        if self._p is None:
            raise RFError(_lib.RF_E_INVALID, "context was destroyed")
        return self._p

    def destroy(self) -> None:
        if getattr(self, "_p", None) is not None:
            load().rf_ctx_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def set_option(self, name: str, value: int) -> None:
        _lib.check(load().rf_ctx_set_option(self._handle(), OPT[name], int(value)))

    def get_option(self, name: str) -> int:
        v = ctypes.c_int64()
        _lib.check(load().rf_ctx_get_option(self._handle(), OPT[name], ctypes.byref(v)))
        return v.value

    @contextlib.contextmanager
    def options(self, **kv):
        """Temporarily set options (A/B measurement, bit-exactness tests of the alternative kernels)."""
        old = {k: self.get_option(k) for k in kv}
        for k, v in kv.items():
            self.set_option(k, v)
        try:
            yield self
        finally:
            for k, v in old.items():
                self.set_option(k, v)

    # ---- G5 collective
    def init_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        _lib.check(load().rf_ctx_init_nccl(self._handle(), bytes(unique_id), int(rank), int(world)))

    def attach_nccl(self, comm_ptr: int, rank: int, world: int) -> None:
        _lib.check(load().rf_ctx_attach_nccl(self._handle(), ctypes.c_void_p(int(comm_ptr)), int(rank), int(world)))

    def attach_peers(self, rank: int, world: int, n_max: int) -> None:
        _lib.check(load().rf_ctx_attach_peers(self._handle(), int(rank), int(world), int(n_max)))

    def peer_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _lib.check(load().rf_ctx_peer_handle(self._handle(), buf))
        return buf.raw

    def open_peers(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(bytes(h).ljust(64, b"\0")[:64] for h in handles)
        _lib.check(load().rf_ctx_open_peers(self._handle(), blob))

    def peer_base(self) -> int:
        p = ctypes.c_void_p()
        _lib.check(load().rf_ctx_peer_base(self._handle(), ctypes.byref(p)))
        return int(p.value)

    def connect_peers(self, bases: Sequence[int]) -> None:
        arr = (ctypes.c_void_p * len(bases))(*[ctypes.c_void_p(int(b)) for b in bases])
        _lib.check(load().rf_ctx_connect_peers(self._handle(), arr))

    def collective(self) -> Tuple[int, int, int]:
        """(rank, world, mode) with mode 0 none, 1 NCCL, 2 peers."""
        r, w, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _lib.check(load().rf_ctx_collective(self._handle(), ctypes.byref(r), ctypes.byref(w), ctypes.byref(m)))
        return r.value, w.value, m.value


def rf_act_leaky_relu(a_plus: float, a_minus: float) -> str:
    """Register Table 2's a₊·max(0, t) + a₋·max(0, −t) (include/rf.h) and return its activation name
    "leaky_relu(a₊,a₋)", usable as `act=` everywhere (the oracle reads the same name)."""
    v = ctypes.c_int()
    _lib.check(load().rf_act_leaky_relu(float(a_plus), float(a_minus), ctypes.byref(v)))
    name = f"leaky_relu({float(a_plus)!r},{float(a_minus)!r})"
    ACT[name] = v.value
    return name


def rf_act_quadratic(a0: float, a1: float, a2: float) -> str:
    """Register Table 2's a₂t² + a₁t + a₀ (include/rf.h) and return its name "quadratic(a₀,a₁,a₂)"."""
    v = ctypes.c_int()
    _lib.check(load().rf_act_quadratic(float(a0), float(a1), float(a2), ctypes.byref(v)))
    name = f"quadratic({float(a0)!r},{float(a1)!r},{float(a2)!r})"
    ACT[name] = v.value
    return name


def rf_nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _lib.check(load().rf_nccl_get_unique_id(buf))
    return buf.raw


def rf_tile_map(n: int, world: int, rank: int):
    """(I, J) of every receive slot of `rank` of the multi-GPU G (include/rf.h G5), int64 numpy (slots, 2);
    (−1, −1) marks padding slots.  Host only, a function of (n, world)."""
    import numpy as np
    cnt = ctypes.c_int64()
    _lib.check(load().rf_tile_map(int(n), RF_PACK_TILE, int(world), int(rank), ctypes.byref(cnt), None))
    ij = np.empty((max(cnt.value, 1), 2), dtype=np.int64)
    _lib.check(load().rf_tile_map(int(n), RF_PACK_TILE, int(world), int(rank), ctypes.byref(cnt),
                                  ij.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return ij[:cnt.value]


# ------------------------------------------------------------------------------------------ host / sizes
def rf_version() -> str:
    return load().rf_version().decode()


def rf_device_supported(device: int = 0) -> bool:
    return bool(load().rf_device_supported(device))


def rf_last_launch_count() -> int:
    return int(load().rf_last_launch_count())


def rf_moments(act: str, tau: float, nodes: int = 0) -> Dict[str, object]:
    lib = load()
    m = rf_moments_t()
    _lib.check(lib.rf_moments(ACT[act], float(tau), int(nodes), ctypes.byref(m)))
    kd = [[m.kd[k][d] for d in range(3)] for k in range(5)]
    return {"tau": m.tau, "kd": kd, "e_sigma_sq": m.e_sigma_sq, "d0": m.d0, "d1": m.d1, "d2": m.d2,
            "nodes": m.nodes, "method": m.method, "quad_err_est": m.quad_err_est, "_struct": m}


def rf_packed_tri_elems(n: int) -> int:
    """Floats of an out="packed_tri" buffer (include/rf.h RF_OUT_PACKED_TRI)."""
    e = ctypes.c_int64()
    _lib.check(load().rf_packed_tri_elems(int(n), ctypes.byref(e)))
    return e.value


def rf_gram_workspace_size(p: int, n: int, m_local: int, prec: str) -> int:
    need = ctypes.c_size_t()
    _lib.check(load().rf_gram_workspace_size(p, n, m_local, PREC[prec], ctypes.byref(need)))
    return need.value


def rf_phi_workspace_size(p: int, n: int, prec: str) -> int:
    need = ctypes.c_size_t()
    _lib.check(load().rf_phi_workspace_size(p, n, PREC[prec], ctypes.byref(need)))
    return need.value


def rf_workspace_size(op: str, p: int, n: int, m_local: int, prec: str, out: str = "upper", ctx=None) -> int:
    """include/rf.h rf_workspace_size: op "gram" or "phi"."""
    need = ctypes.c_size_t()
    _lib.check(load().rf_workspace_size(_cp(ctx), {"gram": 0, "phi": 1}[op], int(p), int(n), int(m_local),
                                        PREC[prec], OUT[out], ctypes.byref(need)))
    return need.value


def rf_phi_row_split(n: int, world: int, rank: int) -> Tuple[int, int]:
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(load().rf_phi_row_split(n, world, rank, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def rf_trf_thresholds(d1: float, d2: float, tau: float, sign2: int = 1) -> Tuple[float, float]:
    """(s−, s+) of σ^ter matching Theorem 1's d1, d2 at τ (Algorithm 1 step 2; include/rf.h)."""
    sm, sp = ctypes.c_double(), ctypes.c_double()
    _lib.check(load().rf_trf_thresholds(float(d1), float(d2), float(tau), int(sign2), ctypes.byref(sm),
                                        ctypes.byref(sp)))
    return sm.value, sp.value


def rf_trf_thresholds_for(act: str, tau: float) -> Tuple[float, float]:
    sm, sp = ctypes.c_double(), ctypes.c_double()
    _lib.check(load().rf_trf_thresholds_for(ACT[act], float(tau), ctypes.byref(sm), ctypes.byref(sp)))
    return sm.value, sp.value


def rf_gram_ter_workspace_size(p: int, n: int, m_local: int) -> int:
    need = ctypes.c_size_t()
    _lib.check(load().rf_gram_ter_workspace_size(p, n, m_local, ctypes.byref(need)))
    return need.value


def rf_ktilde_workspace_size(p: int, n: int, prec: str) -> int:
    need = ctypes.c_size_t()
    _lib.check(load().rf_ktilde_workspace_size(p, n, PREC[prec], ctypes.byref(need)))
    return need.value


def rf_ridge_workspace_size(n_train: int) -> int:
    need = ctypes.c_size_t()
    _lib.check(load().rf_ridge_workspace_size(int(n_train), ctypes.byref(need)))
    return need.value


def rf_profile_enable(on: bool = True) -> None:
    _lib.check(load().rf_profile_enable(1 if on else 0))


def rf_profile_read(max_records: int = 4096):
    """[(kernel name, device ms)] of the launches recorded since the last read (waits for them)."""
    lib = load()
    names = ctypes.create_string_buffer(32 * max_records)
    ms = (ctypes.c_float * max_records)()
    cnt = ctypes.c_int32()
    _lib.check(lib.rf_profile_read(max_records, names, ms, ctypes.byref(cnt)))
    k = min(cnt.value, max_records)
    raw = names.raw
    return [(raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(), float(ms[i])) for i in range(k)]


def rf_profile_timeline(max_records: int = 4096):
    """[(kernel name, start ms relative to the earliest record, device ms)] of the launches recorded since the last
    read (waits for them)."""
    lib = load()
    names = ctypes.create_string_buffer(32 * max_records)
    t0 = (ctypes.c_float * max_records)()
    ms = (ctypes.c_float * max_records)()
    cnt = ctypes.c_int32()
    _lib.check(lib.rf_profile_timeline(max_records, names, t0, ms, ctypes.byref(cnt)))
    k = min(cnt.value, max_records)
    raw = names.raw
    return [(raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(), float(t0[i]), float(ms[i])) for i in range(k)]


# ------------------------------------------------------------------------------------------ compute calls
def rf_estimate_tau(X, ws=None, stream=None, ctx=None) -> float:
    torch = _torch()
    dt = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2}[X.dtype]
    n, p = X.shape
    need = ctypes.c_size_t()
    _lib.check(load().rf_tau_workspace_size(n, ctypes.byref(need)))
    with _on(stream):
        if ws is None:
            ws = torch.empty(need.value, dtype=torch.uint8, device=X.device)
    out = ctypes.c_double()
    _lib.check(load().rf_estimate_tau(_cp(ctx), ctypes.c_void_p(X.data_ptr()), dt, X.stride(0), p, n,
                                      ctypes.byref(out), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                      _stream_ptr(stream)))
    return out.value


def rf_round_bf16(src, out=None, stream=None, ctx=None):
    """G1 for BF16 mode (include/rf.h rf_round_bf16): bf16(src) rounded to nearest even, by the library's kernel.
    src: 2-D float32 CUDA tensor with unit column stride; out: optional bf16 tensor of the same shape."""
    torch = _torch()
    _check_tensor("src", src, torch.float32)
    rows, cols = src.shape
    with _on(stream):
        if out is None:
            out = torch.empty((rows, cols), dtype=torch.bfloat16, device=src.device)
    _check_tensor("out", out, torch.bfloat16)
    if tuple(out.shape) != (rows, cols):
        raise RFError(_lib.RF_E_INVALID, f"out has shape {tuple(out.shape)}, need {(rows, cols)}")
    _lib.check(load().rf_round_bf16(_cp(ctx), ctypes.c_void_p(src.data_ptr()), src.stride(0), rows, cols,
                                    ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream_ptr(stream)))
    return out


def _alloc_out(name, buf, n, out, prec, device, zero=True):
    """Output buffer for `out`: n × n, or the 1-D packed triangle (RF_OUT_PACKED_TRI, ld ignored → 256)."""
    torch = _torch()
    if out == "packed_tri":
        if buf is None:
            buf = torch.empty(rf_packed_tri_elems(n), dtype=_out_dtype(prec), device=device)
        if not buf.is_cuda or buf.dim() != 1 or buf.dtype != _out_dtype(prec) or buf.numel() < rf_packed_tri_elems(n):
            raise RFError(_lib.RF_E_INVALID, f"{name}: packed_tri needs a 1-D CUDA tensor of rf_packed_tri_elems(n)")
        return buf, 256
    if buf is None:
        buf = (torch.zeros if zero else torch.empty)((n, n), dtype=_out_dtype(prec), device=device)
    _check_tensor(name, buf, _out_dtype(prec))
    return buf, buf.stride(0)


def rf_gram(X, W, act: str = "tanh", prec: str = "bf16", out: str = "upper", m_total: Optional[int] = None,
            G=None, ws=None, stream=None, ctx=None):
    """G = (1/m_total) σ(W X)ᵀ σ(W X) over this rank's rows of W (Eq. def_Gram).
    X: (n, p) sample-major CUDA tensor; W: (m_local, p).  Returns G (n, n), or with out="packed_tiles" on a context
    with a collective attached this rank's summed owned tiles (1-D, rf_tile_map order)."""
    torch = _torch()
    dt = _dtype_for(prec)
    _check_tensor("X", X, dt)
    _check_tensor("W", W, dt)
    n, p = X.shape
    m_local = W.shape[0]
    if W.shape[1] != p:
        raise RFError(_lib.RF_E_INVALID, "X and W disagree on p")
    m_total = m_local if m_total is None else int(m_total)
    with _on(stream):
        if out == "packed_tiles":
            if ctx is None:
                raise RFError(_lib.RF_E_INVALID, "out='packed_tiles' needs a Context with a collective attached")
            rank, world, _ = ctx.collective()
            slots = len(rf_tile_map(n, world, rank))
            if G is None:
                G = torch.empty(slots * RF_PACK_TILE * RF_PACK_TILE, dtype=torch.float32, device=X.device)
            if G.dtype != torch.float32 or not G.is_contiguous() or G.numel() < slots * RF_PACK_TILE ** 2:
                raise RFError(_lib.RF_E_INVALID, "packed_tiles: G must be a contiguous float32 tensor of "
                                                 "rf_tile_map slots × 65536 elements")
            ldg = RF_PACK_TILE
        else:
            G, ldg = _alloc_out("G", G, n, out, prec, X.device)
        if ws is None:
            ws = torch.empty(rf_workspace_size("gram", p, n, m_local, prec, out, ctx=ctx), dtype=torch.uint8,
                             device=X.device)
    _lib.check(load().rf_gram(_cp(ctx), ctypes.c_void_p(X.data_ptr()), X.stride(0), ctypes.c_void_p(W.data_ptr()),
                              W.stride(0), p, n, m_local, m_total, ACT[act], PREC[prec], OUT[out],
                              ctypes.c_void_p(G.data_ptr()), ldg, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                              _stream_ptr(stream)))
    return G


def rf_phi_closed_form(X, act: str = "tanh", tau: float = 0.0, mom: Optional[dict] = None, prec: str = "bf16",
                       out: str = "upper", row_begin: int = 0, row_end: Optional[int] = None, Phi=None, ws=None,
                       stream=None, form: int = 1, ctx=None):
    """Φ by EQ1 for pairs i ≤ j, rows i in [row_begin, row_end).  tau <= 0 → Lemma 1 τ̂.
    form = 2: the six-term EQ2 instead (rf_phi_eq2)."""
    torch = _torch()
    lib = load()
    dt = _dtype_for(prec)
    _check_tensor("X", X, dt)
    n, p = X.shape
    row_end = n if row_end is None else int(row_end)
    with _on(stream):
        Phi, ldphi = _alloc_out("Phi", Phi, n, out, prec, X.device)
        if ws is None:
            ws = torch.empty(rf_phi_workspace_size(p, n, prec), dtype=torch.uint8, device=X.device)
    mp = ctypes.byref(mom["_struct"]) if mom is not None else None
    fn = lib.rf_phi_eq2 if form == 2 else lib.rf_phi_closed_form
    _lib.check(fn(_cp(ctx), ctypes.c_void_p(X.data_ptr()), X.stride(0), p, n, ACT[act], float(tau), mp, PREC[prec],
                  OUT[out], int(row_begin), row_end, ctypes.c_void_p(Phi.data_ptr()), ldphi,
                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream)))
    return Phi


def rf_debug_gemm_nt(A, B, prec: str = "bf16", kchunk: int = 0, C=None, stream=None, ctx=None):
    """TEST HOOK: raw C = A·Bᵀ on the tcgen05 mainloop (see include/rf.h)."""
    torch = _torch()
    lib = load()
    dt = _dtype_for(prec)
    _check_tensor("A", A, dt)
    _check_tensor("B", B, dt)
    M, K = A.shape
    N = B.shape[0]
    need = ctypes.c_size_t()
    _lib.check(lib.rf_debug_gemm_workspace_size(M, N, K, PREC[prec], ctypes.byref(need)))
    with _on(stream):
        if C is None:
            C = torch.empty((M, N), dtype=torch.float32, device=A.device)
        ws = torch.empty(need.value, dtype=torch.uint8, device=A.device)
    _lib.check(lib.rf_debug_gemm_nt(_cp(ctx), ctypes.c_void_p(A.data_ptr()), A.stride(0),
                                    ctypes.c_void_p(B.data_ptr()), B.stride(0), M, N, K, PREC[prec], int(kchunk),
                                    ctypes.c_void_p(C.data_ptr()), C.stride(0), ctypes.c_void_p(ws.data_ptr()),
                                    ws.numel(), _stream_ptr(stream)))
    return C


# ------------------------------------------------------------------------------------------ NEXT-1 (TRF)
def rf_ter_features(X, T, eps: float, s_minus: float, s_plus: float, out=None, stream=None, ctx=None):
    """Σ^terᵀ as fp8 E4M3 codes (uint8 n × m_local; 0x38 = +1, 0xB8 = −1, 0 = 0).  X, T: bf16 CUDA tensors."""
    torch = _torch()
    _check_tensor("X", X, torch.bfloat16)
    _check_tensor("T", T, torch.bfloat16)
    n, p = X.shape
    m_local = T.shape[0]
    with _on(stream):
        if out is None:
            ld = (m_local + 15) // 16 * 16
            out = torch.empty((n, ld), dtype=torch.uint8, device=X.device)[:, :m_local]
    _lib.check(load().rf_ter_features(_cp(ctx), ctypes.c_void_p(X.data_ptr()), X.stride(0),
                                      ctypes.c_void_p(T.data_ptr()), T.stride(0), p, n, m_local, float(eps),
                                      float(s_minus), float(s_plus), ctypes.c_void_p(out.data_ptr()), out.stride(0),
                                      _stream_ptr(stream)))
    return out


def rf_gram_ter(X, T, eps: float, s_minus: float, s_plus: float, out: str = "upper", m_total: Optional[int] = None,
                G=None, ws=None, stream=None, ctx=None):
    """G^ter = (1/m_total) Σ^terᵀ Σ^ter (Algorithm 1 step 4) over this rank's rows of T."""
    torch = _torch()
    _check_tensor("X", X, torch.bfloat16)
    _check_tensor("T", T, torch.bfloat16)
    n, p = X.shape
    m_local = T.shape[0]
    m_total = m_local if m_total is None else int(m_total)
    with _on(stream):
        G, ldg = _alloc_out("G", G, n, out, "bf16", X.device)
        if ws is None:
            ws = torch.empty(rf_gram_ter_workspace_size(p, n, m_local), dtype=torch.uint8, device=X.device)
    _lib.check(load().rf_gram_ter(_cp(ctx), ctypes.c_void_p(X.data_ptr()), X.stride(0), ctypes.c_void_p(T.data_ptr()),
                                  T.stride(0), p, n, m_local, m_total, float(eps), float(s_minus), float(s_plus),
                                  OUT[out], ctypes.c_void_p(G.data_ptr()), ldg, ctypes.c_void_p(ws.data_ptr()),
                                  ws.numel(), _stream_ptr(stream)))
    return G


# ------------------------------------------------------------------------------------------ NEXT-2 (K̃)
def rf_ktilde(X, V, A, d0: float, d1: float, d2: float, prec: str = "bf16", out: str = "upper", Kt=None, ws=None,
              stream=None, ctx=None):
    """Theorem 1's K̃ = P(d1·XᵀX + d2·V A Vᵀ + d0·I)P (EQ6).  X: CUDA (n, p) bf16 (prec bf16) or f32 (tf32/3xtf32);
    V: CUDA f32 (n, kv) or None; A: host (kv, kv) array-like."""
    import numpy as np
    torch = _torch()
    _check_tensor("X", X, _dtype_for(prec))
    n, p = X.shape
    kv = 0 if V is None else V.shape[1]
    if V is not None:
        _check_tensor("V", V, torch.float32)
    Ah = np.ascontiguousarray(np.asarray(A if A is not None else np.zeros((0, 0)), dtype=np.float64).reshape(kv, kv))
    with _on(stream):
        if Kt is None:
            Kt = torch.zeros((n, n), dtype=torch.float32, device=X.device)
        if ws is None:
            ws = torch.empty(rf_ktilde_workspace_size(p, n, prec), dtype=torch.uint8, device=X.device)
    _check_tensor("Kt", Kt, torch.float32)
    _lib.check(load().rf_ktilde(_cp(ctx), ctypes.c_void_p(X.data_ptr()), X.stride(0), p, n,
                                ctypes.c_void_p(V.data_ptr() if V is not None else 0), V.stride(0) if V is not None else 1,
                                kv, Ah.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(d0), float(d1), float(d2),
                                PREC[prec], OUT[out], ctypes.c_void_p(Kt.data_ptr()), Kt.stride(0),
                                ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream)))
    return Kt


# ------------------------------------------------------------------------------------------ NEXT-4 (ridge)
def rf_ridge(G, n_train: int, gammas, Y, n_test: Optional[int] = None, ws=None, stream=None, ctx=None):
    """NEXT-4 kernel ridge regression on the stacked Gram G of [X_train; X_test] (include/rf.h rf_ridge).
    G: (n_all, n_all) float32 CUDA tensor (upper triangle read); Y: (n_train, r) float64 CUDA tensor.
    Returns (alpha, Yhat): (len(gammas), n_train, r) and (len(gammas), n_test, r) float64 tensors."""
    torch = _torch()
    _check_tensor("G", G, torch.float32)
    if Y.dim() == 1:
        Y = Y[:, None]
    _check_tensor("Y", Y, torch.float64)
    n_all = G.shape[0]
    n_test = n_all - int(n_train) if n_test is None else int(n_test)
    gam = [float(g) for g in gammas]
    r = Y.shape[1]
    with _on(stream):
        alpha = torch.empty((len(gam), int(n_train), r), dtype=torch.float64, device=G.device)
        Yhat = torch.empty((len(gam), max(n_test, 0), r), dtype=torch.float64, device=G.device)
        if ws is None:   # room to factor up to 16 γ at once, within ≈ 2 GB (include/rf.h rf_ridge)
            one = rf_ridge_workspace_size(n_train)
            k = max(1, min(len(gam), 16, (2 << 30) // (one - 256)))
            ws = torch.empty(256 + k * (one - 256), dtype=torch.uint8, device=G.device)
    garr = (ctypes.c_double * len(gam))(*gam)
    _lib.check(load().rf_ridge(_cp(ctx), ctypes.c_void_p(G.data_ptr()), G.stride(0), int(n_train), n_test, garr,
                               len(gam), ctypes.c_void_p(Y.data_ptr()), Y.stride(0), r,
                               ctypes.c_void_p(alpha.data_ptr()),
                               ctypes.c_void_p(Yhat.data_ptr()) if n_test > 0 else None,
                               ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream)))
    return alpha, Yhat
