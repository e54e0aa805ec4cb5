"""CPU-side checks of the C ABI: the library loads, exports every symbol include/rf.h declares, its
host-only entry points (rf_moments, rf_phi_row_split, workspace sizing) are right, and argument
validation rejects bad calls before touching a device.  No GPU compute here."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_2110_01899_b200 as rf
from paper_2110_01899_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "rf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rf_[a-z0-9_]+)\s*\(", src)))


def test_option_table_matches_header():
    """The binding's context-option names (argument marshalling only) are include/rf.h's rf_opt enum, value for value."""
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "rf.h")).read(), flags=re.S)
    enum = {k: int(v) for k, v in re.findall(r"\bRF_OPT_([A-Z0-9_]+)\s*=\s*(\d+)", src)}
    count = enum.pop("COUNT")
    assert sorted(enum.values()) == list(range(count))
    assert {k.lower(): v for k, v in enum.items()} == _lib.OPT


def test_library_exports_every_declared_symbol():
    lib = rf.load()
    declared = _declared_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SYMBOLS)
    assert "sm_100a" in rf.rf_version()


def test_library_has_tcgen05_and_tma_sass():
    """The shipped .so carries sm_100a tcgen05 MMAs, TMEM loads and TMA loads (SASS names)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "LDTM" in out and "UTMALDG" in out


@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
@pytest.mark.parametrize("tau", [0.5, 1.0, 1.0133, 1.0833, 2.0])
def test_rf_moments_matches_oracle(act, tau):
    """Library Golub–Welsch quadrature vs the oracle's independent Newton-based rule."""
    got = rf.rf_moments(act, tau)
    ref = oracle.moments(act, tau, 512)
    kd = np.array(got["kd"])
    assert np.max(np.abs(kd - ref["kd"])) < 5e-13
    for key in ("e_sigma_sq", "d0", "d1", "d2"):
        assert abs(got[key] - ref[key]) < 5e-13, key
    assert got["quad_err_est"] < 1e-13


def test_rf_moments_fixed_nodes_and_large_tau_fallback():
    m = rf.rf_moments("erf", 1.0, nodes=64)
    assert m["nodes"] == 64
    c = 2 / math.sqrt(math.pi)
    assert abs(m["kd"][0][1] - c / math.sqrt(3.0)) < 1e-14
    big = rf.rf_moments("tanh", 16.0)            # GH cannot reach 1e-13 here → trapezoid
    tr = oracle.moments_trapezoid("tanh", 16.0)
    assert np.max(np.abs(np.array(big["kd"]) - tr) / np.maximum(1.0, np.abs(tr))) < 1e-12


def test_rf_moments_errors():
    with pytest.raises(rf.RFError) as e:
        rf.rf_moments("tanh", -1.0)
    assert e.value.status == _lib.RF_E_INVALID
    with pytest.raises(rf.RFError):
        rf.rf_moments("tanh", float("nan"))
    with pytest.raises(rf.RFError):
        rf.rf_moments("tanh", 1.0, nodes=1)


def test_phi_row_split_covers_and_balances():
    for n in (256, 1000, 131072):
        for world in (1, 2, 3, 8):
            ranges = [rf.rf_phi_row_split(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            for b, e in ranges:
                assert b % 256 == 0 and (e == n or e % 256 == 0)
            if n >= 256 * 8 * world:
                area = [sum(n - i for i in range(b, e)) for b, e in ranges]
                assert max(area) / min(area) < 1.05


def test_workspace_sizes():
    assert rf.rf_gram_workspace_size(784, 4096, 8192, "bf16") >= 4096 * 8192 * 2
    assert rf.rf_gram_workspace_size(784, 4096, 8192, "3xtf32") >= 2 * 4096 * 8192 * 4
    assert rf.rf_phi_workspace_size(512, 131072, "bf16") >= 131072 * 8


def test_validation_rejects_before_any_launch():
    lib = rf.load()
    g = lib.rf_gram(None, None, 64, None, 64, 64, 256, 512, 512, 0, 4, 0, None, 256, None, 0, None)
    assert g == _lib.RF_E_INVALID
    assert b"NULL" in lib.rf_last_error()
    buf = (ctypes.c_char * 4096)()
    addr = ctypes.addressof(buf)
    addr16 = (addr + 15) // 16 * 16
    # p = 100 bf16 with ldx = 100 → 200 B rows, not a multiple of 16 B (TMA stride rule)
    s = lib.rf_gram(None, ctypes.c_void_p(addr16), 100, ctypes.c_void_p(addr16), 104, 100, 8, 8, 8, 0, 4, 0,
                    ctypes.c_void_p(addr16), 8, ctypes.c_void_p(addr16), 16, None)
    assert s == _lib.RF_E_INVALID and b"16 B" in lib.rf_last_error()
    s = lib.rf_gram(None, ctypes.c_void_p(addr16), 64, ctypes.c_void_p(addr16), 64, 64, 8, 8, 4, 0, 4, 0,
                    ctypes.c_void_p(addr16), 8, ctypes.c_void_p(addr16), 16, None)
    assert s == _lib.RF_E_INVALID and b"m_total" in lib.rf_last_error()
    s = lib.rf_gram(None, ctypes.c_void_p(addr16), 64, ctypes.c_void_p(addr16), 64, 64, 8, 8, 8, 42, 4, 0,
                    ctypes.c_void_p(addr16), 8, ctypes.c_void_p(addr16), 16, None)
    assert s == _lib.RF_E_INVALID and b"activation" in lib.rf_last_error()
    # workspace too small
    s = lib.rf_gram(None, ctypes.c_void_p(addr16), 64, ctypes.c_void_p(addr16), 64, 64, 8, 8, 8, 0, 4, 0,
                    ctypes.c_void_p(addr16), 8, ctypes.c_void_p(addr16), 16, None)
    assert s == _lib.RF_E_WORKSPACE
    # Φ row range must start on a 256-row boundary
    s = lib.rf_phi_closed_form(None, ctypes.c_void_p(addr16), 64, 64, 512, 0, 1.0, None, 4, 0, 128, 512,
                               ctypes.c_void_p(addr16), 256, ctypes.c_void_p(addr16), 16, None)
    assert s == _lib.RF_E_INVALID and b"row range" in lib.rf_last_error()


@pytest.mark.parametrize("n", [1, 255, 256, 257, 1300, 65536])
def test_packed_tri_size_and_host_decoder(n):
    """RF_OUT_PACKED_TRI: T(T+1)/2 tiles of 65536 floats; the host decoder (layout.py) places tile (I, J) where
    include/rf.h says, checked on a buffer whose entries encode their own (row, col)."""
    from paper_2110_01899_b200 import layout
    T = -(-n // 256)
    assert rf.rf_packed_tri_elems(n) == T * (T + 1) // 2 * 65536 == layout.packed_tri_elems(n)
    if n > 1300:
        return
    P = np.full(layout.packed_tri_elems(n), -1.0)
    for I in range(T):
        for J in range(I, T):
            base = 65536 * (I * T - I * (I - 1) // 2 + J - I)
            r, c = np.meshgrid(np.arange(256) + 256 * I, np.arange(256) + 256 * J, indexing="ij")
            P[base:base + 65536] = (r * 100000 + c).ravel()
    D = layout.unpack_tri(P, n, out=np.full((n, n), -2.0))
    I, J = np.triu_indices(n)
    assert np.array_equal(D[I, J], I * 100000 + J)
    il = np.tril_indices(n, -1)
    assert np.all(D[il] == -2.0)


def test_packed_tri_validation():
    lib = rf.load()
    e = ctypes.c_int64()
    assert lib.rf_packed_tri_elems(0, ctypes.byref(e)) == _lib.RF_E_INVALID
    buf = (ctypes.c_char * 4096)()
    a16 = (ctypes.addressof(buf) + 15) // 16 * 16
    # fp32 (SIMT) precision cannot write the packed layout
    s = lib.rf_gram(None, ctypes.c_void_p(a16), 64, ctypes.c_void_p(a16), 64, 64, 8, 8, 8, 0, 1, 4,
                    ctypes.c_void_p(a16), 0, ctypes.c_void_p(a16), 16, None)
    assert s == _lib.RF_E_INVALID and b"PACKED_TRI" in lib.rf_last_error()
    # misaligned packed buffer
    s = lib.rf_phi_closed_form(None, ctypes.c_void_p(a16), 64, 64, 512, 0, 1.0, None, 4, 4, 0, 512,
                               ctypes.c_void_p(a16 + 4), 0, ctypes.c_void_p(a16), 16, None)
    assert s == _lib.RF_E_INVALID and b"16-byte" in lib.rf_last_error()
    # centering is not defined for the packed layout: 4 | CENTER is not a valid mode
    s = lib.rf_gram(None, ctypes.c_void_p(a16), 64, ctypes.c_void_p(a16), 64, 64, 8, 8, 8, 0, 4, 6,
                    ctypes.c_void_p(a16), 8, ctypes.c_void_p(a16), 16, None)
    assert s == _lib.RF_E_INVALID and b"output mode" in lib.rf_last_error()


def test_no_cpu_fallback_without_gpu():
    """On a host with no usable sm_100 device a well-formed call fails loudly (never computes on CPU)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = rf.load()
    assert lib.rf_device_supported(0) == 0
    size = rf.rf_phi_workspace_size(64, 256, "bf16")
    ws = (ctypes.c_char * (size + 512))()
    wsa = (ctypes.addressof(ws) + 255) // 256 * 256
    x = (ctypes.c_char * (256 * 64 * 2 + 64))()
    xa = (ctypes.addressof(x) + 15) // 16 * 16
    out = (ctypes.c_char * (256 * 256 * 4 + 64))()
    oa = (ctypes.addressof(out) + 15) // 16 * 16
    s = lib.rf_phi_closed_form(None, ctypes.c_void_p(xa), 64, 64, 256, 0, 1.0, None, 4, 0, 0, 256,
                               ctypes.c_void_p(oa), 256, ctypes.c_void_p(wsa), size, None)
    assert s in (_lib.RF_E_CUDA, _lib.RF_E_UNSUPPORTED)


# ------------------------------------------------------------------------------------------ context (host side)
def test_context_api_validation_without_gpu():
    """The §8(b) context calls validate on the host: options need a context, value ranges are checked, a context on a
    device that is not an sm_100 part is refused, and rf_workspace_size adds the NCCL send buffer only for a
    context with NCCL attached (NULL context: none)."""
    import torch
    lib = rf.load()
    v = ctypes.c_int64()
    assert lib.rf_ctx_set_option(None, 0, 1) == _lib.RF_E_INVALID
    assert lib.rf_ctx_get_option(None, 0, ctypes.byref(v)) == _lib.RF_E_INVALID
    lib.rf_ctx_destroy(None)                                # no-op
    if not torch.cuda.is_available():
        p = ctypes.c_void_p()
        assert lib.rf_ctx_create(0, ctypes.byref(p)) == _lib.RF_E_UNSUPPORTED and not p.value
    assert lib.rf_ctx_attach_peers(None, 0, 2, 1000) == _lib.RF_E_INVALID
    assert lib.rf_ctx_init_nccl(None, b"\0" * 128, 0, 1) == _lib.RF_E_INVALID
    a = rf.rf_workspace_size("gram", 64, 1000, 512, "bf16", "packed_tiles")
    assert a == rf.rf_gram_workspace_size(64, 1000, 512, "bf16")
    assert rf.rf_workspace_size("phi", 64, 1000, 0, "bf16") == rf.rf_phi_workspace_size(64, 1000, "bf16")
    with pytest.raises(rf.RFError):
        rf.rf_workspace_size("gram", 64, 1000, 0, "bf16")


def test_tile_map_small_case_by_hand():
    """n = 600 → T = 3 row tiles, one chunk; the upper tiles row-major are (0,0) (0,1) (0,2) (1,1) (1,2) (2,2) and
    tile u goes to rank u mod 2 at slot u div 2."""
    assert rf.rf_tile_map(600, 1, 0).tolist() == [[0, 0], [0, 1], [0, 2], [1, 1], [1, 2], [2, 2]]
    assert rf.rf_tile_map(600, 2, 0).tolist() == [[0, 0], [0, 2], [1, 2]]
    assert rf.rf_tile_map(600, 2, 1).tolist() == [[0, 1], [1, 1], [2, 2]]
    assert rf.rf_tile_map(600, 4, 3).tolist() == [[1, 1], [-1, -1]]


# ------------------------------------------------------------------------------------------ TRF thresholds (host)
@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
@pytest.mark.parametrize("tau", [0.5, 1.0, 1.0133, 1.0833])
def test_trf_thresholds_for_match_oracle(act, tau):
    from oracle import trf
    sm, sp = rf.rf_trf_thresholds_for(act, tau)
    mo = oracle.moments(act, tau)
    osm, osp = trf.solve_thresholds(mo["d1"], mo["d2"], tau)
    assert abs(sm - osm) < 1e-9 and abs(sp - osp) < 1e-9
    t = trf.ternary_moments(sm, sp, tau)
    assert abs(t["d1"] - mo["d1"]) < 1e-13 and abs(t["d2"] - mo["d2"]) < 1e-13


@pytest.mark.parametrize("tau", [0.5, 1.0])
@pytest.mark.parametrize("sign2", [1, -1])
def test_trf_thresholds_relu_targets(tau, sign2):
    """Table 2 ReLU row as the target; the mirror solution for the other sign of E[σ'']."""
    from oracle import trf
    d1, d2 = 0.25, 1 / (8 * math.pi * tau)
    sm, sp = rf.rf_trf_thresholds(d1, d2, tau, sign2)
    osm, osp = trf.solve_thresholds(d1, d2, tau, sign2=sign2)
    assert abs(sm - osm) < 1e-9 and abs(sp - osp) < 1e-9
    t = trf.ternary_moments(sm, sp, tau)
    assert abs(t["d1"] - d1) < 1e-13 and abs(t["d2"] - d2) < 1e-13
    assert (t["E_s2"] > 0) == (sign2 > 0)


def test_trf_thresholds_sign_function_and_errors():
    sm, sp = rf.rf_trf_thresholds(2 / math.pi, 0.0, 1.0, 1)        # Table 2 sign(t) row: s± = 0
    assert abs(sm) < 1e-7 and abs(sp) < 1e-7
    for bad in [(0.7, 0.0, 1.0), (0.25, 1 / (16 * math.pi), 2.0), (0.1, 0.0, 0.0), (-0.1, 0.0, 1.0)]:
        with pytest.raises(rf.RFError):
            rf.rf_trf_thresholds(*bad, 1)


def test_ridge_validation():
    lib = rf.load()
    need = ctypes.c_size_t()
    assert lib.rf_ridge_workspace_size(1000, ctypes.byref(need)) == 0 and need.value >= 1000 * 1000 * 8
    assert lib.rf_ridge_workspace_size(0, ctypes.byref(need)) == _lib.RF_E_INVALID
    buf = (ctypes.c_char * 4096)()
    a = (ctypes.addressof(buf) + 255) // 256 * 256
    g_ok = (ctypes.c_double * 2)(0.5, 1.0)
    g_bad = (ctypes.c_double * 2)(0.5, 0.0)
    vp = ctypes.c_void_p
    # γ must be > 0
    s = lib.rf_ridge(None, vp(a), 16, 8, 8, g_bad, 2, vp(a), 1, 1, vp(a), vp(a), vp(a), 16, None)
    assert s == _lib.RF_E_INVALID and b"gamma" in lib.rf_last_error()
    # ldg must cover the stacked samples
    s = lib.rf_ridge(None, vp(a), 15, 8, 8, g_ok, 2, vp(a), 1, 1, vp(a), vp(a), vp(a), 16, None)
    assert s == _lib.RF_E_INVALID and b"ldg" in lib.rf_last_error()
    # test predictions need Yhat
    s = lib.rf_ridge(None, vp(a), 16, 8, 8, g_ok, 2, vp(a), 1, 1, vp(a), None, vp(a), 16, None)
    assert s == _lib.RF_E_INVALID and b"Yhat" in lib.rf_last_error()
    # workspace too small
    s = lib.rf_ridge(None, vp(a), 16, 8, 8, g_ok, 2, vp(a), 1, 1, vp(a), vp(a), vp(a), 16, None)
    assert s == _lib.RF_E_WORKSPACE


def test_round_bf16_validation():
    """rf_round_bf16 (G1) validates before touching the device: empty sizes are a no-op, bad arguments fail."""
    lib = rf.load()
    buf = (ctypes.c_char * 4096)()
    a = (ctypes.addressof(buf) + 255) // 256 * 256
    vp = ctypes.c_void_p
    assert lib.rf_round_bf16(None, vp(a), 8, 0, 8, vp(a), 8, None) == 0
    assert lib.rf_round_bf16(None, vp(a), 8, 8, 0, vp(a), 8, None) == 0
    assert lib.rf_round_bf16(None, vp(a), 8, -1, 8, vp(a), 8, None) == _lib.RF_E_INVALID
    assert lib.rf_round_bf16(None, None, 8, 2, 8, vp(a), 8, None) == _lib.RF_E_INVALID
    s = lib.rf_round_bf16(None, vp(a), 7, 2, 8, vp(a), 8, None)
    assert s == _lib.RF_E_INVALID and b"leading" in lib.rf_last_error()
    s = lib.rf_round_bf16(None, vp(a + 2), 8, 2, 8, vp(a), 8, None)
    assert s == _lib.RF_E_INVALID and b"aligned" in lib.rf_last_error()


# ------------------------------------------------------------------------------------------ parametrised Table-2 σ
@pytest.mark.parametrize("spec", [("leaky", 1.0, -0.2), ("leaky", 0.5, 2.0), ("quad", 0.4, -1.3, 0.7),
                                  ("quad", -1.0, 0.0, 2.0)])
@pytest.mark.parametrize("tau", [0.5, 1.0833, 2.0])
def test_param_act_moments_match_oracle_and_table2(spec, tau):
    """rf_act_leaky_relu / rf_act_quadratic (include/rf.h): the library's Stein-form moments of the registered σ
    equal the oracle's and Table 2's closed forms."""
    if spec[0] == "leaky":
        name = rf.rf_act_leaky_relu(spec[1], spec[2])
        ap, am = spec[1], spec[2]
        want = (tau * (ap + am) ** 2 * (math.pi - 2) / (4 * math.pi), (ap - am) ** 2 / 4,
                (ap + am) ** 2 / (8 * math.pi * tau))
    else:
        name = rf.rf_act_quadratic(*spec[1:])
        a0, a1, a2 = spec[1:]
        want = (2 * tau ** 2 * a2 ** 2, a1 ** 2, a2 ** 2)
    got = rf.rf_moments(name, tau)
    ref = oracle.moments(name, tau)
    assert np.max(np.abs(np.array(got["kd"]) - ref["kd"])) < 1e-11 * max(1.0, np.max(np.abs(ref["kd"])))
    for k, w in zip(("d0", "d1", "d2"), want):
        assert abs(got[k] - w) < 1e-11 * max(1.0, abs(w)), (k, got[k], w)


def test_param_act_registration():
    a = rf.rf_act_leaky_relu(1.0, -0.1)
    b = rf.rf_act_leaky_relu(1.0, -0.1)
    assert a == b and rf.ACT[a] == rf.ACT[b] >= 64
    assert rf.ACT[rf.rf_act_quadratic(0.0, 0.0, 1.0)] != rf.ACT[a]
    lib = rf.load()
    v = ctypes.c_int()
    assert lib.rf_act_leaky_relu(float("nan"), 0.0, ctypes.byref(v)) == _lib.RF_E_INVALID
    assert lib.rf_act_quadratic(0.0, float("inf"), 0.0, ctypes.byref(v)) == _lib.RF_E_INVALID
    m = ctypes.c_int()
    assert lib.rf_moments(200, 1.0, 0, None) == _lib.RF_E_INVALID      # an id never registered


def test_dram_traffic_record_matches_the_current_sources():
    """bench.py reports `roofline.traffic` only from an ncu record keyed by the hash of csrc/* and include/rf.h
    (never stale bytes).  The committed record must be the one of the sources as they stand —
    after a kernel change, re-run scripts/ncu_traffic.py on a B200 (or the bench line carries traffic = null)."""
    import json
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    with open(os.path.join(root, "profiles", "ncu_traffic.json")) as f:
        rec = json.load(f)
    h = bench.source_hash()
    assert h in rec, f"no ncu DRAM-traffic record for the current library sources ({h})"
    assert rec[h].get("configs[3]:bf16:w1:K4_syrk", 0) > 17.2e9      # at least K4's compulsory bytes
