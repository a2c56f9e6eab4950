"""ctypes front end of the plain-C oracle (TEST INFRASTRUCTURE ONLY).

Argument marshalling only; every number is computed in fleet_oracle.c.
Every output field is named next to its pin in DESIGN.md §2 "Parity pins, field by field".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liboracle.so")

U32, U64, F64 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
VP = ctypes.c_void_p

OR_VALID, OR_FEASIBLE, OR_HOMO_FEASIBLE = 1, 2, 4

POOL3_DTYPE = np.dtype([
    ("index", "<u4"), ("model", "<u4"), ("gpu", "<u4"), ("b1", "<u4"), ("b2", "<u4"), ("c_long", "<u4"),
    ("flags", "<u4"), ("_pad", "<u4"),
    ("n1", "<u8"), ("n2", "<u8"), ("n3", "<u8"), ("n_reject", "<u8"),
    ("nseq1", "<u8"), ("nseq2", "<u8"), ("nseq3", "<u8"),
    ("inst1", "<u8"), ("inst2", "<u8"), ("inst3", "<u8"), ("inst_homo", "<u8"), ("gpus", "<u8"),
    ("gpus_homo", "<u8"), ("cost", "<f8"), ("cost_homo", "<f8"), ("savings", "<f8"),
])

PEAK_DTYPE = np.dtype([
    ("index", "<u4"), ("model", "<u4"), ("gpu", "<u4"), ("b_short", "<u4"), ("c_short", "<u4"),
    ("c_long", "<u4"), ("flags", "<u4"), ("_pad", "<u4"),
    ("peak_short", "<u8"), ("peak_long", "<u8"), ("peak_homo", "<u8"),
    ("inst_short", "<u8"), ("inst_long", "<u8"), ("inst_homo", "<u8"), ("gpus_dual", "<u8"),
    ("gpus_homo", "<u8"),
    ("lambda_short", "<f8"), ("lambda_long", "<f8"), ("lambda_homo", "<f8"), ("cost_dual", "<f8"),
    ("cost_homo", "<f8"), ("savings", "<f8"),
])

CANDIDATE_DTYPE = np.dtype([
    ("index", "<u4"), ("model", "<u4"), ("gpu", "<u4"), ("b_short", "<u4"),
    ("c_short", "<u4"), ("c_long", "<u4"), ("flags", "<u4"), ("_pad", "<u4"),
    ("nseq_short", "<u8"), ("nseq_long", "<u8"),
    ("n_short", "<u8"), ("n_long", "<u8"), ("n_reject", "<u8"),
    ("mass_short", "<u8"), ("mass_long", "<u8"),
    ("inst_short", "<u8"), ("inst_long", "<u8"), ("inst_homo", "<u8"),
    ("gpus_dual", "<u8"), ("gpus_homo", "<u8"),
    ("alpha", "<f8"), ("rho", "<f8"), ("predicted_savings", "<f8"), ("savings", "<f8"),
    ("cost_dual", "<f8"), ("cost_homo", "<f8"),
    ("occupancy_short", "<f8"), ("occupancy_long", "<f8"),
])

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "or_kv_bytes_per_seq": (U64, [U32, U32, U32, U32, U64]),
        "or_kv_bytes_per_token_per_gpu": (U64, [U32, U32, U32, U32, U32, VP]),
        "or_kv_budget": (U64, [U64, U32, U32, U64, U64]),
        "or_max_seqs": (U64, [U64, U64, U32]),
        "or_count_le": (None, [VP, U64, VP, U32, VP, VP]),
        "or_route": (ctypes.c_int, [U32, U32, U32, U32, VP]),
        "or_route_batch": (None, [VP, U64, U32, U32, U32, VP, VP]),
        "or_pool_instances": (ctypes.c_int, [F64, F64, U64, VP]),
        "or_predicted_savings": (F64, [F64, F64]),
        "or_cost": (F64, [U64, F64, F64]),
        "or_candidate_size": (U32, []),
        "or_sweep": (ctypes.c_int, [VP, U64, U32, VP, U32, VP, VP, VP, VP, U32, VP, U32, VP, U32,
                                    VP, U32, VP, F64, F64, VP, VP]),
        "or_num_threads": (ctypes.c_int, []),
        "or_set_num_threads": (None, [ctypes.c_int]),
        "or_route_ratio": (F64, [F64, F64, F64, F64]),
        "or_pool3_size": (U32, []),
        "or_peak_size": (U32, []),
        "or_sweep_peak": (ctypes.c_int, [VP, VP, U64, U64, U32, VP, U32, VP, VP, VP, VP, U32, VP, U32, VP, U32, VP,
                                         U32, VP, F64, VP, VP]),
        "or_calibrate": (None, [VP, VP, VP, U64, U32, F64, VP, VP, VP, VP, VP, U64, VP, VP]),
        "or_sweep3": (ctypes.c_int, [VP, U64, U32, VP, U32, VP, VP, VP, VP, U32, VP, U32, VP, U32, VP, F64, F64,
                                     VP, VP]),
        "or_estimate_one": (U32, [U32, U32, F64]),
        "or_estimate": (None, [VP, VP, VP, U64, VP, VP, U32, F64, F64, VP]),
        "or_route_batch_est": (None, [VP, VP, VP, VP, U64, VP, VP, U32, F64, F64, U32, U32, U32, VP, VP, VP, VP]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    assert L.or_candidate_size() == CANDIDATE_DTYPE.itemsize, "oracle record layout drift"
    assert L.or_pool3_size() == POOL3_DTYPE.itemsize, "oracle pool3 layout drift"
    assert L.or_peak_size() == PEAK_DTYPE.itemsize, "oracle peak layout drift"
    _lib = L
    return L


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


# ---- Eq. (1)-(2) -----------------------------------------------------------
def kv_bytes_per_seq(n_l, n_h, d_h, b, c_max):
    return int(lib().or_kv_bytes_per_seq(n_l, n_h, d_h, b, c_max))


def kv_bytes_per_token_per_gpu(n_l, n_h, d_h, b, tp):
    rem = ctypes.c_uint64(0)
    q = lib().or_kv_bytes_per_token_per_gpu(n_l, n_h, d_h, b, tp, ctypes.byref(rem))
    return int(q), int(rem.value)


def kv_budget(hbm, u_num, u_den, weights_per_gpu, act_reserve):
    return int(lib().or_kv_budget(hbm, u_num, u_den, weights_per_gpu, act_reserve))


def max_seqs(budget, m_seq_total, tp):
    return int(lib().or_max_seqs(budget, m_seq_total, tp))


# ---- CDF / routing -----------------------------------------------------------
def count_le(L, x):
    L = _u32(L)
    x = _u32(x)
    cnt = np.zeros(len(x), dtype=np.uint64)
    mass = np.zeros(len(x), dtype=np.uint64)
    lib().or_count_le(L.ctypes.data, L.size, x.ctypes.data, x.size, cnt.ctypes.data,
                      mass.ctypes.data)
    return cnt, mass


def route(L, B, c_short, c_long):
    st = ctypes.c_int(0)
    p = lib().or_route(L, B, c_short, c_long, ctypes.byref(st))
    return int(p), int(st.value)


def route_batch(L, B, c_short, c_long, want_decisions=True):
    L = _u32(L)
    dec = np.zeros(L.size, dtype=np.uint8) if want_decisions else None
    counts = np.zeros(5, dtype=np.uint64)
    lib().or_route_batch(L.ctypes.data, L.size, B, c_short, c_long,
                         dec.ctypes.data if dec is not None else None, counts.ctypes.data)
    return dec, counts


# ---- Sec. 3 formulas ----------------------------------------------------------
def pool_instances(lam, mu, nseq):
    inst = ctypes.c_uint64(0)
    ok = lib().or_pool_instances(lam, mu, nseq, ctypes.byref(inst))
    return bool(ok), int(inst.value)


def predicted_savings(alpha, rho):
    return float(lib().or_predicted_savings(alpha, rho))


def cost(gpus, price, hours):
    return float(lib().or_cost(gpus, price, hours))


def num_threads():
    return int(lib().or_num_threads())


def set_num_threads(n):
    lib().or_set_num_threads(int(n))


# ---- the sweep -------------------------------------------------------------------
def config_arrays(cfg):
    """Flatten a synth.configs.Config into the oracle's own argument arrays."""
    arch = np.array([[m.n_layers, m.n_kv_heads, m.head_dim, m.kv_elem_bytes] for m in cfg.models],
                    dtype=np.uint32).ravel()
    gpu_u64 = np.array([[g.hbm_bytes, g.util_num, g.util_den, g.activation_reserve_bytes]
                        for g in cfg.gpus], dtype=np.uint64).ravel()
    price = np.array([g.price_per_gpu_hour for g in cfg.gpus], dtype=np.float64)
    dep = np.array([[d.tp_degree, d.weight_bytes_per_gpu, d.gpus_per_instance] for d in cfg.deploy],
                   dtype=np.uint64).ravel()
    return dict(arch=arch, gpu_u64=gpu_u64, price=price, deploy=dep,
                b=_u32(cfg.b_short), cs=_u32(cfg.c_short), cl=_u32(cfg.c_long),
                windows=_u32(cfg.windows()),
                mu=np.ascontiguousarray(cfg.mu_table().ravel(), dtype=np.float64))


def sweep(cfg, L, rate=None, want_all=True):
    """Evaluate every candidate of cfg on trace L. Returns (all or None, best)."""
    L = _u32(L)
    a = config_arrays(cfg)
    nm = len(cfg.models)
    out = np.zeros(cfg.n_candidates(), dtype=CANDIDATE_DTYPE) if want_all else None
    best = np.zeros(nm, dtype=CANDIDATE_DTYPE)
    rc = lib().or_sweep(
        L.ctypes.data, L.size, nm, a["arch"].ctypes.data, len(cfg.gpus), a["gpu_u64"].ctypes.data,
        a["price"].ctypes.data, a["deploy"].ctypes.data, a["b"].ctypes.data, a["b"].size,
        a["cs"].ctypes.data if a["cs"].size else None, a["cs"].size, a["cl"].ctypes.data,
        a["cl"].size, a["windows"].ctypes.data, a["windows"].size, a["mu"].ctypes.data,
        float(cfg.rate_rps if rate is None else rate), float(cfg.hours_per_year),
        out.ctypes.data if out is not None else None, best.ctypes.data)
    if rc == 1:
        raise ValueError("empty trace")
    if rc != 0:
        raise ValueError(f"or_sweep rc={rc}")
    return out, best


# ---- token-budget estimation (NEXT-1) ------------------------------------------
def route_ratio(c_hat, sigma, gamma, c_floor):
    return float(lib().or_route_ratio(c_hat, sigma, gamma, c_floor))


def estimate_one(nbytes, max_out, cstar):
    return int(lib().or_estimate_one(nbytes, max_out, cstar))


def _est_args(cats):
    c_hat = np.ascontiguousarray([c[0] for c in cats], dtype=np.float64)
    sig = np.ascontiguousarray([c[1] for c in cats], dtype=np.float64)
    return c_hat, sig


def estimate(body, max_out, cat, cats, gamma, c_floor):
    """L_total estimates; cats = [(c_hat, sigma_hat), ...] indexed by category."""
    body, max_out = _u32(body), _u32(max_out)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    c_hat, sig = _est_args(cats)
    out = np.zeros(body.size, dtype=np.uint32)
    lib().or_estimate(body.ctypes.data, max_out.ctypes.data, cat.ctypes.data, body.size, c_hat.ctypes.data,
                      sig.ctypes.data, len(cats), gamma, c_floor, out.ctypes.data)
    return out


def route_batch_est(body, max_out, cat, true_prompt, cats, gamma, c_floor, B, c_short, c_long):
    body, max_out = _u32(body), _u32(max_out)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    tp = _u32(true_prompt) if true_prompt is not None else None
    c_hat, sig = _est_args(cats)
    dec = np.zeros(body.size, dtype=np.uint8)
    lt = np.zeros(body.size, dtype=np.uint32)
    counts = np.zeros(5, dtype=np.uint64)
    mis = np.zeros(2, dtype=np.uint64)
    lib().or_route_batch_est(body.ctypes.data, max_out.ctypes.data, cat.ctypes.data,
                             tp.ctypes.data if tp is not None else None, body.size, c_hat.ctypes.data,
                             sig.ctypes.data, len(cats), gamma, c_floor, B, c_short, c_long, dec.ctypes.data,
                             lt.ctypes.data, counts.ctypes.data, mis.ctypes.data)
    return dec, lt, counts, mis


# ---- NEXT-2: three pools -------------------------------------------------------------
def sweep3(cfg, L, rate=None, want_all=True):
    """Three-pool sweep (B1 < B2 from the B grid, C_L grid); returns (all or None, best)."""
    L = _u32(L)
    a = config_arrays(cfg)
    nb = len(cfg.b_short)
    n_cand = len(cfg.models) * len(cfg.gpus) * len(cfg.c_long) * (nb * (nb - 1) // 2)
    out = np.zeros(n_cand, dtype=POOL3_DTYPE) if want_all else None
    best = np.zeros(len(cfg.models), dtype=POOL3_DTYPE)
    rc = lib().or_sweep3(
        L.ctypes.data, L.size, len(cfg.models), a["arch"].ctypes.data, len(cfg.gpus), a["gpu_u64"].ctypes.data,
        a["price"].ctypes.data, a["deploy"].ctypes.data, a["b"].ctypes.data, a["b"].size, a["cl"].ctypes.data,
        a["cl"].size, a["windows"].ctypes.data, a["windows"].size, a["mu"].ctypes.data,
        float(cfg.rate_rps if rate is None else rate), float(cfg.hours_per_year),
        out.ctypes.data if out is not None else None, best.ctypes.data)
    if rc == 1:
        raise ValueError("empty trace")
    if rc != 0:
        raise ValueError(f"or_sweep3 rc={rc}")
    return out, best


# ---- NEXT-3: calibration replay ------------------------------------------------------------
def calibrate(body, tokens, cat, n_cats, beta=0.95, c0=4.0, s0=0.5, snap_at=50):
    """Sequential EMA replay (Alg. 1 OnResponse). Returns dict of per-category arrays."""
    body, tokens = _u32(body), _u32(tokens)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    c0a = np.ascontiguousarray(np.broadcast_to(np.asarray(c0, dtype=np.float64), (n_cats,)))
    s0a = np.ascontiguousarray(np.broadcast_to(np.asarray(s0, dtype=np.float64), (n_cats,)))
    c_hat = np.zeros(n_cats)
    sig = np.zeros(n_cats)
    nobs = np.zeros(n_cats, dtype=np.uint64)
    sc = np.zeros(n_cats)
    ss = np.zeros(n_cats)
    lib().or_calibrate(body.ctypes.data, tokens.ctypes.data, cat.ctypes.data, body.size, n_cats, beta,
                       c0a.ctypes.data, s0a.ctypes.data, c_hat.ctypes.data, sig.ctypes.data, nobs.ctypes.data,
                       snap_at, sc.ctypes.data, ss.ctypes.data)
    return {"c_hat": c_hat, "sigma": sig, "n_obs": nobs, "snap_c": sc, "snap_sigma": ss}


# ---- NEXT-4: peak-window provisioning --------------------------------------------------------
def sweep_peak(cfg, L, arrival_ns, window_ns, want_all=True):
    L = _u32(L)
    arr = np.ascontiguousarray(arrival_ns, dtype=np.uint64)
    a = config_arrays(cfg)
    out = np.zeros(cfg.n_candidates(), dtype=PEAK_DTYPE) if want_all else None
    best = np.zeros(len(cfg.models), dtype=PEAK_DTYPE)
    rc = lib().or_sweep_peak(
        L.ctypes.data, arr.ctypes.data, L.size, int(window_ns), len(cfg.models), a["arch"].ctypes.data,
        len(cfg.gpus), a["gpu_u64"].ctypes.data, a["price"].ctypes.data, a["deploy"].ctypes.data,
        a["b"].ctypes.data, a["b"].size, a["cs"].ctypes.data if a["cs"].size else None, a["cs"].size,
        a["cl"].ctypes.data, a["cl"].size, a["windows"].ctypes.data, a["windows"].size, a["mu"].ctypes.data,
        float(cfg.hours_per_year), out.ctypes.data if out is not None else None, best.ctypes.data)
    if rc != 0:
        raise ValueError(f"or_sweep_peak rc={rc}")
    return out, best
