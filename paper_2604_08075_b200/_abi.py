"""Thin Python binding of the C ABI in include/fleet_plan.h (argument marshalling
only: every step of the sweep runs in libfleetplan.so's CUDA kernels).

The Python names are the ABI names. There is no fallback: if the native
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLEETPLAN_LIB") or os.path.join(_HERE, "lib", "libfleetplan.so")

FP_ABI_VERSION = 2
FP_FLAG_NO_MASS = 0x1
FP_FLAG_REPLICATED_GRID = 0x2
FP_FLAG_KERNEL_TIMING = 0x4
FP_FLAG_CHECK_ORDER = 0x8
FP_FLAG_COLLECTIVES = 0x10
FP_FLAG_TIME_TRACE = 0x20
FP_FLAG_P2P = 0x40
FP_FLAG_SPECULATE = 0x80
FP_P2P_HANDLE_BYTES = 64
FP_KERNEL_TRACE, FP_KERNEL_EVAL, FP_KERNEL_ROUTE = 0, 1, 2
FP_CAND_VALID, FP_CAND_FEASIBLE, FP_CAND_HOMO_FEASIBLE = 1, 2, 4
STATUS = ["FP_OK", "FP_ERR_INVALID_ARG", "FP_ERR_CONFIG", "FP_ERR_EMPTY_TRACE", "FP_ERR_ALIGNMENT",
          "FP_ERR_OOM", "FP_ERR_CUDA", "FP_ERR_NCCL", "FP_ERR_STATE"]
EXPORTED = ["fleet_plan_create", "route_batch", "sweep_thresholds", "best_split", "sweep_histogram",
            "fleet_plan_info", "fp_kernel_launches", "fleet_plan_destroy", "fp_status_string",
            "fp_last_error", "fp_shard_range", "fp_candidate_range", "fp_merge_best",
            "fp_nccl_get_unique_id", "fp_kernel_time", "fp_kernel_time_reset", "sweep_and_route",
            "sweep_thresholds_raw", "route_batch_raw", "sweep_three_pools", "calibrate_replay",
            "sweep_peak_windows", "fp_p2p_export", "fp_p2p_import", "sweep_and_route_raw",
            "sweep_and_route_graph"]

c_u32, c_u64, c_i32, c_dbl, c_vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p


class fp_model(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("n_layers", c_u32), ("n_kv_heads", c_u32),
                ("head_dim", c_u32), ("kv_elem_bytes", c_u32)]


class fp_gpu(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("hbm_bytes", c_u64), ("util_num", c_u32),
                ("util_den", c_u32), ("activation_reserve_bytes", c_u64), ("price_per_gpu_hour", c_dbl)]


class fp_deploy(ctypes.Structure):
    _fields_ = [("tp_degree", c_u32), ("gpus_per_instance", c_u32), ("weight_bytes_per_gpu", c_u64)]


class fp_grid(ctypes.Structure):
    _fields_ = [("b_short", ctypes.POINTER(c_u32)), ("n_b", c_u32),
                ("c_short", ctypes.POINTER(c_u32)), ("n_cs", c_u32),
                ("c_long", ctypes.POINTER(c_u32)), ("n_cl", c_u32)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(c_u64), c_u64, c_vp)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, c_u64, c_vp)


class fp_collectives(ctypes.Structure):
    _fields_ = [("allreduce_sum_u64", ALLREDUCE_FN), ("allgather_bytes", ALLGATHER_FN), ("user", c_vp)]


class fp_plan_desc(ctypes.Structure):
    _fields_ = [("abi_version", c_u32), ("flags", c_u32),
                ("models", ctypes.POINTER(fp_model)), ("n_models", c_u32),
                ("gpus", ctypes.POINTER(fp_gpu)), ("n_gpus", c_u32),
                ("deploy", ctypes.POINTER(fp_deploy)),
                ("grid", fp_grid),
                ("windows", ctypes.POINTER(c_u32)), ("n_windows", c_u32),
                ("mu_table", ctypes.POINTER(c_dbl)),
                ("hours_per_year", c_dbl),
                ("device", c_i32), ("rank", c_i32), ("world", c_i32),
                ("nccl_unique_id", c_vp),
                ("collectives", ctypes.POINTER(fp_collectives))]


class fp_category_calibration(ctypes.Structure):
    _fields_ = [("c_hat", c_dbl), ("sigma_hat", c_dbl)]


class fp_estimator(ctypes.Structure):
    _fields_ = [("cats", ctypes.POINTER(fp_category_calibration)), ("n_cats", c_u32), ("gamma", c_dbl),
                ("c_floor", c_dbl)]


class fp_raw_trace(ctypes.Structure):
    _fields_ = [("body_bytes", c_vp), ("max_output_tokens", c_vp), ("category", c_vp),
                ("true_prompt_tokens", c_vp)]


class fp_route_counts(ctypes.Structure):
    _fields_ = [("n_short", c_u64), ("n_long", c_u64), ("n_reject", c_u64),
                ("mass_short", c_u64), ("mass_long", c_u64)]


class fp_plan_info(ctypes.Structure):
    _fields_ = [("n_candidates", c_u64), ("cand_first", c_u64), ("cand_count", c_u64),
                ("n_edges", c_u32), ("lut_shift", c_u32), ("lut_cells", c_u32), ("n_windows", c_u32),
                ("device", c_i32), ("rank", c_i32), ("world", c_i32),
                ("sm_count", c_u32), ("k1_grid", c_u32), ("k1_block", c_u32),
                ("nccl_comm_size", c_i32), ("k3_shape", c_u32), ("k3_blocks_per_model", c_u32),
                ("spec_calls", c_u32), ("spec_misses", c_u32)]


# fp_candidate (192 bytes) as a numpy record, field order of fleet_plan.h
FP_CANDIDATE = np.dtype([
    ("index", "<u4"), ("model", "<u4"), ("gpu", "<u4"),
    ("b_short", "<u4"), ("c_short", "<u4"), ("c_long", "<u4"),
    ("flags", "<u4"), ("_pad", "<u4"),
    ("nseq_short", "<u8"), ("nseq_long", "<u8"),
    ("n_short", "<u8"), ("n_long", "<u8"), ("n_reject", "<u8"),
    ("mass_short", "<u8"), ("mass_long", "<u8"),
    ("inst_short", "<u8"), ("inst_long", "<u8"), ("inst_homo", "<u8"),
    ("gpus_dual", "<u8"), ("gpus_homo", "<u8"),
    ("alpha", "<f8"), ("rho", "<f8"), ("predicted_savings", "<f8"), ("savings", "<f8"),
    ("cost_dual", "<f8"), ("cost_homo", "<f8"),
    ("occupancy_short", "<f8"), ("occupancy_long", "<f8"),
])
assert FP_CANDIDATE.itemsize == 192

# fp_pool3_candidate (160 bytes), field order of fleet_plan.h
FP_POOL3 = np.dtype([
    ("index", "<u4"), ("model", "<u4"), ("gpu", "<u4"), ("b1", "<u4"), ("b2", "<u4"), ("c_long", "<u4"),
    ("flags", "<u4"), ("_pad", "<u4"),
    ("n1", "<u8"), ("n2", "<u8"), ("n3", "<u8"), ("n_reject", "<u8"),
    ("nseq1", "<u8"), ("nseq2", "<u8"), ("nseq3", "<u8"),
    ("inst1", "<u8"), ("inst2", "<u8"), ("inst3", "<u8"), ("inst_homo", "<u8"),
    ("gpus", "<u8"), ("gpus_homo", "<u8"),
    ("cost", "<f8"), ("cost_homo", "<f8"), ("savings", "<f8"),
])
assert FP_POOL3.itemsize == 160

# fp_peak_candidate (144 bytes)
FP_PEAK = np.dtype([
    ("index", "<u4"), ("model", "<u4"), ("gpu", "<u4"), ("b_short", "<u4"), ("c_short", "<u4"),
    ("c_long", "<u4"), ("flags", "<u4"), ("_pad", "<u4"),
    ("peak_short", "<u8"), ("peak_long", "<u8"), ("peak_homo", "<u8"),
    ("inst_short", "<u8"), ("inst_long", "<u8"), ("inst_homo", "<u8"), ("gpus_dual", "<u8"),
    ("gpus_homo", "<u8"),
    ("lambda_short", "<f8"), ("lambda_long", "<f8"), ("lambda_homo", "<f8"),
    ("cost_dual", "<f8"), ("cost_homo", "<f8"), ("savings", "<f8"),
])
assert FP_PEAK.itemsize == 144


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "fleet_plan_create": (c_i32, [ctypes.POINTER(fp_plan_desc), ctypes.POINTER(c_vp)]),
        "route_batch": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_u32, c_u32, c_vp, ctypes.POINTER(fp_route_counts), c_vp]),
        "sweep_thresholds": (c_i32, [c_vp, c_vp, c_u64, c_dbl, c_vp, c_vp]),
        "best_split": (c_i32, [c_vp, c_vp]),
        "sweep_histogram": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
        "fleet_plan_info": (c_i32, [c_vp, ctypes.POINTER(fp_plan_info)]),
        "fp_kernel_launches": (c_u64, [c_vp]),
        "fleet_plan_destroy": (None, [c_vp]),
        "fp_status_string": (ctypes.c_char_p, [c_i32]),
        "fp_last_error": (ctypes.c_char_p, [c_vp]),
        "fp_shard_range": (None, [c_u64, c_i32, c_i32, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64)]),
        "fp_candidate_range": (None, [c_u64, c_i32, c_i32, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64)]),
        "fp_merge_best": (None, [c_vp, c_i32, c_u32, c_vp]),
        "fp_nccl_get_unique_id": (c_i32, [c_vp]),
        "fp_p2p_export": (c_i32, [c_vp, c_vp]),
        "fp_p2p_import": (c_i32, [c_vp, c_vp]),
        "fp_kernel_time": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_dbl), ctypes.POINTER(c_u64)]),
        "fp_kernel_time_reset": (c_i32, [c_vp]),
        "sweep_thresholds_raw": (c_i32, [c_vp, ctypes.POINTER(fp_raw_trace), c_u64, ctypes.POINTER(fp_estimator), c_dbl,
                                         c_vp, c_vp]),
        "route_batch_raw": (c_i32, [c_vp, ctypes.POINTER(fp_raw_trace), c_u64, ctypes.POINTER(fp_estimator), c_u32, c_u32,
                                    c_u32, c_vp, c_vp, ctypes.POINTER(fp_route_counts), ctypes.POINTER(c_u64), c_vp]),
        "sweep_and_route_raw": (c_i32, [c_vp, ctypes.POINTER(fp_raw_trace), c_u64, ctypes.POINTER(fp_estimator),
                                        c_dbl, c_u32, c_vp, c_vp, ctypes.POINTER(fp_route_counts), c_vp]),
        "sweep_three_pools": (c_i32, [c_vp, c_dbl, c_vp, c_vp, c_vp]),
        "sweep_peak_windows": (c_i32, [c_vp, c_vp, c_vp, c_u64, c_u64, c_vp, c_vp, c_vp]),
        "calibrate_replay": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_u64, c_u32, c_dbl, c_vp, c_u64, c_vp, c_vp, c_vp,
                                     c_vp]),
        "sweep_and_route": (c_i32, [c_vp, c_vp, c_u64, c_dbl, c_u32, c_vp, c_vp, ctypes.POINTER(fp_route_counts), c_vp]),
        "sweep_and_route_graph": (c_i32, [c_vp, c_vp, c_u64, c_dbl, c_u32, c_vp, c_vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


class FleetPlanError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")
        self.status = status


def _check(status, plan=None):
    if status != 0:
        msg = lib.fp_last_error(plan.handle if plan is not None else None)
        raise FleetPlanError(status, msg.decode() if msg else "")


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


class FleetPlan:
    """Owner of an fp_plan* (destroyed with fleet_plan_destroy)."""

    def __init__(self, handle, n_models, device, keepalive=None):
        self.handle = handle
        self.n_models = n_models
        self.device = device
        self._keepalive = keepalive     # ctypes callbacks of host collectives

    def __del__(self):
        try:
            fleet_plan_destroy(self)
        except Exception:
            pass


def desc_from_config(cfg):
    """Marshal a configuration object (synth.configs.Config or any object with the
    same attributes) into fleet_plan_create keyword arguments."""
    return dict(
        models=[(m.name, m.n_layers, m.n_kv_heads, m.head_dim, m.kv_elem_bytes) for m in cfg.models],
        gpus=[(g.name, g.hbm_bytes, g.util_num, g.util_den, g.activation_reserve_bytes, g.price_per_gpu_hour)
              for g in cfg.gpus],
        deploy=[(d.tp_degree, d.gpus_per_instance, d.weight_bytes_per_gpu) for d in cfg.deploy],
        b_short=cfg.b_short, c_short=cfg.c_short, c_long=cfg.c_long,
        windows=cfg.windows(), mu_table=cfg.mu_table(), hours_per_year=cfg.hours_per_year)


def fleet_plan_create(*, models, gpus, deploy, b_short, c_short, c_long, windows, mu_table,
                      hours_per_year=8760.0, device=0, rank=0, world=1, nccl_unique_id=None, flags=0,
                      collectives=None):
    """collectives: optional object with allreduce_sum_u64(np.ndarray[uint64]) (in place) and
    allgather_bytes(bytes) -> bytes (rank order); replaces NCCL when world > 1."""
    nm, ng = len(models), len(gpus)
    M = (fp_model * nm)(*[fp_model(n.encode()[:31], *a) for (n, *a) in models])
    G = (fp_gpu * ng)(*[fp_gpu(n.encode()[:31], *a) for (n, *a) in gpus])
    D = (fp_deploy * (nm * ng))(*[fp_deploy(*d) for d in deploy])
    b, cs, cl, w = _u32(b_short), _u32(c_short), _u32(c_long), _u32(windows)
    mu = np.ascontiguousarray(np.asarray(mu_table, dtype=np.float64).ravel())
    P = ctypes.POINTER(c_u32)
    desc = fp_plan_desc()
    desc.abi_version = FP_ABI_VERSION
    desc.flags = flags
    desc.models, desc.n_models = M, nm
    desc.gpus, desc.n_gpus = G, ng
    desc.deploy = D
    desc.grid = fp_grid(b.ctypes.data_as(P), b.size, cs.ctypes.data_as(P) if cs.size else None, cs.size,
                        cl.ctypes.data_as(P), cl.size)
    desc.windows, desc.n_windows = w.ctypes.data_as(P), w.size
    desc.mu_table = mu.ctypes.data_as(ctypes.POINTER(c_dbl))
    desc.hours_per_year = hours_per_year
    desc.device, desc.rank, desc.world = device, rank, world
    uid = None
    if nccl_unique_id is not None:
        uid = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        desc.nccl_unique_id = ctypes.cast(uid, c_vp)
    keep = None
    if collectives is not None:
        def _ar(buf, count, user):
            try:
                a = np.ctypeslib.as_array(buf, shape=(count,))
                collectives.allreduce_sum_u64(a)
                return 0
            except Exception:
                return 1

        def _ag(hsend, hrecv, nbytes, user):
            try:
                data = ctypes.string_at(hsend, nbytes)
                out = collectives.allgather_bytes(data)
                ctypes.memmove(hrecv, out, len(out))
                return 0
            except Exception:
                return 1
        coll = fp_collectives(ALLREDUCE_FN(_ar), ALLGATHER_FN(_ag), None)
        desc.collectives = ctypes.pointer(coll)
        keep = (coll, _ar, _ag)
    h = c_vp()
    _check(lib.fleet_plan_create(ctypes.byref(desc), ctypes.byref(h)))
    return FleetPlan(h, nm, device, keepalive=keep)


def _trace_ptr(lengths):
    """(pointer, n, is_device, keepalive) for a torch tensor or numpy array of u32."""
    try:
        import torch
        if isinstance(lengths, torch.Tensor):
            if lengths.dtype not in (torch.int32, torch.uint32):
                raise TypeError("lengths must be an int32/uint32 tensor of L_total values")
            if not lengths.is_contiguous():
                raise ValueError("lengths must be contiguous")
            return lengths.data_ptr(), lengths.numel(), lengths.is_cuda, lengths
    except ImportError:
        pass
    a = np.asarray(lengths)
    if a.dtype not in (np.uint32, np.int32) or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=np.uint32)
    return a.ctypes.data, a.size, False, a


def _stream_handle(stream, device):
    if stream is not None:
        return c_vp(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    import torch
    return c_vp(torch.cuda.current_stream(device).cuda_stream)


def route_batch(plan, lengths, b_short, c_short, c_long, decision=None, want_counts=True, stream=None):
    ptr, n, _, keep = _trace_ptr(lengths)
    dptr = None
    if decision is not None:
        if decision.numel() < n or not decision.is_cuda:
            raise ValueError("decision must be a CUDA uint8 tensor with >= n elements")
        dptr = decision.data_ptr()
    counts = fp_route_counts() if want_counts else None
    _check(lib.route_batch(plan.handle, ptr, n, b_short, c_short, c_long, dptr,
                           ctypes.byref(counts) if counts is not None else None,
                           _stream_handle(stream, plan.device)), plan)
    del keep
    if counts is None:
        return None
    return {k: int(getattr(counts, k)) for k, _ in fp_route_counts._fields_}


def sweep_thresholds(plan, lengths, rate_rps, want_results=False, stream=None):
    ptr, n, _, keep = _trace_ptr(lengths)
    out = None
    if want_results:
        out = np.zeros(fleet_plan_info(plan)["cand_count"], dtype=FP_CANDIDATE)
    _check(lib.sweep_thresholds(plan.handle, ptr, n, float(rate_rps),
                                out.ctypes.data if out is not None else None,
                                _stream_handle(stream, plan.device)), plan)
    del keep
    return out


def best_split(plan):
    out = np.zeros(plan.n_models, dtype=FP_CANDIDATE)
    _check(lib.best_split(plan.handle, out.ctypes.data), plan)
    return out


def sweep_histogram(plan):
    info = fleet_plan_info(plan)
    ne = info["n_edges"]
    edges = np.zeros(ne, dtype=np.uint32)
    cnt = np.zeros(ne + 1, dtype=np.uint64)
    mass = np.zeros(ne + 1, dtype=np.uint64)
    _check(lib.sweep_histogram(plan.handle, edges.ctypes.data, cnt.ctypes.data, mass.ctypes.data), plan)
    return edges, cnt, mass


def fleet_plan_info(plan):
    i = fp_plan_info()
    _check(lib.fleet_plan_info(plan.handle, ctypes.byref(i)), plan)
    return {k: getattr(i, k) for k, _ in fp_plan_info._fields_}


def fp_kernel_launches(plan):
    return int(lib.fp_kernel_launches(plan.handle))


def fleet_plan_destroy(plan):
    if plan is not None and plan.handle:
        lib.fleet_plan_destroy(plan.handle)
        plan.handle = None


def fp_status_string(status):
    return lib.fp_status_string(status).decode()


def fp_shard_range(n_total, rank, world):
    a, b = c_u64(), c_u64()
    lib.fp_shard_range(n_total, rank, world, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def fp_candidate_range(n_candidates, rank, world):
    a, b = c_u64(), c_u64()
    lib.fp_candidate_range(n_candidates, rank, world, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def fp_merge_best(recs, world, n_models):
    recs = np.ascontiguousarray(recs, dtype=FP_CANDIDATE)
    assert recs.size == world * n_models
    out = np.zeros(n_models, dtype=FP_CANDIDATE)
    lib.fp_merge_best(recs.ctypes.data, world, n_models, out.ctypes.data)
    return out


def fp_nccl_get_unique_id():
    buf = ctypes.create_string_buffer(128)
    st = lib.fp_nccl_get_unique_id(buf)
    if st != 0:
        raise FleetPlanError(st, "ncclGetUniqueId failed")
    return buf.raw


def fp_p2p_export(plan):
    """This rank's CUDA IPC handle (FP_P2P_HANDLE_BYTES bytes) of its histogram exchange buffer."""
    buf = ctypes.create_string_buffer(FP_P2P_HANDLE_BYTES)
    _check(lib.fp_p2p_export(plan.handle, buf), plan)
    return buf.raw


def fp_p2p_import(plan, handles):
    """Open every rank's exchange buffer; `handles` = the ranks' fp_p2p_export bytes in rank order."""
    blob = b"".join(handles)
    assert len(blob) == len(handles) * FP_P2P_HANDLE_BYTES
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(lib.fp_p2p_import(plan.handle, buf), plan)


def fp_kernel_time(plan, kind):
    """(total device ms, launches) of kernel `kind` since the last reset."""
    ms, n = c_dbl(), c_u64()
    _check(lib.fp_kernel_time(plan.handle, kind, ctypes.byref(ms), ctypes.byref(n)), plan)
    return ms.value, n.value


def fp_kernel_time_reset(plan):
    _check(lib.fp_kernel_time_reset(plan.handle), plan)


def sweep_and_route(plan, lengths, rate_rps, route_model=0, decision=None, stream=None, want_best=True):
    """Whole workflow in one call; returns (best records [n_models], route counts dict).
    want_best=False (device trace, bin mode): asynchronous, returns (None, None);
    read the records later with best_split()."""
    ptr, n, _, keep = _trace_ptr(lengths)
    dptr = None
    if decision is not None:
        if decision.numel() < n or not decision.is_cuda:
            raise ValueError("decision must be a CUDA uint8 tensor with >= n elements")
        dptr = decision.data_ptr()
    if not want_best:
        _check(lib.sweep_and_route(plan.handle, ptr, n, float(rate_rps), route_model, dptr, None, None,
                                   _stream_handle(stream, plan.device)), plan)
        del keep
        return None, None
    best = np.zeros(plan.n_models, dtype=FP_CANDIDATE)
    counts = fp_route_counts()
    _check(lib.sweep_and_route(plan.handle, ptr, n, float(rate_rps), route_model, dptr, best.ctypes.data,
                               ctypes.byref(counts), _stream_handle(stream, plan.device)), plan)
    del keep
    return best, {k: int(getattr(counts, k)) for k, _ in fp_route_counts._fields_}


def sweep_and_route_graph(plan, lengths, rate_rps, decision, route_model=0, stream=None):
    """sweep_and_route's asynchronous step as the plan's captured CUDA graph
    (device trace and decision tensor; captured on the first call with these
    arguments, replayed after). Read the records with best_split()."""
    if not (hasattr(lengths, "is_cuda") and lengths.is_cuda and lengths.is_contiguous()):
        raise ValueError("sweep_and_route_graph needs a contiguous CUDA trace")
    if decision.numel() < lengths.numel() or not decision.is_cuda:
        raise ValueError("decision must be a CUDA uint8 tensor with >= n elements")
    _check(lib.sweep_and_route_graph(plan.handle, lengths.data_ptr(), lengths.numel(), float(rate_rps), route_model,
                                     decision.data_ptr(), _stream_handle(stream, plan.device)), plan)


# ---- token-budget estimation (NEXT-1) ------------------------------------------------
def _estimator(cats, gamma, c_floor):
    arr = (fp_category_calibration * len(cats))(*[fp_category_calibration(float(c), float(s)) for c, s in cats])
    return fp_estimator(arr, len(cats), float(gamma), float(c_floor)), arr


def _raw(body, max_out, cat, true_prompt=None):
    for t in (body, max_out, cat) + ((true_prompt,) if true_prompt is not None else ()):
        if not (hasattr(t, "is_cuda") and t.is_cuda and t.is_contiguous()):
            raise ValueError("raw columns must be contiguous CUDA tensors")
    if body.numel() != max_out.numel() or body.numel() != cat.numel():
        raise ValueError("raw columns must have the same length")
    return fp_raw_trace(body.data_ptr(), max_out.data_ptr(), cat.data_ptr(),
                        true_prompt.data_ptr() if true_prompt is not None else None), body.numel()


def sweep_thresholds_raw(plan, body, max_out, cat, cats, rate_rps, gamma=1.0, c_floor=0.5, want_results=False,
                         stream=None):
    """Sweep on L_total estimated from (body bytes, max_output, category) in the trace pass.
    cats = [(c_hat, sigma_hat), ...] indexed by category."""
    tr, n = _raw(body, max_out, cat)
    est, keep = _estimator(cats, gamma, c_floor)
    out = np.zeros(fleet_plan_info(plan)["cand_count"], dtype=FP_CANDIDATE) if want_results else None
    _check(lib.sweep_thresholds_raw(plan.handle, ctypes.byref(tr), n, ctypes.byref(est), float(rate_rps),
                                    out.ctypes.data if out is not None else None,
                                    _stream_handle(stream, plan.device)), plan)
    del keep
    return out


def route_batch_raw(plan, body, max_out, cat, cats, b_short, c_short, c_long, true_prompt=None, gamma=1.0,
                    c_floor=0.5, decision=None, l_total=None, stream=None):
    """Route on estimated L_total; returns (counts dict, misroute [short, long] or None)."""
    tr, n = _raw(body, max_out, cat, true_prompt)
    est, keep = _estimator(cats, gamma, c_floor)
    counts = fp_route_counts()
    mis = (c_u64 * 2)()
    _check(lib.route_batch_raw(plan.handle, ctypes.byref(tr), n, ctypes.byref(est), b_short, c_short, c_long,
                               decision.data_ptr() if decision is not None else None,
                               l_total.data_ptr() if l_total is not None else None, ctypes.byref(counts),
                               mis, _stream_handle(stream, plan.device)), plan)
    del keep
    c = {k: int(getattr(counts, k)) for k, _ in fp_route_counts._fields_}
    return c, ([int(mis[0]), int(mis[1])] if true_prompt is not None else None)


def sweep_and_route_raw(plan, body, max_out, cat, cats, rate_rps, route_model=0, decision=None, gamma=1.0,
                        c_floor=0.5, stream=None, want_best=True):
    """The whole workflow on raw columns; returns (best records, counts dict), or
    (None, None) with want_best=False (asynchronous in the speculative form)."""
    tr, n = _raw(body, max_out, cat)
    est, keep = _estimator(cats, gamma, c_floor)
    dptr = None
    if decision is not None:
        if decision.numel() < n or not decision.is_cuda:
            raise ValueError("decision must be a CUDA uint8 tensor with >= n elements")
        dptr = decision.data_ptr()
    if not want_best:
        _check(lib.sweep_and_route_raw(plan.handle, ctypes.byref(tr), n, ctypes.byref(est), float(rate_rps),
                                       route_model, dptr, None, None, _stream_handle(stream, plan.device)), plan)
        del keep
        return None, None
    best = np.zeros(plan.n_models, dtype=FP_CANDIDATE)
    counts = fp_route_counts()
    _check(lib.sweep_and_route_raw(plan.handle, ctypes.byref(tr), n, ctypes.byref(est), float(rate_rps), route_model,
                                   dptr, best.ctypes.data, ctypes.byref(counts),
                                   _stream_handle(stream, plan.device)), plan)
    del keep
    return best, {k: int(getattr(counts, k)) for k, _ in fp_route_counts._fields_}


# ---- NEXT-2: three pools ----------------------------------------------------------------
def sweep_three_pools(plan, rate_rps, want_results=False, n_results=None, stream=None):
    """Three-pool grid over the last sweep's histogram; returns (all or None, best)."""
    out = np.zeros(n_results, dtype=FP_POOL3) if want_results else None
    best = np.zeros(plan.n_models, dtype=FP_POOL3)
    _check(lib.sweep_three_pools(plan.handle, float(rate_rps), out.ctypes.data if out is not None else None,
                                 best.ctypes.data, _stream_handle(stream, plan.device)), plan)
    return out, best


# ---- NEXT-3: calibration replay ---------------------------------------------------------------
def calibrate_replay(plan, body, prompt_tokens, cat, init, beta=0.95, snap_at=50, stream=None):
    """EMA replay of a device feedback stream; init = [(c_hat, sigma_hat), ...] per category.
    Returns dict(c_hat, sigma, n_obs, snap_c, snap_sigma) of numpy arrays."""
    for t in (body, prompt_tokens, cat):
        if not (hasattr(t, "is_cuda") and t.is_cuda and t.is_contiguous()):
            raise ValueError("feedback columns must be contiguous CUDA tensors")
    n = body.numel()
    k = len(init)
    ini = (fp_category_calibration * k)(*[fp_category_calibration(float(c), float(s)) for c, s in init])
    fin = (fp_category_calibration * k)()
    snap = (fp_category_calibration * k)()
    nobs = np.zeros(k, dtype=np.uint64)
    _check(lib.calibrate_replay(plan.handle, body.data_ptr(), prompt_tokens.data_ptr(), cat.data_ptr(), n, k,
                                float(beta), ini, snap_at, fin, nobs.ctypes.data, snap,
                                _stream_handle(stream, plan.device)), plan)
    return {"c_hat": np.array([f.c_hat for f in fin]), "sigma": np.array([f.sigma_hat for f in fin]),
            "n_obs": nobs, "snap_c": np.array([f.c_hat for f in snap]),
            "snap_sigma": np.array([f.sigma_hat for f in snap])}


# ---- NEXT-4: peak-window provisioning -------------------------------------------------------
def sweep_peak_windows(plan, lengths, arrival_ns, window_ns, want_results=False, stream=None):
    """lengths: int32/uint32 CUDA tensor; arrival_ns: int64 CUDA tensor (non-decreasing)."""
    if not (lengths.is_cuda and arrival_ns.is_cuda and lengths.numel() == arrival_ns.numel()):
        raise ValueError("lengths and arrival_ns must be CUDA tensors of equal length")
    out = np.zeros(fleet_plan_info(plan)["n_candidates"], dtype=FP_PEAK) if want_results else None
    best = np.zeros(plan.n_models, dtype=FP_PEAK)
    _check(lib.sweep_peak_windows(plan.handle, lengths.data_ptr(), arrival_ns.data_ptr(), lengths.numel(),
                                  int(window_ns), out.ctypes.data if out is not None else None, best.ctypes.data,
                                  _stream_handle(stream, plan.device)), plan)
    return out, best
