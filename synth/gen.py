"""Trace generation: numpy reference, host-C and CUDA front ends (INPUT MODULE).

A trace is a u32 column of L_total values. Request i of
a trace with seed s and mixture M is

    w0, w1, w2, _ = Philox4x32-10(ctr=(lo32 i, hi32 i, 0, 0), key=(lo32 s, hi32 s))
    c      = #{k : w2 >= M.cut[k]}                 (mixture component)
    L_in   = sample(M.shapes[c].t_in,  w0)
    L_out  = sample(M.shapes[c].t_out, w1)
    L_total = L_in + L_out

with `sample` the table rule in shapes.py. No routing or counting here.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .philox import philox_words
from .shapes import LUT_SIZE, Mixture, mixture

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")


def _sample(table, w):
    q = table.q.astype(np.uint64)
    i = (w >> np.uint32(16)).astype(np.int64)
    if not table.interp:
        return q[i]
    f = (w & np.uint32(0xFFFF)).astype(np.uint64)
    return q[i] + (((q[i + 1] - q[i]) * f) >> np.uint64(16))


def generate_np(mix: Mixture | str, seed: int, first: int, count: int) -> np.ndarray:
    """Numpy reference generator for indices [first, first+count)."""
    if isinstance(mix, str):
        mix = mixture(mix)
    if count == 0:
        return np.zeros(0, dtype=np.uint32)
    w0, w1, w2, _ = philox_words(seed, first, count)
    comp = np.zeros(count, dtype=np.int64)
    for c in mix.cut:
        comp += (w2 >= np.uint32(c)).astype(np.int64)
    out = np.zeros(count, dtype=np.uint64)
    for k, sh in enumerate(mix.shapes):
        m = comp == k
        if m.any():
            out[m] = _sample(sh.t_in, w0[m]) + _sample(sh.t_out, w1[m])
    return out.astype(np.uint32)


@dataclass
class PackedMixture:
    """Flat arrays handed to the C and CUDA generators."""
    luts: np.ndarray      # uint32 [n_comp * 2 * LUT_SIZE]  (comp, in/out, level)
    interp: np.ndarray    # uint8  [n_comp * 2]
    cuts: np.ndarray      # uint32 [max(n_comp-1, 1)]
    n_comp: int


def pack(mix: Mixture | str) -> PackedMixture:
    if isinstance(mix, str):
        mix = mixture(mix)
    n = len(mix.shapes)
    luts = np.zeros((n, 2, LUT_SIZE), dtype=np.uint32)
    interp = np.zeros((n, 2), dtype=np.uint8)
    for k, sh in enumerate(mix.shapes):
        luts[k, 0] = sh.t_in.q
        luts[k, 1] = sh.t_out.q
        interp[k] = (sh.t_in.interp, sh.t_out.interp)
    cuts = np.array(mix.cut if mix.cut else (0,), dtype=np.uint32)
    return PackedMixture(np.ascontiguousarray(luts.ravel()), interp.ravel().copy(), cuts, n)


# ---------------------------------------------------------------- host C ----
_host_lib = None


def _load_host():
    global _host_lib
    if _host_lib is None:
        path = os.path.join(LIB_DIR, "libsynth_host.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.synth_generate_host.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_generate_host.restype = ctypes.c_int
        _host_lib = lib
    return _host_lib


def generate_host(mix: Mixture | str, seed: int, first: int, count: int,
                  out: np.ndarray | None = None) -> np.ndarray:
    """Host-C generator (OpenMP); same words as generate_np."""
    p = pack(mix)
    if out is None:
        out = np.empty(count, dtype=np.uint32)
    assert out.dtype == np.uint32 and out.flags.c_contiguous and out.size >= count
    rc = _load_host().synth_generate_host(
        p.luts.ctypes.data, p.interp.ctypes.data, p.cuts.ctypes.data, p.n_comp,
        seed, first, count, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"synth_generate_host failed rc={rc}")
    return out


# ------------------------------------------------------------------ CUDA ----
_dev_lib = None


def _load_dev():
    global _dev_lib
    if _dev_lib is None:
        path = os.path.join(LIB_DIR, "libsynth_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.synth_generate_device.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
            ctypes.c_void_p]
        lib.synth_generate_device.restype = ctypes.c_int
        _dev_lib = lib
    return _dev_lib


def generate_device(mix: Mixture | str, seed: int, first: int, count: int, out=None,
                    stream=None):
    """CUDA generator writing into a torch uint32/int32 CUDA tensor (returned)."""
    import torch
    p = pack(mix)
    dev = torch.device("cuda", torch.cuda.current_device())
    luts = torch.from_numpy(p.luts.view(np.int32)).to(dev)
    interp = torch.from_numpy(p.interp).to(dev)
    cuts = torch.from_numpy(p.cuts.view(np.int32)).to(dev)
    if out is None:
        out = torch.empty(count, dtype=torch.int32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = _load_dev().synth_generate_device(
        luts.data_ptr(), interp.data_ptr(), cuts.data_ptr(), p.n_comp,
        seed, first, count, out.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_generate_device failed rc={rc}")
    s.synchronize()   # keep the temporary tables alive until the kernel is done
    return out


# ------------------------------------------------------- raw request columns ----
def _raw_tables():
    from .shapes import category_cuts16, ratio_tables
    ratio = np.ascontiguousarray(ratio_tables().ravel())
    cuts = np.array(category_cuts16(), dtype=np.uint32)
    return ratio, cuts, len(category_cuts16()) + 1


def generate_raw_np(mix: Mixture | str, seed: int, first: int, count: int):
    """Numpy reference: (body_bytes u32, max_output u32, category u8, true_prompt u32)."""
    from .shapes import category_cuts16, ratio_tables
    if isinstance(mix, str):
        mix = mixture(mix)
    w0, w1, w2, w3 = philox_words(seed, first, count)
    comp = np.zeros(count, dtype=np.int64)
    for c in mix.cut:
        comp += (w2 >= np.uint32(c)).astype(np.int64)
    lin = np.zeros(count, dtype=np.uint64)
    lout = np.zeros(count, dtype=np.uint64)
    for k, sh in enumerate(mix.shapes):
        m = comp == k
        if m.any():
            lin[m] = _sample(sh.t_in, w0[m])
            lout[m] = _sample(sh.t_out, w1[m])
    lo = (w3 & np.uint32(0xFFFF)).astype(np.int64)
    cat = np.zeros(count, dtype=np.int64)
    for c in category_cuts16():
        cat += (lo >= c).astype(np.int64)
    r = ratio_tables()[cat, (w3 >> np.uint32(16)).astype(np.int64)].astype(np.uint64)
    body = (lin * r + np.uint64(0x8000)) >> np.uint64(16)
    return (body.astype(np.uint32), lout.astype(np.uint32), cat.astype(np.uint8), lin.astype(np.uint32))


def generate_raw_host(mix: Mixture | str, seed: int, first: int, count: int):
    p = pack(mix)
    ratio, cuts, ncat = _raw_tables()
    lib = _load_host()
    f = lib.synth_generate_raw_host
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64] + [ctypes.c_void_p] * 4
    f.restype = ctypes.c_int
    out = (np.empty(count, np.uint32), np.empty(count, np.uint32), np.empty(count, np.uint8),
           np.empty(count, np.uint32))
    rc = f(p.luts.ctypes.data, p.interp.ctypes.data, p.cuts.ctypes.data, p.n_comp, ratio.ctypes.data,
           cuts.ctypes.data, ncat, seed, first, count, *[a.ctypes.data for a in out])
    if rc != 0:
        raise RuntimeError(f"synth_generate_raw_host rc={rc}")
    return out


def generate_raw_device(mix: Mixture | str, seed: int, first: int, count: int):
    """CUDA generator: torch tensors (bytes int32, max_out int32, cat uint8, true_prompt int32)."""
    import torch
    p = pack(mix)
    ratio, cuts, ncat = _raw_tables()
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(dev)  # noqa: E731
    luts, interp, ccuts, rat, catc = t(p.luts), t(p.interp), t(p.cuts), t(ratio), t(cuts)
    out = (torch.empty(count, dtype=torch.int32, device=dev), torch.empty(count, dtype=torch.int32, device=dev),
           torch.empty(count, dtype=torch.uint8, device=dev), torch.empty(count, dtype=torch.int32, device=dev))
    lib = _load_dev()
    f = lib.synth_generate_raw_device
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64] + [ctypes.c_void_p] * 5
    f.restype = ctypes.c_int
    s = torch.cuda.current_stream(dev)
    rc = f(luts.data_ptr(), interp.data_ptr(), ccuts.data_ptr(), p.n_comp, rat.data_ptr(), catc.data_ptr(), ncat,
           seed, first, count, *[o.data_ptr() for o in out], ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_generate_raw_device rc={rc}")
    s.synchronize()
    return out


# ------------------------------------------------------------------- arrivals ----
def gaps_np(seed: int, first: int, count: int, rate_rps: float) -> np.ndarray:
    from .philox import philox4x32_10
    from .shapes import BURST_FACTORS, gap_table
    idx = np.arange(first, first + count, dtype=np.uint64)
    w0, _, _, _ = philox4x32_10(idx & np.uint64(0xFFFFFFFF), idx >> np.uint64(32), 1, 0,
                                seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    g = gap_table(rate_rps).astype(np.uint64)[(w0 >> np.uint32(16)).astype(np.int64)]
    f = np.asarray(BURST_FACTORS, dtype=np.uint64)[((idx >> np.uint64(20)) & np.uint64(7)).astype(np.int64)]
    return ((g * f) >> np.uint64(3)).astype(np.uint32)


def arrivals_host(seed: int, count: int, rate_rps: float) -> np.ndarray:
    """uint64 arrival times (ns) of requests [0, count): inclusive sum of the gaps."""
    from .shapes import BURST_FACTORS, gap_table
    gt = np.ascontiguousarray(gap_table(rate_rps))
    b8 = np.asarray(BURST_FACTORS, dtype=np.uint32)
    g = np.empty(count, dtype=np.uint32)
    lib = _load_host()
    f = lib.synth_gaps_host
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                  ctypes.c_void_p]
    f.restype = ctypes.c_int
    f(gt.ctypes.data, b8.ctypes.data, seed, 0, count, g.ctypes.data)
    return np.cumsum(g, dtype=np.uint64)


def arrivals_device(seed: int, count: int, rate_rps: float):
    """CUDA gaps + an integer prefix sum (torch.cumsum on int64: exact)."""
    import torch
    from .shapes import BURST_FACTORS, gap_table
    dev = torch.device("cuda", torch.cuda.current_device())
    gt = torch.from_numpy(np.ascontiguousarray(gap_table(rate_rps)).view(np.int32)).to(dev)
    b8 = torch.tensor(BURST_FACTORS, dtype=torch.int32, device=dev)
    g = torch.empty(count, dtype=torch.int32, device=dev)
    lib = _load_dev()
    f = lib.synth_gaps_device
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                  ctypes.c_void_p, ctypes.c_void_p]
    f.restype = ctypes.c_int
    s = torch.cuda.current_stream(dev)
    if f(gt.data_ptr(), b8.data_ptr(), seed, 0, count, g.data_ptr(), ctypes.c_void_p(s.cuda_stream)) != 0:
        raise RuntimeError("synth_gaps_device failed")
    out = torch.cumsum(g.to(torch.int64) & 0xFFFFFFFF, dim=0)
    s.synchronize()
    return out
