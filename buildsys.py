"""Native build for every C/CUDA artefact in the repo (used by __graft_entry__.build()).

Targets (all built in-tree so they travel to the GPU box with the snapshot):
  paper_2604_08075_b200/lib/libfleetplan.so  product: C-ABI + sm_100a kernels
  synth/lib/libsynth_gen.so                  input module: CUDA trace generator
  synth/lib/libsynth_host.so                 input module: host-C trace generator
  oracle/lib/liboracle.so                    test infrastructure: the CPU oracle
"""
from __future__ import annotations

import glob
import os
import subprocess

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def _p(*a):
    return os.path.join(ROOT, *a)


def build_oracle(verbose=False, force=False):
    src = [_p("oracle", "fleet_oracle.c")]
    out = _p("oracle", "lib", "liboracle.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if force or _stale(out, src):
        # -ffp-contract=off / no fast-math: fixed fp64 op order (reading R14)
        _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
              "-shared", "-fPIC", "-o", out] + src + ["-lm"], verbose)
    return out


def build_synth(verbose=False, force=False):
    hdr = [_p("synth", "csrc", "synth_philox.h")]
    os.makedirs(_p("synth", "lib"), exist_ok=True)
    host_src = [_p("synth", "csrc", "synth_host.c")]
    host_out = _p("synth", "lib", "libsynth_host.so")
    if force or _stale(host_out, host_src + hdr):
        _run(["gcc", "-std=c11", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", host_out] + host_src,
             verbose)
    gen_src = [_p("synth", "csrc", "synth_gen.cu")]
    gen_out = _p("synth", "lib", "libsynth_gen.so")
    if force or _stale(gen_out, gen_src + hdr):
        _run([NVCC] + ARCH + ["-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-o", gen_out]
             + gen_src, verbose)
    return host_out, gen_out


def build_product(verbose=False, force=False):
    csrc = _p("paper_2604_08075_b200", "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh"))
                  + [_p("include", "fleet_plan.h")])
    if not srcs:
        return None
    out = _p("paper_2604_08075_b200", "lib", "libfleetplan.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if force or _stale(out, srcs + hdrs):
        # --fmad=false: no FMA contraction in the fp64 candidate evaluation (R14)
        _run([NVCC] + ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-shared",
                              "-Xcompiler", "-fPIC", "-I", _p("include"), "-o", out] + srcs
             + ["-ldl"], verbose)
    return out


def build_all(verbose=False, force=False):
    build_oracle(verbose, force)
    build_synth(verbose, force)
    build_product(verbose, force)


if __name__ == "__main__":
    import sys
    build_all(verbose=True, force="-f" in sys.argv)
