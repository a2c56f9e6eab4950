"""Workload configurations C1-C5 and hardware/model presets (INPUT MODULE).

Pure data: model and GPU specs (PAPER.md symbols of Eq. `kv-per-seq` and
`max-seqs`), candidate grids, the profiled-throughput table mu and
the trace recipe. Nothing here routes, counts or sizes a fleet.

mu (requests/s per instance) is an INPUT table, as in the paper ("profiled
throughput"): the paper gives no closed form for
mu(C_max). Two stated generators are provided (reading R5):
  * "table": explicit values (C1 uses Table 1: mu(8K) = 11.2, mu(65K) = 2.8,
    P:691-693);
  * "pow23": mu(C) = mu_ref * (C_ref / C) ** (2/3), an assumption anchored at
    the single paper point (Llama-3-70B, A100, C_ref = 65,536, mu_ref = 2.8)
    that reproduces Table 1's ratio (8 ** (2/3) = 4, "rho in [4, 8]").
The values are computed once on the host in float64 and handed identically to
the oracle and to the GPU path as data.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

GB = 10 ** 9   # the paper's GB is 10^9 bytes (reading R8)


@dataclass(frozen=True)
class Model:
    name: str
    n_layers: int          # n_l
    n_kv_heads: int        # n_h
    head_dim: int          # d_h
    kv_elem_bytes: int     # b_dtype
    weight_bytes: int      # total weight bytes (all GPUs of one instance)


@dataclass(frozen=True)
class Gpu:
    name: str
    hbm_bytes: int         # M_gpu
    util_num: int          # u = util_num / util_den
    util_den: int
    activation_reserve_bytes: int
    price_per_gpu_hour: float


@dataclass(frozen=True)
class Deploy:
    tp_degree: int
    weight_bytes_per_gpu: int    # M_model
    gpus_per_instance: int       # GPUs counted per instance (Q6)


MODELS = {
    # Llama-3-70B, BF16, 80 layers, 8 KV heads, d_h = 128.
    "llama3-70b": Model("llama3-70b", 80, 8, 128, 2, 141_200_000_000),
    # Qwen3-235B-A22B, 94 layers, 4 KV heads, d_h = 128, FP8 weights;
    # BF16 KV (reading R11: 23.5 KB/token/GPU needs b = 2).
    "qwen3-235b-a22b": Model("qwen3-235b-a22b", 94, 4, 128, 2, 235_000_000_000),
    # Stated presets (not in the paper).
    "llama3-8b": Model("llama3-8b", 32, 8, 128, 2, 16_060_000_000),
    "llama3-405b": Model("llama3-405b", 126, 8, 128, 2, 810_000_000_000),
    "mixtral-8x22b": Model("mixtral-8x22b", 56, 8, 128, 2, 281_000_000_000),
}

GPUS = {
    # A100-80GB, $2.21/GPU-hr.  Activation reserve 11.35 GB is the
    # [CONSTRUCTED] value of DESIGN.md reading R10 that makes Eq. `max-seqs`
    # give exactly 16 / 128 sequences at 64K / 8K for Llama-3-70B at TP=8
    # (P:40-43).
    "a100-80g": Gpu("a100-80g", 80 * GB, 9, 10, 11_350_000_000, 2.21),
    # MI300X 192 GB, u = 0.9, activations 10 GB, $3.67/GPU-hr.
    "mi300x-192g": Gpu("mi300x-192g", 192 * GB, 9, 10, 10 * GB, 3.67),
    # B200 (stated): 180 GB HGX part, u = 0.9, 10 GB activations, $6.00/GPU-hr.
    "b200-180g": Gpu("b200-180g", 180 * GB, 9, 10, 10 * GB, 6.00),
}

# Stated tensor-parallel degree per (model, GPU) (P:665 uses TP=2 for
# Llama-3-70B on A100; P:995 uses TP=8 for Qwen3 on MI300X).
TP = {
    ("llama3-8b", "a100-80g"): 1, ("llama3-8b", "b200-180g"): 1, ("llama3-8b", "mi300x-192g"): 1,
    ("llama3-70b", "a100-80g"): 2, ("llama3-70b", "b200-180g"): 2, ("llama3-70b", "mi300x-192g"): 2,
    ("qwen3-235b-a22b", "a100-80g"): 8, ("qwen3-235b-a22b", "b200-180g"): 8,
    ("qwen3-235b-a22b", "mi300x-192g"): 8,
    ("llama3-405b", "a100-80g"): 8, ("llama3-405b", "b200-180g"): 8, ("llama3-405b", "mi300x-192g"): 8,
    ("mixtral-8x22b", "a100-80g"): 4, ("mixtral-8x22b", "b200-180g"): 4,
    ("mixtral-8x22b", "mi300x-192g"): 4,
}

# Stated mu_ref (req/s/instance at C_ref = 65,536) for the pow23 generator.
# Only (llama3-70b, a100-80g) = 2.8 is the paper's (Table 1).
MU_REF = {
    ("llama3-8b", "a100-80g"): 20.0, ("llama3-8b", "b200-180g"): 60.0, ("llama3-8b", "mi300x-192g"): 40.0,
    ("llama3-70b", "a100-80g"): 2.8, ("llama3-70b", "b200-180g"): 8.4, ("llama3-70b", "mi300x-192g"): 5.6,
    ("qwen3-235b-a22b", "a100-80g"): 2.0, ("qwen3-235b-a22b", "b200-180g"): 12.0,
    ("qwen3-235b-a22b", "mi300x-192g"): 9.0,
    ("llama3-405b", "a100-80g"): 0.6, ("llama3-405b", "b200-180g"): 2.0, ("llama3-405b", "mi300x-192g"): 1.4,
    ("mixtral-8x22b", "a100-80g"): 2.0, ("mixtral-8x22b", "b200-180g"): 7.0,
    ("mixtral-8x22b", "mi300x-192g"): 5.0,
}
C_REF = 65536


def default_deploy(m: Model, g: Gpu) -> Deploy:
    tp = TP[(m.name, g.name)]
    return Deploy(tp, m.weight_bytes // tp, tp)


@dataclass(frozen=True)
class Config:
    name: str
    shape: str                  # trace mixture name (synth.shapes)
    seed: int
    n_requests: int
    rate_rps: float             # lambda
    models: tuple
    gpus: tuple
    deploy: tuple               # [n_models][n_gpus] of Deploy (flattened row-major)
    b_short: tuple              # B grid
    c_short: tuple              # C_S grid; empty => C_S = B (Fig. 6 convention)
    c_long: tuple               # C_L grid (= C_H of the homogeneous baseline)
    mu_mode: str = "pow23"      # "pow23" | "pow23cap8" | "table"
    mu_values: dict = field(default_factory=dict)   # table mode: {(m, g, C): mu}
    hours_per_year: float = 8760.0
    description: str = ""

    # ---- derived input arrays (data only) ----
    def windows(self) -> np.ndarray:
        """Sorted unique list of every pool window a candidate can use."""
        w = set(self.c_long) | (set(self.c_short) if self.c_short else set(self.b_short))
        return np.array(sorted(w), dtype=np.uint32)

    def mu_table(self) -> np.ndarray:
        """float64 [n_models][n_gpus][n_windows] requests/s per instance."""
        win = self.windows()
        mu = np.zeros((len(self.models), len(self.gpus), len(win)), dtype=np.float64)
        for i, m in enumerate(self.models):
            for j, g in enumerate(self.gpus):
                for k, c in enumerate(win):
                    if self.mu_mode == "table":
                        mu[i, j, k] = self.mu_values.get((m.name, g.name, int(c)), 0.0)
                    elif self.mu_mode == "pow23cap8":
                        # throughput gain capped at 8x mu_ref ("rho in [4, 8]")
                        r = min((C_REF / float(c)) ** (2.0 / 3.0), 8.0)
                        mu[i, j, k] = MU_REF[(m.name, g.name)] * r
                    else:
                        mu[i, j, k] = MU_REF[(m.name, g.name)] * (C_REF / float(c)) ** (2.0 / 3.0)
        return mu

    def n_cs_eff(self) -> int:
        return len(self.c_short) if self.c_short else 1

    def n_candidates(self) -> int:
        return (len(self.models) * len(self.gpus) * len(self.c_long) * self.n_cs_eff()
                * len(self.b_short))

    def deploy_at(self, i: int, j: int) -> Deploy:
        return self.deploy[i * len(self.gpus) + j]

    def with_n(self, n: int) -> "Config":
        return replace(self, n_requests=n)


def geometric_thresholds(lo: int, hi: int, n: int, multiple: int) -> tuple:
    """n thresholds geometric in [lo, hi], rounded to a multiple (may repeat)."""
    x = lo * (hi / lo) ** (np.arange(n) / (n - 1))
    return tuple(int(max(multiple, round(v / multiple) * multiple)) for v in x)


def make_config(name, shape, seed, n, rate, model_names, gpu_names, b, cs, cl,
                deploy_override=None, **kw) -> Config:
    models = tuple(MODELS[m] for m in model_names)
    gpus = tuple(GPUS[g] for g in gpu_names)
    dep = []
    for m in models:
        for g in gpus:
            d = default_deploy(m, g)
            if deploy_override and (m.name, g.name) in deploy_override:
                d = deploy_override[(m.name, g.name)]
            dep.append(d)
    return Config(name, shape, seed, n, float(rate), models, gpus, tuple(dep),
                  tuple(int(x) for x in b), tuple(int(x) for x in cs), tuple(int(x) for x in cl), **kw)


SEED0 = 20260417


def c1() -> Config:
    """C1: 1,000-request Azure-shaped trace, Llama-3-70B on A100-80GB, one split
    B = C_S = 8,192 vs homogeneous 65,536, mu from Table 1, lambda =
    1,000 req/s (Table 2).  TP=8 for the KV budget (reading R10, the
    [CONSTRUCTED] 16/128 budget) and one counted GPU per instance (Table 2
    counts "GPU instances"; reading R6)."""
    return make_config(
        "C1", "AZ", SEED0 + 1, 1000, 1000.0, ["llama3-70b"], ["a100-80g"],
        [8192], [8192], [65536],
        deploy_override={("llama3-70b", "a100-80g"): Deploy(8, 141_200_000_000 // 8, 1)},
        mu_mode="table",
        mu_values={("llama3-70b", "a100-80g", 8192): 11.2, ("llama3-70b", "a100-80g", 65536): 2.8},
        description="1e3 AZ, Llama-3-70B A100, split 8K vs homogeneous 64K, Table-1 mu")


def c2() -> Config:
    """C2: 10.3M BurstGPT-shaped (AZ) trace, 64 thresholds 512..65,536
    (geometric, multiples of 16), C_S = B, C_L = 65,536, Llama-3-70B TP=2 on B200."""
    return make_config(
        "C2", "AZ", SEED0 + 2, 10_300_000, 1000.0, ["llama3-70b"], ["b200-180g"],
        geometric_thresholds(512, 65536, 64, 16), [], [65536],
        description="10.3M AZ, 64 thresholds 512-64K, Llama-3-70B B200")


C3_MODELS = ["llama3-8b", "llama3-70b", "qwen3-235b-a22b", "llama3-405b", "mixtral-8x22b"]
C3_GPUS = ["a100-80g", "b200-180g", "mi300x-192g"]
C3_CL = [8192, 16384, 24576, 32768, 49152, 65536, 98304, 131072]


def c3(n: int = 100_000_000) -> Config:
    """C3: LMSYS-shaped trace, 5 models x 3 GPUs x 256 thresholds (256 k) x 8 C_L."""
    return make_config(
        "C3", "LM", SEED0 + 3, n, 1000.0, C3_MODELS, C3_GPUS,
        [256 * k for k in range(1, 257)], [], C3_CL,
        description=f"{n:.0e} LM, 5 models x 3 GPUs x 256 B x 8 C_L")


def c4() -> Config:
    """C4: ServeGen mixture, 1e8 requests, full (B, C_S, C_L) grid, Qwen3-235B
    TP=8 on B200, lambda = 10,000."""
    return make_config(
        "C4", "SG", SEED0 + 4, 100_000_000, 10000.0, ["qwen3-235b-a22b"], ["b200-180g"],
        geometric_thresholds(512, 65536, 64, 256),
        [1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072],
        [32768, 49152, 65536, 98304, 131072, 196608, 262144, 524288],
        description="1e8 SG, 64 B x 8 C_S x 8 C_L, Qwen3-235B B200")


C5_MODELS = ["llama3-8b", "llama3-70b", "qwen3-235b-a22b", "mixtral-8x22b"]
C5_GPUS = ["b200-180g", "mi300x-192g"]
C5_CL = [8192, 16384, 32768, 49152, 65536, 98304, 131072, 262144]


def c5(n: int = 1_000_000_000) -> Config:
    """C5: 1e9-request MIX trace, 4 models x 2 GPUs x 64 B x 8 C_L = 4,096
    candidates, lambda = 10,000."""
    return make_config(
        "C5", "MIX", SEED0 + 5, n, 10000.0, C5_MODELS, C5_GPUS,
        geometric_thresholds(512, 65536, 64, 256), [], C5_CL,
        description=f"{n:.0e} MIX, 4 models x 2 GPUs x 64 B x 8 C_L")


def k3_large(n: int = 1_000_000) -> Config:
    """ALU-regime candidate grid: 4 models x 2 GPUs x 512 B x
    64 C_S x 64 C_L = 16,777,216 candidates, all valid (B < C_S < C_L), on a
    short MIX trace. Used to measure K3 candidates/s, not a paper workload."""
    b = [16 * k for k in range(1, 513)]                      # 16 .. 8,192
    cs = [8192 + 384 * k for k in range(1, 65)]              # 8,576 .. 32,768
    cl = [32768 + 3584 * k for k in range(1, 65)]            # 36,352 .. 262,144
    return make_config("K3L", "MIX", SEED0 + 6, n, 10000.0, C5_MODELS, C5_GPUS, b, cs, cl,
                       description="2^24-candidate ALU-regime grid on a 1e6 MIX trace")


def k3_factored(n: int = 400_003) -> Config:
    """Test grid just above the cluster K3 shape's reach (2 models x 2 GPUs x
    96 B x 16 C_S x 20 C_L = 122,880 candidates; > 8,192 per model), so the
    factored K3 shape runs; C_S values are not B or C_L values (extra edges).
    Not a paper workload."""
    b = [64 * k for k in range(1, 97)]
    cs = [6144 + 512 * k for k in range(1, 17)]
    cl = [8192 + 4096 * k for k in range(0, 20)]
    return make_config("K3F", "MIX", SEED0 + 7, n, 10000.0, ["llama3-8b", "qwen3-235b-a22b"],
                       ["b200-180g", "mi300x-192g"], b, cs, cl,
                       description="122,880-candidate factored-shape test grid")


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5, "K3L": k3_large, "K3F": k3_factored}
