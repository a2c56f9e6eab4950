"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path.

Holds none of the method's arithmetic: Philox4x32-10, inverse-CDF length
tables, the trace recipe, and configuration data (presets, grids, mu tables).
"""
from .configs import CONFIGS, Config, GPUS, MODELS  # noqa: F401
from .gen import generate_np, generate_host, generate_device, pack  # noqa: F401
