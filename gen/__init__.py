"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the SST method (no window, STFT, IF,
reassignment or inverse): only the workload definitions of BASELINE.json's
configs C1-C5 and deterministic signal generators.  It is the one
module both sides may use.
"""

from .configs import CONFIGS, Config, get_config  # noqa: F401
from .signals import generate, clean_components, eq30_signal, eq30_true_ifs  # noqa: F401
