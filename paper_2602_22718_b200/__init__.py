"""B200-native planning core of RLHFless (arXiv 2602.22718).

Drop-in GPU implementation of the reference `rollsim` hot path:
shared-prefix dedup, length-aware assignment and cost-aware actor scaling,
behind the C-ABI in include/rs.h (librs_b200.so, sm_100a).
"""
from .lib import ConfigError, DeviceError, Error, ValidationError, context, ensure_built  # noqa: F401

__version__ = "0.1.0"
