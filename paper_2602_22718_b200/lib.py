"""Loader for librs_b200.so (the in-tree CUDA extension) and its contexts.

There is no fallback: if the shared library is missing or no CUDA device is
visible, every call raises. `ensure_built()` compiles the library in-tree
with nvcc (sm_100a) when it is absent, which is what a fresh GPU box needs.
"""
import ctypes as C
import os
import pathlib
import subprocess
import threading

import numpy as np

from . import _abi

PKG_DIR = pathlib.Path(__file__).resolve().parent
REPO = PKG_DIR.parent
LIB_PATH = PKG_DIR / "librs_b200.so"
if os.environ.get("RS_B200_LIB"):  # A/B runs of another build of the same C-ABI
    LIB_PATH = pathlib.Path(os.environ["RS_B200_LIB"]).resolve()

RS_OK, RS_E_VALIDATION, RS_E_CONFIG, RS_E_CUDA, RS_E_NOMEM, RS_E_ARG, RS_E_PLACEMENT, RS_E_PARSE = range(8)


class Error(RuntimeError):
    """rollsim::Error (proj/include/rollsim/errors.hpp:11-14)."""


class ConfigError(Error):
    """rollsim::ConfigError (errors.hpp:17-20)."""


class ValidationError(Error):
    """rollsim::ValidationError (errors.hpp:29-32)."""


class PlacementError(Error):
    """rollsim::PlacementError (errors.hpp:35-38)."""


class ParseError(Error):
    """rollsim::ParseError (errors.hpp:23-26)."""


class DeviceError(Error):
    """CUDA failure inside librs_b200 (no reference equivalent)."""


_lock = threading.Lock()
_lib = None
_ctxs = {}


def ensure_built(force=False):
    """Compile librs_b200.so in-tree if it is missing (nvcc, sm_100a)."""
    if LIB_PATH.exists() and not force:
        return LIB_PATH
    subprocess.run(["make", "-C", str(REPO), "lib", "-j8"], check=True)
    return LIB_PATH


def load():
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(f"{LIB_PATH} is missing: run `make lib` (or __graft_entry__.build())")
            _lib = _abi.bind(C.CDLL(str(LIB_PATH)), _abi.PRODUCT_SIGS)
        return _lib


def check(status):
    if status == RS_OK:
        return
    msg = load().rs_last_error().decode(errors="replace")
    if status == RS_E_VALIDATION:
        raise ValidationError(msg)
    if status == RS_E_CONFIG:
        raise ConfigError(msg)
    if status == RS_E_PLACEMENT:
        raise PlacementError(msg)
    if status == RS_E_PARSE:
        raise ParseError(msg)
    raise DeviceError(f"rs status {status}: {msg}")


class Context:
    """One rs_ctx (device, stream, scratch arena, profile tables)."""

    def __init__(self, device=0):
        lib = load()
        h = C.c_void_p()
        check(lib.rs_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self.lib = lib

    def close(self):
        if self.handle:
            self.lib.rs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr):
        check(self.lib.rs_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def synchronize(self):
        check(self.lib.rs_ctx_synchronize(self.handle))

    def kernel_launches(self):
        v = C.c_uint64()
        check(self.lib.rs_ctx_kernel_launches(self.handle, C.byref(v)))
        return v.value

    def enable_kernel_timing(self, on=True):
        check(self.lib.rs_ctx_enable_kernel_timing(self.handle, 1 if on else 0))

    def reset_kernel_timing(self):
        check(self.lib.rs_ctx_reset_kernel_timing(self.handle))

    def kernel_time(self, name):
        ms, n = C.c_double(), C.c_uint64()
        check(self.lib.rs_ctx_kernel_time(self.handle, name.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value


def context(device=None):
    """Process-wide default context for `device` (default: $LOCAL_RANK or 0)."""
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    with _lock:
        ctx = _ctxs.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _ctxs[device] = ctx
    return ctx


# ----------------------------------------------------------- numpy helpers
def ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def as_i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def profile_struct(batch_knots, context_knots, grid, rho):
    """Build an RsProfile; returns (struct, keepalive)."""
    bk, ck = as_f64(batch_knots), as_f64(context_knots)
    g = as_f64(grid).reshape(-1)
    s = _abi.RsProfile(ptr(bk, C.c_double), len(bk), ptr(ck, C.c_double), len(ck),
                       ptr(g, C.c_double), float(rho))
    return s, (bk, ck, g)
