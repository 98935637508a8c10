"""CPU checks of the drop-in boundary: librs_b200.so loads without a GPU,
exports every entry point include/rs.h declares, fails loudly (no CPU
fallback) when no device is present, and its host-only helpers work."""
import ctypes as C
import pathlib
import re

import numpy as np
import pytest

from paper_2602_22718_b200 import lib

REPO = pathlib.Path(__file__).resolve().parents[1]


def declared():
    text = (REPO / "include" / "rs.h").read_text()
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = lib.load()
    names = declared()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.rs_abi_version() == 1


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lib.DeviceError, match="no CPU fallback"):
        lib.Context(0)


def test_host_only_sweep_select():
    from paper_2602_22718_b200 import sweep
    from oracle_lib import port
    rng = np.random.RandomState(1)
    for _ in range(20):
        st, sc = rng.rand(32) * 50, rng.rand(32)
        lam = float(rng.rand())
        assert sweep.aggregate_pick(st, sc, 100, 3, lam) == port().sweep_select(st, sc, 100, 3, lam)


def test_prefix_index_from_tables_roundtrip():
    from cases import csr
    from oracle_lib import port
    tok, off = csr([[1, 2, 3], [1, 2, 4], [7, 8, 9], [1, 2]])
    info, (n, a, b, c, d) = port().prefix_tables(tok, off)
    L = lib.load()
    h = C.c_void_p()
    P64 = C.POINTER(C.c_int64)
    lib.check(L.rs_prefix_index_from_tables(int(info[0]), int(info[1]), int(info[2]), int(info[3]),
                                            *[x.ctypes.data_as(P64) for x in (n, a, b, c, d)],
                                            C.byref(h)))
    out = C.c_int64()
    lib.check(L.rs_unique_prefix_count(h, 3, C.byref(out)))
    assert out.value == 4
    ln, ex = C.c_int32(), C.c_int32()
    lib.check(L.rs_select_prefix_length(h, 2, 1, 1, 3, C.byref(ln), C.byref(ex)))
    assert (ln.value, ex.value) == port().select_prefix_length(tok, off, 2, 1, 3)
    with pytest.raises(lib.ValidationError):
        lib.check(L.rs_unique_prefix_count(h, 0, C.byref(out)))
    L.rs_prefix_index_free(h)
