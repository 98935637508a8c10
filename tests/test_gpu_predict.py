"""GPU parity for the prediction snapshot (rs_predict_lengths):
LengthHistory::predict / predict_noisy (proj/src/predictor.cpp:52-98)
bitwise against the reference's own LengthHistory (oracle/_ref) or the C
restatement, from host buffers and from device tensors, and chained into the
device sweep without leaving HBM."""
import ctypes as C

import numpy as np
import pytest

from cases import Rng, predictor_cases
from oracle_lib import port, ref
from paper_2602_22718_b200 import _abi
from paper_2602_22718_b200.lib import ConfigError, check, context
from paper_2602_22718_b200.rollsim import (LengthHistory, NoiseModel, default_profile,
                                           predict_lengths)

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def oracle():
    return ref() or port()


def test_predict_host_bitwise():
    for t, (w, a, m, obs, depth, gt, ids, noise) in enumerate(predictor_cases()):
        got = predict_lengths(obs, depth, gt, w, a, m, noise, ids if noise else None)
        want = oracle().predict_lengths(obs, depth, gt, w, a, m, noise, ids)
        assert np.array_equal(bits(got), bits(want)), t


def test_predict_device_tensors_bitwise():
    import torch
    dev = torch.device("cuda", 0)
    for t, (w, a, m, obs, depth, gt, ids, noise) in enumerate(predictor_cases()[:12]):
        enc = [s.encode() for s in ids]
        blob = torch.tensor(np.frombuffer(b"".join(enc), np.uint8).copy(), device=dev)
        off = torch.tensor(np.cumsum([0] + [len(e) for e in enc]), dtype=torch.int64, device=dev)
        got = predict_lengths(torch.tensor(obs, device=dev), torch.tensor(depth, device=dev),
                              torch.tensor(gt, device=dev), w, a, m, noise, (blob, off),
                              device=True)
        want = oracle().predict_lengths(obs, depth, gt, w, a, m, noise, ids)
        assert np.array_equal(bits(got.cpu().numpy()), bits(want)), t


def test_length_history_mirror():
    """observe() bookkeeping on the host + one device snapshot, against the
    reference fed the same means."""
    h = LengthHistory(window=3, alpha=0.4, max_response_len=900)
    rng = Rng(5)
    ids = [f"p{i:06d}" for i in range(200)]
    for step in range(5):
        for pid in ids[: 50 + 30 * step]:
            h.observe(step, pid, [rng.uniform_int(1, 900) for _ in range(rng.uniform_int(1, 4))])
    prompts = [(pid, rng.uniform_int(1, 2000)) for pid in ids]
    noise = NoiseModel("bucket", 0.5, 64, 99)
    for nm in (None, noise):
        got = h.snapshot(prompts, nm)
        obs = np.zeros((200, 3))
        depth = np.zeros(200, np.int32)
        for i, (pid, _) in enumerate(prompts):
            q = h.observations(pid) or []
            depth[i] = len(q)
            obs[i, :len(q)] = q
        want = oracle().predict_lengths(obs, depth, [g for _, g in prompts], 3, 0.4, 900, nm, ids)
        assert np.array_equal(bits(got), bits(want))
    assert h.predict_noisy(prompts[7], noise) == got[7]
    with pytest.raises(ConfigError):
        LengthHistory(window=0)


def test_snapshot_feeds_device_sweep():
    """Predictions computed on the device go straight into rs_sweep_arrays
    (device_ptrs=1): same t_total / cost / N* as the oracle sweep on the
    oracle's predictions."""
    import torch
    dev = torch.device("cuda", 0)
    S, P, w = 3, 1500, 4
    rng = np.random.RandomState(11)
    depth = rng.randint(0, w + 1, S * P).astype(np.int32)
    obs = rng.randint(1, 4000, (S * P, w)).astype(np.float64)
    gt = rng.randint(1, 8000, S * P).astype(np.int32)
    plen = rng.randint(16, 1024, S * P).astype(np.int32)
    d_pred = predict_lengths(torch.tensor(obs, device=dev), torch.tensor(depth, device=dev),
                             torch.tensor(gt, device=dev), w, 0.5, 16384, device=True)
    d_plen = torch.tensor(plen, device=dev)
    Cn = 64
    outs = {k: torch.zeros(S * Cn, dtype=torch.float64, device=dev) for k in ("t", "c")}
    idle = torch.zeros(S * Cn, dtype=torch.int64, device=dev)
    ns = torch.zeros(S, dtype=torch.int32, device=dev)
    hist = torch.zeros(Cn, dtype=torch.int32, device=dev)
    st = torch.zeros(Cn, dtype=torch.float64, device=dev)
    sc = torch.zeros(Cn, dtype=torch.float64, device=dev)
    so = _abi.RsSweepOut(outs["t"].data_ptr(), outs["c"].data_ptr(), idle.data_ptr(),
                         ns.data_ptr(), hist.data_ptr(), st.data_ptr(), sc.data_ptr())
    ctx = context()
    prof = default_profile()
    s, keep = prof.struct()
    check(ctx.lib.rs_sweep_arrays(ctx.handle, d_pred.data_ptr(), d_plen.data_ptr(), S, P,
                                  C.byref(s), 8, 1, Cn, 0.7, 2, C.byref(so), 1))
    torch.cuda.synchronize()
    pred = oracle().predict_lengths(obs, depth, gt, w, 0.5, 16384)
    tt, cc, nstar = port().sweep_arrays(pred, plen, S, P, prof, 8, 1, Cn, 0.7, 2, threads=3)
    assert np.array_equal(bits(outs["t"].cpu().numpy()), bits(tt.ravel()))
    assert np.array_equal(bits(outs["c"].cpu().numpy()), bits(cc.ravel()))
    assert ns.cpu().numpy().tolist() == nstar.tolist()
