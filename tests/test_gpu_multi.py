"""Multi-GPU paths, run on a >= 2-GPU box (gpurun --gpus 2);
skipped when fewer GPUs are visible.

- rs_multi (one process, one host thread per GPU, NCCL clique inside
  librs_b200) against the single-GPU sweep: per-scenario bits identical,
  aggregates within 1e-12, the aggregate pick equal;
- rs_comm + rs_sweep_sharded in two processes (the NCCL id shipped over a
  gloo store), the same comparison;
- two contexts on two devices driven from one thread (device guard);
- `bench.py --gpus 2` relaunches itself under torchrun and reports n_gpus 2.
"""
import ctypes as C
import json
import os
import pathlib
import socket
import subprocess
import sys

import numpy as np
import pytest

from cases import c4_spec
from oracle_lib import port
from paper_2602_22718_b200 import _abi, sweep
from paper_2602_22718_b200.lib import check, context
from paper_2602_22718_b200.rollsim import default_profile

REPO = pathlib.Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


def n_gpus():
    import torch
    return torch.cuda.device_count()


need2 = pytest.mark.skipif("n_gpus() < 2", reason="needs 2 GPUs")

S, P, N_MIN, N_MAX, LAM = 601, 2048, 1, 64, 0.7


def host_out(S, Cn):
    o = {"t_total": np.zeros(S * Cn), "cost": np.zeros(S * Cn), "idle": np.zeros(S * Cn, np.int64),
         "n_star": np.zeros(S, np.int32), "hist": np.zeros(Cn, np.int32), "sum_t": np.zeros(Cn),
         "sum_c": np.zeros(Cn)}
    so = _abi.RsSweepOut(*[o[k].ctypes.data for k in
                           ("t_total", "cost", "idle", "n_star", "hist", "sum_t", "sum_c")])
    return o, so


def single(spec):
    ctx = context(0)
    o, so = host_out(spec.n_scenarios, N_MAX - N_MIN + 1)
    ps, keep = default_profile().struct()
    check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), 8, N_MIN, N_MAX, LAM, 2,
                           C.byref(so), 0))
    return o


def same(a, b, rows=None):
    for k in ("t_total", "cost"):
        x, y = a[k], b[k] if rows is None else b[k][rows]
        assert np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64)), k
    for k in ("idle", "n_star"):
        assert np.array_equal(a[k], b[k] if rows is None else b[k][rows]), k


@need2
def test_multi_sweep_matches_single_gpu():
    spec = c4_spec(S, count=P, first=9)
    want = single(spec)
    m = sweep.Multi([0, 1])
    try:
        got, so = host_out(S, N_MAX - N_MIN + 1)
        ps, keep = default_profile().struct()
        pick = C.c_int32()
        check(m.lib.rs_multi_sweep(m.handle, C.byref(spec), C.byref(ps), 8, N_MIN, N_MAX, LAM, 2,
                                   C.byref(so), C.byref(pick)))
    finally:
        m.close()
    same(got, want)
    assert np.array_equal(got["hist"], want["hist"])
    np.testing.assert_allclose(got["sum_t"], want["sum_t"], rtol=1e-12)
    np.testing.assert_allclose(got["sum_c"], want["sum_c"], rtol=1e-12)
    assert pick.value == sweep.aggregate_pick(want["sum_t"], want["sum_c"], S, N_MIN, LAM)
    # and against the C port on a few scenarios of each rank's block
    for s in (0, 299, 300, 600):
        pred, plen = port().generate_scenarios(c4_spec(1, count=P, first=9 + s))
        tt, cc, ns = port().sweep_arrays(pred, plen, 1, P, default_profile(), 8, N_MIN, N_MAX,
                                         LAM, 2)
        Cn = N_MAX - N_MIN + 1
        assert np.array_equal(got["t_total"][s * Cn:(s + 1) * Cn].view(np.uint64),
                              tt[0].view(np.uint64))
        assert got["n_star"][s] == ns[0]


@need2
def test_two_contexts_one_thread():
    """Calls alternate between contexts of GPU 0 and GPU 1 from one thread:
    each runs on its own device (RS_DEVICE_GUARD) and the caller's current
    device is left untouched."""
    import torch
    from paper_2602_22718_b200.lib import Context
    torch.cuda.set_device(0)
    a, b = Context(0), Context(1)
    spec = c4_spec(40, count=1024, first=3)
    ps, keep = default_profile().struct()
    outs = []
    for ctx in (a, b, a, b):
        o, so = host_out(40, 32)
        check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), 8, 1, 32, LAM, 2,
                               C.byref(so), 0))
        outs.append(o)
    assert torch.cuda.current_device() == 0
    for o in outs[1:]:
        same(o, outs[0])
    a.close()
    b.close()


def _rank(rank, world, port_no, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = context(rank)

    def bcast(bb):
        o = [bb]
        dist.broadcast_object_list(o, src=0)
        return o[0]

    comm = sweep.Comm(ctx, world, rank, bcast)
    spec = c4_spec(S, count=P, first=9)
    s0, s1 = sweep.shard_range(S, world, rank)
    o, so = host_out(s1 - s0, N_MAX - N_MIN + 1)
    ps, keep = default_profile().struct()
    pick = C.c_int32()
    check(ctx.lib.rs_sweep_sharded(ctx.handle, comm.handle, C.byref(spec), C.byref(ps), 8, N_MIN,
                                   N_MAX, LAM, 2, C.byref(so), 0, C.byref(pick)))
    comm.close()
    q.put((rank, s0, s1, o, pick.value))
    dist.barrier()
    dist.destroy_process_group()


@need2
@pytest.mark.timeout(600)
def test_sharded_two_processes_match_single_gpu():
    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port_no = s_.getsockname()[1]
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_rank, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=500) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = single(c4_spec(S, count=P, first=9))
    Cn = N_MAX - N_MIN + 1
    for rank, s0, s1, o, pick in res:
        rows = slice(s0 * Cn, s1 * Cn)
        for k in ("t_total", "cost", "idle"):
            assert np.array_equal(np.asarray(o[k]).view(np.uint64),
                                  np.asarray(want[k][rows]).view(np.uint64)), k
        assert np.array_equal(o["n_star"], want["n_star"][s0:s1])
        assert np.array_equal(o["hist"], want["hist"])
        np.testing.assert_allclose(o["sum_t"], want["sum_t"], rtol=1e-12)
        assert pick == sweep.aggregate_pick(want["sum_t"], want["sum_c"], S, N_MIN, LAM)


@need2
@pytest.mark.timeout(900)
def test_bench_two_gpus_relaunches():
    cmd = [sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--scenarios", "1200", "--parity-samples", "16", "--no-cpu", "--no-dedup", "--no-c5",
           "--no-c3", "--no-arrays", "--no-trace"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=850, cwd=REPO)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["parity_sampled"]["ok"] and line["parity_sampled"]["scenarios"] >= 16
    assert "NCCL INFO" in p.stdout + p.stderr  # the communicator log (rank count visible)
