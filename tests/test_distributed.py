"""CPU multi-process test (gloo, world_size 2) of the sweep sharding and
combine logic (paper_2602_22718_b200/sweep.py). Per-shard partials come from
the CPU oracle, so no GPU is needed; the combined aggregates and the
aggregate N* must equal the single-process sweep."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import c4_spec
from oracle_lib import port
from paper_2602_22718_b200 import sweep
from paper_2602_22718_b200.rollsim import default_profile

S, P, N_MIN, N_MAX, LAM = 12, 384, 1, 24, 0.7


def partials(first, count):
    spec = c4_spec(count, count=P, first=first)
    pred, plen = port().generate_scenarios(spec)
    tt, cc, ns = port().sweep_arrays(pred, plen, count, P, default_profile(), 8, N_MIN, N_MAX,
                                     LAM, 2)
    hist = np.bincount(ns - N_MIN, minlength=N_MAX - N_MIN + 1).astype(np.int32)
    return tt.sum(axis=0), cc.sum(axis=0), hist


def worker(rank, world, port_no, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s0, s1 = sweep.shard_range(S, world, rank)
    st, sc, h = partials(s0, s1 - s0)
    t_st, t_sc, t_h = torch.from_numpy(st), torch.from_numpy(sc), torch.from_numpy(h)
    sweep.combine(t_st, t_sc, t_h)
    pick = sweep.aggregate_pick(t_st.numpy(), t_sc.numpy(), S, N_MIN, LAM)
    q.put((rank, t_st.numpy(), t_sc.numpy(), t_h.numpy(), pick))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_cover():
    for world in (1, 2, 3, 8):
        ranges = [sweep.shard_range(10000, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 10000
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1


@pytest.mark.timeout(300)
def test_gloo_two_ranks_combine_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    st, sc, h = partials(0, S)
    want_pick = sweep.aggregate_pick(st, sc, S, N_MIN, LAM)
    for rank, gst, gsc, gh, pick in res:
        np.testing.assert_allclose(gst, st, rtol=1e-12)
        np.testing.assert_allclose(gsc, sc, rtol=1e-12)
        assert np.array_equal(gh, h)
        assert pick == want_pick
    assert int(h.sum()) == S
    assert port().sweep_select(st, sc, S, N_MIN, LAM) == want_pick


def test_bench_relaunches_under_torchrun():
    """`bench.py --gpus N` without WORLD_SIZE re-executes itself with one
    process per GPU (the driver may launch it either way)."""
    import bench
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "2"], 4, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
