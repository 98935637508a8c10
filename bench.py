"""Benchmark of the B200-native RLHFless planning core (one JSON line).

Headline (BASELINE.json metric, config C4): the cost-aware actor-scaling
sweep — 10,000 Monte-Carlo length scenarios x 256 candidate actor counts,
65,536 prompts x G=8 responses per scenario — reported as scenario x
candidate evals/s. One step = the whole sweep. Scenarios are sharded in
contiguous blocks over ranks (strong scaling: total work fixed); the only
collective is an NCCL all-reduce of the per-candidate aggregates.

  value        device-resident: scenarios generated in HBM, outputs in HBM
  e2e          the public C-ABI call with HOST output buffers (rs_sweep,
               device_ptrs=0): device->host copies inside the timed region
  roofline     dominant kernel (group_eval), CUDA events inside the run
  cpu_baseline the reference's own scale() (oracle/_ref) on host cores
  dedup        secondary metric (C2 prefix dedup, tokens/s), same fields

`--impl reference` runs only the reference CPU arm (rank 0), same metric.
"""
import argparse
import ctypes as C
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

METRIC = "scenario×candidate evals/sec (scaling sweep)"
EVAL_BYTES = 65536 * 12 + 16  # P*(8 B pred + 4 B plen) + 16 B out


def _profile_traffic(key):
    """ncu DRAM read + write per launch of a kernel (profiles/kernel_counters.json), or None."""
    tf = REPO / "profiles" / "kernel_counters.json"
    if not tf.exists():
        return None
    return json.loads(tf.read_text()).get(key)


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every 10 ms from a thread (nvidia-ml-py), so even a 40 ms timed
    region gets samples; `nvidia-smi -lms 200` is the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                  "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device, pci_bus_id=None):
        self.device, self.pci = device, pci_bus_id
        self.sm, self.max_mhz, self.reasons = [], None, set()
        self.stop = threading.Event()
        self.proc = self.t = None
        self.source = None

    def _nvml_loop(self, nv, h):
        masks = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(name for name, m in masks if m and r & m)
            except Exception:  # noqa: BLE001 — sampling must never break the bench
                pass
            self.stop.wait(0.01)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
                except Exception:  # noqa: BLE001
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.t.start()
            self.source = "nvml/10ms"
            return self
        except Exception:  # noqa: BLE001
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.SMI_FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._smi_loop, daemon=True)
            self.t.start()
            self.source = "nvidia-smi/200ms"
        except OSError:
            self.proc = None
        return self

    def _smi_loop(self):
        names = [n for n, _ in self.REASONS[:4]]
        for ln in self.proc.stdout:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                self.sm.append(float(f[1]))
                self.max_mhz = float(f[2])
            except ValueError:
                continue
            self.reasons.update(n for n, v in zip(names, f[5:9]) if v.lower() == "active")

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0, "source": self.source}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return
    from cases import c4_spec
    from oracle_lib import port, ref
    from paper_2602_22718_b200.rollsim import default_profile
    R = ref()
    kind = "reference" if R is not None else "port"
    impl = R if R is not None else port()
    threads = os.cpu_count() or 1
    n_cand = args.n_max - args.n_min + 1
    prof = default_profile()
    times = []
    for step in range(args.warmup + args.steps):
        spec = c4_spec(threads, count=args.prompts, first=step * threads)
        pred, plen = port().generate_scenarios(spec)
        t0 = time.perf_counter()
        impl.sweep_arrays(pred, plen, threads, args.prompts, prof, args.G, args.n_min,
                          args.n_max, args.lam, 2, threads=threads)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    evals = threads * n_cand
    v = evals * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Monte-Carlo scenarios, DESIGN.md §4.1)",
        "config": config(args, world),
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": threads, "kind": kind,
                         "sample": f"{threads} scenarios x {n_cand} candidates per step "
                                   f"(one scenario per thread), {args.prompts} prompts x G={args.G}"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config(args, world):
    return {"workload": f"C4 actor-scaling sweep: {args.scenarios} scenarios x "
                        f"{args.n_max - args.n_min + 1} candidate N, {args.prompts} prompts x "
                        f"G={args.G} per scenario",
            "scenarios": args.scenarios, "candidates": [args.n_min, args.n_max],
            "prompts": args.prompts, "G": args.G, "lambda": args.lam, "gpus_per_actor": 2,
            "profile": "default_profile()", "parallelism": f"scenario-sharded x{world}",
            "l2": "inputs larger than L2 (per-batch scenario structures of several GiB: "
                  "~6 MB per scenario, batches of up to 2,048 scenarios planned in whole waves)"}


# ----------------------------------------------------------------- our arm
def cpu_baseline_sweep(args):
    from cases import c4_spec
    from oracle_lib import port, ref
    from paper_2602_22718_b200.rollsim import default_profile
    R = ref()
    kind = "reference" if R is not None else "port"
    impl = R if R is not None else port()
    threads = os.cpu_count() or 1
    n = threads * args.cpu_rounds
    pred, plen = port().generate_scenarios(c4_spec(n, count=args.prompts, first=0))
    t0 = time.perf_counter()
    impl.sweep_arrays(pred, plen, n, args.prompts, default_profile(), args.G, args.n_min,
                      args.n_max, args.lam, 2, threads=threads)
    dt = time.perf_counter() - t0
    n_cand = args.n_max - args.n_min + 1
    # one thread: the reference's own single-threaded scale(), 2 scenarios
    p1, l1 = port().generate_scenarios(c4_spec(2, count=args.prompts, first=n))
    t1 = time.perf_counter()
    impl.sweep_arrays(p1, l1, 2, args.prompts, default_profile(), args.G, args.n_min,
                      args.n_max, args.lam, 2, threads=1)
    d1 = time.perf_counter() - t1
    return {"value": n * n_cand / dt, "unit": "evals/s", "cores": threads, "kind": kind,
            "cpu_model": cpu_model(),
            "one_thread_value": 2 * n_cand / d1,
            "sample": f"{n} scenarios x {n_cand} candidates ({args.prompts} prompts x G={args.G}), "
                      f"{threads} threads, {dt:.1f} s; one thread: 2 scenarios, {d1:.1f} s"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def counters(key):
    """ncu counters per unit of the dominant kernels (profiles/kernel_counters.json,
    written from a committed `ncu --set full` capture by tools/kernel_counters.py)."""
    f = REPO / "profiles" / "kernel_counters.json"
    if not f.exists():
        return None
    return json.loads(f.read_text()).get(key)


def parity_sample(args, world, rank, S_local, s0, t_total, cost, idle, n_star, n_cand):
    """Bitwise check against the C port, outside the timed region: at N=1
    every scenario of the sweep (~1 minute on the host cores), at N>1 (or
    with --parity-sampled-only) --parity-samples scenarios spread over every
    batch of every rank's block, first and last included."""
    import torch
    from cases import c4_spec
    from oracle_lib import port
    from paper_2602_22718_b200.rollsim import default_profile
    if S_local == 0:
        return 0, True
    full = args.parity_full or (world == 1 and not args.parity_sampled_only)
    want = S_local if full else max(1, -(-args.parity_samples // world))
    idx = np.unique(np.linspace(0, S_local - 1, min(want, S_local)).round().astype(np.int64))
    tt_d = t_total.view(S_local, n_cand).cpu().numpy()
    cc_d = cost.view(S_local, n_cand).cpu().numpy()
    id_d = idle.view(S_local, n_cand).cpu().numpy()
    ns_d = n_star.cpu().numpy()
    threads = max(1, (os.cpu_count() or 1) // world)
    ok = True
    prof = default_profile()
    chunk = 256
    for c0 in range(0, len(idx), chunk):
        sel = idx[c0:c0 + chunk]
        if sel[-1] - sel[0] + 1 == len(sel):  # a contiguous block: one generator call
            pred, plen = port().generate_scenarios(c4_spec(len(sel), count=args.prompts,
                                                           first=s0 + int(sel[0])))
            preds = np.split(pred, len(sel))
        else:
            preds, plens = [], []
            for s in sel:  # each sampled scenario generated by the port itself
                p, l = port().generate_scenarios(c4_spec(1, count=args.prompts, first=s0 + int(s)))
                preds.append(p)
                plens.append(l)
            pred, plen = np.concatenate(preds), np.concatenate(plens)
        tt, cc, ns = port().sweep_arrays(pred, plen, len(sel), args.prompts, prof, args.G,
                                         args.n_min, args.n_max, args.lam, 2, threads=threads)
        ok &= bool(np.array_equal(tt.view(np.uint64), tt_d[sel].view(np.uint64)))
        ok &= bool(np.array_equal(cc.view(np.uint64), cc_d[sel].view(np.uint64)))
        ok &= bool(np.array_equal(ns, ns_d[sel]))
        # idle slot-ticks per scenario on the host threads (the port's C call
        # releases the GIL)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            idles = list(ex.map(lambda p: port().scale_idle(p, None, args.G, args.n_min, args.n_max),
                                preds))
        for j, s in enumerate(sel):
            ok &= bool(np.array_equal(idles[j], id_d[s]))
    return len(idx), ok


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist
    from cases import c4_spec
    from paper_2602_22718_b200 import _abi, sweep
    from paper_2602_22718_b200.lib import check, context, ensure_built
    from paper_2602_22718_b200.rollsim import default_profile

    ensure_built()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = context(local)
    lib = ctx.lib
    # A dedicated torch stream shared with the library so CUDA events order
    # against our kernels (NULL would select the context's own stream).
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    comm = None
    if world > 1:  # librs_b200's own NCCL communicator for the one aggregate all-reduce
        def bcast(b):
            o = [b]
            dist.broadcast_object_list(o, src=0)
            return o[0]
        comm = sweep.Comm(ctx, world, rank, bcast)
    prof = default_profile()
    ps, keep = prof.struct()
    n_cand = args.n_max - args.n_min + 1
    s0, s1 = sweep.shard_range(args.scenarios, world, rank)
    S = s1 - s0
    spec_all = c4_spec(args.scenarios, count=args.prompts, first=0)
    spec_local = c4_spec(S, count=args.prompts, first=s0)
    t_total = torch.empty(max(S, 1) * n_cand, dtype=torch.float64, device=dev)
    cost = torch.empty_like(t_total)
    idle = torch.empty(max(S, 1) * n_cand, dtype=torch.int64, device=dev)
    n_star = torch.empty(max(S, 1), dtype=torch.int32, device=dev)
    agg_t = torch.empty(n_cand, dtype=torch.float64, device=dev)
    agg_c = torch.empty(n_cand, dtype=torch.float64, device=dev)
    agg_h = torch.empty(n_cand, dtype=torch.int32, device=dev)
    out_dev = _abi.RsSweepOut(t_total.data_ptr(), cost.data_ptr(), idle.data_ptr(),
                              n_star.data_ptr(), agg_h.data_ptr(), agg_t.data_ptr(),
                              agg_c.data_ptr())
    pick = C.c_int32()

    def sweep_call(out, device_ptrs):
        if comm is not None:
            check(lib.rs_sweep_sharded(ctx.handle, comm.handle, C.byref(spec_all), C.byref(ps),
                                       args.G, args.n_min, args.n_max, args.lam, 2, C.byref(out),
                                       device_ptrs, C.byref(pick)))
        else:
            check(lib.rs_sweep(ctx.handle, C.byref(spec_local), C.byref(ps), args.G, args.n_min,
                               args.n_max, args.lam, 2, C.byref(out), device_ptrs))

    def step_device():
        sweep_call(out_dev, 1)

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(k):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches()
    pci = None
    try:
        pr = torch.cuda.get_device_properties(local)
        pci = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
    except Exception:  # noqa: BLE001
        pci = None
    with ClockSampler(local, pci) as clk:
        ms = timed(step_device, args.steps)
    launches = (ctx.kernel_launches() - launches0) // args.steps
    # per-kernel attribution: the same steps again with per-kernel CUDA-event
    # timing on (kept out of the timed region above)
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    attr_ms = timed(step_device, args.steps)
    kt = {k: ctx.kernel_time(k) for k in ("group_eval", "fast_build", "group_table", "finish",
                                          "aggregate", "fast_tables", "pack_aggregates")}
    ctx.enable_kernel_timing(False)
    total_evals = args.scenarios * n_cand
    value = total_evals * args.steps / (ms / 1e3)

    # e2e: the same public call with host (pinned) output buffers
    pin = {k: torch.empty(max(S, 1) * n_cand, dtype=t, pin_memory=True)
           for k, t in (("t", torch.float64), ("c", torch.float64), ("i", torch.int64))}
    pin_ns = torch.empty(max(S, 1), dtype=torch.int32, pin_memory=True)
    pin_agg = [torch.empty(n_cand, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    pin_h = torch.empty(n_cand, dtype=torch.int32, pin_memory=True)
    out_host = _abi.RsSweepOut(pin["t"].data_ptr(), pin["c"].data_ptr(), pin["i"].data_ptr(),
                               pin_ns.data_ptr(), pin_h.data_ptr(), pin_agg[0].data_ptr(),
                               pin_agg[1].data_ptr())
    d2h = S * n_cand * 24 + S * 4 + n_cand * 20
    h2d = C.sizeof(spec_all) + 8 * (9 + 5 + 45)
    sweep_call(out_host, 0)
    e2e_steps = max(1, args.steps // 2)
    e2e_ms = timed(lambda: sweep_call(out_host, 0), e2e_steps) / e2e_steps
    e2e = total_evals / (e2e_ms / 1e3)

    # bit-exactness of sampled scenarios of every rank's block (outside timing)
    sweep_call(out_dev, 1)
    torch.cuda.synchronize()
    n_chk, ok = (0, None)
    if args.check:
        n_chk, ok = parity_sample(args, world, rank, S, s0, t_total, cost, idle, n_star, n_cand)
        if world > 1:
            v = torch.tensor([n_chk, 1 if ok else 0], dtype=torch.int64, device=dev)
            dist.all_reduce(v[:1])
            dist.all_reduce(v[1:], op=dist.ReduceOp.MIN)
            n_chk, ok = int(v[0].item()), bool(v[1].item())

    peak, peak_kind = peaks()
    ge_ms, ge_n = kt["group_eval"]
    ge_avg_ms = ge_ms / max(ge_n, 1)
    per_launch_evals = total_evals / world * args.steps / max(ge_n, 1)
    clocks = clk.summary()
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    # The dominant kernel is issue-bound integer + FP64-scalar code (no
    # contraction, DRAM ~3 % busy): its roofline is the SM issue rate, 4 warp
    # instructions per SM per cycle. achieved = ncu's warp instructions per
    # eval (committed capture) x evals per launch / the live launch time.
    inst_pe = counters("group_eval_inst_issued_per_eval")
    dram_pe = counters("group_eval_dram_bytes_per_eval")
    issue_peak = n_sm * 4 * sm_mhz * 1e6 / 1e9  # G warp-inst/s
    achieved_issue = (inst_pe * per_launch_evals / (ge_avg_ms / 1e3) / 1e9) if inst_pe else None
    traffic = dram_pe * per_launch_evals if dram_pe else None
    ref_equiv = per_launch_evals * EVAL_BYTES / (ge_avg_ms / 1e3) / 1e9
    result = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated Monte-Carlo scenarios, DESIGN.md §4.1)",
        "config": config(args, world),
        "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h * world,
                "path": "rs_sweep / rs_sweep_sharded with pinned host outputs (C-ABI)"},
        "roofline": {
            "bound": "issue", "kernel": "group_eval (lockstep_eval_kernel)",
            "achieved": achieved_issue, "peak": issue_peak, "unit": "G warp-inst/s",
            "frac": achieved_issue / issue_peak if achieved_issue else None,
            "inst_issued_per_eval": inst_pe, "sm_mhz": sm_mhz, "sms": n_sm,
            "traffic": traffic,
            "dram_frac": (traffic / (ge_avg_ms / 1e3) / 1e9 / peak) if traffic else None,
            "hbm_peak_gbs": peak, "peak_kind": peak_kind,
            "ref_equiv_frac": ref_equiv / peak,
            "ref_equiv_note": "SURVEY §8d reference-equivalent bytes (786,448 B per eval) / HBM peak; "
                              "reuse accounting, not a bound",
            "launch_ms": ge_avg_ms, "evals_per_launch": per_launch_evals,
            "counters_source": "profiles/kernel_counters.json",
            "kernel_share_of_step": ge_ms / attr_ms if attr_ms else None},
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items() if v[1]},
        "gpu_launches": int(launches),
        "parity_sampled": {"scenarios": n_chk, "ok": ok, "of": args.scenarios,
                           "fields": "t_total, cost, idle_slot_ticks, n_star bitwise vs oracle/rs_oracle.c"},
    }
    if world > 1 and not args.no_c5:
        its, err = bench_c5_replicas(world, rank, local)
        v = torch.tensor([its, 1.0 if err is None else 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(v[:1])
        dist.all_reduce(v[1:], op=dist.ReduceOp.MIN)
        result["c5_replicas"] = {"metric": "C5 iterations/sec, one independent replica per GPU",
                                 "value": float(v[0].item()), "unit": "iterations/s",
                                 "replicas": world, "steps_each": 200, "all_ok": bool(v[1].item())}
    if comm is not None:
        result["n_star_aggregate"] = pick.value
        result["collective"] = "one NCCL all-reduce of 3 x C doubles inside librs_b200 (rs_sweep_sharded)"
    if rank == 0:
        result["clocks"] = clocks
        if world == 1 and not args.no_arrays:
            result["e2e_arrays"] = bench_arrays(args, ctx, torch, dev, ps)
        if world == 1 and not args.no_c3:
            result["c3"] = bench_c3(args)
        if world == 1 and not args.no_dedup:
            result["dedup"] = bench_dedup(args, ctx, torch, dev, stream)
        if world == 1 and not args.no_cpu:
            result["cpu_baseline"] = cpu_baseline_sweep(args)
        if world == 1 and not args.no_c5:
            result["c5"] = bench_c5()
        if world == 1 and not args.no_trace:
            result["trace"] = bench_trace(args, ctx, torch, dev)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:  # last, after every communicator log line
        if world > 1:
            nccl_log_summary()
        sys.stderr.flush()
        print(json.dumps(result), flush=True)


def bench_arrays(args, ctx, torch, dev, ps):
    """The sweep over CALLER arrays (rs_sweep_arrays: the reference API's input
    form, predicted lengths from the caller) with pinned HOST inputs and
    outputs: every step copies S x P x 12 B of inputs in (batch i+1's H2D on
    its own stream while batch i computes) and the results out."""
    from cases import c4_spec
    from paper_2602_22718_b200 import _abi
    from paper_2602_22718_b200.lib import check
    S, P, n_cand = args.arrays_scenarios, args.prompts, args.n_max - args.n_min + 1
    pred = torch.empty(S * P, dtype=torch.float64, pin_memory=True)
    plen = torch.empty(S * P, dtype=torch.int32, pin_memory=True)
    spec = c4_spec(S, count=P, first=0)
    check(ctx.lib.rs_generate_scenarios(ctx.handle, C.byref(spec), C.c_void_p(pred.data_ptr()),
                                        C.c_void_p(plen.data_ptr()), 0))
    outs = [torch.empty(S * n_cand, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    idle = torch.empty(S * n_cand, dtype=torch.int64, pin_memory=True)
    ns = torch.empty(S, dtype=torch.int32, pin_memory=True)
    so = _abi.RsSweepOut(outs[0].data_ptr(), outs[1].data_ptr(), idle.data_ptr(), ns.data_ptr(),
                         None, None, None)

    def call():
        check(ctx.lib.rs_sweep_arrays(ctx.handle, C.c_void_p(pred.data_ptr()),
                                      C.c_void_p(plen.data_ptr()), S, P, C.byref(ps), args.G,
                                      args.n_min, args.n_max, args.lam, 2, C.byref(so), 0))

    call()
    torch.cuda.synchronize()
    k = 2
    t0 = time.perf_counter()
    for _ in range(k):
        call()
    dt = (time.perf_counter() - t0) / k
    return {"metric": METRIC + " from caller arrays", "value": S * n_cand / dt, "unit": "evals/s",
            "ms_per_step": dt * 1e3, "scenarios": S,
            "h2d_bytes_per_step": S * P * 12, "d2h_bytes_per_step": S * n_cand * 24 + S * 4,
            "h2d_gbs": S * P * 12 / dt / 1e9,
            "path": "rs_sweep_arrays, pinned host inputs and outputs (host wall clock)"}


def bench_c3(args):
    """C3 (BASELINE config 3): scale() over one 65,536-prompt x G=8 scenario,
    N in [1, 512], through the C++ drop-in (rollsim::scale over the C-ABI)
    and the unmodified reference, both on this host (build/shim/c3_bench_*)."""
    from cases import c4_spec
    from oracle_lib import port
    out = {}
    pred, plen = port().generate_scenarios(c4_spec(1, count=65536, first=0))
    path = REPO / "gpurun_out" / "c3_scenario.bin"
    path.parent.mkdir(exist_ok=True)
    with open(path, "wb") as f:
        f.write(np.int64(len(pred)).tobytes() + pred.tobytes() + plen.astype(np.int32).tobytes())
    for arm, reps in (("b200", 20), ("ref", 1)):
        exe = REPO / "build" / "shim" / f"c3_bench_{arm}"
        if not exe.exists():
            return {"unavailable": "build/shim not built (make shim)"}
        cmd = [str(exe), str(path), str(reps), "512"] + (["nowarm"] if arm == "ref" else [])
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        if p.returncode != 0:
            return {"unavailable": f"c3_bench_{arm} exit {p.returncode}: {p.stderr[-300:]}"}
        out[arm] = json.loads(p.stdout.strip().splitlines()[-1])
    b, r = out["b200"], out["ref"]
    return {"metric": "C3 scale() calls/sec (65,536 prompts x G=8, N in [1, 512])",
            "value": 1e3 / b["ms_per_call"], "unit": "calls/s", "ms_per_call": b["ms_per_call"],
            "evals_per_s": 512 * 1e3 / b["ms_per_call"],
            "reference_ms_per_call": r["ms_per_call"],
            "identical_to_reference": b["digest"] == r["digest"] and b["n_star"] == r["n_star"],
            "n_star": b["n_star"], "path": "rollsim::scale (C++ drop-in, string ids ranked on the "
                                           "device, groups of N* materialised) vs the reference",
            "cpu_baseline": {"value": 1e3 / r["ms_per_call"], "unit": "calls/s", "cores": 1,
                             "kind": "reference", "sample": "one scale() call, 1 thread"}}


def trace_parity(d_text, tok, off, fmt, n=65536, g=8, seed=1):
    """One parse (outside the timed region) checked against what the text
    encodes (tests/cases.py's generator): the id-sorted token CSR (ids
    p000000.. sort in prompt order), and the step table — one step, the batch
    in the generator's order with its g lengths per prompt."""
    from paper_2602_22718_b200.rollsim import TraceCSR
    tr = TraceCSR(d_text, device=True, fmt=fmt)
    got, st = tr.host(), tr.steps()
    rng = np.random.RandomState(seed + 1)
    order = rng.permutation(n)
    lens = rng.randint(1, 2049, (n, g))
    ok = (np.array_equal(got["tokens"], tok) and np.array_equal(got["offsets"], off)
          and st["step_idx"].tolist() == [0] and np.array_equal(st["entry_prompt"], order)
          and np.array_equal(st["lengths"], lens))
    del tr
    return {"ok": bool(ok), "fields": "tokens, offsets, step entries and lengths bitwise",
            "vs": "the generator of the text (tests/cases.py)"}


def bench_trace(args, ctx, torch, dev):
    """the C2 batch written as a CSV trace (~1 GB of text,
    tests/cases.py c2_trace_text) -> id-sorted token CSR in HBM
    (rs_trace_csr_parse), tokens/s. value: text already in HBM; e2e: from
    pinned host text; cpu_baseline: the reference's trace_from_string on the
    same trace shape cut to 4,096 prompts. The trace carries one step
    scheduling the whole batch (g = 8 rows per prompt, 524,288 step rows),
    parsed into the step table in the same call."""
    from cases import c2_trace_text
    from paper_2602_22718_b200.lib import check
    text, tok, off = c2_trace_text()
    n_tok = int(tok.size)
    d_text = torch.from_numpy(text).to(dev)
    h = C.c_void_p()
    lib = ctx.lib

    def parse(ptr, device):
        check(lib.rs_trace_csr_parse(ctx.handle, C.c_void_p(ptr), text.nbytes, device, C.byref(h)))
        lib.rs_trace_csr_free(h)

    for _ in range(3):
        parse(d_text.data_ptr(), 1)
    k = 10
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        parse(d_text.data_ptr(), 1)
    dev_s = (time.perf_counter() - t0) / k
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    parse(d_text.data_ptr(), 1)
    kt = {n: ctx.kernel_time(n)[0] for n in ("trace_classify", "trace_tokens", "trace_nl_write",
                                             "trace_steprow", "trace_group", "trace_line_flags",
                                             "trace_line_compact", "scan_apply")}
    ctx.enable_kernel_timing(False)
    pt = torch.from_numpy(text).pin_memory()
    parse(pt.data_ptr(), 0)
    t0 = time.perf_counter()
    for _ in range(3):
        parse(pt.data_ptr(), 0)
    host_s = (time.perf_counter() - t0) / 3
    peak, _ = peaks()
    top = max(kt, key=kt.get)
    achieved = text.nbytes / (kt[top] / 1e3) / 1e9  # the dominant pass reads the text once
    parity = trace_parity(d_text, tok, off, "csv")
    out = {"metric": "trace prompt-table parse tokens/sec (CSV -> device CSR)", "value": n_tok / dev_s,
           "unit": "tokens/s", "text_bytes": int(text.nbytes), "ms_per_parse": dev_s * 1e3,
           "config": {"workload": "C2 batch as CSV trace text: 65536 '# prompt' lines x 2560 tokens "
                                  "+ one step of 65536 x 8 rows"},
           "e2e": {"value": n_tok / host_s, "unit": "tokens/s", "h2d_bytes_per_step": int(text.nbytes),
                   "d2h_bytes_per_step": 0},
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "kernel": top,
                        "traffic": (_profile_traffic("trace_tokens_dram_bytes_per_launch")
                                    if top == "trace_tokens" else None),
                        "launch_ms": kt[top], "kernel_ms": kt},
           "parity": parity}
    if not args.no_cpu:
        from oracle_lib import ref
        R = ref()
        if R is not None:
            sample = c2_trace_text(n_prompts=4096)[0].tobytes()
            t0 = time.perf_counter()
            R.trace_prompts(sample)
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": 4096 * 2560 / dt, "unit": "tokens/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"4,096 prompts + 32,768 step rows ({len(sample) / 1e6:.0f} MB), "
                                             f"trace_from_string, {dt:.1f} s"}
    out["jsonl"] = bench_trace_jsonl(args, ctx, torch, dev)
    return out


def bench_trace_jsonl(args, ctx, torch, dev):
    """The same trace in the JSONL form (tests/cases.py c2_trace_jsonl: the
    whole prompt table on one ~1 GB header line, one step object) through
    rs_trace_csr_parse_jsonl; cpu_baseline: the reference's nlohmann reader
    on the same shape cut to 1,024 prompts."""
    from cases import c2_trace_jsonl
    from paper_2602_22718_b200.lib import check
    text, tok, off = c2_trace_jsonl()
    n_tok = int(tok.size)
    d_text = torch.from_numpy(text).to(dev)
    h = C.c_void_p()
    lib = ctx.lib

    def parse(ptr, device):
        check(lib.rs_trace_csr_parse_jsonl(ctx.handle, C.c_void_p(ptr), text.nbytes, device, C.byref(h)))
        lib.rs_trace_csr_free(h)

    for _ in range(2):
        parse(d_text.data_ptr(), 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        parse(d_text.data_ptr(), 1)
    dev_s = (time.perf_counter() - t0) / 5
    pt = torch.from_numpy(text).pin_memory()
    parse(pt.data_ptr(), 0)
    t0 = time.perf_counter()
    for _ in range(3):
        parse(pt.data_ptr(), 0)
    host_s = (time.perf_counter() - t0) / 3
    parity = trace_parity(d_text, tok, off, "jsonl")
    out = {"metric": "trace JSONL parse tokens/sec (JSONL -> device CSR + step table)",
           "value": n_tok / dev_s, "unit": "tokens/s", "text_bytes": int(text.nbytes),
           "ms_per_parse": dev_s * 1e3,
           "config": {"workload": "C2 batch as a JSONL trace: one 65536-prompt header line x 2560 tokens "
                                  "+ one step of 65536 x 8 lengths"},
           "e2e": {"value": n_tok / host_s, "unit": "tokens/s", "h2d_bytes_per_step": int(text.nbytes),
                   "d2h_bytes_per_step": 0},
           "parity": parity}
    if not args.no_cpu:
        from oracle_lib import ref
        R = ref()
        if R is not None:
            sample = c2_trace_jsonl(n_prompts=1024)[0].tobytes()
            t0 = time.perf_counter()
            R.trace_prompts(sample, "jsonl")
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": 1024 * 2560 / dt, "unit": "tokens/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"1,024 prompts + 8,192 lengths ({len(sample) / 1e6:.0f} MB), "
                                             f"trace_from_string(jsonl), {dt:.1f} s"}
    return out


def c5_run(arm, steps, seed=11, checkpoint=None, device=None, timeout=1800, run=None):
    exe = REPO / "build" / "shim" / f"c5_bench_{arm}"
    if not exe.exists():
        return None, "build/shim not built (make shim)"
    env = dict(os.environ)
    if device is not None:
        env["RS_DEVICE"] = str(device)
    cmd = [str(exe), str(steps), "512", str(seed), str(checkpoint or steps), str(run or steps)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    if p.returncode != 0:
        return None, f"c5_bench_{arm} exit {p.returncode}: {p.stderr[-300:]}"
    return json.loads(p.stdout.strip().splitlines()[-1]), None


def bench_c5(steps=1000, compare=50):
    """C5 (BASELINE config 5): the reference's own
    run_training(rlhfless) on default_topology(128, 8, 4) — 1,024 simulated
    GPUs, 512 prompts x G=8 — for the configured 1,000 iterations, linked
    against the drop-in with training.cpp patched as INTEGRATION.md describes
    (c5_bench_train). The unmodified reference (c5_bench_ref) and the drop-in
    under the stock training.cpp (c5_bench_b200) run the first `compare`
    iterations of the same trace; all three must agree bit for bit there
    (digest over those iterations)."""
    train, err = c5_run("train", steps, checkpoint=compare)
    if err:
        return {"unavailable": err}
    ref, err = c5_run("ref", steps, run=compare)  # the same 1,000-step trace, first iterations
    if err:
        return {"unavailable": err}
    b200, err = c5_run("b200", steps, run=compare)
    if err:
        return {"unavailable": err}
    same = train["digest_checkpoint"] == ref["digest"] == b200["digest"]
    return {"metric": "C5 iterations/sec (run_training, simulated 1,024-GPU cluster)",
            "value": train["iterations_per_s"], "unit": "iterations/s", "steps": steps,
            "plan_ms_per_step": train["plan_ms_per_step"],
            "path": "reference run_training, training.cpp + shim/patches/training_b200.patch, "
                    "drop-in planner on the GPU",
            "identical_to_reference_first_steps": {"steps": compare, "ok": same},
            "reference": {"value": ref["iterations_per_s"], "steps": compare,
                          "plan_ms_per_step": ref["plan_ms_per_step"]},
            "dropin_stock_training": {"value": b200["iterations_per_s"], "steps": compare,
                                      "plan_ms_per_step": b200["plan_ms_per_step"]},
            "cpu_baseline": {"value": ref["iterations_per_s"], "unit": "iterations/s", "cores": 1,
                             "kind": "reference", "sample": f"first {compare} iterations"},
            "config": train["config"]}


def bench_c5_replicas(world, rank, local, steps=200):
    """C5 at N GPUs (replicas only — the loop is sequential
    through predictor state, training.cpp:303-317): every rank runs one
    independent replica (seed 11 + rank) on its own GPU; the aggregate is the
    sum of the replicas' iterations/s."""
    r, err = c5_run("train", steps, seed=11 + rank, device=local)
    return (r["iterations_per_s"] if r else 0.0), err


def bench_dedup(args, ctx, torch, dev, stream):
    """C2: PrefixIndex::build over 65,536 x 2,560 tokens (2,048 shared)."""
    from cases import c2_tokens
    from paper_2602_22718_b200.lib import check
    tok, off = c2_tokens()
    n_tok = int(tok.size)
    d_tok = torch.from_numpy(tok).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    h = C.c_void_p()
    lib = ctx.lib

    def build_dev():
        check(lib.rs_prefix_index_build_device(ctx.handle, C.c_void_p(d_tok.data_ptr()),
                                               C.c_void_p(d_off.data_ptr()), len(off) - 1,
                                               C.byref(h)))
        lib.rs_prefix_index_free(h)

    for _ in range(3):
        build_dev()
    k = 20
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        build_dev()
    torch.cuda.synchronize()
    dev_s = (time.perf_counter() - t0) / k
    # per-kernel attribution in a separate pass (event timing off above)
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    for _ in range(5):
        build_dev()
    cmp_ms, cmp_n = ctx.kernel_time("dedup_compare_r0")
    ctx.enable_kernel_timing(False)
    pt = torch.from_numpy(tok).pin_memory()
    po = torch.from_numpy(off).pin_memory()
    tptr = pt.numpy().ctypes.data_as(C.POINTER(C.c_int32))
    optr = po.numpy().ctypes.data_as(C.POINTER(C.c_int64))

    def build_host():
        check(lib.rs_prefix_index_build(ctx.handle, tptr, optr, len(off) - 1, C.byref(h)))
        lib.rs_prefix_index_free(h)

    build_host()
    t0 = time.perf_counter()
    for _ in range(3):
        build_host()
    host_s = (time.perf_counter() - t0) / 3
    peak, _ = peaks()
    r0_ms = cmp_ms / max(cmp_n, 1)
    achieved = n_tok * 4 / (r0_ms / 1e3) / 1e9
    out = {
        "metric": "prefix-dedup tokens/sec", "value": n_tok / dev_s, "unit": "tokens/s",
        "config": {"workload": "C2 prefix dedup: 65536 prompts x (2048 shared + 512 unique) "
                               "tokens, vocab 32000", "tokens": n_tok},
        "ms_per_build": dev_s * 1e3,
        "e2e": {"value": n_tok / host_s, "unit": "tokens/s", "h2d_bytes_per_step": n_tok * 4 + off.nbytes,
                "d2h_bytes_per_step": 5 * 8 * 2562},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _profile_traffic("dedup_compare_r0_dram_bytes_per_launch"),
                     "kernel": "dedup_compare_r0 (round 0, streaming)",
                     "launch_ms": r0_ms, "kernel_share_of_step": r0_ms / (dev_s * 1e3)},
        # the whole build call (host wall clock) against the same roofline:
        # SURVEY §8d's 4 B per token read once
        "build_roofline_frac": n_tok * 4 / dev_s / 1e9 / peak,
    }
    if not args.no_cpu:
        from oracle_lib import port, ref
        R = ref()
        impl = R if R is not None else port()
        t0 = time.perf_counter()
        impl.prefix_curves(tok, off, 1)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": n_tok / dt, "unit": "tokens/s", "cores": 1,
                               "kind": "reference" if R is not None else "port",
                               "sample": f"full C2 input, one PrefixIndex::build, {dt:.1f} s"}
    return out


NCCL_LOG = "/tmp/rs_bench_nccl.%h.%p.log"


def nccl_log_on(env):
    """NCCL's INIT log (rank count, transports) at INFO, even where the image
    presets a quieter NCCL_DEBUG (VERSION / WARN), written to per-process
    files (NCCL's default is stdout, where only the JSON line may go); rank 0
    echoes its key lines to stderr at the end (nccl_log_summary)."""
    if env.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        env["NCCL_DEBUG"] = "INFO"
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if env.get("NCCL_DEBUG_FILE", "") in ("", "/dev/stdout"):
        env["NCCL_DEBUG_FILE"] = NCCL_LOG


def nccl_log_summary():
    """The communicator lines of the NCCL logs (ranks, NVLS / NVLink paths) on stderr."""
    import glob
    keys = ("NVLS", "nRanks", "Init COMPLETE", "P2P/CUMEM", "via P2P", "NCCL version", "comm 0x")
    shown = 0
    for path in sorted(glob.glob("/tmp/rs_bench_nccl.*.log")):
        try:
            with open(path, errors="replace") as f:
                for line in f:
                    if any(k in line for k in keys) and shown < 40:
                        sys.stderr.write(line)
                        shown += 1
            os.remove(path)
        except OSError:
            pass


def relaunch_cmd(argv, n, port):
    """The torchrun command that runs this bench on n ranks (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", str(REPO / "bench.py"), *argv]


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scenarios", type=int, default=10000)
    ap.add_argument("--prompts", type=int, default=65536)
    ap.add_argument("--n-min", type=int, default=1)
    ap.add_argument("--n-max", type=int, default=256)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--lam", type=float, default=0.7)
    ap.add_argument("--cpu-rounds", type=int, default=4)
    ap.add_argument("--arrays-scenarios", type=int, default=2368,
                    help="scenarios of the e2e_arrays line (host inputs: 786 KB each)")
    ap.add_argument("--parity-samples", type=int, default=64)
    ap.add_argument("--parity-full", action="store_true",
                    help="bit-check every scenario (the default at N=1)")
    ap.add_argument("--parity-sampled-only", action="store_true",
                    help="at N=1 too, check only --parity-samples scenarios")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dedup", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-arrays", action="store_true")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--no-check", dest="check", action="store_false")
    raw = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(raw)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (the driver may call
        # `bench.py --gpus N` directly); NCCL's communicator log stays on so
        # the rank count is visible in stderr
        env = dict(os.environ)
        nccl_log_on(env)
        sys.exit(subprocess.call(relaunch_cmd(raw, args.gpus, free_port()), env=env))
    world, rank, local = init_dist()
    if world > 1:  # NCCL's communicator log (ranks, NVLS / NVLink paths)
        nccl_log_on(os.environ)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
