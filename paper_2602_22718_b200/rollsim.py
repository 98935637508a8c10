"""Python mirror of the reference `rollsim` hot-path API over librs_b200.

Same names, argument meaning and error behaviour as the reference C++
library (/root/reference/proj/include/rollsim/{dedup,planner,profile}.hpp),
so tests read like the reference's own. Every computation runs on the GPU
through the C-ABI (include/rs.h); this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi
from .lib import (ConfigError, DeviceError, Error, ParseError, PlacementError,
                  ValidationError, as_f64, as_i32, as_i64, check, context, profile_struct, ptr)

__all__ = [
    "Error", "ConfigError", "ValidationError", "PlacementError", "ParseError", "DeviceError",
    "TraceCSR",
    "ClusterTopology", "default_topology", "PlacementPenalty", "NoiseModel", "LengthHistory",
    "predict_lengths",
    "LatencyProfile", "default_profile", "Prompt", "PrefixIndex", "PrefillCapacity",
    "PrefixSelection", "DedupSavings", "select_prefix_length", "dedup_savings",
    "unique_prefix_count_among", "dedup_map", "block_hashes", "PredictedPrompt",
    "ActorGroup", "ResponseSpec", "assign", "integrate_decode_seconds",
    "estimate_actor_time", "estimate_cost", "ScaleCandidate", "ScaleResult", "scale",
    "lpt", "to_csr", "id_ranks",
]


# ------------------------------------------------------------------ profile
@dataclass
class LatencyProfile:
    """proj/include/rollsim/profile.hpp:17-35 (tpot part)."""
    batch_knots: List[float]
    context_knots: List[float]
    tpot_grid: List[List[float]]
    rho: float = 0.0005
    gpus_per_actor: int = 2

    def struct(self):
        return profile_struct(self.batch_knots, self.context_knots,
                              np.asarray(self.tpot_grid, dtype=np.float64), self.rho)

    def tpot_seconds(self, batch_size, context_len):
        b = np.atleast_1d(as_f64(batch_size))
        c = np.atleast_1d(as_f64(context_len))
        b, c = np.broadcast_arrays(b, c)
        b, c = as_f64(b), as_f64(c)
        out = np.empty(b.shape, np.float64)
        s, keep = self.struct()
        ctx = context()
        check(ctx.lib.rs_tpot_seconds(ctx.handle, C.byref(s), ptr(b, C.c_double),
                                      ptr(c, C.c_double), b.size, ptr(out, C.c_double)))
        return out if np.ndim(batch_size) or np.ndim(context_len) else float(out[0])


def default_profile() -> LatencyProfile:
    """default_profile() (proj/src/profile.cpp:159-185): same grid bits."""
    bk = [1, 2, 4, 8, 16, 32, 64, 128, 256]
    ck = [128, 512, 1024, 2048, 4096]
    grid = [[0.006 + 2e-5 * float(b) + 1.2e-6 * float(c) + 4.5e-8 * float(b) * float(c)
             for c in ck] for b in bk]
    return LatencyProfile([float(x) for x in bk], [float(x) for x in ck], grid, 0.0005, 2)


# -------------------------------------------------------------------- dedup
@dataclass
class Prompt:
    """proj/include/rollsim/workload.hpp:18-25."""
    id: str
    token_ids: Sequence[int]
    ground_truth_len: int = 1

    def prompt_len(self):
        return len(self.token_ids)


def to_csr(prompts):
    """Batch (list of Prompt or token lists) -> (tokens int32, offsets int64)."""
    seqs = [p.token_ids if isinstance(p, Prompt) else p for p in prompts]
    lens = np.fromiter((len(s) for s in seqs), dtype=np.int64, count=len(seqs))
    off = np.zeros(len(seqs) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    tok = np.empty(int(off[-1]), np.int32)
    for i, s in enumerate(seqs):
        tok[off[i]:off[i + 1]] = s
    return tok, off


def _csr_args(batch):
    if isinstance(batch, tuple) and len(batch) == 2:
        tok, off = as_i32(batch[0]), as_i64(batch[1])
    else:
        tok, off = to_csr(batch)
    if tok.size == 0:
        tok = np.zeros(1, np.int32)
    return tok, off


class PrefixIndex:
    """PrefixIndex (proj/include/rollsim/dedup.hpp:20-48) built on the GPU."""

    def __init__(self, handle, ctx):
        self._h = handle
        self._ctx = ctx
        b, mn, mx, tot = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        check(ctx.lib.rs_prefix_index_info(handle, C.byref(b), C.byref(mn), C.byref(mx),
                                           C.byref(tot)))
        self._batch, self._min, self._max, self._total = b.value, mn.value, mx.value, tot.value

    @staticmethod
    def build(batch) -> "PrefixIndex":
        tok, off = _csr_args(batch)
        ctx = context()
        h = C.c_void_p()
        check(ctx.lib.rs_prefix_index_build(ctx.handle, ptr(tok, C.c_int32), ptr(off, C.c_int64),
                                            len(off) - 1, C.byref(h)))
        return PrefixIndex(h, ctx)

    @staticmethod
    def build_device(d_tokens, d_offsets, batch) -> "PrefixIndex":
        ctx = context()
        h = C.c_void_p()
        check(ctx.lib.rs_prefix_index_build_device(ctx.handle, C.c_void_p(d_tokens),
                                                   C.c_void_p(d_offsets), batch, C.byref(h)))
        return PrefixIndex(h, ctx)

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.rs_prefix_index_free(self._h)
                self._h = None
        except Exception:
            pass

    def _acc(self, fn, l):
        out = C.c_int64()
        check(fn(self._h, int(l), C.byref(out)))
        return out.value

    def unique_prefix_count(self, prefix_len):
        return self._acc(self._ctx.lib.rs_unique_prefix_count, prefix_len)

    def unique_prefix_tokens(self, prefix_len):
        return self._acc(self._ctx.lib.rs_unique_prefix_tokens, prefix_len)

    def remainder_tokens(self, prefix_len):
        return self._acc(self._ctx.lib.rs_remainder_tokens, prefix_len)

    def total_prompt_tokens(self):
        return self._total

    def min_prompt_len(self):
        return self._min

    def max_prompt_len(self):
        return self._max

    def batch_size(self):
        return self._batch

    def tables(self):
        m = self._max
        arrs = [np.zeros(m + 1, np.int64)] + [np.zeros(m + 2, np.int64) for _ in range(4)]
        check(self._ctx.lib.rs_prefix_index_tables(self._h, *[ptr(a, C.c_int64) for a in arrs]))
        return arrs


class TraceCSR:
    """The prompt table of a CSV workload trace (csv_from_string,
    proj/src/workload.cpp:169-263) parsed on the GPU into an id-sorted token
    CSR in HBM (rs_trace_csr_parse). `prefix_index()` builds the dedup index
    from that CSR without a host round trip."""

    def __init__(self, text, device=False, fmt="csv"):
        ctx = context()
        self._ctx = ctx
        h = C.c_void_p()
        parse = ctx.lib.rs_trace_csr_parse_jsonl if fmt == "jsonl" else ctx.lib.rs_trace_csr_parse
        if device:  # a torch uint8 CUDA tensor
            check(parse(ctx.handle, C.c_void_p(text.data_ptr()), text.numel(), 1, C.byref(h)))
        else:
            data = text.encode() if isinstance(text, str) else bytes(text)
            buf = C.create_string_buffer(data, len(data))
            check(parse(ctx.handle, buf, len(data), 0, C.byref(h)))
        self._h = h
        n, nt, nb = C.c_int32(), C.c_int64(), C.c_int64()
        g, mp, mr = C.c_int32(), C.c_int32(), C.c_int32()
        check(ctx.lib.rs_trace_csr_info(h, C.byref(n), C.byref(nt), C.byref(nb), C.byref(g),
                                        C.byref(mp), C.byref(mr)))
        self.count, self.n_tokens, self._nb = n.value, nt.value, nb.value
        self.responses_per_prompt, self.max_prompt_len, self.max_response_len = (
            g.value, mp.value, mr.value)

    @staticmethod
    def load(path, fmt=None):
        """load_trace (workload.cpp): the format from the extension unless given."""
        fmt = fmt or ("jsonl" if str(path).endswith(".jsonl") else "csv")
        with open(path, "rb") as f:
            return TraceCSR(f.read(), fmt=fmt)

    def device(self):
        """(tokens, offsets) device pointers, valid while this object lives."""
        t, o = C.c_void_p(), C.c_void_p()
        check(self._ctx.lib.rs_trace_csr_device(self._h, C.byref(t), C.byref(o)))
        return t.value, o.value

    def host(self):
        tok = np.zeros(max(self.n_tokens, 1), np.int32)
        off = np.zeros(self.count + 1, np.int64)
        ids = C.create_string_buffer(max(self._nb, 1))
        ioff = np.zeros(self.count + 1, np.int64)
        gt = np.zeros(max(self.count, 1), np.int32)
        check(self._ctx.lib.rs_trace_csr_copy(self._ctx.handle, self._h, tok.ctypes.data,
                                              off.ctypes.data, ids, ioff.ctypes.data,
                                              gt.ctypes.data))
        raw = ids.raw[:self._nb]
        return {"ids": [raw[ioff[i]:ioff[i + 1]].decode("latin-1") for i in range(self.count)],
                "gt": gt[:self.count], "tokens": tok[:self.n_tokens], "offsets": off}

    def steps(self):
        """The step table (rs_trace_csr_steps_copy): step_idx[S], entry_off[S+1],
        entry_prompt[E] (index into the id-sorted prompts, batch order) and
        lengths[E, g] (actual_lengths in response order)."""
        S, E = C.c_int32(), C.c_int64()
        check(self._ctx.lib.rs_trace_csr_steps_info(self._h, C.byref(S), C.byref(E)))
        S, E, g = S.value, E.value, self.responses_per_prompt
        st = np.zeros(max(S, 1), np.int32)
        eo = np.zeros(S + 1, np.int32)
        ep = np.zeros(max(E, 1), np.int32)
        ln = np.zeros(max(E * g, 1), np.int32)
        check(self._ctx.lib.rs_trace_csr_steps_copy(self._ctx.handle, self._h, st.ctypes.data,
                                                    eo.ctypes.data, ep.ctypes.data, ln.ctypes.data))
        return {"step_idx": st[:S], "entry_off": eo, "entry_prompt": ep[:E],
                "lengths": ln[:E * g].reshape(E, g)}

    def prefix_index(self) -> "PrefixIndex":
        t, o = self.device()
        return PrefixIndex.build_device(t, o, self.count)

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.rs_trace_csr_free(self._h)
                self._h = None
        except Exception:
            pass


@dataclass
class PrefillCapacity:
    max_unique_prefixes: int = 64
    gpu_count: int = 1


@dataclass
class PrefixSelection:
    prefix_len: int = 0
    capacity_exceeded: bool = False


@dataclass
class DedupSavings:
    raw_prefill_tokens: int = 0
    dedup_prefill_tokens: int = 0
    saved_fraction: float = 0.0


def select_prefix_length(index: PrefixIndex, capacity: PrefillCapacity, l_min, l_max):
    ln, ex = C.c_int32(), C.c_int32()
    check(index._ctx.lib.rs_select_prefix_length(index._h, capacity.max_unique_prefixes,
                                                 capacity.gpu_count, l_min, l_max,
                                                 C.byref(ln), C.byref(ex)))
    return PrefixSelection(ln.value, bool(ex.value))


def dedup_savings(index: PrefixIndex, l_star, responses_per_prompt):
    raw, dd, fr = C.c_int64(), C.c_int64(), C.c_double()
    check(index._ctx.lib.rs_dedup_savings(index._h, l_star, responses_per_prompt,
                                          C.byref(raw), C.byref(dd), C.byref(fr)))
    return DedupSavings(raw.value, dd.value, fr.value)


def unique_prefix_count_among(prompts, prefix_len):
    tok, off = _csr_args(prompts)
    ctx = context()
    out = C.c_int64()
    check(ctx.lib.rs_unique_prefix_count_among(ctx.handle, ptr(tok, C.c_int32),
                                               ptr(off, C.c_int64), len(off) - 1,
                                               prefix_len, C.byref(out)))
    return out.value


def dedup_map(prompts, prefix_len):
    tok, off = _csr_args(prompts)
    n = len(off) - 1
    lab = np.zeros(max(n, 1), np.int32)
    ctx = context()
    check(ctx.lib.rs_dedup_map(ctx.handle, ptr(tok, C.c_int32), ptr(off, C.c_int64), n,
                               prefix_len, ptr(lab, C.c_int32)))
    return lab[:n]


def block_hashes(prompts, block_tokens=16):
    tok, off = _csr_args(prompts)
    n = len(off) - 1
    nb = int(sum((int(off[i + 1] - off[i]) + block_tokens - 1) // block_tokens for i in range(n)))
    out = np.zeros(max(nb, 1), np.uint64)
    ctx = context()
    check(ctx.lib.rs_block_hashes(ctx.handle, ptr(tok, C.c_int32), ptr(off, C.c_int64), n,
                                  block_tokens, ptr(out, C.c_uint64)))
    return out[:nb]


# ------------------------------------------------------------------ planner
@dataclass
class PredictedPrompt:
    """proj/include/rollsim/planner.hpp:16-20."""
    id: str
    prompt_len: int = 0
    predicted_len: float = 1.0


@dataclass
class ActorGroup:
    """proj/include/rollsim/planner.hpp:22-28."""
    actor_id: int = 0
    prompt_ids: List[str] = field(default_factory=list)
    prompt_lens: List[int] = field(default_factory=list)
    predicted_lengths: List[float] = field(default_factory=list)
    gpu_count: int = 1


@dataclass
class ResponseSpec:
    prompt_len: int = 0
    target_len: float = 1.0


@dataclass
class ScaleCandidate:
    n_actors: int = 0
    t_total: float = 0.0
    t_penalty: float = 0.0
    cost: float = 0.0
    t_norm: float = 0.0
    c_norm: float = 0.0
    score: float = 0.0


@dataclass
class ScaleResult:
    n_star: int = 0
    candidates: List[ScaleCandidate] = field(default_factory=list)
    groups: List[ActorGroup] = field(default_factory=list)
    actor_times: List[float] = field(default_factory=list)


def id_ranks(ids):
    """Rank of each id under std::string ordering (unsigned bytewise)."""
    keys = [s.encode() for s in ids]
    order = sorted(range(len(keys)), key=keys.__getitem__)
    rank = np.empty(len(keys), np.int32)
    rank[order] = np.arange(len(keys), dtype=np.int32)
    return rank


def _soa(predicted):
    pred = as_f64([p.predicted_len for p in predicted])
    plen = as_i32([p.prompt_len for p in predicted])
    return pred, plen, id_ranks([p.id for p in predicted])


def _groups_from_order(predicted, order, n, gpus):
    P = len(predicted)
    q, r = divmod(P, n)
    groups, pos = [], 0
    for a in range(n):
        size = q + (1 if a < r else 0)
        g = ActorGroup(actor_id=a, gpu_count=gpus)
        for k in order[pos:pos + size]:
            p = predicted[int(k)]
            g.prompt_ids.append(p.id)
            g.prompt_lens.append(p.prompt_len)
            g.predicted_lengths.append(p.predicted_len)
        groups.append(g)
        pos += size
    return groups


def assign(predicted: Sequence[PredictedPrompt], n_actors: int, gpus_per_actor: int):
    """assign (proj/src/planner.cpp:16-51)."""
    ctx = context()
    P = len(predicted)
    pred, _, rank = _soa(predicted) if P else (as_f64([0.0]), None, as_i32([0]))
    order = np.zeros(max(P, 1), np.int32)
    goff = np.zeros(max(n_actors, 0) + 2, np.int32)
    check(ctx.lib.rs_assign(ctx.handle, ptr(pred, C.c_double), ptr(rank, C.c_int32), P,
                            n_actors, ptr(order, C.c_int32), ptr(goff, C.c_int32)))
    return _groups_from_order(predicted, order[:P], n_actors, gpus_per_actor)


def integrate_decode_seconds(responses: Sequence[ResponseSpec], profile: LatencyProfile):
    """integrate_decode_seconds (proj/src/planner.cpp:88-130)."""
    ctx = context()
    n = len(responses)
    plen = as_i32([r.prompt_len for r in responses] or [0])
    tgt = as_f64([r.target_len for r in responses] or [1.0])
    s, keep = profile.struct()
    out = C.c_double()
    check(ctx.lib.rs_integrate_decode_seconds(ctx.handle, ptr(plen, C.c_int32),
                                              ptr(tgt, C.c_double), n, C.byref(s),
                                              C.byref(out)))
    return out.value


def estimate_actor_time(group: ActorGroup, profile: LatencyProfile, responses_per_prompt):
    """estimate_actor_time (proj/src/planner.cpp:132-146)."""
    ctx = context()
    n = len(group.prompt_ids)
    plen = as_i32(list(group.prompt_lens) or [0])
    pred = as_f64(list(group.predicted_lengths) or [1.0])
    s, keep = profile.struct()
    out = C.c_double()
    check(ctx.lib.rs_estimate_actor_time(ctx.handle, ptr(plen, C.c_int32), ptr(pred, C.c_double),
                                         n, C.byref(s), responses_per_prompt, C.byref(out)))
    return out.value


def estimate_cost(groups: Sequence[ActorGroup], profile: LatencyProfile, responses_per_prompt,
                  times_out=None):
    """estimate_cost (proj/src/planner.cpp:148-157)."""
    ctx = context()
    plen = as_i32([l for g in groups for l in g.prompt_lens] or [0])
    pred = as_f64([p for g in groups for p in g.predicted_lengths] or [1.0])
    goff = np.zeros(len(groups) + 1, np.int32)
    goff[1:] = np.cumsum([len(g.prompt_ids) for g in groups]) if groups else []
    gpus = as_i32([g.gpu_count for g in groups] or [0])
    times = np.zeros(max(len(groups), 1), np.float64)
    s, keep = profile.struct()
    out = C.c_double()
    check(ctx.lib.rs_estimate_cost(ctx.handle, ptr(plen, C.c_int32), ptr(pred, C.c_double),
                                   ptr(goff, C.c_int32), ptr(gpus, C.c_int32), len(groups),
                                   C.byref(s), responses_per_prompt, C.byref(out),
                                   ptr(times, C.c_double)))
    if times_out is not None:
        times_out.extend(times[:len(groups)].tolist())
    return out.value


TimePenaltyFn = Callable[[int, List[ActorGroup], List[float]], float]


# ---------------------------------------------------------------- predictor
@dataclass
class NoiseModel:
    """NoiseModel (proj/include/rollsim/predictor.hpp:18-27)."""
    kind: str = "identity"  # or "bucket"
    bucket_accuracy: float = 1.0
    bucket_width: int = 100
    seed: int = 0

    def struct(self):
        return _abi.RsNoiseModel(0 if self.kind == "identity" else 1, float(self.bucket_accuracy),
                                 int(self.bucket_width), int(self.seed) & (2**64 - 1))


def predict_lengths(obs, depth, ground_truth_len, window, alpha, max_response_len,
                    noise: Optional[NoiseModel] = None, ids=None, device=False):
    """Batch LengthHistory::predict / predict_noisy on the GPU
    (rs_predict_lengths). obs: (count, window) oldest-first observation means,
    depth[i] of them valid. With device=True the arrays are torch CUDA tensors
    and the result stays on the device (a float64 tensor)."""
    ctx = context()
    nm = noise.struct() if noise is not None and noise.kind != "identity" else None
    if device:
        import torch
        n = int(depth.numel())
        out = torch.empty(n, dtype=torch.float64, device=depth.device)
        check(ctx.lib.rs_predict_lengths(ctx.handle, obs.data_ptr(), depth.data_ptr(),
                                         ground_truth_len.data_ptr(), n, window, float(alpha),
                                         max_response_len, C.byref(nm) if nm else None,
                                         ids[0].data_ptr() if ids is not None else None,
                                         ids[1].data_ptr() if ids is not None else None, 1,
                                         out.data_ptr()))
        return out
    depth, gt = as_i32(depth), as_i32(ground_truth_len)
    n = len(depth)
    obs = as_f64(np.asarray(obs, np.float64).reshape(-1)) if np.size(obs) else as_f64([0.0])
    out = np.zeros(max(n, 1), np.float64)
    blob = off = None
    if ids is not None:
        enc = [s.encode() for s in ids]
        blob = C.create_string_buffer(b"".join(enc) or b"\0")
        off = as_i64(np.cumsum([0] + [len(e) for e in enc]))
    check(ctx.lib.rs_predict_lengths(ctx.handle, obs.ctypes.data, depth.ctypes.data,
                                     gt.ctypes.data, n, window, float(alpha), max_response_len,
                                     C.byref(nm) if nm else None,
                                     C.cast(blob, C.c_void_p) if blob is not None else None,
                                     off.ctypes.data if off is not None else None, 0,
                                     out.ctypes.data))
    return out[:n]


class LengthHistory:
    """Sliding-window EWMA estimator (proj/include/rollsim/predictor.hpp:30-65).
    observe() keeps the reference's host bookkeeping; predictions run on the
    GPU, one batch per snapshot (snapshot_predictions, training.cpp:53-66)."""

    def __init__(self, window=1, alpha=0.5, max_response_len=2048):
        if window < 1:
            raise ConfigError("predictor window must be >= 1")
        if not alpha > 0 or alpha > 1:
            raise ConfigError("predictor alpha must be in (0, 1]")
        if max_response_len < 1:
            raise ConfigError("predictor max_response_len must be >= 1")
        self._window, self._alpha, self._max = window, alpha, max_response_len
        self._obs, self._last_step = {}, {}

    def window(self):
        return self._window

    def alpha(self):
        return self._alpha

    def max_response_len(self):
        return self._max

    def observe(self, step_idx, prompt_id, lengths):
        """predictor.cpp:33-50: store the step's mean length."""
        if not lengths:
            raise ValidationError(f"observe: empty length list for prompt '{prompt_id}'")
        total = 0.0
        for v in lengths:
            if v < 1 or v > self._max:
                raise ValidationError(f"observe: length out of range for prompt '{prompt_id}': {v}")
            total += v
        q = self._obs.setdefault(prompt_id, [])
        q.append(total / float(len(lengths)))
        del q[:max(0, len(q) - self._window)]
        self._last_step[prompt_id] = step_idx

    def observations(self, prompt_id):
        return self._obs.get(prompt_id)

    def snapshot(self, prompts, noise: Optional[NoiseModel] = None):
        """Predictions for (id, ground_truth_len) pairs, or objects with .id and
        .ground_truth_len, in one device call."""
        items = [(p.id, p.ground_truth_len) if hasattr(p, "id") else tuple(p) for p in prompts]
        n = len(items)
        if n == 0:
            return np.zeros(0, np.float64)
        obs = np.zeros((n, self._window), np.float64)
        depth = np.zeros(n, np.int32)
        for i, (pid, _) in enumerate(items):
            q = self._obs.get(pid) or []
            depth[i] = len(q)
            obs[i, :len(q)] = q
        return predict_lengths(obs, depth, [g for _, g in items], self._window, self._alpha,
                               self._max, noise, [pid for pid, _ in items] if noise else None)

    def predict(self, prompt):
        return float(self.snapshot([prompt])[0])

    def predict_noisy(self, prompt, noise: NoiseModel):
        return float(self.snapshot([prompt], noise)[0])


# ---------------------------------------------------------------- placement
@dataclass
class ClusterTopology:
    """ClusterTopology (proj/include/rollsim/placement.hpp:14-38): GPUs per
    node, two-tier bandwidths (or a full symmetric matrix), learner node and
    its local GPUs. Validated by the library like ClusterTopology::validate."""
    node_gpus: List[int]
    intra_node_bw: float = 2.5e10
    inter_node_bw: float = 3.0e9
    bw_matrix: Optional[List[List[float]]] = None
    learner_node: int = 0
    learner_gpus: List[int] = field(default_factory=lambda: [0, 1, 2, 3])

    def struct(self):
        ng = as_i32(self.node_gpus if self.node_gpus else [0])
        lg = as_i32(self.learner_gpus if self.learner_gpus else [0])
        bw = as_f64(np.asarray(self.bw_matrix, np.float64).ravel()) if self.bw_matrix else None
        t = _abi.RsTopology(len(self.node_gpus), ptr(ng, C.c_int32), float(self.intra_node_bw),
                            float(self.inter_node_bw), ptr(bw, C.c_double) if bw is not None else None,
                            int(self.learner_node), len(self.learner_gpus), ptr(lg, C.c_int32))
        return t, (ng, lg, bw)


def default_topology(node_count=2, gpus_per_node=8, learner_gpu_count=4) -> ClusterTopology:
    """default_topology (placement.cpp:118-128)."""
    return ClusterTopology(node_gpus=[gpus_per_node] * node_count,
                           learner_gpus=list(range(min(learner_gpu_count, gpus_per_node))))


@dataclass
class PlacementPenalty:
    """The TimePenaltyFn plan_rlhfless builds (proj/src/training.cpp:150-164):
    place each candidate on `topology` (placement.cpp:177-291) and charge the
    worst exposed transfer (check_overlap, placement.cpp:339-363), with
    kv bytes = kv_bytes_per_token x the group's prompt tokens
    (transfers_for, training.cpp:68-80). Passed as scale()'s `penalty`, it
    runs on the device for every candidate (rs_scale_placed)."""
    topology: ClusterTopology
    l_prefill_seconds: float
    model_bytes: float = 6e9
    kv_bytes_per_token: float = 36864.0

    def struct(self):
        t, keep = self.topology.struct()
        p = _abi.RsPlacementPenalty(C.pointer(t), float(self.model_bytes),
                                    float(self.kv_bytes_per_token), float(self.l_prefill_seconds))
        return p, (t, keep)


def scale(predicted: Sequence[PredictedPrompt], profile: LatencyProfile, responses_per_prompt,
          n_min, n_max, lambda_, gpus_per_actor, penalty=None, with_lpt=False):
    """scale (proj/src/planner.cpp:159-218). A Python `penalty` is called per
    candidate in ascending N with that candidate's groups and times, like
    TimePenaltyFn (planner.hpp:80-82); a `PlacementPenalty` is evaluated on
    the device instead (rs_scale_placed). with_lpt: also the LPT extension's
    token makespan and idle per candidate on the same predictions
    (res.lpt_makespan, res.lpt_idle)."""
    ctx = context()
    P = len(predicted)
    if P:
        pred, plen, rank = _soa(predicted)
    else:
        pred, plen, rank = as_f64([1.0]), as_i32([0]), as_i32([0])
    Cn = max(n_max - n_min + 1, 1)
    T = max((n_max * (n_max + 1) - (n_min - 1) * n_min) // 2, 1)
    arr = {k: np.zeros(Cn, np.float64) for k in ("t_total", "t_penalty", "cost", "t_norm",
                                                 "c_norm", "score")}
    idle = np.zeros(Cn, np.int64)
    order = np.zeros(max(P, 1), np.int32)
    gt = np.zeros(T, np.float64)
    at = np.zeros(max(n_max, 1), np.float64)
    lpt_mk = np.zeros(Cn, np.int64)
    lpt_idle = np.zeros(Cn, np.int64)
    out = _abi.RsScaleOut(0, *[ptr(arr[k], C.c_double) for k in
                               ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score")],
                          ptr(idle, C.c_int64), ptr(order, C.c_int32), ptr(at, C.c_double),
                          ptr(gt, C.c_double) if callable(penalty) else None,
                          ptr(lpt_mk, C.c_int64) if with_lpt else None,
                          ptr(lpt_idle, C.c_int64) if with_lpt else None)
    s, keep = profile.struct()
    if isinstance(penalty, PlacementPenalty):
        pp, keep_p = penalty.struct()
        check(ctx.lib.rs_scale_placed(ctx.handle, ptr(pred, C.c_double), ptr(plen, C.c_int32),
                                      ptr(rank, C.c_int32), P, C.byref(s), responses_per_prompt,
                                      n_min, n_max, float(lambda_), gpus_per_actor, C.byref(pp),
                                      C.byref(out)))
    else:
        check(ctx.lib.rs_scale(ctx.handle, ptr(pred, C.c_double), ptr(plen, C.c_int32),
                               ptr(rank, C.c_int32), P, C.byref(s), responses_per_prompt, n_min,
                               n_max, float(lambda_), gpus_per_actor, None, C.byref(out)))
    n_star = out.n_star
    if callable(penalty) and not isinstance(penalty, PlacementPenalty):
        pen = np.zeros(Cn, np.float64)
        base = 0
        for i, n in enumerate(range(n_min, n_max + 1)):
            groups = _groups_from_order(predicted, order[:P], n, gpus_per_actor)
            pen[i] = float(penalty(n, groups, gt[base:base + n].tolist()))
            base += n
        ns = C.c_int32()
        check(ctx.lib.rs_scale_select(ctx.handle, ptr(arr["t_total"], C.c_double),
                                      ptr(pen, C.c_double), ptr(arr["cost"], C.c_double), Cn,
                                      n_min, float(lambda_), ptr(arr["t_norm"], C.c_double),
                                      ptr(arr["c_norm"], C.c_double),
                                      ptr(arr["score"], C.c_double), C.byref(ns)))
        arr["t_penalty"] = pen
        n_star = ns.value
        b = (n_star * (n_star - 1) - n_min * (n_min - 1)) // 2
        at[:n_star] = gt[b:b + n_star]
    res = ScaleResult(n_star=n_star)
    for i, n in enumerate(range(n_min, n_max + 1)):
        res.candidates.append(ScaleCandidate(n, arr["t_total"][i], arr["t_penalty"][i],
                                             arr["cost"][i], arr["t_norm"][i], arr["c_norm"][i],
                                             arr["score"][i]))
    res.groups = _groups_from_order(predicted, order[:P], n_star, gpus_per_actor)
    res.actor_times = at[:n_star].tolist()
    res.idle_slot_ticks = idle
    if with_lpt:
        res.lpt_makespan, res.lpt_idle = lpt_mk, lpt_idle
    return res


def lpt(pred, id_rank, responses_per_prompt, n_min, n_max):
    """LPT extension: (makespan, idle) per candidate N."""
    ctx = context()
    pred = as_f64(pred)
    rank = as_i32(id_rank) if id_rank is not None else None
    C_ = n_max - n_min + 1
    mk = np.zeros(max(C_, 1), np.int64)
    idle = np.zeros(max(C_, 1), np.int64)
    check(ctx.lib.rs_lpt(ctx.handle, ptr(pred, C.c_double),
                         ptr(rank, C.c_int32) if rank is not None else None, len(pred),
                         responses_per_prompt, n_min, n_max, ptr(mk, C.c_int64),
                         ptr(idle, C.c_int64)))
    return mk[:C_], idle[:C_]
