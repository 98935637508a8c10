"""TEST INFRASTRUCTURE: loaders for the CPU checkers (oracle/oracle.h).

  port()  -> oracle/build/liboracle_port.so  (C restatement, prefix orc_)
  ref()   -> oracle/_ref/librollsim_ref_capi.so (the reference, prefix ref_)

Both expose the same plain-C surface; `Oracle` wraps it with numpy-friendly
methods that mirror the product calls, so tests compare like with like.
"""
import ctypes as C
import functools
import pathlib
import subprocess

import numpy as np

from paper_2602_22718_b200 import _abi
from paper_2602_22718_b200.lib import as_f64, as_i32, as_i64, ptr

REPO = pathlib.Path(__file__).resolve().parents[1]
PORT_SO = REPO / "oracle" / "build" / "liboracle_port.so"
REF_SO = REPO / "oracle" / "_ref" / "librollsim_ref_capi.so"


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class Oracle:
    def __init__(self, path, prefix):
        self.lib = C.CDLL(str(path))
        self.prefix = prefix
        _abi.bind(self.lib, _abi.ORACLE_SIGS, prefix)
        if prefix == "orc_":
            _abi.bind(self.lib, _abi.PORT_ONLY_SIGS)
        else:
            _abi.bind(self.lib, _abi.REF_ONLY_SIGS)

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _chk(self, st):
        if st:
            raise OracleError(st, self.fn("last_error")().decode(errors="replace"))

    # ---------------------------------------------------------------- dedup
    def prefix_curves(self, tok, off, n_l):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        info = np.zeros(4, np.int64)
        u, t, r = (np.zeros(max(n_l, 1), np.int64) for _ in range(3))
        self._chk(self.fn("prefix_curves")(ptr(tok, C.c_int32), ptr(off, C.c_int64), len(off) - 1,
                                           n_l, ptr(info, C.c_int64), ptr(u, C.c_int64),
                                           ptr(t, C.c_int64), ptr(r, C.c_int64)))
        return info, u[:n_l], t[:n_l], r[:n_l]

    def select_prefix_length(self, tok, off, cap, l_min, l_max, gpus=1):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        ln, ex = C.c_int32(), C.c_int32()
        self._chk(self.fn("select_prefix_length")(ptr(tok, C.c_int32), ptr(off, C.c_int64),
                                                  len(off) - 1, cap, gpus, l_min, l_max,
                                                  C.byref(ln), C.byref(ex)))
        return ln.value, bool(ex.value)

    def dedup_savings(self, tok, off, l_star, g):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        raw, dd, fr = C.c_int64(), C.c_int64(), C.c_double()
        self._chk(self.fn("dedup_savings")(ptr(tok, C.c_int32), ptr(off, C.c_int64), len(off) - 1,
                                           l_star, g, C.byref(raw), C.byref(dd), C.byref(fr)))
        return raw.value, dd.value, fr.value

    def unique_prefix_count_among(self, tok, off, l):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        out = C.c_int64()
        self._chk(self.fn("unique_prefix_count_among")(ptr(tok, C.c_int32), ptr(off, C.c_int64),
                                                       len(off) - 1, l, C.byref(out)))
        return out.value

    # -------------------------------------------------------------- planner
    def tpot_seconds(self, prof, b, c):
        b, c = as_f64(b), as_f64(c)
        out = np.zeros(len(b), np.float64)
        s, keep = prof.struct()
        self._chk(self.fn("tpot_seconds")(C.byref(s), ptr(b, C.c_double), ptr(c, C.c_double),
                                          len(b), ptr(out, C.c_double)))
        return out

    def assign(self, pred, id_rank, n):
        pred = as_f64(pred)
        rank = as_i32(id_rank) if id_rank is not None else None
        P = len(pred)
        order = np.zeros(max(P, 1), np.int32)
        goff = np.zeros(max(n, 0) + 2, np.int32)
        self._chk(self.fn("assign")(ptr(pred, C.c_double),
                                    ptr(rank, C.c_int32) if rank is not None else None, P, n,
                                    ptr(order, C.c_int32), ptr(goff, C.c_int32)))
        return order[:P], goff[:n + 1]

    def integrate(self, plen, target, prof):
        n = len(target)
        plen, target = as_i32(plen if len(plen) else [0]), as_f64(target if len(target) else [1])
        out = C.c_double()
        s, keep = prof.struct()
        self._chk(self.fn("integrate_decode_seconds")(ptr(plen, C.c_int32), ptr(target, C.c_double),
                                                      n, C.byref(s), C.byref(out)))
        return out.value

    def estimate_actor_time(self, plen, pred, prof, g):
        plen, pred = as_i32(plen), as_f64(pred)
        out = C.c_double()
        s, keep = prof.struct()
        self._chk(self.fn("estimate_actor_time")(ptr(plen, C.c_int32), ptr(pred, C.c_double),
                                                 len(pred), C.byref(s), g, C.byref(out)))
        return out.value

    def estimate_cost(self, plen, pred, goff, gpus, prof, g):
        plen, pred, goff, gpus = as_i32(plen), as_f64(pred), as_i32(goff), as_i32(gpus)
        out = C.c_double()
        times = np.zeros(max(len(goff) - 1, 1), np.float64)
        s, keep = prof.struct()
        self._chk(self.fn("estimate_cost")(ptr(plen, C.c_int32), ptr(pred, C.c_double),
                                           ptr(goff, C.c_int32), ptr(gpus, C.c_int32),
                                           len(goff) - 1, C.byref(s), g, C.byref(out),
                                           ptr(times, C.c_double)))
        return out.value, times[:len(goff) - 1]

    def scale(self, pred, plen, id_rank, prof, g, n_min, n_max, lam, gpus, penalty=None):
        pred, plen = as_f64(pred), as_i32(plen)
        rank = as_i32(id_rank) if id_rank is not None else None
        Cn = max(n_max - n_min + 1, 1)
        arrs = [np.zeros(Cn, np.float64) for _ in range(6)]
        order = np.zeros(max(len(pred), 1), np.int32)
        at = np.zeros(max(n_max, 1), np.float64)
        ns = C.c_int32()
        pen = as_f64(penalty) if penalty is not None else None
        s, keep = prof.struct()
        self._chk(self.fn("scale")(ptr(pred, C.c_double), ptr(plen, C.c_int32),
                                   ptr(rank, C.c_int32) if rank is not None else None, len(pred),
                                   C.byref(s), g, n_min, n_max, float(lam), gpus,
                                   ptr(pen, C.c_double) if pen is not None else None,
                                   C.byref(ns), *[ptr(a, C.c_double) for a in arrs],
                                   ptr(order, C.c_int32), ptr(at, C.c_double)))
        keys = ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score")
        out = dict(zip(keys, arrs))
        out.update(n_star=ns.value, order=order[:len(pred)], actor_times=at[:ns.value])
        return out

    def scale_placed(self, pred, plen, id_rank, prof, g, n_min, n_max, lam, gpus, placement):
        """scale() with plan_rlhfless's placement penalty (a PlacementPenalty)."""
        pred, plen = as_f64(pred), as_i32(plen)
        rank = as_i32(id_rank) if id_rank is not None else None
        Cn = max(n_max - n_min + 1, 1)
        arrs = [np.zeros(Cn, np.float64) for _ in range(6)]
        order = np.zeros(max(len(pred), 1), np.int32)
        at = np.zeros(max(n_max, 1), np.float64)
        ns = C.c_int32()
        s, keep = prof.struct()
        pp, keep_p = placement.struct()
        self._chk(self.fn("scale_placed")(ptr(pred, C.c_double), ptr(plen, C.c_int32),
                                          ptr(rank, C.c_int32) if rank is not None else None,
                                          len(pred), C.byref(s), g, n_min, n_max, float(lam), gpus,
                                          C.byref(pp), C.byref(ns),
                                          *[ptr(a, C.c_double) for a in arrs],
                                          ptr(order, C.c_int32), ptr(at, C.c_double)))
        keys = ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score")
        out = dict(zip(keys, arrs))
        out.update(n_star=ns.value, order=order[:len(pred)], actor_times=at[:ns.value])
        return out

    def predict_lengths(self, obs, depth, gt, window, alpha, max_len, noise=None, ids=None):
        """LengthHistory::predict / predict_noisy per prompt. obs: count x window."""
        obs = as_f64(np.asarray(obs, np.float64).reshape(-1) if np.size(obs) else [0.0])
        depth, gt = as_i32(depth), as_i32(gt)
        n = len(depth)
        out = np.zeros(max(n, 1), np.float64)
        nm = noise.struct() if noise is not None else None
        if ids is not None:
            blob = b"".join(s.encode() for s in ids)
            off = as_i64(np.cumsum([0] + [len(s.encode()) for s in ids]))
        else:
            blob, off = None, None
        self._chk(self.fn("predict_lengths")(ptr(obs, C.c_double), ptr(depth, C.c_int32),
                                             ptr(gt, C.c_int32), n, window, float(alpha), max_len,
                                             C.byref(nm) if nm is not None else None, blob,
                                             ptr(off, C.c_int64) if off is not None else None,
                                             ptr(out, C.c_double)))
        return out[:n]

    def trace_format(self, fmt):
        """Reference only: the format trace_prompts / trace_steps read."""
        self.lib.ref_trace_set_format(1 if fmt == "jsonl" else 0)

    def trace_convert(self, text: bytes, fmt_in="csv", fmt_out="jsonl") -> bytes:
        """Reference only: trace_to_string(trace_from_string(text, fmt_in), fmt_out)."""
        n = C.c_int64()
        buf = C.create_string_buffer(text, len(text))
        codes = {"csv": 0, "jsonl": 1}
        self._chk(self.lib.ref_trace_convert(buf, len(text), codes[fmt_in], codes[fmt_out], None, 0,
                                             C.byref(n)))
        out = C.create_string_buffer(max(n.value, 1))
        self._chk(self.lib.ref_trace_convert(buf, len(text), codes[fmt_in], codes[fmt_out], out,
                                             n.value, C.byref(n)))
        return out.raw[:n.value]

    def trace_prompts(self, text: bytes, fmt="csv"):
        """Reference only: the id-sorted prompt table of a CSV / JSONL trace."""
        self.trace_format(fmt)
        info = np.zeros(6, np.int64)
        buf = C.create_string_buffer(text, len(text))
        self._chk(self.lib.ref_trace_prompts(buf, len(text), ptr(info, C.c_int64), None, None, None,
                                             None, None))
        n, nt, nb = (int(x) for x in info[:3])
        tok = np.zeros(max(nt, 1), np.int32)
        off = np.zeros(n + 1, np.int64)
        ids = C.create_string_buffer(max(nb, 1))
        ioff = np.zeros(n + 1, np.int64)
        gt = np.zeros(max(n, 1), np.int32)
        self._chk(self.lib.ref_trace_prompts(buf, len(text), ptr(info, C.c_int64), tok.ctypes.data,
                                             off.ctypes.data, ids, ioff.ctypes.data, gt.ctypes.data))
        raw = ids.raw[:nb]
        return {"ids": [raw[ioff[i]:ioff[i + 1]].decode("latin-1") for i in range(n)],
                "gt": gt[:n], "tokens": tok[:nt], "offsets": off, "g": int(info[3]),
                "max_prompt_len": int(info[4]), "max_response_len": int(info[5])}

    def trace_steps(self, text: bytes, fmt="csv"):
        """Reference only: the step table of a CSV / JSONL trace (ref_trace_steps)."""
        self.trace_format(fmt)
        info = np.zeros(3, np.int64)
        buf = C.create_string_buffer(text, len(text))
        self._chk(self.lib.ref_trace_steps(buf, len(text), ptr(info, C.c_int64), None, None, None,
                                           None))
        S, E, g = (int(x) for x in info)
        st = np.zeros(max(S, 1), np.int32)
        eo = np.zeros(S + 1, np.int32)
        ep = np.zeros(max(E, 1), np.int32)
        ln = np.zeros(max(E * g, 1), np.int32)
        self._chk(self.lib.ref_trace_steps(buf, len(text), ptr(info, C.c_int64), st.ctypes.data,
                                           eo.ctypes.data, ep.ctypes.data, ln.ctypes.data))
        return {"step_idx": st[:S], "entry_off": eo, "entry_prompt": ep[:E],
                "lengths": ln[:E * g].reshape(E, g)}

    def sweep_arrays(self, pred, plen, S, P, prof, g, n_min, n_max, lam, gpus, threads=1):
        pred, plen = as_f64(pred), as_i32(plen)
        Cn = n_max - n_min + 1
        tt = np.zeros(S * Cn, np.float64)
        cc = np.zeros(S * Cn, np.float64)
        ns = np.zeros(S, np.int32)
        s, keep = prof.struct()
        self._chk(self.fn("sweep_arrays")(ptr(pred, C.c_double), ptr(plen, C.c_int32), S, P,
                                          C.byref(s), g, n_min, n_max, float(lam), gpus, threads,
                                          ptr(tt, C.c_double), ptr(cc, C.c_double),
                                          ptr(ns, C.c_int32)))
        return tt.reshape(S, Cn), cc.reshape(S, Cn), ns

    # ------------------------------------------------------- port-only extras
    def generate_scenarios(self, spec):
        n = spec.n_scenarios * spec.count
        pred = np.zeros(max(n, 1), np.float64)
        plen = np.zeros(max(n, 1), np.int32)
        self._chk(self.lib.orc_generate_scenarios(C.byref(spec), ptr(pred, C.c_double),
                                                  ptr(plen, C.c_int32)))
        return pred[:n], plen[:n]

    def scale_idle(self, pred, id_rank, g, n_min, n_max):
        pred = as_f64(pred)
        rank = as_i32(id_rank) if id_rank is not None else None
        out = np.zeros(n_max - n_min + 1, np.int64)
        self._chk(self.lib.orc_scale_idle(ptr(pred, C.c_double),
                                          ptr(rank, C.c_int32) if rank is not None else None,
                                          len(pred), g, n_min, n_max, ptr(out, C.c_int64)))
        return out

    def dedup_map(self, tok, off, l):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        n = len(off) - 1
        lab = np.zeros(max(n, 1), np.int32)
        self._chk(self.lib.orc_dedup_map(ptr(tok, C.c_int32), ptr(off, C.c_int64), n, l,
                                         ptr(lab, C.c_int32)))
        return lab[:n]

    def block_hashes(self, tok, off, k):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        n = len(off) - 1
        nb = int(sum((int(off[i + 1] - off[i]) + k - 1) // k for i in range(n)))
        out = np.zeros(max(nb, 1), np.uint64)
        self._chk(self.lib.orc_block_hashes(ptr(tok, C.c_int32), ptr(off, C.c_int64), n, k,
                                            ptr(out, C.c_uint64)))
        return out[:nb]

    def lpt(self, pred, id_rank, g, n_min, n_max):
        pred = as_f64(pred)
        rank = as_i32(id_rank) if id_rank is not None else None
        Cn = n_max - n_min + 1
        mk = np.zeros(Cn, np.int64)
        idle = np.zeros(Cn, np.int64)
        self._chk(self.lib.orc_lpt(ptr(pred, C.c_double),
                                   ptr(rank, C.c_int32) if rank is not None else None, len(pred),
                                   g, n_min, n_max, ptr(mk, C.c_int64), ptr(idle, C.c_int64)))
        return mk, idle

    def prefix_tables(self, tok, off):
        tok, off = as_i32(tok if len(tok) else [0]), as_i64(off)
        lens = np.diff(off)
        m = int(lens.max()) if len(lens) else 0
        info = np.zeros(4, np.int64)
        arrs = [np.zeros(m + 1, np.int64)] + [np.zeros(m + 2, np.int64) for _ in range(4)]
        self._chk(self.lib.orc_prefix_tables(ptr(tok, C.c_int32), ptr(off, C.c_int64),
                                             len(off) - 1, ptr(info, C.c_int64),
                                             *[ptr(a, C.c_int64) for a in arrs]))
        return info, arrs

    def sweep_select(self, sum_t, sum_c, S, n_min, lam):
        sum_t, sum_c = as_f64(sum_t), as_f64(sum_c)
        ns = C.c_int32()
        self._chk(self.lib.orc_sweep_select(ptr(sum_t, C.c_double), ptr(sum_c, C.c_double), S,
                                            len(sum_t), n_min, float(lam), C.byref(ns)))
        return ns.value


@functools.lru_cache(None)
def port():
    if not PORT_SO.exists():
        subprocess.run(["make", "-C", str(REPO / "oracle"), "port"], check=True,
                       stdout=subprocess.DEVNULL)
    return Oracle(PORT_SO, "orc_")


@functools.lru_cache(None)
def ref():
    """The reference library, or None when it was not built (GPU boxes have no
    /root/reference; the build ships oracle/_ref/ when it was made here)."""
    if not REF_SO.exists():
        ref_src = pathlib.Path("/root/reference/proj/src")
        if ref_src.exists():
            subprocess.run(["make", "-C", str(REPO / "oracle"), "ref", "-j8"], check=True,
                           stdout=subprocess.DEVNULL)
        else:
            return None
    return Oracle(REF_SO, "ref_")
