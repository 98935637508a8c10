"""Seeded test inputs shared by the CPU and GPU suites.

Generators follow the reference tests' own fixtures:
random_batch (proj/tests/test_dedup.cpp:52-65), criterion-2 batches
(proj/tests/acceptance_main.cpp:97-106), constant_profile
(proj/tests/helpers.hpp:38-50), small_profile (proj/tests/test_profile.cpp:26-38).
"""
import numpy as np

from paper_2602_22718_b200 import _abi
from paper_2602_22718_b200.rollsim import LatencyProfile, default_profile

MASK = (1 << 64) - 1


class Rng:
    """rollsim::Rng (proj/include/rollsim/rng.hpp:14-49), integer draws only."""

    def __init__(self, seed):
        self.s = seed & MASK

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self):
        return (self.next_u64() >> 11) * 2.0 ** -53

    def uniform_range(self, lo, hi):
        return lo + (hi - lo) * self.uniform()

    def uniform_int(self, lo, hi):
        return lo + self.next_u64() % (hi - lo + 1)


def csr(seqs):
    off = np.zeros(len(seqs) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs]) if seqs else []
    tok = np.array([t for s in seqs for t in s], dtype=np.int32)
    return tok, off


def random_batch(rng, max_count=14, max_len=10, alphabet=3, min_len=1):
    count = rng.uniform_int(1, max_count)
    return [[rng.uniform_int(0, alphabet - 1) for _ in range(rng.uniform_int(min_len, max_len))]
            for _ in range(count)]


def constant_profile(tpot, rho=0.0005, gpus=2):
    return LatencyProfile([1.0, 4096.0], [1.0, float(1 << 20)], [[tpot, tpot], [tpot, tpot]],
                          rho, gpus)


def small_profile():
    return LatencyProfile([1.0, 4.0, 16.0], [100.0, 1000.0],
                          [[0.010, 0.020], [0.012, 0.026], [0.020, 0.050]], 0.0005, 2)


def profiles():
    return {"default": default_profile(), "small": small_profile(),
            "constant": constant_profile(0.01)}


def random_predicted(rng, count, pred_lo=1.0, pred_hi=400.0, plen_lo=8, plen_hi=400,
                     integer=False):
    pred = [float(rng.uniform_int(int(pred_lo), int(pred_hi))) if integer
            else rng.uniform_range(pred_lo, pred_hi) for _ in range(count)]
    plen = [rng.uniform_int(plen_lo, plen_hi) for _ in range(count)]
    return np.array(pred, np.float64), np.array(plen, np.int32)


def c4_spec(n_scenarios, count=65536, first=0, seed=1234):
    """The C4/C3 Monte-Carlo scenario definition."""
    return _abi.RsScenarioSpec(seed, first, n_scenarios, count, 384.0, 96.0, 16, 1024,
                               1024.0, 1.0, 16384.0)


def c2_tokens(n_prompts=65536, shared=2048, unique=512, vocab=32000, seed=1):
    """C2: Rng(1): a shared system prompt then per-prompt unique suffixes
    (SURVEY.md §8d), vectorised splitmix64."""
    n = shared + n_prompts * unique
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    draws = (z % np.uint64(vocab)).astype(np.int32)
    sys_prompt = draws[:shared]
    uniq = draws[shared:].reshape(n_prompts, unique)
    tok = np.empty((n_prompts, shared + unique), np.int32)
    tok[:, :shared] = sys_prompt
    tok[:, shared:] = uniq
    off = np.arange(n_prompts + 1, dtype=np.int64) * (shared + unique)
    return tok.reshape(-1), off


def placement_cases():
    """(penalty, gpus_per_actor, capacity) triples covering the placement
    rules of proj/src/placement.cpp:177-291: learner-node co-location, node
    ranking by bandwidth (ties by index), a bandwidth matrix, a learner node
    too small to host the heaviest actor, heterogeneous nodes, and penalties
    dominated by model sync or by KV shipping. capacity = actors that fit."""
    from paper_2602_22718_b200.rollsim import ClusterTopology, PlacementPenalty, default_topology
    bw3 = [[4e10, 1e10, 5e9], [1e10, 4e10, 1e10], [5e9, 1e10, 4e10]]
    return [
        (PlacementPenalty(default_topology(2, 8, 4), l_prefill_seconds=0.5, model_bytes=6e10), 2, 8),
        (PlacementPenalty(default_topology(4, 8, 4), l_prefill_seconds=0.05, model_bytes=1e9), 2, 16),
        (PlacementPenalty(ClusterTopology([8, 8, 8], bw_matrix=bw3, learner_node=2,
                                          learner_gpus=[1, 3]), l_prefill_seconds=0.2,
                          model_bytes=3e11), 2, 12),
        (PlacementPenalty(ClusterTopology([1, 4, 4], learner_gpus=[0]), l_prefill_seconds=0.1,
                          model_bytes=4e10), 2, 4),
        (PlacementPenalty(ClusterTopology([4, 6, 2, 8], learner_node=2, learner_gpus=[0, 1]),
                          l_prefill_seconds=1.0, kv_bytes_per_token=4e6), 2, 10),
        (PlacementPenalty(ClusterTopology([3, 5, 7], intra_node_bw=1e10, inter_node_bw=1e10,
                                          learner_node=1, learner_gpus=[4]),
                          l_prefill_seconds=0.0, model_bytes=1e11), 1, 15),
    ]


def predictor_cases():
    """Histories for LengthHistory::predict / predict_noisy
    (proj/src/predictor.cpp:52-98): (window, alpha, max_len, obs, depth,
    ground_truth, ids, noise). Observation means come from integer length
    lists like observe() stores them; some prompts are never observed, some
    estimates clamp at max_len, and bucket noise runs at several accuracies
    (0 forces the wrong-bucket branch), widths and seeds."""
    from paper_2602_22718_b200.rollsim import NoiseModel
    rng = Rng(2718)
    out = []
    for t in range(24):
        window = [1, 2, 3, 5, 8][t % 5]
        alpha = [0.5, 0.3, 1.0, 0.9, 0.125][t % 5]
        max_len = [2048, 700, 16384, 100, 3][t % 5]
        n = rng.uniform_int(1, 300)
        obs = np.zeros((n, window))
        depth = np.zeros(n, np.int32)
        gt = np.zeros(n, np.int32)
        for i in range(n):
            gt[i] = rng.uniform_int(1, max_len + max_len // 2)
            d = rng.uniform_int(0, window) if rng.uniform() < 0.8 else 0
            depth[i] = d
            for k in range(d):
                ls = [rng.uniform_int(1, max_len) for _ in range(rng.uniform_int(1, 8))]
                obs[i, k] = sum(float(x) for x in ls) / len(ls)
        ids = [f"p{rng.uniform_int(0, 999999):06d}-{i}" for i in range(n)]
        noise = None
        if t % 3:
            noise = NoiseModel("bucket", [0.0, 0.25, 0.8, 1.0][t % 4],
                               max(1, min(max_len, [1, 7, 100, 512][t % 4])), rng.next_u64())
        out.append((window, alpha, max_len, obs, depth, gt, ids, noise))
    return out


def trace_csv(prompts, g=1, max_prompt_len=None, max_response_len=None, steps=(), header=True,
              extra_meta=()):
    """A CSV workload trace in the reference's text format (csv_to_string,
    proj/src/workload.cpp:146-167): prompts = [(id, gt, tokens)], steps =
    [(step_idx, [(id, [lengths])])]."""
    lines = ["# rollsim-trace v1", f"# g {g}"]
    if max_prompt_len is not None:
        lines.append(f"# max_prompt_len {max_prompt_len}")
    if max_response_len is not None:
        lines.append(f"# max_response_len {max_response_len}")
    lines += list(extra_meta)
    for pid, gt, toks in prompts:
        lines.append(f"# prompt {pid} {gt} " + " ".join(str(t) for t in toks))
    if header:
        lines.append("step_idx,prompt_id,response_idx,actual_len")
    for st, rows in steps:
        for pid, lens in rows:
            lines += [f"{st},{pid},{r},{v}" for r, v in enumerate(lens)]
    return ("\n".join(lines) + "\n").encode()


def steps_trace(seed, n, n_steps, g=4, max_len=48, interleave=False, max_response_len=2048):
    """A trace with `n_steps` steps (increasing step_idx with gaps), each
    scheduling a random subset of the prompts in a random batch order; with
    `interleave` the rows of a step go response by response across its
    prompts (still in response order per prompt, the reader accepts it).
    Returns (text, prompts, steps) — the steps as trace_csv takes them."""
    rng = np.random.RandomState(seed)
    prompts = [(f"q{i:05d}", int(rng.randint(1, max_response_len + 1)),
                rng.randint(0, 32000, rng.randint(1, max_len + 1)).tolist()) for i in rng.permutation(n)]
    steps, st = [], int(rng.randint(0, 3))
    for _ in range(n_steps):
        pick = rng.permutation(n)[: int(rng.randint(1, n + 1))]
        steps.append((st, [(prompts[i][0], [int(x) for x in rng.randint(1, max_response_len + 1, g)])
                           for i in pick]))
        st += int(rng.randint(1, 4))
    if not interleave:
        return trace_csv(prompts, g=g, max_prompt_len=max_len, steps=steps), prompts, steps
    lines = trace_csv(prompts, g=g, max_prompt_len=max_len).decode().splitlines()
    for st_i, rows in steps:
        lines += [f"{st_i},{pid},{r},{lens[r]}" for r in range(g) for pid, lens in rows]
    return ("\n".join(lines) + "\n").encode(), prompts, steps


def random_trace(seed, n, max_len=64, g=2, shared=0):
    rng = np.random.RandomState(seed)
    head = rng.randint(0, 32000, shared).tolist()
    prompts = []
    for i in rng.permutation(n):
        toks = head + rng.randint(0, 32000, rng.randint(1, max_len + 1)).tolist()
        prompts.append((f"p{i:06d}", int(rng.randint(1, 2048)), toks))
    steps = [(0, [(p[0], [int(x) for x in rng.randint(1, 2048, g)]) for p in prompts[: n // 2]])]
    return trace_csv(prompts, g=g, max_prompt_len=max_len + shared, steps=steps)


def c2_trace_text(n_prompts=65536, shared=2048, unique=512, vocab=32000, seed=1, g=8, rows=True):
    """The C2 batch (c2_tokens) as CSV trace text: '# prompt p%06d 100 '
    then the tokens as zero-padded 5-digit decimals (valid istream integers,
    vocab < 100000), so every line has the same width and numpy builds the
    ~1 GB text directly; with `rows`, one step (step 0) scheduling the whole
    batch in a seeded random order, g rows per prompt ('0,p%06d,r,%04d',
    lengths in [1, 2048]). Returns (text uint8 array, tokens, offsets)."""
    tok, off = c2_tokens(n_prompts, shared, unique, vocab, seed)
    L = shared + unique
    assert vocab <= 100000 and np.all(np.diff(off) == L) and g <= 10
    head = np.frombuffer(f"# g {g}\n# max_prompt_len 4096\n".encode(), np.uint8)
    tail = np.frombuffer(b"step_idx,prompt_id,response_idx,actual_len\n", np.uint8)
    pre = 20  # '# prompt p000000 100'
    width = pre + 6 * L + 1
    body = np.empty((n_prompts, width), np.uint8)
    ids = np.arange(n_prompts)
    body[:, :pre] = np.frombuffer(b"# prompt p000000 100", np.uint8)
    for k in range(6):  # the id digits
        body[:, 15 - k] = ord("0") + (ids // 10 ** k) % 10
    t = tok.reshape(n_prompts, L)
    cols = body[:, pre:pre + 6 * L].reshape(n_prompts, L, 6)
    cols[:, :, 0] = ord(" ")
    for k in range(5):
        cols[:, :, 5 - k] = ord("0") + (t // 10 ** k) % 10
    body[:, -1] = ord("\n")
    parts = [head, body.reshape(-1), tail]
    if rows:
        rng = np.random.RandomState(seed + 1)
        order = np.repeat(rng.permutation(n_prompts), g)
        lens = rng.randint(1, 2049, n_prompts * g)
        r = np.empty((n_prompts * g, 17), np.uint8)  # '0,p000000,r,llll\n'
        r[:] = np.frombuffer(b"0,p000000,0,0000\n", np.uint8)
        for k in range(6):
            r[:, 8 - k] = ord("0") + (order // 10 ** k) % 10
        r[:, 10] = ord("0") + np.tile(np.arange(g), n_prompts)
        for k in range(4):
            r[:, 15 - k] = ord("0") + (lens // 10 ** k) % 10
        parts.append(r.reshape(-1))
    return np.concatenate(parts), tok, off


def c2_trace_jsonl(n_prompts=65536, shared=2048, unique=512, vocab=32000, seed=1, g=8, rows=True):
    """c2_trace_text's trace in the JSONL form (jsonl_to_string's layout:
    the header object on one line, then one step object): tokens
    right-aligned in 5 columns after a comma (JSON whitespace, no leading
    zeros), so numpy writes the ~1 GB line directly. Returns (text uint8
    array, tokens, offsets)."""
    tok, off = c2_tokens(n_prompts, shared, unique, vocab, seed)
    L = shared + unique
    assert vocab <= 100000 and np.all(np.diff(off) == L) and g <= 10

    def digits(x, width):  # right-aligned decimal columns, spaces before the first digit
        x = np.asarray(x)
        out = np.full(x.shape + (width,), ord(" "), np.uint8)
        nz = x.copy()
        for k in range(width):
            col = width - 1 - k
            d = (nz % 10).astype(np.uint8) + ord("0")
            show = (x >= 10 ** k) | (k == 0)
            out[..., col] = np.where(show, d, ord(" "))
            nz //= 10
        return out

    head = f'{{"g":{g},"max_prompt_len":4096,"max_response_len":2048,"prompts":['.encode()
    pre = b'{"ground_truth_len":100,"id":"p000000","token_ids":['
    width = len(pre) + 6 * L - 1 + 2 + 1  # tokens, "]}", ","
    body = np.empty((n_prompts, width), np.uint8)
    body[:, :len(pre)] = np.frombuffer(pre, np.uint8)
    ids = np.arange(n_prompts)
    at = pre.index(b"p000000") + 1
    for k in range(6):
        body[:, at + 5 - k] = ord("0") + (ids // 10 ** k) % 10
    cols = body[:, len(pre):len(pre) + 6 * L].reshape(n_prompts, L, 6)
    cols[:, :, :5] = digits(tok.reshape(n_prompts, L), 5)
    cols[:, :, 5] = ord(",")
    body[:, len(pre) + 6 * L - 1:len(pre) + 6 * L + 1] = np.frombuffer(b"]}", np.uint8)
    body[:, -1] = ord(",")
    flat = body.reshape(-1)[:-1]  # no comma after the last prompt
    parts = [np.frombuffer(head, np.uint8), flat, np.frombuffer(b'],"type":"header"}\n', np.uint8)]
    if rows:
        rng = np.random.RandomState(seed + 1)
        order = rng.permutation(n_prompts)
        lens = rng.randint(1, 2049, (n_prompts, g))
        ent = b'"p000000":[' + b",".join([b"    "] * g) + b"],"
        e = np.empty((n_prompts, len(ent)), np.uint8)
        e[:] = np.frombuffer(ent, np.uint8)
        srt = np.arange(n_prompts)  # map order = id order; prompt order[j] has lens[j]
        inv = np.argsort(order)
        for k in range(6):
            e[:, 7 - k] = ord("0") + (srt // 10 ** k) % 10
        for r in range(g):
            e[:, 11 + 5 * r:15 + 5 * r] = digits(lens[inv, r], 4)
        sch = np.empty((n_prompts, 10), np.uint8)
        sch[:] = np.frombuffer(b'"p000000",', np.uint8)
        for k in range(6):
            sch[:, 7 - k] = ord("0") + (order // 10 ** k) % 10
        parts += [np.frombuffer(b'{"lengths":{', np.uint8), e.reshape(-1)[:-1],
                  np.frombuffer(b'},"scheduled":[', np.uint8), sch.reshape(-1)[:-1],
                  np.frombuffer(b'],"step":0}\n', np.uint8)]
    return np.concatenate(parts), tok, off


def c2_tokens_multi(n_prompts=65536, n_sys=8, shared=2048, unique=512, vocab=32000, seed=1):
    """The C2 variant of SURVEY.md §8d with n_sys distinct system prompts
    (prompt i carries system prompt i mod n_sys), so the prefix tree branches
    at the root as well as after the system prompts."""
    n = n_sys * shared + n_prompts * unique
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    draws = (z % np.uint64(vocab)).astype(np.int32)
    sys_prompts = draws[:n_sys * shared].reshape(n_sys, shared)
    uniq = draws[n_sys * shared:].reshape(n_prompts, unique)
    tok = np.empty((n_prompts, shared + unique), np.int32)
    tok[:, :shared] = sys_prompts[np.arange(n_prompts) % n_sys]
    tok[:, shared:] = uniq
    off = np.arange(n_prompts + 1, dtype=np.int64) * (shared + unique)
    return tok.reshape(-1), off


def long_context_profile():
    """A 32K-context latency profile (context knots to 32,768): its context
    memo (> 4,096 entries) exceeds the lockstep evaluator's shared-memory
    row, so every group of the sweep takes the warp-cooperative evaluator
    reading the tables from global memory."""
    bk = [1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0, 128.0, 256.0]
    ck = [128.0, 1024.0, 4096.0, 16384.0, 32768.0]
    grid = [[0.005 + 1e-5 * b + 2e-7 * c + 1e-10 * b * c for c in ck] for b in bk]
    return LatencyProfile(bk, ck, grid, 0.0005, 2)
