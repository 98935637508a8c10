"""GPU parity for shared-prefix dedup (1): PrefixIndex tables, accessors,
selection, savings, subset counts, dedup map and block hashes, exact against
the CPU oracle and the reference's own known answers."""
import numpy as np
import pytest

import paper_2602_22718_b200.rollsim as rs
from cases import Rng, c2_tokens, csr, random_batch
from oracle_lib import port, ref
from paper_2602_22718_b200.rollsim import PrefillCapacity, PrefixIndex

pytestmark = pytest.mark.gpu


def curves(idx, n):
    return ([idx.unique_prefix_count(l) for l in range(1, n + 1)],
            [idx.unique_prefix_tokens(l) for l in range(1, n + 1)],
            [idx.remainder_tokens(l) for l in range(1, n + 1)])


def check_batch(seqs, n_l=None):
    tok, off = csr(seqs)
    idx = PrefixIndex.build((tok, off))
    n_l = n_l or idx.max_prompt_len() + 2
    info, u, t, r = port().prefix_curves(tok, off, n_l)
    assert [idx.batch_size(), idx.min_prompt_len(), idx.max_prompt_len(),
            idx.total_prompt_tokens()] == info.tolist()
    gu, gt, gr = curves(idx, n_l)
    assert gu == u.tolist() and gt == t.tolist() and gr == r.tolist()
    _, want = port().prefix_tables(tok, off)
    for a, b in zip(idx.tables(), want):
        assert a.tolist() == b.tolist()
    return idx, tok, off


def test_hand_counted():
    """proj/tests/test_dedup.cpp:78-111."""
    idx = PrefixIndex.build([[1, 2, 3], [1, 2, 4], [7, 8, 9]])
    assert [idx.unique_prefix_count(l) for l in (1, 2, 3, 10)] == [2, 2, 3, 3]
    assert idx.total_prompt_tokens() == 9 and idx.batch_size() == 3
    same = PrefixIndex.build([[5, 5, 5]] * 3)
    assert all(same.unique_prefix_count(l) == 1 for l in range(1, 6))
    distinct = PrefixIndex.build([[(i + 1) * 10000 + k for k in range(4)] for i in range(6)])
    assert all(distinct.unique_prefix_count(l) == 6 for l in range(1, 5))
    with pytest.raises(rs.ValidationError):
        PrefixIndex.build([[1]]).unique_prefix_count(0)
    with pytest.raises(rs.ValidationError):
        PrefixIndex.build([[1]]).unique_prefix_tokens(-1)
    with pytest.raises(rs.ValidationError):
        PrefixIndex.build([])
    with pytest.raises(rs.ValidationError):
        PrefixIndex.build([[1, 2], []])


def test_selection_and_savings():
    """proj/tests/test_dedup.cpp:150-274, acceptance criterion 1."""
    idx = PrefixIndex.build([[1, 1, 1], [1, 1, 2], [1, 2, 3], [1, 2, 4]])
    assert rs.select_prefix_length(idx, PrefillCapacity(2), 1, 3) == rs.PrefixSelection(2, False)
    assert rs.select_prefix_length(idx, PrefillCapacity(4), 1, 3) == rs.PrefixSelection(3, False)
    with pytest.raises(rs.ConfigError):
        rs.select_prefix_length(idx, PrefillCapacity(0), 1, 3)
    with pytest.raises(rs.ValidationError):
        rs.select_prefix_length(idx, PrefillCapacity(2), 0, 3)
    with pytest.raises(rs.ValidationError):
        rs.select_prefix_length(idx, PrefillCapacity(2), 3, 2)
    wide = PrefixIndex.build([[(i + 1) * 10000 + k for k in range(3)] for i in range(8)])
    assert rs.select_prefix_length(wide, PrefillCapacity(4), 1, 3) == rs.PrefixSelection(1, True)
    s = rs.dedup_savings(PrefixIndex.build([[1, 2, 3, 4]] * 3), 4, 1)
    assert (s.raw_prefill_tokens, s.dedup_prefill_tokens) == (12, 4)
    s = rs.dedup_savings(PrefixIndex.build([[1, 2], [1, 2, 3]]), 2, 1)
    assert (s.raw_prefill_tokens, s.dedup_prefill_tokens) == (5, 3)
    seqs = [[i * 100 + k for k in range(5 + i)] for i in range(6)]
    idx = PrefixIndex.build(seqs)
    s = rs.dedup_savings(idx, idx.max_prompt_len(), 3)
    assert s.saved_fraction == 2.0 / 3.0  # bitwise, acceptance_main.cpp:72
    with pytest.raises(rs.ValidationError):
        rs.dedup_savings(idx, 3, 0)


def test_random_batches_exact():
    rng = Rng(2026)
    for trial in range(150):
        seqs = random_batch(rng, max_count=24, max_len=14, alphabet=3)
        idx, tok, off = check_batch(seqs, 16)
        cap = rng.uniform_int(1, 8)
        got = rs.select_prefix_length(idx, PrefillCapacity(cap), 1, idx.max_prompt_len())
        assert (got.prefix_len, got.capacity_exceeded) == port().select_prefix_length(
            tok, off, cap, 1, idx.max_prompt_len())
        l = rng.uniform_int(1, 15)
        s = rs.dedup_savings(idx, l, 3)
        assert (s.raw_prefill_tokens, s.dedup_prefill_tokens, s.saved_fraction) == \
            port().dedup_savings(tok, off, l, 3)


def test_larger_structured_batches():
    """Shared heads, nested prefixes, duplicates, unaligned CSR offsets."""
    rng = np.random.RandomState(7)
    for trial in range(8):
        heads = [rng.randint(0, 50, size=rng.randint(1, 700)).tolist() for _ in range(5)]
        seqs = []
        for i in range(rng.randint(50, 3000)):
            h = heads[rng.randint(len(heads))]
            cut = rng.randint(1, len(h) + 1)
            tail = rng.randint(0, 4, size=rng.randint(0, 40)).tolist()
            seqs.append(h[:cut] + tail if rng.rand() < 0.8 else list(h))
        seqs = [s if s else [1] for s in seqs]
        check_batch(seqs)


def test_long_prompts_multi_chunk_tables():
    """Prompts up to ~9,000 tokens: the tables kernel scans depths in several
    chunks (2,048 per chunk) with carried totals."""
    rng = np.random.RandomState(31)
    head = rng.randint(0, 7, size=6000).tolist()
    seqs = []
    for i in range(60):
        cut = rng.randint(1, len(head) + 1)
        seqs.append(head[:cut] + rng.randint(0, 3, size=rng.randint(0, 3000)).tolist())
    seqs = [s if s else [1] for s in seqs]
    idx, _, _ = check_batch(seqs)
    assert idx.max_prompt_len() > 4096


def test_prompts_longer_than_the_histogram_bound():
    """Prompts longer than the first pass's histogram bound (16,384 tokens):
    the build sees the longest prompt in its stats and reruns once with exact
    arrays, taking a larger pinned table block; a short batch built next
    (smaller block from the pool) is exact too."""
    rng = np.random.RandomState(8)
    head = rng.randint(0, 5, size=30000).tolist()
    seqs = [head[:rng.randint(1, len(head) + 1)] + rng.randint(0, 3, size=rng.randint(0, 6000)).tolist()
            for _ in range(24)]
    seqs.append(head + [1] * 5000)
    idx, _, _ = check_batch(seqs)
    assert idx.max_prompt_len() > 16384
    check_batch([[1, 2, 3], [1, 2, 4], [9]])
    tok, off = csr(seqs)
    for l in (16384, 20000, 40000):  # the subset count and the map rerun the same way
        assert rs.unique_prefix_count_among(seqs, l) == port().unique_prefix_count_among(tok, off, l)
        assert rs.dedup_map(seqs, l).tolist() == port().dedup_map(tok, off, l).tolist()


def test_repeated_builds_identical():
    """The refinement runs its rounds in one persistent launch with grid-wide
    barriers and rotating counters; a race there shows up as a build that
    differs from the oracle now and then. Rebuild the same structured batches
    several times and require every build to match exactly."""
    rng = np.random.RandomState(99)
    for trial in range(3):
        heads = [rng.randint(0, 20, size=rng.randint(1, 300)).tolist() for _ in range(4)]
        seqs = []
        for i in range(rng.randint(500, 2500)):
            h = heads[rng.randint(len(heads))]
            cut = rng.randint(1, len(h) + 1)
            seqs.append(h[:cut] + rng.randint(0, 3, size=rng.randint(0, 30)).tolist())
        seqs = [s if s else [1] for s in seqs]
        tok, off = csr(seqs)
        _, want = port().prefix_tables(tok, off)
        for rep in range(6):
            idx = PrefixIndex.build((tok, off))
            for a, b in zip(idx.tables(), want):
                assert a.tolist() == b.tolist(), (trial, rep)


def test_live_indexes_keep_their_tables():
    """A device-built index keeps its tables in its own pinned block (the one
    the tables kernel wrote): later builds, freed indexes and even the
    destruction of the building context leave a live index intact."""
    import ctypes as C
    from paper_2602_22718_b200.lib import Context, check
    rng = np.random.RandomState(5)
    batches = []
    for _ in range(3):
        head = rng.randint(0, 9, size=rng.randint(50, 400)).tolist()
        seqs = [head[:rng.randint(1, len(head) + 1)] + rng.randint(0, 4, size=rng.randint(0, 40)).tolist()
                for _ in range(rng.randint(100, 600))]
        batches.append(csr(seqs))
    live = [PrefixIndex.build(b) for b in batches]
    PrefixIndex.build(batches[0])  # built and freed: its block returns to the pool
    PrefixIndex.build(batches[2])
    for idx, (tok, off) in zip(live, batches):
        _, want = port().prefix_tables(tok, off)
        for a, b in zip(idx.tables(), want):
            assert a.tolist() == b.tolist()
    tok, off = batches[1]
    ctx = Context(0)
    h = C.c_void_p()
    check(ctx.lib.rs_prefix_index_build(ctx.handle, tok.ctypes.data_as(C.POINTER(C.c_int32)),
                                        off.ctypes.data_as(C.POINTER(C.c_int64)), len(off) - 1,
                                        C.byref(h)))
    lib = ctx.lib
    ctx.close()
    idx = PrefixIndex(h, type("Lib", (), {"lib": lib})())  # no context behind it any more
    _, want = port().prefix_tables(tok, off)
    for a, b in zip(idx.tables(), want):
        assert a.tolist() == b.tolist()


def test_status_of_an_earlier_call_does_not_leak():
    """A call that fails on a device-side check (target length < 1 in
    integrate_decode_seconds) leaves its status bits set; the dedup calls that
    follow must report their own status only."""
    from paper_2602_22718_b200.rollsim import ResponseSpec, default_profile
    with pytest.raises(rs.ValidationError):
        rs.integrate_decode_seconds([ResponseSpec(10, 0.0)], default_profile())
    seqs = [[1, 2, 3], [1, 2, 4], [1, 2, 3], [7]]
    assert rs.unique_prefix_count_among(seqs, 3) == 3
    assert rs.dedup_map(seqs, 3).tolist() == [0, 1, 0, 3]
    idx = PrefixIndex.build(csr(seqs))
    assert idx.unique_prefix_count(2) == 2


def test_among_dedup_map_and_hashes():
    rng = Rng(77)
    for trial in range(40):
        seqs = random_batch(rng, max_count=30, max_len=12, alphabet=3)
        tok, off = csr(seqs)
        for l in (1, 3, 7, 20):
            assert rs.unique_prefix_count_among((tok, off), l) == \
                port().unique_prefix_count_among(tok, off, l)
            assert rs.dedup_map((tok, off), l).tolist() == port().dedup_map(tok, off, l).tolist()
        for k in (4, 8, 16):
            assert np.array_equal(rs.block_hashes((tok, off), k), port().block_hashes(tok, off, k))
    assert rs.unique_prefix_count_among([], 4) == 0
    with pytest.raises(rs.ValidationError):
        rs.unique_prefix_count_among([[1]], 0)
    # subset counts equal a fresh index (test_dedup.cpp:294-312)
    seqs = random_batch(Rng(9), max_count=40, max_len=12)
    for l in (1, 3, 7):
        assert rs.unique_prefix_count_among(seqs, l) == PrefixIndex.build(seqs).unique_prefix_count(l)


def test_block_hashes_long_prompts():
    rng = np.random.RandomState(3)
    seqs = [rng.randint(-2**31, 2**31 - 1, size=rng.randint(1, 3000)).tolist() for _ in range(60)]
    tok, off = csr(seqs)
    for k in (16, 64, 128):
        assert np.array_equal(rs.block_hashes((tok, off), k), port().block_hashes(tok, off, k))


@pytest.mark.slow
def test_c2_full_size():
    """C2: 65,536 prompts x (2,048 shared + 512 unique) tokens, vocab 32K.
    Probe answers from SURVEY.md §6: L* = 2048 at b_prefill 64,
    D(2048) = 1, D(2049) = 27,975, D(2050) = 65,532."""
    tok, off = c2_tokens()
    idx = PrefixIndex.build((tok, off))
    assert idx.unique_prefix_count(2048) == 1
    assert idx.unique_prefix_count(2049) == 27975
    assert idx.unique_prefix_count(2050) == 65532
    assert rs.select_prefix_length(idx, PrefillCapacity(64), 1, idx.max_prompt_len()).prefix_len == 2048
    s = rs.dedup_savings(idx, 2048, 8)
    assert abs(s.saved_fraction - 0.974998) < 5e-7
    _, want = port().prefix_tables(tok, off)
    for a, b in zip(idx.tables(), want):
        assert a.tolist() == b.tolist()
