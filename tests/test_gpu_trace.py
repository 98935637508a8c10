"""GPU parity for the trace prompt table (rs_trace_csr_parse):
the '# prompt' metadata of CSV traces parsed on the device, against the
reference's own reader (trace_from_string via oracle/_ref): ids, ground
truths, tokens, limits, the step table (step rows grouped on the device) and
the errors (type, and the message for the step rules), on generated traces,
the reader's edge cases, and a C2-shaped trace whose device CSR feeds the
dedup index."""
import re

import numpy as np
import pytest

from cases import random_trace, steps_trace, trace_csv
from oracle_lib import OracleError, ref
from paper_2602_22718_b200 import rollsim as rs
from paper_2602_22718_b200.lib import ParseError, ValidationError

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(ref() is None, reason="reference not built (oracle/_ref)")]


def same_as_reference(text):
    want = ref().trace_prompts(text)
    tr = rs.TraceCSR(text)
    got = tr.host()
    assert tr.count == len(want["ids"])
    assert got["ids"] == want["ids"]
    assert got["gt"].tolist() == want["gt"].tolist()
    assert got["offsets"].tolist() == want["offsets"].tolist()
    assert np.array_equal(got["tokens"], want["tokens"])
    assert (tr.responses_per_prompt, tr.max_prompt_len, tr.max_response_len) == (
        want["g"], want["max_prompt_len"], want["max_response_len"])
    return tr


def test_random_traces_match_reference():
    for seed in range(6):
        same_as_reference(random_trace(seed, 50 + 40 * seed, max_len=80, shared=seed * 7))


def test_reader_edge_cases_match_reference():
    p = [("b", 5, [1, 2, 3]), ("a", 9, [4])]
    cases = [
        trace_csv(p).replace(b"\n", b"\r\n"),                                  # CRLF
        trace_csv(p).replace(b"# prompt b", b"  \t# prompt b").replace(b"\n", b" \t\n"),
        b"\n\n" + trace_csv(p) + b"\n\n",                                       # blank lines
        trace_csv([("x", 3, ["12-3", 4, "+5", "-6"])]),                        # glued numbers
        trace_csv([("x", 3, ["7abc", 9])]),                                    # garbage ends the list
        trace_csv([("x", "3+6", [1, 2])]),                                     # a token glued to gt
        trace_csv([("x", 3, [1, "99999999999999999999", 2])]),                 # overflow ends the list
        trace_csv([("x", 3, [4294967297, -2147483649, 5])]),                   # narrowed to int
        trace_csv([("x", 3, [1, 2])], extra_meta=["# note anything", "#g 4", "# g 2"]),
        trace_csv([("x", 3, [1, 2]), ("y", 3, [1])], max_prompt_len=2, max_response_len=3),
        trace_csv([]),                                                          # no prompts
        trace_csv(p).replace(b"\n", b"\r"),                                     # CR only: one line
        trace_csv([("x", 3, [1])], extra_meta=["# max_prompt_len x"]),          # num_get stores 0
        trace_csv([("x", 3, [1])], extra_meta=["# max_prompt_len 5000000000"]), # narrowed
        trace_csv([("x", 3, [1])], extra_meta=["# max_response_len 99999999999999999999"]),
        trace_csv([("x", 3, [1])], extra_meta=["# max_response_len -99999999999999999999"]),
        trace_csv([("x", 3, [1])], extra_meta=["# max_prompt_len 7x", "# max_prompt_len 9"]),
        trace_csv([("x", 3, [1])], extra_meta=["# g 99999999999999999999"]),     # g: ParseError
    ]
    for i, text in enumerate(cases):
        try:
            want = ref().trace_prompts(text)
        except OracleError as e:
            with pytest.raises((ParseError, ValidationError)) as got:
                rs.TraceCSR(text)
            assert (e.status == 7) == isinstance(got.value, ParseError), (i, e)
            continue
        same_as_reference(text)


def test_reader_errors_match_reference():
    p = [("b", 5, [1, 2, 3]), ("a", 9, [4])]
    bad = {
        ParseError: [
            trace_csv([("x", "q", [1])]),                                      # gt not a number
            trace_csv(p, header=False),                                         # no column header
            trace_csv(p) + b"# prompt z 1 2\n",                                 # metadata after header
            trace_csv(p).replace(b"actual_len", b"len"),                        # wrong header
            trace_csv(p, extra_meta=["# g x"]),
        ],
        ValidationError: [
            trace_csv([("x", 3, [1]), ("x", 4, [2])]),                          # duplicate id
            trace_csv([("x", 3, [])]),                                          # no tokens
            trace_csv([("x", 3, ["abc"])]),
            trace_csv([("x", 3, [1, 2, 3])], max_prompt_len=2),                # too long
            trace_csv([("x", 0, [1])]),                                         # gt out of range
            trace_csv([("x", 3000, [1])]),
            trace_csv([("x", 3, [1])], g=0),
        ],
    }
    for kind, texts in bad.items():
        for text in texts:
            with pytest.raises(OracleError) as e:
                ref().trace_prompts(text)
            assert e.value.status == (7 if kind is ParseError else 1), text[:80]
            with pytest.raises(kind):
                rs.TraceCSR(text)


@pytest.mark.slow
def test_c2_shaped_trace_to_prefix_index():
    """8,192 prompts x (2,048 shared + 512 unique) tokens as trace text: the
    device CSR equals the reference's parse and builds the same dedup
    tables as the token arrays themselves."""
    from cases import Rng
    rng = Rng(1)
    head = [rng.uniform_int(0, 31999) for _ in range(2048)]
    arr = np.random.RandomState(2).randint(0, 32000, (8192, 512))
    prompts = [(f"p{i:06d}", 100, head + arr[i].tolist()) for i in range(8192)]
    text = trace_csv(prompts, max_prompt_len=4096)
    tr = same_as_reference(text)
    idx = tr.prefix_index()
    direct = rs.PrefixIndex.build([p[2] for p in prompts])
    assert all(np.array_equal(a, b) for a, b in zip(idx.tables(), direct.tables()))
    assert idx.unique_prefix_count(2048) == 1
    assert idx.unique_prefix_count(2049) == len(np.unique(arr[:, 0]))


# ----------------------------------------------------------------- step rows
def same_steps(text):
    want = ref().trace_steps(text)
    got = rs.TraceCSR(text).steps()
    for k in ("step_idx", "entry_off", "entry_prompt", "lengths"):
        assert np.array_equal(got[k], want[k]), k
    return got


def _tail(msg):
    """The message after the reader's origin ('<string>:12: ...' -> '12: ...')."""
    m = re.search(r":(\d+: .*)$", msg)
    return m.group(1) if m else msg.split("] ", 1)[-1]


def same_error(text):
    with pytest.raises(OracleError) as e:
        ref().trace_steps(text)
    kind = ParseError if e.value.status == 7 else ValidationError
    assert e.value.status in (1, 7), e.value
    with pytest.raises(kind) as got:
        rs.TraceCSR(text)
    want_msg = str(e.value).split("] ", 1)[1]
    if kind is ParseError:
        assert _tail(str(got.value)) == _tail(want_msg)
    else:
        assert str(got.value) == want_msg


def test_step_table_matches_reference():
    for seed in range(8):
        text, prompts, steps = steps_trace(seed, 30 + 10 * seed, 1 + seed, g=1 + seed % 5,
                                           interleave=seed % 2 == 1)
        got = same_steps(text)
        assert got["step_idx"].tolist() == [st for st, _ in steps]


def test_step_table_without_rows():
    text = trace_csv([("a", 3, [1, 2])], g=2)
    got = same_steps(text)
    assert len(got["step_idx"]) == 0 and got["entry_off"].tolist() == [0]


def test_step_row_edge_cases_match_reference():
    p = [("b", 5, [1, 2, 3]), ("a", 9, [4])]
    base = trace_csv(p, g=2).decode()
    ok = [
        base + "0,a,0,5\n0,a,1,7\n",
        base + " 0 , a , 0 , 5 \r\n\t0,\ta,1,7\r\n",          # trimmed fields, CRLF
        base + "+3,b,+0,1\n3,b,1,2\n\n\n4,a,0,3\n4,a,1,4\n",   # signs, blank lines
        base + "0,a,0,5\n0,b,0,6\n0,a,1,7\n0,b,1,8\n",        # interleaved prompts
        base + "2147483648,a,0,5\n2147483648,a,1,7\n",          # narrowed step: INT_MIN -> negative
        base + "5,a,0,5\n5,a,1,7\n5,b,0,1\n5,b,1,1\n",
        base + "0,a,0,5\n0,a,1,7\n1,a,0,2\n1,a,1,2\n1,b,0,3\n1,b,1,3\n",
    ]
    for text in ok:
        text = text.encode()
        try:
            same_steps(text)
        except OracleError:
            same_error(text)


def test_step_row_errors_match_reference():
    p = [("b", 5, [1, 2, 3]), ("a", 9, [4])]
    base = trace_csv(p, g=2).decode()
    bad = [
        "0,a,0\n",                                   # 3 fields
        "0,a,0,5,6\n",                               # 5 fields
        "x,a,0,5\n",                                 # step not an integer
        "0,a,0,5x\n",                                # trailing characters
        "0,a,0,\n",                                  # empty field
        "0,a,0,99999999999999999999\n",              # out of range for long
        "0,a,1,5\n",                                 # response_idx must start at 0
        "0,a,0,5\n0,a,0,6\n",                        # repeated response_idx
        "1,a,0,5\n1,a,1,5\n0,b,0,1\n",               # step decreases
        "0,a,0,5\n0,zz,0,1\n0,zz,2,1\n",             # unknown id, out of order: ParseError
        "0,a,0,5\n0,a,1,5\n0,zz,0,1\n0,zz,1,1\n",    # unknown id: ValidationError
        "0,a,0,5\n",                                 # g = 2: one length missing
        "0,a,0,5\n0,a,1,5\n0,a,2,5\n",               # three lengths
        "0,a,0,5\n0,a,1,0\n",                        # length out of range
        "0,a,0,5\n0,a,1,2049\n",
        "-1,a,0,5\n-1,a,1,5\n",                      # first step must be >= 0
        "0,b,0,1\n0,b,1,0\n0,a,0,1\n",               # two bad groups: id order decides
        "0,a,0,5\n0,a,1,5\n1,zz,0,1\n1,zz,1,1\n1,a,0,9\n",
        "0,a,0,5\n# g 3\n",                          # metadata after header
        "0,a,0,5,1\n# g 3\n",                        # a bad row before it wins
    ]
    for rows in bad:
        same_error((base + rows).encode())
    # a bad prompt table outranks bad steps; a bad row outranks both
    same_error(trace_csv([("x", 0, [1])], g=1, steps=[(0, [("x", [0])])]))
    same_error(trace_csv([("x", 0, [1])], g=1).replace(b"actual_len\n", b"actual_len\n0,x\n"))


def test_step_table_device_views():
    import ctypes as C

    import torch
    from paper_2602_22718_b200.lib import check

    class View:  # a raw device int32 array, for torch.as_tensor
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False),
                                             "version": 3}

    text, _, _ = steps_trace(3, 40, 5, g=3)
    tr = rs.TraceCSR(text)
    host = tr.steps()
    views = [C.c_void_p() for _ in range(4)]
    check(tr._ctx.lib.rs_trace_csr_steps_device(tr._h, *[C.byref(v) for v in views]))
    S, E = len(host["step_idx"]), len(host["entry_prompt"])
    for v, n, k in zip(views, (S, S + 1, E, 3 * E), ("step_idx", "entry_off", "entry_prompt", "lengths")):
        dev = torch.as_tensor(View(v.value, n), device="cuda").cpu().numpy()
        assert np.array_equal(dev, host[k].reshape(-1)), k


@pytest.mark.slow
def test_large_step_table_matches_reference():
    """~200k step rows (50 steps x up to 512 prompts x g = 8)."""
    text, _, _ = steps_trace(11, 512, 50, g=8, max_len=16)
    same_steps(text)


def fuzz_csv(seed, n=120, steps=4, g=3, defect=None):
    """A CSV trace in random layouts: blanks and tabs around fields and
    tokens, CRLF, blank lines, signs, glued and overlong numbers in the
    prompt lists; optionally one defect in the step rows."""
    rng = np.random.RandomState(seed)
    sp = lambda: " " * int(rng.randint(0, 3)) + ("\t" if rng.rand() < 0.2 else "")
    lines = [f"# g {g}", "# max_prompt_len 600"]
    ids = [f"id{i:04d}" for i in rng.permutation(n)]
    for pid in ids:
        toks = []
        for _ in range(int(rng.randint(1, 400))):
            r = rng.rand()
            toks.append(str(rng.randint(0, 32000)) if r < 0.9 else
                        ("-" + str(rng.randint(0, 99)) if r < 0.95 else
                         ("+" + str(rng.randint(0, 99)) if r < 0.98 else "12-3")))
        lines.append(sp() + f"# prompt {pid} {int(rng.randint(1, 2048))} " + " ".join(toks) + sp())
        if rng.rand() < 0.05:
            lines.append(sp())
    lines.append(" step_idx , prompt_id,response_idx , actual_len ")
    rows = []
    st = 0
    for _ in range(steps):
        for pid in rng.permutation(ids)[: int(rng.randint(1, n))]:
            for r in range(g):
                rows.append(f"{sp()}{st}{sp()},{sp()}{pid}{sp()},{sp()}{r}{sp()},{sp()}{int(rng.randint(1, 2048))}{sp()}")
        st += int(rng.randint(1, 5))
    if defect is not None and rows:
        i = int(rng.randint(0, len(rows)))
        rows[i] = {"fields": rows[i] + ",9", "int": rows[i].replace(",", ",x", 1),
                   "order": rows[i].replace(",0,", ",1,", 1) if ",0," in rows[i] else rows[i] + ",",
                   "long": rows[i].split(",")[0] + ",idzz,0,1", "len": rows[i].rsplit(",", 1)[0] + ",0"}[defect]
    lines += rows
    text = "\n".join(lines) + "\n"
    if rng.rand() < 0.5:
        text = text.replace("\n", "\r\n")
    return text.encode()


def test_csv_fuzz_layouts():
    for seed in range(6):
        text = fuzz_csv(seed)
        try:
            ref().trace_prompts(text)
        except OracleError as e:
            pytest.fail(f"seed {seed}: the reference rejects it: {e}")
        same_as_reference(text)
        same_steps(text)


def test_csv_fuzz_defects():
    for seed, d in enumerate(["fields", "int", "order", "long", "len"] * 3):
        text = fuzz_csv(100 + seed, n=40, steps=3, defect=d)
        try:
            ref().trace_steps(text)
            same_steps(text)
        except OracleError:
            same_error(text)
