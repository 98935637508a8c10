"""GPU parity for the trace prompt table (rs_trace_csr_parse):
the '# prompt' metadata of CSV traces parsed on the device, against the
reference's own reader (trace_from_string via oracle/_ref): ids, ground
truths, tokens, limits and the error types, on generated traces, the reader's
edge cases, and a C2-shaped trace whose device CSR feeds the dedup index."""
import numpy as np
import pytest

from cases import random_trace, trace_csv
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
