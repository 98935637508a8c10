"""GPU parity for the JSONL trace reader (rs_trace_csr_parse_jsonl,
SURVEY §8f-4) against the reference's own reader (jsonl_from_string through
oracle/_ref, nlohmann::json): prompt tables and step tables of traces the
reference writes (trace_to_string) and of hand-written lines that exercise
nlohmann's grammar and conversions; errors by type (ParseError at a line vs
ValidationError with the validator's message)."""
import json

import numpy as np
import pytest

from cases import random_trace, steps_trace, trace_csv
from oracle_lib import OracleError, ref
from paper_2602_22718_b200 import rollsim as rs
from paper_2602_22718_b200.lib import ParseError, ValidationError

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(ref() is None, reason="reference not built (oracle/_ref)")]


def same(text):
    want_p = ref().trace_prompts(text, "jsonl")
    want_s = ref().trace_steps(text, "jsonl")
    tr = rs.TraceCSR(text, fmt="jsonl")
    got = tr.host()
    assert got["ids"] == want_p["ids"]
    assert got["gt"].tolist() == want_p["gt"].tolist()
    assert got["offsets"].tolist() == want_p["offsets"].tolist()
    assert np.array_equal(got["tokens"], want_p["tokens"])
    assert (tr.responses_per_prompt, tr.max_prompt_len, tr.max_response_len) == (
        want_p["g"], want_p["max_prompt_len"], want_p["max_response_len"])
    steps = tr.steps()
    for k in ("step_idx", "entry_off", "entry_prompt", "lengths"):
        assert np.array_equal(steps[k], want_s[k]), k
    return tr


def same_error(text):
    with pytest.raises(OracleError) as e:
        ref().trace_prompts(text, "jsonl")
    assert e.value.status in (1, 7), e.value
    kind = ParseError if e.value.status == 7 else ValidationError
    with pytest.raises(kind) as got:
        rs.TraceCSR(text, fmt="jsonl")
    want = str(e.value).split("] ", 1)[1]
    if kind is ValidationError:
        assert str(got.value) == want
    else:  # the same line: '<string>:N: ...' / '<trace>:N: ...'
        assert want.split(":")[1] == str(got.value).split(":")[1], (want, str(got.value))


def header(prompts, g=2, **kw):
    h = {"type": "header", "g": g, "prompts": prompts}
    h.update(kw)
    return h


def lines(*objs, raw=()):
    out = [o if isinstance(o, str) else json.dumps(o) for o in objs]
    return ("\n".join(out + list(raw)) + "\n").encode()


P2 = [{"id": "b", "ground_truth_len": 5, "token_ids": [1, 2, 3]},
      {"id": "a", "ground_truth_len": 9, "token_ids": [4]}]


def test_reference_written_traces():
    for seed in range(5):
        text, _, _ = steps_trace(seed, 30 + 20 * seed, 1 + seed, g=1 + seed % 4,
                                 interleave=seed % 2 == 1)
        same(ref().trace_convert(text))
    same(ref().trace_convert(random_trace(7, 200, max_len=60, shared=5)))
    same(ref().trace_convert(trace_csv([("x", 3, [1, 2])], g=2)))


def grammar_cases():
    step = {"step": 0, "scheduled": ["a", "b"], "lengths": {"a": [5, 6], "b": [7, 8]}}
    return [
        lines(header(P2), step),
        # whitespace, key order, unknown members with nested values
        lines(' { "prompts" : %s , "g":2,"x":{"y":[1,{"z":null}],"w":"\\u00e9"},"type":"header"} '
              % json.dumps(P2), step),
        # CRLF, blank lines, tabs
        lines(header(P2), step).replace(b"\n", b"\r\n") + b"\n\t\n",
        # escapes in ids: é, \", \\, a surrogate pair
        lines(header([{"id": "é\"\\\U0001F600", "ground_truth_len": 3, "token_ids": [1]}], g=1),
              {"step": 4, "lengths": {"é\"\\\U0001F600": [2]}}),
        lines('{"type":"header","g":1,"prompts":[{"id":"\\u0061\\/b","ground_truth_len":3,'
              '"token_ids":[1]}]}', '{"step":1,"lengths":{"a/b":[9]}}'),
        # duplicate keys: the last wins (members and prompt fields)
        lines('{"type":"x","g":5,"type":"header","g":2,"prompts":[],"prompts":%s}' % json.dumps(P2),
              '{"step":0,"step":3,"lengths":{"a":[1,1],"b":[2,2],"a":[3,3]}}'),
        lines('{"type":"header","g":1,"prompts":[{"id":"z","id":"q","token_ids":[1],'
              '"ground_truth_len":4,"token_ids":[7,8]}]}'),
        # get<int> from floats, booleans, -0, exponents, uint64 wrap
        lines('{"type":"header","g":2.9,"max_prompt_len":1e3,"max_response_len":2048.5,'
              '"prompts":[{"id":"a","ground_truth_len":true,"token_ids":[-0,1.5,-2.5,true,false,'
              '4294967297,18446744073709551615,-2147483649,3e2,0.25e1,1E+1]}]}',
              '{"step":0,"lengths":{"a":[1.99,2]}}'),
        # "scheduled" absent: the lengths keys in map order; several steps
        lines(header(P2), {"step": 0, "lengths": {"b": [1, 2], "a": [3, 4]}},
              {"step": 9, "scheduled": ["a"], "lengths": {"a": [5, 5]}}),
        # "prompts": null / []
        lines('{"type":"header","g":1,"prompts":null}'),
        lines('{"type":"header","g":1,"prompts":[]}'),
        # long token arrays
        lines(header([{"id": f"p{i}", "ground_truth_len": 7, "token_ids": list(range(i, i + 300))}
                      for i in range(40)], g=1, max_prompt_len=1000)),
    ]


def test_json_grammar_and_conversions():
    for i, text in enumerate(grammar_cases()):
        try:
            ref().trace_prompts(text, "jsonl")
        except OracleError as e:
            pytest.fail(f"case {i}: the reference rejects it: {e}")
        same(text)


def syntax_errors():
    step = '{"step":0,"lengths":{"a":[1,2],"b":[3,4]}}'
    good = json.dumps(header(P2))
    bad = [
        good + "\n" + '{"step":0,"lengths":{"a":[1,2],"b":[3,4],}}',   # trailing comma
        good + "\n" + '{"step":0 "lengths":{}}',                       # missing comma
        good.replace('"g":', '"g" '),                                   # missing colon
        good.replace('"b"', '"b\\x"'),                                  # bad escape
        good.replace('"b"', '"b\\ud800"'),                              # lone surrogate
        good.replace('"b"', '"b\x01"'),                                 # control character
        good.replace("[1, 2, 3]", "[01, 2]"),                           # leading zero
        good.replace("[1, 2, 3]", "[1., 2]"),                           # '1.'
        good.replace("[1, 2, 3]", "[1, 2"),                              # unbalanced
        good + " x",                                                     # trailing content
        good + "\n" + step + "\n" + '{"step":1,"lengths":{"a":[1,2]}',  # unterminated (last line)
        '{"type":"other","g":1,"prompts":[]}',                          # not a header
        '[1,2]',                                                         # not an object
        '{"type":"header","prompts":[]}',                                # no g
        '{"type":"header","g":1}',                                       # no prompts
        '{"type":"header","g":"2","prompts":[]}',                        # g a string
        '{"type":"header","g":1,"prompts":[{"ground_truth_len":1,"token_ids":[1]}]}',   # no id
        '{"type":"header","g":1,"prompts":[{"id":5,"ground_truth_len":1,"token_ids":[1]}]}',
        '{"type":"header","g":1,"prompts":[{"id":"a","ground_truth_len":1,"token_ids":"x"}]}',
        '{"type":"header","g":1,"prompts":[{"id":"a","ground_truth_len":1,"token_ids":[null]}]}',
        '{"type":"header","g":1,"prompts":[3]}',                         # a prompt not an object
        good + "\n" + '{"lengths":{}}',                                  # no step
        good + "\n" + '{"step":0}',                                      # no lengths
        good + "\n" + '{"step":0,"scheduled":"a","lengths":{}}',         # scheduled not an array
        good + "\n" + '{"step":0,"scheduled":[1],"lengths":{}}',         # scheduled element
        good + "\n" + '{"step":0,"lengths":{"a":"x"}}',                  # lengths value
        good + "\n" + good,                                              # a second header
        "",                                                              # no header
        good.encode().replace(b'"b"', b'"b\xff"').decode("latin-1"),     # invalid UTF-8
    ]
    return [t.encode("latin-1") + b"\n" for t in bad]


def test_json_syntax_and_schema_errors():
    for text in syntax_errors():
        same_error(text)


def validation_errors():
    g = json.dumps(header(P2))
    bad = [
        g + "\n" + '{"step":0,"scheduled":["a","zz"],"lengths":{"a":[1,2],"zz":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["a","a"],"lengths":{"a":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["a","b"],"lengths":{"a":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["a"],"lengths":{"b":[1,2]}}',
        g + "\n" + '{"step":0,"lengths":{"a":[1,2,3],"b":[1,2]}}',
        g + "\n" + '{"step":0,"lengths":{"a":[1,0],"b":[1,2]}}',
        g + "\n" + '{"step":3,"lengths":{"a":[1,2]}}\n{"step":3,"lengths":{"a":[1,2]}}',
        g + "\n" + '{"step":-1,"lengths":{"a":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["a","b"],"lengths":{"a":[1],"b":[1,2],"zz":[1,2]}}',
        g + "\n" + '{"step":0,"lengths":{"a":[1,2],"zz":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["a","b"],"lengths":{"a":[1],"zz":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["a","b"],"lengths":{"a":[1,2],"zz":[1,2]}}',
        g + "\n" + '{"step":0,"scheduled":["b","a"],"lengths":{"a":[1,2],"b":[1,2]}}\n'
            '{"step":1,"scheduled":["a"],"lengths":{"a":[1,2],"a":[1]}}',
        g + "\n" + '{"step":0,"lengths":{}}',
        g + "\n" + '{"step":0,"lengths":null}',
        json.dumps(header([{"id": "", "ground_truth_len": 1, "token_ids": [1]}])),
        json.dumps(header(P2 + [{"id": "a", "ground_truth_len": 1, "token_ids": [1]}])),
        json.dumps(header([{"id": "a", "ground_truth_len": 1, "token_ids": []}])),
        json.dumps(header(P2, g=0)),
        json.dumps(header(P2, max_prompt_len=2)),
        json.dumps(header([{"id": "a", "ground_truth_len": 5000, "token_ids": [1]}])),
    ]
    return [t.encode() + b"\n" for t in bad]


def test_validation_errors():
    for text in validation_errors():
        same_error(text)


def test_prompts_as_an_object():
    """Range-for over an object visits its values in key order; of members
    with the same key only the last exists (its schema decides, the earlier
    ones' types do not matter, their syntax does)."""
    pa = '{"id":"a","ground_truth_len":1,"token_ids":[1,2]}'
    pb = '{"id":"b","ground_truth_len":2,"token_ids":[3]}'
    ok = [
        '{"type":"header","g":1,"prompts":{"k":%s,"j":%s}}' % (pa, pb),
        '{"type":"header","g":1,"prompts":{"k":{"id":5},"j":%s,"k":%s}}' % (pb, pa),   # bad, then replaced
        '{"type":"header","g":1,"prompts":{"\\u006b":[1],"k":%s}}' % pa,                # escaped key duplicate
        '{"type":"header","g":1,"prompts":{}}',
        '{"type":"header","g":1,"prompts":{"x":%s,"y":%s,"z":%s}}\n{"step":0,"lengths":{"a":[4],"b":[5]}}'
        % (pa, pb, pb.replace('"b"', '"c"')),
    ]
    for text in ok:
        same(text.encode() + b"\n")
    bad = [
        '{"type":"header","g":1,"prompts":{"k":%s,"k":{"id":5}}}' % pa,     # the last one is bad
        '{"type":"header","g":1,"prompts":{"k":{"id":5,},"k":%s}}' % pa,    # syntax of a dropped one
        '{"type":"header","g":1,"prompts":{"k":%s,"j":3}}' % pa,            # a member not an object
        '{"type":"header","g":1,"prompts":{"k":%s,"j":%s}}' % (pa, pa),     # duplicate prompt ids
    ]
    for text in bad:
        same_error(text.encode() + b"\n")


def test_lengths_as_an_array():
    """items() of an array: keys "0", "1", ... in map (string) order."""
    ids = [{"id": str(i), "ground_truth_len": 3, "token_ids": [i + 1]} for i in range(12)]
    arr = [[i + 1, i + 2] for i in range(12)]
    same(lines(header(ids), {"step": 0, "lengths": arr}))
    same(lines(header(ids), {"step": 0, "scheduled": ["3", "0", "11"], "lengths": {"3": [1, 1], "0": [2, 2], "11": [3, 3]}},
               {"step": 1, "scheduled": [str(i) for i in range(12)], "lengths": arr}))
    same_error(lines(header(P2), {"step": 0, "lengths": [[1, 2], [3, 4]]}))   # "0" is not a prompt
    same_error(lines(header(ids), {"step": 0, "lengths": [[1, 2], [3]]}))     # "1" needs 2 lengths
    same_error(lines(header(ids), {"step": 0, "lengths": [[1, 2], "x"]}))     # an element not an array


@pytest.mark.slow
def test_c2_shaped_jsonl_to_prefix_index():
    """8,192 prompts x 2,560 tokens as one JSONL header line: the device CSR
    equals the reference's parse and feeds the dedup index."""
    from cases import Rng
    rng = Rng(1)
    head = [rng.uniform_int(0, 31999) for _ in range(2048)]
    arr = np.random.RandomState(2).randint(0, 32000, (8192, 512))
    prompts = [(f"p{i:06d}", 100, head + arr[i].tolist()) for i in range(8192)]
    text = ref().trace_convert(trace_csv(prompts, max_prompt_len=4096))
    tr = same(text)
    direct = rs.PrefixIndex.build([p[2] for p in prompts])
    assert all(np.array_equal(a, b) for a, b in zip(tr.prefix_index().tables(), direct.tables()))


def fuzz_arrays(seed, n=300):
    """Prompt token arrays in random JSON layouts (blanks around every comma,
    signs, zeros, 18-digit and longer numbers), long enough to cross the
    warp reader's 512-byte steps anywhere."""
    rng = np.random.RandomState(seed)
    prompts = []
    for i in range(n):
        k = int(rng.randint(1, 400))
        toks = []
        for _ in range(k):
            r = rng.rand()
            if r < 0.05:
                v = "0"
            elif r < 0.1:
                v = "-" + str(rng.randint(0, 10 ** 9))
            elif r < 0.12:
                v = str(rng.randint(10 ** 17, 10 ** 18 - 1))        # 18 digits
            elif r < 0.13:
                v = str(rng.randint(10 ** 18, 2 ** 63 - 1))         # 19: the serial path
            else:
                v = str(rng.randint(0, 40000))
            toks.append(v)
        seps = [" " * int(rng.randint(0, 3)) + "," + "\t" * int(rng.randint(0, 2)) + " " * int(rng.randint(0, 2))
                for _ in range(k - 1)]
        body = toks[0] + "".join(s + t for s, t in zip(seps, toks[1:]))
        arr = "[" + " " * int(rng.randint(0, 3)) + body + " " * int(rng.randint(0, 3)) + "]"
        prompts.append('{"id":"q%05d","ground_truth_len":5,"token_ids":%s}' % (i, arr))
    return prompts


def test_token_arrays_fuzz():
    for seed in range(4):
        prompts = fuzz_arrays(seed)
        text = ('{"type":"header","g":1,"max_prompt_len":400,"prompts":[' + ",".join(prompts) + ']}\n').encode()
        same(text)


def test_token_array_defects_fuzz():
    rng = np.random.RandomState(9)
    defects = ["01", "1 2", "1,,2", "-", "--1", "1-", "0x", "- 1", "1.", ".5", "+1", "00"]
    for trial in range(24):
        prompts = fuzz_arrays(100 + trial, n=40)
        i = int(rng.randint(0, len(prompts)))
        p = prompts[i]
        lo = p.index("[") + 1
        hi = p.index("]")
        cut = [j for j in range(lo, hi) if p[j] == ","]
        at = cut[int(rng.randint(0, len(cut)))] + 1 if cut else lo
        d = defects[trial % len(defects)]
        prompts[i] = p[:at] + d + "," + p[at:] if cut else p[:lo] + d + p[hi:]
        text = ('{"type":"header","g":1,"max_prompt_len":500,"prompts":[' + ",".join(prompts) + ']}\n').encode()
        try:
            ref().trace_prompts(text, "jsonl")
            same(text)  # still valid JSON for the reference (e.g. a float)
        except OracleError:
            same_error(text)


def test_token_array_defects_before_later_errors():
    """The first pass only sizes "token_ids" (commas before the ']'); the
    arrays are read in full later. A defect in the header's arrays must still
    win over an error on a later line, and in "prompts" given as an object
    only the surviving member's array counts."""
    later = ['{"step":0 "lengths":{}}', '{"step":0,"lengths":{"zz":[1,2]}}', '{"step":0}']
    defects = ["[1 2 3 4 5]", "[1,,2]", "[01]", "[1,2,]", "[,]", "[-]", "[1.]", "[ 1 2 ]"]
    for d in defects:
        for last in (False, True):
            ps = [dict(p) for p in P2]
            head = json.dumps(header(ps))
            which = '[4]' if last else '[1, 2, 3]'
            head = head.replace(which, d)
            same_error((head + "\n").encode())
            for step in later:
                same_error((head + "\n" + step + "\n").encode())
    pa = '{"id":"a","ground_truth_len":1,"token_ids":[1,2]}'
    for d in defects:
        bad = pa.replace("[1,2]", d)
        same_error(('{"type":"header","g":1,"prompts":{"k":%s,"k":%s}}\n' % (pa, bad)).encode())
        same_error(('{"type":"header","g":1,"prompts":{"k":%s,"k":%s}}\n' % (bad, pa)).encode())  # syntax
        same_error(('{"type":"header","g":1,"prompts":{"k":%s,"j":%s}}\n{"step":0}\n' % (pa, bad)).encode())
    # a dropped member's array with a type defect (valid JSON) is ignored
    for d in ['["x"]', "[[1]]", "[null]", "[1,[2]]", "[{}]"]:
        same(('{"type":"header","g":1,"prompts":{"k":%s,"k":%s}}\n' % (pa.replace("[1,2]", d), pa)).encode())
        same_error(('{"type":"header","g":1,"prompts":{"k":%s,"k":%s}}\n{"step":0}\n'
                    % (pa, pa.replace("[1,2]", d))).encode())


def test_step_table_built_on_the_device(monkeypatch, capfd):
    """Valid steps (scheduled lists, key order, duplicate keys, several
    steps) take the device step table; a deviation falls back to the host
    path, which reports the reference's error."""
    monkeypatch.setenv("RS_TRACE_PHASES", "1")
    ok = [
        ref().trace_convert(steps_trace(3, 60, 4, g=3)[0]),
        lines(header(P2), {"step": 0, "lengths": {"b": [1, 2], "a": [3, 4], "b": [5, 6]}},
              {"step": 7, "scheduled": ["b", "a"], "lengths": {"a": [1, 1], "b": [2, 2]}}),
    ]
    for text in ok:
        capfd.readouterr()
        same(text)
        assert "steps: device table" in capfd.readouterr().err
    for text in validation_errors()[:6]:
        capfd.readouterr()
        same_error(text)
        assert "steps: device table" not in capfd.readouterr().err


def fuzz_steps(seed, n_prompts=40, n_steps=12, g=3):
    """A header of n_prompts and n_steps step lines, each a random batch
    with a random perturbation (or none): a repeated, missing, extra or
    unknown id, a wrong length count, a length out of range, duplicate
    lengths keys (the last wins), "scheduled" absent or permuted, a step
    index that does not increase."""
    rng = np.random.RandomState(seed)
    ids = [f"q{i:03d}" for i in range(n_prompts)]
    prompts = [{"id": x, "ground_truth_len": 5, "token_ids": [1 + i, 2]} for i, x in enumerate(ids)]
    out = [json.dumps(header(prompts, g=g, max_response_len=100))]
    step = 0
    for _ in range(n_steps):
        step += int(rng.randint(1, 4))
        k = int(rng.randint(1, 9))
        batch = [ids[j] for j in rng.choice(n_prompts, k, replace=False)]
        lens = {x: [int(v) for v in rng.randint(1, 101, g)] for x in batch}
        sched = list(batch)
        items = list(lens.items())
        kind = int(rng.randint(0, 12)) if rng.rand() < 0.35 else -1
        st = step
        if kind == 0:
            sched.append(sched[0])                       # scheduled twice
        elif kind == 1 and len(sched) > 1:
            sched.pop()                                  # lengths not scheduled
        elif kind == 2:
            sched.append("zz")                           # unknown id
        elif kind == 3:
            items[0] = (items[0][0], items[0][1][:-1])   # too few lengths
        elif kind == 4:
            items[-1] = (items[-1][0], [0] * g)          # out of range
        elif kind == 5:
            items[0] = (items[0][0], [101] * g)
        elif kind == 6:
            st = step - 3                                # not increasing
        elif kind == 7:
            items.append(("zz", [1] * g))                # unknown lengths key
        elif kind == 8 and len(items) > 1:
            items = items[:-1]                           # scheduled without lengths
        body_items = ",".join(f'"{x}":{json.dumps(v)}' for x, v in items)
        if kind == 9:                                    # duplicate key, the last one valid
            body_items = f'"{items[0][0]}":[1],' + body_items
        if kind == 10:                                   # duplicate key, the last one invalid
            body_items = body_items + f',"{items[0][0]}":[0]'
        s = '{"step":%d,' % st
        if kind == 11:                                   # "scheduled" permuted or absent
            rng.shuffle(sched)
        if kind != 11 or rng.rand() < 0.5:
            s += '"scheduled":%s,' % json.dumps(sched)
        s += '"lengths":{%s}}' % body_items
        out.append(s)
    return ("\n".join(out) + "\n").encode()


def test_step_table_fuzz():
    for seed in range(40):
        text = fuzz_steps(seed)
        try:
            ref().trace_steps(text, "jsonl")
        except OracleError:
            same_error(text)
            continue
        same(text)
