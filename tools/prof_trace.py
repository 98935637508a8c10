"""Time the trace parse (rs_trace_csr_parse, or rs_trace_csr_parse_jsonl with
`jsonl` as the first argument) per kernel on the C2-shaped trace text
(tests/cases.py c2_trace_text / c2_trace_jsonl)."""
import ctypes as C
import pathlib
import sys
import time

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import os  # noqa: E402
os.environ.setdefault("RS_TRACE_PHASES", "1")
import torch  # noqa: E402
from cases import c2_trace_jsonl, c2_trace_text  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402

t0 = time.perf_counter()
JSONL = len(sys.argv) > 1 and sys.argv[1] == "jsonl"
text, tok, off = (c2_trace_jsonl if JSONL else c2_trace_text)()
print(f"text {text.nbytes / 1e9:.3f} GB built in {time.perf_counter() - t0:.1f} s")
ctx = context(0)
PARSE = ctx.lib.rs_trace_csr_parse_jsonl if JSONL else ctx.lib.rs_trace_csr_parse
d = torch.from_numpy(text).cuda()
h = C.c_void_p()
names = ["jsonl_bs", "jsonl_quote", "jsonl_depth", "jsonl_tok_count", "jsonl_tok_write",
         "jsonl_first_line", "jsonl_lines", "jsonl_child_count", "jsonl_child_check", "jsonl_sizes",
         "jsonl_prompt_check", "jsonl_prompt_write", "jsonl_prompt_tables", "jsonl_step_write", "jsonl_lookup", "scan_reduce", "scan_apply"] if JSONL else [
         "trace_nl_count", "trace_nl_scan", "trace_nl_write", "trace_classify", "trace_tokens",
         "trace_ids", "string_words", "gather_keys", "trace_gather", "trace_steprow", "trace_runs",
         "trace_run_scan", "trace_group_key", "radix_hist", "radix_scan", "radix_scatter", "trace_group",
         "trace_row_err", "trace_group_check", "trace_entry_scan", "trace_step_table",
         "trace_step_lengths"]
for rep in range(4):
    timing = rep == 3
    ctx.enable_kernel_timing(timing)
    ctx.reset_kernel_timing()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(PARSE(ctx.handle, C.c_void_p(d.data_ptr()), text.nbytes, 1, C.byref(h)))
    dt = time.perf_counter() - t0
    ctx.lib.rs_trace_csr_free(h)
    print(f"rep {rep}: device parse {dt * 1e3:.2f} ms ({text.nbytes / dt / 1e9:.1f} GB/s)")
    if timing:
        for n in names:
            ms, k = ctx.kernel_time(n)
            print(f"   {n:16s} {ms:8.3f} ms over {k}")
pt = torch.from_numpy(text).pin_memory()
for rep in range(2):
    t0 = time.perf_counter()
    check(PARSE(ctx.handle, C.c_void_p(pt.data_ptr()), text.nbytes, 0, C.byref(h)))
    dt = time.perf_counter() - t0
    ctx.lib.rs_trace_csr_free(h)
    print(f"host-text parse {dt * 1e3:.2f} ms")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(pt, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch pinned H2D of the text {1e3 * (time.perf_counter() - t0):.2f} ms")
for rep in range(3):
    t0 = time.perf_counter()
    check(PARSE(ctx.handle, C.c_void_p(pt.data_ptr()), text.nbytes, 0, C.byref(h)))
    dt = time.perf_counter() - t0
    ctx.lib.rs_trace_csr_free(h)
    print(f"host-text parse {dt * 1e3:.2f} ms")
