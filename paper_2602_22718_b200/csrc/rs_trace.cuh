// rs_trace.cuh — what the trace readers share (rs_trace.cu: CSV,
// rs_jsonl.cu: JSONL): the handle, stream-ordered temporaries, the newline
// scan and the prompt-table tail (id order, WorkloadTrace::validate's prompt
// rules, the id-ordered token CSR).
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "rs_internal.cuh"

struct rs_trace_csr {
  int32_t count = 0;
  int64_t n_tokens = 0;
  int32_t g = 1, max_prompt_len = 1024, max_response_len = 2048;
  int32_t* d_tokens = nullptr;
  int64_t* d_offsets = nullptr;
  std::vector<char> ids;
  std::vector<int64_t> id_off;
  std::vector<int32_t> gt;
  std::vector<int64_t> offsets;
  // the step table (rs_trace_csr_steps_*)
  int32_t n_steps = 0;
  int64_t n_entries = 0;
  int32_t* d_step_idx = nullptr;
  int32_t* d_entry_off = nullptr;
  int32_t* d_entry_prompt = nullptr;
  int32_t* d_lengths = nullptr;
  // The outputs are stream-ordered allocations, complete when the parse
  // returns. The handle may outlive its context (and the context's streams),
  // so it is freed with the synchronous cudaFree on its own device.
  int device = 0;
  ~rs_trace_csr() {
    void* bufs[6] = {d_tokens, d_offsets, d_step_idx, d_entry_off, d_entry_prompt, d_lengths};
    if (std::all_of(bufs, bufs + 6, [](void* b) { return b == nullptr; })) return;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
    cudaGetLastError();
  }
};

// Stream-ordered temporary (outside the arena, which is re-reserved once the
// prompt table's size is known).
struct AsyncBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~AsyncBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* alloc(cudaStream_t st, size_t count) {
    s = st;
    if (cudaMallocAsync(&p, std::max<size_t>(count * sizeof(T), 16), st) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return static_cast<T*>(p);
  }
};

// RS_TRACE_PHASES=1: host wall time of each parse phase on stderr (tools/prof_trace.py).
struct PhaseClock {
  bool on = std::getenv("RS_TRACE_PHASES") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  [trace phase] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};


namespace rs {

// "<trace>:<line + 1>: what" as RS_E_PARSE (the reader's origin:lineno form).
int trace_parse_error(int64_t line, const std::string& what);

// The text, 16-byte aligned, padded (4 KB: 64 zero bytes, then readable slack), in the context's
// input buffer (host bytes copied, device bytes copied on the device).
int trace_stage_text(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr, char** d_text);

// Line starts of the text (std::getline on '\n'; the last line may be
// empty): *L lines, line_start[L + 1] in *buf.
int trace_line_starts(rs_ctx* ctx, const char* d_text, int64_t n_bytes, AsyncBuf* buf,
                      int64_t** line_start, int64_t* L);

// The prompt table in line order (ids d_ids / d_id_off, token offsets
// d_tok_off, ground truths d_gt, all on the device) -> tr's id-sorted host
// table; *d_perm (P entries, caller-allocated) = the line index of each rank.
int trace_sorted_table(rs_ctx* ctx, rs_trace_csr* tr, int32_t P, int64_t maxid, const char* d_ids,
                       const int64_t* d_id_off, const int64_t* d_tok_off, const int32_t* d_gt,
                       uint32_t* d_perm);

// WorkloadTrace::validate's global and prompt rules (workload.cpp:34-52).
int trace_validate_prompts(const rs_trace_csr* tr);

// The id-ordered token CSR in the handle, gathered from the line-order tokens.
int trace_gather_csr(rs_ctx* ctx, rs_trace_csr* tr, const int32_t* d_tok_line,
                     const int64_t* d_tok_off, const uint32_t* d_perm);

}  // namespace rs
