// rs_trace.cu — the prompt table of a CSV workload trace parsed on the
// device: the '# prompt <id> <ground_truth> <tok>...' metadata
// lines of csv_from_string (proj/src/workload.cpp:169-263) straight into an
// id-sorted token CSR in HBM, ready for rs_prefix_index_build_device, without
// the reference's per-prompt std::vector / string building or the per-call
// ragged gather.
//
// Work split: the bytes are scanned on the device (newlines, then one warp
// per line for its metadata, then one warp per prompt for its tokens); the
// host only handles per-line / per-prompt scalars (line types, counts,
// offsets) and the ids.
//
// Semantics follow the reference reader line by line:
//   * lines are trimmed of " \t\r" (trim, workload.cpp:112-117), empty lines
//     skipped; '#' lines are metadata, the first other line must be the
//     column header, and metadata after it is a ParseError;
//   * "# prompt": `ms >> id >> gt` (ParseError when gt does not parse), then
//     `while (ms >> tok)` — istream integer extraction: optional sign,
//     digits, stop at the first character that is not a digit; a failed
//     extraction (no digits, or out of range for long) ends the list;
//     tokens and gt are narrowed to int;
//   * "# g" / "# max_prompt_len" / "# max_response_len": one integer (the
//     last occurrence wins); other '#' lines are ignored;
//   * prompts are then sorted by id (std::string order) and validated like
//     WorkloadTrace::validate (workload.cpp:34-60): unique non-empty ids,
//     1 <= prompt_len <= max_prompt_len, 1 <= gt <= max_response_len.
// The step rows after the header are not parsed here.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "rs_internal.cuh"
#include "rs_sort.cuh"

namespace rs {

int rank_strings_device(rs_ctx* ctx, const char* d_bytes, const int64_t* d_off, int64_t n,
                        int64_t maxlen, uint32_t* d_perm);
size_t rank_strings_device_bytes(int64_t n, int64_t maxlen);

namespace {

constexpr int64_t kChunk = 64 * 1024;  // bytes per newline-scan block
constexpr int kNlT = 256;

enum LineType : uint8_t { kEmpty = 0, kPrompt, kG, kMaxPrompt, kMaxResponse, kOtherMeta, kBody };

struct LineInfo {
  int64_t id_s;     // prompt id bytes [id_s, id_s + id_len)
  int64_t tok_pos;  // where token extraction starts
  int64_t val;      // gt (prompt) or the value (g / max_*)
  int32_t id_len;
  int32_t ntok;
  uint8_t type;
  uint8_t bad;      // 1: the metadata integer did not parse
  uint8_t serial;   // 1: numbers glued inside a field: tokens parsed by one lane
};

__device__ __forceinline__ bool is_ws(unsigned char c) {  // std::isspace, "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// One istream `>> long` at p (leading whitespace already skipped by the
// caller): returns the position after the digits, or -1 if extraction fails.
__device__ __forceinline__ int64_t parse_long_at(const unsigned char* t, int64_t p, int64_t e,
                                                 long long* v) {
  bool neg = false;
  if (p < e && (t[p] == '+' || t[p] == '-')) {
    neg = t[p] == '-';
    ++p;
  }
  if (p >= e || t[p] < '0' || t[p] > '9') return -1;
  unsigned long long m = 0;
  bool over = false;
  for (; p < e && t[p] >= '0' && t[p] <= '9'; ++p) {
    const unsigned d = t[p] - '0';
    if (m > (0xFFFFFFFFFFFFFFFFULL - d) / 10) over = true;
    else m = m * 10 + d;
  }
  const unsigned long long lim = neg ? 0x8000000000000000ULL : 0x7FFFFFFFFFFFFFFFULL;
  if (over || m > lim) return -1;
  *v = neg ? (long long)(0ULL - m) : (long long)m;
  return p;
}

// SWAR classification of 16 bytes: bit j of each mask is byte i + j.
// Bytes outside [lo, hi) read as whitespace (never digits or signs). i is
// 16-byte aligned; the text buffer is padded, so the load never faults.
struct Mask16 {
  uint32_t ws, dig, sgn;
};

__device__ __forceinline__ uint32_t pack4(uint32_t m) {  // 0xff / 0x00 bytes -> 4 bits
  return (((m >> 7) & 0x01010101u) * 0x01020408u) >> 24;
}

__device__ __forceinline__ Mask16 mask16(const unsigned char* t, int64_t i, int64_t lo, int64_t hi) {
  const uint4 v = *reinterpret_cast<const uint4*>(t + i);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  Mask16 m{0u, 0u, 0u};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t x = w[q];
    // std::isspace in the "C" locale: ' ' and '\t' .. '\r'
    const uint32_t ws = __vcmpeq4(x, 0x20202020u) | (__vcmpgeu4(x, 0x09090909u) & __vcmpleu4(x, 0x0d0d0d0du));
    const uint32_t dg = __vcmpgeu4(x, 0x30303030u) & __vcmpleu4(x, 0x39393939u);
    const uint32_t sg = __vcmpeq4(x, 0x2b2b2b2bu) | __vcmpeq4(x, 0x2d2d2d2du);
    m.ws |= pack4(ws) << (4 * q);
    m.dig |= pack4(dg) << (4 * q);
    m.sgn |= pack4(sg) << (4 * q);
  }
  uint32_t valid = 0xffffu;
  if (i < lo) valid &= lo - i >= 16 ? 0u : 0xffffu << (int)(lo - i);
  if (i + 16 > hi) valid &= hi > i ? 0xffffu >> (int)(16 - (hi - i)) : 0u;
  m.ws = (m.ws | ~valid) & 0xffffu;
  m.dig &= valid;
  m.sgn &= valid;
  return m;
}

__global__ void nl_count_kernel(const char* text, int64_t n, uint32_t* cnt) {
  __shared__ uint32_t part[kNlT / 32];
  const int64_t b0 = blockIdx.x * kChunk, b1 = min(n, b0 + kChunk);
  uint32_t c = 0;
  for (int64_t i = b0 + 16 * threadIdx.x; i < b1; i += 16 * kNlT) {
    if (i + 16 <= b1) {
      const uint4 w = *reinterpret_cast<const uint4*>(text + i);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) c += ((ws[q] >> (8 * bb)) & 0xff) == '\n';
    } else {
      for (int64_t j = i; j < b1; ++j) c += text[j] == '\n';
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kNlT / 32; ++w) s += part[w];
    cnt[blockIdx.x] = s;
  }
}

// line_start[0] = 0; line_start[1 + k] = position after the k-th newline.
// Warp w of a block owns the contiguous eighth of the chunk; lane l holds
// the 16-byte slice l of each 512-byte step, so slices, lanes and warps are
// in byte order and exclusive scans give every newline its index.
__global__ void nl_write_kernel(const char* text, int64_t n, const uint32_t* base,
                                int64_t* line_start) {
  __shared__ uint32_t wtot[kNlT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b0 = blockIdx.x * kChunk, b1 = min(n, b0 + kChunk);
  const int64_t per_w = kChunk / (kNlT / 32);
  const int64_t w0 = min(b1, b0 + w * per_w), w1 = min(b1, w0 + per_w);
  auto slice_mask = [&](int64_t i) -> uint32_t {  // bit j: byte i + j is '\n'
    uint32_t m = 0;
    if (i + 16 <= w1) {
      const uint4 v = *reinterpret_cast<const uint4*>(text + i);
      const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) m |= (uint32_t)(((ws[q] >> (8 * bb)) & 0xff) == '\n') << (4 * q + bb);
    } else {
      for (int64_t j = i; j < w1; ++j) m |= (uint32_t)(text[j] == '\n') << (j - i);
    }
    return m;
  };
  uint32_t tot = 0;
  for (int64_t i = w0 + 16 * lane; i < w1; i += 512) tot += __popc(slice_mask(i));
  tot = warp_sum(tot);
  if (lane == 0) wtot[w] = tot;
  __syncthreads();
  int64_t k = base[blockIdx.x];
  for (int q = 0; q < w; ++q) k += wtot[q];
  for (int64_t s0 = w0; s0 < w1; s0 += 512) {
    const int64_t i = s0 + 16 * lane;
    uint32_t m = i < w1 ? slice_mask(i) : 0u;
    const uint32_t c = __popc(m);
    const uint32_t incl = warp_incl_sum(c);
    int64_t pos = k + incl - c;
    while (m) {
      const int j = __ffs(m) - 1;
      line_start[1 + pos++] = i + j + 1;
      m &= m - 1;
    }
    k += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) line_start[0] = 0;
}

// `while (ms >> tok)` from p, one extraction at a time (the exact stream
// semantics, for lines where numbers are glued together, e.g. "12-3").
__device__ int serial_tokens(const unsigned char* t, int64_t p, int64_t e, int32_t* out) {
  int k = 0;
  for (;;) {
    while (p < e && is_ws(t[p])) ++p;
    long long v;
    const int64_t q = parse_long_at(t, p, e, &v);
    if (q < 0) return k;
    if (out) out[k] = (int32_t)v;
    ++k;
    p = q;
  }
}

// One warp per line: type, and for '# prompt' lines the id, gt and the
// number of tokens istream extraction yields.
__global__ void classify_kernel(const char* text_c, const int64_t* line_start, int64_t L,
                                int64_t n, LineInfo* info) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text_c);
  const int lane = threadIdx.x & 31;
  for (int64_t ln = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; ln < L;
       ln += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t s = line_start[ln];
    int64_t e = ln + 1 < L ? line_start[ln + 1] - 1 : n;  // exclude the '\n'
    LineInfo li{};
    // trim " \t\r" at both ends (sequential: a handful of characters)
    while (s < e && (t[s] == ' ' || t[s] == '\t' || t[s] == '\r')) ++s;
    while (e > s && (t[e - 1] == ' ' || t[e - 1] == '\t' || t[e - 1] == '\r')) --e;
    if (s == e) {
      li.type = kEmpty;
    } else if (t[s] != '#') {
      li.type = kBody;
    } else {
      // key: first word after '#'
      int64_t p = s + 1;
      while (p < e && is_ws(t[p])) ++p;
      int64_t k0 = p;
      while (p < e && !is_ws(t[p])) ++p;
      const int64_t klen = p - k0;
      auto key_is = [&](const char* w, int wl) {
        if (klen != wl) return false;
        for (int i = 0; i < wl; ++i)
          if (t[k0 + i] != (unsigned char)w[i]) return false;
        return true;
      };
      if (key_is("prompt", 6)) {
        li.type = kPrompt;
        while (p < e && is_ws(t[p])) ++p;
        li.id_s = p;
        while (p < e && !is_ws(t[p])) ++p;
        li.id_len = (int32_t)(p - li.id_s);
        while (p < e && is_ws(t[p])) ++p;
        long long gt = 0;
        const int64_t q = li.id_len > 0 ? parse_long_at(t, p, e, &gt) : -1;
        if (q < 0) {
          li.bad = 1;
        } else {
          li.val = gt;
          li.tok_pos = q;
        }
      } else if (key_is("g", 1) || key_is("max_prompt_len", 14) ||
                 key_is("max_response_len", 16)) {
        li.type = klen == 1 ? kG : (klen == 14 ? kMaxPrompt : kMaxResponse);
        while (p < e && is_ws(t[p])) ++p;
        long long v = 0;
        if (parse_long_at(t, p, e, &v) < 0) li.bad = 1;
        li.val = v;
      } else {
        li.type = kOtherMeta;
      }
    }
    // token count of a prompt line, warp-parallel over 32-character chunks:
    // fields start where a non-space follows a space (or the start); the
    // list ends at the first field that does not start with an integer. A
    // field that starts with one but goes on with other characters may hold
    // more numbers ("12-3" is 12, -3): such lines are counted serially.
    if (li.type == kPrompt && !li.bad) {
      // 16 bytes per lane (SWAR masks), 512 per warp step; a 32-bit line
      // position is enough within a step
      const int64_t ts = li.tok_pos;
      int count = 0;       // complete fields so far (warp-uniform)
      int stop = -1;       // tokens when the list ended (warp-uniform)
      int run = 0;         // non-space characters ending the previous step
      uint32_t prev_ws = 1u;
      if (ts < e && !is_ws(t[ts])) li.serial = 1;  // something glued to gt
      for (int64_t b0 = ts & ~(int64_t)15; b0 < e && stop < 0 && !li.serial; b0 += 512) {
        const int64_t i = b0 + 16 * lane;
        const Mask16 m = mask16(t, i, ts, e);
        const uint32_t nonws = ~m.ws & 0xffffu;
        const uint32_t up = __shfl_up_sync(0xffffffffu, m.ws >> 15, 1);
        const uint32_t wsprev = ((m.ws << 1) | (lane == 0 ? prev_ws : up)) & 0xffffu;
        const uint32_t start = nonws & wsprev;
        // a sign opens a number only if a digit follows (istream >> long)
        uint32_t dnext = __shfl_down_sync(0xffffffffu, m.dig & 1u, 1);
        if (lane == 31) {
          const int64_t j = i + 16;
          dnext = j < e && t[j] >= '0' && t[j] <= '9' ? 1u : 0u;
        }
        const uint32_t dig_next = ((m.dig >> 1) | (dnext << 15)) & 0xffffu;
        const uint32_t bad = nonws & ~m.dig & ~(start & m.sgn & dig_next) & 0xffffu;
        // non-space runs: fields of 19+ characters may overflow long, so
        // such lines take the exact path. Run ending at this lane's end:
        // a full lane extends the run from the left.
        const bool full = nonws == 0xffffu;
        const int lead = __ffs(~nonws) - 1;          // leading non-spaces (16 if full)
        const int trail = __clz(~(nonws << 16));     // trailing non-spaces (16 if full)
        int rend = full ? 16 : trail;                // run ending at this lane's end
        bool rfull = full;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int or_ = __shfl_up_sync(0xffffffffu, rend, d);
          const bool of = __shfl_up_sync(0xffffffffu, rfull, d);
          if (lane >= d && rfull) {
            rend += or_;
            rfull = of;
          }
        }
        if (rfull) rend += run;  // the whole prefix of lanes is one run from the previous step
        int left = __shfl_up_sync(0xffffffffu, rend, 1);  // run ending just before this lane
        if (lane == 0) left = run;
        if (__any_sync(0xffffffffu, (!full && left + lead >= 19) || rend >= 19)) {
          li.serial = 1;
          break;
        }
        run = __shfl_sync(0xffffffffu, rend, 31);
        const unsigned badl = __ballot_sync(0xffffffffu, bad != 0u);
        const int pc = __popc(start);
        const int pre = warp_incl_sum(pc) - pc;
        if (badl) {
          const int bl = __ffs(badl) - 1;  // the line's first bad character: lane bl ...
          const uint32_t bbad = __shfl_sync(0xffffffffu, bad, bl);
          const uint32_t bstart = __shfl_sync(0xffffffffu, start, bl);
          const int bpre = __shfl_sync(0xffffffffu, pre, bl);
          const int bit = __ffs(bbad) - 1;  // ... byte bit
          if ((bstart >> bit) & 1u) stop = count + bpre + __popc(bstart & ((1u << bit) - 1u));  // field fails
          else li.serial = 1;  // a number with more characters glued on
        } else {
          count += __shfl_sync(0xffffffffu, pre + pc, 31);
        }
        prev_ws = __shfl_sync(0xffffffffu, m.ws >> 15, 31);
      }
      li.ntok = stop >= 0 ? stop : count;
      if (li.serial) li.ntok = lane == 0 ? serial_tokens(t, ts, e, nullptr) : 0;
    }
    if (lane == 0) info[ln] = li;
  }
}

// One warp per prompt (line order): the token values. Fast-path lines hold
// complete integer fields only: per 1,024-character window the warp records
// its field starts (u16 offsets, shared memory), then every lane parses
// fields lane, lane + 32, ...; serial lines are parsed by one lane.
constexpr int kTokT = 256;
constexpr int kTokWin = 1024;
__global__ void __launch_bounds__(kTokT)
tokens_kernel(const char* text_c, const int64_t* line_start, int64_t L, int64_t n,
              const LineInfo* info, const int32_t* pline, int32_t P, const int64_t* tok_off,
              int32_t* tok) {
  __shared__ uint16_t s_fs[kTokT / 32][kTokWin / 2 + 32];  // fields start after a space: <= 512 per window
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text_c);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint16_t* fs = s_fs[w];
  for (int64_t pi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; pi < P;
       pi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t ln = pline[pi];
    const LineInfo li = info[ln];
    int64_t e = ln + 1 < L ? line_start[ln + 1] - 1 : n;
    while (e > li.tok_pos && (t[e - 1] == ' ' || t[e - 1] == '\t' || t[e - 1] == '\r')) --e;
    int32_t* out = tok + tok_off[pi];
    if (li.serial) {
      if (lane == 0) serial_tokens(t, li.tok_pos, e, out);
      continue;
    }
    int count = 0;
    uint32_t prev_wsm = 1u;
    for (int64_t w0 = li.tok_pos & ~(int64_t)15; w0 < e && count < li.ntok; w0 += kTokWin) {
      int nf = 0;
      for (int c = 0; c < kTokWin; c += 512) {  // 16 bytes per lane (SWAR masks)
        const int64_t i = w0 + c + 16 * lane;
        const Mask16 m = mask16(t, i, li.tok_pos, e);
        const uint32_t up = __shfl_up_sync(0xffffffffu, m.ws >> 15, 1);
        uint32_t start = ~m.ws & ((m.ws << 1) | (lane == 0 ? prev_wsm : up)) & 0xffffu;
        const int pc = __popc(start);
        int pos = nf + warp_incl_sum(pc) - pc;
        while (start) {
          const int j = __ffs(start) - 1;
          fs[pos++] = (uint16_t)(c + 16 * lane + j);
          start &= start - 1;
        }
        nf = __shfl_sync(0xffffffffu, pos, 31);  // lane 31's end = every start so far
        prev_wsm = __shfl_sync(0xffffffffu, m.ws >> 15, 31);
      }
      __syncwarp();
      for (int f = lane; f < nf && count + f < li.ntok; f += 32) {
        // a fast-path field is an integer of < 19 characters (the classify
        // pass sends longer runs to the serial path): no overflow check needed
        int64_t p = w0 + fs[f];
        const bool neg = t[p] == '-';
        p += (t[p] == '-' || t[p] == '+') ? 1 : 0;
        unsigned long long m = 0;
        for (; p < e && t[p] >= '0' && t[p] <= '9'; ++p) m = m * 10u + (unsigned)(t[p] - '0');
        out[count + f] = (int32_t)(neg ? 0ULL - m : m);
      }
      __syncwarp();
      count += nf;
    }
  }
}

__global__ void ids_gather_kernel(const char* text, const LineInfo* info, const int32_t* pline,
                                  int32_t P, const int64_t* id_off, char* ids) {
  for (int64_t pi = blockIdx.x; pi < P; pi += gridDim.x) {
    const LineInfo li = info[pline[pi]];
    for (int j = threadIdx.x; j < li.id_len; j += blockDim.x) ids[id_off[pi] + j] = text[li.id_s + j];
  }
}

// sorted position r takes prompt perm[r]: copy its tokens
__global__ void csr_gather_kernel(const int32_t* src, const int64_t* src_off, const uint32_t* perm,
                                  int32_t P, const int64_t* dst_off, int32_t* dst) {
  for (int64_t r = blockIdx.x; r < P; r += gridDim.x) {
    const int64_t a = src_off[perm[r]], len = src_off[perm[r] + 1] - a;
    for (int64_t j = threadIdx.x; j < len; j += blockDim.x) dst[dst_off[r] + j] = src[a + j];
  }
}

}  // namespace
}  // namespace rs

using namespace rs;

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
  // The outputs are stream-ordered allocations, complete when the parse
  // returns. The handle may outlive its context (and the context's streams),
  // so it is freed with the synchronous cudaFree on its own device.
  int device = 0;
  ~rs_trace_csr() {
    if (!d_tokens && !d_offsets) return;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    if (d_tokens) cudaFree(d_tokens);
    if (d_offsets) cudaFree(d_offsets);
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

static int parse_error(int64_t line, const std::string& what) {
  return fail(RS_E_PARSE, "<trace>:" + std::to_string(line + 1) + ": " + what);
}

extern "C" int rs_trace_csr_parse(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr,
                                  rs_trace_csr** out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out || (!text && n_bytes > 0)) return fail(RS_E_ARG, "NULL argument");
  if (n_bytes < 0) return fail(RS_E_ARG, "negative size");
  *out = nullptr;
  try {
    // 1. the bytes, 16-byte aligned and padded, in the context input buffer
    const size_t need = abytes(n_bytes + 64, 1);
    if (need > ctx->in_cap) {
      RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      if (ctx->in_buf) cudaFree(ctx->in_buf);
      ctx->in_buf = nullptr;
      ctx->in_cap = 0;
      if (cudaMalloc(&ctx->in_buf, need) != cudaSuccess) {
        cudaGetLastError();
        return fail(RS_E_NOMEM, "trace text allocation failed");
      }
      ctx->in_cap = need;
    }
    char* d_text = ctx->in_buf;
    if (n_bytes)
      RS_CUDA_TRY(cudaMemcpyAsync(d_text, text, n_bytes,
                                  device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                  ctx->stream));
    RS_CUDA_TRY(cudaMemsetAsync(d_text + n_bytes, 0, 64, ctx->stream));
    // 2. line starts
    const int64_t nblk = std::max<int64_t>(1, (n_bytes + kChunk - 1) / kChunk);
    RS_TRY(arena_reserve(ctx, abytes(nblk, 4) * 2 + 4096));
    uint32_t* cnt = arena_alloc<uint32_t>(ctx, nblk);
    uint32_t* base = arena_alloc<uint32_t>(ctx, nblk);
    RS_LAUNCH(ctx, "trace_nl_count", nl_count_kernel, (int)nblk, kNlT, 0, d_text, n_bytes, cnt);
    RS_LAUNCH(ctx, "trace_nl_scan", exclusive_scan_u32_kernel, 1, 1024, 0, cnt, base, nblk);
    uint32_t last[2] = {0, 0};
    RS_TRY(d2h(ctx, &last[0], base + nblk - 1, 4));
    RS_TRY(d2h(ctx, &last[1], cnt + nblk - 1, 4));
    RS_TRY(sync_and_check(ctx));
    const int64_t L = (int64_t)last[0] + last[1] + 1;  // lines (the last may be empty)
    AsyncBuf b_ls, b_info;
    int64_t* line_start = b_ls.alloc<int64_t>(ctx->stream, L + 1);
    LineInfo* info = b_info.alloc<LineInfo>(ctx->stream, L);
    if (!line_start || !info) return fail(RS_E_NOMEM, "trace line arrays: allocation failed");
    RS_LAUNCH(ctx, "trace_nl_write", nl_write_kernel, (int)nblk, kNlT, 0, d_text, n_bytes, base,
              line_start);
    // 3. one warp per line
    const int cgrid = (int)std::min<int64_t>((L * 32 + 255) / 256, 64 * (int64_t)ctx->num_sms);
    RS_LAUNCH(ctx, "trace_classify", classify_kernel, std::max(cgrid, 1), 256, 0, d_text,
              line_start, L, n_bytes, info);
    std::vector<LineInfo> h(L);
    RS_TRY(d2h(ctx, h.data(), info, sizeof(LineInfo) * L));
    RS_TRY(sync_and_check(ctx));
    // 4. the metadata region, in line order (errors at the first offending line)
    auto tr = new rs_trace_csr();
    std::unique_ptr<rs_trace_csr> own(tr);
    std::vector<int32_t> pline;
    int64_t header = -1;
    for (int64_t ln = 0; ln < L; ++ln) {
      const LineInfo& li = h[ln];
      if (li.type == kEmpty) continue;
      if (li.type == kBody) {
        if (header < 0) header = ln;
        continue;
      }
      if (header >= 0) return parse_error(ln, "metadata after the column header");
      if (li.type == kPrompt) {
        if (li.bad) return parse_error(ln, "malformed prompt metadata");
        pline.push_back((int32_t)ln);
      } else if (li.type == kG) {
        if (li.bad) return parse_error(ln, "malformed g metadata");
        tr->g = (int32_t)li.val;
      } else if (li.type == kMaxPrompt) {
        if (li.bad) return parse_error(ln, "malformed max_prompt_len metadata");
        tr->max_prompt_len = (int32_t)li.val;
      } else if (li.type == kMaxResponse) {
        if (li.bad) return parse_error(ln, "malformed max_response_len metadata");
        tr->max_response_len = (int32_t)li.val;
      }
    }
    if (header < 0) return fail(RS_E_PARSE, "<trace>: missing column header");
    {  // the header line, trimmed, compared with its spaces removed (workload.cpp:216-224)
      int64_t ls = 0, le = 0;
      RS_TRY(d2h(ctx, &ls, line_start + header, 8));
      if (header + 1 < L) RS_TRY(d2h(ctx, &le, line_start + header + 1, 8));
      RS_TRY(sync_and_check(ctx));
      if (header + 1 >= L) le = n_bytes + 1;
      std::string line((size_t)std::max<int64_t>(0, le - 1 - ls), '\0');
      if (!line.empty()) RS_TRY(d2h(ctx, &line[0], d_text + ls, line.size()));
      RS_TRY(sync_and_check(ctx));
      std::string compact;
      size_t a = line.find_first_not_of(" \t\r"), b = line.find_last_not_of(" \t\r");
      for (size_t i = a; a != std::string::npos && i <= b; ++i)
        if (line[i] != ' ') compact += line[i];
      if (compact != "step_idx,prompt_id,response_idx,actual_len")
        return parse_error(header, "expected column header 'step_idx,prompt_id,response_idx,actual_len'");
    }
    // 5. prompts in line order: token and id offsets
    const int32_t P = (int32_t)pline.size();
    tr->count = P;
    std::vector<int64_t> tok_off(P + 1, 0), id_off(P + 1, 0);
    int64_t maxid = 0;
    for (int32_t i = 0; i < P; ++i) {
      tok_off[i + 1] = tok_off[i] + h[pline[i]].ntok;
      id_off[i + 1] = id_off[i] + h[pline[i]].id_len;
      maxid = std::max<int64_t>(maxid, h[pline[i]].id_len);
    }
    const int64_t T = tok_off[P];
    tr->n_tokens = T;
    // prompt-level device work: the arena, sized now (the line arrays live
    // outside it)
    const size_t more = abytes(P, 4) + abytes(P + 1, 8) * 4 + abytes(T + 1, 4) +
                        abytes(id_off[P] + 1, 1) + abytes(P, 4) +
                        rank_strings_device_bytes(std::max(P, 1), std::max<int64_t>(maxid, 1)) +
                        (1 << 16);
    RS_TRY(arena_reserve(ctx, more));
    int32_t* d_pline = arena_alloc<int32_t>(ctx, std::max(P, 1));
    int64_t* d_tok_off = arena_alloc<int64_t>(ctx, P + 1);
    int64_t* d_id_off = arena_alloc<int64_t>(ctx, P + 1);
    int32_t* d_tok_line = arena_alloc<int32_t>(ctx, T + 1);
    char* d_ids = arena_alloc<char>(ctx, id_off[P] + 1);
    uint32_t* d_perm = arena_alloc<uint32_t>(ctx, std::max(P, 1));
    int64_t* d_sorted_off = arena_alloc<int64_t>(ctx, P + 1);
    if (P > 0) {
      RS_TRY(h2d(ctx, d_pline, pline.data(), 4ull * P));
      RS_TRY(h2d(ctx, d_tok_off, tok_off.data(), 8ull * (P + 1)));
      RS_TRY(h2d(ctx, d_id_off, id_off.data(), 8ull * (P + 1)));
      const int pgrid = (int)std::min<int64_t>(((int64_t)P * 32 + kTokT - 1) / kTokT, 64 * (int64_t)ctx->num_sms);
      RS_LAUNCH(ctx, "trace_tokens", tokens_kernel, pgrid, kTokT, 0, d_text, line_start, L, n_bytes,
                info, d_pline, P, d_tok_off, d_tok_line);
      RS_LAUNCH(ctx, "trace_ids", ids_gather_kernel,
                (int)std::min<int64_t>(P, 16 * (int64_t)ctx->num_sms), 32, 0, d_text, info, d_pline,
                P, d_id_off, d_ids);
      // 6. id order (std::string <) on the device
      RS_TRY(rank_strings_device(ctx, d_ids, d_id_off, P, maxid, d_perm));
    }
    std::vector<uint32_t> perm(P);
    std::vector<char> ids_line(id_off[P]);
    if (P > 0) {
      RS_TRY(d2h(ctx, perm.data(), d_perm, 4ull * P));
      if (!ids_line.empty()) RS_TRY(d2h(ctx, ids_line.data(), d_ids, ids_line.size()));
      RS_TRY(sync_and_check(ctx));
    }
    // 7. sorted prompt table + WorkloadTrace::validate's prompt rules
    tr->offsets.assign(P + 1, 0);
    tr->id_off.assign(P + 1, 0);
    tr->gt.resize(P);
    for (int32_t r = 0; r < P; ++r) {
      const uint32_t i = perm[r];
      tr->offsets[r + 1] = tr->offsets[r] + (tok_off[i + 1] - tok_off[i]);
      tr->id_off[r + 1] = tr->id_off[r] + (id_off[i + 1] - id_off[i]);
      tr->gt[r] = (int32_t)h[pline[i]].val;
    }
    tr->ids.resize(id_off[P]);
    for (int32_t r = 0; r < P; ++r) {
      const uint32_t i = perm[r];
      std::memcpy(tr->ids.data() + tr->id_off[r], ids_line.data() + id_off[i], id_off[i + 1] - id_off[i]);
    }
    if (tr->g < 1) return fail(RS_E_VALIDATION, "responses_per_prompt must be >= 1");
    if (tr->max_prompt_len < 1 || tr->max_response_len < 1)
      return fail(RS_E_VALIDATION, "trace limits must be positive");
    auto id_of = [&](int32_t r) {
      return std::string(tr->ids.data() + tr->id_off[r], tr->ids.data() + tr->id_off[r + 1]);
    };
    for (int32_t r = 0; r < P; ++r) {
      if (r > 0) {  // std::string order: bytes, then length
        const char* pa = tr->ids.data() + tr->id_off[r - 1];
        const char* pb = tr->ids.data() + tr->id_off[r];
        const int64_t la = tr->id_off[r] - tr->id_off[r - 1], lb = tr->id_off[r + 1] - tr->id_off[r];
        const int c = std::memcmp(pa, pb, (size_t)std::min(la, lb));
        if (!(c < 0 || (c == 0 && la < lb)))
          return fail(RS_E_VALIDATION, "prompts not sorted by unique id near '" + id_of(r) + "'");
      }
      const int64_t len = tr->offsets[r + 1] - tr->offsets[r];
      if (len < 1) return fail(RS_E_VALIDATION, "prompt '" + id_of(r) + "' has no tokens");
      if (len > tr->max_prompt_len)
        return fail(RS_E_VALIDATION, "prompt '" + id_of(r) + "' longer than max_prompt_len");
      if (tr->gt[r] < 1 || tr->gt[r] > tr->max_response_len)
        return fail(RS_E_VALIDATION, "prompt '" + id_of(r) + "' ground_truth_len out of range");
    }
    // 8. the id-ordered token CSR, owned by the handle
    tr->device = ctx->device;
    if (cudaMallocAsync(&tr->d_tokens, 4ull * std::max<int64_t>(T, 1), ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&tr->d_offsets, 8ull * (P + 1), ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      return fail(RS_E_NOMEM, "trace CSR allocation failed");
    }
    RS_TRY(h2d(ctx, tr->d_offsets, tr->offsets.data(), 8ull * (P + 1)));
    if (P > 0) {
      RS_TRY(h2d(ctx, d_sorted_off, tr->offsets.data(), 8ull * (P + 1)));
      RS_LAUNCH(ctx, "trace_gather", csr_gather_kernel,
                (int)std::min<int64_t>(P, 16 * (int64_t)ctx->num_sms), 256, 0, d_tok_line,
                d_tok_off, d_perm, P, d_sorted_off, tr->d_tokens);
    }
    RS_TRY(sync_and_check(ctx));
    *out = own.release();
    return RS_OK;
  } catch (const std::bad_alloc&) {
    return fail(RS_E_NOMEM, "host allocation failed");
  }
}

extern "C" int rs_trace_csr_info(const rs_trace_csr* tr, int32_t* count, int64_t* n_tokens,
                                 int64_t* id_bytes, int32_t* g, int32_t* max_prompt_len,
                                 int32_t* max_response_len) {
  if (!tr) return fail(RS_E_ARG, "NULL trace");
  if (count) *count = tr->count;
  if (n_tokens) *n_tokens = tr->n_tokens;
  if (id_bytes) *id_bytes = (int64_t)tr->ids.size();
  if (g) *g = tr->g;
  if (max_prompt_len) *max_prompt_len = tr->max_prompt_len;
  if (max_response_len) *max_response_len = tr->max_response_len;
  return RS_OK;
}

extern "C" int rs_trace_csr_device(const rs_trace_csr* tr, const int32_t** d_tokens,
                                   const int64_t** d_offsets) {
  if (!tr || !d_tokens || !d_offsets) return fail(RS_E_ARG, "NULL argument");
  *d_tokens = tr->d_tokens;
  *d_offsets = tr->d_offsets;
  return RS_OK;
}

extern "C" int rs_trace_csr_copy(rs_ctx* ctx, const rs_trace_csr* tr, int32_t* tokens,
                                 int64_t* offsets, char* id_bytes, int64_t* id_offsets,
                                 int32_t* ground_truth) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !tr) return fail(RS_E_ARG, "NULL argument");
  if (tokens && tr->n_tokens) RS_TRY(d2h(ctx, tokens, tr->d_tokens, 4ull * tr->n_tokens));
  if (offsets) std::memcpy(offsets, tr->offsets.data(), 8ull * (tr->count + 1));
  if (id_bytes && !tr->ids.empty()) std::memcpy(id_bytes, tr->ids.data(), tr->ids.size());
  if (id_offsets) std::memcpy(id_offsets, tr->id_off.data(), 8ull * (tr->count + 1));
  if (ground_truth && tr->count) std::memcpy(ground_truth, tr->gt.data(), 4ull * tr->count);
  return sync_and_check(ctx);
}

extern "C" void rs_trace_csr_free(rs_trace_csr* tr) { delete tr; }
