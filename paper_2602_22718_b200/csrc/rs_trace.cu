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
//   * the step rows after the header (split on ',', 4 trimmed fields, the
//     integers read by std::stol) are parsed one thread per row and grouped
//     by (step run, prompt) with a device radix sort, which checks the
//     reader's response_idx order and the validator's step rules
//     (workload.cpp:53-91) and yields the step table: step_idx per step,
//     the scheduled prompts per step in batch order (indices into the
//     id-sorted table) and their g lengths in response order.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "rs_sort.cuh"
#include "rs_trace.cuh"

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
        if (parse_long_at(t, p, e, &v) < 0) {
          // `ms >> v` failed: "# g" is a ParseError; the max_* keys keep what
          // num_get stored — LONG_MAX / LONG_MIN when the digits overflow,
          // else 0 (an empty field leaves v unset in the reference: 0 here)
          li.bad = 1;
          int64_t q = p;
          const bool neg = q < e && t[q] == '-';
          if (q < e && (t[q] == '+' || t[q] == '-')) ++q;
          v = q < e && t[q] >= '0' && t[q] <= '9' ? (neg ? LLONG_MIN : LLONG_MAX) : 0;
        }
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

// -------------------------------------------------- line bookkeeping --
// The reader's line loop (workload.cpp:178-225) as reductions and one
// compaction over the classified lines, so only scalars cross to the host.
struct LineStat {
  unsigned int header;      // first body line (~0u: none) = the column header
  unsigned int first_bad;   // first malformed '# prompt' / '# g' line before it
  unsigned int meta_after;  // first '#' line after it
  unsigned int last_g, last_mp, last_mr;  // last '# g' / max_* line before it, + 1 (0: none)
  unsigned int maxid;       // longest prompt id
  int bad_type;             // LineType of first_bad
  int header_ok;            // the header line reads step_idx,prompt_id,response_idx,actual_len
  int pad;
  long long g, mp, mr;      // the values of last_g / last_mp / last_mr
  unsigned long long counts;  // prompt lines << 32 | step rows
  unsigned long long n_tok, n_idb;
};

__device__ __forceinline__ void warp_min_u32(unsigned int* addr, unsigned int v) {
  const unsigned int m = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && m != ~0u) atomicMin(addr, m);
}

__global__ void line_header_kernel(const LineInfo* info, int64_t L, LineStat* st) {
  const int64_t L32 = (L + 31) & ~(int64_t)31;  // whole warps for the reductions
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < L32;
       ln += (int64_t)gridDim.x * blockDim.x)
    warp_min_u32(&st->header, ln < L && info[ln].type == kBody ? (unsigned int)ln : ~0u);
}

// prompt lines before the header and body lines after it, as one u64 flag
// (prompt << 32 | row) for a single scan; the rare lines by atomics.
__global__ void line_flags_kernel(const LineInfo* info, int64_t L, LineStat* st,
                                  unsigned long long* flags) {
  const unsigned int header = st->header;
  const int64_t L32 = (L + 31) & ~(int64_t)31;
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < L32;
       ln += (int64_t)gridDim.x * blockDim.x) {
    unsigned int bad = ~0u, after = ~0u;
    if (ln < L) {
      const LineInfo li = info[ln];
      const bool before = (unsigned int)ln < header;
      unsigned long long f = 0;
      if (li.type == kBody) {
        f = (unsigned int)ln > header ? 1ULL : 0ULL;
      } else if (li.type != kEmpty) {
        if (!before) after = (unsigned int)ln;
        else if (li.type == kPrompt) f = 1ULL << 32;
        if (before && li.bad && (li.type == kPrompt || li.type == kG)) bad = (unsigned int)ln;
        if (before && li.type == kG) atomicMax(&st->last_g, (unsigned int)ln + 1);
        if (before && li.type == kMaxPrompt) atomicMax(&st->last_mp, (unsigned int)ln + 1);
        if (before && li.type == kMaxResponse) atomicMax(&st->last_mr, (unsigned int)ln + 1);
      }
      flags[ln] = f;
    }
    warp_min_u32(&st->first_bad, bad);
    warp_min_u32(&st->meta_after, after);
  }
}

__global__ void line_compact_kernel(const LineInfo* info, const unsigned long long* flags,
                                    const unsigned long long* pos, int64_t L, int32_t* pline,
                                    uint32_t* rline, unsigned long long* pntok,
                                    unsigned long long* pidlen, int32_t* pgt, LineStat* st) {
  const int64_t L32 = (L + 31) & ~(int64_t)31;
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < L32;
       ln += (int64_t)gridDim.x * blockDim.x) {
    unsigned int idl = 0, ntok = 0;
    if (ln < L) {
      const unsigned long long f = flags[ln];
      if (f >> 32) {
        const LineInfo li = info[ln];
        const unsigned long long i = pos[ln] >> 32;
        pline[i] = (int32_t)ln;
        pntok[i] = (unsigned long long)li.ntok;
        pidlen[i] = (unsigned long long)li.id_len;
        pgt[i] = (int32_t)li.val;
        idl = (unsigned int)li.id_len;
        ntok = (unsigned int)li.ntok;
      } else if (f) {
        rline[pos[ln] & 0xffffffffULL] = (uint32_t)ln;
      }
    }
    const unsigned int m = __reduce_max_sync(0xffffffffu, idl);
    const unsigned int sid = __reduce_add_sync(0xffffffffu, idl);
    const unsigned int stok = __reduce_add_sync(0xffffffffu, ntok);
    if ((threadIdx.x & 31) == 0 && (sid | stok)) {
      atomicMax(&st->maxid, m);
      atomicAdd(&st->n_idb, (unsigned long long)sid);
      atomicAdd(&st->n_tok, (unsigned long long)stok);
    }
  }
}

// The metadata values and the column header check (workload.cpp:216-224:
// the trimmed line with its spaces removed), one thread.
__global__ void line_meta_kernel(const char* text_c, const int64_t* line_start, const LineInfo* info,
                                 int64_t L, int64_t n, LineStat* st) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text_c);
  if (st->last_g) st->g = info[st->last_g - 1].val;
  if (st->last_mp) st->mp = info[st->last_mp - 1].val;
  if (st->last_mr) st->mr = info[st->last_mr - 1].val;
  if (st->first_bad != ~0u) st->bad_type = info[st->first_bad].type;
  if (st->header == ~0u) return;
  const int64_t h = st->header;
  int64_t s = line_start[h], e = h + 1 < L ? line_start[h + 1] - 1 : n;
  while (s < e && (t[s] == ' ' || t[s] == '\t' || t[s] == '\r')) ++s;
  while (e > s && (t[e - 1] == ' ' || t[e - 1] == '\t' || t[e - 1] == '\r')) --e;
  const char* want = "step_idx,prompt_id,response_idx,actual_len";
  int k = 0;
  bool ok = true;
  for (int64_t i = s; i < e && ok; ++i) {
    if (t[i] == ' ') continue;
    ok = want[k] != 0 && (unsigned char)want[k] == t[i];
    ++k;
  }
  st->header_ok = ok && want[k] == 0;
}

// ---------------------------------------------------------- step rows --
// The body of the CSV trace (csv_from_string, workload.cpp:226-258): after
// the column header every non-empty line is `step_idx,prompt_id,
// response_idx,actual_len` — split on ',' into exactly 4 fields, each
// trimmed of " \t\r", the three integers read by std::stol with nothing
// left over. One thread per line.
struct SRow {
  int64_t id_s;
  int32_t id_len;
  int32_t step, ridx, len;
  int32_t pidx;  // index in the id-sorted prompt table, -1: unknown id
  int32_t code;  // 0 ok, 1: not 4 fields, 2: field 0 / 2 / 3 not an integer
  int32_t nf;    // fields found (code 1)
};

// std::stol(s, &pos) with pos == s.size() on the trimmed field [p, e):
// leading isspace skipped, optional sign, >= 1 digit, no overflow of long,
// nothing after the digits.
__device__ bool stol_exact(const unsigned char* t, int64_t p, int64_t e, long long* v) {
  while (p < e && is_ws(t[p])) ++p;
  const int64_t q = parse_long_at(t, p, e, v);
  return q >= 0 && q == e;
}

__device__ __forceinline__ int id_cmp(const unsigned char* a, int64_t la, const char* b, int64_t lb) {
  const int64_t n = la < lb ? la : lb;
  for (int64_t i = 0; i < n; ++i) {
    const unsigned char cb = (unsigned char)b[i];
    if (a[i] != cb) return a[i] < cb ? -1 : 1;
  }
  return la < lb ? -1 : (la > lb ? 1 : 0);
}

__global__ void steprow_kernel(const char* text_c, const int64_t* line_start, const uint32_t* rline,
                               int64_t R, int64_t L, int64_t n, const char* sids,
                               const int64_t* sid_off, int32_t P, SRow* rows) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text_c);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ln = rline[r];
    int64_t s = line_start[ln];
    int64_t e = ln + 1 < L ? line_start[ln + 1] - 1 : n;
    while (s < e && (t[s] == ' ' || t[s] == '\t' || t[s] == '\r')) ++s;
    while (e > s && (t[e - 1] == ' ' || t[e - 1] == '\t' || t[e - 1] == '\r')) --e;
    SRow row{};
    row.pidx = -1;
    int64_t fs[4], fe[4];
    int nf = 0;
    int64_t a = s;
    for (int64_t i = s; i <= e; ++i)
      if (i == e || t[i] == ',') {
        if (nf < 4) {
          fs[nf] = a;
          fe[nf] = i;
        }
        ++nf;
        a = i + 1;
      }
    row.nf = nf;
    if (nf != 4) {
      row.code = 1;
    } else {
      for (int f = 0; f < 4; ++f) {  // trim " \t\r"
        while (fs[f] < fe[f] && (t[fs[f]] == ' ' || t[fs[f]] == '\t' || t[fs[f]] == '\r')) ++fs[f];
        while (fe[f] > fs[f] && (t[fe[f] - 1] == ' ' || t[fe[f] - 1] == '\t' || t[fe[f] - 1] == '\r')) --fe[f];
      }
      long long v0 = 0, v2 = 0, v3 = 0;
      if (!stol_exact(t, fs[0], fe[0], &v0) || !stol_exact(t, fs[2], fe[2], &v2) ||
          !stol_exact(t, fs[3], fe[3], &v3)) {
        row.code = 2;
      } else {
        row.step = (int32_t)v0;
        row.ridx = (int32_t)v2;
        row.len = (int32_t)v3;
        row.id_s = fs[1];
        row.id_len = (int32_t)(fe[1] - fs[1]);
        int lo = 0, hi = P;  // the id in the sorted prompt table
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const int c = id_cmp(t + row.id_s, row.id_len, sids + sid_off[mid], sid_off[mid + 1] - sid_off[mid]);
          if (c == 0) {
            row.pidx = mid;
            break;
          }
          if (c < 0) hi = mid;
          else lo = mid + 1;
        }
      }
    }
    rows[r] = row;
  }
}

// Rows in order: step decrease (code 3) and run starts (a new StepRecord,
// csv_from_string's `cur->step_idx != step`).
__global__ void row_runs_kernel(SRow* rows, int64_t R, uint32_t* run_head) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t step = rows[r].step;
    const int32_t prev = r > 0 ? rows[r - 1].step : 0;
    run_head[r] = r == 0 || prev != step ? 1u : 0u;
    if (r > 0 && rows[r].code == 0 && rows[r - 1].code == 0 && step < prev) rows[r].code = 3;
  }
}

// The (run, prompt) grouping key of each row (run = exclusive scan of the
// run heads + head - 1); unknown ids get P + row, a group of their own,
// checked on the host.
__global__ void row_group_key_kernel(const SRow* rows, const uint32_t* run_head,
                                     const uint32_t* run_excl, int64_t R, int32_t P,
                                     uint64_t* key, uint32_t* val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const SRow row = rows[r];
    const uint64_t run = run_excl[r] + run_head[r] - 1;
    const uint64_t pk = row.pidx >= 0 ? (uint64_t)row.pidx : (uint64_t)P + (uint64_t)r;
    key[r] = (run << 32) | pk;
    val[r] = (uint32_t)r;
  }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Sorted by (run, prompt, row): the position inside the group is the
// response_idx the reader expects (code 4 otherwise, expected kept in nf);
// group heads flagged in row order.
__global__ void row_group_kernel(SRow* rows, const uint64_t* skey, const uint32_t* srow, int64_t R,
                                 int32_t P, uint32_t* head, uint32_t* gstart) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < R;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = skey[p];
    const int64_t lo = p > 0 && skey[p - 1] == k ? lower_bound_u64(skey, p, k) : p;
    const uint32_t r = srow[p];
    head[r] = p == lo ? 1u : 0u;
    gstart[p] = (uint32_t)lo;
    const bool known = (k & 0xffffffffULL) < (uint64_t)P;
    if (known && rows[r].code == 0 && rows[r].ridx != (int32_t)(p - lo)) {
      rows[r].code = 4;
      rows[r].nf = (int32_t)(p - lo);
    }
  }
}

// First offending row (rows are in line order) and the rows with an id the
// prompt table does not hold.
__global__ void row_err_kernel(const SRow* rows, int64_t R, unsigned long long* stat) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const SRow row = rows[r];
    if (row.code) atomicMin(&stat[0], (unsigned long long)r);
    else if (row.pidx < 0) atomicAdd(&stat[1], 1ULL);
  }
}

// WorkloadTrace::validate's per-prompt step rules (workload.cpp:72-91) on
// each known group: exactly g lengths, each in [1, max_response_len]. The
// first bad group in (step, id) order — the validator's order, the map
// being id-sorted — is the smallest key.
__global__ void group_check_kernel(const SRow* rows, const uint64_t* skey, const uint32_t* srow,
                                   int64_t R, int32_t P, int32_t g, int32_t max_len,
                                   unsigned long long* bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < R;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = skey[p];
    if ((k & 0xffffffffULL) >= (uint64_t)P || (p > 0 && skey[p - 1] == k)) continue;
    int64_t e = p + 1;
    while (e < R && skey[e] == k && e - p <= g) ++e;
    bool ok = e - p == g && (e == R || skey[e] != k);
    for (int64_t q = p; ok && q < e; ++q) {
      const int32_t len = rows[srow[q]].len;
      ok = len >= 1 && len <= max_len;
    }
    if (!ok) atomicMin(bad, (unsigned long long)k);
  }
}

// The step table: run heads give step_idx and the first entry of each step;
// group heads (first appearance of an id in its step) are the entries, in
// scheduled order; every row lands at lengths[entry * g + response_idx].
__global__ void step_table_kernel(const SRow* rows, const uint32_t* run_head, const uint32_t* run_excl,
                                  const uint32_t* head, const uint32_t* epos, int64_t R,
                                  int32_t* step_idx, int32_t* entry_off, int32_t* entry_prompt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (run_head[r]) {
      step_idx[run_excl[r]] = rows[r].step;
      entry_off[run_excl[r]] = (int32_t)epos[r];
    }
    if (head[r]) entry_prompt[epos[r]] = rows[r].pidx;
  }
}

__global__ void step_lengths_kernel(const SRow* rows, const uint32_t* srow, const uint32_t* gstart,
                                    const uint32_t* epos, int64_t R, int32_t g, int32_t* lengths) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < R;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t lo = gstart[p];
    lengths[(int64_t)epos[srow[lo]] * g + (p - lo)] = rows[srow[p]].len;
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

namespace rs {
int trace_parse_error(int64_t line, const std::string& what) {
  return fail(RS_E_PARSE, "<trace>:" + std::to_string(line + 1) + ": " + what);
}
}  // namespace rs

static int parse_error(int64_t line, const std::string& what) { return trace_parse_error(line, what); }

static std::string trim_ws(const std::string& s) {  // trim, workload.cpp:112-117
  const size_t a = s.find_first_not_of(" \t\r");
  if (a == std::string::npos) return "";
  return s.substr(a, s.find_last_not_of(" \t\r") - a + 1);
}

// The step rows of the CSV body (csv_from_string's loop after the column
// header, workload.cpp:226-258) on the device, in two stages so the errors
// come in the reference's order: parse() raises the rows' ParseErrors (the
// caller has already raised the metadata ones before them in line order),
// table() runs after the prompt rules of WorkloadTrace::validate with the
// step rules (workload.cpp:53-91) and writes the step table into the handle.
struct StepRows {
  rs_ctx* ctx;
  rs_trace_csr* tr;
  const char* d_text;
  const char* text;  // the caller's bytes (device memory when device_ptr)
  int device_ptr;
  int64_t n_bytes, L;
  const int64_t* line_start;
  const uint32_t* d_rline = nullptr;  // the R body rows after the header, line order
  int64_t R = 0;
  AsyncBuf buf;
  SRow* rows = nullptr;
  uint32_t *run_head = nullptr, *run_excl = nullptr, *head = nullptr,
           *epos = nullptr, *gstart = nullptr, *srow = nullptr;
  uint64_t* skey = nullptr;
  uint32_t* scan_part = nullptr;
  unsigned long long* stat = nullptr;  // first error row, unknown-id rows, first bad group
  std::vector<SRow> h_rows;            // downloaded only on the error paths
  int64_t first_unknown = -1;

  int grid(int64_t n) const {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 32 * (int64_t)ctx->num_sms));
  }

  std::string line_text(int64_t ln) {
    int64_t a = 0, b = 0;
    if (d2h(ctx, &a, line_start + ln, 8) || (ln + 1 < L && d2h(ctx, &b, line_start + ln + 1, 8)) ||
        sync_and_check(ctx))
      return "";
    b = ln + 1 < L ? b - 1 : n_bytes;
    std::string out((size_t)std::max<int64_t>(0, b - a), '\0');
    if (!out.empty() && (d2h(ctx, &out[0], d_text + a, out.size()) || sync_and_check(ctx))) return "";
    return out;
  }

  int rows_to_host() {
    if ((int64_t)h_rows.size() == R) return RS_OK;
    h_rows.resize(R);
    RS_TRY(d2h(ctx, h_rows.data(), rows, sizeof(SRow) * R));
    return sync_and_check(ctx);
  }

  std::string id_text(const SRow& row) {
    std::string id((size_t)row.id_len, '\0');
    if (row.id_len && d2h(ctx, &id[0], d_text + row.id_s, id.size()) == RS_OK) sync_and_check(ctx);
    return id;
  }

  int64_t line_of(int64_t r) {
    uint32_t ln = 0;
    if (d2h(ctx, &ln, d_rline + r, 4) || sync_and_check(ctx)) return -1;
    return ln;
  }

  // The reader's message for row r (workload.cpp:227-253), rebuilt on the host.
  int row_error(int64_t r, const SRow& row) {
    const int64_t ln = line_of(r);
    if (row.code == 1) return parse_error(ln, "expected 4 fields, got " + std::to_string(row.nf));
    if (row.code == 3) return parse_error(ln, "step indices must not decrease");
    if (row.code == 4)
      return parse_error(ln, "response_idx out of order for prompt '" + id_text(row) + "' (expected " +
                                 std::to_string(row.nf) + ", got " + std::to_string(row.ridx) + ")");
    std::vector<std::string> f(1);
    for (char c : trim_ws(line_text(ln))) {
      if (c == ',') f.emplace_back();
      else f.back() += c;
    }
    for (int i : {0, 2, 3}) {
      const std::string v = trim_ws(f[i]);
      bool ok = true;
      try {
        size_t pos = 0;
        (void)std::stol(v, &pos);
        ok = pos == v.size();
      } catch (const std::exception&) {
        ok = false;
      }
      if (!ok) return parse_error(ln, "expected integer, got '" + v + "'");
    }
    return parse_error(ln, "malformed step row");
  }

  int parse(int64_t meta_after) {
    if (R == 0) return meta_after >= 0 ? parse_error(meta_after, "metadata after the column header") : RS_OK;
    if (R >= (int64_t)INT32_MAX / 2) return fail(RS_E_ARG, "trace has too many step rows");
    const int32_t P = tr->count;
    // device copies of the id-sorted prompt ids for the lookup
    const size_t scratch = radix_sort_scratch_bytes64(R) + scan_scratch_bytes(R, 4);
    const size_t bytes = abytes(R, sizeof(SRow)) + abytes(R, 4) * 6 + abytes(R, 8) + abytes(4, 8) +
                         abytes(tr->ids.size() + 1, 1) + abytes(P + 1, 8) + scratch;
    char* b = buf.alloc<char>(ctx->stream, bytes);
    if (!b) return fail(RS_E_NOMEM, "trace step rows: allocation failed");
    auto carve = [&](size_t n) {
      char* q = b;
      b += n;
      return q;
    };
    rows = (SRow*)carve(abytes(R, sizeof(SRow)));
    run_head = (uint32_t*)carve(abytes(R, 4));
    run_excl = (uint32_t*)carve(abytes(R, 4));
    head = (uint32_t*)carve(abytes(R, 4));
    epos = (uint32_t*)carve(abytes(R, 4));
    gstart = (uint32_t*)carve(abytes(R, 4));
    uint32_t* val = (uint32_t*)carve(abytes(R, 4));
    uint64_t* key = (uint64_t*)carve(abytes(R, 8));
    stat = (unsigned long long*)carve(abytes(4, 8));
    char* d_sids = carve(abytes(tr->ids.size() + 1, 1));
    int64_t* d_sid_off = (int64_t*)carve(abytes(P + 1, 8));
    scan_part = (uint32_t*)carve(scan_scratch_bytes(R, 4));
    char* d_scratch = carve(radix_sort_scratch_bytes64(R));
    if (!tr->ids.empty()) RS_TRY(h2d(ctx, d_sids, tr->ids.data(), tr->ids.size()));
    RS_TRY(h2d(ctx, d_sid_off, tr->id_off.data(), 8ull * (P + 1)));
    const unsigned long long init[4] = {~0ULL, 0ULL, ~0ULL, 0ULL};
    RS_TRY(h2d(ctx, stat, init, sizeof init));
    const int gr = grid(R);
    RS_LAUNCH(ctx, "trace_steprow", steprow_kernel, gr, 256, 0, d_text, line_start, d_rline, R, L,
              n_bytes, d_sids, d_sid_off, P, rows);
    RS_LAUNCH(ctx, "trace_runs", row_runs_kernel, gr, 256, 0, rows, R, run_head);
    RS_TRY(exclusive_scan<uint32_t>(ctx, run_head, run_excl, R, scan_part, nullptr));
    RS_LAUNCH(ctx, "trace_group_key", row_group_key_kernel, gr, 256, 0, rows, run_head, run_excl, R, P,
              key, val);
    RS_TRY(radix_sort_pairs(ctx, key, val, R, d_scratch, &skey, &srow));
    RS_LAUNCH(ctx, "trace_group", row_group_kernel, gr, 256, 0, rows, skey, srow, R, P, head, gstart);
    RS_LAUNCH(ctx, "trace_row_err", row_err_kernel, gr, 256, 0, rows, R, stat);
    unsigned long long st[2];
    RS_TRY(d2h(ctx, st, stat, sizeof st));
    RS_TRY(sync_and_check(ctx));
    int64_t err_r = st[0] == ~0ULL ? R : (int64_t)st[0];
    int64_t host_err = -1;  // an unknown id's response_idx out of order
    if (st[1] > 0) {
      RS_TRY(rows_to_host());
      std::string host_text;
      const char* t = text;
      if (device_ptr) {
        host_text.resize((size_t)n_bytes);
        if (n_bytes) RS_TRY(d2h(ctx, &host_text[0], d_text, (size_t)n_bytes));
        RS_TRY(sync_and_check(ctx));
        t = host_text.data();
      }
      std::map<std::pair<int64_t, std::string>, int32_t> seen;
      int64_t run = -1;
      for (int64_t r = 0; r < err_r; ++r) {
        const SRow& row = h_rows[r];
        if (r == 0 || row.step != h_rows[r - 1].step) ++run;
        if (row.pidx >= 0) continue;
        if (first_unknown < 0) first_unknown = r;
        int32_t& c = seen[{run, std::string(t + row.id_s, t + row.id_s + row.id_len)}];
        if (row.ridx != c) {
          h_rows[r].code = 4;
          h_rows[r].nf = c;
          host_err = r;
          break;
        }
        ++c;
      }
    }
    if (host_err >= 0) err_r = host_err;
    if (err_r < R && (meta_after < 0 || line_of(err_r) < meta_after)) {
      SRow row;
      if (host_err >= 0) row = h_rows[err_r];
      else {
        RS_TRY(d2h(ctx, &row, rows + err_r, sizeof row));
        RS_TRY(sync_and_check(ctx));
      }
      return row_error(err_r, row);
    }
    if (meta_after >= 0) return parse_error(meta_after, "metadata after the column header");
    return RS_OK;
  }

  int table() {
    if (R == 0) return RS_OK;
    const int32_t P = tr->count, g = tr->g;
    const int gr = grid(R);
    RS_LAUNCH(ctx, "trace_group_check", group_check_kernel, gr, 256, 0, rows, skey, srow, R, P, g,
              tr->max_response_len, stat + 2);
    RS_TRY(exclusive_scan<uint32_t>(ctx, head, epos, R, scan_part, nullptr));
    uint32_t tail[4];
    unsigned long long bad = 0;
    SRow row0;
    RS_TRY(d2h(ctx, &tail[0], run_excl + R - 1, 4));
    RS_TRY(d2h(ctx, &tail[1], run_head + R - 1, 4));
    RS_TRY(d2h(ctx, &tail[2], epos + R - 1, 4));
    RS_TRY(d2h(ctx, &tail[3], head + R - 1, 4));
    RS_TRY(d2h(ctx, &bad, stat + 2, 8));
    RS_TRY(d2h(ctx, &row0, rows, sizeof row0));
    RS_TRY(sync_and_check(ctx));
    const int32_t S = (int32_t)(tail[0] + tail[1]);
    const int64_t E = (int64_t)tail[2] + tail[3];
    // WorkloadTrace::validate, step by step (workload.cpp:53-91)
    auto step_err = [&](int32_t step, const std::string& what) {
      return fail(RS_E_VALIDATION, "step " + std::to_string(step) + what);
    };
    if (row0.step <= -1)
      return fail(RS_E_VALIDATION, "step indices must be strictly increasing at step " +
                                       std::to_string(row0.step));
    const int64_t bad_run = bad == ~0ULL ? -1 : (int64_t)(bad >> 32);
    if (first_unknown >= 0) {
      int64_t run = 0;
      for (int64_t r = 1; r <= first_unknown; ++r) run += h_rows[r].step != h_rows[r - 1].step;
      if (bad_run < 0 || run <= bad_run) {
        const SRow& u = h_rows[first_unknown];
        return step_err(u.step, " schedules unknown prompt '" + id_text(u) + "'");
      }
    }
    if (bad_run >= 0) {
      RS_TRY(rows_to_host());
      std::vector<uint64_t> hk(R);
      std::vector<uint32_t> hs(R);
      RS_TRY(d2h(ctx, hk.data(), skey, 8ull * R));
      RS_TRY(d2h(ctx, hs.data(), srow, 4ull * R));
      RS_TRY(sync_and_check(ctx));
      const int64_t lo = std::lower_bound(hk.begin(), hk.end(), (uint64_t)bad) - hk.begin();
      const int64_t hi = std::upper_bound(hk.begin(), hk.end(), (uint64_t)bad) - hk.begin();
      const SRow& first = h_rows[hs[lo]];
      const int32_t pidx = (int32_t)(bad & 0xffffffffULL);
      const std::string id(tr->ids.data() + tr->id_off[pidx], tr->ids.data() + tr->id_off[pidx + 1]);
      if (hi - lo != g)
        return step_err(first.step, " prompt '" + id + "' needs exactly " + std::to_string(g) +
                                        " response lengths");
      for (int64_t q = lo; q < hi; ++q) {
        const int32_t l = h_rows[hs[q]].len;
        if (l < 1 || l > tr->max_response_len)
          return step_err(first.step, " prompt '" + id + "' response length out of range: " +
                                          std::to_string(l));
      }
    }
    // the step table, owned by the handle
    tr->n_steps = S;
    tr->n_entries = E;
    if (cudaMallocAsync(&tr->d_step_idx, 4ull * S, ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&tr->d_entry_off, 4ull * (S + 1), ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&tr->d_entry_prompt, 4ull * std::max<int64_t>(E, 1), ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&tr->d_lengths, 4ull * std::max<int64_t>(E * g, 1), ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      return fail(RS_E_NOMEM, "trace step table allocation failed");
    }
    const int32_t e32 = (int32_t)E;
    RS_TRY(h2d(ctx, tr->d_entry_off + S, &e32, 4));
    RS_LAUNCH(ctx, "trace_step_table", step_table_kernel, gr, 256, 0, rows, run_head, run_excl, head,
              epos, R, tr->d_step_idx, tr->d_entry_off, tr->d_entry_prompt);
    RS_LAUNCH(ctx, "trace_step_lengths", step_lengths_kernel, gr, 256, 0, rows, srow, gstart, epos, R,
              g, tr->d_lengths);
    return RS_OK;
  }
};

extern "C" int rs_trace_csr_parse(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr,
                                  rs_trace_csr** out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out || (!text && n_bytes > 0)) return fail(RS_E_ARG, "NULL argument");
  if (n_bytes < 0) return fail(RS_E_ARG, "negative size");
  *out = nullptr;
  try {
    PhaseClock clk;
    // 1. the bytes; 2. line starts
    char* d_text = nullptr;
    RS_TRY(trace_stage_text(ctx, text, n_bytes, device_ptr, &d_text));
    clk.mark("text");
    AsyncBuf b_ls, b_info;
    int64_t* line_start = nullptr;
    int64_t L = 0;
    RS_TRY(trace_line_starts(ctx, d_text, n_bytes, &b_ls, &line_start, &L));
    clk.mark("line starts");
    LineInfo* info = b_info.alloc<LineInfo>(ctx->stream, L);
    if (!info) return fail(RS_E_NOMEM, "trace line arrays: allocation failed");
    // 3. one warp per line
    if (L >= (int64_t)UINT32_MAX - 1) return fail(RS_E_ARG, "trace has too many lines");
    const int cgrid = (int)std::min<int64_t>((L * 32 + 255) / 256, 64 * (int64_t)ctx->num_sms);
    RS_LAUNCH(ctx, "trace_classify", classify_kernel, std::max(cgrid, 1), 256, 0, d_text,
              line_start, L, n_bytes, info);
    // 4. the line loop's bookkeeping on the device: header, metadata, the
    // prompt lines and the step rows compacted in line order
    AsyncBuf b_lines;
    const size_t lbytes = abytes(1, sizeof(LineStat)) + abytes(L, 8) * 4 + abytes(L, 4) * 3 +
                          scan_scratch_bytes(L, 8);
    char* lb = b_lines.alloc<char>(ctx->stream, lbytes);
    if (!lb) return fail(RS_E_NOMEM, "trace line arrays: allocation failed");
    auto carve = [&](size_t nb) {
      char* q = lb;
      lb += nb;
      return q;
    };
    LineStat* d_st = (LineStat*)carve(abytes(1, sizeof(LineStat)));
    auto* flags = (unsigned long long*)carve(abytes(L, 8));
    auto* pos = (unsigned long long*)carve(abytes(L, 8));
    auto* pntok = (unsigned long long*)carve(abytes(L + 1, 8));   // -> token offsets (line order)
    auto* pidlen = (unsigned long long*)carve(abytes(L + 1, 8));  // -> id offsets
    int32_t* d_pline = (int32_t*)carve(abytes(L, 4));
    uint32_t* d_rline = (uint32_t*)carve(abytes(L, 4));
    int32_t* d_pgt = (int32_t*)carve(abytes(L, 4));
    auto* scan_part = (unsigned long long*)carve(scan_scratch_bytes(L, 8));
    LineStat st0{};
    st0.header = st0.first_bad = st0.meta_after = ~0u;
    st0.g = 1;
    st0.mp = 1024;
    st0.mr = 2048;
    RS_TRY(h2d(ctx, d_st, &st0, sizeof st0));
    const int lgrid = (int)std::max<int64_t>(1, std::min<int64_t>((L + 255) / 256, 32 * (int64_t)ctx->num_sms));
    RS_LAUNCH(ctx, "trace_line_header", line_header_kernel, lgrid, 256, 0, info, L, d_st);
    RS_LAUNCH(ctx, "trace_line_flags", line_flags_kernel, lgrid, 256, 0, info, L, d_st, flags);
    RS_TRY(exclusive_scan<unsigned long long>(ctx, flags, pos, L, scan_part, &d_st->counts));
    RS_LAUNCH(ctx, "trace_line_compact", line_compact_kernel, lgrid, 256, 0, info, flags, pos, L,
              d_pline, d_rline, pntok, pidlen, d_pgt, d_st);
    RS_LAUNCH(ctx, "trace_line_meta", line_meta_kernel, 1, 1, 0, d_text, line_start, info, L, n_bytes,
              d_st);
    LineStat st;
    RS_TRY(d2h(ctx, &st, d_st, sizeof st));
    RS_TRY(sync_and_check(ctx));
    clk.mark("classify + lines");
    auto tr = new rs_trace_csr();
    std::unique_ptr<rs_trace_csr> own(tr);
    tr->device = ctx->device;
    // errors in line order: malformed metadata before the header, then the header
    if (st.first_bad != ~0u)
      return parse_error(st.first_bad, st.bad_type == kG ? "malformed g metadata" : "malformed prompt metadata");
    if (st.header == ~0u) return fail(RS_E_PARSE, "<trace>: missing column header");
    if (!st.header_ok)
      return parse_error(st.header, "expected column header 'step_idx,prompt_id,response_idx,actual_len'");
    tr->g = (int32_t)st.g;
    tr->max_prompt_len = (int32_t)st.mp;
    tr->max_response_len = (int32_t)st.mr;
    const int64_t meta_after = st.meta_after == ~0u ? -1 : (int64_t)st.meta_after;
    StepRows sr{ctx, tr, d_text, text, device_ptr, n_bytes, L, line_start, d_rline,
                (int64_t)(st.counts & 0xffffffffULL)};
    // 5. prompts in line order: token and id offsets (scans in place)
    const int32_t P = (int32_t)(st.counts >> 32);
    const int64_t T = (int64_t)st.n_tok, IDB = (int64_t)st.n_idb;
    const int64_t maxid = st.maxid;
    tr->count = P;
    tr->n_tokens = T;
    RS_TRY(exclusive_scan<unsigned long long>(ctx, pntok, pntok, P, scan_part, pntok + P));
    RS_TRY(exclusive_scan<unsigned long long>(ctx, pidlen, pidlen, P, scan_part, pidlen + P));
    const int64_t* d_tok_off = (const int64_t*)pntok;
    const int64_t* d_id_off = (const int64_t*)pidlen;
    // prompt-level device work: the arena, sized now (the line arrays live
    // outside it)
    const size_t more = abytes(T + 1, 4) + abytes(IDB + 1, 1) + abytes(P, 4) +
                        rank_strings_device_bytes(std::max(P, 1), std::max<int64_t>(maxid, 1)) +
                        (1 << 16);
    RS_TRY(arena_reserve(ctx, more));
    int32_t* d_tok_line = arena_alloc<int32_t>(ctx, T + 1);
    char* d_ids = arena_alloc<char>(ctx, IDB + 1);
    uint32_t* d_perm = arena_alloc<uint32_t>(ctx, std::max(P, 1));
    if (P > 0) {
      const int pgrid = (int)std::min<int64_t>(((int64_t)P * 32 + kTokT - 1) / kTokT, 64 * (int64_t)ctx->num_sms);
      RS_LAUNCH(ctx, "trace_tokens", tokens_kernel, pgrid, kTokT, 0, d_text, line_start, L, n_bytes,
                info, d_pline, P, d_tok_off, d_tok_line);
      RS_LAUNCH(ctx, "trace_ids", ids_gather_kernel,
                (int)std::min<int64_t>(P, 16 * (int64_t)ctx->num_sms), 32, 0, d_text, info, d_pline,
                P, d_id_off, d_ids);
    }
    // 6. id order (std::string <) on the device; 7. the sorted host table
    RS_TRY(trace_sorted_table(ctx, tr, P, maxid, d_ids, d_id_off, d_tok_off, d_pgt, d_perm));
    clk.mark("id rank + sorted table");
    // 8. the step rows' ParseErrors, then the validator
    RS_TRY(sr.parse(meta_after));
    clk.mark("step rows parse");
    RS_TRY(trace_validate_prompts(tr));
    RS_TRY(sr.table());
    clk.mark("step table");
    // 9. the id-ordered token CSR, owned by the handle
    RS_TRY(trace_gather_csr(ctx, tr, d_tok_line, d_tok_off, d_perm));
    clk.mark("CSR gather");
    *out = own.release();
    return RS_OK;
  } catch (const std::bad_alloc&) {
    return fail(RS_E_NOMEM, "host allocation failed");
  }
}

namespace rs {

int trace_stage_text(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr, char** d_text) {
  // 4 KB of slack: the warp scans load whole 512-byte steps (two 1 KB
  // windows in the token scan) past the end of the last line; the bytes
  // beyond the text are masked out, they only have to be readable
  const size_t need = abytes(n_bytes + 4096, 1);
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
  *d_text = ctx->in_buf;
  if (n_bytes)
    RS_CUDA_TRY(cudaMemcpyAsync(*d_text, text, n_bytes,
                                device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                ctx->stream));
  RS_CUDA_TRY(cudaMemsetAsync(*d_text + n_bytes, 0, 64, ctx->stream));
  return RS_OK;
}

int trace_line_starts(rs_ctx* ctx, const char* d_text, int64_t n_bytes, AsyncBuf* buf,
                      int64_t** line_start, int64_t* L_out) {
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
  if (L >= (int64_t)UINT32_MAX - 1) return fail(RS_E_ARG, "trace has too many lines");
  *line_start = buf->alloc<int64_t>(ctx->stream, L + 1);
  if (!*line_start) return fail(RS_E_NOMEM, "trace line arrays: allocation failed");
  RS_LAUNCH(ctx, "trace_nl_write", nl_write_kernel, (int)nblk, kNlT, 0, d_text, n_bytes, base,
            *line_start);
  *L_out = L;
  return RS_OK;
}

int trace_sorted_table(rs_ctx* ctx, rs_trace_csr* tr, int32_t P, int64_t maxid, const char* d_ids,
                       const int64_t* d_id_off, const int64_t* d_tok_off, const int32_t* d_gt,
                       uint32_t* d_perm) {
  std::vector<uint32_t> perm(P);
  std::vector<int64_t> tok_off(P + 1, 0), id_off(P + 1, 0);
  std::vector<int32_t> gt_line(P);
  std::vector<char> ids_line;
  if (P > 0) {
    RS_TRY(rank_strings_device(ctx, d_ids, d_id_off, P, std::max<int64_t>(maxid, 1), d_perm));
    RS_TRY(d2h(ctx, perm.data(), d_perm, 4ull * P));
    RS_TRY(d2h(ctx, tok_off.data(), d_tok_off, 8ull * (P + 1)));
    RS_TRY(d2h(ctx, id_off.data(), d_id_off, 8ull * (P + 1)));
    RS_TRY(d2h(ctx, gt_line.data(), d_gt, 4ull * P));
    RS_TRY(sync_and_check(ctx));
    ids_line.resize(id_off[P]);
    if (!ids_line.empty()) RS_TRY(d2h(ctx, ids_line.data(), d_ids, ids_line.size()));
    RS_TRY(sync_and_check(ctx));
  }
  tr->count = P;
  tr->n_tokens = tok_off[P];
  tr->offsets.assign(P + 1, 0);
  tr->id_off.assign(P + 1, 0);
  tr->gt.resize(P);
  for (int32_t r = 0; r < P; ++r) {
    const uint32_t i = perm[r];
    tr->offsets[r + 1] = tr->offsets[r] + (tok_off[i + 1] - tok_off[i]);
    tr->id_off[r + 1] = tr->id_off[r] + (id_off[i + 1] - id_off[i]);
    tr->gt[r] = gt_line[i];
  }
  tr->ids.resize(id_off[P]);
  for (int32_t r = 0; r < P; ++r) {
    const uint32_t i = perm[r];
    std::memcpy(tr->ids.data() + tr->id_off[r], ids_line.data() + id_off[i], id_off[i + 1] - id_off[i]);
  }
  return RS_OK;
}

int trace_validate_prompts(const rs_trace_csr* tr) {
  if (tr->g < 1) return fail(RS_E_VALIDATION, "responses_per_prompt must be >= 1");
  if (tr->max_prompt_len < 1 || tr->max_response_len < 1)
    return fail(RS_E_VALIDATION, "trace limits must be positive");
  const int32_t P = tr->count;
  auto id_of = [&](int32_t r) {
    return std::string(tr->ids.data() + tr->id_off[r], tr->ids.data() + tr->id_off[r + 1]);
  };
  for (int32_t r = 0; r < P; ++r) {
    if (tr->id_off[r + 1] == tr->id_off[r]) return fail(RS_E_VALIDATION, "prompt with empty id");
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
  return RS_OK;
}

int trace_gather_csr(rs_ctx* ctx, rs_trace_csr* tr, const int32_t* d_tok_line,
                     const int64_t* d_tok_off, const uint32_t* d_perm) {
  const int32_t P = tr->count;
  const int64_t T = tr->n_tokens;
  tr->device = ctx->device;
  if (cudaMallocAsync(&tr->d_tokens, 4ull * std::max<int64_t>(T, 1), ctx->stream) != cudaSuccess ||
      cudaMallocAsync(&tr->d_offsets, 8ull * (P + 1), ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_E_NOMEM, "trace CSR allocation failed");
  }
  RS_TRY(h2d(ctx, tr->d_offsets, tr->offsets.data(), 8ull * (P + 1)));
  if (P > 0)
    RS_LAUNCH(ctx, "trace_gather", csr_gather_kernel,
              (int)std::min<int64_t>(P, 16 * (int64_t)ctx->num_sms), 256, 0, d_tok_line, d_tok_off,
              d_perm, P, (const int64_t*)tr->d_offsets, tr->d_tokens);
  return sync_and_check(ctx);
}

}  // namespace rs

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

extern "C" int rs_trace_csr_steps_info(const rs_trace_csr* tr, int32_t* n_steps, int64_t* n_entries) {
  if (!tr) return fail(RS_E_ARG, "NULL trace");
  if (n_steps) *n_steps = tr->n_steps;
  if (n_entries) *n_entries = tr->n_entries;
  return RS_OK;
}

extern "C" int rs_trace_csr_steps_device(const rs_trace_csr* tr, const int32_t** step_idx,
                                         const int32_t** entry_off, const int32_t** entry_prompt,
                                         const int32_t** lengths) {
  if (!tr) return fail(RS_E_ARG, "NULL trace");
  if (step_idx) *step_idx = tr->d_step_idx;
  if (entry_off) *entry_off = tr->d_entry_off;
  if (entry_prompt) *entry_prompt = tr->d_entry_prompt;
  if (lengths) *lengths = tr->d_lengths;
  return RS_OK;
}

extern "C" int rs_trace_csr_steps_copy(rs_ctx* ctx, const rs_trace_csr* tr, int32_t* step_idx,
                                       int32_t* entry_off, int32_t* entry_prompt, int32_t* lengths) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !tr) return fail(RS_E_ARG, "NULL argument");
  const int64_t S = tr->n_steps, E = tr->n_entries;
  if (step_idx && S) RS_TRY(d2h(ctx, step_idx, tr->d_step_idx, 4ull * S));
  if (entry_off) {
    if (S) RS_TRY(d2h(ctx, entry_off, tr->d_entry_off, 4ull * (S + 1)));
    else entry_off[0] = 0;
  }
  if (entry_prompt && E) RS_TRY(d2h(ctx, entry_prompt, tr->d_entry_prompt, 4ull * E));
  if (lengths && E) RS_TRY(d2h(ctx, lengths, tr->d_lengths, 4ull * E * tr->g));
  return sync_and_check(ctx);
}

extern "C" void rs_trace_csr_free(rs_trace_csr* tr) { delete tr; }
