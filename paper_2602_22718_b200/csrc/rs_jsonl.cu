// rs_jsonl.cu — a JSONL workload trace parsed on the device:
// jsonl_from_string (proj/src/workload.cpp:294-352), one JSON document per
// line read by nlohmann::json, into the same handle as the CSV reader
// (rs_trace.cu): the id-sorted token CSR in HBM and the step table.
//
// Work split.
//   1. Structural index over the whole text, 64 bytes per thread: backslash
//      runs -> escaped characters -> unescaped quotes -> in-string masks (a
//      scan of quote parities) -> bracket depth outside strings (a scan of
//      depth deltas). Two lists come out: every structural character at
//      level <= 1 (the top-level value and its direct members), and every
//      comma at level 2 (the separators of the members' own containers).
//      The states run across lines without a reset: a valid line ends
//      outside strings at depth 0, so a wrong state can only follow a line
//      that is itself an error, which is reported first.
//   2. One thread per line walks the top-level object sequentially: keys,
//      scalars, and each member container jumped over through the level-1
//      list (its matching closer).
//   3. One thread per container child (the spans between the level-2
//      commas): each child is validated as a complete JSON value (array
//      members) or "key": value member (object members) and the schema's
//      fields are extracted — prompt objects, scheduled ids, length lists.
//      A line is valid iff its skeleton and all its children are, whatever
//      the split, so the reader accepts exactly what nlohmann accepts (up to
//      the constructs listed below).
//   4. Prompts: counts -> scans -> writes -> the shared id-order tail
//      (rs_trace.cuh). Steps: the extracted records go to the host, which
//      applies std::map / scheduled-list semantics and WorkloadTrace::validate
//      (workload.cpp:53-91), and the step table is uploaded.
//
// nlohmann semantics kept: whitespace (space, \t, \n, \r); strings with every
// escape, \u surrogate pairs, UTF-8 validation and no raw control
// characters; number grammar; duplicate keys (the last wins); get<int> from
// integers (int64 / uint64 truncation), booleans and floats (truncation,
// INT_MIN out of range); "prompts": null; "lengths": null or an array
// (items() keys "0", "1", ...); "scheduled" absent (the lengths keys in map
// order).
// "prompts" given as an object (its values in key order, the last member
// of a repeated key). Rejected as RS_E_PARSE "unsupported" although nlohmann
// reads them: nesting deeper than 256, and floats converted to int that lie
// within 1e-6 below an integer (where the double rounding decides the result)
// or have a decimal exponent beyond +-60.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "rs_sort.cuh"
#include "rs_trace.cuh"

namespace rs {
size_t rank_strings_device_bytes(int64_t n, int64_t maxlen);
int rank_strings_device(rs_ctx* ctx, const char* d_bytes, const int64_t* d_off, int64_t n,
                        int64_t maxlen, uint32_t* d_perm);

namespace {

constexpr int kJErr = 1;     // a ParseError of the reference reader
constexpr int kJUnsup = 2;   // valid for nlohmann, not read here

// ------------------------------------------------------------ stage 1 ----
// 64-byte words: bitmasks of one character class, bit j = byte 64 w + j,
// four bytes at a time (SWAR byte compares packed to bits).
__device__ __forceinline__ uint32_t pk4(uint32_t m) {  // 0xff / 0x00 bytes -> 4 bits
  return (((m & 0x01010101u) * 0x01020408u) >> 24) & 0xfu;
}
__device__ __forceinline__ void word_masks(const unsigned char* t, int64_t w, int64_t n,
                                           uint64_t* bs, uint64_t* q, uint64_t* op, uint64_t* cl,
                                           uint64_t* cm, uint64_t* co) {
  const uint4* p = reinterpret_cast<const uint4*>(t + 64 * w);
  uint64_t mbs = 0, mq = 0, mop = 0, mcl = 0, mcm = 0, mco = 0;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const uint4 x = p[v];
    const uint32_t wd[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t y = wd[k];
      const int sh = 16 * v + 4 * k;
      mbs |= (uint64_t)pk4(__vcmpeq4(y, 0x5c5c5c5cu)) << sh;                                  // '\\'
      mq |= (uint64_t)pk4(__vcmpeq4(y, 0x22222222u)) << sh;                                   // '"'
      mop |= (uint64_t)pk4(__vcmpeq4(y, 0x7b7b7b7bu) | __vcmpeq4(y, 0x5b5b5b5bu)) << sh;      // '{' '['
      mcl |= (uint64_t)pk4(__vcmpeq4(y, 0x7d7d7d7du) | __vcmpeq4(y, 0x5d5d5d5du)) << sh;      // '}' ']'
      mcm |= (uint64_t)pk4(__vcmpeq4(y, 0x2c2c2c2cu)) << sh;                                  // ','
      mco |= (uint64_t)pk4(__vcmpeq4(y, 0x3a3a3a3au)) << sh;                                  // ':'
    }
  }
  const int64_t left = n - 64 * w;  // bytes of the word inside the text
  const uint64_t in = left >= 64 ? ~0ULL : (left <= 0 ? 0ULL : ((1ULL << left) - 1));
  *bs = mbs & in;
  *q = mq & in;
  *op = mop & in;
  *cl = mcl & in;
  *cm = mcm & in;
  *co = mco & in;
}

// Escaped characters of a word given the parity of the backslash run that
// ends right before it: a character is escaped iff an odd run precedes it.
// Runs are rare, so the loop walks runs, not bytes.
__device__ __forceinline__ uint64_t escaped_of(uint64_t bs, int carry) {
  if (bs == ~0ULL) return 0;  // a word of backslashes: its run goes on into the next word
  uint64_t esc = (carry && !(bs & 1ULL)) ? 1ULL : 0ULL;
  uint64_t m = bs;
  while (m) {
    const int s = __ffsll((long long)m) - 1;   // run start
    const int len = __ffsll((long long)~(m >> s)) - 1;
    const int e = s + len;                      // the character after the run
    if (e < 64 && ((len + (s == 0 ? carry : 0)) & 1)) esc |= 1ULL << e;
    m = e >= 64 ? 0ULL : m & (~0ULL << e);
  }
  return esc;
}

__device__ __forceinline__ uint64_t prefix_xor(uint64_t x) {
  x ^= x << 1;
  x ^= x << 2;
  x ^= x << 4;
  x ^= x << 8;
  x ^= x << 16;
  x ^= x << 32;
  return x;
}

// Word state: trailing backslash run parity, all-backslash flag.
__global__ void js_bs_kernel(const char* text, int64_t n, int64_t W, uint8_t* tail) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint64_t bs, q, op, cl, cm, co;
    word_masks(t, w, n, &bs, &q, &op, &cl, &cm, &co);
    const int lead = __clzll((long long)~bs);  // backslashes at the top of the word
    tail[w] = (uint8_t)((bs == ~0ULL ? 2 : 0) | (lead & 1));
  }
}

// The run parity before word w (words of 64 backslashes pass it through).
__device__ __forceinline__ int esc_carry(const uint8_t* tail, int64_t w) {
  int64_t v = w - 1;
  while (v >= 0 && (tail[v] & 2)) --v;
  return v >= 0 ? (tail[v] & 1) : 0;
}

// Unescaped quotes per word (their parity, for the in-string scan).
__global__ void js_quote_kernel(const char* text, int64_t n, int64_t W, const uint8_t* tail,
                                uint32_t* qpar) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint64_t bs, q, op, cl, cm, co;
    word_masks(t, w, n, &bs, &q, &op, &cl, &cm, &co);
    const uint64_t uq = q & ~escaped_of(bs, esc_carry(tail, w));
    qpar[w] = __popcll((long long)uq) & 1;
  }
}

// Structural characters outside strings; depth delta per word.
__device__ __forceinline__ void outside(const unsigned char* t, int64_t n, int64_t w, const uint8_t* tail,
                                        const uint32_t* qscan, uint64_t* op, uint64_t* cl, uint64_t* cm,
                                        uint64_t* co) {
  uint64_t bs, q;
  word_masks(t, w, n, &bs, &q, op, cl, cm, co);
  const uint64_t uq = q & ~escaped_of(bs, esc_carry(tail, w));
  uint64_t ins = prefix_xor(uq);  // 1 from an opening quote up to (not incl.) its closing one
  if (qscan[w] & 1) ins = ~ins;
  const uint64_t out = ~ins & ~uq;
  *op &= out;
  *cl &= out;
  *cm &= out;
  *co &= out;
}

// (ncl: the word's closers outside strings, so the token pass can skip a
// word that cannot come back to level 2 without reading it)
__global__ void js_depth_kernel(const char* text, int64_t n, int64_t W, const uint8_t* tail,
                                const uint32_t* qscan, unsigned long long* dd, uint8_t* ncl) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint64_t op, cl, cm, co;
    outside(t, n, w, tail, qscan, &op, &cl, &cm, &co);
    const int c = __popcll((long long)cl);
    dd[w] = (unsigned long long)(long long)(__popcll((long long)op) - c);
    ncl[w] = (uint8_t)c;
  }
}

// Tokens at level <= 1 (list A) and commas at level 2 (list B), counted per
// word; a word that holds any keeps them as two bit masks (ma / mb), which
// js_tokens_expand_kernel turns into the lists at the scanned offsets (the
// byte classes are computed once). Level: an opener's depth before it, a
// closer's depth after it, a comma's / colon's depth.
__global__ void js_tokens_kernel(const char* text, int64_t n, int64_t W, const uint8_t* tail,
                                 const uint32_t* qscan, const unsigned long long* dscan, const uint8_t* ncl,
                                 uint32_t* ca, uint32_t* cb, uint64_t* ma, uint64_t* mb) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    long long d = (long long)dscan[w];
    // no token of this word can come back to level 2 (the bulk of the text:
    // the insides of token arrays at depth 4): not read at all
    if (d - ncl[w] > 2) {
      ca[w] = cb[w] = 0;
      continue;
    }
    uint64_t op, cl, cm, co;
    outside(t, n, w, tail, qscan, &op, &cl, &cm, &co);
    uint64_t all = op | cl | cm | co;
    uint64_t a = 0, b = 0;
    while (all) {
      const int j = __ffsll((long long)all) - 1;
      all &= all - 1;
      const uint64_t bit = 1ULL << j;
      long long lev;
      if (op & bit) {
        lev = d;
        ++d;
      } else if (cl & bit) {
        --d;
        lev = d;
      } else {
        lev = d;
      }
      if (lev >= 0 && lev <= 1) a |= bit;
      else if (lev == 2 && (cm & bit)) b |= bit;
    }
    ca[w] = (uint32_t)__popcll((long long)a);
    cb[w] = (uint32_t)__popcll((long long)b);
    if (a | b) {
      ma[w] = a;
      mb[w] = b;
    }
  }
}

__global__ void js_tokens_expand_kernel(const char* text, int64_t W, const uint32_t* ca, const uint32_t* cb,
                                        const uint64_t* ma, const uint64_t* mb, const uint32_t* oa,
                                        const uint32_t* ob, uint64_t* la, int64_t* lb) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    if (!(ca[w] | cb[w])) continue;
    uint64_t a = ma[w], b = mb[w];
    uint32_t ia = oa[w], ib = ob[w];
    while (a) {
      const int64_t pos = 64 * w + __ffsll((long long)a) - 1;
      a &= a - 1;
      la[ia++] = ((uint64_t)pos << 8) | t[pos];
    }
    while (b) {
      lb[ib++] = 64 * w + __ffsll((long long)b) - 1;
      b &= b - 1;
    }
  }
}

// ------------------------------------------------------ JSON scanning ----
struct JIn {
  const unsigned char* t;
  int64_t p, e;
};

__device__ __forceinline__ bool jws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r';
}
__device__ __forceinline__ void skip_ws(JIn& in) {
  while (in.p < in.e && jws(in.t[in.p])) ++in.p;
}
__device__ __forceinline__ int hexv(unsigned char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

// A string at in.p (the opening quote): validated like nlohmann's lexer;
// *len = its unescaped bytes, written to out (nullable, out_cap bytes kept).
// Returns 0 or kJErr.
__device__ int jstring(JIn& in, char* out, int64_t out_cap, int64_t* len) {
  const unsigned char* t = in.t;
  int64_t p = in.p + 1, k = 0;
  auto put = [&](unsigned c) {
    if (out && k < out_cap) out[k] = (char)c;
    ++k;
  };
  for (;;) {
    if (p >= in.e) return kJErr;
    const unsigned c = t[p];
    if (c == '"') {
      ++p;
      break;
    }
    if (c < 0x20) return kJErr;
    if (c == '\\') {
      if (p + 1 >= in.e) return kJErr;
      const unsigned x = t[p + 1];
      p += 2;
      switch (x) {
        case '"': put('"'); break;
        case '\\': put('\\'); break;
        case '/': put('/'); break;
        case 'b': put('\b'); break;
        case 'f': put('\f'); break;
        case 'n': put('\n'); break;
        case 'r': put('\r'); break;
        case 't': put('\t'); break;
        case 'u': {
          auto hex4 = [&](int64_t at, unsigned* v) {
            if (at + 4 > in.e) return false;
            unsigned r = 0;
            for (int i = 0; i < 4; ++i) {
              const int h = hexv(t[at + i]);
              if (h < 0) return false;
              r = r * 16 + (unsigned)h;
            }
            *v = r;
            return true;
          };
          unsigned cp;
          if (!hex4(p, &cp)) return kJErr;
          p += 4;
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            unsigned lo;
            if (p + 2 > in.e || t[p] != '\\' || t[p + 1] != 'u' || !hex4(p + 2, &lo) ||
                lo < 0xDC00 || lo > 0xDFFF)
              return kJErr;
            p += 6;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            return kJErr;
          }
          if (cp < 0x80) {
            put(cp);
          } else if (cp < 0x800) {
            put(0xC0 | (cp >> 6));
            put(0x80 | (cp & 0x3F));
          } else if (cp < 0x10000) {
            put(0xE0 | (cp >> 12));
            put(0x80 | ((cp >> 6) & 0x3F));
            put(0x80 | (cp & 0x3F));
          } else {
            put(0xF0 | (cp >> 18));
            put(0x80 | ((cp >> 12) & 0x3F));
            put(0x80 | ((cp >> 6) & 0x3F));
            put(0x80 | (cp & 0x3F));
          }
          break;
        }
        default:
          return kJErr;
      }
      continue;
    }
    if (c < 0x80) {
      put(c);
      ++p;
      continue;
    }
    // UTF-8 (RFC 3629, as nlohmann's lexer checks it)
    int need;
    unsigned lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) need = 1;
    else if (c == 0xE0) { need = 2; lo = 0xA0; }
    else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) need = 2;
    else if (c == 0xED) { need = 2; hi = 0x9F; }
    else if (c == 0xF0) { need = 3; lo = 0x90; }
    else if (c >= 0xF1 && c <= 0xF3) need = 3;
    else if (c == 0xF4) { need = 3; hi = 0x8F; }
    else return kJErr;
    if (p + need >= in.e) return kJErr;
    put(c);
    for (int i = 1; i <= need; ++i) {
      const unsigned d = t[p + i];
      const unsigned l = i == 1 ? lo : 0x80, h = i == 1 ? hi : 0xBF;
      if (d < l || d > h) return kJErr;
      put(d);
    }
    p += need + 1;
  }
  in.p = p;
  *len = k;
  return 0;
}

// A number at in.p: the JSON grammar, and its value as nlohmann's get<int>
// gives it (*v). Returns 0, kJErr (grammar) or kJUnsup.
__device__ int jnumber(JIn& in, int32_t* v) {
  const unsigned char* t = in.t;
  int64_t p = in.p;
  const bool neg = p < in.e && t[p] == '-';
  if (neg) ++p;
  if (p >= in.e || t[p] < '0' || t[p] > '9') return kJErr;
  const int64_t i0 = p;
  if (t[p] == '0') ++p;
  else
    while (p < in.e && t[p] >= '0' && t[p] <= '9') ++p;
  const int64_t i1 = p;
  int64_t f0 = p, f1 = p;
  bool is_float = false;
  if (p < in.e && t[p] == '.') {
    ++p;
    f0 = p;
    if (p >= in.e || t[p] < '0' || t[p] > '9') return kJErr;
    while (p < in.e && t[p] >= '0' && t[p] <= '9') ++p;
    f1 = p;
    is_float = true;
  }
  long long ex = 0;
  if (p < in.e && (t[p] == 'e' || t[p] == 'E')) {
    ++p;
    bool eneg = false;
    if (p < in.e && (t[p] == '+' || t[p] == '-')) {
      eneg = t[p] == '-';
      ++p;
    }
    if (p >= in.e || t[p] < '0' || t[p] > '9') return kJErr;
    while (p < in.e && t[p] >= '0' && t[p] <= '9') {
      if (ex < 100000) ex = ex * 10 + (t[p] - '0');
      ++p;
    }
    if (eneg) ex = -ex;
    is_float = true;
  }
  in.p = p;
  if (!is_float) {
    unsigned long long m = 0;
    bool over = false;
    for (int64_t i = i0; i < i1; ++i) {
      const unsigned d = t[i] - '0';
      if (m > (0xFFFFFFFFFFFFFFFFULL - d) / 10) over = true;
      else m = m * 10 + d;
    }
    if (neg) {
      if (over || m > 0x8000000000000000ULL) *v = INT32_MIN;  // a float far out of range
      else *v = (int32_t)(long long)(0ULL - m);                // int64, narrowed
    } else {
      *v = over ? INT32_MIN : (int32_t)m;                       // int64 / uint64, narrowed
    }
    return 0;
  }
  // a float: the truncation of the nearest double. value = m * 10^e10 with
  // m the first 18 significant digits (sticky: a nonzero digit dropped)
  unsigned long long m = 0;
  int digits = 0;
  long long e10 = ex;
  bool sticky = false;
  auto digit = [&](unsigned d, bool frac) {
    if (m == 0 && d == 0) {
      if (frac) --e10;
      return;
    }
    if (digits < 18) {
      m = m * 10 + d;
      ++digits;
      if (frac) --e10;
    } else {
      sticky |= d != 0;
      if (!frac) ++e10;
    }
  };
  for (int64_t i = i0; i < i1; ++i) digit(t[i] - '0', false);
  for (int64_t i = f0; i < f1; ++i) digit(t[i] - '0', true);
  if (m == 0) {
    *v = 0;
    return 0;
  }
  if (e10 > 60 || e10 < -60) return kJUnsup;
  if (e10 >= 0) {  // an integer (sticky digits only below it): its range decides
    unsigned long long x = m;
    bool big = false;
    for (long long i = 0; i < e10 && !big; ++i) {
      if (x > 3000000000ULL) big = true;
      else x *= 10;
    }
    if (big || (neg ? x > 2147483648ULL : x >= 2147483648ULL)) *v = INT32_MIN;
    else *v = neg ? (int32_t)(0 - (long long)x) : (int32_t)x;
    return 0;
  }
  const long long k = -e10;
  if (k >= 19) {  // |value| < 0.1
    *v = 0;
    return 0;
  }
  unsigned long long pw = 1;
  for (long long i = 0; i < k; ++i) pw *= 10;
  const unsigned long long ip = m / pw, fr = m % pw;
  // within 1e-6 below the next integer the double rounding decides
  if ((double)(pw - fr) <= 1e-6 * (double)pw || (sticky && fr == pw - 1)) return kJUnsup;
  if (neg ? ip > 2147483648ULL : ip >= 2147483648ULL) *v = INT32_MIN;
  else *v = neg ? (int32_t)(0 - (long long)ip) : (int32_t)ip;
  return 0;
}

__device__ __forceinline__ bool jlit(JIn& in, const char* w, int n) {
  if (in.p + n > in.e) return false;
  for (int i = 0; i < n; ++i)
    if (in.t[in.p + i] != (unsigned char)w[i]) return false;
  in.p += n;
  return true;
}

// Any JSON value at in.p (after whitespace): validated, skipped. An explicit
// 256-level stack (bit = object).
__device__ int jskip(JIn& in) {
  uint64_t stk[4] = {0, 0, 0, 0};
  int depth = 0;
  enum { kValue, kAfter } st = kValue;
  for (;;) {
    skip_ws(in);
    if (st == kValue) {
      if (in.p >= in.e) return kJErr;
      const unsigned char c = in.t[in.p];
      if (c == '{' || c == '[') {
        if (depth >= 256) return kJUnsup;
        const bool obj = c == '{';
        if (obj) stk[depth >> 6] |= 1ULL << (depth & 63);
        else stk[depth >> 6] &= ~(1ULL << (depth & 63));
        ++depth;
        ++in.p;
        skip_ws(in);
        if (in.p < in.e && in.t[in.p] == (obj ? '}' : ']')) {
          ++in.p;
          --depth;
          st = kAfter;
          continue;
        }
        if (obj) {  // first key
          int64_t l;
          if (in.p >= in.e || in.t[in.p] != '"' || jstring(in, nullptr, 0, &l)) return kJErr;
          skip_ws(in);
          if (in.p >= in.e || in.t[in.p] != ':') return kJErr;
          ++in.p;
        }
        continue;  // a value
      }
      if (c == '"') {
        int64_t l;
        if (jstring(in, nullptr, 0, &l)) return kJErr;
      } else if (c == '-' || (c >= '0' && c <= '9')) {
        int32_t v;
        const int r = jnumber(in, &v);
        if (r == kJErr) return kJErr;  // a float outside the int conversion is still a number
      } else if (!(jlit(in, "true", 4) || jlit(in, "false", 5) || jlit(in, "null", 4))) {
        return kJErr;
      }
      st = kAfter;
      continue;
    }
    // after a value
    if (depth == 0) return 0;
    const bool obj = (stk[(depth - 1) >> 6] >> ((depth - 1) & 63)) & 1;
    if (in.p >= in.e) return kJErr;
    const unsigned char c = in.t[in.p];
    if (c == ',') {
      ++in.p;
      if (obj) {
        skip_ws(in);
        int64_t l;
        if (in.p >= in.e || in.t[in.p] != '"' || jstring(in, nullptr, 0, &l)) return kJErr;
        skip_ws(in);
        if (in.p >= in.e || in.t[in.p] != ':') return kJErr;
        ++in.p;
      }
      st = kValue;
    } else if (c == (obj ? '}' : ']')) {
      ++in.p;
      --depth;
    } else {
      return kJErr;
    }
  }
}

// get<int> of the value at in.p: numbers and booleans; kJErr for the rest.
__device__ int jint(JIn& in, int32_t* v) {
  skip_ws(in);
  if (in.p >= in.e) return kJErr;
  const unsigned char c = in.t[in.p];
  if (c == '-' || (c >= '0' && c <= '9')) return jnumber(in, v);
  if (jlit(in, "true", 4)) {
    *v = 1;
    return 0;
  }
  if (jlit(in, "false", 5)) {
    *v = 0;
    return 0;
  }
  return kJErr;  // a string / null / container: type_error (or a syntax error)
}

// get<std::vector<int>> of the value at in.p: count, and write when out.
__device__ int jint_array(JIn& in, int32_t* out, int64_t* count) {
  skip_ws(in);
  if (in.p >= in.e || in.t[in.p] != '[') return kJErr;
  ++in.p;
  int64_t k = 0;
  skip_ws(in);
  if (in.p < in.e && in.t[in.p] == ']') {
    ++in.p;
    *count = 0;
    return 0;
  }
  for (;;) {
    int32_t v;
    const int r = jint(in, &v);
    if (r) return r;
    if (out) out[k] = v;
    ++k;
    skip_ws(in);
    if (in.p >= in.e) return kJErr;
    if (in.t[in.p] == ',') {
      ++in.p;
      continue;
    }
    if (in.t[in.p] == ']') {
      ++in.p;
      break;
    }
    return kJErr;
  }
  *count = k;
  return 0;
}

// A key at in.p (the opening quote), matched against the schema's names:
// returns the index in names (or -1), after the ':' and its whitespace.
__device__ int jkey(JIn& in, const char* const* names, int nn, int* err) {
  char buf[24];
  int64_t len;
  if (in.p >= in.e || in.t[in.p] != '"' || jstring(in, buf, sizeof buf, &len)) {
    *err = kJErr;
    return -1;
  }
  skip_ws(in);
  if (in.p >= in.e || in.t[in.p] != ':') {
    *err = kJErr;
    return -1;
  }
  ++in.p;
  skip_ws(in);
  for (int i = 0; i < nn; ++i) {
    int l = 0;
    while (names[i][l]) ++l;
    if (l != len) continue;
    bool eq = true;
    for (int j = 0; j < l; ++j) eq &= buf[j] == names[i][j];
    if (eq) return i;
  }
  return -1;
}

// ------------------------------------------------------- stage 2: lines --
enum LineKind : int32_t { kLEmpty = 0, kLHeader, kLStep };
enum Role : int32_t { kRValidate = 0, kRPrompts, kRSched, kRLengths };

struct JLine {
  int32_t kind, err;
  int32_t g, mp, mr;  // header values
  int32_t step;       // step line: "step"
  int32_t has_sched;
  int32_t prompts_null;  // header: "prompts": null
  int32_t lengths_null;  // step: "lengths": null
};

struct JCont {
  int64_t open, close;  // the container's brackets
  int32_t line, role, is_obj, pad;
};

__device__ __forceinline__ int64_t lower_a(const uint64_t* a, int64_t n, int64_t pos) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)(a[mid] >> 8) < pos) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void js_first_line_kernel(const char* text, const int64_t* line_start, int64_t L, int64_t n,
                                     unsigned int* first) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < L;
       ln += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = line_start[ln], e = ln + 1 < L ? line_start[ln + 1] - 1 : n;
    bool any = false;
    for (int64_t i = s; i < e && !any; ++i) any = !(t[i] == ' ' || t[i] == '\t' || t[i] == '\r');
    if (any) atomicMin(first, (unsigned int)ln);
  }
}

// One thread per line: the top-level object, member containers jumped over
// (their closer: the next level-1 token). Containers go to a list (count
// via atomicAdd; cont_cap entries at most).
__global__ void js_line_kernel(const char* text, const int64_t* line_start, int64_t L, int64_t n,
                               const unsigned int* first, const uint64_t* la, int64_t na,
                               JLine* lines, JCont* conts, unsigned int* ncont, int64_t cont_cap) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < L;
       ln += (int64_t)gridDim.x * blockDim.x) {
    JLine out{};
    out.g = 0;
    out.mp = 1024;
    out.mr = 2048;
    int64_t s = line_start[ln], e = ln + 1 < L ? line_start[ln + 1] - 1 : n;
    while (s < e && (t[s] == ' ' || t[s] == '\t' || t[s] == '\r')) ++s;
    while (e > s && (t[e - 1] == ' ' || t[e - 1] == '\t' || t[e - 1] == '\r')) --e;
    if (s == e || ln < (int64_t)*first) {
      lines[ln] = out;
      continue;
    }
    const bool header = ln == (int64_t)*first;
    out.kind = header ? kLHeader : kLStep;
    JIn in{t, s, e};
    int err = 0;
    // members seen (last wins): type ok?, g, max_*, prompts / step, scheduled, lengths
    bool has_type = false, type_ok = false, has_g = false, has_prompts = false, has_step = false,
         has_lengths = false;
    int last_role_cont[4] = {-1, -1, -1, -1};  // container index per role (prompts / sched / lengths)
    auto demote = [&](int role) {  // an earlier container of a repeated key: validate only
      if (last_role_cont[role] >= 0) conts[last_role_cont[role]].role = kRValidate;
      last_role_cont[role] = -1;
    };
    auto add_cont = [&](int64_t open, int role) -> int64_t {  // jump to the matching closer
      const int64_t i = lower_a(la, na, open);
      if (i + 1 >= na || (int64_t)(la[i] >> 8) != open) return -1;
      const uint64_t c = la[i + 1];
      const unsigned char oc = t[open], cc = (unsigned char)(c & 0xff);
      if (!((oc == '{' && cc == '}') || (oc == '[' && cc == ']'))) return -1;
      const int64_t close = (int64_t)(c >> 8);
      const unsigned int k = atomicAdd(ncont, 1u);
      if ((int64_t)k < cont_cap) {
        JCont jc{open, close, (int32_t)ln, role, oc == '{' ? 1 : 0, 0};
        conts[k] = jc;
        if (role != kRValidate) last_role_cont[role] = (int)k;
      }
      return close + 1;
    };
    skip_ws(in);
    if (in.p >= in.e || t[in.p] != '{') {
      err = kJErr;  // contains("type") / at("step") need an object
    } else {
      ++in.p;
      skip_ws(in);
      bool first_m = true;
      while (!err) {
        if (in.p < in.e && t[in.p] == '}' && first_m) {
          ++in.p;
          break;
        }
        static const char* const kHdr[] = {"type", "g", "max_prompt_len", "max_response_len", "prompts"};
        static const char* const kStp[] = {"step", "scheduled", "lengths"};
        const int key = header ? jkey(in, kHdr, 5, &err) : jkey(in, kStp, 3, &err);
        if (err) break;
        const unsigned char c = in.p < in.e ? t[in.p] : 0;
        const bool cont = c == '{' || c == '[';
        int role = kRValidate;
        if (header && key == 4) role = kRPrompts;
        if (!header && key == 1) role = kRSched;
        if (!header && key == 2) role = kRLengths;
        if (role != kRValidate) demote(role);
        if (cont) {
          int r2 = role;
          if (role == kRSched && c == '{') r2 = -kJErr;       // get<vector<string>> of an object
          const int64_t np = add_cont(in.p, r2 < 0 ? kRValidate : r2);
          if (np < 0) {
            err = kJErr;
            break;
          }
          if (r2 < 0) err = -r2;
          in.p = np;
          if (header && key == 4) has_prompts = true;
          if (!header && key == 2) has_lengths = true;
          if (!header && key == 1) out.has_sched = 1;
          if (header && key == 0) type_ok = false, has_type = true;
          if ((header && (key == 1 || key == 2 || key == 3)) || (!header && key == 0)) err = kJErr;
        } else {
          // a scalar member
          if (header && key == 0) {
            has_type = true;
            type_ok = false;
            if (c == '"') {
              char buf[8];
              int64_t l;
              JIn tmp = in;
              if (jstring(tmp, buf, sizeof buf, &l)) err = kJErr;
              else type_ok = l == 6 && buf[0] == 'h' && buf[1] == 'e' && buf[2] == 'a' && buf[3] == 'd' &&
                             buf[4] == 'e' && buf[5] == 'r';
            }
            if (!err) err = jskip(in);
          } else if ((header && key >= 1 && key <= 3) || (!header && key == 0)) {
            int32_t v = 0;
            err = jint(in, &v);
            if (!err) {
              if (header && key == 1) {
                out.g = v;
                has_g = true;
              } else if (header && key == 2) {
                out.mp = v;
              } else if (header && key == 3) {
                out.mr = v;
              } else {
                out.step = v;
                has_step = true;
              }
            }
          } else if (role == kRPrompts || role == kRLengths || role == kRSched) {
            // null: no items / prompts; "scheduled": null is a type_error;
            // other scalars: a type_error on the first element
            if (jlit(in, "null", 4)) {
              if (role == kRSched) err = kJErr;
              if (role == kRPrompts) {
                has_prompts = true;
                out.prompts_null = 1;
              }
              if (role == kRLengths) {
                has_lengths = true;
                out.lengths_null = 1;
              }
            } else {
              err = jskip(in);
              if (!err) err = kJErr;
            }
          } else {
            err = jskip(in);
          }
        }
        if (err) break;
        skip_ws(in);
        first_m = false;
        if (in.p < in.e && t[in.p] == ',') {
          ++in.p;
          skip_ws(in);
          continue;
        }
        if (in.p < in.e && t[in.p] == '}') {
          ++in.p;
          break;
        }
        err = kJErr;
      }
      if (!err) {
        skip_ws(in);
        if (in.p != in.e) err = kJErr;  // trailing content
      }
      if (!err && header && !(has_type && type_ok)) err = kJErr;  // "first line must be the header object"
      if (!err && header && (!has_g || !has_prompts)) err = kJErr;  // at("g") / at("prompts")
      if (!err && !header && (!has_step || !has_lengths)) err = kJErr;  // at("step") / at("lengths")
    }
    if (header) out.prompts_null = out.prompts_null && last_role_cont[kRPrompts] < 0;
    else out.lengths_null = out.lengths_null && last_role_cont[kRLengths] < 0;
    out.err = err;
    lines[ln] = out;
  }
}

// ----------------------------------------------------- stage 3: children --
// Children of container ci: the spans between its level-2 commas.
__device__ __forceinline__ int64_t lower_b(const int64_t* b, int64_t n, int64_t pos) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (b[mid] < pos) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void js_child_count_kernel(const char* text, const JCont* conts, int64_t nc, const int64_t* lb,
                                      int64_t nb, unsigned long long* nchild) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
       c += (int64_t)gridDim.x * blockDim.x) {
    const JCont jc = conts[c];
    const int64_t b0 = lower_b(lb, nb, jc.open), b1 = lower_b(lb, nb, jc.close);
    int64_t k = b1 - b0 + 1;
    if (b1 == b0) {  // no separator: empty if only whitespace inside
      bool any = false;
      for (int64_t i = jc.open + 1; i < jc.close && !any; ++i) any = !jws(t[i]);
      if (!any) k = 0;
    }
    nchild[c] = (unsigned long long)k;
  }
}

struct JChild {   // pass-1 results of one child
  int64_t a, e;        // span
  int64_t id_len;      // prompt id / scheduled id / lengths key: unescaped bytes
  int64_t n_int;       // prompt tokens / length values
  int64_t id_at, ints_at;  // where the id string and the int array start (pass 2)
  int64_t key_at;      // "prompts" given as an object: the member's key
  int32_t key_len;     // its unescaped bytes
  int32_t serr;        // its schema error (counts only if no later member repeats the key)
  int32_t gt, err;
  int32_t cont, line;
};

// Every child but the prompt objects (js_prompt_kernel), a thread each.
// Pass 1 (write = false): validate, measure. Pass 2: write the ids and ints
// of the roles in wrole (a bit mask) at their scanned offsets.
template <bool kWrite>
__global__ void js_child_kernel(const char* text, const JCont* conts, const unsigned long long* cscan,
                                int64_t nc, const int64_t* lb, int64_t nb, int64_t total, JChild* ch,
                                const int64_t* id_off, const int64_t* int_off, char* ids, int32_t* ints,
                                unsigned int* first_err, int wrole) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    JChild r{};
    int64_t ci;
    if (kWrite) {
      r = ch[u];
      ci = r.cont;
      if (r.err || !((wrole >> conts[ci].role) & 1)) continue;  // another pass writes it
    } else {  // container of unit u, index inside it
      int64_t lo = 0, hi = nc;  // last container with cscan <= u
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)cscan[mid] <= u) lo = mid;
        else hi = mid;
      }
      ci = lo;
      while (ci + 1 < nc && (int64_t)cscan[ci + 1] <= u) ++ci;
      const JCont jc = conts[ci];
      const int64_t idx = u - (int64_t)cscan[ci];
      const int64_t b0 = lower_b(lb, nb, jc.open), b1 = lower_b(lb, nb, jc.close);
      r.a = idx == 0 ? jc.open + 1 : lb[b0 + idx - 1] + 1;
      r.e = b0 + idx < b1 ? lb[b0 + idx] : jc.close;
      r.cont = (int32_t)ci;
      r.line = jc.line;
    }
    const JCont jc = conts[ci];
    if (jc.role == kRPrompts) continue;  // js_prompt_kernel: a warp per prompt object
    JIn in{t, r.a, r.e};
    int err = 0;
    skip_ws(in);
    if (jc.is_obj) {  // a member: "key": value
      if (jc.role == kRLengths) {
        if (in.p >= in.e || t[in.p] != '"') err = kJErr;
        else {
          r.id_at = in.p;
          int64_t l;
          err = jstring(in, kWrite ? ids + id_off[u] : nullptr, kWrite ? r.id_len : 0, &l);
          r.id_len = l;
        }
        if (!err) {
          skip_ws(in);
          if (in.p >= in.e || t[in.p] != ':') err = kJErr;
          else ++in.p;
        }
        if (!err) {
          skip_ws(in);
          r.ints_at = in.p;
          int64_t k;
          err = jint_array(in, kWrite ? ints + int_off[u] : nullptr, &k);
          r.n_int = k;
        }
      } else {
        int64_t l;
        if (in.p >= in.e || t[in.p] != '"' || jstring(in, nullptr, 0, &l)) err = kJErr;
        if (!err) {
          skip_ws(in);
          if (in.p >= in.e || t[in.p] != ':') err = kJErr;
          else ++in.p;
        }
        if (!err) err = jskip(in);
      }
    } else if (jc.role == kRLengths) {  // "lengths" as an array: items() keys "0", "1", ...
      r.id_len = 0;                      // (the host names them)
      r.ints_at = in.p;
      int64_t k;
      err = jint_array(in, kWrite ? ints + int_off[u] : nullptr, &k);
      r.n_int = k;
    } else if (jc.role == kRSched) {
      if (in.p >= in.e || t[in.p] != '"') {
        err = jskip(in);  // get<std::string> of a non-string: type_error
        if (!err) err = kJErr;
      } else {
        r.id_at = in.p;
        int64_t l;
        err = jstring(in, kWrite ? ids + id_off[u] : nullptr, kWrite ? r.id_len : 0, &l);
        r.id_len = l;
      }
    } else {
      err = jskip(in);
    }
    if (!err) {
      skip_ws(in);
      if (in.p != in.e) err = kJErr;
    }
    if (!kWrite) {
      r.err = err;
      ch[u] = r;
      if (err) atomicMin(first_err, ((unsigned int)r.line << 1) | (err == kJUnsup ? 1u : 0u));
    }
  }
}

// ------------------------------------------- warp-cooperative prompts --
// An int array of plain integers at p (just after its '['), 16 bytes per
// lane, 512 per step: byte classes as masks, every item checked against the
// previous non-blank one (a number after ',' or the '[', a ',' after a
// number, the ']' after a number or the '['), no '-' except at a number's
// start, no leading zero, at most 18 digits. Counts (out == nullptr) or
// writes the first cap values. Returns 0 (with *count and *end, the position after
// the ']') or 1 when the array is not of that form — a float, a boolean, a
// longer number, or a syntax error: the caller's serial path then decides.
__device__ int warp_int_array(const unsigned char* t, int64_t p, int64_t e, int32_t* out, int64_t cap,
                              int64_t* count, int64_t* end) {
  const int lane = threadIdx.x & 31;
  enum : int { kNone = 0, kStart = 1, kNum = 2, kComma = 3 };  // class of the last non-blank byte
  int carry = kStart;    // the '['
  uint32_t prevX = 0, prevM = 0;  // the byte before the step: part of a number / a '-'
  int64_t k = 0;
  for (int64_t b0 = p & ~(int64_t)15;; b0 += 512) {
    if (b0 >= e) return 1;  // no ']' before the end of the span
    const int64_t i = b0 + 16 * lane;
    uint32_t D = 0, M = 0, Z = 0, C = 0, W = 0, E = 0, O = 0;
    {
      const uint4 v = *reinterpret_cast<const uint4*>(t + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t x = w[q];
        const uint32_t dg = __vcmpgeu4(x, 0x30303030u) & __vcmpleu4(x, 0x39393939u);
        const uint32_t mi = __vcmpeq4(x, 0x2d2d2d2du), ze = __vcmpeq4(x, 0x30303030u);
        const uint32_t cm = __vcmpeq4(x, 0x2c2c2c2cu), cl = __vcmpeq4(x, 0x5d5d5d5du);
        const uint32_t ws = __vcmpeq4(x, 0x20202020u) | __vcmpeq4(x, 0x09090909u) |
                            __vcmpeq4(x, 0x0a0a0a0au) | __vcmpeq4(x, 0x0d0d0d0du);
        D |= pk4(dg) << (4 * q);
        M |= pk4(mi) << (4 * q);
        Z |= pk4(ze) << (4 * q);
        C |= pk4(cm) << (4 * q);
        E |= pk4(cl) << (4 * q);
        W |= pk4(ws) << (4 * q);
      }
      uint32_t valid = 0xffffu;
      if (i < p) valid &= p - i >= 16 ? 0u : 0xffffu << (int)(p - i);
      if (i + 16 > e) valid &= e > i ? 0xffffu >> (int)(16 - (e - i)) : 0u;
      D &= valid;
      M &= valid;
      Z &= valid;
      C &= valid;
      E &= valid;
      W = (W & valid) | (~valid & 0xffffu & (i < p ? (p - i >= 16 ? 0xffffu : ((1u << (p - i)) - 1)) : 0u));
      O = ~(D | M | C | E | W) & 0xffffu;  // bytes past e count as other
    }
    // the array ends at the first ']': later bytes do not matter
    const unsigned eb = __ballot_sync(0xffffffffu, E != 0);
    int close_lane = eb ? __ffs(eb) - 1 : 32;
    if (lane > close_lane) D = M = Z = C = E = O = 0, W = 0xffffu;
    if (lane == close_lane) {
      const int j = __ffs(E) - 1;
      const uint32_t keep = (2u << j) - 1;  // up to and with the ']'
      D &= keep;
      M &= keep;
      Z &= keep;
      C &= keep;
      E &= keep;
      O &= keep;
      W = (W & keep) | (~keep & 0xffffu);
    }
    const uint32_t X = D | M;
    const uint32_t up = __shfl_up_sync(0xffffffffu, X >> 15, 1);
    const uint32_t S = X & ~((X << 1) | (lane == 0 ? prevX : up)) & 0xffffu;
    const uint32_t dn = __shfl_down_sync(0xffffffffu, D & 1u, 1);
    const uint32_t d_after = i + 16 < e && t[i + 16] >= '0' && t[i + 16] <= '9' ? 1u : 0u;
    const uint32_t Dn = ((D >> 1) | ((lane == 31 ? d_after : dn) << 15)) & 0xffffu;  // next byte a digit
    const uint32_t mup = __shfl_up_sync(0xffffffffu, M >> 15, 1);
    const uint32_t Mp = ((M << 1) & 0xffffu) | (lane == 0 ? prevM : mup);
    bool bad = O != 0;
    bad |= (M & ~S) != 0;                // '-' inside a number
    bad |= (M & ~Dn) != 0;               // '-' not followed by a digit
    bad |= (Z & (S | Mp) & Dn) != 0;     // leading zero
    // the class of the last non-blank byte before each lane (a "last
    // non-none" scan over the lanes, from the previous step's carry)
    const uint32_t NW = ~W & 0xffffu;
    int last = kNone;
    if (NW) {
      const int j = 31 - __clz(NW);
      last = ((C >> j) & 1) ? kComma : (((E >> j) & 1) ? kNone : kNum);
    }
    int before = last;  // inclusive scan of "the last defined" across the lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, before, d);
      if (lane >= d && before == kNone) before = o;
    }
    // exclusive: the lane before's inclusive value (or the carry)
    int prev = __shfl_up_sync(0xffffffffu, before, 1);
    if (lane == 0) prev = kNone;
    if (prev == kNone) prev = carry;
    // walk this lane's items: starts, commas, the ']'
    uint32_t items = S | C | E;
    int pc = prev;
    uint32_t nw = NW;
    while (items && !bad) {
      const int j = __ffs(items) - 1;
      items &= items - 1;
      // the last non-blank byte below j in this lane, else the carried class
      const uint32_t below = nw & ((1u << j) - 1);
      int cls = pc;
      if (below) {
        const int jb = 31 - __clz(below);
        cls = ((C >> jb) & 1) ? kComma : kNum;
      }
      if ((S >> j) & 1) bad |= !(cls == kComma || cls == kStart);
      else if ((C >> j) & 1) bad |= cls != kNum;
      else bad |= !(cls == kNum || cls == kStart);
    }
    // numbers: each lane parses the ones starting in its bytes. The digit
    // run's length comes from the digit masks (this lane's and the next
    // one's); up to 8 digits are read as one 8-byte window (three aligned
    // words) and converted by SWAR multiply-adds, longer or unbounded runs
    // (past the next lane, or past the step) byte by byte.
    const int ns = __popc(S);
    const int before_n = warp_incl_sum(ns) - ns;
    const uint32_t Dnx = __shfl_down_sync(0xffffffffu, D, 1);
    if (!bad && ns) {
      const uint32_t Dx = D | ((lane == 31 ? d_after : Dnx) << 16);
      const int wend = lane == 31 ? 17 : 32;  // bits of Dx the masks cover
      uint32_t m = S;
      int idx = 0;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const int neg = (M >> j) & 1;
        const int p0 = j + neg;
        int nd = __ffs(~(Dx >> p0)) - 1;  // -1: the run fills the window
        unsigned long long v = 0;
        if (nd >= 1 && nd <= 8 && p0 + nd < wend) {
          const int64_t a = i + p0;
          const uint32_t* wp = reinterpret_cast<const uint32_t*>(t + (a & ~(int64_t)3));
          const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2];
          const int sh = (int)(a & 3) * 8;
          unsigned long long x = ((unsigned long long)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh);
          const int pad = 8 - nd;  // leading '0' bytes: the digits end at byte 7
          if (pad) x = (x << (8 * pad)) | (0x3030303030303030ULL >> (8 * nd));
          x = ((x & 0x0F0F0F0F0F0F0F0FULL) * 2561ULL) >> 8;
          x = ((x & 0x00FF00FF00FF00FFULL) * 6553601ULL) >> 16;
          v = ((x & 0x0000FFFF0000FFFFULL) * 42949672960001ULL) >> 32;
        } else {
          int64_t q = i + p0;
          nd = 0;
          for (; q < e && t[q] >= '0' && t[q] <= '9'; ++q, ++nd) v = v * 10u + (unsigned)(t[q] - '0');
        }
        if (nd > 18) bad = true;
        if (out && !bad && k + before_n + idx < cap) out[k + before_n + idx] = (int32_t)(neg ? 0ULL - v : v);
        ++idx;
      }
    }
    if (__any_sync(0xffffffffu, bad)) return 1;
    k += __shfl_sync(0xffffffffu, before_n + ns, 31);
    // the carry: the class of the last non-blank byte of this step
    const int lastcls = __shfl_sync(0xffffffffu, before, 31);
    if (lastcls != kNone) carry = lastcls;
    prevX = __shfl_sync(0xffffffffu, (X >> 15) & 1u, 31);
    prevM = __shfl_sync(0xffffffffu, (M >> 15) & 1u, 31);
    if (close_lane < 32) {
      const uint32_t ej = (uint32_t)__shfl_sync(0xffffffffu, (uint32_t)(__ffs(E) - 1), close_lane);
      *count = k;
      *end = b0 + 16 * close_lane + ej + 1;
      return 0;
    }
  }
}

// The count-only form of warp_int_array for the first pass: the array ends at
// its first ']', holds (commas + 1) items, or none when only blanks precede
// the ']'. Values and the grammar are not checked here — pass 2 reads the
// same bytes with warp_int_array and reports what it rejects. Returns 1 (the
// caller's serial path decides) when a '[', '{' or '"' comes before the ']'
// or there is no ']' before e: there the first ']' need not be the array's.
// 0x80 in every byte of x equal to the matching byte of c (exact per byte)
__device__ __forceinline__ uint32_t byte_eq(uint32_t x, uint32_t c) {
  const uint32_t y = x ^ c;
  return ~(((y & 0x7f7f7f7fu) + 0x7f7f7f7fu) | y | 0x7f7f7f7fu);
}

__device__ int warp_count_array(const unsigned char* t, int64_t p, int64_t e, int64_t* count, int64_t* end) {
  const int lane = threadIdx.x & 31;
  int64_t commas = 0;
  bool nonblank = false;
  for (int64_t b0 = p & ~(int64_t)15;; b0 += 512) {
    if (b0 >= e) return 1;
    const int64_t i = b0 + 16 * lane;
    if (b0 >= p && b0 + 512 <= e) {
      // a whole step inside the span: byte flags (the high bit of each
      // matching byte), no bit packing; a step holding the ']' is redone
      // below with positions
      const uint4 v = *reinterpret_cast<const uint4*>(t + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t fe = 0, fq = 0, fnb = 0;
      int nc = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t x = w[q];
        fe |= byte_eq(x, 0x5d5d5d5du);
        fq |= byte_eq(x, 0x5b5b5b5bu) | byte_eq(x, 0x7b7b7b7bu) | byte_eq(x, 0x22222222u);
        nc += __popc(byte_eq(x, 0x2c2c2c2cu));
        fnb |= __vcmpgtu4(x, 0x20202020u);  // above ' ': not blank (blank bytes are <= ' ')
      }
      if (!__any_sync(0xffffffffu, fe != 0)) {
        if (__any_sync(0xffffffffu, fq != 0)) return 1;
        commas += __reduce_add_sync(0xffffffffu, (unsigned)nc);
        nonblank |= __any_sync(0xffffffffu, fnb != 0);
        continue;
      }
    }
    uint32_t C = 0, E = 0, W = 0, Q = 0;
    {
      const uint4 v = *reinterpret_cast<const uint4*>(t + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t x = w[q];
        const uint32_t ws = __vcmpeq4(x, 0x20202020u) | __vcmpeq4(x, 0x09090909u) |
                            __vcmpeq4(x, 0x0a0a0a0au) | __vcmpeq4(x, 0x0d0d0d0du);
        const uint32_t nest = __vcmpeq4(x, 0x5b5b5b5bu) | __vcmpeq4(x, 0x7b7b7b7bu) | __vcmpeq4(x, 0x22222222u);
        C |= pk4(__vcmpeq4(x, 0x2c2c2c2cu)) << (4 * q);
        E |= pk4(__vcmpeq4(x, 0x5d5d5d5du)) << (4 * q);
        W |= pk4(ws) << (4 * q);
        Q |= pk4(nest) << (4 * q);
      }
      uint32_t valid = 0xffffu;
      if (i < p) valid &= p - i >= 16 ? 0u : 0xffffu << (int)(p - i);
      if (i + 16 > e) valid &= e > i ? 0xffffu >> (int)(16 - (e - i)) : 0u;
      C &= valid;
      E &= valid;
      Q &= valid;
      W = ~W & valid;  // from here: the non-blank bytes
    }
    const unsigned eb = __ballot_sync(0xffffffffu, E != 0);
    const int close_lane = eb ? __ffs(eb) - 1 : 32;
    uint32_t keep = lane < close_lane ? 0xffffu : 0u;  // the bytes before the ']'
    if (lane == close_lane) keep = (1u << (__ffs(E) - 1)) - 1;
    if (__any_sync(0xffffffffu, (Q & keep) != 0)) return 1;
    commas += __reduce_add_sync(0xffffffffu, (unsigned)__popc(C & keep));
    nonblank |= __any_sync(0xffffffffu, (W & keep) != 0);
    if (close_lane < 32) {
      const uint32_t ej = (uint32_t)__shfl_sync(0xffffffffu, (uint32_t)(__ffs(E) - 1), close_lane);
      *count = nonblank ? commas + 1 : 0;
      *end = b0 + 16 * close_lane + ej + 1;
      return 0;
    }
  }
}

// One warp per prompt object (the children [c0, c0 + P) of the prompts
// container): lane 0 reads the members, the warp reads "token_ids" (serial
// fallback on lane 0 for arrays outside the fast form). kMode 0 (pass 1)
// records the child like js_child_kernel, sizing "token_ids" by its commas
// (warp_count_array); kMode 2 (pass 2) writes the id and the tokens,
// checking the arrays as it goes, and kMode 1 only checks them — the error
// path's pass, so a bad array is reported before an error on a later line.
// Modes 1 and 2 report through first_err like pass 1.
template <int kMode>
__global__ void __launch_bounds__(128, 8) js_prompt_kernel(const char* text, const JCont* conts, const unsigned long long* cscan,
                                 int64_t c0, int64_t P, const int64_t* lb, int64_t nb, int64_t pc,
                                 JChild* ch, const int64_t* id_off, const int64_t* int_off, char* ids,
                                 int32_t* ints, unsigned int* first_err) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  const int lane = threadIdx.x & 31;
  for (int64_t pi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; pi < P;
       pi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t u = c0 + pi;
    JChild r{};
    const JCont jc = conts[pc];
    if (kMode != 0) {
      r = ch[u];
      if (r.err) continue;
      if (kMode == 2 && lane == 0) {
        JIn is{t, r.id_at, r.e};
        int64_t l;
        jstring(is, ids + id_off[u], r.id_len, &l);
      }
      int32_t* out = kMode == 2 ? ints + int_off[u] : nullptr;
      int64_t cnt = 0, endp;
      const int st = warp_int_array(t, r.ints_at + 1, r.e, out, r.n_int, &cnt, &endp);
      if (lane == 0) {
        int err = 0;
        if (st) {  // pass 1's count bounds the writes: items <= commas + 1
          JIn it{t, r.ints_at, r.e};
          err = jint_array(it, out, &cnt);
        }
        if (!err && cnt != r.n_int) err = kJErr;
        if (err) atomicMin(first_err, ((unsigned int)r.line << 1) | (err == kJUnsup ? 1u : 0u));
      }
      continue;
    }
    const int64_t b0 = lower_b(lb, nb, jc.open), b1 = lower_b(lb, nb, jc.close);
    r.a = pi == 0 ? jc.open + 1 : lb[b0 + pi - 1] + 1;
    r.e = b0 + pi < b1 ? lb[b0 + pi] : jc.close;
    r.cont = (int32_t)pc;
    r.line = jc.line;
    // lane 0 walks the members; at "token_ids" the warp reads the array
    JIn in{t, r.a, r.e};
    int err = 0, syn = 0;
    int64_t val_end = -1;  // object members: where the value ends (syntax checked first)
    bool has_id = false, has_gt = false, has_tok = false, open_ok = false;
    if (lane == 0 && jc.is_obj) {
      // "key": value — the key kept for the duplicate rule, the value's JSON
      // checked on its own: a syntax error always counts, a schema error only
      // for the last member with this key (nlohmann keeps the last one)
      skip_ws(in);
      int64_t kl = 0;
      if (in.p >= in.e || t[in.p] != '"') syn = kJErr;
      else {
        r.key_at = in.p;
        syn = jstring(in, nullptr, 0, &kl);
        r.key_len = (int32_t)kl;
      }
      if (!syn) {
        skip_ws(in);
        if (in.p >= in.e || t[in.p] != ':') syn = kJErr;
        else ++in.p;
      }
      if (!syn) {
        skip_ws(in);
        JIn v = in;
        syn = jskip(v);
        if (!syn) {
          skip_ws(v);
          if (v.p != v.e) syn = kJErr;
          val_end = v.p;
        }
      }
      if (syn) in.p = in.e;  // nothing more to read
    }
    syn = __shfl_sync(0xffffffffu, syn, 0);
    if (lane == 0 && !syn) {
      skip_ws(in);
      if (in.p >= in.e || t[in.p] != '{') {
        err = jskip(in);
        if (!err) err = kJErr;
      } else {
        ++in.p;
        skip_ws(in);
        open_ok = true;
      }
    }
    bool done = syn || !__shfl_sync(0xffffffffu, open_ok, 0);
    bool first_m = true;
    while (!done) {
      int key = -1, want_arr = 0;
      int64_t arr_at = 0;
      if (lane == 0) {
        if (first_m && in.p < in.e && t[in.p] == '}') {
          ++in.p;
          done = true;
        } else {
          static const char* const kP[] = {"id", "ground_truth_len", "token_ids"};
          key = jkey(in, kP, 3, &err);
          if (err) {
            done = true;
          } else if (key == 0) {
            if (in.p >= in.e || t[in.p] != '"') {
              err = jskip(in);
              if (!err) err = kJErr;
            } else {
              r.id_at = in.p;
              err = jstring(in, nullptr, 0, &r.id_len);
              has_id = true;
            }
          } else if (key == 1) {
            err = jint(in, &r.gt);
            has_gt = true;
          } else if (key == 2) {
            r.ints_at = in.p;
            has_tok = true;
            if (in.p < in.e && t[in.p] == '[') {
              want_arr = 1;
              arr_at = in.p;
            } else {
              err = jskip(in);
              if (!err) err = kJErr;
            }
          } else {
            err = jskip(in);
          }
        }
      }
      want_arr = __shfl_sync(0xffffffffu, want_arr, 0);
      if (want_arr) {
        arr_at = __shfl_sync(0xffffffffu, arr_at, 0);
        int64_t cnt = 0, endp = 0;
        const int st = warp_count_array(t, arr_at + 1, r.e, &cnt, &endp);
        if (lane == 0) {
          if (st) {
            JIn it{t, arr_at, in.e};
            err = jint_array(it, nullptr, &cnt);
            endp = it.p;
          }
          r.n_int = cnt;
          in.p = endp;
        }
      }
      if (lane == 0 && !done) {
        if (err) {
          done = true;
        } else {
          skip_ws(in);
          if (in.p < in.e && t[in.p] == ',') {
            ++in.p;
            skip_ws(in);
          } else if (in.p < in.e && t[in.p] == '}') {
            ++in.p;
            done = true;
          } else {
            err = kJErr;
            done = true;
          }
        }
      }
      first_m = false;
      done = __shfl_sync(0xffffffffu, done, 0);
    }
    if (lane == 0) {
      if (!err && open_ok && !(has_id && has_gt && has_tok)) err = kJErr;
      if (!err && !jc.is_obj) {
        skip_ws(in);
        if (in.p != in.e) err = kJErr;
      }
      if (jc.is_obj) {  // the schema error waits for the duplicate rule
        r.serr = syn ? 0 : err;
        err = syn;
        (void)val_end;
      }
      r.err = err;
      ch[u] = r;
      if (err) atomicMin(first_err, ((unsigned int)r.line << 1) | (err == kJUnsup ? 1u : 0u));
    }
  }
}

// "prompts" given as an object: the members' keys written out (for the
// string ranking), then the duplicate rule — of the members sharing a key,
// the last one is the prompt; the others are dropped (err = -1, after their
// schema errors are ignored) and the survivors' schema errors reported.
__global__ void js_key_write_kernel(const char* text, const JChild* ch, int64_t c0, int64_t n,
                                    const int64_t* koff, char* keys) {
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const JChild r = ch[c0 + i];
    if (r.err) continue;
    JIn in{t, r.key_at, r.e};
    int64_t l;
    jstring(in, keys + koff[i], r.key_len, &l);
  }
}

__global__ void js_key_sizes_kernel(const JChild* ch, int64_t c0, int64_t n, unsigned long long* kl) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    kl[i] = ch[c0 + i].err ? 0ULL : (unsigned long long)ch[c0 + i].key_len;
}

__global__ void js_key_dedup_kernel(JChild* ch, int64_t c0, int64_t n, const uint32_t* perm,
                                    const char* keys, const int64_t* koff, unsigned int* first_err,
                                    uint32_t* kept) {
  auto same = [&](uint32_t x, uint32_t y) {
    const int64_t lx = koff[x + 1] - koff[x], ly = koff[y + 1] - koff[y];
    if (lx != ly) return false;
    for (int64_t j = 0; j < lx; ++j)
      if (keys[koff[x] + j] != keys[koff[y] + j]) return false;
    return true;
  };
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = perm[r];
    JChild& c = ch[c0 + i];
    if (c.err) {  // a syntax error: already reported
      kept[i] = 0;
      continue;
    }
    bool last = true;  // no later member (higher index) with the same key
    for (int64_t q = r - 1; q >= 0 && same(perm[q], i); --q) last &= perm[q] < i || ch[c0 + perm[q]].err;
    for (int64_t q = r + 1; q < n && same(perm[q], i); ++q) last &= perm[q] < i || ch[c0 + perm[q]].err;
    kept[i] = last ? 1u : 0u;
    if (!last) {
      c.err = -1;  // dropped: no prompt, no error
    } else if (c.serr) {
      c.err = c.serr;
      atomicMin(first_err, ((unsigned int)c.line << 1) | (c.serr == kJUnsup ? 1u : 0u));
    }
  }
}

// Children with no error keep their pass-1 sizes; others count 0.
__global__ void js_sizes_kernel(const JChild* ch, const JCont* conts, int64_t total, int rmask,
                                unsigned long long* idl, unsigned long long* nint) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const JChild r = ch[u];
    const bool mine = !r.err && ((rmask >> conts[r.cont].role) & 1);
    idl[u] = mine ? (unsigned long long)r.id_len : 0ULL;
    nint[u] = mine ? (unsigned long long)r.n_int : 0ULL;
  }
}

// Each scheduled id / lengths key of one role: its index in the id-sorted
// prompt table (binary search, std::string order), -1 when absent.
__global__ void js_lookup_kernel(const JChild* ch, const JCont* conts, int64_t total, int rmask,
                                 const int64_t* id_off, const char* ids, const char* sids,
                                 const int64_t* sid_off, int32_t P, int32_t* pidx) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const JChild r = ch[u];
    if (r.err || !((rmask >> conts[r.cont].role) & 1)) continue;
    const unsigned char* a = reinterpret_cast<const unsigned char*>(ids + id_off[u]);
    const int64_t la = r.id_len;
    int32_t lo = 0, hi = P, found = -1;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      const unsigned char* b = reinterpret_cast<const unsigned char*>(sids + sid_off[mid]);
      const int64_t lb = sid_off[mid + 1] - sid_off[mid];
      int c = 0;
      for (int64_t i = 0; i < (la < lb ? la : lb) && !c; ++i) c = a[i] < b[i] ? -1 : (a[i] > b[i] ? 1 : 0);
      if (!c) c = la < lb ? -1 : (la > lb ? 1 : 0);
      if (!c) {
        found = mid;
        break;
      }
      if (c < 0) hi = mid;
      else lo = mid + 1;
    }
    pidx[u] = found;
  }
}

// ------------------------------------------------ steps on the device --
// The step table without the host (WorkloadTrace::validate's step rules,
// workload.cpp:53-91, over the reader's containers, :304-349): every step
// line's "lengths" children and "scheduled" children become sort keys
// (step line << 32 | prompt table index). Sorted (stable), the last lengths
// child of each key is the one std::map keeps; the distinct keys of a line
// are its lengths map in key order (= id order = table order). A valid step
// has a scheduled list without repeats equal to that key set, g lengths per
// key, each in [1, max_response_len]. Any deviation sets *bad and the host
// path (which reproduces the reference's first error) runs instead.
struct JStepLine {   // per step line, device copy
  int32_t e_off;     // its first entry in the step table
  int32_t sk_start;  // its first scheduled key in the sorted scheduled keys (-1: no "scheduled")
  int32_t dk_start;  // its first distinct lengths key
  int32_t pad;
};

__global__ void js_step_keys_kernel(const JChild* ch, const JCont* conts, const unsigned long long* cscan,
                                    int64_t n, const int64_t* cbase, const int32_t* cstep, const int32_t* pidx,
                                    uint64_t* lk, uint32_t* lv, uint64_t* sk, uint32_t* sv, int* bad) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int c = ch[u].cont;
    const int64_t b = cbase[c];
    if (b < 0) continue;  // not the last "lengths" / "scheduled" of a step line
    const int64_t i = b + (u - (int64_t)cscan[c]);
    const int32_t p = pidx[u];
    if (p < 0) atomicOr(bad, 1);  // an id outside the prompt table
    const uint64_t key = ((uint64_t)cstep[c] << 32) | (uint32_t)max(p, 0);
    if (conts[c].role == kRLengths) {
      lk[i] = key;
      lv[i] = (uint32_t)u;
    } else {
      sk[i] = key;
      sv[i] = (uint32_t)(u - (int64_t)cscan[c]);
    }
  }
}

// flag the last child of each (line, key) run of the sorted lengths keys
__global__ void js_step_ends_kernel(const uint64_t* k, int64_t n, uint32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == n - 1 || k[i + 1] != k[i]) ? 1u : 0u;
}

__global__ void js_step_distinct_kernel(const uint64_t* k, const uint32_t* v, const uint32_t* flag,
                                        const uint32_t* pos, int64_t n, uint64_t* dk, uint32_t* dw,
                                        int32_t* dcnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    dk[pos[i]] = k[i];
    dw[pos[i]] = v[i];
    atomicAdd(&dcnt[k[i] >> 32], 1);
  }
}

// scheduled lines: no repeats, the same sorted keys as the line's lengths,
// entries in batch order; lines without "scheduled": the keys in map order
__global__ void js_step_entries_kernel(const uint64_t* sk, const uint32_t* sv, int64_t nsk, const uint64_t* dk,
                                       const uint32_t* dw, int64_t nd, const JStepLine* sl, int32_t* e_prompt,
                                       uint32_t* e_win, int* bad) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nsk + nd;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (j < nsk) {
      const int s = (int)(sk[j] >> 32);
      const JStepLine L = sl[s];
      if (j > 0 && sk[j - 1] == sk[j]) atomicOr(bad, 2);  // scheduled twice
      const int64_t d = L.dk_start + (j - L.sk_start);
      if (dk[d] != sk[j]) atomicOr(bad, 4);  // lengths and scheduled differ
      const int64_t e = L.e_off + sv[j];
      e_prompt[e] = (int32_t)(sk[j] & 0xffffffffu);
      e_win[e] = dw[d];
    } else {
      const int64_t d = j - nsk;
      const int s = (int)(dk[d] >> 32);
      const JStepLine L = sl[s];
      if (L.sk_start >= 0) continue;
      const int64_t e = L.e_off + (d - L.dk_start);
      e_prompt[e] = (int32_t)(dk[d] & 0xffffffffu);
      e_win[e] = dw[d];
    }
  }
}

__global__ void js_step_lengths_kernel(const uint32_t* e_win, int64_t ne, const unsigned long long* nint,
                                       const unsigned long long* int_off, const int32_t* vals, int G, int max_r,
                                       int32_t* lengths, int* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = e_win[e];
    if ((int64_t)nint[u] != G) {
      atomicOr(bad, 8);
      continue;
    }
    const int32_t* src = vals + int_off[u];
    for (int i = 0; i < G; ++i) {
      const int32_t l = src[i];
      if (l < 1 || l > max_r) atomicOr(bad, 16);
      lengths[e * G + i] = l;
    }
  }
}

// The header's prompts, in child order: their line-order tables for the
// shared tail (token offsets, id offsets, ground truths).
// (kidx: the prompt index of each member, nullptr when every child is one.)
__global__ void js_prompt_tables_kernel(const JChild* ch, int64_t c0, int64_t nkids, const uint32_t* kidx,
                                        const int64_t* id_off, const int64_t* int_off, int64_t* p_id_off,
                                        int64_t* p_tok_off, int32_t* p_gt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nkids;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nkids && ch[c0 + i].err) continue;  // a dropped member
    const int64_t k = kidx ? kidx[i] : i;
    p_id_off[k] = id_off[c0 + i] - id_off[c0];
    p_tok_off[k] = int_off[c0 + i] - int_off[c0];
    if (i < nkids) p_gt[k] = ch[c0 + i].gt;
  }
}

}  // namespace
}  // namespace rs

using namespace rs;

extern "C" int rs_trace_csr_parse_jsonl(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr,
                                        rs_trace_csr** out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out || (!text && n_bytes > 0)) return fail(RS_E_ARG, "NULL argument");
  if (n_bytes < 0) return fail(RS_E_ARG, "negative size");
  *out = nullptr;
  try {
    PhaseClock clk;
    char* d_text = nullptr;
    RS_TRY(trace_stage_text(ctx, text, n_bytes, device_ptr, &d_text));
    AsyncBuf b_ls;
    int64_t* line_start = nullptr;
    int64_t L = 0;
    RS_TRY(trace_line_starts(ctx, d_text, n_bytes, &b_ls, &line_start, &L));
    clk.mark("line starts");
    auto grid = [&](int64_t n) {
      return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 32 * (int64_t)ctx->num_sms));
    };
    // 1. structural index
    const int64_t W = std::max<int64_t>(1, (n_bytes + 63) / 64);
    AsyncBuf b_w;
    const size_t wbytes = abytes(W, 1) * 2 + abytes(W + 1, 4) * 6 + abytes(W + 1, 8) * 4 +
                          scan_scratch_bytes(W + 1, 8) + abytes(8, 8);
    char* wb = b_w.alloc<char>(ctx->stream, wbytes);
    if (!wb) return fail(RS_E_NOMEM, "jsonl structural index: allocation failed");
    auto carve = [&](char*& base, size_t nb) {
      char* q = base;
      base += nb;
      return q;
    };
    uint8_t* tail = (uint8_t*)carve(wb, abytes(W, 1));
    uint8_t* ncl = (uint8_t*)carve(wb, abytes(W, 1));
    uint32_t* qpar = (uint32_t*)carve(wb, abytes(W + 1, 4));
    uint32_t* qscan = (uint32_t*)carve(wb, abytes(W + 1, 4));
    uint32_t* ca = (uint32_t*)carve(wb, abytes(W + 1, 4));
    uint32_t* cb = (uint32_t*)carve(wb, abytes(W + 1, 4));
    uint32_t* oa = (uint32_t*)carve(wb, abytes(W + 1, 4));
    uint32_t* ob = (uint32_t*)carve(wb, abytes(W + 1, 4));
    auto* dd = (unsigned long long*)carve(wb, abytes(W + 1, 8));
    auto* dscan = (unsigned long long*)carve(wb, abytes(W + 1, 8));
    uint64_t* ma = (uint64_t*)carve(wb, abytes(W + 1, 8));  // per word: list A / list B token masks
    uint64_t* mb = (uint64_t*)carve(wb, abytes(W + 1, 8));
    auto* part64 = (unsigned long long*)carve(wb, scan_scratch_bytes(W + 1, 8));
    auto* small = (unsigned int*)carve(wb, abytes(8, 8));  // first line, #containers, first error, totals
    uint32_t* part32 = (uint32_t*)part64;
    const int gw = grid(W);
    RS_LAUNCH(ctx, "jsonl_bs", js_bs_kernel, gw, 256, 0, d_text, n_bytes, W, tail);
    RS_LAUNCH(ctx, "jsonl_quote", js_quote_kernel, gw, 256, 0, d_text, n_bytes, W, tail, qpar);
    RS_TRY(exclusive_scan<uint32_t>(ctx, qpar, qscan, W, part32, nullptr));
    RS_LAUNCH(ctx, "jsonl_depth", js_depth_kernel, gw, 256, 0, d_text, n_bytes, W, tail, qscan, dd, ncl);
    RS_TRY(exclusive_scan<unsigned long long>(ctx, dd, dscan, W, part64, nullptr));
    RS_LAUNCH(ctx, "jsonl_tok_count", js_tokens_kernel, gw, 256, 0, d_text, n_bytes, W, tail, qscan, dscan, ncl,
              ca, cb, ma, mb);
    RS_TRY(exclusive_scan<uint32_t>(ctx, ca, oa, W, part32, oa + W));
    RS_TRY(exclusive_scan<uint32_t>(ctx, cb, ob, W, part32, ob + W));
    uint32_t tot[2];
    RS_TRY(d2h(ctx, &tot[0], oa + W, 4));
    RS_TRY(d2h(ctx, &tot[1], ob + W, 4));
    RS_TRY(sync_and_check(ctx));
    const int64_t NA = tot[0], NB = tot[1];
    AsyncBuf b_lists;
    char* lbuf = b_lists.alloc<char>(ctx->stream, abytes(NA + 1, 8) + abytes(NB + 1, 8));
    if (!lbuf) return fail(RS_E_NOMEM, "jsonl token lists: allocation failed");
    uint64_t* la = (uint64_t*)carve(lbuf, abytes(NA + 1, 8));
    int64_t* lbv = (int64_t*)carve(lbuf, abytes(NB + 1, 8));
    RS_LAUNCH(ctx, "jsonl_tok_write", js_tokens_expand_kernel, gw, 256, 0, d_text, W, (const uint32_t*)ca,
              (const uint32_t*)cb, (const uint64_t*)ma, (const uint64_t*)mb, (const uint32_t*)oa, (const uint32_t*)ob,
              la, lbv);
    clk.mark("structural index");
    // 2. lines
    const int64_t cont_cap = NA / 2 + 1;
    AsyncBuf b_lines;
    char* lnb = b_lines.alloc<char>(ctx->stream, abytes(L, sizeof(JLine)) + abytes(cont_cap, sizeof(JCont)) +
                                                     abytes(cont_cap + 1, 8) * 2 + scan_scratch_bytes(cont_cap + 1, 8));
    if (!lnb) return fail(RS_E_NOMEM, "jsonl line records: allocation failed");
    JLine* d_lines = (JLine*)carve(lnb, abytes(L, sizeof(JLine)));
    JCont* d_conts = (JCont*)carve(lnb, abytes(cont_cap, sizeof(JCont)));
    auto* nchild = (unsigned long long*)carve(lnb, abytes(cont_cap + 1, 8));
    auto* cscan = (unsigned long long*)carve(lnb, abytes(cont_cap + 1, 8));
    auto* cpart = (unsigned long long*)carve(lnb, scan_scratch_bytes(cont_cap + 1, 8));
    const unsigned int init[4] = {~0u, 0u, ~0u, 0u};
    RS_TRY(h2d(ctx, small, init, sizeof init));
    RS_LAUNCH(ctx, "jsonl_first_line", js_first_line_kernel, grid(L), 256, 0, d_text, line_start, L, n_bytes,
              small);
    RS_LAUNCH(ctx, "jsonl_lines", js_line_kernel, grid(L), 128, 0, d_text, line_start, L, n_bytes, small,
              la, NA, d_lines, d_conts, small + 1, cont_cap);
    unsigned int hs[2];
    RS_TRY(d2h(ctx, hs, small, 8));
    RS_TRY(sync_and_check(ctx));
    const int64_t first = hs[0] == ~0u ? -1 : (int64_t)hs[0];
    const int64_t NC = std::min<int64_t>(hs[1], cont_cap);
    // 3. children of every member container
    RS_LAUNCH(ctx, "jsonl_child_count", js_child_count_kernel, grid(NC), 256, 0, d_text, d_conts, NC, lbv, NB,
              nchild);
    RS_TRY(exclusive_scan<unsigned long long>(ctx, nchild, cscan, NC, cpart, cscan + NC));
    unsigned long long nch = 0;
    RS_TRY(d2h(ctx, &nch, cscan + NC, 8));
    RS_TRY(sync_and_check(ctx));
    const int64_t NCH = (int64_t)nch;
    AsyncBuf b_ch;
    char* chb = b_ch.alloc<char>(ctx->stream, abytes(NCH + 1, sizeof(JChild)) + abytes(NCH + 1, 8) * 4 +
                                                  scan_scratch_bytes(NCH + 1, 8));
    if (!chb) return fail(RS_E_NOMEM, "jsonl children: allocation failed");
    JChild* d_ch = (JChild*)carve(chb, abytes(NCH + 1, sizeof(JChild)));
    auto* idl = (unsigned long long*)carve(chb, abytes(NCH + 1, 8));
    auto* nint = (unsigned long long*)carve(chb, abytes(NCH + 1, 8));
    auto* id_off = (unsigned long long*)carve(chb, abytes(NCH + 1, 8));
    auto* int_off = (unsigned long long*)carve(chb, abytes(NCH + 1, 8));
    auto* chpart = (unsigned long long*)carve(chb, scan_scratch_bytes(NCH + 1, 8));
    // the containers (the prompts one gets a warp per prompt object)
    std::vector<JCont> hc(NC);
    std::vector<unsigned long long> hcs(NC + 1, 0);
    if (NC) {
      RS_TRY(d2h(ctx, hc.data(), d_conts, sizeof(JCont) * NC));
      RS_TRY(d2h(ctx, hcs.data(), cscan, 8ull * (NC + 1)));
      RS_TRY(sync_and_check(ctx));
    }
    int64_t pc = -1;  // the prompts container
    for (int64_t c = 0; c < NC; ++c)
      if (hc[c].role == kRPrompts) pc = c;
    const int64_t c0 = pc >= 0 ? (int64_t)hcs[pc] : 0;
    const int64_t nkids = pc >= 0 ? (int64_t)(hcs[pc + 1] - hcs[pc]) : 0;  // prompt objects / members
    const bool pobj = pc >= 0 && hc[pc].is_obj;  // "prompts" given as an object
    int32_t P = (int32_t)nkids;                  // prompts (object: after the duplicate rule)
    auto wgrid = [&](int64_t n) {  // a warp per item, 128-thread blocks
      return (int)std::max<int64_t>(1, std::min<int64_t>((n + 3) / 4, 64 * (int64_t)ctx->num_sms));
    };
    if (NCH > 0)
      RS_LAUNCH(ctx, "jsonl_child_check", js_child_kernel<false>, grid(NCH), 128, 0, d_text, d_conts, cscan, NC,
                lbv, NB, NCH, d_ch, (const int64_t*)nullptr, (const int64_t*)nullptr, (char*)nullptr,
                (int32_t*)nullptr, small + 2, 0);
    if (nkids > 0)
      RS_LAUNCH(ctx, "jsonl_prompt_check", js_prompt_kernel<0>, wgrid(nkids), 128, 0, d_text, d_conts, cscan,
                c0, nkids, lbv, NB, pc, d_ch, (const int64_t*)nullptr, (const int64_t*)nullptr, (char*)nullptr,
                (int32_t*)nullptr, small + 2);
    // "prompts" as an object: nlohmann keeps the last member of each key; the
    // others are neither prompts nor schema errors
    AsyncBuf b_keys;
    uint32_t* kidx = nullptr;  // prompt index of each member (exclusive scan of the survivors)
    if (pobj && nkids > 0) {
      char* q = b_keys.alloc<char>(ctx->stream, abytes(nkids + 1, 8) * 3 + abytes(nkids + 1, 4) * 3 +
                                                    scan_scratch_bytes(nkids + 1, 8));
      if (!q) return fail(RS_E_NOMEM, "jsonl prompt keys: allocation failed");
      auto* kl = (unsigned long long*)carve(q, abytes(nkids + 1, 8));
      auto* koff = (unsigned long long*)carve(q, abytes(nkids + 1, 8));
      auto* kpart = (unsigned long long*)carve(q, scan_scratch_bytes(nkids + 1, 8));
      uint32_t* kperm = (uint32_t*)carve(q, abytes(nkids + 1, 4));
      uint32_t* kept = (uint32_t*)carve(q, abytes(nkids + 1, 4));
      kidx = (uint32_t*)carve(q, abytes(nkids + 1, 4));
      RS_LAUNCH(ctx, "jsonl_key_sizes", js_key_sizes_kernel, grid(nkids), 256, 0, d_ch, c0, nkids, kl);
      RS_TRY(exclusive_scan<unsigned long long>(ctx, kl, koff, nkids, kpart, koff + nkids));
      std::vector<unsigned long long> hkl(nkids);
      unsigned long long kbytes = 0;
      RS_TRY(d2h(ctx, hkl.data(), kl, 8ull * nkids));
      RS_TRY(d2h(ctx, &kbytes, koff + nkids, 8));
      RS_TRY(sync_and_check(ctx));
      int64_t maxk = 1;
      for (unsigned long long v : hkl) maxk = std::max<int64_t>(maxk, (int64_t)v);
      AsyncBuf b_kb;
      char* keys = b_kb.alloc<char>(ctx->stream, kbytes + 1);
      if (!keys) return fail(RS_E_NOMEM, "jsonl prompt keys: allocation failed");
      RS_LAUNCH(ctx, "jsonl_key_write", js_key_write_kernel, grid(nkids), 256, 0, d_text, d_ch, c0, nkids,
                (const int64_t*)koff, keys);
      RS_TRY(arena_reserve(ctx, rank_strings_device_bytes(nkids, maxk) + (1 << 16)));
      RS_TRY(rank_strings_device(ctx, keys, (const int64_t*)koff, nkids, maxk, kperm));
      RS_LAUNCH(ctx, "jsonl_key_dedup", js_key_dedup_kernel, grid(nkids), 256, 0, d_ch, c0, nkids, kperm, keys,
                (const int64_t*)koff, small + 2, kept);
      RS_TRY(exclusive_scan<uint32_t>(ctx, kept, kidx, nkids, (uint32_t*)kpart, kidx + nkids));
      uint32_t np = 0;
      RS_TRY(d2h(ctx, &np, kidx + nkids, 4));
      RS_TRY(sync_and_check(ctx));
      P = (int32_t)np;
    }
    // the first error line over the lines and the children
    std::vector<JLine> hl(L);
    unsigned int cerr = ~0u;
    RS_TRY(d2h(ctx, hl.data(), d_lines, sizeof(JLine) * L));
    RS_TRY(d2h(ctx, &cerr, small + 2, 4));
    RS_TRY(sync_and_check(ctx));
    clk.mark("lines + children");
    int64_t err_line = -1;
    int err_kind = 0;
    auto first_error = [&]() {
      err_line = -1;
      err_kind = 0;
      for (int64_t ln = 0; ln < L; ++ln)
        if (hl[ln].err) {
          err_line = ln;
          err_kind = hl[ln].err;
          break;
        }
      if (cerr != ~0u && (err_line < 0 || (int64_t)(cerr >> 1) < err_line)) {
        err_line = cerr >> 1;
        err_kind = (cerr & 1) ? kJUnsup : kJErr;
      } else if (cerr != ~0u && (int64_t)(cerr >> 1) == err_line && err_kind == kJUnsup && !(cerr & 1)) {
        err_kind = kJErr;
      }
    };
    first_error();
    // pass 1 only sized the "token_ids" arrays: an error at or after the
    // prompts' line waits for their check, which may report an earlier one
    if (err_line >= 0 && nkids > 0 && err_line >= (int64_t)hc[pc].line) {
      RS_LAUNCH(ctx, "jsonl_prompt_verify", js_prompt_kernel<1>, wgrid(nkids), 128, 0, d_text, d_conts, cscan,
                c0, nkids, lbv, NB, pc, d_ch, (const int64_t*)nullptr, (const int64_t*)nullptr, (char*)nullptr,
                (int32_t*)nullptr, small + 2);
      RS_TRY(d2h(ctx, &cerr, small + 2, 4));
      RS_TRY(sync_and_check(ctx));
      first_error();
    }
    if (err_line >= 0)
      return trace_parse_error(err_line, err_kind == kJUnsup ? "JSON construct the device reader does not support"
                                                             : "malformed JSON trace line");
    if (first < 0) return fail(RS_E_PARSE, "<trace>: missing header line");
    // 4. the header's prompts (the container with the prompts role, if any)
    auto tr = new rs_trace_csr();
    std::unique_ptr<rs_trace_csr> own(tr);
    tr->device = ctx->device;
    const JLine& H = hl[first];
    tr->g = H.g;
    tr->max_prompt_len = H.mp;
    tr->max_response_len = H.mr;
    // sizes of every extracted child (per role), scanned, then written
    auto sizes = [&](int rmask) -> int {
      if (NCH == 0) return RS_OK;
      RS_LAUNCH(ctx, "jsonl_sizes", js_sizes_kernel, grid(NCH), 256, 0, d_ch, d_conts, NCH, rmask, idl, nint);
      RS_TRY(exclusive_scan<unsigned long long>(ctx, idl, id_off, NCH, chpart, id_off + NCH));
      RS_TRY(exclusive_scan<unsigned long long>(ctx, nint, int_off, NCH, chpart, int_off + NCH));
      return RS_OK;
    };
    RS_TRY(sizes(1 << kRPrompts));
    unsigned long long ptot[2] = {0, 0};
    if (NCH) {
      RS_TRY(d2h(ctx, &ptot[0], id_off + NCH, 8));
      RS_TRY(d2h(ctx, &ptot[1], int_off + NCH, 8));
      RS_TRY(sync_and_check(ctx));
    }
    const int64_t IDB = (int64_t)ptot[0], T = (int64_t)ptot[1];
    AsyncBuf b_p;
    char* pb = b_p.alloc<char>(ctx->stream, abytes(IDB + 1, 1) + abytes(T + 1, 4) + abytes(P + 1, 8) * 2 +
                                                abytes(P + 1, 4) * 2);
    if (!pb) return fail(RS_E_NOMEM, "jsonl prompts: allocation failed");
    char* d_ids = carve(pb, abytes(IDB + 1, 1));
    int32_t* d_tok = (int32_t*)carve(pb, abytes(T + 1, 4));
    int64_t* p_id_off = (int64_t*)carve(pb, abytes(P + 1, 8));
    int64_t* p_tok_off = (int64_t*)carve(pb, abytes(P + 1, 8));
    int32_t* p_gt = (int32_t*)carve(pb, abytes(P + 1, 4));
    uint32_t* d_perm = (uint32_t*)carve(pb, abytes(P + 1, 4));
    int64_t maxid = 1;
    if (P > 0) {
      RS_LAUNCH(ctx, "jsonl_prompt_write", js_prompt_kernel<2>, wgrid(nkids), 128, 0, d_text, d_conts, cscan,
                c0, nkids, lbv, NB, pc, d_ch, (const int64_t*)id_off, (const int64_t*)int_off, d_ids, d_tok,
                small + 2);
      RS_LAUNCH(ctx, "jsonl_prompt_tables", js_prompt_tables_kernel, grid(nkids + 1), 256, 0, d_ch, c0, nkids,
                (const uint32_t*)kidx, (const int64_t*)id_off, (const int64_t*)int_off, p_id_off, p_tok_off, p_gt);
      std::vector<int64_t> ioff(P + 1);
      RS_TRY(d2h(ctx, ioff.data(), p_id_off, 8ull * (P + 1)));
      RS_TRY(d2h(ctx, &cerr, small + 2, 4));
      RS_TRY(sync_and_check(ctx));
      if (cerr != ~0u)  // a "token_ids" array pass 1 only sized (no other error is left)
        return trace_parse_error(cerr >> 1, (cerr & 1) ? "JSON construct the device reader does not support"
                                                       : "malformed JSON trace line");
      for (int32_t i = 0; i < P; ++i) maxid = std::max<int64_t>(maxid, ioff[i + 1] - ioff[i]);
    }
    RS_TRY(arena_reserve(ctx, rank_strings_device_bytes(std::max(P, 1), maxid) + (1 << 16)));
    RS_TRY(trace_sorted_table(ctx, tr, P, maxid, d_ids, p_id_off, p_tok_off, p_gt, d_perm));
    clk.mark("prompts");
    // 5. steps: the scheduled ids and lengths keys / lists of every step line
    // written on the device (one pass for both roles), the keys resolved
    // against the id-sorted table there, and the records copied to the host
    // through pinned memory in one go
    std::vector<unsigned long long> h_id_off, h_int_off, h_il, h_ni;
    std::vector<char> h_ids;
    std::vector<int32_t> h_ints;
    std::vector<int32_t> hp;  // per child: its index in the id-sorted table (-1: unknown)
    bool any_steps = false;
    for (int64_t ln = 0; ln < L; ++ln) any_steps |= hl[ln].kind == kLStep;
    // The step table on the device (js_step_*_kernel). Sets steps_done when
    // every step is of the valid form; otherwise the host path below runs
    // (it reports the reference's first error). Errors returned here are
    // CUDA / allocation failures only.
    bool steps_done = false;
    auto steps_device = [&](const int32_t* d_pidx, const int32_t* d_vals) -> int {
      const int32_t G = tr->g;
      if (G < 1) return RS_OK;
      std::vector<int64_t> sc_of(L, -1), lc_of(L, -1);  // the last container of each role
      for (int64_t c = 0; c < NC; ++c) {
        if (hc[c].role == kRSched) sc_of[hc[c].line] = c;
        if (hc[c].role == kRLengths) lc_of[hc[c].line] = c;
      }
      std::vector<int64_t> lines;
      std::vector<int64_t> cbase(NC, -1);
      std::vector<int32_t> cstep(NC, 0);
      std::vector<JStepLine> sl;
      int64_t nlk = 0, nsk = 0;
      int prev = -1;
      for (int64_t ln = 0; ln < L; ++ln) {
        if (hl[ln].kind != kLStep) continue;
        if (hl[ln].step <= prev) return RS_OK;  // not strictly increasing
        prev = hl[ln].step;
        const int64_t lc = lc_of[ln], sc = sc_of[ln];
        if (lc < 0 || !hc[lc].is_obj || hcs[lc + 1] == hcs[lc]) return RS_OK;
        const int32_t s = (int32_t)lines.size();
        JStepLine x{0, -1, 0, 0};
        if (hl[ln].has_sched) {
          if (sc < 0 || hcs[sc + 1] == hcs[sc]) return RS_OK;
          x.sk_start = (int32_t)nsk;
          cbase[sc] = nsk;
          cstep[sc] = s;
          nsk += (int64_t)(hcs[sc + 1] - hcs[sc]);
        }
        cbase[lc] = nlk;
        cstep[lc] = s;
        nlk += (int64_t)(hcs[lc + 1] - hcs[lc]);
        lines.push_back(ln);
        sl.push_back(x);
      }
      const int64_t nsl = (int64_t)lines.size();
      if (nsl == 0 || nlk >= INT32_MAX || nsk >= INT32_MAX || NCH >= (int64_t)UINT32_MAX) return RS_OK;
      const int64_t nmax = std::max<int64_t>(nlk, nsk);
      AsyncBuf b;
      char* q = b.alloc<char>(ctx->stream, abytes(NC, 8) + abytes(NC, 4) + abytes(nlk, 8) * 2 + abytes(nlk, 4) * 4 +
                                               abytes(nlk + 1, 4) + abytes(nsk + 1, 8) + abytes(nsk + 1, 4) +
                                               2 * radix_sort_scratch_bytes64(nmax) + scan_scratch_bytes(nlk + 1, 4) +
                                               abytes(nsl, 4) + abytes(nsl, sizeof(JStepLine)) + 64);
      if (!q) return fail(RS_E_NOMEM, "jsonl steps: allocation failed");
      int64_t* d_cbase = (int64_t*)carve(q, abytes(NC, 8));
      int32_t* d_cstep = (int32_t*)carve(q, abytes(NC, 4));
      uint64_t* lk = (uint64_t*)carve(q, abytes(nlk, 8));
      uint64_t* dk = (uint64_t*)carve(q, abytes(nlk, 8));
      uint32_t* lv = (uint32_t*)carve(q, abytes(nlk, 4));
      uint32_t* dw = (uint32_t*)carve(q, abytes(nlk, 4));
      uint32_t* flag = (uint32_t*)carve(q, abytes(nlk, 4));
      uint32_t* e_win = (uint32_t*)carve(q, abytes(nlk, 4));  // entries <= distinct keys (checked below)
      uint32_t* pos = (uint32_t*)carve(q, abytes(nlk + 1, 4));
      uint64_t* sk = (uint64_t*)carve(q, abytes(nsk + 1, 8));
      uint32_t* sv = (uint32_t*)carve(q, abytes(nsk + 1, 4));
      char* sort1 = carve(q, radix_sort_scratch_bytes64(nmax));
      char* sort2 = carve(q, radix_sort_scratch_bytes64(nmax));
      uint32_t* spart = (uint32_t*)carve(q, scan_scratch_bytes(nlk + 1, 4));
      int32_t* dcnt = (int32_t*)carve(q, abytes(nsl, 4));
      JStepLine* d_sl = (JStepLine*)carve(q, abytes(nsl, sizeof(JStepLine)));
      int* d_bad = (int*)carve(q, 64);
      RS_TRY(h2d(ctx, d_cbase, cbase.data(), 8ull * NC));
      RS_TRY(h2d(ctx, d_cstep, cstep.data(), 4ull * NC));
      RS_CUDA_TRY(cudaMemsetAsync(dcnt, 0, 4ull * nsl, ctx->stream));
      RS_CUDA_TRY(cudaMemsetAsync(d_bad, 0, 64, ctx->stream));
      RS_LAUNCH(ctx, "jsonl_step_keys", js_step_keys_kernel, grid(NCH), 256, 0, d_ch, d_conts, cscan, NCH,
                d_cbase, d_cstep, d_pidx, lk, lv, sk, sv, d_bad);
      uint64_t *lks, *sks;
      uint32_t *lvs, *svs;
      RS_TRY(radix_sort_pairs(ctx, lk, lv, nlk, sort1, &lks, &lvs));
      RS_TRY(radix_sort_pairs(ctx, sk, sv, nsk, sort2, &sks, &svs));
      RS_LAUNCH(ctx, "jsonl_step_ends", js_step_ends_kernel, grid(nlk), 256, 0, lks, nlk, flag);
      RS_TRY(exclusive_scan<uint32_t>(ctx, flag, pos, nlk, spart, pos + nlk));
      RS_LAUNCH(ctx, "jsonl_step_distinct", js_step_distinct_kernel, grid(nlk), 256, 0, lks, lvs, flag, pos, nlk,
                dk, dw, dcnt);
      std::vector<int32_t> hcnt(nsl);
      uint32_t nd = 0;
      int bad = 0;
      RS_TRY(d2h(ctx, hcnt.data(), dcnt, 4ull * nsl));
      RS_TRY(d2h(ctx, &nd, pos + nlk, 4));
      RS_TRY(d2h(ctx, &bad, d_bad, 4));
      RS_TRY(sync_and_check(ctx));
      if (bad) return RS_OK;
      // entries per step: the scheduled list, or the keys
      std::vector<int32_t> st_idx(nsl), e_off(nsl + 1, 0);
      int64_t dks = 0;
      for (int64_t s = 0; s < nsl; ++s) {
        const int64_t ln = lines[s];
        int64_t ne = hcnt[s];
        if (hl[ln].has_sched) {
          const int64_t sc = sc_of[ln];
          if ((int64_t)(hcs[sc + 1] - hcs[sc]) != ne) return RS_OK;  // lengths do not cover the batch
        }
        sl[s].dk_start = (int32_t)dks;
        sl[s].e_off = e_off[s];
        dks += hcnt[s];
        if ((int64_t)e_off[s] + ne >= INT32_MAX) return RS_OK;
        e_off[s + 1] = (int32_t)(e_off[s] + ne);
        st_idx[s] = hl[ln].step;
      }
      const int64_t ne = e_off[nsl];
      if (dks != (int64_t)nd || ne > nlk) return RS_OK;
      RS_TRY(h2d(ctx, d_sl, sl.data(), sizeof(JStepLine) * nsl));
      int32_t *d_step_idx = nullptr, *d_entry_off = nullptr, *d_entry_prompt = nullptr, *d_lengths = nullptr;
      auto release = [&]() {
        for (int32_t* p : {d_step_idx, d_entry_off, d_entry_prompt, d_lengths})
          if (p) cudaFreeAsync(p, ctx->stream);
      };
      if (cudaMallocAsync(&d_step_idx, 4ull * nsl, ctx->stream) != cudaSuccess ||
          cudaMallocAsync(&d_entry_off, 4ull * (nsl + 1), ctx->stream) != cudaSuccess ||
          cudaMallocAsync(&d_entry_prompt, 4ull * std::max<int64_t>(ne, 1), ctx->stream) != cudaSuccess ||
          cudaMallocAsync(&d_lengths, 4ull * std::max<int64_t>(ne * G, 1), ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        release();
        return fail(RS_E_NOMEM, "trace step table allocation failed");
      }
      RS_LAUNCH(ctx, "jsonl_step_entries", js_step_entries_kernel, grid(nsk + nd), 256, 0, sks, svs, nsk, dk, dw,
                (int64_t)nd, d_sl, d_entry_prompt, e_win, d_bad);
      RS_LAUNCH(ctx, "jsonl_step_lengths", js_step_lengths_kernel, grid(ne), 256, 0, e_win, ne, nint, int_off,
                d_vals, G, tr->max_response_len, d_lengths, d_bad);
      RS_TRY(h2d(ctx, d_step_idx, st_idx.data(), 4ull * nsl));
      RS_TRY(h2d(ctx, d_entry_off, e_off.data(), 4ull * (nsl + 1)));
      RS_TRY(d2h(ctx, &bad, d_bad, 4));
      RS_TRY(sync_and_check(ctx));
      if (bad) {
        release();
        return RS_OK;
      }
      tr->n_steps = (int32_t)nsl;
      tr->n_entries = ne;
      tr->d_step_idx = d_step_idx;
      tr->d_entry_off = d_entry_off;
      tr->d_entry_prompt = d_entry_prompt;
      tr->d_lengths = d_lengths;
      steps_done = true;
      return RS_OK;
    };
    if (any_steps && NCH > 0) {
      const int smask = (1 << kRSched) | (1 << kRLengths);
      RS_TRY(sizes(smask));
      unsigned long long tt[2];
      RS_TRY(d2h(ctx, &tt[0], id_off + NCH, 8));
      RS_TRY(d2h(ctx, &tt[1], int_off + NCH, 8));
      RS_TRY(sync_and_check(ctx));
      AsyncBuf b_st;
      char* q = b_st.alloc<char>(ctx->stream, abytes(tr->ids.size() + 1, 1) + abytes(P + 1, 8) + abytes(NCH, 4) +
                                                  abytes(tt[0] + 1, 1) + abytes(tt[1] + 1, 4));
      if (!q) return fail(RS_E_NOMEM, "jsonl steps: allocation failed");
      char* d_sids = carve(q, abytes(tr->ids.size() + 1, 1));
      int64_t* d_sid_off = (int64_t*)carve(q, abytes(P + 1, 8));
      int32_t* d_pidx = (int32_t*)carve(q, abytes(NCH, 4));
      char* d_i = carve(q, abytes(tt[0] + 1, 1));
      int32_t* d_n = (int32_t*)carve(q, abytes(tt[1] + 1, 4));
      if (!tr->ids.empty()) RS_TRY(h2d(ctx, d_sids, tr->ids.data(), tr->ids.size()));
      RS_TRY(h2d(ctx, d_sid_off, tr->id_off.data(), 8ull * (P + 1)));
      RS_CUDA_TRY(cudaMemsetAsync(d_pidx, 0xff, 4ull * NCH, ctx->stream));
      RS_LAUNCH(ctx, "jsonl_step_write", js_child_kernel<true>, grid(NCH), 128, 0, d_text, d_conts, cscan, NC,
                lbv, NB, NCH, d_ch, (const int64_t*)id_off, (const int64_t*)int_off, d_i, d_n, small + 2, smask);
      RS_LAUNCH(ctx, "jsonl_lookup", js_lookup_kernel, grid(NCH), 256, 0, d_ch, d_conts, NCH, smask,
                (const int64_t*)id_off, d_i, d_sids, d_sid_off, P, d_pidx);
      RS_TRY(steps_device(d_pidx, d_n));
      if (steps_done) clk.mark("steps: device table");
      if (!steps_done) {  // the host path: the records through one pinned staging area
      const size_t o_il = 0, o_ni = abytes(NCH, 8), o_p = 2 * abytes(NCH, 8), o_i = o_p + abytes(NCH, 4),
                   o_n = o_i + abytes(tt[0] + 1, 1), total_b = o_n + abytes(tt[1] + 1, 4);
      RS_TRY(pinned_reserve(ctx, total_b));
      char* hb = static_cast<char*>(ctx->pinned);
      RS_TRY(d2h(ctx, hb + o_il, idl, 8ull * NCH));
      RS_TRY(d2h(ctx, hb + o_ni, nint, 8ull * NCH));
      RS_TRY(d2h(ctx, hb + o_p, d_pidx, 4ull * NCH));
      if (tt[0]) RS_TRY(d2h(ctx, hb + o_i, d_i, tt[0]));
      if (tt[1]) RS_TRY(d2h(ctx, hb + o_n, d_n, 4ull * tt[1]));
      RS_TRY(sync_and_check(ctx));
      const auto* il = reinterpret_cast<const unsigned long long*>(hb + o_il);
      const auto* ni = reinterpret_cast<const unsigned long long*>(hb + o_ni);
      h_il.assign(il, il + NCH);
      h_ni.assign(ni, ni + NCH);
      hp.assign(reinterpret_cast<const int32_t*>(hb + o_p), reinterpret_cast<const int32_t*>(hb + o_p) + NCH);
      h_ids.assign(hb + o_i, hb + o_i + tt[0]);
      h_ints.assign(reinterpret_cast<const int32_t*>(hb + o_n), reinterpret_cast<const int32_t*>(hb + o_n) + tt[1]);
      h_id_off.assign(NCH + 1, 0);
      h_int_off.assign(NCH + 1, 0);
      for (int64_t u = 0; u < NCH; ++u) {
        h_id_off[u + 1] = h_id_off[u] + h_il[u];
        h_int_off[u + 1] = h_int_off[u] + h_ni[u];
      }
      }
      clk.mark("steps: device records");
    }
    // WorkloadTrace::validate: the prompt rules, then step by step
    RS_TRY(trace_validate_prompts(tr));
    clk.mark("prompt rules");
    if (!steps_done) {  // the host path (a deviation from the device path's valid form)
      // per step line: its containers (the last of each role) and children
      std::vector<int64_t> sched_c(L, -1), len_c(L, -1);
      for (int64_t c = 0; c < NC; ++c) {
        if (hc[c].role == kRSched) sched_c[hc[c].line] = c;
        if (hc[c].role == kRLengths) len_c[hc[c].line] = c;
      }
      auto id_index = [&](const std::string& id) -> int32_t {  // in the id-sorted table
        int32_t lo = 0, hi = tr->count;
        while (lo < hi) {
          const int32_t mid = (lo + hi) >> 1;
          const std::string m(tr->ids.data() + tr->id_off[mid], tr->ids.data() + tr->id_off[mid + 1]);
          if (m < id) lo = mid + 1;
          else if (id < m) hi = mid;
          else return mid;
        }
        return -1;
      };
      std::vector<int32_t> st_idx, e_off{0}, e_prompt, lens;
      int prev_step = -1;
      const int32_t G = tr->g;
      // "lengths" given as an array: nlohmann's items() names the elements
      // "0", "1", ...; their table indices are looked up here
      std::vector<std::string> idx_key(any_steps ? NCH : 0);
      for (int64_t c = 0; c < NC && any_steps; ++c)
        if (hc[c].role == kRLengths && !hc[c].is_obj)
          for (unsigned long long u = hcs[c]; u < hcs[c + 1]; ++u) {
            idx_key[u] = std::to_string(u - hcs[c]);
            hp[u] = id_index(idx_key[u]);
          }
      auto child_id = [&](unsigned long long u) {
        if (!idx_key[u].empty()) return idx_key[u];
        return std::string(h_ids.data() + h_id_off[u], h_ids.data() + h_id_off[u] + h_il[u]);
      };
      auto table_id = [&](int32_t p) {
        return std::string(tr->ids.data() + tr->id_off[p], tr->ids.data() + tr->id_off[p + 1]);
      };
      // per prompt, stamped with the step line: its last lengths child, scheduled
      std::vector<int64_t> last_u(std::max(P, 1), -1), stamp_len(std::max(P, 1), -1),
          stamp_sched(std::max(P, 1), -1);
      for (int64_t ln = 0; ln < L; ++ln) {
        if (hl[ln].kind != kLStep) continue;
        const int step = hl[ln].step;
        const std::string sn = std::to_string(step);
        if (step <= prev_step)
          return fail(RS_E_VALIDATION, "step indices must be strictly increasing at step " + sn);
        prev_step = step;
        // the lengths map (std::map: key order, the last duplicate wins) by
        // table index; a key outside the table takes the string path below
        std::vector<int32_t> keys;
        bool known = true;
        if (len_c[ln] >= 0)
          for (unsigned long long u = hcs[len_c[ln]]; u < hcs[len_c[ln] + 1] && known; ++u) {
            const int32_t p = hp[u];
            if (p < 0) {
              known = false;
              break;
            }
            if (stamp_len[p] != ln) {
              stamp_len[p] = ln;
              keys.push_back(p);
            }
            last_u[p] = (int64_t)u;
          }
        // items() of an array runs in element order (an object's, in key order)
        const bool arr = len_c[ln] >= 0 && !hc[len_c[ln]].is_obj;
        if (known) {
          const std::vector<int32_t> keys_items = arr ? keys : std::vector<int32_t>();
          if ((int64_t)keys.size() * 16 > (int64_t)P) {  // dense: the stamps in table order
            keys.clear();
            for (int32_t p = 0; p < P; ++p)
              if (stamp_len[p] == ln) keys.push_back(p);
          } else {
            std::sort(keys.begin(), keys.end());
          }
          std::vector<int32_t> sched;
          std::vector<unsigned long long> sched_u;
          if (hl[ln].has_sched && sched_c[ln] >= 0) {
            for (unsigned long long u = hcs[sched_c[ln]]; u < hcs[sched_c[ln] + 1]; ++u) {
              sched.push_back(hp[u]);
              sched_u.push_back(u);
            }
          } else if (!hl[ln].has_sched) {
            sched = arr ? keys_items : keys;
          }
          if (sched.empty()) return fail(RS_E_VALIDATION, "step " + sn + " schedules no prompts");
          for (size_t i = 0; i < sched.size(); ++i) {
            const int32_t p = sched[i];
            if (p < 0)
              return fail(RS_E_VALIDATION, "step " + sn + " schedules unknown prompt '" + child_id(sched_u[i]) + "'");
            if (stamp_sched[p] == ln)
              return fail(RS_E_VALIDATION, "step " + sn + " schedules prompt '" + table_id(p) + "' twice");
            stamp_sched[p] = ln;
          }
          if (keys.size() != sched.size())
            return fail(RS_E_VALIDATION, "step " + sn + " lengths do not cover the scheduled batch");
          for (const int32_t p : keys) {
            if (stamp_sched[p] != ln)
              return fail(RS_E_VALIDATION, "step " + sn + " has lengths for unscheduled prompt '" + table_id(p) + "'");
            const unsigned long long u = (unsigned long long)last_u[p];
            if ((int)h_ni[u] != G)
              return fail(RS_E_VALIDATION, "step " + sn + " prompt '" + table_id(p) + "' needs exactly " +
                                               std::to_string(G) + " response lengths");
            for (int64_t i = 0; i < (int64_t)h_ni[u]; ++i) {
              const int l = h_ints[h_int_off[u] + i];
              if (l < 1 || l > tr->max_response_len)
                return fail(RS_E_VALIDATION, "step " + sn + " prompt '" + table_id(p) +
                                                 "' response length out of range: " + std::to_string(l));
            }
          }
          st_idx.push_back(step);
          for (const int32_t p : sched) {
            e_prompt.push_back(p);
            const unsigned long long u = (unsigned long long)last_u[p];
            lens.insert(lens.end(), h_ints.begin() + h_int_off[u], h_ints.begin() + h_int_off[u] + h_ni[u]);
          }
          e_off.push_back((int32_t)e_prompt.size());
          continue;
        }
        // a key outside the prompt table: the reference's containers verbatim
        std::vector<std::string> sched;
        std::map<std::string, std::vector<int>> lmap;
        for (unsigned long long u = hcs[len_c[ln]]; u < hcs[len_c[ln] + 1]; ++u)
          lmap[child_id(u)] = std::vector<int>(h_ints.begin() + h_int_off[u], h_ints.begin() + h_int_off[u] + h_ni[u]);
        if (hl[ln].has_sched && sched_c[ln] >= 0) {
          for (unsigned long long u = hcs[sched_c[ln]]; u < hcs[sched_c[ln] + 1]; ++u) sched.push_back(child_id(u));
        } else if (!hl[ln].has_sched) {
          if (arr)
            for (unsigned long long u = hcs[len_c[ln]]; u < hcs[len_c[ln] + 1]; ++u) sched.push_back(child_id(u));
          else
            for (const auto& kv : lmap) sched.push_back(kv.first);
        }
        if (sched.empty()) return fail(RS_E_VALIDATION, "step " + sn + " schedules no prompts");
        std::set<std::string> seen;
        for (const std::string& id : sched) {
          if (id_index(id) < 0) return fail(RS_E_VALIDATION, "step " + sn + " schedules unknown prompt '" + id + "'");
          if (!seen.insert(id).second)
            return fail(RS_E_VALIDATION, "step " + sn + " schedules prompt '" + id + "' twice");
        }
        if (lmap.size() != sched.size())
          return fail(RS_E_VALIDATION, "step " + sn + " lengths do not cover the scheduled batch");
        for (const auto& kv : lmap) {
          if (!seen.count(kv.first))
            return fail(RS_E_VALIDATION, "step " + sn + " has lengths for unscheduled prompt '" + kv.first + "'");
          if ((int)kv.second.size() != G)
            return fail(RS_E_VALIDATION, "step " + sn + " prompt '" + kv.first + "' needs exactly " +
                                             std::to_string(G) + " response lengths");
          for (int l : kv.second)
            if (l < 1 || l > tr->max_response_len)
              return fail(RS_E_VALIDATION, "step " + sn + " prompt '" + kv.first +
                                               "' response length out of range: " + std::to_string(l));
        }
        return fail(RS_E_VALIDATION, "step " + sn + ": lengths key outside the prompt table");  // unreachable
      }
      clk.mark("steps (host)");
      // the step table, owned by the handle
      tr->n_steps = (int32_t)st_idx.size();
      tr->n_entries = (int64_t)e_prompt.size();
      tr->device = ctx->device;
      if (tr->n_steps > 0) {
        if (cudaMallocAsync(&tr->d_step_idx, 4ull * st_idx.size(), ctx->stream) != cudaSuccess ||
            cudaMallocAsync(&tr->d_entry_off, 4ull * e_off.size(), ctx->stream) != cudaSuccess ||
            cudaMallocAsync(&tr->d_entry_prompt, 4ull * std::max<size_t>(e_prompt.size(), 1), ctx->stream) != cudaSuccess ||
            cudaMallocAsync(&tr->d_lengths, 4ull * std::max<size_t>(lens.size(), 1), ctx->stream) != cudaSuccess) {
          cudaGetLastError();
          return fail(RS_E_NOMEM, "trace step table allocation failed");
        }
        RS_TRY(h2d(ctx, tr->d_step_idx, st_idx.data(), 4ull * st_idx.size()));
        RS_TRY(h2d(ctx, tr->d_entry_off, e_off.data(), 4ull * e_off.size()));
        RS_TRY(h2d(ctx, tr->d_entry_prompt, e_prompt.data(), 4ull * e_prompt.size()));
        RS_TRY(h2d(ctx, tr->d_lengths, lens.data(), 4ull * lens.size()));
      }
    }
    // the id-ordered token CSR
    RS_TRY(trace_gather_csr(ctx, tr, d_tok, p_tok_off, d_perm));
    clk.mark("CSR gather");
    *out = own.release();
    return RS_OK;
  } catch (const std::bad_alloc&) {
    return fail(RS_E_NOMEM, "host allocation failed");
  }
}
