// rs_dedup.cu — shared-prefix dedup (1) of the RLHFless planning core.
//
// Reference: PrefixIndex::build (proj/src/dedup.cpp:30-100) sorts the batch
// lexicographically and counts, per depth, the trie nodes created by each
// distinct prompt after its sorted predecessor (node_diff[lcp+1] += 1,
// node_diff[len+1] -= 1), skipping exact duplicates, then turns the
// difference array and the per-length counts into five prefix tables.
//
// B200 design: no string sort. The multiset of adjacent LCPs
// of the sorted distinct prompts equals sum over trie branch nodes v of
// (deg(v) - 1) copies of depth(v), where deg counts children plus "a prompt
// ends here". We recover every branch node exactly by refining classes of
// prompts that share a verified prefix:
//   class c = (representative r, verified common prefix length l)
//   each member m computes x = lcp(m, r) from l on (warp-cooperative,
//   coalesced 128-bit loads of m; r is hot in L1) and t = m[x] or END;
//   (c, x) names the branch node on r's path at depth x; every distinct t
//   is one extra child -> node_diff[x+1] += 1; members with equal (c, x, t)
//   form the next class with verified prefix x+1 (rep = min index), or a
//   leaf (END, or a single member); exact duplicates of r are dropped.
// Every token of every prompt is read at most once (plus r's, from cache),
// so the pass is HBM-bound on the first round. Grouping uses two
// open-addressing tables keyed (c<<32|x) and (slotA<<33|t) with CAS insert.
// The same refinement with lengths truncated to L gives the dedup map and
// unique_prefix_count_among (dedup.cpp:163-183).
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr uint64_t kEmpty = ~0ULL;
constexpr uint64_t kEnd = 1ULL << 32;  // t value for "prompt ends at x"

// One set of grouping tables: A keyed (class << 32 | x), B keyed
// (slotA << 33 | t) with the branch's smallest member and its count.
struct Tab {
  uint64_t* a_keys;
  uint64_t* b_keys;
  int32_t* b_rep;
  int32_t* b_cnt;
};

struct DedupState {
  int P;
  int maxd;           // histogram depth bound (arrays hold maxd + 2); longer prompts clamp

  const int32_t* tok;
  const int64_t* off;
  int32_t* len;       // effective (possibly truncated) lengths
  int64_t* node_diff; // maxd + 2
  int64_t* end_count; // maxd + 2
  int64_t* len_count; // maxd + 2
  int64_t* stats;     // {INT64_MAX - min, max, total, leaves} (zero-initialised)
  int* flags;         // kernel status bits of this build
  int32_t* labels;    // optional
  // refinement
  int32_t* mem_idx[2];
  int32_t* m_slot[2];  // per member of a round: its B slot, or -1 (exact duplicate)
  Tab tab[3];         // grouping tables, rotating over rounds (fill, read, clear)
  int32_t* counter;   // next member count
};

// Warp-aggregated atomicAdd of `v` (same for all active lanes) at base[idx].
__device__ __forceinline__ void agg_add(int64_t* base, int64_t idx, int64_t v) {
  unsigned act = __activemask();
  unsigned peers = __match_any_sync(act, idx);
  int leader = __ffs(peers) - 1;
  if ((threadIdx.x & 31) == leader)
    atomicAdd((unsigned long long*)(base + idx), (unsigned long long)(v * __popc(peers)));
}

__device__ __forceinline__ uint64_t volatile_load(const uint64_t* p) {
  return *(volatile const uint64_t*)p;
}

__device__ __forceinline__ uint32_t table_insert(uint64_t* keys, uint32_t mask,
                                                 uint64_t key, bool* created) {
  uint32_t h = (uint32_t)hash_u64(key) & mask;
  for (;;) {
    uint64_t cur = volatile_load(keys + h);
    if (cur == key) {
      *created = false;
      return h;
    }
    if (cur == kEmpty) {
      uint64_t prev = atomicCAS((unsigned long long*)(keys + h), kEmpty, key);
      if (prev == kEmpty) {
        *created = true;
        return h;
      }
      if (prev == key) {
        *created = false;
        return h;
      }
    }
    h = (h + 1) & mask;
  }
}

// The lengths (capped at cap_len; min / max / total into stats), the length
// histogram, the root class (rep = prompt 0, the smallest index, verified
// prefix 0; members 1 .. P-1), round 0's table clear and its member count,
// in one pass over max(P, cap0). Histogram indices clamp at maxd + 1: a
// longer prompt makes the host redo the refinement with larger arrays.
__global__ void init_kernel(DedupState st, int32_t cap_len, int strict, int* kc, uint32_t cap0) {
  __shared__ long long s_mn[8], s_mx[8];
  __shared__ unsigned long long s_sum[8];
  const int P = st.P;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid0 == 0) kc[0] = P - 1;
  // rounds 0 and 1 use table sets 0 and 1: cleared with 16-byte stores,
  // four slots per thread (cap0 is a power of two >= 64)
  for (uint32_t q = tid0; q < cap0 / 4; q += stride) {
    const ulonglong2 e2 = make_ulonglong2(kEmpty, kEmpty);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      reinterpret_cast<ulonglong2*>(st.tab[b].a_keys)[2 * q] = e2;
      reinterpret_cast<ulonglong2*>(st.tab[b].a_keys)[2 * q + 1] = e2;
      reinterpret_cast<ulonglong2*>(st.tab[b].b_keys)[2 * q] = e2;
      reinterpret_cast<ulonglong2*>(st.tab[b].b_keys)[2 * q + 1] = e2;
      reinterpret_cast<int4*>(st.tab[b].b_rep)[q] = make_int4(INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX);
      reinterpret_cast<int4*>(st.tab[b].b_cnt)[q] = make_int4(0, 0, 0, 0);
    }
  }
  long long mn = INT64_MAX, mx = 0;
  unsigned long long sum = 0;
  for (uint32_t i = tid0; i < (uint32_t)P; i += stride) {
    const int64_t raw = st.off[i + 1] - st.off[i];
    if (strict && raw < 1) atomicOr(st.flags, kFlagEmptyPrompt);
    int32_t l = (int32_t)(raw < cap_len ? raw : cap_len);
    if (l < 0) l = 0;
    st.len[i] = l;
    mn = l < mn ? l : mn;
    mx = l > mx ? l : mx;
    sum += (unsigned long long)l;
    const int lc = min(l, st.maxd + 1);
    agg_add(st.len_count, lc, 1);
    if (i == 0) {
      atomicAdd((unsigned long long*)&st.node_diff[1], 1ULL);  // first sorted string
      atomicAdd((unsigned long long*)&st.end_count[lc], 1ULL);
      atomicAdd((unsigned long long*)&st.node_diff[min(l + 1, st.maxd + 1)], (unsigned long long)-1LL);
      atomicAdd((unsigned long long*)&st.stats[3], 1ULL);
      if (st.labels) st.labels[0] = 0;
    } else {
      st.mem_idx[0][i - 1] = i;
    }
  }
  // one set of stats atomics per CTA
  if (blockIdx.x * blockDim.x >= (uint32_t)P) return;  // CTA-uniform: no prompts here
  mn = warp_min(mn);
  mx = warp_max(mx);
  sum = warp_sum(sum);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_mn[w] = mn;
    s_mx[w] = mx;
    s_sum[w] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < nw; ++k) {
      mn = s_mn[k] < mn ? s_mn[k] : mn;
      mx = s_mx[k] > mx ? s_mx[k] : mx;
      sum += s_sum[k];
    }
    atomicMax((long long*)&st.stats[0], INT64_MAX - mn);  // min, stored inverted
    atomicMax((long long*)&st.stats[1], mx);
    atomicAdd((unsigned long long*)&st.stats[2], sum);
  }
}

// Exact lcp(m, r) over [l0, n), warp-cooperative. m is streamed with 128-bit
// non-allocating loads when 16B aligned; r is read through L1.
__device__ __forceinline__ int warp_lcp(const int32_t* __restrict__ pm,
                                        const int32_t* __restrict__ pr, int l0, int n) {
  const int lane = threadIdx.x & 31;
  constexpr int kU = 4;               // 4 x 128 tokens in flight per warp
  const uintptr_t am = (uintptr_t)pm;
  // first position whose address in m is 16B aligned, at or below l0
  int align_shift = (int)((am / 4 + l0) & 3);
  const bool r_aligned = (((uintptr_t)pr - am) & 15) == 0;
  int pos = l0 - align_shift;
  while (pos < n) {
    int best = INT32_MAX;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      int p = pos + (u * 32 + lane) * 4;
      int4 a;
      if (p >= 0 && p + 3 < n) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
                     : "l"(pm + p));
      } else {
        a.x = (p + 0 >= 0 && p + 0 < n) ? pm[p + 0] : 0;
        a.y = (p + 1 >= 0 && p + 1 < n) ? pm[p + 1] : 0;
        a.z = (p + 2 >= 0 && p + 2 < n) ? pm[p + 2] : 0;
        a.w = (p + 3 >= 0 && p + 3 < n) ? pm[p + 3] : 0;
      }
      int4 b;
      if (r_aligned && p >= 0 && p + 3 < n) {
        b = __ldg(reinterpret_cast<const int4*>(pr + p));
      } else {
        b.x = (p + 0 >= 0 && p + 0 < n) ? __ldg(pr + p + 0) : 0;
        b.y = (p + 1 >= 0 && p + 1 < n) ? __ldg(pr + p + 1) : 0;
        b.z = (p + 2 >= 0 && p + 2 < n) ? __ldg(pr + p + 2) : 0;
        b.w = (p + 3 >= 0 && p + 3 < n) ? __ldg(pr + p + 3) : 0;
      }
      int e[4] = {a.x, a.y, a.z, a.w};
      int f[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int q = p + j;
        if (q >= l0 && q < n && best == INT32_MAX && e[j] != f[j]) best = q;
      }
    }
    best = warp_min(best);
    if (best != INT32_MAX) return best;
    pos += kU * 128;
  }
  return n;
}

__device__ __forceinline__ uint32_t dev_cap(int K) {
  const uint32_t need = 2u * (uint32_t)K + 2u;
  uint32_t c = 64;
  while (c < need) c <<= 1;
  return c;
}

// Clears the grouping tables for this round (capacity from the device-side
// member count) and the next round's counter.
__device__ __forceinline__ void clear_phase(const Tab& t, uint32_t cap, int bid, int nb) {
  for (uint32_t i = bid * blockDim.x + threadIdx.x; i < cap; i += nb * blockDim.x) {
    t.a_keys[i] = kEmpty;
    t.b_keys[i] = kEmpty;
    t.b_rep[i] = INT32_MAX;
    t.b_cnt[i] = 0;
  }
}

// Record member k's branch (x, t) against representative r of class c.
__device__ __forceinline__ void record_member(const DedupState& st, const Tab& tb, int32_t* mslot,
                                              int64_t k, int m, int c, int r, int x, int lm, int lr,
                                              uint32_t mask) {
  if (x == lm && x == lr) {  // exact duplicate of r: skipped (dedup.cpp:62)
    mslot[k] = -1;
    if (st.labels) st.labels[m] = r;
    return;
  }
  const uint64_t t = x < lm ? (uint64_t)(uint32_t)st.tok[st.off[m] + x] : kEnd;
  bool created;
  const uint32_t sa = table_insert(tb.a_keys, mask, ((uint64_t)c << 32) | (uint32_t)x, &created);
  const uint32_t sb = table_insert(tb.b_keys, mask, ((uint64_t)sa << 33) | t, &created);
  atomicMin(tb.b_rep + sb, m);
  atomicAdd(tb.b_cnt + sb, 1);
  mslot[k] = (int32_t)sb;
}

// Members of rounds >= 1 are compared inside round_phase: one lane per
// member probes the first kProbe tokens past the class LCP (nearly every
// member branches there); members still matching after the probe are handed,
// one at a time, to the whole warp (warp_lcp).
constexpr int kProbe = 4;

// Round 0 (one class, representative = prompt 0): the HBM-bound pass.
// The representative is staged once per CTA in shared memory; every warp
// streams its members through a 2-stage ring of 2 KB windows filled by bulk
// TMA copies (cp.async.bulk, one elected lane, completion on a per-slot
// mbarrier), with no per-lane copy instructions, and compares 512 tokens per
// stage with a warp-min for the first mismatch. Measured at C2 against other
// rings: 2 x 2 KB (42 KB of shared memory, four CTAs per SM by registers) is
// 5 % faster than 2 x 4 KB (three CTAs per SM) and 10 % faster than 4 x 2 KB;
// more resident warps beat a deeper ring.
constexpr int kStreamStages = 2;
constexpr int kStageTok = 512;
constexpr int kStreamWarps = 8;
static_assert(kStageTok % 128 == 0, "a window is whole int4 chunks per lane");
// The representative's first kRepSmemTok tokens are staged in shared memory
// (10 KB: ring + staging still fit three CTAs per SM); the rest, if any, is
// read through L1.
constexpr int kRepSmemTok = 2560;
constexpr int kStreamSmem = (int)sizeof(int32_t) * (kRepSmemTok + kStageTok * kStreamStages * kStreamWarps);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// 1D bulk TMA global -> shared, completing `bytes` on bar (16-byte aligned,
// bytes a multiple of 16).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kStreamWarps * 32)
compare_stream_kernel(DedupState st, const int* kcur) {
  extern __shared__ __align__(16) int32_t sm[];
  __shared__ int2 slot_meta[kStreamWarps][kStreamStages];  // (member, window) per ring slot
  __shared__ __align__(8) uint64_t slot_bar[kStreamWarps][kStreamStages];
  const int K = *kcur;
  if (K <= 0) return;
  const uint32_t mask = dev_cap(K) - 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int lr = st.len[0];
  int32_t* rep_s = sm;  // representative tokens [0, kRepSmemTok)
  int32_t* ring = sm + kRepSmemTok + kStageTok * kStreamStages * wid;
  int2* meta = slot_meta[wid];
  const int32_t* pr = st.tok + st.off[0];
  const int32_t* tok_end = st.tok + st.off[st.P];  // bulk copies must not read past it
  for (int i = threadIdx.x; i < min(lr, kRepSmemTok); i += blockDim.x) rep_s[i] = pr[i];
  // representative token / 16-byte chunk at p (chunks: p % 4 == 0)
  const bool rep_aligned = (((uintptr_t)pr) & 15) == 0;
  auto rep_at = [&](int p) { return p < kRepSmemTok ? rep_s[p] : __ldg(pr + p); };
  auto rep4_at = [&](int p) {
    return p < kRepSmemTok ? *reinterpret_cast<const int4*>(rep_s + p)
                           : __ldg(reinterpret_cast<const int4*>(pr + p));
  };
  uint64_t* bars = slot_bar[wid];
  if (lane == 0)
    for (int q = 0; q < kStreamStages; ++q) mbar_init(&bars[q], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t parity = 0;  // bit s: phase parity to wait for on slot s (warp-uniform)
  // Each warp owns a contiguous block of members (adjacent prompts are
  // adjacent in the CSR) and streams their windows back to back: the issue
  // cursor runs kStreamStages-1 windows ahead of the compare cursor across
  // member boundaries, so the ring never drains between members; windows of
  // a member whose mismatch is already known are not issued.
  const int64_t nw = (int64_t)gridDim.x * kStreamWarps;
  const int64_t gw = (int64_t)blockIdx.x * kStreamWarps + wid;
  const int64_t k_begin = K * gw / nw, k_end = K * (gw + 1) / nw;
  for (int64_t kb0 = k_begin; kb0 < k_end; kb0 += 32) {
    const int cnt = (int)(k_end - kb0 < 32 ? k_end - kb0 : 32);
    int my_m = 0, my_n = 0, my_lm = 0, my_shift = 0, my_nwin = 0;
    unsigned long long my_src = 0;
    if (lane < cnt) {  // lane i holds member kb0 + i
      my_m = st.mem_idx[0][kb0 + lane];
      my_lm = st.len[my_m];
      my_n = min(my_lm, lr);
      const int32_t* pm = st.tok + st.off[my_m];
      my_shift = (int)(((uintptr_t)pm >> 2) & 3);
      my_src = reinterpret_cast<unsigned long long>(pm - my_shift);
      my_nwin = (my_n + my_shift + kStageTok - 1) / kStageTok;
    }
    int im = 0, iwin = 0;           // next window to issue
    int seq_issue = 0, seq_cmp = 0;
    int cur = -1, found = INT32_MAX;  // member being compared, its mismatch
    auto issue_next = [&]() {
      if (im == cur && found != INT32_MAX) {  // mismatch known: skip the rest
        ++im;
        iwin = 0;
      }
      while (im < cnt && iwin >= __shfl_sync(0xffffffffu, my_nwin, im)) {
        ++im;
        iwin = 0;
      }
      const int slot = seq_issue % kStreamStages;
      // the slot was consumed by this warp one window ago (the __syncwarp
      // after its compare); order those generic reads before the async write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (im < cnt) {
        const int n = __shfl_sync(0xffffffffu, my_n, im);
        const int sh = __shfl_sync(0xffffffffu, my_shift, im);
        const int32_t* src = reinterpret_cast<const int32_t*>(__shfl_sync(0xffffffffu, my_src, im)) +
                             iwin * kStageTok;
        int32_t* dst = ring + slot * kStageTok;
        const int need = min(kStageTok, n + sh - iwin * kStageTok);  // tokens this window uses
        const uint32_t bytes = (uint32_t)((need * 4 + 15) & ~15);
        if (src + bytes / 4 <= tok_end) {
          if (lane == 0) {
            meta[slot] = make_int2(im, iwin);
            mbar_arrive_tx(&bars[slot], bytes);
            tma_load_1d(dst, src, bytes, &bars[slot]);
          }
        } else {  // the batch's last window: plain loads up to the end
          for (int j = lane; j < need; j += 32) dst[j] = src + j < tok_end ? src[j] : 0;
          __syncwarp();
          if (lane == 0) {
            meta[slot] = make_int2(im, iwin);
            mbar_arrive(&bars[slot]);
          }
        }
        ++iwin;
      } else if (lane == 0) {
        meta[slot] = make_int2(-1, 0);
        mbar_arrive(&bars[slot]);
      }
      ++seq_issue;
    };
    auto finish = [&](int i) {  // record member i
      const int m = __shfl_sync(0xffffffffu, my_m, i);
      const int lm = __shfl_sync(0xffffffffu, my_lm, i);
      const int n = __shfl_sync(0xffffffffu, my_n, i);
      if (lane == 0)
        record_member(st, st.tab[0], st.m_slot[0], kb0 + i, m, 0, 0, found == INT32_MAX ? n : found,
                      lm, lr, mask);
    };
    for (int s0 = 0; s0 < kStreamStages - 1; ++s0) issue_next();
    for (;;) {
      issue_next();
      const int slot = seq_cmp % kStreamStages;
      mbar_wait(&bars[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      __syncwarp();
      const int2 mw = meta[slot];
      ++seq_cmp;
      if (mw.x < 0) break;  // the issuer ran dry and everything issued is consumed
      if (mw.x != cur) {
        if (cur >= 0) finish(cur);
        cur = mw.x;
        found = INT32_MAX;
      }
      if (found != INT32_MAX) continue;  // already resolved: skip this window
      const int n = __shfl_sync(0xffffffffu, my_n, cur);
      const int sh = __shfl_sync(0xffffffffu, my_shift, cur);
      const int32_t* buf = ring + slot * kStageTok;
      // per int4: a 4-bit mismatch mask over the positions in [0, n); the
      // lane keeps its first mismatch (q ascending = position ascending)
      int best = INT32_MAX;
      if (sh == 0 && rep_aligned) {  // member and representative chunks both 16B aligned
#pragma unroll
        for (int q = 0; q < kStageTok / 128; ++q) {
          const int j = lane + 32 * q;
          const int p = mw.y * kStageTok + 4 * j;
          if (best == INT32_MAX && p < n) {
            const int4 a4 = *reinterpret_cast<const int4*>(buf + 4 * j);
            const int4 b4 = rep4_at(p);
            uint32_t m = (uint32_t)(a4.x != b4.x) | ((uint32_t)(a4.y != b4.y) << 1) |
                         ((uint32_t)(a4.z != b4.z) << 2) | ((uint32_t)(a4.w != b4.w) << 3);
            if (n - p < 4) m &= (1u << (n - p)) - 1;
            if (m) best = p + __ffs(m) - 1;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < kStageTok / 128; ++q) {
          const int j = lane + 32 * q;
          const int p = -sh + mw.y * kStageTok + 4 * j;
          if (best == INT32_MAX && p < n && p + 3 >= 0) {
            const int4 a4 = *reinterpret_cast<const int4*>(buf + 4 * j);
            const int e[4] = {a4.x, a4.y, a4.z, a4.w};
            uint32_t m = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int pos = p + t;
              if (pos >= 0 && pos < n) m |= (uint32_t)(e[t] != rep_at(pos)) << t;
            }
            if (m) best = p + __ffs(m) - 1;
          }
        }
      }
      found = __any_sync(0xffffffffu, best != INT32_MAX) ? warp_min(best) : INT32_MAX;
      __syncwarp();
    }
    if (cur >= 0) finish(cur);
    // drain the windows issued ahead of the last compare (their phases must
    // complete before the slots are reused by the next block of members)
    while (seq_cmp < seq_issue) {
      const int slot = seq_cmp % kStreamStages;
      mbar_wait(&bars[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      ++seq_cmp;
    }
    __syncwarp();
  }
}

// One thread per B slot: branch children, leaves, next classes.
// One phase per round r >= 0 (members in buffer cur, their branches in
// tables tr): every member that is not an exact duplicate looks up its
// branch. The branch's representative (its smallest member) accounts for it
// (dedup.cpp:58-78: one more child of the node at depth x, one leaf of
// length x for END or len[rep] otherwise). Every other member of a branch
// with two or more members and a next token continues: it is appended to
// round r + 1 (class = the branch slot, representative = rep, verified
// prefix x + 1) and compared right away, its branch recorded in tables tn.
__device__ __forceinline__ void round_phase(const DedupState& st, const Tab& tr, const Tab& tn,
                                            uint32_t mask_n, int cur, int K, int* knext, int bid,
                                            int nb) {
  const int nxt = cur ^ 1;
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)nb * (blockDim.x >> 5);
  for (int64_t k0 = ((int64_t)bid * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; k0 < K;
       k0 += W * 32) {
    const int64_t k = k0 + lane;
    bool cont = false;
    int m = 0, rep = 0, sb = 0, x = 0;
    if (k < K) {
      sb = st.m_slot[cur][k];
      if (sb >= 0) {
        m = st.mem_idx[cur][k];
        rep = tr.b_rep[sb];
        const uint64_t key = tr.b_keys[sb];
        const uint64_t t = key & ((1ULL << 33) - 1);
        const bool leaf = t == kEnd || tr.b_cnt[sb] == 1;
        if (m == rep || !leaf) x = (int)(uint32_t)(tr.a_keys[(uint32_t)(key >> 33)] & 0xffffffffULL);
        if (m == rep) {
          agg_add(st.node_diff, min(x + 1, st.maxd + 1), 1);
          const int leaf_len = min(t == kEnd ? x : st.len[rep], st.maxd + 1);
          agg_add(st.end_count, leaf_len, 1);
          agg_add(st.node_diff, min(leaf_len + 1, st.maxd + 1), -1);
          agg_add(st.stats, 3, 1);
        }
        if (leaf || m == rep) {
          if (st.labels) st.labels[m] = rep;
        } else {
          cont = true;
          ++x;  // the class's verified prefix
        }
      }
    }
    // warp-aggregated append to round r + 1
    const unsigned cm = __ballot_sync(0xffffffffu, cont);
    if (!cm) continue;
    const int leader = __ffs(cm) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(knext, __popc(cm));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int kn = base + __popc(cm & ((1u << lane) - 1));
    int lm = 0, lr = 0, n = 0;
    bool slow = false;
    if (cont) {
      st.mem_idx[nxt][kn] = m;
      lm = st.len[m];
      lr = st.len[rep];
      n = min(lm, lr);
      const int32_t* pm = st.tok + st.off[m];
      const int32_t* pr = st.tok + st.off[rep];
      const int lim = min(n, x + kProbe);
      while (x < lim && __ldg(pm + x) == __ldg(pr + x)) ++x;
      slow = x == lim && lim < n;
      if (!slow) record_member(st, tn, st.m_slot[nxt], kn, m, sb, rep, x, lm, lr, mask_n);
    }
    unsigned todo = __ballot_sync(0xffffffffu, slow);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int sm = __shfl_sync(0xffffffffu, m, src);
      const int sr = __shfl_sync(0xffffffffu, rep, src);
      const int sx = __shfl_sync(0xffffffffu, x, src);
      const int sn = __shfl_sync(0xffffffffu, n, src);
      const int xx = warp_lcp(st.tok + st.off[sm], st.tok + st.off[sr], sx, sn);
      if (lane == src) record_member(st, tn, st.m_slot[nxt], kn, m, sb, rep, xx, lm, lr, mask_n);
    }
  }
}

// Grid-wide barrier of the persistent refinement (all CTAs co-resident: the
// kernel is launched cooperatively). A 64-bit arrival counter, zeroed before
// the launch; barrier g completes when it reaches g * gridDim.x. Arrival is a
// release (cumulative over the CTA's writes ordered by the bar.sync before
// it), the poll an acquire, which invalidates the SM's L1: plain loads after
// the barrier see the other CTAs' writes (data written inside the kernel is
// never read through the non-coherent path).
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long* target) {
  *target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    } while (v < *target);
  }
  __syncthreads();
}

// Rounds with at most this many members finish on CTA 0 alone (CTA-wide
// barriers instead of grid-wide ones: the last rounds hold a handful).
constexpr int kSoloMembers = 1024;

// Every round after round 0's compare, in one persistent launch, one grid
// barrier per round: round_phase closes round r and compares round r + 1,
// while the table set of round r + 2 is cleared.
constexpr int kRefineT = 256;

__global__ void __launch_bounds__(kRefineT)
refine_kernel(DedupState st, int* kc, unsigned long long* bar) {
  unsigned long long target = 0;
  int cur = 0;
  bool solo = false;  // CTA 0 alone from here on
  int bid = blockIdx.x, nb = gridDim.x;
  auto sync = [&]() {
    if (solo) {  // the fence also invalidates L1 (table slots changed by atomics at L2)
      __syncthreads();
      if (threadIdx.x == 0) __threadfence();
      __syncthreads();
    } else {
      grid_barrier(bar, &target);
    }
  };
  // round r's branches are in set r % 3; round r + 1 fills set (r + 1) % 3,
  // cleared two phases earlier (the init kernel clears sets 0 and 1) with a
  // capacity from a member count >= its own
  // The member counts rotate the same way: phase r reads kc[r % 3], appends
  // to kc[(r + 1) % 3] and zeroes kc[(r + 2) % 3] (last read in phase r - 1).
  uint32_t capset[3];
  capset[0] = capset[1] = dev_cap(*(volatile int*)kc);
  capset[2] = 0;
  int set = 0;
  for (;;) {
    const int s1 = set == 2 ? 0 : set + 1, s2 = s1 == 2 ? 0 : s1 + 1;
    const int K = *(volatile int*)(kc + set);
    if (K <= 0) break;  // no members left (or a single prompt)
    if (!solo && K <= kSoloMembers) {
      if (blockIdx.x != 0) return;
      solo = true;
      nb = 1;
    }
    if (bid == 0 && threadIdx.x == 0) kc[s2] = 0;
    round_phase(st, st.tab[set], st.tab[s1], capset[s1] - 1, cur, K, kc + s1, bid, nb);
    capset[s2] = dev_cap(K);  // round r + 2 has at most K members
    clear_phase(st.tab[s2], capset[s2], bid, nb);
    sync();
    cur ^= 1;
    set = s1;
  }
}

// The five PrefixIndex tables from the difference array and the counts
// (dedup.cpp:73-98). With x_m = x on depths 1..maxd and 0 elsewhere:
//   nodes[d] = incl(node_diff_m)[d] (0 at d = 0 and d = maxd + 1)
//   scb[d]   = incl(end_count_m)[d] - end_count_m[d]
//   stb[d]   = incl(end_count_m * i)[d] - end_count_m[d] * d
//   lcf[d]   = total(len_count_m) - incl(len_count_m)[d]
//   ltf[d]   = total(len_count_m * i) - incl(len_count_m * i)[d]
// kTabSlices CTAs per table (five independent scans): each thread scans
// kTabIPT consecutive depths, one CTA-wide scan of the thread totals per
// chunk of kTabT * kTabIPT depths; every CTA of a table runs its (cheap)
// scan and writes one slice, so writes into mapped host memory leave from
// 5 x kTabSlices SMs at once. maxd < 0: the longest
// prompt from stats; the tables are written (stride maxd + 2) only if
// maxd <= cap_md. stats_out (nullable) receives {min, max, total, leaves,
// flags}.
constexpr int kTabT = 1024;
constexpr int kTabIPT = 4;
constexpr int kTabSlices = 4;
constexpr int kTabCtas = 5 * kTabSlices;
constexpr int kTabSmem = 8 * kTabT * kTabIPT;  // one chunk staged for coalesced writes

__global__ void __launch_bounds__(kTabT)
tables_kernel(DedupState st, int maxd, int cap_md, int64_t* out, int64_t* stats_out) {
  __shared__ int64_t ws[32];
  extern __shared__ int64_t stage[];  // [kTabT * kTabIPT]
  if (maxd < 0) maxd = (int)st.stats[1];
  const int q = blockIdx.x / kTabSlices, slice = blockIdx.x % kTabSlices;  // table, slice
  if (stats_out && q == 0 && threadIdx.x < 5)
    stats_out[threadIdx.x] = threadIdx.x == 0 ? INT64_MAX - st.stats[0]
                             : threadIdx.x == 4 ? (int64_t)*st.flags : st.stats[threadIdx.x];
  if (maxd > cap_md) return;
  const int n = maxd + 2;  // depths 0 .. maxd + 1
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t* tab = out + (int64_t)q * n;
  const int s_lo = (int)((int64_t)slice * n / kTabSlices), s_hi = (int)((int64_t)(slice + 1) * n / kTabSlices);
  const int64_t* src = q == 0 ? st.node_diff : q <= 2 ? st.end_count : st.len_count;
  const bool weighted = q == 2 || q == 4;  // x * depth
  // totals of the suffix tables: prompts of length >= 1, and all tokens
  const int64_t total = q == 3 ? st.P - st.len_count[0] : q == 4 ? st.stats[2] : 0;
  int64_t carry = 0;
  for (int d0 = 0; d0 < n; d0 += kTabT * kTabIPT) {
    int64_t x[kTabIPT];
    int64_t run = 0;
#pragma unroll
    for (int j = 0; j < kTabIPT; ++j) {
      const int d = d0 + threadIdx.x * kTabIPT + j;
      const int64_t c = d >= 1 && d <= maxd ? src[d] : 0;
      x[j] = weighted ? c * d : c;
      run += x[j];
    }
    const int64_t incl = warp_incl_sum(run);
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int64_t t = ws[lane];
      ws[lane] = warp_incl_sum(t) - t;
    }
    __syncthreads();
    int64_t pre = carry + ws[wid] + incl - run;  // exclusive prefix of this thread
#pragma unroll
    for (int j = 0; j < kTabIPT; ++j) {
      const int d = d0 + threadIdx.x * kTabIPT + j;
      pre += x[j];  // inclusive at d
      int64_t v;
      if (q == 0) v = d >= 1 && d <= maxd ? pre : 0;
      else if (q <= 2) v = pre - x[j];
      else v = total - pre;
      stage[threadIdx.x * kTabIPT + j] = v;
    }
    __syncthreads();
    {  // this CTA's slice of the chunk, consecutive depths per warp
      const int lo = max(d0, s_lo), hi = min(min(d0 + kTabT * kTabIPT, n), s_hi);
      for (int d = lo + threadIdx.x; d < hi; d += kTabT) tab[d] = stage[d - d0];
    }
    // the chunk's total (the last thread's inclusive prefix) carries over
    __syncthreads();
    if (threadIdx.x == kTabT - 1) ws[0] = ws[31] + incl;
    __syncthreads();
    carry += ws[0];
    __syncthreads();
  }
}

uint32_t pow2_at_least(int64_t v) {
  uint32_t c = 64;
  while ((int64_t)c < v) c <<= 1;
  return c;
}

}  // namespace

static int launch_refine(rs_ctx* ctx, DedupState st, int* kc, unsigned long long* bar) {
  int& per_sm = ctx->dev_cache.refine_per_sm;  // per device: the context's
  if (!per_sm) {
    RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_kernel, kRefineT, 0));
    per_sm = std::max(1, std::min(per_sm, 4));
  }
  const int blocks = per_sm * ctx->num_sms;
  void* args[] = {&st, &kc, &bar};
  cudaEvent_t ev = nullptr;
  timer_begin(ctx, "dedup_refine", &ev);
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)refine_kernel, blocks, kRefineT, args, 0, ctx->stream);
  ctx->launches++;
  if (e != cudaSuccess) return fail(RS_E_CUDA, std::string("launch dedup_refine: ") + cudaGetErrorString(e));
  timer_end(ctx, "dedup_refine", ev);
  return RS_OK;
}

// Runs the refinement on device-resident CSR. cap_len = INT32_MAX for the
// full index. Fills node_diff/end_count/len_count/stats (and labels if
// non-null). Everything is queued without a host round trip and
// synchronised once at the end. The histograms are sized by a bound (the
// hint, at least 16,384, at most cap_len); a longer prompt is seen in the
// final stats and the refinement reruns once with the exact size.
// tail (nullable): enqueued after the refinement, before the final
// synchronisation; it writes the four stats to pinned + kStatsOff (else
// they are copied there) and its own output (the index tables: into the
// index's pinned block).
constexpr size_t kPinnedHead = 128;
constexpr int kStatsOff = 4;  // int64 index of the read-back {stats, flags} in pinned
struct RefineTail {
  virtual int enqueue(rs_ctx* ctx, const DedupState& st, int cap_md) = 0;
  virtual void finish(rs_ctx* ctx) = 0;  // after the final synchronisation
};

static int tables_setup(rs_ctx* ctx) {
  bool& done = ctx->dev_cache.tables_ready;
  if (!done) {
    done = true;
  }
  return RS_OK;
}

static int stream_kernel_setup(rs_ctx* ctx, int* blocks_per_sm) {
  int& per_sm = ctx->dev_cache.stream_per_sm;
  if (!per_sm) {
    RS_CUDA_TRY(cudaFuncSetAttribute(compare_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kStreamSmem));
    RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compare_stream_kernel,
                                                              kStreamWarps * 32, kStreamSmem));
    per_sm = std::max(1, per_sm);
  }
  *blocks_per_sm = per_sm;
  return RS_OK;
}

static int dedup_refine(rs_ctx* ctx, const int32_t* d_tok, const int64_t* d_off, int P,
                        int32_t cap_len, int strict, bool want_labels, int32_t max_len_hint,
                        DedupState* out_state, int64_t* h_stats, int32_t* h_labels,
                        RefineTail* tail = nullptr) {
  const uint32_t cap = pow2_at_least(2 * (int64_t)P + 2);
  const size_t base_bytes = abytes(P, 4) + abytes(4, 8) + abytes(P, 4) * 4 +
                            3 * (abytes(cap, 8) * 2 + abytes(cap, 4) * 2) + abytes(P, 4);
  int64_t maxd = std::max<int64_t>(max_len_hint, 16384);
  maxd = std::max<int64_t>(1, std::min<int64_t>(maxd, cap_len));
  int per_sm = 1;
  RS_TRY(stream_kernel_setup(ctx, &per_sm));
  DedupState st{};
  int64_t hs[4];
  for (int attempt = 0; attempt < 2; ++attempt) {
    const int md = (int)maxd;
    // zero-initialised: three histograms, stats, flags, member counts, barrier
    const size_t zh = 3 * ((size_t)md + 2);
    const size_t zwords = zh + 8;
    RS_TRY(arena_reserve(ctx, base_bytes + 8 * abytes(zwords, 8) + (1 << 16)));
    RS_TRY(pinned_reserve(ctx, kPinnedHead));
    st = DedupState{};
    st.P = P;
    st.maxd = md;
    st.tok = d_tok;
    st.off = d_off;
    st.len = arena_alloc<int32_t>(ctx, P);
    int64_t* zero = arena_alloc<int64_t>(ctx, zwords);
    if (!zero) return fail(RS_E_NOMEM, "arena exhausted (dedup)");
    st.node_diff = zero;
    st.end_count = zero + (md + 2);
    st.len_count = zero + 2 * ((int64_t)md + 2);
    for (int b = 0; b < 2; ++b) {
      st.mem_idx[b] = arena_alloc<int32_t>(ctx, std::max(P, 1));
      st.m_slot[b] = arena_alloc<int32_t>(ctx, std::max(P, 1));
    }
    for (int b = 0; b < 3; ++b) {
      st.tab[b].a_keys = arena_alloc<uint64_t>(ctx, cap);
      st.tab[b].b_keys = arena_alloc<uint64_t>(ctx, cap);
      st.tab[b].b_rep = arena_alloc<int32_t>(ctx, cap);
      st.tab[b].b_cnt = arena_alloc<int32_t>(ctx, cap);
    }
    st.stats = zero + zh;
    st.flags = reinterpret_cast<int*>(zero + zh + 4);
    int* kc = reinterpret_cast<int*>(zero + zh + 5);  // member counts of rounds r % 3
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(zero + zh + 7);
    st.counter = kc;
    st.labels = want_labels ? arena_alloc<int32_t>(ctx, std::max(P, 1)) : nullptr;
    if (!st.tab[2].b_cnt || (want_labels && !st.labels)) return fail(RS_E_NOMEM, "arena exhausted (dedup)");
    int64_t* pin = reinterpret_cast<int64_t*>(ctx->pinned);
    RS_CUDA_TRY(cudaMemsetAsync(zero, 0, 8 * zwords, ctx->stream));
    const uint32_t cap0 = pow2_at_least(2 * (int64_t)(P - 1) + 2);  // dev_cap(P - 1)
    const int iblocks = (int)std::max<int64_t>(
        1, std::min<int64_t>((std::max<int64_t>(P, cap0 / 4) + 255) / 256, 8 * ctx->num_sms));
    RS_LAUNCH(ctx, "dedup_init", init_kernel, iblocks, 256, 0, st, cap_len, strict, kc, cap0);
    // round 0 (every member against prompt 0) streams the batch; every later
    // round runs inside one persistent launch (refine_kernel)
    RS_LAUNCH(ctx, "dedup_compare_r0", compare_stream_kernel, per_sm * ctx->num_sms,
              kStreamWarps * 32, kStreamSmem, st, kc);
    RS_TRY(launch_refine(ctx, st, kc, bar));
    if (tail) {
      RS_TRY(tail->enqueue(ctx, st, md));  // writes {stats, flags} to pin + kStatsOff
    } else {
      RS_CUDA_TRY(cudaMemcpyAsync(pin + kStatsOff, st.stats, 5 * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (!tail) pin[kStatsOff] = INT64_MAX - pin[kStatsOff];
    if (ctx->timing) RS_TRY(collect_timers(ctx));
    RS_TRY(flags_to_status((int)pin[kStatsOff + 4]));
    std::memcpy(hs, pin + kStatsOff, sizeof(hs));
    if (hs[1] <= maxd) break;
    maxd = hs[1];  // a prompt longer than the bound: rerun with exact arrays
  }
  if (h_stats) std::memcpy(h_stats, hs, sizeof(hs));
  if (tail) tail->finish(ctx);
  if (h_labels && P > 0) RS_TRY(d2h(ctx, h_labels, st.labels, 4ull * P));
  *out_state = st;
  return RS_OK;
}

}  // namespace rs

using namespace rs;

struct rs_prefix_index {
  int32_t batch = 0, min_len = 0, max_len = 0;
  int64_t total = 0;
  // the five tables, stride max_len + 2 (nodes has max_len + 1 entries)
  const int64_t *nodes = nullptr, *scb = nullptr, *stb = nullptr, *lcf = nullptr, *ltf = nullptr;
  std::vector<int64_t> own;  // storage of an index made from host tables
  // storage of a device-built index: the pinned block the tables kernel
  // wrote (zero-copy), returned to the context's pool on free
  std::shared_ptr<rs::PinnedPool> pool;
  void* blk = nullptr;
  size_t blk_cap = 0;
  ~rs_prefix_index() {
    if (blk) pool->give(blk, blk_cap);
  }
  void view(const int64_t* t) {
    const size_t n = (size_t)max_len + 2;
    nodes = t;
    scb = t + n;
    stb = t + 2 * n;
    lcf = t + 3 * n;
    ltf = t + 4 * n;
  }
};

static int build_index_device(rs_ctx* ctx, const int32_t* d_tok, const int64_t* d_off,
                              int32_t P, rs_prefix_index** out) {
  if (P <= 0) return fail(RS_E_VALIDATION, "prefix index needs a non-empty batch");
  // The tables kernel writes the stats (into the context's pinned staging)
  // and the tables (into the index's own pinned block) through mapped host
  // memory before the refinement's single synchronisation: no copy after it.
  struct Tables : RefineTail {
    rs_prefix_index* idx = nullptr;
    int enqueue(rs_ctx* c, const DedupState& st, int cap_md) override {
      const size_t need = 5 * 8 * ((size_t)cap_md + 2);
      if (idx->blk && idx->blk_cap < need) {  // a rerun with a longer bound
        RS_CUDA_TRY(cudaStreamSynchronize(c->stream));
        idx->pool->give(idx->blk, idx->blk_cap);
        idx->blk = nullptr;
      }
      if (!idx->blk) {
        idx->pool = c->pin_pool;
        idx->blk = c->pin_pool->take(need, &idx->blk_cap);
        if (!idx->blk) return fail(RS_E_NOMEM, "pinned allocation failed");
      }
      int64_t* pin = reinterpret_cast<int64_t*>(c->pinned);
      RS_TRY(tables_setup(c));
      RS_LAUNCH(c, "dedup_tables", tables_kernel, kTabCtas, kTabT, kTabSmem, st, -1, cap_md,
                static_cast<int64_t*>(idx->blk), pin + kStatsOff);
      return RS_OK;
    }
    void finish(rs_ctx* c) override {
      const int64_t* stats = reinterpret_cast<const int64_t*>(c->pinned) + kStatsOff;
      idx->min_len = (int32_t)stats[0];
      idx->max_len = (int32_t)stats[1];
      idx->total = stats[2];
      idx->view(static_cast<const int64_t*>(idx->blk));
    }
  } tab;
  std::unique_ptr<rs_prefix_index> idx(new rs_prefix_index());
  idx->batch = P;
  tab.idx = idx.get();
  DedupState st;
  int64_t stats[4];
  RS_TRY(dedup_refine(ctx, d_tok, d_off, P, INT32_MAX, 1, false, 0, &st, stats, nullptr, &tab));
  *out = idx.release();
  return RS_OK;
}

// Copy a host CSR into the context's grow-only input buffer (outside the
// arena, which the refinement re-reserves): no per-call allocation.
struct DeviceCSR {
  int32_t* tok = nullptr;
  int64_t* off = nullptr;
};

static int upload_csr(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets, int32_t count,
                      DeviceCSR* d) {
  if (count < 0) return fail(RS_E_ARG, "negative count");
  if (!offsets) return fail(RS_E_ARG, "offsets is NULL");
  int64_t ntok = offsets[count] - offsets[0];
  if (ntok < 0) return fail(RS_E_VALIDATION, "offsets must be non-decreasing");
  const size_t tok_bytes = abytes(std::max<int64_t>(ntok, 1) + 4, 4);
  const size_t need = tok_bytes + abytes((size_t)count + 1, 8);
  if (need > ctx->in_cap) {
    RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (ctx->in_buf) cudaFree(ctx->in_buf);
    ctx->in_buf = nullptr;
    ctx->in_cap = 0;
    if (cudaMalloc(&ctx->in_buf, need) != cudaSuccess) {
      cudaGetLastError();
      return fail(RS_E_NOMEM, "device CSR allocation failed");
    }
    ctx->in_cap = need;
  }
  d->tok = reinterpret_cast<int32_t*>(ctx->in_buf);
  d->off = reinterpret_cast<int64_t*>(ctx->in_buf + tok_bytes);
  if (ntok) RS_TRY(h2d(ctx, d->tok, tokens + offsets[0], 4ull * ntok));
  if (offsets[0] == 0) {
    RS_TRY(h2d(ctx, d->off, offsets, 8ull * (count + 1)));
  } else {
    std::vector<int64_t> rel(count + 1);
    for (int32_t i = 0; i <= count; ++i) rel[i] = offsets[i] - offsets[0];
    RS_TRY(h2d(ctx, d->off, rel.data(), 8ull * (count + 1)));
    RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // rel is a local
  }
  return RS_OK;
}

__global__ void block_hash_kernel(const int32_t* tok, const int64_t* off, int P, int K,
                                  const int64_t* hash_off, uint64_t* out) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t kMul = 0x9e3779b97f4a7c15ULL;
  const int lanes_per_block = K / 4 < 32 ? K / 4 : 32;  // K in {4..128}
  const int blocks_per_chunk = 128 / K > 0 ? 128 / K : 1;
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < P; i += W) {
    const int32_t* p = tok + off[i];
    const int64_t len = off[i + 1] - off[i];
    uint64_t* o = out + hash_off[i];
    uint64_t h = 0x243f6a8885a308d3ULL;
    int64_t wb = 0;
    for (int64_t c0 = 0; c0 < len; c0 += 128) {
      // lane covers tokens [c0 + 4*lane, +4); its block is (4*lane)/K
      int64_t q = c0 + 4 * lane;
      int blk = (4 * lane) / K;
      int64_t bstart = c0 + (int64_t)blk * K;
      int64_t bend = bstart + K < len ? bstart + K : len;
      uint64_t acc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t pos = q + j;
        if (pos < bend) {
          // exponent = bend - 1 - pos
          uint64_t e = (uint64_t)(bend - 1 - pos), pw = 1, bse = kMul;
          while (e) {
            if (e & 1) pw *= bse;
            bse *= bse;
            e >>= 1;
          }
          acc += ((uint64_t)(uint32_t)p[pos] + 1) * pw;
        }
      }
      // reduce within the lanes of one block
      for (int o2 = 1; o2 < lanes_per_block; o2 <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2);
      uint64_t m = (uint64_t)(bend - bstart);
      uint64_t bh = hash_u64(acc ^ (m << 56));
      int nblk = (int)std::min<int64_t>(blocks_per_chunk, (len - c0 + K - 1) / K);
      for (int b = 0; b < nblk; ++b) {
        uint64_t v = __shfl_sync(0xffffffffu, bh, b * lanes_per_block);
        h = hash_combine(h, v);
        if (lane == 0) o[wb] = h;
        ++wb;
      }
    }
  }
}

extern "C" {

int rs_prefix_index_build(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets,
                          int32_t batch, rs_prefix_index** out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  *out = nullptr;
  if (batch <= 0) return fail(RS_E_VALIDATION, "prefix index needs a non-empty batch");
  for (int32_t i = 0; i < batch; ++i)
    if (offsets[i + 1] - offsets[i] < 1)
      return fail(RS_E_VALIDATION, "prefix index: empty prompt in batch");
  DeviceCSR d;
  RS_TRY(upload_csr(ctx, tokens, offsets, batch, &d));
  return build_index_device(ctx, d.tok, d.off, batch, out);
}

int rs_prefix_index_build_device(rs_ctx* ctx, const int32_t* d_tokens, const int64_t* d_offsets,
                                 int32_t batch, rs_prefix_index** out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  *out = nullptr;
  return build_index_device(ctx, d_tokens, d_offsets, batch, out);
}

int rs_prefix_index_build_device_async(rs_ctx* ctx, const int32_t* d_tokens,
                                       const int64_t* d_offsets, int32_t batch,
                                       int32_t max_len_cap, int64_t* d_tables, int64_t* d_info) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !d_tables || !d_info) return fail(RS_E_ARG, "NULL argument");
  if (batch <= 0) return fail(RS_E_VALIDATION, "prefix index needs a non-empty batch");
  DedupState st;
  int64_t stats[4];
  RS_TRY(dedup_refine(ctx, d_tokens, d_offsets, batch, INT32_MAX, 1, false, max_len_cap, &st,
                      stats, nullptr));
  if (stats[1] > max_len_cap) return fail(RS_E_ARG, "max_len_cap below the longest prompt");
  RS_TRY(tables_setup(ctx));
  RS_LAUNCH(ctx, "dedup_tables", tables_kernel, kTabCtas, kTabT, kTabSmem, st, max_len_cap, max_len_cap, d_tables,
            nullptr);
  int64_t info[5] = {batch, stats[0], stats[1], stats[2], 0};
  RS_TRY(h2d(ctx, d_info, info, sizeof(info)));
  return RS_OK;
}

void rs_prefix_index_free(rs_prefix_index* idx) { delete idx; }

int rs_prefix_index_from_tables(int32_t batch, int32_t min_len, int32_t max_len, int64_t total,
                                const int64_t* nodes, const int64_t* scb, const int64_t* stb,
                                const int64_t* lcf, const int64_t* ltf, rs_prefix_index** out) {
  if (!out || !nodes || !scb || !stb || !lcf || !ltf) return fail(RS_E_ARG, "NULL argument");
  if (max_len < 0) return fail(RS_E_ARG, "max_len must be >= 0");
  auto* idx = new rs_prefix_index();
  idx->batch = batch;
  idx->min_len = min_len;
  idx->max_len = max_len;
  idx->total = total;
  const size_t n = (size_t)max_len + 2;
  idx->own.resize(5 * n);
  int64_t* t = idx->own.data();
  std::memcpy(t, nodes, 8 * (n - 1));
  t[n - 1] = 0;
  std::memcpy(t + n, scb, 8 * n);
  std::memcpy(t + 2 * n, stb, 8 * n);
  std::memcpy(t + 3 * n, lcf, 8 * n);
  std::memcpy(t + 4 * n, ltf, 8 * n);
  idx->view(t);
  *out = idx;
  return RS_OK;
}

int rs_prefix_index_info(const rs_prefix_index* idx, int32_t* batch, int32_t* min_len,
                         int32_t* max_len, int64_t* total) {
  if (!idx) return fail(RS_E_ARG, "index is NULL");
  if (batch) *batch = idx->batch;
  if (min_len) *min_len = idx->min_len;
  if (max_len) *max_len = idx->max_len;
  if (total) *total = idx->total;
  return RS_OK;
}

// dedup.cpp:102-122
int rs_unique_prefix_count(const rs_prefix_index* idx, int32_t l, int64_t* out) {
  if (!idx || !out) return fail(RS_E_ARG, "NULL argument");
  if (l < 1) return fail(RS_E_VALIDATION, "unique_prefix_count: prefix_len must be >= 1");
  int32_t m = std::min(l, idx->max_len);
  *out = idx->nodes[m] + idx->scb[m];
  return RS_OK;
}

int rs_unique_prefix_tokens(const rs_prefix_index* idx, int32_t l, int64_t* out) {
  if (!idx || !out) return fail(RS_E_ARG, "NULL argument");
  if (l < 1) return fail(RS_E_VALIDATION, "unique_prefix_tokens: prefix_len must be >= 1");
  int32_t m = std::min(l, idx->max_len);
  *out = idx->nodes[m] * m + idx->stb[m];
  return RS_OK;
}

int rs_remainder_tokens(const rs_prefix_index* idx, int32_t l, int64_t* out) {
  if (!idx || !out) return fail(RS_E_ARG, "NULL argument");
  if (l < 1) return fail(RS_E_VALIDATION, "remainder_tokens: prefix_len must be >= 1");
  if (l >= idx->max_len) {
    *out = 0;
    return RS_OK;
  }
  *out = idx->ltf[l] - idx->lcf[l] * l;
  return RS_OK;
}

int rs_prefix_index_tables(const rs_prefix_index* idx, int64_t* nodes, int64_t* scb,
                           int64_t* stb, int64_t* lcf, int64_t* ltf) {
  if (!idx) return fail(RS_E_ARG, "index is NULL");
  const size_t n = (size_t)idx->max_len + 2;
  if (nodes) std::memcpy(nodes, idx->nodes, 8 * (n - 1));
  if (scb) std::memcpy(scb, idx->scb, 8 * n);
  if (stb) std::memcpy(stb, idx->stb, 8 * n);
  if (lcf) std::memcpy(lcf, idx->lcf, 8 * n);
  if (ltf) std::memcpy(ltf, idx->ltf, 8 * n);
  return RS_OK;
}

// dedup.cpp:124-144
int rs_select_prefix_length(const rs_prefix_index* idx, int32_t cap, int32_t gpu_count,
                            int32_t l_min, int32_t l_max, int32_t* len, int32_t* exceeded) {
  (void)gpu_count;  // PrefillCapacity::gpu_count does not enter the math
  if (!idx || !len || !exceeded) return fail(RS_E_ARG, "NULL argument");
  if (l_min < 1 || l_min > l_max)
    return fail(RS_E_VALIDATION, "select_prefix_length: need 1 <= l_min <= l_max");
  if (cap < 1) return fail(RS_E_CONFIG, "prefill capacity must allow at least one prefix");
  int64_t d;
  RS_TRY(rs_unique_prefix_count(idx, l_min, &d));
  if (d > cap) {
    *len = l_min;
    *exceeded = 1;
    return RS_OK;
  }
  int32_t lo = l_min, hi = l_max;
  while (lo < hi) {
    int32_t mid = lo + (hi - lo + 1) / 2;
    RS_TRY(rs_unique_prefix_count(idx, mid, &d));
    if (d <= cap) lo = mid; else hi = mid - 1;
  }
  *len = lo;
  *exceeded = 0;
  return RS_OK;
}

// dedup.cpp:146-161
int rs_dedup_savings(const rs_prefix_index* idx, int32_t l_star, int32_t g, int64_t* raw,
                     int64_t* dedup, double* frac) {
  if (!idx || !raw || !dedup || !frac) return fail(RS_E_ARG, "NULL argument");
  if (g < 1) return fail(RS_E_VALIDATION, "dedup_savings: responses_per_prompt must be >= 1");
  int64_t r = idx->total * (int64_t)g;
  int64_t ut, rem;
  RS_TRY(rs_unique_prefix_tokens(idx, l_star, &ut));
  RS_TRY(rs_remainder_tokens(idx, l_star, &rem));
  *raw = r;
  *dedup = ut + rem;
  *frac = r == 0 ? 0.0 : (double)(r - *dedup) / (double)r;
  return RS_OK;
}

int rs_unique_prefix_count_among(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets,
                                 int32_t count, int32_t prefix_len, int64_t* out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  if (prefix_len < 1)
    return fail(RS_E_VALIDATION, "unique_prefix_count_among: prefix_len must be >= 1");
  if (count <= 0) {
    *out = 0;
    return RS_OK;
  }
  DeviceCSR d;
  RS_TRY(upload_csr(ctx, tokens, offsets, count, &d));
  DedupState st;
  int64_t stats[4];
  RS_TRY(dedup_refine(ctx, d.tok, d.off, count, prefix_len, 0, false, prefix_len, &st, stats,
                      nullptr));  // synchronised, its own status checked
  *out = stats[3];
  return RS_OK;
}

int rs_dedup_map(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets, int32_t count,
                 int32_t prefix_len, int32_t* labels) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !labels) return fail(RS_E_ARG, "NULL argument");
  if (prefix_len < 1) return fail(RS_E_VALIDATION, "dedup_map: prefix_len must be >= 1");
  if (count <= 0) return RS_OK;
  DeviceCSR d;
  RS_TRY(upload_csr(ctx, tokens, offsets, count, &d));
  DedupState st;
  int64_t stats[4];
  return dedup_refine(ctx, d.tok, d.off, count, prefix_len, 0, true, prefix_len, &st, stats,
                      labels);  // synchronised (labels read back), its own status checked
}

int rs_block_hashes(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets, int32_t count,
                    int32_t K, uint64_t* hashes) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !hashes) return fail(RS_E_ARG, "NULL argument");
  if (K < 4 || K > 128 || (K & (K - 1)))
    return fail(RS_E_CONFIG, "block_hashes: block_tokens must be a power of two in [4, 128]");
  if (count <= 0) return RS_OK;
  std::vector<int64_t> hoff(count + 1, 0);
  for (int32_t i = 0; i < count; ++i) {
    int64_t len = offsets[i + 1] - offsets[i];
    if (len < 0) return fail(RS_E_VALIDATION, "offsets must be non-decreasing");
    hoff[i + 1] = hoff[i] + (len + K - 1) / K;
  }
  DeviceCSR d;
  RS_TRY(upload_csr(ctx, tokens, offsets, count, &d));
  RS_TRY(clear_flags(ctx));
  const int64_t nh = hoff[count];
  RS_TRY(arena_reserve(ctx, abytes(count + 1, 8) + abytes(std::max<int64_t>(nh, 1), 8) + 4096));
  int64_t* dho = arena_alloc<int64_t>(ctx, count + 1);
  uint64_t* dh = arena_alloc<uint64_t>(ctx, std::max<int64_t>(nh, 1));
  RS_TRY(h2d(ctx, dho, hoff.data(), 8ull * (count + 1)));
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)count + 7) / 8, 16 * ctx->num_sms));
  RS_LAUNCH(ctx, "block_hashes", block_hash_kernel, blocks, 256, 0, d.tok, d.off, count, K, dho, dh);
  if (nh) RS_TRY(d2h(ctx, hashes, dh, 8ull * nh));
  return sync_and_check(ctx);
}

}  // extern "C"
