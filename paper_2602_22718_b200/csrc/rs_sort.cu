// rs_sort.cu — stable LSD radix sort of (u64 key, u32 value) pairs and a
// single-CTA exclusive scan, used by the generic (unbounded-key) planner
// paths. 8-bit digits, 4096-item tiles; digit passes whose 8 bits do not
// vary across the input are skipped (one AND/OR reduction decides).
#include <algorithm>

#include "rs_sort.cuh"

namespace rs {

namespace {

constexpr int kSortThreads = 256;
constexpr int kItemsPerThread = 16;
constexpr int kTile = kSortThreads * kItemsPerThread;  // 4096
constexpr int kWarpsPerTile = kSortThreads / 32;
constexpr int kItemsPerWarp = kTile / kWarpsPerTile;    // 512

__global__ void key_bits_kernel(const uint64_t* keys, int64_t n,
                                unsigned long long* and_or) {
  uint64_t a = ~0ULL, o = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    a &= k;
    o |= k;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a &= __shfl_xor_sync(0xffffffffu, a, off);
    o |= __shfl_xor_sync(0xffffffffu, o, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAnd(&and_or[0], (unsigned long long)a);
    atomicOr(&and_or[1], (unsigned long long)o);
  }
}

__global__ void __launch_bounds__(kSortThreads)
radix_hist_kernel(const uint64_t* keys, int64_t n, int shift, uint32_t* hist,
                  int ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kTile;
  for (int j = 0; j < kItemsPerThread; ++j) {
    int64_t i = base + j * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
radix_scatter_kernel(const uint64_t* kin, const uint32_t* vin, uint64_t* kout,
                     uint32_t* vout, int64_t n, int shift, const uint32_t* offs,
                     int ntiles) {
  __shared__ uint32_t wcnt[kWarpsPerTile][256];
  __shared__ uint32_t woff[kWarpsPerTile][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) wcnt[w][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * kItemsPerWarp;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint64_t key[kItemsPerThread];
  uint32_t val[kItemsPerThread];
  uint32_t pos[kItemsPerThread];
#pragma unroll
  for (int j = 0; j < kItemsPerThread; ++j) {
    int64_t i = base + j * 32 + lane;
    bool valid = i < n;
    key[j] = valid ? kin[i] : 0;
    val[j] = valid ? vin[i] : 0;
    uint32_t d = valid ? (uint32_t)((key[j] >> shift) & 255) : 256u + lane;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t rank = __popc(peers & lt_mask);
    uint32_t cnt = valid ? wcnt[w][d] : 0;
    pos[j] = cnt + rank;
    __syncwarp();
    if (valid && rank == 0) wcnt[w][d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    int d = threadIdx.x;  // 256 threads == 256 digits
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kWarpsPerTile; ++ww) {
      woff[ww][d] = run;
      run += wcnt[ww][d];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItemsPerThread; ++j) {
    int64_t i = base + j * 32 + lane;
    if (i < n) {
      uint32_t d = (uint32_t)((key[j] >> shift) & 255);
      int64_t dst = (int64_t)offs[(int64_t)d * ntiles + blockIdx.x] + woff[w][d] + pos[j];
      kout[dst] = key[j];
      vout[dst] = val[j];
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(1024)
exclusive_scan_u32_kernel(const uint32_t* in, uint32_t* out, int64_t n) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t t0 = 0; t0 < n; t0 += 1024) {
    int64_t i = t0 + threadIdx.x;
    uint32_t v = i < n ? in[i] : 0;
    uint32_t incl = warp_incl_sum(v);
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      uint32_t x = wsum[lane];
      uint32_t xi = warp_incl_sum(x);
      wsum[lane] = xi - x;
    }
    __syncthreads();
    uint32_t carry = carry_s;
    if (i < n) out[i] = carry + wsum[w] + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry_s = carry + wsum[w] + incl;
    __syncthreads();
  }
}

// ------------------------------------------------------ multi-CTA scan --
// Three launches: per-tile sums, one CTA scanning the tile sums (and the
// total), per-tile scans with the tile base. 512 threads x 8 items per tile.
namespace {
constexpr int kScanT = 512;
constexpr int kScanIPT = 8;
constexpr int64_t kScanTile = kScanT * kScanIPT;

template <class T>
__device__ __forceinline__ T block_excl_sum(T v, T* wsum, T* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T incl = warp_incl_sum(v);
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    const T x = lane < kScanT / 32 ? wsum[lane] : T(0);
    const T xi = warp_incl_sum(x);
    if (lane < kScanT / 32) wsum[lane] = xi - x;
    if (lane == 31) *total = xi;
  }
  __syncthreads();
  return wsum[w] + incl - v;
}

template <class T>
__global__ void __launch_bounds__(kScanT) scan_reduce_kernel(const T* in, int64_t n, T* part) {
  __shared__ T wsum[kScanT / 32];
  __shared__ T tot;
  const int64_t b = blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIPT;
  T v = 0;
#pragma unroll
  for (int j = 0; j < kScanIPT; ++j)
    if (b + j < n) v += in[b + j];
  block_excl_sum(v, wsum, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

template <class T>
__global__ void __launch_bounds__(kScanT) scan_partials_kernel(T* part, int64_t nt, T* total) {
  __shared__ T wsum[kScanT / 32];
  __shared__ T tot;
  T carry = 0;
  for (int64_t t0 = 0; t0 < nt; t0 += kScanT) {
    const int64_t i = t0 + threadIdx.x;
    const T v = i < nt ? part[i] : T(0);
    const T ex = block_excl_sum(v, wsum, &tot);
    if (i < nt) part[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

template <class T>
__global__ void __launch_bounds__(kScanT) scan_apply_kernel(const T* in, T* out, int64_t n, const T* part) {
  __shared__ T wsum[kScanT / 32];
  __shared__ T tot;
  const int64_t b = blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIPT;
  T x[kScanIPT];
  T v = 0;
#pragma unroll
  for (int j = 0; j < kScanIPT; ++j) {
    x[j] = b + j < n ? in[b + j] : T(0);
    v += x[j];
  }
  T run = part[blockIdx.x] + block_excl_sum(v, wsum, &tot);
#pragma unroll
  for (int j = 0; j < kScanIPT; ++j)
    if (b + j < n) {
      out[b + j] = run;
      run += x[j];
    }
}
}  // namespace

size_t scan_scratch_bytes(int64_t n, size_t elem) {
  return abytes((n + kScanTile - 1) / kScanTile + 1, elem);
}

template <class T>
int exclusive_scan(rs_ctx* ctx, const T* in, T* out, int64_t n, T* scratch, T* total) {
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  if (nt == 0) {
    if (total) RS_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(T), ctx->stream));
    return RS_OK;
  }
  RS_LAUNCH(ctx, "scan_reduce", scan_reduce_kernel<T>, (int)nt, kScanT, 0, in, n, scratch);
  RS_LAUNCH(ctx, "scan_partials", scan_partials_kernel<T>, 1, kScanT, 0, scratch, nt, total);
  RS_LAUNCH(ctx, "scan_apply", scan_apply_kernel<T>, (int)nt, kScanT, 0, in, out, n, scratch);
  return RS_OK;
}

template int exclusive_scan<uint32_t>(rs_ctx*, const uint32_t*, uint32_t*, int64_t, uint32_t*, uint32_t*);
template int exclusive_scan<unsigned long long>(rs_ctx*, const unsigned long long*, unsigned long long*,
                                                int64_t, unsigned long long*, unsigned long long*);

size_t radix_sort_scratch_bytes64(int64_t n) {
  int64_t ntiles = (n + kTile - 1) / kTile;
  return abytes(n, 8) + abytes(n, 4) + abytes(256 * ntiles, 4) * 2 + abytes(2, 8) +
         scan_scratch_bytes(256 * ntiles, 4);
}

int radix_sort_pairs(rs_ctx* ctx, uint64_t* keys, uint32_t* vals, int64_t n,
                     char* scratch, uint64_t** out_keys, uint32_t** out_vals) {
  *out_keys = keys;
  *out_vals = vals;
  if (n <= 1) return RS_OK;
  int64_t ntiles = (n + kTile - 1) / kTile;
  char* q = scratch;
  uint64_t* k2 = (uint64_t*)q; q += abytes(n, 8);
  uint32_t* v2 = (uint32_t*)q; q += abytes(n, 4);
  uint32_t* hist = (uint32_t*)q; q += abytes(256 * ntiles, 4);
  uint32_t* offs = (uint32_t*)q; q += abytes(256 * ntiles, 4);
  unsigned long long* ao = (unsigned long long*)q; q += abytes(2, 8);
  uint32_t* scan_part = (uint32_t*)q;
  unsigned long long init[2] = {~0ULL, 0ULL};
  RS_CUDA_TRY(cudaMemcpyAsync(ao, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 4 * ctx->num_sms);
  RS_LAUNCH(ctx, "radix_keybits", key_bits_kernel, blocks, 256, 0, keys, n, ao);
  unsigned long long hb[2];
  RS_CUDA_TRY(cudaMemcpyAsync(hb, ao, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  uint64_t vary = hb[0] ^ hb[1];
  uint64_t* kin = keys;
  uint32_t* vin = vals;
  uint64_t* kout = k2;
  uint32_t* vout = v2;
  for (int shift = 0; shift < 64; shift += 8) {
    if (((vary >> shift) & 255) == 0) continue;
    RS_LAUNCH(ctx, "radix_hist", radix_hist_kernel, (int)ntiles, kSortThreads, 0,
              kin, n, shift, hist, (int)ntiles);
    if (ntiles >= 64) {  // one CTA would walk 256 x ntiles counts alone
      RS_TRY(exclusive_scan<uint32_t>(ctx, hist, offs, 256 * ntiles, scan_part, nullptr));
    } else {
      RS_LAUNCH(ctx, "radix_scan", exclusive_scan_u32_kernel, 1, 1024, 0, hist,
                offs, (int64_t)256 * ntiles);
    }
    RS_LAUNCH(ctx, "radix_scatter", radix_scatter_kernel, (int)ntiles,
              kSortThreads, 0, kin, vin, kout, vout, n, shift, offs, (int)ntiles);
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  *out_keys = kin;
  *out_vals = vin;
  return RS_OK;
}

}  // namespace rs
