// rs_sort.cuh — device sort / scan primitives shared by the planner paths.
#pragma once
#include "rs_internal.cuh"

namespace rs {

// Scratch bytes radix_sort_pairs needs for n items.
size_t radix_sort_scratch_bytes64(int64_t n);

// Stable ascending sort of (keys, vals) on ctx->stream. The result lives in
// *out_keys / *out_vals, which are either the inputs or buffers inside
// `scratch`. Performs one host sync (to skip constant digit passes).
int radix_sort_pairs(rs_ctx* ctx, uint64_t* keys, uint32_t* vals, int64_t n,
                     char* scratch, uint64_t** out_keys, uint32_t** out_vals);

// Multi-CTA exclusive scan on ctx->stream (in == out allowed); *total
// (device, nullable) gets the sum. scratch: scan_scratch_bytes(n, sizeof(T)).
size_t scan_scratch_bytes(int64_t n, size_t elem);
template <class T>
int exclusive_scan(rs_ctx* ctx, const T* in, T* out, int64_t n, T* scratch, T* total);

// Single-CTA exclusive scan (launch with <<<1, 1024>>>).
__global__ void exclusive_scan_u32_kernel(const uint32_t* in, uint32_t* out,
                                          int64_t n);

}  // namespace rs
