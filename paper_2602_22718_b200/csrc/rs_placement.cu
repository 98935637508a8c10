// rs_placement.cu — the placement penalty plan_rlhfless folds into scale()
// (proj/src/training.cpp:150-164), evaluated for every candidate N on the
// device.
//
// Reference semantics, per candidate (placement.cpp:177-291, 339-363):
//   * the heaviest group (first maximum of the estimated times) is placed
//     first, on the learner node when it has room (co-located: no transfer);
//   * the others follow in (time desc, group index asc) order, each on the
//     first node of the bandwidth ranking (bandwidth to the learner desc,
//     index asc) with enough free GPUs;
//   * slack_i = (l_prefill + T_heaviest) - (model/bw_i + kv_i/bw_i + T_i),
//     kv_i = kv_bytes_per_token * (sum of the group's prompt lengths)
//     (transfers_for, training.cpp:68-80); penalty = max(0, max_i -slack_i).
// Every actor of a scale() candidate needs the same gpus_per_actor GPUs, so
// which node the j-th placed actor lands on depends only on j: the host
// replays the first-fit once into per-slot bandwidths, and the device only
// has to rank each group's time among its candidate's groups.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "rs_placement.cuh"

namespace rs {

namespace {

double node_bw(const rs_topology& t, int a, int b) {
  if (t.bw_matrix) return t.bw_matrix[(size_t)a * t.n_nodes + b];
  return a == b ? t.intra_node_bw : t.inter_node_bw;
}

// ClusterTopology::validate (placement.cpp:28-62), same checks and order.
int validate_topology(const rs_topology& t) {
  if (t.n_nodes < 1 || !t.node_gpus) return fail(RS_E_CONFIG, "topology needs at least one node");
  for (int i = 0; i < t.n_nodes; ++i)
    if (t.node_gpus[i] < 1) return fail(RS_E_CONFIG, "every node needs at least one GPU");
  if (!t.bw_matrix) {
    if (!(t.intra_node_bw > 0) || !(t.inter_node_bw > 0))
      return fail(RS_E_CONFIG, "bandwidths must be positive");
    if (t.intra_node_bw < t.inter_node_bw)
      return fail(RS_E_CONFIG, "intra-node bandwidth below inter-node bandwidth");
  } else {
    for (int i = 0; i < t.n_nodes; ++i)
      for (int j = 0; j < t.n_nodes; ++j) {
        const double v = t.bw_matrix[(size_t)i * t.n_nodes + j];
        if (!(v > 0)) return fail(RS_E_CONFIG, "bandwidth matrix entries must be positive");
        if (v != t.bw_matrix[(size_t)j * t.n_nodes + i])
          return fail(RS_E_CONFIG, "bandwidth matrix must be symmetric");
      }
  }
  if (t.learner_node < 0 || t.learner_node >= t.n_nodes)
    return fail(RS_E_CONFIG, "learner_node out of range");
  if (t.n_learner_gpus < 1 || !t.learner_gpus)
    return fail(RS_E_CONFIG, "learner needs at least one GPU");
  for (int k = 0; k < t.n_learner_gpus; ++k)
    if (t.learner_gpus[k] < 0 || t.learner_gpus[k] >= t.node_gpus[t.learner_node])
      return fail(RS_E_CONFIG, "learner GPU index out of range");
  return RS_OK;
}

}  // namespace

int placement_slots(const rs_placement_penalty* pen, int gpus_per_actor, int n_max,
                    PlacementSlots* out) {
  if (!pen || !pen->topology) return fail(RS_E_ARG, "NULL placement penalty / topology");
  const rs_topology& t = *pen->topology;
  RS_TRY(validate_topology(t));
  // validate_transfers (placement.cpp:150-160)
  if (!(pen->model_bytes >= 0) || !std::isfinite(pen->model_bytes))
    return fail(RS_E_CONFIG, "model_bytes must be finite and >= 0");
  if (!(pen->kv_bytes_per_token >= 0) || !std::isfinite(pen->kv_bytes_per_token))
    return fail(RS_E_CONFIG, "kv bytes must be finite and >= 0");
  std::vector<int> rank(t.n_nodes);
  std::iota(rank.begin(), rank.end(), 0);
  std::sort(rank.begin(), rank.end(), [&](int a, int b) {
    const double ba = node_bw(t, a, t.learner_node), bb = node_bw(t, b, t.learner_node);
    if (ba != bb) return ba > bb;
    return a < b;
  });
  std::vector<int> free_gpus(t.node_gpus, t.node_gpus + t.n_nodes);
  out->model_over_bw.assign(n_max, 0.0);
  out->bw.assign(n_max, 1.0);
  out->n_placeable = 0;
  for (int j = 0; j < n_max; ++j) {
    int node = -1;
    if (j == 0 && free_gpus[t.learner_node] >= gpus_per_actor) {
      node = t.learner_node;  // co-located: no model sync, no KV shipping
    } else {
      for (int nd : rank)
        if (free_gpus[nd] >= gpus_per_actor) {
          node = nd;
          break;
        }
    }
    if (node < 0) break;
    free_gpus[node] -= gpus_per_actor;
    const double bw = node_bw(t, node, t.learner_node);
    out->bw[j] = bw;
    out->model_over_bw[j] = pen->model_bytes / bw;
    out->n_placeable = j + 1;
  }
  return RS_OK;
}

// Exclusive prefix sums of the rank-ordered prompt lengths (one CTA).
__global__ void plen_prefix_kernel(const int32_t* plen_r, int64_t n, int64_t* cum) {
  __shared__ long long part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo = min(n, tid * per), hi = min(n, lo + per);
  long long s = 0;
  for (int64_t i = lo; i < hi; ++i) s += plen_r[i];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    long long run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const long long v = part[i];
      part[i] = run;
      run += v;
    }
    cum[n] = run;
  }
  __syncthreads();
  long long run = part[tid];
  for (int64_t i = lo; i < hi; ++i) {
    cum[i] = run;
    run += plen_r[i];
  }
}

constexpr int kPenT = 256;

// One CTA per candidate N. gt holds the candidate's N group times (group
// order), groups are the contiguous rank chunks of assign()
// (planner.cpp:33-49).
__global__ void __launch_bounds__(kPenT)
placement_penalty_kernel(const double* gt, int n_min, int64_t P, const int64_t* cum,
                         const double* model_over_bw, const double* bw, double kvpt,
                         double l_prefill, double* tp) {
  extern __shared__ double s_t[];
  __shared__ double s_v[kPenT / 32];
  __shared__ int s_i[kPenT / 32];
  const int N = n_min + blockIdx.x;
  const double* t = gt + ((int64_t)N * (N - 1) / 2 - (int64_t)n_min * (n_min - 1) / 2);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int g = tid; g < N; g += kPenT) s_t[g] = t[g];
  __syncthreads();
  // heaviest = first maximum (placement.cpp:193-197)
  double bv = -INFINITY;
  int bi = INT32_MAX;
  for (int g = tid; g < N; g += kPenT) {
    const double v = s_t[g];
    if (v > bv || bi == INT32_MAX) {
      bv = v;
      bi = g;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi != INT32_MAX && (bi == INT32_MAX || ov > bv || (ov == bv && oi < bi))) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_v[wid] = bv;
    s_i[wid] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kPenT / 32; ++w)
      if (s_i[w] != INT32_MAX && (bi == INT32_MAX || s_v[w] > bv || (s_v[w] == bv && s_i[w] < bi))) {
        bv = s_v[w];
        bi = s_i[w];
      }
    s_i[0] = bi;
  }
  __syncthreads();
  const int h = s_i[0];
  const double left = dadd(l_prefill, s_t[h]);
  const int64_t q = P / N, rem = P % N;
  double exposed = 0.0;  // std::max(exposed, -slack) from 0 (training.cpp:160-162)
  for (int g = tid; g < N; g += kPenT) {
    if (g == h) continue;
    const double tg = s_t[g];
    int r = 0;  // position among the non-heaviest: (time desc, index asc)
    for (int j = 0; j < N; ++j) {
      const double tj = s_t[j];
      r += (j != h && (tj > tg || (tj == tg && j < g))) ? 1 : 0;
    }
    const int slot = r + 1;
    const int64_t a = g * q + min((int64_t)g, rem), b = a + q + (g < rem ? 1 : 0);
    const double l_kv = ddiv(dmul((double)(cum[b] - cum[a]), kvpt), bw[slot]);
    const double x = dadd(dadd(model_over_bw[slot], l_kv), tg);
    const double v = -dsub(left, x);
    if (exposed < v) exposed = v;
  }
  // max with the same "replace only when strictly greater" rule
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, exposed, o);
    if (exposed < ov) exposed = ov;
  }
  __syncthreads();
  if (lane == 0) s_v[wid] = exposed;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kPenT / 32; ++w)
      if (exposed < s_v[w]) exposed = s_v[w];
    tp[blockIdx.x] = exposed;
  }
}

int placement_penalties(rs_ctx* ctx, const double* gt, const int32_t* plen_r, int64_t P,
                        int n_min, int n_max, const PlacementSlots& slots,
                        const rs_placement_penalty* pen, double* tp) {
  const int C = n_max - n_min + 1;
  int64_t* cum = arena_alloc<int64_t>(ctx, P + 1);
  double* d_lm = arena_alloc<double>(ctx, n_max);
  double* d_bw = arena_alloc<double>(ctx, n_max);
  if (!cum || !d_lm || !d_bw) return fail(RS_E_NOMEM, "arena exhausted (placement)");
  RS_TRY(h2d(ctx, d_lm, slots.model_over_bw.data(), 8 * (size_t)n_max));
  RS_TRY(h2d(ctx, d_bw, slots.bw.data(), 8 * (size_t)n_max));
  RS_LAUNCH(ctx, "plen_prefix", plen_prefix_kernel, 1, 1024, 0, plen_r, P, cum);
  RS_LAUNCH(ctx, "placement_penalty", placement_penalty_kernel, C, kPenT,
            sizeof(double) * n_max, gt, n_min, P, cum, d_lm, d_bw, pen->kv_bytes_per_token,
            pen->l_prefill_seconds, tp);
  return RS_OK;
}

size_t placement_bytes(int64_t P, int n_max) {
  return abytes(P + 1, 8) + 2 * abytes(n_max, 8);
}

}  // namespace rs
