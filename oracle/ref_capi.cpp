// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// Plain-C wrapper over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests and bench.py call the reference's own PrefixIndex::build,
// select_prefix_length, dedup_savings, unique_prefix_count_among, assign,
// integrate_decode_seconds, estimate_actor_time, estimate_cost and scale on
// the same SoA/CSR inputs the C-ABI (include/rs.h) takes. No algorithm lives
// here: every number is produced by the reference code.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "oracle.h"
#include "rollsim/dedup.hpp"
#include "rollsim/errors.hpp"
#include <nlohmann/json.hpp>

#include "rollsim/placement.hpp"
#include "rollsim/predictor.hpp"
#include "rollsim/planner.hpp"
#include "rollsim/profile.hpp"
#include "rollsim/workload.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const rollsim::ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const rollsim::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const rollsim::PlacementError& e) {
    g_err = e.what();
    return 6;
  } catch (const rollsim::ParseError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

rollsim::LatencyProfile to_profile(const rs_profile* p) {
  rollsim::LatencyProfile lp;
  lp.batch_knots.assign(p->batch_knots, p->batch_knots + p->nb);
  lp.context_knots.assign(p->context_knots, p->context_knots + p->nc);
  lp.tpot_grid.resize(p->nb);
  for (int i = 0; i < p->nb; ++i)
    lp.tpot_grid[i].assign(p->tpot_grid + (size_t)i * p->nc,
                           p->tpot_grid + (size_t)(i + 1) * p->nc);
  lp.prefill_token_knots = {1, 1e9};
  lp.prefill_seconds_knots = {1e-4, 1e5};
  lp.rho = p->rho;
  lp.gpus_per_actor = 1;
  return lp;
}

std::vector<rollsim::Prompt> to_prompts(const int32_t* tok, const int64_t* off,
                                        int32_t n) {
  std::vector<rollsim::Prompt> ps(n > 0 ? n : 0);
  for (int32_t i = 0; i < n; ++i) {
    ps[i].id = "q" + std::to_string(i);
    ps[i].token_ids.assign(tok + off[i], tok + off[i + 1]);
  }
  return ps;
}

std::vector<const rollsim::Prompt*> ptrs(const std::vector<rollsim::Prompt>& ps) {
  std::vector<const rollsim::Prompt*> out;
  out.reserve(ps.size());
  for (const auto& p : ps) out.push_back(&p);
  return out;
}

// Ids whose std::string order equals id_rank order.
std::string rank_id(int32_t r) {
  char buf[24];
  std::snprintf(buf, sizeof(buf), "r%010d", r);
  return buf;
}

std::vector<rollsim::PredictedPrompt> to_predicted(const double* pred,
                                                   const int32_t* plen,
                                                   const int32_t* id_rank,
                                                   int32_t count) {
  std::vector<rollsim::PredictedPrompt> v(count > 0 ? count : 0);
  for (int32_t i = 0; i < count; ++i) {
    v[i].id = rank_id(id_rank ? id_rank[i] : i);
    v[i].prompt_len = plen ? plen[i] : 0;
    v[i].predicted_len = pred[i];
  }
  return v;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_tpot_seconds(const rs_profile* p, const double* b, const double* c,
                     int64_t n, double* out) {
  return guarded([&] {
    rollsim::LatencyProfile lp = to_profile(p);
    for (int64_t i = 0; i < n; ++i) out[i] = lp.tpot_seconds(b[i], c[i]);
  });
}

int ref_prefix_curves(const int32_t* tok, const int64_t* off, int32_t batch,
                      int32_t n_l, int64_t* info, int64_t* ucount,
                      int64_t* utokens, int64_t* rem) {
  return guarded([&] {
    auto ps = to_prompts(tok, off, batch);
    rollsim::PrefixIndex idx = rollsim::PrefixIndex::build(ptrs(ps));
    info[0] = idx.batch_size();
    info[1] = idx.min_prompt_len();
    info[2] = idx.max_prompt_len();
    info[3] = idx.total_prompt_tokens();
    for (int32_t l = 1; l <= n_l; ++l) {
      ucount[l - 1] = idx.unique_prefix_count(l);
      utokens[l - 1] = idx.unique_prefix_tokens(l);
      rem[l - 1] = idx.remainder_tokens(l);
    }
  });
}

int ref_select_prefix_length(const int32_t* tok, const int64_t* off,
                             int32_t batch, int32_t cap, int32_t gpus,
                             int32_t l_min, int32_t l_max, int32_t* len,
                             int32_t* exceeded) {
  return guarded([&] {
    auto ps = to_prompts(tok, off, batch);
    rollsim::PrefixIndex idx = rollsim::PrefixIndex::build(ptrs(ps));
    rollsim::PrefixSelection s =
        rollsim::select_prefix_length(idx, {cap, gpus}, l_min, l_max);
    *len = s.prefix_len;
    *exceeded = s.capacity_exceeded ? 1 : 0;
  });
}

int ref_dedup_savings(const int32_t* tok, const int64_t* off, int32_t batch,
                      int32_t l_star, int32_t g, int64_t* raw, int64_t* dedup,
                      double* frac) {
  return guarded([&] {
    auto ps = to_prompts(tok, off, batch);
    rollsim::PrefixIndex idx = rollsim::PrefixIndex::build(ptrs(ps));
    rollsim::DedupSavings s = rollsim::dedup_savings(idx, l_star, g);
    *raw = s.raw_prefill_tokens;
    *dedup = s.dedup_prefill_tokens;
    *frac = s.saved_fraction;
  });
}

int ref_unique_prefix_count_among(const int32_t* tok, const int64_t* off,
                                  int32_t count, int32_t len, int64_t* out) {
  return guarded([&] {
    auto ps = to_prompts(tok, off, count);
    *out = rollsim::unique_prefix_count_among(ptrs(ps), len);
  });
}

int ref_assign(const double* pred, const int32_t* id_rank, int32_t count,
               int32_t n_actors, int32_t* order, int32_t* group_offsets) {
  return guarded([&] {
    auto v = to_predicted(pred, nullptr, id_rank, count);
    for (int32_t i = 0; i < count; ++i) v[i].prompt_len = i;  // carry index
    auto groups = rollsim::assign(v, n_actors, 1);
    int32_t pos = 0;
    for (size_t g = 0; g < groups.size(); ++g) {
      group_offsets[g] = pos;
      for (int idx : groups[g].prompt_lens) order[pos++] = idx;
    }
    group_offsets[groups.size()] = pos;
  });
}

int ref_integrate_decode_seconds(const int32_t* plen, const double* target,
                                 int64_t count, const rs_profile* p,
                                 double* out) {
  return guarded([&] {
    std::vector<rollsim::ResponseSpec> rs(count > 0 ? count : 0);
    for (int64_t i = 0; i < count; ++i) rs[i] = {plen[i], target[i]};
    *out = rollsim::integrate_decode_seconds(std::move(rs), to_profile(p));
  });
}

int ref_estimate_actor_time(const int32_t* plen, const double* pred,
                            int32_t count, const rs_profile* p, int32_t g,
                            double* out) {
  return guarded([&] {
    rollsim::ActorGroup grp;
    for (int32_t i = 0; i < count; ++i) {
      grp.prompt_ids.push_back(rank_id(i));
      grp.prompt_lens.push_back(plen[i]);
      grp.predicted_lengths.push_back(pred[i]);
    }
    *out = rollsim::estimate_actor_time(grp, to_profile(p), g);
  });
}

int ref_estimate_cost(const int32_t* plen, const double* pred,
                      const int32_t* group_offsets, const int32_t* gpu_count,
                      int32_t n_groups, const rs_profile* p, int32_t g,
                      double* cost, double* times) {
  return guarded([&] {
    rollsim::LatencyProfile lp = to_profile(p);
    std::vector<rollsim::ActorGroup> groups(n_groups);
    for (int32_t k = 0; k < n_groups; ++k) {
      groups[k].actor_id = k;
      groups[k].gpu_count = gpu_count[k];
      for (int32_t i = group_offsets[k]; i < group_offsets[k + 1]; ++i) {
        groups[k].prompt_ids.push_back(rank_id(i));
        groups[k].prompt_lens.push_back(plen[i]);
        groups[k].predicted_lengths.push_back(pred[i]);
      }
    }
    *cost = rollsim::estimate_cost(groups, lp, g);
    if (times)
      for (int32_t k = 0; k < n_groups; ++k)
        times[k] = rollsim::estimate_actor_time(groups[k], lp, g);
  });
}

int ref_scale(const double* pred, const int32_t* plen, const int32_t* id_rank,
              int32_t count, const rs_profile* p, int32_t g, int32_t n_min,
              int32_t n_max, double lambda, int32_t gpus,
              const double* t_penalty, int32_t* n_star, double* t_total,
              double* t_pen_out, double* cost, double* t_norm, double* c_norm,
              double* score, int32_t* order, double* actor_times) {
  return guarded([&] {
    auto v = to_predicted(pred, plen, id_rank, count);
    rollsim::TimePenaltyFn pen = nullptr;
    if (t_penalty)
      pen = [&](int n, const std::vector<rollsim::ActorGroup>&,
                const std::vector<double>&) { return t_penalty[n - n_min]; };
    rollsim::ScaleResult r =
        rollsim::scale(v, to_profile(p), g, n_min, n_max, lambda, gpus, pen);
    *n_star = r.n_star;
    for (size_t i = 0; i < r.candidates.size(); ++i) {
      const auto& c = r.candidates[i];
      if (t_total) t_total[i] = c.t_total;
      if (t_pen_out) t_pen_out[i] = c.t_penalty;
      if (cost) cost[i] = c.cost;
      if (t_norm) t_norm[i] = c.t_norm;
      if (c_norm) c_norm[i] = c.c_norm;
      if (score) score[i] = c.score;
    }
    if (actor_times)
      for (size_t i = 0; i < r.actor_times.size(); ++i)
        actor_times[i] = r.actor_times[i];
    if (order) {
      // Map rank ids back to input indices.
      std::vector<int32_t> by_rank;
      if (id_rank) {
        by_rank.assign(count, 0);
        for (int32_t i = 0; i < count; ++i) by_rank[id_rank[i]] = i;
      }
      int32_t pos = 0;
      for (const auto& grp : r.groups)
        for (const std::string& id : grp.prompt_ids) {
          int32_t rk = std::stoi(id.substr(1));
          order[pos++] = id_rank ? by_rank[rk] : rk;
        }
    }
  });
}

// plan_rlhfless's penalty (training.cpp:150-164) around the reference's own
// place() / check_overlap(); transfers as transfers_for (training.cpp:68-80).
int ref_scale_placed(const double* pred, const int32_t* plen, const int32_t* id_rank,
                     int32_t count, const rs_profile* p, int32_t g, int32_t n_min,
                     int32_t n_max, double lambda, int32_t gpus,
                     const rs_placement_penalty* pen, int32_t* n_star, double* t_total,
                     double* t_pen_out, double* cost, double* t_norm, double* c_norm,
                     double* score, int32_t* order, double* actor_times) {
  return guarded([&] {
    const rs_topology& t = *pen->topology;
    rollsim::ClusterTopology topo;
    topo.nodes.clear();
    for (int i = 0; i < t.n_nodes; ++i) topo.nodes.push_back({t.node_gpus[i]});
    topo.intra_node_bw = t.intra_node_bw;
    topo.inter_node_bw = t.inter_node_bw;
    if (t.bw_matrix)
      for (int i = 0; i < t.n_nodes; ++i)
        topo.bw_matrix.emplace_back(t.bw_matrix + (size_t)i * t.n_nodes,
                                    t.bw_matrix + (size_t)(i + 1) * t.n_nodes);
    topo.learner_node = t.learner_node;
    topo.learner_gpus.assign(t.learner_gpus, t.learner_gpus + t.n_learner_gpus);
    rollsim::TimePenaltyFn fn = [&](int n, const std::vector<rollsim::ActorGroup>& groups,
                                    const std::vector<double>& times) {
      rollsim::GenerationPlan probe;
      probe.responses_per_prompt = g;
      probe.prefill_mode = rollsim::PrefillMode::shared_dedup;
      probe.n_actors = n;
      probe.groups = groups;
      probe.est_time_per_actor = times;
      probe.prefill_gpu_count = t.n_learner_gpus;
      rollsim::TransferSizes tr;
      tr.model_bytes = pen->model_bytes;
      tr.kv_bytes_per_actor.clear();
      for (const auto& grp : groups) {
        int64_t tokens = 0;
        for (int pl : grp.prompt_lens) tokens += pl;
        tr.kv_bytes_per_actor.push_back(static_cast<double>(tokens) * pen->kv_bytes_per_token);
      }
      rollsim::PlacementPlan pl = rollsim::place(probe, topo, tr);
      double exposed = 0;
      for (const rollsim::OverlapSlack& s : rollsim::check_overlap(pl, probe, pen->l_prefill_seconds))
        exposed = std::max(exposed, -s.slack);
      return exposed;
    };
    auto v = to_predicted(pred, plen, id_rank, count);
    rollsim::ScaleResult r = rollsim::scale(v, to_profile(p), g, n_min, n_max, lambda, gpus, fn);
    *n_star = r.n_star;
    for (size_t i = 0; i < r.candidates.size(); ++i) {
      const auto& c = r.candidates[i];
      if (t_total) t_total[i] = c.t_total;
      if (t_pen_out) t_pen_out[i] = c.t_penalty;
      if (cost) cost[i] = c.cost;
      if (t_norm) t_norm[i] = c.t_norm;
      if (c_norm) c_norm[i] = c.c_norm;
      if (score) score[i] = c.score;
    }
    if (actor_times)
      for (size_t i = 0; i < r.actor_times.size(); ++i) actor_times[i] = r.actor_times[i];
    if (order) {
      std::vector<int32_t> by_rank;
      if (id_rank) {
        by_rank.assign(count, 0);
        for (int32_t i = 0; i < count; ++i) by_rank[id_rank[i]] = i;
      }
      int32_t pos = 0;
      for (const auto& grp : r.groups)
        for (const std::string& id : grp.prompt_ids) {
          int32_t rk = std::stoi(id.substr(1));
          order[pos++] = id_rank ? by_rank[rk] : rk;
        }
    }
  });
}

// The reference's own LengthHistory, loaded with the same observations
// (LengthHistory::from_json, predictor.cpp:120-133).
int ref_predict_lengths(const double* obs, const int32_t* depth, const int32_t* gt,
                        int32_t count, int32_t window, double alpha, int32_t max_len,
                        const rs_noise_model* noise, const char* id_bytes,
                        const int64_t* id_offsets, double* out) {
  return guarded([&] {
    rollsim::LengthHistory check(window, alpha, max_len);  // constructor validation
    (void)check;
    nlohmann::json j;
    j["window"] = window;
    j["alpha"] = alpha;
    j["max_response_len"] = max_len;
    nlohmann::json o = nlohmann::json::object();
    std::vector<std::string> ids(count);
    for (int32_t i = 0; i < count; ++i) {
      ids[i] = id_bytes ? std::string(id_bytes + id_offsets[i], id_bytes + id_offsets[i + 1])
                        : "p" + std::to_string(i);
      if (depth[i] > 0)
        o[ids[i]] = std::vector<double>(obs + (size_t)i * window, obs + (size_t)i * window + depth[i]);
    }
    j["observations"] = std::move(o);
    rollsim::LengthHistory h = rollsim::LengthHistory::from_json(j);
    rollsim::NoiseModel nm;
    if (noise && noise->kind == 1) {
      nm.kind = rollsim::NoiseModel::Kind::bucket;
      nm.bucket_accuracy = noise->bucket_accuracy;
      nm.bucket_width = noise->bucket_width;
      nm.seed = noise->seed;
    }
    for (int32_t i = 0; i < count; ++i) {
      rollsim::Prompt p;
      p.id = ids[i];
      p.ground_truth_len = gt[i];
      out[i] = nm.kind == rollsim::NoiseModel::Kind::identity ? h.predict(p) : h.predict_noisy(p, nm);
    }
  });
}

// The format ref_trace_prompts / ref_trace_steps read (0 CSV, 1 JSONL).
static rollsim::TraceFormat g_trace_format = rollsim::TraceFormat::csv;
void ref_trace_set_format(int fmt) {
  g_trace_format = fmt == 1 ? rollsim::TraceFormat::jsonl : rollsim::TraceFormat::csv;
}

// trace_to_string(trace_from_string(text, fmt_in), fmt_out) (workload.cpp):
// *out_len gets the size; out (nullable) the bytes when cap allows.
int ref_trace_convert(const char* text, int64_t n_bytes, int fmt_in, int fmt_out, char* out,
                      int64_t cap, int64_t* out_len) {
  return guarded([&] {
    const auto fi = fmt_in == 1 ? rollsim::TraceFormat::jsonl : rollsim::TraceFormat::csv;
    const auto fo = fmt_out == 1 ? rollsim::TraceFormat::jsonl : rollsim::TraceFormat::csv;
    const std::string s =
        rollsim::trace_to_string(rollsim::trace_from_string(std::string(text, text + n_bytes), fi), fo);
    *out_len = (int64_t)s.size();
    if (out && cap >= (int64_t)s.size()) std::copy(s.begin(), s.end(), out);
  });
}

// The prompt table of a trace through the reference's own reader
// (trace_from_string, workload.cpp:355-359): info = {count, n_tokens,
// id_bytes, g, max_prompt_len, max_response_len}; the arrays (nullable) get
// the id-sorted prompts.
int ref_trace_prompts(const char* text, int64_t n_bytes, int64_t* info, int32_t* tokens,
                      int64_t* offsets, char* ids, int64_t* id_offsets, int32_t* gt) {
  return guarded([&] {
    rollsim::WorkloadTrace t =
        rollsim::trace_from_string(std::string(text, text + n_bytes), g_trace_format);
    int64_t ntok = 0, nid = 0;
    for (const auto& p : t.prompts) {
      ntok += (int64_t)p.token_ids.size();
      nid += (int64_t)p.id.size();
    }
    info[0] = (int64_t)t.prompts.size();
    info[1] = ntok;
    info[2] = nid;
    info[3] = t.responses_per_prompt;
    info[4] = t.limits.max_prompt_len;
    info[5] = t.limits.max_response_len;
    int64_t to = 0, io = 0;
    for (size_t i = 0; i < t.prompts.size(); ++i) {
      const auto& p = t.prompts[i];
      if (offsets) offsets[i] = to;
      if (id_offsets) id_offsets[i] = io;
      if (tokens) std::copy(p.token_ids.begin(), p.token_ids.end(), tokens + to);
      if (ids) std::copy(p.id.begin(), p.id.end(), ids + io);
      if (gt) gt[i] = p.ground_truth_len;
      to += (int64_t)p.token_ids.size();
      io += (int64_t)p.id.size();
    }
    if (offsets) offsets[t.prompts.size()] = to;
    if (id_offsets) id_offsets[t.prompts.size()] = io;
  });
}

// The step table of a CSV trace through the reference's own reader: info =
// {n_steps, n_entries, g}; the arrays (nullable) as rs_trace_csr_steps_copy
// lays them out — step_idx, entry_off, the id-sorted index of each
// scheduled prompt in batch order, and its actual_lengths.
int ref_trace_steps(const char* text, int64_t n_bytes, int64_t* info, int32_t* step_idx,
                    int32_t* entry_off, int32_t* entry_prompt, int32_t* lengths) {
  return guarded([&] {
    rollsim::WorkloadTrace t =
        rollsim::trace_from_string(std::string(text, text + n_bytes), g_trace_format);
    int64_t e = 0;
    for (size_t s = 0; s < t.steps.size(); ++s) {
      const rollsim::StepRecord& st = t.steps[s];
      if (step_idx) step_idx[s] = st.step_idx;
      if (entry_off) entry_off[s] = (int32_t)e;
      for (const std::string& id : st.scheduled_prompts) {
        const rollsim::Prompt* p = t.find_prompt(id);
        if (entry_prompt) entry_prompt[e] = (int32_t)(p - t.prompts.data());
        const std::vector<int>& lens = st.actual_lengths.at(id);
        if (lengths) std::copy(lens.begin(), lens.end(), lengths + e * t.responses_per_prompt);
        ++e;
      }
    }
    if (entry_off) entry_off[t.steps.size()] = (int32_t)e;
    info[0] = (int64_t)t.steps.size();
    info[1] = e;
    info[2] = t.responses_per_prompt;
  });
}

int ref_sweep_arrays(const double* pred, const int32_t* plen,
                     int32_t n_scenarios, int32_t count, const rs_profile* p,
                     int32_t g, int32_t n_min, int32_t n_max, double lambda,
                     int32_t gpus, int32_t n_threads, double* t_total,
                     double* cost, int32_t* n_star) {
  if (n_threads < 1) n_threads = 1;
  const int32_t c_n = n_max - n_min + 1;
  std::vector<int> status(n_scenarios, 0);
  std::vector<std::string> errs(n_threads);
  auto work = [&](int tid) {
    for (int32_t s = tid; s < n_scenarios; s += n_threads) {
      status[s] = guarded([&] {
        auto v = to_predicted(pred + (size_t)s * count, plen + (size_t)s * count,
                              nullptr, count);
        rollsim::ScaleResult r =
            rollsim::scale(v, to_profile(p), g, n_min, n_max, lambda, gpus);
        n_star[s] = r.n_star;
        for (int32_t i = 0; i < c_n; ++i) {
          t_total[(size_t)s * c_n + i] = r.candidates[i].t_total;
          cost[(size_t)s * c_n + i] = r.candidates[i].cost;
        }
      });
      if (status[s]) errs[tid] = g_err;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < n_threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int32_t s = 0; s < n_scenarios; ++s)
    if (status[s]) {
      for (auto& e : errs)
        if (!e.empty()) g_err = e;
      return status[s];
    }
  return 0;
}

}  // extern "C"
