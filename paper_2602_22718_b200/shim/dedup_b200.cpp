// dedup_b200.cpp — drop-in replacement for proj/src/dedup.cpp.
//
// Defines the rollsim:: dedup API (proj/include/rollsim/dedup.hpp:20-78)
// on top of librs_b200 (include/rs.h). PrefixIndex keeps the reference's
// private layout; its tables are produced on the GPU by
// rs_prefix_index_build and the O(1) accessors read them.
#include <algorithm>

#include "rollsim/dedup.hpp"
#include "rollsim/errors.hpp"
#include "rs_shim.hpp"

namespace rollsim {

namespace {

// Gather the non-owning prompt pointers into a CSR (the only host work:
// marshalling across the boundary).
void to_csr(const std::vector<const Prompt*>& batch, std::vector<int32_t>* tok,
            std::vector<int64_t>* off) {
  off->assign(batch.size() + 1, 0);
  size_t total = 0;
  for (size_t i = 0; i < batch.size(); ++i) total += batch[i]->token_ids.size();
  tok->resize(std::max<size_t>(total, 1));
  size_t pos = 0;
  for (size_t i = 0; i < batch.size(); ++i) {
    const auto& t = batch[i]->token_ids;
    std::copy(t.begin(), t.end(), tok->begin() + pos);
    pos += t.size();
    (*off)[i + 1] = static_cast<int64_t>(pos);
  }
}

struct Handle {
  rs_prefix_index* h = nullptr;
  ~Handle() { rs_prefix_index_free(h); }
};

}  // namespace

PrefixIndex PrefixIndex::build(const std::vector<const Prompt*>& batch) {
  Handle h;
  const rs_shim::DeviceCsr* dev = rs_shim::device_csr_of(batch);
  if (dev) {  // b200::DeviceTrace::prefix_index: the CSR is already in HBM
    rs_shim::check(rs_prefix_index_build_device(rs_shim::ctx(), dev->tokens, dev->offsets,
                                                dev->count, &h.h));
  } else {
    if (batch.empty()) throw ValidationError("prefix index needs a non-empty batch");
    for (const Prompt* p : batch)
      if (p == nullptr || p->prompt_len() < 1)
        throw ValidationError("prefix index: empty prompt in batch");
    std::vector<int32_t> tok;
    std::vector<int64_t> off;
    to_csr(batch, &tok, &off);
    rs_shim::check(rs_prefix_index_build(rs_shim::ctx(), tok.data(), off.data(),
                                         static_cast<int32_t>(batch.size()), &h.h));
  }
  PrefixIndex idx;
  int32_t bs, mn, mx;
  rs_shim::check(rs_prefix_index_info(h.h, &bs, &mn, &mx, &idx.total_tokens_));
  idx.batch_size_ = bs;
  idx.min_len_ = mn;
  idx.max_len_ = mx;
  idx.nodes_at_depth_.resize(mx + 1);
  idx.short_count_below_.resize(mx + 2);
  idx.short_tokens_below_.resize(mx + 2);
  idx.longer_count_from_.resize(mx + 2);
  idx.longer_tokens_from_.resize(mx + 2);
  rs_shim::check(rs_prefix_index_tables(h.h, idx.nodes_at_depth_.data(),
                                        idx.short_count_below_.data(),
                                        idx.short_tokens_below_.data(),
                                        idx.longer_count_from_.data(),
                                        idx.longer_tokens_from_.data()));
  return idx;
}

int64_t PrefixIndex::unique_prefix_count(int prefix_len) const {
  if (prefix_len < 1) throw ValidationError("unique_prefix_count: prefix_len must be >= 1");
  const int l = std::min(prefix_len, max_len_);
  return nodes_at_depth_[l] + short_count_below_[l];
}

int64_t PrefixIndex::unique_prefix_tokens(int prefix_len) const {
  if (prefix_len < 1) throw ValidationError("unique_prefix_tokens: prefix_len must be >= 1");
  const int l = std::min(prefix_len, max_len_);
  return nodes_at_depth_[l] * l + short_tokens_below_[l];
}

int64_t PrefixIndex::remainder_tokens(int prefix_len) const {
  if (prefix_len < 1) throw ValidationError("remainder_tokens: prefix_len must be >= 1");
  return prefix_len >= max_len_
             ? 0
             : longer_tokens_from_[prefix_len] - longer_count_from_[prefix_len] * prefix_len;
}

// select_prefix_length / dedup_savings (dedup.hpp:63-74) are O(log L) host
// arithmetic over the O(1) accessors; the tables behind them come from the
// GPU. D(L) is non-decreasing, so the deepest feasible L is found by
// bisection on [l_min, l_max].
PrefixSelection select_prefix_length(const PrefixIndex& index, const PrefillCapacity& capacity,
                                     int l_min, int l_max) {
  if (l_min < 1 || l_min > l_max)
    throw ValidationError("select_prefix_length: need 1 <= l_min <= l_max");
  if (capacity.max_unique_prefixes < 1)
    throw ConfigError("prefill capacity must allow at least one prefix");
  const int64_t cap = capacity.max_unique_prefixes;
  if (index.unique_prefix_count(l_min) > cap) return {l_min, true};
  int good = l_min, bad = l_max + 1;  // invariant: D(good) <= cap < D(bad)
  while (bad - good > 1) {
    const int mid = good + (bad - good) / 2;
    (index.unique_prefix_count(mid) <= cap ? good : bad) = mid;
  }
  return {good, false};
}

DedupSavings dedup_savings(const PrefixIndex& index, int l_star, int responses_per_prompt) {
  if (responses_per_prompt < 1)
    throw ValidationError("dedup_savings: responses_per_prompt must be >= 1");
  DedupSavings s;
  s.raw_prefill_tokens = index.total_prompt_tokens() * static_cast<int64_t>(responses_per_prompt);
  s.dedup_prefill_tokens = index.unique_prefix_tokens(l_star) + index.remainder_tokens(l_star);
  if (s.raw_prefill_tokens != 0)
    s.saved_fraction = static_cast<double>(s.raw_prefill_tokens - s.dedup_prefill_tokens) /
                       static_cast<double>(s.raw_prefill_tokens);
  return s;
}

int64_t unique_prefix_count_among(const std::vector<const Prompt*>& prompts, int prefix_len) {
  if (prefix_len < 1)
    throw ValidationError("unique_prefix_count_among: prefix_len must be >= 1");
  if (prompts.empty()) return 0;
  std::vector<int32_t> tok;
  std::vector<int64_t> off;
  to_csr(prompts, &tok, &off);
  int64_t out = 0;
  rs_shim::check(rs_unique_prefix_count_among(rs_shim::ctx(), tok.data(), off.data(),
                                              static_cast<int32_t>(prompts.size()), prefix_len,
                                              &out));
  return out;
}

}  // namespace rollsim
