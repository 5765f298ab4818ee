// treetrain_b200.hpp — header-only C++ wrapper over the C-ABI (treetrain_b200.h) that mirrors the
// reference's C++ API shape (namespace treetrain, /root/reference/proj/core/include/treetrain/) and
// its error behaviour: status codes are rethrown as std::invalid_argument / std::runtime_error
// (model.hpp:334-343, model_io.cpp:60-103) and a non-finite loss as std::runtime_error.
//
// Link: -L<repo>/paper_2602_00482_b200 -ltreetrain_b200  (or dlopen libtreetrain_b200.so).
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "treetrain_b200.h"

namespace treetrain_b200 {

inline void check(int rc) {
  if (rc == TT_OK) return;
  const std::string msg = tt_last_error();
  if (rc == TT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == TT_ERR_OOM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

// TokenSequence (token_sequence.hpp:15-21); seq_id is the position in the input vector.
struct TokenSequence {
  std::vector<int32_t> tokens;
  std::vector<double> weights;
};

struct Csr {
  std::vector<int32_t> tokens;
  std::vector<uint64_t> offsets{0};
  std::vector<double> weights;
  explicit Csr(const std::vector<TokenSequence>& seqs) {
    for (const auto& s : seqs) {
      if (!s.weights.empty() && s.weights.size() != s.tokens.size())
        throw std::invalid_argument("TokenSequence: one weight per token");
      tokens.insert(tokens.end(), s.tokens.begin(), s.tokens.end());
      if (s.weights.empty()) weights.insert(weights.end(), s.tokens.size(), 1.0);
      else weights.insert(weights.end(), s.weights.begin(), s.weights.end());
      offsets.push_back(tokens.size());
    }
  }
};

enum class ChildOrder : int32_t { as_built = 0, lexicographic = 1, subtree_tokens_desc = 2, subtree_tokens_asc = 3 };

// PrefixTree: build_prefix_tree + order_children.
class PrefixTree {
 public:
  explicit PrefixTree(const std::vector<TokenSequence>& seqs, ChildOrder order = ChildOrder::subtree_tokens_desc) {
    Csr c(seqs);
    tt_tree* t = nullptr;
    check(tt_tree_build(c.tokens.data(), c.offsets.data(), c.weights.data(), seqs.size(), &t));
    h_.reset(t);
    check(tt_tree_order_children(t, static_cast<int32_t>(order)));
  }
  uint64_t tree_token_count() const {
    uint64_t n = 0;
    check(tt_tree_stats(h_.get(), &n, nullptr, nullptr, nullptr));
    return n;
  }
  std::string serialize() const { return text(tt_tree_serialize); }
  std::string dfs_trace() const { return text(tt_tree_dfs_trace); }
  const tt_tree* handle() const { return h_.get(); }

 private:
  template <typename F>
  std::string text(F f) const {
    uint64_t n = 0;
    check(f(h_.get(), nullptr, 0, &n));
    std::string s(n, '\0');
    check(f(h_.get(), s.data(), n, &n));
    return s;
  }
  struct Del {
    void operator()(tt_tree* t) const { tt_tree_destroy(t); }
  };
  std::unique_ptr<tt_tree, Del> h_;
};

// SchedulerConfig / TrainStepResult.
using SchedulerConfig = tt_sched_config;
using TrainStepResult = tt_step_result;

// One B200 engine = Parameters + GradientStore + device KV stack on one GPU.
class Engine {
 public:
  Engine(const tt_model_config& cfg, int device = 0) {
    tt_engine* e = nullptr;
    check(tt_engine_create(&cfg, device, &e));
    h_.reset(e);
    check(tt_param_count(&cfg, &n_params_));
  }
  uint64_t param_count() const { return n_params_; }
  // Parameters in for_each_tensor order (model.hpp:42-59).
  void upload_parameters(const std::vector<double>& flat) { check(tt_params_upload_f64(h_.get(), flat.data(), flat.size())); }
  void load_parameters(const std::string& path) { check(tt_params_load_ttpm(h_.get(), path.c_str())); }
  void zero_gradients() { check(tt_grads_zero(h_.get())); }
  std::vector<float> gradients() const {
    std::vector<float> g(n_params_);
    check(tt_grads_download_f32(h_.get(), g.data(), g.size()));
    return g;
  }
  // tree_train_step
  TrainStepResult tree_train_step(const PrefixTree& tree, const SchedulerConfig& sc) {
    TrainStepResult r{};
    check(tt_tree_train_step(h_.get(), tree.handle(), &sc, &r));
    return r;
  }
  // dense_train_step
  TrainStepResult dense_train_step(const std::vector<TokenSequence>& seqs) {
    Csr c(seqs);
    TrainStepResult r{};
    check(tt_dense_train_step(h_.get(), c.tokens.data(), c.offsets.data(), c.weights.data(), seqs.size(), &r));
    return r;
  }
  // forward_segment / backward_segment over the device stack (model.hpp:328, :474)
  std::vector<float> forward_segment(const std::vector<int32_t>& tokens, uint64_t vocab) {
    std::vector<float> logits(tokens.size() * vocab);
    check(tt_segment_push(h_.get(), tokens.data(), tokens.size(), logits.data()));
    return logits;
  }
  void backward_segment(const std::vector<float>* grad_logits) {
    check(tt_segment_pop(h_.get(), grad_logits ? grad_logits->data() : nullptr, nullptr));
  }

 private:
  struct Del {
    void operator()(tt_engine* e) const { tt_engine_destroy(e); }
  };
  std::unique_ptr<tt_engine, Del> h_;
  uint64_t n_params_ = 0;
};

// partition_contiguous: group index per sequence + max group tree cost.
inline std::pair<std::vector<int32_t>, uint64_t> partition_contiguous(const std::vector<TokenSequence>& seqs,
                                                                      uint64_t K) {
  Csr c(seqs);
  std::vector<int32_t> g(seqs.size());
  std::vector<uint64_t> costs(K);
  uint64_t mx = 0, dup = 0;
  check(tt_partition_contiguous(c.tokens.data(), c.offsets.data(), seqs.size(), K, g.data(), costs.data(), &mx, &dup));
  return {g, mx};
}

}  // namespace treetrain_b200
