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

// LossResult of weighted_nll (model.hpp:637-640): loss + grad_logits [n x V].
struct LossResult {
  double loss = 0.0;
  std::vector<float> grad_logits;
};

// One NCCL communicator of the data-parallel step; rank 0 creates the id, the
// launcher ships it to every rank (MPI_Bcast, a TCP store, ...).
class NcclComm {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(TT_NCCL_UNIQUE_ID_BYTES);
    check(tt_nccl_unique_id(id.data()));
    return id;
  }
  NcclComm(const std::vector<uint8_t>& id, int nranks, int rank, int device) {
    if (id.size() != TT_NCCL_UNIQUE_ID_BYTES) throw std::invalid_argument("NcclComm: bad unique id");
    check(tt_nccl_comm_init_rank(id.data(), nranks, rank, device, &c_));
  }
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  ~NcclComm() {
    if (c_) tt_nccl_comm_destroy(c_);
  }
  void* handle() const { return c_; }

 private:
  void* c_ = nullptr;
};

class Engine;

// A prepared tree step (tt_plan_create): schedule, batches, memory plan and metadata resident in HBM;
// execute() any number of times, or execute_async() + wait() to overlap the host's preparation of the
// next step with this one.
class StepPlan {
 public:
  StepPlan(Engine& eng, const PrefixTree& tree, const SchedulerConfig& sc);
  TrainStepResult execute();
  void execute_async();
  TrainStepResult wait();
  std::string trace() const {
    uint64_t n = 0;
    check(tt_plan_trace(h_.get(), nullptr, 0, &n));
    std::string s(n, '\0');
    check(tt_plan_trace(h_.get(), s.data(), n, &n));
    return s;
  }

 private:
  struct Del {
    void operator()(tt_step_plan* p) const { tt_plan_destroy(p); }
  };
  tt_engine* eng_;
  std::unique_ptr<tt_step_plan, Del> h_;
};

// One B200 engine = Parameters + GradientStore + device KV stack on one GPU.
class Engine {
 public:
  Engine(const tt_model_config& cfg, int device = 0) : cfg_(cfg) {
    tt_engine* e = nullptr;
    check(tt_engine_create(&cfg, device, &e));
    h_.reset(e);
    check(tt_param_count(&cfg, &n_params_));
  }
  const tt_model_config& config() const { return cfg_; }
  uint64_t param_count() const { return n_params_; }
  tt_engine* handle() const { return h_.get(); }
  void set_option(const std::string& key, int64_t value) { check(tt_engine_set_option(h_.get(), key.c_str(), value)); }
  // Parameters in for_each_tensor order (model.hpp:42-59).
  void upload_parameters(const std::vector<double>& flat) { check(tt_params_upload_f64(h_.get(), flat.data(), flat.size())); }
  void upload_parameters(const std::vector<float>& flat) { check(tt_params_upload_f32(h_.get(), flat.data(), flat.size())); }
  void load_parameters(const std::string& path) { check(tt_params_load_ttpm(h_.get(), path.c_str())); }
  void zero_gradients() { check(tt_grads_zero(h_.get())); }
  // GradientStore<float> / GradientStore<double> in for_each_tensor order (model.hpp:76-81)
  std::vector<float> gradients() const {
    std::vector<float> g(n_params_);
    check(tt_grads_download_f32(h_.get(), g.data(), g.size()));
    return g;
  }
  std::vector<double> gradients_f64() const {
    std::vector<double> g(n_params_);
    check(tt_grads_download_f64(h_.get(), g.data(), g.size()));
    return g;
  }
  // the reference's reduction of the workers' GradientStores as one NCCL all-reduce
  void allreduce_gradients(const NcclComm& comm) { check(tt_grads_allreduce(h_.get(), comm.handle())); }
  // tree_train_step
  TrainStepResult tree_train_step(const PrefixTree& tree, const SchedulerConfig& sc) {
    TrainStepResult r{};
    check(tt_tree_train_step(h_.get(), tree.handle(), &sc, &r));
    return r;
  }
  StepPlan plan(const PrefixTree& tree, const SchedulerConfig& sc) { return StepPlan(*this, tree, sc); }
  // dense_train_step
  TrainStepResult dense_train_step(const std::vector<TokenSequence>& seqs) {
    Csr c(seqs);
    TrainStepResult r{};
    check(tt_dense_train_step(h_.get(), c.tokens.data(), c.offsets.data(), c.weights.data(), seqs.size(), &r));
    return r;
  }
  // forward_segment over the device stack (model.hpp:328-463): logits [len x V] sized from the
  // engine's own vocab_size; want_kv / want_activations as the reference (model.hpp:328-331)
  std::vector<float> forward_segment(const std::vector<int32_t>& tokens, bool want_kv = true,
                                     bool want_activations = true) {
    std::vector<float> logits(tokens.size() * cfg_.vocab_size);
    check(tt_segment_push_ex(h_.get(), tokens.data(), tokens.size(), want_kv ? 1 : 0, want_activations ? 1 : 0,
                             logits.data()));
    if (want_kv || want_activations) seg_lens_.push_back(tokens.size());
    return logits;
  }
  // forward_segment without the logits download (the loss stays on the device: segment_loss)
  void push_segment(const std::vector<int32_t>& tokens, bool want_kv = true, bool want_activations = true) {
    check(tt_segment_push_ex(h_.get(), tokens.data(), tokens.size(), want_kv ? 1 : 0, want_activations ? 1 : 0,
                             nullptr));
    if (want_kv || want_activations) seg_lens_.push_back(tokens.size());
  }
  // weighted_nll of the top segment's logits on the device (the VISIT); its pop then
  // takes the upstream grad_logits from these pairs. row_off (len + 1 offsets) or empty = one pair per row.
  double segment_loss(const std::vector<int32_t>& targets, const std::vector<double>& weights,
                      const std::vector<uint64_t>& row_off = {}) {
    double loss = 0.0;
    check(tt_segment_loss(h_.get(), row_off.empty() ? nullptr : row_off.data(), targets.data(), weights.data(), &loss));
    return loss;
  }
  // backward_segment (model.hpp:474-633) of the top segment: grad_logits [len x V] or nullptr (zero,
  // or the device pairs of segment_loss). Returns this pop's grad_prefix ([L][2][S][d], K then V) when
  // want_grad_prefix; it is always added into the ancestors' stack rows (KVGrad::add_rows).
  std::vector<float> backward_segment(const std::vector<float>* grad_logits, bool want_grad_prefix = false) {
    if (seg_lens_.empty()) throw std::invalid_argument("backward_segment: empty stack");
    const uint64_t len = seg_lens_.back();
    if (grad_logits && grad_logits->size() != len * cfg_.vocab_size)
      throw std::invalid_argument("backward_segment: grad_logits must be [len x vocab_size]");
    std::vector<float> gp;
    if (want_grad_prefix) {
      uint64_t segs = 0, toks = 0;
      check(tt_stack_depth(h_.get(), &segs, &toks));
      gp.assign(static_cast<size_t>(2) * cfg_.n_layers * (toks - len) * cfg_.d_model, 0.f);  // [L][2][S][d]
    }
    check(tt_segment_pop(h_.get(), grad_logits ? grad_logits->data() : nullptr, want_grad_prefix ? gp.data() : nullptr));
    seg_lens_.pop_back();
    return gp;
  }
  void reset_stack() {
    check(tt_stack_reset(h_.get()));
    seg_lens_.clear();
  }
  // weighted_nll (model.hpp:643-677) on the device over host logits [n x V]
  LossResult weighted_nll(const std::vector<float>& logits, const std::vector<int32_t>& targets,
                          const std::vector<double>& weights, const std::vector<uint64_t>& row_off = {}) {
    if (logits.size() % cfg_.vocab_size != 0) throw std::invalid_argument("weighted_nll: logits must be [n x V]");
    const uint64_t n = logits.size() / cfg_.vocab_size;
    LossResult r;
    r.grad_logits.assign(logits.size(), 0.f);
    check(tt_weighted_nll(h_.get(), logits.data(), n, row_off.empty() ? nullptr : row_off.data(), targets.data(),
                          weights.data(), &r.loss, r.grad_logits.data()));
    return r;
  }

 private:
  struct Del {
    void operator()(tt_engine* e) const { tt_engine_destroy(e); }
  };
  tt_model_config cfg_;
  std::unique_ptr<tt_engine, Del> h_;
  uint64_t n_params_ = 0;
  std::vector<uint64_t> seg_lens_;  // lengths of the pushed segments (the caller's KVView)
};

inline StepPlan::StepPlan(Engine& eng, const PrefixTree& tree, const SchedulerConfig& sc) : eng_(eng.handle()) {
  tt_step_plan* p = nullptr;
  check(tt_plan_create(eng_, tree.handle(), &sc, &p));
  h_.reset(p);
}
inline TrainStepResult StepPlan::execute() {
  TrainStepResult r{};
  check(tt_plan_execute(eng_, h_.get(), &r));
  return r;
}
inline void StepPlan::execute_async() { check(tt_plan_execute_async(eng_, h_.get())); }
inline TrainStepResult StepPlan::wait() {
  TrainStepResult r{};
  check(tt_plan_wait(eng_, h_.get(), &r));
  return r;
}

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
