// extern "C" entry points declared in include/treetrain_b200.h. Each maps onto one reference
// operation (cited per function in the header) and converts exceptions into status codes.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "corpus_io.hpp"
#include "engine.hpp"
#include "prefix_tree.hpp"
#include "ttpm.hpp"

struct tt_tree {
  ttb::PrefixTree t;
};
struct tt_engine {
  std::unique_ptr<ttb::Engine> e;
};
struct tt_step_plan {
  std::unique_ptr<ttb::StepPlan> p;
};

namespace {

std::vector<ttb::SeqView> views(const int32_t* tokens, const uint64_t* offsets, const double* weights, uint64_t n) {
  if (!tokens || !offsets) throw std::invalid_argument("null sequence arrays");
  std::vector<ttb::SeqView> v(n);
  for (uint64_t i = 0; i < n; ++i) {
    if (offsets[i + 1] < offsets[i]) throw std::invalid_argument("sequence offsets must be non-decreasing");
    v[i].tokens = tokens + offsets[i];
    v[i].weights = weights ? weights + offsets[i] : nullptr;
    v[i].len = offsets[i + 1] - offsets[i];
  }
  return v;
}

int copy_out(const std::string& s, char* buf, uint64_t cap, uint64_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const uint64_t n = s.size() < cap ? s.size() : cap;
    std::memcpy(buf, s.data(), n);
  }
  return TT_OK;
}

void fill_plan(const ttb::PartitionPlan& p, uint64_t n, int32_t* group_of_seq, uint64_t* costs, uint64_t* max_cost,
               uint64_t* dup) {
  if (group_of_seq)
    for (size_t g = 0; g < p.groups.size(); ++g)
      for (uint64_t i : p.groups[g]) group_of_seq[i] = static_cast<int32_t>(g);
  (void)n;
  if (costs)
    for (size_t g = 0; g < p.costs.size(); ++g) costs[g] = p.costs[g];
  if (max_cost) *max_cost = p.max_cost;
  if (dup) *dup = p.duplicated;
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null ") + what);
}

// Every engine entry point first selects the engine's GPU: a process may hold engines on several
// devices, and the caller's current device is not necessarily this engine's.
ttb::Engine& use(tt_engine* eng) {
  need(eng, "engine");
  ttb::check_cuda(cudaSetDevice(eng->e->device()), "cudaSetDevice");
  return *eng->e;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ prefix tree
int tt_tree_build(const int32_t* tokens, const uint64_t* offsets, const double* weights, uint64_t n_seqs,
                  tt_tree** out) {
  return ttb::guarded([&] {
    need(out, "out");
    auto t = std::make_unique<tt_tree>();
    t->t = ttb::build_prefix_tree(views(tokens, offsets, weights, n_seqs));
    *out = t.release();
  });
}

int tt_tree_destroy(tt_tree* tree) {
  delete tree;
  return TT_OK;
}

int tt_tree_order_children(tt_tree* tree, int32_t policy) {
  return ttb::guarded([&] {
    need(tree, "tree");
    ttb::order_children(tree->t, policy);
  });
}

int tt_tree_stats(const tt_tree* tree, uint64_t* tree_tokens, uint64_t* num_sequences, uint64_t* num_nodes,
                  uint64_t* max_path_tokens) {
  return ttb::guarded([&] {
    need(tree, "tree");
    if (tree_tokens) *tree_tokens = tree->t.total_tree_tokens;
    if (num_sequences) *num_sequences = tree->t.num_sequences;
    if (num_nodes) *num_nodes = tree->t.nodes.size() - 1;
    if (max_path_tokens) *max_path_tokens = tree->t.nodes[0].max_path_below;
  });
}

int tt_tree_serialize(const tt_tree* tree, char* buf, uint64_t cap, uint64_t* len) {
  return ttb::guarded([&] {
    need(tree, "tree");
    copy_out(ttb::serialize_tree(tree->t), buf, cap, len);
  });
}

int tt_tree_dfs_trace(const tt_tree* tree, char* buf, uint64_t cap, uint64_t* len) {
  return ttb::guarded([&] {
    need(tree, "tree");
    copy_out(ttb::dfs_trace(tree->t), buf, cap, len);
  });
}

// ------------------------------------------------------------------ partitioner
int tt_lexicographic_sort(const int32_t* tokens, const uint64_t* offsets, uint64_t n_seqs, uint64_t* order_out) {
  return ttb::guarded([&] {
    need(order_out, "order_out");
    const auto ord = ttb::lexicographic_order(views(tokens, offsets, nullptr, n_seqs));
    for (size_t i = 0; i < ord.size(); ++i) order_out[i] = ord[i];
  });
}

int tt_partition_contiguous(const int32_t* tokens, const uint64_t* offsets, uint64_t n_seqs, uint64_t K,
                            int32_t* group_of_seq, uint64_t* group_costs, uint64_t* max_cost, uint64_t* duplicated) {
  return ttb::guarded([&] {
    fill_plan(ttb::partition_contiguous(views(tokens, offsets, nullptr, n_seqs), K), n_seqs, group_of_seq,
              group_costs, max_cost, duplicated);
  });
}

int tt_greedy_least_loaded(const int32_t* tokens, const uint64_t* offsets, uint64_t n_seqs, uint64_t K,
                           int32_t cost_mode, int32_t* group_of_seq, uint64_t* group_costs, uint64_t* max_cost,
                           uint64_t* duplicated) {
  return ttb::guarded([&] {
    fill_plan(ttb::greedy_least_loaded(views(tokens, offsets, nullptr, n_seqs), K, cost_mode), n_seqs, group_of_seq,
              group_costs, max_cost, duplicated);
  });
}

// ------------------------------------------------------------------ corpus
struct tt_corpus {
  std::vector<ttb::CorpusSeq> seqs;
};

int tt_corpus_load_jsonl(const char* path, tt_corpus** out) {
  return ttb::guarded([&] {
    need(path, "path");
    need(out, "out");
    auto c = std::make_unique<tt_corpus>();
    c->seqs = ttb::load_corpus_jsonl(path);
    *out = c.release();
  });
}

int tt_corpus_generate(const tt_corpus_spec* spec, tt_corpus** out) {
  return ttb::guarded([&] {
    need(spec, "spec");
    need(out, "out");
    ttb::CorpusSpec sp;
    sp.num_prompts = spec->num_prompts;
    sp.group_size = spec->group_size;
    sp.prompt_len_lo = spec->prompt_len_lo;
    sp.prompt_len_hi = spec->prompt_len_hi;
    sp.response_len_lo = spec->response_len_lo;
    sp.response_len_hi = spec->response_len_hi;
    sp.branch_prob = spec->branch_prob;
    sp.vocab_size = spec->vocab_size;
    sp.seed = spec->seed;
    auto c = std::make_unique<tt_corpus>();
    c->seqs = ttb::gen_corpus(sp);
    *out = c.release();
  });
}

int tt_corpus_from_csr(const int32_t* tokens, const uint64_t* offsets, const double* weights, uint64_t n_seqs,
                       const char* const* seq_ids, tt_corpus** out) {
  return ttb::guarded([&] {
    need(out, "out");
    if (n_seqs > 0) {
      need(tokens, "tokens");
      need(offsets, "offsets");
    }
    auto c = std::make_unique<tt_corpus>();
    c->seqs.resize(n_seqs);
    for (uint64_t i = 0; i < n_seqs; ++i) {
      auto& q = c->seqs[i];
      if (offsets[i + 1] < offsets[i]) throw std::invalid_argument("tt_corpus_from_csr: offsets not ascending");
      q.seq_id = seq_ids && seq_ids[i] ? std::string(seq_ids[i]) : std::to_string(i);
      q.tokens.assign(tokens + offsets[i], tokens + offsets[i + 1]);
      if (weights) q.weights.assign(weights + offsets[i], weights + offsets[i + 1]);
      else q.weights.assign(q.tokens.size(), 1.0);
    }
    *out = c.release();
  });
}

int tt_corpus_save_jsonl(const tt_corpus* corpus, const char* path) {
  return ttb::guarded([&] {
    need(corpus, "corpus");
    need(path, "path");
    ttb::save_corpus_jsonl(path, corpus->seqs);
  });
}

int tt_corpus_size(const tt_corpus* corpus, uint64_t* n_seqs, uint64_t* n_tokens) {
  return ttb::guarded([&] {
    need(corpus, "corpus");
    uint64_t t = 0;
    for (const auto& q : corpus->seqs) t += q.tokens.size();
    if (n_seqs) *n_seqs = corpus->seqs.size();
    if (n_tokens) *n_tokens = t;
  });
}

int tt_corpus_export(const tt_corpus* corpus, int32_t* tokens, uint64_t* offsets, double* weights) {
  return ttb::guarded([&] {
    need(corpus, "corpus");
    uint64_t o = 0;
    for (size_t i = 0; i < corpus->seqs.size(); ++i) {
      const auto& q = corpus->seqs[i];
      if (offsets) offsets[i] = o;
      if (tokens) std::memcpy(tokens + o, q.tokens.data(), q.tokens.size() * sizeof(int32_t));
      if (weights) std::memcpy(weights + o, q.weights.data(), q.weights.size() * sizeof(double));
      o += q.tokens.size();
    }
    if (offsets) offsets[corpus->seqs.size()] = o;
  });
}

int tt_corpus_seq_id(const tt_corpus* corpus, uint64_t i, char* buf, uint64_t buf_len, uint64_t* needed) {
  return ttb::guarded([&] {
    need(corpus, "corpus");
    if (i >= corpus->seqs.size()) throw std::invalid_argument("tt_corpus_seq_id: index out of range");
    const std::string& id = corpus->seqs[i].seq_id;
    if (needed) *needed = id.size() + 1;
    if (buf && buf_len > 0) {
      const size_t n = std::min<size_t>(id.size(), buf_len - 1);
      std::memcpy(buf, id.data(), n);
      buf[n] = '\0';
    }
  });
}

int tt_corpus_destroy(tt_corpus* corpus) {
  delete corpus;
  return TT_OK;
}

// ------------------------------------------------------------------ engine
int tt_param_count(const tt_model_config* cfg, uint64_t* n) {
  return ttb::guarded([&] {
    need(cfg, "cfg");
    uint64_t k = 0;
    for (auto& t : ttb::tensor_specs(*cfg)) {
      uint64_t m = 1;
      for (auto s : t.second) m *= s;
      k += m;
    }
    *n = k;
  });
}

int tt_engine_create(const tt_model_config* cfg, int32_t device, tt_engine** out) {
  return ttb::guarded([&] {
    need(cfg, "cfg");
    need(out, "out");
    auto e = std::make_unique<tt_engine>();
    e->e = std::make_unique<ttb::Engine>(*cfg, device);
    *out = e.release();
  });
}

int tt_engine_destroy(tt_engine* eng) {
  return ttb::guarded([&] {
    if (eng) use(eng);
    delete eng;
  });
}

int tt_engine_stream(tt_engine* eng, void** stream) {
  return ttb::guarded([&] {
    use(eng);
    *stream = eng->e->stream();
  });
}

int tt_params_upload_f32(tt_engine* eng, const float* flat, uint64_t n) {
  return ttb::guarded([&] {
    use(eng);
    need(flat, "flat");
    eng->e->upload_params(flat, n);
  });
}

int tt_params_upload_f64(tt_engine* eng, const double* flat, uint64_t n) {
  return ttb::guarded([&] {
    use(eng);
    need(flat, "flat");
    std::vector<float> f(flat, flat + n);
    eng->e->upload_params(f.data(), n);
  });
}

int tt_params_init_random(tt_engine* eng, uint64_t seed) {
  return ttb::guarded([&] {
    use(eng);
    eng->e->init_random(seed);
  });
}

int tt_params_load_ttpm(tt_engine* eng, const char* path) {
  return ttb::guarded([&] {
    use(eng);
    need(path, "path");
    ttb::TtpmFile f = ttb::read_ttpm(path);
    const tt_model_config& c = eng->e->config();
    if (f.config.vocab_size != c.vocab_size || f.config.d_model != c.d_model || f.config.n_heads != c.n_heads ||
        f.config.n_layers != c.n_layers || f.config.d_ff != c.d_ff)
      throw std::invalid_argument("load_parameters: file config does not match the engine");
    std::vector<float> v(f.values.begin(), f.values.end());
    eng->e->upload_params(v.data(), v.size());
  });
}

int tt_grads_zero(tt_engine* eng) {
  return ttb::guarded([&] {
    use(eng);
    eng->e->grads_zero();
  });
}

int tt_grads_download_f32(tt_engine* eng, float* out, uint64_t n) {
  return ttb::guarded([&] {
    use(eng);
    need(out, "out");
    eng->e->grads_download(out, n);
  });
}

int tt_grads_download_f64(tt_engine* eng, double* out, uint64_t n) {
  return ttb::guarded([&] {
    use(eng);
    need(out, "out");
    eng->e->grads_download_f64(out, n);
  });
}

int tt_grads_allreduce(tt_engine* eng, void* nccl_comm) {
  return ttb::guarded([&] {
    use(eng);
    eng->e->grads_allreduce(nccl_comm);
  });
}

int tt_weighted_nll(tt_engine* eng, const float* logits, uint64_t n, const uint64_t* row_off, const int32_t* targets,
                    const double* weights, double* loss_out, float* grad_logits_out) {
  return ttb::guarded([&] {
    use(eng);
    const double l = eng->e->weighted_nll(logits, n, row_off, targets, weights, grad_logits_out);
    if (loss_out) *loss_out = l;
  });
}

int tt_grads_device_ptr(tt_engine* eng, float** dptr, uint64_t* n) {
  return ttb::guarded([&] {
    use(eng);
    *dptr = eng->e->grads_device();
    *n = eng->e->param_count();
  });
}

int tt_grads_accum_count(tt_engine* eng, uint64_t* count) {
  return ttb::guarded([&] {
    use(eng);
    *count = eng->e->accum_count();
  });
}

int tt_tree_train_step(tt_engine* eng, const tt_tree* tree, const tt_sched_config* sched, tt_step_result* result) {
  return ttb::guarded([&] {
    use(eng);
    need(tree, "tree");
    need(sched, "sched");
    tt_step_result r = eng->e->train_step(tree->t, *sched);
    if (result) *result = r;
  });
}

int tt_dense_train_step(tt_engine* eng, const int32_t* tokens, const uint64_t* offsets, const double* weights,
                        uint64_t n_seqs, tt_step_result* result) {
  return ttb::guarded([&] {
    use(eng);
    ttb::PrefixTree flat = ttb::build_flat_forest(views(tokens, offsets, weights, n_seqs));
    tt_sched_config sc{};
    sc.sibling_batch = 1;  // every sequence is its own root-level leaf: packed varlen batches
    sc.batch_token_budget = 0;  // memory-aware automatic budget
    tt_step_result r = eng->e->train_step(flat, sc);
    if (result) *result = r;
  });
}

int tt_plan_create(tt_engine* eng, const tt_tree* tree, const tt_sched_config* sched, tt_step_plan** out) {
  return ttb::guarded([&] {
    use(eng);
    need(tree, "tree");
    need(sched, "sched");
    need(out, "out");
    auto p = std::make_unique<tt_step_plan>();
    p->p = eng->e->prepare(tree->t, *sched);
    *out = p.release();
  });
}

int tt_plan_execute(tt_engine* eng, tt_step_plan* plan, tt_step_result* result) {
  return ttb::guarded([&] {
    use(eng);
    need(plan, "plan");
    tt_step_result r = eng->e->execute(*plan->p);
    if (result) *result = r;
  });
}

int tt_plan_execute_async(tt_engine* eng, tt_step_plan* plan) {
  return ttb::guarded([&] {
    use(eng);
    need(plan, "plan");
    eng->e->execute_async(*plan->p);
  });
}

int tt_plan_wait(tt_engine* eng, tt_step_plan* plan, tt_step_result* result) {
  return ttb::guarded([&] {
    use(eng);
    need(plan, "plan");
    tt_step_result r = eng->e->wait(*plan->p);
    if (result) *result = r;
  });
}

int tt_plan_trace(const tt_step_plan* plan, char* buf, uint64_t cap, uint64_t* len) {
  return ttb::guarded([&] {
    need(plan, "plan");
    copy_out(plan->p->trace, buf, cap, len);
  });
}

int tt_plan_destroy(tt_step_plan* plan) {
  return ttb::guarded([&] { delete plan; });
}

int tt_engine_set_profiling(tt_engine* eng, int32_t on) {
  return ttb::guarded([&] {
    use(eng);
    eng->e->set_profiling(on != 0);
  });
}

int tt_engine_set_option(tt_engine* eng, const char* key, int64_t value) {
  return ttb::guarded([&] {
    use(eng);
    need(key, "key");
    eng->e->set_option(key, value);
  });
}

int tt_engine_profile(tt_engine* eng, double* ms, double* flops, double* bytes, uint64_t* launches, int32_t reset) {
  return ttb::guarded([&] {
    use(eng);
    const ttb::KStats& k = eng->e->kstats();
    for (int i = 0; i < TT_NUM_KCLASS; ++i) {
      if (ms) ms[i] = k.ms[i];
      if (flops) flops[i] = k.flops[i];
      if (bytes) bytes[i] = k.bytes[i];
      if (launches) launches[i] = k.launches[i];
    }
    if (reset) eng->e->reset_kstats();
  });
}

int tt_engine_profile_gemm_text(tt_engine* eng, char* buf, uint64_t cap, uint64_t* len) {
  return ttb::guarded([&] {
    use(eng);
    copy_out(eng->e->gemm_profile_text(), buf, cap, len);
  });
}

int tt_segment_push(tt_engine* eng, const int32_t* tokens, uint64_t len, float* logits_out) {
  return ttb::guarded([&] {
    use(eng);
    need(tokens, "tokens");
    eng->e->segment_push(tokens, len, true, true, logits_out);
  });
}

int tt_segment_push_ex(tt_engine* eng, const int32_t* tokens, uint64_t len, int32_t want_kv, int32_t want_activations,
                       float* logits_out) {
  return ttb::guarded([&] {
    use(eng);
    need(tokens, "tokens");
    eng->e->segment_push(tokens, len, want_kv != 0, want_activations != 0, logits_out);
  });
}

int tt_segment_loss(tt_engine* eng, const uint64_t* row_off, const int32_t* targets, const double* weights,
                    double* loss_out) {
  return ttb::guarded([&] {
    use(eng);
    const double l = eng->e->segment_loss(row_off, targets, weights);
    if (loss_out) *loss_out = l;
  });
}

int tt_segment_pop(tt_engine* eng, const float* grad_logits, float* grad_prefix_out) {
  return ttb::guarded([&] {
    use(eng);
    eng->e->segment_pop(grad_logits, grad_prefix_out);
  });
}

int tt_stack_reset(tt_engine* eng) {
  return ttb::guarded([&] {
    use(eng);
    eng->e->stack_reset();
  });
}

int tt_stack_depth(tt_engine* eng, uint64_t* segments, uint64_t* tokens) {
  return ttb::guarded([&] {
    use(eng);
    if (segments) *segments = eng->e->stack_segments();
    if (tokens) *tokens = eng->e->stack_tokens();
  });
}

}  // extern "C"
