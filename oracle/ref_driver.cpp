// ORACLE / CPU BASELINE — TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the reference's own model core, compiled in place from
// /root/reference/proj/core/include (read-only; nothing copied) by oracle/Makefile into
// oracle/_ref/libttref.so. All arithmetic is the reference's: forward_segment (model.hpp:328),
// backward_segment (model.hpp:474), weighted_nll (model.hpp:643), init_params (model.hpp:121),
// save/load_parameters (model_io.cpp:44-105), KVView/KVGrad::add_rows (model.hpp:162-207).
// The SPEC-only DFS driver is restated here as an event executor: the caller
// supplies the PUSH/POP event list (tree + order + loss pairs from oracle/treetrain_oracle.py),
// this file runs it with per-frame KVGrad buffers exactly as SPEC.md:208-211,271-276 describe.
#include <treetrain/model.hpp>
#include <treetrain/model_io.hpp>

#include <algorithm>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace treetrain;

extern "C" {
struct ttref_cfg {
  uint64_t vocab_size, d_model, n_heads, n_layers, d_ff, max_position;
};
}

namespace {

thread_local std::string g_err;

ModelConfig to_cfg(const ttref_cfg* c) {
  ModelConfig m;
  m.vocab_size = c->vocab_size;
  m.d_model = c->d_model;
  m.n_heads = c->n_heads;
  m.n_layers = c->n_layers;
  m.d_ff = c->d_ff;
  m.max_position = c->max_position;
  m.validate();
  return m;
}

template <typename T>
Parameters<T> params_from_flat(const ModelConfig& cfg, const double* flat) {
  Parameters<T> p = zero_parameters<T>(cfg);
  std::size_t o = 0;
  for_each_tensor(p, [&](const std::string&, std::vector<T>& d, const std::vector<std::size_t>&) {
    for (auto& v : d) v = T(flat[o++]);
  });
  return p;
}

template <typename T>
void flat_from_params(const Parameters<T>& p, double* out) {
  std::size_t o = 0;
  for_each_tensor(p, [&](const std::string&, const std::vector<T>& d, const std::vector<std::size_t>&) {
    for (auto v : d) out[o++] = double(v);
  });
}

template <typename T>
KVSegment<T> segment_from_flat(const ModelConfig& cfg, const double* k, const double* v, std::size_t S) {
  KVSegment<T> seg;
  seg.start_position = 0;
  seg.length = S;
  for (std::size_t l = 0; l < cfg.n_layers; ++l) {
    Matrix<T> K(S, cfg.d_model), V(S, cfg.d_model);
    for (std::size_t i = 0; i < S * cfg.d_model; ++i) {
      K.data[i] = T(k[l * S * cfg.d_model + i]);
      V.data[i] = T(v[l * S * cfg.d_model + i]);
    }
    seg.keys.push_back(std::move(K));
    seg.values.push_back(std::move(V));
  }
  return seg;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// ---------------------------------------------------------------- event executor
template <typename T>
struct Frame {
  std::size_t start = 0, length = 0;
  KVSegment<T> kv;
  SegmentActivations<T> acts;
  KVGrad<T> grad;  // accumulated dK/dV for this frame's own rows
  Matrix<T> logits;
};

template <typename T>
double run_events(const ModelConfig& cfg, const Parameters<T>& params, GradientStore<T>& grads, uint64_t n_events,
                  const int32_t* ev_type, const uint64_t* ev_tok_off, const int32_t* tokens,
                  const uint64_t* ev_pair_off, const int32_t* pair_rows, const int32_t* pair_tgts,
                  const double* pair_w) {
  std::vector<Frame<T>> stack;
  double total = 0.0;
  for (uint64_t e = 0; e < n_events; ++e) {
    if (ev_type[e] == 0) {  // PUSH: forward_segment from the stack KV
      KVView<T> view;
      std::size_t S = 0;
      for (auto& f : stack) {
        view.push(f.kv);
        S += f.length;
      }
      std::span<const TokenId> tok(tokens + ev_tok_off[e], ev_tok_off[e + 1] - ev_tok_off[e]);
      ForwardResult<T> r = forward_segment(params, view, tok, S, /*want_kv=*/true, /*want_acts=*/true);
      Frame<T> f;
      f.start = S;
      f.length = tok.size();
      f.kv = std::move(*r.kv);
      f.acts = std::move(*r.activations);
      f.grad = KVGrad<T>::zeros(f.length, cfg);
      f.logits = std::move(r.logits);
      stack.push_back(std::move(f));
    } else {  // POP: own loss (deferred) + accumulated KVGrad -> backward_segment
      if (stack.empty()) throw std::invalid_argument("run_events: POP on empty stack");
      Frame<T>& f = stack.back();
      const uint64_t p0 = ev_pair_off[e], p1 = ev_pair_off[e + 1];
      Matrix<T> gl(f.length, cfg.vocab_size);
      bool have = false;
      for (uint64_t p = p0; p < p1; ++p) {  // one weighted_nll term per (row, target, weight)
        Matrix<T> one(1, cfg.vocab_size);
        const std::size_t row = std::size_t(pair_rows[p]);
        for (std::size_t c = 0; c < cfg.vocab_size; ++c) one(0, c) = f.logits(row, c);
        const TokenId tg = pair_tgts[p];
        const double w = pair_w[p];
        LossResult<T> lr = weighted_nll(one, std::span<const TokenId>(&tg, 1), std::span<const double>(&w, 1));
        if (!std::isfinite(lr.loss)) throw std::runtime_error("run_events: non-finite loss");
        total += lr.loss;
        for (std::size_t c = 0; c < cfg.vocab_size; ++c) gl(row, c) += lr.grad_logits(0, c);
        have = true;
      }
      KVView<T> view;
      for (std::size_t i = 0; i + 1 < stack.size(); ++i) view.push(stack[i].kv);
      BackwardUpstream<T> up;
      up.grad_logits = have ? &gl : nullptr;
      up.grad_new_kv = &f.grad;
      KVGrad<T> gp = backward_segment(params, f.acts, view, up, grads);
      for (std::size_t i = 0; i + 1 < stack.size(); ++i)  // scatter grad_prefix into ancestor frames
        stack[i].grad.add_rows(gp, stack[i].start, stack[i].start + stack[i].length, 0);
      stack.pop_back();
    }
  }
  if (!stack.empty()) throw std::invalid_argument("run_events: unbalanced events");
  return total;
}

template <typename T>
int run_events_entry(const ttref_cfg* c, const double* params_flat, uint64_t n_events, const int32_t* ev_type,
                     const uint64_t* ev_tok_off, const int32_t* tokens, const uint64_t* ev_pair_off,
                     const int32_t* pair_rows, const int32_t* pair_tgts, const double* pair_w, double* loss_out,
                     double* grads_out) {
  return guard([&] {
    const ModelConfig cfg = to_cfg(c);
    const Parameters<T> params = params_from_flat<T>(cfg, params_flat);
    GradientStore<T> g = make_gradient_store<T>(cfg);
    *loss_out = run_events<T>(cfg, params, g, n_events, ev_type, ev_tok_off, tokens, ev_pair_off, pair_rows,
                              pair_tgts, pair_w);
    if (grads_out) flat_from_params(g.tensors, grads_out);
  });
}

}  // namespace

extern "C" {

const char* ttref_last_error(void) { return g_err.c_str(); }

int ttref_param_count(const ttref_cfg* c, uint64_t* n) {
  return guard([&] { *n = total_param_count(zero_parameters<double>(to_cfg(c))); });
}

// init_params<double> (model.hpp:121-142): the reference's own deterministic init.
int ttref_init_params(const ttref_cfg* c, uint64_t seed, double* out) {
  return guard([&] { flat_from_params(init_params<double>(to_cfg(c), seed), out); });
}

// save_parameters (model_io.cpp:44-71); dtype 0 = f32, 1 = f64.
int ttref_save_ttpm(const ttref_cfg* c, const double* flat, int dtype, const char* path) {
  return guard([&] {
    const ModelConfig cfg = to_cfg(c);
    if (dtype == 0) save_parameters(params_from_flat<float>(cfg, flat), path);
    else save_parameters(params_from_flat<double>(cfg, flat), path);
  });
}

// load_parameters<double> (model_io.cpp:73-105).
int ttref_load_ttpm_f64(const char* path, ttref_cfg* c_out, double* out, uint64_t cap) {
  return guard([&] {
    Parameters<double> p = load_parameters<double>(path);
    const uint64_t n = total_param_count(p);
    c_out->vocab_size = p.config.vocab_size;
    c_out->d_model = p.config.d_model;
    c_out->n_heads = p.config.n_heads;
    c_out->n_layers = p.config.n_layers;
    c_out->d_ff = p.config.d_ff;
    c_out->max_position = p.config.max_position;
    if (out) {
      if (cap < n) throw std::invalid_argument("ttref_load_ttpm_f64: buffer too small");
      flat_from_params(p, out);
    }
  });
}

// forward_segment<double> with the prefix given as one KV segment [L][S][d].
int ttref_forward_segment_f64(const ttref_cfg* c, const double* params_flat, const double* pk, const double* pv,
                              uint64_t S, const int32_t* tokens, uint64_t len, double* logits_out, double* k_out,
                              double* v_out) {
  return guard([&] {
    const ModelConfig cfg = to_cfg(c);
    const Parameters<double> P = params_from_flat<double>(cfg, params_flat);
    KVSegment<double> seg = segment_from_flat<double>(cfg, pk, pv, S);
    KVView<double> view;
    view.push(seg);
    ForwardResult<double> r = forward_segment(P, view, std::span<const TokenId>(tokens, len), S, true, false);
    std::memcpy(logits_out, r.logits.data.data(), sizeof(double) * r.logits.data.size());
    const std::size_t n = len * cfg.d_model;
    for (std::size_t l = 0; l < cfg.n_layers; ++l) {
      if (k_out) std::memcpy(k_out + l * n, r.kv->keys[l].data.data(), sizeof(double) * n);
      if (v_out) std::memcpy(v_out + l * n, r.kv->values[l].data.data(), sizeof(double) * n);
    }
  });
}

// backward_segment<double>: activations from a fresh forward_segment, then the exact reverse
// pass. grads_inout is added into (flat, for_each_tensor order); grad prefix -> gpk/gpv [L][S][d].
int ttref_backward_segment_f64(const ttref_cfg* c, const double* params_flat, const double* pk, const double* pv,
                               uint64_t S, const int32_t* tokens, uint64_t len, const double* grad_logits,
                               const double* gnk, const double* gnv, double* grads_inout, double* gpk,
                               double* gpv) {
  return guard([&] {
    const ModelConfig cfg = to_cfg(c);
    const Parameters<double> P = params_from_flat<double>(cfg, params_flat);
    KVSegment<double> seg = segment_from_flat<double>(cfg, pk, pv, S);
    KVView<double> view;
    view.push(seg);
    ForwardResult<double> r = forward_segment(P, view, std::span<const TokenId>(tokens, len), S, false, true);
    GradientStore<double> g{params_from_flat<double>(cfg, grads_inout), 0};
    Matrix<double> gl;
    KVGrad<double> gn;
    BackwardUpstream<double> up;
    if (grad_logits) {
      gl = Matrix<double>(len, cfg.vocab_size);
      std::memcpy(gl.data.data(), grad_logits, sizeof(double) * gl.data.size());
      up.grad_logits = &gl;
    }
    if (gnk) {
      KVSegment<double> s2 = segment_from_flat<double>(cfg, gnk, gnv, len);
      gn.length = len;
      gn.keys = s2.keys;
      gn.values = s2.values;
      up.grad_new_kv = &gn;
    }
    KVGrad<double> gp = backward_segment(P, *r.activations, view, up, g);
    flat_from_params(g.tensors, grads_inout);
    const std::size_t n = S * cfg.d_model;
    for (std::size_t l = 0; l < cfg.n_layers; ++l) {
      if (gpk) std::memcpy(gpk + l * n, gp.keys[l].data.data(), sizeof(double) * n);
      if (gpv) std::memcpy(gpv + l * n, gp.values[l].data.data(), sizeof(double) * n);
    }
  });
}

// weighted_nll<double> (model.hpp:643-677).
int ttref_weighted_nll_f64(const double* logits, uint64_t n, uint64_t V, const int32_t* targets,
                           const double* weights, double* loss, double* grad) {
  return guard([&] {
    Matrix<double> L(n, V);
    std::memcpy(L.data.data(), logits, sizeof(double) * n * V);
    LossResult<double> r =
        weighted_nll(L, std::span<const TokenId>(targets, n), std::span<const double>(weights, n));
    *loss = r.loss;
    std::memcpy(grad, r.grad_logits.data.data(), sizeof(double) * n * V);
  });
}

// DFS event list executed with the reference arithmetic at T=double (precision 1) or float (0).
int ttref_run_events(int precision, const ttref_cfg* c, const double* params_flat, uint64_t n_events,
                     const int32_t* ev_type, const uint64_t* ev_tok_off, const int32_t* tokens,
                     const uint64_t* ev_pair_off, const int32_t* pair_rows, const int32_t* pair_tgts,
                     const double* pair_w, double* loss_out, double* grads_out) {
  if (precision == 0)
    return run_events_entry<float>(c, params_flat, n_events, ev_type, ev_tok_off, tokens, ev_pair_off, pair_rows,
                                   pair_tgts, pair_w, loss_out, grads_out);
  return run_events_entry<double>(c, params_flat, n_events, ev_type, ev_tok_off, tokens, ev_pair_off, pair_rows,
                                  pair_tgts, pair_w, loss_out, grads_out);
}

// CPU baseline: `n_threads` workers each run the same event list (one tree per host thread,
// SPEC.md:278) at T=float with private GradientStores; returns wall seconds.
int ttref_run_events_threads(const ttref_cfg* c, const double* params_flat, uint64_t n_events,
                             const int32_t* ev_type, const uint64_t* ev_tok_off, const int32_t* tokens,
                             const uint64_t* ev_pair_off, const int32_t* pair_rows, const int32_t* pair_tgts,
                             const double* pair_w, int n_threads, double* seconds_out, double* loss_out) {
  return guard([&] {
    const ModelConfig cfg = to_cfg(c);
    const Parameters<float> params = params_from_flat<float>(cfg, params_flat);
    std::vector<double> losses(n_threads, 0.0);
    std::vector<std::string> errs(n_threads);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int i = 0; i < n_threads; ++i)
      th.emplace_back([&, i] {
        try {
          GradientStore<float> g = make_gradient_store<float>(cfg);
          losses[i] = run_events<float>(cfg, params, g, n_events, ev_type, ev_tok_off, tokens, ev_pair_off,
                                        pair_rows, pair_tgts, pair_w);
        } catch (const std::exception& e) {
          errs[i] = e.what();
        }
      });
    for (auto& t : th) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    *loss_out = losses.empty() ? 0.0 : losses[0];
  });
}

// CPU baseline at full model shape without a full tree: a model handle holds
// init_params<float> (made once); each slice call runs, on each of n_threads workers,
// forward_segment + weighted_nll + backward_segment of `len` tokens over a random prefix KV of
// S rows. Per-thread setup (prefix KV fill, GradientStore) happens before a barrier and is not
// timed; returns the slowest worker's compute seconds.
struct ttref_model {
  ModelConfig cfg;
  Parameters<float> params;
};

ttref_model* ttref_model_create(const ttref_cfg* c, uint64_t seed) {
  try {
    auto* m = new ttref_model;
    m->cfg = to_cfg(c);
    m->params = init_params<float>(m->cfg, seed);
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ttref_model_destroy(ttref_model* m) { delete m; }

int ttref_model_slice(ttref_model* m, uint64_t S, uint64_t len, int n_threads, uint64_t seed, double* seconds_out) {
  return guard([&] {
    const ModelConfig& cfg = m->cfg;
    if (S + len > cfg.max_position) throw std::invalid_argument("slice exceeds max_position");
    std::vector<std::string> errs(n_threads);
    std::vector<double> secs(n_threads, 0.0);
    std::barrier sync(n_threads);
    std::vector<std::thread> th;
    for (int i = 0; i < n_threads; ++i)
      th.emplace_back([&, i] {
        bool arrived = false;
        try {
          std::mt19937_64 rng(seed + 17 * i + 1);
          std::normal_distribution<double> nd(0.0, 1.0);
          KVSegment<float> seg;
          seg.length = S;
          for (std::size_t l = 0; l < cfg.n_layers; ++l) {
            Matrix<float> K(S, cfg.d_model), V(S, cfg.d_model);
            for (auto& x : K.data) x = float(nd(rng));
            for (auto& x : V.data) x = float(nd(rng));
            seg.keys.push_back(std::move(K));
            seg.values.push_back(std::move(V));
          }
          KVView<float> view;
          view.push(seg);
          std::vector<TokenId> tok(len), tg(len);
          for (auto& t : tok) t = TokenId(rng() % cfg.vocab_size);
          for (auto& t : tg) t = TokenId(rng() % cfg.vocab_size);
          std::vector<double> w(len, 1.0);
          GradientStore<float> g = make_gradient_store<float>(cfg);
          sync.arrive_and_wait();
          arrived = true;
          const auto t0 = std::chrono::steady_clock::now();
          ForwardResult<float> r = forward_segment(m->params, view, std::span<const TokenId>(tok), S, false, true);
          LossResult<float> lr = weighted_nll(r.logits, std::span<const TokenId>(tg), std::span<const double>(w));
          BackwardUpstream<float> up;
          up.grad_logits = &lr.grad_logits;
          backward_segment(m->params, *r.activations, view, up, g);
          secs[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        } catch (const std::exception& e) {
          errs[i] = e.what();
          if (!arrived) sync.arrive_and_drop();
        }
      });
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    *seconds_out = *std::max_element(secs.begin(), secs.end());
  });
}

}  // extern "C"
