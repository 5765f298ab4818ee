// B200 DFS prefix-tree forward/backward engine. See engine.hpp for the HBM layout.
//
//   push  = forward_segment  (model.hpp:328-463)  for a segment batch over the device KV stack
//   visit = weighted_nll     (model.hpp:643-677)  fused LM head + multi-target CE
//   pop   = backward_segment (model.hpp:474-633)  with grad_new_kv = the frame's dK/dV stack rows
//           and grad_prefix added into the ancestors' dK/dV stack rows (KVGrad::add_rows :193-206)
#include "engine.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>

#include "capi_internal.h"
#include "kernels/attention.h"
#include "kernels/elementwise.h"
#include "kernels/gemm.h"
#include "ttpm.hpp"

namespace ttb {

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
constexpr int kQChunkPrefix = 4096;  // tcgen05 dK/dV items over prefix rows (span members)
constexpr int kQChunkOwn = 2048;     // tcgen05 dK/dV items over a member's own rows (causal)

void ck(cudaError_t e, const char* what) { check_cuda(e, what); }

GemmOperand op(const bf16* p, long ld, bool mn) { return GemmOperand{p, ld, mn}; }

}  // namespace

DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}

namespace {
std::atomic<uint64_t> g_alloc_gen{1};
}
uint64_t alloc_generation() { return g_alloc_gen.load(); }

void DevBuf::ensure(size_t n) {
  if (n <= bytes) return;
  g_alloc_gen.fetch_add(1);
  if (p) {
    cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  if (n == 0) return;
  const cudaError_t e = cudaMalloc(&p, n);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw std::bad_alloc();
  }
  bytes = n;
}

Engine::Engine(const tt_model_config& cfg, int device) : cfg_(cfg), device_(device) {
  if (cfg.vocab_size < 1 || cfg.d_model < 1 || cfg.n_heads < 1 || cfg.n_layers < 1 || cfg.d_ff < 1 ||
      cfg.max_position < 1)
    throw std::invalid_argument("ModelConfig: all counts must be >= 1");
  if (cfg.d_model % cfg.n_heads != 0) throw std::invalid_argument("ModelConfig: d_model must be divisible by n_heads");
  V_ = cfg.vocab_size;
  d_ = cfg.d_model;
  H_ = cfg.n_heads;
  L_ = cfg.n_layers;
  F_ = cfg.d_ff;
  dh_ = d_ / H_;
  if (dh_ != 64 && dh_ != 128) throw std::invalid_argument("engine: head_dim must be 64 or 128 on sm_100a");
  if (d_ % 64 || F_ % 64 || V_ % 16)
    throw std::invalid_argument("engine: d_model and d_ff must be multiples of 64, vocab_size of 16");
  if (d_ > 8192) throw std::invalid_argument("engine: d_model must be <= 8192");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaEventCreateWithFlags(&step_done_, cudaEventDisableTiming), "cudaEventCreate");

  // ---- weights (bf16), device layout
  const size_t n_w = V_ * d_ + L_ * (3 * d_ * d_ + d_ * d_ + 2 * d_ * F_) + d_ * V_;
  wbuf_.ensure(n_w * sizeof(bf16));
  bf16* w = wbuf_.as<bf16>();
  emb_ = w;
  w += V_ * d_;
  for (int64_t l = 0; l < L_; ++l) {
    wqkv_.push_back(w);
    w += 3 * d_ * d_;
    wo_.push_back(w);
    w += d_ * d_;
    win_.push_back(w);
    w += d_ * F_;
    wout_.push_back(w);
    w += F_ * d_;
  }
  head_ = w;
  gainbuf_.ensure((2 * L_ + 1) * d_ * sizeof(float));
  float* gp = gainbuf_.as<float>();
  for (int64_t l = 0; l < L_; ++l) {
    attn_g_.push_back(gp + 2 * l * d_);
    mlp_g_.push_back(gp + (2 * l + 1) * d_);
  }
  final_g_ = gp + 2 * L_ * d_;
  k_fill(gp, (2 * L_ + 1) * d_, 1.0f, stream_);

  // ---- sinusoidal PE table, computed like add_positional_encoding (model.hpp:239-248)
  {
    std::vector<float> pe(cfg.max_position * d_);
    for (uint64_t p = 0; p < cfg.max_position; ++p)
      for (int64_t i = 0; 2 * i < d_; ++i) {
        const double freq = std::pow(10000.0, -double(2 * i) / double(d_));
        const double ang = double(p) * freq;
        pe[p * d_ + 2 * i] = float(std::sin(ang));
        if (2 * i + 1 < d_) pe[p * d_ + 2 * i + 1] = float(std::cos(ang));
      }
    pe_.ensure(pe.size() * sizeof(float));
    ck(cudaMemcpy(pe_.p, pe.data(), pe.size() * sizeof(float), cudaMemcpyHostToDevice), "upload PE");
  }

  // ---- GradientStore: flat fp32 in for_each_tensor order
  n_params_ = 0;
  for (auto& t : tensor_specs(cfg_)) {
    uint64_t k = 1;
    for (auto s : t.second) k *= s;
    n_params_ += k;
  }
  grads_.ensure(n_params_ * sizeof(float));
  float* g = grads_.as<float>();
  g_emb_ = g;
  g += V_ * d_;
  for (int64_t l = 0; l < L_; ++l) {
    g_attn_g_.push_back(g);
    g += d_;
    g_wq_.push_back(g);
    g += d_ * d_;
    g_wk_.push_back(g);
    g += d_ * d_;
    g_wv_.push_back(g);
    g += d_ * d_;
    g_wo_.push_back(g);
    g += d_ * d_;
    g_mlp_g_.push_back(g);
    g += d_;
    g_win_.push_back(g);
    g += d_ * F_;
    g_wout_.push_back(g);
    g += F_ * d_;
  }
  g_final_g_ = g;
  g += d_;
  g_head_ = g;
  grads_zero();
  loss_.ensure(sizeof(double));
  ck(cudaMallocHost(&loss_host_, sizeof(double)), "cudaMallocHost");
  ck(cudaStreamSynchronize(stream_), "engine init");
}

Engine::~Engine() {
  cudaStreamSynchronize(stream_);
  if (loss_host_) cudaFreeHost(loss_host_);
  if (meta_host_) cudaFreeHost(meta_host_);
  cudaStreamDestroy(stream_);
  cudaStreamSynchronize(copy_stream_);
  cudaStreamDestroy(copy_stream_);
  for (int i = 0; i < 2; ++i) {
    if (pin_ev_[i]) cudaEventDestroy(pin_ev_[i]);
    if (pin_ring_[i]) cudaFreeHost(pin_ring_[i]);
  }
  for (auto& b : meta_pool_) cudaFree(b.first);
  cudaEventDestroy(step_done_);
}

void Engine::set_option(const std::string& key, int64_t value) {
  if (key == "gemm_2cta") {
    gemm_2cta_ = value != 0 ? 1 : 0;
  } else if (key == "root_batch_tokens") {
    if (value < 0) throw std::invalid_argument("root_batch_tokens must be >= 0");
    root_batch_tokens_ = value;
  } else if (key == "head_chunk_mb") {
    if (value < 1) throw std::invalid_argument("head_chunk_mb must be >= 1");
    head_chunk_bytes_ = value << 20;
    head_cap_rows_ = 0;
  } else if (key == "pdl_auto_elems") {
    if (value < 0) throw std::invalid_argument("pdl_auto_elems must be >= 0");
    pdl_auto_elems_ = static_cast<double>(value);
  } else if (key == "gn_bf16") {
    // 1: grad_normed (dX GEMM -> RMSNorm backward) in bf16 where supported (default); 0: fp32
    gn_bf16_ = value != 0;
  } else if (key == "pdl") {
    // programmatic dependent launch (kernels/launch.cuh): 0 off, 1 every batch, 2 (default) batches of
    // at most pdl_auto_elems activation elements (rows x d_model), where launch latency and kernel prologues are a
    // visible share of each kernel (tools/pdl_ab.py: c1 +4.4%; the c2 step -0.6% with PDL)
    if (value < 0 || value > 2) throw std::invalid_argument("pdl must be 0, 1 or 2");
    pdl_ = static_cast<int>(value);
  } else if (key == "cuda_graph") {
    cuda_graph_ = value != 0;
  } else if (key == "ce_stats") {
    // 1: LM-head GEMM epilogue emits per-32-column softmax statistics, CE reads logits once
    // (default); 0: CE does both passes over the logits row itself
    ce_stats_ = value != 0;
  } else if (key == "plan_timing") {
    plan_timing_ = value != 0;
  } else if (key == "logits_bf16") {
    // 1: LM-head logits as bf16 offsets from their 32-column group max (half the logits traffic;
    // needs ce_stats); 0: fp32 logits
    logits_bf16_ = value != 0;
  } else {
    throw std::invalid_argument("unknown engine option: " + key);
  }
  ++opt_epoch_;
}

// ----------------------------------------------------------------------------- parameters
void Engine::upload_params(const float* flat, uint64_t n) {
  if (n != n_params_) throw std::invalid_argument("params upload: wrong parameter count");
  DevBuf tmp;
  size_t maxt = 0;
  for (auto& t : tensor_specs(cfg_)) {
    uint64_t k = 1;
    for (auto s : t.second) k *= s;
    maxt = std::max<size_t>(maxt, k);
  }
  tmp.ensure(maxt * sizeof(float));
  const float* src = flat;
  auto put = [&](uint64_t rows, uint64_t cols, bf16* dst, long ldd) {
    ck(cudaMemcpyAsync(tmp.p, src, rows * cols * sizeof(float), cudaMemcpyHostToDevice, stream_), "params upload");
    k_f32_to_bf16_2d(tmp.as<float>(), cols, dst, ldd, rows, cols, stream_);
    ck(cudaStreamSynchronize(stream_), "params upload");
    src += rows * cols;
  };
  auto put_t = [&](uint64_t rows, uint64_t cols, bf16* dst, long ldd) {  // transposed device copy
    ck(cudaMemcpyAsync(tmp.p, src, rows * cols * sizeof(float), cudaMemcpyHostToDevice, stream_), "params upload");
    k_f32_to_bf16_2d_t(tmp.as<float>(), cols, dst, ldd, rows, cols, stream_);
    ck(cudaStreamSynchronize(stream_), "params upload");
    src += rows * cols;
  };
  auto put_gain = [&](float* dst) {
    ck(cudaMemcpyAsync(dst, src, d_ * sizeof(float), cudaMemcpyHostToDevice, stream_), "params upload");
    src += d_;
  };
  put(V_, d_, emb_, d_);
  for (int64_t l = 0; l < L_; ++l) {
    put_gain(attn_g_[l]);
    put(d_, d_, wqkv_[l], 3 * d_);           // w_q -> columns [0, d)
    put(d_, d_, wqkv_[l] + d_, 3 * d_);      // w_k -> columns [d, 2d)
    put(d_, d_, wqkv_[l] + 2 * d_, 3 * d_);  // w_v -> columns [2d, 3d)
    put(d_, d_, wo_[l], d_);
    put_gain(mlp_g_[l]);
    put(d_, F_, win_[l], F_);
    put_t(F_, d_, wout_[l], F_);  // device layout W_out^T [d x F] (see forward_batch)
  }
  put_gain(final_g_);
  put(d_, V_, head_, V_);
  ck(cudaStreamSynchronize(stream_), "params upload");
}

void Engine::init_random(uint64_t seed) {
  DevBuf tmp;
  tmp.ensure(std::max<size_t>(V_ * d_, std::max<size_t>(3 * d_ * d_, d_ * F_)) * sizeof(float));
  uint64_t salt = 0;
  auto fill = [&](uint64_t rows, uint64_t cols, bf16* dst, long ldd) {
    k_init_normal(tmp.as<float>(), rows * cols, seed * 1000003ULL + (++salt), 0.02f, stream_);
    k_f32_to_bf16_2d(tmp.as<float>(), cols, dst, ldd, rows, cols, stream_);
  };
  fill(V_, d_, emb_, d_);
  for (int64_t l = 0; l < L_; ++l) {
    fill(d_, 3 * d_, wqkv_[l], 3 * d_);
    fill(d_, d_, wo_[l], d_);
    fill(d_, F_, win_[l], F_);
    fill(d_, F_, wout_[l], F_);  // W_out^T [d x F]
  }
  fill(d_, V_, head_, V_);
  k_fill(gainbuf_.as<float>(), (2 * L_ + 1) * d_, 1.0f, stream_);
  ck(cudaStreamSynchronize(stream_), "init_random");
}

void Engine::grads_zero() {
  ck(cudaMemsetAsync(grads_.p, 0, n_params_ * sizeof(float), stream_), "grads_zero");
  accum_count_ = 0;
}

void Engine::grads_download(float* out, uint64_t n) {
  if (n != n_params_) throw std::invalid_argument("grads download: wrong parameter count");
  ck(cudaMemcpyAsync(out, grads_.p, n * sizeof(float), cudaMemcpyDefault, stream_), "grads download");
  ck(cudaStreamSynchronize(stream_), "grads download");
}

// GradientStore<double> (model.hpp:76-81): the fp32 device gradients widened on the host.
void Engine::grads_download_f64(double* out, uint64_t n) {
  if (n != n_params_) throw std::invalid_argument("grads download: wrong parameter count");
  constexpr uint64_t kChunk = uint64_t(1) << 24;
  std::vector<float> tmp(std::min<uint64_t>(n, kChunk));
  for (uint64_t o = 0; o < n; o += kChunk) {
    const uint64_t m = std::min<uint64_t>(kChunk, n - o);
    ck(cudaMemcpyAsync(tmp.data(), grads_.as<float>() + o, m * sizeof(float), cudaMemcpyDeviceToHost, stream_),
       "grads download");
    ck(cudaStreamSynchronize(stream_), "grads download");
    for (uint64_t i = 0; i < m; ++i) out[o + i] = tmp[i];
  }
}

// ----------------------------------------------------------------------------- memory plan
ActLayout Engine::layout(int64_t n) const {
  ActLayout a;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += align_up(bytes);
    return r;
  };
  a.x = take(n * d_ * 4);
  a.inv1 = take(n * 4);
  a.n1 = take(n * d_ * 2);
  a.q = take(n * d_ * 2);
  a.attn = take(n * d_ * 2);
  a.lse = take(H_ * n * 4);
  a.xmid = take(n * d_ * 4);
  a.inv2 = take(n * 4);
  a.n2 = take(n * d_ * 2);
  a.h = take(n * F_ * 2);
  a.act = take(n * F_ * 2);
  a.per_layer = o;
  o = a.per_layer * L_;
  a.final_x = take(n * d_ * 4);
  a.invf = take(n * 4);
  a.nf = take(n * d_ * 2);
  a.total = o;
  return a;
}

void Engine::ensure_capacity(int64_t rows, size_t arena_bytes, int64_t max_n, int64_t max_loss_rows) {
  if (rows > rows_cap_) {
    if (!seg_stack_.empty()) throw std::runtime_error("engine: KV stack capacity exceeded with a live stack");
    rows_cap_ = rows;
    const size_t kvb = static_cast<size_t>(L_) * rows * d_;
    kst_.ensure(kvb * 2);
    vst_.ensure(kvb * 2);
    dkst_.ensure(kvb * 4);
    dvst_.ensure(kvb * 4);
    ck(cudaMemsetAsync(kst_.p, 0, kvb * 2, stream_), "K stack zero");
    ck(cudaMemsetAsync(vst_.p, 0, kvb * 2, stream_), "V stack zero");
    ck(cudaMemsetAsync(dkst_.p, 0, kvb * 4, stream_), "dK stack zero");
    ck(cudaMemsetAsync(dvst_.p, 0, kvb * 4, stream_), "dV stack zero");
  }
  if (arena_bytes > arena_.bytes) {
    if (!seg_stack_.empty()) throw std::runtime_error("engine: activation arena exceeded with a live stack");
    arena_.ensure(arena_bytes);
  }
  if (max_n > scratch_n_) {
    scratch_n_ = max_n;
    const size_t n = max_n;
    sc_gx_.ensure(n * d_ * 4);
    sc_gxb_.ensure(n * d_ * 2);
    sc_gxf_.ensure(n * d_ * 4);
    sc_gn_.ensure(n * d_ * 4);
    sc_gh_.ensure(n * F_ * 2);
    sc_dO_.ensure(n * d_ * 2);
    sc_D_.ensure(H_ * n * 4);
    sc_dq_.ensure(n * d_ * 4);
    sc_dqkv_.ensure(n * 3 * d_ * 2);
  }
  // LM-head / CE chunk: head_chunk_bytes_ of fp32 logits + bf16 dlogits at most, and no more than a
  // third of the memory still free after the buffers above (at least 2 GB)
  if (head_cap_rows_ == 0 && std::max<int64_t>(max_loss_rows, 1) > head_chunk_) {
    int64_t head_bytes = head_chunk_bytes_;
    size_t free_b = 0, total_b = 0;  // the query is slow: once, not per plan
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      const int64_t room = (static_cast<int64_t>(free_b) + static_cast<int64_t>(sc_logits_.bytes + sc_dlog_.bytes)) / 3;
      head_bytes = std::min<int64_t>(head_bytes, std::max<int64_t>(room, int64_t(2) << 30));
    } else {
      (void)cudaGetLastError();
    }
    head_cap_rows_ = std::max<int64_t>(128, head_bytes / (V_ * 6) / 128 * 128);
  }
  const int64_t cap = head_cap_rows_ > 0 ? head_cap_rows_ : std::max<int64_t>(128, head_chunk_bytes_ / (V_ * 6) / 128 * 128);
  const int64_t chunk = std::min<int64_t>(cap, std::max<int64_t>(max_loss_rows, 1));
  if (chunk > head_chunk_) {
    head_chunk_ = chunk;
    sc_nfl_.ensure(chunk * d_ * 2);
    sc_logits_.ensure(chunk * V_ * 4);
    sc_stats_.ensure(chunk * ((V_ + 31) / 32) * 8);
    sc_dlog_.ensure(chunk * V_ * 2);
    sc_gnf_.ensure(chunk * d_ * 4);
  }
}

uint64_t Engine::stack_tokens() const {
  return seg_stack_.empty() ? 0 : static_cast<uint64_t>(seg_stack_.back().S + seg_stack_.back().n);
}

// Host metadata of one batch: tokens/positions, attention work lists, loss CSR.
void Engine::build_meta(Batch& b, size_t& cursor, std::vector<char>& host) {
  auto put = [&](const void* src, size_t bytes) {
    const size_t off = cursor;
    cursor = align_up(cursor + bytes);
    if (host.capacity() < cursor) host.reserve(std::max(cursor, 2 * host.capacity()));
    if (host.size() < cursor) host.resize(cursor);
    if (bytes) std::memcpy(host.data() + off, src, bytes);
    return off;
  };
  b.qblk128.clear();
  b.kvit128.clear();
  b.kvit128_2.clear();
  for (size_t i = 0; i < b.seg_off.size(); ++i) {
    const int64_t so = b.seg_off[i], end = so + b.seg_len[i];
    for (int64_t q = so; q < end; q += kFwdBlockQ) {
      b.qblk128.insert(b.qblk128.end(), {int32_t(q), int32_t(std::min<int64_t>(q + kFwdBlockQ, end)), int32_t(so), 0});
    }
    // direct_kv (fused kernels): one item per own key block, so each own dK/dV row has a single
    // writer that stores it as bf16 into the packed operand (flag 2); else ranges of kQChunkOwn
    // queries accumulate into the fp32 stack rows (flag 1)
    const bool direct = b.direct_kv;
    const int64_t qchunk = direct ? std::max<int64_t>(b.seg_len[i], 1) : kQChunkOwn;
    for (int64_t kt = 0; kt < b.seg_len[i]; kt += kBwdBlockKV)
      for (int64_t q = so + kt; q < end; q += qchunk) {
        b.kvit128.insert(b.kvit128.end(), {int32_t(b.row0() + so + kt), int32_t(std::min<int64_t>(kBwdBlockKV, b.seg_len[i] - kt)),
                                           int32_t(q), int32_t(std::min<int64_t>(q + qchunk, end))});
        b.kvit128_2.insert(b.kvit128_2.end(), {int32_t(so), direct ? 2 : 1});
      }
  }
  // tcgen05 dK/dV items of the shared prefix rows: every query of every member attends them fully, so
  // one item spans members (fewer items: less per-item fixed cost and fewer red.add passes over the
  // same prefix dK/dV rows)
  {
    int64_t n_rows = 0;
    for (size_t i = 0; i < b.seg_off.size(); ++i) n_rows = std::max<int64_t>(n_rows, b.seg_off[i] + b.seg_len[i]);
    for (int64_t kv = 0; kv < b.S; kv += kBwdBlockKV)
      for (int64_t q = 0; q < n_rows; q += kQChunkPrefix) {
        b.kvit128.insert(b.kvit128.end(), {int32_t(b.pbase + kv), int32_t(std::min<int64_t>(kBwdBlockKV, b.S - kv)), int32_t(q),
                                           int32_t(std::min<int64_t>(q + kQChunkPrefix, n_rows))});
        b.kvit128_2.insert(b.kvit128_2.end(), {0, 0});
      }
  }
  {
    // longest first: the persistent dK/dV kernel deals items to CTAs in snake order (~LPT balance)
    const size_t ni = b.kvit128.size() / 4;
    std::vector<int32_t> order(ni);
    for (size_t i = 0; i < ni; ++i) order[i] = static_cast<int32_t>(i);
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
      return b.kvit128[4 * x + 3] - b.kvit128[4 * x + 2] > b.kvit128[4 * y + 3] - b.kvit128[4 * y + 2];
    });
    std::vector<int32_t> k4(ni * 4), k2(ni * 2);
    for (size_t i = 0; i < ni; ++i) {
      std::memcpy(&k4[4 * i], &b.kvit128[4 * order[i]], 16);
      std::memcpy(&k2[2 * i], &b.kvit128_2[2 * order[i]], 8);
    }
    b.kvit128.swap(k4);
    b.kvit128_2.swap(k2);
  }
  b.o_tok = put(b.tokens.data(), b.tokens.size() * 4);
  b.o_pos = put(b.positions.data(), b.positions.size() * 4);
  b.o_qblk128 = put(b.qblk128.data(), b.qblk128.size() * 4);
  b.o_kvit128 = put(b.kvit128.data(), b.kvit128.size() * 4);
  b.o_kvit128_2 = put(b.kvit128_2.data(), b.kvit128_2.size() * 4);
  b.o_lrows = put(b.loss_rows.data(), b.loss_rows.size() * 4);
  b.o_poff = put(b.pair_off.data(), b.pair_off.size() * 4);
  b.o_ptgt = put(b.pair_tgt.data(), b.pair_tgt.size() * 4);
  b.o_pw = put(b.pair_w.data(), b.pair_w.size() * 8);
}


size_t Engine::upload_staged(const std::vector<char>& host, DevBuf& dst) {
  const size_t bytes = std::max(host.size(), kAlign);
  dst.ensure(bytes);
  ck(cudaStreamSynchronize(stream_), "meta staging");
  if (bytes > meta_host_cap_) {
    if (meta_host_) cudaFreeHost(meta_host_);
    meta_host_ = nullptr;
    ck(cudaMallocHost(&meta_host_, bytes), "cudaMallocHost meta");
    meta_host_cap_ = bytes;
  }
  if (!host.empty()) {
    std::memcpy(meta_host_, host.data(), host.size());
    ck(cudaMemcpyAsync(dst.p, meta_host_, host.size(), cudaMemcpyHostToDevice, stream_), "meta upload");
  }
  return host.size();
}

void Engine::upload_meta(std::vector<Batch*>& batches) {
  std::vector<char> host;
  size_t cursor = 0;
  for (Batch* b : batches) build_meta(*b, cursor, host);
  upload_staged(host, meta_);
  cur_meta_ = meta_.as<char>();
}

cudaEvent_t Engine::event() {
  if (event_next_ == event_pool_.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    event_pool_.push_back(e);
  }
  return event_pool_[event_next_++];
}

void Engine::collect_profile() {
  for (auto& p : pending_) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, p.a, p.b), "cudaEventElapsedTime");
    kstats_.ms[p.cls] += ms;
    kstats_.flops[p.cls] += p.flops;
    kstats_.bytes[p.cls] += p.bytes;
    kstats_.launches[p.cls] += 1;
    if (!p.tag.empty()) {
      TagStat& ts = tag_stats_[p.tag];
      ts.ms += ms;
      ts.flops += p.flops;
      ts.bytes += p.bytes;
      ts.n += 1;
    }
  }
  pending_.clear();
  event_next_ = 0;
}

std::string Engine::gemm_profile_text() const {
  std::vector<std::pair<std::string, TagStat>> v(tag_stats_.begin(), tag_stats_.end());
  std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.second.ms > b.second.ms; });
  std::string out;
  for (const auto& [tag, st] : v) {
    char line[256];
    if (st.flops > 0)
      std::snprintf(line, sizeof(line), "%10.3f ms  n=%6llu  %7.1f TFLOP/s  %s\n", st.ms,
                    static_cast<unsigned long long>(st.n), st.flops / (st.ms * 1e-3) / 1e12, tag.c_str());
    else
      std::snprintf(line, sizeof(line), "%10.3f ms  n=%6llu  %7.1f GB/s     %s\n", st.ms,
                    static_cast<unsigned long long>(st.n), st.bytes / (st.ms * 1e-3) / 1e9, tag.c_str());
    out += line;
  }
  return out;
}

// GEMM launch: algorithmic FLOPs 2MNK; algorithmic bytes = operands once + output (x2 if RMW).
void Engine::gemm(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const EpiParams& e, int splits) {
  double out_b = 2.0;
  if (e.mode == EPI_STORE_F32 || e.mode == EPI_STORE_F32_STATS) out_b = 4.0;
  if (e.mode == EPI_STORE_BF16_STATS) out_b = 2.0;
  if (e.mode == EPI_ADD_F32 || e.mode == EPI_RESID_F32) out_b = 8.0;
  if (e.mode == EPI_SILU || e.mode == EPI_DSILU) out_b = 4.0;
  const double bytes = 2.0 * (double(M) * K + double(N) * K) + out_b * double(M) * N;
  if (profiling_) {
    pending_tag_ = std::to_string(M) + "x" + std::to_string(N) + "x" + std::to_string(K) + (A.mn_major ? " A:mn" : " A:k") +
                   (B.mn_major ? " B:mn" : " B:k") + " epi" + std::to_string(e.mode) + " s" + std::to_string(splits) +
                   (e.mode == EPI_ADD_F32 && e.split_w == 0 && gemm_prefer_transposed(M, N, K) ? " T" : "");
  }
  run(KC_GEMM, 2.0 * M * N * K, bytes, [&] { gemm_bf16(A, B, M, N, K, e, splits, stream_); });
}

// ----------------------------------------------------------------------------- push (forward_segment)
void Engine::forward_batch(const Batch& b, size_t arena_off) {
  const int n = static_cast<int>(b.n);
  set_pdl(pdl_ == 1 || (pdl_ == 2 && static_cast<double>(b.n) * d_ <= pdl_auto_elems_));
  const int d = static_cast<int>(d_), F = static_cast<int>(F_);
  const double nd = double(n) * d_;
  const ActLayout lay = layout(b.n);
  char* base = arena_.as<char>(arena_off);
  auto X = [&](int64_t l) {
    return reinterpret_cast<float*>(l == L_ ? base + lay.final_x : base + l * lay.per_layer + lay.x);
  };
  const size_t kv_layer = static_cast<size_t>(rows_cap_) * d_;
  const float scale = 1.0f / std::sqrt(static_cast<float>(dh_));  // model.hpp:345

  tag("k_embed_pe");
  run(KC_ELEMWISE, 0, nd * 10, [&] {
    k_embed_pe(meta<int32_t>(b.o_tok), meta<int32_t>(b.o_pos), emb_, pe_.as<float>(), X(0), n, d, stream_);
  });
  for (int64_t l = 0; l < L_; ++l) {
    char* Lb = base + l * lay.per_layer;
    float* inv1 = reinterpret_cast<float*>(Lb + lay.inv1);
    bf16* n1 = reinterpret_cast<bf16*>(Lb + lay.n1);
    bf16* q = reinterpret_cast<bf16*>(Lb + lay.q);
    bf16* attn = reinterpret_cast<bf16*>(Lb + lay.attn);
    float* lse = reinterpret_cast<float*>(Lb + lay.lse);
    float* xmid = reinterpret_cast<float*>(Lb + lay.xmid);
    float* inv2 = reinterpret_cast<float*>(Lb + lay.inv2);
    bf16* n2 = reinterpret_cast<bf16*>(Lb + lay.n2);
    bf16* h = reinterpret_cast<bf16*>(Lb + lay.h);
    bf16* act = reinterpret_cast<bf16*>(Lb + lay.act);
    bf16* K = kst_.as<bf16>() + l * kv_layer;
    bf16* Vv = vst_.as<bf16>() + l * kv_layer;

    tag("k_rmsnorm_fwd");
    run(KC_ELEMWISE, 0, nd * 6, [&] { k_rmsnorm_fwd(X(l), attn_g_[l], inv1, n1, n, d, stream_); });  // :376-380
    {  // q,k,v = normed W{q,k,v}; k,v written straight onto the stack rows [S, S+n)  (:381-384)
      EpiParams e;
      e.mode = EPI_STORE_BF16;
      e.split_w = d;
      e.out[0] = q;
      e.out[1] = K + b.row0() * d_;
      e.out[2] = Vv + b.row0() * d_;
      e.ldo[0] = e.ldo[1] = e.ldo[2] = d;
      gemm(op(n1, d, false), op(wqkv_[l], 3 * d, true), n, 3 * d, d, e, 1);
    }
    {  // segment attention over the stack (:386-408)
      AttnFwdArgs a;
      a.q = q;
      a.ldq = d;
      a.k = K;
      a.v = Vv;
      a.ldkv = d;
      a.o = attn;
      a.ldo = d;
      a.lse = lse;
      a.n = n;
      a.H = static_cast<int>(H_);
      a.dh = static_cast<int>(dh_);
      a.S = static_cast<int>(b.S);
      a.pbase = static_cast<int>(b.pbase);
      a.r0 = static_cast<int>(b.row0());
      a.scale = scale;
      a.qblocks = meta<int4>(b.o_qblk128);
      a.nqb = static_cast<int>(b.qblk128.size() / 4);
      tag("attn_fwd_sm100");
      run(KC_ATTN_FWD, 4.0 * d_ * b.attn_ctx, 0, [&] { attn_fwd_sm100(a, rows_cap_, stream_); });
    }
    {  // x_mid = x + attn W_o  (:410-411,427-428)
      EpiParams e;
      e.mode = EPI_RESID_F32;
      e.out[0] = xmid;
      e.ldo[0] = d;
      e.resid = X(l);
      e.ld_resid = d;
      gemm(op(attn, d, false), op(wo_[l], d, true), n, d, d, e, 1);
    }
    tag("k_rmsnorm_fwd");
    run(KC_ELEMWISE, 0, nd * 6, [&] { k_rmsnorm_fwd(xmid, mlp_g_[l], inv2, n2, n, d, stream_); });  // :430-434
    {  // h = normed W_in, act = silu(h)  (:435-444)
      EpiParams e;
      e.mode = EPI_SILU;
      e.out[0] = h;
      e.ldo[0] = F;
      e.out2 = act;
      e.ldo2 = F;
      gemm(op(n2, d, false), op(win_[l], F, true), n, F, d, e, 1);
    }
    {  // x_out = x_mid + act W_out  (:445-448)
      EpiParams e;
      e.mode = EPI_RESID_F32;
      e.out[0] = X(l + 1);
      e.ldo[0] = d;
      e.resid = xmid;
      e.ld_resid = d;
      // W_out is kept transposed on the device ([d x F], K-major B): the N = d output then tiles with
      // the 224-wide pair tiles at d = 896; the grad_hidden GEMM reads it MN-major instead
      gemm(op(act, F, false), op(wout_[l], F, false), n, d, F, e, 1);
    }
  }
  tag("k_rmsnorm_fwd");
  run(KC_ELEMWISE, 0, nd * 6, [&] {  // final norm (:451-455)
    k_rmsnorm_fwd(X(L_), final_g_, reinterpret_cast<float*>(base + lay.invf), reinterpret_cast<bf16*>(base + lay.nf),
                  n, d, stream_);
  });
}

// ----------------------------------------------------------------------------- visit: LM head + weighted CE
// For every loss row (compacted): logits = c W_head (fp32), CE -> loss (fp64) and dlogits (bf16),
// dW_head += c^T dlogits, grad_c = dlogits W_head^T scattered back to the batch rows.
void Engine::head_backward(const Batch& b, const bf16* nf, bool loss_only) {
  const int d = static_cast<int>(d_);
  const int V = static_cast<int>(V_);
  float* gxf = sc_gxf_.as<float>();
  const int64_t m = static_cast<int64_t>(b.loss_rows.size());
  bf16* dlog = sc_dlog_.as<bf16>();
  bf16* nfl = sc_nfl_.as<bf16>();
  float* gnf = sc_gnf_.as<float>();
  // equal chunks (multiples of 128 rows) rather than full ones plus a short tail
  const int64_t nch = (m + head_chunk_ - 1) / head_chunk_;
  const int64_t per = nch <= 1 ? head_chunk_ : std::min<int64_t>(head_chunk_, ((m + nch - 1) / nch + 127) / 128 * 128);
  for (int64_t c0 = 0; c0 < m; c0 += per) {
    const int cm = static_cast<int>(std::min<int64_t>(per, m - c0));
    tag("k_gather_rows_bf16");
    run(KC_ELEMWISE, 0, 4.0 * cm * d, [&] { k_gather_rows_bf16(nf, meta<int32_t>(b.o_lrows) + c0, nfl, cm, d, stream_); });
    const bool lbf = ce_stats_ && logits_bf16_;
    {
      EpiParams e;  // logits = normed_final W_head (model.hpp:460-461) + per-row softmax stats
      e.mode = lbf ? EPI_STORE_BF16_STATS : (ce_stats_ ? EPI_STORE_F32_STATS : EPI_STORE_F32);
      e.out[0] = sc_logits_.p;
      e.ldo[0] = V;
      e.out2 = sc_stats_.p;
      e.ldo2 = (V + 31) / 32;
      gemm(op(nfl, d, false), op(head_, V, true), cm, V, d, e, 1);
    }
    tag("k_ce");
    run(KC_CE, 0, (lbf ? 4.0 : 6.0) * cm * V, [&] {  // weighted_nll (model.hpp:643-677), multi-target rows
      if (lbf)
        k_ce_bf16(sc_logits_.as<bf16>(), cm, V, meta<int32_t>(b.o_poff) + c0, meta<int32_t>(b.o_ptgt),
                  meta<double>(b.o_pw), dlog, loss_.as<double>(), stream_, sc_stats_.as<float2>(), (V + 31) / 32);
      else
        k_ce(sc_logits_.as<float>(), cm, V, meta<int32_t>(b.o_poff) + c0, meta<int32_t>(b.o_ptgt), meta<double>(b.o_pw),
             dlog, loss_.as<double>(), stream_, ce_stats_ ? sc_stats_.as<float2>() : nullptr, (V + 31) / 32);
    });
    if (loss_only) continue;  // the VISIT of a segment-level caller: loss now, gradients at the pop
    {  // dW_head += c^T dlogits  (model.hpp:506)
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = g_head_;
      e.ldo[0] = V;
      gemm(op(nfl, d, true), op(dlog, V, true), d, V, cm, e, gemm_choose_splits(d, V, cm));
    }
    {  // grad_c = dlogits W_head^T  (model.hpp:507-508)
      ck(cudaMemsetAsync(gnf, 0, static_cast<size_t>(cm) * d_ * 4, stream_), "memset");
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = gnf;
      e.ldo[0] = d;
      gemm(op(dlog, V, false), op(head_, V, false), cm, d, V, e, gemm_choose_splits(cm, d, V));
    }
    tag("k_scatter_rows_f32");
    run(KC_ELEMWISE, 0, 8.0 * cm * d, [&] { k_scatter_rows_f32(gnf, meta<int32_t>(b.o_lrows) + c0, gxf, cm, d, stream_); });
  }
}

// Segment API: caller-provided upstream grad_logits [n x V] (BackwardUpstream, model.hpp:465-469).
void Engine::head_backward_dense(const Batch& b, const bf16* nf, const float* host_grad_logits) {
  const int d = static_cast<int>(d_);
  const int V = static_cast<int>(V_);
  float* gxf = sc_gxf_.as<float>();
  bf16* dlog = sc_dlog_.as<bf16>();
  for (int64_t c0 = 0; c0 < b.n; c0 += head_chunk_) {
    const int cm = static_cast<int>(std::min<int64_t>(head_chunk_, b.n - c0));
    ck(cudaMemcpyAsync(sc_logits_.p, host_grad_logits + c0 * V_, static_cast<size_t>(cm) * V_ * 4,
                       cudaMemcpyDefault, stream_),
       "grad_logits upload");
    tag("k_f32_to_bf16_2d");
    run(KC_ELEMWISE, 0, 6.0 * cm * V, [&] { k_f32_to_bf16_2d(sc_logits_.as<float>(), V, dlog, V, cm, V, stream_); });
    {
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = g_head_;
      e.ldo[0] = V;
      gemm(op(nf + c0 * d_, d, true), op(dlog, V, true), d, V, cm, e, gemm_choose_splits(d, V, cm));
    }
    {
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = gxf + c0 * d_;
      e.ldo[0] = d;
      gemm(op(dlog, V, false), op(head_, V, false), cm, d, V, e, gemm_choose_splits(cm, d, V));
    }
  }
}

// ----------------------------------------------------------------------------- pop (backward_segment)
void Engine::backward_batch(const Batch& b, size_t arena_off, const float* host_grad_logits, float* grad_prefix) {
  const int n = static_cast<int>(b.n);
  set_pdl(pdl_ == 1 || (pdl_ == 2 && static_cast<double>(b.n) * d_ <= pdl_auto_elems_));
  const int d = static_cast<int>(d_), F = static_cast<int>(F_);
  const double nd = double(n) * d_;
  const ActLayout lay = layout(b.n);
  char* base = arena_.as<char>(arena_off);
  auto X = [&](int64_t l) {
    return reinterpret_cast<float*>(l == L_ ? base + lay.final_x : base + l * lay.per_layer + lay.x);
  };
  const size_t kv_layer = static_cast<size_t>(rows_cap_) * d_;
  const float scale = 1.0f / std::sqrt(static_cast<float>(dh_));
  float* gx = sc_gx_.as<float>();
  bf16* gxb = sc_gxb_.as<bf16>();
  float* gxf = sc_gxf_.as<float>();
  float* gn = sc_gn_.as<float>();
  // grad_normed (the dX GEMM output the RMSNorm backward consumes once) in bf16 where the TMA-fed
  // RMSNorm backward takes it (d % 8 == 0, d <= 4096): 16 instead of 18 bytes per element there and
  // half the GEMM's store; the residual gradient it is added into stays fp32
  const bool gn16 = gn_bf16_ && rmsnorm_bwd_bf16_gy_ok(d);
  bf16* gnb = sc_gn_.as<bf16>();
  auto norm_bwd = [&](const float* x, const float* inv, const float* gain, float* ggain) {
    if (gn16) k_rmsnorm_bwd(gnb, x, inv, gain, gx, gx, gxb, ggain, n, d, stream_);
    else k_rmsnorm_bwd(gn, x, inv, gain, gx, gx, gxb, ggain, n, d, stream_);
  };
  bf16* gh = sc_gh_.as<bf16>();
  bf16* dO = sc_dO_.as<bf16>();
  float* dq = sc_dq_.as<float>();
  bf16* dqkv = sc_dqkv_.as<bf16>();
  const bf16* nf = reinterpret_cast<const bf16*>(base + lay.nf);

  ck(cudaMemsetAsync(gxf, 0, static_cast<size_t>(n) * d_ * 4, stream_), "memset");
  if (b.full_logits) {
    if (host_grad_logits) head_backward_dense(b, nf, host_grad_logits);
  } else {
    head_backward(b, nf);
  }
  tag("k_rmsnorm_bwd");
  run(KC_ELEMWISE, 0, nd * 14, [&] {  // final-norm backward (model.hpp:509-511)
    k_rmsnorm_bwd(gxf, X(L_), reinterpret_cast<const float*>(base + lay.invf), final_g_, nullptr, gx, gxb, g_final_g_,
                  n, d, stream_);
  });

  for (int64_t l = L_ - 1; l >= 0; --l) {
    char* Lb = base + l * lay.per_layer;
    const float* inv1 = reinterpret_cast<const float*>(Lb + lay.inv1);
    const bf16* n1 = reinterpret_cast<const bf16*>(Lb + lay.n1);
    const bf16* q = reinterpret_cast<const bf16*>(Lb + lay.q);
    const bf16* attn = reinterpret_cast<const bf16*>(Lb + lay.attn);
    const float* lse = reinterpret_cast<const float*>(Lb + lay.lse);
    const float* xmid = reinterpret_cast<const float*>(Lb + lay.xmid);
    const float* inv2 = reinterpret_cast<const float*>(Lb + lay.inv2);
    const bf16* n2 = reinterpret_cast<const bf16*>(Lb + lay.n2);
    const bf16* h = reinterpret_cast<const bf16*>(Lb + lay.h);
    const bf16* act = reinterpret_cast<const bf16*>(Lb + lay.act);
    const bf16* K = kst_.as<bf16>() + l * kv_layer;
    const bf16* Vv = vst_.as<bf16>() + l * kv_layer;
    float* dK = dkst_.as<float>() + l * kv_layer;
    float* dV = dvst_.as<float>() + l * kv_layer;

    {  // dW_out += act^T gx  (model.hpp:524)
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = g_wout_[l];
      e.ldo[0] = d;
      gemm(op(act, F, true), op(gxb, d, true), F, d, n, e, gemm_choose_splits(F, d, n));
    }
    {  // grad_hidden = (gx W_out^T) * silu'(h)  (model.hpp:525-528)
      EpiParams e;
      e.mode = EPI_DSILU;
      e.out[0] = gh;
      e.ldo[0] = F;
      e.aux = h;
      e.ld_aux = F;
      gemm(op(gxb, d, false), op(wout_[l], F, true), n, F, d, e, 1);
    }
    {  // dW_in += normed2^T grad_hidden  (model.hpp:533)
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = g_win_[l];
      e.ldo[0] = F;
      gemm(op(n2, d, true), op(gh, F, true), d, F, n, e, gemm_choose_splits(d, F, n));
    }
    {  // grad_normed2 = grad_hidden W_in^T  (model.hpp:535)
      EpiParams e;
      e.mode = gn16 ? EPI_STORE_BF16 : EPI_STORE_F32;
      e.out[0] = gn;
      e.ldo[0] = d;
      gemm(op(gh, F, false), op(win_[l], F, false), n, d, F, e, 1);
    }
    tag("k_rmsnorm_bwd");
    run(KC_ELEMWISE, 0, nd * (gn16 ? 16 : 18), [&] {  // gx_mid = gx + rmsnorm_bwd (model.hpp:536-539)
      norm_bwd(xmid, inv2, mlp_g_[l], g_mlp_g_[l]);
    });
    {  // dW_o += attn^T gx_mid  (model.hpp:542)
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.out[0] = g_wo_[l];
      e.ldo[0] = d;
      gemm(op(attn, d, true), op(gxb, d, true), d, d, n, e, gemm_choose_splits(d, d, n));
    }
    {  // grad_attn = gx_mid W_o^T  (model.hpp:543-544)
      EpiParams e;
      e.mode = EPI_STORE_BF16;
      e.out[0] = dO;
      e.ldo[0] = d;
      gemm(op(gxb, d, false), op(wo_[l], d, false), n, d, d, e, 1);
    }
    // attention backward (model.hpp:546-604): dQ, and dK/dV added into the stack rows [0, S+n)
    {
      AttnBwdArgs a;
      a.q = q;
      a.dO = dO;
      a.o = attn;
      a.ldq = d;
      a.k = K;
      a.v = Vv;
      a.ldkv = d;
      a.lse = lse;
      a.D = sc_D_.as<float>();
      a.dq = dq;
      a.lddq = d;
      a.dk = dK;
      a.dv = dV;
      a.lddkv = d;
      if (grad_prefix) {  // segment pop: this pop's prefix dK/dV into [L][2][S][d] (rows from pbase = 0)
        a.dk_pre = grad_prefix + (2 * l) * b.S * d_;
        a.dv_pre = grad_prefix + (2 * l + 1) * b.S * d_;
      }
      a.n = n;
      a.H = static_cast<int>(H_);
      a.dh = static_cast<int>(dh_);
      a.S = static_cast<int>(b.S);
      a.pbase = static_cast<int>(b.pbase);
      a.r0 = static_cast<int>(b.row0());
      a.scale = scale;
      if (b.direct_kv) {  // own rows' dK / dV straight into the packed operand (bf16)
        a.dkv16 = dqkv + d;
        a.lddkv16 = 3 * d;
      }
      // fused kernels (dh 64 and 128): dQ partials (one per key block) reduced into the fp32 accumulator,
      // which the D pre-pass zeroes (no memset node between the kernels)
      tag("attn_bwd_sm100");
      run(KC_ATTN_BWD, 8.0 * d_ * b.attn_ctx, 0, [&] {
        attn_bwd_sm100(a, rows_cap_, meta<int4>(b.o_kvit128), meta<int2>(b.o_kvit128_2),
                       static_cast<int>(b.kvit128.size() / 4), stream_);
      });
      launches_ += 1;  // + the D pre-pass
    }
    // pop: consume this batch's dK/dV rows (children + own contributions), zero them for reuse
    if (b.direct_kv) {
      tag("k_pack_dq");  // dK / dV are already in the operand; the stack rows were never written
      run(KC_ELEMWISE, 0, nd * 6, [&] { k_pack_dqkv(dq, nullptr, nullptr, dqkv, n, d, stream_); });
    } else {
      tag("k_pack_dqkv");
      run(KC_ELEMWISE, 0, nd * 26, [&] { k_pack_dqkv(dq, dK + b.row0() * d_, dV + b.row0() * d_, dqkv, n, d, stream_); });
    }
    {  // dW_{q,k,v} += normed1^T [dq | dk | dv]  (model.hpp:610-612)
      EpiParams e;
      e.mode = EPI_ADD_F32;
      e.split_w = d;
      e.out[0] = g_wq_[l];
      e.out[1] = g_wk_[l];
      e.out[2] = g_wv_[l];
      e.ldo[0] = e.ldo[1] = e.ldo[2] = d;
      gemm(op(n1, d, true), op(dqkv, 3 * d, true), d, 3 * d, n, e, gemm_choose_splits(d, 3 * d, n));
    }
    {  // grad_normed1 = dq W_q^T + dk W_k^T + dv W_v^T  (model.hpp:613-618)
      EpiParams e;
      e.mode = gn16 ? EPI_STORE_BF16 : EPI_STORE_F32;
      e.out[0] = gn;
      e.ldo[0] = d;
      gemm(op(dqkv, 3 * d, false), op(wqkv_[l], 3 * d, false), n, d, 3 * d, e, 1);
    }
    tag("k_rmsnorm_bwd");
    run(KC_ELEMWISE, 0, nd * (gn16 ? 16 : 18), [&] {  // gx = gx_mid + rmsnorm_bwd (model.hpp:620-624)
      norm_bwd(X(l), inv1, attn_g_[l], g_attn_g_[l]);
    });
  }
  tag("k_embed_grad");
  run(KC_ELEMWISE, 0, nd * 12, [&] { k_embed_grad(gx, meta<int32_t>(b.o_tok), g_emb_, n, d, stream_); });  // :627-630
  accum_count_ += b.accum_inc;
}

// ----------------------------------------------------------------------------- tree_train_step
// Device bytes one more token of a pushed batch costs: activations (per layer 16d + 4F + 4H + 8,
// plus the final norm), its K/V (bf16) + dK/dV (fp32) stack rows, and pop scratch.
double Engine::bytes_per_token() const {
  const double d = double(d_), F = double(F_), H = double(H_), L = double(L_);
  const double act = L * (16 * d + 4 * F + 4 * H + 8) + 6 * d + 4;
  const double stack = 12 * L * d;
  const double scratch = 26 * d + 2 * F + 4 * H;
  return act + stack + scratch;
}

// Sibling-batch token budget that keeps the step inside HBM: what is free now (plus what this
// engine already holds and can re-purpose) minus the resident path, a head-chunk + safety margin.
uint64_t Engine::auto_batch_budget(uint64_t path_tokens) const {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    (void)cudaGetLastError();
    return 8192;
  }
  const double held = double(arena_.bytes + kst_.bytes + vst_.bytes + dkst_.bytes + dvst_.bytes + sc_gx_.bytes +
                             sc_gxb_.bytes + sc_gxf_.bytes + sc_gn_.bytes + sc_gh_.bytes + sc_dO_.bytes + sc_D_.bytes +
                             sc_dq_.bytes + sc_dqkv_.bytes);
  const double per_tok = bytes_per_token();
  // 6 GB: a 2 GB LM-head chunk + slack; the head chunk grows past 2 GB only into memory left free
  // after the plan's own buffers (ensure_buffers)
  const double avail = 0.85 * (double(free_b) + held) - 6e9 - double(path_tokens) * per_tok;
  const double tok = avail / per_tok;
  return tok < 2048 ? 2048 : static_cast<uint64_t>(tok);
}

std::unique_ptr<StepPlan> Engine::prepare(const PrefixTree& tree, const tt_sched_config& sc, bool transient) {
  const bool timing = plan_timing_;  // option "plan_timing": host-phase timing of prepare() on stderr
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_start = now();
  if (tree.nodes[0].max_path_below > cfg_.max_position)
    throw std::invalid_argument("tree_train_step: path exceeds max_position");
  // every token is both an embedding row and (as the next token of its predecessor) a CE target:
  // reject ids outside [0, V) before anything is uploaded (model.hpp:343,653)
  for (const auto& nd : tree.nodes)
    for (int32_t t : nd.tokens)
      if (t < 0 || static_cast<uint64_t>(t) >= cfg_.vocab_size)
        throw std::invalid_argument("tree_train_step: token id out of vocab range");
  auto plan = std::make_unique<StepPlan>();
  plan->owner = this;
  auto& batches = plan->batches;
  auto& ops = plan->ops;
  const auto pre = preorder(tree);
  std::vector<int32_t> pid(tree.nodes.size(), -1);
  for (size_t i = 0; i < pre.size(); ++i) pid[pre[i]] = static_cast<int32_t>(i);

  // ---- batches + PUSH/POP op list in DFS order
  auto make_batch = [&](const std::vector<int32_t>& members, int64_t S) {
    Batch b;
    b.S = S;
    b.nodes = members;
    int64_t off = 0;
    for (int32_t u : members) {
      const auto& nd = tree.nodes[u];
      const int64_t len = static_cast<int64_t>(nd.tokens.size());
      b.seg_off.push_back(off);
      b.seg_len.push_back(len);
      b.attn_ctx += double(len) * double(S) + 0.5 * double(len) * double(len + 1);
      for (int64_t t = 0; t < len; ++t) {
        b.tokens.push_back(nd.tokens[t]);
        b.positions.push_back(static_cast<int32_t>(S + t));
      }
      LossPairs lp = node_loss_pairs(tree, u, S);  // rows are non-decreasing within a node
      for (size_t k = 0; k < lp.rows.size(); ++k) {
        const int32_t row = static_cast<int32_t>(off + lp.rows[k]);
        if (b.loss_rows.empty() || b.loss_rows.back() != row) {
          b.loss_rows.push_back(row);
          b.pair_off.push_back(static_cast<int32_t>(b.pair_tgt.size()));
        }
        b.pair_tgt.push_back(lp.targets[k]);
        b.pair_w.push_back(lp.weights[k]);
      }
      off += len;
    }
    b.pair_off.push_back(static_cast<int32_t>(b.pair_tgt.size()));
    b.n = off;
    b.accum_inc = static_cast<int>(members.size());
    batches.push_back(std::move(b));
    return static_cast<int>(batches.size() - 1);
  };
  std::string& trace = plan->trace;
  const uint64_t budget = (sc.batch_token_budget == 0 && sc.sibling_batch)
                              ? auto_batch_budget(tree.nodes[0].max_path_below +
                                                  static_cast<uint64_t>(std::max<int64_t>(root_batch_tokens_, 0)))
                              : sc.batch_token_budget;
  // chunk [a, b) of node u (S = the node's start): a chained sub-segment (chunked backward,
  // SPEC.md:234-251); the loss pairs of rows in [a, b) move with it
  auto make_chunk = [&](int32_t u, int64_t S, int64_t a, int64_t e, int accum_inc) {
    Batch b;
    b.S = S + a;
    b.n = e - a;
    b.nodes = {u};
    b.accum_inc = accum_inc;
    b.seg_off = {0};
    b.seg_len = {b.n};
    b.attn_ctx = double(b.n) * double(b.S) + 0.5 * double(b.n) * double(b.n + 1);
    const auto& nd = tree.nodes[u];
    for (int64_t t = a; t < e; ++t) {
      b.tokens.push_back(nd.tokens[t]);
      b.positions.push_back(static_cast<int32_t>(S + t));
    }
    LossPairs lp = node_loss_pairs(tree, u, S);
    for (size_t k = 0; k < lp.rows.size(); ++k) {
      if (lp.rows[k] < a || lp.rows[k] >= e) continue;
      const int32_t row = static_cast<int32_t>(lp.rows[k] - a);
      if (b.loss_rows.empty() || b.loss_rows.back() != row) {
        b.loss_rows.push_back(row);
        b.pair_off.push_back(static_cast<int32_t>(b.pair_tgt.size()));
      }
      b.pair_tgt.push_back(lp.targets[k]);
      b.pair_w.push_back(lp.weights[k]);
    }
    b.pair_off.push_back(static_cast<int32_t>(b.pair_tgt.size()));
    batches.push_back(std::move(b));
    return static_cast<int>(batches.size() - 1);
  };
  const uint64_t chunk = sc.chunk_len;
  auto short_leaf = [&](int32_t c) {
    return tree.nodes[c].children.empty() && (chunk == 0 || tree.nodes[c].tokens.size() <= chunk);
  };
  // one or more batches of consecutive short-leaf children of `parent` (sibling batching), pushed and
  // popped in turn; prefix rows [pbase, pbase + S), own rows from R0 (< 0: right after the prefix)
  auto leaf_runs = [&](const std::vector<int32_t>& ch, size_t i, size_t i_end, int64_t S, int64_t pbase,
                       int64_t R0) {
    while (i < i_end) {
      std::vector<int32_t> run_nodes = {ch[i]};
      uint64_t tok = tree.nodes[ch[i]].tokens.size();
      size_t j = i + 1;
      while (j < i_end && (budget == 0 || tok + tree.nodes[ch[j]].tokens.size() <= budget)) {
        tok += tree.nodes[ch[j]].tokens.size();
        run_nodes.push_back(ch[j++]);
      }
      const int bi = make_batch(run_nodes, S);
      batches[bi].leaf_batch = true;
      batches[bi].direct_kv = true;
      batches[bi].pbase = pbase;
      batches[bi].R0 = R0;
      ops.push_back({bi, OP_FWD, 0});
      ops.push_back({bi, OP_BWD, 0});
      for (int32_t m : run_nodes) trace += "PUSH " + std::to_string(pid[m]) + "\nPOP " + std::to_string(pid[m]) + "\n";
      i = j;
    }
  };
  // a forest root that can join a multi-root batch: unchunked, with children that are all short leaves
  auto root_groupable = [&](int32_t c) {
    const auto& nd = tree.nodes[c];
    if (nd.children.empty() || (chunk != 0 && nd.tokens.size() > chunk)) return false;
    for (int32_t g : nd.children)
      if (!short_leaf(g)) return false;
    return true;
  };
  std::function<void(int32_t, int64_t)> visit = [&](int32_t u, int64_t S) {
    const auto& ch = tree.nodes[u].children;
    size_t i = 0;
    while (i < ch.size()) {
      const int32_t c = ch[i];
      const int64_t len = static_cast<int64_t>(tree.nodes[c].tokens.size());
      if (u == 0 && S == 0 && sc.sibling_batch && root_batch_tokens_ > 0 && root_groupable(c)) {
        // multi-root batch: the prompts of several trees share one push (larger GEMM M, fewer
        // launches); each root's leaf batches then see only that root's rows as their prefix
        std::vector<int32_t> roots = {c};
        int64_t tok = len;
        size_t j = i + 1;
        while (j < ch.size() && root_groupable(ch[j]) &&
               tok + static_cast<int64_t>(tree.nodes[ch[j]].tokens.size()) <= root_batch_tokens_) {
          tok += static_cast<int64_t>(tree.nodes[ch[j]].tokens.size());
          roots.push_back(ch[j++]);
        }
        const int bi = make_batch(roots, 0);
        const int64_t n_roots = batches[bi].n;
        ops.push_back({bi, OP_FWD, 0});
        int64_t off = 0;
        for (int32_t r : roots) {
          const int64_t rl = static_cast<int64_t>(tree.nodes[r].tokens.size());
          const auto& rch = tree.nodes[r].children;
          trace += "PUSH " + std::to_string(pid[r]) + "\n";
          leaf_runs(rch, 0, rch.size(), rl, off, n_roots);
          trace += "POP " + std::to_string(pid[r]) + "\n";
          off += rl;
        }
        ops.push_back({bi, OP_BWD, 0});
        i = j;
      } else if (sc.sibling_batch && short_leaf(c)) {
        size_t j = i + 1;
        while (j < ch.size() && short_leaf(ch[j])) ++j;
        leaf_runs(ch, i, j, S, 0, -1);
        i = j;
      } else if (chunk == 0 || static_cast<uint64_t>(len) <= chunk) {
        const int bi = make_batch({c}, S);
        batches[bi].leaf_batch = tree.nodes[c].children.empty();
        batches[bi].direct_kv = batches[bi].leaf_batch;
        ops.push_back({bi, OP_FWD, 0});
        trace += "PUSH " + std::to_string(pid[c]) + "\n";
        visit(c, S + len);
        ops.push_back({bi, OP_BWD, 0});
        trace += "POP " + std::to_string(pid[c]) + "\n";
        ++i;
      } else {
        // chunked node: forward every chunk (its K/V stays on the stack), keep activations only for
        // the newest chunk; at pop recompute + backward the older chunks newest-first
        std::vector<int> ids;
        for (int64_t a = 0; a < len; a += static_cast<int64_t>(chunk))
          ids.push_back(make_chunk(c, S, a, std::min<int64_t>(len, a + static_cast<int64_t>(chunk)), a == 0 ? 1 : 0));
        for (int id : ids) batches[id].leaf_batch = tree.nodes[c].children.empty();
        trace += "PUSH " + std::to_string(pid[c]) + "\n";
        for (size_t k = 0; k + 1 < ids.size(); ++k) ops.push_back({ids[k], OP_FWD_DISCARD, 0});
        ops.push_back({ids.back(), OP_FWD, 0});
        visit(c, S + len);
        ops.push_back({ids.back(), OP_BWD, 0});
        for (size_t k = ids.size() - 1; k-- > 0;) ops.push_back({ids[k], OP_REFWD_BWD, 0});
        trace += "POP " + std::to_string(pid[c]) + "\n";
        ++i;
      }
    }
  };
  visit(0, 0);

  const auto t_sched = now();
  // ---- memory plan: LIFO arena offsets, stack rows, scratch sizes, counters
  tt_step_result& res = plan->counters;
  size_t top = 0;
  uint64_t live_tok = 0, peak_tok = 0, peak_kv = 0;
  std::vector<size_t> fwd_off(batches.size(), 0);
  for (auto& op : ops) {
    Batch& b = batches[op.b];
    const size_t sz = align_up(layout(b.n).total);
    if (op.code != OP_BWD) {
      plan->rows = std::max<int64_t>(plan->rows, b.row0() + b.n);
      plan->max_n = std::max<int64_t>(plan->max_n, b.n);
      plan->max_loss = std::max<int64_t>(plan->max_loss, static_cast<int64_t>(b.loss_rows.size()));
      // live KV (ledger semantics): childless leaves skip KV storage with leaf_kv_skip
      const uint64_t kv = static_cast<uint64_t>(b.row0()) + ((sc.leaf_kv_skip && b.leaf_batch) ? 0 : b.n);
      peak_kv = std::max(peak_kv, kv);
    }
    switch (op.code) {
      case OP_FWD:
        op.off = fwd_off[op.b] = top;
        top += sz;
        plan->arena_peak = std::max(plan->arena_peak, top);
        live_tok += b.n;
        peak_tok = std::max(peak_tok, live_tok);
        res.forward_tokens += b.n;
        res.num_segments += b.accum_inc;
        res.num_batches += 1;
        break;
      case OP_FWD_DISCARD:  // forward, activations dropped right after (K/V stay on the stack)
        op.off = top;
        plan->arena_peak = std::max(plan->arena_peak, top + sz);
        peak_tok = std::max(peak_tok, live_tok + b.n);
        res.forward_tokens += b.n;
        res.num_batches += 1;
        break;
      case OP_BWD:
        op.off = fwd_off[op.b];
        top = op.off;
        live_tok -= b.n;
        res.backward_tokens += b.n;
        res.num_chunks += 1;
        break;
      case OP_REFWD_BWD:  // recompute the chunk's activations from the stack, then its backward
        op.off = top;
        plan->arena_peak = std::max(plan->arena_peak, top + sz);
        peak_tok = std::max(peak_tok, live_tok + b.n);
        res.recompute_tokens += b.n;
        res.backward_tokens += b.n;
        res.num_chunks += 1;
        res.num_segments += b.accum_inc;
        break;
      default:
        break;
    }
  }
  res.peak_live_kv_tokens = peak_kv;
  res.peak_live_activation_tokens = peak_tok;
  for (auto& s : tree.seq_tokens) res.rollout_tokens += s.size();
  // ---- metadata for every batch, resident in HBM for the plan's lifetime
  std::vector<char> host;
  size_t cursor = 0;
  const auto t_mem = now();
  for (auto& b : batches) build_meta(b, cursor, host);
  const auto t_meta = now();
  if (transient) {
    plan->meta_bytes = upload_staged(host, meta_);
    plan->meta_ptr = meta_.as<char>();
    ck(cudaStreamSynchronize(stream_), "plan upload");
  } else {
    // pinned staging ring + the copy stream + a pooled device buffer: no synchronisation with a step
    // in flight and no per-plan pinning / cudaMalloc
    const size_t need = std::max(host.size(), kAlign);
    size_t best = meta_pool_.size();
    for (size_t i = 0; i < meta_pool_.size(); ++i)
      if (meta_pool_[i].second >= need && (best == meta_pool_.size() || meta_pool_[i].second < meta_pool_[best].second))
        best = i;
    if (best < meta_pool_.size()) {
      plan->meta_dev = meta_pool_[best].first;
      plan->meta_dev_bytes = meta_pool_[best].second;
      meta_pool_.erase(meta_pool_.begin() + static_cast<long>(best));
    } else {
      ck(cudaMalloc(&plan->meta_dev, need), "cudaMalloc plan meta");
      plan->meta_dev_bytes = need;
    }
    plan->release_meta = [this](void* p, size_t n) { retire_meta(p, n); };
    plan->meta_bytes = host.size();
    plan->meta_ptr = static_cast<const char*>(plan->meta_dev);
    if (!host.empty()) {
      const int slot = pin_next_;
      pin_next_ ^= 1;
      if (pin_ev_[slot]) ck(cudaEventSynchronize(pin_ev_[slot]), "staging slot");  // its last upload is done
      if (host.size() > pin_cap_[slot]) {
        if (pin_ring_[slot]) cudaFreeHost(pin_ring_[slot]);
        pin_ring_[slot] = nullptr;
        ck(cudaMallocHost(&pin_ring_[slot], host.size()), "cudaMallocHost plan meta");
        pin_cap_[slot] = host.size();
      }
      std::memcpy(pin_ring_[slot], host.data(), host.size());
      ck(cudaMemcpyAsync(plan->meta_dev, pin_ring_[slot], host.size(), cudaMemcpyHostToDevice, copy_stream_),
         "plan meta upload");
      if (!pin_ev_[slot]) ck(cudaEventCreateWithFlags(&pin_ev_[slot], cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventRecord(pin_ev_[slot], copy_stream_), "staging event");
    }
    ck(cudaEventCreateWithFlags(&plan->uploaded, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(plan->uploaded, copy_stream_), "plan upload event");
  }
  res.h2d_bytes = plan->meta_bytes;
  if (timing) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "prepare: schedule %.1f ms, memory plan %.1f ms, metadata %.1f ms, upload %.1f ms (%zu B)\n",
                 ms(t_start, t_sched), ms(t_sched, t_mem), ms(t_mem, t_meta), ms(t_meta, now()), plan->meta_bytes);
  }
  return plan;
}

// A destroyed plan's device metadata buffer: back to the pool (at most 4 kept), unless a step of that
// plan may still be reading it.
void Engine::retire_meta(void* p, size_t n) {
  if (inflight_) cudaEventSynchronize(step_done_);
  meta_pool_.emplace_back(p, n);
  if (meta_pool_.size() > 4) {
    cudaFree(meta_pool_.front().first);
    meta_pool_.erase(meta_pool_.begin());
  }
}

tt_step_result Engine::execute(StepPlan& plan) {
  execute_async(plan);
  return wait(plan);
}

void Engine::execute_async(StepPlan& plan) {
  if (plan.owner != this) throw std::invalid_argument("plan_execute: the plan was prepared by another engine");
  if (inflight_) throw std::runtime_error("plan_execute: another step is still in flight on this engine");
  if (!seg_stack_.empty()) throw std::runtime_error("tree_train_step: segment stack is not empty");
  issue_step(plan);
  ck(cudaEventRecord(step_done_, stream_), "step event");
  inflight_ = &plan;
}

tt_step_result Engine::wait(StepPlan& plan) {
  if (inflight_ != &plan) throw std::invalid_argument("plan_wait: this plan has no step in flight");
  inflight_ = nullptr;
  ck(cudaEventSynchronize(step_done_), "tree_train_step");
  return finish_step(plan);
}

void Engine::issue_step(StepPlan& plan) {
  ensure_capacity(plan.rows, plan.arena_peak, plan.max_n, plan.max_loss);
  if (plan.uploaded) ck(cudaStreamWaitEvent(stream_, plan.uploaded, 0), "plan upload wait");
  cur_meta_ = plan.meta_ptr;
  step_launches0_ = launches_;
  // First execution eager (sets kernel attributes, proves the plan); from the second one on, the
  // whole op list is one CUDA graph (re-captured if any device buffer was reallocated since).
  const bool use_graph = cuda_graph_ && !profiling_ && plan.warmed;
  if (use_graph && !(plan.graph && plan.graph_gen == alloc_generation() && plan.graph_opts == opt_epoch_)) {
    if (plan.graph) {
      cudaGraphExecDestroy(plan.graph);
      plan.graph = nullptr;
    }
    cudaGraph_t g = nullptr;
    ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "graph capture");
    const uint64_t l0 = launches_;
    try {
      issue_ops(plan);
    } catch (...) {
      cudaStreamEndCapture(stream_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ck(cudaStreamEndCapture(stream_, &g), "graph capture end");
    ck(cudaGraphInstantiate(&plan.graph, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    plan.graph_launches = launches_ - l0;
    launches_ = l0;
    plan.graph_gen = alloc_generation();
    plan.graph_opts = opt_epoch_;
  }
  if (use_graph) {
    ck(cudaGraphLaunch(plan.graph, stream_), "graph launch");
    launches_ += plan.graph_launches;
  } else {
    issue_ops(plan);
    plan.warmed = true;
  }
  ck(cudaGetLastError(), "tree_train_step launch");
  ck(cudaMemcpyAsync(loss_host_, loss_.p, sizeof(double), cudaMemcpyDeviceToHost, stream_), "loss download");
}

tt_step_result Engine::finish_step(StepPlan& plan) {
  collect_profile();
  tt_step_result res = plan.counters;
  res.total_loss = *loss_host_;
  res.num_launches = launches_ - step_launches0_;
  res.d2h_bytes = sizeof(double);
  res.peak_hbm_bytes = wbuf_.bytes + gainbuf_.bytes + pe_.bytes + grads_.bytes + kst_.bytes + vst_.bytes +
                       dkst_.bytes + dvst_.bytes + plan.arena_peak + sc_gx_.bytes + sc_gxb_.bytes + sc_gxf_.bytes +
                       sc_gn_.bytes + sc_gh_.bytes + sc_dO_.bytes + sc_D_.bytes + sc_dq_.bytes + sc_dqkv_.bytes +
                       sc_nfl_.bytes + sc_logits_.bytes + sc_dlog_.bytes + sc_gnf_.bytes + plan.meta_dev_bytes +
                       meta_.bytes;
  arena_peak_ = std::max(arena_peak_, plan.arena_peak);
  if (!std::isfinite(res.total_loss)) throw NonFiniteError("tree_train_step: non-finite loss");
  return res;
}

// Enqueues one step of the plan on the engine stream (no host synchronisation: graph-capturable).
void Engine::issue_ops(const StepPlan& plan) {
  gemm_set_2cta(gemm_2cta_);
  ck(cudaMemsetAsync(loss_.p, 0, sizeof(double), stream_), "memset");
  for (const auto& op : plan.ops) {
    const Batch& b = plan.batches[op.b];
    switch (op.code) {
      case OP_FWD:
      case OP_FWD_DISCARD:
        forward_batch(b, op.off);
        break;
      case OP_BWD:
        backward_batch(b, op.off, nullptr);
        break;
      case OP_REFWD_BWD:
        forward_batch(b, op.off);
        backward_batch(b, op.off, nullptr);
        break;
      default:
        break;
    }
  }
}

tt_step_result Engine::train_step(const PrefixTree& tree, const tt_sched_config& sc) {
  auto plan = prepare(tree, sc, /*transient=*/true);
  last_trace_ = plan->trace;
  return execute(*plan);
}

// ----------------------------------------------------------------------------- segment-level API
void Engine::stack_reset() {
  ck(cudaStreamSynchronize(stream_), "stack_reset");
  seg_stack_.clear();
  arena_top_ = 0;
  if (dkst_.p) {
    ck(cudaMemset(dkst_.p, 0, dkst_.bytes), "memset");
    ck(cudaMemset(dvst_.p, 0, dvst_.bytes), "memset");
  }
}

// forward_segment (model.hpp:328-463) continuing from the device stack. want_kv = false: the
// segment's K/V rows are not kept for descendants (no push on top of it); want_activations = false:
// its activations are dropped right away (its pop recomputes them, the chunked backward's
// recompute). Neither: forward only, the stack is unchanged.
void Engine::segment_push(const int32_t* tokens, uint64_t len, bool want_kv, bool want_acts, float* logits_out) {
  if (len == 0) throw std::invalid_argument("forward_segment: empty token list");
  if (!seg_stack_.empty() && seg_stack_.back().no_kv)
    throw std::invalid_argument("forward_segment: the prefix segment was pushed with want_kv = false");
  const int64_t S = static_cast<int64_t>(stack_tokens());
  if (S + static_cast<int64_t>(len) > static_cast<int64_t>(cfg_.max_position))
    throw std::invalid_argument("forward_segment: position overflow beyond max_position");
  for (uint64_t t = 0; t < len; ++t)
    if (tokens[t] < 0 || static_cast<uint64_t>(tokens[t]) >= cfg_.vocab_size)
      throw std::invalid_argument("forward_segment: token id out of vocab range");
  Batch b;
  b.S = S;
  b.n = static_cast<int64_t>(len);
  b.seg_off = {0};
  b.seg_len = {b.n};
  b.full_logits = true;
  b.no_kv = !want_kv;
  b.has_acts = want_acts;
  b.leaf_batch = !want_kv;
  b.attn_ctx = double(b.n) * double(S) + 0.5 * double(b.n) * double(b.n + 1);
  for (uint64_t t = 0; t < len; ++t) {
    b.tokens.push_back(tokens[t]);
    b.positions.push_back(static_cast<int32_t>(S + t));
  }
  b.pair_off = {0};
  if (seg_stack_.empty()) {
    // first segment: size the stack for max_position rows and the arena for a max_position path
    const int64_t mp = static_cast<int64_t>(cfg_.max_position);
    ensure_capacity(mp, align_up(layout(mp).total) + 64 * align_up(layout(1).total), mp, mp);
  }
  b.arena_off = arena_top_;
  const size_t need = align_up(layout(b.n).total);
  if (arena_top_ + need > arena_.bytes) throw std::runtime_error("segment_push: activation arena exhausted");
  std::vector<Batch*> ptrs;
  for (auto& x : seg_stack_) ptrs.push_back(&x);
  ptrs.push_back(&b);
  upload_meta(ptrs);
  gemm_set_2cta(gemm_2cta_);
  forward_batch(b, b.arena_off);
  if (logits_out) {  // host or device pointer (unified addressing)
    const ActLayout lay = layout(b.n);
    const bf16* nf = arena_.as<bf16>(b.arena_off + lay.nf);
    for (int64_t c0 = 0; c0 < b.n; c0 += head_chunk_) {
      const int64_t cm = std::min<int64_t>(head_chunk_, b.n - c0);
      EpiParams e;
      e.mode = EPI_STORE_F32;
      e.out[0] = sc_logits_.p;
      e.ldo[0] = V_;
      gemm(op(nf + c0 * d_, d_, false), op(head_, V_, true), static_cast<int>(cm), static_cast<int>(V_),
           static_cast<int>(d_), e, 1);
      ck(cudaMemcpyAsync(logits_out + c0 * V_, sc_logits_.p, cm * V_ * 4, cudaMemcpyDefault, stream_),
         "logits download");
    }
  }
  ck(cudaGetLastError(), "segment_push");
  ck(cudaStreamSynchronize(stream_), "segment_push");
  if (!want_kv && !want_acts) return;  // forward only
  if (want_acts) arena_top_ += need;
  seg_stack_.push_back(std::move(b));
}

// weighted_nll (model.hpp:643-677) of the top segment on the device — the VISIT of SPEC.md:225.
// row_off[n + 1] (NULL: one pair per row) indexes (targets, weights) pairs per segment row; pairs of
// weight 0 contribute nothing. The pairs stay with the frame: its pop takes grad_logits from them
// (fused LM-head GEMM + CE, no logits crossing PCIe).
double Engine::segment_loss(const uint64_t* row_off, const int32_t* targets, const double* weights) {
  if (seg_stack_.empty()) throw std::invalid_argument("weighted_nll: empty stack");
  Batch& b = seg_stack_.back();
  if (!b.has_acts) throw std::invalid_argument("weighted_nll: the segment was pushed with want_activations = false");
  if (!targets || !weights) throw std::invalid_argument("weighted_nll: null targets / weights");
  b.loss_rows.clear();
  b.pair_off.clear();
  b.pair_tgt.clear();
  b.pair_w.clear();
  for (int64_t r = 0; r < b.n; ++r) {
    const uint64_t p0 = row_off ? row_off[r] : static_cast<uint64_t>(r);
    const uint64_t p1 = row_off ? row_off[r + 1] : static_cast<uint64_t>(r + 1);
    if (p1 < p0) throw std::invalid_argument("weighted_nll: row offsets must be non-decreasing");
    bool row = false;
    for (uint64_t p = p0; p < p1; ++p) {
      if (targets[p] < 0 || static_cast<uint64_t>(targets[p]) >= cfg_.vocab_size)
        throw std::invalid_argument("weighted_nll: target id out of vocab range");
      if (!std::isfinite(weights[p])) throw std::invalid_argument("weighted_nll: non-finite weight");
      if (weights[p] == 0.0) continue;
      if (!row) {
        b.loss_rows.push_back(static_cast<int32_t>(r));
        b.pair_off.push_back(static_cast<int32_t>(b.pair_tgt.size()));
        row = true;
      }
      b.pair_tgt.push_back(targets[p]);
      b.pair_w.push_back(weights[p]);
    }
  }
  b.pair_off.push_back(static_cast<int32_t>(b.pair_tgt.size()));
  b.full_logits = false;
  b.has_loss = true;
  std::vector<Batch*> ptrs;
  for (auto& x : seg_stack_) ptrs.push_back(&x);
  upload_meta(ptrs);
  gemm_set_2cta(gemm_2cta_);
  ck(cudaMemsetAsync(loss_.p, 0, sizeof(double), stream_), "memset");
  const ActLayout lay = layout(b.n);
  head_backward(b, arena_.as<bf16>(b.arena_off + lay.nf), /*loss_only=*/true);
  ck(cudaMemcpyAsync(loss_host_, loss_.p, sizeof(double), cudaMemcpyDeviceToHost, stream_), "loss download");
  ck(cudaStreamSynchronize(stream_), "weighted_nll");
  if (!std::isfinite(*loss_host_)) throw NonFiniteError("weighted_nll: non-finite loss");
  return *loss_host_;
}

// backward_segment (model.hpp:474-633) of the top segment. Upstream grad_logits: the caller's
// [len x V] (host or device) or, after segment_loss, the device CE of the frame's pairs; grad_new_kv
// is what the segments popped above it added into its dK/dV stack rows. The returned KVGrad
// (grad_prefix, rows [0, S)) is added into the ancestors' rows; with grad_prefix_out (host or
// device, [L][2][S][d] fp32) the attention backward writes it into a separate zeroed buffer that is
// copied out and then added into the stack — the pop's own contribution, not a difference.
void Engine::segment_pop(const float* grad_logits, float* grad_prefix_out) {
  if (seg_stack_.empty()) throw std::invalid_argument("backward_segment: empty stack");
  Batch& b = seg_stack_.back();
  if (b.has_loss && grad_logits)
    throw std::invalid_argument("backward_segment: grad_logits given for a segment whose loss is on the device");
  const bool want_gp = grad_prefix_out && b.S > 0;
  const size_t pre = static_cast<size_t>(b.S) * d_;
  if (want_gp) {
    sc_gpre_.ensure(2 * L_ * pre * sizeof(float));
    ck(cudaMemsetAsync(sc_gpre_.p, 0, 2 * L_ * pre * sizeof(float), stream_), "memset");
  }
  std::vector<Batch*> ptrs;
  for (auto& x : seg_stack_) ptrs.push_back(&x);
  upload_meta(ptrs);
  gemm_set_2cta(gemm_2cta_);
  if (!b.has_acts) {  // recompute the activations from the stack (chunked backward)
    if (b.arena_off + align_up(layout(b.n).total) > arena_.bytes)
      throw std::runtime_error("segment_pop: activation arena exhausted");
    forward_batch(b, b.arena_off);
  }
  backward_batch(b, b.arena_off, grad_logits, want_gp ? sc_gpre_.as<float>() : nullptr);
  if (want_gp) {
    ck(cudaMemcpyAsync(grad_prefix_out, sc_gpre_.p, 2 * L_ * pre * sizeof(float), cudaMemcpyDefault, stream_),
       "grad_prefix download");
    const size_t kv_layer = static_cast<size_t>(rows_cap_) * d_;
    for (int64_t l = 0; l < L_; ++l) {  // KVGrad::add_rows into the ancestors' frames (model.hpp:193-206)
      k_add_f32(dkst_.as<float>() + l * kv_layer, sc_gpre_.as<float>() + (2 * l) * pre, static_cast<long>(pre), stream_);
      k_add_f32(dvst_.as<float>() + l * kv_layer, sc_gpre_.as<float>() + (2 * l + 1) * pre, static_cast<long>(pre),
                stream_);
    }
  }
  ck(cudaGetLastError(), "segment_pop");
  ck(cudaStreamSynchronize(stream_), "segment_pop");
  arena_top_ = b.arena_off;
  seg_stack_.pop_back();
}

// weighted_nll (model.hpp:643-677) as a standalone device operation over caller logits.
double Engine::weighted_nll(const float* logits, uint64_t n, const uint64_t* row_off, const int32_t* targets,
                            const double* weights, float* grad_out) {
  if (n == 0) return 0.0;
  if (!logits || !targets || !weights) throw std::invalid_argument("weighted_nll: null logits / targets / weights");
  std::vector<int32_t> off(n + 1), tgt;
  std::vector<double> w;
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t p0 = row_off ? row_off[r] : r, p1 = row_off ? row_off[r + 1] : r + 1;
    if (p1 < p0) throw std::invalid_argument("weighted_nll: row offsets must be non-decreasing");
    off[r] = static_cast<int32_t>(tgt.size());
    for (uint64_t p = p0; p < p1; ++p) {
      if (targets[p] < 0 || static_cast<uint64_t>(targets[p]) >= cfg_.vocab_size)
        throw std::invalid_argument("weighted_nll: target id out of vocab range");
      if (!std::isfinite(weights[p])) throw std::invalid_argument("weighted_nll: non-finite weight");
      if (weights[p] == 0.0) continue;
      tgt.push_back(targets[p]);
      w.push_back(weights[p]);
    }
  }
  off[n] = static_cast<int32_t>(tgt.size());
  DevBuf meta;
  const size_t o_tgt = align_up(off.size() * 4), o_w = o_tgt + align_up(std::max<size_t>(tgt.size(), 1) * 4);
  meta.ensure(o_w + std::max<size_t>(w.size(), 1) * 8);
  ck(cudaMemcpyAsync(meta.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, stream_), "nll meta");
  if (!tgt.empty()) {
    ck(cudaMemcpyAsync(meta.as<char>(o_tgt), tgt.data(), tgt.size() * 4, cudaMemcpyHostToDevice, stream_), "nll meta");
    ck(cudaMemcpyAsync(meta.as<char>(o_w), w.data(), w.size() * 8, cudaMemcpyHostToDevice, stream_), "nll meta");
  }
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(n), (int64_t(1) << 30) / (V_ * 8)));
  DevBuf lg, gr;
  lg.ensure(static_cast<size_t>(chunk) * V_ * 4);
  gr.ensure(static_cast<size_t>(chunk) * V_ * 4);
  ck(cudaMemsetAsync(loss_.p, 0, sizeof(double), stream_), "memset");
  for (int64_t c0 = 0; c0 < static_cast<int64_t>(n); c0 += chunk) {
    const int64_t cm = std::min<int64_t>(chunk, static_cast<int64_t>(n) - c0);
    ck(cudaMemcpyAsync(lg.p, logits + c0 * V_, static_cast<size_t>(cm) * V_ * 4, cudaMemcpyDefault, stream_), "logits");
    k_ce_f32(lg.as<float>(), static_cast<int>(cm), V_, meta.as<int32_t>() + c0, meta.as<int32_t>(o_tgt),
             meta.as<double>(o_w), gr.as<float>(), loss_.as<double>(), stream_);
    if (grad_out)
      ck(cudaMemcpyAsync(grad_out + c0 * V_, gr.p, static_cast<size_t>(cm) * V_ * 4, cudaMemcpyDefault, stream_),
         "grad_logits");
  }
  ck(cudaGetLastError(), "weighted_nll");
  ck(cudaMemcpyAsync(loss_host_, loss_.p, sizeof(double), cudaMemcpyDeviceToHost, stream_), "loss download");
  ck(cudaStreamSynchronize(stream_), "weighted_nll");
  return *loss_host_;
}

}  // namespace ttb
