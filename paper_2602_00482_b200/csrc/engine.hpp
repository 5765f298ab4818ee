// B200 DFS prefix-tree forward/backward engine (device side of tree_train_step).
//
// HBM layout (one engine per GPU):
//   weights (bf16): embedding [V x d]; per layer Wqkv [d x 3d] (= [Wq | Wk | Wv] column blocks),
//                   Wo [d x d], Win [d x F], Wout [F x d]; head [d x V]; gains (fp32)
//   GradientStore (fp32): one flat buffer in for_each_tensor order (model.hpp:42-59)
//   KV stack (bf16): per layer K,V [rows_cap x d]; stack row = absolute token position on the path
//   dKV stack (fp32): per layer dK,dV [rows_cap x d]; a frame's KVGrad lives on its own rows
//   activation arena: LIFO, one region per pushed segment batch, rewound at pop
//   scratch: per-pop temporaries (largest batch) + LM-head/CE chunk buffers
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/treetrain_b200.h"
#include "kernels/gemm.h"
#include "prefix_tree.hpp"

namespace ttb {

using bf16 = __nv_bfloat16;

// Bumped whenever any DevBuf (re)allocates: CUDA graphs captured before hold stale pointers.
uint64_t alloc_generation();

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void ensure(size_t n);  // grow (contents discarded)
  template <typename T>
  T* as(size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<char*>(p) + byte_off);
  }
};

// One executed segment batch: a single tree node, or a run of sibling childless nodes sharing
// the prefix rows [0, S). Members are laid out contiguously on rows [S, S+n).
struct Batch {
  int64_t S = 0, n = 0;
  // stack rows: the prefix occupies [pbase, pbase + S), the batch's own rows start at row0() (= S
  // unless set: members of a multi-root batch keep their children's prefix at their own rows)
  int64_t pbase = 0, R0 = -1;
  int64_t row0() const { return R0 < 0 ? S : R0; }
  std::vector<int32_t> nodes;
  std::vector<int64_t> seg_off, seg_len;
  // host-built metadata (uploaded once per step)
  std::vector<int32_t> tokens, positions;
  std::vector<int32_t> qblk128;  // int4 per 128-row query block (forward)
  std::vector<int32_t> kvit128, kvit128_2;  // 128-row stack blocks {kv_row0, rows, q_lo, q_hi} / {seg_off, own}
  std::vector<int32_t> loss_rows, pair_off, pair_tgt;
  std::vector<double> pair_w;
  // device offsets (bytes) into the metadata buffer
  size_t o_tok = 0, o_pos = 0, o_qblk128 = 0, o_kvit128 = 0, o_kvit128_2 = 0, o_lrows = 0, o_poff = 0, o_ptgt = 0, o_pw = 0;
  size_t arena_off = 0;
  double attn_ctx = 0;       // sum over query rows of attended keys (S + t + 1): attention FLOP model
  bool full_logits = false;  // segment API: head over all rows with caller-provided grad_logits
  // segment API frame state (forward_segment's want_kv / want_activations, model.hpp:328-331)
  bool no_kv = false;        // pushed with want_kv = false: no segment may be pushed on top of it
  bool has_acts = true;      // activations kept (false: the pop recomputes them from the stack)
  bool has_loss = false;     // weighted_nll pairs set on the device (tt_segment_loss)
  bool leaf_batch = false;   // childless node(s): K/V not kept for descendants (leaf_kv_skip ledger)
  // no contribution reaches the batch's own dK/dV rows before its pop (childless, not a chunk of a
  // chunked node): the attention backward writes their bf16 dK/dV straight into the packed operand
  bool direct_kv = false;
  int accum_inc = 1;         // GradientStore::accum_count increment (nodes completed by this pop)
};

// Step op codes: push (forward, activations kept), push with activations discarded (older chunks of
// a chunked node), pop (backward, activations freed), recompute + pop.
enum OpCode : int { OP_FWD = 0, OP_BWD = 1, OP_FWD_DISCARD = 2, OP_REFWD_BWD = 3 };
struct PlanOp {
  int b;       // batch index
  int code;    // OpCode
  size_t off;  // arena offset of the batch's activations for this op
};

// A prepared tree step: batches, PUSH/POP op list, memory plan, metadata resident in HBM.
// prepare() once, execute() many times (the timed path with inputs already on the device).
struct StepPlan {
  std::vector<Batch> batches;
  std::vector<PlanOp> ops;  // DFS order
  int64_t rows = 0, max_n = 0, max_loss = 0;
  size_t arena_peak = 0;
  const char* meta_ptr = nullptr;  // device metadata (meta_dev, or the engine's step buffer if transient)
  size_t meta_bytes = 0;
  tt_step_result counters{};
  std::string trace;  // logical DFS trace of the executed schedule
  // CUDA graph of the whole op list (captured on the second execute, replayed afterwards)
  bool warmed = false;
  cudaGraphExec_t graph = nullptr;
  uint64_t graph_gen = 0, graph_launches = 0, graph_opts = 0;
  const void* owner = nullptr;  // the Engine that prepared the plan (its buffers are baked in)
  // persistent plans: metadata copied on the engine's copy stream from a pinned staging ring (no host
  // synchronisation, so a plan can be prepared while another step executes) into a device buffer
  // that returns to the engine's pool when the plan is destroyed (no cudaMalloc / cudaFree per step);
  // the first execute orders itself after the copy through `uploaded`
  void* meta_dev = nullptr;
  size_t meta_dev_bytes = 0;
  std::function<void(void*, size_t)> release_meta;
  cudaEvent_t uploaded = nullptr;
  StepPlan() = default;
  StepPlan(const StepPlan&) = delete;
  StepPlan& operator=(const StepPlan&) = delete;
  ~StepPlan() {
    if (graph) cudaGraphExecDestroy(graph);
    if (uploaded) {
      cudaEventSynchronize(uploaded);
      cudaEventDestroy(uploaded);
    }
    if (meta_dev && release_meta) release_meta(meta_dev, meta_dev_bytes);
  }
};

// Per-kernel-class device timing (profiling mode): CUDA events around every launch.
enum KClass { KC_GEMM = 0, KC_ATTN_FWD = 1, KC_ATTN_BWD = 2, KC_ELEMWISE = 3, KC_CE = 4, KC_NUM = 5 };
struct KStats {
  double ms[KC_NUM] = {0, 0, 0, 0, 0};
  double flops[KC_NUM] = {0, 0, 0, 0, 0};
  double bytes[KC_NUM] = {0, 0, 0, 0, 0};
  uint64_t launches[KC_NUM] = {0, 0, 0, 0, 0};
};

struct ActLayout {  // byte offsets of one batch's activations inside its arena region
  size_t per_layer = 0;
  size_t x, inv1, n1, q, attn, lse, xmid, inv2, n2, h, act;  // within a layer block
  size_t final_x, invf, nf;                                  // after the layer blocks
  size_t total = 0;
};

class Engine {
 public:
  Engine(const tt_model_config& cfg, int device);
  ~Engine();

  const tt_model_config& config() const { return cfg_; }
  int device() const { return device_; }
  uint64_t param_count() const { return n_params_; }
  cudaStream_t stream() const { return stream_; }

  void upload_params(const float* flat, uint64_t n);
  void init_random(uint64_t seed);
  void grads_zero();
  void grads_download(float* out, uint64_t n);
  void grads_download_f64(double* out, uint64_t n);
  // in-place sum all-reduce of the GradientStore over an NCCL communicator (ncclComm_t), on the
  // engine stream (SPEC.md:278's worker-order reduction, replaced by one ncclAllReduce)
  void grads_allreduce(void* nccl_comm);
  // weighted_nll (model.hpp:643-677) on the device over caller logits [n x V] (host or device
  // pointer); row_off (n + 1, NULL = one pair per row) indexes targets/weights; grad_out [n x V]
  // fp32 (host or device, may be NULL). Returns the loss (fp64).
  double weighted_nll(const float* logits, uint64_t n, const uint64_t* row_off, const int32_t* targets,
                      const double* weights, float* grad_out);
  float* grads_device() const { return grads_.as<float>(); }
  uint64_t accum_count() const { return accum_count_; }

  tt_step_result train_step(const PrefixTree& tree, const tt_sched_config& sc);
  // transient = the plan is executed once right away (tree_train_step): its metadata goes into an
  // engine-owned buffer reused across steps instead of a fresh allocation per plan
  std::unique_ptr<StepPlan> prepare(const PrefixTree& tree, const tt_sched_config& sc, bool transient = false);
  tt_step_result execute(StepPlan& plan);
  // Asynchronous form: enqueue the step and return; wait() blocks for it and returns the result.
  // One step in flight per engine; prepare() of the next plan may run meanwhile (its metadata goes
  // over the copy stream), which is how a training loop overlaps host planning with the device step.
  void execute_async(StepPlan& plan);
  tt_step_result wait(StepPlan& plan);
  void retire_meta(void* p, size_t n);

  void set_profiling(bool on) { profiling_ = on; }
  void set_option(const std::string& key, int64_t value);
  const KStats& kstats() const { return kstats_; }
  void reset_kstats() {
    kstats_ = KStats{};
    tag_stats_.clear();
  }
  std::string gemm_profile_text() const;
  const std::string& last_trace() const { return last_trace_; }

  // segment level (device stack)
  void segment_push(const int32_t* tokens, uint64_t len, bool want_kv, bool want_acts, float* logits_out);
  double segment_loss(const uint64_t* row_off, const int32_t* targets, const double* weights);
  void segment_pop(const float* grad_logits, float* grad_prefix_out);
  void stack_reset();
  uint64_t stack_segments() const { return seg_stack_.size(); }
  uint64_t stack_tokens() const;

 private:
  // ---- helpers
  ActLayout layout(int64_t n) const;
  double bytes_per_token() const;
  uint64_t auto_batch_budget(uint64_t path_tokens) const;
  void ensure_capacity(int64_t rows, size_t arena_bytes, int64_t max_n, int64_t max_loss_rows);
  void build_meta(Batch& b, size_t& cursor, std::vector<char>& host);
  void upload_meta(std::vector<Batch*>& batches);
  void forward_batch(const Batch& b, size_t arena_off);
  void backward_batch(const Batch& b, size_t arena_off, const float* host_grad_logits, float* grad_prefix = nullptr);
  void head_backward(const Batch& b, const bf16* nf, bool loss_only = false);
  void head_backward_dense(const Batch& b, const bf16* nf, const float* host_grad_logits);
  void gemm(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const EpiParams& e, int splits);
  template <typename T>
  const T* meta(size_t off) const {
    return reinterpret_cast<const T*>(cur_meta_ + off);
  }
  void count(int k = 1) { launches_ += k; }
  void tag(const char* name) {
    if (profiling_) pending_tag_ = name;
  }
  // Launch wrapper: counts the launch and, in profiling mode, brackets it with CUDA events.
  template <typename F>
  void run(KClass cls, double flops, double bytes, F&& launch) {
    if (!profiling_) {
      launch();
      ++launches_;
      return;
    }
    cudaEvent_t a = event(), b = event();
    cudaEventRecord(a, stream_);
    launch();
    cudaEventRecord(b, stream_);
    pending_.push_back({cls, a, b, flops, bytes, pending_tag_});
    pending_tag_.clear();
    ++launches_;
  }
  cudaEvent_t event();
  void collect_profile();
  size_t upload_staged(const std::vector<char>& host, DevBuf& dst);
  void issue_step(StepPlan& plan);       // enqueue one step of a prepared plan (graph or eager)
  tt_step_result finish_step(StepPlan& plan);  // wait for it; loss, counters, non-finite check

  tt_model_config cfg_;
  int device_ = 0;
  int64_t V_, d_, H_, L_, F_, dh_;
  uint64_t n_params_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaStream_t copy_stream_ = nullptr;  // metadata uploads of persistent plans
  // pinned staging ring of the persistent plans' metadata (2 slots: the plan being prepared and the
  // one executing) and the pool of retired plans' device metadata buffers
  void* pin_ring_[2] = {nullptr, nullptr};
  size_t pin_cap_[2] = {0, 0};
  cudaEvent_t pin_ev_[2] = {nullptr, nullptr};
  int pin_next_ = 0;
  std::vector<std::pair<void*, size_t>> meta_pool_;
  cudaEvent_t step_done_ = nullptr;     // end of the step in flight (execute_async / wait)
  const StepPlan* inflight_ = nullptr;
  uint64_t step_launches0_ = 0;

  // parameters (device layout) and gradients
  DevBuf wbuf_;  // all bf16 weights
  bf16 *emb_ = nullptr, *head_ = nullptr;
  std::vector<bf16*> wqkv_, wo_, win_, wout_;
  DevBuf gainbuf_;  // fp32 gains
  std::vector<float*> attn_g_, mlp_g_;
  float* final_g_ = nullptr;
  DevBuf pe_;  // fp32 [max_position x d]
  DevBuf grads_;
  // gradient tensor pointers (into grads_)
  float *g_emb_ = nullptr, *g_final_g_ = nullptr, *g_head_ = nullptr;
  std::vector<float*> g_attn_g_, g_wq_, g_wk_, g_wv_, g_wo_, g_mlp_g_, g_win_, g_wout_;
  uint64_t accum_count_ = 0;

  // stacks / arena / scratch
  int64_t rows_cap_ = 0;
  DevBuf kst_, vst_, dkst_, dvst_;
  DevBuf arena_;
  size_t arena_top_ = 0, arena_peak_ = 0;
  int64_t scratch_n_ = 0, head_chunk_ = 0;
  DevBuf sc_gx_, sc_gxb_, sc_gxf_, sc_gn_, sc_gh_, sc_dO_, sc_D_, sc_dq_, sc_dqkv_;
  DevBuf sc_nfl_, sc_logits_, sc_stats_, sc_dlog_, sc_gnf_;
  DevBuf sc_gpre_;  // segment pop: this pop's grad_prefix by itself ([L][2][S][d] fp32)
  DevBuf meta_;
  DevBuf loss_;
  double* loss_host_ = nullptr;  // pinned
  char* meta_host_ = nullptr;    // pinned staging
  size_t meta_host_cap_ = 0;
  uint64_t launches_ = 0;
  const char* cur_meta_ = nullptr;
  std::string last_trace_;
  bool profiling_ = false;
  bool cuda_graph_ = true;  // replay prepared plans as CUDA graphs (engine option "cuda_graph")
  void issue_ops(const StepPlan& plan);
  bool ce_stats_ = true;
  bool logits_bf16_ = true;
  bool plan_timing_ = false;  // LM-head logits stored bf16 relative to the 32-column group max
  int gemm_2cta_ = 1;
  // programmatic dependent launch (engine option "pdl"): 0 off, 1 on, 2 auto = batches of at most
  // kPdlAutoElems rows x d_model
  int pdl_ = 2;
  bool gn_bf16_ = true;  // engine option "gn_bf16"
  double pdl_auto_elems_ = 2.0 * 1024 * 1024;  // engine option "pdl_auto_elems"
  uint64_t opt_epoch_ = 1;  // bumped by set_option: a plan's CUDA graph is re-captured after a change
  // multi-root batching: consecutive forest roots whose children are all short leaves are pushed as
  // ONE batch of up to this many tokens (0 = off); each root's leaves attend to its own rows
  int64_t root_batch_tokens_ = 4096;
  // LM-head chunk scratch (fp32 logits + bf16 dlogits): larger chunks mean fewer fp32 read-modify-
  // write passes of the V x d head gradient (one per chunk)
  int64_t head_chunk_bytes_ = int64_t(6) << 30;
  int64_t head_cap_rows_ = 0;  // chunk row cap, fixed at the first plan that needs it (0 = not yet)
  KStats kstats_;
  struct Pending {
    KClass cls;
    cudaEvent_t a, b;
    double flops, bytes;
    std::string tag;  // GEMM shape key (profiling detail)
  };
  std::string pending_tag_;
  struct TagStat {
    double ms = 0, flops = 0, bytes = 0;
    uint64_t n = 0;
  };
  std::map<std::string, TagStat> tag_stats_;
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> event_pool_;
  size_t event_next_ = 0;

  // segment-level API state
  std::vector<Batch> seg_stack_;
};

}  // namespace ttb
