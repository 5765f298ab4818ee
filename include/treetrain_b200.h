/*
 * treetrain_b200 — C-ABI of the B200 (sm_100a) DFS prefix-tree forward/backward engine.
 *
 * Drop-in boundary for the reference's header-only C++ API in namespace treetrain
 * (/root/reference/proj/core/include/treetrain/ headers) and for the SPEC-level operations the
 * reference leaves unshipped. Every entry point:
 *   - returns TT_OK (0) or a TT_ERR_* status; no exception crosses the ABI;
 *   - takes plain pointers and sizes (host pointers unless documented otherwise);
 *   - records a message retrievable with tt_last_error() on failure.
 * Status -> reference exception mapping (model.hpp:334-343,483-492,647-655; model_io.cpp:60-103):
 *   TT_ERR_INVALID_ARGUMENT <-> std::invalid_argument, TT_ERR_RUNTIME <-> std::runtime_error,
 *   TT_ERR_NONFINITE <-> the SPEC's abort on non-finite loss.
 *
 * One engine per GPU and per host thread; an engine owns all of its device memory and one
 * CUDA stream and is not re-entrant. Trees are immutable after build/order and may be shared.
 */
#ifndef TREETRAIN_B200_H_
#define TREETRAIN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_OK 0
#define TT_ERR_INVALID_ARGUMENT 1
#define TT_ERR_RUNTIME 2
#define TT_ERR_OOM 3
#define TT_ERR_NONFINITE 4

/* ModelConfig (model_config.hpp:19-27). The engine computes in bf16 operands with fp32
 * accumulation/residual/gradients and fp64 loss, whatever `precision` says; the field is kept so
 * a reference config round-trips (0 = f32, 1 = f64, model_config.hpp:9). */
typedef struct tt_model_config {
  uint64_t vocab_size;
  uint64_t d_model;
  uint64_t n_heads;
  uint64_t n_layers;
  uint64_t d_ff;
  uint64_t max_position;
  int32_t precision;
  int32_t reserved;
} tt_model_config;

/* order_children policies. */
#define TT_ORDER_AS_BUILT 0
#define TT_ORDER_LEXICOGRAPHIC 1
#define TT_ORDER_SUBTREE_TOKENS_DESC 2
#define TT_ORDER_SUBTREE_TOKENS_ASC 3

/* SchedulerConfig plus the B200 sibling-batching switch. */
typedef struct tt_sched_config {
  uint64_t chunk_len;          /* SPEC.md:205; 0 = unlimited (whole segment keeps activations) */
  int32_t leaf_kv_skip;
  int32_t child_order_policy;  /* informational: the tree passed in is already ordered */
  int32_t sibling_batch;       /* run each maximal run of consecutive childless siblings as one
                                  varlen segment batch over the shared prefix (logical DFS order,
                                  trace and results unchanged up to fp32 summation order) */
  int32_t reserved;
  uint64_t batch_token_budget; /* max tokens per sibling batch; 0 = unlimited */
} tt_sched_config;

/* TrainStepResult counters + device measurements. */
typedef struct tt_step_result {
  double total_loss;
  uint64_t forward_tokens;
  uint64_t recompute_tokens;
  uint64_t backward_tokens;
  uint64_t peak_live_kv_tokens;
  uint64_t peak_live_activation_tokens;
  uint64_t num_segments;
  uint64_t num_chunks;
  uint64_t rollout_tokens;   /* sum of sequence lengths covered by the step */
  uint64_t num_batches;      /* executed segment batches (== num_segments without batching) */
  uint64_t num_launches;     /* device kernel launches issued by the step */
  uint64_t peak_hbm_bytes;   /* engine static allocations + activation-arena high-water */
  uint64_t h2d_bytes;        /* host->device bytes of the step (plan metadata: tokens, tables, loss CSR) */
  uint64_t d2h_bytes;        /* device->host bytes of the step (the loss) */
} tt_step_result;

/* ------------------------------------------------------------------ prefix tree */
typedef struct tt_tree tt_tree;

/* build_prefix_tree. Sequence i occupies tokens[offsets[i], offsets[i+1]) and
 * weights[...] (per-token loss weights, TokenSequence token_sequence.hpp:15-21); its seq_id is i. */
int tt_tree_build(const int32_t* tokens, const uint64_t* offsets, const double* weights, uint64_t n_seqs,
                  tt_tree** out);
int tt_tree_destroy(tt_tree* tree);
/* order_children, recursively, stable tie-break by first token ascending. */
int tt_tree_order_children(tt_tree* tree, int32_t policy);
/* tree_token_count and companions. */
int tt_tree_stats(const tt_tree* tree, uint64_t* tree_tokens, uint64_t* num_sequences, uint64_t* num_nodes,
                  uint64_t* max_path_tokens);
/* Canonical pre-order text serialisation (bit-exact structure check) and the DFS PUSH/POP trace. */
int tt_tree_serialize(const tt_tree* tree, char* buf, uint64_t cap, uint64_t* len);
int tt_tree_dfs_trace(const tt_tree* tree, char* buf, uint64_t cap, uint64_t* len);

/* ------------------------------------------------------------------ partitioner */
/* lexicographic_sort: order_out[k] = index of the k-th sequence. */
int tt_lexicographic_sort(const int32_t* tokens, const uint64_t* offsets, uint64_t n_seqs, uint64_t* order_out);
/* partition_contiguous. group_of_seq[i] in [0,K) for input sequence i;
 * group_costs[K] = C(T_j); max_cost; duplicated = sum_j C(T_j) - C(combined). */
int tt_partition_contiguous(const int32_t* tokens, const uint64_t* offsets, uint64_t n_seqs, uint64_t K,
                            int32_t* group_of_seq, uint64_t* group_costs, uint64_t* max_cost,
                            uint64_t* duplicated);
/* greedy_least_loaded; cost_mode 0 = tree_tokens, 1 = raw_tokens. */
int tt_greedy_least_loaded(const int32_t* tokens, const uint64_t* offsets, uint64_t n_seqs, uint64_t K,
                           int32_t cost_mode, int32_t* group_of_seq, uint64_t* group_costs, uint64_t* max_cost,
                           uint64_t* duplicated);

/* ------------------------------------------------------------------ corpus */
/* A rollout corpus: JSON lines {"seq_id": str, "tokens": [int], "weights": [float]} (weights
 * optional: 0 on the first "prompt_len" positions when given, else 1). */
typedef struct tt_corpus tt_corpus;
/* CorpusSpec; lengths uniform in [lo, hi]. */
typedef struct tt_corpus_spec {
  uint64_t num_prompts;
  uint64_t group_size;
  uint64_t prompt_len_lo, prompt_len_hi;
  uint64_t response_len_lo, response_len_hi;
  double branch_prob;
  uint64_t vocab_size;
  uint64_t seed;
} tt_corpus_spec;
int tt_corpus_load_jsonl(const char* path, tt_corpus** out);
/* gen-corpus: deterministic per seed. */
int tt_corpus_generate(const tt_corpus_spec* spec, tt_corpus** out);
/* CSR view in, string ids optional (NULL -> "0", "1", ...). */
int tt_corpus_from_csr(const int32_t* tokens, const uint64_t* offsets, const double* weights, uint64_t n_seqs,
                       const char* const* seq_ids, tt_corpus** out);
int tt_corpus_save_jsonl(const tt_corpus* corpus, const char* path);
int tt_corpus_size(const tt_corpus* corpus, uint64_t* n_seqs, uint64_t* n_tokens);
/* offsets[n_seqs + 1], tokens[n_tokens], weights[n_tokens] (any may be NULL). */
int tt_corpus_export(const tt_corpus* corpus, int32_t* tokens, uint64_t* offsets, double* weights);
/* seq_id of sequence i into buf (NUL-terminated, truncated to buf_len); *needed = strlen + 1. */
int tt_corpus_seq_id(const tt_corpus* corpus, uint64_t i, char* buf, uint64_t buf_len, uint64_t* needed);
int tt_corpus_destroy(tt_corpus* corpus);

/* ------------------------------------------------------------------ engine */
typedef struct tt_engine tt_engine;

int tt_param_count(const tt_model_config* cfg, uint64_t* n);
int tt_engine_create(const tt_model_config* cfg, int32_t device, tt_engine** out);
int tt_engine_destroy(tt_engine* eng);
/* cudaStream_t of the engine (for event timing / stream interop by the caller). */
int tt_engine_stream(tt_engine* eng, void** stream);

/* Parameters in for_each_tensor order (model.hpp:42-59), converted to the device layout. */
int tt_params_upload_f32(tt_engine* eng, const float* flat, uint64_t n);
int tt_params_upload_f64(tt_engine* eng, const double* flat, uint64_t n);
/* Device-side random init: N(0, 0.02) weights, gains 1 (the distribution of model.hpp:119-142;
 * not bitwise the reference's mt19937_64 stream). */
int tt_params_init_random(tt_engine* eng, uint64_t seed);
/* load_parameters (model_io.cpp:73-105): "TTPM" file with f32 or f64 payload. */
int tt_params_load_ttpm(tt_engine* eng, const char* path);

/* GradientStore (model.hpp:76-81): fp32 flat buffer in for_each_tensor order. */
int tt_grads_zero(tt_engine* eng); /* zero_gradients, model.hpp:110-117 */
int tt_grads_download_f32(tt_engine* eng, float* out, uint64_t n);
/* GradientStore<double> (model.hpp:76-81): the fp32 device gradients widened to double. */
int tt_grads_download_f64(tt_engine* eng, double* out, uint64_t n);
int tt_grads_device_ptr(tt_engine* eng, float** dptr, uint64_t* n);
int tt_grads_accum_count(tt_engine* eng, uint64_t* count);

/* weighted_nll (model.hpp:643-677) on the device: logits [n x V] fp32 (host or device pointer),
 * loss = sum_p w_p (lse - logit[target_p]) in fp64, grad_logits_out [n x V] fp32 (host or device,
 * may be NULL) = per row (sum_p w_p) softmax - sum_p w_p onehot(target_p). row_off[n + 1] makes
 * rows multi-target (the tree's node-boundary rows); NULL = one (target, weight) per
 * row, exactly the reference signature. Pairs of weight 0 contribute nothing (model.hpp:658).
 * Errors as the reference: target out of range / non-finite weight -> TT_ERR_INVALID_ARGUMENT. */
int tt_weighted_nll(tt_engine* eng, const float* logits, uint64_t n, const uint64_t* row_off, const int32_t* targets,
                    const double* weights, double* loss_out, float* grad_logits_out);

/* ------------------------------------------------------------------ multi-GPU
 * One process per GPU (or one process driving all GPUs with tt_nccl_comm_init_all), one NCCL
 * communicator per engine, ONE in-place sum all-reduce of the fp32 GradientStore per step — the
 * reduction the reference does across workers in worker order. Communicators are
 * ncclComm_t values passed as void*; libnccl.so.2 is bound at run time (the copy already loaded in
 * the process if any). */
#define TT_NCCL_UNIQUE_ID_BYTES 128
int tt_nccl_unique_id(uint8_t* id_out /* TT_NCCL_UNIQUE_ID_BYTES */);
int tt_nccl_comm_init_rank(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, void** comm_out);
int tt_nccl_comm_init_all(int32_t ndev, const int32_t* devices, void** comms_out);
int tt_nccl_comm_destroy(void* comm);
/* In-place ncclAllReduce(sum, fp32) of the engine's GradientStore on the engine stream; returns
 * after it completed. */
int tt_grads_allreduce(tt_engine* eng, void* nccl_comm);

/* tree_train_step: one DFS push/visit/pop pass over `tree`, gradients added
 * into the engine's GradientStore, loss in result->total_loss. */
int tt_tree_train_step(tt_engine* eng, const tt_tree* tree, const tt_sched_config* sched, tt_step_result* result);
/* dense_train_step: the flat per-sequence baseline on the same engine. */
int tt_dense_train_step(tt_engine* eng, const int32_t* tokens, const uint64_t* offsets, const double* weights,
                        uint64_t n_seqs, tt_step_result* result);

/* tree_train_step split in two: plan (DFS schedule, sibling batches, memory plan, metadata uploaded
 * to HBM once) and execute (the device push/visit/pop pass). A plan may be executed many times;
 * tt_tree_train_step == create + execute + destroy. The plan's logical PUSH/POP trace equals
 * tt_tree_dfs_trace() of the tree. */
typedef struct tt_step_plan tt_step_plan;
int tt_plan_create(tt_engine* eng, const tt_tree* tree, const tt_sched_config* sched, tt_step_plan** out);
int tt_plan_execute(tt_engine* eng, tt_step_plan* plan, tt_step_result* result);
/* Asynchronous execute: enqueue the step and return at once; tt_plan_wait blocks for it and fills the
 * result (loss, counters; TT_ERR_NONFINITE as tt_plan_execute). One step in flight per engine. While
 * it runs, the host may build and tt_plan_create the next step (plan metadata is copied on a separate
 * stream without synchronising the engine), so a training loop overlaps host planning with the
 * device step. tt_plan_execute == execute_async + wait. */
int tt_plan_execute_async(tt_engine* eng, tt_step_plan* plan);
int tt_plan_wait(tt_engine* eng, tt_step_plan* plan, tt_step_result* result);
int tt_plan_trace(const tt_step_plan* plan, char* buf, uint64_t cap, uint64_t* len);
int tt_plan_destroy(tt_step_plan* plan);

/* Per-kernel-class device timing (CUDA events around every launch while enabled).
 * Classes: 0 GEMM (tcgen05), 1 attention fwd, 2 attention bwd, 3 elementwise/stack, 4 CE.
 * Arrays have TT_NUM_KCLASS entries: accumulated ms, algorithmic FLOPs, algorithmic bytes, launches. */
#define TT_NUM_KCLASS 5
int tt_engine_set_profiling(tt_engine* eng, int32_t on);
/* Execution options (results are unchanged up to fp32 summation order; a prepared plan's CUDA graph
 * is re-captured after any change):
 *   "gemm_2cta"          0 = single-CTA GEMM tiles only, 1 = CTA pairs (cta_group::2) where they fit (default)
 *   "root_batch_tokens"  token cap of a multi-root prompt push (default 4096; 0 = one root per push)
 *   "cuda_graph"         0 = eager launches, 1 = capture a prepared plan's op list on its 2nd execute (default)
 *   "ce_stats"           1 = LM-head GEMM emits per-row softmax statistics for CE (default), 0 = CE two-pass
 *   "logits_bf16"        1 = LM-head logits stored bf16 relative to their 32-column group max (default; with
 *                        ce_stats), 0 = fp32 logits (loss / gradients then differ by bf16 rounding only)
 *   "head_chunk_mb"      LM-head / CE scratch budget per loss-row chunk (default 6144, >= 1; capped by free HBM)
 *   "plan_timing"        1 = print the host phases of tt_plan_create (schedule, memory plan, metadata) to stderr
 *   "pdl_auto_elems"     the batch size (rows x d_model elements) up to which pdl = 2 enables PDL (default 2^21)
 *   "gn_bf16"            1 = the grad_normed outputs of the dX GEMMs stored bf16 for the RMSNorm backward (default,
 *                        d_model % 8 == 0 and <= 4096), 0 = fp32 (loss unchanged; gradients differ by bf16 rounding)
 *   "pdl"                programmatic dependent launch of every kernel: 0 = off, 1 = on, 2 = segment batches of
 *                        at most 2^21 rows x d_model elements (default; launch-bound batches gain, large ones not)
 * Unknown keys and out-of-range values return TT_ERR_INVALID_ARGUMENT. */
int tt_engine_set_option(tt_engine* eng, const char* key, int64_t value);
int tt_engine_profile(tt_engine* eng, double* ms, double* flops, double* bytes, uint64_t* launches, int32_t reset);
/* Per-GEMM-shape breakdown of the profiled launches (text, one shape per line, slowest first). */
int tt_engine_profile_gemm_text(tt_engine* eng, char* buf, uint64_t cap, uint64_t* len);

/* ------------------------------------------------------------------ segment level (device KV stack)
 * forward_segment (model.hpp:328-463) continuing from the device stack (KVView of all pushed
 * segments, start_position = current stack length). logits_out: [len x V] fp32, host or device
 * pointer, or NULL. Equivalent to tt_segment_push_ex(..., want_kv = 1, want_activations = 1, ...). */
int tt_segment_push(tt_engine* eng, const int32_t* tokens, uint64_t len, float* logits_out);
/* forward_segment's want_kv / want_activations (model.hpp:328-331, ForwardResult :232-237):
 *   want_kv = 0           the segment's K/V rows are not kept for descendants: pushing on top of it
 *                         fails with TT_ERR_INVALID_ARGUMENT (a childless node, leaf_kv_skip);
 *   want_activations = 0  activations are dropped after the forward; its pop recomputes them from
 *                         the stack before the backward (the chunked backward's recompute);
 *   both 0                forward only (logits): nothing is pushed. */
int tt_segment_push_ex(tt_engine* eng, const int32_t* tokens, uint64_t len, int32_t want_kv, int32_t want_activations,
                       float* logits_out);
/* weighted_nll of the TOP segment's logits, on the device (the VISIT of SPEC.md:225): pairs as in
 * tt_weighted_nll over the segment's rows (row_off[len + 1] or NULL). *loss_out gets the loss now;
 * the segment's pop then takes its upstream grad_logits from these pairs (fused LM-head GEMM + CE,
 * no logits cross PCIe). */
int tt_segment_loss(tt_engine* eng, const uint64_t* row_off, const int32_t* targets, const double* weights,
                    double* loss_out);
/* backward_segment (model.hpp:474-633) of the top segment. Upstream grad_logits: [len x V] fp32
 * (host or device) or NULL (= zero, or the device pairs of tt_segment_loss; giving both is an
 * error). grad_new_kv is the dK/dV the popped segment's rows accumulated from segments popped above
 * it. grad_prefix (the returned KVGrad, rows [0,S)) is added into the ancestors' dK/dV stack rows
 * (KVGrad::add_rows, model.hpp:193-206); grad_prefix_out (host or device, [L][2][S][d] fp32, K then
 * V) additionally receives exactly this pop's contribution when not NULL. */
int tt_segment_pop(tt_engine* eng, const float* grad_logits, float* grad_prefix_out);
int tt_stack_reset(tt_engine* eng);
int tt_stack_depth(tt_engine* eng, uint64_t* segments, uint64_t* tokens);

const char* tt_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* TREETRAIN_B200_H_ */
