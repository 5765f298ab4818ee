"""ctypes loader for libtreetrain_b200.so (the C-ABI in include/treetrain_b200.h).

The product path has no fallback: if the library is missing, every call fails loudly.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtreetrain_b200.so")
_lib = None

c = ctypes
u64, i32, f64, vp = c.c_uint64, c.c_int32, c.c_double, c.c_void_p
P = c.POINTER


class ModelConfigC(c.Structure):
    _fields_ = [("vocab_size", u64), ("d_model", u64), ("n_heads", u64), ("n_layers", u64), ("d_ff", u64),
                ("max_position", u64), ("precision", i32), ("reserved", i32)]


class SchedConfigC(c.Structure):
    _fields_ = [("chunk_len", u64), ("leaf_kv_skip", i32), ("child_order_policy", i32), ("sibling_batch", i32),
                ("reserved", i32), ("batch_token_budget", u64)]


class StepResultC(c.Structure):
    _fields_ = [("total_loss", f64)] + [(n, u64) for n in (
        "forward_tokens", "recompute_tokens", "backward_tokens", "peak_live_kv_tokens",
        "peak_live_activation_tokens", "num_segments", "num_chunks", "rollout_tokens", "num_batches",
        "num_launches", "peak_hbm_bytes", "h2d_bytes", "d2h_bytes")]


class CorpusSpecC(c.Structure):
    _fields_ = [("num_prompts", u64), ("group_size", u64), ("prompt_len_lo", u64), ("prompt_len_hi", u64),
                ("response_len_lo", u64), ("response_len_hi", u64), ("branch_prob", f64), ("vocab_size", u64),
                ("seed", u64)]


EXPORTS = {
    "tt_corpus_load_jsonl": [c.c_char_p, P(vp)],
    "tt_corpus_generate": [P(CorpusSpecC), P(vp)],
    "tt_corpus_from_csr": [P(i32), P(u64), P(f64), u64, P(c.c_char_p), P(vp)],
    "tt_corpus_save_jsonl": [vp, c.c_char_p],
    "tt_corpus_size": [vp, P(u64), P(u64)],
    "tt_corpus_export": [vp, P(i32), P(u64), P(f64)],
    "tt_corpus_seq_id": [vp, u64, c.c_char_p, u64, P(u64)],
    "tt_corpus_destroy": [vp],
    "tt_tree_build": [P(i32), P(u64), P(f64), u64, P(vp)],
    "tt_tree_destroy": [vp],
    "tt_tree_order_children": [vp, i32],
    "tt_tree_stats": [vp, P(u64), P(u64), P(u64), P(u64)],
    "tt_tree_serialize": [vp, c.c_char_p, u64, P(u64)],
    "tt_tree_dfs_trace": [vp, c.c_char_p, u64, P(u64)],
    "tt_lexicographic_sort": [P(i32), P(u64), u64, P(u64)],
    "tt_partition_contiguous": [P(i32), P(u64), u64, u64, P(i32), P(u64), P(u64), P(u64)],
    "tt_greedy_least_loaded": [P(i32), P(u64), u64, u64, i32, P(i32), P(u64), P(u64), P(u64)],
    "tt_param_count": [P(ModelConfigC), P(u64)],
    "tt_engine_create": [P(ModelConfigC), i32, P(vp)],
    "tt_engine_destroy": [vp],
    "tt_engine_stream": [vp, P(vp)],
    "tt_params_upload_f32": [vp, P(c.c_float), u64],
    "tt_params_upload_f64": [vp, P(f64), u64],
    "tt_params_init_random": [vp, u64],
    "tt_params_load_ttpm": [vp, c.c_char_p],
    "tt_grads_zero": [vp],
    "tt_grads_download_f32": [vp, P(c.c_float), u64],
    "tt_grads_download_f64": [vp, P(f64), u64],
    "tt_weighted_nll": [vp, vp, u64, P(u64), P(i32), P(f64), P(f64), vp],
    "tt_nccl_unique_id": [P(c.c_uint8)],
    "tt_nccl_comm_init_rank": [P(c.c_uint8), i32, i32, i32, P(vp)],
    "tt_nccl_comm_init_all": [i32, P(i32), P(vp)],
    "tt_nccl_comm_destroy": [vp],
    "tt_grads_allreduce": [vp, vp],
    "tt_grads_device_ptr": [vp, P(vp), P(u64)],
    "tt_grads_accum_count": [vp, P(u64)],
    "tt_tree_train_step": [vp, vp, P(SchedConfigC), P(StepResultC)],
    "tt_dense_train_step": [vp, P(i32), P(u64), P(f64), u64, P(StepResultC)],
    "tt_plan_create": [vp, vp, P(SchedConfigC), P(vp)],
    "tt_plan_execute": [vp, vp, P(StepResultC)],
    "tt_plan_execute_async": [vp, vp],
    "tt_plan_wait": [vp, vp, P(StepResultC)],
    "tt_plan_trace": [vp, c.c_char_p, u64, P(u64)],
    "tt_plan_destroy": [vp],
    "tt_engine_set_profiling": [vp, i32],
    "tt_engine_set_option": [vp, c.c_char_p, c.c_int64],
    "tt_debug_attn": [c.c_int, c.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, c.c_int, c.c_int, c.c_int, c.c_int,
                      c.c_long, c.c_int, P(c.c_float)],
    "tt_engine_profile": [vp, P(f64), P(f64), P(f64), P(u64), i32],
    "tt_engine_profile_gemm_text": [vp, c.c_char_p, u64, P(u64)],
    "tt_segment_push": [vp, P(i32), u64, vp],
    "tt_segment_push_ex": [vp, P(i32), u64, i32, i32, vp],
    "tt_segment_loss": [vp, P(u64), P(i32), P(f64), P(f64)],
    "tt_segment_pop": [vp, vp, vp],
    "tt_stack_reset": [vp],
    "tt_stack_depth": [vp, P(u64), P(u64)],
    "tt_last_error": [],
    "tt_debug_gemm": [vp, c.c_long, c.c_int, vp, c.c_long, c.c_int, c.c_int, c.c_int, c.c_int, c.c_int, vp, vp, vp,
                      c.c_long, c.c_int, vp, vp, c.c_int],
    "tt_debug_gemm_async": [vp, c.c_long, c.c_int, vp, c.c_long, c.c_int, c.c_int, c.c_int, c.c_int, c.c_int, vp, vp,
                            vp, c.c_long, c.c_int, vp, vp, c.c_int],
    "tt_debug_gemm_splits": [c.c_int, c.c_int, c.c_int],
    "tt_debug_gemm_set_2cta": [c.c_int],
    "tt_debug_gemm_set_transpose": [c.c_int],
    "tt_debug_gemm_force_bn2": [c.c_int],
    "tt_debug_gemm_force_bn1": [c.c_int],
    "tt_debug_attn_set_segments": [c.c_int],
    "tt_debug_rmsnorm_bwd": [vp, vp, vp, vp, vp, vp, vp, vp, c.c_int, c.c_int],
    "tt_debug_rmsnorm_bwd16": [vp, vp, vp, vp, vp, vp, vp, vp, c.c_int, c.c_int],
}


def lib():
    global _lib
    if _lib is None:
        path = LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(path)
        for name, args in EXPORTS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = c.c_char_p if name == "tt_last_error" else c.c_int
        _lib = L
    return _lib
