"""B200-native tensor-parallel forward of low-rank-decomposed LLaMA-3 blocks
(arxiv 2604.17709, "DeInfer").  The product is the C-ABI library libdl.so
(include/dl.h, sources in csrc/); this package is its thin Python binding.
"""
from ._lib import (DL_BF16, DL_DECODE, DL_F32, DL_LAYOUT_DEINFER, DL_LAYOUT_RANK_PARALLEL, DL_MLP_RELU,
                   DL_MLP_SILU_GLU, DL_PREFILL, EXPORTS, dl_deinfer_shard_factors, LowRankKVCache, dl_kv_prepare,
                   dl_decomposed_block_forward_kvlr, dl_decomposed_stack_forward, StackArgs, dl_argmax, BlockWeights, Comm, DLError,  # noqa: F401
                   dl_block_config, dl_block_workspace, dl_comm_create, dl_decomposed_block_forward, dl_dense,
                   dl_device_ok, dl_embedding, dl_lowrank_linear, dl_lowrank_linear_workspace, dl_rmsnorm,
                   dl_tp_plan, dl_tp_shard_factors, dl_version, load, make_block_config,
                   dl_launch_count, dl_profile_begin, dl_profile_end, dl_profile_records,
                   DL_REDUCE_NONE, DL_REDUCE_ALLREDUCE, DL_REDUCE_SCATTER, run_ranks,
                   dl_block_window_bytes)
