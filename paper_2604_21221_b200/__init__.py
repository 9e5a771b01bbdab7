"""B200-native Persistent Block-Sparse Attention (PBSA), the hot path of Sparse Forcing.

Importing the package loads libpbsa_b200.so (sm_100a kernels behind a C ABI, see
include/pbsa_b200.h); there is no CPU fallback.
"""
from .pbsa import (MODE_CACHE_UPDATE, MODE_DENOISE, Memory, PbsaCudaError, PbsaError,  # noqa: F401
                   attention_scale, attention_sparse, attention_sparse_backward, compress_blocks, debug_tile, score_select,
                   latent_blocks, latent_geom, topk_count, TensorIoError, write_tensor,
                   read_tensor, tensor_dims, load_bf16, bsa_fwd_last_plan, debug_set_fault,
                   matmul, masked_softmax_rows, aggregate_scores, select_topk, blockify, unblockify, topc_select,
                   pair_tiles)

__version__ = "0.1.0"
