"""paper_2309_12381_b200 -- B200-native residual-compensated 16-bit optimizer step (arXiv 2309.12381).

The hot path is the CUDA library ``lib/libmpo.so`` (C ABI: include/mpo.h); this package is its
thin binding (``api``), the user-facing optimizers (``optim``) and the data-parallel sharded
driver (``sharded``).  Importing it does not touch the GPU; calling into it without the built
library raises (there is no CPU fallback).
"""
from .api import (AdamParams, SgdParams, TensorTable, mpo_adam_step, mpo_comm_check,  # noqa: F401
                  mpo_fused_backward_hook_step, mpo_grad_sumsq, mpo_p2p_sharded_step, mpo_reconstruct, mpo_sgd_step,
                  mpo_sharded_step, mpo_split, norm_ws_doubles)
from ._lib import MpoError  # noqa: F401
from .optim import ResidualAdamW, ResidualSGD  # noqa: F401
from .sharded import (BucketedShardedOptimizer, BucketLayout, ShardedResidualAdamW, ShardedResidualOptimizer,  # noqa: F401
                      ShardedResidualSGD, ShardLayout)

__all__ = ["mpo_split", "mpo_reconstruct", "mpo_sgd_step", "mpo_adam_step", "mpo_fused_backward_hook_step",
           "mpo_sharded_step", "mpo_p2p_sharded_step", "mpo_grad_sumsq", "mpo_comm_check", "TensorTable", "SgdParams", "AdamParams", "ResidualSGD", "ResidualAdamW",
           "ShardedResidualOptimizer", "ShardedResidualAdamW", "ShardedResidualSGD", "ShardLayout", "BucketedShardedOptimizer", "BucketLayout", "MpoError",
           "norm_ws_doubles"]
