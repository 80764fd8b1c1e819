"""B200-native WallFacer multi-ring attention (arXiv 2407.00611).

The product is libwf.so (C ABI, include/wf.h) built from csrc/; this package is
its thin Python binding.  See DESIGN.md.
"""
from .wf import (SCHED_DIRECT_PULL, SCHED_GATHER_SHUFFLE, Context, WFError, block_bwd, block_fwd, gemm_bf16,  # noqa: F401
                 plan, plan_trace, shard_ranges, workspace_bytes)
