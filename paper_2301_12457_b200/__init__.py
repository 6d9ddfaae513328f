"""B200-native EvoX PSO/CSO generation engine (arXiv 2301.12457).

The hot path (one ask-evaluate-tell generation over X[pop x dim]) runs in the
sm_100a kernels of ``libevox.so`` behind the C-ABI ``include/evox.h``; this
package is the thin ctypes binding.  See DESIGN.md.
"""
from .evox import (CSO, DE, PSO, DEFAULT_BOUNDS, PROBLEMS, EvoxError, evaluate, lib, nccl_unique_id,
                   shard_rows, version)

__all__ = ["PSO", "CSO", "DE", "evaluate", "shard_rows", "nccl_unique_id", "version", "lib",
           "PROBLEMS", "DEFAULT_BOUNDS", "EvoxError"]
