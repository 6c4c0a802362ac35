"""CodecSight hot path on B200 (sm_100a): codec metadata -> pruned visual tokens -> refreshed KV cache.

The compute lives in ``libcodecsight.so`` (hand-written CUDA kernels behind the C ABI of include/codecsight.h).
This package is the thin Python binding (``_abi``) plus per-stream device state (``pipeline``).
"""
from ._abi import (CodecSightError, codecsight_compact, codecsight_kv_refresh, codecsight_score_patches, compact,
                   kv_refresh, kv_workspace_size, ptr_array, score_patches)

__all__ = ["CodecSightError", "codecsight_score_patches", "codecsight_compact", "codecsight_kv_refresh",
           "score_patches", "compact", "kv_refresh", "kv_workspace_size", "ptr_array"]
