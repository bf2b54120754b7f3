"""B200-native hot path of the contrastive-RL (CRL) critic update of arXiv 2408.11052.

The compute lives in libcrl.so (CUDA for sm_100a, C ABI in include/crl.h); this package is
the thin Python binding (argument marshalling only).
"""
from ._lib import (CrlConfig, CrlContext, CrlError, EXPORTED, LIB_PATH, bootstrap_nccl_id,
                   load_library, nccl_unique_id, workspace_size)

__all__ = ["CrlConfig", "CrlContext", "CrlError", "EXPORTED", "LIB_PATH", "bootstrap_nccl_id",
           "load_library", "nccl_unique_id", "workspace_size"]
