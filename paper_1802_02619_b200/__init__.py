"""B200-native permutation of sorted LCO sparse tensors (arXiv 1802.02619 hot path).

The work runs in liblco.so (hand-written sm_100a CUDA behind the C ABI in
include/lco.h); this package is the thin Python binding plus the sharded driver.
"""
from .lco import (FLAG_HIERARCHICAL, FLAG_VALIDATE, LcoError, LcoValueError, Plan, add,
                  compress, fastdiv_host, flatten, lib, mdt_choice, permute, plan, sort,
                  sparsity_class, version)

__all__ = ["FLAG_HIERARCHICAL", "FLAG_VALIDATE", "LcoError", "LcoValueError", "Plan", "add",
           "compress", "fastdiv_host", "flatten", "lib", "mdt_choice", "permute", "plan", "sort",
           "sparsity_class", "version"]
