"""B200-native batched adaptive-LP decoding of LDPC codes (arXiv 0902.0657).

The product is libalp.so (include/alp.h): hand-written sm_100a CUDA kernels behind a
C ABI.  This package is its thin Python binding (api), the in-tree build (build) and
the multi-GPU sharding helpers (dist).  It never imports `oracle/`.
"""
from .api import (AlpError, Code, DecodeResult, StepResult, Workspace, decode, decode_host,
                  default_params, ipm_step_pcg, last_launch_count, launch_info, lib, STATS_DTYPE)

__all__ = ["AlpError", "Code", "DecodeResult", "StepResult", "Workspace", "decode", "decode_host",
           "default_params", "ipm_step_pcg", "last_launch_count", "launch_info", "lib", "STATS_DTYPE"]
