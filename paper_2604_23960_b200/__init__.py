"""B200-native batched multi-robot MotionValidation / FindFirstConflict
(arxiv 2604.23960) behind the C ABI in include/mrv.h.

Modules:
  mrv    -- ctypes binding of libmrv.so (argument marshalling only)
  gen    -- seeded synthetic inputs for BASELINE.json's configs (no method arithmetic)
  dist   -- motion-index sharding + NCCL all-gather of per-motion results
  build  -- nvcc build of libmrv.so for sm_100a
"""
__all__ = ["mrv", "gen", "dist", "build"]
