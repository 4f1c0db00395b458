"""B200-native (sm_100a) RGSW CCMM / PPMM-mod-Q engine for arXiv 2601.17561.

Modules (all compute runs in libirl_b200.so through the C ABI include/irl_capi.h;
there is no CPU fallback):
  modmat  -- irislab::modmat mirror: digit split, small_gemm, gemm_mod_psq, gemm_mod_Q
  ccmm    -- the device-resident CCMM engine (8-slice database) and ccmm_twin
  iris    -- plaintext iris scoring: overlaps, scores, match_db_reference, template files
  fold    -- Alg. 2 fold stage: normalize, folding polynomial + Rot, fold chain, refold
  dist    -- the paper's multi-GPU layout (part dealing, a-part exchange)
  build   -- in-tree nvcc build of libirl_b200.so for sm_100a
"""
