// tcgen05 (5th-gen tensor core) paths for the bf16 configurations.
#pragma once

#include "common.cuh"

namespace vqb {

inline bool tc_supported(int prec, int d, int dh, int T, int Q) {
  (void)prec; (void)d; (void)dh; (void)T; (void)Q;
  return false;
}

inline void tc_gemm(const int64_t*, int64_t, int, int, const void*, int, const int32_t*,
                    const void*, const float*, void*, int, int, const float*, int,
                    const int64_t*, cudaStream_t, int) {}

inline void tc_attention_vq(int, int, int, int, int, int, int, float, const int32_t*,
                            const int32_t*, const int64_t*, const int64_t*, const int32_t*,
                            const int64_t*, const void*, const void*, const float*, int32_t*,
                            cudaStream_t, int, double*) {}

}  // namespace vqb
