/* Kernel-level test hooks of libvqnqs_b200 (tests only; not part of the
 * drop-in surface). Device pointers throughout; synchronous. */
#ifndef VQNQS_B200_DEBUG_H
#define VQNQS_B200_DEBUG_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* out[M x N] = A[M x K] . WT[N x K]^T + bias, epi 0 store bf16, 1 gelu bf16,
 * 2 fp32 residual add (resid [M x N]). use_tc selects tcgen05 vs CUDA cores. */
int vqnqs_debug_gemm_bf16(int64_t M, int N, int K, const void* A, const void* WT,
                          const void* W, const float* bias, void* out, const float* resid,
                          int epi, int use_tc);
/* code[M] = argmin_j |x_m - cb_j|^2 (fp32 x [M x d], fp32 cb [Q x d]). */
int vqnqs_debug_vq(int64_t M, int d, const float* x, const float* cb32, int Q, int32_t* code,
                   int use_tc, unsigned long long* n_rescored);
#ifdef __cplusplus
}
#endif
#endif
