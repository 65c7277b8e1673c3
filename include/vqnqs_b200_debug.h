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
/* The tcgen05 gathered causal attention over an explicit location layout
 * (see csrc/debug_hooks.cuh for the arrays); x = xh + xl per location. */
int vqnqs_debug_tc_attention(int S, int R1, int T, int d, int nh, const int32_t* K,
                             const int32_t* row_t1, const int32_t* row_perm,
                             const int64_t* row_aoff, const int64_t* act_off, int64_t M,
                             const int32_t* I, const int64_t* Uoff, const void* qkv, void* xh,
                             void* xl, float* xn2, float* rr2);
/* Engine test hook: force the VQ code of every active location to the
 * reference's (codes host [n_samples][L][nb+1][T] int16, rows in bond order,
 * -1 = keep the computed code) for the following calls on batches of
 * exactly n_samples; codes = NULL clears. vq_heads = 1. */
typedef struct vqnqs_handle vqnqs_handle;
int vqnqs_debug_set_code_override(vqnqs_handle* h, const int16_t* codes, int64_t n_samples);
#ifdef __cplusplus
}
#endif
#endif
