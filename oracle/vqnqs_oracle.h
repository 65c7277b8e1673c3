/* TEST INFRASTRUCTURE — plain-C restatement of the reference's local-energy
 * path, used only as the parity checker by tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline leg. Never linked into the product.
 *
 * Symbol-for-symbol the same C surface as oracle/ref_harness.cpp (prefix
 * orc_ instead of ref_), so the Python front-end (oracle/oracle.py) drives
 * both through one class. Status codes follow the reference's exception
 * taxonomy (proj/include/vqnqs/common.hpp:14-28): 0 ok, 1 Config, 2 Shape,
 * 3 Capability, 4 Numeric, 5 Usage, 6 other.
 */
#ifndef VQNQS_ORACLE_H
#define VQNQS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_sites, group_size, d_hidden, n_heads, n_blocks;
  int32_t trailing_half_block, vq_enabled, vq_heads, vq_codebook, phase_enabled;
  double vq_init_scale;
} orc_model_desc;

const char* orc_last_error(void);
void orc_set_bf16_products(int on);
void* orc_model_create(const orc_model_desc* d, uint64_t seed, int snap_bf16);
void orc_model_destroy(void* m);
int orc_model_num_params(void* m);
int64_t orc_model_param(void* m, int i, double** data, const char** name);
void* orc_ham_create(int kind, int lattice, int lx, int ly, int marshall,
                     double J, double Gamma);
void orc_ham_destroy(void* h);
int orc_ham_bonds(void* h, int32_t* out, int cap);
int orc_connected_set(void* h, const uint8_t* s, int cap, uint8_t* configs,
                      double* coeffs);
void orc_zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed,
                         uint8_t* out);
int orc_local_energies(void* m, void* h, const uint8_t* configs, int64_t B,
                       int workers, double* e_re, double* e_im, double* logpsi,
                       int64_t* ledger7);
int orc_local_energies_fast(void* m, void* h, const uint8_t* configs,
                            int64_t B, int workers, double* e_re);
int orc_dedup_log_prob(void* m, const uint8_t* configs, int64_t K,
                       const uint8_t* base, double* lp);
int orc_dense_log_prob(void* m, const uint8_t* configs, int64_t K, double* lp);
/* VqTransformer::sample (proj/src/model.cpp:485-525) with Rng(seed):
 * configs [count x n_sites], log_probs [count]. */
int orc_sample(void* m, int count, uint64_t seed, uint8_t* configs, double* log_probs);
int orc_taps(void* m, void* h, const uint8_t* s, int64_t* U, int32_t* codes,
             float* gaps, double* lp, int32_t* I_final);

#ifdef __cplusplus
}
#endif
#endif
