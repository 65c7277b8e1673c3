/* vqnqs_b200 — C ABI of the B200-native local-energy engine.
 *
 * This is the drop-in boundary for the reference's local-energy path. The
 * reference exposes it as C++ (proj/include/vqnqs/trainer.hpp:76-79,
 * proj/include/vqnqs/dedup.hpp:77-93); a C++ caller keeps those signatures by
 * going through the header-only adapter include/vqnqs_b200.hpp, which calls
 * the functions below. Plain pointers and sizes only — no torch, no STL.
 *
 * Status codes mirror the reference's exception taxonomy
 * (proj/include/vqnqs/common.hpp:14-28); the adapter re-throws them as the
 * matching vqnqs::*Error. The message of the last failure on the calling
 * thread is vqnqs_last_error().
 *
 * A handle is bound to one CUDA device and is not thread-safe: serialise
 * calls on it (the reference's worker pool becomes one handle per GPU).
 */
#ifndef VQNQS_B200_H
#define VQNQS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VQNQS_OK = 0,
  VQNQS_CONFIG_ERROR = 1,     /* vqnqs::ConfigError */
  VQNQS_SHAPE_ERROR = 2,      /* vqnqs::ShapeError (check()) */
  VQNQS_CAPABILITY_ERROR = 3, /* vqnqs::CapabilityError */
  VQNQS_NUMERIC_ERROR = 4,    /* vqnqs::NumericError (non-finite E_loc) */
  VQNQS_USAGE_ERROR = 5,      /* vqnqs::UsageError */
  VQNQS_RUNTIME_ERROR = 6     /* CUDA / allocation failure */
};

enum { VQNQS_PREC_FP32 = 0, VQNQS_PREC_BF16 = 1 };

/* Field-for-field subset of vqnqs::ModelConfig
 * (proj/include/vqnqs/model.hpp:13-27); local_dim is fixed at 2. */
typedef struct {
  int32_t n_sites, group_size, d_hidden, n_heads, n_blocks;
  int32_t trailing_half_block, vq_enabled, vq_heads, vq_codebook, phase_enabled;
  double vq_init_scale;
} vqnqs_model_desc;

typedef struct vqnqs_handle vqnqs_handle;

/* Ledger slots, in the order of flops::Ledger's fields
 * (proj/include/vqnqs/flops.hpp:12-44). */
enum {
  VQNQS_LEDGER_PER_LOCATION_DENSE = 0,
  VQNQS_LEDGER_PER_LOCATION_UNIQUE = 1,
  VQNQS_LEDGER_ATTENTION = 2,
  VQNQS_LEDGER_VQ_DISTANCE = 3,
  VQNQS_LEDGER_OTHER = 4,
  VQNQS_LEDGER_PER_LOCATION_DENSE_QUANTIZED = 5,
  VQNQS_LEDGER_PER_LOCATION_UNIQUE_QUANTIZED = 6,
  VQNQS_LEDGER_SLOTS = 7
};

const char* vqnqs_last_error(void);

/* ---- host-side model/lattice helpers (no GPU needed) ---- */

/* Number of parameter tensors and the numel of each, in the reference's
 * parameters() order (proj/src/model.cpp:210-229). numels may be NULL. */
int vqnqs_param_layout(const vqnqs_model_desc* d, int* n_params, int64_t* numels);

/* VqTransformer::init(cfg, Rng(seed)) (proj/src/model.cpp:150-184): fills the
 * caller's float64 buffers (parameters() order, sizes from
 * vqnqs_param_layout). snap_bf16 rounds every value to bf16. */
int vqnqs_init_params(const vqnqs_model_desc* d, uint64_t seed, int snap_bf16,
                      double* const* params);

/* Lattice bonds (proj/src/hamiltonian.cpp:5-35); periodic=1 adds the wrap
 * bonds of SURVEY §8d. ly=0 for chains. Returns the bond count (writes at
 * most cap pairs), or -status. */
int vqnqs_build_lattice(int lx, int ly, int periodic, int32_t* bonds, int cap);

/* Zero-Sz configurations: sample i <- Rng(seed).split(start + i), N/2 up
 * spins shuffled by Fisher-Yates. out is [count x n]. */
int vqnqs_zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed,
                          uint8_t* out);

/* The reference's FLOP ledger for one connected set (flops::Ledger after
 * local_energy_batch, proj/src/dedup.cpp:394-420 with opcost,
 * proj/include/vqnqs/tensor.hpp:81-102) from its size K and the realised
 * unique-row counts U[0..L] (L = blocks incl. a trailing half block).
 * ADDS into ledger7. The engine fills ledgers this way. */
int vqnqs_ledger_from_counts(const vqnqs_model_desc* d, int64_t K, const int64_t* U,
                             int64_t* ledger7);

/* ---- engine ---- */

/* Uploads weights (float64, parameters() order) to `device`, converting to
 * the engine precision. Validates like ModelConfig::validate
 * (proj/src/model.cpp:10-27). Replaces constructing a VqTransformer for the
 * GPU: the handle plays the role of `const VqTransformer&`. */
int vqnqs_gpu_create(const vqnqs_model_desc* d, const double* const* params,
                     int n_params, int precision, int device, vqnqs_handle** out);

/* Heisenberg Hamiltonian on an explicit bond list [nb][2] (the fields
 * connected_set reads, proj/src/hamiltonian.cpp:41-74). TFIM is refused
 * with VQNQS_CAPABILITY_ERROR. Plays the role of `const HamiltonianModel&`. */
int vqnqs_gpu_set_hamiltonian(vqnqs_handle* h, const int32_t* bonds, int nb,
                              int n_sites, int marshall);

/* Replaces VqTransformer::sample(count, rng) with rng = Rng(seed)
 * (proj/src/model.cpp:485-525; proj/include/vqnqs/rng.hpp): ancestral
 * sampling of count configurations, one position per step for all samples
 * at once with a per-block K/V cache on the device. configs: host
 * [count x n_sites] bytes; log_probs: host [count], the sampled
 * configurations' log P (the reference recomputes them with log_prob_batch;
 * here they are accumulated during the draw). Draws use the reference's
 * uniforms in the reference's order, so a configuration differs from the
 * reference's only where a uniform falls within rounding of a CDF step.
 * skip = uniforms of the same Rng(seed) stream already consumed (count x T
 * per earlier batch), so consecutive calls continue one stream. */
int vqnqs_gpu_sample(vqnqs_handle* h, int64_t count, uint64_t seed, uint64_t skip,
                     uint8_t* configs, double* log_probs);

/* ---- the score-function gradient ---- */
typedef struct vqnqs_grad_handle vqnqs_grad_handle;

/* fp32 weights of the model on `device` for the backward pass. */
int vqnqs_grad_create(const vqnqs_model_desc* d, const double* const* params, int n_params,
                      int device, vqnqs_grad_handle** out);
/* grads = d/dtheta sum_i weights[i] log P(configs[i]) — the backward of
 * vmc_gradient (proj/src/trainer.cpp:236-244: build_log_prob, weighted_sum,
 * backward; proj/src/autodiff.cpp) with the straight-through VQ surrogate at
 * temperature vq_tau (Graph::vq_quantize, autodiff.cpp:536-655). grads: host,
 * every parameter's gradient concatenated in parameters() order; log_probs:
 * host [B], the dense log P of each configuration. Deterministic. */
int vqnqs_grad_log_prob(vqnqs_grad_handle* h, const uint8_t* configs, int64_t B,
                        const double* weights, double vq_tau, double* grads,
                        double* log_probs);
int vqnqs_grad_destroy(vqnqs_grad_handle* h);

/* reuse = 1 (default): the compressed path. reuse = 0: the reference's
 * no-reuse regime (dense_local_energy, proj/src/bench.cpp:19-36 — every
 * connected configuration's full T-token forward, no shared prefixes, no
 * unique-row merging); same outputs, used for the no_reuse wall-time series
 * (proj/src/bench.cpp:193) and as an independent self-check. */
int vqnqs_gpu_set_reuse(vqnqs_handle* h, int reuse);

/* Samples per micro-batch ("chunk"). 0 (default) sizes it
 * from a device working-set budget. Results do not depend on it (no
 * reduction mixes samples); it exists for memory control and for the
 * multi-micro-batch parity tests. */
int vqnqs_gpu_set_micro_batch(vqnqs_handle* h, int samples);

/* Replaces local_energies(model, h, batch, ledger)
 * (proj/include/vqnqs/trainer.hpp:76-79, proj/src/trainer.cpp:150-180).
 * configs: host [B x n_sites] bytes (0 = down, 1 = up). Outputs host arrays
 * of B doubles; e_im/logpsi/ledger7 may be NULL. logpsi = 0.5 * log P(s)
 * (proj/src/model.cpp:481-483). ledger7 is ADDED to (like
 * `*ledger += part`, trainer.cpp:177-178). Synchronous. A non-finite E_loc
 * returns VQNQS_NUMERIC_ERROR naming the configuration, like the reference. */
int vqnqs_gpu_local_energies(vqnqs_handle* h, const uint8_t* configs, int64_t B,
                             double* e_re, double* e_im, double* logpsi,
                             int64_t* ledger7);

/* Same, on device buffers (configs, e_re, logpsi on the handle's device),
 * ordered on `stream` (a cudaStream_t, NULL = the handle's own stream).
 * Returns after enqueueing the last kernel for this batch; the ledger (host)
 * is filled after the engine's per-chunk size readbacks. */
int vqnqs_gpu_local_energies_device(vqnqs_handle* h, const uint8_t* d_configs,
                                    int64_t B, double* d_e_re, double* d_logpsi,
                                    int64_t* ledger7, void* stream);

/* Replaces dedup_log_prob(model, configs, base) (proj/include/vqnqs/dedup.hpp:77-79)
 * for the connected set of `base`: per-row log-probs lp[K] in connected_set
 * order (diagonal first, then bond order). Returns K (>0) or -status. */
int vqnqs_gpu_connected_log_probs(vqnqs_handle* h, const uint8_t* base,
                                  double* lp, int cap);

/* Parity taps for a batch (same layout as the oracle's taps):
 *   K[B], U[B*(L+1)], codes[sum_s K_s*T*L] (layer-major per sample:
 *   sample s occupies L*K_s*T entries, [layer][row][pos]),
 *   lp_rows[sum_s K_s] per-row log-probs in connected_set order.
 * Returns 0 or status. Any output pointer may be NULL. */
int vqnqs_gpu_taps(vqnqs_handle* h, const uint8_t* configs, int64_t B,
                   int32_t* K, int64_t* U, int32_t* codes, int64_t codes_cap,
                   double* lp_rows, int64_t lp_cap);

/* ---- multi-GPU statistics (one process per GPU) ---- */

/* An NCCL communicator over the ranks of one job. Rank 0 calls
 * vqnqs_comm_unique_id and shares the VQNQS_COMM_ID_BYTES bytes out of band
 * (MPI, torch.distributed, a file); every rank then calls vqnqs_comm_create
 * with its rank and the CUDA device of its engine. */
typedef struct vqnqs_comm vqnqs_comm;
#define VQNQS_COMM_ID_BYTES 128
int vqnqs_comm_unique_id(char* id);
int vqnqs_comm_create(const char* id, int world, int rank, int device, vqnqs_comm** out);
int vqnqs_comm_destroy(vqnqs_comm* c);

/* estimate_energy's statistics (proj/src/trainer.cpp:200-211 and fill_stats,
 * :184-198) over a batch sharded by sample across the ranks of `comm`: each
 * rank passes its own B configurations (host); stats = {energy (mean Re E),
 * variance (unbiased, two-pass), std_err = sqrt(variance / k), k} over ALL
 * ranks' samples; e_re / logpsi (host [B], nullable) are this rank's; the
 * ledger (nullable) is ADDED the whole job's ledger. The sums are fp64 on the
 * device in a fixed order plus one NCCL allreduce per pass (the only
 * data-path collective). comm = NULL: this process alone. A non-finite E_loc
 * on any rank makes every rank return VQNQS_NUMERIC_ERROR. */
int vqnqs_gpu_estimate_energy(vqnqs_handle* h, vqnqs_comm* comm, const uint8_t* configs,
                              int64_t B, double* e_re, double* logpsi, int64_t* ledger7,
                              double* stats);

/* The same statistics for local energies already on the device (d_e_re [B],
 * this rank's shard, e.g. from vqnqs_gpu_local_energies_device), ordered on
 * `stream` (NULL = the handle's stream); synchronous. */
int vqnqs_gpu_fill_stats_device(vqnqs_handle* h, vqnqs_comm* comm, const double* d_e_re,
                                int64_t B, double* stats, void* stream);

/* Balanced sample shards: owner[i] = the rank that evaluates
 * sample i, dealing samples in decreasing connected-set size
 * K = 1 + #antiparallel bonds to the rank with the least total K so far, so
 * every rank gets about the same number of evaluations. */
int vqnqs_balanced_shards(const uint8_t* configs, int64_t B, int n_sites, const int32_t* bonds,
                          int nb, int world, int32_t* owner);

/* Kernel launches issued by the last local-energies call (own kernels only). */
int64_t vqnqs_gpu_last_launch_count(vqnqs_handle* h);

/* Per-call timings of the last call's dominant kernel family (ms, CUDA events
 * on the engine stream) and its algorithmic work; see DESIGN.md. Slots:
 * [0] attention+VQ ms  [1] their algorithmic flops  [2] launches timed
 * [3] active locations  [4] sum U_b  [5] sum U_{b+1}  [6] VQ ms
 * [7] attention ms  [8] VQ rows re-scored  [9] attention flops
 * [10] VQ distance flops  [11] attention tiles (<= 128 active locations each). */
int vqnqs_gpu_last_profile(vqnqs_handle* h, double* out, int cap);

int vqnqs_gpu_destroy(vqnqs_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* VQNQS_B200_H */
