// Internal interface of the B200 local-energy engine (not part of the ABI;
// the ABI is include/vqnqs_b200.h).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vqnqs_b200.h"

namespace vqb {

// Error taxonomy of the reference (proj/include/vqnqs/common.hpp:14-28),
// carried across the C ABI as status codes.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
struct ConfigError : Error {
  explicit ConfigError(const std::string& m) : Error(VQNQS_CONFIG_ERROR, m) {}
};
struct ShapeError : Error {
  explicit ShapeError(const std::string& m) : Error(VQNQS_SHAPE_ERROR, m) {}
};
struct CapabilityError : Error {
  explicit CapabilityError(const std::string& m) : Error(VQNQS_CAPABILITY_ERROR, m) {}
};
struct NumericError : Error {
  explicit NumericError(const std::string& m) : Error(VQNQS_NUMERIC_ERROR, m) {}
};
struct UsageError : Error {
  explicit UsageError(const std::string& m) : Error(VQNQS_USAGE_ERROR, m) {}
};
struct RuntimeError : Error {
  explicit RuntimeError(const std::string& m) : Error(VQNQS_RUNTIME_ERROR, m) {}
};

struct ParamSpec {
  std::string name;
  int64_t rows, cols;
  int init;  // 0 zeros, 1 ones, 2/3 gaussian
  double scale;
};

uint64_t mix64(uint64_t x);
double round_bf16_host(double x);
void validate(const vqnqs_model_desc& c);
std::vector<ParamSpec> param_layout(const vqnqs_model_desc& c);
void init_params(const vqnqs_model_desc& c, uint64_t seed, bool snap, double* const* out);
std::vector<int32_t> build_lattice(int lx, int ly, bool periodic);
void zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed, uint8_t* out);
// n consecutive Rng(seed).uniform() draws (proj/include/vqnqs/rng.hpp:22).
void rng_uniforms(uint64_t seed, int64_t n, double* out);

// Host-side restatement of the reference ledger for one sample
// (proj/src/flops.cpp:29-72 with the opcost formulas of
// proj/include/vqnqs/tensor.hpp:81-102), from K and the realised unique
// counts U[0..L]. Adds into led[7].
void ledger_add(const vqnqs_model_desc& c, int64_t K, const int64_t* U, int64_t* led);

class EngineImpl;
class GradImpl;
class Comm;

// d/dtheta sum_i w_i log P(s_i) on the GPU
// (proj/src/trainer.cpp:213-246 backward through build_log_prob,
// proj/src/model.cpp:570-603, with the VQ surrogate of autodiff.cpp:536-655).
class GradEngine {
 public:
  GradEngine(const vqnqs_model_desc& d, const double* const* params, int n_params, int device);
  ~GradEngine();
  // grads: parameters() order, concatenated (host); lp: log P per sample (host)
  void log_prob_grad(const uint8_t* configs, int64_t B, const double* weights, double vq_tau,
                     double* grads, double* lp);

 private:
  GradImpl* p_;
};

class Engine {
 public:
  Engine(const vqnqs_model_desc& d, const double* const* params, int n_params, int precision,
         int device);
  ~Engine();
  void set_hamiltonian(const int32_t* bonds, int nb, int n_sites, bool marshall);
  // reuse = false: the no-reuse (dense) regime of proj/src/bench.cpp:19-36 —
  // every row active from position 0, every location its own unique row.
  void set_reuse(bool reuse);
  // samples per micro-batch; 0 = sized from the working-set budget
  void set_micro_batch(int samples);
  // Test hook: force the VQ code of every location to the given one
  // (codes [n][L][nb + 1][T] int16 over rows in bond order, -1 = keep the
  // computed code), for the next calls on batches of exactly n samples, so
  // that values after a flagged near-tie can be compared with the
  // reference's; null clears. vq_heads = 1 only.
  void set_code_override(const int16_t* codes, int64_t n);

  struct Taps {
    int32_t* K = nullptr;       // [B]
    int64_t* U = nullptr;       // [B*(L+1)]
    int32_t* codes = nullptr;   // per sample [L][K_s][T]
    int64_t codes_cap = 0;
    double* lp_rows = nullptr;  // per sample [K_s] row log-probs
    int64_t lp_cap = 0;
  };
  // Device-resident batch. d_configs [B x n], outputs device [B]. ledger7
  // host (added to), may be null. taps optional (host buffers).
  void run_device(const uint8_t* d_configs, int64_t B, double* d_e, double* d_logpsi,
                  int64_t* ledger7, void* stream, Taps* taps);
  // estimate_energy / fill_stats over this rank's shard (host configs);
  // with comm the statistics and ledger are global over all ranks.
  // stats = {energy, variance, std_err, k_total}.
  void estimate(const uint8_t* configs, int64_t B, double* e_re, double* logpsi,
                int64_t* ledger7, Comm* comm, double* stats);
  // fill_stats of device-resident local energies d_e[B] (this rank's
  // shard), global over comm's ranks; synchronous on `stream`.
  void fill_stats_device(const double* d_e, int64_t B, Comm* comm, void* stream, double* stats);
  // Host batch (pinned staging inside).
  void run_host(const uint8_t* configs, int64_t B, double* e_re, double* e_im, double* logpsi,
                int64_t* ledger7, Taps* taps);
  // The autoregressive sampler (VqTransformer::sample, proj/src/model.cpp:
  // 485-525) with Rng(seed): configs [count x n] and log-probs [count], host.
  // skip: uniforms of the Rng(seed) stream already consumed (a later batch of
  // the same stream, as measure_flops draws, proj/src/bench.cpp:84-85).
  void sample(int64_t count, uint64_t seed, uint64_t skip, uint8_t* configs, double* log_probs);
  int64_t last_launches() const;
  int last_profile(double* out, int cap) const;
  const vqnqs_model_desc& desc() const;

 private:
  EngineImpl* p_;
};

}  // namespace vqb
