// C ABI (include/vqnqs_b200.h): exception -> status translation around the
// engine. Mirrors how the reference surfaces failures (typed exceptions,
// proj/include/vqnqs/common.hpp:14-28) as integer status codes plus a
// thread-local message.
#include <algorithm>
#include <cstring>
#include <exception>
#include <vector>
#include <string>

#include "comm.h"
#include "engine.h"
#include "vqnqs_b200_debug.h"

struct vqnqs_handle {
  vqb::Engine* eng;
};
struct vqnqs_grad_handle {
  vqb::GradEngine* g;
};
struct vqnqs_comm {
  vqb::Comm* c;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return VQNQS_OK;
  } catch (const vqb::Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return VQNQS_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VQNQS_RUNTIME_ERROR;
  }
}
}  // namespace

extern "C" {

const char* vqnqs_last_error(void) { return g_err.c_str(); }

int vqnqs_param_layout(const vqnqs_model_desc* d, int* n_params, int64_t* numels) {
  return guarded([&] {
    if (!d) throw vqb::UsageError("null model descriptor");
    auto spec = vqb::param_layout(*d);
    if (n_params) *n_params = int(spec.size());
    if (numels)
      for (size_t i = 0; i < spec.size(); ++i) numels[i] = spec[i].rows * spec[i].cols;
  });
}

int vqnqs_init_params(const vqnqs_model_desc* d, uint64_t seed, int snap_bf16,
                      double* const* params) {
  return guarded([&] {
    if (!d || !params) throw vqb::UsageError("null argument");
    vqb::init_params(*d, seed, snap_bf16 != 0, params);
  });
}

int vqnqs_build_lattice(int lx, int ly, int periodic, int32_t* bonds, int cap) {
  int nb = 0;
  int st = guarded([&] {
    auto b = vqb::build_lattice(lx, ly, periodic != 0);
    nb = int(b.size() / 2);
    if (bonds) std::memcpy(bonds, b.data(), sizeof(int32_t) * 2 * size_t(std::min(nb, cap)));
  });
  return st == 0 ? nb : -st;
}

int vqnqs_zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed, uint8_t* out) {
  return guarded([&] {
    if (n < 1 || count < 0 || !out) throw vqb::UsageError("bad sampler arguments");
    vqb::zero_sz_samples(n, start, count, seed, out);
  });
}

int vqnqs_ledger_from_counts(const vqnqs_model_desc* d, int64_t K, const int64_t* U,
                             int64_t* ledger7) {
  return guarded([&] {
    if (!d || !U || !ledger7) throw vqb::UsageError("null argument");
    vqb::validate(*d);
    vqb::ledger_add(*d, K, U, ledger7);
  });
}

int vqnqs_gpu_create(const vqnqs_model_desc* d, const double* const* params, int n_params,
                     int precision, int device, vqnqs_handle** out) {
  return guarded([&] {
    if (!d || !params || !out) throw vqb::UsageError("null argument");
    *out = nullptr;
    auto* h = new vqnqs_handle{nullptr};
    try {
      h->eng = new vqb::Engine(*d, params, n_params, precision, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int vqnqs_gpu_set_hamiltonian(vqnqs_handle* h, const int32_t* bonds, int nb, int n_sites,
                              int marshall) {
  return guarded([&] {
    if (!h) throw vqb::UsageError("null handle");
    h->eng->set_hamiltonian(bonds, nb, n_sites, marshall != 0);
  });
}

int vqnqs_gpu_sample(vqnqs_handle* h, int64_t count, uint64_t seed, uint64_t skip,
                     uint8_t* configs, double* log_probs) {
  return guarded([&] {
    if (!h || !configs || !log_probs) throw vqb::UsageError("null argument");
    h->eng->sample(count, seed, skip, configs, log_probs);
  });
}

int vqnqs_grad_create(const vqnqs_model_desc* d, const double* const* params, int n_params,
                      int device, vqnqs_grad_handle** out) {
  return guarded([&] {
    if (!d || !params || !out) throw vqb::UsageError("null argument");
    auto* h = new vqnqs_grad_handle{nullptr};
    try {
      h->g = new vqb::GradEngine(*d, params, n_params, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int vqnqs_grad_log_prob(vqnqs_grad_handle* h, const uint8_t* configs, int64_t B,
                        const double* weights, double vq_tau, double* grads, double* log_probs) {
  return guarded([&] {
    if (!h || !configs || !weights || !grads || !log_probs) throw vqb::UsageError("null argument");
    h->g->log_prob_grad(configs, B, weights, vq_tau, grads, log_probs);
  });
}

int vqnqs_grad_destroy(vqnqs_grad_handle* h) {
  return guarded([&] {
    if (h) {
      delete h->g;
      delete h;
    }
  });
}

int vqnqs_gpu_set_reuse(vqnqs_handle* h, int reuse) {
  return guarded([&] {
    if (!h) throw vqb::UsageError("null handle");
    h->eng->set_reuse(reuse != 0);
  });
}

int vqnqs_gpu_set_micro_batch(vqnqs_handle* h, int samples) {
  return guarded([&] {
    if (!h) throw vqb::UsageError("null handle");
    if (samples < 0) throw vqb::ConfigError("micro-batch size must be >= 0");
    h->eng->set_micro_batch(samples);
  });
}

int vqnqs_debug_set_code_override(vqnqs_handle* h, const int16_t* codes, int64_t n_samples) {
  return guarded([&] {
    if (!h) throw vqb::UsageError("null handle");
    h->eng->set_code_override(codes, n_samples);
  });
}

int vqnqs_gpu_local_energies(vqnqs_handle* h, const uint8_t* configs, int64_t B, double* e_re,
                             double* e_im, double* logpsi, int64_t* ledger7) {
  return guarded([&] {
    if (!h || (!configs && B > 0) || (!e_re && B > 0)) throw vqb::UsageError("null argument");
    if (B <= 0) return;
    const int n = h->eng->desc().n_sites;
    for (int64_t i = 0; i < B * n; ++i)
      if (configs[i] > 1) throw vqb::ConfigError("configuration entries must be 0 or 1");
    h->eng->run_host(configs, B, e_re, e_im, logpsi, ledger7, nullptr);
  });
}

int vqnqs_gpu_local_energies_device(vqnqs_handle* h, const uint8_t* d_configs, int64_t B,
                                    double* d_e_re, double* d_logpsi, int64_t* ledger7,
                                    void* stream) {
  return guarded([&] {
    if (!h) throw vqb::UsageError("null handle");
    if (B <= 0) return;
    h->eng->run_device(d_configs, B, d_e_re, d_logpsi, ledger7, stream, nullptr);
  });
}

int vqnqs_gpu_connected_log_probs(vqnqs_handle* h, const uint8_t* base, double* lp, int cap) {
  int K = 0;
  int st = guarded([&] {
    if (!h || !base) throw vqb::UsageError("null argument");
    int32_t Kv = 0;
    std::vector<double> rows(static_cast<size_t>(std::max(cap, 1)) + 4096);
    vqb::Engine::Taps t;
    t.K = &Kv;
    t.lp_rows = rows.data();
    t.lp_cap = int64_t(rows.size());
    double e, lpsi;
    h->eng->run_host(base, 1, &e, nullptr, &lpsi, nullptr, &t);
    K = Kv;
    if (lp) std::memcpy(lp, rows.data(), sizeof(double) * size_t(std::min(K, cap)));
  });
  return st == 0 ? K : -st;
}

int vqnqs_gpu_taps(vqnqs_handle* h, const uint8_t* configs, int64_t B, int32_t* K, int64_t* U,
                   int32_t* codes, int64_t codes_cap, double* lp_rows, int64_t lp_cap) {
  return guarded([&] {
    if (!h || !configs) throw vqb::UsageError("null argument");
    vqb::Engine::Taps t;
    t.K = K;
    t.U = U;
    t.codes = codes;
    t.codes_cap = codes_cap;
    t.lp_rows = lp_rows;
    t.lp_cap = lp_cap;
    std::vector<double> e(static_cast<size_t>(B)), lpsi(static_cast<size_t>(B));
    h->eng->run_host(configs, B, e.data(), nullptr, lpsi.data(), nullptr, &t);
  });
}

int vqnqs_comm_unique_id(char* id) {
  return guarded([&] {
    if (!id) throw vqb::UsageError("null argument");
    static_assert(NCCL_UNIQUE_ID_BYTES == VQNQS_COMM_ID_BYTES, "id size");
    vqb::Comm::unique_id(id);
  });
}

int vqnqs_comm_create(const char* id, int world, int rank, int device, vqnqs_comm** out) {
  return guarded([&] {
    if (!id || !out) throw vqb::UsageError("null argument");
    *out = nullptr;
    auto* c = new vqnqs_comm{nullptr};
    try {
      c->c = new vqb::Comm(id, world, rank, device);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int vqnqs_comm_destroy(vqnqs_comm* c) {
  return guarded([&] {
    if (!c) return;
    delete c->c;
    delete c;
  });
}

int vqnqs_gpu_estimate_energy(vqnqs_handle* h, vqnqs_comm* comm, const uint8_t* configs,
                              int64_t B, double* e_re, double* logpsi, int64_t* ledger7,
                              double* stats) {
  return guarded([&] {
    if (!h || !stats || (!configs && B > 0)) throw vqb::UsageError("null argument");
    if (B < 0) throw vqb::ConfigError("negative batch size");
    const int n = h->eng->desc().n_sites;
    for (int64_t i = 0; i < B * n; ++i)
      if (configs[i] > 1) throw vqb::ConfigError("configuration entries must be 0 or 1");
    h->eng->estimate(configs, B, e_re, logpsi, ledger7, comm ? comm->c : nullptr, stats);
  });
}

int vqnqs_gpu_fill_stats_device(vqnqs_handle* h, vqnqs_comm* comm, const double* d_e_re,
                                int64_t B, double* stats, void* stream) {
  return guarded([&] {
    if (!h || !stats || (!d_e_re && B > 0)) throw vqb::UsageError("null argument");
    h->eng->fill_stats_device(d_e_re, B, comm ? comm->c : nullptr, stream, stats);
  });
}

int vqnqs_balanced_shards(const uint8_t* configs, int64_t B, int n_sites, const int32_t* bonds,
                          int nb, int world, int32_t* owner) {
  return guarded([&] {
    if ((!configs && B > 0) || (!bonds && nb > 0) || !owner) throw vqb::UsageError("null argument");
    if (world < 1) throw vqb::ConfigError("world size must be >= 1");
    // K_s = 1 + antiparallel bonds (the connected-set size, proj/src/hamiltonian.cpp:58-72)
    std::vector<std::pair<int, int64_t>> k(static_cast<size_t>(B));
    for (int64_t i = 0; i < B; ++i) {
      int K = 1;
      const uint8_t* c = configs + i * n_sites;
      for (int b = 0; b < nb; ++b) K += c[bonds[2 * b]] != c[bonds[2 * b + 1]];
      k[static_cast<size_t>(i)] = {K, i};
    }
    // longest-processing-time first: decreasing K (ties: batch order) to the
    // rank with the least total so far (ties: lower rank)
    std::stable_sort(k.begin(), k.end(),
                     [](const std::pair<int, int64_t>& a, const std::pair<int, int64_t>& b) {
                       return a.first > b.first;
                     });
    std::vector<int64_t> load(static_cast<size_t>(world), 0);
    for (const auto& e : k) {
      int r = 0;
      for (int q = 1; q < world; ++q)
        if (load[q] < load[r]) r = q;
      load[r] += e.first;
      owner[e.second] = r;
    }
  });
}

int64_t vqnqs_gpu_last_launch_count(vqnqs_handle* h) { return h ? h->eng->last_launches() : -1; }

int vqnqs_gpu_last_profile(vqnqs_handle* h, double* out, int cap) {
  return h ? h->eng->last_profile(out, cap) : -1;
}

int vqnqs_gpu_destroy(vqnqs_handle* h) {
  return guarded([&] {
    if (!h) return;
    delete h->eng;
    delete h;
  });
}

}  // extern "C"
