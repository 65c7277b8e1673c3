// vqnqs_b200.hpp — header-only C++ adapter that keeps the reference's
// local-energy signatures while running on the B200 engine (C ABI in
// vqnqs_b200.h). Templated on the reference's own types so this header does
// not depend on them:
//
//   Model  = vqnqs::VqTransformer   (proj/include/vqnqs/model.hpp:99-152)
//   Ham    = vqnqs::HamiltonianModel (proj/include/vqnqs/hamiltonian.hpp:28-37)
//   Config = vqnqs::SpinConfiguration (std::vector<uint8_t>)
//   Ledger = vqnqs::flops::Ledger    (proj/include/vqnqs/flops.hpp:12-44)
//
// Drop-in use:
//   #include "vqnqs/trainer.hpp"
//   #define VQNQS_B200_REFERENCE_ERRORS   // re-throw vqnqs::*Error types
//   #include "vqnqs_b200.hpp"
//   auto e = vqnqs_b200::local_energies(model, h, batch, &ledger);
//
// Semantics follow local_energies (proj/src/trainer.cpp:150-180): one complex
// E_loc per configuration, the ledger ADDED to, a non-finite E_loc reported
// as NumericError naming the configuration.
#pragma once

#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "vqnqs_b200.h"

namespace vqnqs_b200 {

[[noreturn]] inline void throw_status(int st) {
  const std::string msg = vqnqs_last_error();
#ifdef VQNQS_B200_REFERENCE_ERRORS
  switch (st) {
    case VQNQS_CONFIG_ERROR: throw vqnqs::ConfigError(msg);
    case VQNQS_SHAPE_ERROR: throw vqnqs::ShapeError(msg);
    case VQNQS_CAPABILITY_ERROR: throw vqnqs::CapabilityError(msg);
    case VQNQS_NUMERIC_ERROR: throw vqnqs::NumericError(msg);
    case VQNQS_USAGE_ERROR: throw vqnqs::UsageError(msg);
    default: throw std::runtime_error(msg);
  }
#else
  throw std::runtime_error("vqnqs_b200 status " + std::to_string(st) + ": " + msg);
#endif
}

inline void check(int st) {
  if (st != VQNQS_OK) throw_status(st);
}

// One model + Hamiltonian resident on one GPU. Not thread-safe (one per
// device / host thread, like the reference's per-worker evaluation).
template <class Model, class Ham>
class Engine {
 public:
  // fp32 by default: the reference computes in double, and only the fp32
  // engine meets the north-star tolerances on every configuration; bf16 is
  // an explicit opt-in.
  Engine(const Model& m, const Ham& h, int precision = VQNQS_PREC_FP32, int device = 0) {
    vqnqs_model_desc d{};
    d.n_sites = m.cfg.n_sites;
    d.group_size = m.cfg.group_size;
    d.d_hidden = m.cfg.d_hidden;
    d.n_heads = m.cfg.n_heads;
    d.n_blocks = m.cfg.n_blocks;
    d.trailing_half_block = m.cfg.trailing_half_block ? 1 : 0;
    d.vq_enabled = m.cfg.vq_enabled ? 1 : 0;
    d.vq_heads = m.cfg.vq_heads;
    d.vq_codebook = m.cfg.vq_codebook;
    d.phase_enabled = m.cfg.phase_enabled ? 1 : 0;
    d.vq_init_scale = m.cfg.vq_init_scale;
    std::vector<const double*> ptrs;
    for (const auto* p : m.parameters()) ptrs.push_back(p->value.data.data());
    check(vqnqs_gpu_create(&d, ptrs.data(), static_cast<int>(ptrs.size()), precision, device,
                           &h_));
    if (h.kind != Ham::Kind::heisenberg) {
      vqnqs_gpu_destroy(h_);
      h_ = nullptr;
#ifdef VQNQS_B200_REFERENCE_ERRORS
      throw vqnqs::CapabilityError("B200 engine: Heisenberg connected sets only");
#else
      throw std::runtime_error("B200 engine: Heisenberg connected sets only");
#endif
    }
    std::vector<int32_t> bonds;
    for (const auto& b : h.lattice.bonds) {
      bonds.push_back(b.first);
      bonds.push_back(b.second);
    }
    n_ = h.n_sites();
    check(vqnqs_gpu_set_hamiltonian(h_, bonds.data(), static_cast<int>(bonds.size() / 2), n_,
                                    h.marshall ? 1 : 0));
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  ~Engine() {
    if (h_) vqnqs_gpu_destroy(h_);
  }

  template <class Config, class Ledger>
  std::vector<std::complex<double>> local_energies(const std::vector<Config>& batch,
                                                   Ledger* ledger = nullptr) {
    const int64_t B = static_cast<int64_t>(batch.size());
    std::vector<uint8_t> flat(static_cast<size_t>(B) * n_);
    for (int64_t i = 0; i < B; ++i) {
      if (static_cast<int>(batch[i].size()) != n_) throw_size();
      for (int j = 0; j < n_; ++j) flat[static_cast<size_t>(i) * n_ + j] = batch[i][j];
    }
    std::vector<double> re(B), im(B);
    int64_t led[VQNQS_LEDGER_SLOTS] = {0, 0, 0, 0, 0, 0, 0};
    check(vqnqs_gpu_local_energies(h_, flat.data(), B, re.data(), im.data(), nullptr, led));
    if (ledger) {
      ledger->per_location_dense += led[VQNQS_LEDGER_PER_LOCATION_DENSE];
      ledger->per_location_unique += led[VQNQS_LEDGER_PER_LOCATION_UNIQUE];
      ledger->attention += led[VQNQS_LEDGER_ATTENTION];
      ledger->vq_distance += led[VQNQS_LEDGER_VQ_DISTANCE];
      ledger->other += led[VQNQS_LEDGER_OTHER];
      ledger->per_location_dense_quantized += led[VQNQS_LEDGER_PER_LOCATION_DENSE_QUANTIZED];
      ledger->per_location_unique_quantized += led[VQNQS_LEDGER_PER_LOCATION_UNIQUE_QUANTIZED];
    }
    std::vector<std::complex<double>> out(B);
    for (int64_t i = 0; i < B; ++i) out[i] = {re[i], im[i]};
    return out;
  }

  // dedup_log_prob over the connected set of `base` (diagonal row first, then
  // bond order), proj/include/vqnqs/dedup.hpp:77-79.
  template <class Config>
  std::vector<double> connected_log_probs(const Config& base) {
    std::vector<double> lp(static_cast<size_t>(4 * n_ + 8));
    const int K = vqnqs_gpu_connected_log_probs(h_, base.data(), lp.data(),
                                                static_cast<int>(lp.size()));
    if (K < 0) throw_status(-K);
    lp.resize(static_cast<size_t>(K));
    return lp;
  }

 private:
  [[noreturn]] static void throw_size() {
#ifdef VQNQS_B200_REFERENCE_ERRORS
    throw vqnqs::ShapeError("configuration size != site count");
#else
    throw std::runtime_error("configuration size != site count");
#endif
  }
  vqnqs_handle* h_ = nullptr;
  int n_ = 0;
};

// Content fingerprint of what an Engine snapshots: every parameter value,
// the bonds and the Marshall flag (64-bit mix over the raw bits).
template <class Model, class Ham>
inline uint64_t fingerprint(const Model& m, const Ham& h) {
  uint64_t x = 0x9E3779B97F4A7C15ull;
  auto mix = [&x](uint64_t v) {
    x ^= v + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
  };
  for (const auto* p : m.parameters())
    for (double v : p->value.data) {
      uint64_t u;
      std::memcpy(&u, &v, sizeof u);
      mix(u);
    }
  for (const auto& b : h.lattice.bonds) mix((uint64_t(uint32_t(b.first)) << 32) | uint32_t(b.second));
  mix(h.marshall ? 1 : 2);
  return x;
}

// Drop-in for vqnqs::local_energies(model, h, batch, ledger)
// (proj/include/vqnqs/trainer.hpp:76-79). Keeps one engine per thread for the
// last (model, Hamiltonian, precision, device) seen. The cache is keyed on the
// CONTENT of model and Hamiltonian, so parameters updated in place between
// calls (a VMC loop) are re-uploaded, never silently stale; hashing the
// weights costs one pass over them per call — hold an Engine directly to
// avoid it.
template <class Model, class Ham>
struct EngineCache {
  const Model* m = nullptr;
  const Ham* h = nullptr;
  uint64_t fp = 0;
  int precision = -1, device = -1;
  std::unique_ptr<Engine<Model, Ham>> eng;
};

template <class Model, class Ham>
inline EngineCache<Model, Ham>& engine_cache() {
  thread_local EngineCache<Model, Ham> c;
  return c;
}

template <class Model, class Ham>
inline void reset_cache() {
  engine_cache<Model, Ham>().eng.reset();
  engine_cache<Model, Ham>().m = nullptr;
}

template <class Model, class Ham, class Config, class Ledger>
std::vector<std::complex<double>> local_energies(const Model& model, const Ham& h,
                                                 const std::vector<Config>& batch,
                                                 Ledger* ledger = nullptr,
                                                 int precision = VQNQS_PREC_FP32,
                                                 int device = 0) {
  auto& c = engine_cache<Model, Ham>();
  const uint64_t fp = fingerprint(model, h);
  if (!c.eng || c.m != &model || c.h != &h || c.fp != fp || c.precision != precision ||
      c.device != device) {
    c.eng.reset();
    c.eng = std::make_unique<Engine<Model, Ham>>(model, h, precision, device);
    c.m = &model;
    c.h = &h;
    c.fp = fp;
    c.precision = precision;
    c.device = device;
  }
  return c.eng->local_energies(batch, ledger);
}

}  // namespace vqnqs_b200
