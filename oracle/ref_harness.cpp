// TEST INFRASTRUCTURE — the reference itself, behind a C ABI for the checkers.
//
// Linked into oracle/_ref/libvqnqs_ref.so together with the UNMODIFIED
// reference sources proj/src/{flops,tensor,hamiltonian,model,dedup}.cpp
// (compiled where they lie under /root/reference by oracle/Makefile) and the
// Eigen shim in oracle/eigen_shim. Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline / --impl reference) load it. Never shipped.
//
// What this file adds around the reference API (nothing here re-implements
// the hot path; everything numeric is the reference's own code):
//   * periodic L x L lattices (horizontals then verticals,
//     row-major, bonds stored (min, max)); the Lattice struct is public and
//     connected_set reads only sites/bonds (proj/src/hamiltonian.cpp:41-74);
//   * the zero-Sz sampler of SURVEY §8d (Rng(seed).split(i), Fisher-Yates);
//   * local_energies restated from proj/src/trainer.cpp:150-180 (trainer.cpp
//     is not linked: it drags in exact.cpp and nlohmann json) — strided
//     std::thread pool, non-finite check, ledger merge in worker order;
//   * a "taps" pass that re-composes dedup_log_prob (proj/src/dedup.cpp:272-323)
//     from the public dedup.hpp functions to expose per-layer unique counts,
//     per-location VQ codes and the top-2 relative distance gap, and checks
//     that its log-probs equal dedup_log_prob's bit for bit;
//   * the checkpoint wire format (proj/src/checkpoint.cpp, linked with the
//     nlohmann json single header found in this image) and the measurement
//     report (measure_flops + emit_table, proj/src/bench.cpp) for the
//     SURVEY §8(f) rank-4 wire formats.
#include <atomic>
#include <cmath>
#include <complex>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include <Eigen/Dense>

#include "vqnqs/autodiff.hpp"
#include "vqnqs/bench.hpp"
#include "vqnqs/checkpoint.hpp"
#include "vqnqs/dedup.hpp"
#include "vqnqs/flops.hpp"
#include "vqnqs/hamiltonian.hpp"
#include "vqnqs/model.hpp"
#include "vqnqs/rng.hpp"

using namespace vqnqs;

extern "C" {

// Same layout as vqnqs_model_desc in include/vqnqs_b200.h.
typedef struct {
  int32_t n_sites, group_size, d_hidden, n_heads, n_blocks;
  int32_t trailing_half_block, vq_enabled, vq_heads, vq_codebook,
      phase_enabled;
  double vq_init_scale;
} ref_model_desc;

}  // extern "C"

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const ShapeError*>(&e)) return 2;
  if (dynamic_cast<const CapabilityError*>(&e)) return 3;
  if (dynamic_cast<const NumericError*>(&e)) return 4;
  if (dynamic_cast<const UsageError*>(&e)) return 5;
  return 6;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

ModelConfig to_cfg(const ref_model_desc& d) {
  ModelConfig c;
  c.n_sites = d.n_sites;
  c.group_size = d.group_size;
  c.d_hidden = d.d_hidden;
  c.n_heads = d.n_heads;
  c.n_blocks = d.n_blocks;
  c.trailing_half_block = d.trailing_half_block != 0;
  c.vq_enabled = d.vq_enabled != 0;
  c.vq_heads = d.vq_heads;
  c.vq_codebook = d.vq_codebook;
  c.phase_enabled = d.phase_enabled != 0;
  c.vq_init_scale = d.vq_init_scale;
  return c;
}

std::vector<SpinConfiguration> unpack(const uint8_t* p, int64_t n, int sites) {
  std::vector<SpinConfiguration> v(static_cast<size_t>(n), SpinConfiguration(static_cast<size_t>(sites)));
  for (int64_t i = 0; i < n; ++i)
    std::memcpy(v[static_cast<size_t>(i)].data(), p + i * sites, static_cast<size_t>(sites));
  return v;
}

void ledger_out(const flops::Ledger& l, int64_t* o) {
  if (!o) return;
  o[0] = l.per_location_dense;
  o[1] = l.per_location_unique;
  o[2] = l.attention;
  o[3] = l.vq_distance;
  o[4] = l.other;
  o[5] = l.per_location_dense_quantized;
  o[6] = l.per_location_unique_quantized;
}

// Same formula as the reference's private op_tag (proj/src/dedup.cpp:17-19);
// only the partition into unique rows matters, never the key values.
uint64_t tag(uint64_t stage, uint64_t block, uint64_t op) {
  return mix64((stage << 32) | (block << 8) | op);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_bf16_products(int on) { Eigen::shim::bf16_products() = on != 0; }

void* ref_model_create(const ref_model_desc* d, uint64_t seed, int snap_bf16) {
  VqTransformer* m = nullptr;
  int st = guarded([&] {
    Rng rng(seed);
    m = new VqTransformer(VqTransformer::init(to_cfg(*d), rng));
    if (snap_bf16)
      for (ad::Parameter* p : m->parameters())
        for (double& x : p->value.data) x = Eigen::shim::round_bf16(x);
  });
  return st == 0 ? m : nullptr;
}

void ref_model_destroy(void* m) { delete static_cast<VqTransformer*>(m); }

int ref_model_num_params(void* m) {
  return int(static_cast<VqTransformer*>(m)->parameters().size());
}

// Returns numel of parameter i (parameters() order, proj/src/model.cpp:210-229)
// and its name; *data points into the model.
int64_t ref_model_param(void* m, int i, double** data, const char** name) {
  auto ps = static_cast<VqTransformer*>(m)->parameters();
  if (i < 0 || i >= int(ps.size())) return -1;
  if (data) *data = ps[static_cast<size_t>(i)]->value.data.data();
  if (name) *name = ps[static_cast<size_t>(i)]->name.c_str();
  return ps[static_cast<size_t>(i)]->value.size();
}

// kind: 0 tfim, 1 heisenberg. lattice: 0 open chain, 1 open grid,
// 2 periodic grid (harness extension), 3 periodic chain (harness extension).
void* ref_ham_create(int kind, int lattice, int lx, int ly, int marshall,
                     double J, double Gamma) {
  HamiltonianModel* h = nullptr;
  int st = guarded([&] {
    h = new HamiltonianModel();
    h->kind = kind == 0 ? HamiltonianModel::Kind::tfim
                        : HamiltonianModel::Kind::heisenberg;
    h->J = J;
    h->Gamma = Gamma;
    h->marshall = marshall != 0;
    if (lattice == 0) {
      h->lattice = build_lattice(Lattice::Kind::chain1d, {lx});
    } else if (lattice == 1) {
      h->lattice = build_lattice(Lattice::Kind::grid2d, {lx, ly});
    } else {
      const bool grid = lattice == 2;
      if (lx < 3 || (grid && ly < 3))
        throw ConfigError("periodic lattices need L >= 3");
      Lattice& lat = h->lattice;
      lat.kind = grid ? Lattice::Kind::grid2d : Lattice::Kind::chain1d;
      lat.dims = grid ? std::vector<int>{lx, ly} : std::vector<int>{lx};
      const int nx = lx, ny = grid ? ly : 1;
      lat.sites = nx * ny;
      auto bond = [&](int a, int b) {
        lat.bonds.emplace_back(std::min(a, b), std::max(a, b));
      };
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) bond(y * nx + x, y * nx + (x + 1) % nx);
      if (grid)
        for (int y = 0; y < ny; ++y)
          for (int x = 0; x < nx; ++x)
            bond(y * nx + x, ((y + 1) % ny) * nx + x);
      lat.sublattice.resize(static_cast<size_t>(lat.sites));
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x)
          lat.sublattice[static_cast<size_t>(y * nx + x)] = uint8_t((x + y) % 2);
    }
  });
  return st == 0 ? h : nullptr;
}

void ref_ham_destroy(void* h) { delete static_cast<HamiltonianModel*>(h); }

int ref_ham_bonds(void* hp, int32_t* out, int cap) {
  auto* h = static_cast<HamiltonianModel*>(hp);
  const int nb = int(h->lattice.bonds.size());
  for (int b = 0; b < nb && b < cap; ++b) {
    out[2 * b] = h->lattice.bonds[static_cast<size_t>(b)].first;
    out[2 * b + 1] = h->lattice.bonds[static_cast<size_t>(b)].second;
  }
  return nb;
}

// connected_set (proj/src/hamiltonian.cpp:41-74). Returns K, or -status.
int ref_connected_set(void* hp, const uint8_t* s, int cap, uint8_t* configs,
                      double* coeffs) {
  auto* h = static_cast<HamiltonianModel*>(hp);
  int K = 0;
  int st = guarded([&] {
    const int n = h->n_sites();
    SpinConfiguration sc(s, s + n);
    ConnectedSet cs = connected_set(*h, sc);
    K = int(cs.entries.size());
    for (int k = 0; k < K && k < cap; ++k) {
      if (configs)
        std::memcpy(configs + int64_t(k) * n, cs.entries[static_cast<size_t>(k)].config.data(),
                    static_cast<size_t>(n));
      if (coeffs) coeffs[k] = cs.entries[static_cast<size_t>(k)].coeff;
    }
  });
  return st == 0 ? K : -st;
}

// Zero-Sz sampler of SURVEY §8d: sample i uses Rng(seed).split(start + i);
// start from N/2 ones then N/2 zeros; Fisher-Yates with below(j+1),
// j = N-1 .. 1 (proj/include/vqnqs/rng.hpp:25,42).
void ref_zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed,
                         uint8_t* out) {
  const Rng master(seed);
  for (int64_t i = 0; i < count; ++i) {
    Rng r = master.split(uint64_t(start + i));
    uint8_t* s = out + i * n;
    for (int j = 0; j < n; ++j) s[j] = j < n / 2 ? 1 : 0;
    for (int j = n - 1; j >= 1; --j) {
      const int t = int(r.below(uint64_t(j) + 1));
      std::swap(s[j], s[t]);
    }
  }
}

// save_checkpoint / load_checkpoint (proj/src/checkpoint.cpp:53-126)
int ref_save_checkpoint(void* mp, const char* path) {
  return guarded([&] { save_checkpoint(*static_cast<VqTransformer*>(mp), path); });
}
void* ref_load_checkpoint(const char* path) {
  VqTransformer* m = nullptr;
  int st = guarded([&] { m = new VqTransformer(load_checkpoint(path)); });
  return st == 0 ? m : nullptr;
}

// measure_flops (proj/src/bench.cpp:65-124) with Rng(seed), then
// emit_table({report}, dir) (:270-290): report.csv / report.json in dir.
int ref_measure_and_emit(void* mp, void* hp, int samples_per_batch, int batches, uint64_t seed,
                         double reference_per_site, const char* dir) {
  return guarded([&] {
    Rng rng(seed);
    auto rep = measure_flops(*static_cast<VqTransformer*>(mp), *static_cast<HamiltonianModel*>(hp),
                             samples_per_batch, batches, rng, reference_per_site);
    emit_table({rep}, dir);
  });
}

// The score-function gradient's backward (proj/src/trainer.cpp:213-246 with
// the sample and its weights given): g = d/dtheta sum_i w_i log P(s_i)
// through build_log_prob (proj/src/model.cpp:570-603) on the reference's own
// tape (proj/src/autodiff.cpp), with its straight-through VQ surrogate.
// grads: every parameter's gradient concatenated in parameters() order;
// lp: the graph's log-probs.
int ref_log_prob_grad(void* mp, const uint8_t* configs, int64_t B, const double* weights,
                      double vq_tau, double* grads, double* lp) {
  auto* m = static_cast<VqTransformer*>(mp);
  return guarded([&] {
    auto batch = unpack(configs, B, m->cfg.n_sites);
    for (auto* p : m->parameters()) p->zero_grad();
    m->cfg.vq_temperature = vq_tau;
    m->cfg.vq_gumbel = false;
    ad::Graph g;
    auto ids = m->build_log_prob(g, batch, nullptr, nullptr);
    const Tensor& lv = g.value(ids);
    for (int64_t i = 0; i < B; ++i) lp[i] = lv.data[size_t(i)];
    auto root = g.weighted_sum(ids, std::vector<double>(weights, weights + B));
    g.backward(root);
    size_t off = 0;
    for (auto* p : m->parameters()) {
      std::copy(p->grad.data.begin(), p->grad.data.end(), grads + off);
      off += p->grad.data.size();
    }
  });
}

// The reference's autoregressive sampler, VqTransformer::sample
// (proj/src/model.cpp:485-525) with Rng(seed): configs [count x n] and the
// recomputed log-probs (log_prob_batch, :398-426).
int ref_sample(void* mp, int count, uint64_t seed, uint8_t* configs, double* log_probs) {
  auto* m = static_cast<VqTransformer*>(mp);
  return guarded([&] {
    Rng rng(seed);
    auto res = m->sample(count, rng);
    const int n = m->cfg.n_sites;
    for (int i = 0; i < count; ++i) {
      std::copy(res.configs[size_t(i)].begin(), res.configs[size_t(i)].end(),
                configs + int64_t(i) * n);
      log_probs[i] = res.log_probs[size_t(i)];
    }
  });
}

// local_energies restated from proj/src/trainer.cpp:150-180 over the
// reference's own local_energy_batch (proj/src/dedup.cpp:394-420).
// logpsi[i] = 0.5 * dedup log-prob of the sample (row 0 of its connected
// set), the quantity log_psi(s) (proj/src/model.cpp:481-483) returns up to
// dense-vs-dedup rounding.
int ref_local_energies(void* mp, void* hp, const uint8_t* configs, int64_t B,
                       int workers, double* e_re, double* e_im, double* logpsi,
                       int64_t* ledger7) {
  auto* m = static_cast<VqTransformer*>(mp);
  auto* h = static_cast<HamiltonianModel*>(hp);
  return guarded([&] {
    const int n = h->n_sites();
    auto batch = unpack(configs, B, n);
    const int W = std::max(1, std::min<int>(workers, int(B)));
    std::vector<flops::Ledger> parts(static_cast<size_t>(W));
    std::vector<std::complex<double>> out(static_cast<size_t>(B));
    std::vector<std::string> errs(static_cast<size_t>(W));
    auto run = [&](int w) {
      try {
        for (int64_t i = w; i < B; i += W) {
          auto r = local_energy_batch(*m, *h, batch[static_cast<size_t>(i)]);
          out[static_cast<size_t>(i)] = r.value;
          parts[static_cast<size_t>(w)] += r.ledger;
          if (logpsi) {
            ConnectedSet cs = connected_set(*h, batch[static_cast<size_t>(i)]);
            // row 0 alone reproduces lp[0] of the full pass only if the
            // per-location math is row-independent, which it is; use the
            // full set anyway so the value is literally the same number.
            std::vector<SpinConfiguration> cf;
            for (auto& e : cs.entries) cf.push_back(e.config);
            logpsi[i] = 0.5 * dedup_log_prob(*m, cf, batch[static_cast<size_t>(i)])[0];
          }
        }
      } catch (const std::exception& e) {
        errs[static_cast<size_t>(w)] = e.what();
      }
    };
    if (W == 1) {
      run(0);
    } else {
      std::vector<std::thread> pool;
      for (int w = 0; w < W; ++w) pool.emplace_back(run, w);
      for (auto& t : pool) t.join();
    }
    for (auto& e : errs)
      if (!e.empty()) throw ShapeError(e);
    for (int64_t i = 0; i < B; ++i) {
      if (!std::isfinite(out[static_cast<size_t>(i)].real()) ||
          !std::isfinite(out[static_cast<size_t>(i)].imag())) {
        std::string s;
        for (uint8_t v : batch[static_cast<size_t>(i)]) s.push_back(v ? '1' : '0');
        throw NumericError("non-finite local energy at configuration " + s);
      }
      e_re[i] = out[static_cast<size_t>(i)].real();
      if (e_im) e_im[i] = out[static_cast<size_t>(i)].imag();
    }
    flops::Ledger tot;
    for (auto& p : parts) tot += p;
    ledger_out(tot, ledger7);
  });
}

// Bare timing loop for the CPU baseline: local_energy_batch only, no taps.
int ref_local_energies_fast(void* mp, void* hp, const uint8_t* configs,
                            int64_t B, int workers, double* e_re) {
  return ref_local_energies(mp, hp, configs, B, workers, e_re, nullptr,
                            nullptr, nullptr);
}

int ref_dedup_log_prob(void* mp, const uint8_t* configs, int64_t K,
                       const uint8_t* base, double* lp) {
  auto* m = static_cast<VqTransformer*>(mp);
  return guarded([&] {
    const int n = m->cfg.n_sites;
    auto cf = unpack(configs, K, n);
    SpinConfiguration b(base, base + n);
    auto v = dedup_log_prob(*m, cf, b);
    std::memcpy(lp, v.data(), sizeof(double) * static_cast<size_t>(K));
  });
}

int ref_dense_log_prob(void* mp, const uint8_t* configs, int64_t K,
                       double* lp) {
  auto* m = static_cast<VqTransformer*>(mp);
  return guarded([&] {
    auto v = m->log_prob_batch(unpack(configs, K, m->cfg.n_sites));
    std::memcpy(lp, v.data(), sizeof(double) * static_cast<size_t>(K));
  });
}

// Taps for one sample s (SURVEY §7 phase 0 step 3). Outputs (caller sizes
// them from K = ref_connected_set(...) and T = seq_len, L = #blocks):
//   U[L+1]            unique rows at the input and after each block
//   codes[L*K*T*H]    VQ picks per (block, location, head); -1 for no-VQ
//   gaps[L*K*T]       min over heads of (d2 - d1) / d1, the relative gap
//                     between the best and second-best squared distance
//   lp[K]             per-row log-probs (bitwise equal to dedup_log_prob)
//   I_final[K*T]      final-stream row index per location
int ref_taps(void* mp, void* hp, const uint8_t* s, int64_t* U, int32_t* codes,
             float* gaps, double* lp, int32_t* I_final) {
  auto* m = static_cast<VqTransformer*>(mp);
  auto* h = static_cast<HamiltonianModel*>(hp);
  return guarded([&] {
    const ModelConfig& cfg = m->cfg;
    if (cfg.phase_enabled) throw CapabilityError("taps: phase not tapped");
    SpinConfiguration base(s, s + h->n_sites());
    ConnectedSet cs = connected_set(*h, base);
    std::vector<SpinConfiguration> configs;
    for (auto& e : cs.entries) configs.push_back(e.config);
    const int64_t K = int64_t(configs.size()), T = cfg.seq_len();
    const int64_t KT = K * T;
    const int64_t d = cfg.d_hidden;

    CompressedBatch x = compress_inputs(*m, configs, base);
    U[0] = x.U();
    for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
      const Block& blk = m->blocks[bi];
      const bool pre_q = m->pre_quantized(int(bi));
      const bool cont_q = m->cont_quantized(int(bi));
      PerLocationOp ln1{LocOp::layer_norm, tag(0, bi, 0), pre_q,
                        [&](const Tensor& t) {
                          return kernels::layer_norm(t, blk.ln1_g.value,
                                                     blk.ln1_b.value, 1e-5);
                        }};
      CompressedBatch hb = apply_per_location(ln1, x);
      auto proj = [&](const ad::Parameter& w, const ad::Parameter& b,
                      uint64_t op) {
        PerLocationOp o{LocOp::linear, tag(0, bi, op), pre_q,
                        [&](const Tensor& t) {
                          return kernels::linear(t, w.value, b.value);
                        }};
        return apply_per_location(o, hb);
      };
      CompressedBatch q = proj(blk.wq, blk.bq, 1);
      CompressedBatch k = proj(blk.wk, blk.bk, 2);
      CompressedBatch v = proj(blk.wv, blk.bv, 3);
      Tensor att = attention_dense(q, k, v, cfg.n_heads, Mask::causal);
      CompressedBatch cat;
      const int H = cfg.vq_heads;
      if (blk.has_vq) {
        // the selection loop of vq_apply_rows (proj/src/model.cpp:292-313),
        // additionally tracking the runner-up distance
        const auto& W = blk.codebook.value;
        const int64_t dh = d / H, Q = W.rows() / H;
        for (int64_t r = 0; r < KT; ++r) {
          float gmin = INFINITY;
          for (int hh = 0; hh < H; ++hh) {
            const double* xr = att.row_ptr(r) + hh * dh;
            int best = 0;
            double b1 = 1e300, b2 = 1e300;
            for (int64_t j = 0; j < Q; ++j) {
              const double* wr = W.row_ptr(hh * Q + j);
              double s2 = 0.0;
              for (int64_t c = 0; c < dh; ++c) {
                const double df = xr[c] - wr[c];
                s2 += df * df;
              }
              if (s2 < b1) {
                b2 = b1;
                b1 = s2;
                best = int(j);
              } else if (s2 < b2) {
                b2 = s2;
              }
            }
            codes[(int64_t(bi) * KT + r) * H + hh] = best;
            const double g = b1 > 0 ? (b2 - b1) / b1 : INFINITY;
            gmin = std::min(gmin, float(g));
          }
          gaps[int64_t(bi) * KT + r] = gmin;
        }
        cat = requantize(att, x, blk.codebook, H, tag(0, bi, 4));
        for (int64_t r = 0; r < KT; ++r)
          for (int hh = 0; hh < H; ++hh) {
            const int c = codes[(int64_t(bi) * KT + r) * H + hh];
            const double* wr = W.row_ptr(hh * (W.rows() / H) + c);
            if (std::memcmp(cat.V.row_ptr(cat.I[static_cast<size_t>(r)]) + hh * (d / H), wr,
                            sizeof(double) * static_cast<size_t>(d / H)) != 0)
              throw NumericError("taps: pick disagrees with requantize");
          }
      } else {
        for (int64_t r = 0; r < KT * H; ++r) codes[int64_t(bi) * KT * H + r] = -1;
        for (int64_t r = 0; r < KT; ++r) gaps[int64_t(bi) * KT + r] = INFINITY;
        cat = densify_attention(att, x, tag(0, bi, 5));
      }
      PerLocationOp cont{
          LocOp::continuation, tag(0, bi, 6), cont_q, [&](const Tensor& t) {
            const int64_t u = t.rows();
            Tensor a({u, d}), r({u, d});
            for (int64_t i = 0; i < u; ++i) {
              std::memcpy(a.row_ptr(i), t.row_ptr(i), sizeof(double) * static_cast<size_t>(d));
              std::memcpy(r.row_ptr(i), t.row_ptr(i) + d,
                          sizeof(double) * static_cast<size_t>(d));
            }
            Tensor o = kernels::linear(a, blk.wo.value, blk.bo.value);
            Tensor y = kernels::add(r, o);
            if (blk.has_ffn) {
              Tensor h2 = kernels::layer_norm(y, blk.ln2_g.value,
                                              blk.ln2_b.value, 1e-5);
              Tensor f = kernels::linear(
                  kernels::gelu(kernels::linear(h2, blk.w1.value, blk.b1.value)),
                  blk.w2.value, blk.b2.value);
              y = kernels::add(y, f);
            }
            return y;
          }};
      x = apply_per_location(cont, cat);
      U[bi + 1] = x.U();
    }
    const bool head_q = m->head_quantized();
    PerLocationOp lnf{LocOp::layer_norm, tag(0, 99, 0), head_q,
                      [&](const Tensor& t) {
                        return kernels::layer_norm(t, m->lnf_g.value,
                                                   m->lnf_b.value, 1e-5);
                      }};
    CompressedBatch hf = apply_per_location(lnf, x);
    PerLocationOp headp{LocOp::linear, tag(0, 99, 1), head_q,
                        [&](const Tensor& t) {
                          return kernels::linear(t, m->head_w.value,
                                                 m->head_b.value);
                        }};
    CompressedBatch logits = apply_per_location(headp, hf);
    if (cfg.last_vocab() < cfg.vocab())
      for (int64_t u = 0; u < logits.U(); ++u)
        if (logits.pos[static_cast<size_t>(u)] == int32_t(T - 1))
          for (int64_t c = cfg.last_vocab(); c < cfg.vocab(); ++c)
            logits.V.at(u, c) = -1e30;
    PerLocationOp lsm{LocOp::output_head, tag(0, 99, 2), head_q,
                      [](const Tensor& t) { return kernels::log_softmax_rows(t); }};
    CompressedBatch lpb = apply_per_location(lsm, logits);
    for (int64_t kk = 0; kk < K; ++kk) {
      const std::vector<int> toks = m->tokenize(configs[static_cast<size_t>(kk)]);
      double acc = 0.0;
      for (int64_t p = 0; p < T; ++p)
        acc += lpb.V.at(lpb.I[static_cast<size_t>(kk * T + p)], toks[static_cast<size_t>(p)]);
      lp[kk] = acc;
    }
    if (I_final)
      for (int64_t l = 0; l < KT; ++l) I_final[l] = lpb.I[static_cast<size_t>(l)];
    auto official = dedup_log_prob(*m, configs, base);
    for (int64_t kk = 0; kk < K; ++kk)
      if (official[static_cast<size_t>(kk)] != lp[kk])
        throw NumericError("taps: re-composed pass differs from dedup_log_prob");
  });
}

}  // extern "C"
