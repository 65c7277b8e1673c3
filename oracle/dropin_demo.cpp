// TEST INFRASTRUCTURE — the drop-in boundary exercised from the reference's
// own C++ types. Builds a vqnqs::VqTransformer and vqnqs::HamiltonianModel
// with the reference's code (oracle/_ref objects), evaluates a batch with
// the reference's local_energy_batch, then calls vqnqs_b200::local_energies
// (include/vqnqs_b200.hpp) with the very same objects and compares.
//
//   dropin_demo L d heads blocks Q batch precision(0 fp32 | 1 bf16)
// exit 0: parity ok; 1: mismatch; 3: no usable GPU (engine refused loudly).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vqnqs/dedup.hpp"
#include "vqnqs/flops.hpp"
#include "vqnqs/hamiltonian.hpp"
#include "vqnqs/model.hpp"
#include "vqnqs/rng.hpp"

#define VQNQS_B200_REFERENCE_ERRORS
#include "vqnqs_b200.hpp"

using namespace vqnqs;

int main(int argc, char** argv) {
  const int L = argc > 1 ? std::atoi(argv[1]) : 4;
  const int d = argc > 2 ? std::atoi(argv[2]) : 32;
  const int heads = argc > 3 ? std::atoi(argv[3]) : 4;
  const int blocks = argc > 4 ? std::atoi(argv[4]) : 2;
  const int Q = argc > 5 ? std::atoi(argv[5]) : 64;
  const int B = argc > 6 ? std::atoi(argv[6]) : 32;
  const int prec = argc > 7 ? std::atoi(argv[7]) : 0;
  ModelConfig cfg;
  cfg.n_sites = L * L;
  cfg.group_size = 2;
  cfg.d_hidden = d;
  cfg.n_heads = heads;
  cfg.n_blocks = blocks;
  cfg.trailing_half_block = false;
  cfg.vq_heads = 1;
  cfg.vq_codebook = Q;
  cfg.vq_init_scale = 1.0 / d;
  Rng rng(0);
  VqTransformer model = VqTransformer::init(cfg, rng);
  HamiltonianModel h;
  h.kind = HamiltonianModel::Kind::heisenberg;
  h.lattice.kind = Lattice::Kind::grid2d;
  h.lattice.dims = {L, L};
  h.lattice.sites = L * L;
  for (int y = 0; y < L; ++y)
    for (int x = 0; x < L; ++x) {
      const int a = y * L + x, b = y * L + (x + 1) % L;
      h.lattice.bonds.emplace_back(std::min(a, b), std::max(a, b));
    }
  for (int y = 0; y < L; ++y)
    for (int x = 0; x < L; ++x) {
      const int a = y * L + x, b = ((y + 1) % L) * L + x;
      h.lattice.bonds.emplace_back(std::min(a, b), std::max(a, b));
    }
  h.lattice.sublattice.resize(L * L);
  std::vector<SpinConfiguration> batch;
  const Rng master(1);
  for (int i = 0; i < B; ++i) {
    Rng r = master.split(uint64_t(i));
    SpinConfiguration s(L * L);
    for (int j = 0; j < L * L; ++j) s[j] = j < L * L / 2 ? 1 : 0;
    for (int j = L * L - 1; j >= 1; --j) std::swap(s[j], s[r.below(uint64_t(j) + 1)]);
    batch.push_back(s);
  }
  // the reference
  std::vector<double> e_ref(B);
  flops::Ledger led_ref;
  for (int i = 0; i < B; ++i) {
    auto r = local_energy_batch(model, h, batch[i]);
    e_ref[i] = r.value.real();
    led_ref += r.ledger;
  }
  // the drop-in, same objects
  flops::Ledger led;
  std::vector<std::complex<double>> e;
  try {
    e = vqnqs_b200::local_energies(model, h, batch, &led, prec, 0);
  } catch (const std::exception& ex) {
    std::printf("NO_GPU: %s\n", ex.what());
    return 3;
  }
  double worst = 0;
  for (int i = 0; i < B; ++i)
    worst = std::max(worst, std::abs(e[i].real() - e_ref[i]) / std::max(1e-12, std::abs(e_ref[i])));
  const bool ledger_eq = led.total_dense() == led_ref.total_dense() &&
                         led.attention == led_ref.attention && led.vq_distance == led_ref.vq_distance;
  std::printf("{\"max_rel_dE\": %.3e, \"ledger_dense_equal\": %d, \"savings\": %.4f}\n", worst,
              int(ledger_eq), double(led.total_dense()) / double(led.total_dedup()));
  return (worst < 1e-4 && ledger_eq) ? 0 : 1;
}
