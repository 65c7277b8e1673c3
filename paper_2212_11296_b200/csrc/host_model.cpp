// Host-side model construction for the engine: parameter layout, seeded
// initialisation, lattices and the zero-Sz sampler. These are the pieces of
// the reference a caller needs to produce the inputs of the hot path; they run
// once per model/batch on the CPU and are not part of the timed step.
//
//   * Rng (mt19937_64 seeded with mix64(seed), hand-rolled uniform/below and
//     Box-Muller, split(stream)) — proj/include/vqnqs/rng.hpp:15-51 and
//     mix64/hash_combine, proj/include/vqnqs/common.hpp:35-45;
//   * VqTransformer::init draw order, proj/src/model.cpp:113-184, and the
//     parameters() order, proj/src/model.cpp:188-229;
//   * build_lattice, proj/src/hamiltonian.cpp:5-35 (+ periodic wrap).
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "engine.h"

namespace vqb {

uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

namespace {

class Rng {
 public:
  explicit Rng(uint64_t seed) : seed_(seed), gen_(mix64(seed)) {}
  uint64_t u64() { return gen_(); }
  double uniform() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return u64() % n; }
  double gaussian() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform(), u2 = uniform();
    while (u1 <= 1e-300) u1 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(t);
    has_spare_ = true;
    return r * std::cos(t);
  }
  Rng split(uint64_t stream) const { return Rng(mix64(seed_ ^ mix64(stream))); }

 private:
  uint64_t seed_;
  std::mt19937_64 gen_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

}  // namespace

double round_bf16_host(double x) {
  float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) {
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&f, &u, 4);
  }
  return static_cast<double>(f);
}

void validate(const vqnqs_model_desc& c) {
  if (c.n_sites < 1) throw ConfigError("n_sites must be positive");
  if (c.group_size < 1 || c.group_size > 16) throw ConfigError("group_size out of range");
  if (c.d_hidden < 1) throw ConfigError("d_hidden must be positive");
  if (c.n_heads < 1 || c.d_hidden % c.n_heads != 0)
    throw ConfigError("d_hidden must divide into n_heads");
  if (c.n_blocks < 0) throw ConfigError("n_blocks must be nonnegative");
  if (c.n_blocks == 0 && !c.trailing_half_block)
    throw ConfigError("model needs at least one block");
  if (c.vq_enabled) {
    if (c.vq_heads < 1 || c.d_hidden % c.vq_heads != 0)
      throw ConfigError("d_hidden must divide into vq_heads");
    if (c.vq_codebook < 1) throw ConfigError("vq_codebook must be positive");
  }
}

// Parameter shapes in parameters() order (proj/src/model.cpp:188-229).
std::vector<ParamSpec> param_layout(const vqnqs_model_desc& c) {
  validate(c);
  std::vector<ParamSpec> out;
  const int64_t d = c.d_hidden, v = int64_t(1) << c.group_size;
  const int64_t T = (c.n_sites + c.group_size - 1) / c.group_size;
  auto add = [&](std::string n, int64_t r, int64_t col, int init, double s) {
    out.push_back({std::move(n), r, col, init, s});
  };
  add("dec.tok_embed", v + 1, d, 2, 0.02);
  add("dec.pos_embed", T, d, 2, 0.02);
  const int nblk = c.n_blocks + (c.trailing_half_block ? 1 : 0);
  for (int b = 0; b < nblk; ++b) {
    const bool half = b == c.n_blocks;
    const std::string p = half ? "dec.half" : "dec.block" + std::to_string(b);
    const bool vq = !half && c.vq_enabled;
    add(p + ".ln1_g", d, 1, 1, 0);
    add(p + ".ln1_b", d, 1, 0, 0);
    for (const char* w : {"q", "k", "v", "o"}) {
      add(p + ".w" + w, d, d, 2, 0.02);
      add(p + ".b" + w, d, 1, 0, 0);
    }
    if (vq) add(p + ".codebook", int64_t(c.vq_heads) * c.vq_codebook, d / c.vq_heads, 3,
                c.vq_init_scale);
    if (!half) {
      add(p + ".ln2_g", d, 1, 1, 0);
      add(p + ".ln2_b", d, 1, 0, 0);
      add(p + ".w1", d, 4 * d, 2, 0.02);
      add(p + ".b1", 4 * d, 1, 0, 0);
      add(p + ".w2", 4 * d, d, 2, 0.02);
      add(p + ".b2", d, 1, 0, 0);
    }
  }
  add("dec.lnf_g", d, 1, 1, 0);
  add("dec.lnf_b", d, 1, 0, 0);
  add("dec.head_w", d, v, 2, 0.02);
  add("dec.head_b", v, 1, 0, 0);
  if (c.phase_enabled) throw CapabilityError("phase network is out of scope for the GPU path");
  return out;
}

// VqTransformer::init draws: tok_embed, pos_embed, then per block
// wq wk wv wo [w1 w2] [codebook], then head_w (model.cpp:113-184).
void init_params(const vqnqs_model_desc& c, uint64_t seed, bool snap, double* const* out) {
  auto spec = param_layout(c);
  for (size_t i = 0; i < spec.size(); ++i) {
    const int64_t n = spec[i].rows * spec[i].cols;
    for (int64_t j = 0; j < n; ++j) out[i][j] = spec[i].init == 1 ? 1.0 : 0.0;
  }
  Rng rng(seed);
  auto draw = [&](const std::string& name, double s) {
    for (size_t i = 0; i < spec.size(); ++i)
      if (spec[i].name == name) {
        const int64_t n = spec[i].rows * spec[i].cols;
        for (int64_t j = 0; j < n; ++j) out[i][j] = s * rng.gaussian();
        return;
      }
  };
  draw("dec.tok_embed", 0.02);
  draw("dec.pos_embed", 0.02);
  const int nblk = c.n_blocks + (c.trailing_half_block ? 1 : 0);
  for (int b = 0; b < nblk; ++b) {
    const bool half = b == c.n_blocks;
    const std::string p = half ? "dec.half" : "dec.block" + std::to_string(b);
    for (const char* w : {".wq", ".wk", ".wv", ".wo"}) draw(p + w, 0.02);
    if (!half) {
      draw(p + ".w1", 0.02);
      draw(p + ".w2", 0.02);
      if (c.vq_enabled) draw(p + ".codebook", c.vq_init_scale);
    }
  }
  draw("dec.head_w", 0.02);
  if (snap)
    for (size_t i = 0; i < spec.size(); ++i) {
      const int64_t n = spec[i].rows * spec[i].cols;
      for (int64_t j = 0; j < n; ++j) out[i][j] = round_bf16_host(out[i][j]);
    }
}

std::vector<int32_t> build_lattice(int lx, int ly, bool periodic) {
  if (lx <= 0 || ly < 0) throw ConfigError("lattice needs positive dimensions");
  const bool grid = ly > 0;
  const int nx = lx, ny = grid ? ly : 1;
  if (periodic && (nx < 3 || (grid && ny < 3)))
    throw ConfigError("periodic lattices need L >= 3");
  std::vector<int32_t> b;
  auto bond = [&](int a, int c) {
    b.push_back(std::min(a, c));
    b.push_back(std::max(a, c));
  };
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      if (x + 1 < nx) bond(y * nx + x, y * nx + x + 1);
      else if (periodic) bond(y * nx + x, y * nx);
    }
  if (grid)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        if (y + 1 < ny) bond(y * nx + x, (y + 1) * nx + x);
        else if (periodic) bond(y * nx + x, x);
      }
  return b;
}

void rng_uniforms(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}

void zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed, uint8_t* out) {
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

}  // namespace vqb
