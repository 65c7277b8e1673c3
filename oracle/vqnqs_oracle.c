/* TEST INFRASTRUCTURE — plain-C restatement ("port") of the reference's
 * local-energy path. Parity checker only: tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline leg load it; the product never does.
 *
 * Every function cites the reference code it restates (paths relative to
 * /root/reference). The floating-point operation order follows the reference
 * (with Eigen products evaluated as the eager k-ascending loop of
 * oracle/eigen_shim), so in double mode this port reproduces the reference
 * bit for bit; tests/test_oracle_port.py pins that against oracle/_ref and
 * the committed golden vectors.
 *
 * bf16 emulation (hard part 1): when enabled, both operands of
 * every product — linear layers (tensor.cpp:43-55), attention scores and the
 * probability-value mix (tensor.cpp:206-207,224) — are rounded
 * double -> fp32 (RNE) -> bf16 (RNE) before multiplying; sums stay in double.
 * This mirrors exactly where the GPU path rounds its fp32 values to bf16.
 *
 * Row keys are EXACT tuples — (position, input token) at the input layer and
 * (residual row, VQ code tuple) after each quantizer — the collision-free
 * equivalent of the reference's 64-bit hash chains (dedup.cpp:61-63,156-159;
 * SURVEY §8a). Unique rows are numbered in first-occurrence order, like the
 * reference's unordered_map emplace loop.
 */
#define _GNU_SOURCE
#include "vqnqs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <setjmp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static _Thread_local char g_err[512];
static _Thread_local jmp_buf* g_jmp;

static void fail(int status, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  longjmp(*g_jmp, status);
}

#define GUARD_BEGIN          \
  jmp_buf jb__;              \
  jmp_buf* prev__ = g_jmp;   \
  int st__ = setjmp(jb__);   \
  if (st__ != 0) {           \
    g_jmp = prev__;          \
    return st__;             \
  }                          \
  g_jmp = &jb__;
#define GUARD_END \
  g_jmp = prev__; \
  return 0;

const char* orc_last_error(void) { return g_err; }

static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s);
  if (!p) fail(6, "out of memory");
  return p;
}

/* ----------------------------------------------- hashing / RNG (common.hpp) */

/* splitmix64 finalizer, proj/include/vqnqs/common.hpp:35-40 */
static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 (the engine inside vqnqs::Rng, proj/include/vqnqs/rng.hpp:15-51) */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int mti;
  uint64_t seed;
  int has_spare;
  double spare;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed) {
  r->seed = seed;
  r->has_spare = 0;
  r->spare = 0.0;
  uint64_t s = mix64(seed); /* Rng(seed) : gen_(mix64(seed)), rng.hpp:20 */
  r->mt[0] = s;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->mti = MT_N;
}

static uint64_t rng_u64(rng_t* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL,
                        A = 0xB5026F5AA96619E9ULL;
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= A;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:25 */
static double rng_uniform(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:28 */
static uint64_t rng_below(rng_t* r, uint64_t n) { return rng_u64(r) % n; }
/* Box-Muller with cached pair, rng.hpp:31-43 */
static double rng_gaussian(rng_t* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = rng_uniform(r), u2 = rng_uniform(r);
  while (u1 <= 1e-300) u1 = rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double t = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(t);
  r->has_spare = 1;
  return rr * cos(t);
}
/* rng.hpp:45 */
static void rng_split(const rng_t* r, uint64_t stream, rng_t* out) {
  rng_init(out, mix64(r->seed ^ mix64(stream)));
}

/* ------------------------------------------------------------ bf16 product */

static int g_bf16 = 0;
void orc_set_bf16_products(int on) { g_bf16 = on != 0; }

static double round_bf16(double x) {
  float f = (float)x;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f;
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* --------------------------------------------------------------- model */

typedef struct {
  double *ln1_g, *ln1_b, *wq, *bq, *wk, *bk, *wv, *bv, *wo, *bo, *cb;
  double *ln2_g, *ln2_b, *w1, *b1, *w2, *b2;
  int has_ffn, has_vq;
} blk_t;

typedef struct {
  char name[48];
  double* data;
  int64_t rows, cols;
} param_t;

typedef struct {
  orc_model_desc c;
  int T, vocab, last_vocab, nblk;
  param_t p[512];
  int np;
  blk_t* blk;
  double *tok_embed, *pos_embed, *lnf_g, *lnf_b, *head_w, *head_b;
} model_t;

static double* add_param(model_t* m, const char* name, int64_t r, int64_t c,
                         int kind /*0 zeros 1 ones 2 randn*/, rng_t* rng,
                         double scale) {
  if (m->np >= 512) fail(1, "too many parameters");
  param_t* p = &m->p[m->np++];
  snprintf(p->name, sizeof p->name, "%s", name);
  p->rows = r;
  p->cols = c;
  p->data = xcalloc((size_t)(r * c), sizeof(double));
  for (int64_t i = 0; i < r * c; ++i)
    p->data[i] = kind == 1 ? 1.0 : kind == 2 ? scale * rng_gaussian(rng) : 0.0;
  return p->data;
}

/* ModelConfig::validate, proj/src/model.cpp:10-27 */
static void validate(const orc_model_desc* c) {
  if (c->n_sites < 1) fail(1, "n_sites must be positive");
  if (c->group_size < 1 || c->group_size > 16) fail(1, "group_size out of range");
  if (c->d_hidden < 1) fail(1, "d_hidden must be positive");
  if (c->n_heads < 1 || c->d_hidden % c->n_heads != 0)
    fail(1, "d_hidden must divide into n_heads");
  if (c->n_blocks < 0) fail(1, "n_blocks must be nonnegative");
  if (c->n_blocks == 0 && !c->trailing_half_block)
    fail(1, "model needs at least one block");
  if (c->vq_enabled) {
    if (c->vq_heads < 1 || c->d_hidden % c->vq_heads != 0)
      fail(1, "d_hidden must divide into vq_heads");
    if (c->vq_codebook < 1) fail(1, "vq_codebook must be positive");
  }
}

/* make_block, proj/src/model.cpp:113-146: draw order wq wk wv wo [w1 w2] [codebook];
 * parameter order collect_block, model.cpp:188-208. We register parameters in
 * parameters() order but draw in init order, so draws happen into the final
 * buffers afterwards. */
static void make_block(model_t* m, const char* prefix, int has_ffn, int has_vq,
                       rng_t* rng, blk_t* b) {
  const int64_t d = m->c.d_hidden;
  char nm[48];
#define NM(s) (snprintf(nm, sizeof nm, "%s.%s", prefix, s), nm)
  b->has_ffn = has_ffn;
  b->has_vq = has_vq;
  b->ln1_g = add_param(m, NM("ln1_g"), d, 1, 1, NULL, 0);
  b->ln1_b = add_param(m, NM("ln1_b"), d, 1, 0, NULL, 0);
  b->wq = add_param(m, NM("wq"), d, d, 0, NULL, 0);
  b->bq = add_param(m, NM("bq"), d, 1, 0, NULL, 0);
  b->wk = add_param(m, NM("wk"), d, d, 0, NULL, 0);
  b->bk = add_param(m, NM("bk"), d, 1, 0, NULL, 0);
  b->wv = add_param(m, NM("wv"), d, d, 0, NULL, 0);
  b->bv = add_param(m, NM("bv"), d, 1, 0, NULL, 0);
  b->wo = add_param(m, NM("wo"), d, d, 0, NULL, 0);
  b->bo = add_param(m, NM("bo"), d, 1, 0, NULL, 0);
  const int64_t dh = has_vq ? d / m->c.vq_heads : 0;
  const int64_t hq = has_vq ? (int64_t)m->c.vq_heads * m->c.vq_codebook : 0;
  b->cb = has_vq ? add_param(m, NM("codebook"), hq, dh, 0, NULL, 0) : NULL;
  if (has_ffn) {
    b->ln2_g = add_param(m, NM("ln2_g"), d, 1, 1, NULL, 0);
    b->ln2_b = add_param(m, NM("ln2_b"), d, 1, 0, NULL, 0);
    b->w1 = add_param(m, NM("w1"), d, 4 * d, 0, NULL, 0);
    b->b1 = add_param(m, NM("b1"), 4 * d, 1, 0, NULL, 0);
    b->w2 = add_param(m, NM("w2"), 4 * d, d, 0, NULL, 0);
    b->b2 = add_param(m, NM("b2"), d, 1, 0, NULL, 0);
  }
#undef NM
  const double s = 0.02;
  double* draw[] = {b->wq, b->wk, b->wv, b->wo};
  for (int i = 0; i < 4; ++i)
    for (int64_t j = 0; j < d * d; ++j) draw[i][j] = s * rng_gaussian(rng);
  if (has_ffn) {
    for (int64_t j = 0; j < 4 * d * d; ++j) b->w1[j] = s * rng_gaussian(rng);
    for (int64_t j = 0; j < 4 * d * d; ++j) b->w2[j] = s * rng_gaussian(rng);
  }
  if (has_vq)
    for (int64_t j = 0; j < hq * dh; ++j)
      b->cb[j] = m->c.vq_init_scale * rng_gaussian(rng);
}

static void model_free(model_t* m) {
  if (!m) return;
  for (int i = 0; i < m->np; ++i) free(m->p[i].data);
  free(m->blk);
  free(m);
}

/* VqTransformer::init, proj/src/model.cpp:150-184 */
void* orc_model_create(const orc_model_desc* d, uint64_t seed, int snap_bf16) {
  model_t* volatile m = NULL;
  jmp_buf jb;
  jmp_buf* prev = g_jmp;
  if (setjmp(jb) != 0) {
    g_jmp = prev;
    model_free(m);
    return NULL;
  }
  g_jmp = &jb;
  validate(d);
  if (d->phase_enabled) fail(3, "oracle port: phase network not restated (out of scope)");
  m = xcalloc(1, sizeof(model_t));
  m->c = *d;
  m->T = (d->n_sites + d->group_size - 1) / d->group_size;
  m->vocab = 1 << d->group_size;
  const int rem = d->n_sites % d->group_size;
  m->last_vocab = rem == 0 ? m->vocab : 1 << rem;
  m->nblk = d->n_blocks + (d->trailing_half_block ? 1 : 0);
  m->blk = xcalloc((size_t)m->nblk, sizeof(blk_t));
  rng_t rng;
  rng_init(&rng, seed);
  const int64_t dd = d->d_hidden, v = m->vocab;
  m->tok_embed = add_param(m, "dec.tok_embed", v + 1, dd, 2, &rng, 0.02);
  m->pos_embed = add_param(m, "dec.pos_embed", m->T, dd, 2, &rng, 0.02);
  for (int b = 0; b < d->n_blocks; ++b) {
    char pre[32];
    snprintf(pre, sizeof pre, "dec.block%d", b);
    make_block(m, pre, 1, d->vq_enabled, &rng, &m->blk[b]);
  }
  if (d->trailing_half_block) make_block(m, "dec.half", 0, 0, &rng, &m->blk[d->n_blocks]);
  m->lnf_g = add_param(m, "dec.lnf_g", dd, 1, 1, NULL, 0);
  m->lnf_b = add_param(m, "dec.lnf_b", dd, 1, 0, NULL, 0);
  m->head_w = add_param(m, "dec.head_w", dd, v, 2, &rng, 0.02);
  m->head_b = add_param(m, "dec.head_b", v, 1, 0, NULL, 0);
  if (snap_bf16)
    for (int i = 0; i < m->np; ++i)
      for (int64_t j = 0; j < m->p[i].rows * m->p[i].cols; ++j)
        m->p[i].data[j] = round_bf16(m->p[i].data[j]);
  g_jmp = prev;
  return m;
}

void orc_model_destroy(void* m) { model_free(m); }
int orc_model_num_params(void* m) { return ((model_t*)m)->np; }
int64_t orc_model_param(void* mp, int i, double** data, const char** name) {
  model_t* m = mp;
  if (i < 0 || i >= m->np) return -1;
  if (data) *data = m->p[i].data;
  if (name) *name = m->p[i].name;
  return m->p[i].rows * m->p[i].cols;
}

/* --------------------------------------------------------- hamiltonian */

typedef struct {
  int kind; /* 0 tfim, 1 heisenberg */
  int n;
  int nb;
  int32_t* bonds;
  double J, Gamma;
  int marshall;
} ham_t;

/* build_lattice (proj/src/hamiltonian.cpp:5-35) plus the periodic extension
 * of SURVEY §8d (horizontals then verticals, row-major, (min,max)). */
void* orc_ham_create(int kind, int lattice, int lx, int ly, int marshall, double J,
                     double Gamma) {
  if (lx <= 0 || (lattice == 1 && ly <= 0) || (lattice == 2 && ly <= 0)) {
    snprintf(g_err, sizeof g_err, "lattice needs positive dimensions");
    return NULL;
  }
  if ((lattice == 2 || lattice == 3) && (lx < 3 || (lattice == 2 && ly < 3))) {
    snprintf(g_err, sizeof g_err, "periodic lattices need L >= 3");
    return NULL;
  }
  ham_t* h = calloc(1, sizeof(ham_t));
  h->kind = kind;
  h->J = J;
  h->Gamma = Gamma;
  h->marshall = marshall;
  const int grid = lattice == 1 || lattice == 2;
  const int nx = lx, ny = grid ? ly : 1;
  h->n = nx * ny;
  h->bonds = calloc((size_t)(4 * h->n + 2), sizeof(int32_t));
  int nb = 0;
#define BOND(a, b)                                 \
  do {                                             \
    int a_ = (a), b_ = (b);                        \
    h->bonds[2 * nb] = a_ < b_ ? a_ : b_;          \
    h->bonds[2 * nb + 1] = a_ < b_ ? b_ : a_;      \
    ++nb;                                          \
  } while (0)
  if (lattice == 0 || lattice == 1) {
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x + 1 < nx; ++x) BOND(y * nx + x, y * nx + x + 1);
    if (grid)
      for (int y = 0; y + 1 < ny; ++y)
        for (int x = 0; x < nx; ++x) BOND(y * nx + x, (y + 1) * nx + x);
  } else {
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) BOND(y * nx + x, y * nx + (x + 1) % nx);
    if (grid)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) BOND(y * nx + x, ((y + 1) % ny) * nx + x);
  }
#undef BOND
  h->nb = nb;
  return h;
}

void orc_ham_destroy(void* hp) {
  ham_t* h = hp;
  if (!h) return;
  free(h->bonds);
  free(h);
}

int orc_ham_bonds(void* hp, int32_t* out, int cap) {
  ham_t* h = hp;
  for (int b = 0; b < h->nb && b < cap; ++b) {
    out[2 * b] = h->bonds[2 * b];
    out[2 * b + 1] = h->bonds[2 * b + 1];
  }
  return h->nb;
}

/* connected_set, proj/src/hamiltonian.cpp:41-74. Writes up to `cap` rows;
 * returns K. */
static int connected(const ham_t* h, const uint8_t* s, int cap, uint8_t* cf, double* co) {
  const int n = h->n;
  int K = 0;
#define ZV(v) (2 * (int)(v)-1)
  if (h->kind == 0) {
    double diag = 0.0;
    for (int b = 0; b < h->nb; ++b)
      diag += (double)(ZV(s[h->bonds[2 * b]]) * ZV(s[h->bonds[2 * b + 1]]));
    if (K < cap) {
      if (cf) memcpy(cf, s, (size_t)n);
      if (co) co[0] = -h->J * diag;
    }
    ++K;
    for (int i = 0; i < n; ++i, ++K)
      if (K < cap) {
        if (cf) {
          memcpy(cf + (size_t)K * n, s, (size_t)n);
          cf[(size_t)K * n + i] = (uint8_t)(1 - s[i]);
        }
        if (co) co[K] = -h->Gamma;
      }
  } else {
    double diag = 0.0;
    const double off = h->marshall ? -0.5 : 0.5;
    if (K < cap && cf) memcpy(cf, s, (size_t)n);
    ++K;
    for (int b = 0; b < h->nb; ++b) {
      const int i = h->bonds[2 * b], j = h->bonds[2 * b + 1];
      diag += 0.25 * (double)(ZV(s[i]) * ZV(s[j]));
      if (s[i] != s[j]) {
        if (K < cap) {
          if (cf) {
            memcpy(cf + (size_t)K * n, s, (size_t)n);
            cf[(size_t)K * n + i] = (uint8_t)(1 - s[i]);
            cf[(size_t)K * n + j] = (uint8_t)(1 - s[j]);
          }
          if (co) co[K] = off;
        }
        ++K;
      }
    }
    if (cap > 0 && co) co[0] = diag;
  }
#undef ZV
  return K;
}

int orc_connected_set(void* hp, const uint8_t* s, int cap, uint8_t* cf, double* co) {
  return connected(hp, s, cap, cf, co);
}

/* Zero-Sz sampler of SURVEY §8d (same definition as ref_zero_sz_samples). */
void orc_zero_sz_samples(int n, int64_t start, int64_t count, uint64_t seed,
                         uint8_t* out) {
  rng_t master, r;
  rng_init(&master, seed);
  for (int64_t i = 0; i < count; ++i) {
    rng_split(&master, (uint64_t)(start + i), &r);
    uint8_t* s = out + i * n;
    for (int j = 0; j < n; ++j) s[j] = j < n / 2 ? 1 : 0;
    for (int j = n - 1; j >= 1; --j) {
      const int t = (int)rng_below(&r, (uint64_t)j + 1);
      uint8_t tmp = s[j];
      s[j] = s[t];
      s[t] = tmp;
    }
  }
}

/* ------------------------------------------------------------- kernels */

typedef struct {
  int64_t pl_dense, pl_unique, att, vq, other, pl_dense_q, pl_unique_q;
} ledger_t;

/* kernels::linear, proj/src/tensor.cpp:43-55 (Eigen product = k-ascending
 * double loop, then the bias row). x:[m x n] with row stride ldx. */
static void linear(const double* x, int64_t ldx, int64_t m, int64_t n,
                   const double* w, const double* b, int64_t p, double* y) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < p; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        double xv = x[i * ldx + k], wv = w[k * p + j];
        if (g_bf16) {
          xv = round_bf16(xv);
          wv = round_bf16(wv);
        }
        s += xv * wv;
      }
      y[i * p + j] = s;
    }
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < p; ++j) y[i * p + j] += b[j];
}

/* kernels::layer_norm, proj/src/tensor.cpp:57-83 */
static void layer_norm(const double* x, int64_t m, int64_t n, const double* g,
                       const double* bta, double* y) {
  for (int64_t r = 0; r < m; ++r) {
    const double* xr = x + r * n;
    double mean = 0.0;
    for (int64_t c = 0; c < n; ++c) mean += xr[c];
    mean /= (double)n;
    double var = 0.0;
    for (int64_t c = 0; c < n; ++c) {
      const double dd = xr[c] - mean;
      var += dd * dd;
    }
    var /= (double)n;
    const double rstd = 1.0 / sqrt(var + 1e-5);
    for (int64_t c = 0; c < n; ++c) y[r * n + c] = (xr[c] - mean) * rstd * g[c] + bta[c];
  }
}

/* kernels::gelu (tanh form), proj/src/tensor.cpp:126-139 */
static double gelu(double v) {
  const double c = 0.7978845608028654;
  const double u = c * (v + 0.044715 * v * v * v);
  return 0.5 * v * (1.0 + tanh(u));
}

/* kernels::log_softmax_rows, proj/src/tensor.cpp:107-124 */
static void log_softmax(double* x, int64_t m, int64_t n) {
  for (int64_t r = 0; r < m; ++r) {
    double* xr = x + r * n;
    double mx = xr[0];
    for (int64_t c = 1; c < n; ++c) mx = mx > xr[c] ? mx : xr[c];
    double sum = 0.0;
    for (int64_t c = 0; c < n; ++c) sum += exp(xr[c] - mx);
    const double lse = mx + log(sum);
    for (int64_t c = 0; c < n; ++c) xr[c] = xr[c] - lse;
  }
}

/* masked_attention for one (sequence, head), proj/src/tensor.cpp:199-231,
 * reading q/k/v rows through the location->row index I (the expand() of
 * dedup.cpp:31-37 without materialising it). */
static void attention_head(const double* q, const double* k, const double* v,
                           int64_t ld, const int32_t* I, int64_t T, int64_t dh,
                           int64_t off, double* S, double* out, int64_t ldo) {
  const double scale = 1.0 / sqrt((double)dh);
  for (int64_t r = 0; r < T; ++r)
    for (int64_t c = 0; c < T; ++c) {
      double s = 0.0;
      const double* qr = q + (int64_t)I[r] * ld + off;
      const double* kc = k + (int64_t)I[c] * ld + off;
      for (int64_t e = 0; e < dh; ++e) {
        double a = qr[e], b = kc[e];
        if (g_bf16) {
          a = round_bf16(a);
          b = round_bf16(b);
        }
        s += a * b;
      }
      S[r * T + c] = s;
    }
  for (int64_t i = 0; i < T * T; ++i) S[i] *= scale;
  for (int64_t r = 0; r < T; ++r)
    for (int64_t c = r + 1; c < T; ++c) S[r * T + c] = -1e30;
  for (int64_t r = 0; r < T; ++r) {
    double* sr = S + r * T;
    double mx = sr[0];
    for (int64_t c = 1; c < T; ++c) mx = mx > sr[c] ? mx : sr[c];
    double sum = 0.0;
    for (int64_t c = 0; c < T; ++c) {
      sr[c] = exp(sr[c] - mx);
      sum += sr[c];
    }
    for (int64_t c = 0; c < T; ++c) sr[c] /= sum;
  }
  for (int64_t r = 0; r < T; ++r)
    for (int64_t e = 0; e < dh; ++e) {
      double s = 0.0;
      for (int64_t c = 0; c < T; ++c) {
        double a = S[r * T + c], b = v[(int64_t)I[c] * ld + off + e];
        if (g_bf16) {
          a = round_bf16(a);
          b = round_bf16(b);
        }
        s += a * b;
      }
      out[r * ldo + off + e] = s;
    }
}

/* ------------------------------------------------------- exact-key dedup */

typedef struct {
  int64_t cap;
  int64_t* slot; /* representative location, -1 empty */
  int32_t* uid;
} table_t;

static void table_init(table_t* t, int64_t n) {
  int64_t cap = 16;
  while (cap < 2 * n + 2) cap <<= 1;
  t->cap = cap;
  t->slot = xcalloc((size_t)cap, sizeof(int64_t));
  t->uid = xcalloc((size_t)cap, sizeof(int32_t));
  for (int64_t i = 0; i < cap; ++i) t->slot[i] = -1;
}
static void table_free(table_t* t) {
  free(t->slot);
  free(t->uid);
}

/* ------------------------------------------------------ compressed forward */

typedef struct {
  int64_t K, T, U, w;
  int32_t* I;   /* K*T */
  double* V;    /* U x w */
  int32_t* pos; /* U */
} stream_t;

static void stream_free(stream_t* s) {
  free(s->I);
  free(s->V);
  free(s->pos);
  memset(s, 0, sizeof *s);
}

typedef struct {
  int64_t* U;      /* [L+1] or NULL */
  int32_t* codes;  /* [L*KT*H] or NULL */
  float* gaps;     /* [L*KT] or NULL */
  int32_t* I_final;
  double* rows;    /* [KT*V] per-location log-softmax rows, or NULL */
} taps_t;

/* tokenize, proj/src/model.cpp:236-248 (little-endian groups) */
static void tokenize(const model_t* m, const uint8_t* s, int* toks) {
  const int g = m->c.group_size;
  for (int p = 0; p < m->T; ++p) toks[p] = 0;
  for (int i = 0; i < m->c.n_sites; ++i) toks[i / g] += (int)s[i] << (i % g);
}

static int64_t per_loc(ledger_t* L, int64_t logical, int64_t actual, int64_t cost,
                       int quant) {
  /* PerLocationScope, proj/src/flops.cpp:29-53 */
  L->pl_unique += cost;
  if (quant) L->pl_unique_q += cost;
  const int64_t dense = (actual > 0 && cost % actual == 0) ? cost / actual * logical : cost;
  L->pl_dense += dense;
  if (quant) L->pl_dense_q += dense;
  return cost;
}

/* dedup_log_prob (proj/src/dedup.cpp:272-323) over one connected set, with
 * compress_inputs (:39-91), run_block (:217-268), requantize (:136-185),
 * densify_attention (:187-211). dense != 0 evaluates the same network with
 * no merging at all, i.e. VqTransformer::log_prob_batch's dense path
 * (proj/src/model.cpp:325-426). */
static void forward(const model_t* m, const uint8_t* configs, int64_t K,
                    const uint8_t* base, int dense, double* lp, ledger_t* led,
                    taps_t* taps) {
  const int64_t T = m->T, KT = K * T, d = m->c.d_hidden, n = m->c.n_sites;
  const int bos = m->vocab;
  const int H = m->c.vq_heads;
  int* toks = xcalloc((size_t)KT, sizeof(int));
  for (int64_t k = 0; k < K; ++k) {
    if (base && !dense) {
      int diff = 0;
      for (int64_t i = 0; i < n; ++i) diff += configs[k * n + i] != base[i];
      if (diff > 2) {
        free(toks);
        fail(5, "connected configuration differs in more than 2 sites");
      }
    }
    tokenize(m, configs + k * n, toks + k * T);
  }
  /* ---- input layer ---- */
  stream_t x = {K, T, 0, d, xcalloc((size_t)KT, 4), NULL, NULL};
  int32_t* row_tok = xcalloc((size_t)KT, 4);
  x.pos = xcalloc((size_t)KT, 4);
  {
    table_t tb;
    table_init(&tb, KT);
    int64_t* rep = xcalloc((size_t)KT, 8);
    for (int64_t k = 0; k < K; ++k)
      for (int64_t p = 0; p < T; ++p) {
        const int64_t l = k * T + p;
        const int tok = p == 0 ? bos : toks[k * T + p - 1];
        if (dense) {
          x.I[l] = (int32_t)x.U;
          x.pos[x.U] = (int32_t)p;
          row_tok[x.U++] = tok;
          continue;
        }
        uint64_t hsh = mix64(((uint64_t)p << 32) ^ (uint64_t)tok);
        int64_t s = (int64_t)(hsh & (uint64_t)(tb.cap - 1));
        for (;;) {
          if (tb.slot[s] < 0) {
            tb.slot[s] = l;
            tb.uid[s] = (int32_t)x.U;
            x.pos[x.U] = (int32_t)p;
            row_tok[x.U] = tok;
            rep[x.U++] = l;
            break;
          }
          const int64_t r = tb.slot[s];
          if (x.pos[tb.uid[s]] == p && row_tok[tb.uid[s]] == tok) break;
          (void)r;
          s = (s + 1) & (tb.cap - 1);
        }
        x.I[l] = tb.uid[s];
      }
    free(rep);
    table_free(&tb);
  }
  x.V = xcalloc((size_t)(x.U * d), sizeof(double));
  for (int64_t u = 0; u < x.U; ++u)
    for (int64_t c = 0; c < d; ++c)
      x.V[u * d + c] = m->tok_embed[row_tok[u] * d + c] + m->pos_embed[x.pos[u] * d + c];
  per_loc(led, KT, x.U, x.U * d, 0);
  if (taps && taps->U) taps->U[0] = x.U;
  free(row_tok);

  double* S = xcalloc((size_t)(T * T), sizeof(double));
  int seen_vq = 0;
  for (int b = 0; b < m->nblk; ++b) {
    const blk_t* B = &m->blk[b];
    const int pre_q = m->c.vq_enabled && seen_vq;
    const int cont_q = m->c.vq_enabled && (seen_vq || B->has_vq);
    const int64_t U = x.U;
    double* h = xcalloc((size_t)(U * d), 8);
    double *q = xcalloc((size_t)(U * d), 8), *kk = xcalloc((size_t)(U * d), 8),
           *v = xcalloc((size_t)(U * d), 8);
    layer_norm(x.V, U, d, B->ln1_g, B->ln1_b, h);
    per_loc(led, KT, U, U * (7 * d + 5), pre_q);
    linear(h, d, U, d, B->wq, B->bq, d, q);
    per_loc(led, KT, U, 2 * U * d * d + U * d, pre_q);
    linear(h, d, U, d, B->wk, B->bk, d, kk);
    per_loc(led, KT, U, 2 * U * d * d + U * d, pre_q);
    linear(h, d, U, d, B->wv, B->bv, d, v);
    per_loc(led, KT, U, 2 * U * d * d + U * d, pre_q);
    free(h);
    /* attention_dense over all K*T locations (always dense) */
    double* att = xcalloc((size_t)(KT * d), 8);
    const int64_t nh = m->c.n_heads, dh = d / nh;
    for (int64_t k = 0; k < K; ++k)
      for (int64_t hh = 0; hh < nh; ++hh)
        attention_head(q, kk, v, d, x.I + k * T, T, dh, hh * dh, S, att + k * T * d, d);
    led->att += K * nh * (4 * T * T * dh + 6 * T * T);
    free(q);
    free(kk);
    free(v);
    /* ---- requantize / densify ---- */
    stream_t y = {K, T, 0, 2 * d, xcalloc((size_t)KT, 4), NULL, xcalloc((size_t)KT, 4)};
    int64_t* rep = xcalloc((size_t)KT, 8);
    if (B->has_vq) {
      /* vq_apply_rows, proj/src/model.cpp:283-319: ties to the lowest index */
      const int64_t vdh = d / H, Q = m->c.vq_codebook;
      int32_t* picks = xcalloc((size_t)(KT * H), 4);
      for (int64_t r = 0; r < KT; ++r) {
        float gmin = INFINITY;
        for (int hh = 0; hh < H; ++hh) {
          const double* xr = att + r * d + hh * vdh;
          int best = 0;
          double b1 = 1e300, b2 = 1e300;
          for (int64_t j = 0; j < Q; ++j) {
            const double* wr = B->cb + (hh * Q + j) * vdh;
            double s2 = 0.0;
            for (int64_t c = 0; c < vdh; ++c) {
              const double df = xr[c] - wr[c];
              s2 += df * df;
            }
            if (s2 < b1) {
              b2 = b1;
              b1 = s2;
              best = (int)j;
            } else if (s2 < b2) {
              b2 = s2;
            }
          }
          picks[r * H + hh] = best;
          const double gg = b1 > 0 ? (b2 - b1) / b1 : INFINITY;
          if ((float)gg < gmin) gmin = (float)gg;
        }
        if (taps && taps->gaps) taps->gaps[(int64_t)b * KT + r] = gmin;
      }
      if (taps && taps->codes) memcpy(taps->codes + (int64_t)b * KT * H, picks, (size_t)(KT * H) * 4);
      led->vq += KT * (int64_t)H * (Q * (3 * vdh + 2) + Q);
      table_t tb;
      table_init(&tb, KT);
      for (int64_t l = 0; l < KT; ++l) {
        if (dense) {
          rep[y.U] = l;
          y.pos[y.U] = x.pos[x.I[l]];
          y.I[l] = (int32_t)y.U++;
          continue;
        }
        uint64_t hsh = mix64((uint64_t)x.I[l]);
        for (int hh = 0; hh < H; ++hh) hsh = mix64(hsh ^ (uint64_t)picks[l * H + hh]);
        int64_t s = (int64_t)(hsh & (uint64_t)(tb.cap - 1));
        for (;;) {
          if (tb.slot[s] < 0) {
            tb.slot[s] = l;
            tb.uid[s] = (int32_t)y.U;
            rep[y.U] = l;
            y.pos[y.U++] = x.pos[x.I[l]];
            break;
          }
          const int64_t r = tb.slot[s];
          int same = x.I[r] == x.I[l];
          for (int hh = 0; same && hh < H; ++hh) same = picks[r * H + hh] == picks[l * H + hh];
          if (same) break;
          s = (s + 1) & (tb.cap - 1);
        }
        y.I[l] = tb.uid[s];
      }
      table_free(&tb);
      y.V = xcalloc((size_t)(y.U * 2 * d), 8);
      for (int64_t u = 0; u < y.U; ++u) {
        const int64_t l = rep[u];
        for (int hh = 0; hh < H; ++hh)
          memcpy(y.V + u * 2 * d + hh * vdh, B->cb + (hh * Q + picks[l * H + hh]) * vdh,
                 (size_t)vdh * 8);
        memcpy(y.V + u * 2 * d + d, x.V + (int64_t)x.I[l] * d, (size_t)d * 8);
      }
      free(picks);
      seen_vq = 1;
    } else {
      if (taps && taps->codes)
        for (int64_t r = 0; r < KT * H; ++r) taps->codes[(int64_t)b * KT * H + r] = -1;
      if (taps && taps->gaps)
        for (int64_t r = 0; r < KT; ++r) taps->gaps[(int64_t)b * KT + r] = INFINITY;
      y.V = xcalloc((size_t)(KT * 2 * d), 8);
      for (int64_t l = 0; l < KT; ++l) {
        y.I[l] = (int32_t)l;
        y.pos[l] = x.pos[x.I[l]];
        memcpy(y.V + l * 2 * d, att + l * d, (size_t)d * 8);
        memcpy(y.V + l * 2 * d + d, x.V + (int64_t)x.I[l] * d, (size_t)d * 8);
      }
      y.U = KT;
    }
    free(rep);
    free(att);
    /* ---- continuation, dedup.cpp:246-267 ---- */
    const int64_t U2 = y.U;
    double* o = xcalloc((size_t)(U2 * d), 8);
    double* xn = xcalloc((size_t)(U2 * d), 8);
    int64_t cost = 0;
    linear(y.V, 2 * d, U2, d, B->wo, B->bo, d, o);
    cost += 2 * U2 * d * d + U2 * d;
    for (int64_t u = 0; u < U2; ++u)
      for (int64_t c = 0; c < d; ++c) xn[u * d + c] = y.V[u * 2 * d + d + c] + o[u * d + c];
    cost += U2 * d;
    if (B->has_ffn) {
      double* h2 = xcalloc((size_t)(U2 * d), 8);
      double* f1 = xcalloc((size_t)(U2 * 4 * d), 8);
      layer_norm(xn, U2, d, B->ln2_g, B->ln2_b, h2);
      cost += U2 * (7 * d + 5);
      linear(h2, d, U2, d, B->w1, B->b1, 4 * d, f1);
      cost += 2 * U2 * d * 4 * d + U2 * 4 * d;
      for (int64_t i = 0; i < U2 * 4 * d; ++i) f1[i] = gelu(f1[i]);
      cost += 10 * U2 * 4 * d;
      linear(f1, 4 * d, U2, 4 * d, B->w2, B->b2, d, h2);
      cost += 2 * U2 * 4 * d * d + U2 * d;
      for (int64_t i = 0; i < U2 * d; ++i) xn[i] = xn[i] + h2[i];
      cost += U2 * d;
      free(h2);
      free(f1);
    }
    per_loc(led, KT, U2, cost, cont_q);
    free(o);
    stream_free(&x);
    x.K = K;
    x.T = T;
    x.U = U2;
    x.w = d;
    x.I = y.I;
    x.pos = y.pos;
    x.V = xn;
    free(y.V);
    if (taps && taps->U) taps->U[b + 1] = U2;
  }
  free(S);
  /* ---- head, dedup.cpp:280-308 ---- */
  const int head_q = m->c.vq_enabled && seen_vq;
  const int64_t U = x.U, V = m->vocab;
  double* hf = xcalloc((size_t)(U * d), 8);
  double* lg = xcalloc((size_t)(U * V), 8);
  layer_norm(x.V, U, d, m->lnf_g, m->lnf_b, hf);
  per_loc(led, KT, U, U * (7 * d + 5), head_q);
  linear(hf, d, U, d, m->head_w, m->head_b, V, lg);
  per_loc(led, KT, U, 2 * U * d * V + U * V, head_q);
  if (m->last_vocab < m->vocab)
    for (int64_t u = 0; u < U; ++u)
      if (x.pos[u] == T - 1)
        for (int64_t c = m->last_vocab; c < V; ++c) lg[u * V + c] = -1e30;
  log_softmax(lg, U, V);
  per_loc(led, KT, U, U * (5 * V + 1), head_q);
  /* gather-sum, dedup.cpp:310-321 */
  led->other += KT;
  for (int64_t k = 0; k < K; ++k) {
    double s = 0.0;
    for (int64_t p = 0; p < T; ++p) s += lg[(int64_t)x.I[k * T + p] * V + toks[k * T + p]];
    lp[k] = s;
  }
  if (taps && taps->I_final) memcpy(taps->I_final, x.I, (size_t)KT * 4);
  if (taps && taps->rows)
    for (int64_t l = 0; l < KT; ++l)
      memcpy(taps->rows + l * V, lg + (int64_t)x.I[l] * V, (size_t)V * 8);
  free(hf);
  free(lg);
  free(toks);
  stream_free(&x);
}

/* -------------------------------------------------------- entry points */

int orc_dedup_log_prob(void* mp, const uint8_t* configs, int64_t K,
                       const uint8_t* base, double* lp) {
  GUARD_BEGIN
  ledger_t led = {0};
  if (K < 1) fail(2, "empty connected set");
  forward(mp, configs, K, base, 0, lp, &led, NULL);
  GUARD_END
}

int orc_dense_log_prob(void* mp, const uint8_t* configs, int64_t K, double* lp) {
  GUARD_BEGIN
  ledger_t led = {0};
  forward(mp, configs, K, NULL, 1, lp, &led, NULL);
  GUARD_END
}

/* VqTransformer::sample, proj/src/model.cpp:485-525: T ancestral steps with
 * Rng(seed); step t reads position t's log-softmax row of the decoder on the
 * sampled prefix (the dense forward of the partially filled configurations:
 * position t depends on tokens < t only, and masked keys add exact zeros),
 * and draws by inverse CDF in sample order (:503-518). log_probs are the
 * dense log-probs of the finished configurations (log_prob_batch, :398-426). */
int orc_sample(void* mp, int count, uint64_t seed, uint8_t* configs, double* log_probs) {
  GUARD_BEGIN
  const model_t* m = mp;
  if (count < 1) fail(1, "sample count must be >= 1");
  const int64_t T = m->T, n = m->c.n_sites, V = m->vocab, g = m->c.group_size;
  rng_t rng;
  rng_init(&rng, seed);
  int* tok = xcalloc((size_t)(count * T), sizeof(int));
  double* rows = xcalloc((size_t)(count * T * V), 8);
  double* lp = xcalloc((size_t)count, 8);
  for (int64_t step = 0; step < T; ++step) {
    for (int64_t i = 0; i < count; ++i)
      for (int64_t j = 0; j < n; ++j) {
        const int64_t p = j / g;
        configs[i * n + j] = p < step ? (uint8_t)((tok[i * T + p] >> (j % g)) & 1) : 0;
      }
    ledger_t led = {0};
    taps_t tp = {0};
    tp.rows = rows;
    forward(m, configs, count, NULL, 1, lp, &led, &tp);
    for (int64_t i = 0; i < count; ++i) {
      const double* row = rows + (i * T + step) * V;
      const double u = rng_uniform(&rng);
      double cum = 0.0;
      int picked = -1, last_pos = 0;
      for (int c = 0; c < m->vocab; ++c) {
        const double pr = exp(row[c]);
        if (pr > 0) last_pos = c;
        cum += pr;
        if (u < cum) {
          picked = c;
          break;
        }
      }
      if (picked < 0) picked = last_pos; /* guard against rounding */
      tok[i * T + step] = picked;
    }
  }
  for (int64_t i = 0; i < count; ++i)
    for (int64_t j = 0; j < n; ++j)
      configs[i * n + j] = (uint8_t)((tok[i * T + j / g] >> (j % g)) & 1);
  {
    ledger_t led = {0};
    forward(m, configs, count, NULL, 1, log_probs, &led, NULL);
  }
  free(tok);
  free(rows);
  free(lp);
  GUARD_END
}

/* local_energy_batch, proj/src/dedup.cpp:394-420 (phase off) */
static double local_energy(const model_t* m, const ham_t* h, const uint8_t* s,
                           double* logpsi, ledger_t* led) {
  const int n = h->n;
  const int K = connected(h, s, 0, NULL, NULL);
  uint8_t* cf = xcalloc((size_t)K * n, 1);
  double* co = xcalloc((size_t)K, 8);
  double* lp = xcalloc((size_t)K, 8);
  connected(h, s, K, cf, co);
  forward(m, cf, K, s, 0, lp, led, NULL);
  double e = 0.0;
  for (int k = 0; k < K; ++k) {
    const double dlp = 0.5 * (lp[k] - lp[0]);
    e += co[k] * exp(dlp);
  }
  if (logpsi) *logpsi = 0.5 * lp[0];
  free(cf);
  free(co);
  free(lp);
  return e;
}

typedef struct {
  const model_t* m;
  const ham_t* h;
  const uint8_t* configs;
  int64_t B;
  int W, w;
  double *e_re, *logpsi;
  ledger_t led;
  int status;
  char err[512];
} job_t;

static void* worker(void* arg) {
  job_t* j = arg;
  jmp_buf jb;
  g_jmp = &jb;
  int st = setjmp(jb);
  if (st != 0) {
    j->status = st;
    snprintf(j->err, sizeof j->err, "%s", g_err);
    return NULL;
  }
  for (int64_t i = j->w; i < j->B; i += j->W)
    j->e_re[i] = local_energy(j->m, j->h, j->configs + i * j->h->n,
                              j->logpsi ? j->logpsi + i : NULL, &j->led);
  return NULL;
}

/* local_energies, proj/src/trainer.cpp:150-180: strided pool, ledgers merged
 * in worker order, non-finite -> NumericError naming the configuration. */
int orc_local_energies(void* mp, void* hp, const uint8_t* configs, int64_t B,
                       int workers, double* e_re, double* e_im, double* logpsi,
                       int64_t* ledger7) {
  const ham_t* h = hp;
  const model_t* m = mp;
  if (h->n != m->c.n_sites) {
    snprintf(g_err, sizeof g_err, "configuration size != site count");
    return 2;
  }
  if (h->kind != 1 && h->kind != 0) return 3;
  int W = workers < 1 ? 1 : workers;
  if (W > B) W = (int)(B > 0 ? B : 1);
  job_t* jobs = calloc((size_t)W, sizeof(job_t));
  pthread_t* th = calloc((size_t)W, sizeof(pthread_t));
  for (int w = 0; w < W; ++w) {
    jobs[w] = (job_t){m, h, configs, B, W, w, e_re, logpsi, {0}, 0, {0}};
    if (W == 1)
      worker(&jobs[w]);
    else
      pthread_create(&th[w], NULL, worker, &jobs[w]);
  }
  if (W > 1)
    for (int w = 0; w < W; ++w) pthread_join(th[w], NULL);
  int st = 0;
  ledger_t tot = {0};
  for (int w = 0; w < W; ++w) {
    if (jobs[w].status && !st) {
      st = jobs[w].status;
      snprintf(g_err, sizeof g_err, "%s", jobs[w].err);
    }
    tot.pl_dense += jobs[w].led.pl_dense;
    tot.pl_unique += jobs[w].led.pl_unique;
    tot.att += jobs[w].led.att;
    tot.vq += jobs[w].led.vq;
    tot.other += jobs[w].led.other;
    tot.pl_dense_q += jobs[w].led.pl_dense_q;
    tot.pl_unique_q += jobs[w].led.pl_unique_q;
  }
  free(jobs);
  free(th);
  if (st) return st;
  for (int64_t i = 0; i < B; ++i) {
    if (!isfinite(e_re[i])) {
      char s[300];
      int n = h->n < 256 ? h->n : 256;
      for (int j = 0; j < n; ++j) s[j] = configs[i * h->n + j] ? '1' : '0';
      s[n] = 0;
      snprintf(g_err, sizeof g_err, "non-finite local energy at configuration %s", s);
      return 4;
    }
    if (e_im) e_im[i] = 0.0;
  }
  if (ledger7) {
    ledger7[0] = tot.pl_dense;
    ledger7[1] = tot.pl_unique;
    ledger7[2] = tot.att;
    ledger7[3] = tot.vq;
    ledger7[4] = tot.other;
    ledger7[5] = tot.pl_dense_q;
    ledger7[6] = tot.pl_unique_q;
  }
  return 0;
}

int orc_local_energies_fast(void* m, void* h, const uint8_t* configs, int64_t B,
                            int workers, double* e_re) {
  return orc_local_energies(m, h, configs, B, workers, e_re, NULL, NULL, NULL);
}

int orc_taps(void* mp, void* hp, const uint8_t* s, int64_t* U, int32_t* codes,
             float* gaps, double* lp, int32_t* I_final) {
  GUARD_BEGIN
  const ham_t* h = hp;
  const int n = h->n;
  const int K = connected(h, s, 0, NULL, NULL);
  uint8_t* cf = xcalloc((size_t)K * n, 1);
  connected(h, s, K, cf, NULL);
  ledger_t led = {0};
  taps_t t = {U, codes, gaps, I_final};
  forward(mp, cf, K, s, 0, lp, &led, &t);
  free(cf);
  GUARD_END
}
