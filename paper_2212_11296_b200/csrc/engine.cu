// Host orchestration of the local-energy pipeline on one B200.
//
// One call = one batch of B sample configurations, processed in micro-batches
// ("chunks") of at most S samples. Per chunk:
//   (a) k_connected / k_scan / k_enumerate   connected sets, active locations
//   (d) k_dedup<0> + k_embed                 unique input rows
//   per block b:
//   (b) LN1 -> QKV GEMM on U_b unique rows   k_layernorm, gemm
//   (b) gathered causal attention            attention over active locations
//   (c) nearest codeword                     vq
//   (d) requantize dedup + gather build      k_dedup<1>, k_build_gather
//   (b) continuation GEMM chain on U_{b+1}   gemm(Wo)+resid, LN2, gemm(W1)+gelu, gemm(W2)+resid
//   (e) LN_f + head + log_softmax, E_loc     k_layernorm, k_head, k_eloc
// The only host synchronisation per chunk is one 16-byte readback of the
// chunk's active-location/table totals (to size the arena) and the final
// U-count readback for the ledger.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "engine.h"
#include "pipeline_kernels.cuh"
#include "simt_kernels.cuh"
#include "tc_attention.cuh"
#include "tc_kernels.cuh"
#include "sampler_kernels.cuh"

namespace vqb {

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                         __FILE__ + ":" + std::to_string(__LINE__));                   \
  } while (0)

namespace {

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void ensure(size_t want) {
    if (want <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t alloc = std::max<size_t>(want + want / 4, 64);
    cudaError_t e = cudaMalloc(&p, alloc * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw RuntimeError(std::string("device allocation failed: ") + cudaGetErrorString(e));
    }
    n = alloc;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct DevBlock {
  bool has_vq, has_ffn;  // full blocks carry both (VQ when vq_enabled); the half block neither
  float *ln1_g, *ln1_b, *bqkv, *bo, *ln2_g, *ln2_b, *b1, *b2, *cb32, *wn2;
  float* pwo;  // per-code continuation table [Q x d]: code_j Wo + bo
  float wmax, werr;
  CUtensorMap tmB;                       // codebook tensor map (tcgen05 VQ)
  void *wqkv, *wo, *w1, *w2, *cbA;       // [in x out] row-major, operand type
  void *wqkvT, *woT, *w1T, *w2T;         // [out x in] (K-major) copies for tcgen05
};

}  // namespace

void ledger_add(const vqnqs_model_desc& c, int64_t K, const int64_t* U, int64_t* led) {
  // proj/src/flops.cpp:29-72 with opcost (tensor.hpp:81-102); the dense
  // shadow scales each per-location segment's exact per-row cost to K*T.
  const int64_t T = (c.n_sites + c.group_size - 1) / c.group_size, KT = K * T;
  const int64_t d = c.d_hidden, V = int64_t(1) << c.group_size;
  auto per_loc = [&](int64_t u, int64_t cost, bool q) {
    led[1] += cost;
    if (q) led[6] += cost;
    const int64_t dense = (u > 0 && cost % u == 0) ? cost / u * KT : cost;
    led[0] += dense;
    if (q) led[5] += dense;
  };
  per_loc(U[0], U[0] * d, false);
  const int nblk = c.n_blocks + (c.trailing_half_block ? 1 : 0);
  bool seen_vq = false;
  for (int b = 0; b < nblk; ++b) {
    const bool half = b == c.n_blocks;
    const bool has_vq = !half && c.vq_enabled;
    const bool pre_q = c.vq_enabled && seen_vq, cont_q = c.vq_enabled && (seen_vq || has_vq);
    const int64_t u = U[b], u2 = U[b + 1];
    per_loc(u, u * (7 * d + 5), pre_q);
    for (int i = 0; i < 3; ++i) per_loc(u, 2 * u * d * d + u * d, pre_q);
    const int64_t nh = c.n_heads, dh = d / nh;
    led[2] += K * nh * (4 * T * T * dh + 6 * T * T);
    if (has_vq) {
      const int64_t H = c.vq_heads, vdh = d / H, Q = c.vq_codebook;
      led[3] += KT * H * (Q * (3 * vdh + 2) + Q);
    }
    int64_t cost = 2 * u2 * d * d + u2 * d + u2 * d;
    if (!half)
      cost += u2 * (7 * d + 5) + 2 * u2 * d * 4 * d + u2 * 4 * d + 10 * u2 * 4 * d +
              2 * u2 * 4 * d * d + u2 * d + u2 * d;
    per_loc(u2, cost, cont_q);
    seen_vq = seen_vq || has_vq;
  }
  const int64_t uL = U[nblk];
  const bool head_q = c.vq_enabled && seen_vq;
  per_loc(uL, uL * (7 * d + 5), head_q);
  per_loc(uL, 2 * uL * d * V + uL * V, head_q);
  per_loc(uL, uL * (5 * V + 1), head_q);
  led[4] += KT;
}

class EngineImpl {
 public:
  vqnqs_model_desc c{};
  int prec = VQNQS_PREC_FP32;
  int dev = 0;
  int sms = 148;
  cudaStream_t own = nullptr;
  int d, nh, dh, Q, H, L, V, T, g, N, lastV;
  int qbits = 1;            // bits per VQ code in the packed tuple key
  bool tuple_pass = false;  // H codes exceed 32 bits: number tuples first
  bool use_tc_gemm = false;  // tcgen05 per-location GEMMs (bf16)
  bool use_tc_vq = false;    // tcgen05 certified-argmin VQ (both precisions)
  bool use_tc_attn = false;  // tcgen05 gathered attention (bf16)
  int attn_cap = 256;        // score columns a tile may need (the attention kernel's TMEM budget)
  unsigned long long* d_rescored = nullptr;
  std::vector<void*> allocs;
  float *tok_embed, *pos_embed, *lnf_g, *lnf_b, *head_b;
  float* zeros_d = nullptr;  // [d] zeros
  void* head_w;
  std::vector<DevBlock> blk;
  // hamiltonian
  int nb = 0;
  bool marshall = true;
  int32_t* d_bonds = nullptr;
  std::vector<int32_t> h_bonds;
  // launch accounting / profile
  int64_t launches = 0;
  double prof[12] = {0};
  // arena
  int S_max = 256;
  DBuf<int32_t> row_perm_;
  DBuf<int32_t> K_, Mact_, row_bond_, row_t1_, tok0_, lrow_, Ucnt_, I_a, I_b, code_, slot_,
      rep_of_, trep_, tuid_, g_code_;
  DBuf<int16_t> lpos_, upos_;
  DBuf<int64_t> row_aoff_, act_off_, tab_off_, Uoff_, tot_, g_res_, attw_;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> lev;  // per-layer stage events, read once per chunk
  DBuf<double> diag_, lpV_, lp_rows_;
  DBuf<unsigned long long> tkey_, ctup_;
  DBuf<int32_t> ckey_;  // packed / numbered VQ code tuples (H > 1)
  DBuf<float> x_a, x_b, y_, att_, xn2_, rr2_;
  DBuf<bf16> att_hi_, att_lo_;
  DBuf<char> h_, qkv_, f1_;
  DBuf<uint8_t> cfg_stage_;
  DBuf<AttnTile> tiles_;
  DBuf<uint8_t> tinfo_;
  VqScratch vqs_;  // deferred VQ re-scoring queue
  DBuf<int32_t> ntiles_;
  DBuf<int32_t> tcnt_;  // attention tiles per sample
  DBuf<int64_t> toff_;  // their exclusive scan, [S] = total
  DBuf<double> out_stage_;
  DBuf<int32_t> taps_codes_;
  size_t tab_cap_n = 0;
  uint8_t* h_pinned_cfg = nullptr;
  size_t h_pinned_cfg_n = 0;
  double* h_pinned_out = nullptr;
  size_t h_pinned_out_n = 0;

  size_t esz() const { return prec == VQNQS_PREC_BF16 ? 2 : 4; }

  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)));
    CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    allocs.push_back(p);
    return p;
  }
  void* upload_op(const std::vector<double>& v) {
    if (prec == VQNQS_PREC_BF16) {
      std::vector<uint16_t> b(v.size());
      for (size_t i = 0; i < v.size(); ++i) {
        float f = static_cast<float>(v[i]);
        uint32_t u;
        std::memcpy(&u, &f, 4);
        if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
        b[i] = static_cast<uint16_t>(u >> 16);
      }
      return upload(b);
    }
    std::vector<float> f(v.begin(), v.end());
    return upload(f);
  }
  float* upload_f(const double* p, int64_t n) {
    std::vector<float> f(p, p + n);
    return upload(f);
  }

  EngineImpl(const vqnqs_model_desc& desc, const double* const* params, int n_params, int precision,
             int device)
      : c(desc), prec(precision), dev(device) {
    auto spec = param_layout(c);
    if (n_params != int(spec.size()))
      throw ShapeError("parameter count " + std::to_string(n_params) + " != " +
                       std::to_string(spec.size()));
    if (c.group_size > 4) throw CapabilityError("GPU path: group_size <= 4");
    if (precision != VQNQS_PREC_FP32 && precision != VQNQS_PREC_BF16)
      throw ConfigError("precision must be fp32 or bf16");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw RuntimeError("no such CUDA device");
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
    d = c.d_hidden;
    nh = c.n_heads;
    dh = d / nh;
    Q = c.vq_codebook;
    H = std::max(1, c.vq_heads);
    L = c.n_blocks + (c.trailing_half_block ? 1 : 0);
    g = c.group_size;
    V = 1 << g;
    N = c.n_sites;
    T = (N + g - 1) / g;
    lastV = (N % g == 0) ? V : 1 << (N % g);
    if (T > 1024 || dh > 256) throw CapabilityError("GPU path: T <= 1024, head dim <= 256");
    use_tc_gemm = tc_gemm_ok(prec, d, d) && tc_gemm_ok(prec, 4 * d, d);
    use_tc_vq = H == 1 && c.vq_enabled && tc_vq_ok(d, Q);
    // dedup key of a location after a VQ: (residual row, code tuple); H codes
    // of ceil(log2 Q) bits pack into the key's low 32 bits when they fit,
    // otherwise the tuple is first numbered by its own exact-key pass
    qbits = 1;
    while ((int64_t(1) << qbits) < Q) ++qbits;
    tuple_pass = H > 1 && H * qbits > 32;
    if (H > 1 && H * qbits > 63)
      throw CapabilityError("GPU path: vq_heads * ceil(log2 vq_codebook) <= 63");
    use_tc_attn = tc_attn_ok(prec, d, dh, T) && !getenv("VQNQS_SIMT_ATTENTION");
    ntiles_.ensure(1);
    CK(cudaMalloc(&d_rescored, sizeof(unsigned long long)));
    allocs.push_back(d_rescored);
    // weights, parameters() order (proj/src/model.cpp:188-229)
    int i = 0;
    auto nxt = [&]() -> const double* { return params[i++]; };
    auto numel = [&](int j) { return spec[j].rows * spec[j].cols; };
    tok_embed = upload_f(nxt(), numel(0));
    pos_embed = upload_f(nxt(), numel(1));
    for (int b = 0; b < L; ++b) {
      DevBlock B{};
      // the trailing half block is attention only (no FFN, no VQ);
      // proj/src/model.cpp:113-184
      B.has_ffn = b < c.n_blocks;
      B.has_vq = B.has_ffn && c.vq_enabled;
      const double* ln1g = nxt();
      const double* ln1b = nxt();
      const double *wq = nxt(), *bq = nxt(), *wk = nxt(), *bk = nxt(), *wv = nxt(), *bv = nxt(),
                   *wo = nxt(), *bo = nxt();
      const double* cb = B.has_vq ? nxt() : nullptr;
      const double *ln2g = nullptr, *ln2b = nullptr, *w1 = nullptr, *b1 = nullptr,
                   *w2 = nullptr, *b2 = nullptr;
      if (B.has_ffn) {
        ln2g = nxt();
        ln2b = nxt();
        w1 = nxt();
        b1 = nxt();
        w2 = nxt();
        b2 = nxt();
      }
      B.ln1_g = upload_f(ln1g, d);
      B.ln1_b = upload_f(ln1b, d);
      std::vector<double> wqkv((size_t)d * 3 * d), bqkv(3 * d);
      for (int r = 0; r < d; ++r)
        for (int cc = 0; cc < d; ++cc) {
          wqkv[(size_t)r * 3 * d + cc] = wq[(size_t)r * d + cc];
          wqkv[(size_t)r * 3 * d + d + cc] = wk[(size_t)r * d + cc];
          wqkv[(size_t)r * 3 * d + 2 * d + cc] = wv[(size_t)r * d + cc];
        }
      for (int cc = 0; cc < d; ++cc) {
        bqkv[cc] = bq[cc];
        bqkv[d + cc] = bk[cc];
        bqkv[2 * d + cc] = bv[cc];
      }
      B.wqkv = upload_op(wqkv);
      B.bqkv = upload_f(bqkv.data(), 3 * d);
      B.wo = upload_op(std::vector<double>(wo, wo + (size_t)d * d));
      B.bo = upload_f(bo, d);
      if (B.has_vq) {
        // codebook [H*Q x d/H] (proj/src/model.cpp:139-142)
        B.cb32 = upload_f(cb, (int64_t)Q * d);
        // bf16 operand copy, |W_j|^2, max |W_j| and the bf16 rounding error
        // of the codebook for the certified argmin (tc_vq.cuh)
        const VqCodebook pc = prepare_codebook(cb, H * Q, d / H);
        B.wn2 = upload(pc.wn2);
        B.wmax = float(pc.wmax);
        B.werr = float(pc.werr);
        if (prec == VQNQS_PREC_BF16) B.cbA = upload(pc.bf);
        else B.cbA = upload_op(std::vector<double>(cb, cb + (size_t)Q * d));
        // the certified-argmin kernel's bf16 codebook operand (in fp32 mode the
        // codebook's bf16 rounding error enters its bound, werr)
        if (use_tc_vq)
          B.tmB = make_tmap_bf16(prec == VQNQS_PREC_BF16 ? B.cbA : upload(pc.bf), uint64_t(Q),
                                 uint64_t(d), 256);
      }
      if (B.has_ffn) {
        B.ln2_g = upload_f(ln2g, d);
        B.ln2_b = upload_f(ln2b, d);
        B.w1 = upload_op(std::vector<double>(w1, w1 + (size_t)d * 4 * d));
        B.b1 = upload_f(b1, 4 * d);
        B.w2 = upload_op(std::vector<double>(w2, w2 + (size_t)4 * d * d));
        B.b2 = upload_f(b2, d);
      }
      if (use_tc_gemm) {
        auto tr = [](const double* w, int rows, int cols) {
          std::vector<double> t((size_t)rows * cols);
          for (int r = 0; r < rows; ++r)
            for (int cc = 0; cc < cols; ++cc) t[(size_t)cc * rows + r] = w[(size_t)r * cols + cc];
          return t;
        };
        B.wqkvT = upload_op(tr(wqkv.data(), d, 3 * d));
        B.woT = upload_op(tr(wo, d, d));
        if (B.has_ffn) {
          B.w1T = upload_op(tr(w1, d, 4 * d));
          B.w2T = upload_op(tr(w2, 4 * d, d));
        }
      }
      blk.push_back(B);
    }
    lnf_g = upload_f(nxt(), d);
    lnf_b = upload_f(nxt(), d);
    head_w = upload_op(std::vector<double>(params[i], params[i] + (size_t)d * V));
    ++i;
    head_b = upload_f(nxt(), V);
    // Per-code continuation tables: o_j = code_j Wo + bo for every codeword,
    // with the same GEMM (and so the same per-row arithmetic) the per-row
    // continuation would run — the values are bit-identical, and the Wo GEMM
    // leaves the per-step path (hard part 7). With H VQ heads the
    // quantized row is H codewords side by side, so a Wo + bo =
    // bo + sum_h code_{h,j_h} Wo[rows of head h]: one [Q x d] table per head
    // (bo folded into head 0's), summed per row by k_cont_ln.
    {
      int64_t* dQ = nullptr;
      float* zeros = nullptr;
      CK(cudaMalloc(&dQ, sizeof(int64_t)));
      const int64_t q64 = Q;
      CK(cudaMemcpy(dQ, &q64, sizeof(int64_t), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&zeros, size_t(Q) * d * sizeof(float)));
      CK(cudaMemset(zeros, 0, size_t(Q) * d * sizeof(float)));
      const int hd = d / H;
      for (auto& B : blk) {
        if (!B.has_vq) continue;
        CK(cudaMalloc(&B.pwo, size_t(H) * Q * d * sizeof(float)));
        allocs.push_back(B.pwo);
        for (int h = 0; h < H; ++h) {
          const size_t aoff = size_t(h) * Q * hd * esz(), boff = size_t(h) * hd * d * esz();
          const void* A = static_cast<const char*>(B.cbA) + aoff;
          const void* W = static_cast<const char*>(B.wo) + boff;
          const void* WT = H == 1 ? B.woT : nullptr;  // tcgen05 needs the full K = d
          float* out = B.pwo + size_t(h) * Q * d;
          const float* bias = h == 0 ? B.bo : zeros;
          if (prec == VQNQS_PREC_BF16)
            gemm<bf16>(dQ, Q, d, hd, A, hd, nullptr, W, WT, bias, out, d, EPI_RESID, zeros, d,
                       nullptr, own);
          else
            gemm<float>(dQ, Q, d, hd, A, hd, nullptr, W, WT, bias, out, d, EPI_RESID, zeros, d,
                        nullptr, own);
        }
      }
      CK(cudaStreamSynchronize(own));
      CK(cudaGetLastError());
      cudaFree(dQ);
      cudaFree(zeros);
    }
    CK(cudaMalloc(&zeros_d, size_t(d) * sizeof(float)));
    allocs.push_back(zeros_d);
    CK(cudaMemset(zeros_d, 0, size_t(d) * sizeof(float)));
  }

  ~EngineImpl() {
    cudaSetDevice(dev);
    for (void* p : allocs) cudaFree(p);
    DBufRelease();
    vqs_.release();
    if (d_bonds) cudaFree(d_bonds);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : lev)
      if (e) cudaEventDestroy(e);
    red_.release();
    if (own) cudaStreamDestroy(own);
    if (h_pinned_cfg) cudaFreeHost(h_pinned_cfg);
    if (h_pinned_out) cudaFreeHost(h_pinned_out);
  }
  void DBufRelease() {
    K_.release(); Mact_.release(); row_bond_.release(); row_t1_.release(); tok0_.release();
    lrow_.release(); Ucnt_.release(); I_a.release(); I_b.release(); code_.release();
    slot_.release(); rep_of_.release(); trep_.release(); tuid_.release(); g_code_.release();
    lpos_.release(); upos_.release(); row_aoff_.release(); act_off_.release(); tab_off_.release();
    Uoff_.release(); tot_.release(); g_res_.release(); attw_.release(); diag_.release(); lpV_.release();
    lp_rows_.release(); tkey_.release(); ctup_.release(); ckey_.release(); x_a.release(); x_b.release(); y_.release();
    att_.release(); xn2_.release(); rr2_.release(); att_hi_.release(); att_lo_.release(); h_.release(); qkv_.release(); f1_.release(); cfg_stage_.release();
    out_stage_.release(); taps_codes_.release();
  }

  bool dense = false;  // no-reuse regime
  int fixed_chunk = 0;  // set_micro_batch: fixed samples per micro-batch (0 = auto)
  // test hook: forced VQ codes [n][L][R1][T] (-1 = keep), see set_code_override
  DBuf<int16_t> ovr_;
  int64_t ovr_n_ = 0, chunk_s0_ = 0;
  void set_code_override(const int16_t* host, int64_t n) {
    CK(cudaSetDevice(dev));
    if (!host || n <= 0) {
      ovr_n_ = 0;
      return;
    }
    if (H != 1) throw CapabilityError("code override supports vq_heads = 1 only");
    const size_t cnt = size_t(n) * L * (nb + 1) * T;
    ovr_.ensure(cnt);
    CK(cudaMemcpy(ovr_.p, host, cnt * sizeof(int16_t), cudaMemcpyHostToDevice));
    ovr_n_ = n;
  }
  void set_micro_batch(int samples) {
    fixed_chunk = samples;
    size_chunks();
  }
  void size_chunks() {
    if (fixed_chunk > 0) {
      S_max = fixed_chunk;
      return;
    }
    // micro-batch size: keep the per-location working set near a fixed budget.
    // ~ active locations per sample: a connected row (about half the bonds)
    // is active from its first changed token on, on average half the tokens;
    // in the no-reuse regime every row is active in full
    const double locs = double(T) + double(nb) * (dense ? 0.5 : 0.25) * double(T);
    const double bytes_per_loc = double(d) * 40.0 + 64.0;
    // working-set budget per micro-batch (VQNQS_CHUNK_GB overrides, for tuning)
    double budget = 80e9;
    if (const char* e = std::getenv("VQNQS_CHUNK_GB")) budget = std::max(1.0, std::atof(e)) * 1e9;
    S_max = int(std::clamp(budget / (locs * bytes_per_loc), 16.0, 4096.0));
  }
  void set_reuse(bool reuse) {
    dense = !reuse;
    size_chunks();
  }
  void set_hamiltonian(const int32_t* bonds, int nbonds, int n_sites, bool m) {
    if (n_sites != N) throw ShapeError("configuration size != site count");
    if (nbonds < 0) throw ConfigError("negative bond count");
    for (int b = 0; b < nbonds; ++b) {
      const int i = bonds[2 * b], j = bonds[2 * b + 1];
      if (i < 0 || j < 0 || i >= N || j >= N || i == j)
        throw ConfigError("bond " + std::to_string(b) + " out of range");
    }
    CK(cudaSetDevice(dev));
    if (k_connected_smem(T, nbonds) > smem_optin_limit())
      throw CapabilityError("GPU path: at most " +
                            std::to_string(smem_optin_limit() / 32 - 1) + " bonds");
    if (d_bonds) cudaFree(d_bonds);
    d_bonds = nullptr;
    h_bonds.assign(bonds, bonds + 2 * nbonds);
    CK(cudaMalloc(&d_bonds, std::max(1, 2 * nbonds) * sizeof(int32_t)));
    CK(cudaMemcpy(d_bonds, bonds, 2 * nbonds * sizeof(int32_t), cudaMemcpyHostToDevice));
    nb = nbonds;
    marshall = m;
    size_chunks();
  }

  // CUDA-core gathered attention (fp32 engine; bf16 engine when the tcgen05
  // kernel does not take the shape): the register-blocked kernel for the head
  // widths of the configurations, the one-query kernel otherwise.
#ifndef VQNQS_ATTQ_NQ32
#define VQNQS_ATTQ_NQ32 2
#endif
  template <typename TA, int DH, int NQ>
  void launch_attention_q(int64_t R, int R1, int T, int d, int nh, float scale, const int32_t* Icur,
                          const int64_t* Uo_cur, const TA* qkv, cudaStream_t st) {
    const size_t asmem =
        (((size_t(T) * (DH + 1) + 3) & ~size_t(3)) + size_t(T) * DH + 4 * size_t(T) * NQ + 4 * NQ * DH) * 4;
    smem_optin(reinterpret_cast<const void*>(k_attention_q<TA, DH, NQ>), asmem);
    k_attention_q<TA, DH, NQ><<<dim3(unsigned(R), nh), 128, asmem, st>>>(
        R1, T, d, scale, K_.p, row_t1_.p, row_aoff_.p, act_off_.p, Icur, Uo_cur, qkv, att_.p);
  }
  template <typename TA>
  void launch_attention_simt(int64_t R, int R1, int T, int d, int dh, int nh, float scale,
                             const int32_t* Icur, const int64_t* Uo_cur, const TA* qkv,
                             cudaStream_t st) {
    switch (dh) {
      case 8: launch_attention_q<TA, 8, 4>(R, R1, T, d, nh, scale, Icur, Uo_cur, qkv, st); return;
      case 16: launch_attention_q<TA, 16, 4>(R, R1, T, d, nh, scale, Icur, Uo_cur, qkv, st); return;
      case 32: launch_attention_q<TA, 32, VQNQS_ATTQ_NQ32>(R, R1, T, d, nh, scale, Icur, Uo_cur, qkv, st); return;
      case 64: launch_attention_q<TA, 64, 2>(R, R1, T, d, nh, scale, Icur, Uo_cur, qkv, st); return;
      default: break;
    }
    const size_t asmem = (size_t(T) * (dh + 1) + size_t(T) * dh + 4 * T + 4 * dh) * 4;
    smem_optin(reinterpret_cast<const void*>(k_attention<TA>), asmem);
    k_attention<TA><<<dim3(unsigned(R), nh), 128, asmem, st>>>(
        R1, T, d, dh, scale, K_.p, row_t1_.p, row_aoff_.p, act_off_.p, Icur, Uo_cur, qkv, att_.p);
  }

  template <typename TA>
  void gemm(const int64_t* Mp, int64_t Mcap, int Nn, int Kk, const void* A, int lda,
            const int32_t* gA, const void* B, const void* BT, const float* bias, void* out, int ldo,
            int epi, const float* resid, int ldr, const int64_t* gR, cudaStream_t st) {
    if (use_tc_gemm && BT) {
      tc_gemm(Mp, Mcap, Nn, Kk, A, lda, gA, BT, bias, out, ldo, epi, resid, ldr, gR, st, sms);
      ++launches;
      return;
    }
    const int64_t tiles = ((Mcap + 63) / 64) * ((Nn + 63) / 64);
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * 8)));
    const TA* a = static_cast<const TA*>(A);
    const TA* b = static_cast<const TA*>(B);
    if (epi == EPI_STORE)
      k_gemm_simt<TA, EPI_STORE><<<grid, 256, 0, st>>>(Mp, Nn, Kk, a, lda, gA, b, bias, out, ldo,
                                                       resid, ldr, gR);
    else if (epi == EPI_GELU)
      k_gemm_simt<TA, EPI_GELU><<<grid, 256, 0, st>>>(Mp, Nn, Kk, a, lda, gA, b, bias, out, ldo,
                                                      resid, ldr, gR);
    else
      k_gemm_simt<TA, EPI_RESID><<<grid, 256, 0, st>>>(Mp, Nn, Kk, a, lda, gA, b, bias, out, ldo,
                                                       resid, ldr, gR);
    ++launches;
  }

  // CUDA-core nearest codeword per location and VQ head (k_vq once per
  // head): codes [M x H]
  void vq_simt(const int64_t* Mp, int64_t Mcap, const float* att, const float* cb32,
               int32_t* code, cudaStream_t st) {
    const int hd = d / H;
    const int LOCS = hd > 384 ? 32 : 64;
    const size_t vsmem = (size_t(LOCS) * (hd + 1) + 32 * size_t(hd + 1) + 2 * 256) * 4;
    const int vgrid =
        int(std::max<int64_t>(1, std::min<int64_t>((Mcap + LOCS - 1) / LOCS, sms * 4)));
    for (int h = 0; h < H; ++h) {
      const float* x = att + size_t(h) * hd;
      const float* cb = cb32 + size_t(h) * Q * hd;
      if (LOCS == 64) {
        smem_optin(reinterpret_cast<const void*>(k_vq<64>), vsmem);
        k_vq<64><<<vgrid, 256, vsmem, st>>>(Mp, hd, d, x, cb, Q, code + h, H);
      } else {
        smem_optin(reinterpret_cast<const void*>(k_vq<32>), vsmem);
        k_vq<32><<<vgrid, 256, vsmem, st>>>(Mp, hd, d, x, cb, Q, code + h, H);
      }
      ++launches;
    }
  }

  template <typename TA>
  void run_chunk(const uint8_t* d_cfg, int S, double* d_e, double* d_logpsi, cudaStream_t st,
                 std::vector<int32_t>& hK, std::vector<int32_t>& hU, Engine::Taps* taps,
                 std::vector<int32_t>* tap_codes, std::vector<int64_t>* tap_act_off,
                 std::vector<int32_t>* tap_t1, std::vector<int64_t>* tap_aoff,
                 std::vector<double>* tap_lp) {
    const int R1 = nb + 1;
    const int64_t R = int64_t(S) * R1;
    K_.ensure(S); attw_.ensure(S); Mact_.ensure(S); diag_.ensure(S); act_off_.ensure(S); tab_off_.ensure(S);
    row_bond_.ensure(R); row_perm_.ensure(R); row_t1_.ensure(R); row_aoff_.ensure(R); tok0_.ensure(int64_t(S) * T);
    Ucnt_.ensure(int64_t(L + 1) * S); Uoff_.ensure(int64_t(L + 1) * S); tot_.ensure(2 * (L + 2));
    int64_t* tot = tot_.p;  // [0] M total, [1] table total, [2+b] U_b total
    const size_t csmem = k_connected_smem(T, nb);
    smem_optin(reinterpret_cast<const void*>(k_connected), csmem);
    k_connected<<<(S * 32 + 127) / 128, 128, csmem, st>>>(S, N, g, T, nb, int(dense), attn_cap,
                                                      d_cfg, d_bonds,
                                                      K_.p, diag_.p,
                                                      row_bond_.p, row_t1_.p, row_aoff_.p, Mact_.p,
                                                      tok0_.p, attw_.p, row_perm_.p);
    k_scan<<<1, 1024, 0, st>>>(S, Mact_.p, act_off_.p, tot + 0, 0);
    k_scan<<<1, 1024, 0, st>>>(S, Mact_.p, tab_off_.p, tot + 1, 1);
    launches += 3;
    int64_t totals[2];
    CK(cudaMemcpyAsync(totals, tot, sizeof(totals), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t M = totals[0], TB = totals[1];
    // arena
    lrow_.ensure(M); lpos_.ensure(M); I_a.ensure(M); I_b.ensure(M); code_.ensure(M * H);
    slot_.ensure(M); rep_of_.ensure(M); g_code_.ensure(M * H); g_res_.ensure(M); upos_.ensure(M);
    if (tkey_.n < size_t(TB)) {
      tkey_.ensure(TB); trep_.ensure(TB); tuid_.ensure(TB);
      CK(cudaMemsetAsync(tkey_.p, 0xFF, tkey_.n * sizeof(unsigned long long), st));
      CK(cudaMemsetAsync(trep_.p, 0x7F, trep_.n * sizeof(int32_t), st));
    }
    x_a.ensure(M * d); x_b.ensure(M * d); y_.ensure(M * d);
    h_.ensure(M * d * esz()); qkv_.ensure(M * 3 * d * esz()); f1_.ensure(M * 4 * d * esz());
    // fp32 attention rows: the CUDA-core attention's output, or the
    // CUDA-core quantizer's input
    if (!use_tc_attn || !use_tc_vq) att_.ensure(M * d);
    if (use_tc_vq || use_tc_attn) {
      att_hi_.ensure(M * d);
      att_lo_.ensure(M * d);
      xn2_.ensure(M);
      rr2_.ensure(M);
    }
    lpV_.ensure(M * V);
    const int64_t Rtot = R * T;
    k_enumerate<<<int((Rtot + 255) / 256), 256, 0, st>>>(S, R1, T, K_.p, row_t1_.p, row_aoff_.p,
                                                         act_off_.p, lrow_.p, lpos_.p);
    // (d) input layer
    int32_t* Icur = I_a.p;
    int32_t* Inext = I_b.p;
    smem_optin(reinterpret_cast<const void*>(k_dedup<0>), dedup_smem_bytes());
    k_dedup<0><<<S, DEDUP_THREADS, dedup_smem_bytes(), st>>>(Mact_.p, act_off_.p, tab_off_.p, tkey_.p, trep_.p, tuid_.p,
                                  slot_.p, lrow_.p, lpos_.p, tok0_.p, row_bond_.p, d_bonds, R1, T,
                                  g, V, nullptr, nullptr, int(dense), Icur, rep_of_.p, Ucnt_.p,
                                  nullptr);
    k_scan<<<1, 1024, 0, st>>>(S, Ucnt_.p, Uoff_.p, tot + 2, 0);
    k_embed<<<S, 256, 0, st>>>(d, R1, T, g, V, Ucnt_.p, Uoff_.p, act_off_.p, rep_of_.p, lrow_.p,
                               lpos_.p, tok0_.p, row_bond_.p, d_bonds, tok_embed, pos_embed, x_a.p);
    launches += 4;
    float* xcur = x_a.p;
    float* xnext = x_b.p;
    float* ybuf = y_.p;
    const int lnGrid = sms * 8;
    const float scale = float(1.0 / std::sqrt(double(dh)));
    for (int b = 0; b < L; ++b) {
      const DevBlock& B = blk[b];
      const int64_t* Mb = tot + 2 + b;
      int32_t* Uc_cur = Ucnt_.p + int64_t(b) * S;
      int64_t* Uo_cur = Uoff_.p + int64_t(b) * S;
      int32_t* Uc_next = Ucnt_.p + int64_t(b + 1) * S;
      int64_t* Uo_next = Uoff_.p + int64_t(b + 1) * S;
      (void)Uc_cur;
      TA* h = reinterpret_cast<TA*>(h_.p);
      TA* qkv = reinterpret_cast<TA*>(qkv_.p);
      TA* f1 = reinterpret_cast<TA*>(f1_.p);
      launch_layernorm<TA>(lnGrid, st, Mb, d, xcur, B.ln1_g, B.ln1_b, h);
      ++launches;
      gemm<TA>(Mb, M, 3 * d, d, h, d, nullptr, B.wqkv, B.wqkvT, B.bqkv, qkv, 3 * d, EPI_STORE,
               nullptr, 0, nullptr, st);
      CK(cudaEventRecord(lev[3 * b + 0], st));
      if (use_tc_attn) {
        // tiles of whole rows (once per chunk; rows do not change across layers)
        if (b == 0) {
          tiles_.ensure(R);
          tcnt_.ensure(S);
          toff_.ensure(S + 1);
          k_build_tiles<<<(S + 127) / 128, 128, 0, st>>>(0, S, R1, T, attn_cap, K_.p, row_t1_.p,
                                                         row_perm_.p, act_off_.p, tcnt_.p, nullptr,
                                                         nullptr, tiles_.p, ntiles_.p);
          k_scan<<<1, 1024, 0, st>>>(S, tcnt_.p, toff_.p, toff_.p + S, 0);
          k_build_tiles<<<(S + 127) / 128, 128, 0, st>>>(1, S, R1, T, attn_cap, K_.p, row_t1_.p,
                                                         row_perm_.p, act_off_.p, tcnt_.p,
                                                         toff_.p, toff_.p + S, tiles_.p, ntiles_.p);
          launches += 3;
        }
        // per-layer tile tables (qkv rows follow this layer's dedup); at most
        // 2 M / 128 + 3 S tiles (a tile and the longest row of the next hold > 128)
        const int64_t tcap = std::min<int64_t>(R, M / 64 + 3 * int64_t(S) + 16);
        tinfo_.ensure(size_t(tcap) * TINFO_BYTES);
        k_tile_info<<<sms * 8, 128, 0, st>>>(tiles_.p, ntiles_.p, R1, T, row_t1_.p, act_off_.p,
                                             lrow_.p, lpos_.p, Icur, Uo_cur, tinfo_.p);
        ++launches;
        const size_t asmem = AttnSmem(T).total + 1024;
        launch_tc_attention(dh, sms, asmem, st, (const uint8_t*)tinfo_.p,
                            (const int32_t*)ntiles_.p, T, d, dh, scale,
                            reinterpret_cast<const bf16*>(qkv), att_hi_.p, att_lo_.p, xn2_.p,
                            rr2_.p);
      } else {
        launch_attention_simt<TA>(R, R1, T, d, dh, nh, scale, Icur, Uo_cur, qkv, st);
      }
      CK(cudaEventRecord(lev[3 * b + 2], st));
      const int64_t* Mn = tot + 3 + b;
      if (B.has_vq) {
        if (use_tc_vq) {
          if (!use_tc_attn) {
            k_vq_prep<<<sms * 8, 256, 0, st>>>(tot + 0, d, att_.p, att_hi_.p, att_lo_.p, xn2_.p,
                                               rr2_.p);
            ++launches;
          }
          tc_vq(tot + 0, M, d, att_hi_.p, att_lo_.p, xn2_.p, rr2_.p, B.tmB, B.cb32, B.wn2, B.wmax,
                B.werr, Q, code_.p, d_rescored, vqs_, st, sms);
          launches += 2;
        } else {
          if (use_tc_attn) {  // x = xh + xl for the CUDA-core quantizer
            k_join_split<<<sms * 8, 256, 0, st>>>(tot + 0, d, att_hi_.p, att_lo_.p, att_.p);
            ++launches;
          }
          vq_simt(tot + 0, M, att_.p, B.cb32, code_.p, st);
        }
        if (ovr_n_ > 0) {  // test hook: the reference's codes at every location
          k_code_override<<<sms * 4, 256, 0, st>>>(tot + 0, lrow_.p, lpos_.p, R1, T, L, b,
                                                   chunk_s0_, ovr_.p, code_.p);
          ++launches;
        }
        CK(cudaEventRecord(lev[3 * b + 1], st));
        if (tap_codes) {
          std::vector<int32_t> hc(size_t(M) * H);
          CK(cudaMemcpyAsync(hc.data(), code_.p, hc.size() * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          tap_codes->insert(tap_codes->end(), hc.begin(), hc.end());
        }
        // requantize (proj/src/dedup.cpp:136-185): key (residual row, codes)
        const int32_t* ckey = code_.p;
        if (H > 1) {
          ckey_.ensure(M);
          if (tuple_pass) {
            ctup_.ensure(M);
            k_pack_codes<<<int((M + 255) / 256), 256, 0, st>>>(tot + 0, H, qbits, code_.p,
                                                               ctup_.p, nullptr);
            smem_optin(reinterpret_cast<const void*>(k_dedup<2>), dedup_smem_bytes());
            k_dedup<2><<<S, DEDUP_THREADS, dedup_smem_bytes(), st>>>(Mact_.p, act_off_.p, tab_off_.p, tkey_.p, trep_.p,
                                          tuid_.p, slot_.p, nullptr, nullptr, nullptr, nullptr,
                                          nullptr, R1, T, g, V, nullptr, nullptr, int(dense),
                                          ckey_.p, rep_of_.p, Uc_next, ctup_.p);
            launches += 2;
          } else {
            k_pack_codes<<<int((M + 255) / 256), 256, 0, st>>>(tot + 0, H, qbits, code_.p,
                                                               nullptr, ckey_.p);
            ++launches;
          }
          ckey = ckey_.p;
        }
        smem_optin(reinterpret_cast<const void*>(k_dedup<1>), dedup_smem_bytes());
        k_dedup<1><<<S, DEDUP_THREADS, dedup_smem_bytes(), st>>>(Mact_.p, act_off_.p, tab_off_.p, tkey_.p, trep_.p, tuid_.p,
                                      slot_.p, nullptr, nullptr, nullptr, nullptr, nullptr, R1, T,
                                      g, V, Icur, ckey, int(dense), Inext, rep_of_.p, Uc_next,
                                      nullptr);
        k_scan<<<1, 1024, 0, st>>>(S, Uc_next, Uo_next, tot + 3 + b, 0);
        k_build_gather<<<S, 256, 0, st>>>(H, Uc_next, Uo_next, Uo_cur, act_off_.p, rep_of_.p,
                                          code_.p, Icur, lpos_.p, g_code_.p, g_res_.p, upos_.p);
        launches += 3;
        // continuation (proj/src/dedup.cpp:246-267): y = r + (code rows Wo + bo)
        // from the per-code tables, fused with LN2
        launch_cont_ln<TA>(lnGrid, st, Mn, d, H, Q, xcur, g_res_.p, g_code_.p, B.pwo,
                                              B.ln2_g, B.ln2_b, ybuf, h);
        ++launches;
        gemm<TA>(Mn, M, 4 * d, d, h, d, nullptr, B.w1, B.w1T, B.b1, f1, 4 * d, EPI_GELU, nullptr,
                 0, nullptr, st);
        gemm<TA>(Mn, M, d, 4 * d, f1, 4 * d, nullptr, B.w2, B.w2T, B.b2, xnext, d, EPI_RESID,
                 ybuf, d, nullptr, st);
        std::swap(xcur, xnext);
      } else {
        // a block without VQ: densify_attention (proj/src/dedup.cpp:187-211),
        // every location its own row (the reference's U = K T; here the
        // active locations, the others being the base row's), then
        // y = r + (att Wo + bo) and, in a full block, the FFN
        CK(cudaEventRecord(lev[3 * b + 1], st));
        if (tap_codes) tap_codes->insert(tap_codes->end(), size_t(M) * H, -1);
        k_densify<<<S, 256, 0, st>>>(Mact_.p, act_off_.p, Uo_cur, Icur, lpos_.p, Inext, g_res_.p,
                                     upos_.p, Uc_next);
        k_scan<<<1, 1024, 0, st>>>(S, Uc_next, Uo_next, tot + 3 + b, 0);
        k_gather_rows<<<lnGrid, 256, 0, st>>>(Mn, d, xcur, g_res_.p, ybuf);
        launches += 3;
        const void* A = att_.p;  // fp32 engine: the fp32 attention rows
        if (prec == VQNQS_PREC_BF16) {
          if (use_tc_attn) {
            A = att_hi_.p;  // bf16(x): the operand the emulated reference rounds to
          } else {
            k_to_bf16<<<lnGrid, 256, 0, st>>>(tot + 0, d, att_.p,
                                              reinterpret_cast<bf16*>(h));
            ++launches;
            A = h;
          }
        }
        gemm<TA>(Mn, M, d, d, A, d, nullptr, B.wo, B.woT, B.bo, xnext, d, EPI_RESID, ybuf, d,
                 nullptr, st);
        if (B.has_ffn) {
          launch_layernorm<TA>(lnGrid, st, Mn, d, xnext, B.ln2_g, B.ln2_b, h);
          ++launches;
          gemm<TA>(Mn, M, 4 * d, d, h, d, nullptr, B.w1, B.w1T, B.b1, f1, 4 * d, EPI_GELU,
                   nullptr, 0, nullptr, st);
          gemm<TA>(Mn, M, d, 4 * d, f1, 4 * d, nullptr, B.w2, B.w2T, B.b2, ybuf, d, EPI_RESID,
                   xnext, d, nullptr, st);
          float* old = xcur;  // the block output is in ybuf
          xcur = ybuf;
          ybuf = xnext;
          xnext = old;
        } else {
          std::swap(xcur, xnext);
        }
      }
      std::swap(Icur, Inext);
    }
    // (e) head and E_loc
    const int64_t* ML = tot + 2 + L;
    TA* h = reinterpret_cast<TA*>(h_.p);
    launch_layernorm<TA>(lnGrid, st, ML, d, xcur, lnf_g, lnf_b, h);
    k_head<TA><<<lnGrid, 256, 0, st>>>(ML, d, V, lastV, T, h, static_cast<const TA*>(head_w),
                                       head_b, upos_.p, lpV_.p);
    double* lp_rows = nullptr;
    if (tap_lp) {
      lp_rows_.ensure(R);
      lp_rows = lp_rows_.p;
    }
    smem_optin(reinterpret_cast<const void*>(k_eloc), size_t(R1) * sizeof(double));
    k_eloc<<<S, ELOC_THREADS, size_t(R1) * sizeof(double), st>>>(S, R1, T, g, V, marshall ? -0.5 : 0.5, K_.p,
                                                 diag_.p, row_bond_.p, row_t1_.p, row_aoff_.p,
                                                 act_off_.p, tok0_.p, d_bonds, Icur,
                                                 Uoff_.p + int64_t(L) * S, lpV_.p, d_e, d_logpsi,
                                                 lp_rows);
    launches += 3;
    CK(cudaGetLastError());
    hK.resize(S);
    hU.resize(size_t(L + 1) * S);
    std::vector<int64_t> haw(S);
    CK(cudaMemcpyAsync(haw.data(), attw_.p, S * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hK.data(), K_.p, S * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hU.data(), Ucnt_.p, hU.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    int32_t h_ntiles = 0;
    if (use_tc_attn)
      CK(cudaMemcpyAsync(&h_ntiles, ntiles_.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (taps) {
      tap_act_off->resize(S);
      tap_t1->resize(R);
      tap_aoff->resize(R);
      CK(cudaMemcpyAsync(tap_act_off->data(), act_off_.p, S * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(tap_t1->data(), row_t1_.p, R * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(tap_aoff->data(), row_aoff_.p, R * 8, cudaMemcpyDeviceToHost, st));
      tap_lp->resize(R);
      CK(cudaMemcpyAsync(tap_lp->data(), lp_rows_.p, R * 8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < L; ++b) {  // per-layer stage timing (no per-layer host sync)
      float ms = 0.f, ma = 0.f;
      CK(cudaEventElapsedTime(&ms, lev[3 * b + 0], lev[3 * b + 1]));
      CK(cudaEventElapsedTime(&ma, lev[3 * b + 0], lev[3 * b + 2]));
      prof[0] += ms;
      prof[2] += 2;
      prof[7] += ma;
      prof[6] += ms - ma;
    }
    // algorithmic work of the attention->VQ stage actually executed
    double aw = 0;
    for (int s2 = 0; s2 < S; ++s2) aw += double(haw[s2]);
    int nvq = 0;
    for (const auto& Bk : blk) nvq += Bk.has_vq ? 1 : 0;
    prof[1] += double(L) * 4.0 * d * aw + double(nvq) * 2.0 * double(d) * Q * double(M);
    prof[9] += double(L) * 4.0 * d * aw;            // attention (QK^T + PV, live keys)
    prof[10] += double(nvq) * 2.0 * double(d) * Q * double(M);  // VQ distance GEMM
    prof[3] += double(M) * L;
    prof[11] += double(h_ntiles) * L;  // attention tiles (<= 128 locations each)
    for (int s2 = 0; s2 < S; ++s2)
      for (int b = 0; b < L; ++b) {
        prof[4] += hU[size_t(b) * S + s2];
        prof[5] += hU[size_t(b + 1) * S + s2];
      }
  }

  void run_device(const uint8_t* d_cfg, int64_t B, double* d_e, double* d_logpsi, int64_t* ledger7,
                  cudaStream_t st, Engine::Taps* taps) {
    if (!d_bonds && nb == 0 && h_bonds.empty())
      throw UsageError("set_hamiltonian must be called before local_energies");
    CK(cudaSetDevice(dev));
    launches = 0;
    for (double& v : prof) v = 0;
    CK(cudaMemsetAsync(d_rescored, 0, sizeof(unsigned long long), st));
    if (!ev[0])
      for (auto& e : ev) CK(cudaEventCreate(&e));
    if (lev.size() < size_t(3 * L)) {
      lev.resize(3 * L, nullptr);
      for (auto& e : lev)
        if (!e) CK(cudaEventCreate(&e));
    }
    int64_t tap_code_pos = 0, tap_lp_pos = 0;
    if (ovr_n_ > 0 && ovr_n_ != B)
      throw UsageError("code override set for " + std::to_string(ovr_n_) +
                       " samples, batch has " + std::to_string(B));
    for (int64_t s0 = 0; s0 < B; s0 += S_max) {
      const int S = int(std::min<int64_t>(S_max, B - s0));
      chunk_s0_ = s0;
      std::vector<int32_t> hK, hU;
      std::vector<int32_t> tcodes;
      std::vector<int64_t> tact, taoff;
      std::vector<int32_t> tt1;
      std::vector<double> tlp;
      if (prec == VQNQS_PREC_BF16)
        run_chunk<bf16>(d_cfg + s0 * N, S, d_e + s0, d_logpsi + s0, st, hK, hU, taps,
                        taps ? &tcodes : nullptr, &tact, &tt1, &taoff, taps ? &tlp : nullptr);
      else
        run_chunk<float>(d_cfg + s0 * N, S, d_e + s0, d_logpsi + s0, st, hK, hU, taps,
                         taps ? &tcodes : nullptr, &tact, &tt1, &taoff, taps ? &tlp : nullptr);
      for (int s = 0; s < S; ++s) {
        std::vector<int64_t> U(L + 1);
        for (int b = 0; b <= L; ++b) U[b] = hU[size_t(b) * S + s];
        // a block without VQ densifies: the reference counts every one of
        // the K T locations as a unique row (the engine computes the active
        // ones; the rest are the base row's, identical by causality)
        for (int b = 0; b < L; ++b)
          if (!blk[b].has_vq) U[b + 1] = int64_t(hK[s]) * T;
        if (ledger7) ledger_add(c, hK[s], U.data(), ledger7);
        if (taps) {
          if (taps->K) taps->K[s0 + s] = hK[s];
          if (taps->U)
            for (int b = 0; b <= L; ++b) taps->U[(s0 + s) * (L + 1) + b] = U[b];
        }
      }
      if (taps) {
        const int R1 = nb + 1;
        const int64_t M = int64_t(tcodes.size()) / std::max(1, L * H);
        for (int s = 0; s < S; ++s) {
          const int Ks = hK[s];
          if (taps->codes) {
            if (tap_code_pos + int64_t(L) * Ks * T * H > taps->codes_cap)
              throw ShapeError("taps: codes buffer too small");
            for (int b = 0; b < L; ++b)
              for (int k = 0; k < Ks; ++k) {
                const int64_t r = int64_t(s) * R1 + k;
                const int a = k == 0 ? 0 : tt1[r] + 1;
                for (int p = 0; p < T; ++p) {
                  const int64_t loc = p < a ? tact[s] + p : tact[s] + taoff[r] + (p - a);
                  for (int hh = 0; hh < H; ++hh)
                    taps->codes[tap_code_pos + ((int64_t(b) * Ks + k) * T + p) * H + hh] =
                        tcodes[(size_t(b) * M + loc) * H + hh];
                }
              }
            tap_code_pos += int64_t(L) * Ks * T * H;
          }
          if (taps->lp_rows) {
            if (tap_lp_pos + Ks > taps->lp_cap) throw ShapeError("taps: lp buffer too small");
            for (int k = 0; k < Ks; ++k) taps->lp_rows[tap_lp_pos + k] = tlp[int64_t(s) * R1 + k];
            tap_lp_pos += Ks;
          }
        }
      }
    }
    unsigned long long resc = 0;
    CK(cudaMemcpyAsync(&resc, d_rescored, sizeof(resc), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    prof[8] = double(resc);
  }

  // ---------------------------------------------------------------- sampler
  template <typename TA>
  void sample_chunk(int B, const double* d_u, int32_t* d_tok, double* d_lp, cudaStream_t st) {
    const size_t es = esz();
    DBuf<float> x, ya, att;
    DBuf<char> h, qkv, f1, kc, vc;
    DBuf<bf16> xh, xl;
    DBuf<float> xn2, rr2;
    DBuf<int32_t> code;
    DBuf<int64_t> dB, iota;
    DBuf<int16_t> pos;
    DBuf<double> lpv;
    x.ensure(size_t(B) * d);
    ya.ensure(size_t(B) * d);
    att.ensure(size_t(B) * d);
    h.ensure(size_t(B) * d * es);
    qkv.ensure(size_t(B) * 3 * d * es);
    f1.ensure(size_t(B) * 4 * d * es);
    kc.ensure(size_t(L) * B * T * d * es);
    vc.ensure(size_t(L) * B * T * d * es);
    code.ensure(size_t(B) * H);
    dB.ensure(1);
    iota.ensure(B);
    pos.ensure(B);
    lpv.ensure(size_t(B) * V);
    if (use_tc_vq) {
      xh.ensure(size_t(B) * d);
      xl.ensure(size_t(B) * d);
      xn2.ensure(B);
      rr2.ensure(B);
    }
    const int64_t b64 = B;
    CK(cudaMemcpyAsync(dB.p, &b64, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    k_iota64<<<(B + 255) / 256, 256, 0, st>>>(B, iota.p);
    const int lnGrid = sms * 8;
    const float scale = float(1.0 / std::sqrt(double(dh)));
    TA* hp = reinterpret_cast<TA*>(h.p);
    TA* qp = reinterpret_cast<TA*>(qkv.p);
    TA* fp = reinterpret_cast<TA*>(f1.p);
    const int awpb = 4;
    const size_t asmem = size_t(awpb) * (dh + T) * sizeof(float);
    smem_optin(reinterpret_cast<const void*>(k_dec_attention<TA>), asmem);
    launches += 2;
    for (int t = 0; t < T; ++t) {
      k_dec_embed<<<B, 128, 0, st>>>(B, d, T, V, t, d_tok, tok_embed, pos_embed, x.p);
      k_fill_i16<<<(B + 255) / 256, 256, 0, st>>>(B, int16_t(t), pos.p);
      launches += 2;
      float* xc = x.p;
      float* xn = ya.p;
      for (int b = 0; b < L; ++b) {
        const DevBlock& Bk = blk[b];
        launch_layernorm<TA>(lnGrid, st, dB.p, d, xc, Bk.ln1_g, Bk.ln1_b, hp);
        gemm<TA>(dB.p, B, 3 * d, d, hp, d, nullptr, Bk.wqkv, Bk.wqkvT, Bk.bqkv, qp, 3 * d,
                 EPI_STORE, nullptr, 0, nullptr, st);
        TA* kcb = reinterpret_cast<TA*>(kc.p) + size_t(b) * B * T * d;
        TA* vcb = reinterpret_cast<TA*>(vc.p) + size_t(b) * B * T * d;
        const int64_t jobs = int64_t(B) * nh;
        k_dec_attention<TA><<<int((jobs + awpb - 1) / awpb), 32 * awpb, asmem, st>>>(
            B, d, nh, T, t, scale, qp, kcb, vcb, att.p);
        launches += 2;
        if (!Bk.has_vq) {
          // no VQ (model.cpp:325-355 with has_vq = false): x += att Wo + bo,
          // then the FFN in a full block
          const void* A = att.p;
          if (prec == VQNQS_PREC_BF16) {
            k_to_bf16<<<lnGrid, 256, 0, st>>>(dB.p, d, att.p, reinterpret_cast<bf16*>(hp));
            ++launches;
            A = hp;
          }
          gemm<TA>(dB.p, B, d, d, A, d, nullptr, Bk.wo, Bk.woT, Bk.bo, xn, d, EPI_RESID, xc, d,
                   nullptr, st);
          if (Bk.has_ffn) {
            launch_layernorm<TA>(lnGrid, st, dB.p, d, xn, Bk.ln2_g, Bk.ln2_b, hp);
            ++launches;
            gemm<TA>(dB.p, B, 4 * d, d, hp, d, nullptr, Bk.w1, Bk.w1T, Bk.b1, fp, 4 * d,
                     EPI_GELU, nullptr, 0, nullptr, st);
            gemm<TA>(dB.p, B, d, 4 * d, fp, 4 * d, nullptr, Bk.w2, Bk.w2T, Bk.b2, xc, d,
                     EPI_RESID, xn, d, nullptr, st);
          } else {
            std::swap(xc, xn);
          }
          continue;
        }
        if (use_tc_vq) {
          k_vq_prep<<<sms * 8, 256, 0, st>>>(dB.p, d, att.p, xh.p, xl.p, xn2.p, rr2.p);
          tc_vq(dB.p, B, d, xh.p, xl.p, xn2.p, rr2.p, Bk.tmB, Bk.cb32, Bk.wn2, Bk.wmax, Bk.werr, Q,
                code.p, nullptr, vqs_, st, sms);
          launches += 3;
        } else {
          vq_simt(dB.p, B, att.p, Bk.cb32, code.p, st);
        }
        // continuation (proj/src/dedup.cpp:246-267) from the per-code Wo tables
        launch_cont_ln<TA>(lnGrid, st, dB.p, d, H, Q, xc, iota.p, code.p, Bk.pwo, Bk.ln2_g,
                                              Bk.ln2_b, y_.p, hp);
        ++launches;
        gemm<TA>(dB.p, B, 4 * d, d, hp, d, nullptr, Bk.w1, Bk.w1T, Bk.b1, fp, 4 * d, EPI_GELU,
                 nullptr, 0, nullptr, st);
        gemm<TA>(dB.p, B, d, 4 * d, fp, 4 * d, nullptr, Bk.w2, Bk.w2T, Bk.b2, xn, d, EPI_RESID,
                 y_.p, d, nullptr, st);
        std::swap(xc, xn);
      }
      launch_layernorm<TA>(lnGrid, st, dB.p, d, xc, lnf_g, lnf_b, hp);
      k_head<TA><<<lnGrid, 256, 0, st>>>(dB.p, d, V, lastV, T, hp, static_cast<const TA*>(head_w),
                                         head_b, pos.p, lpv.p);
      k_dec_sample<<<(B + 127) / 128, 128, 0, st>>>(B, T, V, t, lpv.p, d_u, d_tok, d_lp);
      launches += 3;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
  }

  void sample(int64_t count, uint64_t seed, uint64_t skip, uint8_t* cfg_out, double* lp_out) {
    CK(cudaSetDevice(dev));
    launches = 0;
    cudaStream_t st = own;
    // the reference's draws: step-major, then sample index (model.cpp:497-518)
    std::vector<double> hu(size_t(skip) + size_t(count) * T);
    rng_uniforms(seed, int64_t(hu.size()), hu.data());
    hu.erase(hu.begin(), hu.begin() + int64_t(skip));
    // micro-batches of samples (K/V cache: 2 L T d per sample)
    const double per = double(L) * T * d * esz() * 2 + double(d) * 60;
    const int64_t Bmax = std::max<int64_t>(1, std::min<int64_t>(int64_t(24e9 / per), 65536));
    DBuf<double> du, dlp;
    DBuf<int32_t> dtok;
    DBuf<uint8_t> dcfg;
    for (int64_t s0 = 0; s0 < count; s0 += Bmax) {
      const int B = int(std::min<int64_t>(Bmax, count - s0));
      std::vector<double> cu(size_t(B) * T);
      for (int t = 0; t < T; ++t)
        std::memcpy(cu.data() + size_t(t) * B, hu.data() + size_t(t) * count + s0,
                    size_t(B) * sizeof(double));
      du.ensure(cu.size());
      dlp.ensure(B);
      dtok.ensure(size_t(B) * T);
      dcfg.ensure(size_t(B) * N);
      y_.ensure(size_t(B) * d);
      CK(cudaMemcpyAsync(du.p, cu.data(), cu.size() * sizeof(double), cudaMemcpyHostToDevice,
                         st));
      if (prec == VQNQS_PREC_BF16)
        sample_chunk<bf16>(B, du.p, dtok.p, dlp.p, st);
      else
        sample_chunk<float>(B, du.p, dtok.p, dlp.p, st);
      k_detokenize<<<int((int64_t(B) * N + 255) / 256), 256, 0, st>>>(B, N, g, T, dtok.p, dcfg.p);
      ++launches;
      CK(cudaMemcpyAsync(cfg_out + s0 * N, dcfg.p, size_t(B) * N, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(lp_out + s0, dlp.p, size_t(B) * sizeof(double), cudaMemcpyDeviceToHost,
                         st));
      CK(cudaStreamSynchronize(st));
    }
  }

  void run_host(const uint8_t* configs, int64_t B, double* e_re, double* e_im, double* logpsi,
                int64_t* ledger7, Engine::Taps* taps) {
    CK(cudaSetDevice(dev));
    const size_t nbytes = size_t(B) * N;
    if (h_pinned_cfg_n < nbytes) {
      if (h_pinned_cfg) cudaFreeHost(h_pinned_cfg);
      CK(cudaMallocHost(&h_pinned_cfg, nbytes));
      h_pinned_cfg_n = nbytes;
    }
    if (h_pinned_out_n < size_t(2 * B)) {
      if (h_pinned_out) cudaFreeHost(h_pinned_out);
      CK(cudaMallocHost(&h_pinned_out, 2 * B * sizeof(double)));
      h_pinned_out_n = 2 * B;
    }
    std::memcpy(h_pinned_cfg, configs, nbytes);
    cfg_stage_.ensure(nbytes);
    out_stage_.ensure(2 * B);
    CK(cudaMemcpyAsync(cfg_stage_.p, h_pinned_cfg, nbytes, cudaMemcpyHostToDevice, own));
    run_device(cfg_stage_.p, B, out_stage_.p, out_stage_.p + B, ledger7, own, taps);
    CK(cudaMemcpyAsync(h_pinned_out, out_stage_.p, 2 * B * sizeof(double), cudaMemcpyDeviceToHost,
                       own));
    CK(cudaStreamSynchronize(own));
    for (int64_t i = 0; i < B; ++i) {
      const double e = h_pinned_out[i];
      if (!std::isfinite(e)) {
        std::string s;
        for (int j = 0; j < N; ++j) s.push_back(configs[i * N + j] ? '1' : '0');
        throw NumericError("non-finite local energy at configuration " + s);
      }
      e_re[i] = e;
      if (e_im) e_im[i] = 0.0;
      if (logpsi) logpsi[i] = h_pinned_out[B + i];
    }
  }

  // fill_stats over a device-resident shard e[B] (fp64, fixed order) into
  // red[0..3] (n, sum, #non-finite, centred sum of squares) and, when led is
  // given, the ledger into red[4..10] (int64); with comm every quantity is
  // summed over the ranks (NCCL on stream st). Asynchronous.
  void stats_device(const double* e, int64_t B, Comm* comm, cudaStream_t st, double* red,
                    const int64_t* led) {
    k_stats<<<1, 1024, 0, st>>>(B, e, red, 0);
    if (comm) comm->allreduce_f64(red, 3, st);
    k_stats<<<1, 1024, 0, st>>>(B, e, red, 1);
    if (comm) comm->allreduce_f64(red + 3, 1, st);
    launches += 2;
    if (led) {
      int64_t* dled = reinterpret_cast<int64_t*>(red + 4);
      CK(cudaMemcpyAsync(dled, led, VQNQS_LEDGER_SLOTS * sizeof(int64_t),
                         cudaMemcpyHostToDevice, st));
      if (comm) comm->allreduce_i64(dled, VQNQS_LEDGER_SLOTS, st);
    }
  }

  // fill_stats of a device-resident shard (the device-buffer estimate):
  // stats = {energy, variance, std_err, k}; synchronous on st.
  DBuf<double> red_;
  void fill_stats_device(const double* e, int64_t B, Comm* comm, cudaStream_t st,
                         double* stats) {
    CK(cudaSetDevice(dev));
    red_.ensure(16);
    stats_device(e, B, comm, st, red_.p, nullptr);
    double hr[4];
    CK(cudaMemcpyAsync(hr, red_.p, sizeof(hr), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hr[2] > 0) throw NumericError("non-finite local energy in the batch");
    finish_stats(hr, stats);
  }
  static void finish_stats(const double* hr, double* stats) {
    const int64_t k = int64_t(hr[0] + 0.5);
    if (k < 1) throw ConfigError("k_samples must be >= 1");
    const double var = k > 1 ? hr[3] / double(k - 1) : 0.0;
    stats[0] = hr[1] / hr[0];
    stats[1] = var;
    stats[2] = std::sqrt(var / double(k));
    stats[3] = double(k);
  }

  // estimate_energy's statistics (proj/src/trainer.cpp:200-211 with
  // fill_stats, :184-198) over this rank's shard; with a communicator the
  // sums, the non-finite count and the ledger are reduced over all ranks
  // (NCCL, on the engine stream), so every rank returns the global estimate.
  void estimate(const uint8_t* configs, int64_t B, double* e_re, double* logpsi,
                int64_t* ledger7, Comm* comm, double* stats) {
    CK(cudaSetDevice(dev));
    if (comm && comm->device() != dev)
      throw UsageError("communicator and engine are on different devices");
    const size_t nbytes = size_t(B) * N;
    if (h_pinned_cfg_n < nbytes) {
      if (h_pinned_cfg) cudaFreeHost(h_pinned_cfg);
      CK(cudaMallocHost(&h_pinned_cfg, std::max<size_t>(nbytes, 1)));
      h_pinned_cfg_n = nbytes;
    }
    if (h_pinned_out_n < size_t(2 * B + 16)) {
      if (h_pinned_out) cudaFreeHost(h_pinned_out);
      CK(cudaMallocHost(&h_pinned_out, (2 * B + 16) * sizeof(double)));
      h_pinned_out_n = 2 * B + 16;
    }
    if (nbytes) std::memcpy(h_pinned_cfg, configs, nbytes);
    cfg_stage_.ensure(std::max<size_t>(nbytes, 1));
    out_stage_.ensure(2 * B + 16);
    double* red = out_stage_.p + 2 * B;  // [4] sums, then [8] ledger (int64)
    int64_t led[VQNQS_LEDGER_SLOTS] = {0, 0, 0, 0, 0, 0, 0};
    if (B > 0) {
      CK(cudaMemcpyAsync(cfg_stage_.p, h_pinned_cfg, nbytes, cudaMemcpyHostToDevice, own));
      run_device(cfg_stage_.p, B, out_stage_.p, out_stage_.p + B, led, own, nullptr);
    }
    stats_device(out_stage_.p, B, comm, own, red, led);
    CK(cudaMemcpyAsync(h_pinned_out, out_stage_.p, (2 * B + 4 + VQNQS_LEDGER_SLOTS) *
                       sizeof(double), cudaMemcpyDeviceToHost, own));
    CK(cudaStreamSynchronize(own));
    const double* hr = h_pinned_out + 2 * B;
    for (int64_t i = 0; i < B; ++i) {
      const double e = h_pinned_out[i];
      if (!std::isfinite(e)) {
        std::string s;
        for (int j = 0; j < N; ++j) s.push_back(configs[i * N + j] ? '1' : '0');
        throw NumericError("non-finite local energy at configuration " + s);
      }
    }
    if (hr[2] > 0)  // every rank learns of it through the reduced count
      throw NumericError("non-finite local energy on another rank");
    for (int64_t i = 0; i < B; ++i) {
      if (e_re) e_re[i] = h_pinned_out[i];
      if (logpsi) logpsi[i] = h_pinned_out[B + i];
    }
    finish_stats(hr, stats);
    if (ledger7) {
      const int64_t* gl = reinterpret_cast<const int64_t*>(hr + 4);
      for (int i = 0; i < VQNQS_LEDGER_SLOTS; ++i) ledger7[i] += gl[i];
    }
  }
};

Engine::Engine(const vqnqs_model_desc& d, const double* const* params, int n_params, int precision,
               int device)
    : p_(new EngineImpl(d, params, n_params, precision, device)) {}
Engine::~Engine() { delete p_; }
void Engine::set_reuse(bool reuse) { p_->set_reuse(reuse); }
void Engine::set_micro_batch(int samples) { p_->set_micro_batch(samples); }
void Engine::set_code_override(const int16_t* codes, int64_t n) { p_->set_code_override(codes, n); }
void Engine::fill_stats_device(const double* d_e, int64_t B, Comm* comm, void* stream,
                               double* stats) {
  p_->fill_stats_device(d_e, B, comm, stream ? static_cast<cudaStream_t>(stream) : p_->own,
                        stats);
}
void Engine::estimate(const uint8_t* configs, int64_t B, double* e_re, double* logpsi,
                      int64_t* ledger7, Comm* comm, double* stats) {
  p_->estimate(configs, B, e_re, logpsi, ledger7, comm, stats);
}
void Engine::set_hamiltonian(const int32_t* bonds, int nb, int n_sites, bool marshall) {
  p_->set_hamiltonian(bonds, nb, n_sites, marshall);
}
void Engine::run_device(const uint8_t* d_configs, int64_t B, double* d_e, double* d_logpsi,
                        int64_t* ledger7, void* stream, Taps* taps) {
  p_->run_device(d_configs, B, d_e, d_logpsi, ledger7,
                 stream ? static_cast<cudaStream_t>(stream) : p_->own, taps);
}
void Engine::sample(int64_t count, uint64_t seed, uint64_t skip, uint8_t* configs,
                    double* log_probs) {
  if (count < 1) throw ConfigError("sample count must be >= 1");
  p_->sample(count, seed, skip, configs, log_probs);
}
void Engine::run_host(const uint8_t* configs, int64_t B, double* e_re, double* e_im,
                      double* logpsi, int64_t* ledger7, Taps* taps) {
  p_->run_host(configs, B, e_re, e_im, logpsi, ledger7, taps);
}
int64_t Engine::last_launches() const { return p_->launches; }
int Engine::last_profile(double* out, int cap) const {
  for (int i = 0; i < cap && i < 12; ++i) out[i] = p_->prof[i];
  return 12;
}
const vqnqs_model_desc& Engine::desc() const { return p_->c; }

}  // namespace vqb

// Kernel-level test hooks share this translation unit (header-defined kernels).
#include "debug_hooks.cuh"
