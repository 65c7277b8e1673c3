// Developer probe (not part of the product): per-SM gather throughput of
// 128-byte rows from an L2-resident table into shared memory, by
//   TMA gather4 (cp.async.bulk.tensor ... tile::gather4) from P issuing warps,
//   cp.async 16 B from W warps.
// One CTA per SM, `rows` rows per round, completion waited each round.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2212_11296_b200/csrc scripts/gather_probe.cu -o scripts/_gather_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_common.cuh"
#include "tma.cuh"

using namespace vqb;

constexpr int ROWS = 432;  // one attention item: 128 q + 2 x 152 keys / values

template <int P>
__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap tm, int nrows_tab,
                                                int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  const uint32_t sb = tc::smem_u32(smem);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, P);
    tc::mbar_fence_init();
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  uint32_t ph = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (w < P && tc::elect_one()) {
      const int nops = ROWS / 4;
      const int mine = (nops - w + P - 1) / P;
      tc::mbar_expect_tx(tc::smem_u32(&bar), mine * 512);
      for (int o = w; o < nops; o += P) {
        const int base = (o * 4 * 2654435761u + r * 977) % (nrows_tab - 4);
        tc::tma_gather4(sb + o * 512, &tm, 64 * (r & 3), base, base + 7 % nrows_tab,
                        (base * 3 + 11) % nrows_tab, (base * 5 + 13) % nrows_tab,
                        tc::smem_u32(&bar));
      }
    }
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
  }
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

template <int W>
__global__ void __launch_bounds__(128, 1) k_cpasync(const uint8_t* tab, int nrows_tab, int reps,
                                                    unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sb = tc::smem_u32(smem_raw);
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (tid < 32 * W) {
      for (int e = tid; e < ROWS * 8; e += 32 * W) {
        const int row = e >> 3, c = e & 7;
        const int g = (row * 2654435761u + r * 977) % nrows_tab;
        tc::cp_async16(sb + row * 128 + c * 16, tab + (size_t)g * 1536 + (r & 3) * 128 + c * 16);
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

int main() {
  const int nrows = 1 << 14;  // 16384 rows x 1536 B = 24 MB (L2 resident)
  uint8_t* tab;
  cudaMalloc(&tab, (size_t)nrows * 1536);
  cudaMemset(tab, 1, (size_t)nrows * 1536);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const CUtensorMap tm = make_tmap_bf16(tab, nrows, 768, 1);
  const int smem = ROWS * 128 + 1024, reps = 200;
  auto report = [&](const char* name) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %8.0f cycles per %d rows: %5.1f B/clk/SM\n", name, (double)c / reps, ROWS,
           ROWS * 128.0 * reps / c);
  };
#define TMA(P)                                                                            \
  cudaFuncSetAttribute(k_tma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);     \
  k_tma<P><<<148, 128, smem>>>(tm, nrows, reps, d);                                      \
  report("tma gather4 x" #P);
#define CPA(W)                                                                            \
  cudaFuncSetAttribute(k_cpasync<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  k_cpasync<W><<<148, 128, smem>>>(tab, nrows, reps, d);                                 \
  report("cp.async warps " #W);
  TMA(1) TMA(2) TMA(3) TMA(4) CPA(1) CPA(2) CPA(3) CPA(4)
  return 0;
}
