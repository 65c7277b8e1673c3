"""Developer timing probe: the tcgen05 per-location GEMM (debug entry point)
vs torch.matmul (cuBLAS) at the workloads' shapes."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2212_11296_b200 import _native  # noqa: E402

L = _native.lib()
L.vqnqs_debug_gemm_bf16.restype = C.c_int
L.vqnqs_debug_gemm_bf16.argtypes = [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 6 + [C.c_int] * 2
p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
for (M, N, K, epi) in [(500000, 768, 256, 0), (500000, 1024, 256, 1), (500000, 256, 1024, 2),
                       (200000, 2304, 768, 0), (200000, 3072, 768, 1), (200000, 768, 3072, 2)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(K, N, device="cuda") * 0.05).to(torch.bfloat16)
    WT = W.t().contiguous()
    bias = torch.zeros(N, device="cuda")
    resid = torch.zeros(M, N, device="cuda") if epi == 2 else None
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    for _ in range(2):
        L.vqnqs_debug_gemm_bf16(M, N, K, p(A), p(WT), p(W), p(bias), p(out), p(resid), epi, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        L.vqnqs_debug_gemm_bf16(M, N, K, p(A), p(WT), p(W), p(bias), p(out), p(resid), epi, 1)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 5
    for _ in range(2):
        torch.matmul(A, W)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        torch.matmul(A, W)
    torch.cuda.synchronize()
    tb = (time.perf_counter() - t0) / 5
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} epi={epi}: ours {t*1e3:.2f} ms {fl/t/1e12:.0f} TF/s | "
          f"cuBLAS {tb*1e3:.2f} ms {fl/tb/1e12:.0f} TF/s", flush=True)
