"""Kernel-level numerics on the GPU: tcgen05 GEMM and certified-argmin VQ
against plain PyTorch fp32 references of the same ops (bf16 operands, as the
kernels see them)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _lib():
    from paper_2212_11296_b200 import _native
    L = _native.lib()
    L.vqnqs_debug_gemm_bf16.restype = C.c_int
    L.vqnqs_debug_gemm_bf16.argtypes = [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 6 + \
        [C.c_int, C.c_int]
    L.vqnqs_debug_vq.restype = C.c_int
    L.vqnqs_debug_vq.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_void_p, C.c_int, C.c_void_p]
    return L


def p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 384, 128), (1000, 768, 256),
                                   (77, 1024, 256), (513, 256, 1024), (4096, 2304, 768)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_tc_gemm_matches_torch(M, N, K, epi):
    L = _lib()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(K, N, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    WT = W.t().contiguous()
    bias = torch.randn(N, device="cuda", generator=g) * 0.1
    resid = torch.randn(M, N, device="cuda", generator=g)
    ref = A.float() @ W.float() + bias
    if epi == 1:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if epi == 2:
        ref = resid + ref
    outs = []
    for use_tc in (1, 0):
        out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
        assert L.vqnqs_debug_gemm_bf16(M, N, K, p(A), p(WT), p(W), p(bias), p(out), p(resid),
                                       epi, use_tc) == 0
        outs.append(out.float())
    tc, simt = outs
    tol = 1e-4 if epi == 2 else 1e-2  # bf16 output rounding for epi 0/1
    torch.testing.assert_close(tc, ref, atol=tol * ref.abs().max().item(), rtol=tol)
    torch.testing.assert_close(tc, simt, atol=tol * ref.abs().max().item(), rtol=tol)


@pytest.mark.parametrize("M,d,Q,scale", [(1000, 128, 256, 1 / 128), (513, 256, 512, 1 / 256),
                                         (300, 768, 1024, 1 / 768), (2048, 256, 512, 0.02)])
def test_tc_vq_certified_argmin_equals_fp32_argmin(M, d, Q, scale):
    L = _lib()
    g = torch.Generator(device="cuda").manual_seed(M + d + Q)
    cb = (torch.randn(Q, d, device="cuda", generator=g) * scale).to(torch.bfloat16).float()
    x = torch.randn(M, d, device="cuda", generator=g) * 0.2 + cb[torch.randint(0, Q, (M,),
                                                                              device="cuda",
                                                                              generator=g)]
    # plant exact and near ties
    x[0] = cb[5]
    x[1] = 0.5 * (cb[3] + cb[9])
    codes = []
    resc = torch.zeros(1, dtype=torch.int64, device="cuda")
    for use_tc in (1, 0):
        c = torch.full((M,), -1, dtype=torch.int32, device="cuda")
        assert L.vqnqs_debug_vq(M, d, p(x), p(cb), Q, p(c), use_tc, p(resc)) == 0
        codes.append(c)
    tc, simt = codes
    # exact double distances (the reference's arithmetic on the same fp32 x)
    d2 = ((x.double()[:, None, :] - cb.double()[None, :, :]) ** 2).sum(-1)
    ref = d2.argmin(dim=1).int()
    top2 = d2.topk(2, largest=False).values
    gap = (top2[:, 1] - top2[:, 0]) / top2[:, 0].clamp_min(1e-300)
    # tensor-core path re-scores candidates in double: equals the exact argmin
    assert torch.equal(tc, ref), (tc != ref).nonzero()[:5]
    # the fp32 CUDA-core path may differ only at flagged near-ties
    assert not ((simt != ref) & (gap > 1e-5)).any()
    assert tc[0].item() == 5
    # near-ties are the only rescored rows: a handful per row on average
    assert resc.item() < 4 * M
