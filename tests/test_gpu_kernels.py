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


# (20000, 1024, 256): several row tiles per CTA of the W-stationary kernel (K <= 256, N % 256 == 0);
# N = 384 and K >= 768 take the streaming kernel
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 384, 128), (1000, 768, 256),
                                   (77, 1024, 256), (513, 256, 1024), (4096, 2304, 768),
                                   (20000, 1024, 256)])
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


def _attention_layout(rng, S, T, nb, nh, d, dense=False):
    """A random location layout like k_connected's: per sample a base row
    (all T positions) and K_s - 1 connected rows active from a_k = t1 + 1,
    laid out in a random row order; random unique-row ids I per location."""
    R1 = nb + 1
    K = np.zeros(S, np.int32)
    t1 = np.full(S * R1, -1, np.int32)
    perm = np.zeros(S * R1, np.int32)
    aoff = np.zeros(S * R1, np.int64)
    act_off = np.zeros(S, np.int64)
    Uoff = np.zeros(S, np.int64)
    I, M, U = [], 0, 0
    for s in range(S):
        Ks = int(rng.integers(2, R1 + 1))
        K[s] = Ks
        b = s * R1
        t1[b + 1:b + Ks] = -1 if dense else rng.integers(-1, T - 1, Ks - 1)
        order = np.concatenate([[0], 1 + rng.permutation(Ks - 1)])
        perm[b:b + Ks] = order
        off = 0
        for k in order:
            aoff[b + k] = off
            off += T if k == 0 else T - (t1[b + k] + 1)
        act_off[s] = M
        Us = max(T, off // 3)
        Uoff[s] = U
        ids = rng.integers(0, Us, off).astype(np.int32)
        ids[:T] = rng.permutation(Us)[:T] if Us >= T else np.arange(T)
        I.append(ids)
        M += off
        U += Us
    return dict(S=S, R1=R1, K=K, t1=t1, perm=perm, aoff=aoff, act_off=act_off, Uoff=Uoff,
                I=np.concatenate(I), M=M, U=U)


def _attention_reference(lay, qkv, T, d, nh):
    """softmax(q k^T / sqrt(dh), causal) v per (location, head) in float64 from
    the bf16 q/k/v the kernel reads, with P rounded to bf16 before the value
    product (the kernel's P operand), proj/src/tensor.cpp:199-231 over the
    gathered keys of proj/src/dedup.cpp:31-37,128-134."""
    dh = d // nh
    out = np.zeros((lay["M"], d))
    mag = np.zeros((lay["M"], d))  # sum_t P_t |v_t|: the element's error scale
    scale = 1.0 / np.sqrt(dh)
    for s in range(lay["S"]):
        b = s * lay["R1"]
        base = lay["act_off"][s]
        for k in range(lay["K"][s]):
            a = 0 if k == 0 else lay["t1"][b + k] + 1
            rloc = base + lay["aoff"][b + k]
            keys = np.array([base + t if t < a else rloc + (t - a) for t in range(T)])
            rows = lay["Uoff"][s] + lay["I"][keys]
            for p in range(a, T):
                loc = rloc + (p - a)
                q = qkv[lay["Uoff"][s] + lay["I"][loc]]
                for h in range(nh):
                    sl = slice(h * dh, (h + 1) * dh)
                    kk = qkv[rows[:p + 1], d + h * dh:d + (h + 1) * dh]
                    vv = qkv[rows[:p + 1], 2 * d + h * dh:2 * d + (h + 1) * dh]
                    sc = (kk @ q[sl]) * scale
                    e = np.exp(sc - sc.max())
                    P = torch.tensor(e / e.sum(), dtype=torch.float32).to(torch.bfloat16)
                    out[loc, sl] = P.double().numpy() @ vv
                    mag[loc, sl] = P.double().numpy() @ np.abs(vv)
    return out, mag


@pytest.mark.parametrize("T,d,nh,nb,S,dense", [(50, 128, 8, 20, 3, False),
                                               (128, 256, 8, 24, 2, False),
                                               (72, 128, 4, 12, 3, False),
                                               (18, 64, 4, 9, 4, False),
                                               (128, 256, 8, 6, 2, True)])
def test_tc_attention_matches_gathered_reference(T, d, nh, nb, S, dense):
    """k_tc_attention (the dominant kernel) on its own, against a float64
    gathered causal attention of the same bf16 operands: rows with base/own
    key splits at every first-changed-token position, several rows per tile,
    shared unique rows, and (dense) rows with no base keys."""
    L = _lib()
    L.vqnqs_debug_tc_attention.restype = C.c_int
    L.vqnqs_debug_tc_attention.argtypes = [C.c_int] * 5 + [C.c_void_p] * 5 + [C.c_int64] + \
        [C.c_void_p] * 7
    rng = np.random.default_rng(T * 1000 + d + nb)
    lay = _attention_layout(rng, S, T, nb, nh, d, dense)
    qkv = rng.standard_normal((lay["U"], 3 * d)).astype(np.float32)
    qkv[rng.random(lay["U"]) < 0.1, :d] *= 6.0  # peaked softmax rows
    qkv_b = torch.tensor(qkv).to(torch.bfloat16)
    ref, mag = _attention_reference(lay, qkv_b.double().numpy(), T, d, nh)
    dev = {k: torch.tensor(v).cuda() for k, v in lay.items() if isinstance(v, np.ndarray)}
    qd = qkv_b.cuda()
    M = lay["M"]
    xh = torch.zeros(M, d, dtype=torch.bfloat16, device="cuda")
    xl = torch.zeros_like(xh)
    xn2 = torch.zeros(M, device="cuda")
    rr2 = torch.zeros(M, device="cuda")
    assert L.vqnqs_debug_tc_attention(S, lay["R1"], T, d, nh, p(dev["K"]), p(dev["t1"]),
                                      p(dev["perm"]), p(dev["aoff"]), p(dev["act_off"]), M,
                                      p(dev["I"]), p(dev["Uoff"]), p(qd), p(xh), p(xl),
                                      p(xn2), p(rr2)) == 0
    x = (xh.float() + xl.float()).double().cpu().numpy()
    # error relative to sum_t P_t |v_t| of the element: P is rounded to bf16
    # on both sides, so only a P value within fp32 accumulation error of a
    # bf16 rounding boundary may differ (by 2^-8 of one term)
    rel = np.abs(x - ref) / mag
    print(f"\nT={T} d={d} M={M}: max rel {rel.max():.2e} mean {rel.mean():.2e} "
          f"frac>1e-5 {(rel > 1e-5).mean():.4f}")
    assert rel.max() < 1e-2        # a few bf16 P flips at most (2^-8 of a term each)
    assert rel.mean() < 2e-5       # a systematic 1e-3 error would fail here
    assert (rel > 1e-4).mean() < 0.01
    np.testing.assert_allclose(xn2.double().cpu().numpy(), (x ** 2).sum(1), rtol=2e-5)
