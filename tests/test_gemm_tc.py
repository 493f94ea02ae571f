"""The recurrent path's tensor-core GEMM (gemm_tc.cu, C-ABI marl_gemm_f32):
3xTF32 on tcgen05 against an fp64 matmul of the same fp32 operands, for the
three operand layouts the recurrent collector and BPTT update use (row-major
A . B^T, A . B, and the weight-gradient form D^T . X summed over every row,
which splits K across CTAs), ragged M / N / K, N above one 256-column tile,
beta accumulation, and bitwise determinism of the split-K fold.  The bar is
fp32-level accuracy: max |err| <= 2e-6 * (|A| . |B'|^T) elementwise."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(M, N, K, A, sam, sak, B, sbn, sbk, Cm, ldc, beta):
    import torch
    from paper_2311_10090_b200 import _native
    rc = _native.lib().marl_gemm_f32(M, N, K, C.c_void_p(A.data_ptr()), sam, sak, C.c_void_p(B.data_ptr()), sbn, sbk,
                                    C.c_void_p(Cm.data_ptr()), ldc, C.c_float(beta),
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(rc)
    torch.cuda.synchronize()


def _check(got, a64, b64, c0, beta):
    ref = a64 @ b64.T + (beta * c0 if beta else 0.0)
    scale = np.abs(a64) @ np.abs(b64).T + (np.abs(c0) if beta else 0.0) + 1e-30
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= 2e-6 * scale + 1e-30), float((err / scale).max())


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (127, 64, 18), (4096, 384, 64), (5000, 5, 64), (300, 64, 541),
                                   (2049, 384, 128), (129, 16, 7)])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_gemm_nt(M, N, K, beta):
    import torch
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).cuda()
    B = torch.randn(N, K, generator=g).cuda()
    Cm = torch.randn(M, N, generator=g).cuda()
    c0 = Cm.cpu().numpy().astype(np.float64)
    _gemm(M, N, K, A, K, 1, B, K, 1, Cm, N, beta)
    _check(Cm.cpu().numpy(), A.cpu().double().numpy(), B.cpu().double().numpy(), c0, beta)


@pytest.mark.parametrize("M,N,K", [(4096, 64, 5), (1000, 128, 384), (77, 128, 256)])
def test_gemm_nn_strided(M, N, K):
    """C = A . B with B [K x N] row-major and A a column slice of a wider
    buffer (lda > K), as in the BPTT input gradients."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(3)
    Aw = torch.randn(M, K + 13, generator=g).cuda()
    B = torch.randn(K, N, generator=g).cuda()
    Cm = torch.zeros(M, N).cuda()
    _gemm(M, N, K, Aw[:, 5:], K + 13, 1, B, 1, N, Cm, N, 0.0)
    _check(Cm.cpu().numpy(), Aw[:, 5:5 + K].cpu().double().numpy(), B.cpu().double().numpy().T, 0, 0.0)


@pytest.mark.parametrize("O,I,K", [(64, 18, 200_000), (384, 64, 65_536), (128, 128, 131_072), (5, 64, 1000)])
def test_gemm_tn_split_k_deterministic(O, I, K):
    """G[O x I] = D^T . X over K rows (the weight gradients): split K, folded
    in a fixed order -- two runs are bitwise equal."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(O + I)
    D = torch.randn(K, O, generator=g).cuda()
    X = torch.randn(K, I, generator=g).cuda()
    G1 = torch.zeros(O, I).cuda()
    G2 = torch.zeros(O, I).cuda()
    _gemm(O, I, K, D, 1, O, X, 1, I, G1, I, 0.0)
    _gemm(O, I, K, D, 1, O, X, 1, I, G2, I, 0.0)
    assert torch.equal(G1, G2)
    _check(G1.cpu().numpy(), D.cpu().double().numpy().T, X.cpu().double().numpy().T, 0, 0.0)


@pytest.mark.parametrize("O,I,ldx,K", [(128, 543, 544, 100_000), (64, 300, 300, 70_000)])
def test_gemm_tn_split_k_wide_tiles(O, I, ldx, K):
    """The wide update's dW1 = dZ1^T . X shape: a long K split across CTAs
    with 128-column N tiles (several of them, the last ragged) over a padded
    row pitch -- deterministic and within the fp32 bar."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(O + I)
    D = torch.randn(K, O, generator=g).cuda()
    X = torch.randn(K, ldx, generator=g).cuda()
    G1 = torch.zeros(O, I).cuda()
    G2 = torch.zeros(O, I).cuda()
    _gemm(O, I, K, D, 1, O, X, 1, ldx, G1, I, 0.0)
    _gemm(O, I, K, D, 1, O, X, 1, ldx, G2, I, 0.0)
    assert torch.equal(G1, G2)
    _check(G1.cpu().numpy(), D.cpu().double().numpy().T, X[:, :I].cpu().double().numpy().T, 0, 0.0)
