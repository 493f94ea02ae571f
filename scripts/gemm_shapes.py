"""Time marl_gemm_f32 (3xTF32 tcgen05) on the wide fp32 update's and the
recurrent update's GEMM shapes, beside cuBLAS fp32 SGEMM (torch.matmul, TF32
off) on the same operands.  CUDA events on the default stream, warm L2 only
for operands that fit it.  Usage: python scripts/gemm_shapes.py [M]"""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2311_10090_b200 import _native

L = _native.lib()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
torch.backends.cuda.matmul.allow_tf32 = False


def timeit(f, reps=20):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


p = lambda t: C.c_void_p(t.data_ptr())


def case(name, Mm, N, K, A, sam, sak, B, sbn, sbk, ref):
    Cc = torch.empty(Mm, N, device="cuda")
    us = timeit(lambda: L.marl_gemm_f32(Mm, N, K, p(A), sam, sak, p(B), sbn, sbk, p(Cc), N, 0.0, None))
    ub = timeit(ref)
    gb = 4 * (Mm * K + N * K + Mm * N) / 1e9
    print(f"{name:44s} tc {us:8.1f} us ({gb * 1e6 / us:6.0f} GB/s)   cuBLAS sgemm {ub:8.1f} us")


W, I, ld = 64, 543, 544
X = torch.randn(M, ld, device="cuda")
Xv = X[:, :I]
W1s = torch.randn(2 * W, ld, device="cuda")
case(f"Z1 stacked  {M}x128x543", M, 2 * W, I, X, ld, 1, W1s, ld, 1, lambda: Xv @ W1s[:, :I].t())
D1 = torch.randn(M, 2 * W, device="cuda")
case(f"dW1 stacked 128x543x{M}", 2 * W, I, M, D1, 1, 2 * W, X, 1, ld, lambda: D1.t() @ Xv)
H1 = torch.randn(M, 2 * W, device="cuda")
W2 = torch.randn(W, W, device="cuda")
case(f"Z2 {M}x64x64 (lda 128)", M, W, W, H1, 2 * W, 1, W2, W, 1, lambda: H1[:, :W] @ W2.t())
case(f"dW2 64x64x{M}", W, W, M, D1, 1, 2 * W, H1, 1, 2 * W, lambda: D1[:, :W].t() @ H1[:, :W])
Mr = 24576
E = torch.randn(Mr, 64, device="cuda")
Wx = torch.randn(384, 64, device="cuda")
case(f"rnn gx {Mr}x384x64", Mr, 384, 64, E, 64, 1, Wx, 64, 1, lambda: E @ Wx.t())
Hh = torch.randn(Mr, 128, device="cuda")
Uh = torch.randn(384, 128, device="cuda")
case(f"rnn gh {Mr}x384x128", Mr, 384, 128, Hh, 128, 1, Uh, 128, 1, lambda: Hh @ Uh.t())
Kr = 128 * Mr
Dz = torch.randn(Kr, 512, device="cuda")
Ee = torch.randn(Kr, 64, device="cuda")
case(f"rnn dWx 384x64x{Kr}", 384, 64, Kr, Dz, 1, 512, Ee, 1, 64, lambda: Dz[:, :384].t() @ Ee)
