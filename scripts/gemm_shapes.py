"""Time marl_gemm_f32 on the wide fp32 update's layer-1 shapes (CUDA events,
default stream): Z1 = X . W1^T and dW1 = dZ1^T . X at ld 522 vs a padded ld."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2311_10090_b200 import _native

L = _native.lib()
M, W, I = int(sys.argv[1]) if len(sys.argv) > 1 else 262144, 64, 522


def run(name, f, reps=20):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:40s} {ms * 1e3:8.1f} us")


p = lambda t: C.c_void_p(t.data_ptr())
for ld in (522, 524, 528):
    X = torch.randn(M, ld, device="cuda")
    W1 = torch.randn(W, ld, device="cuda")
    Z = torch.empty(M, W, device="cuda")
    G = torch.empty(W, ld, device="cuda")
    run(f"Z1  M={M} N=64 K=522 ld={ld}", lambda: L.marl_gemm_f32(M, W, I, p(X), ld, 1, p(W1), ld, 1, p(Z), W, 0.0, None))
    run(f"dW1 64x522 K={M} ld={ld}", lambda: L.marl_gemm_f32(W, I, M, p(Z), 1, W, p(X), 1, ld, p(G), ld, 0.0, None))
    idx = torch.randperm(M, device="cuda", dtype=torch.int32)
    run(f"gather torch ld={ld}", lambda: torch.index_select(X, 0, idx))
    del X
