"""Times the tcgen05 GEMM (mpic_test_gemm, fp32-store epilogue) against cuBLAS (torch.matmul)
on the projection shapes of the selective pass. Diagnostic only."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_01960_b200 import _lib

def t_ours(a, w, out, reps=20):
    M, K = a.shape; N = w.shape[0]
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        _lib.check(_lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, 1, out.data_ptr(), s))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, 1, out.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

def t_torch(a, w, reps=20):
    for _ in range(3): a @ w.t()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): a @ w.t()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for M, N, K in [(330, 12288, 4096), (330, 16384, 4096), (330, 4096, 16384), (96, 16384, 4096),
                (512, 16384, 4096), (1024, 16384, 4096), (4096, 4096, 4096), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda")
    to = t_ours(a, w, out); tt = t_torch(a, w)
    fl = 2.0 * M * N * K
    wb = N * K * 2
    print(f"M={M:5d} N={N:5d} K={K:5d}  ours {to*1e3:8.1f} us {fl/to/1e9:7.1f} TF/s {wb/to/1e6:6.0f} GB/s(W)"
          f" | cublas {tt*1e3:8.1f} us {fl/tt/1e9:7.1f} TF/s {wb/tt/1e6:6.0f} GB/s(W)")
