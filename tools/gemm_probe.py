"""Times the tcgen05 GEMM (mpic_test_gemm, fp32-store epilogue) against cuBLAS (torch.matmul)
on the projection shapes of the selective pass. Diagnostic only."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_01960_b200 import _lib

COLD = os.environ.get("COLD") == "1"
_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if COLD else None


BLOCKED = os.environ.get("BLOCKED") == "1"
PATH = 3 if BLOCKED else 1


def t_ours(a, w, out, reps=20, N=None):
    """Mean device time per launch; with COLD=1 the L2 is flushed (256 MB write) before
    each launch and only the launch itself is timed."""
    M, K = a.shape; N = N or w.shape[0]
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        _lib.check(_lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, PATH, out.data_ptr(), s))
    if COLD:
        tot = 0.0
        for _ in range(reps):
            _flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, PATH, out.data_ptr(), s)
            e1.record(); torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, PATH, out.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

def t_torch(a, w, reps=20):
    for _ in range(3): a @ w.t()
    if COLD:
        tot = 0.0
        for _ in range(reps):
            _flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); a @ w.t(); e1.record(); torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): a @ w.t()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

SHAPES = os.environ.get("SHAPES")
_shapes = [tuple(int(v) for v in x.split("x")) for x in SHAPES.split(",")] if SHAPES else None
for M, N, K in _shapes or [(330, 4096, 4096), (330, 12288, 4096), (330, 16384, 4096), (330, 4096, 16384), (96, 16384, 4096),
                (512, 16384, 4096), (1024, 16384, 4096), (4096, 4096, 4096), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda")
    wb = w.view(N // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous() if BLOCKED else w
    to = t_ours(a, wb, out, N=N); tt = t_torch(a, w)
    fl = 2.0 * M * N * K
    wb = N * K * 2
    print(f"M={M:5d} N={N:5d} K={K:5d}  ours {to*1e3:8.1f} us {fl/to/1e9:7.1f} TF/s {wb/to/1e6:6.0f} GB/s(W)"
          f" | cublas {tt*1e3:8.1f} us {fl/tt/1e9:7.1f} TF/s {wb/tt/1e6:6.0f} GB/s(W)")
