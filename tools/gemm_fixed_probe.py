"""Device time of pair-GEMM launches inside a CUDA graph (no host launch overhead):
20 back-to-back launches per shape, config-C projection shapes plus tiny-K shapes that
expose the fixed cost. Diagnostic only; sweep the MPIC_PG_* environment knobs around it."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_01960_b200 import _lib

SHAPES = [(330, 12288, 4096), (330, 4096, 4096), (330, 16384, 4096), (330, 4096, 16384), (330, 16384, 128)]
if os.environ.get("SHAPES"):
    SHAPES = [tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(",")]
# a buffer larger than L2 rotated between launches would flush it; instead every launch of
# the graph reads its own copy of W so the weight stream comes from HBM as in a prefill
NW = 4
res = []
for M, N, K in SHAPES:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(NW)]
    out = torch.empty(M, N, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for w in ws:
            _lib.check(_lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, 1, out.data_ptr(), s.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(20):
            _lib.lib().mpic_test_gemm(a.data_ptr(), ws[i % NW].data_ptr(), M, N, K, 1, out.data_ptr(), s.cuda_stream)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 100 * 1e3
    gbs = N * K * 2 / us / 1e3
    res.append(f"{N}x{K}:{us:.1f}us({gbs:.0f}GB/s)")
    del ws
print(os.environ.get("TAG", ""), " ".join(res))
