"""Pair-GEMM timeline with the production epilogues (MPIC_PG_TS=1): device time per launch
inside a CUDA graph of 20 launches, and CTA 0's timeline of the last one — entry -> prologue
done -> MMAs issued -> epilogue done -> exit (us), plus producer / MMA-issuer wait cycles.
Config-C shapes: QKV (bf16 store), Wo and W2 (residual add), W1 (GELU). Diagnostic only."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_01960_b200 import _lib

L = _lib.lib()
M = int(os.environ.get("M", "330"))
for name, N, K, mode in [("qkv", 12288, 4096, 2), ("qkv-rope", 12288, 4096, 3), ("wo", 4096, 4096, 0), ("w1", 16384, 4096, 1),
                         ("w2", 4096, 16384, 0)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(4)]
    x = torch.randn(M, N, device="cuda")
    xb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()

    def launch(w):
        _lib.check(L.mpic_test_gemm_epi(a.data_ptr(), w.data_ptr(), M, N, K, mode, x.data_ptr(), xb.data_ptr(),
                                        out.data_ptr(), s.cuda_stream))
    with torch.cuda.stream(s):
        for w in ws:
            launch(w)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(20):
            launch(ws[i % 4])
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 100 * 1e3
    ts = np.zeros(16, np.uint64)
    _lib.check(L.mpic_pgemm_timestamps(ts.ctypes.data))
    t = (ts[:5].astype(np.int64) - int(ts[0])) / 1e3
    c = ts[5:11].astype(np.int64)
    print(f"{name} M={M} N={N} K={K}: {us:.1f} us/launch in graph | CTA0: prologue {t[1]:.2f} MMAs issued "
          f"{t[2]:.2f} epilogue done {t[3]:.2f} exit {t[4]:.2f} us | producer waits {c[0]}/{c[1]} cyc, "
          f"MMA waits {c[2]}/{c[3]} cyc ({c[3] / max(t[2] - t[1], 1e-3) / 1e3:.2f} GHz) | warp2: acc wait "
          f"{(int(ts[11]) - int(ts[0])) / 1e3:.2f}->{(int(ts[12]) - int(ts[0])) / 1e3:.2f} us, tmem_ld {c[4]} cyc, epi {c[5]} cyc"
          + (f" | split-K: barrier1 {(int(ts[13]) - int(ts[0])) / 1e3:.2f} pushed {(int(ts[14]) - int(ts[0])) / 1e3:.2f} "
             f"barrier2 {(int(ts[15]) - int(ts[0])) / 1e3:.2f} owner: tmem {ts[9]} stage {ts[10]} resid {ts[12]} cyc"
             if mode == 0 else ""))
    del ws
