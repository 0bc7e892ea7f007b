"""Times the tcgen05 selective attention (mpic_test_attention) on synthetic shapes.
Diagnostic only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01960_b200 import _lib

def run(q, k, v, rows, H, out, reps=10):
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.lib().mpic_test_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.ctypes.data,
                                               q.shape[0], k.shape[0], H, out.data_ptr(), s)
    for _ in range(3): _lib.check(f())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

for name, n, m, H, kind in [("C-layer", 9418, 330, 32, "mpic"),
                            ("148-units", 16384, 128, 148, "tail")]:
    q = torch.randn(m, H * 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(n, H * 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(n, H * 128, device="cuda").to(torch.bfloat16)
    if kind == "mpic":
        segs, rows, at = [], [], 0
        for i in range(4):
            t = 32 + 7 * i; rows += list(range(at, at + t)); at += t
            rows += list(range(at, at + 32)); at += 2304
        rows += list(range(at, at + 32)); rows = np.array(rows, np.uint32)
    else:
        rows = np.arange(n - m, n, dtype=np.uint32)
    out = torch.empty(m, H * 128, device="cuda", dtype=torch.bfloat16)
    us = run(q, k, v, rows, H, out)
    fl = 4.0 * H * 128 * float(np.sum(rows.astype(np.float64) + 1))
    blocks = sum((rows[min(len(rows), t * 128 + 128) - 1] // 128 + 1) for t in range((len(rows) + 127) // 128)) * H
    print(f"{name:18s} n={n:6d} m={m:4d} H={H:3d}: {us:8.1f} us  {fl/us/1e6:7.1f} TFLOP/s  "
          f"{us*148/blocks*1.9e3:7.0f} cycles/block/SM (blocks={blocks})")
