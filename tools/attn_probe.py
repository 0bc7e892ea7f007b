"""Times the tcgen05 selective attention (mpic_test_attention) on synthetic shapes.
Diagnostic only. Cases: the config-C layer (rows of the MPIC-k selection), a steady-state
pair case (every item two 128-row tiles over the same keys) and a single-tile case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_01960_b200 import _lib

def run(q, k, v, rows, H, out, reps=20):
    """Median over 5 batches of `reps` launches, after ~0.5 s of warm-up launches (the SM
    clock ramps up under load; a cold GPU times several times slower)."""
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.lib().mpic_test_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.ctypes.data,
                                               q.shape[0], k.shape[0], H, out.data_ptr(), s)
    _lib.check(f())
    torch.cuda.synchronize()
    import time
    t0 = time.time()
    while time.time() - t0 < 0.5:
        for _ in range(10): f()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = []
    for _ in range(5):
        e0.record()
        for _ in range(reps): f()
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps * 1e3)
    if os.environ.get("MPIC_ATTN_TS"):  # the stamps of every call went to /dev/null: dump one
        os.dup2(_saved_err, 2)
        _lib.check(f()); torch.cuda.synchronize()
        os.dup2(_devnull, 2)
    return float(np.median(res))

_saved_err = os.dup(2)
_devnull = os.open(os.devnull, os.O_WRONLY)
if os.environ.get("MPIC_ATTN_TS"):
    os.dup2(_devnull, 2)

def mpic_rows(imgs=4, T=2304, k=32):
    rows, at = [], 0
    for i in range(imgs):
        t = 32 + 7 * i; rows += list(range(at, at + t)); at += t
        rows += list(range(at, at + k)); at += T
    rows += list(range(at, at + 32)); at += 32
    return np.array(rows, np.uint32), at

cases = sys.argv[1:] or ["C", "pair", "single"]
for name in cases:
    if name == "C":
        rows, n = mpic_rows(); H = 32
    elif name == "E16":
        rows, n = mpic_rows(16); H = 32
    elif name == "pair":
        n, H = 16384, 74; rows = np.arange(n - 256, n, dtype=np.uint32)
    else:
        n, H = 16384, 148; rows = np.arange(n - 128, n, dtype=np.uint32)
    m = len(rows)
    torch.manual_seed(0)
    q = torch.randn(m, H * 128, device="cuda").to(torch.bfloat16)
    kk = torch.randn(n, H * 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(n, H * 128, device="cuda").to(torch.bfloat16)
    out = torch.empty(m, H * 128, device="cuda", dtype=torch.bfloat16)
    us = run(q, kk, v, rows, H, out)
    fl = 4.0 * H * 128 * float(np.sum(rows.astype(np.float64) + 1))
    shift = (-m) % 128
    tiles = (m + 127) // 128
    blocks = 0
    for t in range(tiles):
        last = min(m, 128 * t + 128 - shift) - 1
        blocks += int(rows[last]) // 128 + 1
    blocks *= H
    print(f"{name:8s} n={n:6d} m={m:4d} H={H:3d} cps={os.environ.get('MPIC_ATTN_CHUNKS_PER_SM','3')}: {us:8.1f} us "
          f"{fl/us/1e6:7.1f} TFLOP/s alg, {blocks*4*128**3/us/1e6:7.1f} exec; "
          f"{us*148/blocks*1.9e3:6.0f} cyc per tile-block per SM (tile-blocks={blocks})", flush=True)
    print(f"{name} done", file=sys.stdout, flush=True)
