"""Per-phase device time of one decode step (prefill_extend of one row at the end of a
config-C bf16 cache, 9.4 K context). Diagnostic only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2502_01960_b200 as mp

L, H, D, V, images, k = bench.CONFIGS["C"]
cfg = mp.config(L, H, D, vocab_size=V, image_token_count=images[0], seed=1)
model = mp.Model(cfg, mp.BF16, device=0)
n = 9418
kv = mp.KV(L, n + 8, H, D, mp.BF16, 0)
ws = mp.Workspace(model, 16, n + 8)
for i in range(3):
    mp.prefill_extend(model, ws, [5 + i], n + i, 0, kv)
torch.cuda.synchronize()
mp.profile_enable(True)
mp.profile_collect()
for i in range(3):
    mp.prefill_extend(model, ws, [9 + i], n + 3 + i, 0, kv)
torch.cuda.synchronize()
ph = mp.profile_collect()
mp.profile_enable(False)
print({p: round(v[0] / 3, 4) for p, v in ph.items() if v[1]})
