"""Per-phase device time of one config-C request in fp32 mode (SIMT GEMMs + fp32 attention).
Diagnostic only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2502_01960_b200 as mp

L, H, D, V, images, k = bench.CONFIGS[os.environ.get("CFG", "C")]
h = H * D
cfg = mp.config(L, H, D, vocab_size=V, image_token_count=images[0], seed=1)
model = mp.Model(cfg, mp.F32, device=0)
segs = bench.build_prompt(os.environ.get("CFG", "C"), V, seed=42)
prompt = mp.Prompt.from_segments(segs)
n = prompt.n
m = len(mp.select_tokens(prompt, mp.POLICY_MPIC_K, k))
ws = mp.Workspace(model, m, n)
g = np.random.default_rng(1)
chunks = []
for t in images:
    kv = mp.KV(L, t, H, D, mp.F32, 0)
    r = g.random((t, h), dtype=np.float32) - 0.5
    kv.upload(np.broadcast_to(r, (L, t, h)), np.broadcast_to(r, (L, t, h)))
    chunks.append(kv)
linked = mp.KV(L, n, H, D, mp.F32, 0)
mp.request_prefill(model, ws, prompt, chunks, linked, k=k)
mp.profile_enable(True)
mp.profile_collect()
mp.request_prefill(model, ws, prompt, chunks, linked, k=k)
torch.cuda.synchronize()
ph = mp.profile_collect()
mp.profile_enable(False)
print({p: round(v[0], 3) for p, v in ph.items() if v[1]})
