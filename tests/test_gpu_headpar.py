"""Head-parallel request on one B200: P virtual ranks, each with its head
slice of the weights and of the request cache, run layer by layer with the reduce-scatter /
all-gather done in torch (headpar.prefill_local). Their logits and caches must match the
single-GPU request on the same inputs (bf16 tolerance)."""
import numpy as np
import pytest
import torch

import paper_2502_01960_b200 as mp
from paper_2502_01960_b200 import headpar

pytestmark = pytest.mark.gpu


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("world", [2, 4])
def test_head_parallel_matches_single_gpu(world):
    L, H, D, V = 2, 8, 128, 4096
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=256, seed=5)
    rng = np.random.default_rng(world)
    segs = [("text", rng.integers(0, V - 1, 40).tolist()), ("image", rng.bytes(32), 256),
            ("text", rng.integers(0, V - 1, 23).tolist()), ("image", rng.bytes(32), 256),
            ("text", rng.integers(0, V - 1, 17).tolist())]
    prompt = mp.Prompt.from_segments(segs)
    h = H * D
    chunks_host = [(rng.random((L, 256, h), dtype=np.float32) - 0.5,
                    rng.random((L, 256, h), dtype=np.float32) - 0.5) for _ in range(2)]
    # single GPU
    model = mp.Model(cfg, mp.BF16)
    ws = mp.Workspace(model, 256, prompt.n)
    chunks = [mp.KV.from_host(k, v, H, D, mp.BF16) for k, v in chunks_host]
    linked = mp.KV(L, prompt.n, H, D, mp.BF16)
    ref_logits, ref_sel = mp.request_prefill(model, ws, prompt, chunks, linked, k=32)
    ref_k, ref_v = linked.download()
    # P virtual ranks
    stream = torch.cuda.current_stream().cuda_stream
    engines = [headpar.HeadParallelRank(cfg, r, world, max_rows=256, max_ctx=prompt.n) for r in range(world)]
    caches = [e.linked_cache(prompt.n) for e in engines]
    for e, c in zip(engines, caches):
        sel = e.prepare(prompt, chunks, c, mp.POLICY_MPIC_K, 32, stream)
        assert np.array_equal(sel, ref_sel)
    logits = headpar.prefill_local(engines, L)
    assert rel_err(logits, ref_logits) < 1e-2
    # the ranks' head slices of the request cache are the single-GPU cache
    hs = h // world
    for r, c in enumerate(caches):
        k, v = c.download()
        assert rel_err(k, ref_k[:, :, r * hs:(r + 1) * hs]) < 1e-2
        assert rel_err(v, ref_v[:, :, r * hs:(r + 1) * hs]) < 1e-2
