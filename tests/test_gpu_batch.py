"""Batched varlen requests (mpic_request_prefill_batch): several MPIC-k requests in one
selective pass over one concatenated cache, each checked against the plain-C oracle run on
that request alone (bf16 bar: max rel <= 1e-2)."""
import numpy as np
import pytest

import oracle
from helpers import rand_hash, rel_err

pytestmark = pytest.mark.gpu

mp = pytest.importorskip("paper_2502_01960_b200")


def _requests(rng, L, H, D, V, layouts):
    reqs = []
    for layout in layouts:
        segs, ck, cv = [], [], []
        for kind, ln in layout:
            if kind == "t":
                segs.append(("text", rng.integers(0, V - 1, ln).tolist()))
            else:
                segs.append(("image", rand_hash(rng), ln))
                ck.append(rng.random((L, ln, H * D), dtype=np.float32) - 0.5)
                cv.append(rng.random((L, ln, H * D), dtype=np.float32) - 0.5)
        reqs.append((segs, ck, cv))
    return reqs


@pytest.mark.parametrize("layouts", [
    [[("t", 20), ("i", 300), ("t", 40)], [("t", 7), ("i", 200), ("t", 30), ("i", 250), ("t", 9)],
     [("t", 150)], [("t", 33), ("i", 520), ("t", 12)]],
    [[("t", 64), ("i", 700), ("t", 64), ("i", 700), ("t", 32)]] * 3,
])
def test_batch_matches_oracle_per_request(layouts):
    L, H, D, V, k = 2, 4, 128, 4096, 32
    cfg_o = oracle.Config(L, H, D, H * D, V, 64, 10000.0, 3)
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=64, seed=3)
    o = oracle.OracleC()
    om = o.model(cfg_o)
    rng = np.random.default_rng(len(layouts))
    reqs = _requests(rng, L, H, D, V, layouts)
    refs = []
    for segs, ck, cv in reqs:
        po = oracle.make_prompt(segs)
        po.chunk_k.extend(ck)
        po.chunk_v.extend(cv)
        po.chunk_base.extend([0] * len(ck))
        sel = o.select(po, 0, k)  # MPIC-k
        ak, av = o.assemble(cfg_o, po, False)
        rk, rv, lg = om.selective(cfg_o, po, sel, ak, av)
        refs.append((sel, ak, rk, rv, lg))

    m = mp.Model(cfg, mp.BF16)
    prompts = [mp.Prompt.from_segments(segs) for segs, _, _ in reqs]
    ns = [p.n for p in prompts]
    ws = mp.Workspace(m, sum(len(r[0]) for r in refs), sum(ns))
    chunks = [[mp.KV.from_host(a, b, H, D, mp.BF16) for a, b in zip(ck, cv)] for _, ck, cv in reqs]
    linked = mp.KV(L, sum(ns), H, D, mp.BF16)
    logits, mrows = mp.request_prefill_batch(m, ws, prompts, chunks, linked, k=k)
    kb, vb = linked.download()
    off = 0
    for r, (sel, ak, rk, rv, lg) in enumerate(refs):
        assert mrows[r] == len(sel)
        assert rel_err(logits[r], lg) < 1e-2, (r, rel_err(logits[r], lg))
        rows = off + np.asarray(sel, np.int64)
        assert rel_err(kb[-1][rows], rk[-1][sel]) < 1e-2
        assert rel_err(vb[-1][rows], rv[-1][sel]) < 1e-2
        img = np.setdiff1d(np.arange(ns[r]), sel)  # assembled (reused) rows: the chunks in bf16
        if img.size:
            assert rel_err(kb[0][off + img], ak[0][img]) < 1e-2
        off += ns[r]


def test_batch_of_one_equals_single_request():
    L, H, D, V = 2, 2, 128, 512
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=64, seed=5)
    rng = np.random.default_rng(5)
    (segs, ck, cv), = _requests(rng, L, H, D, V, [[("t", 40), ("i", 333), ("t", 20)]])
    m = mp.Model(cfg, mp.BF16)
    p = mp.Prompt.from_segments(segs)
    ws = mp.Workspace(m, p.n, p.n)
    chunks = [mp.KV.from_host(a, b, H, D, mp.BF16) for a, b in zip(ck, cv)]
    l1 = mp.KV(L, p.n, H, D, mp.BF16)
    single, sel = mp.request_prefill(m, ws, p, chunks, l1, k=32)
    l2 = mp.KV(L, p.n, H, D, mp.BF16)
    batch, mrows = mp.request_prefill_batch(m, ws, [p], [chunks], l2, k=32)
    assert mrows[0] == len(sel)
    assert rel_err(batch[0], single) < 1e-3


@pytest.mark.parametrize("reposition", [mp.AS_STORED, mp.REROTATE])
def test_batch_matches_single_requests(reposition):
    """Each request of a batch against the same request run alone on the GPU (Rerotate too:
    a chunk's rotation delta stays relative to its own request)."""
    L, H, D, V = 2, 2, 128, 1024
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=64, seed=9)
    rng = np.random.default_rng(9)
    reqs = _requests(rng, L, H, D, V, [[("t", 12), ("i", 180), ("t", 5), ("i", 90), ("t", 7)],
                                       [("t", 40)], [("t", 3), ("i", 257), ("t", 30)]])
    m = mp.Model(cfg, mp.BF16)
    prompts = [mp.Prompt.from_segments(segs) for segs, _, _ in reqs]
    ns = [p.n for p in prompts]
    ws = mp.Workspace(m, sum(ns), sum(ns))
    chunks = [[mp.KV.from_host(a, b, H, D, mp.BF16) for a, b in zip(ck, cv)] for _, ck, cv in reqs]
    big = mp.KV(L, sum(ns), H, D, mp.BF16)
    logits, mrows = mp.request_prefill_batch(m, ws, prompts, chunks, big, k=16, reposition=reposition)
    kb, vb = big.download()
    off = 0
    for r, p in enumerate(prompts):
        one = mp.KV(L, p.n, H, D, mp.BF16)
        lg, sel = mp.request_prefill(m, ws, p, chunks[r], one, k=16, reposition=reposition)
        k1, v1 = one.download()
        assert mrows[r] == len(sel)
        # same kernels, different GEMM tilings (sum(m) rows vs m): bf16 rounding flips only
        assert rel_err(logits[r], lg) < 1e-2, (r, rel_err(logits[r], lg))
        assert rel_err(kb[:, off:off + p.n], k1) < 1e-2
        assert rel_err(vb[:, off:off + p.n], v1) < 1e-2
        off += p.n


def test_batch_more_chunks_than_one_assembly_launch():
    """A batch whose requests carry more image chunks (300) than one assembly launch stages
    (256 descriptors): the assembly runs in descriptor groups, and every request still matches
    the same request run alone (assembled rows exactly, logits within bf16 rounding)."""
    L, H, D, V = 1, 2, 128, 512
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=16, seed=11)
    rng = np.random.default_rng(11)
    layouts = [[("t", 3), ("i", 16), ("t", 2), ("i", 16), ("t", 4)]] * 150
    reqs = _requests(rng, L, H, D, V, layouts)
    m = mp.Model(cfg, mp.BF16)
    prompts = [mp.Prompt.from_segments(segs) for segs, _, _ in reqs]
    ns = [p.n for p in prompts]
    ws = mp.Workspace(m, sum(ns), sum(ns))
    chunks = [[mp.KV.from_host(a, b, H, D, mp.BF16) for a, b in zip(ck, cv)] for _, ck, cv in reqs]
    assert sum(len(c) for c in chunks) == 300
    big = mp.KV(L, sum(ns), H, D, mp.BF16)
    logits, mrows = mp.request_prefill_batch(m, ws, prompts, chunks, big, k=4)
    kb, _ = big.download()
    off = 0
    for r in (0, 77, 127, 128, 149):  # requests on both sides of the 256-descriptor boundary
        p = prompts[r]
        one = mp.KV(L, p.n, H, D, mp.BF16)
        lg, sel = mp.request_prefill(m, ws, p, chunks[r], one, k=4)
        k1, _ = one.download()
        o = sum(ns[:r])
        assert mrows[r] == len(sel)
        img = np.setdiff1d(np.arange(p.n), sel)
        assert np.array_equal(kb[:, o + img], k1[:, img])
        assert rel_err(logits[r], lg) < 1e-2, (r, rel_err(logits[r], lg))
