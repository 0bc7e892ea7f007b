"""Shared test fixtures: seeded random prompts whose image chunks are standalone
precomputes made by the oracle (make_image_entry, proj/tests/test_util.h:44-60)."""
from __future__ import annotations

import numpy as np

import oracle
from oracle import Config, make_prompt


def tiny_config(seed: int = 7) -> Config:
    """proj/tests/test_util.h:14-24"""
    return Config(3, 2, 8, 16, 101, 8, 10000.0, seed)


def rand_hash(rng) -> bytes:
    return rng.integers(0, 256, 32, dtype=np.uint8).tobytes()


def build_prompt(o: oracle.OracleC, om: oracle.OracleModel, cfg: Config, layout, rng,
                 bases=None, ns: str = "u"):
    """layout: list of ('t', len) / ('i', len). Image chunks are oracle prefills at base 0
    (or bases[i])."""
    segs, chunks = [], []
    for kind, ln in layout:
        if kind == "t":
            segs.append(("text", rng.integers(0, cfg.vocab_size - 1, ln).tolist()))
        else:
            h = rand_hash(rng)
            segs.append(("image", h, ln))
            chunks.append(h)
    p = make_prompt(segs, ns)
    for i, h in enumerate(chunks):
        base = 0 if bases is None else bases[i]
        ids = o.image_ids(cfg, h, [s for s in segs if s[0] == "image"][i][2])
        k, v, _ = om.prefill(ids, base)
        p.chunk_k.append(k)
        p.chunk_v.append(v)
        p.chunk_base.append(base)
    return p


def random_layout(rng, max_tokens=64, max_text=8, max_img=10):
    """random_mixed_prompt's shape (proj/tests/test_util.h:69-101): 1-4 segments, ends in
    text."""
    layout, budget = [], max_tokens
    for _ in range(int(rng.integers(1, 5))):
        if budget <= 1:
            break
        if rng.integers(0, 2) == 0:
            ln = min(int(rng.integers(1, max_text + 1)), budget - 1)
            layout.append(("t", ln))
        else:
            ln = min(int(rng.integers(1, max_img + 1)), budget - 1)
            layout.append(("i", ln))
        budget -= ln
    layout.append(("t", max(1, min(int(rng.integers(1, max_text + 1)), budget))))
    return layout


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(b).max(), 1e-30)
    return float(np.abs(a - b).max() / den)
