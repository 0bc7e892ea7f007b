"""Generate tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref, built
from /root/reference/proj/src). Run in the build container:

    python oracle/gen_golden.py

The fixtures pin the plain-C oracle and the B200 path to the reference's own outputs on
seeded inputs; the GPU box never needs /root/reference. TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import Config, make_prompt  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def rand_hash(rng):
    return rng.integers(0, 256, 32, dtype=np.uint8).tobytes()


def random_chunk(seed, L, T, h):
    """Seeded U(-0.5, 0.5) chunk KV, regenerable bit-identically by the tests."""
    g = np.random.default_rng(seed)
    k = (g.random((L, T, h)) - 0.5).astype(np.float32)
    v = (g.random((L, T, h)) - 0.5).astype(np.float32)
    return k, v


def prompt_with_chunks(rm, cfg, layout, rng, bases=None, chunk_seed=None):
    segs, hs = [], []
    for kind, ln in layout:
        if kind == "t":
            segs.append(("text", rng.integers(0, cfg.vocab_size - 1, ln).tolist()))
        else:
            h = rand_hash(rng)
            segs.append(("image", h, ln))
            hs.append((h, ln))
    p = make_prompt(segs, "u")
    for i, (h, ln) in enumerate(hs):
        base = 0 if bases is None else bases[i]
        if chunk_seed is None:
            k, v, _ = rm.prefill(rm.image_ids(h, ln), base)
        else:
            k, v = random_chunk(chunk_seed + i, cfg.n_layers, ln, cfg.hidden_dim)
        p.chunk_k.append(k)
        p.chunk_v.append(v)
        p.chunk_base.append(base)
    return p


def dump_case(rm, cfg, p, name, policies, rerotate_too=True, full=True):
    d = {}
    d[f"{name}.kinds"] = p.kinds
    d[f"{name}.lens"] = p.lens
    d[f"{name}.text_ids"] = p.text_ids
    d[f"{name}.hashes"] = p.hashes
    d[f"{name}.chunk_base"] = np.array(p.chunk_base, np.uint32)
    d[f"{name}.flat"] = rm.flatten(p)
    for tag, (pol, k, g) in policies.items():
        sel = rm.select(p, pol, k, g)
        d[f"{name}.sel.{tag}"] = sel
    for rr in ([False, True] if rerotate_too else [False]):
        for tag, (pol, k, g) in policies.items():
            sel = d[f"{name}.sel.{tag}"]
            if len(sel) == 0 or sel[-1] != p.n - 1:
                continue
            res = rm.link_and_prefill(p, sel=sel, rerotate=rr)
            key = f"{name}.{'rr' if rr else 'as'}.{tag}"
            d[f"{key}.logits"] = res["logits"]
            d[f"{key}.slots"] = res["slots"]
            if full:
                d[f"{key}.k"] = res["k"]
                d[f"{key}.v"] = res["v"]
            else:
                d[f"{key}.k_sha"] = np.frombuffer(hashlib.sha256(res["k"].tobytes()).digest(),
                                                  np.uint8)
                # last 8 recomputed rows of the last layer, for tolerance checks
                d[f"{key}.k_last_sel"] = res["k"][-1][sel[-8:]]
                d[f"{key}.v_last_sel"] = res["v"][-1][sel[-8:]]
        asm = rm.link_and_prefill(p, sel=None, rerotate=rr)
        key = f"{name}.{'rr' if rr else 'as'}"
        d[f"{key}.asm_sha_k"] = np.frombuffer(hashlib.sha256(asm["asm_k"].tobytes()).digest(),
                                              np.uint8)
        d[f"{key}.asm_sha_v"] = np.frombuffer(hashlib.sha256(asm["asm_v"].tobytes()).digest(),
                                              np.uint8)
        if full:
            d[f"{key}.asm_k"] = asm["asm_k"]
            d[f"{key}.asm_v"] = asm["asm_v"]
    return d


def main():
    os.makedirs(OUT, exist_ok=True)
    r = oracle.RefLib()
    policies = {"k2": (0, 2, False), "k0": (0, 0, False), "text": (1, 0, False),
                "all": (2, 0, False), "g7": (0, 7, True), "k99": (0, 99, False)}

    # tiny: proj/tests/test_util.h:14-24 shape, full tensors.
    cfg = Config(3, 2, 8, 16, 101, 8, 10000.0, 7)
    rm = r.model(cfg)
    rng = np.random.default_rng(2025)
    d = {"tiny.cfg": np.array([3, 2, 8, 16, 101, 8, 7], np.uint64),
         "tiny.fingerprint": np.array([r.fingerprint(cfg)], np.uint64),
         "tiny.checksum": np.array([rm.checksum()], np.uint64)}
    for w in range(8):
        d[f"tiny.w{w}.l0"] = rm.weight(w, 0).copy()
    d["tiny.w7.l2"] = rm.weight(7, 2).copy()
    h = rand_hash(rng)
    d["tiny.img_hash"] = np.frombuffer(h, np.uint8)
    d["tiny.img_ids"] = rm.image_ids(h, 40)
    ids = rng.integers(0, cfg.vocab_size, 24).astype(np.int32)
    k, v, lg = rm.prefill(ids, 3)
    d.update({"tiny.prefill.ids": ids, "tiny.prefill.k": k, "tiny.prefill.v": v,
              "tiny.prefill.logits": lg})
    layouts = [[("t", 3), ("i", 5), ("t", 2)],
               [("i", 7), ("t", 5)],
               [("t", 4), ("i", 6), ("t", 3), ("i", 9), ("t", 2)],
               [("i", 5), ("i", 5), ("t", 1)],
               [("t", 12)]]
    for ci, lay in enumerate(layouts):
        bases = [3 * j for j in range(sum(1 for x in lay if x[0] == "i"))] if ci == 2 else None
        p = prompt_with_chunks(rm, cfg, lay, rng, bases)
        d.update(dump_case(rm, cfg, p, f"tiny.c{ci}", policies))
    np.savez_compressed(os.path.join(OUT, "tiny.npz"), **d)

    # config A shape at reduced image length: L2 H8 D64 V4096, 2 images of
    # 96 tokens interleaved with text, k=32. Large tensors stored as digests + slices.
    cfg = Config(2, 8, 64, 512, 4096, 96, 10000.0, 1)
    rm = r.model(cfg)
    rng = np.random.default_rng(42)
    lay = [("t", 32), ("i", 96), ("t", 39), ("i", 96), ("t", 32)]
    p = prompt_with_chunks(rm, cfg, lay, rng, chunk_seed=1000)
    d = {"a.cfg": np.array([2, 8, 64, 512, 4096, 96, 1], np.uint64),
         "a.chunk_seed": np.array([1000], np.uint64)}
    d.update(dump_case(rm, cfg, p, "a", {"k32": (0, 32, False), "all": (2, 0, False)},
                       full=False))
    np.savez_compressed(os.path.join(OUT, "config_a96.npz"), **d)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
