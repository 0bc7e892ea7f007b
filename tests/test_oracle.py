"""The checker itself: the plain-C oracle (oracle/mpic_oracle.c) against the reference's
own outputs — the committed golden fixtures generated from the unmodified reference build
(oracle/gen_golden.py) and, when oracle/_ref was built here, the live reference library.
Integer outputs bit-exact; float outputs within 1e-5 max-abs (the reference tests' own
tolerance, proj/tests/test_linker.cpp:437-439)."""
import os

import numpy as np
import pytest

import oracle
from oracle import Config, Prompt
from helpers import tiny_config

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def o():
    return oracle.OracleC()


@pytest.fixture(scope="module")
def g():
    return dict(np.load(os.path.join(GOLD, "tiny.npz")))


def load_prompt(g, name):
    p = Prompt(g[f"{name}.kinds"], g[f"{name}.lens"], g[f"{name}.text_ids"], g[f"{name}.hashes"])
    p.chunk_base = [int(x) for x in g[f"{name}.chunk_base"]]
    return p


def test_fingerprint_and_weights_bit_exact(o, g):
    cfg = tiny_config()
    assert o.fingerprint(cfg) == int(g["tiny.fingerprint"][0])
    om = o.model(cfg)
    for w in range(8):
        assert np.array_equal(om.weight(w, 0), g[f"tiny.w{w}.l0"]), w
    assert np.array_equal(om.weight(7, 2), g["tiny.w7.l2"])


def test_image_ids_bit_exact(o, g):
    ids = o.image_ids(tiny_config(), g["tiny.img_hash"].tobytes(), 40)
    assert np.array_equal(ids, g["tiny.img_ids"])


def test_selection_known_answers(o):
    """proj/tests/test_linker.cpp:37-89 known answers."""
    p = oracle.make_prompt([("text", [1, 2, 3]), ("image", bytes(32), 5), ("text", [4, 5])])
    assert o.select(p, 0, 2).tolist() == [0, 1, 2, 3, 4, 8, 9]
    assert o.select(p, 0, 0).tolist() == [0, 1, 2, 8, 9]
    assert o.select(p, 1).tolist() == [0, 1, 2, 8, 9]
    assert len(o.select(p, 0, 99)) == p.n
    assert len(o.select(p, 3)) == 0
    q = oracle.make_prompt([("image", bytes(32), 5), ("image", bytes([1] * 32), 5), ("text", [1])])
    assert o.select(q, 0, 7, True).tolist() == [0, 1, 2, 3, 4, 5, 6, 10]
    for k in range(6):  # nesting
        assert set(o.select(p, 0, k)) <= set(o.select(p, 0, k + 1))


@pytest.mark.parametrize("ci", range(5))
def test_selection_and_flatten_golden(o, g, ci):
    name = f"tiny.c{ci}"
    p = load_prompt(g, name)
    assert np.array_equal(o.flatten(tiny_config(), p), g[f"{name}.flat"])
    for tag, (pol, k, glob) in {"k2": (0, 2, False), "k0": (0, 0, False), "text": (1, 0, False),
                                "all": (2, 0, False), "g7": (0, 7, True),
                                "k99": (0, 99, False)}.items():
        assert np.array_equal(o.select(p, pol, k, glob), g[f"{name}.sel.{tag}"]), tag


def test_prefill_golden(o, g):
    om = o.model(tiny_config())
    k, v, lg = om.prefill(g["tiny.prefill.ids"], 3)
    assert np.abs(k - g["tiny.prefill.k"]).max() < 1e-5
    assert np.abs(v - g["tiny.prefill.v"]).max() < 1e-5
    assert np.abs(lg - g["tiny.prefill.logits"]).max() < 1e-5


@pytest.mark.parametrize("ci", range(5))
@pytest.mark.parametrize("rr", [False, True])
def test_assembly_and_selective_golden(o, g, ci, rr):
    """Chunks in the fixture are the reference's own precomputes, so assembly is checked
    bit-exactly (AsStored and Rerotate), the selective pass within 1e-5."""
    cfg = tiny_config()
    name = f"tiny.c{ci}"
    p = load_prompt(g, name)
    # chunks = rows of the reference's assembled cache at each image's segment offset
    asm_k, asm_v = g[f"{name}.as.asm_k"], g[f"{name}.as.asm_v"]
    for (s, e), kind in zip(p.bounds(), p.kinds):
        if kind == 1:
            p.chunk_k.append(np.ascontiguousarray(asm_k[:, s:e]))
            p.chunk_v.append(np.ascontiguousarray(asm_v[:, s:e]))
    key = f"{name}.{'rr' if rr else 'as'}"
    ok, ov = o.assemble(cfg, p, rr)
    assert np.array_equal(ok, g[f"{key}.asm_k"])
    assert np.array_equal(ov, g[f"{key}.asm_v"])
    om = o.model(cfg)
    for tag in ["k2", "k0", "text", "all", "g7"]:
        if f"{key}.{tag}.logits" not in g:
            continue
        sel = g[f"{name}.sel.{tag}"]
        kk, vv, lg = om.selective(cfg, p, sel, ok, ov)
        assert np.abs(lg - g[f"{key}.{tag}.logits"]).max() < 1e-5, tag
        assert np.abs(kk - g[f"{key}.{tag}.k"]).max() < 1e-5, tag
        assert np.abs(vv - g[f"{key}.{tag}.v"]).max() < 1e-5, tag


@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference(o):
    r = oracle.RefLib()
    rng = np.random.default_rng(5)
    cfg = Config(2, 4, 16, 64, 300, 8, 10000.0, 11)
    assert o.fingerprint(cfg) == r.fingerprint(cfg)
    om, rm = o.model(cfg), r.model(cfg)
    assert all(np.array_equal(om.weight(w, 1 if w > 1 else 0), rm.weight(w, 1 if w > 1 else 0))
               for w in range(8))
    ids = rng.integers(0, cfg.vocab_size, 40).astype(np.int32)
    k1, v1, l1 = om.prefill(ids, 5)
    k2, v2, l2 = rm.prefill(ids, 5)
    assert max(np.abs(k1 - k2).max(), np.abs(v1 - v2).max(), np.abs(l1 - l2).max()) < 1e-5


@pytest.mark.skipif(not os.path.exists(os.path.join(oracle.REF_DIR, "tests", "test_linker")),
                    reason="reference test binaries not built")
@pytest.mark.parametrize("suite", ["test_model", "test_cache", "test_linker", "test_transfer"])
def test_reference_suites_pass_on_reference(suite):
    """The reference's own doctest suites pass on the oracle build (sanity of the shim)."""
    import subprocess
    r = subprocess.run([os.path.join(oracle.REF_DIR, "tests", suite)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("policy,k", [(0, 4), (2, 0)])
def test_fp64_restatement_matches_reference(policy, k):
    """oracle/fp64.py (selective pass in float64, reference_model.h arithmetic) agrees with
    the reference's fp32 selective_prefill to fp32 rounding on a mixed prompt."""
    from oracle.fp64 import selective_prefill_f64
    r = oracle.RefLib()
    cfg = Config(3, 4, 16, 64, 211, 12, 10000.0, 5)
    rm = r.model(cfg)
    rng = np.random.default_rng(policy + 3)
    segs = [("text", rng.integers(0, 210, 7).tolist()), ("image", rng.bytes(32), 12),
            ("text", rng.integers(0, 210, 5).tolist()), ("image", rng.bytes(32), 12),
            ("text", rng.integers(0, 210, 4).tolist())]
    p = oracle.make_prompt(segs)
    for seg in segs:
        if seg[0] == "image":
            kk, vv, _ = rm.prefill(rm.image_ids(seg[1], 12), 0)
            p.chunk_k.append(kk)
            p.chunk_v.append(vv)
            p.chunk_base.append(0)
    sel = rm.select(p, policy, k)
    res = rm.link_and_prefill(p, sel=sel)
    flat = rm.flatten(p)
    lg, kf, vf = selective_prefill_f64(rm.weight, 3, 4, 16, 10000.0, flat[sel], sel, res["asm_k"], res["asm_v"])
    den = np.abs(lg).max()
    assert np.abs(lg - res["logits"]).max() / den < 1e-5
    assert np.abs(kf - res["k"][:, sel]).max() < 1e-5 and np.abs(vf - res["v"][:, sel]).max() < 1e-5
