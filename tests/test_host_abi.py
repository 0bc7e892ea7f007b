"""CPU-side checks of the product library: it loads without a GPU, exports every symbol
the C ABI header declares, its host-side integer logic (fingerprint, image ids,
selection, flatten) is bit-exact with the reference's golden outputs, and it refuses to
run the compute path without an sm_100 device (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

import paper_2502_01960_b200 as mp
from paper_2502_01960_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_symbols():
    names = set()
    for hdr in ["include/mpic_b200.h"]:
        txt = open(os.path.join(ROOT, hdr)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(mpic_[a-z0-9_]+)\s*\(", txt))
    return names


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared_symbols()) if not hasattr(L, n)]
    assert not missing, missing
    assert declared_symbols() <= set(_lib.SIGNATURES), "python binding misses a symbol"


def tiny():
    return mp.config(3, 2, 8, vocab_size=101, image_token_count=8, seed=7)


@pytest.fixture(scope="module")
def g():
    return dict(np.load(os.path.join(GOLD, "tiny.npz")))


def test_fingerprint_and_image_ids(g):
    assert mp.fingerprint(tiny()) == int(g["tiny.fingerprint"][0])
    ids = mp.image_token_ids(tiny(), g["tiny.img_hash"].tobytes(), 40)
    assert np.array_equal(ids, g["tiny.img_ids"])


@pytest.mark.parametrize("ci", range(5))
def test_selection_and_flatten_bit_exact(g, ci):
    name = f"tiny.c{ci}"
    p = mp.Prompt(g[f"{name}.kinds"], g[f"{name}.lens"], g[f"{name}.text_ids"], g[f"{name}.hashes"])
    assert np.array_equal(mp.flatten_ids(tiny(), p), g[f"{name}.flat"])
    for tag, (pol, k, glob) in {"k2": (0, 2, False), "k0": (0, 0, False), "text": (1, 0, False),
                                "all": (2, 0, False), "g7": (0, 7, True),
                                "k99": (0, 99, False)}.items():
        assert np.array_equal(mp.select_tokens(p, pol, k, glob), g[f"{name}.sel.{tag}"]), tag


def test_selection_known_answers():
    p = mp.Prompt.from_segments([("text", [1, 2, 3]), ("image", bytes(32), 5), ("text", [4, 5])])
    assert mp.select_tokens(p, mp.POLICY_MPIC_K, 2).tolist() == [0, 1, 2, 3, 4, 8, 9]
    assert mp.select_tokens(p, mp.POLICY_TEXT_ONLY).tolist() == [0, 1, 2, 8, 9]
    assert len(mp.select_tokens(p, mp.POLICY_PREFIX_ONLY)) == 0
    q = mp.Prompt.from_segments([("image", bytes(32), 5), ("image", bytes(32), 5), ("text", [1])])
    assert mp.select_tokens(q, mp.POLICY_MPIC_K, 7, True).tolist() == [0, 1, 2, 3, 4, 5, 6, 10]


def test_error_contract_on_host():
    empty = mp.Prompt.from_segments([("text", [])])
    with pytest.raises(mp.MpicError) as e:
        mp.select_tokens(empty)
    assert e.value.kind == "validation_error"
    bad = mp.config(2, 2, 8, hidden_dim=15)
    assert _lib.lib().mpic_config_validate(C.byref(bad)) == 1  # config_error


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(mp.MpicError) as e:
        mp.Model(tiny())
    assert e.value.kind == "no_device"


def test_nccl_unique_id_without_gpu():
    """The head-parallel plumbing resolves NCCL at run time (dlopen): an id can be created on
    a host without a GPU, and it is MPIC_NCCL_ID_BYTES long and fresh each call."""
    from paper_2502_01960_b200 import headpar
    a, b = headpar.nccl_unique_id(), headpar.nccl_unique_id()
    assert len(a) == 128 and a != b


def test_write_mpic_v3_layer_crcs(tmp_path):
    """.mpic v3 (this library's writer): header, K then V payload, the per-layer CRC table
    (crc_k[L], crc_v[L]), then the CRC32 of everything before it; v1 keeps the reference's
    layout (no table)."""
    import struct
    import zlib
    cfg = mp.config(3, 2, 8, vocab_size=101, image_token_count=5, seed=7)
    rng = np.random.default_rng(1)
    k = rng.random((3, 5, 16), dtype=np.float32)
    v = rng.random((3, 5, 16), dtype=np.float32)
    for bf16, crcs in ((False, True), (True, True), (False, False)):
        path = tmp_path / f"c{int(bf16)}{int(crcs)}.mpic"
        mp.write_mpic(str(path), cfg, bytes(range(32)), k, v, bf16=bf16, layer_crcs=crcs)
        b = path.read_bytes()
        ver = struct.unpack_from("<I", b, 4)[0]
        assert ver == (3 if crcs else (2 if bf16 else 1))
        assert b[24:56] == bytes(range(32))
        assert struct.unpack_from("<I", b, len(b) - 4)[0] == zlib.crc32(b[:-4])
        seg = 5 * 16 * (2 if bf16 else 4)
        if crcs:
            table = struct.unpack_from("<6I", b, len(b) - 4 - 24)
            for i in range(6):
                assert table[i] == zlib.crc32(b[84 + i * seg:84 + (i + 1) * seg])
            assert len(b) == 84 + 6 * seg + 24 + 4
        else:
            assert len(b) == 84 + 6 * seg + 4
