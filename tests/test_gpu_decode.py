"""Decode after a prefill (decode_step, proj/src/model.cpp:356-367: extend_rows of one row at
the end of the cache) on the B200 path, against the plain-C oracle's prefill of the whole
sequence (oracle/mpic_oracle.c): the cache holds the prompt's K/V (bf16 or fp32), each
decoded token is one mpic_prefill_extend row at position n, n+1, ... In bf16 mode with
head_dim 128 this runs the tcgen05 GEMMs at M = 1 token and the tcgen05 attention with one
query row. Tolerances: 1e-4 (fp32), 1e-2 (bf16) relative on the logits of every decoded
token; the K/V rows the decode appended are checked too."""
import numpy as np
import pytest

import oracle
import paper_2502_01960_b200 as mp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,tol", [(mp.F32, 1e-4), (mp.BF16, 1e-2)], ids=["f32", "bf16"])
@pytest.mark.parametrize("n,steps", [(300, 3), (1100, 2)])
def test_decode_after_prefill(dtype, tol, n, steps):
    L, H, D, V = 2, 4, 128, 4096
    cfg_o = oracle.Config(L, H, D, H * D, V, 64, 10000.0, 3)
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=64, seed=3)
    ids = np.random.default_rng(n).integers(0, V - 1, n + steps).astype(np.int32)
    om = oracle.OracleC().model(cfg_o)
    model = mp.Model(cfg, dtype, device=0)
    ws = mp.Workspace(model, max(n, 16), n + steps)
    kv = mp.KV(L, n + steps, H, D, dtype)
    mp.prefill_extend(model, ws, ids[:n], 0, 0, kv)  # the prompt: rows [0, n)
    for i in range(steps):
        got = mp.prefill_extend(model, ws, ids[n + i:n + i + 1], n + i, 0, kv)  # one decoded token
        ref_k, ref_v, ref = om.prefill(ids[:n + i + 1], 0)
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        assert err < tol, (i, err)
    k, v = kv.download()
    for a, b in ((k, ref_k), (v, ref_v)):
        row = a[:, n:n + steps].astype(np.float64)
        want = b[:, n:n + steps].astype(np.float64)
        assert float(np.abs(row - want).max() / np.abs(want).max()) < tol
