"""Head-parallel decomposition on CPU with world_size 2 (gloo): headpar.prefill_layers with
TorchComm drives a plain-torch fp32 engine (head slices of Wq/Wk/Wv/Wo, FFN on a row slice),
and the logits must equal the same engine run on one rank. This checks the row split, the
padding, the reduce-scatter/all-gather data movement and the last-row owner logic that the
B200 engine (HeadParallelRank) uses with NCCL."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2502_01960_b200 import headpar

L, H, D, V, N_CTX = 2, 4, 8, 61, 40


def weights(seed=3):
    g = torch.Generator().manual_seed(seed)
    h = H * D
    w = {"emb": torch.randn(V, h, generator=g), "lm": torch.randn(V, h, generator=g) / h ** 0.5}
    for l in range(L):
        for nm, shp in (("wq", (h, h)), ("wk", (h, h)), ("wv", (h, h)), ("wo", (h, h)),
                        ("w1", (4 * h, h)), ("w2", (h, 4 * h))):
            w[f"{nm}{l}"] = torch.randn(*shp, generator=g) / shp[1] ** 0.5
    return w


class TorchEngine:
    """fp32 restatement of one rank's share (positions = cache rows, no RoPE)."""

    def __init__(self, rank, world, rows, ids, kv0):
        self.w, self.rank, self.world = weights(), rank, world
        self.rows, self.m = rows, len(rows)
        self.mr, self.m_pad = headpar.row_split(self.m, world)
        h = H * D
        self.hl = H // world
        self.cols = slice(rank * self.hl * D, (rank + 1) * self.hl * D)
        self.k = kv0[0][:, :, self.cols].clone()
        self.v = kv0[1][:, :, self.cols].clone()
        self.x = torch.zeros(self.m_pad, h)
        self.x[:self.m] = self.w["emb"][ids]
        self.xb_all = self.x.clone()
        self.partial = torch.zeros(self.m_pad, h)
        self.reduced = torch.zeros(self.mr, h)

    def attn(self, l):
        w, c, m = self.w, self.cols, self.m
        xb = self.xb_all[:m]
        q, k, v = xb @ w[f"wq{l}"][c].T, xb @ w[f"wk{l}"][c].T, xb @ w[f"wv{l}"][c].T
        self.k[l, self.rows], self.v[l, self.rows] = k, v
        out = torch.zeros(m, self.hl * D)
        for hd in range(self.hl):
            s = slice(hd * D, (hd + 1) * D)
            sc = q[:, s] @ self.k[l][:, s].T / D ** 0.5
            mask = torch.arange(N_CTX)[None, :] > torch.as_tensor(self.rows)[:, None]
            out[:, s] = torch.softmax(sc.masked_fill(mask, float("-inf")), -1) @ self.v[l][:, s]
        self.partial.zero_()
        self.partial[:m] = out @ w[f"wo{l}"][:, c].T

    def ffn(self, l, reduced, row0, rows):
        w = self.w
        x = self.x[row0:row0 + rows]
        x += reduced
        x += torch.nn.functional.gelu(x @ w[f"w1{l}"].T, approximate="tanh") @ w[f"w2{l}"].T
        self.xb_all[row0:row0 + rows] = x

    def logits(self, row):
        return (self.w["lm"] @ self.x[row]).numpy()


def inputs():
    g = torch.Generator().manual_seed(7)
    rows = np.sort(np.random.default_rng(1).choice(N_CTX - 1, 10, replace=False)).tolist() + [N_CTX - 1]
    ids = torch.randint(0, V, (len(rows),), generator=g)
    kv0 = (torch.randn(L, N_CTX, H * D, generator=g), torch.randn(L, N_CTX, H * D, generator=g))
    return rows, ids, kv0


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows, ids, kv0 = inputs()
        eng = TorchEngine(rank, world, rows, ids, kv0)
        res = headpar.prefill_layers(eng, headpar.TorchComm(), L)
        if res is not None:
            out.put(res)
    finally:
        dist.destroy_process_group()


def test_head_parallel_decomposition_gloo():
    rows, ids, kv0 = inputs()

    class Solo:
        rank, world = 0, 1

        def reduce_scatter(self, partial, out):
            out.copy_(partial[:out.shape[0]])

        def all_gather_rows(self, full, mr):
            pass

    ref = headpar.prefill_layers(TorchEngine(0, 1, rows, ids, kv0), Solo(), L)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-4)


def test_row_split():
    assert headpar.row_split(330, 8) == (42, 336)
    assert headpar.row_split(1896, 8) == (237, 1896)
    assert headpar.row_split(5, 4) == (2, 8)
