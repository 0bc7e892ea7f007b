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


def _case(seed=11, L=2, H=8, D=128, V=4096, img=256):
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=img, seed=5)
    rng = np.random.default_rng(seed)
    segs = [("text", rng.integers(0, V - 1, 40).tolist()), ("image", rng.bytes(32), img),
            ("text", rng.integers(0, V - 1, 23).tolist()), ("image", rng.bytes(32), img),
            ("text", rng.integers(0, V - 1, 17).tolist())]
    h = H * D
    chunks_host = [(rng.random((L, img, h), dtype=np.float32) - 0.5,
                    rng.random((L, img, h), dtype=np.float32) - 0.5) for _ in range(2)]
    return cfg, segs, chunks_host


def test_hp_request_in_library_nccl():
    """mpic_hp_request: the whole head-parallel request in C++ with the collectives on a
    library-created NCCL communicator (P = 1: one GPU per gpurun box). It must equal the
    step-by-step Python driver (same kernels, same data movement) bit for bit, stay identical
    when the layer loop is replayed from its CUDA graph, and match the single-GPU request."""
    cfg, segs, chunks_host = _case()
    L, H, D = cfg.n_layers, cfg.n_heads, cfg.head_dim
    prompt = mp.Prompt.from_segments(segs)
    chunks = [mp.KV.from_host(k, v, H, D, mp.BF16) for k, v in chunks_host]
    model = mp.Model(cfg, mp.BF16)
    ws = mp.Workspace(model, 256, prompt.n)
    ref_logits, ref_sel = mp.request_prefill(model, ws, prompt, chunks, mp.KV(L, prompt.n, H, D, mp.BF16), k=32)
    stream = torch.cuda.current_stream().cuda_stream
    e = headpar.HeadParallelRank(cfg, 0, 1, max_rows=256, max_ctx=prompt.n)
    c_py = e.linked_cache(prompt.n)
    e.prepare(prompt, chunks, c_py, mp.POLICY_MPIC_K, 32, stream)
    py_logits = headpar.prefill_local([e], L)
    comm = headpar.NcclComm(0, 1)
    c_lib = e.linked_cache(prompt.n)
    outs = []
    for _ in range(3):  # eager, captured, replayed
        logits, sel = e.request(prompt, chunks, c_lib, k=32, stream=stream, comm=comm)
        assert np.array_equal(sel, ref_sel)
        outs.append(logits)
    for o in outs:
        assert np.array_equal(o, py_logits)
    assert all(np.array_equal(a, b) for a, b in zip(c_lib.download(), c_py.download()))
    assert rel_err(outs[0], ref_logits) < 1e-2
    nc, _ = e.request(prompt, chunks, c_lib, k=32, stream=stream, comm=None)  # P = 1 without NCCL
    assert np.array_equal(nc, py_logits)
    comm.close()
    # the workspace must hold P * ceil(m / P) rows (the all-gather target)
    small = headpar.HeadParallelRank(cfg, 0, 1, max_rows=64, max_ctx=prompt.n)
    with pytest.raises(mp.MpicError):
        small.request(prompt, chunks, small.linked_cache(prompt.n), k=32, stream=stream)


def _hp_worker(rank, world, port, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg, segs, chunks_host = _case()
        L, H, D = cfg.n_layers, cfg.n_heads, cfg.head_dim
        prompt = mp.Prompt.from_segments(segs)
        chunks = [mp.KV.from_host(k, v, H, D, mp.BF16) for k, v in chunks_host]
        e = headpar.HeadParallelRank(cfg, rank, world, max_rows=256, max_ctx=prompt.n)
        cache = e.linked_cache(prompt.n)
        stream = torch.cuda.current_stream().cuda_stream
        e.prepare(prompt, chunks, cache, mp.POLICY_MPIC_K, 32, stream)
        out = headpar.prefill_layers(e, headpar.TorchComm(), L)
        torch.cuda.synchronize()
        q.put((rank, None if out is None else out.tolist(), [a.tolist() for a in cache.download()]))
    finally:
        dist.destroy_process_group()


def test_head_parallel_two_processes():
    """Two processes (ranks 0, 1 of a gloo group sharing the one B200): the B200 engine with
    real inter-process collectives (TorchComm) equals the P = 2 single-process decomposition
    bit for bit and the single-GPU request within the bf16 tolerance."""
    import socket
    import torch.multiprocessing as tmp
    cfg, segs, chunks_host = _case()
    L, H, D = cfg.n_layers, cfg.n_heads, cfg.head_dim
    prompt = mp.Prompt.from_segments(segs)
    chunks = [mp.KV.from_host(k, v, H, D, mp.BF16) for k, v in chunks_host]
    model = mp.Model(cfg, mp.BF16)
    ref_logits, _ = mp.request_prefill(model, mp.Workspace(model, 256, prompt.n), prompt, chunks,
                                       mp.KV(L, prompt.n, H, D, mp.BF16), k=32)
    stream = torch.cuda.current_stream().cuda_stream
    engines = [headpar.HeadParallelRank(cfg, r, 2, max_rows=256, max_ctx=prompt.n) for r in range(2)]
    caches = [e.linked_cache(prompt.n) for e in engines]
    for e, c in zip(engines, caches):
        e.prepare(prompt, chunks, c, mp.POLICY_MPIC_K, 32, stream)
    local = headpar.prefill_local(engines, L)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, logits, cache = q.get(timeout=300)
        res[r] = (logits, cache)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    got = [res[r][0] for r in range(2) if res[r][0] is not None]
    assert len(got) == 1
    got = np.array(got[0], np.float32)
    assert np.array_equal(got, local)
    assert rel_err(got, ref_logits) < 1e-2
    for r in range(2):
        k, v = caches[r].download()
        assert np.array_equal(np.array(res[r][1][0], np.float32), k)
        assert np.array_equal(np.array(res[r][1][1], np.float32), v)
