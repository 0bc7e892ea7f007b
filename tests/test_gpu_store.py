"""The tiered chunk store on the device (mpic_store_*): CacheStore
(proj/include/mpic/cache.h:70-133, proj/src/cache.cpp:203-461) with the Device tier in HBM,
LRU demotion Device -> Host (pinned) -> Disk (.mpic v3) by entry-count budgets, the GPU CRC32
(bit-exact with zlib), and prepare's fault semantics (transfer.cpp:83-145): a miss and an entry
that fails its checks are computed on the device. Every request from the store must give
exactly the outputs of mpic_request_prefill on the same chunks."""
import os
import zlib

import numpy as np
import pytest
import torch

import paper_2502_01960_b200 as mp
from test_gpu_parity import _computed_chunk, _files_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 7, 8, 4095, 32768, 32769, 100003, 3 * 32768])
def test_crc32_device_matches_zlib(n):
    g = np.random.default_rng(n)
    data = g.integers(0, 256, n, dtype=np.uint8)
    buf = torch.from_numpy(data).cuda() if n else torch.zeros(1, dtype=torch.uint8, device="cuda")
    off = 1 if n > 2 else 0  # also an unaligned start
    want = zlib.crc32(data[off:].tobytes())
    assert mp.crc32_device(buf.data_ptr() + off, n - off) == want


@pytest.mark.parametrize("nplanes,plane", [(1, 4096), (3, 32 * 4096), (2, 33 * 4096), (4, 4608 * 4096 // 16)])
def test_crc32_pieces_warp_kernel(nplanes, plane):
    """The files loader's GPU CRC: 128 KB pieces of 4 KB-multiple planes, each folded by one warp
    (GF(2) 'append 4 KB' operator), combined on the host — bit-exact with zlib per plane."""
    from paper_2502_01960_b200 import _lib
    g = np.random.default_rng(plane + nplanes)
    data = g.integers(0, 256, nplanes * plane, dtype=np.uint8)
    buf = torch.from_numpy(data).cuda()
    got = [mp.crc32_planes_device(buf.data_ptr(), plane, nplanes)[i] for i in range(nplanes)]
    want = [zlib.crc32(data[i * plane:(i + 1) * plane].tobytes()) for i in range(nplanes)]
    assert got == want


def _want(m, ws, p, chunks, L, H, D):
    linked = mp.KV(L, p.n, H, D, m.dtype)
    logits, sel = mp.request_prefill(m, ws, p, chunks, linked, k=32)
    return logits, sel, linked.download()


def _got(store, ws, p, L, H, D, dtype):
    linked = mp.KV(L, p.n, H, D, dtype)
    logits, sel, st = store.request(ws, p, linked, k=32)
    return logits, sel, linked.download(), list(st)


def _same(a, b):
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])
    assert all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))


@pytest.mark.parametrize("dtype", [mp.BF16, mp.F32], ids=["bf16", "f32"])
def test_store_tiers_and_lru(tmp_path, dtype):
    """put -> Device; budgets 1/1 demote the least recently used entry to Host, then to a
    .mpic v3 file on disk; a request promotes every chunk back to HBM (GPU-checked) and gives
    the outputs of the device-resident request bit for bit; the file the store wrote is read by
    the disk loader (mpic_request_prefill_files) as LOADED with the same outputs."""
    cfg, m, segs, p, chunks = _files_case(dtype)
    L, H, D = cfg.n_layers, cfg.n_heads, cfg.head_dim
    h0, h1 = segs[1][1], segs[3][1]
    ws = mp.Workspace(m, 128, p.n)
    dev = [mp.KV.from_host(k, v, H, D, dtype) for k, v in chunks]
    want = _want(m, ws, p, dev, L, H, D)

    st = mp.Store(m, str(tmp_path), device_budget=1, host_budget=1)
    st.put(h0, dev[0])
    assert st.tier(h0) == mp.TIER_DEVICE
    st.put(h1, dev[1])  # h0 is the LRU Device entry -> Host
    assert (st.tier(h0), st.tier(h1)) == (mp.TIER_HOST, mp.TIER_DEVICE)
    st.demote(h0, mp.TIER_DISK)
    assert st.tier(h0) == mp.TIER_DISK
    fp = "%016x" % mp.fingerprint(cfg)
    path = os.path.join(str(tmp_path), "", fp, h0.hex() + ".mpic")
    assert os.path.exists(path)
    with open(path, "rb") as f:
        assert int.from_bytes(f.read(8)[4:], "little") == 3

    got = _got(st, ws, p, L, H, D, dtype)
    assert got[3] == [mp.CHUNK_LOADED] * 2
    _same(got, want)
    # after the request (both chunks were promoted to Device) the budgets demote again: the
    # least recently used of the two (h0, fetched first) goes to Host
    assert (st.tier(h0), st.tier(h1)) == (mp.TIER_HOST, mp.TIER_DEVICE)
    got = _got(st, ws, p, L, H, D, dtype)
    _same(got, want)

    # the store's file is a valid .mpic v3 for the disk loader
    lf = mp.KV(L, p.n, H, D, dtype)
    other = os.path.join(str(tmp_path), "c1.mpic")
    mp.write_mpic(other, cfg, h1, *chunks[1], bf16=dtype == mp.BF16)
    logits, sel, status = mp.request_prefill_files(m, ws, p, [path, other], lf, k=32, with_status=True)
    assert list(status) == [mp.CHUNK_LOADED] * 2
    assert np.array_equal(logits, want[0])
    st.close()


def test_store_misses_and_fallbacks(tmp_path):
    """A miss is computed on the device (COMPUTED) and kept in the Device tier; a Disk entry
    whose file was corrupted (a flipped payload byte: caught by the GPU check of the layer
    CRCs after the H2D) or removed is a FALLBACK and computed: the outputs equal the request
    given the computed chunks."""
    cfg, m, segs, p, chunks = _files_case()
    L, H, D = cfg.n_layers, cfg.n_heads, cfg.head_dim
    h0, h1 = segs[1][1], segs[3][1]
    ws = mp.Workspace(m, 128, p.n)
    dev = [mp.KV.from_host(k, v, H, D, mp.BF16) for k, v in chunks]
    comp = [_computed_chunk(m, cfg, h, 160) for h in (h0, h1)]

    st = mp.Store(m, str(tmp_path), device_budget=8, host_budget=8)
    got = _got(st, ws, p, L, H, D, mp.BF16)
    assert got[3] == [mp.CHUNK_COMPUTED] * 2
    _same(got, _want(m, ws, p, comp, L, H, D))
    assert st.tier(h0) == st.tier(h1) == mp.TIER_DEVICE
    got = _got(st, ws, p, L, H, D, mp.BF16)  # now hits
    assert got[3] == [mp.CHUNK_LOADED] * 2
    _same(got, _want(m, ws, p, comp, L, H, D))

    # stored chunks, h0 on disk with one payload byte flipped
    st.put(h0, dev[0])
    st.put(h1, dev[1])
    st.demote(h0, mp.TIER_DISK)
    fp = "%016x" % mp.fingerprint(cfg)
    path = os.path.join(str(tmp_path), "", fp, h0.hex() + ".mpic")
    with open(path, "r+b") as f:
        f.seek(84 + 1000)
        b = f.read(1)
        f.seek(84 + 1000)
        f.write(bytes([b[0] ^ 0x10]))
    got = _got(st, ws, p, L, H, D, mp.BF16)
    assert got[3] == [mp.CHUNK_FALLBACK, mp.CHUNK_LOADED]
    _same(got, _want(m, ws, p, [comp[0], dev[1]], L, H, D))
    assert st.tier(h0) == mp.TIER_DEVICE  # the computed chunk replaced the corrupt entry

    # a Disk entry whose file is gone
    st.put(h0, dev[0])
    st.demote(h0, mp.TIER_DISK)
    os.unlink(path)
    got = _got(st, ws, p, L, H, D, mp.BF16)
    assert got[3] == [mp.CHUNK_FALLBACK, mp.CHUNK_LOADED]
    _same(got, _want(m, ws, p, [comp[0], dev[1]], L, H, D))

    # no disk tier: a Host-tier victim is dropped (a later request computes it)
    st2 = mp.Store(m, None, device_budget=0, host_budget=0)
    st2.put(h0, dev[0])
    assert st2.tier(h0) == -1
    st2.put(h1, dev[1])
    assert st2.tier(h1) == -1
    got = _got(st2, ws, p, L, H, D, mp.BF16)
    assert got[3] == [mp.CHUNK_COMPUTED] * 2
    st.close()
    st2.close()


def test_store_errors(tmp_path):
    cfg, m, segs, p, chunks = _files_case()
    L, H, D = cfg.n_layers, cfg.n_heads, cfg.head_dim
    st = mp.Store(m, str(tmp_path))
    with pytest.raises(mp.MpicError) as e:
        st.demote(segs[1][1], mp.TIER_HOST)
    assert e.value.kind == "not_found_error"
    wrong = mp.KV(L, 100, H, D, mp.BF16)  # token_count 100 for a 160-token image segment
    st.put(segs[1][1], wrong)
    with pytest.raises(mp.MpicError) as e:
        st.request(mp.Workspace(m, 128, p.n), p, mp.KV(L, p.n, H, D, mp.BF16), k=32)
    assert e.value.kind == "link_error"
    st.close()
