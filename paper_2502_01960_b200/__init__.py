"""B200-native MPIC partial-reuse prefill (arxiv 2502.01960) — Python host binding.

The product is the native library ``lib/libmpic_b200.so`` (sm_100a CUDA kernels + the C
ABI declared in ``include/mpic_b200.h`` + the C++ ``mpic::`` host API declared in
``include/mpic/*.h``). This module is a thin ctypes mirror of the reference's public
interface (``proj/include/mpic/*.h``) for Python callers, tests and the bench: same
names, argument meaning and error classes. Every call goes to the native library; if it
is missing the call raises ``ExtensionMissing`` (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._lib import (ChunkRef, ExtensionMissing, ModelConfig, MpicError, PolicyDesc, PromptDesc,
                   check, lib)

__all__ = ["ModelConfig", "Model", "KV", "Workspace", "Prompt", "MpicError", "ExtensionMissing", "Store",
           "F32", "BF16", "AS_STORED", "REROTATE", "POLICY_MPIC_K", "POLICY_TEXT_ONLY",
           "POLICY_ALL", "POLICY_PREFIX_ONLY", "config", "fingerprint", "image_token_ids",
           "select_tokens", "flatten_ids", "assemble", "selective_prefill", "prefill_extend",
           "request_prefill", "request_prefill_host", "last_launch_count", "HostBuffer", "to_bf16_bits", "request_prefill_files", "write_mpic",
           "CHUNK_LOADED", "CHUNK_COMPUTED", "CHUNK_FALLBACK"]

F32, BF16 = 0, 1
AS_STORED, REROTATE = 0, 1
POLICY_MPIC_K, POLICY_TEXT_ONLY, POLICY_ALL, POLICY_PREFIX_ONLY = 0, 1, 2, 3


def config(n_layers=2, n_heads=2, head_dim=8, hidden_dim=None, vocab_size=256,
           image_token_count=16, rope_base=10000.0, seed=0) -> ModelConfig:
    """mpic::ModelConfig with the reference's defaults (config.h:7-15)."""
    if hidden_dim is None:
        hidden_dim = n_heads * head_dim
    return ModelConfig(n_layers, n_heads, head_dim, hidden_dim, vocab_size, image_token_count,
                       rope_base, seed)


def fingerprint(cfg: ModelConfig) -> int:
    return int(lib().mpic_config_fingerprint(C.byref(cfg)))


def last_launch_count() -> int:
    """Kernels launched by the last library call on this thread."""
    return int(lib().mpic_last_launch_count())


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(getattr(stream, "cuda_stream", stream))


class Model:
    """Device-resident model: build_model (model.cpp:103-123) synthesised on the GPU."""

    def __init__(self, cfg: ModelConfig, dtype: int = F32, device: int = 0, weights=None):
        self.cfg, self.dtype, self.device = cfg, dtype, device
        h = C.c_void_p()
        if weights is None:
            check(lib().mpic_model_create(C.byref(cfg), device, dtype, C.byref(h)))
        else:
            emb, lm, layers = weights
            self._keep = [np.ascontiguousarray(a, np.float32) for a in [emb, lm] + list(layers)]
            ptrs = (C.c_void_p * len(layers))(*[a.ctypes.data for a in self._keep[2:]])
            check(lib().mpic_model_upload(C.byref(cfg), device, dtype, self._keep[0].ctypes.data,
                                          self._keep[1].ctypes.data, ptrs, C.byref(h)))
        self.handle = h.value

    def close(self):
        if getattr(self, "handle", None):
            try:
                lib().mpic_model_destroy(self.handle)
            except Exception:  # interpreter shutdown: module globals may be gone
                pass
            self.handle = None

    __del__ = close

    def weight(self, which: int, layer: int = 0) -> np.ndarray:
        c = self.cfg
        h = c.hidden_dim
        shape = {0: (c.vocab_size, h), 1: (c.vocab_size, h), 6: (4 * h, h),
                 7: (h, 4 * h)}.get(which, (h, h))
        out = np.zeros(shape, np.float32)
        check(lib().mpic_model_download_weight(self.handle, which, layer, out.ctypes.data))
        return out


class KV:
    """Device KV tensor [L][T][H][D] (KvTensor, tensor.h:11-55)."""

    def __init__(self, L, T, H, D, dtype=F32, device=0):
        h = C.c_void_p()
        check(lib().mpic_kv_alloc(L, T, H, D, dtype, device, C.byref(h)))
        self.handle, self.shape, self.dtype = h.value, (L, T, H * D), dtype

    @classmethod
    def from_host(cls, k: np.ndarray, v: np.ndarray, H: int, D: int, dtype=F32, device=0,
                  stream=None):
        L, T = k.shape[0], k.shape[1]
        kv = cls(L, T, H, D, dtype, device)
        kv.upload(k, v, stream)
        return kv

    def upload(self, k, v, stream=None):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        assert k.size == self.shape[0] * self.shape[1] * self.shape[2]
        check(lib().mpic_kv_upload(self.handle, k.ctypes.data, v.ctypes.data, _stream_ptr(stream)))

    def download(self, stream=None):
        k = np.zeros(self.shape, np.float32)
        v = np.zeros(self.shape, np.float32)
        check(lib().mpic_kv_download(self.handle, k.ctypes.data, v.ctypes.data,
                                     _stream_ptr(stream)))
        return k, v

    def device_ptrs(self):
        k, v = C.c_void_p(), C.c_void_p()
        check(lib().mpic_kv_device_ptrs(self.handle, C.byref(k), C.byref(v)))
        return k.value, v.value

    def close(self):
        if getattr(self, "handle", None):
            try:
                lib().mpic_kv_free(self.handle)
            except Exception:  # interpreter shutdown: module globals may be gone
                pass
            self.handle = None

    __del__ = close


class Workspace:
    def __init__(self, model: Model, max_rows: int, max_ctx: int = 0):
        h = C.c_void_p()
        check(lib().mpic_workspace_create(model.handle, max_rows, max_ctx, C.byref(h)))
        self.handle, self.model = h.value, model

    def close(self):
        if getattr(self, "handle", None):
            try:
                lib().mpic_workspace_destroy(self.handle)
            except Exception:  # interpreter shutdown: module globals may be gone
                pass
            self.handle = None

    __del__ = close


class HostBuffer:
    """Pinned host memory (cudaMallocHost) viewed as a numpy array."""

    def __init__(self, shape, dtype=np.float32):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        check(lib().mpic_host_alloc(max(n, 1), C.byref(p)))
        self.ptr = p.value
        buf = (C.c_uint8 * max(n, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def close(self):
        if getattr(self, "ptr", None):
            self.array = None
            lib().mpic_host_free(self.ptr)
            self.ptr = None

    __del__ = close


@dataclass
class Prompt:
    """SegmentedPrompt (linker.h:14-54) as flat arrays: kinds 0=text/1=image, lens,
    concatenated text ids, 32-byte content hash per image."""

    kinds: np.ndarray
    lens: np.ndarray
    text_ids: np.ndarray
    hashes: np.ndarray

    @classmethod
    def from_segments(cls, segments):
        """segments: ('text', ids) or ('image', hash32, token_count)."""
        kinds, lens, text, hashes = [], [], [], []
        for seg in segments:
            if seg[0] == "text":
                kinds.append(0)
                lens.append(len(seg[1]))
                text.extend(int(t) for t in seg[1])
            else:
                kinds.append(1)
                lens.append(int(seg[2]))
                hashes.append(np.frombuffer(bytes(seg[1]), np.uint8))
        return cls(np.array(kinds, np.uint8), np.array(lens, np.uint32), np.array(text, np.int32),
                   np.concatenate(hashes) if hashes else np.zeros(0, np.uint8))

    @property
    def n(self) -> int:
        return int(self.lens.sum())

    def desc(self) -> PromptDesc:
        self._keep = [np.ascontiguousarray(self.kinds, np.uint8),
                      np.ascontiguousarray(self.lens, np.uint32),
                      np.ascontiguousarray(self.text_ids if self.text_ids.size else np.zeros(1),
                                           np.int32),
                      np.ascontiguousarray(self.hashes if self.hashes.size else np.zeros(32),
                                           np.uint8)]
        return PromptDesc(len(self.kinds), *[a.ctypes.data for a in self._keep])


def image_token_ids(cfg: ModelConfig, hash32: bytes, count: int) -> np.ndarray:
    out = np.zeros(count, np.int32)
    h = np.frombuffer(bytes(hash32), np.uint8).copy()
    check(lib().mpic_image_token_ids(C.byref(cfg), h.ctypes.data, count, out.ctypes.data))
    return out


def select_tokens(prompt: Prompt, policy: int = POLICY_MPIC_K, k: int = 32,
                  global_budget: bool = False) -> np.ndarray:
    out = np.zeros(max(prompt.n, 1), np.uint32)
    m = C.c_uint32()
    pol = PolicyDesc(policy, k, int(global_budget))
    check(lib().mpic_select_tokens(C.byref(prompt.desc()), C.byref(pol), out.ctypes.data,
                                   C.byref(m)))
    return out[:m.value].copy()


def flatten_ids(cfg: ModelConfig, prompt: Prompt) -> np.ndarray:
    out = np.zeros(prompt.n, np.int32)
    check(lib().mpic_flatten_ids(C.byref(cfg), C.byref(prompt.desc()), out.ctypes.data))
    return out


def assemble(chunks, dst: KV, reposition: int = AS_STORED, rope_base: float = 10000.0,
             zero_gaps: bool = True, stream=None):
    """chunks: list of (KV src, src_row0, dst_row0, rows, position_base)."""
    arr = (ChunkRef * max(len(chunks), 1))(
        *[ChunkRef(c[0].handle, c[1], c[2], c[3], c[4]) for c in chunks])
    check(lib().mpic_assemble(_stream_ptr(stream), arr, len(chunks), dst.handle, reposition,
                              rope_base, int(zero_gaps)))


def selective_prefill(model: Model, ws: Workspace, ids, rows, kv: KV, stream=None) -> np.ndarray:
    ids = np.ascontiguousarray(ids, np.int32)
    rows = np.ascontiguousarray(rows, np.uint32)
    logits = np.zeros(model.cfg.vocab_size, np.float32)
    check(lib().mpic_selective_prefill(model.handle, ws.handle, ids.ctypes.data, rows.ctypes.data,
                                       len(ids), kv.handle, logits.ctypes.data,
                                       _stream_ptr(stream)))
    return logits


def prefill_extend(model: Model, ws: Workspace, ids, start: int, position_base: int, kv: KV,
                   stream=None) -> np.ndarray:
    ids = np.ascontiguousarray(ids, np.int32)
    logits = np.zeros(model.cfg.vocab_size, np.float32)
    check(lib().mpic_prefill_extend(model.handle, ws.handle, ids.ctypes.data, len(ids), start,
                                    position_base, kv.handle, logits.ctypes.data,
                                    _stream_ptr(stream)))
    return logits


def request_prefill(model: Model, ws: Workspace, prompt: Prompt, chunks, linked: KV,
                    policy: int = POLICY_MPIC_K, k: int = 32, global_budget: bool = False,
                    reposition: int = AS_STORED, position_bases=None, stream=None):
    """select_tokens -> assemble_linked_cache -> selective_prefill with device-resident
    chunks (one KV per image segment). Returns (logits, selected rows)."""
    n_img = int((prompt.kinds == 1).sum())
    arr = (C.c_void_p * max(n_img, 1))(*[c.handle for c in chunks])
    pb = np.ascontiguousarray(position_bases if position_bases is not None else np.zeros(n_img),
                              np.uint32)
    logits = np.zeros(model.cfg.vocab_size, np.float32)
    sel = np.zeros(prompt.n, np.uint32)
    m = C.c_uint32()
    pol = PolicyDesc(policy, k, int(global_budget))
    check(lib().mpic_request_prefill(model.handle, ws.handle, C.byref(prompt.desc()),
                                     C.byref(pol), arr, reposition, pb.ctypes.data, linked.handle,
                                     logits.ctypes.data, sel.ctypes.data, C.byref(m),
                                     _stream_ptr(stream)))
    return logits, sel[:m.value].copy()


def request_prefill_batch(model: Model, ws: Workspace, prompts, chunks, linked: KV,
                          policy: int = POLICY_MPIC_K, k: int = 32, global_budget: bool = False,
                          reposition: int = AS_STORED, stream=None):
    """Batched varlen form of request_prefill (mpic_request_prefill_batch): `chunks[r]` lists
    request r's image chunks. Request r's cache is rows [off_r, off_r + n_r) of `linked`
    (off_r = sum of the earlier prompts' n). Returns (logits [nreq][vocab], rows per request)."""
    descs = (PromptDesc * len(prompts))(*[p.desc() for p in prompts])
    flat = [c.handle for cs in chunks for c in cs]
    arr = (C.c_void_p * max(len(flat), 1))(*flat)
    logits = np.zeros((len(prompts), model.cfg.vocab_size), np.float32)
    m = np.zeros(len(prompts), np.uint32)
    pol = PolicyDesc(policy, k, int(global_budget))
    check(lib().mpic_request_prefill_batch(model.handle, ws.handle, descs, len(prompts), C.byref(pol), arr,
                                           reposition, linked.handle, logits.ctypes.data, m.ctypes.data,
                                           _stream_ptr(stream)))
    return logits, m


def request_prefill_host(model: Model, ws: Workspace, prompt: Prompt, chunk_k, chunk_v,
                         linked: KV, policy: int = POLICY_MPIC_K, k: int = 32,
                         global_budget: bool = False, reposition: int = AS_STORED,
                         position_bases=None, stream=None, logits_out=None):
    """Same request with chunk KV in host memory ([L][len][h] arrays, ideally pinned
    HostBuffers): the loader streams them layer by layer to HBM. fp32 arrays are the .mpic
    v1 payload; bf16 chunks (numpy uint16 bit patterns, HostBuffer(..., np.uint16)) are the
    model-dtype Host tier with half the PCIe bytes. A None chunk is a miss: the library
    computes it on the device (the image's standalone prefill at position base 0) while the
    other chunks stream in (prepare's compute lane, transfer.cpp:119-127)."""
    n_img = len(chunk_k)
    present = [a for a in chunk_k if a is not None]
    dt = BF16 if present and present[0].dtype == np.uint16 else (model.dtype if not present else F32)
    kp = (C.c_void_p * max(n_img, 1))(*[None if a is None else a.ctypes.data for a in chunk_k])
    vp = (C.c_void_p * max(n_img, 1))(*[None if a is None else a.ctypes.data for a in chunk_v])
    pb = np.ascontiguousarray(position_bases if position_bases is not None else np.zeros(n_img),
                              np.uint32)
    logits = logits_out if logits_out is not None else np.zeros(model.cfg.vocab_size, np.float32)
    sel = np.zeros(prompt.n, np.uint32)
    m = C.c_uint32()
    pol = PolicyDesc(policy, k, int(global_budget))
    check(lib().mpic_request_prefill_host2(model.handle, ws.handle, C.byref(prompt.desc()),
                                           C.byref(pol), kp, vp, dt, pb.ctypes.data, reposition,
                                           linked.handle, logits.ctypes.data, sel.ctypes.data,
                                           C.byref(m), _stream_ptr(stream)))
    return logits, sel[:m.value].copy()


def request_prefill_files(model: Model, ws: Workspace, prompt: Prompt, paths, linked: KV,
                          policy: int = POLICY_MPIC_K, k: int = 32, global_budget: bool = False,
                          reposition: int = AS_STORED, stream=None, with_status: bool = False):
    """Same request with every image chunk read from its .mpic file by the disk loader
    (mpic_request_prefill_files2): disk -> pinned ring -> HBM per layer, CRC-checked. A path
    of None or a missing file is a miss, an unusable file (bad header, other model, wrong
    content hash, CRC mismatch) a fallback: both are computed on the device instead
    (prepare's semantics, transfer.cpp:83-145). with_status=True also returns the per-chunk
    outcome (CHUNK_LOADED / CHUNK_COMPUTED / CHUNK_FALLBACK)."""
    n_img = len(paths)
    enc = [None if p is None else os.fsencode(p) for p in paths]
    arr = (C.c_char_p * max(n_img, 1))(*enc)
    logits = np.zeros(model.cfg.vocab_size, np.float32)
    sel = np.zeros(prompt.n, np.uint32)
    status = np.zeros(max(n_img, 1), np.uint32)
    m = C.c_uint32()
    pol = PolicyDesc(policy, k, int(global_budget))
    check(lib().mpic_request_prefill_files2(model.handle, ws.handle, C.byref(prompt.desc()), C.byref(pol),
                                            C.cast(arr, C.c_void_p), reposition, linked.handle,
                                            logits.ctypes.data, sel.ctypes.data, C.byref(m),
                                            status.ctypes.data, _stream_ptr(stream)))
    if with_status:
        return logits, sel[:m.value].copy(), status[:n_img].copy()
    return logits, sel[:m.value].copy()


CHUNK_LOADED, CHUNK_COMPUTED, CHUNK_FALLBACK = 0, 1, 2
TIER_DEVICE, TIER_HOST, TIER_DISK = 0, 1, 2


class Store:
    """Tiered chunk store on the device (mpic_store_*, CacheStore of
    proj/include/mpic/cache.h:70-133): Device tier in HBM, Host tier in pinned memory, Disk
    tier as .mpic v3 files under `dir` (None: no disk tier), LRU demotion by entry-count
    budgets (cache.cpp:426-461), per-layer CRC32s computed and checked on the GPU."""

    def __init__(self, model: "Model", dir: str | None = None, device_budget: int = 64, host_budget: int = 256):
        h = C.c_void_p()
        check(lib().mpic_store_create(model.handle, dir.encode() if dir else None, device_budget, host_budget,
                                      C.byref(h)))
        self.handle, self.model = h.value, model

    @staticmethod
    def _hash(content_hash: bytes):
        b = bytes(content_hash)
        assert len(b) == 32
        return C.create_string_buffer(b, 32)

    def put(self, content_hash: bytes, kv: "KV", position_base: int = 0, ns: str = ""):
        check(lib().mpic_store_put(self.handle, self._hash(content_hash), ns.encode(), kv.handle, position_base))

    def tier(self, content_hash: bytes, ns: str = "") -> int:
        """TIER_DEVICE / TIER_HOST / TIER_DISK, or -1 when absent (tier_of)."""
        t = C.c_int()
        check(lib().mpic_store_tier(self.handle, self._hash(content_hash), ns.encode(), C.byref(t)))
        return t.value

    def demote(self, content_hash: bytes, tier: int, ns: str = ""):
        check(lib().mpic_store_demote(self.handle, self._hash(content_hash), ns.encode(), tier))

    def remove(self, content_hash: bytes, ns: str = ""):
        check(lib().mpic_store_remove(self.handle, self._hash(content_hash), ns.encode()))

    def request(self, ws: "Workspace", prompt: "Prompt", linked: "KV", policy: int = POLICY_MPIC_K, k: int = 32,
                global_budget: bool = False, reposition: int = AS_STORED, ns: str = "", stream=None):
        """prepare + selective_prefill from the store (mpic_store_request). Returns
        (logits, selected rows, per-image chunk status)."""
        n_img = int((prompt.kinds == 1).sum())
        logits = np.zeros(self.model.cfg.vocab_size, np.float32)
        sel = np.zeros(prompt.n, np.uint32)
        status = np.zeros(max(n_img, 1), np.uint32)
        m = C.c_uint32()
        pol = PolicyDesc(policy, k, int(global_budget))
        check(lib().mpic_store_request(self.handle, ws.handle, C.byref(prompt.desc()), C.byref(pol), ns.encode(),
                                       reposition, linked.handle, logits.ctypes.data, sel.ctypes.data, C.byref(m),
                                       status.ctypes.data, _stream_ptr(stream)))
        return logits, sel[:m.value].copy(), status[:n_img].copy()

    def close(self):
        if getattr(self, "handle", None):
            try:
                lib().mpic_store_destroy(self.handle)
            except Exception:  # interpreter shutdown
                pass
            self.handle = None

    def __del__(self):
        self.close()


def crc32_planes_device(ptr: int, plane_bytes: int, n_planes: int, stream=None) -> list:
    """Per-plane CRC32s of consecutive device planes, computed as the disk loader does."""
    out = np.zeros(max(n_planes, 1), np.uint32)
    check(lib().mpic_crc32_planes_device(ptr, plane_bytes, n_planes, out.ctypes.data, _stream_ptr(stream)))
    return [int(x) for x in out[:n_planes]]


def crc32_device(ptr: int, n: int, stream=None) -> int:
    """zlib-compatible CRC32 of n bytes at a device address (the store's GPU CRC kernel)."""
    c = C.c_uint32()
    check(lib().mpic_crc32_device(ptr, n, C.byref(c), _stream_ptr(stream)))
    return c.value


def write_mpic(path, cfg: ModelConfig, content_hash: bytes, k: np.ndarray, v: np.ndarray,
               position_base: int = 0, ns: str = "", bf16: bool = False, layer_crcs: bool = True):
    """Write one chunk as a .mpic container (proj/src/cache.cpp:97-125): an fp32 or a bf16
    payload (uint16 bit patterns), then — layer_crcs=True, version 3 — a table of per-layer
    CRC32s (crc_k[L], crc_v[L]; the disk loader verifies each layer on the GPU), then the
    CRC32 of all preceding bytes. layer_crcs=False writes v1 (fp32, the reference's own
    format) or v2 (bf16)."""
    import struct
    import zlib
    L, T, h = k.shape
    D = cfg.head_dim
    fnv = 0xcbf29ce484222325
    for b in ns.encode():
        fnv = ((fnv ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    version = 3 if layer_crcs else (2 if bf16 else 1)
    header = (b"MPIC" + struct.pack("<IQQ", version, fingerprint(cfg), fnv) + bytes(content_hash)
              + struct.pack("<IIIII", position_base, L, T, h // D, D) + bytes([1 if bf16 else 0]) + bytes(7))
    crc = zlib.crc32(header)
    table = []
    with open(path, "wb") as f:
        f.write(header)
        for a in (k, v):
            for l in range(L):  # layer by layer keeps the host copy small
                buf = (to_bf16_bits(a[l]) if bf16 else np.ascontiguousarray(a[l], np.float32)).tobytes()
                crc = zlib.crc32(buf, crc)
                table.append(zlib.crc32(buf))
                f.write(buf)
        if layer_crcs:
            tb = struct.pack(f"<{len(table)}I", *table)
            crc = zlib.crc32(tb, crc)
            f.write(tb)
        f.write(struct.pack("<I", crc & 0xFFFFFFFF))


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) as uint16 bit patterns."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


PHASES = ["assemble", "embed", "qkv", "attn", "wo", "w1", "w2", "cast", "lm_head"]


def profile_enable(on: bool = True):
    """Per-phase CUDA-event timing inside the library (mpic_profile_enable)."""
    check(lib().mpic_profile_enable(int(on)))


def profile_collect() -> dict:
    """{phase: (summed ms, instances)} since the last collect (mpic_profile_collect)."""
    ms = np.zeros(len(PHASES), np.float64)
    cnt = np.zeros(len(PHASES), np.uint32)
    check(lib().mpic_profile_collect(ms.ctypes.data, cnt.ctypes.data))
    return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(PHASES)}
