"""Checker-side bindings (TEST INFRASTRUCTURE ONLY).

Two CPU implementations of the MPIC partial-reuse path, loaded through ctypes:

* ``OracleC`` — the plain-C restatement in ``oracle/mpic_oracle.c`` (always built);
* ``RefLib``  — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` into ``oracle/_ref``
  (present only when that build ran; it travels to the GPU box as a prebuilt .so).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu/reference legs
may import this package. The product path (``paper_2502_01960_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


@dataclass
class Config:
    """Mirror of mpic::ModelConfig (proj/include/mpic/config.h:7-24)."""

    n_layers: int = 2
    n_heads: int = 2
    head_dim: int = 8
    hidden_dim: int = 16
    vocab_size: int = 256
    image_token_count: int = 16
    rope_base: float = 10000.0
    seed: int = 0

    def u6(self) -> np.ndarray:
        return np.array([self.n_layers, self.n_heads, self.head_dim, self.hidden_dim,
                         self.vocab_size, self.image_token_count], dtype=np.uint32)


@dataclass
class Prompt:
    """Segmented prompt as flat arrays (kinds 0=text 1=image, per-segment lengths,
    concatenated text ids, 32-byte content hash per image)."""

    kinds: np.ndarray
    lens: np.ndarray
    text_ids: np.ndarray
    hashes: np.ndarray
    ns: str = ""
    chunk_k: list = field(default_factory=list)  # per image [L][len][h] float32
    chunk_v: list = field(default_factory=list)
    chunk_base: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return int(self.lens.sum())

    @property
    def n_images(self) -> int:
        return int((self.kinds == 1).sum())

    def bounds(self):
        out, at = [], 0
        for ln in self.lens:
            out.append((at, at + int(ln)))
            at += int(ln)
        return out


def make_prompt(segments, ns: str = "") -> Prompt:
    """segments: list of ('text', ids) or ('image', hash32 bytes, count)."""
    kinds, lens, text, hashes = [], [], [], []
    for seg in segments:
        if seg[0] == "text":
            kinds.append(0)
            lens.append(len(seg[1]))
            text.extend(int(t) for t in seg[1])
        else:
            kinds.append(1)
            lens.append(int(seg[2]))
            hashes.append(np.frombuffer(bytes(seg[1]), dtype=np.uint8))
    return Prompt(np.array(kinds, np.uint8), np.array(lens, np.uint32),
                  np.array(text, np.int32),
                  np.concatenate(hashes).astype(np.uint8) if hashes else np.zeros(0, np.uint8),
                  ns)


class OracleC:
    """Bindings to oracle/_ref/libmpic_oracle.so (built from oracle/mpic_oracle.c)."""

    class _Cfg(C.Structure):
        _fields_ = [("n_layers", C.c_uint32), ("n_heads", C.c_uint32), ("head_dim", C.c_uint32),
                    ("hidden_dim", C.c_uint32), ("vocab_size", C.c_uint32),
                    ("image_token_count", C.c_uint32), ("rope_base", C.c_float),
                    ("seed", C.c_uint64)]

    def __init__(self, path: str | None = None):
        path = path or os.path.join(REF_DIR, "libmpic_oracle.so")
        if not os.path.exists(path):
            build_oracle()
        L = self.lib = C.CDLL(path)
        L.mo_fnv1a64.restype = C.c_uint64
        L.mo_fnv1a64.argtypes = [_u8p, C.c_size_t]
        L.mo_fingerprint.restype = C.c_uint64
        L.mo_fingerprint.argtypes = [C.POINTER(self._Cfg)]
        L.mo_counter_hash.restype = C.c_uint64
        L.mo_counter_hash.argtypes = [C.c_uint64] * 3
        L.mo_crc32.restype = C.c_uint32
        L.mo_crc32.argtypes = [_u8p, C.c_size_t]
        L.mo_model_create.restype = C.c_void_p
        L.mo_model_create.argtypes = [C.POINTER(self._Cfg)]
        L.mo_model_free.argtypes = [C.c_void_p]
        L.mo_model_weight.restype = C.POINTER(C.c_float)
        L.mo_model_weight.argtypes = [C.c_void_p, C.c_int, C.c_uint32]
        L.mo_image_ids.argtypes = [C.POINTER(self._Cfg), _u8p, C.c_uint32, _i32p]
        L.mo_select.restype = C.c_uint32
        L.mo_select.argtypes = [C.c_uint32, _u8p, _u32p, C.c_int, C.c_uint32, C.c_int, _u32p]
        L.mo_assemble.argtypes = [C.POINTER(self._Cfg), C.c_uint32, _u8p, _u32p,
                                  C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _u32p, C.c_int,
                                  _f32p, _f32p]
        L.mo_selective_core.restype = C.c_int
        L.mo_selective_core.argtypes = [C.c_void_p, _i32p, _u32p, _u32p, C.c_uint32, _f32p, _f32p,
                                        C.c_uint32, _f32p]

    def cfg(self, c: Config):
        return self._Cfg(c.n_layers, c.n_heads, c.head_dim, c.hidden_dim, c.vocab_size,
                         c.image_token_count, c.rope_base, c.seed)

    def fingerprint(self, c: Config) -> int:
        return int(self.lib.mo_fingerprint(C.byref(self.cfg(c))))

    def crc32(self, b: bytes) -> int:
        a = np.frombuffer(b, np.uint8).copy()
        return int(self.lib.mo_crc32(a, a.size))

    def image_ids(self, c: Config, hash32: bytes, count: int) -> np.ndarray:
        out = np.zeros(count, np.int32)
        self.lib.mo_image_ids(C.byref(self.cfg(c)), np.frombuffer(bytes(hash32), np.uint8).copy(),
                              count, out)
        return out

    def flatten(self, c: Config, p: Prompt) -> np.ndarray:
        parts, ti, hi = [], 0, 0
        for k, ln in zip(p.kinds, p.lens):
            ln = int(ln)
            if k == 0:
                parts.append(p.text_ids[ti:ti + ln])
                ti += ln
            else:
                parts.append(self.image_ids(c, p.hashes[32 * hi:32 * hi + 32].tobytes(), ln))
                hi += 1
        return np.concatenate(parts).astype(np.int32)

    def select(self, p: Prompt, policy: int = 0, k: int = 32, glob: bool = False) -> np.ndarray:
        out = np.zeros(max(p.n, 1), np.uint32)
        m = self.lib.mo_select(len(p.kinds), p.kinds, p.lens, policy, k, int(glob), out)
        return out[:m].copy()

    def model(self, c: Config) -> "OracleModel":
        return OracleModel(self, c)

    def assemble(self, c: Config, p: Prompt, rerotate: bool = False):
        n, row = p.n, c.n_heads * c.head_dim
        ok = np.zeros((c.n_layers, n, row), np.float32)
        ov = np.zeros_like(ok)
        ks = [np.ascontiguousarray(x, np.float32) for x in p.chunk_k]
        vs = [np.ascontiguousarray(x, np.float32) for x in p.chunk_v]
        kp = (C.c_void_p * max(len(ks), 1))(*[x.ctypes.data for x in ks])
        vp = (C.c_void_p * max(len(vs), 1))(*[x.ctypes.data for x in vs])
        base = np.array(p.chunk_base or [0], np.uint32)
        self.lib.mo_assemble(C.byref(self.cfg(c)), len(p.kinds), p.kinds, p.lens, kp, vp, base,
                             int(rerotate), ok, ov)
        return ok, ov


class OracleModel:
    def __init__(self, o: OracleC, c: Config):
        self.o, self.c = o, c
        self.h = o.lib.mo_model_create(C.byref(o.cfg(c)))
        if not self.h:
            raise ValueError("invalid model config")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.mo_model_free(self.h)
            self.h = None

    def weight(self, which: int, layer: int = 0) -> np.ndarray:
        c = self.c
        h = c.hidden_dim
        shape = {0: (c.vocab_size, h), 1: (c.vocab_size, h), 6: (4 * h, h), 7: (h, 4 * h)}.get(
            which, (h, h))
        ptr = self.o.lib.mo_model_weight(self.h, which, layer)
        return np.ctypeslib.as_array(ptr, shape=shape)

    def core(self, ids, rows, rope_pos, kv_k, kv_v):
        """Selective/extend core; kv_k/kv_v [L][n_ctx][h] updated in place. Returns logits."""
        ids = np.ascontiguousarray(ids, np.int32)
        rows = np.ascontiguousarray(rows, np.uint32)
        rope_pos = np.ascontiguousarray(rope_pos, np.uint32)
        logits = np.zeros(self.c.vocab_size, np.float32)
        rc = self.o.lib.mo_selective_core(self.h, ids, rows, rope_pos, len(ids), kv_k, kv_v,
                                          kv_k.shape[1], logits)
        if rc != 0:
            raise ValueError(f"oracle core failed ({rc})")
        return logits

    def prefill(self, ids, base: int = 0):
        """Standalone precompute: prefill_extend(ids, {}, base) (model.cpp:334-349)."""
        n = len(ids)
        kv_k = np.zeros((self.c.n_layers, n, self.c.hidden_dim), np.float32)
        kv_v = np.zeros_like(kv_k)
        rows = np.arange(n, dtype=np.uint32)
        logits = self.core(ids, rows, rows + base, kv_k, kv_v)
        return kv_k, kv_v, logits

    def selective(self, c: Config, p: Prompt, sel, asm_k, asm_v):
        """selective_prefill (linker.cpp:316-353) on copies of the assembled KV."""
        flat = self.o.flatten(c, p)
        kk, vv = asm_k.copy(), asm_v.copy()
        sel = np.asarray(sel, np.uint32)
        logits = self.core(flat[sel], sel, sel, kk, vv)
        return kk, vv, logits


class RefLib:
    """Bindings to oracle/_ref/libmpic_refcapi.so — the unmodified reference built from
    /root/reference/proj/src (see oracle/Makefile and oracle/ref_capi.cpp)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(REF_DIR, "libmpic_refcapi.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_fingerprint.restype = C.c_uint64
        L.ref_fingerprint.argtypes = [_u32p, C.c_float, C.c_uint64]
        L.ref_model_create.argtypes = [_u32p, C.c_float, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_weight.restype = C.POINTER(C.c_float)
        L.ref_model_weight.argtypes = [C.c_void_p, C.c_int, C.c_uint32]
        L.ref_weight_checksum.restype = C.c_uint64
        L.ref_weight_checksum.argtypes = [C.c_void_p]
        L.ref_image_ids.argtypes = [C.c_void_p, _u8p, C.c_uint32, _i32p]
        L.ref_prefill.argtypes = [C.c_void_p, _i32p, C.c_uint32, C.c_uint32, _f32p, _f32p, _f32p]
        L.ref_entries_create.restype = C.c_void_p
        L.ref_entries_free.argtypes = [C.c_void_p]
        L.ref_entries_add.argtypes = [C.c_void_p, C.c_void_p, _u8p, C.c_char_p, C.c_uint32,
                                      C.c_uint32, _f32p, _f32p]
        L.ref_select.argtypes = [C.c_void_p, C.c_uint32, _u8p, _u32p, _i32p, _u8p, C.c_int,
                                 C.c_uint32, C.c_int, _u32p, C.POINTER(C.c_uint32)]
        L.ref_flatten.argtypes = [C.c_void_p, C.c_uint32, _u8p, _u32p, _i32p, _u8p, _i32p]
        L.ref_link_and_prefill.argtypes = [C.c_void_p, C.c_uint32, _u8p, _u32p, _i32p, _u8p,
                                           C.c_char_p, C.c_void_p, C.c_int, C.c_void_p,
                                           C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_serialize_entry.restype = C.c_uint64
        L.ref_serialize_entry.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]

    def check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def set_threads(self, n: int):
        self.lib.ref_set_threads(n)

    def fingerprint(self, c: Config) -> int:
        return int(self.lib.ref_fingerprint(c.u6(), c.rope_base, c.seed))

    def model(self, c: Config) -> "RefModel":
        return RefModel(self, c)


def _ptr(a):
    return None if a is None else a.ctypes.data


class RefModel:
    def __init__(self, r: RefLib, c: Config):
        self.r, self.c = r, c
        h = C.c_void_p()
        r.check(r.lib.ref_model_create(c.u6(), c.rope_base, c.seed, C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_model_free(self.h)
            self.h = None

    def weight(self, which: int, layer: int = 0) -> np.ndarray:
        c = self.c
        h = c.hidden_dim
        shape = {0: (c.vocab_size, h), 1: (c.vocab_size, h), 6: (4 * h, h), 7: (h, 4 * h)}.get(
            which, (h, h))
        return np.ctypeslib.as_array(self.r.lib.ref_model_weight(self.h, which, layer), shape=shape)

    def checksum(self) -> int:
        return int(self.r.lib.ref_weight_checksum(self.h))

    def image_ids(self, hash32: bytes, count: int) -> np.ndarray:
        out = np.zeros(count, np.int32)
        self.r.lib.ref_image_ids(self.h, np.frombuffer(bytes(hash32), np.uint8).copy(), count, out)
        return out

    def prefill(self, ids, base: int = 0):
        ids = np.ascontiguousarray(ids, np.int32)
        n = len(ids)
        k = np.zeros((self.c.n_layers, n, self.c.hidden_dim), np.float32)
        v = np.zeros_like(k)
        logits = np.zeros(self.c.vocab_size, np.float32)
        self.r.check(self.r.lib.ref_prefill(self.h, ids, n, base, k, v, logits))
        return k, v, logits

    def select(self, p: Prompt, policy: int = 0, k: int = 32, glob: bool = False) -> np.ndarray:
        out = np.zeros(max(p.n, 1), np.uint32)
        m = C.c_uint32()
        hashes = p.hashes if p.hashes.size else np.zeros(32, np.uint8)
        self.r.check(self.r.lib.ref_select(self.h, len(p.kinds), p.kinds, p.lens,
                                           p.text_ids if p.text_ids.size else np.zeros(1, np.int32),
                                           hashes, policy, k, int(glob), out, C.byref(m)))
        return out[:m.value].copy()

    def flatten(self, p: Prompt) -> np.ndarray:
        out = np.zeros(p.n, np.int32)
        hashes = p.hashes if p.hashes.size else np.zeros(32, np.uint8)
        self.r.check(self.r.lib.ref_flatten(self.h, len(p.kinds), p.kinds, p.lens,
                                            p.text_ids if p.text_ids.size else np.zeros(1, np.int32),
                                            hashes, out))
        return out

    def entries(self, p: Prompt):
        e = self.r.lib.ref_entries_create()
        ns = p.ns.encode()
        for i in range(p.n_images):
            k = np.ascontiguousarray(p.chunk_k[i], np.float32)
            v = np.ascontiguousarray(p.chunk_v[i], np.float32)
            self.r.lib.ref_entries_add(e, self.h, p.hashes[32 * i:32 * i + 32].copy(), ns,
                                       k.shape[1], p.chunk_base[i], k, v)
        return e

    def link_and_prefill(self, p: Prompt, sel=None, rerotate: bool = False, want_asm=True,
                         want_final=True, entries=None):
        """assemble_linked_cache then (when sel is given) selective_prefill. Returns dict."""
        c, n = self.c, p.n
        shape = (c.n_layers, n, c.hidden_dim)
        own = entries is None
        e = self.entries(p) if own else entries
        try:
            ak = np.zeros(shape, np.float32) if want_asm else None
            av = np.zeros(shape, np.float32) if want_asm else None
            fk = np.zeros(shape, np.float32) if want_final else None
            fv = np.zeros(shape, np.float32) if want_final else None
            slots = np.zeros(3 * n, np.uint32)
            logits = np.zeros(c.vocab_size, np.float32)
            ms = np.zeros(2, np.float64)
            sel_a = None if sel is None else np.ascontiguousarray(sel, np.uint32)
            hashes = p.hashes if p.hashes.size else np.zeros(32, np.uint8)
            self.r.check(self.r.lib.ref_link_and_prefill(
                self.h, len(p.kinds), p.kinds, p.lens,
                p.text_ids if p.text_ids.size else np.zeros(1, np.int32), hashes, p.ns.encode(),
                e, int(rerotate), _ptr(sel_a), 0 if sel_a is None else len(sel_a), _ptr(ak),
                _ptr(av), _ptr(fk), _ptr(fv), slots.ctypes.data, logits.ctypes.data,
                ms.ctypes.data))
        finally:
            if own:
                self.r.lib.ref_entries_free(e)
        return dict(asm_k=ak, asm_v=av, k=fk, v=fv, slots=slots.reshape(n, 3), logits=logits,
                    ms_assemble=float(ms[0]), ms_selective=float(ms[1]))

    def serialize_entry(self, entries, idx: int) -> bytes:
        n = self.r.lib.ref_serialize_entry(entries, idx, None)
        buf = np.zeros(n, np.uint8)
        self.r.lib.ref_serialize_entry(entries, idx, buf.ctypes.data)
        return buf.tobytes()


def build_oracle(with_ref: bool | None = None) -> None:
    """Compile the checker: always the C restatement; the reference library too when
    /root/reference is present (this container only — the GPU box uses the prebuilt
    files that travel with the snapshot)."""
    targets = ["_ref/libmpic_oracle.so"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/src")
    if with_ref:
        targets += ["ref", "reftests"]
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2502_01960_b200", "lib",
                                       "libmpic_b200.so")):
            targets.append("conformance")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def have_ref() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libmpic_refcapi.so"))
