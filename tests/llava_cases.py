"""LLaVA-width parity cases (SURVEY §8(c) parity protocol): the bench's own workloads at
depth L', run through the B200 path and through the UNMODIFIED reference build
(oracle/_ref, proj/src assemble_linked_cache + selective_prefill) on identical inputs.

Inputs (identical bytes on both sides):
  * weights: build_model(seed 1) — the reference builds its own; the GPU synthesises the
    same values on the device (bit-exact, tests/test_gpu_parity.py);
  * prompt: bench.build_prompt(config) — the seeded ids and content hashes of the bench;
  * chunk KV: each image's standalone precompute prefill_extend(image_token_ids(hash), base 0)
    (test_util.h:44-60 make_image_entry), computed ONCE here by the B200 fp32 path and handed
    as the same fp32 arrays to the reference and to the B200 request (the bf16 mode rounds
    them to bf16 on upload, as its Device tier stores them). Hot-path parity therefore does
    not depend on miss-path parity.

Used by tests/test_gpu_llava.py (gated depths) and tools/depth_sweep.py (L' = 16, 32,
reported beside CPU-vs-fp64)."""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2502_01960_b200 as mp  # noqa: E402
from bench import CONFIGS, build_prompt  # noqa: E402


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


class Case:
    """One bench workload at depth `layers` (None = the config's own depth)."""

    def __init__(self, name: str, layers: int | None = None, k: int | None = None,
                 chunk_source: str = "b200"):
        L, H, D, V, images, kk = CONFIGS[name]
        self.name = name
        self.L = layers or L
        self.H, self.D, self.V, self.images = H, D, V, images
        self.k = kk if k is None else k
        self.h = H * D
        self.segs = build_prompt(name, V)
        self.cfg = mp.config(self.L, H, D, vocab_size=V, image_token_count=images[0], seed=1)
        self.ocfg = oracle.Config(self.L, H, D, self.h, V, images[0], 10000.0, 1)
        self.prompt = mp.Prompt.from_segments(self.segs)
        self.n = self.prompt.n
        self.chunk_source = chunk_source  # "b200" (fp32 SIMT prefill) or "reference"
        self.chunks = None   # [(k, v)] fp32 [L][T][h]
        self.ref = None      # reference outputs

    # -- inputs ------------------------------------------------------------------------
    def make_chunks(self):
        """Standalone precompute of every image: on the B200 fp32 path (SIMT, fp32), or
        with the reference's own prefill_extend (small configs)."""
        if self.chunks is not None:
            return self.chunks
        if self.chunk_source == "reference":
            rm = oracle.RefLib().model(self.ocfg)
            self.chunks = [rm.prefill(rm.image_ids(seg[1], seg[2]), 0)[:2] for seg in self.segs
                           if seg[0] == "image"]
            return self.chunks
        m32 = mp.Model(self.cfg, mp.F32)
        ws = mp.Workspace(m32, max(self.images))
        self.chunks = []
        for seg in self.segs:
            if seg[0] != "image":
                continue
            T = seg[2]
            ids = mp.image_token_ids(self.cfg, seg[1], T)
            kv = mp.KV(self.L, T, self.H, self.D, mp.F32)
            mp.prefill_extend(m32, ws, ids, 0, 0, kv)
            self.chunks.append(kv.download())
            kv.close()
        ws.close()
        m32.close()
        return self.chunks

    # -- the reference ---------------------------------------------------------------------
    def run_reference(self, threads: int | None = None, want_f64: bool = False):
        """assemble_linked_cache + selective_prefill of the unmodified reference (fp32,
        OpenBLAS); optionally the fp64 restatement (oracle/fp64.py) on the same assembled
        cache."""
        if self.ref is not None and (not want_f64 or "f64_logits" in self.ref):
            return self.ref
        r = oracle.RefLib()
        r.set_threads(threads or os.cpu_count() or 8)
        t0 = time.time()
        rm = r.model(self.ocfg)
        t_build = time.time() - t0
        p = oracle.make_prompt(self.segs, "")
        for k, v in self.make_chunks():
            p.chunk_k.append(k)
            p.chunk_v.append(v)
            p.chunk_base.append(0)
        sel = rm.select(p, 0, self.k)
        flat = rm.flatten(p)
        res = rm.link_and_prefill(p, sel=sel, want_asm=want_f64, want_final=True)
        out = dict(sel=sel, logits=res["logits"], k_sel=res["k"][:, sel].copy(),
                   v_sel=res["v"][:, sel].copy(), ms_selective=res["ms_selective"],
                   ms_assemble=res["ms_assemble"], s_build=t_build)
        # unselected rows: the assembled chunk rows (AsStored) — keep a digest-sized sample
        unsel = np.setdiff1d(np.arange(self.n), sel)
        pick = unsel[:: max(1, len(unsel) // 257)]
        out["unsel_rows"] = pick
        out["k_unsel"] = res["k"][:, pick].copy()
        out["v_unsel"] = res["v"][:, pick].copy()
        if want_f64:
            from oracle.fp64 import selective_prefill_f64
            t1 = time.time()
            lg, kf, vf = selective_prefill_f64(rm.weight, self.L, self.H, self.D, 10000.0, flat[sel], sel,
                                               res["asm_k"], res["asm_v"])
            out.update(f64_logits=lg, f64_k_sel=kf, f64_v_sel=vf, s_f64=time.time() - t1)
        del res
        self.ref = out
        return out

    # -- the B200 path -----------------------------------------------------------------
    def run_b200(self, dtype: int, path: str = "device"):
        """One MPIC-k request through the C ABI. path: 'device' (chunks HBM-resident, the
        bench's `value` leg), 'host' (bf16 bits in pinned host memory, the e2e leg)."""
        m = mp.Model(self.cfg, dtype)
        ws = mp.Workspace(m, 2048, self.n)
        linked = mp.KV(self.L, self.n, self.H, self.D, dtype)
        chunks = self.make_chunks()
        if path == "device":
            kvs = [mp.KV.from_host(k, v, self.H, self.D, dtype) for k, v in chunks]
            logits, sel = mp.request_prefill(m, ws, self.prompt, kvs, linked, k=self.k)
            for kv in kvs:
                kv.close()
        else:
            pins = []
            bits = dtype == mp.BF16
            for k, v in chunks:
                hk = mp.HostBuffer(k.shape, np.uint16 if bits else np.float32)
                hv = mp.HostBuffer(v.shape, np.uint16 if bits else np.float32)
                hk.array[...] = mp.to_bf16_bits(k) if bits else k
                hv.array[...] = mp.to_bf16_bits(v) if bits else v
                pins += [hk, hv]
            logits, sel = mp.request_prefill_host(m, ws, self.prompt, [x.array for x in pins[0::2]],
                                                  [x.array for x in pins[1::2]], linked, k=self.k)
        k_all, v_all = linked.download()
        ref_unsel = self.ref["unsel_rows"] if self.ref is not None else None
        out = dict(logits=logits, sel=sel, k_sel=k_all[:, sel].copy(), v_sel=v_all[:, sel].copy())
        if ref_unsel is not None:
            out["k_unsel"] = k_all[:, ref_unsel].copy()
            out["v_unsel"] = v_all[:, ref_unsel].copy()
        del k_all, v_all
        linked.close()
        ws.close()
        m.close()
        return out

    def compare(self, got, ref, f64: bool = False) -> dict:
        key = "f64_" if f64 else ""
        return dict(logits=rel_err(got["logits"], ref[key + "logits"]),
                    k_sel=rel_err(got["k_sel"], ref[key + "k_sel"]),
                    v_sel=rel_err(got["v_sel"], ref[key + "v_sel"]),
                    argmax_equal=bool(np.argmax(got["logits"]) == np.argmax(ref[key + "logits"])))


def bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()
