"""fp64 selective prefill (TEST INFRASTRUCTURE ONLY — the checker, never the product).

Restates the reference's selective pass (`proj/src/linker.cpp:35-135`) with the arithmetic
of its straight-line fp64 model (`proj/tests/reference_model.h:53-131`): every product,
RoPE angle, softmax and GELU in float64, weights and cached K/V widened from their fp32
values. The reference's own tests use that model as the independent oracle for prefill and
cache reuse (`test_model.cpp:202-231`, `test_linker.cpp:204-220`); here it gives the
"CPU vs fp64" envelope SURVEY §8(c)(4) gates the deep LLaVA-width runs on.

numpy (BLAS float64 GEMMs), so a 32-layer LLaVA-width request runs in seconds.
"""
from __future__ import annotations

import numpy as np

# weight ids of oracle.RefModel.weight / OracleModel.weight
EMB, LM_HEAD, WQ, WK, WV, WO, W1, W2 = range(8)


def _rope(x: np.ndarray, pos: np.ndarray, n_heads: int, head_dim: int, base: float) -> None:
    """reference_model.h:21-35 (ref_rope) on rows x[i] at positions pos[i], in place."""
    i = np.arange(0, head_dim - 1, 2, dtype=np.float64)
    freq = np.power(float(base), -i / head_dim)               # std::pow(base, -i/D)
    theta = pos.astype(np.float64)[:, None] * freq[None, :]   # position * freq
    c, s = np.cos(theta), np.sin(theta)
    xv = x.reshape(x.shape[0], n_heads, head_dim)
    x0 = xv[:, :, 0::2].copy()
    x1 = xv[:, :, 1::2].copy()
    xv[:, :, 0::2] = x0 * c[:, None, :] - x1 * s[:, None, :]
    xv[:, :, 1::2] = x0 * s[:, None, :] + x1 * c[:, None, :]


def _gelu(x: np.ndarray) -> np.ndarray:
    """reference_model.h:48-50 (ref_gelu)."""
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


def selective_prefill_f64(weight, n_layers: int, n_heads: int, head_dim: int, rope_base: float,
                          ids_sel, sel, asm_k: np.ndarray, asm_v: np.ndarray, want_kv: bool = True):
    """weight(which, layer) -> fp32 array ([out][in], row-major); ids_sel/sel: the selected
    rows' token ids and global indices (ascending; position = index, linker.cpp:67-70);
    asm_k/asm_v: the assembled cache [L][n][h] (fp32). Returns (logits f64 [V],
    k_sel f64 [L][m][h], v_sel f64 [L][m][h]) — the recomputed rows of every layer."""
    sel = np.asarray(sel, np.int64)
    ids_sel = np.asarray(ids_sel, np.int64)
    m = len(sel)
    h = n_heads * head_dim
    emb = weight(EMB, 0)
    x = emb[ids_sel].astype(np.float64)                       # embed_tokens (model.cpp:89-99)
    k_out = np.zeros((n_layers, m, h)) if want_kv else None
    v_out = np.zeros((n_layers, m, h)) if want_kv else None
    inv = 1.0 / np.sqrt(float(head_dim))
    for l in range(n_layers):
        q = x @ weight(WQ, l).astype(np.float64).T
        k = x @ weight(WK, l).astype(np.float64).T
        v = x @ weight(WV, l).astype(np.float64).T
        _rope(q, sel, n_heads, head_dim, rope_base)
        _rope(k, sel, n_heads, head_dim, rope_base)
        # every selected row is scattered before any attention of the layer (linker.cpp:64-78)
        K = asm_k[l].astype(np.float64)
        V = asm_v[l].astype(np.float64)
        K[sel] = k
        V[sel] = v
        if want_kv:
            k_out[l] = k
            v_out[l] = v
        n_ctx = int(sel[-1]) + 1
        attn = np.zeros((m, h))
        col = np.arange(n_ctx)
        mask = col[None, :] <= sel[:, None]                   # causal count pos_i + 1
        for hh in range(n_heads):
            sl = slice(hh * head_dim, (hh + 1) * head_dim)
            s = (q[:, sl] @ K[:n_ctx, sl].T) * inv
            s = np.where(mask, s, -np.inf)
            s -= s.max(axis=1, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=1, keepdims=True)
            attn[:, sl] = p @ V[:n_ctx, sl]
        del K, V
        x += attn @ weight(WO, l).astype(np.float64).T
        f = _gelu(x @ weight(W1, l).astype(np.float64).T)
        x += f @ weight(W2, l).astype(np.float64).T
    logits = weight(LM_HEAD, 0).astype(np.float64) @ x[-1]
    return logits, k_out, v_out
