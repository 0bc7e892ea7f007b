"""Kernel-level numerics: the tcgen05 GEMM and the SIMT GEMM against a plain PyTorch fp32
reference of the same bf16 operands (fp32 accumulation both sides)."""
import ctypes as C

import numpy as np

import pytest
import torch

import paper_2502_01960_b200 as mp
from paper_2502_01960_b200 import _lib

pytestmark = pytest.mark.gpu


def run_gemm(a, w, path):
    M, K = a.shape
    N = w.shape[0]
    out = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().mpic_test_gemm(a.data_ptr(), w.data_ptr(), M, N, K, path,
                                         out.data_ptr(), s))
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (17, 256, 128), (96, 512, 512),
                                   (330, 1024, 512), (512, 256, 1024), (600, 384, 256),
                                   (1100, 128, 192), (330, 4096, 4096),
                                   # persistent pair GEMM: one piece, two pieces, groups;
                                   # stream-K splits at 1 .. many pairs per tile
                                   (256, 256, 64), (257, 512, 128), (330, 12288, 4096),
                                   (330, 4096, 16384), (96, 16384, 512), (2000, 1024, 320),
                                   (513, 768, 4096), (48, 256, 12288)])
@pytest.mark.parametrize("path", [1, 2, 0])
def test_gemm_vs_torch(M, N, K, path):
    if path == 2 and N % 256:
        pytest.skip("blocked weights feed the pair GEMM (N % 256 == 0)")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = (torch.rand(M, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    w = (torch.rand(N, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    ref = a.float() @ w.float().t()
    out = run_gemm(a, w, path)
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    # fp32 accumulation of K products: the rounding envelope grows with K (and with the
    # order the partial sums are combined in), so the bound scales with K / 4096
    assert err < 1e-5 * max(1.0, K / 4096), err


@pytest.mark.parametrize("M,N,K", [(1, 256, 64), (17, 256, 96), (330, 12288, 4096), (330, 4096, 4096),
                                   (330, 16384, 4096), (330, 4096, 16384), (96, 4096, 4096),
                                   (600, 512, 256), (1100, 768, 1024)])
def test_gemm_3xtf32_vs_fp64(M, N, K):
    """The fp32 mode's tensor-core GEMM (3xTF32: hi/lo tf32 split, three tcgen05 kind::tf32
    products per step, fp32 TMEM accumulation) is as close to the exact (fp64) product as
    the SIMT FFMA GEMM it replaces."""
    g = torch.Generator(device="cuda").manual_seed(M * 5 + N + K)
    a = torch.rand(M, K, device="cuda", generator=g) - 0.5
    w = (torch.rand(N, K, device="cuda", generator=g) - 0.5) / K ** 0.5
    ref = a.double() @ w.double().t()
    scale = ref.abs().max().item()
    err_tc = (run_gemm(a, w, 4).double() - ref).abs().max().item() / scale
    err_simt = (run_gemm(a, w, 5).double() - ref).abs().max().item() / scale
    print(f"3xTF32 {M}x{N}x{K}: tc {err_tc:.3e} simt {err_simt:.3e}")
    # measured: 3e-7 .. 7e-7 (SIMT 1e-7 .. 1.3e-6); one accumulation chain over all of K
    # (no segments) gave 3e-5 .. 6e-5 — the tensor core truncates its fp32 accumulation
    assert err_tc < 2e-6, (err_tc, err_simt)
    assert err_tc < 4 * err_simt + 5e-7, (err_tc, err_simt)


@pytest.mark.parametrize("M,N,K", [(330, 4096, 4096), (96, 1024, 2048), (600, 512, 256),
                                   (330, 16384, 512)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_gemm_epilogues_vs_torch(M, N, K, mode):
    """Fused epilogues of the tcgen05 GEMM: residual add (+ bf16 copy), GELU (tanh form,
    proj/src/model.cpp:85-87), plain bf16 store."""
    g = torch.Generator(device="cuda").manual_seed(M + N * 3 + K + mode)
    a = (torch.rand(M, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    w = (torch.rand(N, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    y = a.float() @ w.float().t()
    x = torch.rand(M, N, device="cuda", generator=g) - 0.5
    xb = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    x_in = x.clone()
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().mpic_test_gemm_epi(a.data_ptr(), w.data_ptr(), M, N, K, mode, x.data_ptr(),
                                             xb.data_ptr(), out.data_ptr(), s))
    torch.cuda.synchronize()
    if mode == 0:
        ref = x_in + y
        assert (x - ref).abs().max().item() / ref.abs().max().item() < 1e-5
        assert torch.equal(xb, x.to(torch.bfloat16))
    else:
        ref = torch.nn.functional.gelu(y, approximate="tanh") if mode == 1 else y
        err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
        assert err < 1e-2, err


def run_attention(q, k, v, rows, H):
    m, n = q.shape[0], k.shape[0]
    out = torch.zeros(m, H * 128, dtype=torch.bfloat16, device="cuda")
    r = np.ascontiguousarray(rows, np.uint32)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().mpic_test_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), r.ctypes.data,
                                              m, n, H, out.data_ptr(), s))
    torch.cuda.synchronize()
    return out


def attention_ref(q, k, v, rows, H):
    """Plain PyTorch fp32: softmax(q k^T / sqrt(128)) v with key j <= rows[i]."""
    m, n = q.shape[0], k.shape[0]
    qf = q.float().view(m, H, 128).transpose(0, 1)
    kf = k.float().view(n, H, 128).transpose(0, 1)
    vf = v.float().view(n, H, 128).transpose(0, 1)
    s = (qf @ kf.transpose(1, 2)) * (1.0 / 128 ** 0.5)
    mask = torch.arange(n, device="cuda")[None, :] > torch.as_tensor(rows.astype(np.int64), device="cuda")[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    return (torch.softmax(s, -1) @ vf).transpose(0, 1).reshape(m, H * 128)


@pytest.mark.parametrize("n,m,H", [(300, 40, 2), (1000, 130, 3), (9418, 330, 4), (4000, 600, 1)])
def test_attention_vs_torch(n, m, H):
    g = torch.Generator(device="cuda").manual_seed(n + m)
    q = torch.randn(m, H * 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(n, H * 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(n, H * 128, device="cuda", generator=g).to(torch.bfloat16)
    rows = np.sort(np.random.default_rng(m).choice(n - 1, m - 1, replace=False)).astype(np.uint32)
    rows = np.append(rows, n - 1).astype(np.uint32)
    out = run_attention(q, k, v, rows, H)
    ref = attention_ref(q, k, v, rows, H)
    err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err


def rope_table(pos, D, base=10000.0):
    """(cos, sin) per row and pair as the reference computes them: theta = pos * base^(-i/D)
    in double, then float (proj/src/model.cpp:46-62)."""
    i = torch.arange(0, D - 1, 2, dtype=torch.float64)
    theta = torch.as_tensor(pos, dtype=torch.float64)[:, None] * torch.pow(torch.tensor(base, dtype=torch.float64), -i / D)
    return torch.stack([torch.cos(theta).float(), torch.sin(theta).float()], dim=-1).contiguous()


def rope_ref(x, cs, H, D):
    """model.cpp:46-62 in fp32 on [M][h] rows."""
    xv = x.view(x.shape[0], H, D // 2, 2)
    c, s = cs[:, None, :, 0], cs[:, None, :, 1]
    x0, x1 = xv[..., 0], xv[..., 1]
    return torch.stack([x0 * c - x1 * s, x0 * s + x1 * c], dim=-1).reshape(x.shape)


@pytest.mark.parametrize("cfg_name", ["C", "A", "B"])
def test_qkv_rope_scatter_vs_torch(cfg_name):
    """K3 exactly as a layer runs it at the bench configs' tiling (config C: M = 330 rows =
    one 176 + 160 token group, 48 tiles of 256 features): Wqkv GEMM + RoPE of q and k at each
    row's position + scatter of k, v into the cache planes at the selected rows
    (linker.cpp:59-78). Against torch fp32 on the same bf16 operands and (cos, sin) table;
    cache rows that are not selected must be untouched."""
    import bench
    L, H, D, V, images, k = bench.CONFIGS[cfg_name]
    h = H * D
    p = mp.Prompt.from_segments(bench.build_prompt(cfg_name, V))
    sel = mp.select_tokens(p, mp.POLICY_MPIC_K, k)
    M, n = len(sel), p.n
    g = torch.Generator(device="cuda").manual_seed(M + n)
    a = (torch.rand(M, h, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    w = ((torch.rand(3 * h, h, device="cuda", generator=g) - 0.5) / 32).to(torch.bfloat16)
    rows = torch.as_tensor(sel.astype(np.int64), device="cuda").to(torch.int32)
    cs = rope_table(sel.astype(np.float64), D).cuda()
    kk = (torch.rand(n, h, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    vv = (torch.rand(n, h, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    k0, v0 = kk.clone(), vv.clone()
    q = torch.zeros(M, h, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().mpic_test_qkv(a.data_ptr(), w.data_ptr(), M, h, h, D, rows.data_ptr(), cs.data_ptr(),
                                        q.data_ptr(), kk.data_ptr(), vv.data_ptr(), s))
    torch.cuda.synchronize()
    y = a.float() @ w.float().t()
    q_ref = rope_ref(y[:, :h].contiguous(), cs, H, D)
    k_ref = rope_ref(y[:, h:2 * h].contiguous(), cs, H, D)
    v_ref = y[:, 2 * h:]
    ri = rows.long()
    for got, ref in ((q.float(), q_ref), (kk[ri].float(), k_ref), (vv[ri].float(), v_ref)):
        # fp32 epilogue then one bf16 rounding: within one bf16 ulp of the fp32 reference
        # (plus the fp32 accumulation-order envelope)
        tol = ref.abs() * 2.0 ** -7 + 1e-5 * ref.abs().max()
        assert ((got - ref).abs() <= tol).all(), (got - ref).abs().max()
    other = torch.ones(n, dtype=torch.bool, device="cuda")
    other[ri] = False
    assert torch.equal(kk[other], k0[other]) and torch.equal(vv[other], v0[other])
