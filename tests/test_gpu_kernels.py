"""Kernel-level numerics: the tcgen05 GEMM and the SIMT GEMM against a plain PyTorch fp32
reference of the same bf16 operands (fp32 accumulation both sides)."""
import ctypes as C

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
                                   (1100, 128, 192), (330, 4096, 4096)])
@pytest.mark.parametrize("path", [1, 0])
def test_gemm_vs_torch(M, N, K, path):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = (torch.rand(M, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    w = (torch.rand(N, K, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    ref = a.float() @ w.float().t()
    out = run_gemm(a, w, path)
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
