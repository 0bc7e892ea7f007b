"""End-to-end parity at the north-star width (SURVEY §8(c) parity protocol):
the bench's own workloads through the B200 C ABI against the UNMODIFIED reference build
(proj/src linker.cpp:35-135 via oracle/_ref) on identical inputs (tests/llava_cases.py).

  * config A exactly (L2 H8 D64 V4096, 2x576 images, n=1255, m=167);
  * config C (LLaVA-1.6: H32 D128 V32000, 4x2304 images, n=9418, m=330) at depth
    L' in {1, 2, 4, 8}, chunks HBM-resident (the bench's `value` leg, linking inside
    attention) and, at L'=2, from pinned host memory (the e2e leg);
  * config B (LLaVA-1.5: 1x576 image, n=640, m=96) at its full 32 layers in fp32 mode,
    gated at max(1e-4, 4 x CPU-vs-fp64) (oracle/fp64.py).

Tolerances (north star): max|gpu - ref| / max|ref| <= 1e-4 in fp32 mode, <= 1e-2 in bf16
mode, on the first-token logits and on the K/V of every recomputed row at every layer.
Unselected rows are the assembled chunk rows: bit-exact (fp32) / RNE-bf16 of them (bf16).
The bf16 32-layer numbers are reported by tools/depth_sweep.py, not gated."""
import numpy as np
import pytest

import oracle
import paper_2502_01960_b200 as mp
from llava_cases import Case, bf16_round

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref (reference build) missing")]

TOL = {mp.F32: 1e-4, mp.BF16: 1e-2}
_cases = {}


def case(name, layers=None, **kw):
    key = (name, layers)
    if key not in _cases:
        if len(_cases) >= 2:  # keep host memory bounded (L'=8 at config C holds ~10 GB)
            _cases.pop(next(iter(_cases)))
        c = Case(name, layers, **kw)
        c.run_reference()
        _cases[key] = c
    return _cases[key]


def check(c, got, dtype, label):
    ref = c.ref
    assert np.array_equal(got["sel"], ref["sel"]), "recompute set differs from the reference"
    e = c.compare(got, ref)
    print(f"{label}: {e}")
    tol = TOL[dtype]
    assert e["logits"] <= tol, (label, e)
    assert e["k_sel"] <= tol and e["v_sel"] <= tol, (label, e)
    if dtype == mp.F32:
        assert np.array_equal(got["k_unsel"], ref["k_unsel"]) and np.array_equal(got["v_unsel"], ref["v_unsel"])
    else:
        assert np.array_equal(got["k_unsel"], bf16_round(ref["k_unsel"]))
        assert np.array_equal(got["v_unsel"], bf16_round(ref["v_unsel"]))


@pytest.mark.parametrize("dtype", [mp.F32, mp.BF16], ids=["f32", "bf16"])
def test_config_a_exact(dtype):
    c = case("A", chunk_source="reference")
    assert c.n == 1255 and len(c.ref["sel"]) == 167
    check(c, c.run_b200(dtype), dtype, f"A {dtype}")


@pytest.mark.parametrize("depth", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", [mp.F32, mp.BF16], ids=["f32", "bf16"])
def test_config_c_depth(depth, dtype):
    c = case("C", depth)
    assert c.n == 9418 and len(c.ref["sel"]) == 330
    check(c, c.run_b200(dtype), dtype, f"C L'={depth} {dtype}")


@pytest.mark.parametrize("dtype", [mp.F32, mp.BF16], ids=["f32", "bf16"])
def test_config_c_host_tier(dtype):
    """The e2e leg (chunks in pinned host memory, per-layer H2D overlapped with compute)."""
    c = case("C", 2)
    check(c, c.run_b200(dtype, path="host"), dtype, f"C L'=2 host {dtype}")


def test_config_b_full_depth_fp32():
    c = Case("B")
    ref = c.run_reference(want_f64=True)
    assert c.n == 640 and len(ref["sel"]) == 96
    got = c.run_b200(mp.F32)
    e = c.compare(got, ref)
    cpu_f64 = c.compare({"logits": ref["logits"], "k_sel": ref["k_sel"], "v_sel": ref["v_sel"]}, ref, f64=True)
    gpu_f64 = c.compare(got, ref, f64=True)
    print(f"B L=32 f32: gpu-vs-cpu {e}; cpu-vs-fp64 {cpu_f64}; gpu-vs-fp64 {gpu_f64}")
    for key in ("logits", "k_sel", "v_sel"):
        assert e[key] <= max(1e-4, 4 * cpu_f64[key]), (key, e, cpu_f64)
