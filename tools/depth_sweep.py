"""Depth sweep of end-to-end parity at LLaVA width.

For config C (and optionally B) at each depth L', runs the unmodified reference
(assemble_linked_cache + selective_prefill, fp32 OpenBLAS), the fp64 restatement of the
same selective pass (oracle/fp64.py, reference_model.h arithmetic) and the B200 path in
fp32 and bf16 mode on identical inputs (tests/llava_cases.py), and reports
  GPU-vs-CPU, CPU-vs-fp64 and GPU-vs-fp64 max relative errors on the logits and on the
  recomputed rows' K/V of every layer, plus argmax agreement.
fp32 gate: GPU-vs-CPU <= max(1e-4, 4 x CPU-vs-fp64).

    python tools/depth_sweep.py --config C --depths 16 32 --out gpurun_out/depth_sweep.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from llava_cases import Case  # noqa: E402

import paper_2502_01960_b200 as mp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C")
    ap.add_argument("--depths", type=int, nargs="+", default=[16, 32])
    ap.add_argument("--f32-only", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "depth_sweep.json"))
    args = ap.parse_args()
    rows = []
    for d in args.depths:
        t0 = time.time()
        c = Case(args.config, d)
        ref = c.run_reference(want_f64=True)
        cpu_f64 = c.compare({k: ref[k] for k in ("logits", "k_sel", "v_sel")}, ref, f64=True)
        row = dict(config=args.config, depth=d, n=c.n, m=len(ref["sel"]), cpu_vs_f64=cpu_f64,
                   ref_selective_s=ref["ms_selective"] / 1e3, f64_s=ref.get("s_f64"))
        for dt, name in [(mp.F32, "f32"), (mp.BF16, "bf16")][: 1 if args.f32_only else 2]:
            got = c.run_b200(dt)
            assert (got["sel"] == ref["sel"]).all()
            row[f"gpu_{name}_vs_cpu"] = c.compare(got, ref)
            row[f"gpu_{name}_vs_f64"] = c.compare(got, ref, f64=True)
            if dt == mp.F32:
                row["f32_gate"] = {k: max(1e-4, 4 * cpu_f64[k]) for k in ("logits", "k_sel", "v_sel")}
                row["f32_pass"] = all(row["gpu_f32_vs_cpu"][k] <= row["f32_gate"][k]
                                      for k in ("logits", "k_sel", "v_sel"))
            del got
        row["wall_s"] = time.time() - t0
        print(json.dumps(row), flush=True)
        rows.append(row)
        del c, ref
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
