"""Prints the A/B table of tools/bench_ab.sh: ms/step and per-phase ms per env assignment."""
import glob, json, os, sys
d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "bench_*.log")), key=lambda x: int(x.split("_")[-1].split(".")[0])):
    env = open(f.replace(".log", ".env")).read().strip() or "(default)"
    line = [l for l in open(f) if l.startswith("{")]
    if not line:
        print(f"{env:40s} no result"); continue
    j = json.loads(line[-1])
    ph = j.get("phases", {})
    parts = " ".join(f"{k} {v['ms_per_step']:.3f}" for k, v in ph.items() if isinstance(v, dict) and "ms_per_step" in v)
    print(f"{env:40s} {j['ms_per_step']:.3f} ms | {parts}")
