"""Summarise bench lines of an A/B run: python tools/bench_table.py gpurun_out/<tag>"""
import glob, json, os, sys
d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "bench_*.log"))):
    env = open(f[:-4] + ".env").read().strip() if os.path.exists(f[:-4] + ".env") else ""
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, env, "NO JSON", open(f).read()[-300:]); continue
    r = json.loads(lines[-1])
    ph = {k: v.get("ms_per_step") for k, v in r.get("phases", {}).items() if isinstance(v, dict) and "ms_per_step" in v}
    print(f"{os.path.basename(f):14s} {env:30s} {r['ms_per_step']:7.3f} ms", " ".join(f"{k}={v}" for k, v in ph.items()))
