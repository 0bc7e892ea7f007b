"""Summarise MPIC_ATTN_TS logs (tools/attn_probe.py output): kernel span from the per-CTA
start/end stamps of the last launch, a least-squares per-block cost fit, and the median
softmax phase times of CTA 0. Diagnostic only."""
import re, sys
import numpy as np

def summarise(path):
    lines = open(path).read().splitlines()
    groups, cur = [], []
    for l in lines:
        if l.startswith("cta    0 ") and cur:
            groups.append(cur); cur = []
        if l.startswith("cta"):
            cur.append(l)
    groups.append(cur)
    g = groups[-1]
    if not g:
        return f"{path}: no CTA stamps"
    rows = []
    for l in g:
        m = re.search(r"start\s+([\d.]+) end\s+([\d.]+) us  head \d+ b0 (\d+) tiles \d+/(\d+) b1 (\d+)/(\d+)", l)
        if not m:
            continue
        s, e, b0, t1, b10, b11 = m.groups()
        n0 = int(b10) - int(b0); n1 = int(b11) - int(b0) if int(t1) != 999 else 0
        rows.append((float(s), float(e), max(n0, n1) - min(n0, n1) if n1 else n0, min(n0, n1) if n1 else 0))
    span = max(r[1] for r in rows)
    ph = []
    for l in g:
        m = re.search(r"start\s+([\d.]+) end\s+([\d.]+).*mma0\s+(-?[\d.]+) lastmma\s+(-?[\d.]+) epi\s+(-?[\d.]+) epi_end\s+(-?[\d.]+)", l)
        if m:
            s0, e0, a, b, c, d = map(float, m.groups())
            if min(a, b, c, d) >= 0:
                ph.append((a - s0, b - a, c - b, d - c, e0 - d))
    phase_txt = ""
    if ph:
        pm = np.median(np.array(ph), axis=0)
        phase_txt = (f"; per CTA median: start->mma0 {pm[0]:.2f}, mma loop {pm[1]:.2f}, lastmma->epi {pm[2]:.2f}, "
                     f"epilogue {pm[3]:.2f}, epi->end {pm[4]:.2f} us")
    A = np.array([[1, r[2], r[3]] for r in rows], float)
    y = np.array([r[1] - r[0] for r in rows])
    coef = np.linalg.lstsq(A, y, rcond=None)[0]
    sm = [l for l in lines if l.startswith("j=")]
    ph = []
    for l in sm[-40:]:
        v = [float(x) for x in re.findall(r"(-?[\d.]+)", l.split("|")[1])]
        if min(v) >= 0:
            ph.append((v[1] - v[0], v[2] - v[1], v[3] - v[2], v[4] - v[0]))
    phs = np.median(np.array(ph), axis=0) if ph else [float("nan")] * 4
    return (f"{path}: span {span:6.1f} us, sum/148 {y.sum()/148:6.1f}; fit setup {coef[0]:.2f} single-blk {coef[1]:.2f} "
            f"pair-blk {coef[2]:.2f} us{phase_txt}; CTA0 softmax ld {phs[0]:.2f} max {phs[1]:.2f} exp {phs[2]:.2f} total {phs[3]:.2f} us")

for p in sys.argv[1:]:
    print(summarise(p))
