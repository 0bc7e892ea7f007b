"""Summarise ncu outputs into markdown for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv> [steps]   per-kernel share of a step
  python tools/ncu_summary.py full <prof.ncu-rep>               key SOL metrics per captured launch
"""
import csv
import collections
import io
import subprocess
import sys


def launches(path, steps=1):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e3  # us
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
    for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {c} | {us:.1f} | {us / c:.2f} | {100 * us / tot:.1f}% |")
    print(f"\ntotal kernel time {tot:.1f} us over {len(rows)} launches "
          f"({tot / steps:.1f} us per step if {steps} steps were captured)")


UNIT = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
        "Gbyte": 1e3, "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0, "cycle/nsecond": 1.0,
        "cycle/usecond": 1e-3, "%": 1.0, "register/thread": 1.0, "": 1.0}
METRICS = [
    ("gpu__time_duration.sum", "us", None),
    ("sm__cycles_elapsed.avg.per_second", "SM GHz", None),
    ("dram__bytes_read.sum", "DRAM rd MB", None),
    ("dram__bytes_write.sum", "DRAM wr MB", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", None),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %", None),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %", None),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", None),
    ("launch__registers_per_thread", "regs", None),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[0]
    idx = [hdr.index(m) if m in hdr else -1 for m, _, _ in METRICS]
    print("| kernel | grid | " + " | ".join(h for _, h, _ in METRICS) + " |")
    print("|---|---|" + "---|" * len(METRICS))
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
        vals = []
        for i, (_, _, sc) in zip(idx, METRICS):
            try:
                f = sc if sc is not None else UNIT.get(r[1][i], float("nan"))
                vals.append(f"{float(row[i].replace(',', '')) * f:.2f}" if i >= 0 else "-")
            except ValueError:
                vals.append(row[i])
        print(f"| `{name}` | {row[hdr.index('Grid Size')]} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)
    else:
        full(sys.argv[2])
