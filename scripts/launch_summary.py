"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_{read,write}.sum --csv
--log-file): per kernel name, launches, average duration, share of device time, DRAM bytes per
launch and their rate against the measured HBM peak.

    python scripts/launch_summary.py launches.csv [hbm_gbs] [first_launches] > summary.txt

first_launches: keep only the first that many launches of the library's step kernels (pos::, the
device-trace init excluded) — the eager warm-up steps, before bench.py's isolated-kernel section.
"""
import csv
import collections
import sys

path = sys.argv[1]
hbm = float(sys.argv[2]) if len(sys.argv) > 2 else 6551.0
lines = [l for l in open(path) if not l.startswith("==")]
rows = list(csv.DictReader(lines))
if len(sys.argv) > 3:
    keep, ids = int(sys.argv[3]), []
    for r in rows:
        if "pos::" in r["Kernel Name"] and "ktrace_init" not in r["Kernel Name"] and r["ID"] not in ids:
            ids.append(r["ID"])
    ids = set(ids[:keep])
    rows = [r for r in rows if r["ID"] in ids]
acc = collections.defaultdict(lambda: {"n": set(), "t": 0.0, "b": 0.0})
for r in rows:
    k = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    u = r.get("Metric Unit", "")
    a = acc[k]
    a["n"].add(r["ID"])
    if r["Metric Name"] == "gpu__time_duration.sum":
        a["t"] += v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(u, 1.0)
    elif r["Metric Name"].startswith("dram__bytes"):
        a["b"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
tot = sum(a["t"] for a in acc.values())
print(f"# {path}: {sum(len(a['n']) for a in acc.values())} launches, serialised (cold, one at a time)")
print("# launches  avg_us  share_of_device_time  DRAM_MB_per_launch  DRAM_GB/s  frac_of_%g  kernel" % hbm)
for k, a in sorted(acc.items(), key=lambda kv: -kv[1]["t"]):
    n = len(a["n"])
    gbs = a["b"] / (a["t"] * 1e3) if a["t"] else 0.0
    print(f"{n:4d} {a['t'] / n:9.1f} {100 * a['t'] / tot:6.1f}% {a['b'] / n / 1e6:10.2f} {gbs:9.1f} {gbs / hbm:6.3f}  {k[:90]}")
