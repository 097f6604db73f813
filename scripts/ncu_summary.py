"""Print the key metrics of an ncu report (raw page) for the kernels it holds."""
import csv, subprocess, sys

WANT = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.max"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print("#", name[:100])
    for w in WANT + [x for x in sys.argv[2:]]:
        if w in h:
            i = h.index(w)
            print(f"  {w:70s} {r[i]:>14s} {units[i]}")
