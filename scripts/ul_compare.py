"""Per-layer comparison of gpu_unet_libs.sh launch lists: python scripts/ul_compare.py base desc ..."""
import csv
import sys


def load(n):
    rows = [r for r in csv.reader(open(f"gpurun_out/ul_{n}.csv")) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki].split("(")[0].replace("void nar::", ""), float(r[vi]) / 1000) for r in rows[1:]
            if "nar::" in r[ki]]


names = sys.argv[1:]
data = [load(n) for n in names]
n_layers = len(data[0]) // 3  # prof_unet --frames 1 runs 3 forwards (2 warm-up)
print(f"{'kernel':34s}" + "".join(f"{n:>9s}" for n in names))
for i in range(n_layers):
    vals = [sum(d[i + k * n_layers][1] for k in range(3)) / 3 for d in data]
    print(f"{data[0][i][0]:34s}" + "".join(f"{v:9.1f}" for v in vals))
print(f"{'total':34s}" + "".join(f"{sum(x for _, x in d) / 3:9.1f}" for d in data))
