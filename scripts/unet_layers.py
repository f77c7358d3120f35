"""Print per-launch times of the last U-Net forward in gpurun_out/unet_launches.csv."""
import csv
rows = [r for r in csv.reader(open("gpurun_out/unet_launches.csv")) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
by = {}
for r in rows[1:]:
    by.setdefault(int(r[iid]), {"name": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
seq = list(by.values())
starts = [i for i, k in enumerate(seq) if "head_pyramid" in k["name"]]
last = seq[starts[-1]:]
tot = 0
for k in last:
    t = k["gpu__time_duration.sum"] / 1e3
    tot += t
    print(f"{k['name'].split('(')[0].replace('void nar::', ''):40s} {t:7.1f} us  rd {k.get('dram__bytes_read.sum', 0) / 1e6:6.1f} MB  wr {k.get('dram__bytes_write.sum', 0) / 1e6:6.1f} MB")
print(f"total {tot:.1f} us")
