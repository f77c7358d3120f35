"""Per-layer U-Net table from ncu launch lists: python scripts/unet_table.py gpurun_out/unet_it_d0.csv [more.csv ...]"""
import csv
import sys

NAMES = ["head", "enc0a", "enc0b", "enc1a", "enc1b", "enc2a", "enc2b", "enc3a", "enc3b", "enc4a",
         "enc4b", "dec3a", "dec3b", "dec2a", "dec2b", "dec1a", "dec1b", "dec0a", "dec0b"]


def load(f):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    by = {}
    for r in rows[1:]:
        by.setdefault(int(r[iid]), {"name": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
    seq = list(by.values())
    st = [i for i, k in enumerate(seq) if "head_pyramid" in k["name"]]
    return seq[st[-1]:]


ds = [load(f) for f in sys.argv[1:]]
tot = [0.0] * len(ds)
for j, k in enumerate(ds[0]):
    t = [d[j]["gpu__time_duration.sum"] / 1e3 for d in ds]
    tot = [a + b for a, b in zip(tot, t)]
    nm = k["name"].split("(")[0].replace("void nar::", "").replace("void ", "")
    print(f"{(NAMES[j] if j < len(NAMES) else '?'):6s} {nm[:26]:26s} " + " ".join(f"{x:6.1f}" for x in t)
          + f"  tc%={k.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}"
          f" iss%={k.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}"
          f" rd={k.get('dram__bytes_read.sum', 0) / 1e6:6.1f} wr={k.get('dram__bytes_write.sum', 0) / 1e6:6.1f}")
print("total", " ".join(f"{x:6.1f}" for x in tot))
