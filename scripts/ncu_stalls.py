"""Summarise an `ncu --page source --csv --print-source sass` export: stall
reasons over the kernel and the hottest SASS lines with their top reasons."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
seen, data = set(), []
for r in rows[2:]:
    if len(r) == len(hdr) and r[0] != "Address" and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
f = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for h in reasons:
        tot[h] += f(r[hdr.index(h)])
allv = sum(tot.values())
print("stall reasons (% of samples):", ", ".join(f"{k[6:]} {v / allv * 100:.1f}" for k, v in tot.most_common(10)))
i_s = hdr.index("Warp Stall Sampling (All Samples)")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for r in sorted(data, key=lambda r: -f(r[i_s]))[:n]:
    c = Counter({h[6:]: f(r[hdr.index(h)]) for h in reasons})
    top = ", ".join(f"{k} {v:.0f}" for k, v in c.most_common(2) if v)
    print(f"{r[0][-5:]} {f(r[i_s]) / allv * 100:5.1f}%  {r[1][:70]:70s} {top}")
