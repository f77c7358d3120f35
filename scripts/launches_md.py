"""profiles/<tag>_launches.md from gpurun_out/ev_launches.csv (scripts/gpu_r02_evidence.sh):
per-launch device time and DRAM bytes of one C2 frame and one U-Net forward."""
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(tag):
    rows = [r for r in csv.reader(open(ROOT / "gpurun_out" / "ev_launches.csv")) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    by = {}
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        by.setdefault(int(r[iid]), {"name": r[ik]})[r[im]] = v
    seq = list(by.values())
    names = [k["name"].split("(")[0].replace("void ", "").replace("nar::", "") for k in seq]
    hp = [i for i, n in enumerate(names) if "head_pyramid" in n]
    res = [i for i, n in enumerate(names) if "resolve" in n and (not hp or i < hp[0])]
    end, start = res[-1], res[-2] + 1
    out = [f"# {tag}: per-launch device time of one C2 frame and one U-Net forward (ncu, cold-cache, serialised)", "",
           "Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
           "--clock-control none python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-gsplat "
           "--no-parity` (the pipeline frames of that command follow the raster frames). Shares are of "
           "the serialised launch list; the bench line's CUDA-event times are the live numbers.", "",
           "| # | kernel | us | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
    tot = sum(seq[i]["gpu__time_duration.sum"] for i in range(start, end + 1)) / 1e3
    rend = rbytes = 0.0
    for j, i in enumerate(range(start, end + 1)):
        k = seq[i]
        t = k["gpu__time_duration.sum"] / 1e3
        if "resolve" not in names[i] and "fill" not in names[i]:
            rend += t
            rbytes += k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        out.append(f"| {j} | {names[i]} | {t:.1f} | {t / tot * 100:.1f}% | "
                   f"{k['dram__bytes_read.sum'] / 1e6:.1f} | {k['dram__bytes_write.sum'] / 1e6:.1f} |")
    out += ["", f"Frame total {tot:.1f} us; render kernels (seed, pre-test passes, Hi-Z refreshes) {rend:.1f} us "
            f"= {rend / tot * 100:.1f}% of the frame; their DRAM traffic {rbytes / 1e9:.3f} GB per frame vs "
            "4.200 GB algorithmic (350M x 12 B).", ""]
    u0, ut = hp[-1], 0.0
    out += ["## U-Net forward (last pipeline frame)", "", "| kernel | us | DRAM read MB | DRAM write MB |",
            "|---|---|---|---|"]
    for i in range(u0, min(u0 + 19, len(seq))):
        k = seq[i]
        t = k["gpu__time_duration.sum"] / 1e3
        ut += t
        out.append(f"| {names[i]} | {t:.1f} | {k['dram__bytes_read.sum'] / 1e6:.1f} | "
                   f"{k['dram__bytes_write.sum'] / 1e6:.1f} |")
    out += ["", f"U-Net launches total {ut:.1f} us serialised (CUDA events in the bench line: "
            "pipeline.unet_ms_median; programmatic dependent launch overlaps each conv's prologue with "
            "the previous one's tail, which a serialised ncu list cannot show).", ""]
    (ROOT / "profiles" / f"{tag}_launches.md").write_text("\n".join(out))
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
