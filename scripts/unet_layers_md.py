"""profiles/<tag>_unet_layers.md from the U-Net probe launch lists (scripts/gpu_unet_iter.sh):
gpurun_out/unet_it_d{0,3,5,6}.csv = normal / loads only / MMAs only / epilogue only."""
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
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


def shapes(W=1920, H=1088, cin=4):
    w = [16, 32, 64, 128, 128]
    out = {}
    for k in range(5):
        px = (W >> k) * (H >> k)
        ci = cin if k == 0 else w[k - 1] + cin
        # algorithmic bf16 bytes: inputs read once, output once, + pooled output
        pool = px // 4 * w[k] * 2 if k < 4 else 0
        inb = px * (cin if k == 0 else cin) * 2 + (px // 4 * 4 * w[k - 1] * 2 // 4 if k else 0)
        out[f"enc{k}a"] = (px, ci, w[k], px * ci * 2 + px * w[k] * 2)
        out[f"enc{k}b"] = (px, w[k], w[k], px * w[k] * 2 * 2 + pool)
    for k in range(3, -1, -1):
        px = (W >> k) * (H >> k)
        up = px // 4 * w[k + 1] * 2
        out[f"dec{k}a"] = (px, w[k + 1] + w[k], w[k], up + px * w[k] * 2 + px * w[k] * 2)
        out[f"dec{k}b"] = (px, w[k], w[k], px * w[k] * 2 + (px * 3 * 4 if k == 0 else px * w[k] * 2))
    return out


def main(tag):
    d = {m: load(ROOT / "gpurun_out" / f"unet_it_d{m}.csv") for m in (0, 3, 5, 6)}
    sh = shapes()
    lines = [f"# {tag}: U-Net forward at 1920x1088 (C4 CNN stage), per layer", "",
             "ncu launch lists of `scripts/prof_unet.py --frames 1` (`--clock-control none`, serialised, "
             "cold cache): `gpu__time_duration`, `sm__pipe_tensor_cycles_active` (% of peak, active "
             "cycles), DRAM read+write vs the algorithmic bf16 bytes (inputs read once, outputs written "
             "once). The last three columns time the same launch with parts of the pipeline switched "
             "off (`NAR_TC_DEBUG`, timing only): loads only (TMA halo + weights), MMAs only, epilogue "
             "only. GFLOP = 2*M*K*N of the gated conv (K = 9*Cin, N = 2*Cout); TF/s against 1626 "
             "(burst bf16, MEASURED_PEAKS.json).", "",
             "| layer | kernel | M px | K | N | GFLOP | us | TF/s | tensor % | DRAM MB | algo MB | loads-only us | MMA-only us | epilogue-only us |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    tot = {"t": 0, "gf": 0, "t3": 0, "t5": 0, "t6": 0, "dram": 0, "algo": 0}
    for j, k in enumerate(d[0]):
        nm = NAMES[j]
        kn = k["name"].split("(")[0].replace("void nar::", "").replace("void ", "").replace("nar::", "")
        t = k["gpu__time_duration.sum"] / 1e3
        dram = (k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)) / 1e6
        tc = k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0)
        t3, t5, t6 = (d[m][j]["gpu__time_duration.sum"] / 1e3 for m in (3, 5, 6))
        tot["t"] += t
        tot["dram"] += dram
        if nm == "head":
            lines.append(f"| head+pyramid | {kn} | 2088960 | - | - | - | {t:.1f} | - | - | {dram:.1f} | 62.7 | - | - | - |")
            tot["algo"] += 62.7
            continue
        px, ci, co, ab = sh[nm]
        gf = 2 * px * 9 * ci * 2 * co / 1e9
        tot["gf"] += gf
        tot["algo"] += ab / 1e6
        tot["t3"] += t3
        tot["t5"] += t5
        tot["t6"] += t6
        lines.append(f"| {nm} | {kn} | {px} | {9 * ci} | {2 * co} | {gf:.1f} | {t:.1f} | "
                     f"{gf / t * 1e3:.0f} | {tc:.0f} | {dram:.1f} | {ab / 1e6:.1f} | {t3:.1f} | {t5:.1f} | {t6:.1f} |")
    lines.append(f"| **total** | | | | | {tot['gf']:.1f} | {tot['t']:.1f} | {tot['gf'] / tot['t'] * 1e3:.0f} | | "
                 f"{tot['dram']:.0f} | {tot['algo']:.0f} | {tot['t3']:.0f} | {tot['t5']:.0f} | {tot['t6']:.0f} |")
    (ROOT / "profiles" / f"{tag}_unet_layers.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
