"""profiles/<tag>_full_ncu.md from the `ncu --set full` captures of scripts/gpu_r02_full.sh
(gpurun_out/full_*.ncu-rep): speed-of-light, memory, issue and occupancy figures, the top
stall reasons (source page) and the dram traffic of each captured launch."""
import csv
import io
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CAPS = [("full_c2_pre", "C2: last pre-test render pass (122M points, 1080p)"),
        ("full_c4_tma", "C4: a dense exact-kernel render pass (122M terrain points)"),
        ("full_dec0a", "U-Net dec0a (gated_conv_tc<32>, 1920x1088, 3 chunks incl. paired up2)"),
        ("full_dec0b", "U-Net dec0b (gated_conv_tc<32> with the fused out head, 1920x1088)"),
        ("full_enc1b", "U-Net enc1b (gated_conv_tc<64>, 960x544)")]
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Issued Ipc Active", "SM Busy",
        "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "L2 Hit Rate"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", str(rep), *args], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    out = {}
    for r in rows[1:]:
        if len(r) > h.index("Metric Value"):  # (rows without rule columns are shorter)
            out.setdefault(r[h.index("Metric Name")], (r[h.index("Metric Value")], r[h.index("Metric Unit")]))
    return out, rows[1][h.index("Kernel Name")] if len(rows) > 1 else "?"


def raw(rep, names):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h = rows[0]
    return {n: f"{rows[2][h.index(n)]} {rows[1][h.index(n)]}" if n in h else "" for n in names}


def stalls(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(rows) < 3:
        return ""
    h = rows[1]
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = Counter()
    for r in rows[2:]:
        if len(r) == len(h) and r[0] != "Address":
            for c in reasons:
                try:
                    tot[c] += float(r[h.index(c)])
                except ValueError:
                    pass
    s = sum(tot.values()) or 1.0
    return ", ".join(f"{k[6:]} {v / s * 100:.0f} %" for k, v in tot.most_common(5))


def main(tag):
    out = [f"# {tag}: `ncu --set full` captures of the dominant kernels (one launch each)", "",
           "`scripts/gpu_r02_full.sh` (`--clock-control none --import-source on`); figures from "
           "`ncu -i <rep> --page details/raw/source`. Serialised, cold-cache single launches: the "
           "bench lines' CUDA-event times are the live numbers.", ""]
    for name, what in CAPS:
        rep = ROOT / "gpurun_out" / f"{name}.ncu-rep"
        if not rep.exists():
            continue
        d, kname = details(rep)
        rw = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum"])
        out += [f"## {what}", "", f"`{kname[:110]}`", "", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in d:
                out.append(f"| {k} | {d[k][0]} {d[k][1]} |")
        out.append(f"| DRAM read / write | {rw['dram__bytes_read.sum']} / {rw['dram__bytes_write.sum']} |")
        st = stalls(rep)
        if st:
            out.append(f"| top stall reasons (warp samples) | {st} |")
        out.append("")
    (ROOT / "profiles" / f"{tag}_full_ncu.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
