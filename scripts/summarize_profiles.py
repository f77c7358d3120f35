"""Condense the ncu outputs of scripts/gpu_profiles.sh into profiles/ (tracked).

  python scripts/summarize_profiles.py <round-tag>

Reads gpurun_out/bench_launches.csv (gpu__time_duration + DRAM bytes of every
launch of `bench.py --steps 3 --warmup 3 --no-e2e --no-cpu`) and the --set full
captures gpurun_out/<tag>_render_full.ncu-rep / <tag>_conv_full.ncu-rep, and
writes profiles/<tag>_launches.md, profiles/<tag>_render_ncu.md,
profiles/<tag>_conv_ncu.md and profiles/render_traffic.json (per-frame DRAM
bytes of the render kernels, consumed by bench.py's roofline.traffic).
"""

import csv
import json
import subprocess
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def launches(tag):
    rows = [r for r in csv.reader(open(OUT / "bench_launches.csv")) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    by = OrderedDict()
    for r in rows[1:]:
        by.setdefault(int(r[iid]), {"name": r[ik]})[r[im]] = num(r[iv])
    seq = list(by.values())
    short = lambda n: n.split("(")[0].replace("void ", "").replace("nar::", "")
    # frames of the timed bench loop: render launches ... resolve_kernel
    frames, cur = [], []
    for k in seq:
        cur.append(k)
        if "resolve_kernel" in k["name"]:
            frames.append(cur)
            cur = []
    frame = frames[min(4, len(frames) - 1)]  # a timed raster frame (after 3 warm-ups)
    tot = sum(k["gpu__time_duration.sum"] for k in frame)
    lines = [f"# {tag}: per-launch device time of one C2 frame (ncu, cold-cache, serialised)",
             "", "Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none python bench.py --steps 3 --warmup 3 "
             "--no-e2e --no-cpu` (the pipeline frames of that command follow the raster frames).",
             "", "| # | kernel | us | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
    rt_bytes = 0.0
    for i, k in enumerate(frame):
        t = k["gpu__time_duration.sum"] / 1e3
        rd = (k.get("dram__bytes_read.sum") or 0) / 1e6
        wr = (k.get("dram__bytes_write.sum") or 0) / 1e6
        if "render" in k["name"] or "hiz_kernel" in k["name"]:
            rt_bytes += (k.get("dram__bytes_read.sum") or 0) + (k.get("dram__bytes_write.sum") or 0)
        lines.append(f"| {i} | {short(k['name'])} | {t:.1f} | {100 * k['gpu__time_duration.sum'] / tot:.1f}% | {rd:.1f} | {wr:.1f} |")
    rsum = sum(k["gpu__time_duration.sum"] for k in frame if "render" in k["name"] or "hiz" in k["name"])
    lines += ["", f"Frame total {tot / 1e3:.1f} us; render kernels (seed, pre-test passes, Hi-Z refreshes) "
              f"{rsum / 1e3:.1f} us = {100 * rsum / tot:.1f}% of the frame; their DRAM traffic "
              f"{rt_bytes / 1e9:.3f} GB per frame vs 4.200 GB algorithmic (350M x 12 B)."]
    # U-Net launches of one pipeline frame
    unet_kernel = lambda k: any(t in k["name"] for t in ("gated_conv", "head_pyramid", "pool_bf16",
                                                           "out_head"))
    starts = [i for i, k in enumerate(seq) if "head_pyramid" in k["name"]]
    last = []
    if starts:
        for k in seq[starts[-1]:]:
            if not unet_kernel(k):
                break
            last.append(k)
    if last:
        ut = sum(k["gpu__time_duration.sum"] for k in last)
        lines += ["", "## U-Net forward (last pipeline frame)", "",
                  "| kernel | us | DRAM read MB | DRAM write MB |", "|---|---|---|---|"]
        for k in last:
            lines.append(f"| {short(k['name'])} | {k['gpu__time_duration.sum'] / 1e3:.1f} | "
                         f"{(k.get('dram__bytes_read.sum') or 0) / 1e6:.1f} | "
                         f"{(k.get('dram__bytes_write.sum') or 0) / 1e6:.1f} |")
        lines.append(f"\nU-Net total {ut / 1e3:.1f} us (413.7 GFLOP -> {413.7e9 / (ut * 1e-9) / 1e12:.0f} TFLOP/s)")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    json.dump({"workload": "c2", "bytes_per_launch": rt_bytes,
               "note": f"DRAM read+write of all render launches of one C2 frame ({tag}, ncu)"},
              open(PROF / "render_traffic.json", "w"), indent=1)
    print("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"]


def full(tag, kind, title):
    rep = OUT / f"{tag}_{kind}_full.ncu-rep"
    if not rep.exists():
        return
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    d = {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}
    st = [(h, num(v[1])) for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled")
          and not h.endswith("not_issued") and num(v[1])]
    tot = sum(x for _, x in st) or 1
    lines = [f"# {tag}: {title} (ncu --set full, one launch)", "", "| metric | value | unit |",
             "|---|---|---|"]
    for k in WANT:
        if k in d:
            lines.append(f"| {k} | {d[k][1]} | {d[k][0]} |")
    lines += ["", "Top warp-stall reasons (share of sampled stalls):", ""]
    for h, x in sorted(st, key=lambda t: -t[1])[:8]:
        lines.append(f"- {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * x / tot:.1f}%")
    (PROF / f"{tag}_{kind}_ncu.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    PROF.mkdir(exist_ok=True)
    launches(tag)
    full(tag, "render", "render_pre_kernel, the last (largest) pre-test pass of a C2 frame")
    full(tag, "conv", "gated_conv_tc<32> (enc0b, level 0, 1920x1088x16 -> 16)")
