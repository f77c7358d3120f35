"""profiles/<tag>_render_ncu.md from gpurun_out/rprof_<w>.csv (scripts/gpu_render_prof.sh):
the last frame's render passes + resolve with DRAM bytes and the L2 reduction / read counters."""
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WL = {"c2": ("C2: 350M uniform points, 1920x1080, storage order", 350e6),
      "c4": ("C4: 350M terrain points (oblique), 1920x1080, storage order", 350e6),
      "c5": ("C5 per-GPU shard at N=8: 250M uniform points, 3840x2160", 250e6)}


def load(f):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
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
    # frames end with the resolve; keep the last frame
    ends = [i for i, k in enumerate(seq) if "resolve" in k["name"]]
    start = ends[-2] + 1 if len(ends) > 1 else 0
    return seq[start:ends[-1] + 1]


def main(tag):
    out = [f"# {tag}: render passes of one frame -- DRAM and L2 traffic of the keybuf fold", "",
           "`ncu --metrics ... --clock-control none` on `bench.py --steps 1 --warmup 3` (the last, "
           "timed frame; serialised, cold cache). RED = `lts__t_sectors_op_red` (the fire-and-forget "
           "`atomicMin` of _native.pyx:76-77 lands in L2 as a reduction), RED req = "
           "`lts__t_requests_srcunit_tex_op_red`, SM reads = `lts__t_sectors_srcunit_tex_op_read` "
           "(L2 sectors read by loads issued from the SMs: keybuf early-z, coarse depth; the TMA point "
           "stream is not in it), hit % = `lts__t_sector_hit_rate`, fp64 % = "
           "`sm__pipe_fp64_cycles_active`. G/s columns are per second of that launch.", ""]
    for w, (desc, npts) in WL.items():
        f = ROOT / "gpurun_out" / f"rprof_{w}.csv"
        if not f.exists():
            continue
        seq = load(f)
        out += [f"## {desc}", "",
                "| # | kernel | us | DRAM rd MB | DRAM rd GB/s | RED sectors (M) | RED G/s | RED req (M) | SM reads (M sectors) | SM reads G/s | L2 hit % | issue % | fp64 % |",
                "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        tot_t = tot_rd = tot_red = tot_rds = 0.0
        for i, k in enumerate(seq):
            t = k.get("gpu__time_duration.sum", 0) / 1e3
            rd = k.get("dram__bytes_read.sum", 0) / 1e6
            red = k.get("lts__t_sectors_op_red.sum", 0) / 1e6
            req = k.get("lts__t_requests_srcunit_tex_op_red.sum", 0) / 1e6
            rds = k.get("lts__t_sectors_srcunit_tex_op_read.sum", 0) / 1e6
            nm = k["name"].split("(")[0].replace("void ", "")
            if "resolve" not in nm:
                tot_t += t
                tot_rd += rd
                tot_red += red
                tot_rds += rds
            g = (lambda x: x / t * 1e3) if t else (lambda x: 0.0)  # M per us -> G/s
            out.append(f"| {i} | {nm} | {t:.1f} | {rd:.1f} | {rd / t * 1e3 if t else 0:.0f} | "
                       f"{red:.2f} | {g(red):.1f} | {req:.2f} | {rds:.2f} | {g(rds):.1f} | "
                       f"{k.get('lts__t_sector_hit_rate.pct', 0):.1f} | "
                       f"{k.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                       f"{k.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):.0f} |")
        alg = npts * 12 / 1e6
        out += ["", f"Render (all passes + Hi-Z refreshes): {tot_t:.1f} us, DRAM read {tot_rd:.0f} MB vs "
                f"{alg:.0f} MB algorithmic ({tot_rd / alg:.2f}x), {alg / tot_t:.2f} TB/s algorithmic "
                f"= {alg / tot_t / 6.5533:.2f} of the measured 6553 GB/s; {tot_red:.1f}M RED sectors "
                f"({tot_red / tot_t * 1e3:.0f} G/s averaged over the render), {tot_rds:.1f}M SM-read sectors "
                f"({tot_rds / tot_t * 1e3:.0f} G/s).", ""]
    (ROOT / "profiles" / f"{tag}_render_ncu.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
