"""Profiling driver: C2-sized render (+ resolve) frames on the device path,
timed with CUDA events.  Used under ncu (one GPU) and for quick A/B runs.

  python scripts/prof_render.py [--points N] [--frames F] [--sorted] [--terrain] [--unet]
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=350_000_000)
    ap.add_argument("--frames", type=int, default=5)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--sorted", action="store_true", help="pixel-coherent (sorted) point order")
    ap.add_argument("--unet", action="store_true")
    ap.add_argument("--terrain", action="store_true", help="C4 height-field cloud and camera")
    ap.add_argument("--morton", action="store_true", help="Morton-reorder the cloud first")
    ap.add_argument("--no-hiz", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    dev = torch.device("cuda", 0)
    gen = bench.make_terrain if args.terrain else bench.make_uniform
    pos, rgb = gen(args.points, dev, 1234)
    if args.sorted:
        key = ((pos[:, 0] + 1) * 1023).long() * 4096 + ((pos[:, 2] + 1) * 1023).long()
        order = torch.argsort(key)
        pos, rgb = pos[order].contiguous(), rgb[order].contiguous()
        del order, key
    cloud = DeviceCloud.from_tensors(pos, {"rgb": rgb})
    if args.morton:
        from paper_2407_19097_b200.preprocess import morton_reorder

        cloud = morton_reorder(cloud)
        del pos, rgb
    eye = (0.0, -1.6, 1.2) if args.terrain else (0.0, -2.2, 1.0)
    cam = look_at(eye, (0, 0, 0), Intrinsics(width=args.width, height=args.height))
    r = Renderer(args.width, args.height, device=dev, pad_multiple=16)
    r.use_hiz = not args.no_hiz
    sel = StreamSelection(rgb=True, depth=True)
    out = r.alloc_outputs(4)
    net = None
    if args.unet:
        from paper_2407_19097_b200.neural import UNet, UNetConfig, init_params

        cfg = UNetConfig(input_channels=4)
        net = UNet(cfg, init_params(cfg), device=dev)
        y = torch.empty(out["data"].shape[:2] + (3,), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    ts = []
    for f in range(args.frames):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        r.render(cloud, cam)
        e[1].record()
        r.resolve(cloud, cam, sel, out=out)
        e[2].record()
        if net is not None:
            net.forward_into(out["data"], y)
        e[3].record()
        torch.cuda.synchronize()
        ts.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])))
    for t in ts:
        print(f"render {t[0]:.3f} ms  resolve {t[1]:.3f} ms  unet {t[2]:.3f} ms  "
              f"-> {args.points / t[0] / 1e6:.1f} Gpts/s render")


if __name__ == "__main__":
    main()
