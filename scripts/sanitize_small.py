"""Small calls of every device entry point, for compute-sanitizer.

  compute-sanitizer --tool memcheck python scripts/sanitize_small.py all
  compute-sanitizer --tool racecheck python scripts/sanitize_small.py render

Run by tests/test_sanitizer_gpu.py.  Sizes are tiny (sanitized kernels run
10-100x slower) but every kernel family launches: render (plain, Hi-Z seed +
pre-test passes forced by NAR_RENDER_PASS_UNITS, the host-staged path),
resolve (RGB+D fast path, the general 16-channel path, zero-copy attributes
from pinned host memory at the stream's first/last bytes), the fused
composite + resolve over several keybufs, the U-Net (head/pyramid + every
tcgen05 conv shape of a small network), the standalone gated conv, the
Gaussian-splat blend and the Morton keys.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NAR_RENDER_PASS_UNITS", "8")


def render_cases():
    import numpy as np
    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection, rasterize

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    n = 60_000 + 37  # a sub-unit tail
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    vel = rng.normal(size=(n, 3)).astype(np.float32)
    tmp = rng.normal(size=(n, 1)).astype(np.float32)
    cam = look_at((0.2, -2.2, 1.0), (0, 0, 0), Intrinsics(width=96, height=72))
    sel = StreamSelection(rgb=True, depth=True)
    full = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, scalars=("t",),
                           coverage_channel=True)
    pc = PointCloud(pos, [Stream("rgb", "u8", rgb), Stream("velocity", "f32", vel),
                          Stream("t", "f32", tmp)])
    rasterize(pc, cam, sel)             # host path, device rgb upload
    rasterize(pc, cam, full)            # general resolve
    pcp = PointCloud(pos, [Stream("rgb", "u8", rgb)], pinned=True)
    rasterize(pcp, cam, sel)            # zero-copy rgb gathers, incl. the last point's bytes
    parts = [PointCloud(pos[a:b], [Stream("rgb", "u8", rgb[a:b]), Stream("velocity", "f32", vel[a:b])])
             for a, b in ((0, 20_000), (20_000, 41_111), (41_111, n))]
    dc = DeviceCloud.from_clouds(parts, device=dev)
    r = Renderer(96, 72, device=dev, pad_multiple=16)
    for _ in range(3):                  # multi-stream Hi-Z passes (forced), stats readback
        r.rasterize(dc, cam, StreamSelection(rgb=True, depth=True, vel2d=True))
    torch.cuda.synchronize()
    return r, dc, cam


def peers_case(r, dc, cam):
    import torch

    from paper_2407_19097_b200.msr import Renderer, StreamSelection

    sel = StreamSelection(rgb=True, depth=True)
    dev = r.device
    rs = [Renderer(96, 72, device=dev, signed_keys=False, pad_multiple=16) for _ in range(3)]
    for k, rk in enumerate(rs):
        from paper_2407_19097_b200.msr import DeviceCloud

        rk.render(DeviceCloud([dc.segments[k]], dc.meta, dev), cam)
    out = rs[0].alloc_outputs(4)
    rows = out["data"].shape[0]
    for a, b in ((0, rows // 2), (rows // 2, rows)):
        rs[0].resolve(dc, cam, sel, out=out, peers=[x.keybuf.data_ptr() for x in rs], rows=(a, b))
    torch.cuda.synchronize()


def unet_cases():
    import numpy as np

    from paper_2407_19097_b200.neural import (UNetConfig, build_pyramid, forward, gated_conv,
                                              init_params)

    rng = np.random.default_rng(1)
    for base in (16, 20):
        cfg = UNetConfig(input_channels=4, base_channels=base)
        x = rng.uniform(0, 1, (1, 48, 80, 4)).astype(np.float32)
        forward(x, init_params(cfg), cfg)
    x = rng.uniform(0, 1, (40, 72, 12)).astype(np.float32)
    w = rng.normal(size=(3, 3, 12, 24)).astype(np.float32) * 0.1
    gated_conv(x, w, np.zeros(24, np.float32), w, np.ones(24, np.float32))
    build_pyramid(rng.uniform(size=(1, 32, 48, 4)).astype(np.float32), levels=5)


def misc_cases():
    import numpy as np
    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.gsplat import build_splats, prepare_splats, splat_blend_image
    from paper_2407_19097_b200.preprocess import morton_keys_device

    rng = np.random.default_rng(2)
    n = 3000
    xy = rng.uniform(-1, 1, (n, 2))
    pc = PointCloud(np.c_[xy, 0.1 * np.sin(3 * xy[:, 0])].astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8))])
    cam = look_at((0.0, -1.6, 1.2), (0, 0, 0), Intrinsics(width=80, height=60))
    mu, abc, boxes, col, op, _ = prepare_splats(build_splats(pc, "terrain"), cam)
    splat_blend_image(mu, abc, boxes, col, op, 80, 60)
    morton_keys_device(torch.from_numpy(pc.positions).cuda())
    torch.cuda.synchronize()


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    r, dc, cam = render_cases()
    if what == "all":
        peers_case(r, dc, cam)
        unet_cases()
        misc_cases()
    print("sanitize_small done:", what)


if __name__ == "__main__":
    main()
