"""Tail imbalance of the pre-test passes (library built with -DNAR_RENDER_TRACE):
renders the C2 cloud once per NAR_RENDER_MAX_PASSES setting and prints the spread of
per-warp finish times of the LAST pre-test launch of the frame."""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import bench
    from paper_2407_19097_b200 import _lib
    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    dev = torch.device("cuda", 0)
    pos, rgb = bench.make_uniform(350_000_000, dev, seed=1234)
    cloud = DeviceCloud.from_tensors(pos)
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=1920, height=1080))
    r = Renderer(1920, 1080, device=dev)
    lib = _lib.load()
    n = 148 * 24
    buf = (ctypes.c_ulonglong * n)()
    for frame in range(3):
        r.clear()
        r.render(cloud, cam)
        torch.cuda.synchronize()
    assert lib.nar_debug_render_trace(buf, n) == 0
    t = np.array(buf, dtype=np.float64)
    t = t[t > 0]
    t -= t.min()
    print(f"last pass: warps {len(t)}, finish spread {t.max() / 1e3:.1f} us, p50 {np.percentile(t, 50) / 1e3:.1f}, "
          f"p90 {np.percentile(t, 90) / 1e3:.1f}, p99 {np.percentile(t, 99) / 1e3:.1f}")


if __name__ == "__main__":
    main()
