"""rasterize() stage times for a pinned PointCloud vs a stock pageable one (registered in
place by the first call): nar_render_host alone, the host rgb gather alone, and the full
call (C2: 350M points at 1080p)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_19097_b200 import _lib, msr
from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at

n = 350_000_000
dev = torch.device("cuda", 0)
pos, rgb = bench.make_uniform(n, dev, 1)
host_pos, host_rgb = pos.cpu().numpy(), rgb.cpu().numpy()
cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=1920, height=1080))
sel = msr.StreamSelection(rgb=True, depth=True)
main = torch.cuda.current_stream()
for name, pc in (("pageable", PointCloud(host_pos, [Stream("rgb", "u8", host_rgb)])),
                 ("pinned", PointCloud(host_pos, [Stream("rgb", "u8", host_rgb)], pinned=True))):
    msr.rasterize(pc, cam, sel)  # registers pageable arrays, warms pools
    r = msr._renderer_for(1920, 1080, dev)
    kc = cam.kernel_camera()
    ts = {"render_host": [], "gather": [], "rasterize": []}
    for _ in range(3):
        torch.cuda.synchronize()
        a = time.perf_counter()
        _lib.call("nar_render_host", r.keybuf.data_ptr(), pc.positions.ctypes.data, pc.count,
                  C.c_uint64(0), C.byref(kc), r.domain, int(main.cuda_stream))
        main.synchronize()
        ts["render_host"].append((time.perf_counter() - a) * 1e3)
        a = time.perf_counter()
        msr._host_gather(r, pc, sel, main, msr._keys_to_host(r, main))
        main.synchronize()
        ts["gather"].append((time.perf_counter() - a) * 1e3)
        r.clear()
        a = time.perf_counter()
        msr.rasterize(pc, cam, sel)
        ts["rasterize"].append((time.perf_counter() - a) * 1e3)
    print(name, {k: round(min(v), 2) for k, v in ts.items()},
          "pos ptr % 4096 =", pc.positions.ctypes.data % 4096, flush=True)
