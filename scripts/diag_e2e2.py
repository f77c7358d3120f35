"""Stage times of rasterize() on pinned host buffers (C2): render_host, resolve
with zero-copy attribute gathers, D2H of the FeatureImage, host clone."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_19097_b200 import _lib
from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
from paper_2407_19097_b200.msr import (DeviceCloud, StreamSelection, _Mapped, _StreamMeta,
                                       _renderer_for)

n = 350_000_000
dev = torch.device("cuda", 0)
pos, rgb = bench.make_uniform(n, dev, 1)
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pos)
hr = torch.empty((n, 3), dtype=torch.uint8, pin_memory=True); hr.copy_(rgb)
cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=1920, height=1080))
r = _renderer_for(1920, 1080, dev)
kc = cam.kernel_camera()
sel = StreamSelection(rgb=True, depth=True)
main = torch.cuda.current_stream()
mp = _lib.mapped_pointer(hr.numpy().ctypes.data)
meta = {"rgb": _StreamMeta("rgb", "u8", 3)}
for mode in ("mapped", "device"):
    streams = {"rgb": _Mapped(mp, (n, 3)) if mode == "mapped" else rgb}
    cloud = DeviceCloud([{"begin": 0, "count": n, "positions": None, "streams": streams}], meta, dev)
    for it in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        _lib.call("nar_render_host", r.keybuf.data_ptr(), hp.numpy().ctypes.data, n, C.c_uint64(0),
                  C.byref(kc), r.domain, int(main.cuda_stream))
        ev[1].record()
        res = r.resolve(cloud, cam, sel, stream=main)
        ev[2].record()
        host = {k: torch.empty(getattr(res, k).shape, dtype=getattr(res, k).dtype, pin_memory=True)
                for k in ("data", "coverage", "index_plane", "depth")}
        for k in host:
            host[k].copy_(getattr(res, k), non_blocking=True)
        ev[3].record()
        main.synchronize()
        t = time.perf_counter()
        own = {k: host[k].clone().numpy() for k in host}
        tc = (time.perf_counter() - t) * 1e3
        print(mode, "render_host %.2f resolve %.2f d2h %.2f clone %.2f ms" % (
            ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), tc))
