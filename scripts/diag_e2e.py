"""Break down the e2e rasterize() time on pinned host buffers."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_19097_b200 import _lib
from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
from paper_2407_19097_b200.msr import StreamSelection, rasterize, _renderer_for

n = 350_000_000
dev = torch.device("cuda", 0)
pos, rgb = bench.make_uniform(n, dev, 1)
hp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True); hp.copy_(pos)
hr = torch.empty((n, 3), dtype=torch.uint8, pin_memory=True); hr.copy_(rgb)
print("pinned?", hp.is_pinned(), torch.from_numpy(hp.numpy()).is_pinned())
def t(f, k=3):
    f(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k * 1e3
print("torch H2D pos ms", t(lambda: pos.copy_(hp, non_blocking=True)))
print("torch H2D pos via from_numpy ms", t(lambda: torch.from_numpy(hp.numpy()).to(dev, non_blocking=True)))
print("torch H2D rgb via from_numpy ms", t(lambda: torch.from_numpy(hr.numpy()).to(dev, non_blocking=True)))
cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=1920, height=1080))
r = _renderer_for(1920, 1080, dev)
kc = cam.kernel_camera()
def rh():
    _lib.call("nar_render_host", r.keybuf.data_ptr(), hp.numpy().ctypes.data, n, C.c_uint64(0), C.byref(kc), 0, int(torch.cuda.current_stream().cuda_stream))
print("nar_render_host ms", t(rh))
pc = PointCloud.__new__(PointCloud)
pc.positions, pc.pinned = hp.numpy(), True
s = Stream.__new__(Stream); s.name, s.format, s.data = "rgb", "u8", hr.numpy()
pc.streams = [s]
sel = StreamSelection(rgb=True, depth=True)
print("rasterize ms", t(lambda: rasterize(pc, cam, sel)))
import cProfile, pstats
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(2): rasterize(pc, cam, sel)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
