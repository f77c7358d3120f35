"""Host-side cost of one rasterize() call on the C2 cloud: cProfile of 5 calls (the
C calls' own time is GPU / DMA waiting; the rest is Python)."""
import cProfile, pstats, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2407_19097_b200 import msr
from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at

n = 350_000_000
dev = torch.device("cuda", 0)
pos, rgb = bench.make_uniform(n, dev, 1)
pc = PointCloud(pos.cpu().numpy(), [Stream("rgb", "u8", rgb.cpu().numpy())], pinned=True)
cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=1920, height=1080))
sel = msr.StreamSelection(rgb=True, depth=True)
for _ in range(3):
    fi = msr.rasterize(pc, cam, sel)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    fi = msr.rasterize(pc, cam, sel)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
