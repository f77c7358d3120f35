import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
        return cache[name]

    return load


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    # the product must load its own library on a GPU box -- never fall back
    from paper_2407_19097_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)


def random_case(golden, ci):
    """Product-side PointCloud / camera / selection for golden random case ci."""
    from paper_2407_19097_b200.geometry import CameraPose, Intrinsics, PointCloud, Stream
    from paper_2407_19097_b200.msr import StreamSelection

    g = golden("raster_random")
    p = f"c{ci}/"
    W, H = (int(v) for v in g[p + "wh"])
    pc = PointCloud(g[p + "positions"], [Stream("rgb", "u8", g[p + "rgb"]),
                                         Stream("velocity", "f32", g[p + "velocity"]),
                                         Stream("temp", "f32", g[p + "temp"]),
                                         Stream("mask", "u8", g[p + "mask"])])
    cam = CameraPose(g[p + "campos"], g[p + "R"],
                     Intrinsics(fov_y_deg=float(g[p + "fov"]), width=W, height=H))
    sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, scalars=("temp", "mask"),
                          coverage_channel=True, velocity_scale=float(g[p + "velocity_scale"]))
    return pc, cam, sel, g, p


def ulp_diff_f32(a, b):
    """Elementwise distance in f32 ulps (monotone integer mapping)."""
    ai = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    bi = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi)
