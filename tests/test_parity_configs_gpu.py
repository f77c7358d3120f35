"""Parity at the configurations bench.py times (BASELINE.json configs C3, C4).

* C4's U-Net: the full 1920x1088 frame of a rendered terrain G-buffer through
  the tcgen05 network vs the f32 oracle forward (oracle.forward restates
  neural/model.py:194-204 and the conv of neural/autodiff.py:267-288) --
  PSNR >= 50 dB and max |err| <= 2e-2 (bf16 operands, f32 accumulation).
* C3's render: 4 x 100M Lagrangian-like points in 4 device buffers rendered
  concurrently on 4 CUDA streams (Hi-Z multi-pass schedule engaged on every
  buffer, one shared coarse-depth scratch) vs the oracle render + resolve of
  the concatenated cloud with base indices 0, 100M, 200M, 300M
  (_kernels/__init__.py:81-87): bit-exact keybuf, planes and rgb/d channels,
  vel2d within 1 f32 ulp.
* The same 4-stream schedule forced onto small buffers (NAR_RENDER_PASS_UNITS),
  across several scenes.
"""

import os

import numpy as np
import pytest

import oracle
from conftest import ulp_diff_f32

pytestmark = pytest.mark.gpu

PSNR_MIN = 50.0
MAX_ABS = 2e-2
THREADS = os.cpu_count() or 4


def _terrain_gbuffer(dev, n=40_000_000):
    """RGB+D G-buffer of a C4-style terrain (bench.make_terrain, oblique camera)
    at 1920x1080, padded to 1920x1088 by the resolve (pad_to_multiple(16))."""
    import bench
    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    pos, rgb = bench.make_terrain(n, dev, seed=1234)
    cloud = DeviceCloud.from_tensors(pos, {"rgb": rgb})
    cam = look_at((0.0, -1.6, 1.2), (0, 0, 0), Intrinsics(width=1920, height=1080))
    r = Renderer(1920, 1080, device=dev, pad_multiple=16)
    img = r.rasterize(cloud, cam, StreamSelection(rgb=True, depth=True))
    return img.data  # (1088, 1920, 4) f32 on the device


def test_unet_c4_frame_vs_f32_oracle(cuda):
    import torch

    from paper_2407_19097_b200.neural import UNet, UNetConfig, init_params

    x = _terrain_gbuffer(cuda)
    assert tuple(x.shape) == (1088, 1920, 4)
    cov = float((x[..., 3] > 0).float().mean())
    # the oblique C4 view: terrain fills the lower ~40 % of the frame, sky above
    assert cov > 0.3, f"terrain G-buffer covers only {cov:.2f} of the frame"
    cfg = UNetConfig(input_channels=4)  # C4: random init, init_seed=0
    params = init_params(cfg)
    net = UNet(cfg, params, device=cuda)
    y = torch.empty((1088, 1920, 3), dtype=torch.float32, device=cuda)
    net.forward_into(x, y)
    y = y.cpu().numpy()
    ref = oracle.forward(x.cpu().numpy()[None], params, cfg)[0]
    err = np.abs(y - ref)
    p = oracle.psnr(y, ref)
    assert p >= PSNR_MIN, f"PSNR {p:.1f} dB"
    assert float(err.max()) <= MAX_ABS, f"max |err| {float(err.max()):.3g}"


def _c3_parts(dev, per_stream, steps=100):
    import bench

    parts = []
    for s in range(4):
        p, c, v = bench.make_trajectories(per_stream, dev, seed=s)
        parts.append((p, c, v))
    return parts


def _check_multistream(dev, parts, cam, frames=2):
    import torch

    from paper_2407_19097_b200.geometry import PointCloud, Stream
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection, _StreamMeta

    segs, begin = [], 0
    for p, c, v in parts:
        segs.append({"begin": begin, "positions": p, "streams": {"rgb": c, "velocity": v}})
        begin += int(p.shape[0])
    meta = {"rgb": _StreamMeta("rgb", "u8", 3), "velocity": _StreamMeta("velocity", "f32", 3)}
    cloud = DeviceCloud(segs, meta, dev)
    sel = StreamSelection(rgb=True, depth=True, vel2d=True)
    W, H = cam.intrinsics.width, cam.intrinsics.height
    r = Renderer(W, H, device=dev)
    whole = PointCloud(torch.cat([p for p, _, _ in parts]).cpu().numpy(),
                       [Stream("rgb", "u8", torch.cat([c for _, c, _ in parts]).cpu().numpy()),
                        Stream("velocity", "f32", torch.cat([v for _, _, v in parts]).cpu().numpy())])
    ref = oracle.rasterize(whole, cam, sel, threads=THREADS)
    for _ in range(frames):  # later frames: pass statistics may switch kernels
        r.render(cloud, cam)  # 4 buffers, 4 CUDA streams, one shared Hi-Z scratch
        assert np.array_equal(r.keys(), ref["keybuf"])
        img = r.resolve(cloud, cam, sel).to_host()
        torch.cuda.synchronize()
        assert np.array_equal(img.index_plane, ref["index_plane"])
        assert np.array_equal(img.depth, ref["depth"])
        assert np.array_equal(img.data[..., :4], ref["data"][..., :4])
        assert ulp_diff_f32(img.data[..., 4:], ref["data"][..., 4:]).max() <= 1


def test_c3_full_scale_multistream_hiz(cuda):
    """The benched C3 frame: 4 x 100M points, 1080p, RGB+D+Vel2D."""
    from paper_2407_19097_b200.geometry import Intrinsics, look_at

    parts = _c3_parts(cuda, 100_000_000)
    cam = look_at((0.0, -2.6, 1.4), (0, 0, 0), Intrinsics(width=1920, height=1080))
    _check_multistream(cuda, parts, cam)


@pytest.mark.parametrize("scene", range(4))
def test_multistream_hiz_forced_small(cuda, scene, monkeypatch):
    """Four concurrent buffers with the seed + pre-test passes forced on small
    clouds (NAR_RENDER_PASS_UNITS), random cameras incl. inside the cloud."""
    import bench
    from paper_2407_19097_b200.geometry import Intrinsics, look_at

    monkeypatch.setenv("NAR_RENDER_PASS_UNITS", "40")
    rng = np.random.default_rng(100 + scene)
    parts = []
    for s in range(4):
        n = int(rng.integers(300_000, 900_000)) // 100 * 100
        parts.append(bench.make_trajectories(n, cuda, seed=10 * scene + s))
    eye = tuple(float(v) for v in rng.uniform(-2.5, 2.5, 3))
    if scene == 3:
        eye = (0.1, 0.05, 0.0)  # inside the cloud
    W, H = int(rng.integers(64, 700)), int(rng.integers(64, 500))
    cam = look_at(eye, (0, 0, 0), Intrinsics(fov_y_deg=float(rng.uniform(30, 100)),
                                                width=W, height=H))
    _check_multistream(cuda, parts, cam, frames=3)
