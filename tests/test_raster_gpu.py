"""Parity of the CUDA MSR path (render + resolve) against the reference.

Golden fixtures come from the real reference (tests/golden/make_golden.py);
larger randomized sweeps compare against the oracle restatement, which
tests/test_oracle.py pins to those fixtures.  Bar: bit-exact keybufs, index /
depth / coverage planes and rgb / d / scalar / coverage channels; vel2d /
vel3d channels within 1 f32 ulp (BLAS / libm ordering).
"""

import numpy as np
import pytest

import oracle
from conftest import random_case, ulp_diff_f32

pytestmark = pytest.mark.gpu

VEL = slice(4, 12)          # v2x..v3m in the full 16-channel selection
EXACT = [0, 1, 2, 3, 12, 13, 14, 15]


def check_feature_image(fi, ref_data, ref_index, ref_depth, ref_cov):
    assert np.array_equal(fi.index_plane, ref_index)
    assert np.array_equal(fi.depth, ref_depth)
    assert np.array_equal(fi.coverage, ref_cov)
    C = ref_data.shape[-1]
    if C == 16:
        assert np.array_equal(fi.data[..., EXACT], ref_data[..., EXACT])
        assert ulp_diff_f32(fi.data[..., VEL], ref_data[..., VEL]).max() <= 1
    else:
        assert np.array_equal(fi.data, ref_data)


def test_kat(cuda, golden):
    from paper_2407_19097_b200.geometry import CameraPose, Intrinsics, PointCloud, Stream
    from paper_2407_19097_b200.msr import StreamSelection, rasterize

    g = golden("raster_kat")
    cam = CameraPose(g["camera/pos"], g["camera/R"], Intrinsics(width=16, height=16))
    for name in ("empty", "depth", "tie"):
        pc = PointCloud(g[f"{name}/positions"], [Stream("rgb", "u8", g[f"{name}/rgb"])])
        fi = rasterize(pc, cam, StreamSelection(rgb=True, depth=True))
        check_feature_image(fi, g[f"{name}/data"], g[f"{name}/index_plane"], g[f"{name}/depth"],
                            g[f"{name}/coverage"])


@pytest.mark.parametrize("ci", range(6))
def test_golden_random(cuda, golden, ci):
    from paper_2407_19097_b200 import _kernels
    from paper_2407_19097_b200.msr import rasterize

    pc, cam, sel, g, p = random_case(golden, ci)
    i = cam.intrinsics
    kb = _kernels.zbuffer_render(pc.positions, cam.orientation, cam.position, i.focal_px, i.cx,
                                 i.cy, i.near, i.far, i.width, i.height)
    assert np.array_equal(kb, g[p + "keybuf"])
    fi = rasterize(pc, cam, sel)
    check_feature_image(fi, g[p + "data"], g[p + "index_plane"], g[p + "depth"], g[p + "coverage"])


@pytest.mark.parametrize("ci", [0, 3, 5])
def test_golden_random_pinned_zero_copy(cuda, golden, ci):
    """Pinned host clouds: attributes (and positions for vel2d) are read in
    place by the resolve instead of uploaded -- same framebuffers."""
    from paper_2407_19097_b200.geometry import PointCloud, Stream
    from paper_2407_19097_b200.msr import rasterize

    pc, cam, sel, g, p = random_case(golden, ci)
    pp = PointCloud(pc.positions, [Stream(s.name, s.format, s.data) for s in pc.streams],
                    pinned=True)
    fi = rasterize(pp, cam, sel)
    check_feature_image(fi, g[p + "data"], g[p + "index_plane"], g[p + "depth"], g[p + "coverage"])


def test_nonfinite(cuda, golden):
    from paper_2407_19097_b200 import _kernels
    from paper_2407_19097_b200.geometry import Intrinsics

    g = golden("raster_nonfinite")
    i = Intrinsics(width=64, height=64)
    kb = _kernels.zbuffer_render(g["positions"], g["R"], g["campos"], i.focal_px, i.cx, i.cy,
                                 i.near, i.far, 64, 64)
    assert np.array_equal(kb, g["keybuf"])


def test_c1_checksum(cuda, golden):
    """Config C1 (1M uniform, 512^2): sha256 of the reference keybuf."""
    import hashlib

    from paper_2407_19097_b200 import _kernels
    from paper_2407_19097_b200.geometry import Intrinsics, look_at

    g = golden("raster_c1_hash")
    pos = np.random.default_rng(0).uniform(-1, 1, (1_000_000, 3)).astype(np.float32)
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=512, height=512))
    i = cam.intrinsics
    kb = _kernels.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                 i.near, i.far, 512, 512)
    assert hashlib.sha256(kb.tobytes()).digest() == g["keybuf_sha256"].tobytes()


def _random_scene(seed, n, W, H):
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at

    rng = np.random.default_rng(seed)
    scale = 10.0 ** rng.uniform(-2, 3)
    pos = (rng.uniform(-1, 1, (n, 3)) * scale).astype(np.float32)
    k = n // 20
    pos[rng.integers(0, n, k)] = pos[rng.integers(0, n, k)]
    eye = rng.normal(size=3)
    eye = eye / np.linalg.norm(eye) * scale * rng.uniform(0.5, 4.0)
    cam = look_at(eye, rng.uniform(-0.2, 0.2, 3) * scale,
                  Intrinsics(fov_y_deg=rng.uniform(20, 120), width=W, height=H,
                             near=float(scale * rng.uniform(1e-4, 0.5))))
    pc = PointCloud(pos, [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8)),
                          Stream("velocity", "f32", rng.normal(size=(n, 3)) * scale)])
    return pc, cam


@pytest.mark.parametrize("seed", range(40))
def test_random_sweep_vs_oracle(cuda, seed):
    """SPEC acceptance #1 style sweep: 10^3..10^5 points, random cameras and
    scales (incl. cameras inside the cloud), bit-identical keybufs."""
    from paper_2407_19097_b200.msr import StreamSelection, rasterize

    rng = np.random.default_rng(1000 + seed)
    n = int(10 ** rng.uniform(3, 5))
    W, H = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    pc, cam = _random_scene(seed, n, W, H)
    sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, velocity_scale=2.5)
    ref = oracle.rasterize(pc, cam, sel)
    fi = rasterize(pc, cam, sel)
    assert np.array_equal(fi.index_plane, ref["index_plane"])
    assert np.array_equal(fi.depth, ref["depth"])
    assert np.array_equal(fi.data[..., :4], ref["data"][..., :4])
    assert ulp_diff_f32(fi.data[..., 4:], ref["data"][..., 4:]).max() <= 1


def test_unaligned_and_tail(cuda):
    """Views at odd offsets (no 16-byte alignment) take the non-TMA kernel;
    counts not a multiple of the tile take the tail kernel."""
    from paper_2407_19097_b200 import _kernels

    pc, cam = _random_scene(7, 50_001, 97, 61)
    i = cam.intrinsics
    buf = np.empty((pc.count + 1) * 3 + 1, np.float32)
    view = buf[1:1 + pc.count * 3].reshape(-1, 3)
    view[...] = pc.positions
    assert view.ctypes.data % 16 != 0
    args = (cam.orientation, cam.position, i.focal_px, i.cx, i.cy, i.near, i.far, 97, 61)
    ref = oracle.zbuffer_render(pc.positions, *args)
    kb = np.full(97 * 61, _kernels.EMPTY_KEY, np.uint64)
    _kernels.zbuffer_accumulate(kb, view, 0, *args)
    assert np.array_equal(kb, ref)
    assert np.array_equal(_kernels.zbuffer_render(pc.positions, *args), ref)


def test_base_index_and_accumulate_in_place(cuda):
    """zbuffer_accumulate folds into an existing buffer with a base index, like
    the reference's per-chunk calls (_kernels/__init__.py:84-87)."""
    from paper_2407_19097_b200 import _kernels

    pc, cam = _random_scene(3, 30_000, 64, 64)
    i = cam.intrinsics
    args = (cam.orientation, cam.position, i.focal_px, i.cx, i.cy, i.near, i.far, 64, 64)
    kb = np.full(64 * 64, _kernels.EMPTY_KEY, np.uint64)
    for lo, hi in [(0, 10_000), (10_000, 25_000), (25_000, 30_000)]:
        _kernels.zbuffer_accumulate(kb, np.ascontiguousarray(pc.positions[lo:hi]), lo, *args)
    assert np.array_equal(kb, oracle.zbuffer_render(pc.positions, *args))
    # index wrap: base_index above 2^32 keeps the low 32 bits
    kb2 = np.full(64 * 64, _kernels.EMPTY_KEY, np.uint64)
    _kernels.zbuffer_accumulate(kb2, pc.positions, (1 << 32) + 5, *args)
    ref2 = np.full(64 * 64, _kernels.EMPTY_KEY, np.uint64)
    oracle.zbuffer_accumulate(ref2, pc.positions, (1 << 32) + 5, *args)
    assert np.array_equal(kb2, ref2)


def test_device_multistream_equals_concatenated(cuda):
    """C3 semantics: 4 point buffers on 4 CUDA streams == rasterize of the
    concatenation with base indices 0, n0, n0+n1, ..."""
    import torch

    from paper_2407_19097_b200.geometry import PointCloud, Stream
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    parts = []
    for s in range(4):
        pc, cam = _random_scene(50, 20_000 + 1000 * s, 120, 90)
        parts.append(pc)
    allpos = np.concatenate([p.positions for p in parts])
    whole = PointCloud(allpos, [Stream("rgb", "u8", np.concatenate([p.stream("rgb").data for p in parts])),
                                Stream("velocity", "f32", np.concatenate([p.stream("velocity").data for p in parts]))])
    sel = StreamSelection(rgb=True, depth=True, vel2d=True)
    ref = oracle.rasterize(whole, cam, sel)
    dc = DeviceCloud.from_clouds(parts, device=cuda)
    r = Renderer(120, 90, device=cuda)
    for signed in (False, True):
        r = Renderer(120, 90, device=cuda, signed_keys=signed)
        for _ in range(2):  # second frame checks the fused keybuf re-clear
            img = r.rasterize(dc, cam, sel).to_host()
            torch.cuda.synchronize()
            assert np.array_equal(img.index_plane, ref["index_plane"])
            assert np.array_equal(img.data[..., :4], ref["data"][..., :4])
            assert ulp_diff_f32(img.data[..., 4:], ref["data"][..., 4:]).max() <= 1
        r.render(dc, cam)
        assert np.array_equal(r.keys(), ref["keybuf"])
        r.clear()


@pytest.mark.parametrize("order", ["storage", "sorted"])
def test_large_scale_properties(cuda, order):
    """Full-size checks (50M points at 1080p): the Hi-Z multi-pass render equals
    the single-pass render, which equals the CPU oracle on all 50M points; a
    3-shard composite (unaligned shard starts) equals the whole render."""
    import os

    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    n = 50_000_000
    g = torch.Generator(device=cuda).manual_seed(5)
    pos = torch.rand((n, 3), device=cuda, generator=g) * 2 - 1
    if order == "sorted":  # pixel-coherent order: heavy Hi-Z rejection and atomic contention
        key = ((pos[:, 0] + 1) * 1023).long() * 4096 + ((pos[:, 2] + 1) * 1023).long()
        pos = pos[torch.argsort(key)].contiguous()
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=1920, height=1080))
    hiz = Renderer(1920, 1080, device=cuda)
    hiz.render(DeviceCloud.from_tensors(pos), cam)
    kw = hiz.keys()
    plain = Renderer(1920, 1080, device=cuda)
    plain.use_hiz = False
    plain.render(DeviceCloud.from_tensors(pos), cam)
    assert np.array_equal(plain.keys(), kw)
    i = cam.intrinsics
    ref = oracle.zbuffer_render(pos.cpu().numpy(), cam.orientation, cam.position, i.focal_px, i.cx,
                                i.cy, i.near, i.far, 1920, 1080, threads=os.cpu_count() or 4)
    assert np.array_equal(kw, ref)
    parts = Renderer(1920, 1080, device=cuda)
    bounds = [0, 12_345_678, 30_000_001, n]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        parts.render(DeviceCloud.from_tensors(pos[lo:hi], begin=lo), cam)
    assert np.array_equal(parts.keys(), kw)


def test_pixel_snap_boundaries(cuda):
    """Points constructed to project exactly onto (and 1-2 ulp around) pixel
    boundaries and the image border: the certified f32 snap must defer every
    one of them to the exact f64 path (bit-exact keys)."""
    from paper_2407_19097_b200 import _kernels
    from paper_2407_19097_b200.geometry import CameraPose, Intrinsics

    W, H = 160, 120
    intr = Intrinsics(fov_y_deg=53.13010235415598, width=W, height=H)  # f ~= 120
    cam = CameraPose(np.zeros(3), np.eye(3), intr)
    f, cx, cy = intr.focal_px, intr.cx, intr.cy
    rng = np.random.default_rng(11)
    n = 200_000
    z = rng.uniform(0.5, 40.0, n)
    kx = rng.integers(-2, W + 2, n)
    ky = rng.integers(-2, H + 2, n)
    # T = cx + f*x/z + 0.5 == k  <=>  x = (k - 0.5 - cx) * z / f
    x = (kx - 0.5 - cx) * z / f
    y = (ky - 0.5 - cy) * z / f
    pos = np.stack([x, y, z], 1).astype(np.float32)
    bump = rng.integers(-2, 3, (n, 3)).astype(np.int32)
    pos = (pos.view(np.int32) + bump).view(np.float32)  # +-2 ulp jitter
    args = (cam.orientation, cam.position, f, cx, cy, intr.near, intr.far, W, H)
    ref = oracle.zbuffer_render(pos, *args, threads=4)
    assert np.array_equal(_kernels.zbuffer_render(pos, *args), ref)


@pytest.mark.parametrize("seed", range(24))
def test_hiz_pretest_multipass_vs_oracle(cuda, seed, monkeypatch):
    """The Hi-Z schedule (seed pass, then passes through the f32 pre-test with
    the dilated coarse depth) forced onto small clouds: random scales, far
    offsets from the origin, cameras inside the cloud, wide/narrow FOV,
    duplicates -- keybuf bit-identical to the oracle."""
    import os

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    monkeypatch.setenv("NAR_RENDER_PASS_UNITS", "48")
    rng = np.random.default_rng(7000 + seed)
    n = int(10 ** rng.uniform(5.3, 6.3))
    W, H = int(rng.integers(16, 640)), int(rng.integers(16, 480))
    scale = 10.0 ** rng.uniform(-2, 3)
    offset = rng.normal(size=3) * scale * (10.0 ** rng.uniform(0, 3) if seed % 3 == 0 else 0.0)
    pos = rng.uniform(-1, 1, (n, 3)) * scale
    if seed % 4 == 1:  # clustered surfaces: many near-equal depths
        pos[:, 2] = np.round(pos[:, 2] / scale * 8) / 8 * scale
    pos = (pos + offset).astype(np.float32)
    k = n // 10
    pos[rng.integers(0, n, k)] = pos[rng.integers(0, n, k)]
    eye = rng.normal(size=3)
    eye = eye / np.linalg.norm(eye) * scale * rng.uniform(0.3 if seed % 2 else 1.5, 4.0) + offset
    cam = look_at(eye, rng.uniform(-0.2, 0.2, 3) * scale + offset,
                  Intrinsics(fov_y_deg=rng.uniform(15, 130), width=W, height=H,
                             near=float(scale * rng.uniform(1e-4, 0.3))))
    import torch

    r = Renderer(W, H, device=cuda)
    r.render(DeviceCloud.from_tensors(torch.from_numpy(pos).to(cuda)), cam)
    i = cam.intrinsics
    ref = oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                i.near, i.far, W, H, threads=os.cpu_count() or 4)
    assert np.array_equal(r.keys(), ref)


def test_host_path_chunked_hiz(cuda):
    """nar_render_host over 20M host points (three 8 Mi-point staging chunks;
    chunks 2 and 3 are tested against the Hi-Z of the earlier ones) gives the
    same keybuf as the CPU oracle and as the plain single-pass device render."""
    import os

    import torch

    from paper_2407_19097_b200 import _kernels
    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    n = 20_000_000
    rng = np.random.default_rng(12)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    cam = look_at((0.3, -2.0, 0.9), (0, 0, 0), Intrinsics(width=1280, height=720))
    i = cam.intrinsics
    kb = _kernels.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                 i.near, i.far, 1280, 720)
    ref = oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                i.near, i.far, 1280, 720, threads=os.cpu_count() or 4)
    assert np.array_equal(kb, ref)  # the host path vs the CPU oracle
    plain = Renderer(1280, 720, device=cuda)
    plain.use_hiz = False
    plain.render(DeviceCloud.from_tensors(torch.from_numpy(pos).to(cuda)), cam)
    assert np.array_equal(kb, plain.keys())


def test_rasterize_thread_safe(cuda, golden):
    """Concurrent rasterize() calls (same resolution -> one cached renderer) give
    the same frames as serial calls."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2407_19097_b200.msr import rasterize

    cases = [random_case(golden, ci) for ci in (0, 1, 4)]  # all 64x64
    serial = [rasterize(pc, cam, sel).data for pc, cam, sel, _, _ in cases]
    with ThreadPoolExecutor(max_workers=6) as ex:
        futs = [ex.submit(rasterize, pc, cam, sel) for _ in range(4) for pc, cam, sel, _, _ in cases]
        got = [f.result().data for f in futs]
    for i, g in enumerate(got):
        assert np.array_equal(g, serial[i % len(cases)])


@pytest.mark.parametrize("case", ["wide_fov", "huge_width"])
def test_exact_only_paths_vs_oracle(cuda, case, monkeypatch):
    """Cameras outside the f32 pre-test bounds (170 deg FOV) or the certified-snap
    bounds (70000 px wide: every point takes the exact f64 path), through the
    forced multi-pass Hi-Z schedule -- keybufs bit-identical to the oracle."""
    import os

    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    monkeypatch.setenv("NAR_RENDER_PASS_UNITS", "48")
    rng = np.random.default_rng(99)
    n = 600_000
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    if case == "wide_fov":
        intr = Intrinsics(fov_y_deg=170.0, width=320, height=240)
    else:
        intr = Intrinsics(fov_y_deg=40.0, width=70000, height=3)
    cam = look_at((0.3, -2.5, 0.7), (0, 0, 0), intr)
    r = Renderer(intr.width, intr.height, device=cuda)
    r.render(DeviceCloud.from_tensors(torch.from_numpy(pos).to(cuda)), cam)
    i = cam.intrinsics
    ref = oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                i.near, i.far, i.width, i.height, threads=os.cpu_count() or 4)
    assert np.array_equal(r.keys(), ref)


def test_pass_kernel_choice_over_frames(cuda, monkeypatch):
    """2.5-D cloud (height field seen obliquely): most points pass the coarse
    test, so after the statistics of the first render come back the passes
    switch to the exact kernel (render 17 collects again).  Every frame of both
    choices must equal the oracle; a volumetric cloud interleaved on another
    renderer keeps its own statistics."""
    import os

    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    monkeypatch.setenv("NAR_RENDER_PASS_UNITS", "48")
    rng = np.random.default_rng(5)
    n = 900_000
    xy = rng.uniform(-1, 1, (n, 2))
    z = 0.15 * np.sin(3 * xy[:, 0]) * np.cos(2 * xy[:, 1])
    terrain = np.column_stack([xy, z]).astype(np.float32)
    volume = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    cam = look_at((0.0, -1.6, 1.2), (0, 0, 0), Intrinsics(width=320, height=200))
    i = cam.intrinsics
    refs, rends, clouds = [], [], []
    for pos in (terrain, volume):
        refs.append(oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx,
                                          i.cy, i.near, i.far, 320, 200,
                                          threads=os.cpu_count() or 4))
        rends.append(Renderer(320, 200, device=cuda))
        clouds.append(DeviceCloud.from_tensors(torch.from_numpy(pos).to(cuda)))
    for frame in range(20):
        for r, c, ref in zip(rends, clouds, refs):
            r.clear()
            r.render(c, cam)
            assert np.array_equal(r.keys(), ref), frame
            torch.cuda.synchronize()  # lets the statistics copy land


@pytest.mark.parametrize("W,H", [(3840, 2160), (7680, 4320)])
def test_hiz_large_frames_multipass(cuda, monkeypatch, W, H):
    """4K and 8K frames take 16- and 32-pixel coarse blocks (vectorised Hi-Z row
    scans of 9 and 17 loads); the forced multi-pass schedule must stay exact."""
    import os

    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    monkeypatch.setenv("NAR_RENDER_PASS_UNITS", "96")
    rng = np.random.default_rng(W)
    n = 1_500_000
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    pos[: n // 2, 2] = np.round(pos[: n // 2, 2] * 4) / 4  # layered surfaces
    cam = look_at((0.2, -2.4, 0.9), (0, 0, 0), Intrinsics(width=W, height=H))
    i = cam.intrinsics
    ref = oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                i.near, i.far, W, H, threads=os.cpu_count() or 4)
    r = Renderer(W, H, device=cuda)
    c = DeviceCloud.from_tensors(torch.from_numpy(pos).to(cuda))
    for _ in range(2):  # the second render may switch passes to the exact kernel
        r.clear()
        r.render(c, cam)
        torch.cuda.synchronize()
        assert np.array_equal(r.keys(), ref)


def test_resolve_rejects_mismatched_outputs(cuda):
    """Caller-provided G-buffers are validated (the kernel writes through raw
    pointers): a wrong channel count, plane shape or dtype raises ValueError."""
    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    pos = torch.rand((5000, 3), device=cuda) * 2 - 1
    rgb = torch.randint(0, 256, (5000, 3), dtype=torch.uint8, device=cuda)
    cloud = DeviceCloud.from_tensors(pos, {"rgb": rgb})
    cam = look_at((0.0, -2.5, 1.0), (0, 0, 0), Intrinsics(width=64, height=48))
    r = Renderer(64, 48, device=cuda)
    sel = StreamSelection(rgb=True, depth=True)
    r.render(cloud, cam)
    with pytest.raises(ValueError, match="out\\['data'\\]"):
        r.resolve(cloud, cam, sel, out=r.alloc_outputs(1))
    bad = r.alloc_outputs(4)
    bad["depth"] = torch.empty((48, 64), dtype=torch.float64, device=cuda)
    with pytest.raises(ValueError, match="depth"):
        r.resolve(cloud, cam, sel, out=bad)
    bad = r.alloc_outputs(4)
    bad["coverage"] = torch.empty((47, 64), dtype=torch.uint8, device=cuda)
    with pytest.raises(ValueError, match="coverage"):
        r.resolve(cloud, cam, sel, out=bad)
    good = r.resolve(cloud, cam, sel, out=r.alloc_outputs(4))
    assert good.data.shape == (48, 64, 4)


def test_rasterize_output_pool_ownership(cuda):
    """rasterize() returns arrays in pooled pinned buffers: an image that is
    still referenced is never overwritten by later calls, and released sets
    are reused."""
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import StreamSelection, _renderer_for, rasterize

    rng = np.random.default_rng(17)
    n = 100_000
    sel = StreamSelection(rgb=True, depth=True)
    cam = look_at((0.3, -2.4, 0.8), (0, 0, 0), Intrinsics(width=96, height=64))
    clouds = [PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                         [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8))])
              for _ in range(3)]
    refs = [oracle.rasterize(pc, cam, sel) for pc in clouds]
    kept = [rasterize(pc, cam, sel) for pc in clouds]  # all three alive at once
    for img, ref in zip(kept, refs):
        assert np.array_equal(img.data, ref["data"])
        assert np.array_equal(img.index_plane, ref["index_plane"])
    view = kept[0].depth[:10]  # a view keeps its set busy after the image is dropped
    del kept, img
    r = _renderer_for(96, 64, cuda)
    before = len(r._host_pool)
    again = [rasterize(pc, cam, sel) for pc in clouds[1:]]
    assert len(r._host_pool) == before  # released sets were reused, no new ones pooled
    assert np.array_equal(view, refs[0]["depth"][:10])
    for img, ref in zip(again, refs[1:]):
        assert np.array_equal(img.data, ref["data"])


def test_resolve_without_planes(cuda):
    """resolve(out=alloc_outputs(C, planes=False)) writes only the CNN input (the neural
    pipeline's path): the channel data equals a full resolve's, the planes are None and
    to_host() refuses."""
    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    rng = np.random.default_rng(11)
    n = 300_000
    pc = PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8))])
    cloud = DeviceCloud.from_clouds([pc], device=cuda)
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=200, height=136))
    sel = StreamSelection(rgb=True, depth=True)
    r = Renderer(200, 136, device=cuda, pad_multiple=16)
    r.render(cloud, cam)
    full = r.resolve(cloud, cam, sel, clear=False)
    lean = r.resolve(cloud, cam, sel, out=r.alloc_outputs(4, planes=False))
    torch.cuda.synchronize()
    assert torch.equal(full.data, lean.data)
    assert lean.coverage is None and lean.index_plane is None and lean.depth is None
    with pytest.raises(ValueError):
        lean.to_host()


def test_resolve_planes_only_and_row_bands(cuda):
    """resolve(out={planes}) writes the coverage / index / depth planes alone (no channel
    data, no attribute reads) and leaves the keybuf when clear=False; the per-pixel-rgb
    resolve over row bands then reproduces a full resolve's channel data band by band."""
    import torch

    from paper_2407_19097_b200 import _lib
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    rng = np.random.default_rng(12)
    n = 300_000
    rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    pc = PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32), [Stream("rgb", "u8", rgb)])
    cloud = DeviceCloud.from_clouds([pc], device=cuda)
    W, H = 200, 136
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=W, height=H))
    sel = StreamSelection(rgb=True, depth=True)
    r = Renderer(W, H, device=cuda, pad_multiple=16)
    r.render(cloud, cam)
    full = r.resolve(cloud, cam, sel, clear=False)
    planes = {k: v for k, v in r.alloc_outputs(4).items() if k != "data"}
    p = r.resolve(cloud, cam, sel, out=planes, clear=False)
    keys = r.keybuf.cpu().numpy().view(np.uint64)
    for k in ("coverage", "index_plane", "depth"):
        assert torch.equal(getattr(p, k), getattr(full, k)), k
    assert p.data is None
    # per-pixel rgb words (the host gather's output) + banded resolves
    pix = np.zeros(W * H, np.uint32)
    assert _lib.load().nar_host_gather_rgb(keys.ctypes.data, W * H, r.domain, rgb.ctypes.data, 3,
                                           0, n, pix.ctypes.data) == 0
    pix_dev = torch.from_numpy(pix.view(np.int32)).to(cuda)
    data = torch.full_like(full.data, float("nan"))
    rows_pad = full.data.shape[0]
    for y0, y1 in ((0, 50), (50, 51), (51, H), (H, rows_pad)):
        r.resolve(cloud, cam, sel, out={"data": data}, pix_rgb=pix_dev, rows=(y0, y1), clear=False)
    torch.cuda.synchronize()
    assert torch.equal(data.view(torch.int32), full.data.view(torch.int32))


@pytest.mark.parametrize("W,H", [(640, 360), (1920, 1080), (3840, 2160)])
def test_hiz_refresh_kernels_agree(cuda, monkeypatch, W, H):
    """The coalesced Hi-Z refresh (hiz_rows_kernel, default for even widths) writes the
    same coarse table as the one-row-per-thread kernel (NAR_HIZ_ROWS=0) -- compared
    after the same forced multi-pass render (the table then holds the last refresh)."""
    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer

    monkeypatch.setenv("NAR_RENDER_PASS_UNITS", "200")
    rng = np.random.default_rng(W)
    pos = torch.from_numpy(rng.uniform(-1, 1, (2_000_000, 3)).astype(np.float32)).to(cuda)
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=W, height=H))
    tables, keys = [], []
    for mode in ("0", "1"):
        monkeypatch.setenv("NAR_HIZ_ROWS", mode)
        r = Renderer(W, H, device=cuda)
        r.hiz.zero_()  # the scratch tail beyond the table stays untouched
        r.render(DeviceCloud.from_tensors(pos), cam)
        torch.cuda.synchronize()
        tables.append(r.hiz.clone())
        keys.append(r.keys())
    assert np.array_equal(keys[0], keys[1])
    assert torch.equal(tables[0], tables[1])


@pytest.mark.gpu
@pytest.mark.parametrize("pinned,arity", [(False, 3), (True, 3), (False, 4)])
def test_rasterize_host_gather_matches_zero_copy(cuda, monkeypatch, pinned, arity):
    """rasterize()'s host-side gather of the winners' rgb (nar_host_gather_rgb +
    nar_resolve_pixrgb) gives the same FeatureImage as the resolve kernel's own
    zero-copy gather, and both equal the oracle (RGB and RGBA u8 streams)."""
    from paper_2407_19097_b200 import msr
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at

    rng = np.random.default_rng(21)
    n = 3_000_000
    pc = PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, arity), dtype=np.uint8))],
                    pinned=pinned)
    cam = look_at((0.3, -2.4, 1.1), (0, 0, 0), Intrinsics(width=640, height=360))
    sel = msr.StreamSelection(rgb=True, depth=True)
    monkeypatch.setattr(msr, "_HOST_GATHER", False)
    a = msr.rasterize(pc, cam, sel)
    a = (a.data.copy(), a.index_plane.copy())
    monkeypatch.setattr(msr, "_HOST_GATHER", True)
    b = msr.rasterize(pc, cam, sel)
    assert getattr(msr._renderer_for(640, 360, torch_device()), "_hg", None) is not None
    np.testing.assert_array_equal(b.index_plane, a[1])
    assert np.array_equal(b.data.view(np.uint32), a[0].view(np.uint32))
    ref = oracle.rasterize(pc, cam, sel)
    np.testing.assert_array_equal(b.index_plane, ref["index_plane"])
    assert np.array_equal(b.data, ref["data"])


def torch_device():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


@pytest.mark.gpu
@pytest.mark.parametrize("wh", [(31, 7), (1, 1), (97, 3)])
def test_rasterize_host_gather_odd_frames(cuda, wh):
    """The banded host gather on tiny / odd frames (fewer rows than bands, one pixel)
    equals the oracle."""
    from paper_2407_19097_b200 import msr
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at

    W, H = wh
    rng = np.random.default_rng(W * 100 + H)
    n = 20_000
    pc = PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8))])
    cam = look_at((0.2, -2.5, 0.9), (0, 0, 0), Intrinsics(width=W, height=H))
    sel = msr.StreamSelection(rgb=True, depth=True)
    fi = msr.rasterize(pc, cam, sel)
    ref = oracle.rasterize(pc, cam, sel)
    np.testing.assert_array_equal(fi.index_plane, ref["index_plane"])
    assert np.array_equal(fi.data, ref["data"])
