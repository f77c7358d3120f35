"""§8f rows on the GPU: Morton keys / reorder (nar_morton_keys kernel),
NARPC -> DeviceCloud upload, f16 checkpoints driving the tensor-core U-Net,
and the render_neural composition with StageTimings.

Bars: Morton keys and the permutation bit-exact vs the reference
(tests/golden/preprocess.npz) and the pinned oracle at 8M points; framebuffers
bit-exact vs the oracle; U-Net outputs PSNR >= 50 dB, max|err| <= 2e-2.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

PSNR_MIN = 50.0
MAX_ABS = 2e-2


@pytest.fixture(scope="module")
def pre(golden):
    return golden("preprocess")


@pytest.mark.parametrize("name", ["uniform", "flat", "dups", "single"])
def test_morton_keys_golden(cuda, pre, name):
    import torch

    from paper_2407_19097_b200.geometry import PointCloud, Stream
    from paper_2407_19097_b200.preprocess import morton_keys_device, morton_reorder

    pos = pre[f"morton/{name}/positions"]
    keys = morton_keys_device(torch.from_numpy(pos).to(cuda)).cpu().numpy().view(np.uint64)
    assert np.array_equal(keys, pre[f"morton/{name}/keys"])
    order = pre[f"morton/{name}/order"]
    tag = np.arange(len(pos), dtype=np.float32)[:, None]
    pc = PointCloud(pos, [Stream("tag", "f32", tag)])
    ro = morton_reorder(pc)
    assert np.array_equal(ro.positions, pos[order])
    assert np.array_equal(ro.stream("tag").data[:, 0].astype(np.int64), order)


@pytest.mark.parametrize("kind", ["uniform", "terrain"])
def test_morton_large_vs_oracle(cuda, kind):
    import torch

    from paper_2407_19097_b200.msr import DeviceCloud
    from paper_2407_19097_b200.preprocess import morton_keys_device, morton_reorder

    rng = np.random.default_rng(11)
    n = 8_000_000
    if kind == "uniform":
        pos = rng.uniform(-100, 250, (n, 3)).astype(np.float32)
    else:  # clustered, with many exact duplicates
        base = rng.normal(0, 1, (n // 4, 3)).astype(np.float32) * [50, 50, 2]
        pos = np.repeat(base, 4, axis=0)[rng.permutation(n)].astype(np.float32)
    pd = torch.from_numpy(pos).to(cuda)
    keys = morton_keys_device(pd).cpu().numpy().view(np.uint64)
    ref = oracle.morton_keys(pos)
    assert np.array_equal(keys, ref)
    cloud = DeviceCloud.from_tensors(pd, {"id": torch.arange(n, device=cuda,
                                                             dtype=torch.float32)[:, None]})
    ro = morton_reorder(cloud)
    order = np.argsort(ref, kind="stable")
    got = ro.segments[0]["streams"]["id"][:, 0].cpu().numpy().astype(np.int64)
    assert np.array_equal(got, order)


def test_morton_order_render_invariance(cuda):
    """Reordering changes point indices, never which surface each pixel shows:
    depth planes equal, and the reordered frame is bit-exact vs the oracle."""
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import StreamSelection, rasterize
    from paper_2407_19097_b200.preprocess import morton_reorder

    rng = np.random.default_rng(3)
    n = 400_000
    pc = PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8))])
    cam = look_at((0.4, -2.3, 1.1), (0, 0, 0), Intrinsics(width=320, height=240))
    sel = StreamSelection(rgb=True, depth=True)
    a = rasterize(pc, cam, sel)
    ro = morton_reorder(pc)
    b = rasterize(ro, cam, sel)
    assert np.array_equal(a.depth, b.depth)
    ref = oracle.rasterize(ro, cam, sel)
    assert np.array_equal(b.data, ref["data"])
    assert np.array_equal(b.index_plane, ref["index_plane"])


def test_narpc_device_load(cuda, pre, tmp_path):
    from paper_2407_19097_b200.geometry import look_at, Intrinsics
    from paper_2407_19097_b200.msr import Renderer, StreamSelection
    from paper_2407_19097_b200.preprocess import load_pointcloud

    p = tmp_path / "a.narpc"
    p.write_bytes(bytes(pre["narpc/file"]))
    cloud = load_pointcloud(p, device=cuda)
    host = load_pointcloud(p)
    assert cloud.count == host.count
    assert np.array_equal(cloud.segments[0]["positions"].cpu().numpy(), host.positions)
    cam = look_at((0, -9, 3), (0, 0, 0), Intrinsics(width=64, height=48))
    sel = StreamSelection(rgb=True, depth=True, vel3d=True, scalars=("temperature",))
    img = Renderer(64, 48, device=cuda).rasterize(cloud, cam, sel).to_host()
    ref = oracle.rasterize(host, cam, sel)
    assert np.array_equal(img.data, ref["data"])
    assert np.array_equal(img.index_plane, ref["index_plane"])


def test_f16_checkpoint_forward(cuda, pre, tmp_path):
    from paper_2407_19097_b200.checkpoint import load_checkpoint
    from paper_2407_19097_b200.neural import forward

    p = tmp_path / "q.narck"
    p.write_bytes(bytes(pre["ckpt/clean_f16_file"]))
    st = load_checkpoint(p)
    y = forward(pre["ckpt/x"], st.params, st.config)
    ref = pre["ckpt/y_f16"]
    assert oracle.psnr(y, ref) >= PSNR_MIN
    assert np.max(np.abs(y - ref)) <= MAX_ABS


def test_render_neural_and_bench(cuda, pre, tmp_path):
    from paper_2407_19097_b200.checkpoint import load_checkpoint
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.neural import pad_to_multiple
    from paper_2407_19097_b200.pipeline import StageTimings, bench, render_neural

    p = tmp_path / "q.narck"
    p.write_bytes(bytes(pre["ckpt/clean_f16_file"]))
    rng = np.random.default_rng(9)
    n = 250_000
    pc = PointCloud(rng.uniform(-1, 1, (n, 3)).astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8))])
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=200, height=120))
    rgb, t = render_neural(pc, cam, p)
    assert isinstance(t, StageTimings) and rgb.shape == (120, 200, 3)
    assert t.msr_ms > 0 and t.transfer_proc_ms > 0 and t.unet_ms > 0
    st = load_checkpoint(p)
    from paper_2407_19097_b200.msr import StreamSelection

    fi = oracle.rasterize(pc, cam, StreamSelection(rgb=True, depth=True))
    x, (h, w) = pad_to_multiple(fi["data"], 16)
    ref = oracle.forward(x[None], st.params, st.config)[0, :h, :w]
    assert oracle.psnr(rgb, ref) >= PSNR_MIN
    assert np.max(np.abs(rgb - ref)) <= MAX_ABS
    med = bench(pc, cam, p, frames=5, warmup=2)
    assert med["fps"] > 0 and med["total_ms"] > 0


def test_feature_dump_from_device(cuda, pre, tmp_path):
    import torch

    from paper_2407_19097_b200.preprocess import load_features, save_features

    data = pre["feat/data"]
    padded = torch.zeros((16, 32, 5), device=cuda)
    padded[:13, :21] = torch.from_numpy(data).to(cuda)
    save_features(("r", "g", "b", "d", "coverage"), padded, tmp_path / "d.feat", 13, 21)
    assert (tmp_path / "d.feat").read_bytes() == bytes(pre["feat/file"])
    names, back = load_features(tmp_path / "d.feat")
    assert np.array_equal(back, data)
