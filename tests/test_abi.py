"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/nar_b200.h declares, and the host-side API mirrors the
reference's names, channel layout and error behaviour.  No kernel launches."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2407_19097_b200 import _kernels, _lib
from paper_2407_19097_b200.errors import ConfigurationError
from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
from paper_2407_19097_b200.msr import StreamSelection

HEADER = Path(__file__).resolve().parents[1] / "include" / "nar_b200.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(nar_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    from paper_2407_19097_b200 import build

    build.build()
    lib = _lib.load()
    assert b"sm_100a" in lib.nar_version()


def test_every_declared_symbol_is_exported_and_bound():
    lib = C.CDLL(str(_lib.LIB_PATH))
    declared = header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(declared)


def test_header_structs_match_ctypes():
    # sizes of the ABI structs as laid out by the C compiler
    assert C.sizeof(_lib.Camera) == 8 * 17 + 8
    assert C.sizeof(_lib.Segment) == 8 * (5 + _lib.MAX_SCALARS)
    assert C.sizeof(_lib.ResolveOut) == 8 + 8 + 8 * 3 + 8


def test_no_device_means_clean_status():
    n = C.c_int32(-1)
    rc = _lib.load().nar_device_count(C.byref(n))
    assert rc == 0 and n.value >= 0


def test_backend_names():
    """_kernels/__init__.py:45-53 names: "native" is an alias of the CUDA build
    (the compiled backend a drop-in caller asks for), "python" is not built
    (RuntimeError, like the reference's missing native module), others are
    unknown (ValueError)."""
    assert _kernels.BACKEND == "cuda"
    assert _kernels._resolve(None) == "cuda"
    assert _kernels._resolve("native") == "cuda"
    with pytest.raises(RuntimeError, match="not part of this build"):
        _kernels._resolve("python")
    with pytest.raises(ValueError):
        _kernels._resolve("opencl")
    assert _kernels.EMPTY_KEY == np.uint64(2 ** 64 - 1)


def test_invalid_arguments_map_to_value_error():
    kb = np.zeros(4, np.uint64)
    with pytest.raises(ValueError):
        _kernels.zbuffer_accumulate(kb, np.zeros((3, 3), np.float64), 0, np.eye(3), np.zeros(3),
                                    1, 1, 1, 0.1, 10, 2, 2)
    with pytest.raises(ValueError):  # C-ABI side validation, before any CUDA call
        _lib.check(_lib.load().nar_zbuffer_accumulate(kb.ctypes.data, None, 0, 0, None, None, 1.0,
                                                      1.0, 1.0, 0.1, 10.0, 2, 2))


def test_channel_layout_is_reference_order():
    rng = np.random.default_rng(0)
    pc = PointCloud(rng.uniform(size=(5, 3)),
                    [Stream("rgb", "u8", np.zeros((5, 3))), Stream("velocity", "f32", np.zeros((5, 3))),
                     Stream("temp", "f32", np.zeros((5, 1))), Stream("mask", "u8", np.zeros((5, 2)))])
    sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, scalars=("temp", "mask"),
                          coverage_channel=True)
    assert sel.channel_names(pc) == ("r", "g", "b", "d", "v2x", "v2y", "v2t", "v2m", "v3x", "v3y",
                                     "v3z", "v3m", "temp", "mask0", "mask1", "coverage")
    sel.validate(pc)
    with pytest.raises(ConfigurationError):
        StreamSelection(scalars=("nope",)).validate(pc)
    with pytest.raises(ConfigurationError):
        StreamSelection(rgb=True, rgb_stream="x").validate(pc)
    big = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True,
                          scalars=("temp", "mask", "temp"), coverage_channel=True)
    with pytest.raises(ConfigurationError):
        big.validate(pc)


def test_camera_contract():
    cam = look_at((0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=512, height=512))
    R = cam.orientation
    assert np.allclose(R @ R.T, np.eye(3))
    kc = cam.kernel_camera()
    assert kc.width == 512 and kc.cx == 256.0
    assert kc.f == pytest.approx(256.0 / np.tan(np.radians(30.0)))
    with pytest.raises(ValueError):
        Intrinsics(near=0.0)


def test_pointcloud_limits():
    from paper_2407_19097_b200.errors import CapacityError

    with pytest.raises(CapacityError):
        PointCloud(np.zeros((1, 3)), [Stream(f"s{i}", "u8", np.zeros((1, 1))) for i in range(9)])
    with pytest.raises(ValueError):
        PointCloud(np.zeros((2, 3)), [Stream("rgb", "u8", np.zeros((3, 3)))])


@pytest.mark.gpu
def test_plain_c_consumer(cuda, tmp_path):
    """tests/c/abi_consumer (gcc, only include/nar_b200.h + libnar_b200.so + cudart):
    host-parity and device entry points from C, checked against the oracle."""
    import struct
    import subprocess

    import oracle
    from paper_2407_19097_b200 import build as b
    from paper_2407_19097_b200.geometry import Intrinsics, look_at

    exe = b.C_CONSUMER if b.C_CONSUMER.exists() else b.build_c_consumer()
    rng = np.random.default_rng(21)
    n, W, H = 200_000, 160, 120
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    cam = look_at((0.2, -2.3, 0.9), (0, 0, 0), Intrinsics(width=W, height=H))
    i = cam.intrinsics
    fin, fout = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(fin, "wb") as f:
        f.write(struct.pack("<qii", n, W, H))
        f.write(np.ascontiguousarray(cam.orientation, np.float64).tobytes())
        f.write(np.ascontiguousarray(cam.position, np.float64).tobytes())
        f.write(struct.pack("<5d", i.focal_px, i.cx, i.cy, i.near, i.far))
        f.write(pos.tobytes() + rgb.tobytes())
    res = subprocess.run([str(exe), str(fin), str(fout)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    raw = fout.read_bytes()
    npix = W * H
    kb_host = np.frombuffer(raw, np.uint64, npix, 0)
    kb_dev = np.frombuffer(raw, np.uint64, npix, npix * 8)
    data = np.frombuffer(raw, np.float32, npix * 4, npix * 16).reshape(H, W, 4)
    ref = oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                i.near, i.far, W, H)
    assert np.array_equal(kb_host, ref) and np.array_equal(kb_dev, ref)
    from paper_2407_19097_b200.geometry import PointCloud, Stream
    from paper_2407_19097_b200.msr import StreamSelection

    want = oracle.rasterize(PointCloud(pos, [Stream("rgb", "u8", rgb)]), cam,
                            StreamSelection(rgb=True, depth=True))["data"]
    assert np.array_equal(data, want)


def test_host_gather_rgb_semantics():
    """nar_host_gather_rgb (host code, no GPU): per pixel the winner's rgb bytes packed
    c0 | c1 << 8 | c2 << 16; 0 for empty keys and winners outside [begin, begin+count);
    signed-domain keys are un-flipped first.  Large enough to run on the thread pool."""
    rng = np.random.default_rng(11)
    count, begin, arity = 50_000, 1000, 4
    rgb = rng.integers(0, 256, (count, arity), dtype=np.uint8)
    npix = 300_000
    idx = rng.integers(0, begin + count + 500, npix).astype(np.uint64)
    depth = rng.integers(1, 2**31, npix).astype(np.uint64)
    keys = (depth << np.uint64(32)) | idx
    empty = rng.random(npix) < 0.1
    keys[empty] = np.uint64(0xFFFFFFFFFFFFFFFF)
    inside = ~empty & (idx >= begin) & (idx < begin + count)
    rows = np.where(inside, idx.astype(np.int64) - begin, 0)
    want = np.where(inside, rgb[rows, 0].astype(np.uint32) | (rgb[rows, 1].astype(np.uint32) << 8)
                    | (rgb[rows, 2].astype(np.uint32) << 16), 0).astype(np.uint32)
    lib = _lib.load()
    for domain, k in ((_lib.KEYS_UNSIGNED, keys), (_lib.KEYS_SIGNED, keys ^ np.uint64(_lib.SIGN_FLIP))):
        k = np.ascontiguousarray(k)
        out = np.full(npix, 0xDEADBEEF, np.uint32)
        assert lib.nar_host_gather_rgb(k.ctypes.data, npix, domain, rgb.ctypes.data, arity,
                                       C.c_uint64(begin), count, out.ctypes.data) == 0
        np.testing.assert_array_equal(out, want)
