"""Pin the CPU oracle against golden vectors produced by the real reference.

These run on CPU only (no GPU): the oracle must reproduce the reference's own
outputs before it is trusted as the checker for the CUDA path.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import random_case


@pytest.fixture(scope="module", autouse=True)
def _build():
    oracle.build()


def test_kat_render_and_resolve(golden):
    from paper_2407_19097_b200.geometry import CameraPose, Intrinsics, PointCloud, Stream
    from paper_2407_19097_b200.msr import StreamSelection

    g = golden("raster_kat")
    cam = CameraPose(g["camera/pos"], g["camera/R"], Intrinsics(width=16, height=16))
    sel = StreamSelection(rgb=True, depth=True)
    for name in ("empty", "depth", "tie"):
        pc = PointCloud(g[f"{name}/positions"], [Stream("rgb", "u8", g[f"{name}/rgb"])])
        out = oracle.rasterize(pc, cam, sel)
        for k in ("data", "index_plane", "depth", "coverage"):
            assert np.array_equal(out[k], g[f"{name}/{k}"]), (name, k)
    # the contract itself
    assert g["empty/coverage"].sum() == 0
    assert set(np.unique(g["depth/index_plane"])) == {-1, 1}
    assert set(np.unique(g["tie/index_plane"])) >= {2}
    assert 7 not in set(np.unique(g["tie/index_plane"]))


@pytest.mark.parametrize("ci", range(6))
def test_random_cases_match_reference(golden, ci):
    pc, cam, sel, g, p = random_case(golden, ci)
    out = oracle.rasterize(pc, cam, sel, threads=3)
    assert np.array_equal(out["keybuf"], g[p + "keybuf"])
    for k in ("index_plane", "depth", "coverage"):
        assert np.array_equal(out[k], g[p + k]), k
    # the oracle calls the same numpy routines as the reference: exact
    assert np.array_equal(out["data"], g[p + "data"])


@pytest.mark.parametrize("ci", [0, 3])
def test_numpy_statement_equals_c(golden, ci):
    pc, cam, sel, g, p = random_case(golden, ci)
    i = cam.intrinsics
    kb = np.full(i.width * i.height, oracle.EMPTY_KEY, np.uint64)
    oracle.zbuffer_accumulate_numpy(kb, pc.positions, 0, cam.orientation, cam.position,
                                    i.focal_px, i.cx, i.cy, i.near, i.far, i.width, i.height)
    assert np.array_equal(kb, g[p + "keybuf"])


def test_nonfinite_culled_like_python_backend(golden):
    g = golden("raster_nonfinite")
    from paper_2407_19097_b200.geometry import Intrinsics

    i = Intrinsics(width=64, height=64)
    kb = oracle.zbuffer_render(g["positions"], g["R"], g["campos"], i.focal_px, i.cx, i.cy,
                               i.near, i.far, 64, 64, threads=2)
    assert np.array_equal(kb, g["keybuf"])


def test_reference_kernel_equals_port(golden):
    if oracle.ref_native() is None:
        pytest.skip("oracle/_ref not built (no /root/reference)")
    pc, cam, sel, g, p = random_case(golden, 1)
    i = cam.intrinsics
    args = (pc.positions, cam.orientation, cam.position, i.focal_px, i.cx, i.cy, i.near, i.far,
            i.width, i.height)
    a = oracle.zbuffer_render(*args, threads=4, impl="reference")
    b = oracle.zbuffer_render(*args, threads=1, impl="port")
    assert np.array_equal(a, b)
    assert np.array_equal(a, g[p + "keybuf"])


def test_c1_hash(golden):
    """1M uniform points at 512^2: checksum of the reference keybuf."""
    from paper_2407_19097_b200.geometry import Intrinsics, look_at

    g = golden("raster_c1_hash")
    pos = np.random.default_rng(0).uniform(-1, 1, (1_000_000, 3)).astype(np.float32)
    assert hashlib.sha256(pos.tobytes()).digest() == g["positions_sha256"].tobytes()
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=512, height=512))
    i = cam.intrinsics
    kb = oracle.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                               i.near, i.far, 512, 512, threads=4)
    assert hashlib.sha256(kb.tobytes()).digest() == g["keybuf_sha256"].tobytes()


def _cfg(cin, base, seed):
    from paper_2407_19097_b200.neural import UNetConfig

    return UNetConfig(input_channels=cin, base_channels=base, init_seed=seed)


@pytest.mark.parametrize("ui", range(3))
def test_unet_params_and_forward(golden, ui):
    g = golden("unet")
    p = f"u{ui}/"
    cin, H, W, base, seed = (int(v) for v in g[p + "cfg"])
    cfg = _cfg(cin, base, seed)
    P = oracle.init_params(cfg)
    for k, v in P.items():
        assert np.array_equal(v.reshape(-1)[:16], g[p + "param_head/" + k]), k
        assert v.astype(np.float64).sum() == pytest.approx(float(g[p + "param_sum/" + k]), abs=1e-9)
    y = oracle.forward(g[p + "x"], P, cfg)
    # same numpy/BLAS routines as the reference: equal up to BLAS blocking noise
    assert np.max(np.abs(y - g[p + "y"])) < 1e-6


def test_pyramid_fixture(golden):
    g = golden("unet")
    lvl = [g[f"pyramid/{k}"][0] for k in range(5)]
    for k in range(1, 5):
        assert np.array_equal(oracle.avg_pool2(lvl[k - 1]), lvl[k])
