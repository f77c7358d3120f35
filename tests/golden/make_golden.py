"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the dev container (needs /root/reference; nothing here runs on the GPU
box):  python tests/golden/make_golden.py

The reference package is copied to a temporary directory and built there
(``setup.py build_ext --inplace``; /root/reference is read-only), then imported
and called through its public API:
  * nar.msr.rasterize (backend="native", threads=4 -- identical to 1 thread by
    the reference's own determinism contract) and
    nar._kernels.zbuffer_render for the keybufs;
  * backend="python" for the non-finite-input case, whose native behaviour is
    undefined (SURVEY.md trap 4);
  * nar.neural.forward with nar.neural.init_params for the U-Net.
Fixtures hold inputs and outputs, so the tests need no reference at run time.
"""

from __future__ import annotations

import hashlib
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")


def build_reference() -> Path:
    dst = Path(tempfile.gettempdir()) / "nar_ref_golden_build"
    if not (dst / "src" / "nar" / "_kernels").exists() or not list(
            (dst / "src" / "nar" / "_kernels").glob("_native*.so")):
        shutil.rmtree(dst, ignore_errors=True)
        shutil.copytree(REF, dst)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst,
                       check=True, capture_output=True)
    return dst / "src"


def scene(rng, n, width, height, dup_frac=0.05):
    """Random cloud with rgb/velocity/scalar streams and some exact duplicates
    (equal depths -> index tie-break), plus a random look-at camera."""
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    nd = int(n * dup_frac)
    if nd:
        src = rng.integers(0, n, nd)
        dst = rng.integers(0, n, nd)
        pos[dst] = pos[src]
    rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    vel = rng.normal(0, 1, (n, 3)).astype(np.float32)
    vel[: max(1, n // 100)] = 0.0  # zero-velocity sentinel rows
    temp = rng.normal(0, 3, (n, 1)).astype(np.float32)
    mask = rng.integers(0, 256, (n, 2), dtype=np.uint8)
    r = rng.uniform(1.6, 3.5)
    th = rng.uniform(0, 2 * np.pi)
    eye = np.array([r * np.cos(th), r * np.sin(th), rng.uniform(-1.5, 1.5)])
    target = rng.uniform(-0.3, 0.3, 3)
    fov = float(rng.uniform(35, 90))
    return pos, rgb, vel, temp, mask, eye, target, fov


def main() -> None:
    sys.path.insert(0, str(build_reference()))
    import nar
    from nar import _kernels
    from nar.geometry import Intrinsics, PointCloud, Stream, look_at
    from nar.msr import StreamSelection, rasterize
    from nar.neural import UNetConfig, build_pyramid, forward, init_params
    from nar.neural.autodiff import Tensor

    assert nar.kernel_backend == "native"
    rng = np.random.default_rng(20240719)

    # ---- rasterize known-answer tests -----------------------
    kat = {}
    cam = look_at((0.0, 0.0, -5.0), (0.0, 0.0, 0.0), Intrinsics(width=16, height=16))
    sel = StreamSelection(rgb=True, depth=True)
    cases = {
        "empty": np.zeros((0, 3), np.float32),
        # two points on the optical axis at depths 5 and 3 -> depth-3 point (index 1) wins
        "depth": np.array([[0, 0, 0], [0, 0, -2]], np.float32),
        # equal depth, indices 7 and 2 -> index 2 wins
        "tie": np.array([[5, 5, 5]] * 2 + [[0, 0, 0]] + [[5, 5, 5]] * 4 + [[0, 0, 0]],
                        np.float32),
    }
    for name, pos in cases.items():
        rgb = (np.arange(len(pos) * 3, dtype=np.uint8).reshape(-1, 3) * 7)
        pc = PointCloud(pos, [Stream("rgb", "u8", rgb)])
        fi = rasterize(pc, cam, sel, backend="native", threads=1)
        kat[f"{name}/positions"] = pos
        kat[f"{name}/rgb"] = rgb
        kat[f"{name}/data"] = fi.data
        kat[f"{name}/index_plane"] = fi.index_plane
        kat[f"{name}/depth"] = fi.depth
        kat[f"{name}/coverage"] = fi.coverage
    kat["camera/R"] = cam.orientation
    kat["camera/pos"] = cam.position
    np.savez_compressed(OUT / "raster_kat.npz", **kat)

    # ---- randomized full-selection cases --------------------------------------
    rnd = {}
    specs = [(2000, 64, 64), (10000, 64, 64), (10000, 80, 48), (6000, 37, 53),
             (10000, 64, 64), (3000, 128, 96)]
    for ci, (n, W, H) in enumerate(specs):
        pos, rgb, vel, temp, mask, eye, target, fov = scene(rng, n, W, H)
        vs = float(rng.uniform(0.5, 3.0))
        pc = PointCloud(pos, [Stream("rgb", "u8", rgb), Stream("velocity", "f32", vel),
                              Stream("temp", "f32", temp), Stream("mask", "u8", mask)])
        cam = look_at(eye, target, Intrinsics(fov_y_deg=fov, width=W, height=H))
        sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True,
                              scalars=("temp", "mask"), coverage_channel=True,
                              velocity_scale=vs)
        fi = rasterize(pc, cam, sel, backend="native", threads=4)
        fi1 = rasterize(pc, cam, sel, backend="native", threads=1)
        assert np.array_equal(fi.data, fi1.data)
        i = cam.intrinsics
        kb = _kernels.zbuffer_render(pc.positions, cam.orientation, cam.position, i.focal_px,
                                     i.cx, i.cy, i.near, i.far, W, H, threads=3,
                                     backend="native")
        p = f"c{ci}/"
        rnd.update({p + "positions": pos, p + "rgb": rgb, p + "velocity": vel,
                    p + "temp": temp, p + "mask": mask, p + "eye": eye, p + "target": target,
                    p + "fov": np.float64(fov), p + "wh": np.array([W, H]),
                    p + "velocity_scale": np.float64(vs), p + "keybuf": kb,
                    p + "data": fi.data, p + "index_plane": fi.index_plane,
                    p + "depth": fi.depth, p + "coverage": fi.coverage,
                    p + "R": cam.orientation, p + "campos": cam.position})
    rnd["n_cases"] = np.int64(len(specs))
    np.savez_compressed(OUT / "raster_random.npz", **rnd)

    # ---- non-finite inputs: python semantics (NaN/inf culled) ------------------
    pos = rng.uniform(-1, 1, (4000, 3)).astype(np.float32)
    pos[::97, 0] = np.nan
    pos[::89, 1] = np.inf
    pos[::83, 2] = -np.inf
    cam = look_at((0.3, -2.5, 0.8), (0, 0, 0), Intrinsics(width=64, height=64))
    i = cam.intrinsics
    kb = _kernels.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                 i.near, i.far, 64, 64, threads=1, backend="python")
    np.savez_compressed(OUT / "raster_nonfinite.npz", positions=pos, R=cam.orientation,
                        campos=cam.position, keybuf=kb)

    # ---- large case: hash only (inputs regenerated from a seed) ----------------
    g = np.random.default_rng(0)
    pos = g.uniform(-1, 1, (1_000_000, 3)).astype(np.float32)
    cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=512, height=512))
    i = cam.intrinsics
    kb = _kernels.zbuffer_render(pos, cam.orientation, cam.position, i.focal_px, i.cx, i.cy,
                                 i.near, i.far, 512, 512, threads=8, backend="native")
    np.savez_compressed(OUT / "raster_c1_hash.npz",
                        positions_sha256=np.frombuffer(hashlib.sha256(pos.tobytes()).digest(),
                                                       np.uint8),
                        keybuf_sha256=np.frombuffer(hashlib.sha256(kb.tobytes()).digest(),
                                                    np.uint8),
                        covered=np.int64((kb != np.uint64(2**64 - 1)).sum()))

    # ---- U-Net forward ---------------------------------------------------------
    net = {}
    for ci, (cin, H, W, base) in enumerate([(4, 32, 32, 16), (8, 48, 64, 16), (4, 16, 16, 4)]):
        cfg = UNetConfig(input_channels=cin, init_seed=ci, base_channels=base)
        params = init_params(cfg)
        x = rng.uniform(0, 1, (1, H, W, cin)).astype(np.float32)
        x[:, :, : W // 5] = 0.0  # background band
        y = forward(Tensor(x), {k: Tensor(v) for k, v in params.items()}, cfg).data
        p = f"u{ci}/"
        net.update({p + "cfg": np.array([cin, H, W, base, ci]), p + "x": x, p + "y": y})
        # parameter fingerprints (the oracle re-derives params from the seed)
        for k, v in params.items():
            net[p + "param_head/" + k] = v.reshape(-1)[:16]
            net[p + "param_sum/" + k] = np.float64(v.astype(np.float64).sum())
    pyr = build_pyramid(Tensor(rng.uniform(0, 1, (1, 32, 48, 3)).astype(np.float32)))
    for k, t in enumerate(pyr):
        net[f"pyramid/{k}"] = t.data
    np.savez_compressed(OUT / "unet.npz", **net)
    # ---- preprocessing: Morton order, NARPC files, checkpoints ----
    import io as _io
    import os as _os

    from nar.geometry import load_pointcloud, morton_keys, morton_reorder, save_pointcloud
    from nar.neural.checkpoint import (load_checkpoint, quantize_checkpoint, save_checkpoint,
                                       weight_payload_bytes)
    from nar.neural.model import ModelState

    pre = {}
    clouds = {
        "uniform": rng.uniform(-3, 5, (8000, 3)).astype(np.float32),
        "flat": np.c_[rng.uniform(0, 1, (5000, 2)), np.full(5000, 0.25)].astype(np.float32),
        "dups": np.repeat(rng.uniform(-1, 1, (700, 3)).astype(np.float32), 7, axis=0)[
            rng.permutation(4900)],
        "single": np.array([[1.5, -2.0, 0.125]], np.float32),
    }
    for name, pos in clouds.items():
        pc = PointCloud(pos, [Stream("rgb", "u8", rng.integers(0, 256, (len(pos), 3),
                                                                 dtype=np.uint8))])
        keys = morton_keys(pc)
        order = np.argsort(keys, kind="stable")
        ro = morton_reorder(pc)
        assert np.array_equal(ro.positions, pos[order])
        pre[f"morton/{name}/positions"] = pos
        pre[f"morton/{name}/keys"] = keys
        pre[f"morton/{name}/order"] = order
    n = 257
    pc = PointCloud(rng.normal(0, 2, (n, 3)).astype(np.float32),
                    [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8)),
                     Stream("velocity", "f32", rng.normal(0, 1, (n, 3)).astype(np.float32)),
                     Stream("temperature", "f32", rng.normal(0, 1, (n, 1)).astype(np.float32))])
    tmp = Path(tempfile.mkdtemp())
    save_pointcloud(pc, tmp / "a.narpc")
    back = load_pointcloud(tmp / "a.narpc")
    assert np.array_equal(back.positions, pc.positions)
    pre["narpc/file"] = np.frombuffer((tmp / "a.narpc").read_bytes(), np.uint8)
    pre["narpc/positions"] = pc.positions
    for s_ in pc.streams:
        pre[f"narpc/stream/{s_.name}"] = s_.data
    save_pointcloud(PointCloud(np.zeros((0, 3), np.float32)), tmp / "e.narpc")
    pre["narpc/empty_file"] = np.frombuffer((tmp / "e.narpc").read_bytes(), np.uint8)

    cfg = UNetConfig(input_channels=4, channel_names=("r", "g", "b", "d"), base_channels=4, max_channels=32,
                     init_seed=5)
    st = ModelState.initialize(cfg)
    st.step = 1234
    st.params["enc0a.f_w"][0, 0, 0, :2] = [70000.0, -1e6]  # saturates in f16
    for k in ("head.w", "head.b", "out.w", "out.b"):  # the rest stay zero (small file)
        st.m[k] = rng.normal(0, 1e-3, st.m[k].shape).astype(np.float32)
        st.v[k] = rng.uniform(0, 1e-6, st.v[k].shape).astype(np.float32)
    save_checkpoint(st, tmp / "f32.narck")
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sat = quantize_checkpoint(st, tmp / "f16.narck")
    pre["ckpt/f32_file"] = np.frombuffer((tmp / "f32.narck").read_bytes(), np.uint8)
    pre["ckpt/f16_file"] = np.frombuffer((tmp / "f16.narck").read_bytes(), np.uint8)
    pre["ckpt/saturated"] = np.int64(sat)
    pre["ckpt/payload_f32"] = np.int64(weight_payload_bytes(tmp / "f32.narck"))
    pre["ckpt/payload_f16"] = np.int64(weight_payload_bytes(tmp / "f16.narck"))
    q = load_checkpoint(tmp / "f16.narck", expected_config=cfg)
    st.params["enc0a.f_w"][0, 0, 0, :2] = 0.0
    q.params["enc0a.f_w"][0, 0, 0, :2] = 0.0
    save_checkpoint(ModelState(cfg, q.params, step=7), tmp / "q.narck", precision="f16")
    pre["ckpt/clean_f16_file"] = np.frombuffer((tmp / "q.narck").read_bytes(), np.uint8)
    x = rng.uniform(0, 1, (1, 48, 80, 4)).astype(np.float32)
    x[:, :, :20] = 0.0
    pre["ckpt/x"] = x
    pre["ckpt/y_f16"] = forward(Tensor(x), {k: Tensor(v) for k, v in q.params.items()},
                                cfg).data
    from nar.msr.feature_io import save_features

    feat = rng.normal(0, 1, (13, 21, 5)).astype(np.float32)
    save_features(("r", "g", "b", "d", "coverage"), feat, tmp / "f.feat")
    pre["feat/data"] = feat
    pre["feat/file"] = np.frombuffer((tmp / "f.feat").read_bytes(), np.uint8)
    shutil.rmtree(tmp)
    np.savez_compressed(OUT / "preprocess.npz", **pre)

    # ---- Gaussian splats (gsplat/renderer.py, _kernels splat_blend_image) ---------
    from nar import _kernels as K
    from nar.gsplat import build_splats, render_gsplat
    from nar.gsplat.renderer import _prepare_splats

    gs = {}
    n = 3000
    W, H = 160, 120
    mu = np.c_[rng.uniform(-10, W + 10, n), rng.uniform(-10, H + 10, n)]
    A = rng.normal(0, 1, (n, 2, 2))
    cov = np.einsum("nij,nkj->nik", A, A) * rng.uniform(0.5, 40, n)[:, None, None] + 0.3 * np.eye(2)
    det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] ** 2
    inv_abc = np.stack([cov[:, 1, 1], -cov[:, 0, 1], cov[:, 0, 0]], axis=1) / det[:, None]
    lam = np.linalg.eigvalsh(cov)[:, 1]
    r3 = 3.0 * np.sqrt(lam)
    boxes = np.stack([np.clip(np.floor(mu[:, 0] - r3), 0, W - 1), np.clip(np.ceil(mu[:, 0] + r3), 0, W - 1),
                      np.clip(np.floor(mu[:, 1] - r3), 0, H - 1), np.clip(np.ceil(mu[:, 1] + r3), 0, H - 1)],
                     axis=1).astype(np.int64)
    color = rng.uniform(0, 1, (n, 3))
    opac = rng.uniform(0.05, 0.99, n)
    img_native = K.splat_blend_image(mu, inv_abc, boxes, color, opac, W, H, threads=4, backend="native")
    img_py = K.splat_blend_image(mu, inv_abc, boxes, color, opac, W, H, backend="python")
    assert np.allclose(img_native, img_py, rtol=0, atol=1e-12)
    gs.update({"blend/mu": mu, "blend/inv_abc": inv_abc, "blend/boxes": boxes, "blend/color": color,
               "blend/opacity": opac, "blend/wh": np.array([W, H]), "blend/rgb": img_native})
    for style in ("vector_field", "terrain"):
        m = 2500
        pos = rng.normal(0, 1, (m, 3)).astype(np.float32) * [1.0, 1.0, 0.3]
        streams = [Stream("rgb", "u8", rng.integers(0, 256, (m, 3), dtype=np.uint8)),
                   Stream("velocity", "f32", rng.normal(0, 1, (m, 3)).astype(np.float32))]
        pc = PointCloud(pos.astype(np.float32), streams)
        cam = look_at((0.5, -4.0, 2.0), (0, 0, 0), Intrinsics(width=128, height=96))
        sp = build_splats(pc, style)
        img, cnt = render_gsplat(sp, cam, threads=4, backend="native", return_counters=True)
        prep = _prepare_splats(sp, cam)
        p = f"{style}/"
        gs.update({p + "positions": pos.astype(np.float32), p + "rgb": streams[0].data,
                   p + "velocity": streams[1].data, p + "R": cam.orientation,
                   p + "campos": cam.position, p + "cov": sp.covariances, p + "colors": sp.colors,
                   p + "opacities": sp.opacities, p + "img": img,
                   p + "counters": np.array([cnt["total"], cnt["culled"], cnt["skipped_singular"]]),
                   p + "prep_mu": prep[0], p + "prep_inv_abc": prep[1], p + "prep_boxes": prep[2]})
    np.savez_compressed(OUT / "gsplat.npz", **gs)

    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
