"""CPU oracle for the NAR hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (paper_2407_19097_b200) imports this module.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference
arm may use it, and only as the checker or the timed CPU reference -- never
as the thing measured for the GPU path.

Contents (each cites the reference file:line it restates):
  * zbuffer_accumulate / zbuffer_render -- C restatement (oracle/zbuffer.c) of
    _kernels/_native.pyx:32-77 and the chunked dispatch _kernels/__init__.py:56-94;
    ``impl="reference"`` runs the reference's own Cython kernel compiled from
    /root/reference by oracle/build_ref.sh into oracle/_ref/.
  * rasterize -- numpy restatement of msr/rasterizer.py:123-188 (decode + resolve),
    with msr/velocity.py:17-48 and geometry/camera.py:154-166.
  * init_params / forward -- numpy f32 restatement of neural/model.py:65-204 and the
    forward ops of neural/autodiff.py:186-288 (im2col + BLAS conv).

  * splat_blend -- numpy restatement of the Gaussian-splat blend
    (_kernels/python_impl.py:56-89 semantics, _native.pyx association).
  * morton_keys / morton_order -- numpy restatement of geometry/morton.py:9-46
    (21-bit f64 quantisation over the cloud AABB, magic-number bit spread,
    stable argsort).

Pinning: tests/test_oracle.py checks every function here against golden
vectors produced by the real reference (tests/golden/make_golden.py, committed
fixtures under tests/golden/), so parity is pinned, not assumed.
"""

from __future__ import annotations

import ctypes as C
import importlib.util
import math
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_DIR = HERE / "_ref"
EMPTY_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)
REFERENCE_ROOT = Path("/root/reference")


# ---------------------------------------------------------------------------
# build
# ---------------------------------------------------------------------------
def build(force: bool = False) -> None:
    """Compile the C restatement; compile the reference's Cython kernel into
    oracle/_ref when /root/reference is present (this container only)."""
    src = HERE / "zbuffer.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                        str(src), "-o", str(LIB), "-lm"], check=True)
    if REFERENCE_ROOT.exists() and (force or _ref_module_path() is None):
        subprocess.run(["bash", str(HERE / "build_ref.sh")], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        vp, d, i64, u64, i32 = C.c_void_p, C.c_double, C.c_int64, C.c_uint64, C.c_int
        L.oracle_zbuffer_accumulate.argtypes = [vp, vp, i64, u64, vp, vp, d, d, d, d, d, i32, i32]
        L.oracle_zbuffer_accumulate.restype = None
        L.oracle_zbuffer_render_mt.argtypes = [vp, vp, i64, vp, vp, d, d, d, d, d, i32, i32, i32]
        L.oracle_zbuffer_render_mt.restype = C.c_int
        _lib = L
    return _lib


def _ref_module_path():
    if not REF_DIR.exists():
        return None
    for p in REF_DIR.glob("_native*.so"):
        return p
    return None


_ref_native = None


def ref_native():
    """The reference's compiled Cython kernel module (oracle/_ref), or None."""
    global _ref_native
    if _ref_native is None:
        p = _ref_module_path()
        if p is None:
            return None
        spec = importlib.util.spec_from_file_location("_native", p)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _ref_native = mod
    return _ref_native


# ---------------------------------------------------------------------------
# render (_native.pyx:32-77, _kernels/__init__.py:56-94)
# ---------------------------------------------------------------------------
def _prep(positions, R, campos):
    pos = np.ascontiguousarray(positions, np.float32).reshape(-1, 3)
    R = np.ascontiguousarray(R, np.float64).reshape(3, 3)
    campos = np.ascontiguousarray(campos, np.float64).reshape(3)
    return pos, R, campos


def zbuffer_accumulate(keybuf, positions, base_index, R, campos, f, cx, cy, near, far,
                       width, height):
    pos, R, campos = _prep(positions, R, campos)
    lib().oracle_zbuffer_accumulate(keybuf.ctypes.data, pos.ctypes.data, len(pos),
                                    int(base_index) & 0xFFFFFFFFFFFFFFFF, R.ctypes.data,
                                    campos.ctypes.data, f, cx, cy, near, far, width, height)


def zbuffer_accumulate_numpy(keybuf, positions, base_index, R, campos, f, cx, cy, near, far,
                             width, height):
    """Vectorised numpy statement (same f64 op order; python_impl.py:17-53)."""
    pos, R, campos = _prep(positions, R, campos)
    p = pos.astype(np.float64)
    w0, w1, w2 = p[:, 0] - campos[0], p[:, 1] - campos[1], p[:, 2] - campos[2]
    uz = w0 * R[2, 0] + w1 * R[2, 1] + w2 * R[2, 2]
    ux = w0 * R[0, 0] + w1 * R[0, 1] + w2 * R[0, 2]
    uy = w0 * R[1, 0] + w1 * R[1, 1] + w2 * R[1, 2]
    keep = (uz > near) & (uz < far)
    z = np.where(keep, uz, 1.0)
    with np.errstate(invalid="ignore"):
        px = np.floor(cx + f * (ux / z) + 0.5)
        py = np.floor(cy + f * (uy / z) + 0.5)
        keep &= (px >= 0) & (px < width) & (py >= 0) & (py < height)
    sel = np.nonzero(keep)[0]
    pix = (py[sel] * width + px[sel]).astype(np.int64)
    hi = uz[sel].astype(np.float32).view(np.uint32).astype(np.uint64) << np.uint64(32)
    lo = (sel.astype(np.uint64) + np.uint64(base_index)) & np.uint64(0xFFFFFFFF)
    np.minimum.at(keybuf, pix, hi | lo)


def zbuffer_render(positions, R, campos, f, cx, cy, near, far, width, height, threads=1,
                   impl: str = "port"):
    """Full render pass.  impl="port": C restatement (pthreads);
    impl="reference": the reference's Cython kernel from oracle/_ref driven by
    the reference's chunk/thread-pool dispatch restated here."""
    pos, R, campos = _prep(positions, R, campos)
    n = len(pos)
    npix = int(width) * int(height)
    if impl == "port":
        keybuf = np.full(npix, EMPTY_KEY, np.uint64)
        lib().oracle_zbuffer_render_mt(keybuf.ctypes.data, pos.ctypes.data, n, R.ctypes.data,
                                       campos.ctypes.data, f, cx, cy, near, far, width, height,
                                       int(threads))
        return keybuf
    if impl != "reference":
        raise ValueError(impl)
    nat = ref_native()
    if nat is None:
        raise RuntimeError("oracle/_ref not built")
    nt = max(1, min(int(threads or 1), max(n, 1)))

    def chunk(lo, hi):
        buf = np.full(npix, EMPTY_KEY, np.uint64)
        if hi > lo:
            nat.zbuffer_accumulate(buf, pos[lo:hi], lo, R, campos, f, cx, cy, near, far,
                                   int(width), int(height))
        return buf

    if nt == 1 or n == 0:
        return chunk(0, n)
    bounds = np.linspace(0, n, nt + 1).astype(np.int64)
    with ThreadPoolExecutor(max_workers=nt) as ex:
        bufs = list(ex.map(lambda b: chunk(int(b[0]), int(b[1])), zip(bounds[:-1], bounds[1:])))
    return np.minimum.reduce(bufs)


# ---------------------------------------------------------------------------
# resolve (rasterizer.py:123-188, velocity.py:17-48, camera.py:154-166)
# ---------------------------------------------------------------------------
def _as_float(stream_data, fmt):
    if fmt == "u8":
        return stream_data.astype(np.float32) / np.float32(255.0)
    return stream_data.astype(np.float32)


def projection_jacobians(R, campos, f, points):
    p = np.asarray(points, np.float64).reshape(-1, 3)
    u = (p - campos) @ R.T
    uz = u[:, 2]
    s = (f / uz ** 2)[:, None]
    J = np.empty((len(p), 2, 3), np.float64)
    J[:, 0, :] = (uz[:, None] * R[0] - u[:, 0:1] * R[2]) * s
    J[:, 1, :] = (uz[:, None] * R[1] - u[:, 1:2] * R[2]) * s
    return J


def encode_vel2d_batch(R, campos, f, points, velocities, scale=1.0):
    J = projection_jacobians(R, campos, f, points)
    vp = np.einsum("nij,nj->ni", J, np.asarray(velocities, np.float64).reshape(-1, 3))
    mag = np.hypot(vp[:, 0], vp[:, 1])
    theta = np.where(mag < 1e-9, 0.0, np.arctan2(-vp[:, 1], vp[:, 0]))
    return np.stack([vp[:, 0] / scale, vp[:, 1] / scale, theta, mag / scale], axis=1)


def encode_vel3d(v, scale=1.0):
    v = np.asarray(v, np.float64).reshape(-1, 3)
    out = np.empty((len(v), 4), np.float64)
    out[:, :3] = v
    out[:, 3] = np.linalg.norm(v, axis=1)
    return out / scale


def resolve(keybuf, pc, cam, sel):
    """Decode + channel fill from a keybuf; returns dict of planes."""
    intr = cam.intrinsics
    W, H = intr.width, intr.height
    covered = keybuf != EMPTY_KEY
    win = (keybuf[covered] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    index_plane = np.full(H * W, -1, np.int64)
    index_plane[covered] = win
    depth = np.zeros(H * W, np.float32)
    depth[covered] = (keybuf[covered] >> np.uint64(32)).astype(np.uint32).view(np.float32)
    names = sel.channel_names(pc)
    data = np.zeros((H * W, len(names)), np.float32)
    col = 0
    if sel.rgb:
        s = pc.stream(sel.rgb_stream)
        data[covered, col:col + 3] = _as_float(s.data[win], s.format)[:, :3]
        col += 3
    if sel.depth:
        data[covered, col] = np.float32(intr.near) / depth[covered]
        np.clip(data[:, col], 0.0, 1.0, out=data[:, col])
        col += 1
    if sel.vel2d or sel.vel3d:
        s = pc.stream(sel.velocity_stream)
        v = _as_float(s.data[win], s.format)[:, :3].astype(np.float64)
    if sel.vel2d:
        data[covered, col:col + 4] = encode_vel2d_batch(
            cam.orientation, cam.position, intr.focal_px, pc.positions[win], v,
            sel.velocity_scale).astype(np.float32)
        col += 4
    if sel.vel3d:
        data[covered, col:col + 4] = encode_vel3d(v, sel.velocity_scale).astype(np.float32)
        col += 4
    for name in sel.scalars:
        s = pc.stream(name)
        data[covered, col:col + s.arity] = _as_float(s.data[win], s.format)
        col += s.arity
    if sel.coverage_channel:
        data[:, col] = covered.astype(np.float32)
        col += 1
    return {"data": data.reshape(H, W, len(names)), "coverage": covered.reshape(H, W).astype(np.uint8),
            "index_plane": index_plane.reshape(H, W), "depth": depth.reshape(H, W),
            "channel_names": names}


def rasterize(pc, cam, sel, threads=1, impl="port"):
    intr = cam.intrinsics
    kb = zbuffer_render(pc.positions, cam.orientation, cam.position, intr.focal_px, intr.cx,
                        intr.cy, intr.near, intr.far, intr.width, intr.height, threads=threads,
                        impl=impl)
    out = resolve(kb, pc, cam, sel)
    out["keybuf"] = kb
    return out


# ---------------------------------------------------------------------------
# U-Net forward (model.py:65-204, autodiff.py:186-288), numpy f32
# ---------------------------------------------------------------------------
def unet_width(cfg, level):
    return min(cfg.base_channels * cfg.channel_multiplier ** level, cfg.max_channels)


def init_params(cfg):
    """Seeded Kaiming-uniform init in the reference's draw order (model.py:70-100)."""
    rng = np.random.default_rng(cfg.init_seed)
    P = {}
    cin = cfg.input_channels
    if cfg.use_descriptor_head:
        P["head.w"] = np.eye(cin, dtype=np.float32)
        P["head.b"] = np.zeros(cin, np.float32)

    def draw(shape, fan):
        b = np.sqrt(6.0 / fan)
        return rng.uniform(-b, b, shape).astype(np.float32)

    def gated(name, ci, co):
        P[f"{name}.f_w"] = draw((3, 3, ci, co), 9 * ci)
        P[f"{name}.f_b"] = np.zeros(co, np.float32)
        P[f"{name}.g_w"] = draw((3, 3, ci, co), 9 * ci)
        P[f"{name}.g_b"] = np.ones(co, np.float32)

    for k in range(cfg.levels):
        ci = cin if k == 0 else unet_width(cfg, k - 1) + cin
        gated(f"enc{k}a", ci, unet_width(cfg, k))
        gated(f"enc{k}b", unet_width(cfg, k), unet_width(cfg, k))
    for k in range(cfg.levels - 2, -1, -1):
        gated(f"dec{k}a", unet_width(cfg, k + 1) + unet_width(cfg, k), unet_width(cfg, k))
        gated(f"dec{k}b", unet_width(cfg, k), unet_width(cfg, k))
    P["out.w"] = draw((unet_width(cfg, 0), cfg.output_channels), unet_width(cfg, 0))
    P["out.b"] = np.zeros(cfg.output_channels, np.float32)
    return P


def conv3x3(x, w, b):
    """'same' cross-correlation, x (H,W,Ci) f32, w (3,3,Ci,Co) HWIO (autodiff.py:260-288)."""
    h, wd, ci = x.shape
    xp = np.pad(x, ((1, 1), (1, 1), (0, 0)))
    win = np.lib.stride_tricks.sliding_window_view(xp, (3, 3), axis=(0, 1))
    cols = np.ascontiguousarray(win.transpose(0, 1, 3, 4, 2)).reshape(h * wd, -1)
    return (cols @ w.reshape(-1, w.shape[-1]) + b).reshape(h, wd, -1)


def elu(x):
    return np.where(x > 0, x, np.exp(np.minimum(x, 0.0)) - 1.0).astype(x.dtype)


def sigmoid(x):
    return (1.0 / (1.0 + np.exp(-x))).astype(x.dtype)


def avg_pool2(x):
    h, w, c = x.shape
    return x.reshape(h // 2, 2, w // 2, 2, c).mean(axis=(1, 3)).astype(x.dtype)


def up2(x):
    return np.repeat(np.repeat(x, 2, axis=0), 2, axis=1)


def gated(P, name, x):
    return elu(conv3x3(x, P[f"{name}.f_w"], P[f"{name}.f_b"])) * sigmoid(
        conv3x3(x, P[f"{name}.g_w"], P[f"{name}.g_b"]))


def forward(features, P, cfg):
    """features (N,H,W,C) or (H,W,C) f32 -> (N,H,W,out) f32."""
    x = np.asarray(features, np.float32)
    squeeze = x.ndim == 3
    if squeeze:
        x = x[None]
    outs = []
    for img in x:
        h, w, c = img.shape
        if cfg.use_descriptor_head:
            img = (img.reshape(-1, c) @ P["head.w"] + P["head.b"]).reshape(h, w, c)
        pyr = [img]
        for _ in range(cfg.levels - 1):
            pyr.append(avg_pool2(pyr[-1]))
        skips, y = [], None
        for k in range(cfg.levels):
            inp = pyr[0] if k == 0 else np.concatenate([avg_pool2(y), pyr[k]], axis=-1)
            y = gated(P, f"enc{k}b", gated(P, f"enc{k}a", inp))
            skips.append(y)
        for k in range(cfg.levels - 2, -1, -1):
            y = gated(P, f"dec{k}b", gated(P, f"dec{k}a",
                                            np.concatenate([up2(y), skips[k]], axis=-1)))
        logits = y.reshape(-1, y.shape[-1]) @ P["out.w"] + P["out.b"]
        outs.append(sigmoid(logits).reshape(h, w, -1))
    out = np.stack(outs)
    return out[0] if squeeze else out


def psnr(a, b):
    """metrics.py:27-36 (100 dB cap)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    m = float(np.mean((a - b) ** 2))
    if m == 0.0:
        return 100.0
    return min(10.0 * math.log10(1.0 / m), 100.0)


# ---- Morton order (geometry/morton.py) ---------------------------------------------

_SPREAD = [(32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
           (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)]


def _spread21(q):
    """morton.py:12-20: two zero bits between each of the low 21 bits."""
    x = q.astype(np.uint64) & np.uint64(0x1FFFFF)
    for sh, mask in _SPREAD:
        x = (x | (x << np.uint64(sh))) & np.uint64(mask)
    return x


def morton_keys(positions, lo=None, hi=None):
    """morton.py:23-37: keys over the cloud AABB (pointcloud.py:38-44 min/max)."""
    p = np.asarray(positions, np.float32)
    if lo is None:
        lo, hi = p.min(axis=0).astype(np.float64), p.max(axis=0).astype(np.float64)
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    ext = np.where(hi > lo, hi - lo, 1.0)
    with np.errstate(invalid="ignore"):
        q = np.floor((p.astype(np.float64) - lo) / ext * float(1 << 21)).astype(np.int64)
    q = np.clip(q, 0, (1 << 21) - 1)
    return _spread21(q[:, 0]) | (_spread21(q[:, 1]) << np.uint64(1)) | (
        _spread21(q[:, 2]) << np.uint64(2))


def morton_order(positions):
    """morton.py:40-46: the stable permutation ``morton_reorder`` applies."""
    if len(positions) == 0:
        return np.zeros(0, np.int64)
    return np.argsort(morton_keys(positions), kind="stable")


# ---- Gaussian splat blending (_kernels/python_impl.py:56-89, _native.pyx:80-159) --------

MIN_TRANSMITTANCE = 1.0 / 255.0


def splat_blend(mu, inv_abc, boxes, color, opacity, width, height):
    """Sequential front-to-back blend, one splat at a time over its clipped box:
    per pixel q = a dx^2 + 2 b dy dx + c dy^2, alpha = op * exp(-q/2); pixels whose
    transmittance is below 1/255 no longer accumulate.  (H, W, 3) f64."""
    rgb = np.zeros((height, width, 3), np.float64)
    trans = np.ones((height, width), np.float64)
    for i in range(len(mu)):
        x0, x1, y0, y1 = (int(v) for v in boxes[i])
        dx = np.arange(x0, x1 + 1, dtype=np.float64) - mu[i, 0]
        dy = np.arange(y0, y1 + 1, dtype=np.float64) - mu[i, 1]
        a, b, c = inv_abc[i]
        q = a * (dx[None, :] * dx[None, :]) + (2.0 * b * dy[:, None]) * dx[None, :] + c * (dy[:, None] * dy[:, None])
        alpha = opacity[i] * np.exp(-0.5 * q)
        tb = trans[y0:y1 + 1, x0:x1 + 1]
        on = tb >= MIN_TRANSMITTANCE
        rgb[y0:y1 + 1, x0:x1 + 1] += np.where(on, alpha * tb, 0.0)[:, :, None] * color[i]
        tb *= np.where(on, 1.0 - alpha, 1.0)
    return rgb


def splat_blend_reference(mu, inv_abc, boxes, color, opacity, width, height, tile_size=16,
                          threads=1):
    """The reference's native blend (oracle/_ref `splat_blend_tiles`) behind the
    CSR tile binning and tile-range thread split of _kernels/__init__.py:123-166,
    restated here (pair list in splat order, stable sort by tile).  CPU baseline
    and cross-check of the GPU blend."""
    nat = ref_native()
    if nat is None:
        raise RuntimeError("oracle/_ref not built")
    ts = int(tile_size)
    tiles_x, tiles_y = (width + ts - 1) // ts, (height + ts - 1) // ts
    n_tiles = tiles_x * tiles_y
    b = np.asarray(boxes, np.int64)
    tx0, tx1, ty0, ty1 = b[:, 0] // ts, b[:, 1] // ts, b[:, 2] // ts, b[:, 3] // ts
    sx = (tx1 - tx0 + 1).astype(np.int64)
    cnt = sx * (ty1 - ty0 + 1)
    sid = np.repeat(np.arange(len(b), dtype=np.int64), cnt)
    off = np.arange(len(sid)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    tile = (ty0[sid] + off // sx[sid]) * tiles_x + tx0[sid] + off % sx[sid]
    order = np.argsort(tile, kind="stable")
    tile_splats = sid[order]
    tile_offsets = np.searchsorted(tile[order], np.arange(n_tiles + 1)).astype(np.int64)
    rgb = np.zeros((height * width, 3), np.float64)
    trans = np.ones(height * width, np.float64)
    args = (np.ascontiguousarray(mu, np.float64), np.ascontiguousarray(inv_abc, np.float64),
            np.ascontiguousarray(b, np.int32), np.ascontiguousarray(color, np.float64),
            np.ascontiguousarray(opacity, np.float64), tile_offsets, tile_splats)

    def span(t0, t1):
        nat.splat_blend_tiles(rgb, trans, *args, int(width), int(height), ts, tiles_x,
                              int(t0), int(t1))

    nt = max(1, min(int(threads or 1), n_tiles))
    if nt == 1:
        span(0, n_tiles)
    else:
        bounds = np.linspace(0, n_tiles, nt + 1).astype(np.int64)
        with ThreadPoolExecutor(max_workers=nt) as ex:
            list(ex.map(lambda se: span(se[0], se[1]), zip(bounds[:-1], bounds[1:])))
    return rgb.reshape(height, width, 3)
