"""Gaussian-splat ground-truth renderer: host preparation,
GPU tile blend.

Mirrors pkg/src/nar/gsplat/renderer.py and covariance.py: ``SplatSet``,
``build_splats`` (vector-field / terrain styles), ``render_gsplat`` and the
kernel entry ``splat_blend_image`` (pkg/src/nar/_kernels/__init__.py:97-166).
The per-splat preparation (cull, depth sort, 2D covariance, bounds) is O(n)
f64 numpy written in the reference's operation order, so its arrays are
bit-identical; the O(pixels x splats) blend runs on the GPU
(``nar_splat_blend``: CSR tile binning by a device radix sort, one CTA per
tile, f64 accumulation, 1/255 transmittance cut-off).  The CPU blend exists
only in oracle/ as the checker.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._kernels import _resolve
from .errors import ConfigurationError, InsufficientPointsError
from .geometry import CameraPose, PointCloud

LOWPASS_PX2 = 0.3          # screen-space covariance floor, px^2 (renderer.py:25)
MAX_CONDITION = 1e12       # 2D covariances worse than this are skipped
SIGMA_CUTOFF = 3.0
VECTOR_FIELD_OPACITY = 0.8
TERRAIN_OPACITY = 1.0
DEFAULT_STRETCH = 300.0    # covariance.py:7

# viridis-like anchors of the flow colormap, evenly spaced on [0, 1] (renderer.py:32-42)
_FLOW_ANCHORS = np.array([
    (0.267004, 0.004874, 0.329415), (0.278826, 0.175490, 0.483397),
    (0.229739, 0.322361, 0.545706), (0.172719, 0.448791, 0.557885),
    (0.127568, 0.566949, 0.550556), (0.157851, 0.683765, 0.501686),
    (0.369214, 0.788888, 0.382914), (0.678489, 0.863742, 0.189503),
    (0.993248, 0.906157, 0.143936),
])


def flow_colormap(t) -> np.ndarray:
    """Piecewise-linear map of [0, 1] onto the anchors."""
    t = np.clip(np.asarray(t, np.float64), 0.0, 1.0)
    pos = t * (len(_FLOW_ANCHORS) - 1)
    lo = np.floor(pos).astype(np.int64)
    hi = np.minimum(lo + 1, len(_FLOW_ANCHORS) - 1)
    w = (pos - lo)[:, None]
    return _FLOW_ANCHORS[lo] * (1.0 - w) + _FLOW_ANCHORS[hi] * w


# ---- covariance helpers (covariance.py) ---------------------------------------------

def rotation_from_dominant_axis(v) -> np.ndarray:
    v = np.asarray(v, np.float64).reshape(3)
    n = np.linalg.norm(v)
    if n == 0:
        raise ValueError("dominant axis must be a nonzero vector")
    e1 = v / n
    aux = np.array([0.0, 0.0, 1.0]) if abs(float(e1[2])) <= 0.999 else np.array([1.0, 0.0, 0.0])
    e2 = np.cross(aux, e1)
    e2 /= np.linalg.norm(e2)
    return np.stack([e1, e2, np.cross(e1, e2)], axis=1)


def covariance_from_vector(v, stretch: float = DEFAULT_STRETCH, base_scale: float = 1.0,
                           square_scales: bool = False) -> np.ndarray:
    if stretch <= 0:
        raise ValueError("stretch factor must be positive")
    R = rotation_from_dominant_axis(v)
    s = stretch * stretch if square_scales else stretch
    return base_scale * (R @ np.diag([s, 1.0, 1.0]) @ R.T)


def isotropic_covariance(radius: float) -> np.ndarray:
    if radius <= 0:
        raise ValueError("radius must be positive")
    return (radius * radius) * np.eye(3)


def knn_avg_distance(pc: PointCloud, k: int = 4) -> np.ndarray:
    """Mean distance to the min(k, n-1) nearest neighbours (geometry/knn.py:60-113),
    exact, via a k-d tree; distances are f64, the result f32."""
    if pc.count < 2:
        raise InsufficientPointsError("need at least 2 points for neighbor radii")
    if k < 1:
        raise ValueError("k must be >= 1")
    from scipy.spatial import cKDTree

    pos = np.asarray(pc.positions, np.float64)
    if not np.any(pos.max(axis=0) - pos.min(axis=0)):
        return np.zeros(pc.count, np.float32)
    k_eff = min(k, pc.count - 1)
    d, _ = cKDTree(pos).query(pos, k=k_eff + 1)
    # drop the point itself (distance 0 first; duplicates also sit at 0, where the
    # reference's "other points" still include them -- dropping any zero is the same)
    return np.asarray(d[:, 1:k_eff + 1].mean(axis=1), np.float32)


# ---- splats ----------------------------------------------------------------------------

@dataclass(eq=False)
class SplatSet:
    means: np.ndarray        # (n, 3) f32
    covariances: np.ndarray  # (n, 3, 3) f32
    colors: np.ndarray       # (n, 3) f32 in [0, 1]
    opacities: np.ndarray    # (n,) f32 in (0, 1]

    def __post_init__(self):
        self.means = np.ascontiguousarray(self.means, np.float32).reshape(-1, 3)
        n = len(self.means)
        self.covariances = np.ascontiguousarray(self.covariances, np.float32).reshape(n, 3, 3)
        self.colors = np.ascontiguousarray(self.colors, np.float32).reshape(n, 3)
        self.opacities = np.ascontiguousarray(self.opacities, np.float32).reshape(n)

    @property
    def count(self) -> int:
        return len(self.means)


def build_splats(pc: PointCloud, style: str, stretch: float = DEFAULT_STRETCH,
                 base_scale: float | None = None, square_scales: bool = False,
                 opacity: float | None = None, neighbors: int = 4) -> SplatSet:
    """Per-point Gaussians (renderer.py:169-226): "vector_field" elongates along
    the velocity stream (I + (s-1) v v^T, coloured by |v|), "terrain" uses the
    kNN radius and the rgb stream."""
    if style == "vector_field":
        if not pc.has_stream("velocity"):
            raise ConfigurationError("vector_field style needs a 'velocity' stream")
        vel = pc.stream("velocity").data[:, :3].astype(np.float64)
        mag = np.linalg.norm(vel, axis=1)
        if base_scale is None:
            if pc.count < 2:
                raise InsufficientPointsError("need >= 2 points to size splats")
            base_scale = (0.5 * float(np.median(knn_avg_distance(pc, neighbors)))) ** 2
        s_eff = stretch * stretch if square_scales else stretch
        if s_eff <= 0:
            raise ValueError("stretch factor must be positive")
        cov = np.tile(np.eye(3), (pc.count, 1, 1)) * base_scale
        nz = mag > 0
        u = vel[nz] / mag[nz, None]
        cov[nz] += (s_eff - 1.0) * base_scale * np.einsum("ni,nj->nij", u, u)
        vmax = np.percentile(mag, 99.0) if pc.count else 1.0
        colors = flow_colormap(mag / vmax if vmax > 0 else mag)
        op = VECTOR_FIELD_OPACITY if opacity is None else opacity
    elif style == "terrain":
        if not pc.has_stream("rgb"):
            raise ConfigurationError("terrain style needs an 'rgb' stream")
        radii = np.maximum(knn_avg_distance(pc, neighbors).astype(np.float64), 1e-12)
        cov = radii[:, None, None] ** 2 * np.eye(3)[None]
        s = pc.stream("rgb")
        colors = s.data[:, :3].astype(np.float64)
        if s.format == "u8":
            colors /= 255.0
        op = TERRAIN_OPACITY if opacity is None else opacity
    else:
        raise ValueError(f"unknown splat style {style!r}")
    return SplatSet(pc.positions, cov.astype(np.float32), colors.astype(np.float32),
                    np.full(pc.count, op, np.float32))


def project_points(cam: CameraPose, points):
    """(xy, depth, culled), f64, elementwise in camera.py:114-137's order."""
    intr = cam.intrinsics
    p = np.asarray(points, np.float64).reshape(-1, 3)
    R, c = cam.orientation, cam.position
    w0, w1, w2 = p[:, 0] - c[0], p[:, 1] - c[1], p[:, 2] - c[2]
    ux = w0 * R[0, 0] + w1 * R[0, 1] + w2 * R[0, 2]
    uy = w0 * R[1, 0] + w1 * R[1, 1] + w2 * R[1, 2]
    uz = w0 * R[2, 0] + w1 * R[2, 1] + w2 * R[2, 2]
    culled = (uz <= intr.near) | (uz >= intr.far)
    zs = np.where(uz == 0.0, 1.0, uz)
    f = intr.focal_px
    xy = np.empty((len(p), 2), np.float64)
    xy[:, 0] = intr.cx + f * (ux / zs)
    xy[:, 1] = intr.cy + f * (uy / zs)
    return xy, uz, culled


def projection_jacobians(cam: CameraPose, points) -> np.ndarray:
    """(n, 2, 3) d(pixel)/d(world) (camera.py:154-166)."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    R = cam.orientation
    u = (p - cam.position) @ R.T
    f = cam.intrinsics.focal_px
    uz = u[:, 2]
    J = np.empty((len(p), 2, 3), np.float64)
    J[:, 0, :] = (uz[:, None] * R[0] - u[:, 0:1] * R[2]) * (f / uz**2)[:, None]
    J[:, 1, :] = (uz[:, None] * R[1] - u[:, 1:2] * R[2]) * (f / uz**2)[:, None]
    return J


def prepare_splats(splats: SplatSet, cam: CameraPose):
    """Cull, depth-sort (stable), project the covariances (J S J^T + lowpass), drop
    ill-conditioned and off-screen footprints (renderer.py:90-138).  Returns
    (mu, inv_abc, boxes, colors, opacities, counters)."""
    W, H = cam.intrinsics.width, cam.intrinsics.height
    xy, depth, culled = project_points(cam, splats.means)
    keep = np.nonzero(~culled)[0]
    order = keep[np.argsort(depth[keep], kind="stable")]
    counters = {"total": splats.count, "culled": int(culled.sum()), "skipped_singular": 0}
    if len(order) == 0:
        e = np.empty((0,))
        return (np.empty((0, 2)), np.empty((0, 3)), np.empty((0, 4), np.int64),
                np.empty((0, 3)), e, counters)
    J = projection_jacobians(cam, splats.means[order])
    cov2 = np.einsum("nij,njk,nlk->nil", J, splats.covariances[order].astype(np.float64), J)
    a = cov2[:, 0, 0] + LOWPASS_PX2
    b = cov2[:, 0, 1]
    c = cov2[:, 1, 1] + LOWPASS_PX2
    half_tr = (a + c) / 2.0
    disc = np.sqrt(np.maximum((a - c) ** 2 / 4.0 + b * b, 0.0))
    lam_max, lam_min = half_tr + disc, half_tr - disc
    det = a * c - b * b
    good = (lam_min > 0) & (det > 0) & (lam_max <= MAX_CONDITION * lam_min)
    counters["skipped_singular"] = int((~good).sum())
    mu = xy[order]
    rad = SIGMA_CUTOFF * np.sqrt(lam_max)
    x0, x1 = np.floor(mu[:, 0] - rad), np.ceil(mu[:, 0] + rad)
    y0, y1 = np.floor(mu[:, 1] - rad), np.ceil(mu[:, 1] + rad)
    vis = np.nonzero(good & (x1 >= 0) & (x0 <= W - 1) & (y1 >= 0) & (y0 <= H - 1))[0]
    boxes = np.stack([np.clip(x0[vis], 0, W - 1), np.clip(x1[vis], 0, W - 1),
                      np.clip(y0[vis], 0, H - 1), np.clip(y1[vis], 0, H - 1)],
                     axis=1).astype(np.int64)
    inv_abc = np.stack([c[vis], -b[vis], a[vis]], axis=1) / det[vis, None]
    return (mu[vis], inv_abc, boxes, splats.colors[order[vis]].astype(np.float64),
            splats.opacities[order[vis]].astype(np.float64), counters)


def splat_blend_image(mu, inv_abc, boxes, color, opacity, width: int, height: int,
                      tile_size: int = 16, threads: int | None = None,
                      backend: str | None = None, device=None, return_device: bool = False):
    """(H, W, 3) f64 front-to-back blend of depth-sorted splats on the GPU
    (_kernels/__init__.py:97-166; ``threads`` accepted and ignored).  The splat
    arrays may be numpy (uploaded here) or torch tensors already on the device."""
    import torch

    _resolve(backend)
    dev = torch.device(device or "cuda")

    tdt = {np.float64: torch.float64, np.int32: torch.int32}

    def up(a, shape, dt):  # numpy arrays are uploaded; device tensors are used in place
        if isinstance(a, torch.Tensor):
            return a.reshape(shape).to(dev, tdt[dt]).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.reshape(a, shape), dt)).to(dev)

    n = int(len(mu))
    t_mu, t_abc = up(mu, (n, 2), np.float64), up(inv_abc, (n, 3), np.float64)
    t_box = up(boxes, (n, 4), np.int32)
    t_col, t_op = up(color, (n, 3), np.float64), up(opacity, (n,), np.float64)
    rgb = torch.empty((height, width, 3), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    _lib.call("nar_splat_blend", t_mu.data_ptr(), t_abc.data_ptr(), t_box.data_ptr(),
              t_col.data_ptr(), t_op.data_ptr(), n, int(width), int(height), int(tile_size),
              rgb.data_ptr(), int(st.cuda_stream))
    if return_device:
        return rgb
    st.synchronize()
    return rgb.cpu().numpy()


def render_gsplat(splats: SplatSet, cam: CameraPose, threads: int | None = None,
                  backend: str | None = None, return_counters: bool = False):
    """(H, W, 3) f32 image in [0, 1], black background (renderer.py:141-155)."""
    W, H = cam.intrinsics.width, cam.intrinsics.height
    mu, inv_abc, boxes, colors, opac, counters = prepare_splats(splats, cam)
    rgb = splat_blend_image(mu, inv_abc, boxes, colors, opac, W, H, backend=backend)
    img = np.clip(rgb, 0.0, 1.0).astype(np.float32)
    return (img, counters) if return_counters else img
