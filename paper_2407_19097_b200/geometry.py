"""Cameras and point clouds as consumed by the MSR kernels.

API-compatible with the reference's ``nar.geometry`` types on the hot path:
``Intrinsics`` / ``CameraPose`` / ``look_at`` (pkg/src/nar/geometry/camera.py:26-96)
and ``PointCloud`` / ``Stream`` (pkg/src/nar/geometry/pointcloud.py:65-131).

B200 additions: ``PointCloud(..., pinned=True)`` places positions and streams
in page-locked host memory so the per-frame H2D copy is an async DMA, and
``PointCloud.to_device()`` uploads the cloud once into a resident
``DeviceCloud`` (positions f32 AoS, streams (n, arity) in their stored dtype).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .errors import CapacityError, FormatError

MAX_STREAMS = 8
_DTYPES = {"u8": np.uint8, "f32": np.float32}


# ---------------------------------------------------------------------------
# camera (camera.py:26-96)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Intrinsics:
    """Square-pixel pinhole model; principal point at the image centre."""

    fov_y_deg: float = 60.0
    near: float = 0.1
    far: float = 2.0e5
    width: int = 512
    height: int = 512

    def __post_init__(self):
        if not (0.0 < self.near < self.far):
            raise ValueError(f"need 0 < near < far, got {self.near}, {self.far}")
        if not (0.0 < self.fov_y_deg < 180.0):
            raise ValueError(f"bad vertical FOV {self.fov_y_deg}")

    @property
    def focal_px(self) -> float:
        half = math.radians(self.fov_y_deg) / 2.0
        return (self.height / 2.0) / math.tan(half)

    @property
    def cx(self) -> float:
        return self.width / 2.0

    @property
    def cy(self) -> float:
        return self.height / 2.0


@dataclass(frozen=True, eq=False)
class CameraPose:
    """World->camera pose; orientation rows are the camera right/down/forward axes."""

    position: np.ndarray
    orientation: np.ndarray
    intrinsics: Intrinsics = field(default_factory=Intrinsics)

    def __post_init__(self):
        pos = np.asarray(self.position, np.float64).reshape(3)
        rot = np.asarray(self.orientation, np.float64).reshape(3, 3)
        dev = float(np.max(np.abs(rot.T @ rot - np.eye(3))))
        if dev > 1e-6:
            raise ValueError(f"orientation not orthonormal (|R^T R - I| = {dev:.2e})")
        object.__setattr__(self, "position", pos)
        object.__setattr__(self, "orientation", rot)

    @property
    def forward(self) -> np.ndarray:
        return self.orientation[2]

    def with_intrinsics(self, intr: Intrinsics) -> "CameraPose":
        return replace(self, intrinsics=intr)

    def kernel_camera(self):
        """The C-ABI ``nar_camera`` for this pose (cached per pose: a frame-rate
        loop builds it once; the key includes the arrays' bytes, so an in-place
        edit of position / orientation is still seen)."""
        from . import _lib

        i = self.intrinsics
        key = (self.position.tobytes(), self.orientation.tobytes(), i)
        cached = self.__dict__.get("_kc")
        if cached is not None and cached[0] == key:
            return cached[1]
        kc = _lib.make_camera(self.orientation.reshape(-1), self.position, i.focal_px,
                              i.cx, i.cy, i.near, i.far, i.width, i.height)
        object.__setattr__(self, "_kc", (key, kc))
        return kc


def _unit(v: np.ndarray) -> np.ndarray:
    n = float(np.linalg.norm(v))
    if n == 0.0:
        raise ValueError("cannot normalize zero vector")
    return v / n


def look_at(position, target, intrinsics: Intrinsics | None = None) -> CameraPose:
    """Pose at ``position`` looking at ``target`` with world +z up (+y when the
    view is near vertical), same basis construction as camera.py:82-96."""
    eye = np.asarray(position, np.float64)
    fwd = _unit(np.asarray(target, np.float64) - eye)
    up = np.array([0.0, 0.0, 1.0])
    if abs(float(fwd @ up)) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = _unit(np.cross(fwd, up))
    down = np.cross(fwd, right)
    return CameraPose(eye, np.stack([right, down, fwd]), intrinsics or Intrinsics())


def pose_from_yaw_pitch(position, yaw_deg: float, pitch_deg: float,
                        intrinsics: Intrinsics | None = None) -> CameraPose:
    yaw, pitch = math.radians(yaw_deg), math.radians(pitch_deg)
    d = np.array([math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw),
                  -math.sin(pitch)])
    eye = np.asarray(position, np.float64)
    return look_at(eye, eye + d, intrinsics)


# ---------------------------------------------------------------------------
# point cloud (pointcloud.py:65-131)
# ---------------------------------------------------------------------------
def _pinned_empty(shape, dtype) -> np.ndarray:
    """numpy view of page-locked host memory (torch's caching host allocator)."""
    import torch

    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.uint8): torch.uint8}[np.dtype(dtype)]
    t = torch.empty(tuple(shape), dtype=tdt, pin_memory=True)
    arr = t.numpy()
    # keep the torch storage alive as long as the array lives
    return _PinnedArray(arr, t)


class _PinnedArray(np.ndarray):
    def __new__(cls, arr, owner):
        obj = arr.view(cls)
        obj._owner = owner
        return obj

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


@dataclass
class Stream:
    """Named per-point attribute block of shape (count, arity), u8 or f32."""

    name: str
    format: str
    data: np.ndarray

    def __post_init__(self):
        if self.format not in _DTYPES:
            raise FormatError(f"unknown stream format {self.format!r}")
        self.data = np.ascontiguousarray(self.data, dtype=_DTYPES[self.format])
        if self.data.ndim != 2:
            raise ValueError("stream data must be (count, arity)")

    @property
    def arity(self) -> int:
        return int(self.data.shape[1])


class PointCloud:
    """Positions (n, 3) f32 AoS plus up to eight attribute streams."""

    def __init__(self, positions: np.ndarray, streams: list[Stream] | None = None,
                 pinned: bool = False):
        pos = np.ascontiguousarray(positions, dtype=np.float32).reshape(-1, 3)
        streams = list(streams or [])
        if len(streams) > MAX_STREAMS:
            raise CapacityError(f"{len(streams)} streams exceed the limit of {MAX_STREAMS}")
        for s in streams:
            if len(s.data) != len(pos):
                raise ValueError(f"stream {s.name!r} has {len(s.data)} rows for {len(pos)} points")
        if pinned:
            p = _pinned_empty(pos.shape, np.float32)
            p[...] = pos
            pos = p
            pinned_streams = []
            for s in streams:
                d = _pinned_empty(s.data.shape, s.data.dtype)
                d[...] = s.data
                st = Stream.__new__(Stream)
                st.name, st.format, st.data = s.name, s.format, d
                pinned_streams.append(st)
            streams = pinned_streams
        self.positions = pos
        self.streams = streams
        self.pinned = pinned

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])

    def stream_names(self) -> list[str]:
        return [s.name for s in self.streams]

    def has_stream(self, name: str) -> bool:
        return any(s.name == name for s in self.streams)

    def stream(self, name: str) -> Stream:
        for s in self.streams:
            if s.name == name:
                return s
        raise KeyError(f"no stream named {name!r}")

    def take(self, indices: np.ndarray) -> "PointCloud":
        return PointCloud(self.positions[indices],
                          [Stream(s.name, s.format, s.data[indices]) for s in self.streams])

    def to_device(self, device=None, streams: list[str] | None = None):
        from .msr import DeviceCloud

        return DeviceCloud.from_host(self, device=device, streams=streams)

    def __repr__(self):
        desc = ", ".join(f"{s.name}:{s.format}x{s.arity}" for s in self.streams)
        return f"PointCloud(count={self.count}, streams=[{desc}])"
