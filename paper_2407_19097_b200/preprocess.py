"""Data path into the hot path: NARPC files -> device, GPU Morton order.

* ``load_pointcloud`` / ``save_pointcloud``: the NARPC container of
  pkg/src/nar/geometry/pointcloud.py:143-199 (magic "NARPC\\0", u16 version,
  u64 count, u8 stream count, stream headers, f32 positions, stream payloads),
  with the reference's error behaviour (FormatError / CorruptError /
  CapacityError).  ``device=`` uploads the payload straight into a resident
  ``DeviceCloud`` (the positions block is already the kernel's f32 AoS layout).
* ``save_features`` / ``load_features``: the feature-dump container of
  pkg/src/nar/msr/feature_io.py:12-43 (u32 W, u32 H, u16 C, channel names,
  then channel-major f32 planes); ``save_features`` also takes a device
  G-buffer (the padded CNN input) and writes its image extent.
* ``morton_reorder``: pkg/src/nar/geometry/morton.py:9-46 on the GPU -- keys by
  the ``nar_morton_keys`` kernel (f64 quantisation, bit-identical), then a
  stable sort; indices change exactly as the reference's ``pc.take(order)``.
"""

from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _lib
from .errors import CapacityError, CorruptError, FormatError
from .geometry import MAX_STREAMS, PointCloud, Stream

NARPC_MAGIC = b"NARPC\0"
NARPC_VERSION = 1
_CODES = {"u8": 0, "f32": 1}
_NAMES = {0: "u8", 1: "f32"}


def save_pointcloud(pc: PointCloud, path) -> None:
    with open(path, "wb") as f:
        f.write(NARPC_MAGIC)
        f.write(struct.pack("<HQB", NARPC_VERSION, pc.count, len(pc.streams)))
        for s in pc.streams:
            nb = s.name.encode("utf-8")
            if len(nb) > 255:
                raise ValueError(f"stream name too long: {s.name!r}")
            f.write(struct.pack("<B", len(nb)) + nb + struct.pack("<BB", _CODES[s.format], s.arity))
        f.write(np.ascontiguousarray(pc.positions, "<f4").tobytes())
        for s in pc.streams:
            f.write(np.ascontiguousarray(s.data, "<f4" if s.format == "f32" else "u1").tobytes())


def _layout(raw) -> tuple[int, list, int]:
    """Parse the NARPC header; returns (count, [(name, fmt, arity, offset)], end)
    with the payload offsets of the positions block (first) and every stream."""
    def fail(n, at):
        raise CorruptError(f"truncated file: wanted {n} bytes at offset {at}")

    if len(raw) < 6:
        fail(6, 0)
    if bytes(raw[:6]) != NARPC_MAGIC:
        raise FormatError("bad magic, not a NARPC file")
    if len(raw) < 17:
        fail(11, 6)
    version, count, n_streams = struct.unpack_from("<HQB", raw, 6)
    if version != NARPC_VERSION:
        raise FormatError(f"unsupported NARPC version {version}")
    if n_streams > MAX_STREAMS:
        raise CapacityError(f"file declares {n_streams} streams (limit {MAX_STREAMS})")
    at, heads = 17, []
    for _ in range(n_streams):
        if at + 1 > len(raw):
            fail(1, at)
        ln = raw[at]
        if at + 3 + ln > len(raw):
            fail(ln + 2, at + 1)
        name = bytes(raw[at + 1:at + 1 + ln]).decode("utf-8")
        code, arity = raw[at + 1 + ln], raw[at + 2 + ln]
        if code not in _NAMES:
            raise FormatError(f"unknown stream format code {code}")
        heads.append((name, _NAMES[code], arity))
        at += 3 + ln
    blocks = [("positions", "f32", 3, at)]
    at += count * 12
    for name, fmt, arity in heads:
        blocks.append((name, fmt, arity, at))
        at += count * arity * (4 if fmt == "f32" else 1)
    if at > len(raw):
        fail(at - len(raw), len(raw))
    if at < len(raw):
        raise CorruptError(f"{len(raw) - at} trailing bytes after payload")
    return count, blocks, at


def load_pointcloud(path, device=None, pinned: bool = False):
    """Parse a NARPC file (pointcloud.py:160-199).  Returns a host ``PointCloud``
    (optionally in pinned memory), or with ``device=`` a ``DeviceCloud``
    resident on that GPU (payload blocks copied straight from the file image)."""
    raw = memoryview(open(path, "rb").read())
    count, blocks, _ = _layout(raw)
    arrs = [(name, fmt, np.frombuffer(raw, "<f4" if fmt == "f32" else "u1", count * arity,
                                      off).reshape(count, arity))
            for name, fmt, arity, off in blocks]
    (_, _, pos), streams = arrs[0], arrs[1:]
    if device is not None:
        import torch

        from .msr import DeviceCloud, _StreamMeta

        dev = torch.device(device)
        up = lambda a: torch.from_numpy(np.array(a)).to(dev)
        seg = {"begin": 0, "positions": up(pos), "streams": {n: up(d) for n, _, d in streams}}
        meta = {n: _StreamMeta(n, fmt, d.shape[1]) for n, fmt, d in streams}
        return DeviceCloud([seg], meta, dev)
    return PointCloud(np.array(pos), [Stream(n, fmt, np.array(d)) for n, fmt, d in streams],
                      pinned=pinned)


def _aabb(positions) -> tuple[np.ndarray, np.ndarray]:
    """pointcloud.py:38-44 Aabb.of_points: per-axis min / max as f64."""
    import torch

    if positions.shape[0] == 0:
        return np.full(3, np.inf), np.full(3, -np.inf)
    lo, hi = torch.aminmax(positions, dim=0)
    return lo.double().cpu().numpy(), hi.double().cpu().numpy()


def morton_keys_device(positions, lo=None, hi=None):
    """63-bit Morton keys (int64 tensor) of device positions (n, 3) f32."""
    import torch

    from .msr import _check_positions

    _check_positions(positions)

    if lo is None or hi is None:
        lo, hi = _aabb(positions)
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    keys = torch.empty(positions.shape[0], dtype=torch.int64, device=positions.device)
    _lib.call("nar_morton_keys", positions.data_ptr(), int(positions.shape[0]), lo.ctypes.data,
              hi.ctypes.data, keys.data_ptr(), _lib.stream_handle(None))
    return keys


def morton_reorder(cloud):
    """Stable reorder by Morton key (morton.py:40-46) of a host PointCloud (computed
    on the GPU, returned on the host) or of a single-buffer DeviceCloud."""
    import torch

    from .msr import DeviceCloud

    if isinstance(cloud, DeviceCloud):
        if len(cloud.segments) != 1:
            raise ValueError("morton_reorder needs a single-buffer DeviceCloud")
        sg = cloud.segments[0]
        if sg["count"] == 0:
            return cloud
        order = torch.sort(morton_keys_device(sg["positions"]), stable=True).indices
        seg = {"begin": sg["begin"], "positions": sg["positions"][order].contiguous(),
               "streams": {n: t[order].contiguous() for n, t in sg["streams"].items()}}
        return DeviceCloud([seg], cloud.meta, cloud.device)
    if cloud.count == 0:
        return cloud
    pos_d = torch.from_numpy(np.ascontiguousarray(cloud.positions)).cuda()
    order = torch.sort(morton_keys_device(pos_d), stable=True).indices.cpu().numpy()
    return cloud.take(order)


# ---- feature dumps (msr/feature_io.py) ---------------------------------------------

def save_features(names, data, path, height: int | None = None, width: int | None = None) -> None:
    """Write (H, W, C) f32 planes channel-major (feature_io.py:12-23).  ``data`` may
    be a numpy array or a device tensor (e.g. a DeviceFeatureImage's padded
    ``data``); ``height``/``width`` crop it to the image extent."""
    if hasattr(data, "detach"):
        data = data.detach()
        if height is not None:
            data = data[:height, :width]
        planes = data.permute(2, 0, 1).contiguous().cpu().numpy()
    else:
        data = np.asarray(data)
        if height is not None:
            data = data[:height, :width]
        planes = np.ascontiguousarray(np.moveaxis(data, 2, 0))
    c, h, w = planes.shape
    names = tuple(names)
    if c != len(names):
        raise ValueError(f"{len(names)} channel names for {c} planes")
    head = [struct.pack("<IIH", w, h, c)]
    for n in names:
        nb = n.encode("utf-8")
        head.append(struct.pack("<B", len(nb)) + nb)
    with open(path, "wb") as f:
        f.write(b"".join(head))
        f.write(np.ascontiguousarray(planes, "<f4").tobytes())


def load_features(path):
    """(names, (H, W, C) f32) from a feature dump; CorruptError on a short header
    or a payload of the wrong size (feature_io.py:26-43)."""
    raw = memoryview(open(path, "rb").read())
    if len(raw) < 10:
        raise CorruptError("feature dump too short for header")
    w, h, c = struct.unpack_from("<IIH", raw, 0)
    off, names = 10, []
    for _ in range(c):
        if off >= len(raw):
            raise CorruptError("feature dump truncated in the channel names")
        n = raw[off]
        names.append(bytes(raw[off + 1:off + 1 + n]).decode("utf-8"))
        off += 1 + n
    want = w * h * c * 4
    if len(raw) - off != want:
        raise CorruptError(f"feature dump payload is {len(raw) - off} bytes, wanted {want}")
    planes = np.frombuffer(raw, "<f4", count=w * h * c, offset=off).reshape(c, h, w)
    return tuple(names), np.ascontiguousarray(np.moveaxis(planes, 0, 2))

