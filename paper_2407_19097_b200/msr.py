"""Multi-Stream Rasterizer on B200: render (project + early-z) and resolve.

Reference API kept (pkg/src/nar/msr/rasterizer.py:27-188):
``StreamSelection``, ``FeatureImage``, ``rasterize(pc, cam, sel, threads=None,
backend=None)``.  ``rasterize`` on a host ``PointCloud`` is the drop-in: it
uploads the points (chunked H2D overlapped with the render kernel), renders
into a device keybuf, resolves on the device and returns host planes that are
bit-identical to the reference's for the rgb / d / scalar / coverage channels
and the index / depth / coverage planes (vel channels: <= 1 f32 ulp, see
DESIGN.md).

The device-resident path for throughput (the benchmark's ``value``) is
``DeviceCloud`` + ``Renderer``: the cloud is uploaded once, each frame runs
``nar_render`` once per point buffer -- one CUDA stream per data stream, all
folding into one keybuf with atomics -- then one ``nar_resolve`` launch that
also re-clears the keybuf for the next frame.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._kernels import EMPTY_KEY, _resolve
from .errors import ConfigurationError
from .geometry import CameraPose, PointCloud

MAX_CHANNELS = 16
VEL2D_CHANNELS = ("v2x", "v2y", "v2t", "v2m")
VEL3D_CHANNELS = ("v3x", "v3y", "v3z", "v3m")
_FMT = {"u8": _lib.FMT_U8, "f32": _lib.FMT_F32}


@dataclass(frozen=True)
class StreamSelection:
    """Which point attributes become raster channels (rasterizer.py:27-91)."""

    rgb: bool = True
    depth: bool = False
    vel2d: bool = False
    vel3d: bool = False
    scalars: tuple[str, ...] = ()
    coverage_channel: bool = False
    velocity_scale: float = 1.0
    rgb_stream: str = "rgb"
    velocity_stream: str = "velocity"

    def channel_names(self, pc=None) -> tuple[str, ...]:
        out: list[str] = []
        if self.rgb:
            out.extend(("r", "g", "b"))
        if self.depth:
            out.append("d")
        if self.vel2d:
            out.extend(VEL2D_CHANNELS)
        if self.vel3d:
            out.extend(VEL3D_CHANNELS)
        for name in self.scalars:
            ar = pc.stream(name).arity if (pc is not None and pc.has_stream(name)) else 1
            out.extend([name] if ar == 1 else [f"{name}{i}" for i in range(ar)])
        if self.coverage_channel:
            out.append("coverage")
        return tuple(out)

    def validate(self, pc) -> None:
        if self.rgb and not pc.has_stream(self.rgb_stream):
            raise ConfigurationError(f"selection needs stream {self.rgb_stream!r}")
        if (self.vel2d or self.vel3d) and not pc.has_stream(self.velocity_stream):
            raise ConfigurationError(f"selection needs stream {self.velocity_stream!r}")
        for name in self.scalars:
            if not pc.has_stream(name):
                raise ConfigurationError(f"selection needs stream {name!r}")
        n = len(self.channel_names(pc))
        if n > MAX_CHANNELS:
            raise ConfigurationError(f"{n} channels exceed the limit of {MAX_CHANNELS}")

    def needed_streams(self) -> list[str]:
        names = []
        if self.rgb:
            names.append(self.rgb_stream)
        if self.vel2d or self.vel3d:
            names.append(self.velocity_stream)
        names.extend(self.scalars)
        return list(dict.fromkeys(names))

    def to_dict(self) -> dict:
        return {"rgb": self.rgb, "depth": self.depth, "vel2d": self.vel2d, "vel3d": self.vel3d,
                "scalars": list(self.scalars), "coverage_channel": self.coverage_channel,
                "velocity_scale": self.velocity_scale, "rgb_stream": self.rgb_stream,
                "velocity_stream": self.velocity_stream}

    @staticmethod
    def from_dict(d: dict) -> "StreamSelection":
        d = dict(d)
        d["scalars"] = tuple(d.get("scalars", ()))
        return StreamSelection(**d)


@dataclass(eq=False)
class FeatureImage:
    """Raster output (rasterizer.py:94-113): (H, W, C) f32 planes + bookkeeping."""

    width: int
    height: int
    channel_names: tuple[str, ...]
    data: np.ndarray
    coverage: np.ndarray
    index_plane: np.ndarray
    depth: np.ndarray = field(default=None)

    def plane(self, name: str) -> np.ndarray:
        return self.data[:, :, self.channel_names.index(name)]

    def rgb(self) -> np.ndarray:
        if not {"r", "g", "b"} <= set(self.channel_names):
            raise ConfigurationError("feature image has no RGB channels")
        return np.stack([self.plane("r"), self.plane("g"), self.plane("b")], axis=-1)


# ---------------------------------------------------------------------------
# device-resident clouds
# ---------------------------------------------------------------------------
class _StreamMeta:
    __slots__ = ("name", "format", "arity")

    def __init__(self, name, fmt, arity):
        self.name, self.format, self.arity = name, fmt, arity


class DeviceCloud:
    """Point buffers resident in HBM; each buffer is one data stream / segment.

    ``segments[k]`` = dict(begin, positions (n,3) f32 tensor, streams {name: tensor}).
    Segment k's points carry global indices ``begin .. begin+n-1`` (the base
    index of the reference's chunked render, _kernels/__init__.py:81-87).
    """

    def __init__(self, segments: list[dict], meta: dict[str, _StreamMeta], device):
        if len(segments) > _lib.MAX_SEGMENTS:
            raise ConfigurationError(f"at most {_lib.MAX_SEGMENTS} point buffers per cloud")
        self.segments = segments
        self.meta = meta
        self.device = device
        for s in segments:
            s.setdefault("count", int(s["positions"].shape[0]) if s.get("positions") is not None else 0)
        self.count = sum(s["count"] for s in segments)
        end = max((s["begin"] + s["count"] for s in segments), default=0)
        if end > 1 << 32:
            raise ConfigurationError("global point indices must fit in 32 bits")

    # -- construction -------------------------------------------------------
    @staticmethod
    def _upload(arr: np.ndarray, device):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(arr))
        return t.to(device, non_blocking=True)

    @classmethod
    def from_host(cls, pc: PointCloud, device=None, streams: list[str] | None = None,
                  begin: int = 0) -> "DeviceCloud":
        return cls.from_clouds([pc], device=device, streams=streams, begins=[begin])

    @classmethod
    def from_clouds(cls, clouds: list[PointCloud], device=None, streams: list[str] | None = None,
                    begins: list[int] | None = None) -> "DeviceCloud":
        """Multi-stream cloud: one device buffer per input cloud.  Default base
        indices are the running sums of the counts, so rendering equals the
        reference ``rasterize`` of the concatenated cloud."""
        import torch

        device = torch.device(device or "cuda")
        if begins is None:
            begins, acc = [], 0
            for pc in clouds:
                begins.append(acc)
                acc += pc.count
        meta: dict[str, _StreamMeta] = {}
        segs = []
        for pc, b in zip(clouds, begins):
            names = streams if streams is not None else pc.stream_names()
            st = {}
            for name in names:
                s = pc.stream(name)
                m = meta.setdefault(name, _StreamMeta(name, s.format, s.arity))
                if (m.format, m.arity) != (s.format, s.arity):
                    raise ConfigurationError(f"stream {name!r} differs between point buffers")
                st[name] = cls._upload(s.data, device)
            segs.append({"begin": int(b), "positions": cls._upload(pc.positions, device),
                         "streams": st})
        return cls(segs, meta, device)

    @classmethod
    def from_tensors(cls, positions, streams: dict | None = None, formats: dict | None = None,
                     begin: int = 0) -> "DeviceCloud":
        """Wrap device tensors generated in place (no host copy).  The kernels read
        them through raw pointers, so layouts are checked here: positions (n, 3)
        float32, streams (n, arity) uint8 / float32, all contiguous on one GPU."""
        import torch

        _check_positions(positions)
        n = int(positions.shape[0])
        meta, st = {}, {}
        for name, t in (streams or {}).items():
            if (not isinstance(t, torch.Tensor) or t.dim() != 2 or int(t.shape[0]) != n
                    or not t.is_contiguous() or t.device != positions.device
                    or t.dtype not in (torch.uint8, torch.float32)):
                raise ValueError(f"stream {name!r} must be a contiguous (n, arity) uint8 or "
                                 f"float32 tensor on {positions.device} with n = {n}")
            fmt = (formats or {}).get(name, "u8" if str(t.dtype) == "torch.uint8" else "f32")
            if (fmt == "u8") != (t.dtype == torch.uint8):
                raise ValueError(f"stream {name!r}: format {fmt!r} does not match {t.dtype}")
            meta[name] = _StreamMeta(name, fmt, int(t.shape[1]))
            st[name] = t
        return cls([{"begin": int(begin), "positions": positions, "streams": st}], meta,
                   positions.device)

    def has_stream(self, name: str) -> bool:
        return name in self.meta

    def stream(self, name: str) -> _StreamMeta:
        if name not in self.meta:
            raise KeyError(f"no stream named {name!r}")
        return self.meta[name]


@dataclass
class DeviceFeatureImage:
    """Device tensors of one resolved frame (see FeatureImage)."""

    width: int
    height: int
    channel_names: tuple[str, ...]
    data: object          # torch (data_h, data_w, C) f32 (padded extent)
    coverage: object      # torch (H, W) u8, or None (not resolved)
    index_plane: object   # torch (H, W) i64, or None
    depth: object         # torch (H, W) f32, or None

    def to_host(self) -> FeatureImage:
        d = self.data[: self.height, : self.width].cpu().numpy()
        if self.coverage is None or self.index_plane is None or self.depth is None:
            raise ValueError("this frame was resolved without its coverage / index / depth planes")
        return FeatureImage(self.width, self.height, self.channel_names, np.ascontiguousarray(d),
                            self.coverage.cpu().numpy(), self.index_plane.cpu().numpy(),
                            self.depth.cpu().numpy())


def _selection_struct(sel: StreamSelection, cloud) -> "_lib.Selection":
    s = _lib.Selection()
    s.rgb, s.depth, s.vel2d, s.vel3d = int(sel.rgb), int(sel.depth), int(sel.vel2d), int(sel.vel3d)
    s.coverage_channel = int(sel.coverage_channel)
    if sel.rgb:
        m = cloud.stream(sel.rgb_stream)
        s.rgb_format, s.rgb_arity = _FMT[m.format], m.arity
        if not (m.arity == 1 or m.arity >= 3):
            raise ValueError(f"rgb stream of arity {m.arity} cannot fill 3 channels")
    if sel.vel2d or sel.vel3d:
        m = cloud.stream(sel.velocity_stream)
        s.vel_format, s.vel_arity = _FMT[m.format], m.arity
    if len(sel.scalars) > _lib.MAX_SCALARS:
        raise ConfigurationError("too many scalar streams")
    s.n_scalars = len(sel.scalars)
    for q, name in enumerate(sel.scalars):
        m = cloud.stream(name)
        s.scalar_format[q], s.scalar_arity[q] = _FMT[m.format], m.arity
    s.velocity_scale = float(sel.velocity_scale)
    return s


def _segments_struct(cloud: DeviceCloud, sel: StreamSelection):
    arr = (_lib.Segment * _lib.MAX_SEGMENTS)()
    for k, sg in enumerate(cloud.segments):
        a = arr[k]
        a.begin = sg["begin"]
        a.count = sg["count"]
        a.positions = sg["positions"].data_ptr() if sg.get("positions") is not None else None
        st = sg["streams"]
        if sel.rgb:
            a.rgb = st[sel.rgb_stream].data_ptr()
        if sel.vel2d or sel.vel3d:
            a.velocity = st[sel.velocity_stream].data_ptr()
        for q, name in enumerate(sel.scalars):
            a.scalars[q] = st[name].data_ptr()
    return arr


class Renderer:
    """Per-resolution frame state: the u64 keybuf (kept EMPTY between frames)
    and the CUDA streams used for multi-stream rendering."""

    def __init__(self, width: int, height: int, device=None, signed_keys: bool = False,
                 pad_multiple: int | None = None):
        import torch

        self.width, self.height = int(width), int(height)
        self.device = torch.device(device or "cuda")
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.domain = _lib.KEYS_SIGNED if signed_keys else _lib.KEYS_UNSIGNED
        self.empty = (_lib.EMPTY_KEY ^ _lib.SIGN_FLIP) if signed_keys else _lib.EMPTY_KEY
        npix = self.width * self.height
        self.keybuf = torch.empty(npix, dtype=torch.int64, device=self.device)
        nb = C.c_size_t(0)
        _lib.check(_lib.load().nar_hiz_scratch_bytes(self.width, self.height, C.byref(nb)))
        self.hiz = torch.empty(int(nb.value) // 4, dtype=torch.int32, device=self.device)
        self.use_hiz = True
        self.pad_multiple = pad_multiple
        self._lock = threading.Lock()  # rasterize() serialises calls sharing this renderer
        self._streams: list = []
        self.clear()

    @property
    def npix(self) -> int:
        return self.width * self.height

    def clear(self, stream=None) -> None:
        with _lib.on_device(self.device.index):
            _lib.call("nar_keybuf_fill", self.keybuf.data_ptr(), self.npix,
                      C.c_uint64(self.empty), _lib.stream_handle(stream, self.device.index))

    def _check_cam(self, cam: CameraPose):
        i = cam.intrinsics
        if (i.width, i.height) != (self.width, self.height):
            raise ValueError("camera resolution differs from the renderer's")
        return cam.kernel_camera()

    def render(self, cloud: DeviceCloud, cam: CameraPose, stream=None,
               multi_stream: bool = True) -> None:
        """Fold every point buffer of ``cloud`` into the keybuf; with several
        buffers and ``multi_stream`` each renders on its own CUDA stream."""
        with _lib.on_device(self.device.index):
            self._render(cloud, cam, stream, multi_stream)

    def _render(self, cloud, cam, stream, multi_stream) -> None:
        import torch

        kc = self._check_cam(cam)
        segs = cloud.segments

        def launch(sg, handle, has_frame):
            n = int(sg["positions"].shape[0])
            if self.use_hiz:
                _lib.call("nar_render_hiz", self.keybuf.data_ptr(), self.hiz.data_ptr(),
                          sg["positions"].data_ptr(), n, C.c_uint64(sg["begin"]), C.byref(kc),
                          self.domain, int(has_frame), handle)
            else:
                _lib.call("nar_render", self.keybuf.data_ptr(), sg["positions"].data_ptr(), n,
                          C.c_uint64(sg["begin"]), C.byref(kc), self.domain, handle)

        if len(segs) <= 1 or not multi_stream:
            handle = _lib.stream_handle(stream, self.device.index)
            for k, sg in enumerate(segs):
                launch(sg, handle, k > 0)
            return
        main = stream or torch.cuda.current_stream(self.device)
        while len(self._streams) < len(segs):
            self._streams.append(torch.cuda.Stream(self.device))
        start = torch.cuda.Event()
        start.record(main)
        for sg, st in zip(segs, self._streams):
            st.wait_event(start)
            launch(sg, int(st.cuda_stream), False)
        for st in self._streams[: len(segs)]:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)

    def alloc_outputs(self, n_channels: int, planes: bool = True):
        """G-buffer tensors for resolve(out=...).  ``planes=False``: only the (padded)
        channel data -- the coverage / index / depth planes are then not written
        (the neural pipeline feeds the CNN from ``data`` alone)."""
        import torch

        H, W = self.height, self.width
        m = self.pad_multiple or 1
        ph, pw = H + (-H) % m, W + (-W) % m
        dev = self.device
        out = {"data": torch.empty((ph, pw, n_channels), dtype=torch.float32, device=dev)}
        if planes:
            out.update({"coverage": torch.empty((H, W), dtype=torch.uint8, device=dev),
                        "index_plane": torch.empty((H, W), dtype=torch.int64, device=dev),
                        "depth": torch.empty((H, W), dtype=torch.float32, device=dev)})
        return out

    def resolve(self, cloud: DeviceCloud, cam: CameraPose, sel: StreamSelection, out=None,
                stream=None, clear: bool = True, owner_only: bool = False,
                peers: list[int] | None = None, rows: tuple[int, int] | None = None,
                pix_rgb=None) -> DeviceFeatureImage:
        """Decode + channel fill.  ``peers`` (device addresses of keybufs, e.g.
        other GPUs' buffers mapped here) makes it the fused composite + resolve
        (``nar_resolve_peers``): the pixel key is the min over them, and only the
        output ``rows`` [r0, r1) are written.  ``out`` tensors may themselves be
        peer buffers (``_Mapped``) so a rank writes its slice straight into the
        root's G-buffer.  ``pix_rgb`` (device int32 (H*W,)): the winners' rgb bytes per
        pixel, gathered on the host (``nar_host_gather_rgb``; RGB+D only)."""
        sel.validate(cloud)
        kc = self._check_cam(cam)
        names = sel.channel_names(cloud)
        if out is None:
            out = self.alloc_outputs(len(names))
        else:
            _check_outputs(out, len(names), self.height, self.width)
        ro = _lib.ResolveOut()
        if "data" in out:  # (absent: the planes alone)
            ro.data = out["data"].data_ptr()
            ro.data_h, ro.data_w = int(out["data"].shape[0]), int(out["data"].shape[1])
        # planes are optional (nar_resolve_out: NULL = not written)
        ro.coverage = out["coverage"].data_ptr() if "coverage" in out else None
        ro.index_plane = out["index_plane"].data_ptr() if "index_plane" in out else None
        ro.depth = out["depth"].data_ptr() if "depth" in out else None
        ro.owner_only, ro.clear_keybuf = int(owner_only), int(clear)
        s = _selection_struct(sel, cloud)
        segs = _segments_struct(cloud, sel)
        with _lib.on_device(self.device.index):
            if pix_rgb is not None:
                r0, r1 = rows if rows is not None else (0, -1)
                _lib.call("nar_resolve_pixrgb", self.keybuf.data_ptr(), int(r0), int(r1),
                          C.byref(kc), self.domain, C.byref(s), segs, len(cloud.segments),
                          C.byref(ro), pix_rgb.data_ptr(),
                          _lib.stream_handle(stream, self.device.index))
            else:
                self._resolve_call(kc, s, segs, len(cloud.segments), ro, stream, peers, rows)
        return DeviceFeatureImage(self.width, self.height, names, out.get("data"),
                                  out.get("coverage"), out.get("index_plane"), out.get("depth"))

    def _resolve_call(self, kc, s, segs, nseg, ro, stream, peers, rows) -> None:
        if peers is None:
            _lib.call("nar_resolve", self.keybuf.data_ptr(), C.byref(kc), self.domain, C.byref(s),
                      segs, nseg, C.byref(ro), _lib.stream_handle(stream, self.device.index))
        else:
            arr = (C.c_void_p * len(peers))(*[int(p) for p in peers])
            r0, r1 = rows if rows is not None else (0, -1)
            _lib.call("nar_resolve_peers", arr, len(peers), int(r0), int(r1), C.byref(kc),
                      self.domain, C.byref(s), segs, nseg, C.byref(ro),
                      _lib.stream_handle(stream, self.device.index))

    def rasterize(self, cloud: DeviceCloud, cam: CameraPose, sel: StreamSelection, out=None,
                  stream=None) -> DeviceFeatureImage:
        self.render(cloud, cam, stream=stream)
        return self.resolve(cloud, cam, sel, out=out, stream=stream)

    def keys(self) -> np.ndarray:
        """Current keybuf as host uint64 in the reference (unsigned) layout."""
        k = self.keybuf.cpu().numpy().view(np.uint64)
        if self.domain == _lib.KEYS_SIGNED:
            k = k ^ np.uint64(_lib.SIGN_FLIP)
        return k


class _Mapped:
    """A host array's device address (mapped pinned memory), tensor-like enough
    for the segment table."""

    def __init__(self, ptr: int, shape):
        self._ptr, self.shape = ptr, tuple(shape)

    def data_ptr(self) -> int:
        return self._ptr


_renderers: dict = {}


def _check_positions(positions) -> None:
    import torch

    if (not isinstance(positions, torch.Tensor) or not positions.is_cuda
            or positions.dtype != torch.float32 or positions.dim() != 2
            or int(positions.shape[1]) != 3 or not positions.is_contiguous()):
        raise ValueError("positions must be a contiguous (n, 3) float32 CUDA tensor")


def _check_outputs(out: dict, n_channels: int, H: int, W: int) -> None:
    """Caller-provided G-buffer tensors must match the selection and the frame:
    the kernel writes through raw pointers, so a mismatch would corrupt memory."""
    import torch

    if not any(k in out for k in ("data", "coverage", "index_plane", "depth")):
        raise ValueError("out needs 'data' and / or planes")
    d = out.get("data")
    if d is not None:
        ds = tuple(d.shape)
        if len(ds) != 3 or ds[2] != n_channels or ds[0] < H or ds[1] < W:
            raise ValueError(f"out['data'] must be (>= {H}, >= {W}, {n_channels}) for this "
                             f"selection, got {ds}")
    want = {"data": torch.float32, "coverage": torch.uint8, "index_plane": torch.int64,
            "depth": torch.float32}
    for k, dt in want.items():
        if k not in out:  # optional: data or planes not written
            continue
        t = out[k]
        if k != "data" and tuple(t.shape) != (H, W):
            raise ValueError(f"out[{k!r}] must be ({H}, {W}), got {tuple(t.shape)}")
        if isinstance(t, torch.Tensor) and (t.dtype != dt or not t.is_contiguous()
                                            or (isinstance(d, torch.Tensor) and t.device != d.device)):
            raise ValueError(f"out[{k!r}] must be a contiguous {dt} tensor on the data's device")


def _renderer_for(width: int, height: int, device) -> Renderer:
    key = (width, height, str(device))
    r = _renderers.get(key)
    if r is None:
        if len(_renderers) > 8:
            _renderers.clear()
        r = _renderers[key] = Renderer(width, height, device)
    return r


def rasterize(pc: PointCloud, cam: CameraPose, sel: StreamSelection, threads: int | None = None,
              backend: str | None = None) -> FeatureImage:
    """Render + resolve a host point cloud on the GPU (rasterizer.py:123-188).

    ``threads`` is accepted for signature compatibility and ignored.  Points
    are copied host->device inside this call (async DMA when pinned); with a
    ``PointCloud(..., pinned=True)`` the attribute streams are not copied at
    all -- the resolve reads the winners' attributes in place.  Thread-safe:
    calls sharing a resolution share one cached Renderer and are serialised.
    """
    import torch

    _resolve(backend)
    sel.validate(pc)
    intr = cam.intrinsics
    dev = torch.device("cuda", torch.cuda.current_device())
    r = _renderer_for(intr.width, intr.height, dev)
    with r._lock:
        return _rasterize(pc, cam, sel, r, dev)


def _rasterize(pc: PointCloud, cam: CameraPose, sel: StreamSelection, r: "Renderer", dev):
    import torch

    intr = cam.intrinsics
    W, H = intr.width, intr.height
    main = torch.cuda.current_stream(dev)
    kc = cam.kernel_camera()
    names = sel.needed_streams()
    # Large pageable arrays (a stock caller's numpy PointCloud) are page-locked
    # in place on first use and stay registered while the arrays live, so the
    # points go up by async DMA and the attributes are read zero-copy, exactly
    # as for PointCloud(..., pinned=True) (NAR_HOST_REGISTER=0 disables this).
    if not getattr(pc, "pinned", False):
        _lib.ensure_registered(pc.positions)
        for n in names:
            _lib.ensure_registered(pc.stream(n).data)
    # Attribute streams in mapped pinned memory are not uploaded: the resolve
    # gathers just the winners' attributes through their device address
    # (zero-copy over PCIe).  Pageable streams go up on a side stream while the
    # points stream through nar_render_host's chunk pipeline on the main stream.
    if getattr(r, "_side", None) is None:
        r._side = torch.cuda.Stream(dev)
    side = r._side
    side.wait_stream(main)
    segs_streams, pos_dev = {}, None
    with torch.cuda.stream(side):
        for n in names:
            d = pc.stream(n).data
            mp = _lib.mapped_pointer(d.ctypes.data) if d.size else None
            segs_streams[n] = (_Mapped(mp, d.shape) if mp is not None else
                               torch.from_numpy(d).to(dev, non_blocking=True))
        if sel.vel2d:
            mp = _lib.mapped_pointer(pc.positions.ctypes.data) if pc.count else None
            pos_dev = (_Mapped(mp, pc.positions.shape) if mp is not None else
                       torch.from_numpy(pc.positions).to(dev, non_blocking=True))
    _lib.call("nar_render_host", r.keybuf.data_ptr(), pc.positions.ctypes.data, pc.count,
              C.c_uint64(0), C.byref(kc), r.domain, int(main.cuda_stream))
    main.wait_stream(side)
    meta = {n: _StreamMeta(n, pc.stream(n).format, pc.stream(n).arity) for n in names}
    cloud = DeviceCloud([{"begin": 0, "count": pc.count, "positions": pos_dev,
                          "streams": segs_streams}], meta, dev)
    # D2H straight into pinned arrays that the returned FeatureImage owns: a
    # pool of output sets on the renderer, recycled once no FeatureImage views
    # them any more (no host-side copy, no page faults on fresh memory)
    if _host_gather_applies(pc, sel):
        # the planes do not need the attributes: they are resolved and go down
        # while the host threads gather the winners' rgb (_host_gather)
        chans = sel.channel_names(pc)
        devo = getattr(r, "_dev_out", None)
        if devo is None or devo["data"].shape[-1] != len(chans):
            devo = r._dev_out = r.alloc_outputs(len(chans))
        # in row bands: the keys of every band go down first; then, band by band, the
        # host threads gather while the previous band's words go up, resolve and come
        # back down (NAR_GATHER_BANDS, default 4)
        data_h = int(devo["data"].shape[0])
        nb = max(1, min(_GATHER_BANDS, H))
        edges = [H * b // nb for b in range(nb + 1)]
        evs = [_keys_to_host(r, main, edges[b] * W, edges[b + 1] * W) for b in range(nb)]
        r.resolve(cloud, cam, sel, out={k: devo[k] for k in _OUT_KEYS[1:]}, stream=main,
                  clear=False)
        res = DeviceFeatureImage(W, H, chans, devo["data"], devo["coverage"], devo["index_plane"],
                                 devo["depth"])
        host = _pinned_outputs(r, res)
        for k in _OUT_KEYS[1:]:
            torch.from_numpy(host[k]).copy_(devo[k], non_blocking=True)
        for b in range(nb):
            y0, y1 = edges[b], (edges[b + 1] if b + 1 < nb else data_h)  # (+ padding rows)
            pix = _host_gather(r, pc, sel, main, evs[b], edges[b] * W, edges[b + 1] * W)
            r.resolve(cloud, cam, sel, out={"data": devo["data"]}, stream=main, pix_rgb=pix,
                      rows=(y0, y1))
            torch.from_numpy(host["data"][y0:y1]).copy_(devo["data"][y0:y1], non_blocking=True)
    else:
        res = r.resolve(cloud, cam, sel, stream=main)
        host = _pinned_outputs(r, res)
        for k in _OUT_KEYS:
            torch.from_numpy(host[k]).copy_(getattr(res, k), non_blocking=True)
    main.synchronize()  # also keeps the uploaded tensors alive until consumed
    names_out = sel.channel_names(pc)
    data = host["data"]
    if data.shape[:2] != (H, W):
        data = np.ascontiguousarray(data[:H, :W])
    else:
        data = data[...]
    return FeatureImage(W, H, names_out, data, host["coverage"][...], host["index_plane"][...],
                        host["depth"][...])


_OUT_KEYS = ("data", "coverage", "index_plane", "depth")
# host-thread gather of the winners' attributes: on by default where there are enough
# host cores to beat the zero-copy PCIe reads (~1.6-2.5 ms on 16 cores vs ~4.7 ms)
_HOST_GATHER = os.environ.get("NAR_HOST_GATHER", "1" if (os.cpu_count() or 1) >= 8 else "0") != "0"
_GATHER_BANDS = int(os.environ.get("NAR_GATHER_BANDS", "4"))


def _host_gather_applies(pc: PointCloud, sel: StreamSelection) -> bool:
    """RGB+D frames of a host cloud with a contiguous u8 rgb stream (NAR_HOST_GATHER)."""
    if not (_HOST_GATHER and sel.rgb and sel.depth and not (sel.vel2d or sel.vel3d)
            and not sel.coverage_channel and not sel.scalars and pc.count > 0):
        return False
    st = pc.stream(sel.rgb_stream)
    return (st.format == "u8" and st.arity >= 3 and st.data.dtype == np.uint8
            and st.data.flags.c_contiguous)


def _hg_buffers(r: "Renderer") -> dict:
    import torch

    npix = r.width * r.height
    hg = getattr(r, "_hg", None)
    if hg is None or hg["keys"].numel() != npix:
        hg = r._hg = {"keys": torch.empty(npix, dtype=torch.int64, pin_memory=True),
                      "pix": torch.empty(npix, dtype=torch.int32, pin_memory=True),
                      "dev": torch.empty(npix, dtype=torch.int32, device=r.device)}
    return hg


def _keys_to_host(r: "Renderer", main, p0: int = 0, p1: int | None = None):
    """Keybuf words [p0, p1) copied down on ``main``; returns the event of that copy."""
    import torch

    hg = _hg_buffers(r)
    p1 = r.width * r.height if p1 is None else p1
    with torch.cuda.stream(main):
        hg["keys"][p0:p1].copy_(r.keybuf[p0:p1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(main)
    return ev


def _host_gather(r: "Renderer", pc: PointCloud, sel: StreamSelection, main, keys_ready,
                 p0: int = 0, p1: int | None = None):
    """The winners' rgb of pixels [p0, p1) of an RGB+D frame of a host cloud, gathered
    by host threads: once the keybuf copy (8 B per pixel) has landed,
    ``nar_host_gather_rgb`` reads each winner's 3 bytes from the caller's array (~1.6 ms
    for 2M pixels on 16 cores) and the packed per-pixel words go back up (4 B per pixel)
    on ``main`` -- instead of ~2M zero-copy PCIe reads by the resolve kernel (~4.7 ms)."""
    import torch

    hg = _hg_buffers(r)
    p1 = r.width * r.height if p1 is None else p1
    st = pc.stream(sel.rgb_stream)
    keys_ready.synchronize()
    _lib.call("nar_host_gather_rgb", hg["keys"].data_ptr() + 8 * p0, p1 - p0, r.domain,
              st.data.ctypes.data, st.arity, C.c_uint64(0), pc.count,
              hg["pix"].data_ptr() + 4 * p0)
    with torch.cuda.stream(main):
        hg["dev"][p0:p1].copy_(hg["pix"][p0:p1], non_blocking=True)
    return hg["dev"]


def _pinned_outputs(r: "Renderer", res) -> dict:
    """A free set of pinned host arrays shaped like ``res`` (a device FeatureImage).

    Each array in a set is the numpy owner of a pinned torch buffer; the arrays
    handed out are views (``.base`` is the owner), so a set is free again when
    the owners' reference counts drop back to the pool's own references.
    """
    import sys

    import torch

    pool = getattr(r, "_host_pool", None)
    if pool is None:
        pool = r._host_pool = []
    shapes = {k: tuple(getattr(res, k).shape) for k in _OUT_KEYS}
    pool[:] = [h for h in pool if all(h[k].shape == shapes[k] for k in _OUT_KEYS)]
    for h in pool:
        # references: the set dict + getrefcount's argument
        if all(sys.getrefcount(h[k]) <= 2 for k in _OUT_KEYS):
            return h
    h = {k: torch.empty(shapes[k], dtype=getattr(res, k).dtype, pin_memory=True).numpy()
         for k in _OUT_KEYS}
    if len(pool) < 4:  # beyond 4 live images, fresh sets are not pooled
        pool.append(h)
    return h
