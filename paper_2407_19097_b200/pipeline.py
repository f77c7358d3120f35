"""Full NAR inference frame: MSR -> channel packing -> U-Net.

``render_neural(pc, cam, checkpoint)`` is the SPEC-level composition the
reference package documents but does not ship: rasterize,
pack the selected channels into the zero-padded CNN input, run the U-Net,
crop, and report ``StageTimings`` with the paper's Table-4 split
(PAPER.md:257-276): ``msr_ms`` = render kernels, ``transfer_proc_ms`` = resolve
(decode + channel fill + padding, written straight into the CNN input), and
``unet_ms`` = head + pyramid + U-Net.  Each stage is timed with CUDA events on
the frame's stream.  ``NeuralRenderer`` keeps the cloud, keybuf, buffers and
packed weights resident for frame-rate use; ``bench`` gives medians over warm
frames.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass

import numpy as np

from .msr import DeviceCloud, Renderer, StreamSelection
from .neural import UNet, UNetConfig


@dataclass
class StageTimings:
    msr_ms: float
    transfer_proc_ms: float
    unet_ms: float

    @property
    def total_ms(self) -> float:
        return self.msr_ms + self.transfer_proc_ms + self.unet_ms


def selection_from_channels(names, velocity_scale: float = 1.0) -> StreamSelection:
    """Invert StreamSelection.channel_names (msr/rasterizer.py:40-60): the built-in
    groups by their channel names, the rest as scalar streams ("temp",
    "mask0", "mask1" -> scalars ("temp", "mask"))."""
    names = tuple(names)
    groups = dict(rgb="r" in names, depth="d" in names, vel2d="v2x" in names,
                  vel3d="v3x" in names, coverage_channel="coverage" in names)
    known = set(StreamSelection(**groups).channel_names())
    scalars = []
    for n in names:
        if n in known:
            continue
        stem = n.rstrip("0123456789")
        base = stem if stem and stem != n else n
        if base not in scalars:
            scalars.append(base)
    return StreamSelection(**groups, scalars=tuple(scalars), velocity_scale=velocity_scale)


def _model(checkpoint):
    from .checkpoint import ModelState, load_checkpoint

    if isinstance(checkpoint, ModelState):
        return checkpoint.config, checkpoint.params
    if isinstance(checkpoint, tuple):
        return checkpoint
    st = load_checkpoint(checkpoint)
    return st.config, st.params


class NeuralRenderer:
    """Resident state for repeated neural frames at one resolution."""

    def __init__(self, width: int, height: int, config: UNetConfig, params: dict,
                 sel: StreamSelection | None = None, device=None):
        import torch

        self.device = torch.device(device or "cuda")
        self.width, self.height = width, height
        self.sel = sel or selection_from_channels(config.channel_names or ("r", "g", "b", "d"))
        self.renderer = Renderer(width, height, device=self.device, pad_multiple=16)
        self.net = UNet(config, params, device=self.device)
        self.config = config
        self._out = None

    def frame(self, cloud: DeviceCloud, cam, stream=None):
        """One frame; returns (device (H_pad, W_pad, 3) f32 image, StageTimings)."""
        import torch

        st = stream or torch.cuda.current_stream(self.device)
        names = self.sel.channel_names(cloud)
        if len(names) != self.config.input_channels:
            raise ValueError(f"selection gives {len(names)} channels, network expects "
                             f"{self.config.input_channels}")
        if self._out is None or self._out["data"].shape[-1] != len(names):
            # the CNN input only: the coverage / index / depth planes are not written
            self._out = self.renderer.alloc_outputs(len(names), planes=False)
            ph, pw = self._out["data"].shape[:2]
            self._rgb = torch.empty((ph, pw, self.config.output_channels), dtype=torch.float32,
                                    device=self.device)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(st)
        self.renderer.render(cloud, cam, stream=st)
        ev[1].record(st)
        self.renderer.resolve(cloud, cam, self.sel, out=self._out, stream=st)
        ev[2].record(st)
        self.net.forward_into(self._out["data"], self._rgb, stream=st)
        ev[3].record(st)
        ev[3].synchronize()
        t = StageTimings(ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                         ev[2].elapsed_time(ev[3]))
        return self._rgb, t


def render_neural(pc, cam, checkpoint, sel: StreamSelection | None = None):
    """(RGB image (H, W, 3) f32 numpy in (0, 1), StageTimings) for one view
    (SPEC.md:562-570).  ``pc``: PointCloud (uploaded) or DeviceCloud;
    ``checkpoint``: NARCK path, ModelState or (UNetConfig, params)."""
    config, params = _model(checkpoint)
    cloud = pc if isinstance(pc, DeviceCloud) else pc.to_device()
    i = cam.intrinsics
    nr = NeuralRenderer(i.width, i.height, config, params, sel=sel, device=cloud.device)
    rgb, t = nr.frame(cloud, cam)
    return rgb[: i.height, : i.width].cpu().numpy(), t


def bench(pc, cam, checkpoint, frames: int = 20, warmup: int = 3,
          sel: StreamSelection | None = None) -> dict:
    """Median StageTimings over `frames` warm frames."""
    config, params = _model(checkpoint)
    cloud = pc if isinstance(pc, DeviceCloud) else pc.to_device()
    i = cam.intrinsics
    nr = NeuralRenderer(i.width, i.height, config, params, sel=sel, device=cloud.device)
    for _ in range(warmup):
        nr.frame(cloud, cam)
    ts = [nr.frame(cloud, cam)[1] for _ in range(frames)]
    med = {k: statistics.median(getattr(t, k) for t in ts)
           for k in ("msr_ms", "transfer_proc_ms", "unet_ms")}
    med["total_ms"] = statistics.median(t.total_ms for t in ts)
    med["fps"] = 1e3 / med["total_ms"]
    med["frames"] = frames
    return med
