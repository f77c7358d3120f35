"""Gated U-Net post-processing network on B200 tcgen05 tensor cores.

Reference API kept (pkg/src/nar/neural/model.py): ``UNetConfig``,
``init_params``, ``pad_to_multiple``, ``build_pyramid``-compatible shapes and
``forward(features, params, config)``.  The forward pass runs entirely in
libnar_b200.so (``nar_unet_*``): bf16 activations and weights, f32
accumulation in TMEM, one implicit-GEMM kernel per gated conv with the
elu(f)*sigmoid(g) epilogue fused, concat / 2x2 average-pool / nearest
upsample fused into the operand loads.  Parity contract vs the f32 reference:
PSNR >= 50 dB and max |err| <= 2e-2 (tests/test_unet_gpu.py).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError

PYRAMID_LEVELS = 5


@dataclass(frozen=True)
class UNetConfig:
    """Network shape (model.py:26-62); widths min(base * mult^k, max)."""

    input_channels: int
    channel_names: tuple[str, ...] = ()
    levels: int = PYRAMID_LEVELS
    base_channels: int = 16
    channel_multiplier: int = 2
    max_channels: int = 128
    output_channels: int = 3
    use_descriptor_head: bool = True
    init_seed: int = 0

    def width(self, level: int) -> int:
        return min(self.base_channels * self.channel_multiplier ** level, self.max_channels)

    def to_dict(self) -> dict:
        return {"input_channels": self.input_channels, "channel_names": list(self.channel_names),
                "levels": self.levels, "base_channels": self.base_channels,
                "channel_multiplier": self.channel_multiplier, "max_channels": self.max_channels,
                "output_channels": self.output_channels,
                "use_descriptor_head": self.use_descriptor_head, "init_seed": self.init_seed}

    @staticmethod
    def from_dict(d: dict) -> "UNetConfig":
        d = dict(d)
        d["channel_names"] = tuple(d.get("channel_names", ()))
        return UNetConfig(**d)

    def hash(self) -> str:
        return hashlib.sha256(json.dumps(self.to_dict(), sort_keys=True).encode()).hexdigest()


def layer_names(cfg: UNetConfig) -> list[str]:
    enc = [f"enc{k}{s}" for k in range(cfg.levels) for s in "ab"]
    dec = [f"dec{k}{s}" for k in range(cfg.levels - 2, -1, -1) for s in "ab"]
    return enc + dec


def layer_shapes(cfg: UNetConfig) -> dict[str, tuple[int, int]]:
    """(c_in, c_out) of every gated conv (model.py:89-97)."""
    cin, w = cfg.input_channels, cfg.width
    out = {}
    for k in range(cfg.levels):
        out[f"enc{k}a"] = (cin if k == 0 else w(k - 1) + cin, w(k))
        out[f"enc{k}b"] = (w(k), w(k))
    for k in range(cfg.levels - 2, -1, -1):
        out[f"dec{k}a"] = (w(k + 1) + w(k), w(k))
        out[f"dec{k}b"] = (w(k), w(k))
    return out


def init_params(config: UNetConfig) -> dict[str, np.ndarray]:
    """Seeded parameters with the reference's draw order (model.py:70-100):
    Kaiming-uniform conv weights (bound sqrt(6/fan_in), HWIO), zero f biases,
    +1 gate biases, identity descriptor head."""
    rng = np.random.default_rng(config.init_seed)
    params: dict[str, np.ndarray] = {}
    c = config.input_channels
    if config.use_descriptor_head:
        params["head.w"] = np.eye(c, dtype=np.float32)
        params["head.b"] = np.zeros(c, np.float32)
    shapes = layer_shapes(config)
    for name in layer_names(config):
        ci, co = shapes[name]
        bound = np.sqrt(6.0 / (9 * ci))
        params[f"{name}.f_w"] = rng.uniform(-bound, bound, (3, 3, ci, co)).astype(np.float32)
        params[f"{name}.f_b"] = np.zeros(co, np.float32)
        params[f"{name}.g_w"] = rng.uniform(-bound, bound, (3, 3, ci, co)).astype(np.float32)
        params[f"{name}.g_b"] = np.ones(co, np.float32)
    w0 = config.width(0)
    bound = np.sqrt(6.0 / w0)
    params["out.w"] = rng.uniform(-bound, bound, (w0, config.output_channels)).astype(np.float32)
    params["out.b"] = np.zeros(config.output_channels, np.float32)
    return params


def pad_to_multiple(img: np.ndarray, multiple: int = 16):
    """Zero-pad (H, W, C) bottom/right to multiples (model.py:207-215);
    returns (padded, (H, W))."""
    h, w = img.shape[:2]
    ph, pw = (-h) % multiple, (-w) % multiple
    if ph or pw:
        img = np.pad(img, ((0, ph), (0, pw)) + ((0, 0),) * (img.ndim - 2))
    return img, (h, w)


# ---------------------------------------------------------------------------
# device network (libnar_b200.so nar_unet_*)
# ---------------------------------------------------------------------------
# ---- standalone ops on the GPU (model.py:135-163) ------------------------------------

def _dev_f32(x):
    """(tensor on cuda f32 contiguous, was_torch)."""
    import torch

    data = getattr(x, "data", x) if not hasattr(x, "device") else x
    if isinstance(data, torch.Tensor):
        return data.to("cuda", torch.float32).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(data, np.float32)).cuda(), False


def _images(t):
    """Iterate the (H, W, C) images of a (.., H, W, C) tensor."""
    return t.reshape((-1,) + tuple(t.shape[-3:]))


def conv1x1_head(x, w, b):
    """Per-pixel affine y = x @ w + b (model.py:135-143) with the fused head kernel.
    ``x`` (..., H, W, C), ``w`` (C, C), ``b`` (C,).  H, W any."""
    return build_pyramid(x, levels=1, head=(w, b))[0]


def build_pyramid(t, levels: int = 5, head=None):
    """Levels 0..levels-1 of 2x2 averages (model.py:146-155) in f32 on the GPU
    (optionally after the descriptor head ``head=(w, b)``).  Returns a list of
    arrays / tensors like the input kind."""
    import torch

    x, was_torch = _dev_f32(t)
    ch = int(x.shape[-1])
    H, W = int(x.shape[-3]), int(x.shape[-2])
    div = 2 ** (levels - 1)
    if H % div or W % div:
        raise ValueError(f"spatial dims {H}x{W} not divisible by {div}")
    if head is not None:
        hw, _ = _dev_f32(head[0])
        hb, _ = _dev_f32(head[1])
        if tuple(hw.shape) != (ch, ch) or tuple(hb.shape) != (ch,):
            raise ConfigurationError(f"head weights must be ({ch},{ch}) and ({ch},)")
    lead = tuple(x.shape[:-3])
    imgs = _images(x)
    outs = [torch.empty((imgs.shape[0], H >> k, W >> k, ch), dtype=torch.float32, device=x.device)
            for k in range(levels)]
    st = torch.cuda.current_stream(x.device)
    for i in range(imgs.shape[0]):
        arr = (C.c_void_p * levels)(*[o[i].data_ptr() for o in outs])
        _lib.call("nar_head_pyramid", imgs[i].data_ptr(), H, W, ch,
                  hw.data_ptr() if head is not None else None,
                  hb.data_ptr() if head is not None else None, int(head is not None), levels,
                  arr, int(st.cuda_stream))
    res = [o.reshape(lead + tuple(o.shape[1:])) for o in outs]
    if was_torch:
        return res
    st.synchronize()
    return [r.cpu().numpy() for r in res]


def gated_conv(x, f_w, f_b, g_w, g_b):
    """elu(conv3x3(x, f_w) + f_b) * sigmoid(conv3x3(x, g_w) + g_b), same padding
    (model.py:158-163), on the tensor cores (bf16 operands, f32 accumulation)."""
    import torch

    xd, was_torch = _dev_f32(x)
    fw = np.ascontiguousarray(getattr(f_w, "data", f_w), np.float32)
    gw = np.ascontiguousarray(getattr(g_w, "data", g_w), np.float32)
    fb = np.ascontiguousarray(getattr(f_b, "data", f_b), np.float32)
    gb = np.ascontiguousarray(getattr(g_b, "data", g_b), np.float32)
    cin = int(xd.shape[-1])
    if fw.shape[:3] != (3, 3, cin) or gw.shape != fw.shape:
        raise ConfigurationError(f"gated conv kernels must be (3,3,{cin},Cout)")
    cout = int(fw.shape[3])
    if fb.shape != (cout,) or gb.shape != (cout,):
        raise ConfigurationError("gated conv biases must be (Cout,)")
    lead = tuple(xd.shape[:-3])
    H, W = int(xd.shape[-3]), int(xd.shape[-2])
    imgs = _images(xd)
    out = torch.empty((imgs.shape[0], H, W, cout), dtype=torch.float32, device=xd.device)
    st = torch.cuda.current_stream(xd.device)
    for i in range(imgs.shape[0]):
        _lib.call("nar_gated_conv", imgs[i].data_ptr(), H, W, cin, fw.ctypes.data, fb.ctypes.data,
                  gw.ctypes.data, gb.ctypes.data, cout, out[i].data_ptr(), int(st.cuda_stream))
    out = out.reshape(lead + (H, W, cout))
    return out if was_torch else out.cpu().numpy()


def _config_struct(cfg: UNetConfig) -> "_lib.UNetConfigC":
    c = _lib.UNetConfigC()
    c.input_channels, c.levels = cfg.input_channels, cfg.levels
    c.base_channels, c.channel_multiplier = cfg.base_channels, cfg.channel_multiplier
    c.max_channels, c.output_channels = cfg.max_channels, cfg.output_channels
    c.use_descriptor_head = int(cfg.use_descriptor_head)
    return c


class UNet:
    """Packed bf16 weights on the device plus a reusable workspace.

    ``params`` is the reference parameter dict (HWIO f32 numpy arrays, names as
    in model.py:70-100); they are validated and packed once at construction.
    """

    def __init__(self, config: UNetConfig, params: dict, device=None):
        import torch

        self.config = config
        self.device = torch.device(device or "cuda")
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.nar_unet_create(C.byref(_config_struct(config)), C.byref(h)))
        self._h = h
        expected = set(["out.w", "out.b"])
        if config.use_descriptor_head:
            expected |= {"head.w", "head.b"}
        for n in layer_names(config):
            expected |= {f"{n}.f_w", f"{n}.f_b", f"{n}.g_w", f"{n}.g_b"}
        missing = expected - set(params)
        if missing:
            raise ConfigurationError(f"missing parameters: {sorted(missing)[:4]}")
        with torch.cuda.device(self.device):
            for name in sorted(expected):
                a = _host_param(params[name])
                _lib.check(lib.nar_unet_set_param(self._h, name.encode(), a.ctypes.data, a.size))
        self._ws = {}
        self._graphs: dict = {}  # (x, out, H, W) -> CUDA graph of one forward (or False)
        self._seen: set = set()

    def _workspace(self, H: int, W: int):
        import torch

        key = (H, W)
        if key not in self._ws:
            n = C.c_size_t(0)
            _lib.check(_lib.load().nar_unet_workspace_bytes(self._h, H, W, C.byref(n)))
            self._ws[key] = torch.empty(int(n.value), dtype=torch.uint8, device=self.device)
        return self._ws[key]

    def forward_into(self, x, out, stream=None) -> None:
        """x: device f32 (H, W, Cin) (or (1,H,W,Cin)); out: device f32 (H, W, out)."""
        H, W = int(x.shape[-3]), int(x.shape[-2])
        if int(x.shape[-1]) != self.config.input_channels:
            raise ConfigurationError(
                f"model expects {self.config.input_channels} channels, "
                f"features have {int(x.shape[-1])}")
        if not (x.is_contiguous() and out.is_contiguous()):
            raise ValueError("forward_into needs contiguous tensors")
        import torch

        n_out = self.config.output_channels
        if x.dtype != torch.float32 or out.dtype != torch.float32:
            raise ValueError("forward_into needs float32 tensors")
        if x.device != self.device or out.device != self.device:
            raise ValueError(f"forward_into needs tensors on {self.device}")
        if tuple(out.shape[-3:]) != (H, W, n_out) or out.numel() != H * W * n_out:
            raise ValueError(f"out must be ({H}, {W}, {n_out}), got {tuple(out.shape)}")
        if x.numel() != H * W * int(x.shape[-1]):
            raise ValueError("forward_into takes one image (H, W, C) or (1, H, W, C)")
        ws = self._workspace(H, W)
        # graphs need a torch stream (None: the current one); raw handles stay eager
        # (and not while the caller captures a graph of its own: the launches join it)
        graphs = (_UNET_GRAPHS and (stream is None or isinstance(stream, torch.cuda.Stream))
                  and not torch.cuda.is_current_stream_capturing())
        key = (x.data_ptr(), out.data_ptr(), H, W)
        g = self._graphs.get(key) if graphs else None
        if g is None and graphs and key in self._seen:
            # second call on the same buffers: capture the 20 launches once and
            # replay them from now on (no per-launch host cost; the programmatic
            # dependent edges between the convs are kept in the graph)
            g = self._capture(x, out, ws, H, W, stream)
        if g is not None and g is not False:
            with torch.cuda.stream(stream or torch.cuda.current_stream(self.device)):
                g.replay()  # on the caller's stream, like the eager launches
            return
        if graphs:
            self._seen.add(key)
        self._launch(x, out, ws, H, W, stream)

    def _launch(self, x, out, ws, H: int, W: int, stream) -> None:
        with _lib.on_device(self.device.index):  # weights upload + launches on self.device
            _lib.check(_lib.load().nar_unet_forward(
                self._h, x.data_ptr(), H, W, out.data_ptr(), ws.data_ptr(), ws.numel(),
                _lib.stream_handle(stream, self.device.index)))

    def _capture(self, x, out, ws, H: int, W: int, stream):
        """A CUDA graph of one forward on these exact buffers (the weights and the
        workspace are the network's own and never move), or False (not retried)."""
        import torch

        key = (x.data_ptr(), out.data_ptr(), H, W)
        if len(self._graphs) >= 8:
            self._graphs.pop(next(iter(self._graphs)))
        caller = stream or torch.cuda.current_stream(self.device)
        try:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.device)
            side.wait_stream(caller)
            with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                self._launch(x, out, ws, H, W, None)
            caller.wait_stream(side)
        except Exception:  # capture not possible here: stay eager for this key
            g = False
        self._graphs[key] = g
        return g

    def __call__(self, x):
        import torch

        x = x.to(self.device, torch.float32).contiguous()
        squeeze = x.dim() == 3
        if squeeze:
            x = x[None]
        outs = []
        for img in x:
            o = torch.empty(img.shape[:2] + (self.config.output_channels,), dtype=torch.float32,
                            device=self.device)
            self.forward_into(img, o)
            outs.append(o)
        y = torch.stack(outs)
        return y[0] if squeeze else y

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.nar_unet_destroy(self._h)
        except Exception:
            pass


_nets: dict = {}
# UNet.forward_into replays a CUDA graph of the forward on buffers it has seen
# before (NAR_UNET_GRAPH=0: plain launches every call)
_UNET_GRAPHS = os.environ.get("NAR_UNET_GRAPH", "1") != "0"


def _host_param(v) -> np.ndarray:
    """A parameter value as a host f32 array: numpy arrays, reference autodiff
    Tensors (``.data``) and torch tensors (any device) alike."""
    if hasattr(v, "detach"):
        v = v.detach().cpu().numpy()
    elif hasattr(v, "data") and not isinstance(v, np.ndarray):
        v = v.data
    return np.ascontiguousarray(v, dtype=np.float32)


def _params_digest(params: dict) -> tuple:
    """Content key of a parameter dict: (name, shape, crc32 of the bytes) per
    entry.  crc32 runs over the buffers in place at several GB/s (~2 ms for the
    default 10 MB network), so a dict updated in place still repacks."""
    import zlib

    key = []
    for name in sorted(params):
        a = _host_param(params[name])
        key.append((name, a.shape, zlib.crc32(memoryview(a).cast("B"))))
    return tuple(key)


def forward(features, params: dict, config: UNetConfig):
    """Full inference path (model.py:194-204): descriptor head, pyramid, U-Net.

    ``features``: (N, H, W, C) f32 -- a torch tensor (returns a tensor on the
    network's device), a reference autodiff ``Tensor`` (returns the same type
    wrapping the numpy result, so ``.data`` is an ndarray as in model.py:194),
    or a numpy array (returns numpy).  H and W must be multiples of
    2^(levels-1); use ``pad_to_multiple`` first, as the reference does.
    """
    import torch

    data = getattr(features, "data", features) if not hasattr(features, "device") else features
    shape = tuple(data.shape)
    if shape[-1] != config.input_channels:
        raise ConfigurationError(f"model expects {config.input_channels} channels, "
                                 f"features have {shape[-1]}")
    div = 2 ** (config.levels - 1)
    if shape[-3] % div or shape[-2] % div:
        raise ValueError(f"spatial dims {shape[-3]}x{shape[-2]} not divisible by {div}")
    # packed weights are cached per (config, parameter contents): a dict updated in
    # place (new arrays or mutated ones) repacks, as the reference reads params
    # on every call
    key = (config, _params_digest(params))
    net = _nets.get(key)
    if net is None:
        if len(_nets) > 4:
            _nets.clear()
        net = _nets[key] = UNet(config, params)
    if isinstance(data, torch.Tensor):
        return net(data)
    x = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32))
    y = net(x.to(net.device)).cpu().numpy()
    if data is not features:  # a reference Tensor in -> the same Tensor type out
        return type(features)(y)
    return y
