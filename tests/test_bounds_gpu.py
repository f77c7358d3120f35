"""Out-of-bounds checks without compute-sanitizer (closed on this GPU pool):
every buffer a kernel writes is a view inside a larger allocation whose guard
bands hold a canary pattern, inputs sit at the very end of their allocations,
and after render / resolve / fused composite / U-Net / standalone conv calls
the canaries must be untouched and the results equal to the oracle.  The
zero-copy rgb gather is checked at both ends of a mapped pinned allocation
whose stream starts one byte into a page and ends at the allocation's last
byte (an over-read there would leave the allocation).  The reference itself
has no bounds checks at all (_native.pyx:1, boundscheck=False)."""

import ctypes as C

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements of canary on each side
CANARY = {1: 0xA5, 4: 0x5A5AA5A5, 8: 0x5A5AA5A5A5A55A5A}


def _guarded(shape, dtype, dev):
    """(view, checker): a contiguous view of `shape` inside a canary-filled buffer."""
    import torch

    n = int(np.prod(shape))
    esize = torch.empty(0, dtype=dtype).element_size()
    raw_t = {1: torch.uint8, 4: torch.int32, 8: torch.int64}[esize]
    buf = torch.empty(n + 2 * GUARD, dtype=raw_t, device=dev)
    can = CANARY[esize]
    if esize > 1 and can >= 1 << (8 * esize - 1):
        can -= 1 << (8 * esize)
    buf.fill_(can)
    view = buf[GUARD:GUARD + n].view(dtype).view(shape)

    def intact():
        return bool((buf[:GUARD] == can).all()) and bool((buf[GUARD + n:] == can).all())

    return view, intact


def test_render_resolve_guard_bands(cuda):
    import torch

    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    rng = np.random.default_rng(7)
    n = 2_000_003
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    rgb = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    vel = rng.normal(size=(n, 3)).astype(np.float32)
    cam = look_at((0.3, -2.1, 0.8), (0, 0, 0), Intrinsics(width=333, height=211))
    pc = PointCloud(pos, [Stream("rgb", "u8", rgb), Stream("velocity", "f32", vel)])
    for sel in (StreamSelection(rgb=True, depth=True),
                StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True,
                                coverage_channel=True)):
        ref = oracle.rasterize(pc, cam, sel, threads=8)
        # inputs at the end of their allocations (no slack after the last point)
        dpos = torch.from_numpy(pos).to(cuda)
        dc = DeviceCloud.from_tensors(dpos, {"rgb": torch.from_numpy(rgb).to(cuda),
                                             "velocity": torch.from_numpy(vel).to(cuda)})
        r = Renderer(333, 211, device=cuda, pad_multiple=16)
        kb, kb_ok = _guarded((333 * 211,), torch.int64, cuda)
        kb.copy_(r.keybuf)
        r.keybuf = kb
        C_ = len(sel.channel_names(pc))
        outs, checks = {}, []
        for k, shape, dt in (("data", (224, 336, C_), torch.float32),
                             ("coverage", (211, 333), torch.uint8),
                             ("index_plane", (211, 333), torch.int64),
                             ("depth", (211, 333), torch.float32)):
            outs[k], ok = _guarded(shape, dt, cuda)
            checks.append(ok)
        for _ in range(2):
            r.render(dc, cam)
            img = r.resolve(dc, cam, sel, out=outs)
        torch.cuda.synchronize()
        assert kb_ok() and all(ok() for ok in checks), "a guard band was overwritten"
        h = img.to_host()
        assert np.array_equal(h.index_plane, ref["index_plane"])
        assert np.array_equal(h.data[..., :4], ref["data"][..., :4])
        assert bool((outs["data"][211:] == 0).all()) and bool((outs["data"][:, 333:] == 0).all())


def test_unet_and_conv_guard_bands(cuda):
    import torch

    from paper_2407_19097_b200.neural import UNet, UNetConfig, init_params

    for base in (16, 20):
        cfg = UNetConfig(input_channels=4, base_channels=base)
        params = init_params(cfg)
        net = UNet(cfg, params, device=cuda)
        x, x_ok = _guarded((96, 160, 4), torch.float32, cuda)
        x.copy_(torch.rand((96, 160, 4), device=cuda))
        y, y_ok = _guarded((96, 160, 3), torch.float32, cuda)
        net.forward_into(x, y)
        torch.cuda.synchronize()
        assert x_ok() and y_ok()
        ref = oracle.forward(x.cpu().numpy()[None], params, cfg)[0]
        assert oracle.psnr(y.cpu().numpy(), ref) >= 50.0


def test_zero_copy_gather_at_allocation_edges(cuda):
    """rgb in mapped pinned memory: the stream starts 1 byte into its page and
    its last byte is the allocation's last byte; the first and last points win
    pixels, so the resolve gathers exactly those edge bytes."""
    from paper_2407_19097_b200 import _lib
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at
    from paper_2407_19097_b200.msr import StreamSelection, rasterize

    n = 4095  # 3 * 4095 + 1 = 12286 bytes -> allocation of exactly 3 pages
    size = 3 * n + 1
    pages = (size + 4095) // 4096 * 4096
    ptr = C.c_void_p()
    _lib.call("nar_host_alloc", C.byref(ptr), pages)
    try:
        raw = np.ctypeslib.as_array((C.c_uint8 * pages).from_address(ptr.value))
        off = pages - 3 * n  # the stream ends at the allocation's last byte
        rgb = raw[off:off + 3 * n].reshape(n, 3)
        rng = np.random.default_rng(3)
        rgb[:] = rng.integers(0, 256, (n, 3), dtype=np.uint8)
        pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        cam = look_at((0.0, -2.2, 1.0), (0, 0, 0), Intrinsics(width=64, height=48))
        # first and last point straight in front of the camera, nearest of all
        d = np.asarray(cam.orientation)[2]
        eye = np.asarray(cam.position)
        pos[0] = (eye + 0.5 * d).astype(np.float32)
        pos[-1] = (eye + 0.6 * d + 0.05 * np.asarray(cam.orientation)[0]).astype(np.float32)
        pc = PointCloud(pos, [Stream("rgb", "u8", rgb)])  # rgb stays in mapped memory
        assert pc.stream("rgb").data.ctypes.data == ptr.value + off
        sel = StreamSelection(rgb=True, depth=True)
        fi = rasterize(pc, cam, sel)
        ref = oracle.rasterize(pc, cam, sel)
        assert {0, n - 1} <= set(np.unique(fi.index_plane).tolist())
        assert np.array_equal(fi.index_plane, ref["index_plane"])
        assert np.array_equal(fi.data, ref["data"])
        # unaligned stream start: the same with the stream beginning 1 byte into the page
        rgb2 = raw[1:1 + 3 * n].reshape(n, 3)
        rgb2[:] = rgb.copy()
        pc2 = PointCloud(pos, [Stream("rgb", "u8", rgb2)])
        fi2 = rasterize(pc2, cam, sel)
        ref2 = oracle.rasterize(pc2, cam, sel)
        assert np.array_equal(fi2.data, ref2["data"])
    finally:
        _lib.call("nar_host_free", ptr)
