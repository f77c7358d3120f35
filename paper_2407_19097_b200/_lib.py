"""ctypes binding of ``libnar_b200.so`` (declared in include/nar_b200.h).

This is the Python side of the drop-in boundary: plain pointers and sizes
cross the ABI, statuses come back as ints and are raised here as the
reference's exception types.  There is no fallback: if the library cannot be
loaded, every entry point raises ``RuntimeError("cuda kernels are not
built")`` -- the wording of the reference's missing-native-backend error
(pkg/src/nar/_kernels/__init__.py:48-50).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigurationError

LIB_PATH = Path(__file__).resolve().parent / "libnar_b200.so"

NAR_OK, NAR_ERR_INVALID, NAR_ERR_CUDA, NAR_ERR_CONFIG, NAR_ERR_NOMEM = 0, 1, 2, 3, 4
EMPTY_KEY = 0xFFFFFFFFFFFFFFFF
SIGN_FLIP = 0x8000000000000000
KEYS_UNSIGNED, KEYS_SIGNED = 0, 1
MAX_SEGMENTS = 8
MAX_SCALARS = 8
MAX_CHANNELS = 16
FMT_U8, FMT_F32 = 0, 1


class Camera(C.Structure):
    _fields_ = [
        ("R", C.c_double * 9),
        ("campos", C.c_double * 3),
        ("f", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("near_", C.c_double),
        ("far_", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class Segment(C.Structure):
    _fields_ = [
        ("begin", C.c_int64),
        ("count", C.c_int64),
        ("positions", C.c_void_p),
        ("rgb", C.c_void_p),
        ("velocity", C.c_void_p),
        ("scalars", C.c_void_p * MAX_SCALARS),
    ]


class Selection(C.Structure):
    _fields_ = [
        ("rgb", C.c_int32),
        ("depth", C.c_int32),
        ("vel2d", C.c_int32),
        ("vel3d", C.c_int32),
        ("coverage_channel", C.c_int32),
        ("rgb_format", C.c_int32),
        ("rgb_arity", C.c_int32),
        ("vel_format", C.c_int32),
        ("vel_arity", C.c_int32),
        ("n_scalars", C.c_int32),
        ("scalar_format", C.c_int32 * MAX_SCALARS),
        ("scalar_arity", C.c_int32 * MAX_SCALARS),
        ("velocity_scale", C.c_double),
    ]


class ResolveOut(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("data_h", C.c_int32),
        ("data_w", C.c_int32),
        ("coverage", C.c_void_p),
        ("index_plane", C.c_void_p),
        ("depth", C.c_void_p),
        ("owner_only", C.c_int32),
        ("clear_keybuf", C.c_int32),
    ]


class UNetConfigC(C.Structure):
    _fields_ = [
        ("input_channels", C.c_int32),
        ("levels", C.c_int32),
        ("base_channels", C.c_int32),
        ("channel_multiplier", C.c_int32),
        ("max_channels", C.c_int32),
        ("output_channels", C.c_int32),
        ("use_descriptor_head", C.c_int32),
    ]


_vp, _i32, _i64, _u64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); this table is the ABI surface (tests check that
# every function declared in include/nar_b200.h appears here and is exported)
SIGNATURES = {
    "nar_version": (C.c_char_p, []),
    "nar_last_error": (C.c_char_p, []),
    "nar_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "nar_host_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "nar_host_free": (C.c_int, [_vp]),
    "nar_launch_count": (C.c_uint64, []),
    "nar_splat_blend": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "nar_host_mapped_pointer": (C.c_int, [_vp, C.POINTER(C.c_void_p)]),
    "nar_host_register": (C.c_int, [_vp, C.c_size_t]),
    "nar_host_unregister": (C.c_int, [_vp]),
    "nar_zbuffer_accumulate": (
        C.c_int,
        [_vp, _vp, _i64, _u64, _vp, _vp, _d, _d, _d, _d, _d, _i32, _i32],
    ),
    "nar_keybuf_fill": (C.c_int, [_vp, _i64, _u64, _vp]),
    "nar_render": (C.c_int, [_vp, _vp, _i64, _u64, C.POINTER(Camera), _i32, _vp]),
    "nar_render_host": (C.c_int, [_vp, _vp, _i64, _u64, C.POINTER(Camera), _i32, _vp]),
    "nar_hiz_scratch_bytes": (C.c_int, [_i32, _i32, C.POINTER(C.c_size_t)]),
    "nar_render_hiz": (C.c_int, [_vp, _vp, _vp, _i64, _u64, C.POINTER(Camera), _i32, _i32, _vp]),
    "nar_morton_keys": (C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "nar_resolve": (
        C.c_int,
        [_vp, C.POINTER(Camera), _i32, C.POINTER(Selection), C.POINTER(Segment), _i32,
         C.POINTER(ResolveOut), _vp],
    ),
    "nar_resolve_peers": (
        C.c_int,
        [C.POINTER(C.c_void_p), _i32, _i32, _i32, C.POINTER(Camera), _i32, C.POINTER(Selection),
         C.POINTER(Segment), _i32, C.POINTER(ResolveOut), _vp],
    ),
    "nar_host_gather_rgb": (C.c_int, [_vp, _i64, _i32, _vp, _i32, _u64, _i64, _vp]),
    "nar_resolve_pixrgb": (
        C.c_int,
        [_vp, _i32, _i32, C.POINTER(Camera), _i32, C.POINTER(Selection), C.POINTER(Segment), _i32,
         C.POINTER(ResolveOut), _vp, _vp],
    ),
    "nar_unet_create": (C.c_int, [C.POINTER(UNetConfigC), C.POINTER(C.c_void_p)]),
    "nar_head_pyramid": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _i32, _i32,
                                   C.POINTER(C.c_void_p), _vp]),
    "nar_gated_conv": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "nar_unet_destroy": (C.c_int, [_vp]),
    "nar_unet_set_param": (C.c_int, [_vp, C.c_char_p, _vp, _i64]),
    "nar_unet_workspace_bytes": (C.c_int, [_vp, _i32, _i32, C.POINTER(C.c_size_t)]),
    "nar_unet_forward": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, C.c_size_t, _vp]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None
_load_error: str | None = None


def load() -> C.CDLL:
    """Load (once) and return the library; raise RuntimeError if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("NAR_B200_LIB", str(LIB_PATH))
        try:
            lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
        except OSError as e:  # not built / wrong platform
            _load_error = str(e)
            raise RuntimeError(f"cuda kernels are not built ({e})") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def available() -> bool:
    try:
        load()
        return True
    except RuntimeError:
        return False


def check(rc: int) -> None:
    if rc == NAR_OK:
        return
    msg = (load().nar_last_error() or b"").decode(errors="replace")
    if rc == NAR_ERR_INVALID:
        raise ValueError(msg)
    if rc == NAR_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == NAR_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def device_count() -> int:
    n = C.c_int32(0)
    call("nar_device_count", C.byref(n))
    return int(n.value)


def make_camera(R, campos, f, cx, cy, near, far, width, height) -> Camera:
    cam = Camera()
    flat = [float(v) for row in R for v in row] if hasattr(R, "__len__") and hasattr(R[0], "__len__") else [float(v) for v in R]
    if len(flat) != 9:
        raise ValueError("R must be 3x3")
    cam.R[:] = flat
    cp = [float(v) for v in campos]
    if len(cp) != 3:
        raise ValueError("campos must have 3 entries")
    cam.campos[:] = cp
    cam.f, cam.cx, cam.cy = float(f), float(cx), float(cy)
    cam.near_, cam.far_ = float(near), float(far)
    cam.width, cam.height = int(width), int(height)
    return cam


def stream_handle(stream, device_index: int | None = None) -> int:
    """cudaStream_t of a torch.cuda.Stream (or None -> torch's current stream of
    ``device_index``, default the current device)."""
    import torch

    if stream is None:  # the raw handle, without building a Stream object
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        idx = torch.cuda.current_device() if device_index is None else device_index
        if raw is not None:
            return int(raw(idx))
        stream = torch.cuda.current_stream(idx)
    return int(stream.cuda_stream)


class on_device:
    """Makes CUDA device ``index`` current for the enclosed library calls (the
    library keys its per-device state and launches on the current device);
    a no-op when it already is."""

    __slots__ = ("index", "prev")

    def __init__(self, index: int | None):
        self.index = index

    def __enter__(self):
        import torch

        self.prev = torch.cuda.current_device()
        if self.index is not None and self.index != self.prev:
            torch.cuda.set_device(self.index)
        return self

    def __exit__(self, *exc):
        import torch

        if self.index is not None and self.index != self.prev:
            torch.cuda.set_device(self.prev)
        return False


# ---- in-place page locking of caller arrays (msr.rasterize's pageable path) ----
REGISTER_MIN_BYTES = 64 << 20
_registered: dict = {}  # data pointer -> (nbytes, weakref.finalize)
_reg_lock = threading.Lock()


def _unregister(ptr: int) -> None:
    with _reg_lock:
        if _registered.pop(ptr, None) is not None and _lib is not None:
            _lib.nar_host_unregister(C.c_void_p(ptr))


def ensure_registered(arr) -> bool:
    """Page-lock a large pageable numpy array in place (cudaHostRegister, mapped)
    so it behaves like pinned memory: async DMA and zero-copy kernel reads.  The
    registration lives as long as the array object (a weakref finalizer undoes
    it before numpy frees the buffer).  Returns False (array left pageable) for
    small arrays, when NAR_HOST_REGISTER=0, or when the driver refuses."""
    import weakref

    if arr.nbytes < REGISTER_MIN_BYTES or os.environ.get("NAR_HOST_REGISTER", "1") == "0":
        return False
    ptr = int(arr.ctypes.data)
    with _reg_lock:
        if ptr in _registered:
            return _registered[ptr][0] >= arr.nbytes
        if load().nar_host_register(C.c_void_p(ptr), arr.nbytes) != NAR_OK:
            return False
        try:
            fin = weakref.finalize(arr, _unregister, ptr)
        except TypeError:  # no weakref support: undo, stay pageable
            _lib.nar_host_unregister(C.c_void_p(ptr))
            return False
        fin.atexit = False
        _registered[ptr] = (arr.nbytes, fin)
    return True


def mapped_pointer(host_ptr: int):
    """Device address of mapped pinned host memory, or None (pageable memory)."""
    out = C.c_void_p()
    if load().nar_host_mapped_pointer(C.c_void_p(host_ptr), C.byref(out)) != 0:
        return None
    return out.value


def launch_count() -> int:
    """Kernels launched by libnar_b200 so far (bench.py's gpu_launches)."""
    return int(load().nar_launch_count())

