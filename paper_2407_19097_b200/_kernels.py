"""Kernel-backend surface, mirroring pkg/src/nar/_kernels/__init__.py.

The reference picks an implementation module by name ("native" Cython loop or
"python" numpy twin, ``_resolve`` at :45-53).  This build has exactly one
backend, ``"cuda"``: the sm_100a kernels behind libnar_b200.so; the reference
name ``"native"`` is an alias of it (a drop-in caller asking for the compiled
backend gets this one), ``"python"`` raises ``RuntimeError`` (not built: there
is no CPU fallback) and any other name ``ValueError``, as in the reference; a
missing library raises ``RuntimeError("cuda kernels are not built")``.

``zbuffer_render`` keeps the reference signature (``threads`` is accepted
for compatibility; the GPU render has no thread-count knob and its result is
order independent, like the reference's chunked min-merge).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

EMPTY_KEY = np.uint64(_lib.EMPTY_KEY)
BACKEND = "cuda"


def available_backends() -> list[str]:
    return ["cuda"] if _lib.available() else []


def _resolve(backend: str | None) -> str:
    """Backend names (reference _kernels/__init__.py:45-53): ``"cuda"`` and the
    reference's ``"native"`` (this build *is* the compiled backend a caller
    asks for by that name) select the sm_100a kernels; ``"python"`` -- the
    reference's numpy twin -- raises RuntimeError, as the reference does for a
    backend that is not built (there is no CPU path here); anything else
    raises ValueError."""
    name = backend or BACKEND
    if name == "python":
        raise RuntimeError("python kernels are not part of this build (no CPU fallback); "
                           "use backend='cuda'")
    if name not in ("cuda", "native"):
        raise ValueError(f"unknown kernel backend {name!r}")
    _lib.load()
    return "cuda"


def _as_f64_3x3(R) -> np.ndarray:
    R = np.ascontiguousarray(R, dtype=np.float64)
    if R.shape != (3, 3):
        raise ValueError(f"R must be (3, 3), got {R.shape}")
    return R


def zbuffer_accumulate(keybuf: np.ndarray, positions: np.ndarray, base_index: int, R, campos,
                       f: float, cx: float, cy: float, near: float, far: float, width: int,
                       height: int) -> None:
    """In-place twin of ``_native.zbuffer_accumulate`` (_native.pyx:32-77) on host
    buffers: keybuf (H*W,) u64 writable, positions (n, 3) f32 C-contiguous."""
    if not (isinstance(keybuf, np.ndarray) and keybuf.dtype == np.uint64 and keybuf.flags.c_contiguous
            and keybuf.flags.writeable):
        raise ValueError("keybuf must be a writable C-contiguous uint64 array")
    if keybuf.size != int(width) * int(height):
        raise ValueError("keybuf size does not match width*height")
    if not (isinstance(positions, np.ndarray) and positions.dtype == np.float32
            and positions.ndim == 2 and positions.shape[1] == 3 and positions.flags.c_contiguous):
        raise ValueError("positions must be a C-contiguous (n, 3) float32 array")
    R = _as_f64_3x3(R)
    campos = np.ascontiguousarray(campos, dtype=np.float64).reshape(3)
    _lib.call("nar_zbuffer_accumulate", keybuf.ctypes.data, positions.ctypes.data,
              int(positions.shape[0]), C.c_uint64(int(base_index) & 0xFFFFFFFFFFFFFFFF),
              R.ctypes.data, campos.ctypes.data, float(f), float(cx), float(cy), float(near),
              float(far), int(width), int(height))


def zbuffer_render(positions: np.ndarray, R, campos, f: float, cx: float, cy: float,
                   near: float, far: float, width: int, height: int,
                   threads: int | None = None, backend: str | None = None) -> np.ndarray:
    """Full render pass -> (H*W,) packed min-(depth, index) keys
    (reference: _kernels/__init__.py:56-94)."""
    _resolve(backend)
    pos = np.ascontiguousarray(positions, dtype=np.float32).reshape(-1, 3)
    keybuf = np.full(int(width) * int(height), EMPTY_KEY, np.uint64)
    if len(pos):
        zbuffer_accumulate(keybuf, pos, 0, R, campos, f, cx, cy, near, far, width, height)
    return keybuf
