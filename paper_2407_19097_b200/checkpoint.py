"""NARCK checkpoints -> device U-Net weights (pkg/src/nar/neural/checkpoint.py).

Container (little-endian): magic "NARCK", u16 version, u8 precision (0 f32,
1 f16 weights), u64 step, SHA-256 of the tensor section, then tensors as
(u8 name_len, name, u8 ndim, u32 dims..., payload); the model config rides
along as the JSON-bytes tensor "__config__".  Loading verifies magic, version
and hash (CheckpointError otherwise) and, if given, config compatibility --
the reference's behaviour (checkpoint.py:85-148).  f16 ("quantized", App. C)
weights are widened to f32 on the host and packed to bf16 for the tensor
cores by ``neural.UNet``.
"""

from __future__ import annotations

import hashlib
import io
import json
import struct
import warnings
from dataclasses import dataclass, field

import numpy as np

from .errors import CheckpointError
from .neural import UNetConfig

MAGIC = b"NARCK"
VERSION = 1
F16_MAX = 65504.0
_CONFIG_KEY = "__config__"


@dataclass
class ModelState:
    """Parameters (+ optimizer moments for resume) and step (model.py:103-132)."""

    config: UNetConfig
    params: dict
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    step: int = 0

    @staticmethod
    def initialize(config: UNetConfig) -> "ModelState":
        from .neural import init_params

        params = init_params(config)
        return ModelState(config, params, {k: np.zeros_like(p) for k, p in params.items()},
                          {k: np.zeros_like(p) for k, p in params.items()})


def _put(buf: io.BytesIO, name: str, arr: np.ndarray) -> None:
    nb = name.encode("utf-8")
    buf.write(struct.pack("<B", len(nb)) + nb + struct.pack("<B", arr.ndim))
    for d in arr.shape:
        buf.write(struct.pack("<I", d))
    buf.write(arr.tobytes())


def save_checkpoint(state: ModelState, path, precision: str = "f32") -> int:
    """Write a checkpoint; returns how many weights saturated to the f16 range."""
    if precision not in ("f32", "f16"):
        raise ValueError(f"precision must be f32 or f16, got {precision!r}")
    buf = io.BytesIO()
    _put(buf, _CONFIG_KEY, np.frombuffer(json.dumps(state.config.to_dict(), sort_keys=True).encode(),
                                         np.uint8))
    sat = 0
    for name, p in state.params.items():
        p = np.asarray(p, np.float32)
        if precision == "f16":
            sat += int((np.abs(p) > F16_MAX).sum())
            _put(buf, f"param/{name}", np.clip(p, -F16_MAX, F16_MAX).astype("<f2"))
        else:
            _put(buf, f"param/{name}", p.astype("<f4"))
    if precision == "f32":
        for tag, d in (("adam_m", state.m), ("adam_v", state.v)):
            for name, p in d.items():
                _put(buf, f"{tag}/{name}", np.asarray(p, "<f4"))
    section = buf.getvalue()
    if sat:
        warnings.warn(f"{sat} weight values saturated to the fp16 range")
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<HBQ", VERSION, 1 if precision == "f16" else 0, state.step))
        f.write(hashlib.sha256(section).digest() + section)
    return sat


def _walk(section: bytes, precision: int):
    """Yield (name, dtype, shape, payload offset) for every tensor record."""
    off = 0
    while off < len(section):
        ln = section[off]
        name = section[off + 1:off + 1 + ln].decode("utf-8")
        ndim = section[off + 1 + ln]
        shape = struct.unpack_from(f"<{ndim}I", section, off + 2 + ln)
        off += 2 + ln + 4 * ndim
        if name == _CONFIG_KEY:
            dt = np.dtype("u1")
        else:
            dt = np.dtype("<f2" if precision == 1 and name.startswith("param/") else "<f4")
        yield name, dt, shape, off
        off += (int(np.prod(shape)) if ndim else 1) * dt.itemsize


def _open(path):
    raw = open(path, "rb").read()
    if raw[:5] != MAGIC:
        raise CheckpointError("not a checkpoint file (bad magic)")
    if len(raw) < 48:
        raise CheckpointError("truncated checkpoint header")
    version, precision, step = struct.unpack_from("<HBQ", raw, 5)
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}")
    return raw, precision, step


def load_checkpoint(path, expected_config: UNetConfig | None = None) -> ModelState:
    """checkpoint.py:85-148: verify magic / version / SHA-256, rebuild the state."""
    raw, precision, step = _open(path)
    section = raw[48:]
    if hashlib.sha256(section).digest() != raw[16:48]:
        raise CheckpointError("integrity hash mismatch (corrupt or tampered file)")
    try:
        tensors = {name: np.frombuffer(section, dt, int(np.prod(shape)) if shape else 1,
                                       off).reshape(shape)
                   for name, dt, shape, off in _walk(section, precision)}
    except (struct.error, ValueError, IndexError) as e:
        raise CheckpointError(f"malformed tensor section: {e}") from None
    if _CONFIG_KEY not in tensors:
        raise CheckpointError("checkpoint carries no config")
    config = UNetConfig.from_dict(json.loads(tensors.pop(_CONFIG_KEY).tobytes().decode()))
    if expected_config is not None and config.to_dict() != expected_config.to_dict():
        raise CheckpointError(f"incompatible checkpoint: config hash {config.hash()[:12]} "
                              f"!= expected {expected_config.hash()[:12]}")
    groups = {"param": {}, "adam_m": {}, "adam_v": {}}
    for key, t in tensors.items():
        tag, _, name = key.partition("/")
        if tag in groups:
            groups[tag][name] = t.astype(np.float32)
    params, m, v = groups["param"], groups["adam_m"], groups["adam_v"]
    if not m:
        m = {k: np.zeros_like(p) for k, p in params.items()}
        v = {k: np.zeros_like(p) for k, p in params.items()}
    return ModelState(config, params, m, v, step)


def weight_payload_bytes(path) -> int:
    """Bytes of the param/ payloads only (checkpoint.py:151-180; App. C size claim)."""
    raw, precision, _ = _open(path)
    return sum((int(np.prod(shape)) if shape else 1) * dt.itemsize
               for name, dt, shape, _ in _walk(raw[48:], precision) if name.startswith("param/"))


def quantize_checkpoint(state: ModelState, path) -> int:
    return save_checkpoint(state, path, precision="f16")
