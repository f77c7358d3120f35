"""Multi-GPU MSR: point-sharded render + min-composite over NVLink.

The reference's only parallelism is point-chunk data parallelism with private
z-buffers merged by ``np.minimum.reduce`` (pkg/src/nar/_kernels/__init__.py:
81-94).  The B200 version shards the cloud across GPUs the same way:

* rank r owns the contiguous global index range [begin_r, begin_r + n_r) and
  renders it into a local keybuf in the *signed* key domain (key ^ 2^63, in
  which unsigned order equals int64 order);
* ``composite_keys`` all-reduces the keybufs with int64 MIN (NCCL over
  NVLink/NVSwitch; exact, order independent -- the same min-merge);
* every rank resolves only the pixels whose winner it owns (``owner_only``),
  all other pixels' channels are written as +0.0;
* ``reduce_planes`` sums the channel planes' int32 bit patterns onto the root:
  exactly one rank contributes a non-zero pattern per pixel, so the integer
  sum reproduces the owner's float bits exactly (a float SUM could flip the
  sign of -0.0).

Coverage, index and depth planes derive from the composited keys and are
identical on every rank.  The helpers take plain torch tensors and a process
group, so the same code runs over gloo on CPU in the tests.
"""

from __future__ import annotations

import numpy as np

SIGN_FLIP = 0x8000000000000000
EMPTY_SIGNED = np.int64(0x7FFFFFFFFFFFFFFF)  # EMPTY_KEY ^ SIGN_FLIP


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n points for `rank` (np.linspace bounds, as
    the reference chunks points, _kernels/__init__.py:91)."""
    lo = int(np.floor(n * rank / world))
    hi = int(np.floor(n * (rank + 1) / world))
    return lo, hi


def to_signed(keys_u64: np.ndarray) -> np.ndarray:
    """Unsigned reference keys -> signed-domain int64 view."""
    return (np.asarray(keys_u64, np.uint64) ^ np.uint64(SIGN_FLIP)).view(np.int64)


def from_signed(keys_i64: np.ndarray) -> np.ndarray:
    return np.asarray(keys_i64, np.int64).view(np.uint64) ^ np.uint64(SIGN_FLIP)


def composite_keys(keybuf, group=None) -> None:
    """In-place int64 MIN all-reduce of a signed-domain keybuf (torch int64)."""
    import torch.distributed as dist

    dist.all_reduce(keybuf, op=dist.ReduceOp.MIN, group=group)


def reduce_planes(data, dst: int = 0, group=None) -> None:
    """Sum the int32 bit patterns of owner-only f32 planes onto `dst`."""
    import torch
    import torch.distributed as dist

    if data.dtype != torch.float32:
        raise ValueError("reduce_planes expects float32 planes")
    dist.reduce(data.view(torch.int32), dst=dst, op=dist.ReduceOp.SUM, group=group)


class ShardedRenderer:
    """One rank's part of a sharded frame (device tensors, NCCL group)."""

    def __init__(self, width: int, height: int, device=None, pad_multiple: int | None = None,
                 group=None):
        from .msr import Renderer

        self.r = Renderer(width, height, device=device, signed_keys=True,
                          pad_multiple=pad_multiple)
        self.group = group

    def frame(self, cloud, cam, sel, out=None, root: int = 0):
        """Render the local shard, composite, owner-resolve, reduce to root.
        Returns the DeviceFeatureImage (complete on `root`)."""
        self.r.render(cloud, cam)
        composite_keys(self.r.keybuf, self.group)
        img = self.r.resolve(cloud, cam, sel, out=out, owner_only=True)
        reduce_planes(img.data, dst=root, group=self.group)
        return img
