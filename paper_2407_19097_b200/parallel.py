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


def row_slice(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) of the padded output resolved by `rank` in the fused path."""
    return rows * rank // world, rows * (rank + 1) // world


class PeerShardedRenderer:
    """Fused composite + resolve over peer memory, no NCCL on
    the data path.

    The rank's keybuf, its shard (positions + attribute streams) and the root's
    output G-buffer live in symmetric memory (``torch.distributed._symmetric_
    memory``: every rank maps every other rank's buffers over NVLink).  A frame
    is: render the local shard into the local keybuf; a device-side barrier;
    ``nar_resolve_peers`` on this rank's row slice -- min over all ranks'
    keybufs, winners' attributes gathered from their owners' shards, channels
    stored straight into the root's G-buffer, every keybuf's slice reset for
    the next frame; a barrier.  Each rank thus reads 1/P of every keybuf
    (16.6 MB inbound per rank at 1080p in total) instead of all-reducing the
    whole buffer and then reducing the planes.
    """

    def __init__(self, width: int, height: int, shard, group=None, pad_multiple: int = 16,
                 root: int = 0, shard_is_symmetric: bool = False):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        from .msr import DeviceCloud, Renderer, _Mapped

        self.group = group or dist.group.WORLD
        self.rank, self.world = dist.get_rank(self.group), dist.get_world_size(self.group)
        self.root = root
        dev = shard.device
        self.r = Renderer(width, height, device=dev, pad_multiple=pad_multiple)
        npix = width * height
        # keybuf in symmetric memory (the renderer renders into it)
        kb = symm.empty(npix, dtype=torch.int64, device=dev)
        kb.copy_(self.r.keybuf)
        self._kh = symm.rendezvous(kb, self.group)
        self.r.keybuf = kb
        self.keybufs = [int(p) for p in self._kh.buffer_ptrs]
        # shard arrays in symmetric memory (equal shapes on all ranks: padded to the max)
        sg = shard.segments[0]
        counts = [None] * self.world
        dist.all_gather_object(counts, (int(sg["begin"]), int(sg["count"])), group=self.group)
        nmax = max(c for _, c in counts)
        self._hold = []

        # A shard the caller allocated in symmetric memory (whole symm.empty
        # buffers, equal counts on all ranks -- ``shard_is_symmetric``) is mapped
        # as is; otherwise it is copied into symmetric buffers once.
        in_place = bool(shard_is_symmetric) and len({c for _, c in counts}) == 1
        flags = [None] * self.world
        dist.all_gather_object(flags, in_place, group=self.group)
        in_place = all(flags)

        def share(t):
            if in_place:
                buf = t
            else:
                buf = symm.empty((nmax,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
                buf[: t.shape[0]].copy_(t)
            h = symm.rendezvous(buf, self.group)
            self._hold.append((buf, h))
            return buf, [int(p) for p in h.buffer_ptrs]

        pos, pos_ptrs = share(sg["positions"])
        names = sorted(sg["streams"])
        st_local, st_ptrs = {}, {}
        for n in names:
            st_local[n], st_ptrs[n] = share(sg["streams"][n])
        self.local = DeviceCloud([{"begin": sg["begin"], "count": sg["count"],
                                   "positions": pos[: sg["count"]],
                                   "streams": {n: st_local[n][: sg["count"]] for n in names}}],
                                 shard.meta, dev)
        segs = []
        for r, (b, c) in enumerate(counts):
            segs.append({"begin": b, "count": c,
                         "positions": _Mapped(pos_ptrs[r], (c, 3)),
                         "streams": {n: _Mapped(st_ptrs[n][r], (c,) + tuple(sg["streams"][n].shape[1:]))
                                     for n in names}})
        self.all = DeviceCloud(segs, shard.meta, dev)
        self._out = None

    def _outputs(self, C: int):
        """Root's G-buffer planes in symmetric memory; every rank writes its slice."""
        import torch
        import torch.distributed._symmetric_memory as symm

        from .msr import _Mapped

        if self._out is not None and self._out[0] == C:
            return self._out[1], self._out[2]
        ph, pw = self.r.alloc_outputs(C)["data"].shape[:2]
        H, W = self.r.height, self.r.width
        dev = self.r.device
        local, peer = {}, {}
        for k, shape, dt in (("data", (ph, pw, C), torch.float32), ("coverage", (H, W), torch.uint8),
                             ("index_plane", (H, W), torch.int64), ("depth", (H, W), torch.float32)):
            buf = symm.empty(shape, dtype=dt, device=dev)
            h = symm.rendezvous(buf, self.group)
            self._hold.append((buf, h))
            local[k] = buf
            peer[k] = _Mapped(int(h.buffer_ptrs[self.root]), shape)
        self._out = (C, local, peer)
        return local, peer

    def frame(self, cam, sel):
        """One sharded frame; returns the root's output dict (complete on root)."""
        names = sel.channel_names(self.all)
        local, peer = self._outputs(len(names))
        self.r.render(self.local, cam)
        self._kh.barrier(channel=0)
        rows = local["data"].shape[0]
        self.r.resolve(self.all, cam, sel, out=peer, peers=self.keybufs,
                       rows=row_slice(rows, self.rank, self.world))
        self._kh.barrier(channel=1)
        return local
