"""Multi-process (world_size 2, gloo, CPU) checks of the sharded composite.

The GPU render/resolve kernels cannot run here, so each rank produces its
shard's keybuf and owner-only planes with the CPU oracle; the product's
composite (int64 MIN all-reduce in the signed key domain) and plane reduction
(int32 SUM of float bit patterns) must then reproduce the single-process
reference exactly -- the property the NCCL path relies on.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from paper_2407_19097_b200.geometry import Intrinsics, PointCloud, Stream, look_at

    rng = np.random.default_rng(123)
    n = 40_000
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    pos[rng.integers(0, n, 2000)] = pos[rng.integers(0, n, 2000)]  # cross-shard ties
    vel = rng.normal(size=(n, 3)).astype(np.float32)
    vel[::7] = -0.0
    pc = PointCloud(pos, [Stream("rgb", "u8", rng.integers(0, 256, (n, 3), dtype=np.uint8)),
                          Stream("velocity", "f32", vel)])
    cam = look_at((0.3, -2.4, 1.1), (0, 0, 0), Intrinsics(width=96, height=72))
    return pc, cam


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_19097_b200 import parallel
        from paper_2407_19097_b200.msr import StreamSelection

        pc, cam = _scene()
        i = cam.intrinsics
        lo, hi = parallel.shard_range(pc.count, rank, world)
        kb = np.full(i.width * i.height, oracle.EMPTY_KEY, np.uint64)
        oracle.zbuffer_accumulate(kb, pc.positions[lo:hi], lo, cam.orientation, cam.position,
                                  i.focal_px, i.cx, i.cy, i.near, i.far, i.width, i.height)
        t = torch.from_numpy(parallel.to_signed(kb).copy())
        parallel.composite_keys(t)
        comp = parallel.from_signed(t.numpy())
        # owner-only resolve of the composited frame, emulated with the oracle
        sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, velocity_scale=1.5)
        full = oracle.resolve(comp, pc, cam, sel)
        owned = (full["index_plane"] >= lo) & (full["index_plane"] < hi)
        planes = np.where(owned[..., None], full["data"], np.float32(0.0)).astype(np.float32)
        pt = torch.from_numpy(np.ascontiguousarray(planes))
        parallel.reduce_planes(pt, dst=0)
        if rank == 0:
            q.put((comp, pt.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_composite_equals_single_process():
    pc, cam = _scene()
    from paper_2407_19097_b200.msr import StreamSelection

    sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, velocity_scale=1.5)
    ref = oracle.rasterize(pc, cam, sel)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    comp, planes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(comp, ref["keybuf"])
    # bit-exact including the sign of zero (int32 SUM of bit patterns)
    assert np.array_equal(planes.view(np.int32), ref["data"].view(np.int32))


def test_shard_ranges_cover_and_match_reference_chunking():
    from paper_2407_19097_b200 import parallel

    for n in (0, 1, 7, 1000, 350_000_000):
        for w in (1, 2, 3, 4, 8):
            rs = [parallel.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            ref = np.linspace(0, n, w + 1).astype(np.int64)
            assert [r[0] for r in rs] == list(ref[:-1])


def test_signed_domain_preserves_order():
    from paper_2407_19097_b200 import parallel

    rng = np.random.default_rng(0)
    k = rng.integers(0, 2 ** 63, 10_000, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 10_000, dtype=np.uint64)
    k = np.concatenate([k, [np.uint64(0), np.uint64(2 ** 64 - 1), np.uint64(2 ** 63)]])
    s = parallel.to_signed(k)
    assert np.array_equal(np.argsort(k, kind="stable"), np.argsort(s, kind="stable"))
    assert np.array_equal(parallel.from_signed(s), k)
    assert s[-2] == parallel.EMPTY_SIGNED


def _nccl_worker(port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        from paper_2407_19097_b200.msr import DeviceCloud, Renderer
        from paper_2407_19097_b200.parallel import ShardedRenderer
        from paper_2407_19097_b200.msr import StreamSelection

        torch.cuda.set_device(0)
        pc, cam = _scene()
        i = cam.intrinsics
        cloud = DeviceCloud.from_host(pc)
        sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, velocity_scale=1.5)
        sr = ShardedRenderer(i.width, i.height)
        img = sr.frame(cloud, cam, sel)
        ref = Renderer(i.width, i.height).rasterize(cloud, cam, sel)
        q.put((img.data.cpu().numpy(), ref.data.cpu().numpy(),
               img.index_plane.cpu().numpy(), ref.index_plane.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_single_rank_sharded_frame(cuda):
    """The NCCL path on the GPU (signed key domain render, int64 MIN all-reduce,
    owner-only resolve, int32 SUM reduce) with one rank equals the plain frame."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    got, ref, gi, ri = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert np.array_equal(gi, ri)
    assert np.array_equal(got.view(np.int32), ref.view(np.int32))


@pytest.mark.gpu
def test_fused_composite_resolve_virtual_ranks(cuda):
    """nar_resolve_peers over several keybufs (the kernel a rank runs on its peers'
    mapped buffers; here three shards rendered into three local buffers) with the
    rows split into slices == the plain single-buffer frame, bit-exact."""
    import torch

    from paper_2407_19097_b200 import parallel
    from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection

    pc, cam = _scene()
    i = cam.intrinsics
    sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, velocity_scale=1.5)
    whole = DeviceCloud.from_host(pc)
    ref = Renderer(i.width, i.height, pad_multiple=16).rasterize(whole, cam, sel)
    world = 3
    shards, rens = [], []
    for r in range(world):
        lo, hi = parallel.shard_range(pc.count, r, world)
        from paper_2407_19097_b200.geometry import PointCloud, Stream

        sub = PointCloud(pc.positions[lo:hi], [Stream(s.name, s.format, s.data[lo:hi])
                                               for s in pc.streams])
        shards.append(DeviceCloud.from_host(sub, begin=lo))
        rn = Renderer(i.width, i.height, pad_multiple=16)
        rn.render(shards[-1], cam)
        rens.append(rn)
    segs = [sg for sh in shards for sg in sh.segments]
    cloud = DeviceCloud(segs, shards[0].meta, cuda)
    out = rens[0].alloc_outputs(len(sel.channel_names(cloud)))
    peers = [rn.keybuf.data_ptr() for rn in rens]
    ph = out["data"].shape[0]
    cuts = [0, ph // 3, 2 * ph // 3, ph]
    for r in range(world):
        rens[r].resolve(cloud, cam, sel, out=out, peers=peers, rows=(cuts[r], cuts[r + 1]))
    torch.cuda.synchronize()
    assert torch.equal(out["index_plane"], ref.index_plane)
    assert torch.equal(out["data"].view(torch.int32), ref.data.view(torch.int32))
    for rn in rens:  # slices cleared every keybuf
        assert bool((rn.keybuf == rn.keybuf[0]).all())


def _peer_worker(port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2407_19097_b200.msr import DeviceCloud, Renderer, StreamSelection
        from paper_2407_19097_b200.parallel import PeerShardedRenderer

        pc, cam = _scene()
        i = cam.intrinsics
        cloud = DeviceCloud.from_host(pc)
        sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True, velocity_scale=1.5)
        pr = PeerShardedRenderer(i.width, i.height, cloud)
        outs = [pr.frame(cam, sel) for _ in range(2)]  # second frame: keybuf was re-cleared
        torch.cuda.synchronize()
        ref = Renderer(i.width, i.height, pad_multiple=16).rasterize(cloud, cam, sel)
        q.put((outs[1]["data"].cpu().numpy(), ref.data.cpu().numpy(),
               outs[1]["index_plane"].cpu().numpy(), ref.index_plane.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_sharded_frame_single_rank(cuda):
    """The symmetric-memory fused path end to end with one rank (peer pointer =
    own buffer): equals the plain frame, twice in a row."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_peer_worker, args=(_free_port(), q))
    p.start()
    got, ref, gi, ri = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert np.array_equal(gi, ri)
    assert np.array_equal(got.view(np.int32), ref.view(np.int32))
