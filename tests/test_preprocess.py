"""Data formats on either side of the hot path, CPU parts.

NARPC point-cloud files (geometry/pointcloud.py:143-199) and NARCK checkpoints
(neural/checkpoint.py) written by the REAL reference (tests/golden/preprocess.npz,
tests/golden/make_golden.py) must load to the same arrays and re-save to the
same bytes; the reference's error types on damaged files; the Morton oracle is
pinned against the reference's morton_keys / morton_reorder.
"""

import struct

import numpy as np
import pytest

import oracle
from paper_2407_19097_b200 import checkpoint as ck
from paper_2407_19097_b200 import preprocess as pp
from paper_2407_19097_b200.errors import CapacityError, CheckpointError, CorruptError, FormatError
from paper_2407_19097_b200.geometry import PointCloud, Stream


@pytest.fixture(scope="module")
def pre(golden):
    return golden("preprocess")


def _write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(bytes(data))
    return p


# ---- NARPC ---------------------------------------------------------------------------

def test_narpc_reference_file_loads(pre, tmp_path):
    pc = pp.load_pointcloud(_write(tmp_path, "a.narpc", pre["narpc/file"]))
    assert np.array_equal(pc.positions, pre["narpc/positions"])
    assert [s.name for s in pc.streams] == ["rgb", "velocity", "temperature"]
    for s in pc.streams:
        ref = pre[f"narpc/stream/{s.name}"]
        assert s.data.dtype == ref.dtype and np.array_equal(s.data, ref)


def test_narpc_save_is_byte_identical(pre, tmp_path):
    pc = PointCloud(pre["narpc/positions"],
                    [Stream("rgb", "u8", pre["narpc/stream/rgb"]),
                     Stream("velocity", "f32", pre["narpc/stream/velocity"]),
                     Stream("temperature", "f32", pre["narpc/stream/temperature"])])
    pp.save_pointcloud(pc, tmp_path / "b.narpc")
    assert (tmp_path / "b.narpc").read_bytes() == bytes(pre["narpc/file"])
    pp.save_pointcloud(PointCloud(np.zeros((0, 3), np.float32)), tmp_path / "e.narpc")
    assert (tmp_path / "e.narpc").read_bytes() == bytes(pre["narpc/empty_file"])
    assert pp.load_pointcloud(tmp_path / "e.narpc").count == 0


@pytest.mark.gpu
def test_narpc_pinned_load(cuda, pre, tmp_path):
    pc = pp.load_pointcloud(_write(tmp_path, "a.narpc", pre["narpc/file"]), pinned=True)
    assert np.array_equal(pc.positions, pre["narpc/positions"])


def test_narpc_errors(pre, tmp_path):
    raw = bytearray(pre["narpc/file"])
    with pytest.raises(FormatError):
        pp.load_pointcloud(_write(tmp_path, "m", b"NARPX\0" + raw[6:]))
    bad = bytearray(raw)
    bad[6:8] = struct.pack("<H", 2)
    with pytest.raises(FormatError):
        pp.load_pointcloud(_write(tmp_path, "v", bad))
    bad = bytearray(raw)
    bad[16] = 9
    with pytest.raises(CapacityError):
        pp.load_pointcloud(_write(tmp_path, "c", bad))
    bad = bytearray(raw)
    bad[17 + 1 + 3] = 7  # format code of the first stream ("rgb")
    with pytest.raises(FormatError):
        pp.load_pointcloud(_write(tmp_path, "f", bad))
    for cut in (3, 10, 19, len(raw) - 1):
        with pytest.raises(CorruptError, match="truncated"):
            pp.load_pointcloud(_write(tmp_path, f"t{cut}", raw[:cut]))
    with pytest.raises(CorruptError, match="trailing"):
        pp.load_pointcloud(_write(tmp_path, "x", raw + b"\0\0"))


# ---- checkpoints -----------------------------------------------------------------------

def _ref_state(pre):
    from paper_2407_19097_b200.neural import UNetConfig

    cfg = UNetConfig(input_channels=4, channel_names=("r", "g", "b", "d"), base_channels=4,
                     max_channels=32, init_seed=5)
    return cfg


def test_checkpoint_reference_files_load(pre, tmp_path):
    cfg = _ref_state(pre)
    st = ck.load_checkpoint(_write(tmp_path, "f32", pre["ckpt/f32_file"]), expected_config=cfg)
    assert st.step == 1234 and st.config == cfg
    ref = oracle.init_params(cfg)
    assert set(st.params) == set(ref)
    for k, v in st.params.items():
        want = ref[k].copy()
        if k == "enc0a.f_w":
            want[0, 0, 0, :2] = [70000.0, -1e6]
        assert v.dtype == np.float32 and np.array_equal(v, want), k
    assert np.any(st.m["head.w"] != 0) and not np.any(st.m["enc0a.f_w"])
    q = ck.load_checkpoint(_write(tmp_path, "f16", pre["ckpt/f16_file"]))
    assert q.params["enc0a.f_w"][0, 0, 0, 0] == 65504.0
    assert q.params["enc0a.f_w"][0, 0, 0, 1] == -65504.0
    assert not np.any(q.m["head.w"])  # moments dropped in f16 files
    for k, v in q.params.items():
        assert np.array_equal(v, st.params[k].clip(-65504, 65504).astype(np.float16)
                              .astype(np.float32)), k


def test_checkpoint_save_is_byte_identical(pre, tmp_path):
    st = ck.load_checkpoint(_write(tmp_path, "f32", pre["ckpt/f32_file"]))
    ck.save_checkpoint(st, tmp_path / "a")
    assert (tmp_path / "a").read_bytes() == bytes(pre["ckpt/f32_file"])
    with pytest.warns(UserWarning, match="saturated"):
        sat = ck.quantize_checkpoint(st, tmp_path / "b")
    assert sat == int(pre["ckpt/saturated"]) == 2
    assert (tmp_path / "b").read_bytes() == bytes(pre["ckpt/f16_file"])
    assert ck.weight_payload_bytes(tmp_path / "a") == int(pre["ckpt/payload_f32"])
    assert ck.weight_payload_bytes(tmp_path / "b") == int(pre["ckpt/payload_f16"])
    assert 2 * int(pre["ckpt/payload_f16"]) == int(pre["ckpt/payload_f32"])
    with pytest.raises(ValueError):
        ck.save_checkpoint(st, tmp_path / "c", precision="bf16")


def test_checkpoint_errors(pre, tmp_path):
    from paper_2407_19097_b200.neural import UNetConfig

    raw = bytearray(pre["ckpt/f16_file"])
    with pytest.raises(CheckpointError, match="magic"):
        ck.load_checkpoint(_write(tmp_path, "m", b"NARCX" + raw[5:]))
    bad = bytearray(raw)
    bad[5:7] = struct.pack("<H", 3)
    with pytest.raises(CheckpointError, match="version"):
        ck.load_checkpoint(_write(tmp_path, "v", bad))
    bad = bytearray(raw)
    bad[1000] ^= 0x40
    with pytest.raises(CheckpointError, match="hash"):
        ck.load_checkpoint(_write(tmp_path, "h", bad))
    with pytest.raises(CheckpointError, match="hash"):
        ck.load_checkpoint(_write(tmp_path, "t", raw[:-10]))
    with pytest.raises(CheckpointError, match="incompatible"):
        ck.load_checkpoint(_write(tmp_path, "ok", raw),
                           expected_config=UNetConfig(input_channels=4, base_channels=4))


# ---- Morton oracle pinned to the reference --------------------------------------------

@pytest.mark.parametrize("name", ["uniform", "flat", "dups", "single"])
def test_morton_oracle_matches_reference(pre, name):
    pos = pre[f"morton/{name}/positions"]
    assert np.array_equal(oracle.morton_keys(pos), pre[f"morton/{name}/keys"])
    assert np.array_equal(oracle.morton_order(pos), pre[f"morton/{name}/order"])


def test_selection_from_channels():
    from paper_2407_19097_b200.msr import StreamSelection
    from paper_2407_19097_b200.pipeline import selection_from_channels

    for sel in (StreamSelection(rgb=True, depth=True),
                StreamSelection(rgb=True, depth=True, vel2d=True, coverage_channel=True),
                StreamSelection(depth=True, vel3d=True)):
        assert selection_from_channels(sel.channel_names()) == sel


# ---- feature dumps ---------------------------------------------------------------------

def test_feature_dump_roundtrip_and_errors(pre, tmp_path):
    names = ("r", "g", "b", "d", "coverage")
    got_names, data = pp.load_features(_write(tmp_path, "f.feat", pre["feat/file"]))
    assert got_names == names and np.array_equal(data, pre["feat/data"])
    pp.save_features(names, pre["feat/data"], tmp_path / "g.feat")
    assert (tmp_path / "g.feat").read_bytes() == bytes(pre["feat/file"])
    raw = bytes(pre["feat/file"])
    with pytest.raises(CorruptError):
        pp.load_features(_write(tmp_path, "s", raw[:8]))
    with pytest.raises(CorruptError):
        pp.load_features(_write(tmp_path, "t", raw[:-4]))
    with pytest.raises(ValueError):
        pp.save_features(names[:4], pre["feat/data"], tmp_path / "x.feat")


def test_device_buffer_validation_cpu():
    """Layout checks in front of the raw-pointer kernels run without a GPU: CPU
    tensors, wrong dtypes or shapes and mismatched streams raise ValueError."""
    import torch

    from paper_2407_19097_b200.msr import DeviceCloud, _check_outputs, _check_positions

    with pytest.raises(ValueError):
        _check_positions(torch.zeros((4, 3)))  # not on a GPU
    with pytest.raises(ValueError):
        DeviceCloud.from_tensors(torch.zeros((4, 3), dtype=torch.float64))
    with pytest.raises(ValueError):
        pp.morton_keys_device(torch.zeros((4, 2)))
    ok = {"data": torch.zeros((8, 8, 4)), "coverage": torch.zeros((6, 7), dtype=torch.uint8),
          "index_plane": torch.zeros((6, 7), dtype=torch.int64), "depth": torch.zeros((6, 7))}
    _check_outputs(ok, 4, 6, 7)
    with pytest.raises(ValueError, match="data"):
        _check_outputs(ok, 3, 6, 7)
    with pytest.raises(ValueError, match="index_plane"):
        _check_outputs(dict(ok, index_plane=torch.zeros((6, 7), dtype=torch.int32)), 4, 6, 7)
    with pytest.raises(ValueError, match="depth"):
        _check_outputs(dict(ok, depth=torch.zeros((7, 6))), 4, 6, 7)
