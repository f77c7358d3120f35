"""INTEGRATION.md section 2, executed: the maintainer patch (a ``cuda_impl``
backend module plus one ``_resolve`` branch) applied to a temporary copy of
the reference package installed in baseline/_ref, then the reference's own
``nar.msr.rasterize(..., backend="cuda")`` and ``nar._kernels.zbuffer_render``
checked against the golden fixtures the unpatched reference produced.

The patch text is taken from INTEGRATION.md itself, so the documented binding
is what runs.  Skipped when baseline/_ref (the pip --target install of the
reference) is absent."""

import importlib
import re
import shutil
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref" / "nar"


def _blocks():
    text = (ROOT / "INTEGRATION.md").read_text()
    return re.findall(r"```python\n(.*?)```", text, re.S)


@pytest.fixture(scope="module")
def patched_nar(tmp_path_factory, cuda):
    if not (REF / "__init__.py").exists():
        pytest.skip("baseline/_ref (installed reference package) not present")
    tmp = tmp_path_factory.mktemp("refpatch")
    shutil.copytree(REF, tmp / "nar")
    blocks = _blocks()
    impl = next(b for b in blocks if "cuda_impl.py" in b)
    impl = impl.replace("/path/to/paper_2407_19097_b200/libnar_b200.so",
                        str(ROOT / "paper_2407_19097_b200" / "libnar_b200.so"))
    (tmp / "nar" / "_kernels" / "cuda_impl.py").write_text(impl)
    branch = next(b for b in blocks if 'if name == "cuda"' in b)
    init = tmp / "nar" / "_kernels" / "__init__.py"
    src = init.read_text()
    anchor = '    if name == "python":\n'
    assert anchor in src, "reference _resolve changed shape"
    init.write_text(src.replace(anchor, branch.rstrip("\n") + "\n" + anchor, 1))
    saved = {k: v for k, v in sys.modules.items() if k == "nar" or k.startswith("nar.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, str(tmp))
    try:
        yield importlib.import_module("nar")
    finally:
        sys.path.remove(str(tmp))
        for k in [k for k in sys.modules if k == "nar" or k.startswith("nar.")]:
            del sys.modules[k]
        sys.modules.update(saved)


def test_patched_reference_rasterize_cuda(patched_nar, golden):
    nar = patched_nar
    from nar.geometry import CameraPose, Intrinsics, PointCloud, Stream
    from nar.msr import StreamSelection, rasterize

    g = golden("raster_random")
    for ci in range(6):
        p = f"c{ci}/"
        W, H = (int(v) for v in g[p + "wh"])
        pc = PointCloud(g[p + "positions"], [Stream("rgb", "u8", g[p + "rgb"]),
                                             Stream("velocity", "f32", g[p + "velocity"]),
                                             Stream("temp", "f32", g[p + "temp"]),
                                             Stream("mask", "u8", g[p + "mask"])])
        cam = CameraPose(g[p + "campos"], g[p + "R"],
                         Intrinsics(fov_y_deg=float(g[p + "fov"]), width=W, height=H))
        sel = StreamSelection(rgb=True, depth=True, vel2d=True, vel3d=True,
                              scalars=("temp", "mask"), coverage_channel=True,
                              velocity_scale=float(g[p + "velocity_scale"]))
        i = cam.intrinsics
        kb = nar._kernels.zbuffer_render(pc.positions, cam.orientation, cam.position, i.focal_px,
                                         i.cx, i.cy, i.near, i.far, W, H, backend="cuda")
        assert np.array_equal(kb, g[p + "keybuf"])
        fi = rasterize(pc, cam, sel, backend="cuda")  # the reference resolve on GPU keys
        assert np.array_equal(fi.index_plane, g[p + "index_plane"])
        assert np.array_equal(fi.data, g[p + "data"])  # same numpy resolve: bit-identical
    with pytest.raises(ValueError):
        nar._kernels.zbuffer_render(np.zeros((1, 3), np.float32), np.eye(3), np.zeros(3), 1, 1, 1,
                                    0.1, 10, 4, 4, backend="nope")
