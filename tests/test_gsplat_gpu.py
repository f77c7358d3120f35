"""GPU tile blend (nar_splat_blend) vs the REAL reference's native blend and the
oracle.  f64 accumulation with the reference's association; only exp() may
differ from libm in the last ulp, so the bar is max |err| <= 1e-9 on the f64
image (a transmittance cut-off flipped by one ulp could move a pixel by at most
1/255 of a colour, which the tests would also catch)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(golden):
    return golden("gsplat")


@pytest.mark.parametrize("tile", [8, 16, 32])
def test_blend_matches_reference(cuda, gs, tile):
    from paper_2407_19097_b200.gsplat import splat_blend_image

    W, H = (int(v) for v in gs["blend/wh"])
    rgb = splat_blend_image(gs["blend/mu"], gs["blend/inv_abc"], gs["blend/boxes"],
                            gs["blend/color"], gs["blend/opacity"], W, H, tile_size=tile)
    assert rgb.shape == (H, W, 3) and rgb.dtype == np.float64
    assert np.max(np.abs(rgb - gs["blend/rgb"])) <= 1e-9


@pytest.mark.parametrize("style", ["vector_field", "terrain"])
def test_render_gsplat_matches_reference(cuda, gs, style):
    from paper_2407_19097_b200.geometry import CameraPose, Intrinsics
    from paper_2407_19097_b200.gsplat import SplatSet, render_gsplat

    p = f"{style}/"
    sp = SplatSet(gs[p + "positions"], gs[p + "cov"], gs[p + "colors"], gs[p + "opacities"])
    cam = CameraPose(gs[p + "campos"], gs[p + "R"], Intrinsics(width=128, height=96))
    img, cnt = render_gsplat(sp, cam, return_counters=True)
    assert img.dtype == np.float32 and img.shape == (96, 128, 3)
    assert np.max(np.abs(img - gs[p + "img"])) <= 1e-6
    assert [cnt["total"], cnt["culled"], cnt["skipped_singular"]] == list(gs[p + "counters"])


def test_blend_large_vs_oracle_and_empty(cuda):
    from paper_2407_19097_b200.gsplat import splat_blend_image

    rng = np.random.default_rng(8)
    n, W, H = 40_000, 333, 211  # ragged tiles
    mu = np.c_[rng.uniform(0, W, n), rng.uniform(0, H, n)]
    s = rng.uniform(0.3, 25.0, n)
    inv_abc = np.c_[1 / s, rng.uniform(-0.1, 0.1, n) / s, 1 / s]
    r = np.ceil(3 * np.sqrt(s))
    boxes = np.c_[np.clip(mu[:, 0] - r, 0, W - 1), np.clip(mu[:, 0] + r, 0, W - 1),
                  np.clip(mu[:, 1] - r, 0, H - 1), np.clip(mu[:, 1] + r, 0, H - 1)].astype(np.int64)
    color = rng.uniform(0, 1, (n, 3))
    opac = rng.uniform(0.01, 0.9, n)
    got = splat_blend_image(mu, inv_abc, boxes, color, opac, W, H)
    ref = oracle.splat_blend(mu, inv_abc, boxes, color, opac, W, H)
    assert np.max(np.abs(got - ref)) <= 1e-9
    empty = splat_blend_image(np.zeros((0, 2)), np.zeros((0, 3)), np.zeros((0, 4), np.int64),
                              np.zeros((0, 3)), np.zeros(0), 40, 30)
    assert empty.shape == (30, 40, 3) and not empty.any()


def test_blend_device_resident_inputs(cuda, gs):
    """Splat arrays already on the device (the bench's resident case) give the
    same image as the numpy inputs, to the last bit."""
    import torch

    from paper_2407_19097_b200.gsplat import splat_blend_image

    W, H = (int(v) for v in gs["blend/wh"])
    arrs = [gs[f"blend/{k}"] for k in ("mu", "inv_abc", "boxes", "color", "opacity")]
    host = splat_blend_image(*arrs, W, H)
    dev = splat_blend_image(*[torch.from_numpy(np.ascontiguousarray(a)).to(cuda) for a in arrs],
                            W, H, device=cuda, return_device=True)
    assert np.array_equal(dev.cpu().numpy(), host)
