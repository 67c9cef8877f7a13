"""GPU: secondary-ray effects (reference render_ray.py:310-489)
against the reference's own trace_effects outputs (tests/golden/golden_effects.npz,
generator tests/golden/make_golden_effects.py)."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import load_golden_scene

pytestmark = pytest.mark.gpu
HERE = Path(__file__).parent / "golden"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(scope="module")
def fx():
    return np.load(HERE / "golden_effects.npz"), json.loads((HERE / "golden_effects.json").read_text())


@pytest.mark.parametrize("bounces", [1, 2, 3])
def test_trace_effects_matches_reference(fx, bounces):
    from paper_2507_18713_b200 import render_ray as RY
    g, meta = fx
    sc = load_golden_scene("rand300")
    oc = RY.build_scene_octrees(sc)
    spheres = [RY.InjectedSphere(**s) for s in meta["spheres"]]
    col = RY.trace_effects(sc, oc, g["fx_o"], g["fx_d"], g["fx_t"], spheres, meta["sun"], max_bounces=bounces,
                           background=tuple(meta["background"]))
    np.testing.assert_allclose(col.cpu().numpy(), g[f"fx_color_b{bounces}"], rtol=0, atol=1e-4)


def test_trace_effects_without_spheres_is_volume_rendering(fx):
    from paper_2507_18713_b200 import render_ray as RY
    g, meta = fx
    sc = load_golden_scene("rand300")
    oc = RY.build_scene_octrees(sc)
    col = RY.trace_effects(sc, oc, g["fx_o"], g["fx_d"], g["fx_t"], [], meta["sun"], max_bounces=2)
    np.testing.assert_allclose(col.cpu().numpy(), g["fx_color_nospheres"], rtol=0, atol=1e-4)
    rec = RY.integrate_rays(sc, oc, g["fx_o"], g["fx_d"])
    np.testing.assert_allclose(col.cpu().numpy(), rec.out_color.double().cpu().numpy(), rtol=0, atol=1e-12)


def test_effects_validation():
    """render_ray.py:322-330, :374-375."""
    from paper_2507_18713_b200 import render_ray as RY
    with pytest.raises(ValueError, match="radius must be positive"):
        RY.InjectedSphere([0, 0, 0], 0.0, "mirror")
    with pytest.raises(ValueError, match="unknown material"):
        RY.InjectedSphere([0, 0, 0], 1.0, "chrome")
    with pytest.raises(ValueError, match="index of refraction"):
        RY.InjectedSphere([0, 0, 0], 1.0, "glass", ior=0.5)
    with pytest.raises(ValueError, match="max_bounces"):
        RY.trace_effects(None, None, np.zeros((1, 3)), np.array([[1.0, 0, 0]]), 0.0, [], [0, 0, 1], max_bounces=0)
