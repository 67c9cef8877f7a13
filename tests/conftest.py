import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden.npz")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden_meta.json").read_text())


def load_golden_scene(name):
    from paper_2507_18713_b200.scene import load_scene
    return load_scene(GOLDEN / "scenes" / name)[0]


def oracle_voxels(scene):
    from oracle import salf_oracle as O
    b, v = scene.bounds, scene.static
    return O.Voxels.from_grid(b.aabb_min, b.aabb_max, b.base_edge, v.level, v.ijk, v.w_s, v.w_c,
                              v.w_sh, v.log_a, v.log_b, mode=scene.density_mode)


def oracle_camera(d):
    from oracle import salf_oracle as O
    return O.Camera(d["kind"], d["width"], d["height"], d.get("fx", 0.0), d.get("fy", 0.0),
                    d.get("cx", 0.0), d.get("cy", 0.0), d.get("distortion", (0, 0, 0, 0)),
                    d.get("position", (0, 0, 0)), d.get("quaternion", (1, 0, 0, 0)),
                    d.get("readout_duration", 0.0), d.get("linear_velocity", (0, 0, 0)),
                    d.get("angular_velocity", (0, 0, 0)))


def oracle_lidar(d):
    from oracle import salf_oracle as O
    return O.Lidar(d["beam_elevations"], d.get("azimuth_start", 0.0), d.get("azimuth_end", 2 * np.pi),
                   d["steps"], d.get("scan_period", 0.1), d.get("position", (0, 0, 0)),
                   d.get("quaternion", (1, 0, 0, 0)), d.get("linear_velocity", (0, 0, 0)),
                   d.get("angular_velocity", (0, 0, 0)))


def grads_close_normwise(a: dict, b: dict):
    """GPU-vs-GPU consistency only (atomic vs deterministic order, sharded vs
    unsharded): max|a-b| / max|b| per parameter class.  Reference parity uses
    assert_grads (elementwise, tests/parity.py)."""
    worst = 0.0
    for k in ("w_s", "w_c", "w_sh", "log_a", "log_b"):
        x, y = np.asarray(a[k], np.float64), np.asarray(b[k], np.float64)
        scale = max(np.abs(y).max(), 1e-30)
        e = np.abs(x - y).max() / scale
        worst = max(worst, e)
    return worst


def assert_grads(got: dict, want: dict, mag: dict | None = None):
    """Elementwise gradient parity: |a-b| <= 1e-4 |b| + 1e-5 mag + 1e-9 max|b|
    per element (mag: the oracle's conditioning scale, tests/parity.py)."""
    from parity import assert_ok, grad_report
    return assert_ok(grad_report(got, want, mag))


def assert_image(got, want, name=""):
    """Elementwise image parity: |a-b| <= 1e-4 |b| + 1e-7, NaN masks identical."""
    from parity import assert_ok, image_report
    return assert_ok(image_report(got, want, name))


def magnitude(rec, vox, d_color, d_depth):
    from oracle import salf_oracle as O
    from parity import grad_magnitude
    return grad_magnitude(O, rec, vox, np.asarray(d_color, np.float64).reshape(-1, 3),
                          np.asarray(d_depth, np.float64).reshape(-1))
