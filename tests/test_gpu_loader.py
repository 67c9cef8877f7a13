"""GPU: salf.v1 records decoded on the device (container.py)
equal the host loader's DeviceScene bit for bit; the octree built from the
device arrays equals the host build; reference error messages."""

import shutil
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
SCENES = Path(__file__).parent / "golden" / "scenes"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("name", ["rand300", "rand400m", "fd10"])
def test_device_loader_matches_host(name):
    from paper_2507_18713_b200.device import DeviceScene, load_device_scene
    from paper_2507_18713_b200.octree import build_octree, build_octree_from_device
    from paper_2507_18713_b200.scene import load_scene
    sc, _ = load_scene(SCENES / name)
    ref = DeviceScene.from_scene(sc)
    ds = load_device_scene(SCENES / name)
    n = sc.static.n
    assert ds.n == n
    assert torch.equal(ds.geo[:n], ref.geo[:n]) and torch.equal(ds.prm[:n], ref.prm[:n])
    torch.testing.assert_close(ds.aux[:n], ref.aux[:n], rtol=1e-15, atol=0)
    np.testing.assert_array_equal(ds.level.cpu().numpy(), sc.static.level)
    np.testing.assert_array_equal(ds.ijk.cpu().numpy(), sc.static.ijk)
    np.testing.assert_array_equal(ds.params[:, 0:4].cpu().numpy(), sc.static.w_s)
    np.testing.assert_array_equal(ds.params[:, 26].cpu().numpy(), sc.static.log_b)
    a = build_octree(sc.static)
    b = build_octree_from_device(ds.level, ds.ijk, ds.bounds)
    assert torch.equal(a.nodes, b.nodes) and a.max_depth == b.max_depth


def test_device_loader_full_size():
    """S1M (1,023,816 records, 124 MB) decoded on the device == host path."""
    from paper_2507_18713_b200.device import DeviceScene, load_device_scene
    from paper_2507_18713_b200.scenes import DATA, get_scene
    sc = get_scene("S1M", "init")
    path = DATA / "S1M_init"
    if not (path / "voxels.bin").exists():
        pytest.skip("scene cache not present")
    ref = DeviceScene.from_scene(sc)
    ds = load_device_scene(path)
    n = sc.static.n
    assert torch.equal(ds.geo[:n], ref.geo[:n]) and torch.equal(ds.prm[:n], ref.prm[:n])


def test_device_loader_errors(tmp_path):
    """container.py:56-59, :91-99: truncated file, non-finite field, duplicate cells."""
    from paper_2507_18713_b200.device import load_device_scene
    from paper_2507_18713_b200.scene import VOXEL_DTYPE, ContainerError
    src = SCENES / "rand300"
    for case in ("trunc", "nan", "dup"):
        dst = tmp_path / case
        shutil.copytree(src, dst)
        raw = np.fromfile(dst / "voxels.bin", dtype=VOXEL_DTYPE)
        if case == "trunc":
            (dst / "voxels.bin").write_bytes(raw.tobytes()[:-5])
            with pytest.raises(ContainerError, match="size mismatch"):
                load_device_scene(dst)
        elif case == "nan":
            raw["w_sh"][17, 1, 2] = np.nan
            raw["log_a"][3] = np.inf
            raw.tofile(dst / "voxels.bin")
            with pytest.raises(ContainerError, match="non-finite values in field 'w_sh'"):
                load_device_scene(dst)
        else:
            raw["level"][5], raw["ijk"][5] = raw["level"][9], raw["ijk"][9]
            raw.tofile(dst / "voxels.bin")
            with pytest.raises(ContainerError, match="duplicate voxel cells"):
                load_device_scene(dst)
