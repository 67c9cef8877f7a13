"""GPU octree build against the reference's node table
(octree.py:54-125, golden fixtures) and the host DFS build, bit-exact."""

import numpy as np
import pytest

from conftest import load_golden_scene

pytestmark = pytest.mark.gpu


def _same(a, b):
    np.testing.assert_array_equal(a.nodes_id, b.nodes_id)
    np.testing.assert_array_equal(a.nodes_leaf, b.nodes_leaf)
    assert a.max_depth == b.max_depth
    assert a.root_edge == b.root_edge
    np.testing.assert_array_equal(a.root_min, b.root_min)


def test_device_build_matches_reference_goldens(golden):
    from paper_2507_18713_b200.octree import build_octree_device
    from paper_2507_18713_b200.scenes import make_init_scene
    t = build_octree_device(load_golden_scene("rand400m").static)
    np.testing.assert_array_equal(t.nodes_id, golden["march_nodes_id"])
    np.testing.assert_array_equal(t.nodes_leaf, golden["march_nodes_leaf"])
    t = build_octree_device(make_init_scene("S20k").static)
    np.testing.assert_array_equal(t.nodes_id, golden["c1_nodes_id"])
    np.testing.assert_array_equal(t.nodes_leaf, golden["c1_nodes_leaf"])


@pytest.mark.parametrize("name", ["rand400", "rand300", "rand400m", "rand300i", "fd10", "rand60s", "actors"])
def test_device_build_matches_host_build(name):
    from paper_2507_18713_b200.octree import build_octree, build_octree_device
    sc = load_golden_scene(name)
    _same(build_octree_device(sc.static), build_octree(sc.static))
    for a in getattr(sc, "actors", []):
        _same(build_octree_device(a.voxels), build_octree(a.voxels))


def test_device_build_full_size_s1m():
    from paper_2507_18713_b200.octree import build_octree, build_octree_device
    from paper_2507_18713_b200.scenes import get_scene
    v = get_scene("S1M").static
    _same(build_octree_device(v), build_octree(v))


def _with_cells(v, level, ijk):
    from paper_2507_18713_b200.scene import SparseVoxelSet
    n = len(level)
    return SparseVoxelSet(v.bounds).set_arrays(level, ijk, np.zeros((n, 4)), np.zeros((n, 3, 3)),
                                                np.zeros((n, 3, 4)), np.zeros(n), np.zeros(n))


def test_device_build_errors_and_empty():
    from paper_2507_18713_b200.octree import build_octree, build_octree_device
    v = load_golden_scene("rand400m").static
    # a coarse voxel whose cell contains a stored finer voxel
    fine = int(np.argmax(v.level))
    assert v.level[fine] > 0
    w = _with_cells(v, np.r_[v.level, v.level[fine] - 1], np.r_[v.ijk, (v.ijk[fine] >> 1)[None]])
    with pytest.raises(ValueError, match="contains another"):
        build_octree(w)
    with pytest.raises(ValueError, match="contains another"):
        build_octree_device(w)
    e = _with_cells(v, np.zeros(0, np.uint8), np.zeros((0, 3), np.int32))
    _same(build_octree_device(e), build_octree(e))
    one = _with_cells(v, v.level[:1], v.ijk[:1])
    _same(build_octree_device(one), build_octree(one))
