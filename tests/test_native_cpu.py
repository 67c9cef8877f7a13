"""CPU-side checks of the native library: it loads without a GPU, exports every
symbol include/salf_b200.h declares, and its host octree build reproduces the
reference's node table (no CUDA needed for that entry point)."""

import re
from pathlib import Path

import ctypes
import numpy as np
import pytest

from conftest import ROOT, load_golden_scene


def _header_symbols():
    text = (ROOT / "include" / "salf_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|size_t|char\s*\*|const char\s*\*)\s*\*?\s*(salf_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_exports_header_symbols():
    from paper_2507_18713_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = _header_symbols()
    assert len(syms) >= 14, syms
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/salf_b200.h but not exported"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"


def _build(scene):
    from paper_2507_18713_b200 import _lib
    lib = _lib.load(require_cuda=False)
    v = scene.static
    b = scene.bounds
    ext = b.aabb_max - b.aabb_min
    m = max(0, int(np.ceil(np.log2(max(ext.max(), 1e-300) / b.base_edge) - 1e-12)))
    lv = np.ascontiguousarray(v.level.astype(np.uint8))
    ijk = np.ascontiguousarray(v.ijk.astype(np.int32))
    nn, md = ctypes.c_int64(0), ctypes.c_int32(0)
    assert lib.salf_octree_build_host(v.n, lv.ctypes.data, ijk.ctypes.data, m, None, 0,
                                      ctypes.byref(nn), ctypes.byref(md)) == 0
    nodes = np.empty(nn.value, np.int32)
    assert lib.salf_octree_build_host(v.n, lv.ctypes.data, ijk.ctypes.data, m, nodes.ctypes.data,
                                      nodes.size, ctypes.byref(nn), ctypes.byref(md)) == 0
    ids = np.where(nodes >= 0, nodes, np.where(nodes == -1, -1, -nodes.astype(np.int64) - 2))
    leaf = np.where(nodes >= 0, 0, np.where(nodes == -1, -1, 1))
    return ids, leaf


def test_native_octree_build_matches_reference(golden):
    ids, leaf = _build(load_golden_scene("rand400m"))
    np.testing.assert_array_equal(ids, golden["march_nodes_id"])
    np.testing.assert_array_equal(leaf, golden["march_nodes_leaf"])


def test_native_octree_build_c1_scene(golden):
    from paper_2507_18713_b200.scenes import make_init_scene
    ids, leaf = _build(make_init_scene("S20k"))
    np.testing.assert_array_equal(ids, golden["c1_nodes_id"])
    np.testing.assert_array_equal(leaf, golden["c1_nodes_leaf"])


def test_scene_generator_matches_reference_cli_bytes():
    import hashlib
    import json
    from paper_2507_18713_b200.scene import records_from_set
    from paper_2507_18713_b200.scenes import make_init_scene
    dig = json.loads((ROOT / "tests" / "golden" / "scene_digests.json").read_text())
    for name in ("S20k", "S1M"):
        sc = make_init_scene(name)
        assert hashlib.sha256(records_from_set(sc.static).tobytes()).hexdigest() == dig[name], name


def test_container_roundtrip_byte_identical(tmp_path):
    from paper_2507_18713_b200.scene import load_scene, save_scene
    src = ROOT / "tests" / "golden" / "scenes" / "rand400"
    sc, _ = load_scene(src)
    save_scene(sc, tmp_path / "s")
    assert (tmp_path / "s" / "voxels.bin").read_bytes() == (src / "voxels.bin").read_bytes()
    assert (tmp_path / "s" / "meta.json").read_text() == (src / "meta.json").read_text()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_18713_b200 import render_raster
    from paper_2507_18713_b200.sensors import CameraModel
    sc = load_golden_scene("rand400")
    with pytest.raises(RuntimeError, match="CUDA"):
        render_raster.rasterize_scene(sc, CameraModel("pinhole", 8, 8, 8.0, 8.0, 4.0, 4.0))


def test_fastmath_exp_expm1_accuracy(tmp_path):
    """csrc/salf_fastmath.h (the exp/expm1 the render kernels use), compiled
    on the host with FMA contraction off: exp <= 1 ulp, expm1 <= 1.1 ulp on the
    render path's range (x <= 0), specials (NaN, +-inf, 0, overflow) exact."""
    import subprocess
    exe = tmp_path / "fmc"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", str(ROOT / "tools" / "fastmath_check.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "300000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def _integration_snippet():
    text = (ROOT / "INTEGRATION.md").read_text()
    return re.findall(r"```python\n(.*?)```", text, flags=re.S)[0]


def test_integration_snippet_structs_match_abi():
    """The ctypes binding documented in INTEGRATION.md runs as written and its
    structs have the C ABI's layout (field names, offsets, sizes)."""
    from paper_2507_18713_b200 import _lib
    ns = {"LIB_PATH": str(_lib.LIB_PATH)}
    exec(compile(_integration_snippet(), "INTEGRATION.md", "exec"), ns)
    for doc, abi in ((ns["_Scene"], _lib.SceneT), (ns["_Camera"], _lib.CameraT)):
        assert ctypes.sizeof(doc) == ctypes.sizeof(abi)
        assert [f[0] for f in doc._fields_] == [f[0] for f in abi._fields_]
        for name, _ in abi._fields_:
            assert getattr(doc, name).offset == getattr(abi, name).offset, name
