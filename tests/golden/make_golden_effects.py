"""Golden fixtures for the secondary-ray effects, generated
by the REFERENCE implementation itself (render_ray.py:310-489, trace_effects).

Run in the build container (where the read-only reference is importable):

    python tests/golden/make_golden_effects.py

Camera rays over the committed golden scene rand300 with one sphere of each
material (mirror, glass, opaque) placed inside the volume, plus a sun
direction so volume points occluded by a sphere are shadowed.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from salf import container as R_io  # noqa: E402
from salf import render_ray as R_ray  # noqa: E402
from salf import sensors as R_sen  # noqa: E402
from salf.synthetic import look_at_quaternion  # noqa: E402

SPHERES = [
    dict(center=[4.2, 3.9, 3.0], radius=1.1, material="mirror"),
    dict(center=[2.6, 5.4, 4.4], radius=0.9, material="glass", ior=1.5),
    dict(center=[5.6, 2.3, 4.9], radius=0.7, material="opaque", albedo=[0.8, 0.3, 0.1]),
    dict(center=[3.3, 2.4, 2.2], radius=0.5, material="glass", ior=1.0),
]
SUN = [0.3, -0.5, 0.8]


def main():
    sc = R_io.load_scene(HERE / "scenes" / "rand300")
    oc = R_ray.build_scene_octrees(sc)
    pos = np.array([11.3, 9.7, 7.1])
    cam = R_sen.CameraModel(kind="pinhole", width=40, height=30, fx=34.0, fy=34.0, cx=20.0, cy=15.0,
                            position=pos, quaternion=look_at_quaternion(pos, [4.0, 4.0, 3.5]))
    rays = R_sen.camera_rays(cam)
    spheres = [R_ray.InjectedSphere(**s) for s in SPHERES]
    out = {}
    for bounces in (1, 2, 3):
        col = R_ray.trace_effects(sc, oc, rays.origins, rays.dirs, rays.t_stamps, spheres, SUN,
                                  max_bounces=bounces, background=(0.1, 0.15, 0.2))
        out[f"fx_color_b{bounces}"] = col
    col = R_ray.trace_effects(sc, oc, rays.origins, rays.dirs, rays.t_stamps, [], SUN, max_bounces=2)
    out["fx_color_nospheres"] = col
    out.update(fx_o=rays.origins, fx_d=rays.dirs, fx_t=rays.t_stamps)
    np.savez_compressed(HERE / "golden_effects.npz", **out)
    (HERE / "golden_effects.json").write_text(json.dumps({"spheres": SPHERES, "sun": SUN,
                                                          "background": [0.1, 0.15, 0.2]}, indent=1) + "\n")
    print("wrote", HERE / "golden_effects.npz")


if __name__ == "__main__":
    main()
