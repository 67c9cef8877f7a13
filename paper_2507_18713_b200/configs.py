"""The BASELINE.json workloads as concrete sensors.

C1  S20k, cam_eval_000 scaled to 256^2 (bench.scale_camera), raster forward.
C2  S1M, 1920x1080 pinhole, 70 deg HFOV, raster forward + backward.
C3  S1M, 128-beam spinning LiDAR, 1800 azimuth steps (230,400 rays).
C4  S2M, 1920x1080 equidistant fisheye + rolling shutter, ray path.
C5  S1M, 8 C2-style cameras (yaw 0, 45, ... deg) + 2 C3 LiDARs, training step.
Sensor origins sit off the grid planes (the reference marcher
crawls when an origin lies exactly on a voxel face with an axis-aligned ray).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .sensors import CameraModel, LidarModel, look_at_quaternion

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"
C2_POS = np.array([-3.01, 0.013, 1.6])
C2_TARGET = np.array([2.0, 0.0, 0.8])


def c1_camera() -> CameraModel:
    meta = json.loads((GOLDEN / "golden_meta.json").read_text())
    return CameraModel.from_dict(meta["c1_cam"])


def c2_camera(yaw_deg: float = 0.0, width: int = 1920, height: int = 1080) -> CameraModel:
    f = 0.5 * width / np.tan(0.5 * np.deg2rad(70.0))
    pos = C2_POS.copy()
    if yaw_deg:
        # orbit the look-at target, keeping the C2 distance and height
        rel = pos[:2] - C2_TARGET[:2]
        a = np.deg2rad(yaw_deg)
        rot = np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]])
        pos[:2] = C2_TARGET[:2] + rot @ rel
    return CameraModel(kind="pinhole", width=width, height=height, fx=f, fy=f, cx=width / 2.0,
                       cy=height / 2.0, position=pos, quaternion=look_at_quaternion(pos, C2_TARGET))


def c3_lidar(position=(0.0137, -0.0213, 1.3)) -> LidarModel:
    return LidarModel(beam_elevations=np.deg2rad(np.linspace(-25.0, 15.0, 128)), steps=1800,
                      scan_period=0.1, position=np.asarray(position, np.float64),
                      linear_velocity=np.array([5.0, 0.0, 0.0]))


def c4_camera(width: int = 1920, height: int = 1080) -> CameraModel:
    return CameraModel(kind="fisheye_equidistant", width=width, height=height, fx=600.0, fy=600.0,
                       cx=width / 2.0, cy=height / 2.0, distortion=(0.05, -0.01, 0.002, 0.0),
                       position=C2_POS.copy(), quaternion=look_at_quaternion(C2_POS, C2_TARGET),
                       readout_duration=0.03, linear_velocity=np.array([10.0, 0.0, 0.0]),
                       angular_velocity=np.array([0.0, 0.0, 0.2]))


def c5_rig():
    cams = [c2_camera(yaw) for yaw in range(0, 360, 45)]
    lidars = [c3_lidar(), c3_lidar(position=(-1.4863, 0.5187, 1.3))]
    return cams, lidars
