"""CPU oracle for the SaLF render hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package's render path
(`/root/reference/pkg/src/salf`, "the reference" below).  It exists to check
the CUDA path, never to serve it: only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s CPU-baseline leg may import it.  The product package
(`paper_2507_18713_b200`) never imports anything from here.

Parity pinning: every function below is checked against the reference itself
(imported in the build container) through golden vectors committed under
`tests/golden/` (generator: `tests/golden/make_golden.py`) and against the
reference test-suite's own known answers (octree dump table, SH constants,
brute-force march oracle, scalar composite oracle, finite differences) in
`tests/test_oracle.py`.

Floating-point operation order follows the reference's NumPy expressions
(including the summation orders NumPy's `einsum`/`matmul` use on x86) so that
the integer outputs -- tile CSR, sort order, ray/voxel hit lists -- are
bit-identical and the float outputs agree to ~1e-12.
"""

from __future__ import annotations

import numpy as np
from scipy.special import expit

# ---------------------------------------------------------------------------
# constants (reference: scene.py:28-35, render_ray.py:31-33, render_raster.py:29-34,
# octree.py:29-31)
SH_C0 = 0.2820947918
SH_C1 = 0.4886025119
ALPHA_MAX = 1.0 - 1e-12
STOP_THRESHOLD = 0.99
DEPTH_WEIGHT_MIN = 0.5
TILE_SIZE = 16
NEAR_PLANE = 0.05
EPS_ADVANCE = 1e-4
MIN_EDGE_FACTOR = 64
MAX_ROUNDS = 200_000
PINHOLE, FISHEYE, EQUIRECT = "pinhole", "fisheye_equidistant", "equirect"

# corner order: x fastest, then y, then z (render_raster.py:32-34)
CUBE_OFFSETS = np.array([[sx, sy, sz] for sz in (-0.5, 0.5) for sy in (-0.5, 0.5)
                         for sx in (-0.5, 0.5)])


# ---------------------------------------------------------------------------
# rotations (reference rotations.py:19-71)

def quat_to_matrix(q):
    """rotations.py:19-33."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    m = np.empty(q.shape[:-1] + (3, 3))
    m[..., 0, 0] = 1 - 2 * (y * y + z * z)
    m[..., 0, 1] = 2 * (x * y - w * z)
    m[..., 0, 2] = 2 * (x * z + w * y)
    m[..., 1, 0] = 2 * (x * y + w * z)
    m[..., 1, 1] = 1 - 2 * (x * x + z * z)
    m[..., 1, 2] = 2 * (y * z - w * x)
    m[..., 2, 0] = 2 * (x * z - w * y)
    m[..., 2, 1] = 2 * (y * z + w * x)
    m[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return m


def axis_angle_matrix(rotvec):
    """Rodrigues matrix, rotations.py:53-71 (I + sin K + (1 - cos) K K)."""
    rotvec = np.asarray(rotvec, dtype=np.float64)
    ang = np.linalg.norm(rotvec, axis=-1, keepdims=True)
    small = ang < 1e-12
    ax = rotvec / np.where(small, 1.0, ang)
    kx, ky, kz = ax[..., 0], ax[..., 1], ax[..., 2]
    zero = np.zeros_like(kx)
    k = np.stack([np.stack([zero, -kz, ky], -1),
                  np.stack([kz, zero, -kx], -1),
                  np.stack([-ky, kx, zero], -1)], -2)
    ang = ang[..., None]
    return np.broadcast_to(np.eye(3), k.shape) + np.sin(ang) * k + (1.0 - np.cos(ang)) * (k @ k)


# ---------------------------------------------------------------------------
# voxel geometry + local field (reference scene.py:57-58, 186-194, 229-284)

def level_edge(base_edge, level):
    return base_edge / np.exp2(np.asarray(level, dtype=np.float64))


def voxel_centers(aabb_min, base_edge, level, ijk):
    edge = level_edge(base_edge, level)
    return np.asarray(aabb_min, np.float64) + (np.asarray(ijk).astype(np.float64) + 0.5) * edge[..., None]


def eval_sdf(x, w_s):
    """scene.py:229-232  W_s . [x, 1]."""
    return np.einsum("...i,...i->...", w_s[..., :3], x) + w_s[..., 3]


def sdf_to_density(s, a, b):
    """scene.py:235-242  a/2 (1 + sign(s)(1 - exp(-|s|/b)))."""
    return 0.5 * a * (1.0 + np.sign(s) * (1.0 - np.exp(-np.abs(s) / b)))


def sh_basis(omega):
    """scene.py:256-267  (C0, C1 y, C1 z, C1 x); unit-norm check."""
    omega = np.asarray(omega, dtype=np.float64)
    if np.any(np.abs(np.linalg.norm(omega, axis=-1) - 1.0) > 1e-6):
        raise ValueError("view direction must be unit norm")
    g = np.empty(omega.shape[:-1] + (4,))
    g[..., 0] = SH_C0
    g[..., 1] = SH_C1 * omega[..., 1]
    g[..., 2] = SH_C1 * omega[..., 2]
    g[..., 3] = SH_C1 * omega[..., 0]
    return g


def eval_color(x, omega, w_c, w_sh):
    """scene.py:270-279  sigmoid(W_c x + W_sh gamma(omega))."""
    z = np.einsum("...ij,...j->...i", w_c, x) + np.einsum("...ij,...j->...i", w_sh, sh_basis(omega))
    return expit(z)


def segment_opacity(sigma, delta):
    """scene.py:282-284  min(1 - exp(-sigma delta), 1 - 1e-12)."""
    return np.minimum(-np.expm1(-np.asarray(sigma, np.float64) * delta), ALPHA_MAX)


def density(mode, s, log_a, log_b):
    if mode == "sdf":
        return sdf_to_density(s, np.exp(log_a), np.exp(log_b))
    return np.exp(s)


# ---------------------------------------------------------------------------
# a flat voxel set: the oracle's input type (plain arrays, static scenes only)

class Voxels:
    """Flat static voxel list: centers (M,3) f64, edges (M,), params (f64)."""

    def __init__(self, centers, edges, w_s, w_c, w_sh, log_a, log_b, mode="sdf",
                 level=None, ijk=None, aabb_min=None, base_edge=None, aabb_max=None):
        self.centers = np.asarray(centers, np.float64)
        self.edges = np.asarray(edges, np.float64)
        self.w_s = np.asarray(w_s, np.float64)
        self.w_c = np.asarray(w_c, np.float64)
        self.w_sh = np.asarray(w_sh, np.float64)
        self.log_a = np.asarray(log_a, np.float64)
        self.log_b = np.asarray(log_b, np.float64)
        self.mode = mode
        self.level, self.ijk = level, ijk
        self.aabb_min, self.aabb_max, self.base_edge = aabb_min, aabb_max, base_edge

    @property
    def n(self):
        return self.centers.shape[0]

    @classmethod
    def from_grid(cls, aabb_min, aabb_max, base_edge, level, ijk, w_s, w_c, w_sh, log_a,
                  log_b, mode="sdf"):
        level = np.asarray(level, np.uint8)
        ijk = np.asarray(ijk, np.int32).reshape(-1, 3)
        return cls(voxel_centers(aabb_min, base_edge, level, ijk), level_edge(base_edge, level),
                   w_s, w_c, w_sh, log_a, log_b, mode, level=level, ijk=ijk,
                   aabb_min=np.asarray(aabb_min, np.float64),
                   aabb_max=np.asarray(aabb_max, np.float64), base_edge=float(base_edge))


# ---------------------------------------------------------------------------
# sensors (reference sensors.py:101-232)

class Camera:
    def __init__(self, kind, width, height, fx=0.0, fy=0.0, cx=0.0, cy=0.0,
                 distortion=(0.0, 0.0, 0.0, 0.0), position=(0, 0, 0), quaternion=(1, 0, 0, 0),
                 readout_duration=0.0, linear_velocity=(0, 0, 0), angular_velocity=(0, 0, 0)):
        self.kind, self.width, self.height = kind, int(width), int(height)
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.distortion = tuple(float(k) for k in distortion)
        self.position = np.asarray(position, np.float64)
        self.quaternion = np.asarray(quaternion, np.float64)
        self.readout_duration = float(readout_duration)
        self.linear_velocity = np.asarray(linear_velocity, np.float64)
        self.angular_velocity = np.asarray(angular_velocity, np.float64)

    def rotation_matrix(self):
        return quat_to_matrix(self.quaternion)


class Lidar:
    def __init__(self, beam_elevations, azimuth_start=0.0, azimuth_end=2 * np.pi, steps=360,
                 scan_period=0.1, position=(0, 0, 0), quaternion=(1, 0, 0, 0),
                 linear_velocity=(0, 0, 0), angular_velocity=(0, 0, 0)):
        self.beam_elevations = np.atleast_1d(np.asarray(beam_elevations, np.float64))
        self.azimuth_start, self.azimuth_end = float(azimuth_start), float(azimuth_end)
        self.steps, self.scan_period = int(steps), float(scan_period)
        self.position = np.asarray(position, np.float64)
        self.quaternion = np.asarray(quaternion, np.float64)
        self.linear_velocity = np.asarray(linear_velocity, np.float64)
        self.angular_velocity = np.asarray(angular_velocity, np.float64)


def fisheye_forward(theta, k):
    t2 = theta * theta
    return theta * (1.0 + t2 * (k[0] + t2 * (k[1] + t2 * (k[2] + t2 * k[3]))))


def invert_fisheye(theta_d, k, theta_max=np.pi, iters=88):
    """sensors.py:106-121  bisection on [0, theta_max]."""
    valid = (theta_d >= 0) & (theta_d <= fisheye_forward(np.float64(theta_max), k))
    lo = np.zeros_like(theta_d)
    hi = np.full_like(theta_d, theta_max)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        up = fisheye_forward(mid, k) >= theta_d
        hi = np.where(up, mid, hi)
        lo = np.where(up, lo, mid)
    return 0.5 * (lo + hi), valid


def camera_rays(cam: Camera, t0=0.0):
    """gen_camera_rays + apply_rolling_shutter (sensors.py:129-190).

    Returns dict(origins, dirs, t_stamps, valid, shape)."""
    v, u = np.mgrid[0:cam.height, 0:cam.width].astype(np.float64)
    u = u.ravel() + 0.5
    v = v.ravel() + 0.5
    n = u.shape[0]
    valid = np.ones(n, dtype=bool)
    if cam.kind == PINHOLE:
        d = np.stack([(u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy, np.ones(n)], axis=1)
    elif cam.kind == FISHEYE:
        xn = (u - cam.cx) / cam.fx
        yn = (v - cam.cy) / cam.fy
        theta, valid = invert_fisheye(np.hypot(xn, yn), cam.distortion)
        phi = np.arctan2(yn, xn)
        st = np.sin(theta)
        d = np.stack([st * np.cos(phi), st * np.sin(phi), np.cos(theta)], axis=1)
    elif cam.kind == EQUIRECT:
        az = 2.0 * np.pi * (u - cam.width / 2.0) / cam.width
        el = -np.pi * (v - cam.height / 2.0) / cam.height
        d = np.stack([np.sin(az) * np.cos(el), -np.sin(el), np.cos(az) * np.cos(el)], axis=1)
    else:
        raise ValueError(f"unknown camera kind {cam.kind!r}")
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    dirs = d @ cam.rotation_matrix().T
    origins = np.broadcast_to(cam.position, (n, 3)).copy()
    t_stamps = np.full(n, float(t0))
    if cam.readout_duration > 0.0:
        rows = np.repeat(np.arange(cam.height), cam.width).astype(np.float64)
        frac = rows / (cam.height - 1) if cam.height > 1 else np.zeros_like(rows)
        dt = cam.readout_duration * frac
        origins = origins + dt[:, None] * cam.linear_velocity
        if np.any(cam.angular_velocity != 0.0):
            dirs = np.einsum("nij,nj->ni", axis_angle_matrix(dt[:, None] * cam.angular_velocity), dirs)
        t_stamps = t_stamps[0] + dt
    return dict(origins=origins, dirs=dirs, t_stamps=t_stamps, valid=valid,
                shape=(cam.height, cam.width))


def lidar_rays(lidar: Lidar, t0=0.0):
    """gen_lidar_rays (sensors.py:193-232): beam-major (beams, steps)."""
    nb, steps = lidar.beam_elevations.shape[0], lidar.steps
    j = np.arange(steps, dtype=np.float64)
    az = lidar.azimuth_start + (lidar.azimuth_end - lidar.azimuth_start) * j / steps
    dt = lidar.scan_period * j / steps
    el = lidar.beam_elevations[:, None]
    azg = az[None, :]
    d_s = np.stack([np.cos(el) * np.cos(azg), np.cos(el) * np.sin(azg),
                    np.broadcast_to(np.sin(el), (nb, steps))], axis=2).reshape(-1, 3)
    r0 = quat_to_matrix(lidar.quaternion)
    dtf = np.tile(dt, nb)
    if np.any(lidar.angular_velocity != 0.0):
        rm = np.einsum("nij,jk->nik", axis_angle_matrix(dtf[:, None] * lidar.angular_velocity), r0)
        dirs = np.einsum("nij,nj->ni", rm, d_s)
    else:
        dirs = d_s @ r0.T
    origins = lidar.position + dtf[:, None] * lidar.linear_velocity
    return dict(origins=origins, dirs=dirs, t_stamps=t0 + dtf, valid=np.ones(nb * steps, bool),
                shape=(nb, steps))


# ---------------------------------------------------------------------------
# slab test (reference octree.py:175-194)

def ray_box_range(o, d, bmin, bmax):
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        ta = (bmin - o) * inv
        tb = (bmax - o) * inv
    near = np.minimum(ta, tb)
    far = np.maximum(ta, tb)
    zero = d == 0.0
    inside = (o >= bmin) & (o <= bmax)
    near = np.where(zero, np.where(inside, -np.inf, np.inf), near)
    far = np.where(zero, np.where(inside, np.inf, -np.inf), far)
    return near.max(axis=-1), far.min(axis=-1)


# ---------------------------------------------------------------------------
# rasterizer (reference render_raster.py:97-301)

def project_voxels(vox: Voxels, cam: Camera, near=NEAR_PLANE):
    """render_raster.py:97-129 -> rect_min, rect_max (M,2), z_center, culled."""
    if cam.kind != PINHOLE:
        raise ValueError(f"rasterizer supports pinhole cameras only, got {cam.kind!r}")
    r = cam.rotation_matrix()
    corners = vox.centers[:, None, :] + CUBE_OFFSETS[None] * vox.edges[:, None, None]
    pc = (corners - cam.position) @ r
    z = pc[..., 2]
    zc = ((vox.centers - cam.position) @ r)[:, 2]
    culled = np.all(z <= near, axis=1)
    straddle = ~culled & np.any(z <= near, axis=1)
    front = z > near
    with np.errstate(divide="ignore", invalid="ignore"):
        u = np.where(front, cam.fx * pc[..., 0] / z + cam.cx, np.inf)
        v = np.where(front, cam.fy * pc[..., 1] / z + cam.cy, np.inf)
        umin, vmin = u.min(axis=1), v.min(axis=1)
        u = np.where(front, u, -np.inf)
        v = np.where(front, v, -np.inf)
        umax, vmax = u.max(axis=1), v.max(axis=1)
    rmin = np.stack([umin, vmin], 1)
    rmax = np.stack([umax, vmax], 1)
    rmin[straddle] = 0.0
    rmax[straddle] = (cam.width, cam.height)
    rmin[culled] = np.nan
    rmax[culled] = np.nan
    return rmin, rmax, zc, culled


def cull_and_bin(vox: Voxels, cam: Camera, tile=TILE_SIZE, near=NEAR_PLANE, window=None,
                 tiles=None, proj=None):
    """render_raster.py:143-182 -> (tiles_x, tiles_y, offsets int64[T+1], entries int64).

    `window=(tx0, ty0, tx1, ty1)` (inclusive tile rectangle) bins only those
    tiles; their lists are identical to the full binning's (tiles are
    independent), the others come out empty.  Used to time bounded samples.
    `tiles` (iterable of tile ids) does the same for an arbitrary tile set
    without expanding the other tiles' instances: each list is the visible
    voxels whose span covers the tile, ordered by lexsort((vid, z)) -- the
    reference's lexsort((vid, z, tile)) restricted to one tile.  `proj` reuses
    a project_voxels() result (same camera and near plane)."""
    rmin, rmax, zc, culled = project_voxels(vox, cam, near) if proj is None else proj
    tx_n = -(-cam.width // tile)
    ty_n = -(-cam.height // tile)
    nt = tx_n * ty_n
    with np.errstate(invalid="ignore"):
        u_lo = np.maximum(np.ceil(rmin[:, 0] - 0.5), 0)
        u_hi = np.minimum(np.floor(rmax[:, 0] - 0.5), cam.width - 1)
        v_lo = np.maximum(np.ceil(rmin[:, 1] - 0.5), 0)
        v_hi = np.minimum(np.floor(rmax[:, 1] - 0.5), cam.height - 1)
        vis = ~culled & (u_lo <= u_hi) & (v_lo <= v_hi)
    idx = np.flatnonzero(vis)
    if idx.size == 0:
        return tx_n, ty_n, np.zeros(nt + 1, np.int64), np.zeros(0, np.int64)
    x0 = (u_lo[idx] // tile).astype(np.int64)
    x1 = (u_hi[idx] // tile).astype(np.int64)
    y0 = (v_lo[idx] // tile).astype(np.int64)
    y1 = (v_hi[idx] // tile).astype(np.int64)
    if tiles is not None:
        counts = np.zeros(nt, np.int64)
        lists = []
        for t in sorted(set(int(t) for t in tiles)):
            ty, tx = divmod(t, tx_n)
            sel = idx[(x0 <= tx) & (tx <= x1) & (y0 <= ty) & (ty <= y1)]
            sel = sel[np.lexsort((sel, zc[sel]))]
            counts[t] = sel.size
            lists.append(sel)
        offsets = np.zeros(nt + 1, np.int64)
        np.cumsum(counts, out=offsets[1:])
        ent = np.concatenate(lists) if lists else np.zeros(0, np.int64)
        return tx_n, ty_n, offsets, ent.astype(np.int64)
    if window is not None:
        x0, y0 = np.maximum(x0, window[0]), np.maximum(y0, window[1])
        x1, y1 = np.minimum(x1, window[2]), np.minimum(y1, window[3])
        k = (x0 <= x1) & (y0 <= y1)
        idx, x0, x1, y0, y1 = idx[k], x0[k], x1[k], y0[k], y1[k]
        if idx.size == 0:
            return tx_n, ty_n, np.zeros(nt + 1, np.int64), np.zeros(0, np.int64)
    nx, ny = x1 - x0 + 1, y1 - y0 + 1
    cnt = nx * ny
    vid = np.repeat(idx, cnt)
    k = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    nxr = np.repeat(nx, cnt)
    tid = (np.repeat(y0, cnt) + k // nxr) * tx_n + np.repeat(x0, cnt) + k % nxr
    order = np.lexsort((vid, zc[vid], tid))
    offsets = np.zeros(nt + 1, np.int64)
    np.cumsum(np.bincount(tid[order], minlength=nt), out=offsets[1:])
    return tx_n, ty_n, offsets, vid[order]


def pixel_rays(cam: Camera, near=NEAR_PLANE):
    """(dirs, t_near) of every pixel (render_raster.py:212-215); reusable across calls (pix_rays=)."""
    return _pixel_rays(cam, near)


def _pixel_rays(cam: Camera, near):
    rays = camera_rays(Camera(cam.kind, cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy,
                              position=cam.position, quaternion=cam.quaternion))
    dirs = rays["dirs"]
    t_near = near / (dirs @ cam.rotation_matrix())[:, 2]
    return dirs, t_near


def _pair_segments(vox: Voxels, origin, dirs, t_near, pix, vid):
    """Per (pixel, voxel) pair: exact segment + fields (render_raster.py:185-253)."""
    with np.errstate(over="ignore", invalid="ignore"):
        o = origin[None, :] - vox.centers[vid]
        d = dirs[pix]
        half = 0.5 * vox.edges[vid]
        t_in, t_out = ray_box_range(o, d, -half[:, None], half[:, None])
        t0 = np.maximum(np.maximum(t_in, t_near[pix]), 0.0)
        hit = t_out > t0 + 1e-12
        delta = np.where(hit, t_out - t0, 0.0)
        t_mid = np.where(hit, 0.5 * (t0 + t_out), 0.0)
        x = (o + t_mid[:, None] * d) / (0.5 * vox.edges[vid])[:, None]
        s = eval_sdf(x, vox.w_s[vid])
        sigma = density(vox.mode, s, vox.log_a[vid], vox.log_b[vid])
        alpha = np.where(hit, segment_opacity(sigma, delta), 0.0)
        color = np.where(hit[:, None], eval_color(x, d, vox.w_c[vid], vox.w_sh[vid]), 0.0)
    return hit, t0, t_out, t_mid, x, s, sigma, alpha, color


def rasterize(vox: Voxels, cam: Camera, background=(0.0, 0.0, 0.0), tile=TILE_SIZE,
              near=NEAR_PLANE, stop_threshold=STOP_THRESHOLD, rows=None, window=None, tiles=None,
              proj=None, pix_rays=None):
    """render_raster.py:201-301, tile by tile.

    `rows=(r0, r1)` restricts work to tile rows r0..r1-1 and `window` to a
    tile rectangle (bounded CPU-baseline samples; other pixels keep zero
    accumulators)."""
    bg = np.asarray(background, np.float64)
    h, w = cam.height, cam.width
    if rows is not None and window is None:
        window = (0, rows[0], -(-w // tile) - 1, rows[1] - 1)
    tx_n, ty_n, offsets, entries = cull_and_bin(vox, cam, tile, near, window, tiles, proj)
    dirs, t_near = _pixel_rays(cam, near) if pix_rays is None else pix_rays
    keep = 1.0 - stop_threshold
    acc_c = np.zeros((h * w, 3))
    acc_l = np.zeros(h * w)
    acc_w = np.zeros(h * w)
    acc_t = np.zeros(h * w)
    for ty in range(ty_n):
        for tx in range(tx_n):
            t = ty * tx_n + tx
            ent = entries[offsets[t]:offsets[t + 1]]
            if ent.size == 0:
                continue
            rr = np.arange(ty * tile, min((ty + 1) * tile, h))
            cc = np.arange(tx * tile, min((tx + 1) * tile, w))
            px = (rr[:, None] * w + cc[None, :]).ravel()
            npx, ne = px.size, ent.size
            hit, t0, t1, tm, x, s, sig, alpha, color = _pair_segments(
                vox, cam.position, dirs, t_near, np.repeat(px, ne), np.tile(ent, npx))
            a = np.clip(alpha, 0.0, ALPHA_MAX).reshape(npx, ne)
            lg = np.log1p(-a)
            lt = np.cumsum(np.concatenate([np.zeros((npx, 1)), lg], axis=1), axis=1)
            tb = np.exp(lt[:, :-1])
            inc = tb > keep
            wgt = np.where(inc, tb * a, 0.0)
            acc_c[px] += np.cumsum(wgt[:, :, None] * color.reshape(npx, ne, 3), axis=1)[:, -1]
            acc_l[px] += np.cumsum(np.where(inc, lg, 0.0), axis=1)[:, -1]
            acc_w[px] += np.cumsum(wgt, axis=1)[:, -1]
            acc_t[px] += np.cumsum(wgt * tm.reshape(npx, ne), axis=1)[:, -1]
    t_fin = np.exp(acc_l)
    color = acc_c + t_fin[:, None] * bg
    with np.errstate(invalid="ignore", divide="ignore"):
        depth = np.where(acc_w > DEPTH_WEIGHT_MIN, acc_t / acc_w, np.nan)
    return dict(color=color.reshape(h, w, 3), opacity=(1.0 - t_fin).reshape(h, w),
                depth=depth.reshape(h, w), weight_sum=acc_w.reshape(h, w),
                t_final=t_fin.reshape(h, w))


def raster_records(vox: Voxels, cam: Camera, background=(0.0, 0.0, 0.0), tile=TILE_SIZE,
                   near=NEAR_PLANE, stop_threshold=STOP_THRESHOLD, window=None, tiles=None,
                   proj=None, pix_rays=None):
    """Raster pairs restated as ray-path records (one ray per pixel, row-major).

    The reference has no raster backward; its gradient is defined by
    composing reference functions: the hit pairs of each pixel in tile-list
    order (t0 = max(t_in, t_near, 0)), composited by `_composite`
    (render_ray.py:86-114) and differentiated by `backward_records`
    (backward.py:35-101).  Misses carry alpha = 0 and drop out exactly."""
    h, w = cam.height, cam.width
    tx_n, ty_n, offsets, entries = cull_and_bin(vox, cam, tile, near, window, tiles, proj)
    dirs, t_near = _pixel_rays(cam, near) if pix_rays is None else pix_rays
    chunks = []
    for t in range(tx_n * ty_n):
        ent = entries[offsets[t]:offsets[t + 1]]
        if ent.size == 0:
            continue
        ty, tx = divmod(t, tx_n)
        rr = np.arange(ty * tile, min((ty + 1) * tile, h))
        cc = np.arange(tx * tile, min((tx + 1) * tile, w))
        px = (rr[:, None] * w + cc[None, :]).ravel()
        pp, vv = np.repeat(px, ent.size), np.tile(ent, px.size)
        hit, t0, t1, tm, x, s, sig, alpha, color = _pair_segments(
            vox, cam.position, dirs, t_near, pp, vv)
        chunks.append((pp[hit], vv[hit], t0[hit], t1[hit], x[hit], s[hit], sig[hit],
                       alpha[hit], color[hit]))
    if chunks:
        cat = [np.concatenate([c[i] for c in chunks]) for i in range(9)]
        order = np.argsort(cat[0], kind="stable")  # by pixel, tile-list order within
        ray, vid, t0, t1, x, s, sig, alpha, color = [c[order] for c in cat]
    else:
        ray = vid = np.zeros(0, np.int64)
        t0 = t1 = s = sig = alpha = np.zeros(0)
        x = color = np.zeros((0, 3))
    omega = dirs[ray]
    return _make_records(h * w, ray, vid, t0, t1, x, omega, s, sig, alpha, color,
                         np.asarray(background, np.float64), stop_threshold, vox.mode)


# ---------------------------------------------------------------------------
# octree (reference octree.py:54-295)

class Octree:
    def __init__(self, nodes_id, nodes_leaf, root_min, root_edge, max_depth):
        self.nodes_id, self.nodes_leaf = nodes_id, nodes_leaf
        self.root_min, self.root_edge, self.max_depth = root_min, root_edge, max_depth

    @property
    def n_nodes(self):
        return self.nodes_id.shape[0]


def build_octree(vox: Voxels) -> Octree:
    """octree.py:54-125: DFS linear layout, children in blocks of 8.

    The node numbering follows the reference's LIFO stack (children pushed
    0..7, so octant 7 of the newest block is expanded first)."""
    ext = vox.aabb_max - vox.aabb_min
    m = max(0, int(np.ceil(np.log2(max(ext.max(), 1e-300) / vox.base_edge) - 1e-12)))
    root_edge = vox.base_edge * 2.0 ** m
    n = vox.n
    if n == 0:
        return Octree(np.array([-1], np.int64), np.array([-1], np.int8),
                      vox.aabb_min.copy(), root_edge, m)
    level = vox.level.astype(np.int64)
    cells = vox.ijk.astype(np.int64)
    depth = m + level
    if vox.edges.min() < MIN_EDGE_FACTOR * EPS_ADVANCE:
        raise ValueError(f"voxel edge {vox.edges.min():.3g} m below the marching floor "
                         f"{MIN_EDGE_FACTOR * EPS_ADVANCE:.3g} m")
    keys = (level << 54) ^ (cells[:, 0] << 36) ^ (cells[:, 1] << 18) ^ cells[:, 2]
    if len(np.unique(keys)) != n:
        raise ValueError("duplicate voxel cells in the set")
    if np.any(vox.centers < vox.aabb_min) or np.any(vox.centers > vox.aabb_max):
        raise ValueError("voxel outside scene bounds")
    ids = [-1]
    leaf = [-1]
    stack = [(0, 0, np.arange(n))]
    while stack:
        node, dep, sel = stack.pop()
        if sel.size == 0:
            continue  # stays (-1, -1)
        if np.any(depth[sel] == dep):
            if sel.size > 1:
                raise ValueError("stored voxel contains another stored voxel")
            ids[node], leaf[node] = int(sel[0]), 1
            continue
        off = len(ids)
        ids[node], leaf[node] = off, 0
        ids.extend([-1] * 8)
        leaf.extend([-1] * 8)
        sh = depth[sel] - dep - 1
        b = (cells[sel] >> sh[:, None]) & 1
        ch = b[:, 0] + 2 * b[:, 1] + 4 * b[:, 2]
        for c in range(8):
            stack.append((off + c, dep + 1, sel[ch == c]))
    return Octree(np.array(ids, np.int64), np.array(leaf, np.int8), vox.aabb_min.copy(),
                  root_edge, m + int(level.max()))


def dump_table(tree: Octree) -> str:
    """octree.py:128-133."""
    rows = ["index is_leaf id_or_offset"]
    rows += [f"{i} {int(tree.nodes_leaf[i])} {int(tree.nodes_id[i])}" for i in range(tree.n_nodes)]
    return "\n".join(rows) + "\n"


def query_batch(tree: Octree, p):
    """octree.py:136-166: root-to-leaf descent -> (flag, vid, corner, edge)."""
    p = np.atleast_2d(np.asarray(p, np.float64))
    u = (p - tree.root_min) / tree.root_edge
    if np.any(u < -1e-9) or np.any(u > 1.0 + 1e-9):
        raise ValueError("query point outside the octree root cube")
    u = np.clip(u, 0.0, 1.0)
    n = p.shape[0]
    node = np.zeros(n, np.int64)
    corner = np.broadcast_to(tree.root_min, (n, 3)).copy()
    edge = np.full(n, tree.root_edge)
    live = np.arange(n)
    while live.size:
        live = live[tree.nodes_leaf[node[live]] == 0]
        if live.size == 0:
            break
        bits = u[live] >= 0.5
        node[live] = tree.nodes_id[node[live]] + (bits[:, 0] + 2 * bits[:, 1] + 4 * bits[:, 2])
        edge[live] *= 0.5
        corner[live] += bits * edge[live, None]
        u[live] = 2.0 * u[live] - bits
    flag = tree.nodes_leaf[node]
    return flag, np.where(flag == 1, tree.nodes_id[node], -1), corner, edge


def march(tree: Octree, origins, dirs, t_max=np.inf, alpha_fn=None,
          stop_threshold=STOP_THRESHOLD):
    """Lockstep epsilon-marching (octree.py:214-295, render_ray.py:136-158).

    Returns (ray, vid, t0, t1) in per-ray march order.  When `alpha_fn` is
    given, a ray stops after the round in which the running product of
    (1 - alpha) of its segments drops to <= 1 - stop_threshold (the
    reference's early termination)."""
    o = np.atleast_2d(np.asarray(origins, np.float64))
    d = np.atleast_2d(np.asarray(dirs, np.float64))
    if np.any(np.abs(np.linalg.norm(d, axis=1) - 1.0) > 1e-6):
        raise ValueError("ray directions must be unit norm")
    n = o.shape[0]
    t_max = np.broadcast_to(np.asarray(t_max, np.float64), (n,)).copy()
    rmax = tree.root_min + tree.root_edge
    t_in, t_out = ray_box_range(o, d, tree.root_min, rmax)
    t_cur = np.maximum(t_in, 0.0)
    t_end = np.minimum(t_out, t_max)
    active = np.flatnonzero((t_out > t_cur) & (t_cur < t_max) & np.isfinite(t_cur))
    t_run = np.ones(n)
    out = []
    rounds = 0
    while active.size:
        rounds += 1
        if rounds > MAX_ROUNDS:
            raise RuntimeError("octree marching failed to terminate")
        idx = active
        p = o[idx] + t_cur[idx, None] * d[idx]
        flag, vid, corner, edge = query_batch(tree, p)
        _, far = ray_box_range(p, d[idx], corner, corner + edge[:, None])
        t_cur[idx] += np.maximum(far, 0.0) + EPS_ADVANCE
        h = flag == 1
        if np.any(h):
            hi = idx[h]
            a_in, a_out = ray_box_range(o[hi], d[hi], corner[h], corner[h] + edge[h, None])
            s0 = np.maximum(a_in, 0.0)
            s1 = np.minimum(a_out, t_max[hi])
            k = s1 > s0 + 1e-12
            seg = (hi[k], vid[h][k], s0[k], s1[k])
            if seg[0].size:
                out.append(seg)
        else:
            seg = None
        done = t_cur[idx] >= np.minimum(t_end[idx], t_max[idx])
        active = idx[~done]
        if alpha_fn is not None and seg is not None and seg[0].size:
            a = alpha_fn(*seg)
            t_run[seg[0]] *= 1.0 - np.clip(a, 0.0, ALPHA_MAX)
            sat = seg[0][t_run[seg[0]] <= 1.0 - stop_threshold]
            if sat.size:
                active = np.setdiff1d(active, sat)
    if not out:
        return (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), np.zeros(0))
    ray, vid, t0, t1 = (np.concatenate([s[i] for s in out]) for i in range(4))
    order = np.argsort(ray, kind="stable")
    return ray[order], vid[order], t0[order], t1[order]


def march_batch(tree: Octree, origins, dirs, t_max=np.inf):
    """octree.py:276-295: all segments, sorted by (ray, t0) with stable ties."""
    ray, vid, t0, t1 = march(tree, origins, dirs, t_max)
    order = np.lexsort((t0, ray))
    return ray[order], vid[order], t0[order], t1[order]


# ---------------------------------------------------------------------------
# ray integration (reference render_ray.py:86-239, static scenes)

def _geometry(vox: Voxels, o, d, ray, vid, t0, t1):
    """render_ray.py:117-133 (identity voxel rotation)."""
    tm = 0.5 * (t0 + t1)
    pts = o[ray] + tm[:, None] * d[ray]
    x = (pts - vox.centers[vid]) * (2.0 / vox.edges[vid][:, None])
    s = eval_sdf(x, vox.w_s[vid])
    sig = density(vox.mode, s, vox.log_a[vid], vox.log_b[vid])
    return x, d[ray], s, sig, segment_opacity(sig, t1 - t0)


def composite(ray, alpha, color, t_mid, n_rays, background, stop_threshold=STOP_THRESHOLD):
    """render_ray.py:86-114 (log-space prefix per ray, freeze at T <= 1 - stop)."""
    keep = 1.0 - stop_threshold
    a = np.clip(alpha, 0.0, ALPHA_MAX)
    s = np.log1p(-a)
    cs = np.cumsum(s)
    cnt = np.bincount(ray, minlength=n_rays)
    starts = np.concatenate([[0], np.cumsum(cnt)])
    base = np.repeat(np.concatenate([[0.0], cs])[starts[:-1]], cnt)
    tb = np.exp((cs - s) - base)
    inc = tb > keep
    w = np.where(inc, tb * a, 0.0)
    col = np.stack([np.bincount(ray, weights=w * color[:, c], minlength=n_rays)
                    for c in range(3)], 1).astype(np.float64)
    t_fin = np.exp(np.bincount(ray, weights=np.where(inc, s, 0.0), minlength=n_rays))
    col += t_fin[:, None] * background
    wsum = np.bincount(ray, weights=w, minlength=n_rays).astype(np.float64)
    dnum = np.bincount(ray, weights=w * t_mid, minlength=n_rays).astype(np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        depth = np.where(wsum > DEPTH_WEIGHT_MIN, dnum / wsum, np.nan)
    return tb, inc, col, 1.0 - t_fin, depth, wsum, t_fin, starts


def _make_records(n_rays, ray, vid, t0, t1, x, omega, s, sig, alpha, color, bg, stop, mode):
    tb, inc, col, op, depth, wsum, t_fin, starts = composite(
        ray, alpha, color, 0.5 * (t0 + t1), n_rays, bg, stop)
    return dict(n_rays=n_rays, ray=ray, vid=vid, t0=t0, t1=t1, x=x, omega=omega, s_field=s,
                sigma=sig, alpha=alpha, color=color, t_before=tb, included=inc,
                out_color=col, opacity=op, depth=depth, weight_sum=wsum, t_final=t_fin,
                background=bg, density_mode=mode, group_start=starts)


def integrate_rays(vox: Voxels, tree: Octree, origins, dirs, t_max=np.inf,
                   background=(0.0, 0.0, 0.0), stop_threshold=STOP_THRESHOLD):
    """render_ray.py:161-239 for a static scene (early stop enabled)."""
    o = np.atleast_2d(np.asarray(origins, np.float64))
    d = np.atleast_2d(np.asarray(dirs, np.float64))

    def alpha_fn(ray, vid, t0, t1):
        return _geometry(vox, o, d, ray, vid, t0, t1)[4]

    ray, vid, t0, t1 = march(tree, o, d, t_max, alpha_fn, stop_threshold)
    order = np.lexsort((vid, t0, ray))
    ray, vid, t0, t1 = ray[order], vid[order], t0[order], t1[order]
    if ray.size:
        x, omega, s, sig, alpha = _geometry(vox, o, d, ray, vid, t0, t1)
        color = eval_color(x, omega, vox.w_c[vid], vox.w_sh[vid])
    else:
        x = omega = color = np.zeros((0, 3))
        s = sig = alpha = np.zeros(0)
    return _make_records(o.shape[0], ray, vid, t0, t1, x, omega, s, sig, alpha, color,
                         np.asarray(background, np.float64), stop_threshold, vox.mode)


def render_lidar_ranges(vox, tree, rays):
    rec = integrate_rays(vox, tree, rays["origins"], rays["dirs"])
    return rec["depth"].reshape(rays["shape"])


def render_rays_image(vox, tree, rays, background=(0.0, 0.0, 0.0), stop_threshold=STOP_THRESHOLD):
    """render_ray.py:275-294: valid rays only, background elsewhere."""
    h, w = rays["shape"]
    color = np.zeros((h * w, 3))
    color[:] = np.asarray(background, np.float64)
    opacity = np.zeros(h * w)
    depth = np.full(h * w, np.nan)
    sel = np.flatnonzero(rays["valid"])
    rec = integrate_rays(vox, tree, rays["origins"][sel], rays["dirs"][sel],
                         background=background, stop_threshold=stop_threshold)
    color[sel], opacity[sel], depth[sel] = rec["out_color"], rec["opacity"], rec["depth"]
    return color.reshape(h, w, 3), opacity.reshape(h, w), depth.reshape(h, w)


# ---------------------------------------------------------------------------
# backward (reference backward.py:26-101, static owner) + L1 seeds (losses.py:22-46)

def backward_records(rec, vox: Voxels, d_color, d_depth, magnitude=False, x_floor=0.0):
    """Dense per-voxel gradients {w_s (M,4), w_c (M,3,3), w_sh (M,3,4), log_a, log_b}.

    `magnitude=True` (test-side conditioning, no reference counterpart) returns
    instead, per gradient element, the sum over segments of the ABSOLUTE values
    of the terms the reference adds (each product taken with |.| factors, the
    suffix sum of |A w|).  It is the scale against which any finite-precision
    evaluation of that sum is conditioned: an element that is a near-cancelling
    sum of large terms cannot be reproduced to 1e-4 of its own (small) value by
    any fp32 or reordered fp64 implementation, only to a fraction of this scale.
    `x_floor` adds the resolution of the quantities that cross zero inside a
    voxel: the local coordinates x (in [-1, 1]) count as |x| + x_floor and the
    SDF value s as |s| + x_floor |w_s|_1 (a chord entering and leaving through
    the two x faces has x_0 = 0 exactly; its fp64 value is rounding noise)."""
    if magnitude:
        return _backward_magnitude(rec, vox, d_color, d_depth, x_floor)
    m = vox.n
    g = dict(w_s=np.zeros((m, 4)), w_c=np.zeros((m, 3, 3)), w_sh=np.zeros((m, 3, 4)),
             log_a=np.zeros(m), log_b=np.zeros(m))
    ray = rec["ray"]
    if ray.size == 0:
        return g
    inc = rec["included"]
    a = np.clip(rec["alpha"], 0.0, ALPHA_MAX)
    tb = rec["t_before"]
    w = np.where(inc, tb * a, 0.0)
    tm = 0.5 * (rec["t0"] + rec["t1"])
    delta = rec["t1"] - rec["t0"]
    ok = rec["weight_sum"] > 0.5
    dd = np.where(ok, d_depth, 0.0)
    dep = np.where(ok, rec["depth"], 0.0)
    ws = np.where(ok, rec["weight_sum"], 1.0)
    A = np.einsum("nc,nc->n", d_color[ray], rec["color"]) + dd[ray] * (tm - dep[ray]) / ws[ray]
    tail = np.einsum("nc,c->n", d_color, rec["background"]) * rec["t_final"]
    vals = np.where(inc, A * w, 0.0)
    cs = np.cumsum(vals)
    gs = rec["group_start"]
    suffix = np.repeat(cs[np.maximum(gs[1:] - 1, 0)], np.diff(gs)) - cs
    g_alpha = np.where(inc, A * tb - (suffix + tail[ray]) / (1.0 - a), 0.0)
    g_sigma = g_alpha * delta * np.exp(-rec["sigma"] * delta)
    g_z = d_color[ray] * w[:, None] * rec["color"] * (1.0 - rec["color"])
    gamma = sh_basis(rec["omega"])
    xh = np.concatenate([rec["x"], np.ones((ray.size, 1))], axis=1)
    vid = rec["vid"]
    if rec["density_mode"] == "sdf":
        ap, bp = np.exp(vox.log_a[vid]), np.exp(vox.log_b[vid])
        s = rec["s_field"]
        e = np.exp(-np.abs(s) / bp)
        ds = np.where(s == 0.0, 0.0, g_sigma * (ap / (2.0 * bp)) * e)
        np.add.at(g["log_a"], vid, g_sigma * rec["sigma"])
        np.add.at(g["log_b"], vid, g_sigma * (-(ap / (2.0 * bp)) * s * e))
        np.add.at(g["w_s"], vid, ds[:, None] * xh)
    else:
        np.add.at(g["w_s"], vid, (g_sigma * rec["sigma"])[:, None] * xh)
    np.add.at(g["w_c"], vid, np.einsum("ni,nj->nij", g_z, rec["x"]))
    np.add.at(g["w_sh"], vid, np.einsum("ni,nj->nij", g_z, gamma))
    return g


def _backward_magnitude(rec, vox: Voxels, d_color, d_depth, x_floor=0.0):
    """backward_records(..., magnitude=True): the chain of backward.py:52-100
    with every factor replaced by its absolute value (x and s floored)."""
    m = vox.n
    g = dict(w_s=np.zeros((m, 4)), w_c=np.zeros((m, 3, 3)), w_sh=np.zeros((m, 3, 4)),
             log_a=np.zeros(m), log_b=np.zeros(m))
    ray = rec["ray"]
    if ray.size == 0:
        return g
    inc = rec["included"]
    a = np.clip(rec["alpha"], 0.0, ALPHA_MAX)
    tb = rec["t_before"]
    w = np.where(inc, tb * a, 0.0)
    tm = 0.5 * (rec["t0"] + rec["t1"])
    delta = rec["t1"] - rec["t0"]
    ok = rec["weight_sum"] > 0.5
    dd = np.abs(np.where(ok, d_depth, 0.0))
    dep = np.where(ok, rec["depth"], 0.0)
    ws = np.where(ok, rec["weight_sum"], 1.0)
    dc = np.abs(d_color)
    A = np.einsum("nc,nc->n", dc[ray], np.abs(rec["color"])) + dd[ray] * np.abs(tm - dep[ray]) / ws[ray]
    tail = np.einsum("nc,c->n", dc, np.abs(rec["background"])) * rec["t_final"]
    vals = np.where(inc, A * w, 0.0)
    cs = np.cumsum(vals)
    gs = rec["group_start"]
    suffix = np.abs(np.repeat(cs[np.maximum(gs[1:] - 1, 0)], np.diff(gs)) - cs)
    g_alpha = np.where(inc, A * tb + (suffix + tail[ray]) / (1.0 - a), 0.0)
    g_sigma = g_alpha * delta * np.exp(-rec["sigma"] * delta)
    g_z = dc[ray] * w[:, None] * np.abs(rec["color"] * (1.0 - rec["color"]))
    gamma = np.abs(sh_basis(rec["omega"]))
    xa = np.abs(rec["x"]) + x_floor
    xh = np.concatenate([xa, np.ones((ray.size, 1))], axis=1)
    vid = rec["vid"]
    if rec["density_mode"] == "sdf":
        ap, bp = np.exp(vox.log_a[vid]), np.exp(vox.log_b[vid])
        s = rec["s_field"]
        sa = np.abs(s) + x_floor * np.abs(vox.w_s[vid]).sum(axis=1)
        e = np.exp(-np.abs(s) / bp)
        ds = g_sigma * (ap / (2.0 * bp)) * e
        np.add.at(g["log_a"], vid, g_sigma * np.abs(rec["sigma"]))
        np.add.at(g["log_b"], vid, g_sigma * ((ap / (2.0 * bp)) * sa * e))
        np.add.at(g["w_s"], vid, ds[:, None] * xh)
    else:
        np.add.at(g["w_s"], vid, (g_sigma * np.abs(rec["sigma"]))[:, None] * xh)
    np.add.at(g["w_c"], vid, np.einsum("ni,nj->nij", g_z, xa))
    np.add.at(g["w_sh"], vid, np.einsum("ni,nj->nij", g_z, gamma))
    return g


def loss_color_seed(out_color, gt, mask):
    """losses.py:22-31: dL/dC = sign(C - gt) / (rays x 3)."""
    d = np.zeros_like(out_color)
    idx = np.flatnonzero(mask)
    if idx.size:
        diff = out_color[idx] - gt
        d[idx] = np.sign(diff) / diff.size
    return d


def loss_depth_seed(depth, gt, mask):
    """losses.py:34-46: dL/dD = sign(D - gt) / #valid."""
    d = np.zeros(depth.shape[0])
    idx = np.flatnonzero(mask)
    if idx.size == 0:
        return d
    ok = np.isfinite(depth[idx]) & np.isfinite(gt)
    idx = idx[ok]
    if idx.size:
        d[idx] = np.sign(depth[idx] - gt[ok]) / idx.size
    return d


# ---------------------------------------------------------------------------
# rest of the training step (reference optim.py:43-62, losses.py:49-249)

def adam_step(params, grads, m, v, step, lr=0.01, lr_decay=0.8, every=800, b1=0.9, b2=0.999,
              eps=1e-8):
    """optim.py:48-62 on dicts of arrays; `step` is the count before this update."""
    rate = lr * lr_decay ** (step // every)
    t = step + 1
    c1, c2 = 1.0 - b1 ** t, 1.0 - b2 ** t
    for k in params:
        m[k] = b1 * m[k] + (1.0 - b1) * grads[k]
        v[k] = b2 * v[k] + (1.0 - b2) * grads[k] * grads[k]
        params[k] -= rate * (m[k] / c1) / (np.sqrt(v[k] / c2) + eps)
    return rate


def loss_eikonal(vox: Voxels, idx):
    """losses.py:49-60."""
    g = np.zeros_like(vox.w_s)
    if idx.size == 0:
        return 0.0, g
    w = vox.w_s[idx, :3]
    nrm = np.linalg.norm(w, axis=1)
    ok = nrm > 1e-12
    gr = np.zeros_like(w)
    gr[ok] = (np.sign(nrm - 1.0) / idx.size)[ok, None] * (w[ok] / nrm[ok, None])
    np.add.at(g[:, :3], idx, gr)
    return float(np.abs(nrm - 1.0).mean()), g


def _density_grad_parts(vox, vid, s):
    a, b = np.exp(vox.log_a[vid]), np.exp(vox.log_b[vid])
    return a, b, sdf_to_density(s, a, b)


def loss_empty(vox: Voxels, outer):
    """losses.py:210-249 (lowest 20% centre opacities of outer voxels)."""
    g = dict(w_s=np.zeros_like(vox.w_s), log_a=np.zeros_like(vox.log_a), log_b=np.zeros_like(vox.log_b))
    if outer.size == 0:
        return 0.0, g
    s = vox.w_s[outer, 3]
    edge = vox.edges[outer]
    a, b, sig = _density_grad_parts(vox, outer, s)
    alpha = -np.expm1(-sig * edge)
    k = max(1, int(np.ceil(0.2 * outer.size)))
    order = np.argsort(alpha, kind="stable")[:k]
    sel = outer[order]
    g_sig = (1.0 / k) * edge[order] * np.exp(-sig[order] * edge[order])
    e = np.exp(-np.abs(s[order]) / b[order])
    k2 = a[order] / (2.0 * b[order])
    ds = np.where(s[order] == 0.0, 0.0, g_sig * k2 * e)
    np.add.at(g["w_s"], (sel, 3), ds)
    np.add.at(g["log_a"], sel, g_sig * sig[order])
    np.add.at(g["log_b"], sel, g_sig * (-k2 * s[order] * e))
    return float(alpha[order].mean()), g


def loss_opacity_lidar(vox: Voxels, tree: Octree, points, delta=0.2):
    """losses.py:188-226."""
    g = dict(w_s=np.zeros_like(vox.w_s), log_a=np.zeros_like(vox.log_a), log_b=np.zeros_like(vox.log_b))
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    rmax = tree.root_min + tree.root_edge
    pts = pts[np.all((pts >= tree.root_min) & (pts <= rmax), axis=1)]
    if pts.shape[0] == 0:
        return 0.0, g
    _f, vid, _c, _e = query_batch(tree, pts)
    keep = vid >= 0
    vid, pts = vid[keep], pts[keep]
    if vid.size == 0:
        return 0.0, g
    x = (pts - vox.centers[vid]) * (2.0 / vox.edges[vid][:, None])
    s = eval_sdf(x, vox.w_s[vid])
    a, b, sig = _density_grad_parts(vox, vid, s)
    alpha = -np.expm1(-sig * delta)
    n = vid.size
    g_sig = (-delta * np.exp(-sig * delta)) / n
    e = np.exp(-np.abs(s) / b)
    k2 = a / (2.0 * b)
    ds = np.where(s == 0.0, 0.0, g_sig * k2 * e)
    np.add.at(g["w_s"], vid, ds[:, None] * np.concatenate([x, np.ones((n, 1))], axis=1))
    np.add.at(g["log_a"], vid, g_sig * sig)
    np.add.at(g["log_b"], vid, g_sig * (-k2 * s * e))
    return float(np.mean(1.0 - alpha)), g


def feature_backward(rec, vox: Voxels, feat, dF, d_depth, magnitude=False, x_floor=0.0):
    """Reverse mode of a blended per-voxel feature F = sum_i w_i f_vid_i (the
    LiDAR intensity / ray-drop extension; no reference code):
    the same chain as backward_records (backward.py:52-100) with the colour
    replaced by f and no background term, plus the expected-depth term.
    Returns ({w_s, log_a, log_b}, feature grads (M, 8)).  `magnitude=True`:
    the conditioning scales instead (backward_records(..., magnitude=True))."""
    if magnitude:
        return _feature_magnitude(rec, vox, feat, dF, d_depth, x_floor)
    m = vox.n
    g = dict(w_s=np.zeros((m, 4)), log_a=np.zeros(m), log_b=np.zeros(m))
    fg = np.zeros((m, 8))
    ray = rec["ray"]
    if ray.size == 0:
        return g, fg
    inc = rec["included"]
    a = np.clip(rec["alpha"], 0.0, ALPHA_MAX)
    tb = rec["t_before"]
    w = np.where(inc, tb * a, 0.0)
    tm = 0.5 * (rec["t0"] + rec["t1"])
    delta = rec["t1"] - rec["t0"]
    ok = rec["weight_sum"] > 0.5
    dd = np.where(ok, d_depth, 0.0)
    dep = np.where(ok, rec["depth"], 0.0)
    ws = np.where(ok, rec["weight_sum"], 1.0)
    vid = rec["vid"]
    A = np.einsum("nc,nc->n", dF[ray], feat[vid]) + dd[ray] * (tm - dep[ray]) / ws[ray]
    vals = np.where(inc, A * w, 0.0)
    cs = np.cumsum(vals)
    gs = rec["group_start"]
    suffix = np.repeat(cs[np.maximum(gs[1:] - 1, 0)], np.diff(gs)) - cs
    g_alpha = np.where(inc, A * tb - suffix / (1.0 - a), 0.0)
    g_sigma = g_alpha * delta * np.exp(-rec["sigma"] * delta)
    xh = np.concatenate([rec["x"], np.ones((ray.size, 1))], axis=1)
    ap, bp = np.exp(vox.log_a[vid]), np.exp(vox.log_b[vid])
    s = rec["s_field"]
    e = np.exp(-np.abs(s) / bp)
    ds = np.where(s == 0.0, 0.0, g_sigma * (ap / (2.0 * bp)) * e)
    np.add.at(g["w_s"], vid, ds[:, None] * xh)
    np.add.at(g["log_a"], vid, g_sigma * rec["sigma"])
    np.add.at(g["log_b"], vid, g_sigma * (-(ap / (2.0 * bp)) * s * e))
    np.add.at(fg, vid, w[:, None] * dF[ray])
    return g, fg


def _feature_magnitude(rec, vox: Voxels, feat, dF, d_depth, x_floor=0.0):
    """feature_backward's chain with every factor replaced by its absolute value."""
    m = vox.n
    g = dict(w_s=np.zeros((m, 4)), log_a=np.zeros(m), log_b=np.zeros(m))
    fg = np.zeros((m, 8))
    ray = rec["ray"]
    if ray.size == 0:
        return g, fg
    inc = rec["included"]
    a = np.clip(rec["alpha"], 0.0, ALPHA_MAX)
    tb = rec["t_before"]
    w = np.where(inc, tb * a, 0.0)
    tm = 0.5 * (rec["t0"] + rec["t1"])
    delta = rec["t1"] - rec["t0"]
    ok = rec["weight_sum"] > 0.5
    dd = np.abs(np.where(ok, d_depth, 0.0))
    dep = np.where(ok, rec["depth"], 0.0)
    ws = np.where(ok, rec["weight_sum"], 1.0)
    vid = rec["vid"]
    adF = np.abs(dF)
    A = np.einsum("nc,nc->n", adF[ray], np.abs(feat[vid])) + dd[ray] * np.abs(tm - dep[ray]) / ws[ray]
    vals = np.where(inc, A * w, 0.0)
    cs = np.cumsum(vals)
    gs = rec["group_start"]
    suffix = np.abs(np.repeat(cs[np.maximum(gs[1:] - 1, 0)], np.diff(gs)) - cs)
    g_alpha = np.where(inc, A * tb + suffix / (1.0 - a), 0.0)
    g_sigma = g_alpha * delta * np.exp(-rec["sigma"] * delta)
    xh = np.concatenate([np.abs(rec["x"]) + x_floor, np.ones((ray.size, 1))], axis=1)
    ap, bp = np.exp(vox.log_a[vid]), np.exp(vox.log_b[vid])
    s = rec["s_field"]
    sa = np.abs(s) + x_floor * np.abs(vox.w_s[vid]).sum(axis=1)
    e = np.exp(-np.abs(s) / bp)
    ds = g_sigma * (ap / (2.0 * bp)) * e
    np.add.at(g["w_s"], vid, ds[:, None] * xh)
    np.add.at(g["log_a"], vid, g_sigma * np.abs(rec["sigma"]))
    np.add.at(g["log_b"], vid, g_sigma * ((ap / (2.0 * bp)) * sa * e))
    np.add.at(fg, vid, w[:, None] * adF[ray])
    return g, fg


# ---------------------------------------------------------------------------
# densify / prune round (reference densify.py:39-94, optim.py:35-40)

PRUNE_OPACITY = 0.005
SPLIT_DENOMINATOR = 8 * 5
CHILD_OFFSETS = np.array([[x, y, z] for z in (0, 1) for y in (0, 1) for x in (0, 1)], np.int64)


def center_opacity(w_s, log_a, log_b, edges, mode="sdf"):
    """densify.py:39-46: 1 - exp(-sigma(centre) edge), sigma from the bias w_s[3]."""
    s = np.asarray(w_s)[:, 3]
    sigma = sdf_to_density(s, np.exp(log_a), np.exp(log_b)) if mode == "sdf" else np.exp(s)
    return -np.expm1(-sigma * edges)


def densify_and_prune(level, ijk, params: dict, edges, grad_norms, budget, max_levels, mode="sdf",
                      prune_opacity=PRUNE_OPACITY):
    """densify.py:53-94.  Returns (new level, new ijk, new params, keep_idx, n_split).

    Prune = centre opacity < prune_opacity; split count
    max(0, (budget + n_prune - n) // 40); candidates ranked by gradient norm
    descending, ties by index (lexsort), finest-level voxels skipped; kept
    voxels first (index order), then 8 children per split voxel (split order
    ascending, child offsets x fastest) inheriting every parameter."""
    n = level.shape[0]
    opa = center_opacity(params["w_s"], params["log_a"], params["log_b"], edges, mode)
    prune = opa < prune_opacity
    n_prune = int(prune.sum())
    want = max(0, (budget + n_prune - n) // SPLIT_DENOMINATOR)
    eligible = ~prune & (level.astype(np.int64) < max_levels - 1)
    order = np.lexsort((np.arange(n), -np.asarray(grad_norms)))
    split_idx = np.sort(order[eligible[order]][:want])
    split = np.zeros(n, bool)
    split[split_idx] = True
    keep_idx = np.flatnonzero(~prune & ~split)
    child_level = np.repeat(level[split_idx].astype(np.int64) + 1, 8).astype(np.uint8)
    child_ijk = (ijk[split_idx].astype(np.int64)[:, None, :] * 2 + CHILD_OFFSETS[None]).reshape(-1, 3)
    new_level = np.concatenate([level[keep_idx], child_level])
    new_ijk = np.concatenate([ijk[keep_idx], child_ijk.astype(np.int32)])
    new_params = {k: np.concatenate([v[keep_idx], np.repeat(v[split_idx], 8, axis=0)])
                  for k, v in params.items()}
    if new_level.shape[0] > budget:
        raise RuntimeError(f"densification exceeded the budget: {new_level.shape[0]} > {budget}")
    return new_level, new_ijk, new_params, keep_idx, int(split_idx.size)


def adam_remap(moments: dict, keep_idx, n_split):
    """optim.py:35-40: kept voxels' moments carried over, children zeroed."""
    return {k: np.concatenate([v[keep_idx], np.zeros((8 * n_split,) + v.shape[1:], v.dtype)])
            for k, v in moments.items()}
