// salf_sensors.cu -- ray generation (reference sensors.py:101-232, rotations.py:53-71).
// fp64 throughout; one thread per ray.  Transcendentals (sin/cos/atan2/hypot)
// are CUDA's (<= 1-2 ulp from NumPy's), so rays agree with the reference to
// ~1e-16 relative; hit-list parity tests feed identical rays to both sides.
#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {

struct CamDev {
  salf_camera_t c;
  bool spin;  // any angular velocity component non-zero
};

__device__ __forceinline__ double fisheye_fwd(double th, const double *k) {
  const double t2 = __dmul_rn(th, th);
  return __dmul_rn(th, __dadd_rn(1.0, __dmul_rn(t2, __dadd_rn(k[0], __dmul_rn(t2, __dadd_rn(k[1],
                                __dmul_rn(t2, __dadd_rn(k[2], __dmul_rn(t2, k[3])))))))));
}

// axis_angle_matrix (rotations.py:53-71): I + sin(a) K + (1 - cos a) K K.
__device__ __forceinline__ void rodrigues(const double rv[3], double R[9]) {
  const double ang = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(rv[0], rv[0]), __dmul_rn(rv[1], rv[1])), __dmul_rn(rv[2], rv[2])));
  const double den = ang < 1e-12 ? 1.0 : ang;
  const double ax = __ddiv_rn(rv[0], den), ay = __ddiv_rn(rv[1], den), az = __ddiv_rn(rv[2], den);
  const double K[9] = {0.0, -az, ay, az, 0.0, -ax, -ay, ax, 0.0};
  const double s = sin(ang), c1 = __dsub_rn(1.0, cos(ang));
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double kk = __dadd_rn(__dadd_rn(__dmul_rn(K[3 * i], K[j]), __dmul_rn(K[3 * i + 1], K[3 + j])),
                                  __dmul_rn(K[3 * i + 2], K[6 + j]));
      R[3 * i + j] = __dadd_rn(__dadd_rn(i == j ? 1.0 : 0.0, __dmul_rn(s, K[3 * i + j])), __dmul_rn(c1, kk));
    }
}

// einsum("nij,nj->ni") in NumPy's order (p0 + p2) + p1.
__device__ __forceinline__ void matvec_es(const double R[9], const double v[3], double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    out[i] = __dadd_rn(__dadd_rn(__dmul_rn(R[3 * i], v[0]), __dmul_rn(R[3 * i + 2], v[2])), __dmul_rn(R[3 * i + 1], v[1]));
}

__global__ void k_camera_rays(CamDev cd, double *__restrict__ origins, double *__restrict__ dirs,
                              double *__restrict__ tst, uint8_t *__restrict__ valid, int64_t *__restrict__ keys) {
  const salf_camera_t &c = cd.c;
  const int64_t n = (int64_t)c.width * c.height;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int row = (int)(i / c.width), col = (int)(i % c.width);
  const double u = (double)col + 0.5, v = (double)row + 0.5;
  double d[3];
  bool ok = true;
  if (c.kind == SALF_PINHOLE) {
    d[0] = __ddiv_rn(__dsub_rn(u, c.cx), c.fx);
    d[1] = __ddiv_rn(__dsub_rn(v, c.cy), c.fy);
    d[2] = 1.0;
  } else if (c.kind == SALF_FISHEYE) {
    const double xn = __ddiv_rn(__dsub_rn(u, c.cx), c.fx), yn = __ddiv_rn(__dsub_rn(v, c.cy), c.fy);
    const double td = hypot(xn, yn), phi = atan2(yn, xn);
    ok = (td >= 0.0) && (td <= fisheye_fwd(M_PI, c.k));
    double lo = 0.0, hi = M_PI;
    for (int it = 0; it < 88; ++it) {  // invert_fisheye bisection (sensors.py:106-121)
      const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
      if (fisheye_fwd(mid, c.k) >= td) hi = mid; else lo = mid;
    }
    const double th = __dmul_rn(0.5, __dadd_rn(lo, hi));
    const double st = sin(th);
    d[0] = __dmul_rn(st, cos(phi));
    d[1] = __dmul_rn(st, sin(phi));
    d[2] = cos(th);
  } else {
    const double az = __ddiv_rn(__dmul_rn(2.0 * M_PI, __dsub_rn(u, __ddiv_rn((double)c.width, 2.0))), (double)c.width);
    const double el = __ddiv_rn(__dmul_rn(-M_PI, __dsub_rn(v, __ddiv_rn((double)c.height, 2.0))), (double)c.height);
    d[0] = __dmul_rn(sin(az), cos(el));
    d[1] = -sin(el);
    d[2] = __dmul_rn(cos(az), cos(el));
  }
  const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
  for (int k = 0; k < 3; ++k) d[k] = __ddiv_rn(d[k], nrm);
  double w[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) w[k] = mm_row(d, c.rot, k);  // d_cam @ R.T
  double o[3] = {c.position[0], c.position[1], c.position[2]};
  double ts = c.t0;
  if (c.readout_duration > 0.0) {  // apply_rolling_shutter (sensors.py:164-182)
    const double frac = c.height > 1 ? __ddiv_rn((double)row, (double)(c.height - 1)) : 0.0;
    const double dt = __dmul_rn(c.readout_duration, frac);
#pragma unroll
    for (int k = 0; k < 3; ++k) o[k] = __dadd_rn(o[k], __dmul_rn(dt, c.linear_velocity[k]));
    if (cd.spin) {
      double rv[3], R[9], r[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) rv[k] = __dmul_rn(dt, c.angular_velocity[k]);
      rodrigues(rv, R);
      matvec_es(R, w, r);
      w[0] = r[0]; w[1] = r[1]; w[2] = r[2];
    }
    ts = __dadd_rn(c.t0, dt);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    origins[3 * i + k] = o[k];
    dirs[3 * i + k] = w[k];
  }
  if (tst) tst[i] = ts;
  if (valid) valid[i] = ok ? 1 : 0;
  if (keys) {  // RayBatch.keys = (row, col), sensors.py:157-160
    keys[2 * i] = row;
    keys[2 * i + 1] = col;
  }
}

__global__ void k_lidar_rays(salf_lidar_t l, bool spin, const double *__restrict__ elev, double *__restrict__ origins,
                             double *__restrict__ dirs, double *__restrict__ tst, int64_t *__restrict__ keys,
                             uint8_t *__restrict__ valid) {
  const int64_t n = (int64_t)l.n_beams * l.steps;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int beam = (int)(i / l.steps), j = (int)(i % l.steps);
  const double jd = (double)j;
  // az = a0 + (a1 - a0) * j / steps ; dt = period * j / steps (sensors.py:201-203)
  const double az = __dadd_rn(l.azimuth_start,
                              __ddiv_rn(__dmul_rn(__dsub_rn(l.azimuth_end, l.azimuth_start), jd), (double)l.steps));
  const double dt = __ddiv_rn(__dmul_rn(l.scan_period, jd), (double)l.steps);
  const double el = elev[beam];
  const double ds[3] = {__dmul_rn(cos(el), cos(az)), __dmul_rn(cos(el), sin(az)), sin(el)};
  double w[3];
  if (spin) {
    double rv[3], R[9], M[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) rv[k] = __dmul_rn(dt, l.angular_velocity[k]);
    rodrigues(rv, R);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        M[3 * a + b] = __dadd_rn(__dadd_rn(__dmul_rn(R[3 * a], l.rot[b]), __dmul_rn(R[3 * a + 2], l.rot[6 + b])),
                                 __dmul_rn(R[3 * a + 1], l.rot[3 + b]));
    matvec_es(M, ds, w);
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) w[k] = mm_row(ds, l.rot, k);  // d_sensor @ r0.T
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    origins[3 * i + k] = __dadd_rn(l.position[k], __dmul_rn(dt, l.linear_velocity[k]));
    dirs[3 * i + k] = w[k];
  }
  if (tst) tst[i] = __dadd_rn(l.t0, dt);
  if (keys) {  // RayBatch.keys = (beam, step), sensors.py:228-231
    keys[2 * i] = beam;
    keys[2 * i + 1] = j;
  }
  if (valid) valid[i] = 1;
}

}  // namespace salf

using namespace salf;

extern "C" int salf_camera_rays(const salf_camera_t *cam, double *origins, double *dirs, double *t_stamps,
                                uint8_t *valid, void *stream) {
  SALF_TRY {
    if (cam->width < 1 || cam->height < 1) return set_error(SALF_EINVAL, "image dimensions must be at least 1");
    if (cam->kind < 0 || cam->kind > 2) return set_error(SALF_EINVAL, "unknown camera kind %d", cam->kind);
    CamDev cd;
    cd.c = *cam;
    cd.spin = cam->angular_velocity[0] != 0.0 || cam->angular_velocity[1] != 0.0 || cam->angular_velocity[2] != 0.0;
    const int64_t n = (int64_t)cam->width * cam->height;
    k_camera_rays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(cd, origins, dirs, t_stamps, valid,
                                                                                  nullptr);
    return check_cuda("salf_camera_rays");
  }
  SALF_CATCH
}

extern "C" int salf_camera_batch(const salf_camera_t *cam, double *origins, double *dirs, double *t_stamps,
                                 uint8_t *valid, int64_t *keys, void *stream) {
  SALF_TRY {
    if (cam->width < 1 || cam->height < 1) return set_error(SALF_EINVAL, "image dimensions must be at least 1");
    if (cam->kind < 0 || cam->kind > 2) return set_error(SALF_EINVAL, "unknown camera kind %d", cam->kind);
    CamDev cd;
    cd.c = *cam;
    cd.spin = cam->angular_velocity[0] != 0.0 || cam->angular_velocity[1] != 0.0 || cam->angular_velocity[2] != 0.0;
    const int64_t n = (int64_t)cam->width * cam->height;
    k_camera_rays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(cd, origins, dirs, t_stamps, valid,
                                                                                  keys);
    return check_cuda("salf_camera_batch");
  }
  SALF_CATCH
}

extern "C" int salf_lidar_rays(const salf_lidar_t *lidar, const double *beam_elevations, double *origins, double *dirs,
                               double *t_stamps, void *stream) {
  SALF_TRY {
    if (lidar->steps < 1) return set_error(SALF_EINVAL, "steps must be at least 1");
    if (!(lidar->scan_period > 0)) return set_error(SALF_EINVAL, "scan_period must be positive");
    const bool spin = lidar->angular_velocity[0] != 0.0 || lidar->angular_velocity[1] != 0.0 ||
                      lidar->angular_velocity[2] != 0.0;
    const int64_t n = (int64_t)lidar->n_beams * lidar->steps;
    if (n == 0) return SALF_OK;
    k_lidar_rays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*lidar, spin, beam_elevations, origins,
                                                                                 dirs, t_stamps, nullptr, nullptr);
    return check_cuda("salf_lidar_rays");
  }
  SALF_CATCH
}

extern "C" int salf_lidar_batch(const salf_lidar_t *lidar, const double *beam_elevations, double *origins,
                                double *dirs, double *t_stamps, int64_t *keys, uint8_t *valid, void *stream) {
  SALF_TRY {
    if (lidar->steps < 1) return set_error(SALF_EINVAL, "steps must be at least 1");
    if (!(lidar->scan_period > 0)) return set_error(SALF_EINVAL, "scan_period must be positive");
    const bool spin = lidar->angular_velocity[0] != 0.0 || lidar->angular_velocity[1] != 0.0 ||
                      lidar->angular_velocity[2] != 0.0;
    const int64_t n = (int64_t)lidar->n_beams * lidar->steps;
    if (n == 0) return SALF_OK;
    k_lidar_rays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*lidar, spin, beam_elevations, origins,
                                                                                 dirs, t_stamps, keys, valid);
    return check_cuda("salf_lidar_batch");
  }
  SALF_CATCH
}
