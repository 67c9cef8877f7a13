// salf_bench.cu -- FP64 / FP32 peak probes for the ALU rooflines reported by
// bench.py (MEASURED_PEAKS.json only holds HBM and bf16 tensor peaks).
// Independent FMA chains, one launch per call.
#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {
__global__ void k_fp64_peak(double *out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1.0, a2 = a0 + 2.0, a3 = a0 + 3.0, a4 = a0 + 4.0, a5 = a0 + 5.0,
         a6 = a0 + 6.0, a7 = a0 + 7.0;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (r == 12345.0) out[blockIdx.x] = r;  // keep the chains alive
}
__global__ void k_fp32_peak(float *out, int iters, float seed) {
  float a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = seed + threadIdx.x + k;
  const float m = 0.9999f, c = 1e-4f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = __fmaf_rn(a[k], m, c);
  }
  float t = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) t += a[k];
  if (t == 12345.0f) out[blockIdx.x] = t;  // keep the chains alive
}
}  // namespace salf

using namespace salf;

// Launches grid x 256 threads, each 64 * iters DFMA (2 flops each).
extern "C" int salf_fp64_peak(double *scratch, int32_t grid, int32_t iters, void *stream) {
  SALF_TRY {
    k_fp64_peak<<<grid, 256, 0, (cudaStream_t)stream>>>(scratch, iters, 0.5);
    return check_cuda("salf_fp64_peak");
  }
  SALF_CATCH
}

// Launches grid x 256 threads, each 64 * iters FFMA (2 flops each).
extern "C" int salf_fp32_peak(float *scratch, int32_t grid, int32_t iters, void *stream) {
  SALF_TRY {
    k_fp32_peak<<<grid, 256, 0, (cudaStream_t)stream>>>(scratch, iters, 0.5f);
    return check_cuda("salf_fp32_peak");
  }
  SALF_CATCH
}
