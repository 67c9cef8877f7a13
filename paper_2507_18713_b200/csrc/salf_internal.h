// salf_internal.h -- host-side error plumbing shared by the C ABI entry points.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <exception>
#include <algorithm>

#include "../../include/salf_b200.h"

namespace salf {

// thread-local last-error message (salf_last_error)
char *error_buffer();

inline int set_error(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(error_buffer(), 1024, fmt, ap);
  va_end(ap);
  return code;
}

inline int check_cuda(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SALF_ECUDA, "%s: %s", where, cudaGetErrorString(e));
  return SALF_OK;
}

inline const char *camera_kind_repr(int kind) {
  switch (kind) {
    case SALF_PINHOLE: return "'pinhole'";
    case SALF_FISHEYE: return "'fisheye_equidistant'";
    case SALF_EQUIRECT: return "'equirect'";
    default: return "'unknown'";
  }
}

// Ordered (deterministic) reduction of per-row 27-vectors into the (M, 27)
// f64 gradient buffer (salf_raster.cu); row_vid == n_vox marks an unused row.
size_t det_reduce_workspace_bytes(int64_t n_rows, int64_t n_vox);
int det_reduce_rows(int64_t n_rows, const uint32_t *row_vid, const float *rows, int64_t n_vox, double *grad,
                    void *workspace, size_t workspace_bytes, cudaStream_t st);

}  // namespace salf

#define SALF_TRY try
#define SALF_CATCH                                                                  \
  catch (const std::exception &ex) {                                                \
    return salf::set_error(SALF_ECUDA, "internal error: %s", ex.what());            \
  }                                                                                 \
  catch (...) {                                                                     \
    return salf::set_error(SALF_ECUDA, "internal error");                           \
  }
