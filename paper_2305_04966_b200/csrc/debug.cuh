// debug.cuh — NACC_DEBUG device-precondition checks (debug.cu).  In release
// builds NACC_DEBUG_CHECK(...) compiles to nothing.
#pragma once
#include "common.cuh"

#ifndef NACC_DEBUG
#define NACC_DEBUG 0
#endif

#if NACC_DEBUG
namespace nacc {
nacc_status debug_check_rays(const float *rays_d, int64_t n, cudaStream_t stream);
nacc_status debug_check_sigma(const float *sigma, int64_t n, const char *name, cudaStream_t stream);
nacc_status debug_check_alpha(const float *alpha, int64_t n, cudaStream_t stream);
nacc_status debug_check_packed(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                               int64_t n_samples, cudaStream_t stream);
nacc_status debug_check_rows_ascending(const float *e, int64_t n_rows, int32_t m1, cudaStream_t stream);
}  // namespace nacc
#define NACC_DEBUG_CHECK(call)            \
  do {                                    \
    const nacc_status s_ = (call);        \
    if (s_ != NACC_OK) return s_;         \
  } while (0)
#else
#define NACC_DEBUG_CHECK(call) \
  do {                         \
  } while (0)
#endif
