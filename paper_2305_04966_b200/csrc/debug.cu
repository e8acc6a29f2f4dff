// debug.cu — the NACC_DEBUG build's device-precondition checks (SURVEY §8(b)
// "Validation and errors"): the release build validates host arguments only;
// libnacc_debug.so (built with -DNACC_DEBUG=1, loaded when NACC_DEBUG=1) also
// checks, before each entry point launches anything, the device preconditions
// the header states and synchronises:
//   * rays_d unit length, |‖d‖ − 1| < 1e-5 ("normalized directions";
//     S:41; reading #8: t is in units of ‖d‖);
//   * σ (and proposal σ) >= 0 and finite;
//   * packed intervals: every ray's [start, start + count) inside [0, n_samples),
//     t0 <= t1 per interval and t1_i <= t0_{i+1} within a ray (ascending,
//     non-overlapping);
//   * α in [0, 1] (alpha compositing, reading #16);
//   * resampling edges non-decreasing per ray (reading #13).
// A violation makes the call return NACC_ERR_INVALID_ARGUMENT with the first
// offending index in nacc_last_error() and launch nothing else.
#include <cstdio>

#include "common.cuh"
#include "debug.cuh"

#if NACC_DEBUG
namespace nacc {

namespace {
// first offending index (+1) per check; 0 = clean
__global__ void check_rays_kernel(const float *__restrict__ d, int64_t n, unsigned long long *bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = d[3 * i], y = d[3 * i + 1], z = d[3 * i + 2];
  const double nn = sqrt(x * x + y * y + z * z);
  if (!(fabs(nn - 1.0) < 1e-5)) atomicMin(bad, (unsigned long long)i + 1);
}

__global__ void check_nonneg_kernel(const float *__restrict__ v, int64_t n, unsigned long long *bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float s = v[i];
  if (!(s >= 0.0f) || isinf(s)) atomicMin(bad, (unsigned long long)i + 1);
}

__global__ void check_unit_interval_kernel(const float *__restrict__ v, int64_t n, unsigned long long *bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float a = v[i];
  if (!(a >= 0.0f && a <= 1.0f)) atomicMin(bad, (unsigned long long)i + 1);
}

// one thread per ray: its run lies inside the arrays and its intervals ascend without overlap
__global__ void check_packed_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                    const float *__restrict__ t0, const float *__restrict__ t1, int64_t n_samples,
                                    unsigned long long *bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const int64_t st = packed_info[2 * r], cnt = packed_info[2 * r + 1];
  if (st < 0 || cnt < 0 || st + cnt > n_samples) {
    atomicMin(bad, (unsigned long long)r + 1);
    return;
  }
  if (!t0 || !t1) return;
  for (int64_t i = 0; i < cnt; ++i) {
    const float a = t0[st + i], b = t1[st + i];
    if (!(a <= b) || (i + 1 < cnt && !(b <= t0[st + i + 1]))) {
      atomicMin(bad, (unsigned long long)r + 1);
      return;
    }
  }
}

// one thread per row: edges[r][0..m] non-decreasing
__global__ void check_rows_kernel(const float *__restrict__ e, int64_t n_rows, int32_t m1, unsigned long long *bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  for (int32_t j = 0; j + 1 < m1; ++j)
    if (!(e[r * m1 + j] <= e[r * m1 + j + 1])) {
      atomicMin(bad, (unsigned long long)r + 1);
      return;
    }
}

template <typename Launch>
nacc_status run_check(const char *what, cudaStream_t stream, Launch launch) {
  unsigned long long *bad = nullptr;
  if (cudaMallocAsync(&bad, sizeof(unsigned long long), stream) != cudaSuccess) {
    set_error(std::string("NACC_DEBUG: allocation failed checking ") + what);
    return NACC_ERR_CUDA;
  }
  const unsigned long long init = ~0ull;
  cudaMemcpyAsync(bad, &init, sizeof(init), cudaMemcpyHostToDevice, stream);
  launch(bad);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, stream);
  cudaFreeAsync(bad, stream);
  const cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    set_error(std::string("NACC_DEBUG: ") + cudaGetErrorString(e));
    return NACC_ERR_CUDA;
  }
  if (h != ~0ull) {
    char buf[160];
    snprintf(buf, sizeof(buf), "NACC_DEBUG: precondition violated: %s (first index %llu)", what, h - 1);
    set_error(buf);
    return NACC_ERR_INVALID_ARGUMENT;
  }
  return NACC_OK;
}

unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }
}  // namespace

nacc_status debug_check_rays(const float *rays_d, int64_t n, cudaStream_t stream) {
  if (n <= 0 || !rays_d) return NACC_OK;
  return run_check("rays_d must be unit length (|‖d‖ - 1| < 1e-5)", stream, [&](unsigned long long *bad) {
    check_rays_kernel<<<blocks_for(n), 256, 0, stream>>>(rays_d, n, bad);
  });
}

nacc_status debug_check_sigma(const float *sigma, int64_t n, const char *name, cudaStream_t stream) {
  if (n <= 0 || !sigma) return NACC_OK;
  return run_check(name, stream, [&](unsigned long long *bad) {
    check_nonneg_kernel<<<blocks_for(n), 256, 0, stream>>>(sigma, n, bad);
  });
}

nacc_status debug_check_alpha(const float *alpha, int64_t n, cudaStream_t stream) {
  if (n <= 0 || !alpha) return NACC_OK;
  return run_check("alphas must lie in [0, 1]", stream, [&](unsigned long long *bad) {
    check_unit_interval_kernel<<<blocks_for(n), 256, 0, stream>>>(alpha, n, bad);
  });
}

nacc_status debug_check_packed(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                               int64_t n_samples, cudaStream_t stream) {
  if (n_rays <= 0 || !packed_info) return NACC_OK;
  return run_check("packed samples: runs inside [0, n_samples), t0 <= t1, ascending non-overlapping per ray", stream,
                   [&](unsigned long long *bad) {
                     check_packed_kernel<<<blocks_for(n_rays), 256, 0, stream>>>(packed_info, n_rays, t0, t1,
                                                                                n_samples, bad);
                   });
}

nacc_status debug_check_rows_ascending(const float *e, int64_t n_rows, int32_t m1, cudaStream_t stream) {
  if (n_rows <= 0 || !e) return NACC_OK;
  return run_check("s_edges must be non-decreasing per ray", stream, [&](unsigned long long *bad) {
    check_rows_kernel<<<blocks_for(n_rows), 256, 0, stream>>>(e, n_rows, m1, bad);
  });
}

}  // namespace nacc
#endif  // NACC_DEBUG
