// filter.cu — §4.2 "No Gradient Filtering": samples whose entering
// transmittance is below ε are dropped before the differentiable pass.
// Per ray the kept set is a prefix (S_i never decreases; reading #9), so the
// filter is a per-ray cut (sequential fp64 sum, early exit) + exclusive scan of
// the cuts + a compacting copy of the prefixes.
#include "common.cuh"

namespace nacc {

// one thread per ray: walk the ray in order, accumulating S_i = Σ_{j<i} σ_j δ_j
// in fp64 exactly as the definition (σ_j δ_j is exact in fp64, so the sum is
// the sequential one), and stop at the first S_i > L.  Only the samples up to
// the cut are read (the kept prefix plus one), four loads in flight.
__global__ void __launch_bounds__(256) filter_cut_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                         const float *__restrict__ t0, const float *__restrict__ t1,
                                                         const float *__restrict__ sigma, double L,
                                                         int32_t *__restrict__ cut_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const longlong2 pi = __ldg(reinterpret_cast<const longlong2 *>(packed_info) + r);
  const int64_t st = pi.x, cnt = pi.y;
  double S = 0.0;
  int64_t cut = cnt;
  for (int64_t i = 0; i < cnt; i += 4) {
    float a[4], b[4], c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool in = i + j < cnt;
      a[j] = in ? __ldg(t0 + st + i + j) : 0.f;
      b[j] = in ? __ldg(t1 + st + i + j) : 0.f;
      c[j] = in ? __ldg(sigma + st + i + j) : 0.f;
    }
    bool done = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!done && i + j < cnt) {
        if (S > L) {
          cut = i + j;
          done = true;
        } else {
          S = __dadd_rn(S, __dmul_rn((double)c[j], __dsub_rn((double)b[j], (double)a[j])));
        }
      }
    }
    if (done) break;
  }
  cut_out[r] = (int32_t)cut;
}

// block of 256 consecutive rays: their kept prefixes are contiguous in the
// output; each thread copies output positions, locating its ray by binary
// search over the block's output starts (in shared memory)
constexpr int kCopyRays = 256;

__global__ void __launch_bounds__(kCopyRays) filter_copy_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                                const float *__restrict__ t0,
                                                                const float *__restrict__ t1,
                                                                const int64_t *__restrict__ packed_out,
                                                                const int64_t *__restrict__ total, int64_t capacity,
                                                                float *__restrict__ t0_out, float *__restrict__ t1_out,
                                                                int32_t *__restrict__ ray_id_out) {
  __shared__ int64_t s_out[kCopyRays + 1];
  __shared__ int64_t s_in[kCopyRays];
  if (*total > capacity) return;
  const int64_t r0 = (int64_t)blockIdx.x * kCopyRays;
  const int nr = (int)min((int64_t)kCopyRays, n_rays - r0);
  const int t = threadIdx.x;
  if (t < nr) {
    const longlong2 po = __ldg(reinterpret_cast<const longlong2 *>(packed_out) + r0 + t);
    s_out[t] = po.x;
    s_in[t] = __ldg(packed_info + 2 * (r0 + t));
    if (t == nr - 1) s_out[nr] = po.x + po.y;
  }
  __syncthreads();
  const int64_t p0 = s_out[0], p1 = s_out[nr];
  for (int64_t p = p0 + t; p < p1; p += kCopyRays) {
    int lo = 0, hi = nr - 1;  // largest k with s_out[k] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_out[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int64_t src = s_in[lo] + (p - s_out[lo]);
    t0_out[p] = __ldg(t0 + src);
    t1_out[p] = __ldg(t1 + src);
    ray_id_out[p] = (int32_t)(r0 + lo);
  }
}

static size_t filter_ws_layout(int64_t n, int32_t **cuts, void **scan_ws, void *base) {
  const size_t a = align_up((size_t)n * 4, 256);
  if (base) {
    *cuts = static_cast<int32_t *>(base);
    *scan_ws = static_cast<char *>(base) + a;
  }
  return a + scan_workspace_bytes(n);
}

}  // namespace nacc

using namespace nacc;

extern "C" {

size_t nacc_filter_workspace_bytes(int64_t n_rays) {
  if (n_rays < 0) return 0;
  return filter_ws_layout(n_rays, nullptr, nullptr, nullptr);
}

nacc_status nacc_filter_early_stop(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                                   const float *sigma, int64_t n_samples, double neg_log_eps,
                                   int64_t *packed_info_out, float *t0_out, float *t1_out, int32_t *ray_id_out,
                                   int64_t capacity, int64_t *total, void *ws, size_t ws_bytes,
                                   cudaStream_t stream) {
  clear_error();
  NACC_REQUIRE(n_rays >= 0 && n_rays < (1ll << 31), "n_rays must be in [0, 2^31)");
  NACC_REQUIRE(n_samples >= 0 && capacity >= 0, "n_samples and capacity must be >= 0");
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  NACC_REQUIRE(total, "total must be non-NULL");
  if (n_rays == 0) {
    NACC_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), stream));
    return NACC_OK;
  }
  NACC_REQUIRE(packed_info && packed_info_out && aligned(packed_info, 16) && aligned(packed_info_out, 16),
               "packed_info / packed_info_out must be non-NULL and 16-byte aligned");
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma), "t0, t1, sigma must be non-NULL");
  NACC_REQUIRE(capacity == 0 || (t0_out && t1_out && ray_id_out), "outputs must be non-NULL when capacity > 0");
  NACC_REQUIRE(ws && ws_bytes >= nacc_filter_workspace_bytes(n_rays), "workspace too small");
  int32_t *cuts;
  void *scan_ws;
  filter_ws_layout(n_rays, &cuts, &scan_ws, ws);
  filter_cut_kernel<<<grid_for(n_rays, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma, neg_log_eps, cuts);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  NACC_CUDA(scan_counts_to_packed(cuts, n_rays, packed_info_out, total, scan_ws, stream));
  if (capacity > 0) {
    filter_copy_kernel<<<grid_for(n_rays, kCopyRays), kCopyRays, 0, stream>>>(
        packed_info, n_rays, t0, t1, packed_info_out, total, capacity, t0_out, t1_out, ray_id_out);
    count_launch(1);
    NACC_CHECK_LAUNCH();
  }
  return NACC_OK;
}

}  // extern "C"
