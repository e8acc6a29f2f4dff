// filter.cu — §4.2 "No Gradient Filtering": samples whose entering
// transmittance is below ε are dropped before the differentiable pass.
// Per ray the kept set is a prefix (S_i never decreases; reading #9), so the
// filter is a per-ray cut (fp64 segmented scan) + exclusive scan + prefix copy.
#include "common.cuh"

namespace nacc {

// one warp per ray: cut[r] = min{i : S_i > L}, S_i = Σ_{j<i} σ_j (t1_j - t0_j) in fp64
__global__ void __launch_bounds__(256) filter_cut_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                         const float *__restrict__ t0, const float *__restrict__ t1,
                                                         const float *__restrict__ sigma, double L,
                                                         int32_t *__restrict__ cut_out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  double carry = 0.0;
  int64_t cut = cnt;
  for (int64_t base = 0; base < cnt; base += 32) {
    const int64_t i = base + lane;
    double s = 0.0;
    if (i < cnt) {
      const int64_t q = st + i;
      s = (double)__ldg(sigma + q) * ((double)__ldg(t1 + q) - (double)__ldg(t0 + q));
    }
    const double incl = warp_incl_scan(s);
    double excl = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) excl = 0.0;
    const double S = carry + excl;
    const unsigned b = __ballot_sync(kFull, (i < cnt) && (S > L));
    if (b) {
      cut = base + __ffs(b) - 1;
      break;
    }
    carry += __shfl_sync(kFull, incl, 31);
  }
  if (lane == 0) cut_out[r] = (int32_t)cut;
}

// one warp per ray: copy the kept prefix to its packed position
__global__ void __launch_bounds__(256) filter_copy_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                          const float *__restrict__ t0, const float *__restrict__ t1,
                                                          const int64_t *__restrict__ packed_out,
                                                          const int64_t *__restrict__ total, int64_t capacity,
                                                          float *__restrict__ t0_out, float *__restrict__ t1_out,
                                                          int32_t *__restrict__ ray_id_out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  if (*total > capacity) return;
  const int64_t src = packed_info[2 * r];
  const longlong2 po = reinterpret_cast<const longlong2 *>(packed_out)[r];
  for (int64_t i = lane; i < po.y; i += 32) {
    t0_out[po.x + i] = __ldg(t0 + src + i);
    t1_out[po.x + i] = __ldg(t1 + src + i);
    ray_id_out[po.x + i] = (int32_t)r;
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
  const int blocks = grid_for(n_rays * 32, 256);
  filter_cut_kernel<<<blocks, 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma, neg_log_eps, cuts);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  NACC_CUDA(scan_counts_to_packed(cuts, n_rays, packed_info_out, total, scan_ws, stream));
  if (capacity > 0) {
    filter_copy_kernel<<<blocks, 256, 0, stream>>>(packed_info, n_rays, t0, t1, packed_info_out, total, capacity,
                                                   t0_out, t1_out, ray_id_out);
    count_launch(1);
    NACC_CHECK_LAUNCH();
  }
  return NACC_OK;
}

}  // extern "C"
