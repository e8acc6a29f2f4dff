// pdfloss.cu — proposal supervision: the PDF-matching (histogram-bound) loss
// that trains the proposal estimator (the paper names Mip-NeRF 360's "PDF
// matching loss"; form [ext], reading #21).  Dense per-ray
// histograms; one warp per ray, the proposal histogram staged in shared
// memory with its fp64 prefix sums.
//   forward : B_i = C[hi_i] − C[lo_i], C_j = Σ_{k<j} ŵ_k, lo_i = #{j : t̂_{j+1} <= t_i},
//             hi_i = #{j : t̂_j < t_{i+1}};  loss = Σ_i max(0, w_i − B_i)² / (w_i + ε)
//   backward: a_i = −2 g max(0, w_i − B_i)/(w_i + ε); the final intervals that
//             overlap proposal bin j form the contiguous range [i_lo(j), i_hi(j))
//             (edges ascending), so g_ŵ_j = A[i_hi(j)] − A[i_lo(j)] with A the
//             fp64 prefix sums of a — no atomics, deterministic.
#include "common.cuh"

namespace nacc {

constexpr int kPdfWarps = 4;

// first index k in [0, n) with a[k] > v (a ascending)
__device__ __forceinline__ int upper_bound_f(const float *a, int n, float v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] > v) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}
// first index k in [0, n) with a[k] >= v
__device__ __forceinline__ int lower_bound_f(const float *a, int n, float v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] >= v) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// exclusive fp64 prefix sums of v[0..n) into P[0..n] by one warp
__device__ __forceinline__ void warp_prefix(const float *v, int n, double *P, bool from_global) {
  const int lane = threadIdx.x & 31;
  double carry = 0.0;
  for (int base = 0; base < n; base += 32) {
    const int j = base + lane;
    const double x = j < n ? (double)(from_global ? __ldg(v + j) : v[j]) : 0.0;
    const double incl = warp_incl_scan(x);
    if (j < n) P[j + 1] = carry + incl;
    carry += __shfl_sync(kFull, incl, 31);
  }
  if (lane == 0) P[0] = 0.0;
  __syncwarp();
}

__device__ __forceinline__ double pdf_residual(const float *th, const double *C, int np, float a, float b, float w) {
  const int lo = upper_bound_f(th + 1, np, a);  // #{j : t̂_{j+1} <= a}
  const int hi = lower_bound_f(th, np, b);      // #{j : t̂_j < b}
  const double B = hi > lo ? C[hi] - C[lo] : 0.0;
  return (double)w - B;
}

__global__ void __launch_bounds__(kPdfWarps * 32) pdf_loss_kernel(int64_t n_rays, int nf, const float *__restrict__ t,
                                                                   const float *__restrict__ w, int np,
                                                                   const float *__restrict__ th,
                                                                   const float *__restrict__ wh, double eps,
                                                                   float *__restrict__ loss) {
  extern __shared__ double sm_d[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * kPdfWarps + warp;
  if (r >= n_rays) return;
  double *C = sm_d + (size_t)warp * (np + 1);
  float *e = reinterpret_cast<float *>(sm_d + (size_t)kPdfWarps * (np + 1)) + (size_t)warp * (np + 1);
  for (int j = lane; j <= np; j += 32) e[j] = __ldg(th + r * (int64_t)(np + 1) + j);
  warp_prefix(wh + r * (int64_t)np, np, C, true);
  const float *tr = t + r * (int64_t)(nf + 1);
  const float *wr = w + r * (int64_t)nf;
  double acc = 0.0;
  for (int i = lane; i < nf; i += 32) {
    const float wi = __ldg(wr + i);
    const double res = pdf_residual(e, C, np, __ldg(tr + i), __ldg(tr + i + 1), wi);
    if (res > 0.0) acc += res * res / ((double)wi + eps);
  }
  acc = warp_sum(acc);
  if (lane == 0) loss[r] = (float)acc;
}

__global__ void __launch_bounds__(kPdfWarps * 32) pdf_loss_bwd_kernel(
    int64_t n_rays, int nf, const float *__restrict__ t, const float *__restrict__ w, int np,
    const float *__restrict__ th, const float *__restrict__ wh, double eps, const float *__restrict__ g_loss,
    float *__restrict__ g_wh) {
  extern __shared__ double sm_d[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * kPdfWarps + warp;
  if (r >= n_rays) return;
  const int mx = max(nf, np);
  double *C = sm_d + (size_t)warp * 2 * (mx + 1);  // proposal prefix sums, then A (final-interval prefix)
  double *A = C + (mx + 1);
  float *e = reinterpret_cast<float *>(sm_d + (size_t)kPdfWarps * 2 * (mx + 1)) + (size_t)warp * (nf + np + 2);
  float *tf = e + (np + 1);
  for (int j = lane; j <= np; j += 32) e[j] = __ldg(th + r * (int64_t)(np + 1) + j);
  for (int i = lane; i <= nf; i += 32) tf[i] = __ldg(t + r * (int64_t)(nf + 1) + i);
  warp_prefix(wh + r * (int64_t)np, np, C, true);
  const float *wr = w + r * (int64_t)nf;
  const double g = (double)__ldg(g_loss + r);
  double carry = 0.0;
  for (int base = 0; base < nf; base += 32) {
    const int i = base + lane;
    double a = 0.0;
    if (i < nf) {
      const float wi = __ldg(wr + i);
      const double res = pdf_residual(e, C, np, tf[i], tf[i + 1], wi);
      if (res > 0.0) a = -2.0 * g * res / ((double)wi + eps);
    }
    const double incl = warp_incl_scan(a);
    if (i < nf) A[i + 1] = carry + incl;
    carry += __shfl_sync(kFull, incl, 31);
  }
  if (lane == 0) A[0] = 0.0;
  __syncwarp();
  float *gr = g_wh + r * (int64_t)np;
  for (int j = lane; j < np; j += 32) {
    // final intervals overlapping (t̂_j, t̂_{j+1}): t_{i+1} > t̂_j and t_i < t̂_{j+1}
    const int i_lo = upper_bound_f(tf + 1, nf, e[j]);   // first i with t_{i+1} > t̂_j
    const int i_hi = lower_bound_f(tf, nf, e[j + 1]);   // first i with t_i >= t̂_{j+1}
    gr[j] = i_hi > i_lo ? (float)(A[i_hi] - A[i_lo]) : 0.f;
  }
}

static nacc_status check_pdf(int64_t n_rays, int32_t nf, int32_t np, double eps) {
  NACC_REQUIRE(n_rays >= 0, "n_rays must be >= 0");
  NACC_REQUIRE(nf >= 1 && np >= 1, "nf and np must be >= 1");
  NACC_REQUIRE(std::isfinite(eps) && eps > 0.0, "eps must be > 0");
  return NACC_OK;
}

}  // namespace nacc

using namespace nacc;

extern "C" {

nacc_status nacc_pdf_loss(int64_t n_rays, int32_t nf, const float *t, const float *w, int32_t np, const float *th,
                          const float *wh, double eps, float *loss, cudaStream_t stream) {
  clear_error();
  nacc_status st = check_pdf(n_rays, nf, np, eps);
  if (st != NACC_OK) return st;
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(t && w && th && wh && loss, "t, w, th, wh, loss must be non-NULL");
  const size_t smem = (size_t)kPdfWarps * (np + 1) * (8 + 4);
  if (smem > 227 * 1024) {
    set_error("nacc_pdf_loss: np too large for shared memory");
    return NACC_ERR_UNSUPPORTED;
  }
  if (smem > 48 * 1024)
    NACC_CUDA(cudaFuncSetAttribute(pdf_loss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  pdf_loss_kernel<<<grid_for(n_rays, kPdfWarps), kPdfWarps * 32, smem, stream>>>(n_rays, nf, t, w, np, th, wh, eps,
                                                                                 loss);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_pdf_loss_bwd(int64_t n_rays, int32_t nf, const float *t, const float *w, int32_t np,
                              const float *th, const float *wh, double eps, const float *g_loss, float *g_wh,
                              cudaStream_t stream) {
  clear_error();
  nacc_status st = check_pdf(n_rays, nf, np, eps);
  if (st != NACC_OK) return st;
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(t && w && th && wh && g_loss && g_wh, "t, w, th, wh, g_loss, g_wh must be non-NULL");
  const int mx = nf > np ? nf : np;
  const size_t smem = (size_t)kPdfWarps * (2 * (mx + 1) * 8 + (nf + np + 2) * 4);
  if (smem > 227 * 1024) {
    set_error("nacc_pdf_loss_bwd: nf/np too large for shared memory");
    return NACC_ERR_UNSUPPORTED;
  }
  if (smem > 48 * 1024)
    NACC_CUDA(cudaFuncSetAttribute(pdf_loss_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  pdf_loss_bwd_kernel<<<grid_for(n_rays, kPdfWarps), kPdfWarps * 32, smem, stream>>>(n_rays, nf, t, w, np, th, wh,
                                                                                     eps, g_loss, g_wh);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

}  // extern "C"
