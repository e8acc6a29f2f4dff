// occgrid.cu — the occupancy-grid estimator update 𝓕 (Eq. 4):
// EMA σ^k = γ σ^{k-1} + (1-γ) σ_query (reading #21) or max-decay
// (S:305), then binarisation σ̂ = 1[σ > τ] (τ or min(τ, mean), #22).
// The caller evaluates σ at the jittered cell points between
// nacc_occgrid_points and nacc_occgrid_update (and, on several GPUs,
// all-reduces the fresh values with MAX; reading #25).
#include "common.cuh"

namespace nacc {

struct LevelBoxes {
  int levels, res;
  double lo[8][3], hi[8][3];  // fp32 boxes widened to fp64
};

static LevelBoxes make_boxes(const nacc_grid &g) {
  LevelBoxes b{};
  b.levels = g.levels;
  b.res = g.res;
  for (int a = 0; a < 3; ++a) {
    const double lo0 = (double)g.roi[a], hi0 = (double)g.roi[3 + a];
    const double ctr = (lo0 + hi0) / 2.0, half = (hi0 - lo0) / 2.0;
    for (int l = 0; l < g.levels; ++l) {
      const double sc = std::ldexp(1.0, l);
      b.lo[l][a] = (double)(float)(ctr - half * sc);
      b.hi[l][a] = (double)(float)(ctr + half * sc);
    }
  }
  return b;
}

__global__ void __launch_bounds__(256) points_kernel(LevelBoxes b, uint32_t key0, uint32_t key1, uint32_t step,
                                                     int jitter, int64_t cell_begin, int64_t cell_count,
                                                     float *__restrict__ xyz) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cell_count) return;
  const int64_t R = b.res, R3 = R * R * R;
  const int64_t cell = cell_begin + q;
  const int l = (int)(cell / R3);
  const int64_t idx = cell - (int64_t)l * R3;
  const int64_t ijk[3] = {idx % R, (idx / R) % R, idx / (R * R)};
  double xi[3] = {0.5, 0.5, 0.5};
  if (jitter) {
    const u32x4 rnd = philox4x32_10(u32x4{(uint32_t)idx, step, (uint32_t)l, 2u}, key0, key1);
    xi[0] = u24(rnd.x);
    xi[1] = u24(rnd.y);
    xi[2] = u24(rnd.z);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double cw = __ddiv_rn(__dsub_rn(b.hi[l][a], b.lo[l][a]), (double)R);
    const double x = __dadd_rn(b.lo[l][a], __dmul_rn(__dadd_rn((double)ijk[a], xi[a]), cw));
    xyz[3 * q + a] = __double2float_rn(x);
  }
}

// dynamic scenes (reading #20): draw j of the per-cell timestamp
__global__ void __launch_bounds__(256) times_kernel(int R, uint32_t key0, uint32_t key1, uint32_t step, uint32_t draw,
                                                    int64_t cell_begin, int64_t cell_count, float *__restrict__ t) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cell_count) return;
  const int64_t R3 = (int64_t)R * R * R;
  const int64_t cell = cell_begin + q;
  const int l = (int)(cell / R3);
  const int64_t idx = cell - (int64_t)l * R3;
  const u32x4 rnd = philox4x32_10(u32x4{(uint32_t)idx, step, (uint32_t)l, 16u + draw}, key0, key1);
  t[q] = (float)u24(rnd.x);
}

// fresh = max(fresh, v): merge of time draws (and the shape of the cross-rank MAX)
__global__ void __launch_bounds__(256) max_merge_kernel(float *__restrict__ dst, const float *__restrict__ src,
                                                        int64_t n) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n && ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    float4 a = *reinterpret_cast<float4 *>(dst + i);
    const float4 b = __ldg(reinterpret_cast<const float4 *>(src + i));
    a.x = b.x > a.x ? b.x : a.x;
    a.y = b.y > a.y ? b.y : a.y;
    a.z = b.z > a.z ? b.z : a.z;
    a.w = b.w > a.w ? b.w : a.w;
    *reinterpret_cast<float4 *>(dst + i) = a;
  } else {
    for (int64_t j = i; j < i + 4 && j < n; ++j) {
      const float b = __ldg(src + j);
      if (b > dst[j]) dst[j] = b;
    }
  }
}

constexpr int kUpdThreads = 256;

// EMA / max-decay; optional direct binarisation (fixed τ); per-block fp64 sums
__global__ void __launch_bounds__(kUpdThreads) update_kernel(float *__restrict__ density, const float *__restrict__ fresh,
                                                             int64_t n, int rule, double gam, double one_m,
                                                             int write_bits, double tau, uint32_t *__restrict__ bits,
                                                             double *__restrict__ partial) {
  __shared__ double red[kUpdThreads / 32];
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float nd = 0.f;
  if (q < n) {
    const double prev = (double)density[q], v = (double)__ldg(fresh + q);
    const double a = __dmul_rn(gam, prev);
    double x;
    if (rule == NACC_UPDATE_EMA) x = __dadd_rn(a, __dmul_rn(one_m, v));
    else x = a > v ? a : v;
    nd = __double2float_rn(x);
    density[q] = nd;
  }
  if (write_bits) {
    const unsigned b = __ballot_sync(kFull, q < n && (double)nd > tau);
    if ((threadIdx.x & 31) == 0 && q < n) bits[q >> 5] = b;
  }
  double s = warp_sum((double)nd);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < kUpdThreads / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) mean_kernel(const double *__restrict__ partial, int64_t nb, int64_t n,
                                                    double *__restrict__ mean_out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = red[threadIdx.x];
    t = warp_sum(t);
    if (threadIdx.x == 0) *mean_out = n > 0 ? t / (double)n : 0.0;
  }
}

__global__ void __launch_bounds__(256) binarize_kernel(const float *__restrict__ density, int64_t n, double tau,
                                                       const double *__restrict__ mean, uint32_t *__restrict__ bits) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double t = mean ? fmin(tau, *mean) : tau;
  const unsigned b = __ballot_sync(kFull, q < n && (double)density[q] > t);
  if ((threadIdx.x & 31) == 0 && q < n) bits[q >> 5] = b;
}

static nacc_status check_grid(const nacc_grid *grid) {
  NACC_REQUIRE(grid, "grid must be non-NULL");
  NACC_REQUIRE(grid->levels >= 1 && grid->levels <= 8, "levels must be in 1..8");
  NACC_REQUIRE(grid->res >= 1, "res must be >= 1");
  NACC_REQUIRE((int64_t)grid->levels * grid->res * grid->res * grid->res < (1ll << 31), "levels*res^3 must be < 2^31");
  for (int a = 0; a < 3; ++a)
    NACC_REQUIRE(std::isfinite(grid->roi[a]) && std::isfinite(grid->roi[3 + a]) && grid->roi[a] < grid->roi[3 + a],
                 "roi must be finite with lo < hi");
  return NACC_OK;
}

}  // namespace nacc

using namespace nacc;

extern "C" {

nacc_status nacc_occgrid_points(const nacc_grid *grid, uint64_t seed, int64_t step, int32_t jitter,
                                int64_t cell_begin, int64_t cell_count, float *xyz, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_grid(grid);
  if (s != NACC_OK) return s;
  const int64_t n = (int64_t)grid->levels * grid->res * grid->res * grid->res;
  NACC_REQUIRE(cell_begin >= 0 && cell_count >= 0 && cell_begin + cell_count <= n, "cell range out of bounds");
  if (cell_count == 0) return NACC_OK;
  NACC_REQUIRE(xyz && aligned(xyz, 4), "xyz must be non-NULL");
  points_kernel<<<grid_for(cell_count, 256), 256, 0, stream>>>(make_boxes(*grid), (uint32_t)(seed & 0xffffffffu),
                                                                (uint32_t)(seed >> 32), (uint32_t)step, jitter,
                                                                cell_begin, cell_count, xyz);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

size_t nacc_occgrid_workspace_bytes(const nacc_grid *grid) {
  if (!grid || grid->levels < 1 || grid->res < 1) return 0;
  const int64_t n = (int64_t)grid->levels * grid->res * grid->res * grid->res;
  return align_up((size_t)ceil_div(n, kUpdThreads) * 8, 256) + 256;
}

nacc_status nacc_occgrid_update(const nacc_grid *grid, float *density, const float *fresh, nacc_update_rule rule,
                                float decay, float threshold, nacc_thresh_rule thresh_rule, uint32_t *bits,
                                double *mean, void *ws, size_t ws_bytes, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_grid(grid);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(rule == NACC_UPDATE_EMA || rule == NACC_UPDATE_MAX_DECAY, "unknown update rule");
  NACC_REQUIRE(thresh_rule == NACC_THRESH_FIXED || thresh_rule == NACC_THRESH_MIN_MEAN, "unknown threshold rule");
  NACC_REQUIRE(decay >= 0.0f && decay <= 1.0f, "decay must be in [0, 1]");
  NACC_REQUIRE(std::isfinite(threshold), "threshold must be finite");
  NACC_REQUIRE(density && fresh && bits, "density, fresh, bits must be non-NULL");
  NACC_REQUIRE(aligned(density, 4) && aligned(fresh, 4) && aligned(bits, 4), "arrays must be 4-byte aligned");
  NACC_REQUIRE(ws && ws_bytes >= nacc_occgrid_workspace_bytes(grid), "workspace too small");
  const int64_t n = (int64_t)grid->levels * grid->res * grid->res * grid->res;
  const int64_t nb = ceil_div(n, kUpdThreads);
  double *partial = static_cast<double *>(ws);
  double *mean_ws = reinterpret_cast<double *>(static_cast<char *>(ws) + align_up((size_t)nb * 8, 256));
  double *mean_dst = mean ? mean : mean_ws;
  const double gam = (double)decay, one_m = 1.0 - gam;
  const int direct = thresh_rule == NACC_THRESH_FIXED;
  update_kernel<<<(unsigned)nb, kUpdThreads, 0, stream>>>(density, fresh, n, (int)rule, gam, one_m, direct,
                                                          (double)threshold, bits, partial);
  mean_kernel<<<1, 1024, 0, stream>>>(partial, nb, n, mean_dst);
  count_launch(2);
  if (!direct) {
    binarize_kernel<<<grid_for(n, 256), 256, 0, stream>>>(density, n, (double)threshold, mean_dst, bits);
    count_launch(1);
  }
  NACC_CHECK_LAUNCH();
  NACC_CUDA(grid_prepare(*grid, bits, stream));  // refresh the march's skip mask
  return NACC_OK;
}

nacc_status nacc_occgrid_times(const nacc_grid *grid, uint64_t seed, int64_t step, int32_t draw,
                               int64_t cell_begin, int64_t cell_count, float *times, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_grid(grid);
  if (s != NACC_OK) return s;
  const int64_t n = (int64_t)grid->levels * grid->res * grid->res * grid->res;
  NACC_REQUIRE(cell_begin >= 0 && cell_count >= 0 && cell_begin + cell_count <= n, "cell range out of bounds");
  NACC_REQUIRE(draw >= 0, "draw must be >= 0");
  if (cell_count == 0) return NACC_OK;
  NACC_REQUIRE(times && aligned(times, 4), "times must be non-NULL");
  times_kernel<<<grid_for(cell_count, 256), 256, 0, stream>>>(grid->res, (uint32_t)(seed & 0xffffffffu),
                                                             (uint32_t)(seed >> 32), (uint32_t)step, (uint32_t)draw,
                                                             cell_begin, cell_count, times);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_max_merge(float *dst, const float *src, int64_t n, cudaStream_t stream) {
  clear_error();
  NACC_REQUIRE(n >= 0, "n must be >= 0");
  if (n == 0) return NACC_OK;
  NACC_REQUIRE(dst && src && aligned(dst, 4) && aligned(src, 4), "dst and src must be non-NULL");
  max_merge_kernel<<<grid_for(ceil_div(n, 4), 256), 256, 0, stream>>>(dst, src, n);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

}  // extern "C"
