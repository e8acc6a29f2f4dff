// march.cu — occupancy-grid ray marching into packed intervals (Alg. 1
// nerfacc.sampling; spatial skipping; sample as interval
// and packed tensor).  DESIGN.md §6 describes the kernel design.
//
// Membership of lattice interval k (readings #1-#3; normative fp32 ops):
//   m_k = fmaf(k + 0.5, Δt, near_r)            (uniform lattice), or
//   t_{k+1} = t_k + min(max(t_k c, Δt), Δt_max), m_k = t_k + 0.5 dt_k  (cone)
//   x_a  = fmaf(m_k, d_a, o_a)
//   l*   = first level l with lo_l <= x < hi_l on every axis
//   u_a  = (x_a - lo_{l*,a}) * s_{l*,a},  i_a = clamp(floor(u_a), 0, R-1)
//   P(k) = m_k < far_r  and  l* exists  and  bit[l*][i]
// The k range each warp scans is a conservative fp64 slab bound (±2 steps
// around the padded outermost box); membership alone decides emission.
#include "common.cuh"

namespace nacc {

struct GridConst {
  int levels, res;
  float lo[8][3], hi[8][3], s[8][3];
  double olo[3], ohi[3];  // outermost box padded by 1e-4*width + 1e-6 (fp64)
};

struct MarchConst {
  float near_plane, far_plane, step, max_step, cone;
  int stratified;
  uint32_t key0, key1;
};

static GridConst make_grid_const(const nacc_grid &g) {
  GridConst c{};
  c.levels = g.levels;
  c.res = g.res;
  for (int a = 0; a < 3; ++a) {
    const double lo0 = (double)g.roi[a], hi0 = (double)g.roi[3 + a];
    const double ctr = (lo0 + hi0) / 2.0, half = (hi0 - lo0) / 2.0;
    for (int l = 0; l < g.levels; ++l) {
      const double sc = std::ldexp(1.0, l);
      c.lo[l][a] = (float)(ctr - half * sc);
      c.hi[l][a] = (float)(ctr + half * sc);
      c.s[l][a] = (float)((double)g.res / ((double)c.hi[l][a] - (double)c.lo[l][a]));
    }
    const int L = g.levels - 1;
    const double w = (double)c.hi[L][a] - (double)c.lo[L][a];
    const double pad = 1e-4 * w + 1e-6;
    c.olo[a] = (double)c.lo[L][a] - pad;
    c.ohi[a] = (double)c.hi[L][a] + pad;
  }
  return c;
}

// -------------------------------------------------------------------------- device
__device__ __forceinline__ bool occupied(const GridConst &g, const uint32_t *__restrict__ bits,
                                         float m, float ox, float oy, float oz, float dx, float dy,
                                         float dz) {
  const float x = __fmaf_rn(m, dx, ox), y = __fmaf_rn(m, dy, oy), z = __fmaf_rn(m, dz, oz);
  int l = 0;
  for (; l < g.levels; ++l) {
    if (g.lo[l][0] <= x && x < g.hi[l][0] && g.lo[l][1] <= y && y < g.hi[l][1] &&
        g.lo[l][2] <= z && z < g.hi[l][2])
      break;
  }
  if (l == g.levels) return false;
  const int R = g.res;
  int ix = (int)floorf(__fmul_rn(__fsub_rn(x, g.lo[l][0]), g.s[l][0]));
  int iy = (int)floorf(__fmul_rn(__fsub_rn(y, g.lo[l][1]), g.s[l][1]));
  int iz = (int)floorf(__fmul_rn(__fsub_rn(z, g.lo[l][2]), g.s[l][2]));
  ix = min(max(ix, 0), R - 1);
  iy = min(max(iy, 0), R - 1);
  iz = min(max(iz, 0), R - 1);
  const uint32_t q = (uint32_t)l * (uint32_t)(R * R * R) + (uint32_t)ix + (uint32_t)R * ((uint32_t)iy + (uint32_t)R * (uint32_t)iz);
  return (__ldg(bits + (q >> 5)) >> (q & 31u)) & 1u;
}

struct RaySetup {
  float ox, oy, oz, dx, dy, dz, near_r, far_r;
  bool hit;
  double t_lo, t_hi;
};

__device__ __forceinline__ RaySetup ray_setup(const GridConst &g, const MarchConst &p,
                                              const float *__restrict__ rays_o,
                                              const float *__restrict__ rays_d,
                                              const float *__restrict__ t_min,
                                              const float *__restrict__ t_max, int64_t r) {
  RaySetup s;
  s.ox = __ldg(rays_o + 3 * r);
  s.oy = __ldg(rays_o + 3 * r + 1);
  s.oz = __ldg(rays_o + 3 * r + 2);
  s.dx = __ldg(rays_d + 3 * r);
  s.dy = __ldg(rays_d + 3 * r + 1);
  s.dz = __ldg(rays_d + 3 * r + 2);
  float nr = t_min ? __ldg(t_min + r) : p.near_plane;
  if (p.stratified) {
    const u32x4 rnd = philox4x32_10(u32x4{(uint32_t)(uint64_t)r, (uint32_t)((uint64_t)r >> 32), 0u, 0u}, p.key0, p.key1);
    nr = __double2float_rn(__dadd_rn((double)nr, __dmul_rn(u24(rnd.x), (double)p.step)));
  }
  s.near_r = nr;
  s.far_r = t_max ? __ldg(t_max + r) : p.far_plane;
  // fp64 slab against the padded outermost box (conservative k range only)
  const double o[3] = {s.ox, s.oy, s.oz}, d[3] = {s.dx, s.dy, s.dz};
  double tmin = -INFINITY, tmax = INFINITY;
  bool hit = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (d[a] != 0.0) {
      double ta = (g.olo[a] - o[a]) / d[a], tb = (g.ohi[a] - o[a]) / d[a];
      if (ta > tb) {
        const double tt = ta;
        ta = tb;
        tb = tt;
      }
      tmin = fmax(tmin, ta);
      tmax = fmin(tmax, tb);
    } else if (!(g.olo[a] <= o[a] && o[a] < g.ohi[a])) {
      hit = false;
    }
  }
  s.t_lo = fmax(tmin, (double)s.near_r);
  s.t_hi = fmin(tmax, (double)s.far_r);
  s.hit = hit && (s.t_hi > s.t_lo);
  return s;
}

// k range of the uniform lattice that can hold emitted intervals
__device__ __forceinline__ void uniform_k_range(const RaySetup &s, float step, int64_t &kb, int64_t &ke) {
  const double dt = (double)step, nr = (double)s.near_r;
  const double fb = floor((s.t_lo - nr) / dt - 0.5) - 2.0;
  const double fe = ceil((s.t_hi - nr) / dt) + 3.0;
  kb = fb > 0.0 ? (int64_t)fb : 0;
  const double cap = (double)(1 << 24);
  ke = fe < cap ? (fe > 0.0 ? (int64_t)fe : 0) : (int64_t)(1 << 24);
}

// first index k in [0, K) with tab[k] >= v (tab ascending)
__device__ __forceinline__ int64_t lower_bound(const float *__restrict__ tab, int64_t K, double v) {
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((double)__ldg(tab + mid) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// cone lattice table: tab[0..K] = t_0..t_K, K = number of intervals whose
// midpoint is < far and whose start is <= t_cap (+3 slack intervals)
constexpr int64_t kConeTableMax = 1 << 20;

struct ConeHeader {
  int64_t K;
  int32_t overflow;
  uint32_t t_cap_bits;
};

__global__ void cone_tcap_kernel(GridConst g, MarchConst p, const float *__restrict__ rays_o,
                                 const float *__restrict__ rays_d, const float *__restrict__ t_max,
                                 int64_t n_rays, ConeHeader *hdr) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float v = 0.0f;
  if (r < n_rays) {
    RaySetup s = ray_setup(g, p, rays_o, rays_d, nullptr, t_max, r);
    if (s.hit) v = (float)s.t_hi;
  }
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.0f) atomicMax(&hdr->t_cap_bits, __float_as_uint(v));
}

__global__ void cone_table_kernel(MarchConst p, ConeHeader *hdr, float *__restrict__ tab) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const float t_cap = __uint_as_float(hdr->t_cap_bits);
  float t = p.near_plane;
  int64_t k = 0;
  int extra = 0;
  int32_t overflow = 0;
  tab[0] = t;
  for (;;) {
    const float dt = fminf(fmaxf(__fmul_rn(t, p.cone), p.step), p.max_step);
    const float m = __fadd_rn(t, __fmul_rn(0.5f, dt));
    const float tn = __fadd_rn(t, dt);
    if (!(m < p.far_plane)) break;
    if (t > t_cap && ++extra > 3) break;
    if (k + 1 >= kConeTableMax) {
      overflow = 1;
      break;
    }
    tab[k + 1] = tn;
    ++k;
    t = tn;
  }
  hdr->K = k;
  hdr->overflow = overflow;
}

template <bool kCone, bool kFill>
__global__ void __launch_bounds__(256) march_kernel(GridConst g, MarchConst p,
                                                    const uint32_t *__restrict__ bits,
                                                    const float *__restrict__ rays_o,
                                                    const float *__restrict__ rays_d,
                                                    const float *__restrict__ t_min,
                                                    const float *__restrict__ t_max, int64_t n_rays,
                                                    const ConeHeader *__restrict__ hdr,
                                                    const float *__restrict__ tab,
                                                    int32_t *__restrict__ counts,
                                                    const int64_t *__restrict__ packed_info,
                                                    const int64_t *__restrict__ total, int64_t capacity,
                                                    float *__restrict__ t0, float *__restrict__ t1,
                                                    int32_t *__restrict__ ray_id) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  if (kFill && total && *total > capacity) return;
  int64_t out = 0;
  if (kFill) out = packed_info[2 * r];
  int32_t cnt = 0;
  const RaySetup s = ray_setup(g, p, rays_o, rays_d, t_min, t_max, r);
  if (s.hit) {
    int64_t kb, ke;
    if (kCone) {
      const int64_t K = hdr->K;
      kb = lower_bound(tab + 1, K, s.t_lo) - 2;  // first k with t_{k+1} >= t_lo, minus slack
      if (kb < 0) kb = 0;
      ke = lower_bound(tab, K + 1, s.t_hi) + 2;  // first k with t_k >= t_hi, plus slack
      if (ke > K) ke = K;
    } else {
      uniform_k_range(s, p.step, kb, ke);
    }
    for (int64_t k0 = kb; k0 < ke; k0 += 32) {
      const int64_t k = k0 + lane;
      bool pred = false, stop = false;
      float ta = 0.f, tb = 0.f;
      if (k < ke) {
        float m;
        if (kCone) {
          ta = __ldg(tab + k);
          tb = __ldg(tab + k + 1);
          const float dt = fminf(fmaxf(__fmul_rn(ta, p.cone), p.step), p.max_step);
          m = __fadd_rn(ta, __fmul_rn(0.5f, dt));
        } else {
          m = __fmaf_rn((float)k + 0.5f, p.step, s.near_r);
        }
        if (!(m < s.far_r)) stop = true;
        else pred = occupied(g, bits, m, s.ox, s.oy, s.oz, s.dx, s.dy, s.dz);
      }
      const unsigned b = __ballot_sync(kFull, pred);
      if (kFill && pred) {
        if (!kCone) {
          ta = __fmaf_rn((float)k, p.step, s.near_r);
          tb = __fmaf_rn((float)(k + 1), p.step, s.near_r);
        }
        const int64_t q = out + cnt + __popc(b & ((1u << lane) - 1u));
        t0[q] = ta;
        t1[q] = tb;
        ray_id[q] = (int32_t)r;
      }
      cnt += __popc(b);
      if (__any_sync(kFull, stop)) break;
    }
  }
  if (!kFill && lane == 0) counts[r] = cnt;
}

__global__ void capacity_status_kernel(const int64_t *total, int64_t capacity, const ConeHeader *hdr,
                                       int32_t *status) {
  int32_t st = (*total > capacity) ? NACC_ERR_INSUFFICIENT_CAPACITY : NACC_OK;
  if (hdr && hdr->overflow) st = NACC_ERR_UNSUPPORTED;
  *status = st;
}

// -------------------------------------------------------------------------- host
struct MarchWs {
  int32_t *counts;
  void *scan_ws;
  ConeHeader *hdr;
  float *tab;
};

static size_t march_ws_layout(const nacc_march &p, int64_t n, MarchWs *w, void *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  const size_t o_counts = take((size_t)n * 4);
  const size_t o_scan = take(scan_workspace_bytes(n));
  size_t o_hdr = 0, o_tab = 0;
  const bool cone = p.cone_angle > 0.0f;
  if (cone) {
    o_hdr = take(sizeof(ConeHeader));
    o_tab = take((size_t)(kConeTableMax + 1) * 4);
  }
  if (w && base) {
    char *b = static_cast<char *>(base);
    w->counts = reinterpret_cast<int32_t *>(b + o_counts);
    w->scan_ws = b + o_scan;
    w->hdr = cone ? reinterpret_cast<ConeHeader *>(b + o_hdr) : nullptr;
    w->tab = cone ? reinterpret_cast<float *>(b + o_tab) : nullptr;
  }
  return off;
}

static nacc_status validate(const nacc_grid *grid, const uint32_t *bits, const nacc_march *p,
                            const float *rays_o, const float *rays_d, const float *t_min,
                            int64_t n_rays, void *ws, size_t ws_bytes) {
  NACC_REQUIRE(grid && p, "grid and params must be non-NULL");
  NACC_REQUIRE(grid->levels >= 1 && grid->levels <= 8, "levels must be in 1..8");
  NACC_REQUIRE(grid->res >= 1, "res must be >= 1");
  NACC_REQUIRE((int64_t)grid->levels * grid->res * grid->res * grid->res < (1ll << 31),
               "levels*res^3 must be < 2^31");
  for (int a = 0; a < 3; ++a)
    NACC_REQUIRE(std::isfinite(grid->roi[a]) && std::isfinite(grid->roi[3 + a]) &&
                     grid->roi[a] < grid->roi[3 + a],
                 "roi must be finite with lo < hi");
  NACC_REQUIRE(std::isfinite(p->step) && p->step > 0.0f, "step must be > 0 and finite");
  NACC_REQUIRE(p->cone_angle >= 0.0f && std::isfinite(p->cone_angle), "cone_angle must be >= 0");
  NACC_REQUIRE(!(p->cone_angle > 0.0f) || (p->max_step >= p->step), "max_step must be >= step");
  NACC_REQUIRE(std::isfinite(p->near_plane) && !std::isnan(p->far_plane), "near/far must be numbers");
  NACC_REQUIRE(n_rays >= 0 && n_rays < (1ll << 31), "n_rays must be in [0, 2^31)");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(bits && rays_o && rays_d, "bits, rays_o, rays_d must be non-NULL");
  NACC_REQUIRE(aligned(bits, 4) && aligned(rays_o, 4) && aligned(rays_d, 4), "arrays must be 4-byte aligned");
  NACC_REQUIRE(ws && ws_bytes >= nacc_sampling_occgrid_workspace_bytes(grid, p, n_rays),
               "workspace too small");
  if (p->cone_angle > 0.0f && (t_min || p->stratified)) return NACC_ERR_UNSUPPORTED;
  return NACC_OK;
}

static MarchConst make_march_const(const nacc_march &p) {
  MarchConst m;
  m.near_plane = p.near_plane;
  m.far_plane = p.far_plane;
  m.step = p.step;
  m.max_step = p.max_step;
  m.cone = p.cone_angle;
  m.stratified = p.stratified;
  m.key0 = (uint32_t)(p.seed & 0xffffffffu);
  m.key1 = (uint32_t)(p.seed >> 32);
  return m;
}

static nacc_status launch_march(bool fill, const nacc_grid *grid, const uint32_t *bits,
                                const nacc_march *params, const float *rays_o, const float *rays_d,
                                const float *t_min, const float *t_max, int64_t n_rays,
                                int64_t *packed_info, float *t0, float *t1, int32_t *ray_id,
                                int64_t capacity, int64_t *total, int32_t *status_out, void *ws,
                                cudaStream_t stream, bool build_table) {
  MarchWs w;
  march_ws_layout(*params, n_rays, &w, ws);
  const GridConst g = make_grid_const(*grid);
  const MarchConst p = make_march_const(*params);
  const bool cone = params->cone_angle > 0.0f;
  if (cone && build_table) {
    NACC_CUDA(cudaMemsetAsync(w.hdr, 0, sizeof(ConeHeader), stream));
    cone_tcap_kernel<<<grid_for(n_rays, 256), 256, 0, stream>>>(g, p, rays_o, rays_d, t_max, n_rays, w.hdr);
    cone_table_kernel<<<1, 32, 0, stream>>>(p, w.hdr, w.tab);
    count_launch(2);
    NACC_CHECK_LAUNCH();
  }
  const int blocks = grid_for(n_rays * 32, 256);
  if (!fill) {
    if (cone)
      march_kernel<true, false><<<blocks, 256, 0, stream>>>(g, p, bits, rays_o, rays_d, t_min, t_max, n_rays, w.hdr, w.tab,
                                                            w.counts, nullptr, nullptr, 0, nullptr, nullptr, nullptr);
    else
      march_kernel<false, false><<<blocks, 256, 0, stream>>>(g, p, bits, rays_o, rays_d, t_min, t_max, n_rays, w.hdr, w.tab,
                                                             w.counts, nullptr, nullptr, 0, nullptr, nullptr, nullptr);
    count_launch(1);
    NACC_CHECK_LAUNCH();
    NACC_CUDA(scan_counts_to_packed(w.counts, n_rays, packed_info, total, w.scan_ws, stream));
    if (status_out) {
      capacity_status_kernel<<<1, 1, 0, stream>>>(total, capacity, w.hdr, status_out);
      count_launch(1);
    }
    NACC_CHECK_LAUNCH();
  }
  if (t0 && t1 && ray_id) {
    if (cone)
      march_kernel<true, true><<<blocks, 256, 0, stream>>>(g, p, bits, rays_o, rays_d, t_min, t_max, n_rays, w.hdr, w.tab,
                                                           nullptr, packed_info, fill ? nullptr : total, capacity, t0, t1, ray_id);
    else
      march_kernel<false, true><<<blocks, 256, 0, stream>>>(g, p, bits, rays_o, rays_d, t_min, t_max, n_rays, w.hdr, w.tab,
                                                            nullptr, packed_info, fill ? nullptr : total, capacity, t0, t1, ray_id);
    count_launch(1);
    NACC_CHECK_LAUNCH();
  }
  return NACC_OK;
}

}  // namespace nacc

using namespace nacc;

extern "C" {

size_t nacc_sampling_occgrid_workspace_bytes(const nacc_grid *grid, const nacc_march *params,
                                             int64_t n_rays) {
  if (!grid || !params || n_rays < 0) return 0;
  return march_ws_layout(*params, n_rays, nullptr, nullptr);
}

nacc_status nacc_sampling_occgrid(const nacc_grid *grid, const uint32_t *bits, const nacc_march *params,
                                  const float *rays_o, const float *rays_d, const float *t_min,
                                  const float *t_max, int64_t n_rays, int64_t *packed_info, float *t0,
                                  float *t1, int32_t *ray_id, int64_t capacity, int64_t *total,
                                  int32_t *status_out, void *ws, size_t ws_bytes, cudaStream_t stream) {
  clear_error();
  nacc_status st = validate(grid, bits, params, rays_o, rays_d, t_min, n_rays, ws, ws_bytes);
  if (st != NACC_OK) return st;
  NACC_REQUIRE(total && capacity >= 0, "total must be non-NULL and capacity >= 0");
  if (n_rays == 0) {
    NACC_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), stream));
    if (status_out) NACC_CUDA(cudaMemsetAsync(status_out, 0, sizeof(int32_t), stream));
    return NACC_OK;
  }
  NACC_REQUIRE(packed_info && aligned(packed_info, 16), "packed_info must be non-NULL and 16-byte aligned");
  NACC_REQUIRE((!t0 && !t1 && !ray_id) || (t0 && t1 && ray_id), "t0, t1, ray_id: all or none");
  return launch_march(false, grid, bits, params, rays_o, rays_d, t_min, t_max, n_rays, packed_info, t0, t1,
                      ray_id, capacity, total, status_out, ws, stream, true);
}

nacc_status nacc_sampling_occgrid_fill(const nacc_grid *grid, const uint32_t *bits, const nacc_march *params,
                                       const float *rays_o, const float *rays_d, const float *t_min,
                                       const float *t_max, int64_t n_rays, const int64_t *packed_info,
                                       float *t0, float *t1, int32_t *ray_id, void *ws, size_t ws_bytes,
                                       cudaStream_t stream) {
  clear_error();
  nacc_status st = validate(grid, bits, params, rays_o, rays_d, t_min, n_rays, ws, ws_bytes);
  if (st != NACC_OK) return st;
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(packed_info && t0 && t1 && ray_id, "packed_info, t0, t1, ray_id must be non-NULL");
  // the cone table lives in the workspace of the preceding nacc_sampling_occgrid call; rebuild it
  return launch_march(true, grid, bits, params, rays_o, rays_d, t_min, t_max, n_rays,
                      const_cast<int64_t *>(packed_info), t0, t1, ray_id, 0, nullptr, nullptr, ws, stream,
                      true);
}

}  // extern "C"
