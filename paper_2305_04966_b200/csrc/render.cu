// render.cu — the transmittance estimator and compositing of Eq. 2
// discretised as in P:246 (reading #11), forward and backward:
//   δ_i = t1_i - t0_i, s_i = σ_i δ_i, S_i = Σ_{j<i} s_j (fp64 segmented scan),
//   T_i = exp(-S_i), α_i = 1 - exp(-s_i), w_i = T_i α_i, w_i = 0 once S_i > -ln ε,
//   color = Σ w rgb, opacity = Σ w, depth = Σ w m / max(opacity, 1e-10).
// Backward (t detached P:78):
//   g_σ_i = δ_i (g_w_i T_i (1-α_i) - Σ_{j>i} g_w_j w_j) for live samples,
// with Σ_{j>i} g_w_j w_j = R - Σ_{j<=i} g_w_j w_j and R = <g_C,C> + g_O' O + g_N N
// taken from the forward's fp64 per-ray sums (ctx), so one forward-order pass
// suffices.  Fused path: flat ray-aligned tiles (segscan.cuh); granular and
// fallback paths: one warp per ray, 32 consecutive samples per step.
#include "common.cuh"
#include "debug.cuh"
#include "segscan.cuh"

namespace nacc {

struct Chunk {
  bool valid, live;
  float t0, t1, sig;
  double delta, s, S;  // S = entering optical depth
};

// loads lane's sample of chunk `base`, performs the segmented scan step and
// advances the carry; returns the chunk's state for this lane
__device__ __forceinline__ Chunk load_chunk(const float *__restrict__ t0, const float *__restrict__ t1,
                                            const float *__restrict__ sigma, int64_t st, int64_t cnt,
                                            int64_t base, double L, double &carry) {
  const int lane = threadIdx.x & 31;
  Chunk c;
  const int64_t i = base + lane;
  c.valid = i < cnt;
  c.t0 = c.t1 = c.sig = 0.f;
  c.delta = c.s = 0.0;
  if (c.valid) {
    const int64_t q = st + i;
    c.t0 = __ldg(t0 + q);
    c.t1 = __ldg(t1 + q);
    c.sig = __ldg(sigma + q);
    c.delta = (double)c.t1 - (double)c.t0;
    c.s = (double)c.sig * c.delta;
  }
  const double incl = warp_incl_scan(c.s);
  double excl = __shfl_up_sync(kFull, incl, 1);
  if (lane == 0) excl = 0.0;
  c.S = carry + excl;
  c.live = c.valid && !(c.S > L);
  carry += __shfl_sync(kFull, incl, 31);
  return c;
}

// fp64: the depth gradient divides by the opacity, so weights must carry
// fp64 precision for the backward's R - P_i difference
__device__ __forceinline__ double trans_of(double S) { return exp(-S); }
__device__ __forceinline__ double alpha_of(double s) { return -expm1(-s); }

// ------------------------------------------------------------------ fused forward
__global__ void __launch_bounds__(256) render_fwd_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                         const float *__restrict__ t0, const float *__restrict__ t1,
                                                         const float *__restrict__ sigma, const float *__restrict__ rgb,
                                                         double L, float *__restrict__ color,
                                                         float *__restrict__ opacity, float *__restrict__ depth,
                                                         double *__restrict__ ctx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  double carry = 0.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, O = 0.0, N = 0.0;
  for (int64_t base = 0; base < cnt; base += 32) {
    const Chunk c = load_chunk(t0, t1, sigma, st, cnt, base, L, carry);
    if (c.live) {
      const double w = trans_of(c.S) * alpha_of(c.s);
      const int64_t q = st + base + lane;
      if (rgb) {
        C0 += w * (double)__ldg(rgb + 3 * q);
        C1 += w * (double)__ldg(rgb + 3 * q + 1);
        C2 += w * (double)__ldg(rgb + 3 * q + 2);
      }
      O += w;
      N += w * (0.5 * ((double)c.t0 + (double)c.t1));
    }
    if (carry > L) break;  // every later sample has S > L: w = 0
  }
  C0 = warp_sum(C0);
  C1 = warp_sum(C1);
  C2 = warp_sum(C2);
  O = warp_sum(O);
  N = warp_sum(N);
  if (lane == 0) {
    if (color) {
      color[3 * r] = (float)C0;
      color[3 * r + 1] = (float)C1;
      color[3 * r + 2] = (float)C2;
    }
    if (opacity) opacity[r] = (float)O;
    if (depth) depth[r] = (float)(N / fmax(O, 1e-10));
    if (ctx) {
      double *cx = ctx + 5 * r;
      cx[0] = C0;
      cx[1] = C1;
      cx[2] = C2;
      cx[3] = O;
      cx[4] = N;
    }
  }
}

// ------------------------------------------------------------------ fused backward
__global__ void __launch_bounds__(256) render_bwd_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                         const float *__restrict__ t0, const float *__restrict__ t1,
                                                         const float *__restrict__ sigma, const float *__restrict__ rgb,
                                                         double L, const double *__restrict__ ctx,
                                                         const float *__restrict__ g_color,
                                                         const float *__restrict__ g_opacity,
                                                         const float *__restrict__ g_depth,
                                                         float *__restrict__ g_sigma, float *__restrict__ g_rgb) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  double C0, C1, C2, O, N;
  if (ctx) {
    const double *cx = ctx + 5 * r;
    C0 = cx[0];
    C1 = cx[1];
    C2 = cx[2];
    O = cx[3];
    N = cx[4];
  } else {  // recompute the forward sums
    double carry = 0.0;
    C0 = C1 = C2 = O = N = 0.0;
    for (int64_t base = 0; base < cnt; base += 32) {
      const Chunk c = load_chunk(t0, t1, sigma, st, cnt, base, L, carry);
      if (c.live) {
        const double w = trans_of(c.S) * alpha_of(c.s);
        const int64_t q = st + base + lane;
        if (rgb) {
          C0 += w * (double)__ldg(rgb + 3 * q);
          C1 += w * (double)__ldg(rgb + 3 * q + 1);
          C2 += w * (double)__ldg(rgb + 3 * q + 2);
        }
        O += w;
        N += w * (0.5 * ((double)c.t0 + (double)c.t1));
      }
      if (carry > L) break;
    }
    C0 = warp_sum(C0);
    C1 = warp_sum(C1);
    C2 = warp_sum(C2);
    O = warp_sum(O);
    N = warp_sum(N);
  }
  const double gc0 = g_color ? (double)g_color[3 * r] : 0.0;
  const double gc1 = g_color ? (double)g_color[3 * r + 1] : 0.0;
  const double gc2 = g_color ? (double)g_color[3 * r + 2] : 0.0;
  const double gO = g_opacity ? (double)g_opacity[r] : 0.0;
  const double gD = g_depth ? (double)g_depth[r] : 0.0;
  double gN, gOp;
  if (O > 1e-10) {
    gN = gD / O;
    gOp = gO - gD * (N / O) / O;
  } else {
    gN = gD / 1e-10;
    gOp = gO;
  }
  const double R = gc0 * C0 + gc1 * C1 + gc2 * C2 + gOp * O + gN * N;
  double carry = 0.0, P = 0.0;
  bool dead = false;
  for (int64_t base = 0; base < cnt; base += 32) {
    const int64_t i = base + lane, q = st + i;
    if (dead) {  // past the cut: zero gradients, no loads
      if (i < cnt) {
        g_sigma[q] = 0.f;
        if (g_rgb) {
          g_rgb[3 * q] = 0.f;
          g_rgb[3 * q + 1] = 0.f;
          g_rgb[3 * q + 2] = 0.f;
        }
      }
      continue;
    }
    const Chunk c = load_chunk(t0, t1, sigma, st, cnt, base, L, carry);
    double gw = 0.0, w = 0.0, T = 0.0, ea = 0.0;
    float r0 = 0.f, r1 = 0.f, r2 = 0.f;
    if (c.live) {
      T = trans_of(c.S);
      ea = exp(-c.s);  // 1 - α
      w = T * alpha_of(c.s);
      if (rgb) {
        r0 = __ldg(rgb + 3 * q);
        r1 = __ldg(rgb + 3 * q + 1);
        r2 = __ldg(rgb + 3 * q + 2);
      }
      gw = gc0 * r0 + gc1 * r1 + gc2 * r2 + gOp + gN * (0.5 * ((double)c.t0 + (double)c.t1));
    }
    const double v = gw * w;
    const double incl = warp_incl_scan(v);
    const double Q = R - (P + incl);  // Σ_{j>i} g_w_j w_j
    P += __shfl_sync(kFull, incl, 31);
    if (c.valid) {
      const double gs = c.live ? gw * T * ea - Q : 0.0;
      g_sigma[q] = (float)(c.delta * gs);
      if (g_rgb) {
        g_rgb[3 * q] = (float)(w * gc0);
        g_rgb[3 * q + 1] = (float)(w * gc1);
        g_rgb[3 * q + 2] = (float)(w * gc2);
      }
    }
    dead = carry > L;
  }
}

// Per-thread view of 4 consecutive packed samples.
struct Items {
  int64_t q0;
  bool valid[4], head[4], tail[4];
  float t0[4], t1[4], sg[4];
  int32_t rid[4];
};

// ------------------------------------------------------------------ warp-tile fused render
// Each warp owns the rays whose first sample lies in its 256-sample tile and
// walks them in chunks of 32 lanes x 4 consecutive samples (float4 loads);
// fp64 warp-level segmented scans (no shared memory, no block barriers) carry
// the open ray across chunks.  Extra warps zero the outputs of empty rays.
#ifndef NACC_RENDER_TILE
#define NACC_RENDER_TILE 512  // samples per warp tile (A/B on 3.8 M samples: 128 / 256 / 512 / 768 / 1024 -> fwd+bwd 177 / 151 / 141 / 157 / 140 us)
#endif
#ifndef NACC_RENDER_BPS
#define NACC_RENDER_BPS 4  // blocks per SM of the tile kernels (A/B: 2 / 3 / 4 -> bwd 88.4 / 81.7 / 79.7 us)
#endif
#ifndef NACC_RENDER_COLORONLY
#define NACC_RENDER_COLORONLY 1  // build parameter: colour-loss backward without the per-ray constants kernel
#endif
#ifndef NACC_RENDER_GRIDX
#define NACC_RENDER_GRIDX 2  // build parameter: grid of the tile kernels as a multiple of the resident blocks
                             // (2: a second wave balances the forward's tiles; CFG2 fwd 60.3 -> 59.5 us)
#endif
#ifndef NACC_RENDER_TPROD
#define NACC_RENDER_TPROD 1  // build parameter: T_{j+1} = T_j e^{-s_j} within a thread's items
#endif
#ifndef NACC_RENDER_RAYCACHE
#define NACC_RENDER_RAYCACHE 1  // build parameter: backward loads per-ray constants once per run of the ray
#endif
#ifndef NACC_RENDER_FASTEXP
#define NACC_RENDER_FASTEXP 1  // build parameter: e^{-s} by exp_neg below (0: the CUDA math library exp)
#endif
// e^{-s} for s >= 0 in fp64 to ~2e-13 relative: the fused tile kernels need T = Π e^{-s_j} to
// ~1e-9 over a 5000-sample ray (abs 1e-5 bars on T and w, rel 1e-3 on gradients), not to the
// last fp64 ulp, so a Cody-Waite reduction e^{-s} = 2^n e^r, |r| <= ln2/2, and a degree-10
// Taylor polynomial (remainder |r|^11/11! < 2.2e-13) replace the library exp's ~39 instructions
// with ~19.  s > 708 returns 0 (e^{-708} ~ 1e-308).
__device__ __forceinline__ double exp_neg(double s) {
  const double x = -s;
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: x*log2(e) + magic holds round(x*log2(e))
  const double kd = __fma_rn(x, 1.4426950408889634, magic);
  const int n = __double2loint(kd);
  const double nd = kd - magic;
  double r = __fma_rn(nd, -6.93147180369123816490e-01, x);  // ln2 split in two (Cody-Waite)
  r = __fma_rn(nd, -1.90821492927058770002e-10, r);
  double p = 2.7557319223985893e-07;  // 1/10!
  p = __fma_rn(p, r, 2.7557319223985888e-06);
  p = __fma_rn(p, r, 2.4801587301587302e-05);
  p = __fma_rn(p, r, 1.9841269841269841e-04);
  p = __fma_rn(p, r, 1.3888888888888889e-03);
  p = __fma_rn(p, r, 8.3333333333333332e-03);
  p = __fma_rn(p, r, 4.1666666666666664e-02);
  p = __fma_rn(p, r, 1.6666666666666666e-01);
  p = __fma_rn(p, r, 0.5);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  const double scale = __hiloint2double((n + 1023) << 20, 0);  // 2^n, n >= -1022 below the cutoff
  return s > 708.0 ? 0.0 : p * scale;
}

// e^{-s} of one interval (1 - alpha)
__device__ __forceinline__ double interval_ea(double s) {
#if NACC_RENDER_FASTEXP
  return exp_neg(s);
#else
  return exp(-s);
#endif
}
__device__ __forceinline__ double trans_first(double S) {  // T of a thread's first item
#if NACC_RENDER_FASTEXP
  return exp_neg(S);
#else
  return exp(-S);
#endif
}
constexpr int64_t kWarpTile = NACC_RENDER_TILE;  // samples per warp tile of the forward (build parameter)
#ifndef NACC_RENDER_BWD_TILE
#define NACC_RENDER_BWD_TILE 1024  // backward tile (A/B on 3.8 M samples: 512 / 1024 -> 71.5 / 68.6 us)
#endif
constexpr int64_t kWarpTileBwd = NACC_RENDER_BWD_TILE;
#ifndef NACC_RENDER_L2PF
#define NACC_RENDER_L2PF 0  // build parameter: TMA bulk L2 prefetch of the warp's next tile (A/B: slower)
#endif

// One bulk-copy-engine prefetch of [p, p + n floats) into L2 (cp.async.bulk.prefetch.L2,
// SASS UBLKPF): 16-byte aligned start, size a multiple of 16 B.
__device__ __forceinline__ void l2_prefetch_floats(const void *p, int64_t n_floats) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uint32_t bytes = (uint32_t)((n_floats * 4 + 15) & ~(int64_t)15);
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}
constexpr int kWarpChunk = 128;

// lane 0 prefetches the raw sample range of warp tile wt (plus a chunk of slack past its end,
// where the ray-aligned tile usually extends) into L2 while the warp works on its current tile
__device__ __forceinline__ void prefetch_tile(int64_t wt, int64_t N, const float *t0, const float *t1,
                                              const float *sigma, const int32_t *ray_id, const float *rgb,
                                              int64_t tile = kWarpTile) {
  if (!NACC_RENDER_L2PF || (threadIdx.x & 31) != 0) return;
  const int64_t a = wt * tile;
  if (a >= N) return;
  const int64_t b = min(a + tile + kWarpChunk, N);
  const int64_t a4 = a & ~(int64_t)3, n = b - a4;
  l2_prefetch_floats(t0 + a4, n);
  l2_prefetch_floats(t1 + a4, n);
  l2_prefetch_floats(sigma + a4, n);
  l2_prefetch_floats(ray_id + a4, n);
  if (rgb) l2_prefetch_floats(rgb + 3 * a4, 3 * n);
}

template <bool kVec>
__device__ __forceinline__ void load_items_warp(Items &it, int64_t c0, int64_t B, int64_t E,
                                                const float *__restrict__ t0, const float *__restrict__ t1,
                                                const float *__restrict__ sigma, const int32_t *__restrict__ ray_id,
                                                int32_t &carry_rid) {
  const int lane = threadIdx.x & 31;
  const int64_t q0 = c0 + (int64_t)lane * 4;
  it.q0 = q0;
  const bool full = kVec && q0 >= B && q0 + 3 < E;
  if (full) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(t0 + q0));
    const float4 b = __ldg(reinterpret_cast<const float4 *>(t1 + q0));
    const float4 c = __ldg(reinterpret_cast<const float4 *>(sigma + q0));
    const int4 d = __ldg(reinterpret_cast<const int4 *>(ray_id + q0));
    it.t0[0] = a.x; it.t0[1] = a.y; it.t0[2] = a.z; it.t0[3] = a.w;
    it.t1[0] = b.x; it.t1[1] = b.y; it.t1[2] = b.z; it.t1[3] = b.w;
    it.sg[0] = c.x; it.sg[1] = c.y; it.sg[2] = c.z; it.sg[3] = c.w;
    it.rid[0] = d.x; it.rid[1] = d.y; it.rid[2] = d.z; it.rid[3] = d.w;
#pragma unroll
    for (int j = 0; j < 4; ++j) it.valid[j] = true;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = q0 + j;
      it.valid[j] = q >= B && q < E;
      it.t0[j] = it.valid[j] ? __ldg(t0 + q) : 0.f;
      it.t1[j] = it.valid[j] ? __ldg(t1 + q) : 0.f;
      it.sg[j] = it.valid[j] ? __ldg(sigma + q) : 0.f;
      it.rid[j] = it.valid[j] ? __ldg(ray_id + q) : -1;
    }
  }
  // neighbours through shuffles; the chunk's first lane uses the previous chunk's last ray,
  // the last lane loads the next sample's ray
  int32_t prev = __shfl_up_sync(kFull, it.rid[3], 1);
  if (lane == 0) prev = carry_rid;
  int32_t next = __shfl_down_sync(kFull, it.rid[0], 1);
  if (lane == 31) next = (q0 + 4 < E) ? __ldg(ray_id + q0 + 4) : -2;
  carry_rid = __shfl_sync(kFull, it.rid[3], 31);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int32_t pr = j == 0 ? prev : it.rid[j - 1];
    const int32_t nx = j == 3 ? next : (it.valid[j + 1] ? it.rid[j + 1] : -2);
    it.head[j] = it.valid[j] && (it.q0 + j == B || it.rid[j] != pr);
    it.tail[j] = it.valid[j] && (it.q0 + j + 1 == E || it.rid[j] != nx);
  }
}

__device__ __forceinline__ void load_rgb4(float col[12], const Items &it, const float *__restrict__ rgb, bool vec) {
  if (vec && it.valid[0] && it.valid[3]) {
    const float4 *p = reinterpret_cast<const float4 *>(rgb + 3 * it.q0);
    const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    col[0] = a.x; col[1] = a.y; col[2] = a.z; col[3] = a.w; col[4] = b.x; col[5] = b.y;
    col[6] = b.z; col[7] = b.w; col[8] = c.x; col[9] = c.y; col[10] = c.z; col[11] = c.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) col[3 * j + ch] = it.valid[j] ? __ldg(rgb + 3 * (it.q0 + j) + ch) : 0.f;
  }
}

// entering optical depth of the thread's items (fp64 warp segmented exclusive scan)
__device__ __forceinline__ void warp_items_S(const Items &it, double s[4], double S[4], Seg<1> &carry) {
  Seg<1> agg = seg_identity<1>();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    s[j] = it.valid[j] ? (double)it.sg[j] * ((double)it.t1[j] - (double)it.t0[j]) : 0.0;
    Seg<1> x;
    x.f = it.head[j];
    x.v[0] = s[j];
    agg = seg_combine(agg, x);
  }
  Seg<1> run = warp_seg_excl<1>(agg, carry);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    S[j] = it.head[j] ? 0.0 : run.v[0];
    run.v[0] = (it.head[j] ? 0.0 : run.v[0]) + s[j];
  }
}

// Per-ray sums of the forward, all fp64: O and N (the backward's depth term
// divides by O, so R - P must keep fp64 precision) and colour (an fp32 sum
// over a 5000-sample ray misses the 1e-4 bar).  Same operator as Seg<K>.
#ifndef NACC_SEGM_FMA
#define NACC_SEGM_FMA 1  // build parameter: the 5-value operator as one DFMA per value (fwd 64.5 -> 62.3 us)
#endif
struct SegM {
  int f;
  double o, n;
  double c0, c1, c2;
};
__device__ __forceinline__ SegM segm_identity() { return SegM{0, 0.0, 0.0, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ SegM segm_combine(const SegM &a, const SegM &b) {
  SegM r;
  r.f = a.f | b.f;
#if NACC_SEGM_FMA
  const double keep = b.f ? 0.0 : 1.0;  // one DFMA per value: fma(a, 1, b) = a + b, fma(a, 0, b) = b
  r.o = __fma_rn(a.o, keep, b.o);
  r.n = __fma_rn(a.n, keep, b.n);
  r.c0 = __fma_rn(a.c0, keep, b.c0);
  r.c1 = __fma_rn(a.c1, keep, b.c1);
  r.c2 = __fma_rn(a.c2, keep, b.c2);
#else
  r.o = b.f ? b.o : a.o + b.o;
  r.n = b.f ? b.n : a.n + b.n;
  r.c0 = b.f ? b.c0 : a.c0 + b.c0;
  r.c1 = b.f ? b.c1 : a.c1 + b.c1;
  r.c2 = b.f ? b.c2 : a.c2 + b.c2;
#endif
  return r;
}
__device__ __forceinline__ SegM segm_shfl_up(const SegM &x, int o) {
  SegM y;
  y.f = __shfl_up_sync(kFull, x.f, o);
  y.o = __shfl_up_sync(kFull, x.o, o);
  y.n = __shfl_up_sync(kFull, x.n, o);
  y.c0 = __shfl_up_sync(kFull, x.c0, o);
  y.c1 = __shfl_up_sync(kFull, x.c1, o);
  y.c2 = __shfl_up_sync(kFull, x.c2, o);
  return y;
}
__device__ __forceinline__ SegM segm_shfl(const SegM &x, int src) {
  SegM y;
  y.f = __shfl_sync(kFull, x.f, src);
  y.o = __shfl_sync(kFull, x.o, src);
  y.n = __shfl_sync(kFull, x.n, src);
  y.c0 = __shfl_sync(kFull, x.c0, src);
  y.c1 = __shfl_sync(kFull, x.c1, src);
  y.c2 = __shfl_sync(kFull, x.c2, src);
  return y;
}
__device__ __forceinline__ SegM warp_segm_excl(const SegM &x, SegM &carry) {
  const int lane = threadIdx.x & 31;
  SegM incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const SegM y = segm_shfl_up(incl, o);
    if (lane >= o) incl = segm_combine(y, incl);
  }
  SegM ex = segm_shfl_up(incl, 1);
  if (lane == 0) ex = segm_identity();
  const SegM res = segm_combine(carry, ex);
  carry = segm_combine(carry, segm_shfl(incl, 31));
  return res;
}
__device__ __forceinline__ SegM segm_item(const Items &it, int j, double w, const float *col) {
  SegM x;
  x.f = it.head[j];
  x.o = w;
  x.n = w * (0.5 * ((double)it.t0[j] + (double)it.t1[j]));
  x.c0 = w * (double)col[3 * j];
  x.c1 = w * (double)col[3 * j + 1];
  x.c2 = w * (double)col[3 * j + 2];
  return x;
}

__device__ __forceinline__ void render_fwd_out(const SegM &v, int64_t r, float *__restrict__ color,
                                               float *__restrict__ opacity, float *__restrict__ depth,
                                               double *__restrict__ ctx) {
  if (color) {
    color[3 * r] = (float)v.c0;
    color[3 * r + 1] = (float)v.c1;
    color[3 * r + 2] = (float)v.c2;
  }
  if (opacity) opacity[r] = (float)v.o;
  // depth = N / max(O, 1e-10) in fp32 (rel 1e-4 bar; an fp64 division was ~3 % of the kernel)
  if (depth) depth[r] = __fdiv_rn((float)v.n, (float)fmax(v.o, 1e-10));
  if (ctx) {
    ctx[5 * r] = v.c0;
    ctx[5 * r + 1] = v.c1;
    ctx[5 * r + 2] = v.c2;
    ctx[5 * r + 3] = v.o;
    ctx[5 * r + 4] = v.n;
  }
}

template <bool kVec>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) render_fwd_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ t0, const float *__restrict__ t1, const float *__restrict__ sigma,
    const float *__restrict__ rgb, double L, float *__restrict__ color, float *__restrict__ opacity,
    float *__restrict__ depth, double *__restrict__ ctx) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw * 32 + lane; r < n_rays; r += nw * 32) {  // rays without samples
    if (packed_info[2 * r + 1] == 0) {
      if (color) { color[3 * r] = 0.f; color[3 * r + 1] = 0.f; color[3 * r + 2] = 0.f; }
      if (opacity) opacity[r] = 0.f;
      if (depth) depth[r] = 0.f;
      if (ctx) for (int k = 0; k < 5; ++k) ctx[5 * r + k] = 0.0;
    }
  }
  // persistent warps stride over the tiles in use (N from packed_info: the launch is sized by
  // the resident capacity, not by the arrays' capacity)
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);  // in bounds after an overflowed march
  for (int64_t wt = gw; wt * kWarpTile < N; wt += nw) {
    prefetch_tile(wt + nw, N, t0, t1, sigma, ray_id, rgb);
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTile, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTile, N);
    if (B >= E) continue;
    Seg<1> carryS = seg_identity<1>();
    SegM carryC = segm_identity();
    int32_t carry_rid = -1;
    for (int64_t c0 = B & ~(int64_t)3; c0 < E; c0 += kWarpChunk) {
      Items it;
      load_items_warp<kVec>(it, c0, B, E, t0, t1, sigma, ray_id, carry_rid);
      double s[4], S[4];
      warp_items_S(it, s, S, carryS);
      float col[12];
      load_rgb4(col, it, rgb, kVec);
      // One pass over the items: a ray whose head lies in this lane is summed
      // here and written at its tail; only the lane's leading run (the ray
      // entering from earlier lanes) waits for the warp scan.
      SegM cur = segm_identity();  // sums since the lane start or its last head
      SegM lead;                   // the leading run up to its tail, if that tail is in this lane
      int64_t lead_r = -1;
      // T of the thread's first item from its optical depth, later items by the product
      // T_{j+1} = T_j e^{-s_j} (one fp64 exp per item instead of two)
      double Tn = trans_first(S[0]);
  #pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool live = it.valid[j] && !(S[j] > L);
        const double ea = interval_ea(s[j]);
        const double T = NACC_RENDER_TPROD ? ((j > 0 && it.head[j]) ? 1.0 : Tn) : exp(-S[j]);
        Tn = T * ea;
        const double w = live ? T * (1.0 - ea) : 0.0;
        cur = segm_combine(cur, segm_item(it, j, w, col));
        if (it.tail[j]) {
          if (cur.f) render_fwd_out(cur, it.rid[j], color, opacity, depth, ctx);
          else {
            lead = cur;
            lead_r = it.rid[j];
          }
        }
      }
      const SegM enter = warp_segm_excl(cur, carryC);
      if (lead_r >= 0) render_fwd_out(segm_combine(enter, lead), lead_r, color, opacity, depth, ctx);
    }
  }
}

// Granular weights (render_weights) on the same ray-aligned warp tiles as the fused forward:
// the fp64 segmented scan of σδ gives each item's entering S, T by the product chain from one
// e^{-S} per thread, α = 1 - e^{-s}, w = T α (0 past the early stop); 12 B/sample out as float4
// runs.  Needs ray_id and the contiguous packing (nacc_render_weights_fwd_flat).
template <bool kVec>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) weights_fwd_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ t0, const float *__restrict__ t1, const float *__restrict__ sigma, double L,
    float *__restrict__ weights, float *__restrict__ trans, float *__restrict__ alphas) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);
  for (int64_t wt = gw; wt * kWarpTile < N; wt += nw) {
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTile, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTile, N);
    if (B >= E) continue;
    Seg<1> carryS = seg_identity<1>();
    int32_t carry_rid = -1;
    for (int64_t c0 = B & ~(int64_t)3; c0 < E; c0 += kWarpChunk) {
      Items it;
      load_items_warp<kVec>(it, c0, B, E, t0, t1, sigma, ray_id, carry_rid);
      double s[4], S[4];
      warp_items_S(it, s, S, carryS);
      float wv[4], tv[4], av[4];
      double Tn = trans_first(S[0]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double ea = interval_ea(s[j]);
        const double T = (j > 0 && it.head[j]) ? 1.0 : Tn;
        Tn = T * ea;
        const double a = 1.0 - ea;
        const bool live = it.valid[j] && !(S[j] > L);
        wv[j] = live ? (float)(T * a) : 0.f;
        tv[j] = (float)T;
        av[j] = (float)a;
      }
      if (kVec && it.valid[0] && it.valid[3]) {
        *reinterpret_cast<float4 *>(weights + it.q0) = make_float4(wv[0], wv[1], wv[2], wv[3]);
        if (trans) *reinterpret_cast<float4 *>(trans + it.q0) = make_float4(tv[0], tv[1], tv[2], tv[3]);
        if (alphas) *reinterpret_cast<float4 *>(alphas + it.q0) = make_float4(av[0], av[1], av[2], av[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!it.valid[j]) continue;
          weights[it.q0 + j] = wv[j];
          if (trans) trans[it.q0 + j] = tv[j];
          if (alphas) alphas[it.q0 + j] = av[j];
        }
      }
    }
  }
}

// accumulate_along_rays on the ray-aligned flat tiles (kC = 1..4 channels): lane-sequential fp64
// sums of w v over 4 consecutive samples, rays written at their tails when their head is in the
// lane, the leading run through the fp64 warp segmented scan (Seg<kC>).  Needs ray_id and the
// contiguous packing (nacc_accumulate_along_rays_flat).
template <int kC>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) accumulate_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ weights, const float *__restrict__ values, float *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw * 32 + lane; r < n_rays; r += nw * 32)  // rays without samples
    if (packed_info[2 * r + 1] == 0)
#pragma unroll
      for (int c = 0; c < kC; ++c) out[r * kC + c] = 0.f;
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);
  for (int64_t wt = gw; wt * kWarpTile < N; wt += nw) {
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTile, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTile, N);
    if (B >= E) continue;
    Seg<kC> carry = seg_identity<kC>();
    int32_t carry_rid = -1;
    for (int64_t c0 = B & ~(int64_t)3; c0 < E; c0 += kWarpChunk) {
      const int64_t q0 = c0 + (int64_t)lane * 4;
      bool valid[4], head[4], tail[4];
      int32_t rid[4];
      float w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t q = q0 + j;
        valid[j] = q >= B && q < E;
        w[j] = valid[j] ? __ldg(weights + q) : 0.f;
        rid[j] = valid[j] ? __ldg(ray_id + q) : -1;
      }
      int32_t prev = __shfl_up_sync(kFull, rid[3], 1);
      if (lane == 0) prev = carry_rid;
      int32_t next = __shfl_down_sync(kFull, rid[0], 1);
      if (lane == 31) next = (q0 + 4 < E) ? __ldg(ray_id + q0 + 4) : -2;
      carry_rid = __shfl_sync(kFull, rid[3], 31);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int32_t pr = j == 0 ? prev : rid[j - 1];
        const int32_t nx = j == 3 ? next : (valid[j + 1] ? rid[j + 1] : -2);
        head[j] = valid[j] && (q0 + j == B || rid[j] != pr);
        tail[j] = valid[j] && (q0 + j + 1 == E || rid[j] != nx);
      }
      Seg<kC> cur = seg_identity<kC>(), lead;
      int32_t lead_r = -1;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        Seg<kC> x;
        x.f = head[j];
#pragma unroll
        for (int c = 0; c < kC; ++c)
          x.v[c] = valid[j] ? (double)w[j] * (values ? (double)__ldg(values + (q0 + j) * kC + c) : 1.0) : 0.0;
        cur = seg_combine(cur, x);
        if (tail[j]) {
          if (cur.f) {
#pragma unroll
            for (int c = 0; c < kC; ++c) out[(int64_t)rid[j] * kC + c] = (float)cur.v[c];
          } else {
            lead = cur;
            lead_r = rid[j];
          }
        }
      }
      const Seg<kC> enter = warp_seg_excl<kC>(cur, carry);
      if (lead_r >= 0) {
        const Seg<kC> t = seg_combine(enter, lead);
#pragma unroll
        for (int c = 0; c < kC; ++c) out[(int64_t)lead_r * kC + c] = (float)t.v[c];
      }
    }
  }
}

// its backward needs no scan: g_w_i = Σ_c g_out[r_i][c] v_i[c], g_v_i = w_i g_out[r_i], one
// thread per sample with the sample's ray from ray_id
__global__ void __launch_bounds__(256) accumulate_bwd_flat_kernel(const int32_t *__restrict__ ray_id,
                                                                  int64_t n_samples, const float *__restrict__ weights,
                                                                  const float *__restrict__ values, int C,
                                                                  const float *__restrict__ g_out,
                                                                  float *__restrict__ g_weights,
                                                                  float *__restrict__ g_values) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n_samples;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = __ldg(ray_id + q);
    const float w = __ldg(weights + q);
    double gw = 0.0;
    for (int c = 0; c < C; ++c) {
      const float g = __ldg(g_out + r * C + c);
      gw += (double)g * (values ? (double)__ldg(values + q * C + c) : 1.0);
      if (g_values) g_values[q * C + c] = w * g;
    }
    if (g_weights) g_weights[q] = (float)gw;
  }
}

// Alpha compositing forward on the ray-aligned flat tiles: an fp64 segmented exclusive product
// scan of (1 - α) (lane-sequential over 4 samples, then across the warp with the chunk carry);
// w = T α unless T < ε_T.  Needs ray_id and the contiguous packing.
struct SegP {
  int f;
  double v;
};
__device__ __forceinline__ SegP segp_combine(const SegP &a, const SegP &b) {
  return SegP{a.f | b.f, b.f ? b.v : a.v * b.v};
}
__device__ __forceinline__ SegP warp_segp_excl(const SegP &x, SegP &carry) {
  const int lane = threadIdx.x & 31;
  SegP incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    SegP y;
    y.f = __shfl_up_sync(kFull, incl.f, o);
    y.v = __shfl_up_sync(kFull, incl.v, o);
    if (lane >= o) incl = segp_combine(y, incl);
  }
  SegP ex{__shfl_up_sync(kFull, incl.f, 1), __shfl_up_sync(kFull, incl.v, 1)};
  if (lane == 0) ex = SegP{0, 1.0};
  const SegP res = segp_combine(carry, ex);
  carry = segp_combine(carry, SegP{__shfl_sync(kFull, incl.f, 31), __shfl_sync(kFull, incl.v, 31)});
  return res;
}

template <bool kVec>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) weights_alpha_fwd_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ alphas, double eps_T, float *__restrict__ weights, float *__restrict__ trans) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);
  for (int64_t wt = gw; wt * kWarpTile < N; wt += nw) {
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTile, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTile, N);
    if (B >= E) continue;
    SegP carry{0, 1.0};
    int32_t carry_rid = -1;
    for (int64_t c0 = B & ~(int64_t)3; c0 < E; c0 += kWarpChunk) {
      const int64_t q0 = c0 + (int64_t)lane * 4;
      bool valid[4], head[4];
      int32_t rid[4];
      float a[4];
      const bool full = kVec && q0 >= B && q0 + 3 < E;
      if (full) {
        const float4 av = __ldg(reinterpret_cast<const float4 *>(alphas + q0));
        const int4 rv = __ldg(reinterpret_cast<const int4 *>(ray_id + q0));
        a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
        rid[0] = rv.x; rid[1] = rv.y; rid[2] = rv.z; rid[3] = rv.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) valid[j] = true;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t q = q0 + j;
          valid[j] = q >= B && q < E;
          a[j] = valid[j] ? __ldg(alphas + q) : 0.f;
          rid[j] = valid[j] ? __ldg(ray_id + q) : -1;
        }
      }
      int32_t prev = __shfl_up_sync(kFull, rid[3], 1);
      if (lane == 0) prev = carry_rid;
      carry_rid = __shfl_sync(kFull, rid[3], 31);
      SegP agg{0, 1.0};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        head[j] = valid[j] && (q0 + j == B || rid[j] != (j == 0 ? prev : rid[j - 1]));
        agg = segp_combine(agg, SegP{head[j], 1.0 - (double)a[j]});
      }
      SegP run = warp_segp_excl(agg, carry);
      float wv[4], tv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double T = head[j] ? 1.0 : run.v;
        run.v = T * (1.0 - (double)a[j]);
        wv[j] = !(T < eps_T) ? (float)(T * (double)a[j]) : 0.f;
        tv[j] = (float)T;
      }
      if (full) {
        *reinterpret_cast<float4 *>(weights + q0) = make_float4(wv[0], wv[1], wv[2], wv[3]);
        if (trans) *reinterpret_cast<float4 *>(trans + q0) = make_float4(tv[0], tv[1], tv[2], tv[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!valid[j]) continue;
          weights[q0 + j] = wv[j];
          if (trans) trans[q0 + j] = tv[j];
        }
      }
    }
  }
}

// Granular weights backward on the flat tiles (samples with ray_id): pass 1 over the warp's tile
// sums v = g_w w + g_T T per ray (lane sums, the leading run through the warp scan) into the
// workspace R[ray]; pass 2 recomputes S, T, w and the inclusive prefix P of v, Q = R - P is
// Σ_{j>i} v_j, g_σ = δ (g_w T (1 - α)[live] - Q).  The tile owns whole rays, so a warp reads only
// the R it wrote.
template <bool kVec>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) weights_bwd_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ t0, const float *__restrict__ t1, const float *__restrict__ sigma, double L,
    const float *__restrict__ g_weights, const float *__restrict__ g_trans, float *__restrict__ g_sigma,
    double *__restrict__ Rws) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);
  auto gload4 = [&](const float *__restrict__ a, const Items &it, float o[4]) {
    if (kVec && it.valid[0] && it.valid[3]) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(a + it.q0));
      o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = it.valid[j] ? __ldg(a + it.q0 + j) : 0.f;
    }
  };
  for (int64_t wt = gw; wt * kWarpTile < N; wt += nw) {
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTile, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTile, N);
    if (B >= E) continue;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      Seg<1> carryS = seg_identity<1>(), carryV = seg_identity<1>();
      int32_t carry_rid = -1;
      for (int64_t c0 = B & ~(int64_t)3; c0 < E; c0 += kWarpChunk) {
        Items it;
        load_items_warp<kVec>(it, c0, B, E, t0, t1, sigma, ray_id, carry_rid);
        double s[4], S[4];
        warp_items_S(it, s, S, carryS);
        float gwv[4], gtv[4] = {0.f, 0.f, 0.f, 0.f};
        gload4(g_weights, it, gwv);
        if (g_trans) gload4(g_trans, it, gtv);
        double v[4], gwTea[4];
        double Tn = trans_first(S[0]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double ea = interval_ea(s[j]);
          const double T = (j > 0 && it.head[j]) ? 1.0 : Tn;
          Tn = T * ea;
          const bool live = it.valid[j] && !(S[j] > L);
          v[j] = it.valid[j] ? (live ? (double)gwv[j] * (T * (1.0 - ea)) : 0.0) + (double)gtv[j] * T : 0.0;
          gwTea[j] = live ? (double)gwv[j] * T * ea : 0.0;
        }
        if (pass == 0) {  // per-ray totals R into the workspace
          Seg<1> cur = seg_identity<1>(), lead;
          int32_t lead_r = -1;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            Seg<1> x;
            x.f = it.head[j];
            x.v[0] = v[j];
            cur = seg_combine(cur, x);
            if (it.tail[j]) {
              if (cur.f) Rws[it.rid[j]] = cur.v[0];
              else {
                lead = cur;
                lead_r = it.rid[j];
              }
            }
          }
          const Seg<1> enter = warp_seg_excl<1>(cur, carryV);
          if (lead_r >= 0) Rws[lead_r] = seg_combine(enter, lead).v[0];
        } else {  // gradients from Q = R - P (inclusive prefix of v)
          Seg<1> agg = seg_identity<1>();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            Seg<1> x;
            x.f = it.head[j];
            x.v[0] = v[j];
            agg = seg_combine(agg, x);
          }
          Seg<1> run = warp_seg_excl<1>(agg, carryV);
          float gs[4];
          int32_t cr = -1;
          double R = 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            run.v[0] = (it.head[j] ? 0.0 : run.v[0]) + v[j];
            gs[j] = 0.f;
            if (it.valid[j]) {
              if (it.rid[j] != cr) {
                R = Rws[it.rid[j]];
                cr = it.rid[j];
              }
              gs[j] = (float)(((double)it.t1[j] - (double)it.t0[j]) * (gwTea[j] - (R - run.v[0])));
            }
          }
          if (kVec && it.valid[0] && it.valid[3]) {
            *reinterpret_cast<float4 *>(g_sigma + it.q0) = make_float4(gs[0], gs[1], gs[2], gs[3]);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (it.valid[j]) g_sigma[it.q0 + j] = gs[j];
          }
        }
      }
      __syncwarp();  // pass 2 reads the totals this warp wrote in pass 1
    }
  }
}

// Alpha compositing backward on the flat tiles (samples with ray_id).  Per warp tile: a forward
// pass stores T (fp64 segmented product scan of 1 - α) to the workspace; a reverse pass over the
// tile's chunks forms Λ_k = Σ_{i>k} ([live_i] g_w_i α_i + g_T_i) Π_{k<j<i} (1 - α_j) by suffix
// composition of the affine maps x -> c + (1 - α) x (division-free, α = 1 safe), a ray's head
// resetting the map to the constant 0 (so no segment flags are needed across lanes), and
// g_α = [live] g_w T - T Λ.  T is read back through L2 (__ldcg): another warp's reverse pass may
// have cached a shared line in L1 before this warp wrote it.
template <bool kVec>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) weights_alpha_bwd_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ alphas, double eps_T, const float *__restrict__ g_weights,
    const float *__restrict__ g_trans, double *__restrict__ T64, float *__restrict__ g_alphas) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);
  auto load4 = [&](const int32_t *ri, const float *a, int64_t q0, int64_t B, int64_t E, float av[4], int32_t rid[4],
                   bool valid[4]) {
    if (kVec && q0 >= B && q0 + 3 < E) {
      const float4 x = __ldg(reinterpret_cast<const float4 *>(a + q0));
      const int4 y = __ldg(reinterpret_cast<const int4 *>(ri + q0));
      av[0] = x.x; av[1] = x.y; av[2] = x.z; av[3] = x.w;
      rid[0] = y.x; rid[1] = y.y; rid[2] = y.z; rid[3] = y.w;
#pragma unroll
      for (int j = 0; j < 4; ++j) valid[j] = true;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        valid[j] = q0 + j >= B && q0 + j < E;
        av[j] = valid[j] ? __ldg(a + q0 + j) : 0.f;
        rid[j] = valid[j] ? __ldg(ri + q0 + j) : -1;
      }
    }
  };
  for (int64_t wt = gw; wt * kWarpTile < N; wt += nw) {
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTile, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTile, N);
    if (B >= E) continue;
    const int64_t cfirst = B & ~(int64_t)3;
    // forward: T of every sample of the tile
    SegP carry{0, 1.0};
    int32_t carry_rid = -1;
    for (int64_t c0 = cfirst; c0 < E; c0 += kWarpChunk) {
      const int64_t q0 = c0 + (int64_t)lane * 4;
      float a[4];
      int32_t rid[4];
      bool valid[4];
      load4(ray_id, alphas, q0, B, E, a, rid, valid);
      int32_t prev = __shfl_up_sync(kFull, rid[3], 1);
      if (lane == 0) prev = carry_rid;
      carry_rid = __shfl_sync(kFull, rid[3], 31);
      bool head[4];
      SegP agg{0, 1.0};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        head[j] = valid[j] && (q0 + j == B || rid[j] != (j == 0 ? prev : rid[j - 1]));
        agg = segp_combine(agg, SegP{head[j], 1.0 - (double)a[j]});
      }
      SegP run = warp_segp_excl(agg, carry);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double T = head[j] ? 1.0 : run.v;
        run.v = T * (1.0 - (double)a[j]);
        if (valid[j]) T64[q0 + j] = T;
      }
    }
    __syncwarp();
    // reverse: Λ by suffix composition, chunk by chunk from the tile's end
    double lam_carry = 0.0;  // Λ entering the chunk from its right (0 at the tile's end: a ray ends there)
    const int64_t clast = cfirst + ((E - 1 - cfirst) / kWarpChunk) * kWarpChunk;
    for (int64_t c0 = clast; c0 >= cfirst; c0 -= kWarpChunk) {
      const int64_t q0 = c0 + (int64_t)lane * 4;
      float a[4];
      int32_t rid[4];
      bool valid[4];
      load4(ray_id, alphas, q0, B, E, a, rid, valid);
      // the previous sample's ray (for the heads): item q0 - 1, from the left lane or memory
      int32_t prev = __shfl_up_sync(kFull, rid[3], 1);
      if (lane == 0) prev = (q0 > B && q0 - 1 < E) ? __ldg(ray_id + q0 - 1) : -1;
      double T[4], c[4], am[4];
      bool head[4], live[4];
      float gwv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        head[j] = valid[j] && (q0 + j == B || rid[j] != (j == 0 ? prev : rid[j - 1]));
        T[j] = valid[j] ? __ldcg(T64 + q0 + j) : 0.0;
        live[j] = valid[j] && !(T[j] < eps_T);
        gwv[j] = valid[j] ? __ldg(g_weights + q0 + j) : 0.f;
        const double gt = (valid[j] && g_trans) ? (double)__ldg(g_trans + q0 + j) : 0.0;
        am[j] = valid[j] ? 1.0 - (double)a[j] : 1.0;  // identity past the tile's end
        c[j] = (live[j] ? (double)gwv[j] * (double)a[j] : 0.0) + gt;
      }
      // the lane's map from Λ of its last item to Λ of the sample before its first: through items
      // 3..0, x -> head ? 0 : c + am x
      double A = 1.0, Bv = 0.0;
#pragma unroll
      for (int j = 3; j >= 0; --j) {
        if (head[j]) {
          A = 0.0;
          Bv = 0.0;
        } else {
          Bv = c[j] + am[j] * Bv;
          A = am[j] * A;
        }
      }
      // exclusive suffix composition over the lanes to the right: X = Λ of the lane's last item
      double SA = A, SB = Bv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double a2 = __shfl_down_sync(kFull, SA, o), b2 = __shfl_down_sync(kFull, SB, o);
        if (lane + o < 32) {
          SB = SB + SA * b2;
          SA = SA * a2;
        }
      }
      double Ae = __shfl_down_sync(kFull, SA, 1), Be = __shfl_down_sync(kFull, SB, 1);
      if (lane == 31) {
        Ae = 1.0;
        Be = 0.0;
      }
      double lam = Be + Ae * lam_carry;  // Λ of item 3
      float ga[4];
#pragma unroll
      for (int j = 3; j >= 0; --j) {
        ga[j] = valid[j] ? (float)((live[j] ? (double)gwv[j] * T[j] : 0.0) - T[j] * lam) : 0.f;
        lam = head[j] ? 0.0 : c[j] + am[j] * lam;  // Λ of item j - 1
      }
      if (kVec && q0 >= B && q0 + 3 < E) {
        *reinterpret_cast<float4 *>(g_alphas + q0) = make_float4(ga[0], ga[1], ga[2], ga[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (valid[j]) g_alphas[q0 + j] = ga[j];
      }
      const double A0 = __shfl_sync(kFull, SA, 0), B0 = __shfl_sync(kFull, SB, 0);
      lam_carry = B0 + A0 * lam_carry;
    }
  }
}

// persistent grid for the tile kernels: all resident at once (3 blocks of 256 per SM)
static unsigned resident_blocks(int64_t want) {
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 1;
  }
  const int64_t cap = (int64_t)n_sm * NACC_RENDER_BPS * NACC_RENDER_GRIDX;
  return (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
}

struct RayGrad {
  double gc0, gc1, gc2, gOp, gN, R;
};

__device__ __forceinline__ RayGrad ray_grad(int64_t r, const double *__restrict__ ctx, const float *__restrict__ g_color,
                                            const float *__restrict__ g_opacity, const float *__restrict__ g_depth) {
  RayGrad q;
  const double *cx = ctx + 5 * r;
  const double C0 = __ldg(cx), C1 = __ldg(cx + 1), C2 = __ldg(cx + 2), O = __ldg(cx + 3), Nn = __ldg(cx + 4);
  q.gc0 = g_color ? (double)__ldg(g_color + 3 * r) : 0.0;
  q.gc1 = g_color ? (double)__ldg(g_color + 3 * r + 1) : 0.0;
  q.gc2 = g_color ? (double)__ldg(g_color + 3 * r + 2) : 0.0;
  const double gO = g_opacity ? (double)__ldg(g_opacity + r) : 0.0;
  const double gD = g_depth ? (double)__ldg(g_depth + r) : 0.0;
  if (O > 1e-10) {
    const double inv = 1.0 / O;
    q.gN = gD * inv;
    q.gOp = gO - gD * Nn * inv * inv;
  } else {
    q.gN = gD * 1e10;
    q.gOp = gO;
  }
  q.R = q.gc0 * C0 + q.gc1 * C1 + q.gc2 * C2 + q.gOp * O + q.gN * Nn;
  return q;
}

// per-ray constants of the backward, once per ray: g_C (as floats), and
// (g_O', g_N, R) in fp64, with R = <g_C, C> + g_O' O + g_N N (see header)
__global__ void __launch_bounds__(256) ray_grad_kernel(int64_t n_rays, const double *__restrict__ ctx,
                                                       const float *__restrict__ g_color,
                                                       const float *__restrict__ g_opacity,
                                                       const float *__restrict__ g_depth, float4 *__restrict__ gcv,
                                                       double2 *__restrict__ gq) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const RayGrad q = ray_grad(r, ctx, g_color, g_opacity, g_depth);
  gcv[r] = make_float4((float)q.gc0, (float)q.gc1, (float)q.gc2, 0.f);
  gq[2 * r] = make_double2(q.gOp, q.gN);
  gq[2 * r + 1] = make_double2(q.R, 0.0);
}

// kColorOnly (g_opacity = g_depth = NULL, the colour-loss case): g_O' = g_N = 0, so the per-ray
// constants are g_C itself and R = <g_C, C>, read directly (g_color, ctx) instead of from the
// ray_grad_kernel workspace, whose launch and 100 B per ray are skipped; the arithmetic is the same
// (the zero terms add +0).
template <bool kVec, bool kColorOnly = false>
__global__ void __launch_bounds__(256, NACC_RENDER_BPS) render_bwd_warp_kernel(
    const int64_t *__restrict__ packed_info, const int32_t *__restrict__ ray_id, int64_t n_rays, int64_t n_samples,
    const float *__restrict__ t0, const float *__restrict__ t1, const float *__restrict__ sigma,
    const float *__restrict__ rgb, double L, const float4 *__restrict__ gcv, const double2 *__restrict__ gq,
    float *__restrict__ g_sigma, float *__restrict__ g_rgb, const float *__restrict__ g_color = nullptr,
    const double *__restrict__ ctx = nullptr) {
  auto ray_gc = [&](int32_t r) {
    if (kColorOnly)
      return make_float4(__ldg(g_color + 3 * (int64_t)r), __ldg(g_color + 3 * (int64_t)r + 1),
                         __ldg(g_color + 3 * (int64_t)r + 2), 0.f);
    return __ldg(gcv + r);
  };
  auto ray_R = [&](int32_t r, const float4 &gc) {
    if (kColorOnly) {
      const double *cx = ctx + 5 * (int64_t)r;
      return (double)gc.x * __ldg(cx) + (double)gc.y * __ldg(cx + 1) + (double)gc.z * __ldg(cx + 2);
    }
    return __ldg(gq + 2 * (int64_t)r + 1).x;
  };
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t N = min(packed_end(packed_info, n_rays), n_samples);  // in bounds after an overflowed march
  for (int64_t wt = gw; wt * kWarpTileBwd < N; wt += nw) {
    prefetch_tile(wt + nw, N, t0, t1, sigma, ray_id, rgb, kWarpTileBwd);
    const int64_t B = snap_to_ray(packed_info, ray_id, wt * kWarpTileBwd, N);
    const int64_t E = snap_to_ray(packed_info, ray_id, (wt + 1) * kWarpTileBwd, N);
    if (B >= E) continue;
    Seg<1> carryS = seg_identity<1>(), carryP = seg_identity<1>();
    int32_t carry_rid = -1;
    for (int64_t c0 = B & ~(int64_t)3; c0 < E; c0 += kWarpChunk) {
      Items it;
      load_items_warp<kVec>(it, c0, B, E, t0, t1, sigma, ray_id, carry_rid);
      double s[4], S[4];
      warp_items_S(it, s, S, carryS);
      // phase A: per item g_w w (scan input), w and g_w T (1-α); the only state kept
      double w[4], gwTea[4];
      unsigned live = 0;
      Seg<1> agg = seg_identity<1>();
      {
        float col[12];
        load_rgb4(col, it, rgb, kVec);
        double Tn = trans_first(S[0]);  // T_{j+1} = T_j e^{-s_j}, as in the forward
        // per-ray constants, loaded once per run of the ray within the thread's items
        int32_t cr = -1;
        float4 gc = make_float4(0.f, 0.f, 0.f, 0.f);
        double2 gon = make_double2(0.0, 0.0);
  #pragma unroll
        for (int j = 0; j < 4; ++j) {
          w[j] = 0.0;
          gwTea[j] = 0.0;
          double v = 0.0;
          const double ea = interval_ea(s[j]);
          const double T = NACC_RENDER_TPROD ? ((j > 0 && it.head[j]) ? 1.0 : Tn) : exp(-S[j]);
          Tn = T * ea;
          if (it.valid[j] && !(S[j] > L)) {
            live |= 1u << j;
            if (!NACC_RENDER_RAYCACHE || it.rid[j] != cr) {
              gc = ray_gc(it.rid[j]);
              if (!kColorOnly) gon = __ldg(gq + 2 * (int64_t)it.rid[j]);
              cr = it.rid[j];
            }
            w[j] = T * (1.0 - ea);
            const double gw =
                kColorOnly ? (double)gc.x * col[3 * j] + (double)gc.y * col[3 * j + 1] + (double)gc.z * col[3 * j + 2]
                           : (double)gc.x * col[3 * j] + (double)gc.y * col[3 * j + 1] + (double)gc.z * col[3 * j + 2] +
                                 gon.x + gon.y * (0.5 * ((double)it.t0[j] + (double)it.t1[j]));
            v = gw * w[j];
            gwTea[j] = gw * T * ea;
          }
          s[j] = v;
          Seg<1> x;
          x.f = it.head[j];
          x.v[0] = v;
          agg = seg_combine(agg, x);
        }
      }
      Seg<1> run = warp_seg_excl<1>(agg, carryP);
      float gs[4], gr[12];
      int32_t cr = -1;
      float4 gc = make_float4(0.f, 0.f, 0.f, 0.f);
      double R = 0.0;
  #pragma unroll
      for (int j = 0; j < 4; ++j) {
        run.v[0] = (it.head[j] ? 0.0 : run.v[0]) + s[j];
        gs[j] = 0.f;
        gr[3 * j] = gr[3 * j + 1] = gr[3 * j + 2] = 0.f;
        if (live & (1u << j)) {
          if (!NACC_RENDER_RAYCACHE || it.rid[j] != cr) {
            gc = ray_gc(it.rid[j]);
            R = ray_R(it.rid[j], gc);
            cr = it.rid[j];
          }
          const double Q = R - run.v[0];  // Σ_{i>j} g_w_i w_i of the ray
          gs[j] = (float)(((double)it.t1[j] - (double)it.t0[j]) * (gwTea[j] - Q));
          gr[3 * j] = (float)(w[j] * gc.x);
          gr[3 * j + 1] = (float)(w[j] * gc.y);
          gr[3 * j + 2] = (float)(w[j] * gc.z);
        }
      }
      if (kVec && it.valid[0] && it.valid[3]) {
        *reinterpret_cast<float4 *>(g_sigma + it.q0) = make_float4(gs[0], gs[1], gs[2], gs[3]);
        if (g_rgb) {
          float4 *pp = reinterpret_cast<float4 *>(g_rgb + 3 * it.q0);
          pp[0] = make_float4(gr[0], gr[1], gr[2], gr[3]);
          pp[1] = make_float4(gr[4], gr[5], gr[6], gr[7]);
          pp[2] = make_float4(gr[8], gr[9], gr[10], gr[11]);
        }
      } else {
  #pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!it.valid[j]) continue;
          g_sigma[it.q0 + j] = gs[j];
          if (g_rgb)
  #pragma unroll
            for (int ch = 0; ch < 3; ++ch) g_rgb[3 * (it.q0 + j) + ch] = gr[3 * j + ch];
        }
      }
    }
  }
}

// ------------------------------------------------------------------ granular weights
__global__ void __launch_bounds__(256) weights_fwd_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                          const float *__restrict__ t0, const float *__restrict__ t1,
                                                          const float *__restrict__ sigma, double L,
                                                          float *__restrict__ weights, float *__restrict__ trans,
                                                          float *__restrict__ alphas) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  double carry = 0.0;
  for (int64_t base = 0; base < cnt; base += 32) {
    const Chunk c = load_chunk(t0, t1, sigma, st, cnt, base, L, carry);
    if (c.valid) {
      const int64_t q = st + base + lane;
      const double T = trans_of(c.S), a = alpha_of(c.s);
      weights[q] = c.live ? (float)(T * a) : 0.f;
      if (trans) trans[q] = (float)T;
      if (alphas) alphas[q] = (float)a;
    }
  }
}

__global__ void __launch_bounds__(256) weights_bwd_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                          const float *__restrict__ t0, const float *__restrict__ t1,
                                                          const float *__restrict__ sigma, double L,
                                                          const float *__restrict__ g_weights,
                                                          const float *__restrict__ g_trans,
                                                          float *__restrict__ g_sigma) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  // pass 1: R = Σ_j (g_w_j w_j + g_T_j T_j)
  double carry = 0.0, R = 0.0;
  for (int64_t base = 0; base < cnt; base += 32) {
    const Chunk c = load_chunk(t0, t1, sigma, st, cnt, base, L, carry);
    if (c.valid) {
      const int64_t q = st + base + lane;
      const double T = trans_of(c.S);
      if (c.live) R += (double)__ldg(g_weights + q) * (T * alpha_of(c.s));
      if (g_trans) R += (double)__ldg(g_trans + q) * T;
    }
  }
  R = warp_sum(R);
  // pass 2: prefix P_i = Σ_{j<=i}, Q_i = R - P_i
  carry = 0.0;
  double P = 0.0;
  for (int64_t base = 0; base < cnt; base += 32) {
    const Chunk c = load_chunk(t0, t1, sigma, st, cnt, base, L, carry);
    const int64_t q = st + base + lane;
    double v = 0.0, gwTa = 0.0;
    if (c.valid) {
      const double T = trans_of(c.S);
      const double gw = (double)__ldg(g_weights + q);
      if (c.live) {
        v += gw * (T * alpha_of(c.s));
        gwTa = gw * T * exp(-c.s);
      }
      if (g_trans) v += (double)__ldg(g_trans + q) * T;
    }
    const double incl = warp_incl_scan(v);
    const double Q = R - (P + incl);
    P += __shfl_sync(kFull, incl, 31);
    if (c.valid) g_sigma[q] = (float)(c.delta * (gwTa - Q));
  }
}

// ------------------------------------------------------------------ alpha compositing
// One warp per ray, chunks of 32 samples (readings #16-#17).  Forward: fp64
// multiplicative warp scan of (1 − α) carried across chunks.  Backward: pass 1
// recomputes T into the fp64 workspace; pass 2 walks the chunks from the end
// with a warp suffix scan of the affine maps x -> c_k + (1 − α_k) x, which
// yields Λ_k = Σ_{i>k} c_i Π_{k<j<i} (1 − α_j) without any division.
__device__ __forceinline__ double warp_excl_prod(double v, double &total) {
  const int lane = threadIdx.x & 31;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl *= y;
  }
  double ex = __shfl_up_sync(kFull, incl, 1);
  if (lane == 0) ex = 1.0;
  total = __shfl_sync(kFull, incl, 31);
  return ex;
}

__global__ void __launch_bounds__(256) weights_alpha_fwd_kernel(const int64_t *__restrict__ packed_info,
                                                                int64_t n_rays, const float *__restrict__ alphas,
                                                                double eps_T, float *__restrict__ weights,
                                                                float *__restrict__ trans,
                                                                double *__restrict__ trans64) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  double carry = 1.0;
  for (int64_t base = 0; base < cnt; base += 32) {
    const int64_t i = base + lane, q = st + i;
    const bool valid = i < cnt;
    const double a = valid ? (double)__ldg(alphas + q) : 0.0;
    double tot;
    const double T = carry * warp_excl_prod(1.0 - a, tot);
    carry *= tot;
    if (valid) {
      if (weights) weights[q] = !(T < eps_T) ? (float)(T * a) : 0.f;
      if (trans) trans[q] = (float)T;
      if (trans64) trans64[q] = T;
    }
  }
}

__global__ void __launch_bounds__(256) weights_alpha_bwd_kernel(const int64_t *__restrict__ packed_info,
                                                                int64_t n_rays, const float *__restrict__ alphas,
                                                                double eps_T, const float *__restrict__ g_weights,
                                                                const float *__restrict__ g_trans,
                                                                const double *__restrict__ trans64,
                                                                float *__restrict__ g_alphas) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  double carry = 0.0;  // Λ of the last sample before the chunk processed next = M of its first sample
  for (int64_t base = ((cnt - 1) / 32) * 32; base >= 0 && cnt > 0; base -= 32) {
    const int64_t i = base + lane, q = st + i;
    const bool valid = i < cnt;
    double a = 1.0, c = 0.0, T = 0.0, gw = 0.0;  // identity map past the ray's end
    bool live = false;
    if (valid) {
      const double al = (double)__ldg(alphas + q);
      T = __ldg(trans64 + q);
      live = !(T < eps_T);
      gw = (double)__ldg(g_weights + q);
      a = 1.0 - al;
      c = (live ? gw * al : 0.0) + (g_trans ? (double)__ldg(g_trans + q) : 0.0);
    }
    // suffix composition of x -> c + a x over lanes lane..31 (inclusive)
    double A = a, Bv = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double a2 = __shfl_down_sync(kFull, A, o), b2 = __shfl_down_sync(kFull, Bv, o);
      if (lane + o < 32) {
        Bv = Bv + A * b2;
        A = A * a2;
      }
    }
    // Λ_k = (maps of lanes > lane) applied to the carry: exclusive suffix
    double Ae = __shfl_down_sync(kFull, A, 1), Be = __shfl_down_sync(kFull, Bv, 1);
    if (lane == 31) {
      Ae = 1.0;
      Be = 0.0;
    }
    const double Lam = Be + Ae * carry;
    if (valid) g_alphas[q] = (float)((live ? gw * T : 0.0) - T * Lam);
    const double A0 = __shfl_sync(kFull, A, 0), B0 = __shfl_sync(kFull, Bv, 0);
    carry = B0 + A0 * carry;
  }
}

// ------------------------------------------------------------------ accumulate_along_rays
template <int kC>
__global__ void __launch_bounds__(256) accumulate_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                         const float *__restrict__ weights,
                                                         const float *__restrict__ values, int C,
                                                         float *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  if (kC > 0) {
    double acc[kC > 0 ? kC : 1];
#pragma unroll
    for (int c = 0; c < kC; ++c) acc[c] = 0.0;
    for (int64_t i = lane; i < cnt; i += 32) {
      const int64_t q = st + i;
      const double w = (double)__ldg(weights + q);
#pragma unroll
      for (int c = 0; c < kC; ++c) acc[c] += w * (values ? (double)__ldg(values + q * kC + c) : 1.0);
    }
#pragma unroll
    for (int c = 0; c < kC; ++c) {
      const double v = warp_sum(acc[c]);
      if (lane == 0) out[r * kC + c] = (float)v;
    }
  } else {
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int64_t i = lane; i < cnt; i += 32) {
        const int64_t q = st + i;
        acc += (double)__ldg(weights + q) * (double)__ldg(values + q * C + c);
      }
      acc = warp_sum(acc);
      if (lane == 0) out[r * C + c] = (float)acc;
    }
  }
}

__global__ void __launch_bounds__(256) accumulate_bwd_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                             const float *__restrict__ weights,
                                                             const float *__restrict__ values, int C,
                                                             const float *__restrict__ g_out,
                                                             float *__restrict__ g_weights,
                                                             float *__restrict__ g_values) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const longlong2 pi = reinterpret_cast<const longlong2 *>(packed_info)[r];
  const int64_t st = pi.x, cnt = pi.y;
  for (int64_t i = lane; i < cnt; i += 32) {
    const int64_t q = st + i;
    const float w = __ldg(weights + q);
    double gw = 0.0;
    for (int c = 0; c < C; ++c) {
      const float g = __ldg(g_out + r * C + c);
      gw += (double)g * (values ? (double)__ldg(values + q * C + c) : 1.0);
      if (g_values) g_values[q * C + c] = w * g;
    }
    if (g_weights) g_weights[q] = (float)gw;
  }
}

static nacc_status check_packed(const int64_t *packed_info, int64_t n_rays, int64_t n_samples) {
  NACC_REQUIRE(n_rays >= 0 && n_rays < (1ll << 31), "n_rays must be in [0, 2^31)");
  NACC_REQUIRE(n_samples >= 0, "n_samples must be >= 0");
  NACC_REQUIRE(n_rays == 0 || (packed_info && aligned(packed_info, 16)),
               "packed_info must be non-NULL and 16-byte aligned");
  return NACC_OK;
}

}  // namespace nacc

using namespace nacc;

extern "C" {

nacc_status nacc_render_fwd(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays, const float *t0,
                            const float *t1, const float *sigma, const float *rgb, int64_t n_samples,
                            double neg_log_eps, float *color, float *opacity, float *depth, double *ctx,
                            cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma), "t0, t1, sigma must be non-NULL");
  NACC_REQUIRE(!ctx || aligned(ctx, 8), "ctx must be 8-byte aligned");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  if (ray_id && rgb) {
    const int64_t n_wtiles = ceil_div(n_samples, kWarpTile);
    const int64_t warps = n_wtiles > ceil_div(n_rays, 32) ? n_wtiles : ceil_div(n_rays, 32);
    const bool vec = aligned(t0, 16) && aligned(t1, 16) && aligned(sigma, 16) && aligned(rgb, 16) &&
                     aligned(ray_id, 16);
    const unsigned blocks = resident_blocks(ceil_div(warps * 32, 256));
    if (vec)
      render_fwd_warp_kernel<true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                               rgb, neg_log_eps, color, opacity, depth, ctx);
    else
      render_fwd_warp_kernel<false><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                                rgb, neg_log_eps, color, opacity, depth, ctx);
  } else {
    render_fwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma, rgb,
                                                                       neg_log_eps, color, opacity, depth, ctx);
  }
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_bwd(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays, const float *t0,
                            const float *t1, const float *sigma, const float *rgb, int64_t n_samples,
                            double neg_log_eps, const double *ctx, const float *g_color, const float *g_opacity,
                            const float *g_depth, float *g_sigma, float *g_rgb, void *ws, size_t ws_bytes,
                            cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0 || n_samples == 0) return NACC_OK;
  NACC_REQUIRE(t0 && t1 && sigma && g_sigma, "t0, t1, sigma, g_sigma must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  if (ray_id && rgb && ctx) {
    NACC_REQUIRE(ws && ws_bytes >= nacc_render_bwd_workspace_bytes(n_rays), "workspace too small");
    float4 *gcv = static_cast<float4 *>(ws);
    double2 *gq = reinterpret_cast<double2 *>(static_cast<char *>(ws) + align_up((size_t)n_rays * 16, 256));
    const bool color_only = NACC_RENDER_COLORONLY && g_color && !g_opacity && !g_depth;
    if (!color_only)
      ray_grad_kernel<<<grid_for(n_rays, 256), 256, 0, stream>>>(n_rays, ctx, g_color, g_opacity, g_depth, gcv, gq);
    const int64_t n_wtiles = ceil_div(n_samples, kWarpTileBwd);
    const bool vec = aligned(t0, 16) && aligned(t1, 16) && aligned(sigma, 16) && aligned(rgb, 16) &&
                     aligned(ray_id, 16) && aligned(g_sigma, 16) && (!g_rgb || aligned(g_rgb, 16));
    const unsigned blocks = resident_blocks(ceil_div(n_wtiles * 32, 256));
    if (color_only && vec)
      render_bwd_warp_kernel<true, true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1,
                                                                     sigma, rgb, neg_log_eps, gcv, gq, g_sigma, g_rgb,
                                                                     g_color, ctx);
    else if (color_only)
      render_bwd_warp_kernel<false, true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1,
                                                                      sigma, rgb, neg_log_eps, gcv, gq, g_sigma, g_rgb,
                                                                      g_color, ctx);
    else if (vec)
      render_bwd_warp_kernel<true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                               rgb, neg_log_eps, gcv, gq, g_sigma, g_rgb);
    else
      render_bwd_warp_kernel<false><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                                rgb, neg_log_eps, gcv, gq, g_sigma, g_rgb);
    if (!color_only) count_launch(1);
  } else {
    render_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma, rgb,
                                                                       neg_log_eps, ctx, g_color, g_opacity, g_depth,
                                                                       g_sigma, g_rgb);
  }
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

size_t nacc_render_bwd_workspace_bytes(int64_t n_rays) {
  if (n_rays < 0) return 0;
  return align_up((size_t)n_rays * 16, 256) + (size_t)n_rays * 32 + 256;
}

nacc_status nacc_render_weights_fwd(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                                    const float *sigma, int64_t n_samples, double neg_log_eps, float *weights,
                                    float *trans, float *alphas, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma && weights), "t0, t1, sigma, weights must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  weights_fwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma,
                                                                      neg_log_eps, weights, trans, alphas);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

size_t nacc_render_weights_bwd_flat_workspace_bytes(int64_t n_rays) {
  return n_rays < 0 ? 0 : (size_t)n_rays * sizeof(double);
}

nacc_status nacc_render_weights_bwd_flat(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                                         const float *t0, const float *t1, const float *sigma, int64_t n_samples,
                                         double neg_log_eps, const float *g_weights, const float *g_trans,
                                         float *g_sigma, void *ws, size_t ws_bytes, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0 || n_samples == 0) return NACC_OK;
  NACC_REQUIRE(ray_id && t0 && t1 && sigma && g_weights && g_sigma,
               "ray_id, t0, t1, sigma, g_weights, g_sigma must be non-NULL");
  NACC_REQUIRE(ws && ws_bytes >= nacc_render_weights_bwd_flat_workspace_bytes(n_rays) && aligned(ws, 8),
               "workspace too small");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  const bool vec = aligned(t0, 16) && aligned(t1, 16) && aligned(sigma, 16) && aligned(ray_id, 16) &&
                   aligned(g_weights, 16) && (!g_trans || aligned(g_trans, 16)) && aligned(g_sigma, 16);
  const unsigned blocks = resident_blocks(ceil_div(ceil_div(n_samples, kWarpTile) * 32, 256));
  double *R = static_cast<double *>(ws);
  if (vec)
    weights_bwd_warp_kernel<true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                              neg_log_eps, g_weights, g_trans, g_sigma, R);
  else
    weights_bwd_warp_kernel<false><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                               neg_log_eps, g_weights, g_trans, g_sigma, R);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_weights_bwd(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                                    const float *sigma, int64_t n_samples, double neg_log_eps,
                                    const float *g_weights, const float *g_trans, float *g_sigma,
                                    cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma && g_weights && g_sigma),
               "t0, t1, sigma, g_weights, g_sigma must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  weights_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma,
                                                                      neg_log_eps, g_weights, g_trans, g_sigma);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_weights_fwd_flat(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                                         const float *t0, const float *t1, const float *sigma, int64_t n_samples,
                                         double neg_log_eps, float *weights, float *trans, float *alphas,
                                         cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0 || n_samples == 0) return NACC_OK;
  NACC_REQUIRE(ray_id && t0 && t1 && sigma && weights, "ray_id, t0, t1, sigma, weights must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  const int64_t n_wtiles = ceil_div(n_samples, kWarpTile);
  const bool vec = aligned(t0, 16) && aligned(t1, 16) && aligned(sigma, 16) && aligned(ray_id, 16) &&
                   aligned(weights, 16) && (!trans || aligned(trans, 16)) && (!alphas || aligned(alphas, 16));
  const unsigned blocks = resident_blocks(ceil_div(n_wtiles * 32, 256));
  if (vec)
    weights_fwd_warp_kernel<true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                              neg_log_eps, weights, trans, alphas);
  else
    weights_fwd_warp_kernel<false><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, t0, t1, sigma,
                                                               neg_log_eps, weights, trans, alphas);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_weights_alpha_fwd_flat(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                                               const float *alphas, int64_t n_samples, double neg_log_eps,
                                               float *weights, float *trans, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0 || n_samples == 0) return NACC_OK;
  NACC_REQUIRE(ray_id && alphas && weights, "ray_id, alphas and weights must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_alpha(alphas, n_samples, stream));
  const bool vec = aligned(alphas, 16) && aligned(ray_id, 16) && aligned(weights, 16) && (!trans || aligned(trans, 16));
  const unsigned blocks = resident_blocks(ceil_div(ceil_div(n_samples, kWarpTile) * 32, 256));
  if (vec)
    weights_alpha_fwd_warp_kernel<true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, alphas,
                                                                     std::exp(-neg_log_eps), weights, trans);
  else
    weights_alpha_fwd_warp_kernel<false><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, alphas,
                                                                      std::exp(-neg_log_eps), weights, trans);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_weights_alpha_fwd(const int64_t *packed_info, int64_t n_rays, const float *alphas,
                                          int64_t n_samples, double neg_log_eps, float *weights, float *trans,
                                          cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (alphas && weights), "alphas and weights must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_alpha(alphas, n_samples, stream));
  weights_alpha_fwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, alphas,
                                                                            std::exp(-neg_log_eps), weights, trans,
                                                                            nullptr);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

size_t nacc_render_weights_alpha_bwd_workspace_bytes(int64_t n_samples) {
  return n_samples > 0 ? align_up((size_t)n_samples * 8, 256) : 256;
}

nacc_status nacc_render_weights_alpha_bwd_flat(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                                               const float *alphas, int64_t n_samples, double neg_log_eps,
                                               const float *g_weights, const float *g_trans, float *g_alphas,
                                               void *ws, size_t ws_bytes, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0 || n_samples == 0) return NACC_OK;
  NACC_REQUIRE(ray_id && alphas && g_weights && g_alphas, "ray_id, alphas, g_weights, g_alphas must be non-NULL");
  NACC_REQUIRE(ws && ws_bytes >= nacc_render_weights_alpha_bwd_workspace_bytes(n_samples) && aligned(ws, 8),
               "workspace too small");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_alpha(alphas, n_samples, stream));
  const double eps_T = std::exp(-neg_log_eps);
  const bool vec = aligned(alphas, 16) && aligned(ray_id, 16) && aligned(g_alphas, 16);
  const unsigned blocks = resident_blocks(ceil_div(ceil_div(n_samples, kWarpTile) * 32, 256));
  double *T64 = static_cast<double *>(ws);
  if (vec)
    weights_alpha_bwd_warp_kernel<true><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, alphas,
                                                                     eps_T, g_weights, g_trans, T64, g_alphas);
  else
    weights_alpha_bwd_warp_kernel<false><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, alphas,
                                                                      eps_T, g_weights, g_trans, T64, g_alphas);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_weights_alpha_bwd(const int64_t *packed_info, int64_t n_rays, const float *alphas,
                                          int64_t n_samples, double neg_log_eps, const float *g_weights,
                                          const float *g_trans, float *g_alphas, void *ws, size_t ws_bytes,
                                          cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (alphas && g_weights && g_alphas), "alphas, g_weights, g_alphas must be non-NULL");
  NACC_REQUIRE(ws && ws_bytes >= nacc_render_weights_alpha_bwd_workspace_bytes(n_samples) && aligned(ws, 8),
               "workspace too small");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_alpha(alphas, n_samples, stream));
  const double eps_T = std::exp(-neg_log_eps);
  double *T64 = static_cast<double *>(ws);
  weights_alpha_fwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, alphas, eps_T,
                                                                            nullptr, nullptr, T64);
  weights_alpha_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, alphas, eps_T,
                                                                            g_weights, g_trans, T64, g_alphas);
  count_launch(2);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_accumulate_along_rays(const int64_t *packed_info, int64_t n_rays, const float *weights,
                                       const float *values, int32_t C, int64_t n_samples, float *out,
                                       cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(C >= 1 && C <= 64, "C must be in 1..64");
  NACC_REQUIRE(values || C == 1, "values == NULL requires C == 1");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(out && (n_samples == 0 || weights), "weights and out must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  const int blocks = grid_for(n_rays * 32, 256);
  switch (C) {
    case 1: accumulate_kernel<1><<<blocks, 256, 0, stream>>>(packed_info, n_rays, weights, values, C, out); break;
    case 2: accumulate_kernel<2><<<blocks, 256, 0, stream>>>(packed_info, n_rays, weights, values, C, out); break;
    case 3: accumulate_kernel<3><<<blocks, 256, 0, stream>>>(packed_info, n_rays, weights, values, C, out); break;
    case 4: accumulate_kernel<4><<<blocks, 256, 0, stream>>>(packed_info, n_rays, weights, values, C, out); break;
    default: accumulate_kernel<0><<<blocks, 256, 0, stream>>>(packed_info, n_rays, weights, values, C, out); break;
  }
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_accumulate_along_rays_flat(const int64_t *packed_info, const int32_t *ray_id, int64_t n_rays,
                                            const float *weights, const float *values, int32_t C, int64_t n_samples,
                                            float *out, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(C >= 1 && C <= 64, "C must be in 1..64");
  NACC_REQUIRE(values || C == 1, "values == NULL requires C == 1");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(out && (n_samples == 0 || (weights && ray_id)), "weights, ray_id and out must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  if (C > 4 || n_samples == 0) return nacc_accumulate_along_rays(packed_info, n_rays, weights, values, C, n_samples,
                                                                 out, stream);
  const unsigned blocks = resident_blocks(std::max(ceil_div(n_samples, kWarpTile), ceil_div(n_rays, 32)) * 32 / 256 + 1);
  switch (C) {
    case 1: accumulate_warp_kernel<1><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, weights, values, out); break;
    case 2: accumulate_warp_kernel<2><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, weights, values, out); break;
    case 3: accumulate_warp_kernel<3><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, weights, values, out); break;
    default: accumulate_warp_kernel<4><<<blocks, 256, 0, stream>>>(packed_info, ray_id, n_rays, n_samples, weights, values, out); break;
  }
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_accumulate_along_rays_bwd_flat(const int32_t *ray_id, int64_t n_rays, const float *weights,
                                                const float *values, int32_t C, int64_t n_samples,
                                                const float *g_out, float *g_weights, float *g_values,
                                                cudaStream_t stream) {
  clear_error();
  NACC_REQUIRE(n_rays >= 0 && n_rays < (1ll << 31) && n_samples >= 0, "sizes must be >= 0 (n_rays < 2^31)");
  NACC_REQUIRE(C >= 1 && C <= 64, "C must be in 1..64");
  NACC_REQUIRE(values || (C == 1 && !g_values), "values == NULL requires C == 1 and g_values == NULL");
  if (n_rays == 0 || n_samples == 0) return NACC_OK;
  NACC_REQUIRE(ray_id && weights && g_out, "ray_id, weights and g_out must be non-NULL");
  const int64_t blocks = std::min(ceil_div(n_samples, (int64_t)256), (int64_t)148 * 16);
  accumulate_bwd_flat_kernel<<<(unsigned)blocks, 256, 0, stream>>>(ray_id, n_samples, weights, values, C, g_out,
                                                                   g_weights, g_values);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_accumulate_along_rays_bwd(const int64_t *packed_info, int64_t n_rays, const float *weights,
                                           const float *values, int32_t C, int64_t n_samples, const float *g_out,
                                           float *g_weights, float *g_values, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(C >= 1 && C <= 64, "C must be in 1..64");
  NACC_REQUIRE(values || (C == 1 && !g_values), "values == NULL requires C == 1 and g_values == NULL");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(g_out && (n_samples == 0 || weights), "weights and g_out must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, nullptr, nullptr, n_samples, stream));
  accumulate_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, weights, values, C,
                                                                         g_out, g_weights, g_values);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

}  // extern "C"
