// resample.cu — the proposal estimator's inverse-transform sampling
// (Eq. 1) of the CDF F = 1 - T (Eq. 3; "compute
// the CDF directly using 1 - T(t)"), piecewise linear in s (P:257,
// readings #16-#19).  One warp per ray; the ray's normalised CDF lives in
// shared memory, each lane inverts 1/32 of the output edges by binary search.
#include <type_traits>

#include "common.cuh"
#include "debug.cuh"

namespace nacc {

// 1/x for x in the fp32 normal range: fp32 reciprocal refined by one fp64 Newton step
// (relative error ~2^-46, far below the resampler's tolerances; no fp64 division)
__device__ __forceinline__ double rcp_fast(double x) {
  if (!(fabs(x) >= 1e-30 && fabs(x) <= 1e30)) return 1.0 / x;  // outside fp32's normal range (s = 1, t_f = inf)
  const double y0 = (double)__frcp_rn((float)x);
  return __fma_rn(y0, __fma_rn(-x, y0, 1.0), y0);
}

__device__ __forceinline__ double phi(int map, double s, double tn, double inv_tn, double inv_tf, double tf) {
  if (map == NACC_MAP_IDENTITY) return tn + s * (tf - tn);
  return rcp_fast((1.0 - s) * inv_tn + s * inv_tf);
}

// the same Φ when the caller knows 1/t = (1 - s)/t_n + s/t_f lies in fp32's normal range for
// every s it passes (lindisp, both 1/t_n and 1/t_f normal, s in [0, 1]): no range check
__device__ __forceinline__ double phi_normal(int map, double s, double tn, double inv_tn, double inv_tf, double tf) {
  if (map == NACC_MAP_IDENTITY) return tn + s * (tf - tn);
  const double x = (1.0 - s) * inv_tn + s * inv_tf;
  const double y0 = (double)__frcp_rn((float)x);
  return __fma_rn(y0, __fma_rn(-x, y0, 1.0), y0);
}

// 1 - e^{-S} for S >= 0 in fp32 (the CDF of Eq. 3): a degree-6 Taylor polynomial below 1/4
// (relative error < 5e-8), 1 - ex2(-S log2 e) above (F > 0.22, error < 6e-7 relative)
__device__ __forceinline__ float one_minus_exp_neg(float S) {
  if (S < 0.25f) {
    float p = 1.0f / 720.0f;
    p = __fmaf_rn(p, -S, 1.0f / 120.0f);
    p = __fmaf_rn(p, -S, 1.0f / 24.0f);
    p = __fmaf_rn(p, -S, 1.0f / 6.0f);
    p = __fmaf_rn(p, -S, 0.5f);
    p = __fmaf_rn(p, -S, 1.0f);
    return S * p;
  }
  return 1.0f - __expf(-S);
}

#ifndef NACC_RESAMPLE_WARPS
#define NACC_RESAMPLE_WARPS 4  // build parameter: rays (warps) per block
#endif
#ifndef NACC_RESAMPLE_MINB
#define NACC_RESAMPLE_MINB 11  // build parameter: min resident blocks per SM in the launch bounds (A/B: 1 / 8 / 9 / 10 / 11 / 12:
                               // 112.7/57.4, 113.0/57.4, 109.6/55.4, 108.5/53.4, 106.5/53.4, 106.5/53.3 us)
#endif
constexpr int kResampleWarps = NACC_RESAMPLE_WARPS;

// per-launch constants computed once on the host
struct ResampleConst {
  double inv_tn, inv_tf;  // 1/t_n, 1/t_f (0 for t_f = inf); unused with per-ray spans
  double inv_n;           // 1/n_out
  double s_thr;           // -log1p(-1e-12): S_m > s_thr <=> F_m = 1 - e^{-S_m} > 1e-12 (reading #16)
  int top;                // largest power of two <= n_in - 1 (0 for n_in = 1)
};
#ifndef NACC_RESAMPLE_F32DT
#define NACC_RESAMPLE_F32DT 1  // build parameter: interval lengths by the fp32 product identities (cdf_items)
#endif
#ifndef NACC_RESAMPLE_ITEMS
#define NACC_RESAMPLE_ITEMS 1  // build parameter: sigma CDF with consecutive edges per lane (0: 32-edge windows)
#endif

// The sigma CDF with kIPL consecutive intervals per lane (n_in <= 32 kIPL): each lane maps its
// edges through Φ, forms s_j = σ_j (t_{j+1} - t_j) and their running sum in fp64, one fp64 warp
// scan of the lane totals gives every S_{j+1}; F[j+1] = 1 - e^{-S_{j+1}} is normalised by F_m in
// registers before it is stored (the same arithmetic as the windowed path, one scan per ray
// instead of one per 32 edges).  Returns the total S_m (every lane).
// 1/t = (1 - s)/t_n + s/t_f in fp32 from itn = 1/t_n, itf = 1/t_f: both terms >= 0, so no
// cancellation (the form 1/t_n + s (1/t_f - 1/t_n) loses the small 1/t near s = 1)
__device__ __forceinline__ float lin_x(float s, float itn, float itf) {
  return __fmaf_rn(s, itf, __fmul_rn(__fsub_rn(1.0f, s), itn));
}

// kMode 0: t_j = Φ(s_j) in fp64 and s_j = σ_j (t_{j+1} - t_j) in fp64 (any map and range).
// kMode 1 (lindisp, every t in [1e-15, 1e15]) and 2 (identity): t_{j+1} - t_j from the exact
// identities 1/x_j - 1/x_{j+1} = (x_{j+1} - x_j) / (x_j x_{j+1}) with x = 1/t linear in s (lin_x), i.e.
// Δt_j = Δs_j (1/t_n - 1/t_f) t_j t_{j+1}, and Δt_j = Δs_j (t_f - t_n): no cancellation, so fp32
// gives Δt_j to a few ulps (the fp64 path needs fp64 only because it subtracts two t's); the lane's
// running sums are fp32 (at most 8 terms), the cross-lane scan fp64 (reading #29).
template <int kIPL, int kMode, typename PhiE>
__device__ __forceinline__ double cdf_items(int n_in, const float *__restrict__ er, const float *__restrict__ sr,
                                            float *e, float *F, PhiE phi_e, float xa, float xb, float dc,
                                            double s_thr, bool &uniform) {
  const int lane = threadIdx.x & 31;
  const int j0 = lane * kIPL;
  float ev[kIPL + 1], sv[kIPL];
#pragma unroll
  for (int k = 0; k < kIPL; ++k) {
    const int j = j0 + k;
    ev[k] = j <= n_in ? __ldg(er + j) : 0.f;
    sv[k] = j < n_in ? __ldg(sr + j) : 0.f;
  }
  ev[kIPL] = j0 + kIPL <= n_in ? __ldg(er + j0 + kIPL) : 0.f;
#pragma unroll
  for (int k = 0; k < kIPL; ++k)
    if (j0 + k <= n_in) e[j0 + k] = ev[k];
  if (j0 + kIPL == n_in) e[n_in] = ev[kIPL];
  float f[kIPL];  // 1 - e^{-S_{j+1}} (unnormalised)
  double run = 0.0, incl;
  if constexpr (kMode == 0) {
    double tk = phi_e((double)ev[0]);
    double loc[kIPL];
#pragma unroll
    for (int k = 0; k < kIPL; ++k) {
      const double tk1 = phi_e((double)ev[k + 1]);
      run += j0 + k < n_in ? (double)sv[k] * (tk1 - tk) : 0.0;
      loc[k] = run;
      tk = tk1;
    }
    incl = warp_incl_scan(run);
    const double base = incl - run;
#pragma unroll
    for (int k = 0; k < kIPL; ++k) f[k] = one_minus_exp_neg((float)(base + loc[k]));
  } else {
    auto rcp = [](float x) {  // 1/x to 1 ulp (x normal)
      float y;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
      return y;
    };
    float tk = kMode == 1 ? rcp(lin_x(ev[0], xa, xb)) : 0.f;
    float loc[kIPL], runf = 0.f;
#pragma unroll
    for (int k = 0; k < kIPL; ++k) {
      const float ds = __fsub_rn(ev[k + 1], ev[k]);
      float dt;
      if (kMode == 1) {
        const float tk1 = rcp(lin_x(ev[k + 1], xa, xb));
        dt = __fmul_rn(__fmul_rn(__fmul_rn(ds, dc), tk), tk1);
        tk = tk1;
      } else {
        dt = __fmul_rn(ds, dc);
      }
      runf = __fadd_rn(runf, j0 + k < n_in ? __fmul_rn(sv[k], dt) : 0.f);
      loc[k] = runf;
    }
    run = (double)runf;
    incl = warp_incl_scan(run);
    const float basef = (float)(incl - run);
#pragma unroll
    for (int k = 0; k < kIPL; ++k) f[k] = one_minus_exp_neg(__fadd_rn(basef, loc[k]));
  }
  // F non-decreasing edge by edge (the scan's tree-order sums and the fp32 1 - e^{-S} can each
  // step back by an ulp): a running max within the lane, then across the lanes
#pragma unroll
  for (int k = 1; k < kIPL; ++k) f[k] = fmaxf(f[k], f[k - 1]);
  float mx = f[kIPL - 1];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(kFull, mx, o);
    if (lane >= o) mx = fmaxf(mx, y);
  }
  const float before = __shfl_up_sync(kFull, mx, 1);
  if (lane > 0)
#pragma unroll
    for (int k = 0; k < kIPL; ++k) f[k] = fmaxf(f[k], before);
  const double total = __shfl_sync(kFull, incl, 31);
  uniform = !(total > s_thr);  // F_m = 1 - e^{-S_m} > 1e-12 <=> S_m > -log1p(-1e-12) (host constant)
  const float Fm = one_minus_exp_neg((float)total), rFm = __frcp_rn(Fm);
#pragma unroll
  for (int k = 0; k < kIPL; ++k) {
    const int j = j0 + k;
    if (j < n_in) F[j + 1] = uniform ? f[k] : (j + 1 == n_in ? 1.0f : fminf(__fmul_rn(f[k], rFm), 1.0f));
  }
  if (lane == 0) F[0] = 0.f;
  __syncwarp();
  return total;
}

template <bool kRanged, int kIPL>
__global__ void __launch_bounds__(kResampleWarps * 32, NACC_RESAMPLE_MINB) importance_kernel(
    int64_t n_rays, int n_in, const float *__restrict__ s_edges, const float *__restrict__ sigma,
    const float *__restrict__ cdf, int map, double tn, double tf, const float *__restrict__ tn_r,
    const float *__restrict__ tf_r, int n_out, int stratified, uint32_t key0, uint32_t key1,
    float *__restrict__ s_out, float *__restrict__ t_out, ResampleConst rc) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * kResampleWarps + warp;
  if (r >= n_rays) return;
  float *e = smem + (size_t)warp * 2 * (n_in + 1);
  float *F = e + (n_in + 1);
  const float *er = s_edges + r * (int64_t)(n_in + 1);
  if (kRanged) {  // per-ray span (combined estimator, reading #19)
    tn = (double)__ldg(tn_r + r);
    tf = (double)__ldg(tf_r + r);
    if (!(tf > tn)) {  // culled: uniform s edges, every t at t_near
      const double e0 = (double)__ldg(er), em = (double)__ldg(er + n_in);
      for (int i = lane; i <= n_out; i += 32) {
        s_out[r * (int64_t)(n_out + 1) + i] = (float)(e0 + (em - e0) * ((double)i / (double)n_out));
        if (t_out) t_out[r * (int64_t)(n_out + 1) + i] = (float)tn;
      }
      return;
    }
  }
  // launch constants from the host (1/t_n, 1/t_f, 1/n, ...); per-ray spans compute their own
  const double inv_tn = kRanged ? 1.0 / tn : rc.inv_tn, inv_tf = kRanged ? (isinf(tf) ? 0.0 : 1.0 / tf) : rc.inv_tf;
  bool uniform = false, normal = false;
  int tmode = 0;  // t_out: 0 Φ in fp64; 1 lindisp 1/lin_x(s, 1/t_n, 1/t_f) in fp32; 2 identity t_n + s w in fp32
  float xa = 0.f, xb = 0.f;
  if constexpr (kIPL > 0) {  // sigma input, n_in <= 32 kIPL
    const float *sr = sigma + r * (int64_t)n_in;
    const bool in01 = __ldg(er) >= 0.f && __ldg(er + n_in) <= 1.f;
    normal = map == NACC_MAP_LINDISP && fmin(inv_tn, inv_tf) >= 1e-30 && fmax(inv_tn, inv_tf) <= 1e30 && in01;
    auto phi_n = [&](double sv) { return phi_normal(map, sv, tn, inv_tn, inv_tf, tf); };
    if (NACC_RESAMPLE_F32DT && normal && fmin(inv_tn, inv_tf) >= 1e-15 && fmax(inv_tn, inv_tf) <= 1e15) {
      tmode = 1;
      xa = (float)inv_tn;
      xb = (float)inv_tf;
      cdf_items<kIPL, 1>(n_in, er, sr, e, F, phi_n, xa, xb, (float)(inv_tn - inv_tf), rc.s_thr, uniform);
    } else if (NACC_RESAMPLE_F32DT && map == NACC_MAP_IDENTITY && in01 && tf - tn <= 1e15) {
      tmode = 2;
      xa = (float)tn;
      xb = (float)(tf - tn);
      cdf_items<kIPL, 2>(n_in, er, sr, e, F, phi_n, 0.f, 0.f, xb, rc.s_thr, uniform);
    } else if (normal)
      cdf_items<kIPL, 0>(n_in, er, sr, e, F, phi_n, 0.f, 0.f, 0.f, rc.s_thr, uniform);
    else
      cdf_items<kIPL, 0>(n_in, er, sr, e, F, [&](double sv) { return phi(map, sv, tn, inv_tn, inv_tf, tf); }, 0.f,
                         0.f, 0.f, rc.s_thr, uniform);
  } else {
    for (int j = lane; j <= n_in; j += 32) e[j] = __ldg(er + j);
    __syncwarp();
    if (sigma) {
      const float *sr = sigma + r * (int64_t)n_in;
      double carry = 0.0;
      // t of every edge once: lane l holds t(e[base + l]); t(e[j + 1]) comes from the next lane,
      // and for lane 31 from lane 0 of the next window (computed one window ahead)
      // every edge's 1/t in fp32's normal range (the common case): Φ without the range check
      normal = map == NACC_MAP_LINDISP && fmin(inv_tn, inv_tf) >= 1e-30 && fmax(inv_tn, inv_tf) <= 1e30 &&
               e[0] >= 0.f && e[n_in] <= 1.f;
      auto phi_e = [&](double sv) {
        return normal ? phi_normal(map, sv, tn, inv_tn, inv_tf, tf) : phi(map, sv, tn, inv_tn, inv_tf, tf);
      };
      double ta = lane <= n_in ? phi_e((double)e[lane]) : 0.0;
      for (int base = 0; base < n_in; base += 32) {
        const int j = base + lane;
        const double tnext = j + 32 <= n_in ? phi_e((double)e[j + 32]) : 0.0;
        const double dn = __shfl_down_sync(kFull, ta, 1), wn = __shfl_sync(kFull, tnext, 0);
        const double tb = lane < 31 ? dn : wn;
        double s = 0.0;
        if (j < n_in) s = (double)__ldg(sr + j) * (tb - ta);
        ta = tnext;
        const double incl = warp_incl_scan(s);
        if (j < n_in) F[j + 1] = one_minus_exp_neg((float)(carry + incl));
        carry += __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) F[0] = 0.f;
      uniform = !(carry > rc.s_thr);
      __syncwarp();
      if (!uniform) {  // F / F_m by one reciprocal (within an ulp of the quotient); F_m / F_m = 1 exactly
        const float Fm = F[n_in], rFm = __frcp_rn(Fm);
        for (int j = lane; j < n_in; j += 32) F[j] = fminf(__fmul_rn(F[j], rFm), 1.0f);  // monotone, <= 1
        __syncwarp();
        if (lane == 0) F[n_in] = 1.0f;
      }
    } else {
      const float *cr = cdf + r * (int64_t)(n_in + 1);
      const float c0 = __ldg(cr), cm = __ldg(cr + n_in);
      uniform = !((double)cm - (double)c0 > 1e-12);
      if (!uniform) {
        const float den = __fsub_rn(cm, c0);
        for (int j = lane; j <= n_in; j += 32) F[j] = __fdiv_rn(__fsub_rn(__ldg(cr + j), c0), den);
      }
    }
  }
  if (uniform) {
    __syncwarp();
    const float e0 = e[0], den = __fsub_rn(e[n_in], e0);
    for (int j = lane; j <= n_in; j += 32) F[j] = __fdiv_rn(__fsub_rn(e[j], e0), den);
  }
  __syncwarp();
  const double inv_n = rc.inv_n;
  float *so = s_out + r * (int64_t)(n_out + 1);
  float *to = t_out ? t_out + r * (int64_t)(n_out + 1) : nullptr;
  int n_search = n_out + 1;
  const int top = rc.top;  // binary-lifting first step: the largest power of two <= n_in - 1
  if (!stratified) {
    // u = 1 at i = n_out: the smallest j in [0, n_in-1] with F[j+1] >= 1.  {j : F[j+1] >= 1} is a
    // suffix of the bins (F monotone, F[n_in] = 1), so scan 32-bin windows from the end and stop
    // at the first window holding a bin below 1
    int jl = 0;
    for (int b0 = n_in - 32;; b0 -= 32) {
      const int j = b0 + lane;
      const unsigned m = __ballot_sync(kFull, j < 0 || F[j + 1] >= 1.0f);
      if (m != kFull) {
        jl = b0 + 32 - __clz(~m);  // one past the highest bin below 1
        break;
      }
      if (b0 <= 0) break;  // every bin reaches 1: j = 0
    }
    if (lane == 0) {
      const double s = (double)e[jl + 1];
      so[n_out] = (float)s;
      if (to) to[n_out] = (float)phi(map, s, tn, inv_tn, inv_tf, tf);
    }
    n_search = n_out;
  }
  for (int i = lane; i < n_search; i += 32) {
    double u;
    if (stratified) {
      const u32x4 rnd = philox4x32_10(u32x4{(uint32_t)(uint64_t)r, (uint32_t)((uint64_t)r >> 32), (uint32_t)i, 1u},
                                      key0, key1);
      u = ((double)i + u24(rnd.x)) / (double)(n_out + 1);
    } else {
      u = (double)i * inv_n;  // i / n within an ulp, < 1
    }
    // largest j in [0, n_in-1] with F[j] <= u, i.e. F[j] <= uf, the largest float <= u (exact)
    // (binary lifting from the largest power of two <= n_in - 1: a fixed, uniform trip count)
    const float uf = __double2float_rd(u);
    int lo = 0;
    for (int step = top; step > 0; step >>= 1)
      if (lo + step < n_in && F[lo + step] <= uf) lo += step;
    // linear within the bin in fp32 (reading #29): F[lo] <= u < F[lo + 1], so the fraction lies in
    // [0, 1); each step rounds once (back error ~1e-7 plus the output's own rounding), and the
    // clamp to the bin keeps the edges non-decreasing across bins
    const float Fj = F[lo], Fj1 = F[lo + 1], ej = e[lo], ej1 = e[lo + 1];
    const float d = __fsub_rn(Fj1, Fj);
    const float num = (float)(u - (double)Fj);
    const float frac = d >= 1e-30f ? __fmul_rn(num, __frcp_rn(d)) : (float)((double)num / (double)d);
    const float sf = fminf(__fmaf_rn(fminf(frac, 1.0f), __fsub_rn(ej1, ej), ej), ej1);
    so[i] = sf;
    // s lies between two edges: with every edge's 1/t normal, so is Φ(s)'s
    if (to) {
      if (tmode == 1) {  // 1/x to 1 ulp (x in [1e-15, 1e15]): t to ~2 ulps, Δs-equivalent ~1e-7
        float y;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(lin_x(sf, xa, xb)));
        to[i] = y;
      } else if (tmode == 2) {
        to[i] = __fmaf_rn(sf, xb, xa);
      } else {
        const double s = (double)sf;
        to[i] = (float)(normal ? phi_normal(map, s, tn, inv_tn, inv_tf, tf) : phi(map, s, tn, inv_tn, inv_tf, tf));
      }
    }
  }
}

static nacc_status launch_importance(int64_t n_rays, int32_t n_in, const float *s_edges, const float *sigma,
                                     const float *cdf, nacc_map map, double t_near, double t_far,
                                     const float *tn_r, const float *tf_r, int32_t n_out, int32_t stratified,
                                     uint64_t seed, float *s_out, float *t_out, cudaStream_t stream) {
  NACC_REQUIRE(s_edges && s_out, "s_edges and s_out must be non-NULL");
  const int ipl = NACC_RESAMPLE_ITEMS && sigma && n_in <= 256 ? (n_in + 31) / 32 : 0;
  const size_t smem = (size_t)kResampleWarps * 2 * (n_in + 1) * sizeof(float);
  if (smem > 227 * 1024) {
    set_error("nacc_importance_sample: n_in too large for shared memory");
    return NACC_ERR_UNSUPPORTED;
  }
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  ResampleConst rc;
  rc.inv_tn = tn_r ? 0.0 : 1.0 / t_near;
  rc.inv_tf = tn_r ? 0.0 : (std::isinf(t_far) ? 0.0 : 1.0 / t_far);
  rc.inv_n = 1.0 / (double)n_out;
  rc.s_thr = -std::log1p(-1e-12);
  rc.top = 0;
  while (n_in > 1 && 2 * rc.top <= n_in - 1) rc.top = rc.top ? 2 * rc.top : 1;
  nacc_status st = NACC_OK;
  auto go = [&](auto ranged, auto items) {
    constexpr bool kR = decltype(ranged)::value;
    constexpr int kI = decltype(items)::value;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(importance_kernel<kR, kI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
      set_error("nacc_importance_sample: cudaFuncSetAttribute failed");
      st = NACC_ERR_CUDA;
      return;
    }
    importance_kernel<kR, kI><<<grid_for(n_rays, kResampleWarps), kResampleWarps * 32, smem, stream>>>(
        n_rays, n_in, s_edges, sigma, cdf, (int)map, t_near, t_far, tn_r, tf_r, n_out, stratified, k0, k1, s_out,
        t_out, rc);
  };
  auto by_items = [&](auto ranged) {
    using I = std::integral_constant<int, 0>;
    switch (ipl) {
      case 1: go(ranged, std::integral_constant<int, 1>{}); break;
      case 2: go(ranged, std::integral_constant<int, 2>{}); break;
      case 3: go(ranged, std::integral_constant<int, 3>{}); break;
      case 4: go(ranged, std::integral_constant<int, 4>{}); break;
      case 5: go(ranged, std::integral_constant<int, 5>{}); break;
      case 6: go(ranged, std::integral_constant<int, 6>{}); break;
      case 7: go(ranged, std::integral_constant<int, 7>{}); break;
      case 8: go(ranged, std::integral_constant<int, 8>{}); break;
      default: go(ranged, I{});
    }
  };
  if (tn_r) by_items(std::true_type{});
  else by_items(std::false_type{});
  if (st != NACC_OK) return st;
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

static nacc_status check_importance(int64_t n_rays, int32_t n_in, const float *sigma, const float *cdf, nacc_map map,
                                    int32_t n_out) {
  NACC_REQUIRE(n_rays >= 0, "n_rays must be >= 0");
  NACC_REQUIRE(n_in >= 1 && n_out >= 1, "n_in and n_out must be >= 1");
  NACC_REQUIRE((sigma != nullptr) != (cdf != nullptr), "exactly one of sigma / cdf must be non-NULL");
  NACC_REQUIRE(map == NACC_MAP_IDENTITY || map == NACC_MAP_LINDISP, "unknown map");
  return NACC_OK;
}

}  // namespace nacc

using namespace nacc;

extern "C" {

nacc_status nacc_importance_sample(int64_t n_rays, int32_t n_in, const float *s_edges, const float *sigma,
                                   const float *cdf, nacc_map map, double t_near, double t_far, int32_t n_out,
                                   int32_t stratified, uint64_t seed, float *s_out, float *t_out,
                                   cudaStream_t stream) {
  clear_error();
  nacc_status st = check_importance(n_rays, n_in, sigma, cdf, map, n_out);
  if (st != NACC_OK) return st;
  NACC_REQUIRE(std::isfinite(t_near) && t_near > 0.0 && t_far > t_near, "need 0 < t_near < t_far");
  NACC_REQUIRE(map == NACC_MAP_LINDISP || std::isfinite(t_far), "identity map needs a finite t_far");
  if (n_rays == 0) return NACC_OK;
  NACC_DEBUG_CHECK(debug_check_rows_ascending(s_edges, n_rays, n_in + 1, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, sigma ? n_rays * n_in : 0, "proposal sigma must be >= 0 and finite", stream));
  return launch_importance(n_rays, n_in, s_edges, sigma, cdf, map, t_near, t_far, nullptr, nullptr, n_out,
                           stratified, seed, s_out, t_out, stream);
}

nacc_status nacc_importance_sample_ranged(int64_t n_rays, int32_t n_in, const float *s_edges, const float *sigma,
                                          const float *cdf, nacc_map map, const float *t_near, const float *t_far,
                                          int32_t n_out, int32_t stratified, uint64_t seed, float *s_out,
                                          float *t_out, cudaStream_t stream) {
  clear_error();
  nacc_status st = check_importance(n_rays, n_in, sigma, cdf, map, n_out);
  if (st != NACC_OK) return st;
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(t_near && t_far, "t_near and t_far must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_rows_ascending(s_edges, n_rays, n_in + 1, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, sigma ? n_rays * n_in : 0, "proposal sigma must be >= 0 and finite", stream));
  return launch_importance(n_rays, n_in, s_edges, sigma, cdf, map, 0.0, 0.0, t_near, t_far, n_out, stratified,
                           seed, s_out, t_out, stream);
}

}  // extern "C"
