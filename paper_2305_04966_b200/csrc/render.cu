// render.cu — the transmittance estimator and compositing of Eq. 2
// discretised as in P:246 (reading #11), forward and backward:
//   δ_i = t1_i - t0_i, s_i = σ_i δ_i, S_i = Σ_{j<i} s_j (fp64 segmented scan),
//   T_i = exp(-S_i), α_i = 1 - exp(-s_i), w_i = T_i α_i, w_i = 0 once S_i > -ln ε,
//   color = Σ w rgb, opacity = Σ w, depth = Σ w m / max(opacity, 1e-10).
// Backward (t detached P:78):
//   g_σ_i = δ_i (g_w_i T_i (1-α_i) - Σ_{j>i} g_w_j w_j) for live samples,
// with Σ_{j>i} g_w_j w_j = R - Σ_{j<=i} g_w_j w_j and R = <g_C,C> + g_O' O + g_N N
// taken from the forward's fp64 per-ray sums (ctx), so one forward-order pass
// suffices.  One warp per ray; 32 consecutive samples per step.
#include "common.cuh"

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

__device__ __forceinline__ float trans_of(double S) { return expf(-(float)S); }
__device__ __forceinline__ float alpha_of(double s) { return -expm1f(-(float)s); }

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
      const double w = (double)(trans_of(c.S) * alpha_of(c.s));
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
        const double w = (double)(trans_of(c.S) * alpha_of(c.s));
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
    double gw = 0.0, w = 0.0;
    float r0 = 0.f, r1 = 0.f, r2 = 0.f, T = 0.f, ea = 0.f;
    if (c.live) {
      T = trans_of(c.S);
      ea = expf(-(float)c.s);  // 1 - α
      w = (double)(T * alpha_of(c.s));
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
      const double gs = c.live ? gw * (double)T * (double)ea - Q : 0.0;
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
      const float T = trans_of(c.S), a = alpha_of(c.s);
      weights[q] = c.live ? T * a : 0.f;
      if (trans) trans[q] = T;
      if (alphas) alphas[q] = a;
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
      const float T = trans_of(c.S);
      if (c.live) R += (double)__ldg(g_weights + q) * (double)(T * alpha_of(c.s));
      if (g_trans) R += (double)__ldg(g_trans + q) * (double)T;
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
      const float T = trans_of(c.S);
      const double gw = (double)__ldg(g_weights + q);
      if (c.live) {
        v += gw * (double)(T * alpha_of(c.s));
        gwTa = gw * (double)T * (double)expf(-(float)c.s);
      }
      if (g_trans) v += (double)__ldg(g_trans + q) * (double)T;
    }
    const double incl = warp_incl_scan(v);
    const double Q = R - (P + incl);
    P += __shfl_sync(kFull, incl, 31);
    if (c.valid) g_sigma[q] = (float)(c.delta * (gwTa - Q));
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

nacc_status nacc_render_fwd(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                            const float *sigma, const float *rgb, int64_t n_samples, double neg_log_eps,
                            float *color, float *opacity, float *depth, double *ctx, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma), "t0, t1, sigma must be non-NULL");
  NACC_REQUIRE(!ctx || aligned(ctx, 8), "ctx must be 8-byte aligned");
  render_fwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma, rgb,
                                                                     neg_log_eps, color, opacity, depth, ctx);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

nacc_status nacc_render_bwd(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                            const float *sigma, const float *rgb, int64_t n_samples, double neg_log_eps,
                            const double *ctx, const float *g_color, const float *g_opacity,
                            const float *g_depth, float *g_sigma, float *g_rgb, cudaStream_t stream) {
  clear_error();
  nacc_status s = check_packed(packed_info, n_rays, n_samples);
  if (s != NACC_OK) return s;
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma && g_sigma), "t0, t1, sigma, g_sigma must be non-NULL");
  render_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma, rgb,
                                                                     neg_log_eps, ctx, g_color, g_opacity, g_depth,
                                                                     g_sigma, g_rgb);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
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
  weights_fwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma,
                                                                      neg_log_eps, weights, trans, alphas);
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
  weights_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, t0, t1, sigma,
                                                                      neg_log_eps, g_weights, g_trans, g_sigma);
  count_launch(1);
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
  accumulate_bwd_kernel<<<grid_for(n_rays * 32, 256), 256, 0, stream>>>(packed_info, n_rays, weights, values, C,
                                                                         g_out, g_weights, g_values);
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

}  // extern "C"
