/*
 * oracle.c — the CPU oracle for the packed-sample volume-rendering hot path
 * of NerfAcc (arXiv 2305.04966).  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain C11, one sequential loop per ray, fp64 arithmetic.  OpenMP only
 * splits independent rays/cells across threads; every per-ray or per-cell
 * result is computed by one thread in program order, so results do not depend
 * on the thread count.  No blocking, fusion or reordering
 * beyond what the cited definitions state.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

void or_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).                         */
/* ------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0;
    k1 += W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

double or_u24(uint32_t x) { return (double)(x >> 8) * (1.0 / 16777216.0); }

static void philox_seed(uint64_t seed, uint32_t key[2]) {
  key[0] = (uint32_t)(seed & 0xffffffffu);
  key[1] = (uint32_t)(seed >> 32);
}

/* ------------------------------------------------------------------------ */
/* O1: slab test (reading #7).  Box is half-open [lo, hi).           */
/* ------------------------------------------------------------------------ */
int or_ray_aabb(const double o[3], const double d[3], const double lo[3], const double hi[3],
                double near, double far, double *t_enter, double *t_exit) {
  double tmin = -INFINITY, tmax = INFINITY;
  for (int a = 0; a < 3; ++a) {
    if (d[a] != 0.0) {
      double ta = (lo[a] - o[a]) / d[a];
      double tb = (hi[a] - o[a]) / d[a];
      if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
      if (ta > tmin) tmin = ta;
      if (tb < tmax) tmax = tb;
    } else {
      /* the axis admits every t when the origin lies inside the slab */
      if (!(lo[a] <= o[a] && o[a] < hi[a])) return 0;
    }
  }
  double te = tmin > near ? tmin : near;
  double tx = tmax < far ? tmax : far;
  if (!(tx > te)) return 0;
  *t_enter = te;
  *t_exit = tx;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Φ: s-space <-> t-space.                                   */
/* ------------------------------------------------------------------------ */
double or_contract(int map, double s, double tn, double tf) {
  if (map == 0) return tn + s * (tf - tn);
  /* 1/t = (1 - s)/tn + s/tf   (1/tf = 0 when tf is infinite) */
  double inv_tf = isinf(tf) ? 0.0 : 1.0 / tf;
  return 1.0 / ((1.0 - s) / tn + s * inv_tf);
}

double or_uncontract(int map, double t, double tn, double tf) {
  if (map == 0) return (t - tn) / (tf - tn);
  double inv_tf = isinf(tf) ? 0.0 : 1.0 / tf;
  return (1.0 / t - 1.0 / tn) / (inv_tf - 1.0 / tn);
}

/* ------------------------------------------------------------------------ */
/* O2-O4: occupancy-grid marching (P:240 spatial skipping; P:74-83 intervals,  */
/* packed tensor; readings #1-#5, #26-#27).                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
  int L, R;
  float lo[8][3], hi[8][3]; /* fp32 level boxes */
  float s[8][3];            /* fp32 R / (hi - lo), rounded once from fp64 */
  double olo[3], ohi[3];    /* outermost box padded, fp64 (fast k-range only) */
  double centre[3], halfdiag;
} gctx;

static void grid_ctx(const or_grid *g, gctx *c) {
  c->L = g->levels;
  c->R = g->res;
  double hd2 = 0.0;
  for (int a = 0; a < 3; ++a) {
    double lo0 = (double)g->roi[a], hi0 = (double)g->roi[3 + a];
    double ctr = (lo0 + hi0) / 2.0, half = (hi0 - lo0) / 2.0;
    for (int l = 0; l < g->levels; ++l) {
      double sc = ldexp(1.0, l); /* level-l box = centre ± half·2^l (reading #4) */
      c->lo[l][a] = (float)(ctr - half * sc);
      c->hi[l][a] = (float)(ctr + half * sc);
      c->s[l][a] = (float)((double)g->res / ((double)c->hi[l][a] - (double)c->lo[l][a]));
    }
    int lo_l = g->levels - 1;
    double w = (double)c->hi[lo_l][a] - (double)c->lo[lo_l][a];
    double pad = 1e-4 * w + 1e-6;
    c->olo[a] = (double)c->lo[lo_l][a] - pad;
    c->ohi[a] = (double)c->hi[lo_l][a] + pad;
    c->centre[a] = ctr;
    hd2 += (half * ldexp(1.0, lo_l)) * (half * ldexp(1.0, lo_l));
  }
  c->halfdiag = sqrt(hd2);
}

/* O3: membership predicate P(k) at the fp32 midpoint m (reading #2, #3).
 * x_a = fmaf(m, d_a, o_a); l* = first level whose half-open box holds x;
 * u_a = (x_a - lo_a) * s_a in fp32; i_a = clamp(floor(u_a), 0, R-1). */
static int member(const gctx *c, const uint8_t *occ, float m, const float o[3], const float d[3]) {
  float x[3];
  for (int a = 0; a < 3; ++a) x[a] = fmaf(m, d[a], o[a]);
  int lstar = -1;
  for (int l = 0; l < c->L; ++l) {
    int in = 1;
    for (int a = 0; a < 3; ++a)
      if (!(c->lo[l][a] <= x[a] && x[a] < c->hi[l][a])) in = 0;
    if (in) { lstar = l; break; }
  }
  if (lstar < 0) return 0;
  int64_t i[3];
  for (int a = 0; a < 3; ++a) {
    float u = (x[a] - c->lo[lstar][a]) * c->s[lstar][a];
    int64_t ia = (int64_t)floorf(u);
    if (ia < 0) ia = 0;
    if (ia > c->R - 1) ia = c->R - 1;
    i[a] = ia;
  }
  int64_t R = c->R;
  return occ[(int64_t)lstar * R * R * R + i[0] + R * (i[1] + R * i[2])] != 0;
}

/* per-ray near plane after optional stratified jitter (reading #1) */
static float ray_near(const or_march *p, const float *t_min, int64_t r) {
  float nr = t_min ? t_min[r] : p->near_plane;
  if (p->stratified) {
    uint32_t key[2], ctr[4] = {(uint32_t)(r & 0xffffffffu), (uint32_t)((uint64_t)r >> 32), 0u, 0u},
                     out[4];
    philox_seed(p->seed, key);
    or_philox4x32_10(ctr, key, out);
    double xi = or_u24(out[0]);
    nr = (float)((double)nr + xi * (double)p->step);
  }
  return nr;
}

/* fp32 rounding (to nearest, ties to even) of the exact real a + b, where a and
 * b are doubles (reading #3: lattice values are the fp32 of the exact value).
 * The fp64 sum s may itself be rounded; a double rounding differs from the
 * single one only when s lands exactly on a tie between two fp32 neighbours
 * while the exact sum does not, so the tie is broken by the sign of the exact
 * error e = (a + b) - s (Knuth's TwoSum). */
static float f32_exact_sum(double a, double b) {
  double s = a + b;
  double a1 = s - b, b1 = s - a1;
  double e = (a - a1) + (b - b1);
  float r = (float)s;
  if (e != 0.0) {
    float lo = (float)s, hi = (float)s;
    if ((double)r > s) lo = nextafterf(r, -INFINITY);
    else if ((double)r < s) hi = nextafterf(r, INFINITY);
    if (lo != hi && s - (double)lo == (double)hi - s) r = e > 0.0 ? hi : lo;
  }
  return r;
}

/* Uniform lattice value near_r + (k + half/2)·Δt rounded once to fp32 (reading
 * #1, #3): t_k for half = 0, the midpoint m_k for half = 1. */
float or_lattice_point(float near_r, float step, int64_t k, int32_t half) {
  return f32_exact_sum((double)near_r, ((double)k + 0.5 * (double)half) * (double)step);
}

/* One ray.  Returns the number of emitted intervals; writes them when t0 != NULL. */
static int64_t march_ray(const gctx *c, const uint8_t *occ, const or_march *p, const float o[3],
                         const float d[3], float near_r, float far_r, int brute, int32_t rid,
                         float *t0, float *t1, int32_t *ray_id) {
  int64_t n = 0;
  double od[3] = {o[0], o[1], o[2]}, dd[3] = {d[0], d[1], d[2]};
  /* range bound for the brute force: beyond T_stop no point of the ray can
   * lie inside the sphere that contains the outermost box */
  double dist = 0.0, dn = 0.0;
  for (int a = 0; a < 3; ++a) {
    dist += (od[a] - c->centre[a]) * (od[a] - c->centre[a]);
    dn += dd[a] * dd[a];
  }
  dist = sqrt(dist);
  dn = sqrt(dn);
  double dtmax = p->cone_angle > 0.0f ? (double)p->max_step : (double)p->step;
  double T_stop = (dn > 0.0 ? (dist + c->halfdiag) / dn * (1.0 + 1e-6) : 0.0) + 2.0 * dtmax + 1e-3;
  double t_lo = -INFINITY, t_hi = INFINITY;
  if (!brute) {
    if (!or_ray_aabb(od, dd, c->olo, c->ohi, (double)near_r, (double)far_r, &t_lo, &t_hi)) return 0;
  }
  if (p->cone_angle == 0.0f) {
    const double dt = (double)p->step, nr = (double)near_r;
    int64_t k_begin = 0, k_end = (int64_t)1 << 24;
    if (!brute) {
      double kb = floor((t_lo - nr) / dt - 0.5) - 2.0;
      double ke = ceil((t_hi - nr) / dt) + 3.0;
      k_begin = kb > 0.0 ? (int64_t)kb : 0;
      if (ke < (double)k_end) k_end = ke > 0.0 ? (int64_t)ke : 0;
    }
    /* lattice indices k < 2^24 (header of nacc.h); (k + 1/2)·Δt and k·Δt are exact
     * fp64 products (25 x 24 bits), the sums with near_r are rounded once to fp32 */
    for (int64_t k = k_begin; k < k_end; ++k) {
      double tk = nr + (double)k * dt;
      if (brute && tk > T_stop) break;
      float m = or_lattice_point(near_r, p->step, k, 1);
      if (!(m < far_r)) break;
      if (member(c, occ, m, o, d)) {
        if (t0) {
          t0[n] = or_lattice_point(near_r, p->step, k, 0);
          t1[n] = or_lattice_point(near_r, p->step, k + 1, 0);
          ray_id[n] = rid;
        }
        ++n;
      }
    }
  } else {
    /* cone recurrence in fp32 (reading #5): dt_k = min(max(t_k c, Δt_min), Δt_max) */
    float t = near_r;
    for (int64_t k = 0; k < ((int64_t)1 << 24); ++k) {
      float dt = fminf(fmaxf(t * p->cone_angle, p->step), p->max_step);
      float m = t + 0.5f * dt;
      float tn = t + dt;
      if (!(m < far_r)) break;
      if (brute) {
        if ((double)t > T_stop) break;
      } else {
        if ((double)m > t_hi + 2.0 * (double)dt) break;
      }
      int test = brute || ((double)m >= t_lo - 2.0 * (double)dt);
      if (test && member(c, occ, m, o, d)) {
        if (t0) {
          t0[n] = t;
          t1[n] = tn;
          ray_id[n] = rid;
        }
        ++n;
      }
      t = tn;
    }
  }
  return n;
}

void or_march_count(const or_grid *g, const uint8_t *occ, const or_march *p, const float *rays_o,
                    const float *rays_d, const float *t_min, const float *t_max, int64_t n_rays,
                    int brute, int64_t *counts) {
  gctx c;
  grid_ctx(g, &c);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    float nr = ray_near(p, t_min, r);
    float fr = t_max ? t_max[r] : p->far_plane;
    counts[r] = march_ray(&c, occ, p, rays_o + 3 * r, rays_d + 3 * r, nr, fr, brute, (int32_t)r,
                          NULL, NULL, NULL);
  }
}

void or_march_fill(const or_grid *g, const uint8_t *occ, const or_march *p, const float *rays_o,
                   const float *rays_d, const float *t_min, const float *t_max, int64_t n_rays,
                   int brute, const int64_t *start, float *t0, float *t1, int32_t *ray_id) {
  gctx c;
  grid_ctx(g, &c);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    float nr = ray_near(p, t_min, r);
    float fr = t_max ? t_max[r] : p->far_plane;
    int64_t s = start[r];
    march_ray(&c, occ, p, rays_o + 3 * r, rays_d + 3 * r, nr, fr, brute, (int32_t)r, t0 + s,
              t1 + s, ray_id + s);
  }
}

/* ------------------------------------------------------------------------ */
/* O5: no-gradient filtering ("samples with transmittance below 10^-4 are */
/* disregarded"; reading #9: entering T, strict, prefix cut).       */
/* ------------------------------------------------------------------------ */
void or_filter_cut(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                   const double *sigma, double neg_log_eps, int64_t *counts_out,
                   double *margin_out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    double S = 0.0, margin = INFINITY;
    int64_t cut = cnt;
    for (int64_t i = 0; i < cnt; ++i) {
      double mg = fabs(S - neg_log_eps);
      if (mg < margin) margin = mg;
      if (S > neg_log_eps) { cut = i; break; } /* entering T_i = e^{-S_i} < eps */
      S += (double)sigma[s + i] * ((double)t1[s + i] - (double)t0[s + i]);
    }
    counts_out[r] = cut;
    if (margin_out) margin_out[r] = margin;
  }
}

/* ------------------------------------------------------------------------ */
/* O6: render forward — Eq. 2 discretised (reading #11):   */
/* δ_i = t1 - t0, s_i = σ_i δ_i, T_i = exp(-Σ_{j<i} s_j), α_i = 1 - exp(-s_i), */
/* w_i = T_i α_i; C = Σ w c, O = Σ w, D = Σ w m / max(O, 1e-10) (reading #12). */
/* Early stop: w_i = 0 once the entering optical depth exceeds -ln ε.   */
/* ------------------------------------------------------------------------ */
void or_render_fwd(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                   const double *sigma, const double *rgb, double neg_log_eps, double *trans,
                   double *alphas, double *weights, double *color, double *opacity,
                   double *depth) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    double S = 0.0, C[3] = {0.0, 0.0, 0.0}, O = 0.0, N = 0.0;
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t q = s + i;
      double delta = (double)t1[q] - (double)t0[q];
      double si = (double)sigma[q] * delta;
      double T = exp(-S);
      double alpha = -expm1(-si);
      double w = (S > neg_log_eps) ? 0.0 : T * alpha;
      double mid = ((double)t0[q] + (double)t1[q]) / 2.0;
      if (trans) trans[q] = T;
      if (alphas) alphas[q] = alpha;
      if (weights) weights[q] = w;
      if (rgb)
        for (int ch = 0; ch < 3; ++ch) C[ch] += w * (double)rgb[3 * q + ch];
      O += w;
      N += w * mid;
      S += si;
    }
    if (color)
      for (int ch = 0; ch < 3; ++ch) color[3 * r + ch] = C[ch];
    if (opacity) opacity[r] = O;
    if (depth) depth[r] = N / (O > 1e-10 ? O : 1e-10);
  }
}

/* ------------------------------------------------------------------------ */
/* O7: render backward (the field receives gradients through σ and    */
/* rgb; t is detached).  Chain rule on the O6 definitions:              */
/*   ∂w_i/∂s_i = T_i (1-α_i),  ∂w_j/∂s_i = -w_j (j > i),  g_σ_i = δ_i g_s_i.   */
/* Depth D = N / max(O, 1e-10): where O > 1e-10, ∂D/∂N = 1/O, ∂D/∂O = -D/O;   */
/* otherwise ∂D/∂N = 1e10, ∂D/∂O = 0 (reading #15).                           */
/* ------------------------------------------------------------------------ */
void or_render_bwd(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                   const double *sigma, const double *rgb, double neg_log_eps, const double *g_color,
                   const double *g_opacity, const double *g_depth, double *g_sigma, double *g_rgb) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    /* recompute the forward pass */
    double O = 0.0, N = 0.0, S = 0.0;
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t q = s + i;
      double delta = (double)t1[q] - (double)t0[q];
      double si = (double)sigma[q] * delta;
      double w = (S > neg_log_eps) ? 0.0 : exp(-S) * -expm1(-si);
      O += w;
      N += w * (((double)t0[q] + (double)t1[q]) / 2.0);
      S += si;
    }
    double gC[3] = {0.0, 0.0, 0.0};
    if (g_color)
      for (int ch = 0; ch < 3; ++ch) gC[ch] = (double)g_color[3 * r + ch];
    double gO = g_opacity ? (double)g_opacity[r] : 0.0;
    double gD = g_depth ? (double)g_depth[r] : 0.0;
    double gN, gOp;
    if (O > 1e-10) {
      double D = N / O;
      gN = gD / O;
      gOp = gO - gD * D / O;
    } else {
      gN = gD / 1e-10;
      gOp = gO;
    }
    /* per-sample g_w, w, T, α */
    double *gw = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    double *wv = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    double *Tv = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    double *av = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    int *live = (int *)malloc(sizeof(int) * (cnt > 0 ? cnt : 1));
    S = 0.0;
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t q = s + i;
      double delta = (double)t1[q] - (double)t0[q];
      double si = (double)sigma[q] * delta;
      live[i] = !(S > neg_log_eps);
      Tv[i] = exp(-S);
      av[i] = -expm1(-si);
      wv[i] = live[i] ? Tv[i] * av[i] : 0.0;
      double mid = ((double)t0[q] + (double)t1[q]) / 2.0;
      double g = gOp + gN * mid;
      if (rgb)
        for (int ch = 0; ch < 3; ++ch) g += gC[ch] * (double)rgb[3 * q + ch];
      gw[i] = g;
      S += si;
    }
    double Q = 0.0; /* Q_i = Σ_{j>i} g_w_j w_j, by a reverse loop */
    for (int64_t i = cnt - 1; i >= 0; --i) {
      int64_t q = s + i;
      double delta = (double)t1[q] - (double)t0[q];
      double gs = live[i] ? gw[i] * Tv[i] * (1.0 - av[i]) - Q : 0.0;
      g_sigma[q] = live[i] ? delta * gs : 0.0;
      if (g_rgb)
        for (int ch = 0; ch < 3; ++ch) g_rgb[3 * q + ch] = wv[i] * gC[ch];
      Q += gw[i] * wv[i];
    }
    free(gw); free(wv); free(Tv); free(av); free(live);
  }
}

void or_weights_bwd(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                    const double *sigma, double neg_log_eps, const double *g_weights,
                    const double *g_trans, double *g_sigma) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    double *Tv = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    double *av = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    int *live = (int *)malloc(sizeof(int) * (cnt > 0 ? cnt : 1));
    double S = 0.0;
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t q = s + i;
      double si = (double)sigma[q] * ((double)t1[q] - (double)t0[q]);
      live[i] = !(S > neg_log_eps);
      Tv[i] = exp(-S);
      av[i] = -expm1(-si);
      S += si;
    }
    /* w_i is masked to 0 past the cut (a constant there); T_i is the true
     * transmittance everywhere, so its gradient reaches every earlier σ. */
    double Qw = 0.0, QT = 0.0; /* Σ_{j>i} g_w_j w_j and Σ_{j>i} g_T_j T_j */
    for (int64_t i = cnt - 1; i >= 0; --i) {
      int64_t q = s + i;
      double delta = (double)t1[q] - (double)t0[q];
      double w = live[i] ? Tv[i] * av[i] : 0.0;
      double gwi = (double)g_weights[q];
      double gs = (live[i] ? gwi * Tv[i] * (1.0 - av[i]) : 0.0) - Qw - QT;
      g_sigma[q] = delta * gs;
      Qw += gwi * w;
      if (g_trans) QT += (double)g_trans[q] * Tv[i];
    }
    free(Tv); free(av); free(live);
  }
}

/* ------------------------------------------------------------------------ */
/* Alpha compositing.                       */
/* ------------------------------------------------------------------------ */
void or_weights_alpha_fwd(const int64_t *packed_info, int64_t n_rays, const double *alpha,
                          double neg_log_eps, double *weights, double *trans) {
  const double eps_T = exp(-neg_log_eps);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    double T = 1.0;
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t q = s + i;
      int live = !(T < eps_T);
      weights[q] = live ? T * alpha[q] : 0.0;
      if (trans) trans[q] = T;
      T *= 1.0 - alpha[q];
    }
  }
}

void or_weights_alpha_bwd(const int64_t *packed_info, int64_t n_rays, const double *alpha,
                          double neg_log_eps, const double *g_weights, const double *g_trans,
                          double *g_alpha) {
  const double eps_T = exp(-neg_log_eps);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    double *Tv = (double *)malloc(sizeof(double) * (cnt > 0 ? cnt : 1));
    int *live = (int *)malloc(sizeof(int) * (cnt > 0 ? cnt : 1));
    double T = 1.0;
    for (int64_t i = 0; i < cnt; ++i) {
      Tv[i] = T;
      live[i] = !(T < eps_T);
      T *= 1.0 - alpha[s + i];
    }
    for (int64_t k = 0; k < cnt; ++k) {
      double g = live[k] ? g_weights[s + k] * Tv[k] : 0.0;
      double P = Tv[k]; /* Π_{j<i, j≠k} (1 − α_j) for i = k + 1 */
      for (int64_t i = k + 1; i < cnt; ++i) {
        double c = (live[i] ? g_weights[s + i] * alpha[s + i] : 0.0) + (g_trans ? g_trans[s + i] : 0.0);
        g -= c * P;
        P *= 1.0 - alpha[s + i];
      }
      g_alpha[s + k] = g;
    }
    free(Tv); free(live);
  }
}

/* ------------------------------------------------------------------------ */
/* accumulate_along_rays (Alg. 1 outputs): segmented sums.           */
/* ------------------------------------------------------------------------ */
void or_accumulate(const int64_t *packed_info, int64_t n_rays, const double *weights,
                   const double *values, int32_t C, double *out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    for (int32_t c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int64_t i = 0; i < cnt; ++i) {
        double v = values ? (double)values[(s + i) * C + c] : 1.0;
        acc += (double)weights[s + i] * v;
      }
      out[r * C + c] = acc;
    }
  }
}

void or_accumulate_bwd(const int64_t *packed_info, int64_t n_rays, const double *weights,
                       const double *values, int32_t C, const double *g_out, double *g_weights,
                       double *g_values) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    int64_t s = packed_info[2 * r], cnt = packed_info[2 * r + 1];
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t q = s + i;
      double gw = 0.0;
      for (int32_t c = 0; c < C; ++c) {
        double v = values ? (double)values[q * C + c] : 1.0;
        gw += (double)g_out[r * C + c] * v;
        if (g_values) g_values[q * C + c] = (double)weights[q] * (double)g_out[r * C + c];
      }
      g_weights[q] = gw;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* O8: inverse-transform resampling (Eq. 1) of the CDF F = 1 - T   */
/* (Eq. 3; "compute the CDF directly using 1 - T(t)"),      */
/* piecewise linear in s (reading #19), normalised (reading #16).      */
/* ------------------------------------------------------------------------ */
static void cdf_hat_ray(int32_t n_in, const double *e, const double *sg, const double *cdf, int map,
                        double tn, double tf, double *F) {
  if (sg) {
    double S = 0.0;
    F[0] = 0.0;
    for (int32_t j = 0; j < n_in; ++j) {
      double ta = or_contract(map, (double)e[j], tn, tf);
      double tb = or_contract(map, (double)e[j + 1], tn, tf);
      S += (double)sg[j] * (tb - ta);
      F[j + 1] = -expm1(-S); /* F = 1 - T */
    }
    double Fm = F[n_in];
    if (Fm > 1e-12) {
      for (int32_t j = 0; j <= n_in; ++j) F[j] = F[j] / Fm;
      return;
    }
  } else {
    double F0 = (double)cdf[0], Fm = (double)cdf[n_in];
    if (Fm - F0 > 1e-12) {
      for (int32_t j = 0; j <= n_in; ++j) F[j] = ((double)cdf[j] - F0) / (Fm - F0);
      return;
    }
  }
  /* no mass: uniform in s (reading #16) */
  double e0 = (double)e[0], em = (double)e[n_in];
  for (int32_t j = 0; j <= n_in; ++j) F[j] = ((double)e[j] - e0) / (em - e0);
}

void or_importance_cdf(int64_t n_rays, int32_t n_in, const double *s_edges, const double *sigma,
                       const double *cdf, int map, double t_near, double t_far, double *cdf_hat) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r)
    cdf_hat_ray(n_in, s_edges + r * (n_in + 1), sigma ? sigma + r * n_in : NULL,
                cdf ? cdf + r * (n_in + 1) : NULL, map, t_near, t_far, cdf_hat + r * (n_in + 1));
}

/* One ray of O8 with its own [t_near, t_far]. */
static void importance_ray(int64_t r, int32_t n_in, const double *s_edges, const double *sigma,
                           const double *cdf, int map, double t_near, double t_far, int32_t n_out,
                           int32_t stratified, const uint32_t key[2], double *s_out, double *t_out) {
  const double *e = s_edges + r * (n_in + 1);
  if (!(t_far > t_near)) {
    /* culled ray (empty span, reading #19): uniform edges in s, every t at t_near */
    for (int32_t i = 0; i <= n_out; ++i) {
      s_out[r * (n_out + 1) + i] = e[0] + (e[n_in] - e[0]) * ((double)i / (double)n_out);
      if (t_out) t_out[r * (n_out + 1) + i] = t_near;
    }
    return;
  }
  double *F = (double *)malloc(sizeof(double) * (n_in + 1));
  cdf_hat_ray(n_in, e, sigma ? sigma + r * n_in : NULL, cdf ? cdf + r * (n_in + 1) : NULL, map,
              t_near, t_far, F);
  for (int32_t i = 0; i <= n_out; ++i) {
    double u;
    if (stratified) {
      uint32_t ctr[4] = {(uint32_t)(r & 0xffffffffu), (uint32_t)((uint64_t)r >> 32), (uint32_t)i,
                         1u},
               out[4];
      or_philox4x32_10(ctr, key, out);
      u = ((double)i + or_u24(out[0])) / (double)(n_out + 1);
    } else {
      u = (double)i / (double)n_out;
    }
    double s;
    if (u >= 1.0) {
      /* u = 1: the end of the mass, smallest j with F̂_{j+1} = 1 */
      int32_t j = 0;
      while (j < n_in - 1 && F[j + 1] < 1.0) ++j;
      s = (double)e[j + 1];
    } else {
      /* the unique j with F̂_j <= u < F̂_{j+1}: the largest j with F̂_j <= u */
      int32_t j = 0;
      for (int32_t k = 0; k < n_in; ++k)
        if (F[k] <= u) j = k;
      double ej = (double)e[j], ej1 = (double)e[j + 1];
      s = ej + (u - F[j]) / (F[j + 1] - F[j]) * (ej1 - ej);
    }
    s_out[r * (n_out + 1) + i] = s;
    if (t_out) t_out[r * (n_out + 1) + i] = or_contract(map, s, t_near, t_far);
  }
  free(F);
}

void or_importance_sample(int64_t n_rays, int32_t n_in, const double *s_edges, const double *sigma,
                          const double *cdf, int map, double t_near, double t_far, int32_t n_out,
                          int32_t stratified, uint64_t seed, double *s_out, double *t_out) {
  uint32_t key[2];
  philox_seed(seed, key);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r)
    importance_ray(r, n_in, s_edges, sigma, cdf, map, t_near, t_far, n_out, stratified, key, s_out,
                   t_out);
}

void or_importance_sample_ranged(int64_t n_rays, int32_t n_in, const double *s_edges,
                                 const double *sigma, const double *cdf, int map,
                                 const double *t_near, const double *t_far, int32_t n_out,
                                 int32_t stratified, uint64_t seed, double *s_out, double *t_out) {
  uint32_t key[2];
  philox_seed(seed, key);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r)
    importance_ray(r, n_in, s_edges, sigma, cdf, map, t_near[r], t_far[r], n_out, stratified, key,
                   s_out, t_out);
}

/* Combined estimator, grid stage (reading #18): the span of
 * the intervals nerfacc.sampling emits for the ray, by marching it. */
void or_ray_bounds(const or_grid *g, const uint8_t *occ, const or_march *p, const float *rays_o,
                   const float *rays_d, const float *t_min, const float *t_max, int64_t n_rays,
                   float *t_near, float *t_far) {
  gctx c;
  grid_ctx(g, &c);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    float nr = ray_near(p, t_min, r);
    float fr = t_max ? t_max[r] : p->far_plane;
    int64_t n = march_ray(&c, occ, p, rays_o + 3 * r, rays_d + 3 * r, nr, fr, 0, (int32_t)r, NULL,
                          NULL, NULL);
    t_near[r] = 0.0f;
    t_far[r] = 0.0f;
    if (n > 0) {
      float *a = (float *)malloc(sizeof(float) * n), *b = (float *)malloc(sizeof(float) * n);
      int32_t *id = (int32_t *)malloc(sizeof(int32_t) * n);
      march_ray(&c, occ, p, rays_o + 3 * r, rays_d + 3 * r, nr, fr, 0, (int32_t)r, a, b, id);
      t_near[r] = a[0];
      t_far[r] = b[n - 1];
      free(a); free(b); free(id);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Proposal supervision loss (reading #21 [ext]): the definition, O(nf·np).   */
/* ------------------------------------------------------------------------ */
static double pdf_bound(int32_t np, const double *th, const double *wh, double a, double b) {
  double B = 0.0;
  for (int32_t j = 0; j < np; ++j)
    if (th[j] < b && th[j + 1] > a) B += wh[j];
  return B;
}

void or_pdf_loss(int64_t n_rays, int32_t nf, const double *t, const double *w, int32_t np,
                 const double *th, const double *wh, double eps, double *loss) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    const double *tr = t + r * (nf + 1), *wr = w + r * nf, *hr = th + r * (np + 1), *vr = wh + r * np;
    double L = 0.0;
    for (int32_t i = 0; i < nf; ++i) {
      double res = wr[i] - pdf_bound(np, hr, vr, tr[i], tr[i + 1]);
      if (res > 0.0) L += res * res / (wr[i] + eps);
    }
    loss[r] = L;
  }
}

void or_pdf_loss_bwd(int64_t n_rays, int32_t nf, const double *t, const double *w, int32_t np,
                     const double *th, const double *wh, double eps, const double *g_loss,
                     double *g_wh) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rays; ++r) {
    const double *tr = t + r * (nf + 1), *wr = w + r * nf, *hr = th + r * (np + 1), *vr = wh + r * np;
    double *gr = g_wh + r * np;
    for (int32_t j = 0; j < np; ++j) gr[j] = 0.0;
    for (int32_t i = 0; i < nf; ++i) {
      double res = wr[i] - pdf_bound(np, hr, vr, tr[i], tr[i + 1]);
      if (!(res > 0.0)) continue;
      double c = -2.0 * g_loss[r] * res / (wr[i] + eps);
      for (int32_t j = 0; j < np; ++j)
        if (hr[j] < tr[i + 1] && hr[j + 1] > tr[i]) gr[j] += c;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* O9: occupancy-grid estimator update (P:240-241 EMA and threshold;          */
/* S:251-268; readings #20-#23).                                             */
/* ------------------------------------------------------------------------ */
void or_occgrid_points(const or_grid *g, uint64_t seed, int64_t step, int32_t jitter,
                       int64_t cell_begin, int64_t cell_count, float *xyz) {
  gctx c;
  grid_ctx(g, &c);
  uint32_t key[2];
  philox_seed(seed, key);
  const int64_t R = g->res, R3 = R * R * R;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < cell_count; ++q) {
    int64_t cell = cell_begin + q;
    int64_t l = cell / R3, idx = cell % R3;
    int64_t i[3] = {idx % R, (idx / R) % R, idx / (R * R)};
    double xi[3] = {0.5, 0.5, 0.5};
    if (jitter) {
      uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)step, (uint32_t)l, 2u}, out[4];
      or_philox4x32_10(ctr, key, out);
      for (int a = 0; a < 3; ++a) xi[a] = or_u24(out[a]);
    }
    for (int a = 0; a < 3; ++a) {
      double lo = (double)c.lo[l][a], hi = (double)c.hi[l][a];
      double cw = (hi - lo) / (double)R;
      xyz[3 * q + a] = (float)(lo + ((double)i[a] + xi[a]) * cw);
    }
  }
}

void or_occgrid_times(const or_grid *g, uint64_t seed, int64_t step, int32_t draw,
                      int64_t cell_begin, int64_t cell_count, float *times) {
  uint32_t key[2];
  philox_seed(seed, key);
  const int64_t R = g->res, R3 = R * R * R;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < cell_count; ++q) {
    int64_t cell = cell_begin + q;
    int64_t l = cell / R3, idx = cell % R3;
    uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)step, (uint32_t)l, 16u + (uint32_t)draw}, out[4];
    or_philox4x32_10(ctr, key, out);
    times[q] = (float)or_u24(out[0]);
  }
}

void or_occgrid_update(const or_grid *g, float *density, const float *fresh, int32_t rule,
                       float decay, float threshold, int32_t thresh_rule, uint8_t *occ_bits,
                       double *mean_out) {
  const int64_t R = g->res, n = (int64_t)g->levels * R * R * R;
  const double gam = (double)decay, one_m = 1.0 - gam;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < n; ++q) {
    double prev = (double)density[q], v = (double)fresh[q];
    double nd;
    if (rule == 0) {
      double a = gam * prev; /* σ^k = γ σ^{k-1} + (1-γ) σ_query */
      double b = one_m * v;
      nd = a + b;
    } else {
      double a = gam * prev; /* max-decay variant */
      nd = a > v ? a : v;
    }
    density[q] = (float)nd;
  }
  double sum = 0.0;
  for (int64_t q = 0; q < n; ++q) sum += (double)density[q];
  double mean = n > 0 ? sum / (double)n : 0.0;
  double tau = (double)threshold;
  if (thresh_rule == 1 && mean < tau) tau = mean;
  if (mean_out) *mean_out = mean;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < n; ++q) occ_bits[q] = ((double)density[q] > tau) ? 1 : 0; /* σ̂ = 1[σ > τ] */
}

/* ------------------------------------------------------------------------ */
/* O10 (validation only): analytic fields and the quadrature renderer.        */
/* ------------------------------------------------------------------------ */
double or_field_sigma(int kind, const double *prm, double sigma0, const double x[3]) {
  if (kind == 0) {
    for (int a = 0; a < 3; ++a)
      if (!(prm[a] <= x[a] && x[a] <= prm[3 + a])) return 0.0;
    return sigma0;
  }
  double r2 = 0.0;
  for (int a = 0; a < 3; ++a) r2 += (x[a] - prm[a]) * (x[a] - prm[a]);
  return r2 <= prm[3] * prm[3] ? sigma0 : 0.0;
}

void or_render_quadrature(int kind, const double *prm, double sigma0, const double o[3],
                          const double d[3], double t_a, double t_b, int64_t n_quad,
                          double *opacity, double *depth) {
  double dt = (t_b - t_a) / (double)n_quad, S = 0.0, O = 0.0, N = 0.0;
  for (int64_t i = 0; i < n_quad; ++i) {
    double ta = t_a + (double)i * dt, tb = t_a + (double)(i + 1) * dt, m = 0.5 * (ta + tb);
    double x[3] = {o[0] + m * d[0], o[1] + m * d[1], o[2] + m * d[2]};
    double si = or_field_sigma(kind, prm, sigma0, x) * (tb - ta);
    double w = exp(-S) * -expm1(-si);
    O += w;
    N += w * m;
    S += si;
  }
  *opacity = O;
  *depth = N / (O > 1e-10 ? O : 1e-10);
}
