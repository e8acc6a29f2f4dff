/*
 * oracle.h — plain, slow, obviously-correct CPU reference for the NerfAcc
 * packed-sample volume-rendering hot path (arXiv 2305.04966).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product (paper_2305_04966_b200/, include/nacc.h) never links, imports or
 * executes anything under oracle/, and this file includes nothing from it.
 *
 * Citation convention: P:n = /root/reference/PAPER.md line n (with section,
 * equation or algorithm); S:n = /root/reference/SPEC.md line n; "reading #k"
 * = DESIGN.md §3 (readings of the paper where it is silent or garbled).
 *
 * Precision: fp64 throughout, except where floating point decides an integer
 * (lattice membership, cell index): there both sides take the decision in the
 * kernel's precision, fp32, with the exact op sequence stated below
 * (reading #3).  Build flags: -O2 -fno-fast-math -ffp-contract=off,
 * so the only fused multiply-adds are the explicit fma()/fmaf() calls.
 *
 * Parity status per function (DESIGN.md §4 lists the pins):
 *   or_philox4x32_10      pinned (Random123 known-answer vectors)
 *   or_ray_aabb           pinned
 *   or_march_*            pinned (all-empty, all-occupied closed form,
 *                         brute force, sphere closed form, invariants);
 *                         cascade + cone readings #4/#5: pinned only by
 *                         reductions and brute force (no paper values)
 *   or_filter_early_stop  pinned (monotonicity, P:86 bound)
 *   or_render_fwd/bwd     pinned (closed forms, finite differences)
 *   or_accumulate_*       pinned (closed forms)
 *   or_weights_alpha_*    pinned (closed form, density-path equivalence, telescoping, finite differences)
 *   or_importance_sample  pinned (KS, strata, backward error)
 *   or_importance_sample_ranged, or_ray_bounds  pinned (reduction to the pinned
 *                         scalar sampler / march, slab closed form, culling)
 *   or_occgrid_*          pinned
 *   or_occgrid_times      pinned (Philox KAT via or_philox4x32_10, u24 grid, uniformity)
 *   or_pdf_loss(_bwd)     pinned (self-bound zero, single-bin closed form, coarsening bound, FD)
 */
#ifndef NACC_ORACLE_H
#define NACC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Philox4x32-10 counter-based generator (Salmon et al. 2011); both sides
 * implement it independently (task rule ③).  key[0] = low 32 bits of the seed,
 * key[1] = high 32 bits. */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* uniform in [0,1): (x >> 8) * 2^-24 */
double or_u24(uint32_t x);

/* O1 slab test.  Returns 1 and writes [t_enter, t_exit] if the ray
 * meets the half-open box [lo, hi) over t in [near, far]; 0 otherwise. */
int or_ray_aabb(const double o[3], const double d[3], const double lo[3], const double hi[3],
                double near, double far, double *t_enter, double *t_exit);

/* Lindisp / identity contraction Φ(s).  map 0 = identity
 * t = tn + s (tf - tn); map 1 = reciprocal depth 1/t = (1-s)/tn + s/tf. */
double or_contract(int map, double s, double tn, double tf);
double or_uncontract(int map, double t, double tn, double tf);

/* Occupancy-grid description (level-l box = centre ± half·2^l, reading #4). */
typedef struct {
  int32_t levels;
  int32_t res;
  float roi[6]; /* lo_x lo_y lo_z hi_x hi_y hi_z of level 0 */
} or_grid;

typedef struct {
  float near_plane, far_plane; /* defaults when t_min/t_max are NULL */
  float step;                  /* Δt (uniform) or Δt_min (cone) */
  float max_step;              /* Δt_max (cone only) */
  float cone_angle;            /* c; 0 = uniform lattice */
  int32_t stratified;          /* jitter the lattice anchor per ray */
  uint64_t seed;
} or_march;

/* Uniform lattice value fp32(near_r + (k + half/2)·Δt), the exact real rounded
 * once (reading #3): t_k (half = 0) or the midpoint m_k (half = 1).  Pinned
 * against exact rationals, including fp64 double-rounding ties. */
float or_lattice_point(float near_r, float step, int64_t k, int32_t half);

/* O2-O4: every lattice interval whose midpoint lies in an occupied cell, in
 * ray/t order ("sample as interval", "packed tensor"; P:240 skipping).
 * occ: uint8 per cell, level-major, x-fastest (reading #27).
 * brute = 1 evaluates the membership predicate for every k >= 0 up to a bound
 * past which no point can lie in the outermost box (the definition);
 * brute = 0 restricts k to the fp64 slab interval ±2 steps (the fast oracle).
 * Pass 1: or_march_count(..., counts) writes count per ray.
 * Pass 2: or_march_fill(..., start, t0, t1, ray_id) writes the samples at
 * start[r] .. start[r]+count[r]-1. */
void or_march_count(const or_grid *g, const uint8_t *occ, const or_march *p,
                    const float *rays_o, const float *rays_d, const float *t_min,
                    const float *t_max, int64_t n_rays, int brute, int64_t *counts);
void or_march_fill(const or_grid *g, const uint8_t *occ, const or_march *p,
                   const float *rays_o, const float *rays_d, const float *t_min,
                   const float *t_max, int64_t n_rays, int brute, const int64_t *start,
                   float *t0, float *t1, int32_t *ray_id);

/* O5 no-gradient early-stop filter (reading #9).
 * Per ray: keep the prefix of samples whose ENTERING optical depth S_i
 * satisfies S_i <= neg_log_eps.  Writes the kept count per ray into
 * counts_out and, for samples i < cut, the margin |S_i - neg_log_eps| minimum
 * into margin_out[r] (NULL allowed). */
void or_filter_cut(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                   const double *sigma, double neg_log_eps, int64_t *counts_out,
                   double *margin_out);

/* O6 render forward (Eq. 2, discretised as P:246 with the
 * index typo read as σ(t_j), reading #11).  Per-sample outputs (NULL allowed):
 * trans T_i, alphas α_i, weights w_i.  Per-ray: color[3], opacity, depth,
 * and the fp64 sums (C[3], O, N) in ctx[5] (NULL allowed). */
void or_render_fwd(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                   const double *sigma, const double *rgb /* [N][3] or NULL */, double neg_log_eps,
                   double *trans, double *alphas, double *weights, double *color,
                   double *opacity, double *depth);

/* O7 render backward (t detached P:78).  Given upstream gradients of
 * color/opacity/depth (any may be NULL = 0), writes g_sigma and g_rgb. */
void or_render_bwd(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                   const double *sigma, const double *rgb, double neg_log_eps,
                   const double *g_color, const double *g_opacity, const double *g_depth,
                   double *g_sigma, double *g_rgb);

/* Transmittance estimator backward from per-sample weight (and optional
 * transmittance) gradients: g_sigma_i = δ_i (g_w_i T_i (1-α_i) - Σ_{j>i} g_w_j w_j
 * - Σ_{j>i} g_T_j T_j). */
void or_weights_bwd(const int64_t *packed_info, int64_t n_rays, const double *t0, const double *t1,
                    const double *sigma, double neg_log_eps, const double *g_weights,
                    const double *g_trans /* NULL allowed */, double *g_sigma);

/* Alpha compositing for fields that supply α per interval (SDF-based fields,
 * P:61; "accumulating them through alpha-composition"; SURVEY §8(f)
 * row 2): T_i = Π_{j<i} (1 − α_j), sequential fp64 product; w_i = T_i α_i for
 * live samples, 0 once T_i < ε_T with ε_T = exp(−neg_log_eps) (DESIGN.md
 * reading #27).  trans may be NULL. */
void or_weights_alpha_fwd(const int64_t *packed_info, int64_t n_rays, const double *alpha,
                          double neg_log_eps, double *weights, double *trans);

/* Its backward, the product rule written out (no division, so α = 1 is
 * safe): g_α_k = [live_k] g_w_k T_k − Σ_{i>k} ([live_i] g_w_i α_i + g_T_i)
 * Π_{j<i, j≠k} (1 − α_j); the liveness mask is a constant (reading #28).
 * O(n²) per ray.  g_trans may be NULL. */
void or_weights_alpha_bwd(const int64_t *packed_info, int64_t n_rays, const double *alpha,
                          double neg_log_eps, const double *g_weights, const double *g_trans,
                          double *g_alpha);

/* accumulate_along_rays: out[r][c] = Σ_i w_i v_i[c] (values NULL = ones). */
void or_accumulate(const int64_t *packed_info, int64_t n_rays, const double *weights,
                   const double *values, int32_t C, double *out);
void or_accumulate_bwd(const int64_t *packed_info, int64_t n_rays, const double *weights,
                       const double *values, int32_t C, const double *g_out, double *g_weights,
                       double *g_values /* NULL allowed */);

/* O8 inverse-CDF resampling of interval edges in s-space (Eq. 1 P:191-195,
 * CDF = 1 - T Eq. 3, s-space P:257; readings #16-19).
 * Exactly one of sigma [n_rays][n_in] / cdf [n_rays][n_in+1] is non-NULL.
 * Writes s_out [n_rays][n_out+1] and, if non-NULL, t_out = Φ(s_out). */
void or_importance_sample(int64_t n_rays, int32_t n_in, const double *s_edges, const double *sigma,
                          const double *cdf, int map, double t_near, double t_far, int32_t n_out,
                          int32_t stratified, uint64_t seed, double *s_out, double *t_out);
/* The same with a per-ray [t_near_r, t_far_r] (the combined estimator's
 * proposal stage); a ray with !(t_far_r > t_near_r) is culled:
 * s_out uniform over [e_0, e_m], t_out = t_near_r (reading #19). */
void or_importance_sample_ranged(int64_t n_rays, int32_t n_in, const double *s_edges,
                                 const double *sigma, const double *cdf, int map,
                                 const double *t_near, const double *t_far, int32_t n_out,
                                 int32_t stratified, uint64_t seed, double *s_out, double *t_out);
/* Combined estimator, grid stage ("stacking an occupancy grid on top
 * of the proposal network ... reduce the number of rays and shrink the
 * near-far plane"; reading #18): per ray, t_near = t0 of the first
 * interval or_march emits and t_far = t1 of its last; both 0 when it emits
 * none (the ray is culled). */
void or_ray_bounds(const or_grid *g, const uint8_t *occ, const or_march *p, const float *rays_o,
                   const float *rays_d, const float *t_min, const float *t_max, int64_t n_rays,
                   float *t_near, float *t_far);
/* the normalised CDF F̂ the sampler inverts (for backward-error checks) */
void or_importance_cdf(int64_t n_rays, int32_t n_in, const double *s_edges, const double *sigma,
                       const double *cdf, int map, double t_near, double t_far, double *cdf_hat);

/* Proposal supervision (the paper names Mip-NeRF 360's
 * "PDF matching loss" that trains the proposal network; its form is
 * [ext], reading #21).  Dense per-ray histograms: final edges t
 * [n][nf+1] with weights w [n][nf]; proposal edges th [n][np+1] with weights
 * wh [n][np].  B_i = Σ_j wh_j over the proposal intervals overlapping
 * (t_i, t_{i+1}) (th_j < t_{i+1} and th_{j+1} > t_i); loss_r = Σ_i
 * max(0, w_i − B_i)² / (w_i + eps).  The backward returns g_wh only (w is a
 * stop-gradient target): g_wh_j = −2 g_loss_r Σ_{i overlapping j} max(0, w_i − B_i) / (w_i + eps). */
void or_pdf_loss(int64_t n_rays, int32_t nf, const double *t, const double *w, int32_t np,
                 const double *th, const double *wh, double eps, double *loss);
void or_pdf_loss_bwd(int64_t n_rays, int32_t nf, const double *t, const double *w, int32_t np,
                     const double *th, const double *wh, double eps, const double *g_loss,
                     double *g_wh);

/* O9 occupancy-grid update (readings #20-23).
 * Points: x = lo_l + (i + ξ)(hi_l - lo_l)/R with ξ from Philox(seed, (i_cell, step, l, 0)),
 * or ξ = 1/2 when jitter == 0. */
void or_occgrid_points(const or_grid *g, uint64_t seed, int64_t step, int32_t jitter,
                       int64_t cell_begin, int64_t cell_count, float *xyz);
/* Dynamic scenes (one grid shared across frames holds "the maximum
 * opacity at this area over all the timestamps"; reading
 * #20): draw j of the per-cell timestamp, t = u24(Philox(seed, (i_cell, step,
 * l, 16 + j)).x) in [0, 1).  The caller evaluates σ(x, t) per draw and merges
 * the draws with MAX before the update. */
void or_occgrid_times(const or_grid *g, uint64_t seed, int64_t step, int32_t draw,
                      int64_t cell_begin, int64_t cell_count, float *times);
/* rule 0 = EMA, 1 = max-decay; thresh_rule 0 = fixed τ, 1 = min(τ, mean).
 * density is updated in place; occ_bits receives one uint8 per cell. */
void or_occgrid_update(const or_grid *g, float *density, const float *fresh, int32_t rule,
                       float decay, float threshold, int32_t thresh_rule, uint8_t *occ_bits,
                       double *mean_out);

/* O10 validation-only: analytic fields and the n_quad uniform
 * quadrature renderer.  kind 0 = constant box (params: lo[3],
 * hi[3]), kind 1 = sphere (centre[3], radius). */
double or_field_sigma(int kind, const double *params, double sigma0, const double x[3]);
void or_render_quadrature(int kind, const double *params, double sigma0, const double o[3],
                          const double d[3], double t_a, double t_b, int64_t n_quad,
                          double *opacity, double *depth);

int or_num_threads(void);
void or_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
