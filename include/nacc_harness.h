/*
 * nacc_harness.h — test/bench HARNESS, not part of the product ABI.
 *
 * The library never evaluates a radiance field (Alg. 1 passes the NeRF as
 * density_fn / rgb_density_fn callbacks).  To run whole synthetic
 * pipeline steps on the GPU the bench needs a stand-in NeRF: a dense
 * cell-centre lattice (σ, r, g, b) with trilinear interpolation,
 * optionally queried through the Mip-NeRF-360 contraction (DESIGN.md reading
 * #6), plus the MSE loss gradient of Alg. 1 line 48.  Same error conventions
 * as nacc.h; all pointers are device pointers.
 */
#ifndef NACC_HARNESS_H
#define NACC_HARNESS_H
#include <stdint.h>
#include <cuda_runtime_api.h>
#include "nacc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* σ (and rgb if non-NULL) at interval midpoints m = (t0+t1)/2 of packed
 * samples: x = o[ray_id] + m d[ray_id].  lattice: [res^3][4] fp32 (x fastest)
 * over [lo, hi]^3; zero outside; contracted != 0 queries contract(x). */
nacc_status naccx_field_at_samples(const float *lattice, int32_t res, float lo, float hi,
                                   int32_t contracted, const float *rays_o, const float *rays_d,
                                   const float *t0, const float *t1, const int32_t *ray_id,
                                   int64_t n, const int64_t *n_dev, float *sigma, float *rgb,
                                   cudaStream_t stream);
/* n is the arrays' capacity; n_dev (device int64, NULL = n) the count in use. */

/* σ only, from a density-only lattice [res^3] fp32 (same interpolation). */
nacc_status naccx_sigma_at_samples(const float *sigma_lattice, int32_t res, float lo, float hi,
                                   int32_t contracted, const float *rays_o, const float *rays_d,
                                   const float *t0, const float *t1, const int32_t *ray_id,
                                   int64_t n, const int64_t *n_dev, float *sigma,
                                   cudaStream_t stream);

/* out[i] = scale * σ(xyz[i]) for the occupancy-grid update (v = σ·Δt). */
nacc_status naccx_field_at_points(const float *lattice, int32_t res, float lo, float hi,
                                  int32_t contracted, const float *xyz, int64_t n, float scale,
                                  float *out, cudaStream_t stream);

/* g_color = 2 (color - gt) / (3 n): gradient of F.mse_loss (Alg. 1 line 48). */
nacc_status naccx_mse_grad(const float *color, const float *gt, int64_t n_rays, float *g_color,
                           cudaStream_t stream);

/* The same lattice in texture memory, sampled with hardware trilinear
 * filtering (8-bit fractional weights).  naccx_tex_create copies the lattice
 * (synchronises `stream`) and returns an opaque handle. */
nacc_status naccx_tex_create(const float *lattice, int32_t res, uint64_t *handle, cudaStream_t stream);
void naccx_tex_destroy(uint64_t handle);
nacc_status naccx_tex_at_samples(uint64_t handle, float lo, float hi, int32_t contracted,
                                 const float *rays_o, const float *rays_d, const float *t0,
                                 const float *t1, const int32_t *ray_id, int64_t n,
                                 const int64_t *n_dev, float *sigma, float *rgb,
                                 cudaStream_t stream);

uint64_t naccx_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
