// field.cu — bench/test harness: the synthetic stand-in for the user's NeRF
// (Alg. 1 density_fn / rgb_density_fn).  Not part of libnacc.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "nacc_harness.h"

namespace {
std::atomic<uint64_t> g_launches{0};

__device__ __forceinline__ float4 lattice_at(const float4 *__restrict__ lat, int R, float lo, float hi, int contracted,
                                             float x, float y, float z) {
  if (contracted) {
    const float n = sqrtf(x * x + y * y + z * z);
    if (n > 1.0f) {
      const float s = (2.0f - 1.0f / n) / n;
      x *= s;
      y *= s;
      z *= s;
    }
  }
  if (!(x >= lo && x <= hi && y >= lo && y <= hi && z >= lo && z <= hi)) return make_float4(0.f, 0.f, 0.f, 0.f);
  const float sc = (float)R / (hi - lo);
  float u[3] = {(x - lo) * sc - 0.5f, (y - lo) * sc - 0.5f, (z - lo) * sc - 0.5f};
  int i0[3];
  float f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    u[a] = fminf(fmaxf(u[a], 0.0f), (float)(R - 1));
    i0[a] = min((int)floorf(u[a]), R - 2);
    f[a] = u[a] - (float)i0[a];
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
    const float w = (dx ? f[0] : 1.f - f[0]) * (dy ? f[1] : 1.f - f[1]) * (dz ? f[2] : 1.f - f[2]);
    const float4 v = __ldg(lat + (i0[0] + dx) + R * ((i0[1] + dy) + R * (i0[2] + dz)));
    acc.x += w * v.x;
    acc.y += w * v.y;
    acc.z += w * v.z;
    acc.w += w * v.w;
  }
  return acc;
}

// density-only lattice: one float per cell (the density query of Alg. 1 line 30
// does not need colour); same interpolation as lattice_at
__device__ __forceinline__ float lattice_sigma_at(const float *__restrict__ lat, int R, float lo, float hi,
                                                  int contracted, float x, float y, float z) {
  if (contracted) {
    const float n = sqrtf(x * x + y * y + z * z);
    if (n > 1.0f) {
      const float s = (2.0f - 1.0f / n) / n;
      x *= s;
      y *= s;
      z *= s;
    }
  }
  if (!(x >= lo && x <= hi && y >= lo && y <= hi && z >= lo && z <= hi)) return 0.f;
  const float sc = (float)R / (hi - lo);
  float u[3] = {(x - lo) * sc - 0.5f, (y - lo) * sc - 0.5f, (z - lo) * sc - 0.5f};
  int i0[3];
  float f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    u[a] = fminf(fmaxf(u[a], 0.0f), (float)(R - 1));
    i0[a] = min((int)floorf(u[a]), R - 2);
    f[a] = u[a] - (float)i0[a];
  }
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
    const float w = (dx ? f[0] : 1.f - f[0]) * (dy ? f[1] : 1.f - f[1]) * (dz ? f[2] : 1.f - f[2]);
    acc += w * __ldg(lat + (i0[0] + dx) + R * ((i0[1] + dy) + R * (i0[2] + dz)));
  }
  return acc;
}

// 4 consecutive samples per thread (vector loads); consecutive samples of a ray
// usually share the 2x2x2 corner block, whose values are reused
__global__ void field_sigma_kernel(const float *__restrict__ lat, int R, float lo, float hi, int contracted,
                                   const float *__restrict__ o, const float *__restrict__ d,
                                   const float *__restrict__ t0, const float *__restrict__ t1,
                                   const int32_t *__restrict__ rid, int64_t n, const int64_t *__restrict__ n_dev,
                                   float *__restrict__ sigma) {
  const int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t nn = n_dev ? min(n, *n_dev) : n;
  if (q0 >= nn) return;
  const bool vec = q0 + 3 < nn && ((reinterpret_cast<uintptr_t>(t0) | reinterpret_cast<uintptr_t>(t1) |
                                    reinterpret_cast<uintptr_t>(rid) | reinterpret_cast<uintptr_t>(sigma)) & 15) == 0;
  float a[4], b[4], out[4];
  int32_t ri[4];
  if (vec) {
    const float4 A = __ldg(reinterpret_cast<const float4 *>(t0 + q0)), Bv = __ldg(reinterpret_cast<const float4 *>(t1 + q0));
    const int4 Ri = __ldg(reinterpret_cast<const int4 *>(rid + q0));
    a[0] = A.x; a[1] = A.y; a[2] = A.z; a[3] = A.w;
    b[0] = Bv.x; b[1] = Bv.y; b[2] = Bv.z; b[3] = Bv.w;
    ri[0] = Ri.x; ri[1] = Ri.y; ri[2] = Ri.z; ri[3] = Ri.w;
  } else {
    for (int j = 0; j < 4; ++j) {
      const bool in = q0 + j < nn;
      a[j] = in ? __ldg(t0 + q0 + j) : 0.f;
      b[j] = in ? __ldg(t1 + q0 + j) : 0.f;
      ri[j] = in ? __ldg(rid + q0 + j) : -1;
    }
  }
  int32_t cur = -1;
  float ox = 0, oy = 0, oz = 0, dx = 0, dy = 0, dz = 0;
  int cached = -1;
  float cv[8];
  const float sc = (float)R / (hi - lo);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    out[j] = 0.f;
    if (ri[j] < 0) continue;
    if (ri[j] != cur) {
      cur = ri[j];
      ox = __ldg(o + 3 * cur); oy = __ldg(o + 3 * cur + 1); oz = __ldg(o + 3 * cur + 2);
      dx = __ldg(d + 3 * cur); dy = __ldg(d + 3 * cur + 1); dz = __ldg(d + 3 * cur + 2);
    }
    const float m = 0.5f * (a[j] + b[j]);
    float x = ox + m * dx, y = oy + m * dy, z = oz + m * dz;
    if (contracted) {
      const float nr = sqrtf(x * x + y * y + z * z);
      if (nr > 1.0f) {
        const float s2 = (2.0f - 1.0f / nr) / nr;
        x *= s2; y *= s2; z *= s2;
      }
    }
    if (!(x >= lo && x <= hi && y >= lo && y <= hi && z >= lo && z <= hi)) continue;
    float u[3] = {(x - lo) * sc - 0.5f, (y - lo) * sc - 0.5f, (z - lo) * sc - 0.5f};
    int i0[3];
    float f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      u[k] = fminf(fmaxf(u[k], 0.0f), (float)(R - 1));
      i0[k] = min((int)floorf(u[k]), R - 2);
      f[k] = u[k] - (float)i0[k];
    }
    const int base = i0[0] + R * (i0[1] + R * i0[2]);
    if (base != cached) {
      cached = base;
#pragma unroll
      for (int c = 0; c < 8; ++c) cv[c] = __ldg(lat + base + (c & 1) + R * (((c >> 1) & 1) + R * (c >> 2)));
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ddx = c & 1, ddy = (c >> 1) & 1, ddz = c >> 2;
      acc += (ddx ? f[0] : 1.f - f[0]) * (ddy ? f[1] : 1.f - f[1]) * (ddz ? f[2] : 1.f - f[2]) * cv[c];
    }
    out[j] = acc;
  }
  if (vec) {
    *reinterpret_cast<float4 *>(sigma + q0) = make_float4(out[0], out[1], out[2], out[3]);
  } else {
    for (int j = 0; j < 4; ++j)
      if (q0 + j < nn) sigma[q0 + j] = out[j];
  }
}

__global__ void field_samples_kernel(const float4 *__restrict__ lat, int R, float lo, float hi, int contracted,
                                     const float *__restrict__ o, const float *__restrict__ d,
                                     const float *__restrict__ t0, const float *__restrict__ t1,
                                     const int32_t *__restrict__ rid, int64_t n, const int64_t *__restrict__ n_dev,
                                     float *__restrict__ sigma, float *__restrict__ rgb) {
  const int64_t nn = n_dev ? min(n, *n_dev) : n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = __ldg(rid + i);
    const float m = 0.5f * (__ldg(t0 + i) + __ldg(t1 + i));
    const float x = __ldg(o + 3 * r) + m * __ldg(d + 3 * r);
    const float y = __ldg(o + 3 * r + 1) + m * __ldg(d + 3 * r + 1);
    const float z = __ldg(o + 3 * r + 2) + m * __ldg(d + 3 * r + 2);
    const float4 v = lattice_at(lat, R, lo, hi, contracted, x, y, z);
    sigma[i] = v.x;
    if (rgb) {
      rgb[3 * i] = v.y;
      rgb[3 * i + 1] = v.z;
      rgb[3 * i + 2] = v.w;
    }
  }
}

__global__ void field_points_kernel(const float4 *__restrict__ lat, int R, float lo, float hi, int contracted,
                                    const float *__restrict__ xyz, int64_t n, float scale, float *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 v = lattice_at(lat, R, lo, hi, contracted, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  out[i] = scale * v.x;
}

__global__ void mse_grad_kernel(const float *__restrict__ c, const float *__restrict__ gt, int64_t n3, float k,
                                float *__restrict__ g) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) g[i] = k * (c[i] - gt[i]);
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }
// grid-stride kernels driven by a device count: cap the launch at a few waves
inline unsigned blocks_capped(int64_t n) {
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 1;
  }
  const int64_t b = (n + 255) / 256, cap = (int64_t)n_sm * 32;
  return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}
}  // namespace

extern "C" {

nacc_status naccx_field_at_samples(const float *lattice, int32_t res, float lo, float hi, int32_t contracted,
                                   const float *rays_o, const float *rays_d, const float *t0, const float *t1,
                                   const int32_t *ray_id, int64_t n, const int64_t *n_dev, float *sigma, float *rgb,
                                   cudaStream_t stream) {
  if (n < 0 || res < 2 || !(hi > lo)) return NACC_ERR_INVALID_ARGUMENT;
  if (n == 0) return NACC_OK;
  if (!lattice || !rays_o || !rays_d || !t0 || !t1 || !ray_id || !sigma) return NACC_ERR_INVALID_ARGUMENT;
  field_samples_kernel<<<n_dev ? blocks_capped(n) : blocks_for(n), 256, 0, stream>>>(reinterpret_cast<const float4 *>(lattice), res, lo, hi,
                                                          contracted, rays_o, rays_d, t0, t1, ray_id, n, n_dev, sigma,
                                                          rgb);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? NACC_OK : NACC_ERR_CUDA;
}

nacc_status naccx_field_at_points(const float *lattice, int32_t res, float lo, float hi, int32_t contracted,
                                  const float *xyz, int64_t n, float scale, float *out, cudaStream_t stream) {
  if (n < 0 || res < 2 || !(hi > lo)) return NACC_ERR_INVALID_ARGUMENT;
  if (n == 0) return NACC_OK;
  if (!lattice || !xyz || !out) return NACC_ERR_INVALID_ARGUMENT;
  field_points_kernel<<<blocks_for(n), 256, 0, stream>>>(reinterpret_cast<const float4 *>(lattice), res, lo, hi,
                                                         contracted, xyz, n, scale, out);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? NACC_OK : NACC_ERR_CUDA;
}

nacc_status naccx_mse_grad(const float *color, const float *gt, int64_t n_rays, float *g_color, cudaStream_t stream) {
  if (n_rays < 0) return NACC_ERR_INVALID_ARGUMENT;
  if (n_rays == 0) return NACC_OK;
  if (!color || !gt || !g_color) return NACC_ERR_INVALID_ARGUMENT;
  mse_grad_kernel<<<blocks_for(3 * n_rays), 256, 0, stream>>>(color, gt, 3 * n_rays, 2.0f / (3.0f * (float)n_rays),
                                                              g_color);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? NACC_OK : NACC_ERR_CUDA;
}

nacc_status naccx_sigma_at_samples(const float *sigma_lattice, int32_t res, float lo, float hi, int32_t contracted,
                                   const float *rays_o, const float *rays_d, const float *t0, const float *t1,
                                   const int32_t *ray_id, int64_t n, const int64_t *n_dev, float *sigma,
                                   cudaStream_t stream) {
  if (n < 0 || res < 2 || !(hi > lo)) return NACC_ERR_INVALID_ARGUMENT;
  if (n == 0) return NACC_OK;
  if (!sigma_lattice || !rays_o || !rays_d || !t0 || !t1 || !ray_id || !sigma) return NACC_ERR_INVALID_ARGUMENT;
  field_sigma_kernel<<<blocks_for((n + 3) / 4), 256, 0, stream>>>(sigma_lattice, res, lo, hi, contracted, rays_o,
                                                                  rays_d, t0, t1, ray_id, n, n_dev, sigma);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? NACC_OK : NACC_ERR_CUDA;
}

}  // extern "C"

// ---------------------------------------------------------------- texture-unit field
// The same cell-centre lattice held in 3-D CUDA arrays and sampled by the
// texture unit (hardware trilinear filtering, clamp-to-edge, unnormalised
// coordinates: texel i is centred at i + 0.5, so u = (x - lo) R / (hi - lo) is
// the cell-centre lattice coordinate of the numpy field).  Hardware filtering
// uses 8-bit fractional weights, which is fine for a stand-in NeRF.
struct TexField {
  cudaArray_t a_sig = nullptr, a_rgba = nullptr;
  cudaTextureObject_t t_sig = 0, t_rgba = 0;
  int res = 0;
};

extern "C" nacc_status naccx_tex_create(const float *lattice, int32_t res, uint64_t *handle, cudaStream_t stream) {
  if (!lattice || res < 2 || !handle) return NACC_ERR_INVALID_ARGUMENT;
  TexField *f = new TexField();
  f->res = res;
  const cudaExtent ext = make_cudaExtent(res, res, res);
  cudaChannelFormatDesc d1 = cudaCreateChannelDesc<float>(), d4 = cudaCreateChannelDesc<float4>();
  if (cudaMalloc3DArray(&f->a_sig, &d1, ext) != cudaSuccess || cudaMalloc3DArray(&f->a_rgba, &d4, ext) != cudaSuccess) {
    delete f;
    return NACC_ERR_CUDA;
  }
  // rgba lattice: copy the (σ, r, g, b) float4 lattice as is; σ-only: strided copy of the first channel
  cudaMemcpy3DParms c4 = {};
  c4.srcPtr = make_cudaPitchedPtr(const_cast<float *>(lattice), (size_t)res * 16, res, res);
  c4.dstArray = f->a_rgba;
  c4.extent = ext;
  c4.kind = cudaMemcpyDeviceToDevice;
  float *sig = nullptr;
  if (cudaMemcpy3DAsync(&c4, stream) != cudaSuccess || cudaMalloc(&sig, (size_t)res * res * res * 4) != cudaSuccess)
    return NACC_ERR_CUDA;
  if (cudaMemcpy2DAsync(sig, 4, lattice, 16, 4, (size_t)res * res * res, cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
    return NACC_ERR_CUDA;
  cudaMemcpy3DParms c1 = {};
  c1.srcPtr = make_cudaPitchedPtr(sig, (size_t)res * 4, res, res);
  c1.dstArray = f->a_sig;
  c1.extent = ext;
  c1.kind = cudaMemcpyDeviceToDevice;
  if (cudaMemcpy3DAsync(&c1, stream) != cudaSuccess) return NACC_ERR_CUDA;
  cudaStreamSynchronize(stream);
  cudaFree(sig);
  for (int which = 0; which < 2; ++which) {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = which ? f->a_rgba : f->a_sig;
    cudaTextureDesc td = {};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModeLinear;
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    if (cudaCreateTextureObject(which ? &f->t_rgba : &f->t_sig, &rd, &td, nullptr) != cudaSuccess) return NACC_ERR_CUDA;
  }
  *handle = reinterpret_cast<uint64_t>(f);
  return NACC_OK;
}

extern "C" void naccx_tex_destroy(uint64_t handle) {
  TexField *f = reinterpret_cast<TexField *>(handle);
  if (!f) return;
  cudaDestroyTextureObject(f->t_sig);
  cudaDestroyTextureObject(f->t_rgba);
  cudaFreeArray(f->a_sig);
  cudaFreeArray(f->a_rgba);
  delete f;
}

__device__ __forceinline__ bool tex_coord(float lo, float hi, float sc, int contracted, float &x, float &y, float &z) {
  if (contracted) {
    const float n = sqrtf(x * x + y * y + z * z);
    if (n > 1.0f) {
      const float s = (2.0f - 1.0f / n) / n;
      x *= s;
      y *= s;
      z *= s;
    }
  }
  if (!(x >= lo && x <= hi && y >= lo && y <= hi && z >= lo && z <= hi)) return false;
  x = (x - lo) * sc;
  y = (y - lo) * sc;
  z = (z - lo) * sc;
  return true;
}

template <bool kRGB>
__global__ void tex_samples_kernel(cudaTextureObject_t tex, int R, float lo, float hi, int contracted,
                                   const float *__restrict__ o, const float *__restrict__ d,
                                   const float *__restrict__ t0, const float *__restrict__ t1,
                                   const int32_t *__restrict__ rid, int64_t n, const int64_t *__restrict__ n_dev,
                                   float *__restrict__ sigma, float *__restrict__ rgb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (n_dev && i >= *n_dev)) return;
  const int64_t r = __ldg(rid + i);
  const float m = 0.5f * (__ldg(t0 + i) + __ldg(t1 + i));
  float x = __ldg(o + 3 * r) + m * __ldg(d + 3 * r);
  float y = __ldg(o + 3 * r + 1) + m * __ldg(d + 3 * r + 1);
  float z = __ldg(o + 3 * r + 2) + m * __ldg(d + 3 * r + 2);
  const bool in = tex_coord(lo, hi, (float)R / (hi - lo), contracted, x, y, z);
  if (kRGB) {
    const float4 v = in ? tex3D<float4>(tex, x, y, z) : make_float4(0.f, 0.f, 0.f, 0.f);
    sigma[i] = v.x;
    rgb[3 * i] = v.y;
    rgb[3 * i + 1] = v.z;
    rgb[3 * i + 2] = v.w;
  } else {
    sigma[i] = in ? tex3D<float>(tex, x, y, z) : 0.f;
  }
}

// density only, 4 consecutive samples per thread (vector loads/stores, four
// independent texture fetches in flight)
constexpr int kTexQuads = 1;  // quads of samples per thread and iteration (2 measured slower)

#ifndef NACCX_TEX_MINB
#define NACCX_TEX_MINB 1  // build parameter: min resident 256-thread blocks per SM (register cap)
#endif
__global__ void __launch_bounds__(256, NACCX_TEX_MINB) tex_sigma4_kernel(cudaTextureObject_t tex, int R, float lo, float hi, int contracted,
                                  const float *__restrict__ o, const float *__restrict__ d,
                                  const float *__restrict__ t0, const float *__restrict__ t1,
                                  const int32_t *__restrict__ rid, int64_t n, const int64_t *__restrict__ n_dev,
                                  float *__restrict__ sigma) {
  const int64_t nn = n_dev ? min(n, *n_dev) : n;
  const float sc = (float)R / (hi - lo);
  constexpr int kS = 4 * kTexQuads;
  for (int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kS; q0 < nn;
       q0 += (int64_t)gridDim.x * blockDim.x * kS) {
    float a[kS], b[kS], out[kS];
    int32_t ri[kS];
    const bool full = q0 + kS - 1 < nn;
    if (full) {
#pragma unroll
      for (int g = 0; g < kTexQuads; ++g) {
        const float4 A = __ldg(reinterpret_cast<const float4 *>(t0 + q0) + g);
        const float4 Bv = __ldg(reinterpret_cast<const float4 *>(t1 + q0) + g);
        const int4 Ri = __ldg(reinterpret_cast<const int4 *>(rid + q0) + g);
        a[4 * g] = A.x; a[4 * g + 1] = A.y; a[4 * g + 2] = A.z; a[4 * g + 3] = A.w;
        b[4 * g] = Bv.x; b[4 * g + 1] = Bv.y; b[4 * g + 2] = Bv.z; b[4 * g + 3] = Bv.w;
        ri[4 * g] = Ri.x; ri[4 * g + 1] = Ri.y; ri[4 * g + 2] = Ri.z; ri[4 * g + 3] = Ri.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kS; ++j) {
        const bool in = q0 + j < nn;
        a[j] = in ? __ldg(t0 + q0 + j) : 0.f;
        b[j] = in ? __ldg(t1 + q0 + j) : 0.f;
        ri[j] = in ? __ldg(rid + q0 + j) : 0;
      }
    }
    float ox = 0.f, oy = 0.f, oz = 0.f, dx = 0.f, dy = 0.f, dz = 0.f;
#pragma unroll
    for (int j = 0; j < kS; ++j) {
      const int64_t r = ri[j];
      if (j == 0 || ri[j] != ri[j - 1]) {  // samples are grouped by ray: reload only on a new ray
        ox = __ldg(o + 3 * r);
        oy = __ldg(o + 3 * r + 1);
        oz = __ldg(o + 3 * r + 2);
        dx = __ldg(d + 3 * r);
        dy = __ldg(d + 3 * r + 1);
        dz = __ldg(d + 3 * r + 2);
      }
      const float m = 0.5f * (a[j] + b[j]);
      float x = ox + m * dx;
      float y = oy + m * dy;
      float z = oz + m * dz;
      const bool in = tex_coord(lo, hi, sc, contracted, x, y, z);
      out[j] = in ? tex3D<float>(tex, x, y, z) : 0.f;
    }
    if (full) {
#pragma unroll
      for (int g = 0; g < kTexQuads; ++g)
        reinterpret_cast<float4 *>(sigma + q0)[g] = make_float4(out[4 * g], out[4 * g + 1], out[4 * g + 2],
                                                                out[4 * g + 3]);
    } else {
      for (int j = 0; j < kS; ++j)
        if (q0 + j < nn) sigma[q0 + j] = out[j];
    }
  }
}

extern "C" nacc_status naccx_tex_at_samples(uint64_t handle, float lo, float hi, int32_t contracted, const float *rays_o,
                                 const float *rays_d, const float *t0, const float *t1, const int32_t *ray_id,
                                 int64_t n, const int64_t *n_dev, float *sigma, float *rgb, cudaStream_t stream) {
  TexField *f = reinterpret_cast<TexField *>(handle);
  if (!f || n < 0 || !(hi > lo)) return NACC_ERR_INVALID_ARGUMENT;
  if (n == 0) return NACC_OK;
  if (rgb)
    tex_samples_kernel<true><<<blocks_for(n), 256, 0, stream>>>(f->t_rgba, f->res, lo, hi, contracted, rays_o, rays_d,
                                                                t0, t1, ray_id, n, n_dev, sigma, rgb);
  else if (((reinterpret_cast<uintptr_t>(t0) | reinterpret_cast<uintptr_t>(t1) | reinterpret_cast<uintptr_t>(ray_id) |
              reinterpret_cast<uintptr_t>(sigma)) & 15) == 0)
    tex_sigma4_kernel<<<n_dev ? blocks_capped((n + 4 * kTexQuads - 1) / (4 * kTexQuads))
                                    : blocks_for((n + 4 * kTexQuads - 1) / (4 * kTexQuads)), 256, 0, stream>>>(f->t_sig, f->res, lo, hi, contracted, rays_o, rays_d,
                                                                    t0, t1, ray_id, n, n_dev, sigma);
  else
    tex_samples_kernel<false><<<blocks_for(n), 256, 0, stream>>>(f->t_sig, f->res, lo, hi, contracted, rays_o, rays_d,
                                                                 t0, t1, ray_id, n, n_dev, sigma, nullptr);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? NACC_OK : NACC_ERR_CUDA;
}

extern "C" uint64_t naccx_launch_count(void) { return g_launches.load(); }


