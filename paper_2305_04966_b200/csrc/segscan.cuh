// segscan.cuh — warp-wide segmented scans over packed samples (ray-aligned tiles).
//
// A "segment" is one ray's run of consecutive samples in the packed tensor
// (P:83).  Warps own ray-aligned sample ranges, process them in chunks of
// 32 lanes x 4 samples, and carry the open segment across chunks, so no
// cross-warp look-back is needed.  Values are fp64 (readings #9, #11).
#pragma once
#include "common.cuh"

#ifndef NACC_SEG_FMA
#define NACC_SEG_FMA 0  // build parameter: segmented-sum operator as one DFMA per value (A/B on the render
                        // kernels: fwd 64.5 -> 62.3 us, bwd 69.4 -> 71.7 us; the 5-value SegM keeps it)
#endif

namespace nacc {

template <int K>
struct Seg {
  int f;        // 1 if a segment head lies in the covered range
  double v[K];  // sums since the last head (or since the start)
};

template <int K>
__device__ __forceinline__ Seg<K> seg_identity() {
  Seg<K> r;
  r.f = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) r.v[k] = 0.0;
  return r;
}

// associative segmented-sum operator: a then b
template <int K>
__device__ __forceinline__ Seg<K> seg_combine(const Seg<K> &a, const Seg<K> &b) {
  Seg<K> r;
  r.f = a.f | b.f;
#if NACC_SEG_FMA
  // a's sums continue into b unless b holds a head: fma(a, 1, b) = a + b rounded once and
  // fma(a, 0, b) = b exactly (finite a), one DFMA instead of a DADD and a two-word select
  const double keep = b.f ? 0.0 : 1.0;
#pragma unroll
  for (int k = 0; k < K; ++k) r.v[k] = __fma_rn(a.v[k], keep, b.v[k]);
#else
#pragma unroll
  for (int k = 0; k < K; ++k) r.v[k] = b.f ? b.v[k] : a.v[k] + b.v[k];
#endif
  return r;
}

template <int K>
__device__ __forceinline__ Seg<K> seg_shfl_up(const Seg<K> &x, int o) {
  Seg<K> y;
  y.f = __shfl_up_sync(kFull, x.f, o);
#pragma unroll
  for (int k = 0; k < K; ++k) y.v[k] = __shfl_up_sync(kFull, x.v[k], o);
  return y;
}

template <int K>
__device__ __forceinline__ Seg<K> warp_seg_incl(Seg<K> x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Seg<K> y = seg_shfl_up(x, o);
    if (lane >= o) x = seg_combine(y, x);
  }
  return x;
}

// Exclusive warp-wide segmented scan seeded with `carry` (the open segment of
// the previous chunk); advances `carry` to the chunk's inclusive total.
template <int K>
__device__ __forceinline__ Seg<K> warp_seg_excl(const Seg<K> &x, Seg<K> &carry) {
  const int lane = threadIdx.x & 31;
  const Seg<K> incl = warp_seg_incl(x);
  Seg<K> ex = seg_shfl_up(incl, 1);
  if (lane == 0) ex = seg_identity<K>();
  const Seg<K> res = seg_combine(carry, ex);
  Seg<K> last;
  last.f = __shfl_sync(kFull, incl.f, 31);
#pragma unroll
  for (int k = 0; k < K; ++k) last.v[k] = __shfl_sync(kFull, incl.v[k], 31);
  carry = seg_combine(carry, last);
  return res;
}

// number of samples in use: end of the last ray's run
__device__ __forceinline__ int64_t packed_end(const int64_t *__restrict__ packed_info, int64_t n_rays) {
  const longlong2 pi = __ldg(reinterpret_cast<const longlong2 *>(packed_info) + (n_rays - 1));
  return pi.x + pi.y;
}

// Ray-aligned tile boundary: the first ray start at or after sample q.
__device__ __forceinline__ int64_t snap_to_ray(const int64_t *__restrict__ packed_info,
                                               const int32_t *__restrict__ ray_id, int64_t q, int64_t N) {
  if (q >= N) return N;
  if (q <= 0) return 0;
  const int64_t r = __ldg(ray_id + q);
  const longlong2 pi = __ldg(reinterpret_cast<const longlong2 *>(packed_info) + r);
  return pi.x == q ? q : pi.x + pi.y;
}

}  // namespace nacc
