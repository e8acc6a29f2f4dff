// lookback.cuh — single-pass exclusive scan across thread blocks (decoupled
// look-back): tiles take increasing ids from an atomic counter, publish their
// aggregate, and warp 0 walks back over predecessors (32 at a time) until it
// finds an inclusive prefix.  Used by the packing steps (start = exclusive
// prefix sum of counts) so count, scan and write happen in one kernel.
#pragma once
#include "common.cuh"

#ifndef NACC_LB_STATS
#define NACC_LB_STATS 0  // debug build: count look-back polls (nacc_debug_lb_stats)
#endif
#ifndef NACC_LB_NS0
#define NACC_LB_NS0 256  // first back-off of a look-back wait (ns); doubles up to NACC_LB_NSMAX (swept)
#endif
#ifndef NACC_LB_NSMAX
#define NACC_LB_NSMAX 4096
#endif

namespace nacc {

#if NACC_LB_STATS
// debug build only: [0] resolves, [1] poll iterations, [2] iterations that slept, [3] tiles walked
__device__ unsigned long long g_lb_stats[4];
#endif

struct LookbackWs {
  unsigned int tile_counter;
  unsigned int pad;
  unsigned long long status[1];  // [n_tiles]: (value << 2) | flag, flag 1 = aggregate, 2 = inclusive prefix
};

// The flag and the value share one 64-bit word and nothing else is read on the
// strength of the flag, so relaxed (strong, gpu-scope) accesses suffice; an
// acquire load would add an L1 invalidation (CCTL.IVALL) per spin iteration,
// evicting the occupancy bits the march keeps in L1.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// one warp: publish this tile's aggregate (tile 0 publishes its inclusive prefix)
__device__ __forceinline__ void lookback_publish(unsigned long long *st, int64_t tile, long long agg) {
  if ((threadIdx.x & 31) == 0) st_relaxed(st + tile, ((unsigned long long)agg << 2) | (tile == 0 ? 2ull : 1ull));
}

// one warp: after lookback_publish(tile, agg), walk back over the predecessors
// (32 at a time) to this tile's exclusive prefix, publish the inclusive one
// and return the exclusive one.  Only the predecessors nearer than the nearest
// published inclusive prefix are waited for (not the slowest of the 32 read).
// Predecessors publish their aggregates without waiting on anything, so the
// walk always terminates.
__device__ __forceinline__ long long lookback_resolve(unsigned long long *st, int64_t tile, long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  long long excl = 0;
  int64_t j = tile - 1;  // lanes look at tiles j, j-1, ..., j-31
  unsigned ns = NACC_LB_NS0;
  for (;;) {
    const int64_t idx = j - lane;
    const unsigned long long w = idx >= 0 ? ld_relaxed(st + idx) : 2ull;  // before tile 0: inclusive 0
    const unsigned m2 = __ballot_sync(kFull, (w & 3ull) == 2ull);
    const unsigned m0 = __ballot_sync(kFull, (w & 3ull) == 0ull);
    const int last = m2 ? __ffs(m2) - 1 : 31;  // nearest predecessor with an inclusive prefix
    const unsigned need = last == 31 ? kFull : ((2u << last) - 1u);
#if NACC_LB_STATS
    if (lane == 0) {
      atomicAdd(&g_lb_stats[1], 1ull);
      if (m0 & need) atomicAdd(&g_lb_stats[2], 1ull);
      else atomicAdd(&g_lb_stats[3], (unsigned long long)(last + 1));
    }
#endif
    if (m0 & need) {  // a tile we need has not published yet: back off and re-read the window
      __nanosleep(ns);
      ns = ns < NACC_LB_NSMAX ? 2 * ns : ns;
      continue;
    }
    long long v = lane <= last ? (long long)(w >> 2) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    excl += v;
    if (m2) break;
    j -= 32;
  }
  if (lane == 0) st_relaxed(st + tile, ((unsigned long long)(excl + agg) << 2) | 2ull);
#if NACC_LB_STATS
  if (lane == 0) atomicAdd(&g_lb_stats[0], 1ull);
#endif
  return excl;
}

}  // namespace nacc
