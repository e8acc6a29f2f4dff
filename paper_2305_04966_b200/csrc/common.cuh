// common.cuh — shared device helpers of libnacc (sm_100a).  Product code:
// nothing here is shared with oracle/ (which is plain C with its own Philox).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <string>

#include "nacc.h"

namespace nacc {

// ---------------------------------------------------------------- error state
void set_error(const std::string &msg);
void clear_error();
void count_launch(int n = 1);

#define NACC_REQUIRE(cond, msg)                                   \
  do {                                                            \
    if (!(cond)) {                                                \
      ::nacc::set_error(std::string(__func__) + ": " + (msg));     \
      return NACC_ERR_INVALID_ARGUMENT;                           \
    }                                                             \
  } while (0)

#define NACC_CHECK_LAUNCH()                                                        \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess) {                                                       \
      ::nacc::set_error(std::string(__func__) + ": " + cudaGetErrorString(e_));     \
      return NACC_ERR_CUDA;                                                        \
    }                                                                              \
  } while (0)

#define NACC_CUDA(call)                                                            \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ::nacc::set_error(std::string(__func__) + ": " + cudaGetErrorString(e_));     \
      return NACC_ERR_CUDA;                                                        \
    }                                                                              \
  } while (0)

inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- Philox4x32-10
struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}
// 24-bit uniform in [0,1) as an exact double
__device__ __forceinline__ double u24(uint32_t x) { return (double)(x >> 8) * (1.0 / 16777216.0); }

// ---------------------------------------------------------------- warp scans
__device__ __forceinline__ double warp_incl_scan(double v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double n = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ int64_t warp_incl_scan_i64(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t n = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// ---------------------------------------------------------------- launch helpers
inline int grid_for(int64_t work_items, int per_block, int64_t cap = (1ll << 31) - 1) {
  int64_t g = ceil_div(work_items, per_block);
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// occupancy bitfield auxiliary skip mask (gridaux.cu)
constexpr int kMacroCells = 4;  // fine cells per macro cell and axis
#ifndef NACC_MARCH_WIN
#define NACC_MARCH_WIN 9  // largest fine-mask window (cells per axis) of cascaded grids
#endif
#ifndef NACC_MARCH_WIN1
#define NACC_MARCH_WIN1 5  // largest window of single-level grids (a 16-point segment of the CFG2 lattice spans <= 5)
#endif
constexpr int kFineWin = NACC_MARCH_WIN;
// windows w = 2..grid_fine_win(g) are built: cascades (cone lattices: a 16-point segment can span up to ~9
// cells per axis; A/B on CFG3 with 5 / 7 / 9: 2.72 / 2.39 / 2.36 ms) and single-level grids (CFG2: 5 / 9 equal)
int grid_fine_win(const nacc_grid &g);
bool grid_skip_enabled(const nacc_grid &g);
int64_t grid_aux_offset_words(const nacc_grid &g);   // start of the private region (gridaux.cu)
int64_t grid_mask2_offset_words(const nacc_grid &g);  // the macro skip mask
bool grid_fine_mask_enabled(const nacc_grid &g);      // single level: fine dilated mask present
int64_t grid_mask3_offset_words(const nacc_grid &g);  // the fine (3-cell dilated) skip mask
constexpr int kAuxHeaderWords = 64;                  // per-level occupied index boxes + world box
constexpr int kAuxBoxWord = 48;                      // 6 floats: padded world box of all occupied cells
cudaError_t grid_prepare(const nacc_grid &g, uint32_t *bits, cudaStream_t stream);

}  // namespace nacc
