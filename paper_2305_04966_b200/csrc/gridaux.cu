// gridaux.cu — the occupancy bitfield's auxiliary region.
//
// After the public fine bits (cell q -> bit q & 31 of word q >> 5, nacc.h) the
// bitfield buffer holds library-private data used by the march to skip empty
// space, rebuilt when the bits change (nacc_occgrid_update,
// nacc_grid_prepare), not on every march:
//   header (64 words): per level the index box of its occupied cells (int32
//     x0,y0,z0,x1,y1,z1 at 6l) and the world box enclosing every occupied cell
//     of every level, padded (6 floats at word 48; lo > hi when none is);
//   mask2 (when skipping is enabled): for every macro cell m (4^3 fine cells)
//     of every level, the OR of the fine bits of macro cells m + {0,1}^3,
//     i.e. of the fine cells [4m, 4m + 8)^3 clipped to the level;
//   mask3 (every grid with skipping; per level): for every fine cell c and every
//     window size w = 2..W (W = grid_fine_win: 9 for cascades, 5 for one level), the OR and the AND of the fine bits of
//     cells c + {0..w-1}^3 clipped to the level, at the fine resolution, stored as
//     OR_2, AND_2, OR_3, AND_3, ..., OR_W, AND_W (the march's segment test picks the
//     window of its segment's cell span: a 16-point segment spans at most 5 cells
//     per axis on the CFG lattices; a tighter window skips and solidifies more);
#include "common.cuh"

#include <type_traits>

namespace nacc {

bool grid_skip_enabled(const nacc_grid &g) { return g.res % kMacroCells == 0 && g.res >= 2 * kMacroCells; }

int64_t grid_aux_offset_words(const nacc_grid &g) {
  const int64_t cells = (int64_t)g.levels * g.res * g.res * g.res;
  return ceil_div(ceil_div(cells, 32), 64) * 64;  // 256-byte aligned
}

int64_t grid_mask2_offset_words(const nacc_grid &g) { return grid_aux_offset_words(g) + kAuxHeaderWords; }

static int64_t mask2_words(const nacc_grid &g) {
  const int64_t M = g.res / kMacroCells;
  return ceil_div(ceil_div((int64_t)g.levels * M * M * M, 32), 64) * 64;
}

bool grid_fine_mask_enabled(const nacc_grid &g) { return grid_skip_enabled(g); }

int grid_fine_win(const nacc_grid &g) { return g.levels > 1 ? kFineWin : (kFineWin < NACC_MARCH_WIN1 ? kFineWin : NACC_MARCH_WIN1); }

int64_t grid_mask3_offset_words(const nacc_grid &g) { return grid_mask2_offset_words(g) + mask2_words(g); }

static int64_t mask3_words(const nacc_grid &g) {  // one mask, every level (level-major, R^3 bits each)
  return ceil_div(ceil_div((int64_t)g.levels * g.res * g.res * g.res, 32), 64) * 64;
}

static int64_t grid_aux_words(const nacc_grid &g) {
  if (!grid_skip_enabled(g)) return kAuxHeaderWords;
  const int64_t w = kAuxHeaderWords + mask2_words(g);
  if (!grid_fine_mask_enabled(g)) return w;
  return w + 2 * (grid_fine_win(g) - 1) * mask3_words(g);  // OR and AND window masks per window size 2..W
}

__global__ void bbox_init_kernel(int32_t *__restrict__ hdr, int levels, int R) {
  const int i = threadIdx.x;
  if (i < 6 * levels) hdr[i] = (i % 6) < 3 ? R : -1;
}

// thread per fine word: index box of its set bits, reduced per level
__global__ void __launch_bounds__(256) bbox_kernel(const uint32_t *__restrict__ bits, int levels, int R,
                                                   int32_t *__restrict__ hdr) {
  const int64_t R3 = (int64_t)R * R * R, cells = (int64_t)levels * R3;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t w = q < (cells + 31) / 32 ? bits[q] : 0u;
  int lo[3] = {R, R, R}, hi[3] = {-1, -1, -1}, lv = -1;
  while (w) {
    const int b = __ffs(w) - 1;
    w &= w - 1u;
    const int64_t cell = q * 32 + b;
    if (cell >= cells) break;
    const int l = (int)(cell / R3);
    const int64_t idx = cell - (int64_t)l * R3;
    const int c[3] = {(int)(idx % R), (int)((idx / R) % R), (int)(idx / ((int64_t)R * R))};
    if (l != lv && lv >= 0) {  // the word straddles levels: flush the previous level
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        atomicMin(hdr + 6 * lv + a, lo[a]);
        atomicMax(hdr + 6 * lv + 3 + a, hi[a]);
        lo[a] = R;
        hi[a] = -1;
      }
    }
    lv = l;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = min(lo[a], c[a]);
      hi[a] = max(hi[a], c[a]);
    }
  }
  // warp pre-reduction when every lane holding bits is on one level
  const unsigned has = __ballot_sync(kFull, lv >= 0);
  if (!has) return;
  const int l0 = __shfl_sync(kFull, lv, __ffs(has) - 1);
  if (__all_sync(kFull, lv < 0 || lv == l0)) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo[a] = min(lo[a], __shfl_xor_sync(kFull, lo[a], o));
        hi[a] = max(hi[a], __shfl_xor_sync(kFull, hi[a], o));
      }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        atomicMin(hdr + 6 * l0 + a, lo[a]);
        atomicMax(hdr + 6 * l0 + 3 + a, hi[a]);
      }
  } else if (lv >= 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(hdr + 6 * lv + a, lo[a]);
      atomicMax(hdr + 6 * lv + 3 + a, hi[a]);
    }
  }
}

// world box of all occupied cells: level l's box is lo_l + [i0, i1 + 1] * (hi_l - lo_l) / R,
// widened by 1e-4 of the outermost width + 1e-6 (far above the fp32 error of P(k)'s positions)
struct LevelBox {
  double lo[8][3], hi[8][3];
};
__global__ void bbox_world_kernel(int32_t *__restrict__ hdr, LevelBox b, int levels, int R) {
  if (threadIdx.x != 0) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int l = 0; l < levels; ++l) {
    const int32_t *h = hdr + 6 * l;
    if (h[3] < 0) continue;  // level without occupied cells
    for (int a = 0; a < 3; ++a) {
      const double cw = (b.hi[l][a] - b.lo[l][a]) / R;
      lo[a] = fmin(lo[a], b.lo[l][a] + h[a] * cw);
      hi[a] = fmax(hi[a], b.lo[l][a] + (h[3 + a] + 1) * cw);
    }
  }
  float *wb = reinterpret_cast<float *>(hdr + kAuxBoxWord);
  for (int a = 0; a < 3; ++a) {
    const double pad = 1e-4 * (b.hi[levels - 1][a] - b.lo[levels - 1][a]) + 1e-6;
    wb[a] = lo[a] <= hi[a] ? (float)(lo[a] - pad) : INFINITY;
    wb[3 + a] = lo[a] <= hi[a] ? (float)(hi[a] + pad) : -INFINITY;
  }
}

__global__ void mask2_kernel(uint32_t *__restrict__ bits, int levels, int R, int64_t aux_off) {
  const int M = R / kMacroCells;
  const int64_t M3 = (int64_t)M * M * M, n = (int64_t)levels * M3;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool on = false;
  if (q < n) {
    const int l = (int)(q / M3);
    const int64_t m = q - l * M3;
    const int mx = (int)(m % M), my = (int)((m / M) % M), mz = (int)(m / ((int64_t)M * M));
    const int x0 = mx * kMacroCells, nx = min(2 * kMacroCells, R - x0);
    const uint32_t xmask = (nx >= 32) ? 0xffffffffu : ((1u << nx) - 1u);
    for (int z = mz * kMacroCells; z < min(mz * kMacroCells + 2 * kMacroCells, R) && !on; ++z)
      for (int y = my * kMacroCells; y < min(my * kMacroCells + 2 * kMacroCells, R) && !on; ++y) {
        const int64_t s = (int64_t)l * R * R * R + x0 + (int64_t)R * (y + (int64_t)R * z);
        const int off = (int)(s & 31);
        uint32_t v = bits[s >> 5] >> off;
        if (off + nx > 32) v |= bits[(s >> 5) + 1] << (32 - off);
        on = (v & xmask) != 0u;
      }
  }
  const unsigned b = __ballot_sync(kFull, on);
  if ((threadIdx.x & 31) == 0 && q < n) bits[aux_off + (q >> 5)] = b;
}

// thread per fine cell (one level): the OR (kAnd = false) or the AND (kAnd = true) of the
// bits of cells c + {0..W-1}^3; cells outside the grid count as empty (an AND window that
// leaves the grid is 0)
template <bool kAnd, int kW>
__global__ void __launch_bounds__(256) mask3_kernel(uint32_t *__restrict__ bits, int levels, int R, int64_t off) {
  const int64_t R3 = (int64_t)R * R * R, n = levels * R3;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool on = false;
  if (q < n) {
    const int64_t lbase = (q / R3) * R3, ql = q - lbase;  // the cell's level: windows stay inside it
    const int x = (int)(ql % R), y = (int)((ql / R) % R), z = (int)(ql / ((int64_t)R * R));
    const int nx = min(kW, R - x);
    const uint32_t xmask = (1u << nx) - 1u;
    if (kAnd) {
      on = x + kW <= R && y + kW <= R && z + kW <= R;
      for (int zz = z; zz < z + kW && on; ++zz)
        for (int yy = y; yy < y + kW && on; ++yy) {
          const int64_t s = lbase + x + (int64_t)R * (yy + (int64_t)R * zz);
          const int o = (int)(s & 31);
          uint32_t v = __ldg(bits + (s >> 5)) >> o;
          if (o + kW > 32) v |= __ldg(bits + (s >> 5) + 1) << (32 - o);
          on = (v & xmask) == xmask;
        }
    } else {
      for (int zz = z; zz < min(z + kW, R) && !on; ++zz)
        for (int yy = y; yy < min(y + kW, R) && !on; ++yy) {
          const int64_t s = lbase + x + (int64_t)R * (yy + (int64_t)R * zz);
          const int o = (int)(s & 31);
          uint32_t v = __ldg(bits + (s >> 5)) >> o;
          if (o + nx > 32) v |= __ldg(bits + (s >> 5) + 1) << (32 - o);
          on = (v & xmask) != 0u;
        }
    }
  }
  const unsigned b = __ballot_sync(kFull, on);
  if ((threadIdx.x & 31) == 0 && q < n) bits[off + (q >> 5)] = b;
}

// Row-wise variant (R % 32 == 0): thread per output word, i.e. 32 cells of one x-row; the
// x-window is W shifted copies of the row's word and its successor, then OR (AND) over the
// W x W rows of the window.  Same bits as mask3_kernel, 32x fewer loads.
template <bool kAnd, int kW>
__global__ void __launch_bounds__(256) mask3_rows_kernel(uint32_t *__restrict__ bits, int levels, int R, int64_t off) {
  const int64_t R3 = (int64_t)R * R * R, nw = levels * R3 / 32;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nw) return;
  const int64_t lbase = (q * 32 / R3) * R3, c0 = q * 32 - lbase;
  const int x0 = (int)(c0 % R), y = (int)((c0 / R) % R), z = (int)(c0 / ((int64_t)R * R));
  const bool last_word = x0 + 32 >= R;
  uint32_t acc = kAnd ? 0xffffffffu : 0u;
  if (kAnd && (y + kW > R || z + kW > R)) acc = 0u;
  for (int zz = z; zz < min(z + kW, R) && (!kAnd || acc); ++zz)
    for (int yy = y; yy < min(y + kW, R); ++yy) {
      const int64_t wi = (lbase + x0 + (int64_t)R * (yy + (int64_t)R * zz)) >> 5;
      const uint32_t w = __ldg(bits + wi), wn = last_word ? 0u : __ldg(bits + wi + 1);
      uint32_t d = w;
#pragma unroll
      for (int k = 1; k < kW; ++k) {
        const uint32_t sh = (w >> k) | (wn << (32 - k));
        d = kAnd ? (d & sh) : (d | sh);
      }
      acc = kAnd ? (acc & d) : (acc | d);
    }
  bits[off + q] = acc;
}

cudaError_t grid_prepare(const nacc_grid &g, uint32_t *bits, cudaStream_t stream) {
  int32_t *hdr = reinterpret_cast<int32_t *>(bits + grid_aux_offset_words(g));
  const int64_t cells = (int64_t)g.levels * g.res * g.res * g.res;
  LevelBox lb;
  for (int a = 0; a < 3; ++a) {
    const double lo0 = (double)g.roi[a], hi0 = (double)g.roi[3 + a];
    const double ctr = (lo0 + hi0) / 2.0, half = (hi0 - lo0) / 2.0;
    for (int l = 0; l < g.levels; ++l) {  // the march's fp32 level boxes
      lb.lo[l][a] = (double)(float)(ctr - half * std::ldexp(1.0, l));
      lb.hi[l][a] = (double)(float)(ctr + half * std::ldexp(1.0, l));
    }
  }
  bbox_init_kernel<<<1, 64, 0, stream>>>(hdr, g.levels, g.res);
  bbox_kernel<<<grid_for(ceil_div(cells, 32), 256), 256, 0, stream>>>(bits, g.levels, g.res, hdr);
  bbox_world_kernel<<<1, 32, 0, stream>>>(hdr, lb, g.levels, g.res);
  count_launch(3);
  if (grid_skip_enabled(g)) {
    const int M = g.res / kMacroCells;
    const int64_t n = (int64_t)g.levels * M * M * M;
    mask2_kernel<<<grid_for(n, 256), 256, 0, stream>>>(bits, g.levels, g.res, grid_mask2_offset_words(g));
    count_launch(1);
  }
  if (grid_fine_mask_enabled(g)) {
    const int64_t n = (int64_t)g.levels * g.res * g.res * g.res;
    const int64_t o3 = grid_mask3_offset_words(g), mw = mask3_words(g);
    auto masks = [&](auto wtag) {
      constexpr int W = decltype(wtag)::value;
      const int64_t o_or = o3 + 2 * (W - 2) * mw, o_and = o_or + mw;
      if (g.res % 32 == 0) {
        mask3_rows_kernel<false, W><<<grid_for(n / 32, 256), 256, 0, stream>>>(bits, g.levels, g.res, o_or);
        mask3_rows_kernel<true, W><<<grid_for(n / 32, 256), 256, 0, stream>>>(bits, g.levels, g.res, o_and);
      } else {
        mask3_kernel<false, W><<<grid_for(n, 256), 256, 0, stream>>>(bits, g.levels, g.res, o_or);
        mask3_kernel<true, W><<<grid_for(n, 256), 256, 0, stream>>>(bits, g.levels, g.res, o_and);
      }
      count_launch(2);
    };
    static_assert(kFineWin >= 2 && kFineWin <= 9, "window sizes 2..9");
    masks(std::integral_constant<int, 2>{});
    const int W = grid_fine_win(g);
    if (W >= 3) masks(std::integral_constant<int, 3 <= kFineWin ? 3 : 2>{});
    if (W >= 4) masks(std::integral_constant<int, 4 <= kFineWin ? 4 : 2>{});
    if (W >= 5) masks(std::integral_constant<int, 5 <= kFineWin ? 5 : 2>{});
    if (W >= 6) masks(std::integral_constant<int, 6 <= kFineWin ? 6 : 2>{});
    if (W >= 7) masks(std::integral_constant<int, 7 <= kFineWin ? 7 : 2>{});
    if (W >= 8) masks(std::integral_constant<int, 8 <= kFineWin ? 8 : 2>{});
    if (W >= 9) masks(std::integral_constant<int, 9 <= kFineWin ? 9 : 2>{});
  }
  return cudaGetLastError();
}

}  // namespace nacc

using namespace nacc;

extern "C" {

size_t nacc_grid_bits_bytes(const nacc_grid *grid) {
  if (!grid || grid->levels < 1 || grid->levels > 8 || grid->res < 1) return 0;
  const int64_t cells = (int64_t)grid->levels * grid->res * grid->res * grid->res;
  if (cells >= (1ll << 31)) return 0;
  return (size_t)(grid_aux_offset_words(*grid) + grid_aux_words(*grid)) * 4;
}

nacc_status nacc_grid_prepare(const nacc_grid *grid, uint32_t *bits, cudaStream_t stream) {
  clear_error();
  NACC_REQUIRE(nacc_grid_bits_bytes(grid) > 0, "invalid grid");
  NACC_REQUIRE(bits && aligned(bits, 4), "bits must be non-NULL and 4-byte aligned");
  NACC_CUDA(grid_prepare(*grid, bits, stream));
  return NACC_OK;
}

}  // extern "C"
