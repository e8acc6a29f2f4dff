// gridaux.cu — the occupancy bitfield's auxiliary skip mask.
//
// After the public fine bits (cell q -> bit q & 31 of word q >> 5, nacc.h) the
// bitfield buffer holds a library-private mask used by the march to skip empty
// space: for every macro cell m (4^3 fine cells) of every level,
// mask2[m] = OR of the fine bits of macro cells m + {0,1}^3, i.e. of the fine
// cells [4m, 4m + 8)^3 clipped to the level.  It depends only on the fine bits,
// so it is rebuilt when they change (nacc_occgrid_update, nacc_grid_prepare),
// not on every march.
#include "common.cuh"

namespace nacc {

bool grid_skip_enabled(const nacc_grid &g) { return g.res % kMacroCells == 0 && g.res >= 2 * kMacroCells; }

int64_t grid_aux_offset_words(const nacc_grid &g) {
  const int64_t cells = (int64_t)g.levels * g.res * g.res * g.res;
  return ceil_div(ceil_div(cells, 32), 64) * 64;  // 256-byte aligned
}

static int64_t grid_aux_words(const nacc_grid &g) {
  if (!grid_skip_enabled(g)) return 0;
  const int64_t M = g.res / kMacroCells;
  return ceil_div((int64_t)g.levels * M * M * M, 32);
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

cudaError_t grid_prepare(const nacc_grid &g, uint32_t *bits, cudaStream_t stream) {
  if (!grid_skip_enabled(g)) return cudaSuccess;
  const int M = g.res / kMacroCells;
  const int64_t n = (int64_t)g.levels * M * M * M;
  mask2_kernel<<<grid_for(n, 256), 256, 0, stream>>>(bits, g.levels, g.res, grid_aux_offset_words(g));
  count_launch(1);
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
