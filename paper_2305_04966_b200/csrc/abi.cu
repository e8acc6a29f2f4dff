// abi.cu — error state, version, launch counter, exclusive scan used by the
// packing steps ("packed tensor": start = exclusive prefix sum of counts).

#include "common.cuh"

namespace nacc {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

// ---------------------------------------------------------------- block scan (1024 threads)
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// exclusive block-wide scan of one int64 per thread; returns the exclusive
// prefix and writes the block total to *block_total
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *smem, int64_t *block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  int64_t incl = warp_incl_scan_i64(v);
  if (lane == 31) smem[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t s = lane < nwarps ? smem[lane] : 0;
    int64_t si = warp_incl_scan_i64(s);
    if (lane < nwarps) smem[lane] = si - s;
    if (lane == 31) smem[32] = si;
  }
  __syncthreads();
  int64_t r = smem[warp] + incl - v;
  *block_total = smem[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) tile_sums_kernel(const int32_t *__restrict__ counts,
                                                                 int64_t n, int64_t *__restrict__ sums) {
  __shared__ int64_t smem[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) v += counts[base + i];
  int64_t tot;
  block_excl_scan(v, smem, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// single block: exclusive scan of the tile sums in place, total to *total
__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(int64_t *__restrict__ sums,
                                                                 int64_t nb, int64_t *__restrict__ total) {
  __shared__ int64_t smem[33];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? sums[i] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan(v, smem, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) tile_apply_kernel(const int32_t *__restrict__ counts,
                                                                  int64_t n, const int64_t *__restrict__ offsets,
                                                                  int64_t *__restrict__ packed_info,
                                                                  int64_t *__restrict__ total) {
  __shared__ int64_t smem[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t c[kScanItems];
  int64_t v = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    c[i] = base + i < n ? counts[base + i] : 0;
    v += c[i];
  }
  int64_t tot;
  int64_t ex = block_excl_scan(v, smem, &tot);
  int64_t run = (offsets ? offsets[blockIdx.x] : 0) + ex;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) {
      reinterpret_cast<longlong2 *>(packed_info)[base + i] = make_longlong2(run, c[i]);
      run += c[i];
    }
  }
  if (!offsets && total && threadIdx.x == 0) *total = tot;
}

size_t scan_workspace_bytes(int64_t n) { return align_up((size_t)ceil_div(n, kScanTile) * 8, 256); }

cudaError_t scan_counts_to_packed(const int32_t *counts, int64_t n, int64_t *packed_info,
                                  int64_t *total, void *ws, cudaStream_t stream) {
  const int64_t nb = ceil_div(n, kScanTile);
  if (nb <= 1) {
    tile_apply_kernel<<<1, kScanThreads, 0, stream>>>(counts, n, nullptr, packed_info, total);
    count_launch(1);
    return cudaGetLastError();
  }
  int64_t *sums = static_cast<int64_t *>(ws);
  tile_sums_kernel<<<(unsigned)nb, kScanThreads, 0, stream>>>(counts, n, sums);
  scan_sums_kernel<<<1, kScanThreads, 0, stream>>>(sums, nb, total);
  tile_apply_kernel<<<(unsigned)nb, kScanThreads, 0, stream>>>(counts, n, sums, packed_info, nullptr);
  count_launch(3);
  return cudaGetLastError();
}

}  // namespace nacc

extern "C" {

const char *nacc_last_error(void) { return nacc::g_last_error.c_str(); }
int nacc_abi_version(void) { return NACC_ABI_VERSION; }
uint64_t nacc_launch_count(void) { return nacc::g_launches.load(std::memory_order_relaxed); }

size_t nacc_grid_bits_bytes(const nacc_grid *grid) {
  if (!grid || grid->levels < 1 || grid->levels > 8 || grid->res < 1) return 0;
  const int64_t cells = (int64_t)grid->levels * grid->res * grid->res * grid->res;
  if (cells >= (1ll << 31)) return 0;
  return (size_t)nacc::ceil_div(cells, 32) * 4;
}

}  // extern "C"
