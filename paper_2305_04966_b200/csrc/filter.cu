// filter.cu — §4.2 "No Gradient Filtering": samples whose entering
// transmittance is below ε are dropped before the differentiable pass.
// Per ray the kept set is a prefix (S_i never decreases; reading #9), so the
// filter is a per-ray cut (sequential fp64 sum, early exit) + exclusive scan of
// the cuts + a compacting copy (two kernels after a memset, no host sync).
#include "common.cuh"
#include "debug.cuh"

namespace nacc {

// Pass 1: one thread per ray walks its samples in order, accumulating
// S_i = Σ_{j<i} σ_j δ_j in fp64 exactly as the definition (σ_j δ_j is exact in
// fp64, so this is the sequential sum), stopping at the first S_i > L; only the
// kept prefix plus a few samples are read.  Each block also reduces its cuts.
#ifndef NACC_FILTER_RAYS
#define NACC_FILTER_RAYS 256  // build parameter: rays per copy block / group sum
#endif
constexpr int kFiltRays = NACC_FILTER_RAYS;


// Small blocks (two warps) and per-warp atomic adds into the 256-ray group
// sums: rays of very different lengths no longer hold a 256-thread block (and
// its resources) at a barrier until the longest one is done.
constexpr int kCutThreads = 64;
// Samples read per step of a ray's walk: 4 at first, doubling up to kCutBatch
// (build parameter; 4 = fixed quads measured fastest on CFG2: 74.6 us vs 76.0 for
// 8 and 78.3 for 16 -- the overread costs more than the saved round trips).
#ifndef NACC_FILTER_BATCH
#define NACC_FILTER_BATCH 4
#endif
constexpr int kCutBatch = NACC_FILTER_BATCH;
#ifndef NACC_FILTER_MINB
#define NACC_FILTER_MINB 1  // build parameter: min resident 64-thread blocks per SM of the sector walk
                            // (A/B 1 / 16 / 24 / 32: 67.2 / 65.9 / 115 / 144 us, within noise up to 16)
#endif
#ifndef NACC_FILTER_SECTOR
#define NACC_FILTER_SECTOR 1  // build parameter: sector-aligned walk when the arrays are 32-byte aligned
#endif

// a warp's cut total into its 256-ray group sum and into the sum of the group's 32-group super
// group (block_sums + nb), from which the copy kernel forms every group's offset directly
__device__ __forceinline__ void add_group_sum(int64_t *block_sums, int64_t nb, int64_t g, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long *>(block_sums + g), (unsigned long long)v);
  atomicAdd(reinterpret_cast<unsigned long long *>(block_sums + nb + (g >> 5)), (unsigned long long)v);
}

__global__ void __launch_bounds__(kCutThreads) filter_cut_kernel(const int64_t *__restrict__ packed_info, int64_t n_rays,
                                                                 const float *__restrict__ t0,
                                                                 const float *__restrict__ t1,
                                                                 const float *__restrict__ sigma, int64_t n_samples,
                                                                 double L, int32_t *__restrict__ cut_out,
                                                                 int64_t *__restrict__ block_sums, int64_t nb) {
  const int64_t r = (int64_t)blockIdx.x * kCutThreads + threadIdx.x;
  int64_t cut = 0;
  if (r < n_rays) {
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2 *>(packed_info) + r);
    // a packed_info written past the input's capacity (device-count mode after an overflowed
    // march) is clamped to the n_samples readable samples; the result is invalid but in bounds
    const int64_t st = min((int64_t)pi.x, n_samples), cnt = min((int64_t)(pi.x + pi.y), n_samples) - st;
    double S = 0.0;
    cut = cnt;
    int nb = 4;
    for (int64_t i = 0; i < cnt; i += nb, nb = min(2 * nb, kCutBatch)) {
      float a[kCutBatch], b[kCutBatch], c[kCutBatch];
#pragma unroll
      for (int j = 0; j < kCutBatch; ++j) {
        const bool in = j < nb && i + j < cnt;
        a[j] = in ? __ldg(t0 + st + i + j) : 0.f;
        b[j] = in ? __ldg(t1 + st + i + j) : 0.f;
        c[j] = in ? __ldg(sigma + st + i + j) : 0.f;
      }
      bool done = false;
#pragma unroll
      for (int j = 0; j < kCutBatch; ++j) {
        if (!done && j < nb && i + j < cnt) {
          if (S > L) {
            cut = i + j;
            done = true;
          } else {
            S = __dadd_rn(S, __dmul_rn((double)c[j], __dsub_rn((double)b[j], (double)a[j])));
          }
        }
      }
      if (done) break;
    }
    cut_out[r] = (int32_t)cut;
  }
  const int64_t tot = warp_sum_i64(cut);
  const int64_t r_warp = r - (threadIdx.x & 31);
  if ((threadIdx.x & 31) == 0 && tot)
    add_group_sum(block_sums, nb, r_warp / kFiltRays, tot);
}

// Pass 1, sector-aligned variant: the walk reads whole 32-byte sectors (8 floats, two
// float4 loads per array) starting at the sector that holds the ray's first sample, so
// every DRAM sector fetched is used in full (the unaligned quads above straddle two).
// Software-pipelined: the next sector's loads are issued before the current one is
// summed, so a long ray's walk costs one DRAM latency plus its arithmetic, not one
// latency per sector (the kernel's time was the longest rays' dependent walks).
// Needs 32-byte-aligned t0 / t1 / sigma; reads stay inside the arrays.
struct Sector {
  float a[8], b[8], c[8];
};

__device__ __forceinline__ void load_sector(Sector &v, const float *__restrict__ t0, const float *__restrict__ t1,
                                            const float *__restrict__ sigma, int64_t q, int64_t n_samples) {
  if (q + 8 <= n_samples) {  // whole sector inside the arrays
    const float4 *pa = reinterpret_cast<const float4 *>(t0 + q), *pb = reinterpret_cast<const float4 *>(t1 + q),
                 *pc = reinterpret_cast<const float4 *>(sigma + q);
    const float4 a0 = __ldg(pa), a1 = __ldg(pa + 1), b0 = __ldg(pb), b1 = __ldg(pb + 1), c0 = __ldg(pc),
                 c1 = __ldg(pc + 1);
    v.a[0] = a0.x; v.a[1] = a0.y; v.a[2] = a0.z; v.a[3] = a0.w; v.a[4] = a1.x; v.a[5] = a1.y; v.a[6] = a1.z; v.a[7] = a1.w;
    v.b[0] = b0.x; v.b[1] = b0.y; v.b[2] = b0.z; v.b[3] = b0.w; v.b[4] = b1.x; v.b[5] = b1.y; v.b[6] = b1.z; v.b[7] = b1.w;
    v.c[0] = c0.x; v.c[1] = c0.y; v.c[2] = c0.z; v.c[3] = c0.w; v.c[4] = c1.x; v.c[5] = c1.y; v.c[6] = c1.z; v.c[7] = c1.w;
  } else {  // the arrays' last, partial sector: element loads (no padding is required)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool in = q + j < n_samples;
      v.a[j] = in ? __ldg(t0 + q + j) : 0.f;
      v.b[j] = in ? __ldg(t1 + q + j) : 0.f;
      v.c[j] = in ? __ldg(sigma + q + j) : 0.f;
    }
  }
}

__global__ void __launch_bounds__(kCutThreads, NACC_FILTER_MINB) filter_cut_sector_kernel(
    const int64_t *__restrict__ packed_info, int64_t n_rays, const float *__restrict__ t0,
    const float *__restrict__ t1, const float *__restrict__ sigma, int64_t n_samples, double L,
    int32_t *__restrict__ cut_out, int64_t *__restrict__ block_sums, int64_t nb) {
  const int64_t r = (int64_t)blockIdx.x * kCutThreads + threadIdx.x;
  int64_t cut = 0;
  if (r < n_rays) {
    const longlong2 pi = __ldg(reinterpret_cast<const longlong2 *>(packed_info) + r);
    // a packed_info written past the input's capacity (device-count mode after an overflowed
    // march) is clamped to the n_samples readable samples; the result is invalid but in bounds
    const int64_t st = min((int64_t)pi.x, n_samples), e = min((int64_t)(pi.x + pi.y), n_samples);
    double S = 0.0;
    cut = e - st;
    int64_t q = st & ~(int64_t)7;
    Sector cur, nxt;
    if (q < e) load_sector(cur, t0, t1, sigma, q, n_samples);
    while (q < e) {
      const int64_t qn = q + 8;
      if (qn < e) load_sector(nxt, t0, t1, sigma, qn, n_samples);  // in flight while `cur` is summed
      bool done = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!done && q + j >= st && q + j < e) {
          if (S > L) {
            cut = q + j - st;
            done = true;
          } else {
            S = __dadd_rn(S, __dmul_rn((double)cur.c[j], __dsub_rn((double)cur.b[j], (double)cur.a[j])));
          }
        }
      }
      if (done) break;
      cur = nxt;
      q = qn;
    }
    cut_out[r] = (int32_t)cut;
  }
  const int64_t tot = warp_sum_i64(cut);
  const int64_t r_warp = r - (threadIdx.x & 31);
  if ((threadIdx.x & 31) == 0 && tot)
    add_group_sum(block_sums, nb, r_warp / kFiltRays, tot);
}

// Pass 2: blocks of 256 consecutive rays scan their cuts (+ the group's offset, from the group and
// super-group sums of pass 1; block 0 writes the total)
// into packed_info', then copy the kept prefixes, which are contiguous in the
// output; each thread locates its ray by binary search over the block's output
// starts in shared memory, so stores are coalesced.
__global__ void __launch_bounds__(kFiltRays) filter_copy_kernel(
    const int64_t *__restrict__ packed_info, int64_t n_rays, const float *__restrict__ t0,
    const float *__restrict__ t1, const int32_t *__restrict__ cuts, const int64_t *__restrict__ block_off,
    int64_t nb, int64_t *__restrict__ total, int64_t capacity, int64_t *__restrict__ packed_out,
    float *__restrict__ t0_out, float *__restrict__ t1_out, int32_t *__restrict__ ray_id_out, int vec) {
  __shared__ int64_t s_out[kFiltRays + 1];
  __shared__ int64_t s_in[kFiltRays];
  __shared__ int64_t s_w[kFiltRays / 32];
  const int64_t r0 = (int64_t)blockIdx.x * kFiltRays;
  const int nr = (int)min((int64_t)kFiltRays, n_rays - r0);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __shared__ int64_t s_pre[2];  // this group's output offset, the grand total
  if (warp == 0) {
    // offset = the super groups before this one + the groups before this one in its super group
    const int64_t b = blockIdx.x, sb = b >> 5, nsb = (nb + 31) >> 5;
    int64_t pre = 0, tot = 0;
    for (int64_t k = lane; k < nsb; k += 32) {
      const int64_t v = block_off[nb + k];
      tot += v;
      if (k < sb) pre += v;
    }
    const int64_t gq = (sb << 5) + lane;
    if (gq < b) pre += block_off[gq];
    pre = warp_sum_i64(pre);
    tot = warp_sum_i64(tot);
    if (lane == 0) {
      s_pre[0] = pre;
      s_pre[1] = tot;
      if (b == 0) *total = tot;
    }
  }
  const int64_t c = t < nr ? (int64_t)cuts[r0 + t] : 0;
  const int64_t incl = warp_incl_scan_i64(c);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int64_t wbase = s_pre[0];
  for (int w = 0; w < warp; ++w) wbase += s_w[w];
  const int64_t out = wbase + incl - c;
  if (t < nr) {
    reinterpret_cast<longlong2 *>(packed_out)[r0 + t] = make_longlong2(out, c);
    s_out[t] = out;
    s_in[t] = __ldg(packed_info + 2 * (r0 + t));  // cut <= the clamped count: sources stay < n_samples
    if (t == nr - 1) s_out[nr] = out + c;
  }
  __syncthreads();
  if (t0_out == nullptr || s_pre[1] > capacity) return;
  const int64_t p0 = s_out[0], p1 = s_out[nr];
  // four consecutive outputs per thread: one binary search, then a forward walk; the
  // stores of a full aligned quad are float4 / int4
  for (int64_t p4 = (p0 & ~(int64_t)3) + 4 * (int64_t)t; p4 < p1; p4 += 4 * kFiltRays) {
    const int64_t pa = p4 > p0 ? p4 : p0;
    int lo = 0, hi = nr - 1;  // largest k with s_out[k] <= pa
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_out[mid] <= pa) lo = mid;
      else hi = mid - 1;
    }
    float a[4], b[4];
    int32_t id[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t p = p4 + j;
      a[j] = b[j] = 0.f;
      id[j] = 0;
      if (p >= p0 && p < p1) {
        while (lo + 1 < nr && s_out[lo + 1] <= p) ++lo;
        const int64_t src = s_in[lo] + (p - s_out[lo]);
        a[j] = __ldg(t0 + src);
        b[j] = __ldg(t1 + src);
        id[j] = (int32_t)(r0 + lo);
      }
    }
    if (vec && p4 >= p0 && p4 + 3 < p1) {
      *reinterpret_cast<float4 *>(t0_out + p4) = make_float4(a[0], a[1], a[2], a[3]);
      *reinterpret_cast<float4 *>(t1_out + p4) = make_float4(b[0], b[1], b[2], b[3]);
      *reinterpret_cast<int4 *>(ray_id_out + p4) = make_int4(id[0], id[1], id[2], id[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t p = p4 + j;
        if (p >= p0 && p < p1) {
          t0_out[p] = a[j];
          t1_out[p] = b[j];
          ray_id_out[p] = id[j];
        }
      }
    }
  }
}

static size_t filter_ws_layout(int64_t n, int32_t **cuts, int64_t **bsums, void *base) {
  const size_t a = align_up((size_t)n * 4, 256);
  if (base) {
    *cuts = static_cast<int32_t *>(base);
    *bsums = reinterpret_cast<int64_t *>(static_cast<char *>(base) + a);
  }
  const int64_t nb = ceil_div(n, kFiltRays);
  return a + align_up(8 * (size_t)(nb + ceil_div(nb, 32)), 256);  // group sums, then super-group sums
}

}  // namespace nacc

using namespace nacc;

extern "C" {

size_t nacc_filter_workspace_bytes(int64_t n_rays) {
  if (n_rays < 0) return 0;
  return filter_ws_layout(n_rays, nullptr, nullptr, nullptr);
}

nacc_status nacc_filter_early_stop(const int64_t *packed_info, int64_t n_rays, const float *t0, const float *t1,
                                   const float *sigma, int64_t n_samples, double neg_log_eps,
                                   int64_t *packed_info_out, float *t0_out, float *t1_out, int32_t *ray_id_out,
                                   int64_t capacity, int64_t *total, void *ws, size_t ws_bytes,
                                   cudaStream_t stream) {
  clear_error();
  NACC_REQUIRE(n_rays >= 0 && n_rays < (1ll << 31), "n_rays must be in [0, 2^31)");
  NACC_REQUIRE(n_samples >= 0 && capacity >= 0, "n_samples and capacity must be >= 0");
  NACC_REQUIRE(!std::isnan(neg_log_eps), "neg_log_eps must not be NaN");
  NACC_REQUIRE(total, "total must be non-NULL");
  if (n_rays == 0) {
    NACC_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), stream));
    return NACC_OK;
  }
  NACC_REQUIRE(packed_info && packed_info_out && aligned(packed_info, 16) && aligned(packed_info_out, 16),
               "packed_info / packed_info_out must be non-NULL and 16-byte aligned");
  NACC_REQUIRE(n_samples == 0 || (t0 && t1 && sigma), "t0, t1, sigma must be non-NULL");
  NACC_REQUIRE(capacity == 0 || (t0_out && t1_out && ray_id_out), "outputs must be non-NULL when capacity > 0");
  NACC_REQUIRE(ws && ws_bytes >= nacc_filter_workspace_bytes(n_rays), "workspace too small");
  NACC_DEBUG_CHECK(debug_check_packed(packed_info, n_rays, t0, t1, n_samples, stream));
  NACC_DEBUG_CHECK(debug_check_sigma(sigma, n_samples, "sigma must be >= 0 and finite", stream));
  int32_t *cuts;
  int64_t *bsums;
  filter_ws_layout(n_rays, &cuts, &bsums, ws);
  const int64_t nb = ceil_div(n_rays, kFiltRays);
  NACC_CUDA(cudaMemsetAsync(bsums, 0, 8 * (size_t)(nb + ceil_div(nb, 32)), stream));
  if (NACC_FILTER_SECTOR && aligned(t0, 32) && aligned(t1, 32) && aligned(sigma, 32))
    filter_cut_sector_kernel<<<(unsigned)ceil_div(n_rays, kCutThreads), kCutThreads, 0, stream>>>(
        packed_info, n_rays, t0, t1, sigma, n_samples, neg_log_eps, cuts, bsums, nb);
  else
    filter_cut_kernel<<<(unsigned)ceil_div(n_rays, kCutThreads), kCutThreads, 0, stream>>>(
        packed_info, n_rays, t0, t1, sigma, n_samples, neg_log_eps, cuts, bsums, nb);
  filter_copy_kernel<<<(unsigned)nb, kFiltRays, 0, stream>>>(packed_info, n_rays, t0, t1, cuts, bsums, nb, total, capacity,
                                                             packed_info_out, capacity > 0 ? t0_out : nullptr, t1_out,
                                                             ray_id_out,
                                                             aligned(t0_out, 16) && aligned(t1_out, 16) &&
                                                                 aligned(ray_id_out, 16));
  count_launch(2);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

}  // extern "C"
