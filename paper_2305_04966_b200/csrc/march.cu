// march.cu — occupancy-grid ray marching into packed intervals (Alg. 1
// nerfacc.sampling; spatial skipping; sample as interval
// and packed tensor).  DESIGN.md §6 describes the kernel design.
//
// Membership of lattice interval k (readings #1-#3; normative fp32 ops):
//   m_k = fmaf(k + 0.5, Δt, near_r)            (uniform lattice), or
//   t_{k+1} = t_k + min(max(t_k c, Δt), Δt_max), m_k = t_k + 0.5 dt_k  (cone)
//   x_a  = fmaf(m_k, d_a, o_a)
//   l*   = first level l with lo_l <= x < hi_l on every axis
//   u_a  = (x_a - lo_{l*,a}) * s_{l*,a},  i_a = clamp(floor(u_a), 0, R-1)
//   P(k) = m_k < far_r  and  l* exists  and  bit[l*][i]
// The k range each warp scans is a conservative fp32 slab bound (±2 steps
// around the padded outermost box); membership alone decides emission.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "debug.cuh"
#include "lookback.cuh"

#ifndef NACC_MARCH_MAGICFLOOR
#define NACC_MARCH_MAGICFLOOR 0  // build parameter: floor by FADD.RZ instead of F2I for interior points
#endif
#ifndef NACC_MARCH_FINEMASK
#define NACC_MARCH_FINEMASK 1  // build parameter: segment test on the fine window masks (0: macro test only)
#endif
#ifndef NACC_MARCH_SHAREDENDS
#define NACC_MARCH_SHAREDENDS 1  // build parameter: segment ends from the next lane's start (fine mask)
#endif
#ifndef NACC_MARCH_SOLID
#define NACC_MARCH_SOLID 1  // build parameter: segments in an all-occupied 3^3 window skip P(k)
#endif
#ifndef NACC_MARCH_MINB
#define NACC_MARCH_MINB 6  // build parameter: min resident blocks per SM in the fused march's launch bounds (A/B 7 -> 6: CFG2 168 -> 166 us, CFG3 2.99 -> 2.75 ms)
#endif
#ifndef NACC_MARCH_PREFETCH
#define NACC_MARCH_PREFETCH 0  // build parameter: L1 prefetch of interior segments' bit words
#endif

namespace nacc {

struct GridConst {
  int levels, res;
  uint32_t r3w, mw;  // bit words per level (R^3 / 32); words per window mask (levels * r3w, 64-word aligned)
  int win;           // largest window mask (cells per axis, grid_fine_win)
  float lo[8][3], hi[8][3], s[8][3];
  float olo[3], ohi[3];  // outermost box padded by 1e-4*width + 1e-6
};

struct MarchConst {
  float near_plane, far_plane, step, max_step, cone, inv_step;
  int stratified;
  uint32_t key0, key1;
};

static GridConst make_grid_const(const nacc_grid &g) {
  GridConst c{};
  c.levels = g.levels;
  c.res = g.res;
  c.r3w = (uint32_t)((int64_t)g.res * g.res * g.res / 32);
  c.mw = (uint32_t)((((int64_t)g.levels * c.r3w + 63) / 64) * 64);
  c.win = grid_fine_win(g);
  for (int a = 0; a < 3; ++a) {
    const double lo0 = (double)g.roi[a], hi0 = (double)g.roi[3 + a];
    const double ctr = (lo0 + hi0) / 2.0, half = (hi0 - lo0) / 2.0;
    for (int l = 0; l < g.levels; ++l) {
      const double sc = std::ldexp(1.0, l);
      c.lo[l][a] = (float)(ctr - half * sc);
      c.hi[l][a] = (float)(ctr + half * sc);
      c.s[l][a] = (float)((double)g.res / ((double)c.hi[l][a] - (double)c.lo[l][a]));
    }
    const int L = g.levels - 1;
    const double w = (double)c.hi[L][a] - (double)c.lo[L][a];
    const double pad = 1e-4 * w + 1e-6;
    c.olo[a] = (float)((double)c.lo[L][a] - pad);
    c.ohi[a] = (float)((double)c.hi[L][a] + pad);
  }
  return c;
}

// -------------------------------------------------------------------------- device
// kL1: single-level grid (the level search reduces to the box-0 test)
__device__ __forceinline__ bool in_level_box(const GridConst &g, int l, float x, float y, float z) {
  return g.lo[l][0] <= x && x < g.hi[l][0] && g.lo[l][1] <= y && y < g.hi[l][1] && g.lo[l][2] <= z && z < g.hi[l][2];
}

// l* = the first level whose half-open box holds x.  The boxes are nested (centre ± half·2^l,
// each bound rounded once to fp32, monotone in l), so membership is monotone in l and a binary
// search over the levels returns exactly the linear search's l*.
template <bool kL1>
__device__ __forceinline__ int level_of(const GridConst &g, float x, float y, float z) {
  if (kL1) return in_level_box(g, 0, x, y, z) ? 0 : -1;
  int lo = 0, hi = g.levels;  // l* in [lo, hi]; hi == levels: in no box
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (in_level_box(g, mid, x, y, z)) hi = mid;
    else lo = mid + 1;
  }
  return lo < g.levels ? lo : -1;
}

// P(k) for the fp32 midpoint m (readings #2, #3): the normative op sequence
template <bool kL1>
__device__ __forceinline__ bool occupied(const GridConst &g, const uint32_t *__restrict__ bits, float m, float ox,
                                         float oy, float oz, float dx, float dy, float dz) {
  const float x = __fmaf_rn(m, dx, ox), y = __fmaf_rn(m, dy, oy), z = __fmaf_rn(m, dz, oz);
  const int l = level_of<kL1>(g, x, y, z);
  if (l < 0) return false;
  const int R = g.res;
  int ix = (int)floorf(__fmul_rn(__fsub_rn(x, g.lo[l][0]), g.s[l][0]));
  int iy = (int)floorf(__fmul_rn(__fsub_rn(y, g.lo[l][1]), g.s[l][1]));
  int iz = (int)floorf(__fmul_rn(__fsub_rn(z, g.lo[l][2]), g.s[l][2]));
  ix = min(max(ix, 0), R - 1);
  iy = min(max(iy, 0), R - 1);
  iz = min(max(iz, 0), R - 1);
  const uint32_t q = (uint32_t)l * (uint32_t)(R * R * R) + (uint32_t)ix +
                     (uint32_t)R * ((uint32_t)iy + (uint32_t)R * (uint32_t)iz);
  return (__ldg(bits + (q >> 5)) >> (q & 31u)) & 1u;
}

// ---------------------------------------------------------------- empty-space skipping
// A segment of kSeg consecutive lattice points whose first and last midpoints
// are A and B is skipped only if no point of it can be emitted: both ends lie
// in the same level l, the segment's box does not reach the finer box l-1, and
// the 2x2x2-macro-cell neighbourhood (macro = 4^3 fine cells) containing the
// segment's bounding box holds no occupied cell.  Points of the segment lie on
// the segment AB (monotone lattice), so they share its bounding box; positions
// use the same fp32 ops as P(k) and a 1e-3 macro-cell margin covers rounding.
#ifndef NACC_MARCH_SEG
#define NACC_MARCH_SEG 16
#endif
#ifndef NACC_MARCH_SEG_CASCADE
#define NACC_MARCH_SEG_CASCADE 16
#endif
// lattice points per segment (8 or 16; build parameters): single-level grids (fine mask, whose
// window NACC_MARCH_WIN must hold a segment's cell range) and cascades (macro test)
constexpr int seg_len(bool l1) { return l1 ? NACC_MARCH_SEG : NACC_MARCH_SEG_CASCADE; }
static_assert(NACC_MARCH_SEG == 8 || NACC_MARCH_SEG == 16, "segment length");
static_assert(NACC_MARCH_SEG_CASCADE == 8 || NACC_MARCH_SEG_CASCADE == 16, "segment length");
constexpr int kMacro = kMacroCells;  // fine cells per macro cell and axis
// segment-test flag (cascades): every point of the segment lies in level (code >> 4) & 7 or the
// next one, so P(k) needs at most two box tests instead of the level search
constexpr int kTwoLevels = 0x100;
constexpr float kSegEps = 1e-3f;

#ifndef NACC_MARCH_STATS
#define NACC_MARCH_STATS 0  // debug build: count segment classes (nacc_debug_march_stats)
#endif
#if NACC_MARCH_STATS
// [0] owner slots tested, [1] skipped, [2] solid (direct), [3] queued code 1 (interior), [4] queued code 2,
// [5] evaluation passes, [6] writer passes, [7] tiles, [8] phase-1 passes, [9] emitted points of evaluated
// segments; why segments are evaluated: [10] an end outside every box, [11] two adjacent levels,
// [12] a level gap, [13] the finer box within reach, [14] span > the largest window, [15] window not
// interior; evaluated segments that came out [16] full / [17] empty
__device__ unsigned long long g_march_stats[18];
#define MSTAT(i, v) atomicAdd(&g_march_stats[i], (unsigned long long)(v))
#else
#define MSTAT(i, v) ((void)0)
#endif

// The same decision at the fine resolution (reading #22).  The points of a
// segment have positions x and cell coordinates u = (x - lo) * s computed by
// the normative fp32 ops of P(k), each of which is monotone in m (RN rounding
// is monotone), so every point's floor(u) lies between the endpoints' floors,
// exactly, per axis.  With at most W = g.win cells per axis that range lies
// in c + {0..W-1}^3, c = the clamped low corner, and mask3[c] (the OR of those
// W^3 fine bits) being 0 proves no point is emitted.  A segment whose floors lie
// in [0, R-2] on every axis is inside the box (u >= 0 <=> x >= lo exactly;
// u < R-1 keeps x below hi by a cell), so its points skip the box test and the
// clamp.  Cascades run this on level l once both ends are known to lie in l and
// the segment misses the finer box (segment_test below).
__device__ __forceinline__ void cell_floors(const GridConst &g, const float X[3], int f[3], int l = 0) {
#pragma unroll
  for (int a = 0; a < 3; ++a) f[a] = (int)floorf(__fmul_rn(__fsub_rn(X[a], g.lo[l][a]), g.s[l][a]));
}

// the fine test from the endpoints' cell floors (ia: first point, ib: last point or any later one)
__device__ __forceinline__ int segment_test_floors(const GridConst &g, const uint32_t *__restrict__ bits,
                                                   const uint32_t *__restrict__ mask3, const int ia[3],
                                                   const int ib[3], int l = 0) {
  const int R = g.res;
  int c[3], span = 0;
  bool interior = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int lo = min(ia[a], ib[a]), hi = max(ia[a], ib[a]);
    if (hi - lo > g.win - 1) {  // longer than the largest window: evaluate
      MSTAT(14, 1);
      return 2;
    }
    if (hi < 0 || lo > R) return 0;          // every point outside the box on this axis
    interior = interior && lo >= 0 && hi <= R - 2;
    c[a] = min(max(lo, 0), R - 1);
    span = max(span, hi - lo);
  }
  const uint32_t q = (uint32_t)c[0] + (uint32_t)R * ((uint32_t)c[1] + (uint32_t)R * (uint32_t)c[2]);
  // the window of the segment's cell span, w = span + 1 cells per axis: OR_w at
  // mask3 + 2 (w - 2) masks, AND_w right after (gridaux.cu); a segment inside one cell (w = 1)
  // reads the cell's own fine bit for both
  const uint32_t *orm = span == 0 ? bits : mask3 + 2u * (uint32_t)(span - 1) * g.mw;
  const uint32_t *andm = span == 0 ? bits : orm + g.mw;
  const uint32_t wi = (uint32_t)l * g.r3w + (q >> 5);
  if (!((__ldg(orm + wi) >> (q & 31u)) & 1u)) return 0;
  if (!interior) {
    MSTAT(15, 1);
    return 2;
  }
  // solid window: every cell the points can fall in is occupied, so every point is a member
  // (subject only to k < ke and m < far)
  if (NACC_MARCH_SOLID && ((__ldg(andm + wi) >> (q & 31u)) & 1u)) return 3;
  return 1;
}

__device__ __forceinline__ int segment_test_fine(const GridConst &g, const uint32_t *__restrict__ bits,
                                                 const uint32_t *__restrict__ mask3, const float A[3],
                                                 const float B[3]) {
  int ia[3], ib[3];
  cell_floors(g, A, ia);
  cell_floors(g, B, ib);
  return segment_test_floors(g, bits, mask3, ia, ib);
}

// Returns 0 (skip the segment), 1 (evaluate; the segment lies inside the
// single level's box with margin, so P(k) can skip the box test) or 2
// (evaluate with the full predicate).
// la_in / lb_in: the ends' levels when the caller has them (level_of), else -2
template <bool kL1>
__device__ __forceinline__ int segment_test(const GridConst &g, const uint32_t *__restrict__ bits,
                                            const uint32_t *__restrict__ mask2, int M,
                                            const uint32_t *__restrict__ mask3, const float A[3], const float B[3],
                                            int la_in = -2, int lb_in = -2) {
  int la = 0;
  if (!kL1) {
    // does the segment's bounding box (padded) reach box l?  Every point of the segment lies in
    // that box (per-axis monotone fp32 positions), so "no" proves no point is in box l
    auto meets = [&](int l) {
      bool m = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float lo = fminf(A[a], B[a]), hi = fmaxf(A[a], B[a]);
        const float pad = kSegEps * (g.hi[l][a] - g.lo[l][a]);
        m = m && hi >= g.lo[l][a] - pad && lo <= g.hi[l][a] + pad;
      }
      return m;
    };
    la = la_in != -2 ? la_in : level_of<false>(g, A[0], A[1], A[2]);
    const int lb = lb_in != -2 ? lb_in : level_of<false>(g, B[0], B[1], B[2]);
    if (la < 0 || lb < 0) {
      MSTAT(10, 1);
      return 2;
    }
    if (la != lb) {
      // ends in adjacent levels and box lo - 1 out of reach: every point's level is lo or lo + 1
      // (both ends lie in the convex box lo + 1), flagged for the two-box evaluation
      const int lo = min(la, lb);
      if (max(la, lb) == lo + 1 && (lo == 0 || !meets(lo - 1))) {
        MSTAT(11, 1);
        return 2 | (lo << 4) | kTwoLevels;
      }
      MSTAT(12, 1);
      return 2;
    }
    if (la >= 1 && meets(la - 1)) {
      MSTAT(13, 1);
      return 2;
    }
    if (mask3 != nullptr) {  // every point lies in level la (convex box, finer box clear): its fine window
      int ia[3], ib[3];
      cell_floors(g, A, ia, la);
      cell_floors(g, B, ib, la);
      const int code = segment_test_floors(g, bits, mask3, ia, ib, la);
      // a non-interior window still knows the level: the two-box evaluation's first box holds
      return code | (la << 4) | (code == 2 ? kTwoLevels : 0);
    }
  }
  int i0[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float sm = g.s[la][a] * (1.0f / kMacro);
    const float ua = (A[a] - g.lo[la][a]) * sm, ub = (B[a] - g.lo[la][a]) * sm;
    const int lo = (int)floorf(fminf(ua, ub) - kSegEps), hi = (int)floorf(fmaxf(ua, ub) + kSegEps);
    // single level: a segment reaching outside [0, M) macro cells (with margin) touches the box faces
    if (kL1 && (lo < 0 || hi >= M)) return 2;
    if (hi - lo > 1) return 2;
    i0[a] = min(max(lo, 0), M - 1);
  }
  const uint32_t q = (uint32_t)la * (uint32_t)(M * M * M) + (uint32_t)i0[0] +
                     (uint32_t)M * ((uint32_t)i0[1] + (uint32_t)M * (uint32_t)i0[2]);
  if (!((__ldg(mask2 + (q >> 5)) >> (q & 31u)) & 1u)) return 0;
  return kL1 ? 1 : 2;
}

// P(k) for a point known to lie inside the (single) level box by a margin far
// above the fp32 error: the box test is skipped, the rest is the normative
// sequence of occupied()
__device__ __forceinline__ bool occupied_interior(const GridConst &g, const uint32_t *__restrict__ bits, float m,
                                                  float ox, float oy, float oz, float dx, float dy, float dz,
                                                  int l = 0) {
  const float x = __fmaf_rn(m, dx, ox), y = __fmaf_rn(m, dy, oy), z = __fmaf_rn(m, dz, oz);
  const int R = g.res;
  // the segment test proved every point in level l's box with floor(u) in [0, R-2] (and
  // outside the finer box), so l* = l and the clamp is the identity
#if NACC_MARCH_MAGICFLOOR
  // floor of u in [0, 2^23) without the conversion unit: u + 2^23 rounded toward zero holds
  // floor(u) in its mantissa (bit-identical to floorf there)
  const int ix = __float_as_int(__fadd_rz(__fmul_rn(__fsub_rn(x, g.lo[l][0]), g.s[l][0]), 8388608.0f)) - 0x4B000000;
  const int iy = __float_as_int(__fadd_rz(__fmul_rn(__fsub_rn(y, g.lo[l][1]), g.s[l][1]), 8388608.0f)) - 0x4B000000;
  const int iz = __float_as_int(__fadd_rz(__fmul_rn(__fsub_rn(z, g.lo[l][2]), g.s[l][2]), 8388608.0f)) - 0x4B000000;
#else
  const int ix = (int)floorf(__fmul_rn(__fsub_rn(x, g.lo[l][0]), g.s[l][0]));
  const int iy = (int)floorf(__fmul_rn(__fsub_rn(y, g.lo[l][1]), g.s[l][1]));
  const int iz = (int)floorf(__fmul_rn(__fsub_rn(z, g.lo[l][2]), g.s[l][2]));
#endif
  const uint32_t q = (uint32_t)l * (uint32_t)(R * R * R) + (uint32_t)ix +
                     (uint32_t)R * ((uint32_t)iy + (uint32_t)R * (uint32_t)iz);
  return (__ldg(bits + (q >> 5)) >> (q & 31u)) & 1u;
}

// P(k) for a point whose level is known to be lo or lo + 1 (kTwoLevels segments): the normative
// l* is the first of the nested boxes holding x, so two box tests replace the level search
__device__ __forceinline__ bool occupied_two(const GridConst &g, const uint32_t *__restrict__ bits, float m,
                                             float ox, float oy, float oz, float dx, float dy, float dz, int lo) {
  const float x = __fmaf_rn(m, dx, ox), y = __fmaf_rn(m, dy, oy), z = __fmaf_rn(m, dz, oz);
  int l = -1;
  if (in_level_box(g, lo, x, y, z)) l = lo;
  else if (lo + 1 < g.levels && in_level_box(g, lo + 1, x, y, z)) l = lo + 1;
  if (l < 0) return false;
  const int R = g.res;
  int ix = (int)floorf(__fmul_rn(__fsub_rn(x, g.lo[l][0]), g.s[l][0]));
  int iy = (int)floorf(__fmul_rn(__fsub_rn(y, g.lo[l][1]), g.s[l][1]));
  int iz = (int)floorf(__fmul_rn(__fsub_rn(z, g.lo[l][2]), g.s[l][2]));
  ix = min(max(ix, 0), R - 1);
  iy = min(max(iy, 0), R - 1);
  iz = min(max(iz, 0), R - 1);
  const uint32_t q = (uint32_t)l * (uint32_t)(R * R * R) + (uint32_t)ix +
                     (uint32_t)R * ((uint32_t)iy + (uint32_t)R * (uint32_t)iz);
  return (__ldg(bits + (q >> 5)) >> (q & 31u)) & 1u;
}

// ---------------------------------------------------------------- per-ray setup
struct RaySetup {
  float ox, oy, oz, dx, dy, dz, near_r, far_r, t_lo, t_hi;
  bool hit;
};

// The slab only bounds the k range (±2 steps of slack around the outermost box
// padded by 1e-4 of its width), so fp32 with reciprocals is conservative
// enough: its error (~1e-6 of t) is far below the slack.  P(k) decides.
// The slab box is the outermost level box intersected with the padded world
// box of all occupied cells (gridaux.cu), so rays stop scanning where no cell
// of any level can be occupied.
__device__ __forceinline__ RaySetup ray_setup(const GridConst &g, const MarchConst &p, const float *__restrict__ obox,
                                              const float *__restrict__ rays_o, const float *__restrict__ rays_d,
                                              const float *__restrict__ t_min, const float *__restrict__ t_max,
                                              int64_t r) {
  RaySetup s;
  s.ox = __ldg(rays_o + 3 * r);
  s.oy = __ldg(rays_o + 3 * r + 1);
  s.oz = __ldg(rays_o + 3 * r + 2);
  s.dx = __ldg(rays_d + 3 * r);
  s.dy = __ldg(rays_d + 3 * r + 1);
  s.dz = __ldg(rays_d + 3 * r + 2);
  float nr = t_min ? __ldg(t_min + r) : p.near_plane;
  if (p.stratified) {
    const u32x4 rnd =
        philox4x32_10(u32x4{(uint32_t)(uint64_t)r, (uint32_t)((uint64_t)r >> 32), 0u, 0u}, p.key0, p.key1);
    nr = __double2float_rn(__dadd_rn((double)nr, __dmul_rn(u24(rnd.x), (double)p.step)));
  }
  s.near_r = nr;
  s.far_r = t_max ? __ldg(t_max + r) : p.far_plane;
  const float o[3] = {s.ox, s.oy, s.oz}, d[3] = {s.dx, s.dy, s.dz};
  float tmin = -INFINITY, tmax = INFINITY;
  bool hit = __ldg(obox) <= __ldg(obox + 3);  // false when no cell is occupied
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float blo = fmaxf(g.olo[a], __ldg(obox + a)), bhi = fminf(g.ohi[a], __ldg(obox + 3 + a));
    if (fabsf(d[a]) > 1e-30f) {
      const float inv = __frcp_rn(d[a]);
      float ta = (blo - o[a]) * inv, tb = (bhi - o[a]) * inv;
      tmin = fmaxf(tmin, fminf(ta, tb));
      tmax = fminf(tmax, fmaxf(ta, tb));
    } else if (!(blo <= o[a] && o[a] < bhi)) {
      hit = false;
    }
  }
  s.t_lo = fmaxf(tmin, s.near_r);
  s.t_hi = fminf(tmax, s.far_r);
  s.hit = hit && (s.t_hi > s.t_lo);
  return s;
}

// k range of the uniform lattice that can hold emitted intervals: ±2 steps of
// slack plus 2^-20 of the index itself, which covers the relative error of the
// fp32 slab and of this division (a few ulps) up to the 2^24 index cap
__device__ __forceinline__ void uniform_k_range(const RaySetup &s, const MarchConst &p, int64_t &kb, int64_t &ke) {
  const float xb = (s.t_lo - s.near_r) * p.inv_step, xe = (s.t_hi - s.near_r) * p.inv_step;
  const float fb = floorf(xb - 0.5f - fabsf(xb) * 0x1p-20f) - 2.0f;
  const float fe = ceilf(xe + fabsf(xe) * 0x1p-20f) + 3.0f;
  const float cap = (float)(1 << 24);
  kb = fb > 0.0f ? (int64_t)fminf(fb, cap) : 0;
  ke = fe > 0.0f ? (int64_t)fminf(fe, cap) : 0;
}

// first index k in [0, K) with tab[k] >= v (tab ascending)
__device__ __forceinline__ int64_t lower_bound(const float *__restrict__ tab, int64_t K, float v) {
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(tab + mid) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// cone lattice table: tab[0..K] = t_0..t_K, K = number of intervals whose
// midpoint is < far and whose start is <= t_cap (+3 slack intervals)
constexpr int64_t kConeTableMax = 1 << 20;

struct ConeHeader {
  int64_t K;
  int32_t overflow;
  uint32_t t_cap_bits;
};

__global__ void cone_tcap_kernel(GridConst g, MarchConst p, const float *__restrict__ obox, const float *__restrict__ rays_o,
                                 const float *__restrict__ rays_d, const float *__restrict__ t_max,
                                 int64_t n_rays, ConeHeader *hdr) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float v = 0.0f;
  if (r < n_rays) {
    RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, nullptr, t_max, r);
    if (s.hit) v = s.t_hi;
  }
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.0f) atomicMax(&hdr->t_cap_bits, __float_as_uint(v));
}

__global__ void cone_table_kernel(MarchConst p, ConeHeader *hdr, float *__restrict__ tab) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const float t_cap = __uint_as_float(hdr->t_cap_bits);
  float t = p.near_plane;
  int64_t k = 0;
  int extra = 0;
  int32_t overflow = 0;
  tab[0] = t;
  for (;;) {
    const float dt = fminf(fmaxf(__fmul_rn(t, p.cone), p.step), p.max_step);
    const float m = __fadd_rn(t, __fmul_rn(0.5f, dt));
    const float tn = __fadd_rn(t, dt);
    if (!(m < p.far_plane)) break;
    if (t > t_cap && ++extra > 3) break;
    if (k + 1 >= kConeTableMax) {
      overflow = 1;
      break;
    }
    tab[k + 1] = tn;
    ++k;
    t = tn;
  }
  hdr->K = k;
  hdr->overflow = overflow;
}

// Uniform lattice midpoint m_k = fp32(near_r + (k + 1/2)Δt), the exact value
// rounded once (reading #3).  For k < 2^23, k + 1/2 is an fp32 and one fmaf is
// that rounding.  Above (lattice indices go up to 2^24), (k + 1/2)Δt is an
// exact fp64 product (25 x 24 bits) and the fp64 sum with near_r is rounded
// to fp32 with the tie fixed by the sign of its TwoSum error (a double rounding
// differs from the single one only on an exact fp32 tie).
__device__ __noinline__ float lattice_mid_wide(int k, float step, float near_r) {
  const double a = (double)near_r, b = __dmul_rn((double)k + 0.5, (double)step);
  const double s = __dadd_rn(a, b);
  const double a1 = __dsub_rn(s, b), b1 = __dsub_rn(s, a1);
  const double e = __dadd_rn(__dsub_rn(a, a1), __dsub_rn(b, b1));
  float r = __double2float_rn(s);
  if (e != 0.0) {
    const float lo = __double2float_rd(s), hi = __double2float_ru(s);
    if (lo != hi && __dsub_rn(s, (double)lo) == __dsub_rn((double)hi, s)) r = e > 0.0 ? hi : lo;
  }
  return r;
}

__device__ __forceinline__ float lattice_mid_uniform(int k, float step, float near_r) {
  if (k < (1 << 23)) return __fmaf_rn((float)k + 0.5f, step, near_r);
  return lattice_mid_wide(k, step, near_r);
}

// the same for code paths that know every index they see is < 2^23 (kWide = false)
template <bool kWide>
__device__ __forceinline__ float lattice_mid_u(int k, float step, float near_r) {
  return kWide ? lattice_mid_uniform(k, step, near_r) : __fmaf_rn((float)k + 0.5f, step, near_r);
}

// midpoint of lattice interval k (uniform or cone table)
template <bool kCone>
__device__ __forceinline__ float lattice_mid(const MarchConst &p, const RaySetup &s, const float *__restrict__ tab,
                                             int k) {
  if (kCone) {
    const float ta = __ldg(tab + k);
    const float dt = fminf(fmaxf(__fmul_rn(ta, p.cone), p.step), p.max_step);
    return __fadd_rn(ta, __fmul_rn(0.5f, dt));
  }
  return lattice_mid_uniform(k, p.step, s.near_r);
}

template <bool kCone>
__device__ __forceinline__ void lattice_ends(const MarchConst &p, float near_r, const float *__restrict__ tab,
                                             int k, float &ta, float &tb) {
  if (kCone) {
    ta = __ldg(tab + k);
    tb = __ldg(tab + k + 1);
  } else {
    ta = __fmaf_rn((float)k, p.step, near_r);
    tb = __fmaf_rn((float)(k + 1), p.step, near_r);
  }
}

// Traverse one ray with one warp.  Each step the 32 lanes test 32 segments of
// kSeg lattice points (kSkip), the flagged segments are compacted through the
// warp's shared `seglist` and evaluated exactly, 4 segments = 32 points per
// pass, in increasing k.  emit(ballot, pred, k) is called once per pass by all
// lanes.  Returns the ray's count.
template <bool kCone, bool kSkip, bool kL1, typename Emit>
__device__ __forceinline__ int32_t traverse_ray(const GridConst &g, const MarchConst &p,
                                                const uint32_t *__restrict__ bits,
                                                const uint32_t *__restrict__ mask2, int M,
                                                const uint32_t *__restrict__ mask3, const RaySetup &s,
                                                const ConeHeader *__restrict__ hdr, const float *__restrict__ tab,
                                                int *seglist, int &kb_out, int &ke_out, Emit emit) {
  const int lane = threadIdx.x & 31;
  int32_t cnt = 0;
  kb_out = ke_out = 0;
  if (!s.hit) return 0;
  int kb, ke;  // lattice indices are < 2^24 (fp32-exact), so int32 throughout
  if (kCone) {
    const int K = (int)hdr->K;
    kb = (int)lower_bound(tab + 1, K, s.t_lo) - 2;  // first k with t_{k+1} >= t_lo, minus slack
    if (kb < 0) kb = 0;
    ke = (int)lower_bound(tab, K + 1, s.t_hi) + 2;  // first k with t_k >= t_hi, plus slack
    if (ke > K) ke = K;
  } else {
    int64_t b64, e64;
    uniform_k_range(s, p, b64, e64);
    kb = (int)b64;
    ke = (int)e64;
  }
  kb_out = kb;
  ke_out = ke;
  constexpr int kSeg = seg_len(kL1);
  constexpr int kSegPerPass = 32 / kSeg;  // segments evaluated per 32-lane pass
  constexpr int kSpan = kSkip ? 32 * kSeg : 32;
  // shared endpoints (uniform single-level lattice, fine mask): every lane computes the cell
  // floors of its segment's first point only; a segment's range is closed by the next lane's
  // first point (a later point: still a superset by monotonicity), so a window holds 31
  // segments and lane 31 only supplies the last end
  const bool shared = NACC_MARCH_SHAREDENDS && kSkip && kL1 && !kCone && mask3 != nullptr;
  const int span = shared ? 31 * kSeg : kSpan;
  for (int k0 = kb; k0 < ke; k0 += span) {
    int nseg = 1;
    if (kSkip && shared) {
      const int ks = k0 + lane * kSeg;
      const float m = lattice_mid<false>(p, s, tab, ks);
      const float X[3] = {__fmaf_rn(m, s.dx, s.ox), __fmaf_rn(m, s.dy, s.oy), __fmaf_rn(m, s.dz, s.oz)};
      int fa[3], fb[3];
      cell_floors(g, X, fa);
#pragma unroll
      for (int a = 0; a < 3; ++a) fb[a] = __shfl_down_sync(kFull, fa[a], 1);
      int code = 0;
      if (lane < 31 && ks < ke) code = segment_test_floors(g, bits, mask3, fa, fb);
      const bool flag = code != 0;
      const unsigned F = __ballot_sync(kFull, flag);
      if (flag) seglist[__popc(F & ((1u << lane) - 1u))] = lane | (code == 1 ? 0x100 : (code == 3 ? 0x300 : 0));
      __syncwarp();
      nseg = __popc(F);
    } else if (kSkip) {
      const int ks = k0 + lane * kSeg;
      bool flag = false;
      int code = 0, lvl = 0;
      if (ks < ke) {
        const int kl = min(ks + kSeg - 1, ke - 1);
        const float ma = lattice_mid<kCone>(p, s, tab, ks), mb = lattice_mid<kCone>(p, s, tab, kl);
        const float A[3] = {__fmaf_rn(ma, s.dx, s.ox), __fmaf_rn(ma, s.dy, s.oy), __fmaf_rn(ma, s.dz, s.oz)};
        const float B[3] = {__fmaf_rn(mb, s.dx, s.ox), __fmaf_rn(mb, s.dy, s.oy), __fmaf_rn(mb, s.dz, s.oz)};
        code = (kL1 && mask3 != nullptr) ? segment_test_fine(g, bits, mask3, A, B)
                                          : segment_test<kL1>(g, bits, mask2, M, mask3, A, B);
        lvl = (code >> 4) & 7;  // cascades: the level every point of the segment lies in
        code &= 15;
        flag = code != 0;
#if NACC_MARCH_PREFETCH
        if (code == 1) {  // interior segment: warm L1 with the bit words its points will read
          const int R = g.res;
          int ia[3], ib[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            ia[a] = min(max((int)floorf((A[a] - g.lo[0][a]) * g.s[0][a]), 0), R - 1);
            ib[a] = min(max((int)floorf((B[a] - g.lo[0][a]) * g.s[0][a]), 0), R - 1);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t q = (uint32_t)ia[0] + (uint32_t)R * ((uint32_t)((c & 1) ? ib[1] : ia[1]) +
                                                                (uint32_t)R * (uint32_t)((c & 2) ? ib[2] : ia[2]));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(bits + (q >> 5)));
          }
        }
#endif
      }
      const unsigned F = __ballot_sync(kFull, flag);
      if (flag)
        seglist[__popc(F & ((1u << lane) - 1u))] = lane | (code == 1 ? 0x100 : (code == 3 ? 0x300 : 0)) | (lvl << 12);
      __syncwarp();
      nseg = __popc(F);
    }
    // lane (lane % kSeg) of segment list entry idx: its point k and P(k)
    auto eval = [&](int idx, int &k) -> bool {
      bool interior = false, solid = false;
      int lv = 0;
      if (kSkip) {
        const int e = idx < nseg ? seglist[idx] : 0;
        k = idx < nseg ? k0 + (e & 0xff) * kSeg + (lane % kSeg) : ke;
        interior = (e & 0x100) != 0;
        solid = (e & 0x200) != 0;
        lv = kL1 ? 0 : (e >> 12) & 7;
      } else {
        k = k0 + lane;
      }
      bool pred = false;
      if (k < ke) {
        const float m = lattice_mid<kCone>(p, s, tab, k);
        if (m < s.far_r)
          pred = solid ? true
                       : (interior ? occupied_interior(g, bits, m, s.ox, s.oy, s.oz, s.dx, s.dy, s.dz, lv)
                                   : occupied<kL1>(g, bits, m, s.ox, s.oy, s.oz, s.dx, s.dy, s.dz));
      }
      return pred;
    };
    // two passes of 4 segments per iteration (independent chains for ILP), emitted in k order
    for (int first = 0; first < nseg; first += (kSkip ? 2 * kSegPerPass : 32)) {
      int ka, kb2;
      const bool pa = eval(first + lane / kSeg, ka);
      if (kSkip && first + kSegPerPass < nseg) {
        const bool pb = eval(first + kSegPerPass + lane / kSeg, kb2);
        const unsigned ba = __ballot_sync(kFull, pa);
        emit(ba, pa, ka, cnt);
        cnt += __popc(ba);
        const unsigned bb = __ballot_sync(kFull, pb);
        emit(bb, pb, kb2, cnt);
        cnt += __popc(bb);
      } else {
        const unsigned ba = __ballot_sync(kFull, pa);
        emit(ba, pa, ka, cnt);
        cnt += __popc(ba);
      }
    }
    if (kSkip) __syncwarp();
  }
  return cnt;
}

// ---------------------------------------------------------------- fused single-pass march
// Persistent warps; a tile = kTRays consecutive rays, handed out by an atomic
// counter.  Phase 1 of a tile treats the segments of ALL its rays as one flat
// list, so a warp pass never idles lanes at the end of a ray:
//   ray j covers slots [base_j, base_j + nseg_j] -- one slot per 16-point
//   segment q < nseg_j of its k range [kb_j, ke_j), plus one terminal slot that
//   only supplies the next point; every lane computes the position (and cell
//   floors) of its slot's first point, and an owner lane (lanes 0..30, not a
//   terminal) tests its segment against the window masks with the next lane's
//   point as the segment's far end (a later point: a superset by monotonicity,
//   reading #22).  A pass advances 31 slots.
// Flagged segments get entries, in (ray, k) order, in the warp's shared entry
// buffer: (j << (16 + kQBits)) | (q << 16) | mask of the segment's emitted points.  A
// solid segment (every point provably a member, all < ke and < far) writes its
// full mask at once; the others are queued and evaluated exactly, two
// segments per 32-lane pass, filling in their masks.  Per-ray counts
// accumulate in shared memory; the tile's total is published for the
// decoupled look-back.  Phase 2 of the PREVIOUS tile (software pipeline:
// its predecessors have had a tile's time to publish) resolves its output
// offset, writes packed_info, and streams its entries into contiguous
// (t0, t1, ray_id) runs, 32 lattice points per pass.  A tile whose entries
// overflow the buffer (or with a ray longer than 2^16 points) is counted and
// written by direct traversal instead (traverse_ray).
#ifndef NACC_MARCH_WPAIR
#define NACC_MARCH_WPAIR 1  // build parameter: writer with two consecutive lattice points per lane (0 off,
                            // 1 cones / cascades: CFG3 2.236 -> 2.182 ms; 2 every grid: CFG2 161.5 -> 163.1 us)
#endif
#ifndef NACC_MARCH_NOLOOKBACK
#define NACC_MARCH_NOLOOKBACK 0  // timing experiment only (wrong output): no look-back
#endif
#ifndef NACC_MARCH_TRAYS
#define NACC_MARCH_TRAYS 16  // build parameter: rays per tile
#endif
#ifndef NACC_MARCH_ECAP
#define NACC_MARCH_ECAP 384  // build parameter: entries (flagged 16-point segments) per tile buffer (A/B 256 / 320 /
                             // 384 / 512 / 768: CFG3 5.76 / 2.21 / 2.12 / 2.19 / 2.51 ms, CFG2 161 us at <= 512)
#endif
#ifndef NACC_MARCH_WARPS
#define NACC_MARCH_WARPS 4  // build parameter: warps per block of the fused march
#endif
constexpr int kFWarps = NACC_MARCH_WARPS, kTRays = NACC_MARCH_TRAYS, kECap = NACC_MARCH_ECAP;
// cone lattices and cascades give long rays (up to ~900 points, 57 segments): half the rays per
// tile, so a tile's entries fit the buffer even when every segment is flagged
constexpr int tile_rays(bool cone, bool l1) { return (cone || !l1) ? kTRays / 2 : kTRays; }
constexpr int kTSeg = 16;   // lattice points per segment / entry mask bits
constexpr int kEvCap = 64;  // queued segments awaiting evaluation
static_assert(kTRays <= 32, "one lane per ray of a tile");
// entry = (j << (16 + kQBits)) | (q << 16) | 16-bit mask: ray index j, segment index q
constexpr int kJBits = kTRays > 16 ? 5 : 4;
constexpr int kQBits = 16 - kJBits;
constexpr uint32_t kQMask = (1u << kQBits) - 1u;
__device__ __forceinline__ uint32_t ent_pack(int j, int q, uint32_t mask) {
  return ((uint32_t)j << (16 + kQBits)) | ((uint32_t)q << 16) | mask;
}
__device__ __forceinline__ int ent_j(uint32_t e) { return (int)(e >> (16 + kQBits)); }
__device__ __forceinline__ int ent_k16(uint32_t e) { return (int)((e >> 12) & (kQMask << 4)); }  // 16 q
// queued segment = slot (10 bits) | j | q | code (2 bits, at 26) | level (3 bits, at 28)
__device__ __forceinline__ uint32_t evq_pack(int slot, int j, int q, int code, int lvl) {
  return (uint32_t)min(slot, 1023) | ((uint32_t)j << 10) | ((uint32_t)q << (10 + kJBits)) | ((uint32_t)code << 26) |
         ((uint32_t)lvl << 28);
}
static_assert(kECap <= 1024, "10-bit entry slot in the evaluation queue");
static_assert(NACC_MARCH_SEG == kTSeg && NACC_MARCH_SEG_CASCADE == kTSeg, "16-point segments");

struct TileBuf {                 // one tile in flight (per warp, double-buffered)
  float4 od[kTRays][2];          // (ox, oy, oz, near_r), (dx, dy, dz, far_r)
  int2 kr[kTRays];               // (kb, ke)
  int cnt[kTRays];               // emitted samples per ray
  uint32_t ent[kECap];           // entries, (ray, k) order
};

// uniform lattice midpoint / ends with the per-ray anchor (cone: the shared table)
template <bool kCone, bool kWide>
__device__ __forceinline__ float tile_mid(const MarchConst &p, float near_r, const float *__restrict__ tab, int k) {
  if (kCone) {
    const float ta = __ldg(tab + k);
    const float dt = fminf(fmaxf(__fmul_rn(ta, p.cone), p.step), p.max_step);
    return __fadd_rn(ta, __fmul_rn(0.5f, dt));
  }
  return lattice_mid_u<kWide>(k, p.step, near_r);
}

// Phase 2 of a tile (the fused kernel's software pipeline, one tile behind phase 1): the
// tile's output offset is `excl`; writes packed_info and streams its entries (or, for an
// overflowed tile, traverses its rays again).
template <bool kCone, bool kSkip, bool kL1>
__device__ __forceinline__ void tile_write(const TileBuf &T, int n_ent_t, bool over, int c_lane, int64_t tile,
                                           long long excl, long long agg, const GridConst &g, const MarchConst &p,
                                           const uint32_t *__restrict__ bits, const uint32_t *__restrict__ mask2,
                                           int M, const uint32_t *__restrict__ mask3, const float *__restrict__ obox,
                                           const float *__restrict__ rays_o, const float *__restrict__ rays_d,
                                           const float *__restrict__ t_min, const float *__restrict__ t_max,
                                           int64_t n_rays, const ConeHeader *__restrict__ hdr,
                                           const float *__restrict__ tab, int64_t *__restrict__ packed_info,
                                           int64_t capacity, float *__restrict__ t0, float *__restrict__ t1,
                                           int32_t *__restrict__ ray_id, int *seglist, float **obase) {
  constexpr int kR = tile_rays(kCone, kL1);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t r_base = tile * kR;
  const int c = lane < kR ? c_lane : 0;
  long long incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  const long long run = excl + incl - c;
  if (lane < kR && r_base + lane < n_rays)
    reinterpret_cast<longlong2 *>(packed_info)[r_base + lane] = make_longlong2(run, c);
  if (t0 != nullptr && excl + agg <= capacity) {
    if (!over) {
      const int n_ent = n_ent_t;
      // the tile's output bases through shared memory, opaque to the optimiser, so every store
      // is one 32-bit-offset IMAD.WIDE from a base register (the compiler otherwise re-associated
      // excl + pos into a 64-bit add chain per store)
      if (lane == 0) {
        obase[0] = t0 + excl;
        obase[1] = t1 + excl;
        obase[2] = reinterpret_cast<float *>(ray_id + excl);
      }
      __syncwarp();
      float *const o0 = obase[0], *const o1 = obase[1];
      int32_t *const oid = reinterpret_cast<int32_t *>(obase[2]);
      int carry = 0;  // samples written so far in the tile
      if constexpr (NACC_MARCH_WPAIR == 2 || (NACC_MARCH_WPAIR == 1 && (kCone || !kL1))) {
      // two consecutive lattice points per lane, four entries per pass: one entry decode, one
      // k, three lattice ends and one output position per two samples; the points' output slots
      // come from two ballots (a lane's two samples are consecutive in the output)
      const int b2 = (lane & 7) * 2;
      for (int e = 0; e < n_ent; e += 4) {
        const int idx = e + (lane >> 3);
        const uint32_t ent = idx < n_ent ? T.ent[idx] : 0u;
        const bool s0 = (ent >> b2) & 1u, s1 = (ent >> (b2 + 1)) & 1u;
        const unsigned B0 = __ballot_sync(kFull, s0), B1 = __ballot_sync(kFull, s1);
        if (NACC_MARCH_STATS && lane == 0) MSTAT(6, 1);
        if (s0 || s1) {
          const int j = ent_j(ent);
          const int pos = carry + __popc(B0 & lt) + __popc(B1 & lt);
          const int k = T.kr[j].x + ent_k16(ent) + b2;  // kb_j + 16 q + b2
          const int32_t rid = (int32_t)(r_base + j);
          float ta, tb, tc;
          if (kCone) {
            ta = __ldg(tab + k);
            tb = __ldg(tab + k + 1);
            tc = s1 ? __ldg(tab + k + 2) : 0.f;
          } else {
            const float nr = T.od[j][0].w;
            ta = __fmaf_rn((float)k, p.step, nr);
            tb = __fmaf_rn((float)(k + 1), p.step, nr);
            tc = __fmaf_rn((float)(k + 2), p.step, nr);
          }
          if (s0) {
            o0[pos] = ta;
            o1[pos] = tb;
            oid[pos] = rid;
          }
          if (s1) {
            const int p1 = pos + (s0 ? 1 : 0);
            o0[p1] = tb;
            o1[p1] = tc;
            oid[p1] = rid;
          }
        }
        carry += __popc(B0) + __popc(B1);
      }
      } else {
      const int b = lane & 15;
      for (int e = 0; e < n_ent; e += 2) {
        const int idx = e + (lane >> 4);
        const uint32_t ent = idx < n_ent ? T.ent[idx] : 0u;
        const bool set = (ent >> b) & 1u;
        const unsigned bal = __ballot_sync(kFull, set);  // both entries' masks, in output order
        if (NACC_MARCH_STATS && lane == 0) MSTAT(6, 1);
        if (set) {
          const int j = ent_j(ent);
          const int pos = carry + __popc(bal & lt);
          const int k = T.kr[j].x + ent_k16(ent) + b;  // kb_j + 16 q + b
          float ta, tb2;
          lattice_ends<kCone>(p, T.od[j][0].w, tab, k, ta, tb2);
          o0[pos] = ta;
          o1[pos] = tb2;
          oid[pos] = (int32_t)(r_base + j);
        }
        carry += __popc(bal);
      }
      }
    } else {  // overflowed tile: traverse again, writing directly
      for (int jj = 0; jj < kR; ++jj) {
        const int64_t r = r_base + jj;
        if (r >= n_rays) break;
        const long long rj = __shfl_sync(kFull, run, jj);
        const RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, t_min, t_max, r);
        int kb0, ke0;
        traverse_ray<kCone, kSkip, kL1>(g, p, bits, mask2, M, mask3, s, hdr, tab, seglist, kb0, ke0,
                                        [&](unsigned bb, bool pred, int k, int32_t cnt) {
                                          if (pred) {
                                            const int64_t qq = rj + cnt + __popc(bb & lt);
                                            float ta, tb2;
                                            lattice_ends<kCone>(p, s.near_r, tab, k, ta, tb2);
                                            t0[qq] = ta;
                                            t1[qq] = tb2;
                                            ray_id[qq] = (int32_t)r;
                                          }
                                        });
      }
    }
  }
  __syncwarp();  // the buffer is refilled next
}

// kBounds: the combined estimator's per-ray span (nacc_occgrid_ray_bounds) from the same phase 1 --
// the first and the last emitted point of each ray from its first and last entries with a set bit
// -- with no look-back and no writer (t0 / t1 carry t_near / t_far).
template <bool kCone, bool kSkip, bool kL1, bool kBounds = false>
__global__ void __launch_bounds__(kFWarps * 32, NACC_MARCH_MINB) march_fused_kernel(
    GridConst g, MarchConst p, const uint32_t *__restrict__ bits, const uint32_t *__restrict__ mask2, int M,
    const uint32_t *__restrict__ mask3, const float *__restrict__ obox, const float *__restrict__ rays_o,
    const float *__restrict__ rays_d, const float *__restrict__ t_min, const float *__restrict__ t_max,
    int64_t n_rays, int64_t n_tiles, const ConeHeader *__restrict__ hdr, const float *__restrict__ tab,
    LookbackWs *__restrict__ lb, int64_t *__restrict__ packed_info, int64_t *__restrict__ total, int64_t capacity,
    int32_t *__restrict__ status_out, float *__restrict__ t0, float *__restrict__ t1, int32_t *__restrict__ ray_id,
    unsigned long long *__restrict__ n_alive = nullptr) {
  constexpr int kR = tile_rays(kCone, kL1);  // rays per tile
  __shared__ int s_efirst[kBounds ? kFWarps : 1][kTRays], s_elast[kBounds ? kFWarps : 1][kTRays];
  __shared__ TileBuf tb[kFWarps][2];
  __shared__ uint32_t evq[kFWarps][kEvCap];
  __shared__ int seglist[kFWarps][32];  // direct traversal (overflowed tiles)
  __shared__ float *obase[kFWarps][3];   // a tile's output bases (phase 2)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const bool fine = kSkip && kL1 && !kCone && mask3 != nullptr;  // single-level fine-mask test on shared floors
  const int K = kCone ? (int)hdr->K : 0;
  // the previous tile, pending its phase 2 (lane j < kR: ray j)
  int64_t prev_tile = -1;
  int prev_c = 0, prev_ne = 0;
  long long prev_agg = 0;
  bool prev_over = false;
  int buf = 0;
  for (;;) {
    unsigned int tile32 = 0;
    if (lane == 0) tile32 = atomicAdd(&lb->tile_counter, 1u);
    const int64_t tile = (int64_t)__shfl_sync(kFull, tile32, 0);
    const bool have = tile < n_tiles;
    if (kBounds && !have) break;
    int cur_c = 0, cur_ne = 0;
    long long cur_agg = 0;
    bool cur_over = false;
    if (have) {
      // ---------------- phase 1 of `tile`
      TileBuf &T = tb[warp][buf];
      const int64_t r_base = tile * kR;
      int kb = 0, ke = 0, nseg = 0;
      bool longray = false;
      if (lane < kR) {
        if (r_base + lane < n_rays) {
          const RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, t_min, t_max, r_base + lane);
          if (s.hit) {
            if (kCone) {
              kb = max((int)lower_bound(tab + 1, K, s.t_lo) - 2, 0);
              ke = min((int)lower_bound(tab, K + 1, s.t_hi) + 2, K);
            } else {
              int64_t b64, e64;
              uniform_k_range(s, p, b64, e64);
              kb = (int)b64;
              ke = (int)e64;
            }
            if (ke < kb) ke = kb;
            nseg = (ke - kb + kTSeg - 1) / kTSeg;
          }
          T.od[lane][0] = make_float4(s.ox, s.oy, s.oz, s.near_r);
          T.od[lane][1] = make_float4(s.dx, s.dy, s.dz, s.far_r);
        }
        T.kr[lane] = make_int2(kb, ke);
        T.cnt[lane] = 0;
        longray = nseg > (int)kQMask;
      }
      // flat slot list: ray j owns slots [base_j, base_j + nseg_j], every ray at least one
      const int nslot = lane < kR ? nseg + 1 : 0;
      int sbase = nslot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, sbase, o);
        if (lane >= o) sbase += v;
      }
      const int total_slots = __shfl_sync(kFull, sbase, 31);
      sbase -= nslot;  // exclusive
      cur_over = __any_sync(kFull, longray);
      __syncwarp();
      int n_ent = 0, npend = 0;
      // lattice indices >= 2^23 anywhere in the tile (far origins): the exact wide midpoint
      const bool wide = !kCone && __any_sync(kFull, lane < kR && ke + kTSeg > (1 << 23));
      auto phase1 = [&](auto wide_tag) {
      constexpr bool kW = decltype(wide_tag)::value;
      auto evaluate = [&](int n_eval) {  // the first n_eval queued segments, two per 32-lane pass
        for (int e0 = 0; e0 < n_eval; e0 += 2) {
          const int idx = e0 + (lane >> 4);
          const uint32_t qe = idx < n_eval ? evq[warp][idx] : 0u;
          const int j = (qe >> 10) & ((1 << kJBits) - 1), q = (qe >> (10 + kJBits)) & kQMask, code = (qe >> 26) & 3,
                    lv = kL1 ? 0 : (qe >> 28) & 7;  // single level: a constant (no indexed constant loads)
          const bool two = !kL1 && (qe >> 31);
          const int2 kr = T.kr[j];
          const int k = kr.x + q * kTSeg + (lane & 15);
          bool pred = false;
          if (idx < n_eval && k < kr.y) {
            const float4 A = T.od[j][0], D = T.od[j][1];
            const float m = tile_mid<kCone, kW>(p, A.w, tab, k);
            if (m < D.w)
              pred = code == 3 ? true
                               : (code == 1 ? occupied_interior(g, bits, m, A.x, A.y, A.z, D.x, D.y, D.z, lv)
                                  : (two ? occupied_two(g, bits, m, A.x, A.y, A.z, D.x, D.y, D.z, lv)
                                         : occupied<kL1>(g, bits, m, A.x, A.y, A.z, D.x, D.y, D.z)));
          }
          const unsigned bal = __ballot_sync(kFull, pred);
          if (NACC_MARCH_STATS && lane == 0) {
            MSTAT(5, 1);
            MSTAT(9, __popc(bal));
          }
          if ((lane & 15) == 0 && idx < n_eval) {
            const uint32_t half = (lane ? bal >> 16 : bal) & 0xFFFFu;
            const int slot = qe & 1023;
            if (slot < kECap) T.ent[slot] = ent_pack(j, q, half);
            if (NACC_MARCH_STATS) {
              if (half == 0xFFFFu) MSTAT(16, 1);
              if (half == 0u) MSTAT(17, 1);
            }
            atomicAdd(&T.cnt[j], __popc(half));
          }
        }
        __syncwarp();
      };
      {
        for (int P = 0; P < total_slots; P += 31) {
          // slot P + lane -> (ray j, segment q)
          const int sb_in = (lane < kR && sbase > P && sbase < P + 32) ? (1 << (sbase - P)) : 0;
          const unsigned starts = __reduce_or_sync(kFull, (unsigned)sb_in);
          const int jP = __popc(__ballot_sync(kFull, lane < kR && sbase <= P)) - 1;
          const int j = min(jP + __popc(starts & ((2u << lane) - 1u)), kR - 1);
          const int bj = __shfl_sync(kFull, sbase, j);
          const int kbj = __shfl_sync(kFull, kb, j), kej = __shfl_sync(kFull, ke, j), nsj = __shfl_sync(kFull, nseg, j);
          const int q = P + lane - bj;
          const bool valid = P + lane < total_slots;
          const bool owner = lane < 31 && valid && q < nsj;
          const int ks = kbj + q * kTSeg;
          const float4 A = T.od[j][0], D = T.od[j][1];
          // first point of the slot (terminal slot: the point after the ray's last segment)
          const float m = tile_mid<kCone, kW>(p, A.w, tab, kCone ? min(ks, K) : ks);
          const float X[3] = {__fmaf_rn(m, D.x, A.x), __fmaf_rn(m, D.y, A.y), __fmaf_rn(m, D.z, A.z)};
          int code = 0, lvl = 0;
          bool two = false;
          if (!kSkip) {
            code = owner ? 2 : 0;
          } else if (fine) {
            int fa[3], fb[3];
            cell_floors(g, X, fa);
#pragma unroll
            for (int a = 0; a < 3; ++a) fb[a] = __shfl_down_sync(kFull, fa[a], 1);
            if (owner) code = segment_test_floors(g, bits, mask3, fa, fb);
          } else {
            float Y[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) Y[a] = __shfl_down_sync(kFull, X[a], 1);
            // cascades: every slot's first point gets its level once; the segment's far end is
            // the next slot's first point, so its level comes from the next lane
            int la = -2, lb = -2;
            if (!kL1) {
              la = level_of<false>(g, X[0], X[1], X[2]);
              lb = __shfl_down_sync(kFull, la, 1);
            }
            if (owner) {
              code = (kL1 && mask3 != nullptr) ? segment_test_fine(g, bits, mask3, X, Y)
                                                : segment_test<kL1>(g, bits, mask2, M, mask3, X, Y, la, lb);
              two = (code & kTwoLevels) != 0;
              lvl = (code >> 4) & 7;
              code &= 15;
            }
          }
          const bool flag = code != 0;
          bool direct = false;
          if (code == 3 && ks + kTSeg <= kej) direct = tile_mid<kCone, kW>(p, A.w, tab, ks + kTSeg - 1) < D.w;
          const unsigned F = __ballot_sync(kFull, flag), Dm = __ballot_sync(kFull, direct);
          if (NACC_MARCH_STATS) {
            const unsigned Ow = __ballot_sync(kFull, owner);
            const unsigned C1 = __ballot_sync(kFull, code == 1 && !direct);
            if (lane == 0) {
              MSTAT(0, __popc(Ow));
              MSTAT(1, __popc(Ow & ~F));
              MSTAT(2, __popc(Dm));
              MSTAT(3, __popc(C1));
              MSTAT(4, __popc(F & ~Dm & ~C1));
              MSTAT(8, 1);
            }
          }
          const int slot = n_ent + __popc(F & lt);
          if (direct) {
            if (slot < kECap) T.ent[slot] = ent_pack(j, q, 0xFFFFu);
            atomicAdd(&T.cnt[j], kTSeg);
          } else if (flag) {
            evq[warp][npend + __popc((F & ~Dm) & lt)] = evq_pack(slot, j, q, code, lvl) | (two ? 0x80000000u : 0u);
          }
          n_ent += __popc(F);
          npend += __popc(F & ~Dm);
          __syncwarp();
          if (npend >= 32) {  // keep the queue short: evaluate whole passes, keep the remainder
            constexpr int kPerPass = 2;
            const int ne = npend & ~(kPerPass - 1);
            evaluate(ne);
            const int rest = npend - ne;
            const uint32_t keep = lane < rest ? evq[warp][ne + lane] : 0u;
            __syncwarp();
            if (lane < rest) evq[warp][lane] = keep;
            __syncwarp();
            npend = rest;
          }
        }
        evaluate(npend);
      }
      };  // phase1
      if (!cur_over) {
        if (wide) phase1(std::true_type{});
        else phase1(std::false_type{});
        cur_over = n_ent > kECap;
      }
      if constexpr (kBounds) {
        if (!cur_over) {  // each ray's first / last entry with a set bit, by shared atomics
          if (lane < kR) {
            s_efirst[warp][lane] = 0x7fffffff;
            s_elast[warp][lane] = -1;
          }
          __syncwarp();
          for (int e0 = 0; e0 < n_ent; e0 += 32) {
            const int e = e0 + lane;
            const uint32_t ent = e < n_ent ? T.ent[e] : 0u;
            if (ent & 0xFFFFu) {
              atomicMin(&s_efirst[warp][ent_j(ent)], e);
              atomicMax(&s_elast[warp][ent_j(ent)], e);
            }
          }
          __syncwarp();
          if (lane < kR && r_base + lane < n_rays) {
            float ta = 0.f, tb = 0.f;
            const int el = s_elast[warp][lane];
            if (el >= 0) {
              const uint32_t eF = T.ent[s_efirst[warp][lane]], eL = T.ent[el];
              const int kf = T.kr[lane].x + ent_k16(eF) + (__ffs(eF & 0xFFFFu) - 1);
              const int kl = T.kr[lane].x + ent_k16(eL) + (31 - __clz(eL & 0xFFFFu));
              float x, y;
              lattice_ends<kCone>(p, T.od[lane][0].w, tab, kf, ta, x);
              lattice_ends<kCone>(p, T.od[lane][0].w, tab, kl, y, tb);
              if (n_alive) atomicAdd(n_alive, 1ull);
            }
            t0[r_base + lane] = ta;
            t1[r_base + lane] = tb;
          }
        } else {  // an overflowed tile: traverse its rays
          for (int jj = 0; jj < kR; ++jj) {
            if (r_base + jj >= n_rays) break;
            const RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, t_min, t_max, r_base + jj);
            int kfirst = -1, klast = -1, kb0, ke0;
            traverse_ray<kCone, kSkip, kL1>(g, p, bits, mask2, M, mask3, s, hdr, tab, seglist[warp], kb0, ke0,
                                            [&](unsigned b, bool pred, int k, int32_t cnt) {
                                              if (b) {
                                                const int kf = __shfl_sync(kFull, k, __ffs(b) - 1);
                                                klast = __shfl_sync(kFull, k, 31 - __clz(b));
                                                if (kfirst < 0) kfirst = kf;
                                              }
                                            });
            if (lane == 0) {
              float ta = 0.f, tb = 0.f;
              if (klast >= 0) {
                float x, y;
                lattice_ends<kCone>(p, s.near_r, tab, kfirst, ta, x);
                lattice_ends<kCone>(p, s.near_r, tab, klast, y, tb);
                if (n_alive) atomicAdd(n_alive, 1ull);
              }
              t0[r_base + jj] = ta;
              t1[r_base + jj] = tb;
            }
          }
        }
        __syncwarp();
        continue;  // no look-back, no writer
      }
      if (cur_over) {  // count by direct traversal (phase 2 writes the same way)
        for (int jj = 0; jj < kR; ++jj) {
          if (r_base + jj >= n_rays) break;
          const RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, t_min, t_max, r_base + jj);
          int kb0, ke0;
          const int32_t c = traverse_ray<kCone, kSkip, kL1>(g, p, bits, mask2, M, mask3, s, hdr, tab, seglist[warp],
                                                            kb0, ke0, [](unsigned, bool, int, int32_t) {});
          if (lane == 0) T.cnt[jj] = c;
        }
        __syncwarp();
      }
      __syncwarp();
      cur_c = lane < kR ? T.cnt[lane] : 0;
      int agg = cur_c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(kFull, agg, o);
      cur_agg = agg;
      cur_ne = n_ent;
      lookback_publish(lb->status, tile, cur_agg);
      if (NACC_MARCH_STATS && lane == 0) MSTAT(7, 1);
    }
    if (prev_tile >= 0) {
      // ---------------- phase 2 of the previous tile (buffer buf ^ 1)
#if NACC_MARCH_NOLOOKBACK  // timing experiment only: every tile writes at offset 0 (wrong output)
      const long long excl = 0;
#else
      const long long excl = lookback_resolve(lb->status, prev_tile, prev_agg);
#endif
      if (prev_tile == n_tiles - 1 && lane == 0) {
        *total = excl + prev_agg;
        if (status_out) {
          int32_t stt = (excl + prev_agg > capacity) ? NACC_ERR_INSUFFICIENT_CAPACITY : NACC_OK;
          if (hdr && hdr->overflow) stt = NACC_ERR_UNSUPPORTED;
          *status_out = stt;
        }
      }
      tile_write<kCone, kSkip, kL1>(tb[warp][buf ^ 1], prev_ne, prev_over, prev_c, prev_tile, excl, prev_agg, g, p,
                                    bits, mask2, M, mask3, obox, rays_o, rays_d, t_min, t_max, n_rays, hdr, tab,
                                    packed_info, capacity, t0, t1, ray_id, seglist[warp], obase[warp]);
    }
    if (!have) break;
    prev_tile = tile;
    prev_c = cur_c;
    prev_ne = cur_ne;
    prev_agg = cur_agg;
    prev_over = cur_over;
    buf ^= 1;
  }
}

// ---------------------------------------------------------------- fill from a given packed_info
template <bool kCone, bool kSkip, bool kL1>
__global__ void __launch_bounds__(256) march_fill_kernel(GridConst g, MarchConst p, const uint32_t *__restrict__ bits,
                                                         const uint32_t *__restrict__ mask2, int M,
                                                         const uint32_t *__restrict__ mask3,
                                                         const float *__restrict__ obox,
                                                         const float *__restrict__ rays_o,
                                                         const float *__restrict__ rays_d,
                                                         const float *__restrict__ t_min,
                                                         const float *__restrict__ t_max, int64_t n_rays,
                                                         const ConeHeader *__restrict__ hdr,
                                                         const float *__restrict__ tab,
                                                         const int64_t *__restrict__ packed_info,
                                                         float *__restrict__ t0, float *__restrict__ t1,
                                                         int32_t *__restrict__ ray_id) {
  __shared__ int seglist[8][32];
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const int64_t out = packed_info[2 * r];
  const RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, t_min, t_max, r);
  int kb0, ke0;
  traverse_ray<kCone, kSkip, kL1>(g, p, bits, mask2, M, mask3, s, hdr, tab, seglist[threadIdx.x >> 5], kb0, ke0,
                                  [&](unsigned b, bool pred, int k, int32_t cnt) {
                                    if (pred) {
                                      const int64_t q = out + cnt + __popc(b & ((1u << lane) - 1u));
                                      float ta, tb;
                                      lattice_ends<kCone>(p, s.near_r, tab, k, ta, tb);
                                      t0[q] = ta;
                                      t1[q] = tb;
                                      ray_id[q] = (int32_t)r;
                                    }
                                  });
}

// ---------------------------------------------------------------- per-ray span (combined estimator)
// One warp per ray: the same traversal, keeping only the first and last
// emitted lattice index (reading #18).
template <bool kCone, bool kSkip, bool kL1>
__global__ void __launch_bounds__(128) march_bounds_kernel(
    GridConst g, MarchConst p, const uint32_t *__restrict__ bits, const uint32_t *__restrict__ mask2, int M,
    const uint32_t *__restrict__ mask3, const float *__restrict__ obox, const float *__restrict__ rays_o, const float *__restrict__ rays_d,
    const float *__restrict__ t_min, const float *__restrict__ t_max, int64_t n_rays,
    const ConeHeader *__restrict__ hdr, const float *__restrict__ tab, float *__restrict__ t_near,
    float *__restrict__ t_far, unsigned long long *__restrict__ n_alive) {
  __shared__ int seglist[4][32];
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rays) return;
  const RaySetup s = ray_setup(g, p, obox, rays_o, rays_d, t_min, t_max, r);
  int kfirst = -1, klast = -1, kb0, ke0;
  traverse_ray<kCone, kSkip, kL1>(g, p, bits, mask2, M, mask3, s, hdr, tab, seglist[threadIdx.x >> 5], kb0, ke0,
                                  [&](unsigned b, bool pred, int k, int32_t cnt) {
                                    if (b) {
                                      const int kf = __shfl_sync(kFull, k, __ffs(b) - 1);
                                      klast = __shfl_sync(kFull, k, 31 - __clz(b));
                                      if (kfirst < 0) kfirst = kf;
                                    }
                                  });
  if (lane == 0) {
    float ta = 0.f, tb = 0.f;
    if (klast >= 0) {
      float x, y;
      lattice_ends<kCone>(p, s.near_r, tab, kfirst, ta, x);
      lattice_ends<kCone>(p, s.near_r, tab, klast, y, tb);
      if (n_alive) atomicAdd(n_alive, 1ull);
    }
    t_near[r] = ta;
    t_far[r] = tb;
  }
}

// -------------------------------------------------------------------------- host
struct MarchWs {
  LookbackWs *lb;
  ConeHeader *hdr;
  float *tab;
};

static int64_t fused_tiles(int64_t n, bool cone, bool l1) { return ceil_div(n, (int64_t)tile_rays(cone, l1)); }

// persistent grid: every warp resident at once (look-back needs no more; the
// counter hands out tiles in order of arrival)
static unsigned fused_blocks(int64_t n_tiles, bool cone, bool skip, bool l1) {
  static int per_sm[8] = {0, 0, 0, 0, 0, 0, 0, 0}, n_sm = 0;
  const int v = (cone ? 4 : 0) | (skip ? 2 : 0) | (l1 ? 1 : 0);
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  if (per_sm[v] == 0) {
    const void *fn = nullptr;
    switch (v) {
      case 0: fn = (const void *)march_fused_kernel<false, false, false>; break;
      case 1: fn = (const void *)march_fused_kernel<false, false, true>; break;
      case 2: fn = (const void *)march_fused_kernel<false, true, false>; break;
      case 3: fn = (const void *)march_fused_kernel<false, true, true>; break;
      case 4: fn = (const void *)march_fused_kernel<true, false, false>; break;
      case 5: fn = (const void *)march_fused_kernel<true, false, true>; break;
      case 6: fn = (const void *)march_fused_kernel<true, true, false>; break;
      default: fn = (const void *)march_fused_kernel<true, true, true>; break;
    }
    // experiment hooks: NACC_MARCH_CARVEOUT (% of the unified L1/shared array given to shared
    // memory) and NACC_MARCH_BPS (resident blocks per SM)
    if (const char *e = getenv("NACC_MARCH_CARVEOUT"))
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e));
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kFWarps * 32, 0);
    if (const char *e = getenv("NACC_MARCH_BPS")) b = atoi(e) < b ? atoi(e) : b;
    per_sm[v] = b > 0 ? b : 1;
  }
  const int64_t want = ceil_div(n_tiles, (int64_t)kFWarps);
  const int64_t cap = (int64_t)per_sm[v] * (n_sm > 0 ? n_sm : 1);
  return (unsigned)(want < cap ? want : cap);
}

static size_t march_ws_layout(const nacc_grid &g, const nacc_march &p, int64_t n, MarchWs *w, void *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  const size_t o_lb = take(8 + 8 * (size_t)fused_tiles(n, p.cone_angle > 0.0f, g.levels == 1));
  size_t o_hdr = 0, o_tab = 0;
  const bool cone = p.cone_angle > 0.0f;
  if (cone) {
    o_hdr = take(sizeof(ConeHeader));
    o_tab = take((size_t)(kConeTableMax + 1) * 4);
  }
  if (w && base) {
    char *b = static_cast<char *>(base);
    w->lb = reinterpret_cast<LookbackWs *>(b + o_lb);
    w->hdr = cone ? reinterpret_cast<ConeHeader *>(b + o_hdr) : nullptr;
    w->tab = cone ? reinterpret_cast<float *>(b + o_tab) : nullptr;
  }
  return off;
}

static nacc_status validate(const nacc_grid *grid, const uint32_t *bits, const nacc_march *p,
                            const float *rays_o, const float *rays_d, const float *t_min,
                            int64_t n_rays, void *ws, size_t ws_bytes) {
  NACC_REQUIRE(grid && p, "grid and params must be non-NULL");
  NACC_REQUIRE(grid->levels >= 1 && grid->levels <= 8, "levels must be in 1..8");
  NACC_REQUIRE(grid->res >= 1, "res must be >= 1");
  NACC_REQUIRE((int64_t)grid->levels * grid->res * grid->res * grid->res < (1ll << 31),
               "levels*res^3 must be < 2^31");
  for (int a = 0; a < 3; ++a)
    NACC_REQUIRE(std::isfinite(grid->roi[a]) && std::isfinite(grid->roi[3 + a]) &&
                     grid->roi[a] < grid->roi[3 + a],
                 "roi must be finite with lo < hi");
  NACC_REQUIRE(std::isfinite(p->step) && p->step > 0.0f, "step must be > 0 and finite");
  NACC_REQUIRE(p->cone_angle >= 0.0f && std::isfinite(p->cone_angle), "cone_angle must be >= 0");
  NACC_REQUIRE(!(p->cone_angle > 0.0f) || (p->max_step >= p->step), "max_step must be >= step");
  NACC_REQUIRE(std::isfinite(p->near_plane) && !std::isnan(p->far_plane), "near/far must be numbers");
  NACC_REQUIRE(n_rays >= 0 && n_rays < (1ll << 31), "n_rays must be in [0, 2^31)");
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(bits && rays_o && rays_d, "bits, rays_o, rays_d must be non-NULL");
  NACC_REQUIRE(aligned(bits, 4) && aligned(rays_o, 4) && aligned(rays_d, 4), "arrays must be 4-byte aligned");
  NACC_REQUIRE(ws && ws_bytes >= nacc_sampling_occgrid_workspace_bytes(grid, p, n_rays),
               "workspace too small");
  if (p->cone_angle > 0.0f && (t_min || p->stratified)) return NACC_ERR_UNSUPPORTED;
  return NACC_OK;
}

static MarchConst make_march_const(const nacc_march &p) {
  MarchConst m;
  m.near_plane = p.near_plane;
  m.far_plane = p.far_plane;
  m.step = p.step;
  m.max_step = p.max_step;
  m.cone = p.cone_angle;
  m.inv_step = 1.0f / p.step;
  m.stratified = p.stratified;
  m.key0 = (uint32_t)(p.seed & 0xffffffffu);
  m.key1 = (uint32_t)(p.seed >> 32);
  return m;
}

#define NACC_DISPATCH3(KERNEL, GRID, BLOCK, STREAM, ...)                                         \
  do {                                                                                           \
    if (cone && skip && l1) KERNEL<true, true, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);     \
    else if (cone && skip) KERNEL<true, true, false><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);     \
    else if (cone && l1) KERNEL<true, false, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);       \
    else if (cone) KERNEL<true, false, false><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);            \
    else if (skip && l1) KERNEL<false, true, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);       \
    else if (skip) KERNEL<false, true, false><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);            \
    else if (l1) KERNEL<false, false, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);              \
    else KERNEL<false, false, false><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);                     \
  } while (0)

// the fused kernel in bounds mode
#define NACC_DISPATCH3B(KERNEL, GRID, BLOCK, STREAM, ...)                                              \
  do {                                                                                                 \
    if (cone && skip && l1) KERNEL<true, true, true, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);     \
    else if (cone && skip) KERNEL<true, true, false, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);     \
    else if (cone && l1) KERNEL<true, false, true, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);       \
    else if (cone) KERNEL<true, false, false, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);            \
    else if (skip && l1) KERNEL<false, true, true, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);       \
    else if (skip) KERNEL<false, true, false, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);            \
    else if (l1) KERNEL<false, false, true, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);              \
    else KERNEL<false, false, false, true><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);                     \
  } while (0)
#ifndef NACC_MARCH_FUSED_BOUNDS
#define NACC_MARCH_FUSED_BOUNDS 2  // build parameter: ray bounds from the fused kernel's phase 1 (0: one warp per ray,
                                   // 1: single-level grids, 2: every grid)
#endif

enum MarchMode { kModeFused = 0, kModeFill = 1, kModeBounds = 2 };

static nacc_status launch_march(int mode, const nacc_grid *grid, const uint32_t *bits,
                                const nacc_march *params, const float *rays_o, const float *rays_d,
                                const float *t_min, const float *t_max, int64_t n_rays,
                                int64_t *packed_info, float *t0, float *t1, int32_t *ray_id,
                                int64_t capacity, int64_t *total, int32_t *status_out, void *ws,
                                cudaStream_t stream, unsigned long long *n_alive = nullptr) {
  MarchWs w;
  march_ws_layout(*grid, *params, n_rays, &w, ws);
  const GridConst g = make_grid_const(*grid);
  const MarchConst p = make_march_const(*params);
  const bool cone = params->cone_angle > 0.0f;
  const bool skip = grid_skip_enabled(*grid);
  const bool l1 = grid->levels == 1;
  const int M = grid->res / kMacro;
  // built by nacc_grid_prepare / nacc_occgrid_update (gridaux.cu)
  const uint32_t *mask2 = bits + grid_mask2_offset_words(*grid);
  // fine dilated mask (single level; build option NACC_MARCH_FINEMASK, 0 = macro test only)
  const uint32_t *mask3 =
      (NACC_MARCH_FINEMASK && grid_fine_mask_enabled(*grid)) ? bits + grid_mask3_offset_words(*grid) : nullptr;
  const float *obox = reinterpret_cast<const float *>(bits + grid_aux_offset_words(*grid) + kAuxBoxWord);
  if (cone) {  // shared cone lattice table (reading #5)
    NACC_CUDA(cudaMemsetAsync(w.hdr, 0, sizeof(ConeHeader), stream));
    cone_tcap_kernel<<<grid_for(n_rays, 256), 256, 0, stream>>>(g, p, obox, rays_o, rays_d, t_max, n_rays, w.hdr);
    cone_table_kernel<<<1, 32, 0, stream>>>(p, w.hdr, w.tab);
    count_launch(2);
    NACC_CHECK_LAUNCH();
  }
  // the fused kernel's phase 1 (CFG2 182.7 -> 117.7 us, CFG3 1.96 -> 1.89 ms with 384-entry buffers)
  if (mode == kModeBounds && NACC_MARCH_FUSED_BOUNDS && (l1 || NACC_MARCH_FUSED_BOUNDS == 2)) {  // t0/t1: t_near/t_far
    if (n_alive) NACC_CUDA(cudaMemsetAsync(n_alive, 0, sizeof(unsigned long long), stream));
    const int64_t n_tiles = fused_tiles(n_rays, cone, l1);
    NACC_CUDA(cudaMemsetAsync(w.lb, 0, 8, stream));  // the tile counter
    NACC_DISPATCH3B(march_fused_kernel, fused_blocks(n_tiles, cone, skip, l1), kFWarps * 32, stream, g, p, bits,
                    mask2, M, mask3, obox, rays_o, rays_d, t_min, t_max, n_rays, n_tiles, w.hdr, w.tab, w.lb,
                    nullptr, nullptr, 0, nullptr, t0, t1, nullptr, n_alive);
  } else if (mode == kModeBounds) {  // t0 / t1 carry t_near / t_far
    if (n_alive) NACC_CUDA(cudaMemsetAsync(n_alive, 0, sizeof(unsigned long long), stream));
    NACC_DISPATCH3(march_bounds_kernel, (unsigned)grid_for(n_rays * 32, 128), 128, stream, g, p, bits, mask2, M, mask3,
                   obox, rays_o, rays_d, t_min, t_max, n_rays, w.hdr, w.tab, t0, t1, n_alive);
  } else if (mode == kModeFused) {
    const int64_t n_tiles = fused_tiles(n_rays, cone, l1);
    NACC_CUDA(cudaMemsetAsync(w.lb, 0, 8 + 8 * (size_t)n_tiles, stream));
    NACC_DISPATCH3(march_fused_kernel, fused_blocks(n_tiles, cone, skip, l1), kFWarps * 32, stream, g, p, bits,
                   mask2, M, mask3, obox, rays_o, rays_d, t_min, t_max, n_rays, n_tiles, w.hdr, w.tab, w.lb,
                   packed_info, total, capacity, status_out, t0, t1, ray_id);
  } else {
    NACC_DISPATCH3(march_fill_kernel, (unsigned)grid_for(n_rays * 32, 256), 256, stream, g, p, bits, mask2, M, mask3,
                   obox, rays_o, rays_d, t_min, t_max, n_rays, w.hdr, w.tab, packed_info, t0, t1, ray_id);
  }
  count_launch(1);
  NACC_CHECK_LAUNCH();
  return NACC_OK;
}

}  // namespace nacc

using namespace nacc;

extern "C" {

size_t nacc_sampling_occgrid_workspace_bytes(const nacc_grid *grid, const nacc_march *params,
                                             int64_t n_rays) {
  if (!grid || !params || n_rays < 0) return 0;
  return march_ws_layout(*grid, *params, n_rays, nullptr, nullptr);
}

nacc_status nacc_sampling_occgrid(const nacc_grid *grid, const uint32_t *bits, const nacc_march *params,
                                  const float *rays_o, const float *rays_d, const float *t_min,
                                  const float *t_max, int64_t n_rays, int64_t *packed_info, float *t0,
                                  float *t1, int32_t *ray_id, int64_t capacity, int64_t *total,
                                  int32_t *status_out, void *ws, size_t ws_bytes, cudaStream_t stream) {
  clear_error();
  nacc_status st = validate(grid, bits, params, rays_o, rays_d, t_min, n_rays, ws, ws_bytes);
  if (st != NACC_OK) return st;
  NACC_REQUIRE(total && capacity >= 0, "total must be non-NULL and capacity >= 0");
  if (n_rays == 0) {
    NACC_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), stream));
    if (status_out) NACC_CUDA(cudaMemsetAsync(status_out, 0, sizeof(int32_t), stream));
    return NACC_OK;
  }
  NACC_REQUIRE(packed_info && aligned(packed_info, 16), "packed_info must be non-NULL and 16-byte aligned");
  NACC_REQUIRE((!t0 && !t1 && !ray_id) || (t0 && t1 && ray_id), "t0, t1, ray_id: all or none");
  NACC_DEBUG_CHECK(debug_check_rays(rays_d, n_rays, stream));
  return launch_march(kModeFused, grid, bits, params, rays_o, rays_d, t_min, t_max, n_rays, packed_info, t0, t1,
                      ray_id, capacity, total, status_out, ws, stream);
}

nacc_status nacc_sampling_occgrid_fill(const nacc_grid *grid, const uint32_t *bits, const nacc_march *params,
                                       const float *rays_o, const float *rays_d, const float *t_min,
                                       const float *t_max, int64_t n_rays, const int64_t *packed_info,
                                       float *t0, float *t1, int32_t *ray_id, void *ws, size_t ws_bytes,
                                       cudaStream_t stream) {
  clear_error();
  nacc_status st = validate(grid, bits, params, rays_o, rays_d, t_min, n_rays, ws, ws_bytes);
  if (st != NACC_OK) return st;
  if (n_rays == 0) return NACC_OK;
  NACC_REQUIRE(packed_info && t0 && t1 && ray_id, "packed_info, t0, t1, ray_id must be non-NULL");
  NACC_DEBUG_CHECK(debug_check_rays(rays_d, n_rays, stream));
  // the cone table lives in the workspace; it is rebuilt here
  return launch_march(kModeFill, grid, bits, params, rays_o, rays_d, t_min, t_max, n_rays,
                      const_cast<int64_t *>(packed_info), t0, t1, ray_id, 0, nullptr, nullptr, ws, stream);
}

nacc_status nacc_occgrid_ray_bounds(const nacc_grid *grid, const uint32_t *bits, const nacc_march *params,
                                   const float *rays_o, const float *rays_d, const float *t_min,
                                   const float *t_max, int64_t n_rays, float *t_near, float *t_far,
                                   uint64_t *n_alive, void *ws, size_t ws_bytes, cudaStream_t stream) {
  clear_error();
  nacc_status st = validate(grid, bits, params, rays_o, rays_d, t_min, n_rays, ws, ws_bytes);
  if (st != NACC_OK) return st;
  if (n_rays == 0) {
    if (n_alive) NACC_CUDA(cudaMemsetAsync(n_alive, 0, sizeof(uint64_t), stream));
    return NACC_OK;
  }
  NACC_REQUIRE(t_near && t_far && aligned(t_near, 4) && aligned(t_far, 4), "t_near and t_far must be non-NULL");
  return launch_march(kModeBounds, grid, bits, params, rays_o, rays_d, t_min, t_max, n_rays, nullptr, t_near, t_far,
                      nullptr, 0, nullptr, nullptr, ws, stream, reinterpret_cast<unsigned long long *>(n_alive));
}

#if NACC_MARCH_STATS
// debug build only: read and reset the segment counters (g_march_stats above)
void nacc_debug_march_stats(unsigned long long *out18) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out18, g_march_stats, 18 * sizeof(unsigned long long));
  const unsigned long long z[18] = {};
  cudaMemcpyToSymbol(g_march_stats, z, sizeof(z));
}
#endif

#if NACC_LB_STATS
// debug build only: read and reset the look-back counters (resolves, polls, sleeping polls, tiles walked)
void nacc_debug_lb_stats(unsigned long long *out4) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out4, g_lb_stats, 4 * sizeof(unsigned long long));
  const unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_lb_stats, z, sizeof(z));
}
#endif

}  // extern "C"
