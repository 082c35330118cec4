// Render record layout shared by the forward and backward rasterizer passes.
//
// The record is the B200 counterpart of rasterizer.RasterRecord
// (rasterizer.py:64-91): instead of per-tile [G,256] float64 alpha matrices
// (15 GB at 200k Gaussians) it keeps O(K + pairs + pixels) state and the
// backward pass recomputes alphas from the projected Gaussians.
#pragma once
#include "common.cuh"
#include "scan_sort.cuh"

namespace fs4d {

constexpr int kTile = 16;
constexpr int kTilePixels = kTile * kTile;
constexpr int kHistTilesSmem = 6144;  // per-block shared histogram capacity (24 KB)
constexpr float kQSkip = 11.0825270270270f;  // 2 ln 255 (rasterizer.py:212)

// The forward blend and the backward replay evaluate a Gaussian at a pixel the
// same way: exp(-q/2) = 2^power with power = a' dx^2 + b' dx dy + c' dy^2 for
// the conic pre-scaled once per staged Gaussian (a' = -log2(e)/2 a, b' =
// -log2(e) b, c' = -log2(e)/2 c), and q > 2 ln 255 <=> power < kPowSkip.
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kPowSkip = -0.5f * kLog2e * kQSkip;
__device__ __forceinline__ float4 scaled_conic(const float4& co) {
  return make_float4(-0.5f * kLog2e * co.x, -kLog2e * co.y, -0.5f * kLog2e * co.z, co.w);
}
// back to (a, b, c, opacity) up to a few ulps -- for the conservative strip cull only
__device__ __forceinline__ float4 unscaled_conic(const float4& cs) {
  return make_float4(cs.x * (-2.f / kLog2e), cs.y * (-1.f / kLog2e), cs.z * (-2.f / kLog2e), cs.w);
}
// The projected mean is kept as fp32 hi + lo (u = hi + lo to ~1e-12 px) and
// staged relative to the tile origin (ox, oy): the per-pair offsets
// dx = (col - ox) - m.x are then exact to ~1e-6 px, where a single fp32 u
// carries half an ulp of error (3e-5 px at u ~ 640) into every alpha.  The
// forward blend, the backward replay and the tile-alpha replay all use it.
__device__ __forceinline__ float2 tile_rel_mean(const float4& m, float ox, float oy) {
  return make_float2((m.x - ox) + m.z, (m.y - oy) + m.w);
}
// explicit rounding: every kernel that evaluates a pair (forward blend,
// backward replay, tile-alpha replay) gets the same bits, whatever FMA
// contraction the compiler would pick in each context
__device__ __forceinline__ float gauss_power(const float4& cs, float dx, float dy) {
  float p = __fmul_rn(__fmul_rn(cs.x, dx), dx);
  p = __fmaf_rn(__fmul_rn(cs.y, dx), dy, p);
  return __fmaf_rn(__fmul_rn(cs.z, dy), dy, p);
}
// 1/x to ~1 ulp (MUFU.RCP, no IEEE-division slow path).  The backward replay
// recovers T_exc = T / (1 - alpha) with it; 1 - alpha lies in [0.01, 1).
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct RenderLayout {
  int64_t K = 0, cap = 0;
  int H = 0, W = 0, D = 0, ntx = 0, nty = 0, ntiles = 0, tile_bits = 0, acc_stride = 0;
  int depth_final = 0;
  // per Gaussian (source-indexed): projected record, fp64 depth, depth-sort
  // keys/values (the global order is only materialised for export/backward)
  size_t xy, conic_o, pix_rect, tile_rect, rgbz, cov_r, z64, dkeys0, dkeys1, dvals0, dvals1, rank_of, clamp_mask;
  size_t dtable;  // depth-ordered binning: per (256-Gaussian block, tile) counts / slots
  // tiles: counts, append cursors, segment offsets, [start, end) ranges
  size_t tcnt, tcur, toff64, ranges, tperm;
  // pairs: 64-bit (depth bits, source index) keys and the sorted source indices
  size_t pkey64, pvals0;
  // pixels
  size_t tfinal, last;
  // counters and scratch
  size_t counters, scratch, scratch_bytes;
  // backward accumulators [K, acc_stride]
  size_t accum;
  size_t total;
};

// counters (uint32 words at layout.counters)
enum { CNT_VISIBLE = 0, CNT_PAIRS64 = 2 /* u64 at words 2..3 */, CNT_PAIRS_CLAMPED = 4, CNT_BIG_TILES = 5, CNT_WORDS = 8 };

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Conservative warp-level cull: can any pixel of the NR-row strip [r0, r0+NR) x
// [c0, c0+15] pass the per-pixel tests (inside pix_rect, q <= 2 ln 255,
// o exp(-q/2) >= alpha_skip)?  Row by row, q(dx) is a parabola with minimum
// (c - b^2/a) dy^2 at dx* = -b dy / a, so the admissible columns are
// mu_x + dx* +- sqrt((Q - q_min)/a) with Q = min(2 ln 255, 2 ln(o/skip)).
// Q gets a 1e-3 relative and the column interval a 0.02 pixel margin, far
// above the fp32 rounding of either side, so no Gaussian the exact per-pixel
// test accepts is ever culled: the pixel decisions stay exactly k_blend's.
// The per-Gaussian constants of the strip cull below, computed once when the
// Gaussian is staged instead of by every warp that tests it: (Q, 1/a,
// c - b^2/a, b/a) of the conic (a, b, c) and opacity; Q < 0 marks a Gaussian
// whose opacity is below alpha_skip (it hits nothing).
__device__ __forceinline__ float4 strip_consts(const float4& co, float alpha_skip) {
  if (co.w < alpha_skip) return make_float4(-1.f, 0.f, 0.f, 0.f);
  const float Q = fminf(kQSkip, 2.f * __logf(co.w * fast_rcp(alpha_skip))) * 1.001f + 1e-3f;
  const float inv_a = fast_rcp(co.x);
  return make_float4(Q, inv_a, co.z - co.y * co.y * inv_a, co.y * inv_a);
}
template <int NR>
__device__ __forceinline__ bool strip_hits_c(const int4& pr, const float2& mm, const float4& sc, int r0, int c0) {
  const float xlo = (float)max(c0, pr.x) - 0.02f, xhi = (float)min(c0 + kTile - 1, pr.y) + 0.02f;
  bool hit = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int row = r0 + r;
    if (row < pr.z || row > pr.w) continue;
    const float dy = (float)row - mm.y;
    const float qmin = sc.z * dy * dy;
    if (!(qmin <= sc.x)) continue;
    const float h = fast_sqrt((sc.x - qmin) * sc.y) + 0.02f;
    const float xc = mm.x - sc.w * dy;
    const float lo = fmaxf(xc - h, xlo), hi = fminf(xc + h, xhi);
    hit |= ceilf(lo) <= floorf(hi);
  }
  return hit;
}

template <int NR>
__device__ __forceinline__ bool strip_hits(const int4& pr, const float2& mm, const float4& co, int r0, int c0,
                                           float alpha_skip) {
  if (co.w < alpha_skip) return false;
  // approximate rcp / sqrt / log (~1e-6 relative): far inside the margins
  const float Q = fminf(kQSkip, 2.f * __logf(co.w * fast_rcp(alpha_skip))) * 1.001f + 1e-3f;
  const float inv_a = fast_rcp(co.x), schur = co.z - co.y * co.y * inv_a;
  const float xlo = (float)max(c0, pr.x) - 0.02f, xhi = (float)min(c0 + kTile - 1, pr.y) + 0.02f;
  bool hit = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int row = r0 + r;
    if (row < pr.z || row > pr.w) continue;
    const float dy = (float)row - mm.y;
    const float qmin = schur * dy * dy;
    if (qmin > Q) continue;
    const float h = fast_sqrt((Q - qmin) * inv_a) + 0.02f;
    const float xc = mm.x - co.y * dy * inv_a;
    const float lo = fmaxf(xc - h, xlo), hi = fminf(xc + h, xhi);
    hit |= ceilf(lo) <= floorf(hi);
  }
  return hit;
}


inline RenderLayout make_layout(const Fs4dRecordInfo& info) {
  RenderLayout L;
  L.K = info.K;
  L.cap = info.pair_capacity;
  L.H = info.height;
  L.W = info.width;
  L.D = info.D;
  L.ntx = (int)ceil_div(L.W, kTile);
  L.nty = (int)ceil_div(L.H, kTile);
  L.ntiles = L.ntx * L.nty;
  int bits = 0;
  while ((1ll << bits) < (int64_t)L.ntiles) ++bits;
  L.tile_bits = bits;
  // ping-pong parity after the radix passes over 32-bit depth keys
  L.depth_final = (int)(ceil_div(32, kMaxRadixBits) & 1);
  L.acc_stride = (int)ceil_div(10 + L.D, 32) * 32;
  const int64_t K = L.K > 0 ? L.K : 1;
  const int64_t cap = L.cap > 0 ? L.cap : 1;
  const int64_t npix = (int64_t)L.H * L.W > 0 ? (int64_t)L.H * L.W : 1;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.xy = take(K * 16);
  L.conic_o = take(K * 16);
  L.pix_rect = take(K * 16);
  L.tile_rect = take(K * 16);
  L.rgbz = take(K * 16);
  L.cov_r = take(K * 16);
  L.z64 = take(K * 8);
  L.dkeys0 = take(K * 4);
  L.dkeys1 = take(K * 4);
  L.dvals0 = take(K * 4);
  L.dvals1 = take(K * 4);
  L.rank_of = take(K * 4);
  L.clamp_mask = take(K * 4);
  const int64_t nt = L.ntiles > 0 ? L.ntiles : 1;
  L.tcnt = take(nt * 4);
  L.tcur = take(nt * 4);
  L.toff64 = take(nt * 8);
  L.ranges = take(nt * 8);
  L.tperm = take(nt * 4);  // tiles by decreasing pair count (CTA launch order)
  L.pkey64 = take(cap * 8);
  L.dtable = take((size_t)((K + 255) / 256) * nt * 4);
  L.pvals0 = take(cap * 4);
  L.tfinal = take(npix * 4);
  L.last = take(npix * 4);
  L.counters = take(CNT_WORDS * 4);
  size_t s1 = scan_scratch_bytes(K > nt ? K : nt), s2 = radix_scratch_bytes(K);
  L.scratch_bytes = s1 > s2 ? s1 : s2;
  L.scratch = take(L.scratch_bytes);
  L.accum = take((size_t)K * L.acc_stride * 4);
  L.total = o;
  return L;
}

template <typename T>
__host__ __device__ inline T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + off);
}

// binning.cu: per-tile pair segments sorted by (depth, index) -> ranges + pvals0
void bin_tiles_device(const RenderLayout& L, void* ws, const int4* tile_rect, const uint32_t* dkeys,
                      const double* z64, uint32_t* counters, int32_t* status, cudaStream_t s);
// render_fwd.cu: global stable depth order of the visible set (export / backward)
const uint32_t* depth_order(const RenderLayout& L, void* ws, cudaStream_t s, bool with_rank = true);

}  // namespace fs4d
