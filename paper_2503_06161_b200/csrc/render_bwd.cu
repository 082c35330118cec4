// Backward rasterizer: per-tile back-to-front replay + projection chain.
//
// Reference: rasterizer.render_backward (rasterizer.py:320-452) and
// gaussians.covariance_backward / rotmat_backward / normalize_backward
// (gaussians.py:156-218).
//   k_blend_bwd       tile loop  rasterizer.py:349-393  (fp32, warp butterfly
//                     reduction + one coalesced red.global per warp/Gaussian)
//   k_preprocess_bwd  projection chain rasterizer.py:395-451 (fp64)
#include <stdlib.h>

#include "render_common.cuh"
#include "scan_sort.cuh"
#include "sh.cuh"

namespace fs4d {

struct BwdArgs {
  int H, W, ntx, D, acc_stride, nvals;
  float alpha_cap, alpha_skip, stop;
  float bg0, bg1, bg2;
  const uint2* ranges;
  const int32_t* tperm;  // tiles by decreasing pair count (from the forward record), or null
  const uint32_t* pvals;
  const float4* xy;  // (u hi, v hi, u lo, v lo)
  const float4* conic_o;
  const int4* pix_rect;
  const float4* rgbz;
  const float* features;
  const float* tfinal;
  const int32_t* last;
  const float* dC;
  const float* dD;
  const float* dF;
  const float* dA;
  float* accum;
  float* part;  // deterministic mode: per (pair, row-split CTA) partial sums [cap][SUBB][nvals]
};

// Reduce v[0..31] over the warp; afterwards lane L holds the warp sum of v[L].
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < n / 2; ++k) {
      float send = upper ? v[k] : v[k + n / 2];
      float keep = upper ? v[k + n / 2] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// Per-Gaussian warp sum of NROW*2 (<= 32) lane values through shared memory:
// lane l stores (v[2m], v[2m+1]) at row m, then lane 2m+h sums value 2m+h over
// lanes 16h..16h+15 with 8 LDS.128 + FADD2s and adds its partner's half with
// one shuffle.  ~40 instructions against ~124 (SHFL + 2 SEL + FADD per step)
// for the register transpose.  Row stride 68 words and the h-rotated read
// order keep both the STS.64 and LDS.128 phases bank-conflict free.
// Returns the sum of value `lane` (lanes >= 2*NROW: 0).
constexpr int kRedRowStride = 68;
template <int NROW>
__device__ __forceinline__ float warp_smem_reduce(const float (&v)[2 * NROW], float* wred, int lane) {
  __syncwarp();
#pragma unroll
  for (int m = 0; m < NROW; ++m)
    *reinterpret_cast<float2*>(wred + m * kRedRowStride + 2 * lane) = make_float2(v[2 * m], v[2 * m + 1]);
  __syncwarp();
  const int h = lane & 1;
  float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
  if (lane < 2 * NROW) {
    const float* row = wred + (lane >> 1) * kRedRowStride + 32 * h;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 q = *reinterpret_cast<const float4*>(row + 4 * ((j + 4 * h) & 7));
      acc = __fadd2_rn(acc, make_float2(q.x, q.y));
      acc2 = __fadd2_rn(acc2, make_float2(q.z, q.w));
    }
    acc = __fadd2_rn(acc, acc2);
  }
  const float keep = h ? acc.y : acc.x, send = h ? acc.x : acc.y;
  return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

template <int DC>
__global__ void __launch_bounds__(kTilePixels) k_blend_bwd(BwdArgs a) {
  constexpr int B = DC >= 64 ? 128 : kTilePixels;  // Gaussians staged per batch
  __shared__ float2 s_xy[B];
  __shared__ float4 s_co[B];
  __shared__ int4 s_pr[B];
  __shared__ float4 s_rgbz[B];
  __shared__ uint32_t s_g[B];
  __shared__ __align__(16) float s_f[DC > 0 ? B * DC : 1];
  __shared__ int s_maxlast;

  const int tile = a.tperm ? a.tperm[blockIdx.x] : blockIdx.x;
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  const int col = tx * kTile + (threadIdx.x & (kTile - 1));
  const int row = ty * kTile + (threadIdx.x / kTile);
  const int lane = threadIdx.x & 31;
  const bool inside = col < a.W && row < a.H;
  const uint2 rg = a.ranges[tile];
  if (rg.y <= rg.x) return;
  const int64_t pix = (int64_t)row * a.W + col;
  const float ox = (float)(tx * kTile), oy = (float)(ty * kTile);  // tile origin (tile_rel_mean)
  const float fc = (float)(col - tx * kTile), fr = (float)(row - ty * kTile);

  float T = 1.f, Tfin = 1.f;
  int lastj = -1;
  float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, dd = 0.f, da = 0.f;
  float df[DC > 0 ? DC : 1];
#pragma unroll
  for (int c = 0; c < (DC > 0 ? DC : 1); ++c) df[c] = 0.f;
  if (inside) {
    T = Tfin = a.tfinal[pix];
    lastj = a.last[pix];
    if (a.dC) { dc0 = a.dC[3 * pix]; dc1 = a.dC[3 * pix + 1]; dc2 = a.dC[3 * pix + 2]; }
    if (a.dD) dd = a.dD[pix];
    if (a.dA) da = a.dA[pix];
    if (DC > 0 && a.dF) {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (c < a.D) df[c] = a.dF[pix * a.D + c];
    }
  }
  const float vpix = dc0 * a.bg0 + dc1 * a.bg1 + dc2 * a.bg2 - da;  // dL/dT_final
  float suffix = 0.f;

  if (threadIdx.x == 0) s_maxlast = -1;
  __syncthreads();
  atomicMax(&s_maxlast, lastj);
  __syncthreads();
  const int maxlast = s_maxlast;
  if (maxlast < (int)rg.x) return;
  const int wlast = __reduce_max_sync(0xffffffffu, lastj);
  const int wrow0 = ty * kTile + (threadIdx.x >> 5) * 2;  // this warp's two pixel rows
  const int tcol0 = tx * kTile;

  const int nv = a.nvals;
  const uint32_t hi = (uint32_t)(maxlast + 1) < rg.y ? (uint32_t)(maxlast + 1) : rg.y;
  for (int64_t bend = hi; bend > (int64_t)rg.x; bend -= B) {
    const int64_t bstart = bend - B > (int64_t)rg.x ? bend - B : (int64_t)rg.x;
    const int cnt = (int)(bend - bstart);
    __syncthreads();
    if ((int)threadIdx.x < cnt) {
      const uint32_t g = a.pvals[bstart + threadIdx.x];
      s_g[threadIdx.x] = g;
      s_xy[threadIdx.x] = tile_rel_mean(a.xy[g], ox, oy);
      s_co[threadIdx.x] = a.conic_o[g];
      s_pr[threadIdx.x] = a.pix_rect[g];
      s_rgbz[threadIdx.x] = a.rgbz[g];
      if (DC > 0) {
        const float* src = a.features + (int64_t)g * a.D;
        float* dst = s_f + threadIdx.x * DC;
        for (int c = 0; c < DC; ++c) dst[c] = c < a.D ? src[c] : 0.f;
      }
    }
    __syncthreads();
    // warp-level culling (as in k_blend): keep the staged Gaussians whose
    // pixel rectangle meets this warp's two pixel rows and that lie at or
    // before the warp's last contributor, then walk them back to front
#pragma unroll 1
    for (int m = (cnt - 1) / 32; m >= 0; --m) {
     unsigned bits;
     {
      const int kk = m * 32 + lane;
      bool hit = false;
      if (kk < cnt && bstart + kk <= (int64_t)wlast) {
        const int4 pr = s_pr[kk];
        hit = pr.w >= wrow0 && pr.z <= wrow0 + 1 && pr.y >= tcol0 && pr.x <= tcol0 + kTile - 1;
      }
      bits = __ballot_sync(0xffffffffu, hit);
     }
     while (bits) {
      const int bit = 31 - __clz(bits);
      bits &= ~(1u << bit);
      const int k = m * 32 + bit;
      const int64_t j = bstart + k;
      bool live = inside && j <= (int64_t)lastj;
      float v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = 0.f;
      float vf[DC > 0 ? DC : 1];
#pragma unroll
      for (int c = 0; c < (DC > 0 ? DC : 1); ++c) vf[c] = 0.f;
      if (live) {
        const int4 pr = s_pr[k];
        live = !(col < pr.x || col > pr.y || row < pr.z || row > pr.w);
      }
      float dx = 0.f, dy = 0.f, gv = 0.f, araw = 0.f, al = 0.f;
      float4 co = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live) {
        const float2 m = s_xy[k];
        co = s_co[k];
        dx = fc - m.x;
        dy = fr - m.y;
        const float pw = gauss_power(scaled_conic(co), dx, dy);  // same scaling as the forward's staging
        live = !(pw < kPowSkip);
        if (live) {
          gv = fast_exp2(pw);
          araw = co.w * gv;
          al = fminf(araw, a.alpha_cap);
          live = al >= a.alpha_skip;
        }
      }
      if (live) {
        const float4 cz = s_rgbz[k];
        const float om = 1.f - al;
        const float rom = fast_rcp(om);
        const float Texc = T * rom;
        const float w = al * Texc;
        float uval = cz.x * dc0 + cz.y * dc1 + cz.z * dc2 + cz.w * dd;
        if (DC > 0) {
          const float* f = s_f + k * DC;
#pragma unroll
          for (int c = 0; c < DC; ++c) {
            uval += f[c] * df[c];
            vf[c] = w * df[c];
          }
        }
        const float dal = uval * Texc - (suffix + Tfin * vpix) * rom;
        suffix += w * uval;
        T = Texc;
        const float dar = araw < a.alpha_cap ? dal : 0.f;
        const float dq = -0.5f * gv * dar * co.w;
        v[0] = w * dc0;
        v[1] = w * dc1;
        v[2] = w * dc2;
        v[3] = w * dd;
        v[4] = dar * gv;
        v[5] = dq * dx * dx;
        v[6] = dq * dx * dy;
        v[7] = dq * dy * dy;
        v[8] = -2.f * dq * (co.x * dx + co.y * dy);
        v[9] = -2.f * dq * (co.y * dx + co.z * dy);
      }
      if (!__any_sync(0xffffffffu, live)) continue;
      float* dst = a.accum + (int64_t)s_g[k] * a.acc_stride;
      // chunk 0: values 0..31 (10 fixed + first 22 feature channels)
#pragma unroll
      for (int c = 0; c < 22; ++c)
        if (c < DC) v[10 + c] = vf[c];
      {
        float r = warp_transpose_reduce(v, lane);
        if (lane < nv && r != 0.f) red_add(dst + lane, r);
      }
      // further chunks of 32 feature channels
#pragma unroll
      for (int base = 22; base < DC; base += 32) {
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = (base + c < DC) ? vf[base + c] : 0.f;
        float r = warp_transpose_reduce(v, lane);
        if (10 + base + lane < nv && r != 0.f) red_add(dst + 10 + base + lane, r);
      }
     }
    }
  }
}

// Same replay with PX vertically adjacent pixels per thread (256/PX threads
// per tile, a warp covers 2*PX pixel rows).  The per-Gaussian warp reduction
// -- the kernel's dominant cost -- is then shared by PX times as many pixels.
template <int SUBB>
__device__ __forceinline__ int ty_sub_rows(int sub) { return sub * (kTile / SUBB); }

// SUBB > 1 splits a tile's rows over SUBB CTAs (each replays the whole list
// for its 16/SUBB rows): CTAs of one or two warps have no cross-warp batch
// barrier to wait on, and more of them fit per SM.
// DET: instead of red.global.add, every warp leaves its per-Gaussian sums in
// shared memory, the CTA adds its warps in a fixed order at the end of each
// staged batch and stores one partial per (pair, CTA) -- k_det_gather then
// sums a Gaussian's partials in tile order: bitwise reproducible gradients.
// (an index prefetch + cp.async staging as in k_blend was measured equal at
// 8 CTAs/SM and slower unconstrained: 142 registers, 2.44 vs 1.96 ms / step)
template <int DC, int PX, int SUBB, bool DET = false>
#ifdef FS4D_BWD_MINB  // A/B knob: minimum resident CTAs per SM (caps registers)
__global__ void __launch_bounds__(kTilePixels / PX / SUBB, FS4D_BWD_MINB) k_blend_bwd2(BwdArgs a) {
#else
__global__ void __launch_bounds__(kTilePixels / PX / SUBB) k_blend_bwd2(BwdArgs a) {
#endif
  constexpr int NT = kTilePixels / PX / SUBB;
  constexpr int B = NT;  // Gaussians staged per batch
  constexpr int NF = DC > 0 ? DC : 1;
  constexpr int NVMAX = 10 + NF;
  __shared__ float s_acc[DET ? (NT / 32) * B * NVMAX : 1];
  // the staged batch as ONE shared array (reads of Gaussian k off one base
  // with immediate offsets, as in k_blend): 16-byte rows [5 + DC/4][B] --
  // conic + opacity, scaled conic (gauss_power, same evaluation as the
  // forward), pixel rectangle, rgb + depth, strip-cull constants (once per
  // staged Gaussian, not per warp), feature quads (channel-quad-
  // major) -- then the tile-relative means (8 B) and the source indices
  constexpr int kRows = 5 + (DC > 0 ? (DC + 3) / 4 : 0);
  __shared__ __align__(16) float4 s_stage[kRows * B + B / 2 + B / 4];
  float4* const s_co = s_stage;
  float4* const s_cs = s_stage + B;
  int4* const s_pr = reinterpret_cast<int4*>(s_stage + 2 * B);
  float4* const s_rgbz = s_stage + 3 * B;
  float4* const s_sc = s_stage + 4 * B;  // strip-cull constants (strip_consts)
  float4* const s_f4 = s_stage + 5 * B;
  float2* const s_xy = reinterpret_cast<float2*>(s_stage + kRows * B);
  uint32_t* const s_g = reinterpret_cast<uint32_t*>(s_stage + kRows * B + B / 2);
  constexpr int NROW = (10 + DC + 1) / 2;  // per-Gaussian values, in float2 rows
  __shared__ __align__(16) float s_red[NT / 32][NROW * kRedRowStride];
  __shared__ int s_maxlast;

  const int tile = a.tperm ? a.tperm[blockIdx.x / SUBB] : blockIdx.x / SUBB;
  const int rsub = ty_sub_rows<SUBB>(blockIdx.x % SUBB);
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  const int col = tx * kTile + (threadIdx.x & (kTile - 1));
  const int row0 = ty * kTile + rsub + (threadIdx.x / kTile) * PX;
  float* wred = s_red[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const uint2 rg = a.ranges[tile];
  if (rg.y <= rg.x) return;
  const float ox = (float)(tx * kTile), oy = (float)(ty * kTile);  // tile origin (tile_rel_mean)
  const float fc = (float)(col - tx * kTile);

  bool inside[PX];
  float T[PX], Tfin[PX], suffix[PX], vpix[PX], dc0[PX], dc1[PX], dc2[PX], dd[PX];
  int lastj[PX];
  float df[PX][NF];
  int mylast = -1;
#pragma unroll
  for (int p = 0; p < PX; ++p) {
    const int row = row0 + p;
    inside[p] = col < a.W && row < a.H;
    T[p] = Tfin[p] = 1.f;
    lastj[p] = -1;
    dc0[p] = dc1[p] = dc2[p] = dd[p] = 0.f;
    float dA = 0.f;
#pragma unroll
    for (int c = 0; c < NF; ++c) df[p][c] = 0.f;
    if (inside[p]) {
      const int64_t pix = (int64_t)row * a.W + col;
      T[p] = Tfin[p] = a.tfinal[pix];
      lastj[p] = a.last[pix];
      if (a.dC) {
        dc0[p] = a.dC[3 * pix];
        dc1[p] = a.dC[3 * pix + 1];
        dc2[p] = a.dC[3 * pix + 2];
      }
      if (a.dD) dd[p] = a.dD[pix];
      if (a.dA) dA = a.dA[pix];
      if (DC > 0 && a.dF) {
#pragma unroll
        for (int c = 0; c < NF; ++c)
          if (c < a.D) df[p][c] = a.dF[pix * a.D + c];
      }
    }
    vpix[p] = dc0[p] * a.bg0 + dc1[p] * a.bg1 + dc2[p] * a.bg2 - dA;  // dL/dT_final
    suffix[p] = 0.f;
    mylast = max(mylast, lastj[p]);
  }

  if (threadIdx.x == 0) s_maxlast = -1;
  __syncthreads();
  atomicMax(&s_maxlast, mylast);
  __syncthreads();
  const int maxlast = s_maxlast;
  const int nv = a.nvals;
  const uint32_t hi = (uint32_t)(maxlast + 1) < rg.y ? (uint32_t)(maxlast + 1) : rg.y;
  const int sidx = blockIdx.x % SUBB;
  if (DET) {  // pairs this CTA never stages (behind every pixel's last contributor): zero partials
    const uint32_t z0 = maxlast < (int)rg.x ? rg.x : hi;
    for (int64_t e = threadIdx.x; e < (int64_t)(rg.y - z0) * nv; e += NT)
      a.part[((int64_t)(z0 + e / nv) * SUBB + sidx) * nv + e % nv] = 0.f;
  }
  if (maxlast < (int)rg.x) return;
  const int wlast = __reduce_max_sync(0xffffffffu, mylast);
  const int wrow0 = ty * kTile + rsub + (threadIdx.x >> 5) * 2 * PX;  // this warp's 2*PX pixel rows
  const int tcol0 = tx * kTile;
  float* wacc = DET ? s_acc + (threadIdx.x >> 5) * B * NVMAX : nullptr;

  for (int64_t bend = hi; bend > (int64_t)rg.x; bend -= B) {
    const int64_t bstart = bend - B > (int64_t)rg.x ? bend - B : (int64_t)rg.x;
    const int cnt = (int)(bend - bstart);
    __syncthreads();
    if ((int)threadIdx.x < cnt) {
      const uint32_t g = a.pvals[bstart + threadIdx.x];
      s_g[threadIdx.x] = g;
      s_xy[threadIdx.x] = tile_rel_mean(a.xy[g], ox, oy);
      const float4 cog = a.conic_o[g];
      s_co[threadIdx.x] = cog;
      s_cs[threadIdx.x] = scaled_conic(cog);
      s_sc[threadIdx.x] = strip_consts(cog, a.alpha_skip);
      s_pr[threadIdx.x] = a.pix_rect[g];
      s_rgbz[threadIdx.x] = a.rgbz[g];
      if (DC > 0) {
        const float* src = a.features + (int64_t)g * a.D;
        if ((a.D & 3) == 0 && a.D >= DC) {
#pragma unroll
          for (int c = 0; c < DC; c += 4) s_f4[(c / 4) * B + threadIdx.x] = __ldg(reinterpret_cast<const float4*>(src + c));
        } else {
          for (int c = 0; c < DC; c += 4) {
            float q[4];
            for (int i = 0; i < 4; ++i) q[i] = c + i < a.D ? src[c + i] : 0.f;
            s_f4[(c / 4) * B + threadIdx.x] = make_float4(q[0], q[1], q[2], q[3]);
          }
        }
      }
    }
    __syncthreads();
    if (DET)
      for (int e = lane; e < cnt * NVMAX; e += 32) wacc[e] = 0.f;
#pragma unroll 1
    for (int m = (cnt - 1) / 32; m >= 0; --m) {
      unsigned bits;
      {
        const int kk = m * 32 + lane;
        bool hit = false;
        if (kk < cnt && bstart + kk <= (int64_t)wlast) {
          const int4 pr = s_pr[kk];
          hit = pr.w >= wrow0 && pr.z <= wrow0 + 2 * PX - 1 && pr.y >= tcol0 && pr.x <= tcol0 + kTile - 1;
          if (hit) {
            const float2 mr = s_xy[kk];
            hit = strip_hits_c<2 * PX>(pr, make_float2(mr.x + ox, mr.y + oy), s_sc[kk], wrow0, tcol0);
          }
        }
        bits = __ballot_sync(0xffffffffu, hit);
      }
      while (bits) {
        const int bit = 31 - __clz(bits);
        bits &= ~(1u << bit);
        const int k = m * 32 + bit;
        const int64_t j = bstart + k;
        const int4 pr = s_pr[k];
        const float2 mxy = s_xy[k];
        const float4 co = s_co[k];
        float v[2 * NROW];
#pragma unroll
        for (int c = 0; c < 2 * NROW; ++c) v[c] = 0.f;
        bool any = false;
#pragma unroll
        for (int p = 0; p < PX; ++p) {
          const int row = row0 + p;
          bool live = inside[p] && j <= (int64_t)lastj[p] &&
                      !(col < pr.x || col > pr.y || row < pr.z || row > pr.w);
          if (!live) continue;
          const float dx = fc - mxy.x, dy = (float)(row - ty * kTile) - mxy.y;
          const float pw = gauss_power(s_cs[k], dx, dy);
          if (pw < kPowSkip) continue;
          const float gv = fast_exp2(pw);
          const float araw = co.w * gv;
          const float al = fminf(araw, a.alpha_cap);
          if (al < a.alpha_skip) continue;
          any = true;
          const float4 cz = s_rgbz[k];
          const float om = 1.f - al;
          const float rom = fast_rcp(om);
          const float Texc = T[p] * rom;
          const float w = al * Texc;
          float uval = cz.x * dc0[p] + cz.y * dc1[p] + cz.z * dc2[p] + cz.w * dd[p];
          if (DC > 0) {
#pragma unroll
            for (int c4 = 0; c4 < NF; c4 += 4) {
              const float4 fq = s_f4[(c4 / 4) * B + k];
              const float f[4] = {fq.x, fq.y, fq.z, fq.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int c = c4 + i;
                if (c < NF) {
                  uval += f[i] * df[p][c];
                  if (c < 22) v[10 + c] += w * df[p][c];
                }
              }
            }
          }
          const float dal = uval * Texc - (suffix[p] + Tfin[p] * vpix[p]) * rom;
          suffix[p] += w * uval;
          T[p] = Texc;
          const float dar = araw < a.alpha_cap ? dal : 0.f;
          const float dq = -0.5f * gv * dar * co.w;
          v[0] += w * dc0[p];
          v[1] += w * dc1[p];
          v[2] += w * dc2[p];
          v[3] += w * dd[p];
          v[4] += dar * gv;
          v[5] += dq * dx * dx;
          v[6] += dq * dx * dy;
          v[7] += dq * dy * dy;
          v[8] += -2.f * dq * (co.x * dx + co.y * dy);
          v[9] += -2.f * dq * (co.y * dx + co.z * dy);
        }
        if (!__any_sync(0xffffffffu, any)) continue;
        const float r = warp_smem_reduce<NROW>(v, wred, lane);
        if (DET) {
          if (lane < nv) wacc[k * NVMAX + lane] = r;
        } else {
          float* dst = a.accum + (int64_t)s_g[k] * a.acc_stride;
          if (lane < nv && r != 0.f) red_add(dst + lane, r);
        }
      }
    }
    if (DET) {  // this batch's partials: warps added in index order, one store per (pair, CTA)
      __syncthreads();
      for (int e = threadIdx.x; e < cnt * nv; e += NT) {
        const int k = e / nv, q = e - k * nv;
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) sum += s_acc[(w * B + k) * NVMAX + q];
        a.part[((bstart + k) * SUBB + sidx) * nv + q] = sum;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// deterministic mode: per-Gaussian pair slots and the ordered gather
// ---------------------------------------------------------------------------
__global__ void k_det_counts(const int4* __restrict__ tile_rect, int64_t K, uint32_t* __restrict__ cnt) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= K) return;
  const int4 r = tile_rect[g];
  cnt[g] = (r.y >= r.x && r.w >= r.z) ? (uint32_t)((r.y - r.x + 1) * (r.w - r.z + 1)) : 0u;
}

// slot[pfx[g] + i] = the pair index of Gaussian g in the i-th tile of its
// rectangle (row-major): one CTA per tile walks the tile's list
__global__ void k_det_slots(const uint2* __restrict__ ranges, const uint32_t* __restrict__ pvals, int ntx,
                            const int4* __restrict__ tile_rect, const uint64_t* __restrict__ pfx, int64_t cap,
                            uint32_t* __restrict__ slot) {
  const int t = blockIdx.x;
  const uint2 rg = ranges[t];
  const int tx = t % ntx, ty = t / ntx;
  for (uint32_t j = rg.x + threadIdx.x; j < rg.y; j += blockDim.x) {
    const uint32_t g = pvals[j];
    const int4 r = tile_rect[g];
    const uint64_t q = pfx[g] + (uint64_t)((ty - r.z) * (r.y - r.x + 1) + (tx - r.x));
    if (q < (uint64_t)cap) slot[q] = j;  // (an overflowed frame is reported by the forward's status)
  }
}

// accum[g] = sum over g's tiles (row-major), then over the row-split CTAs, of
// the partials -- a fixed order; one warp per Gaussian, lane = value
__global__ void k_det_gather(const int4* __restrict__ tile_rect, int64_t K, const uint64_t* __restrict__ pfx,
                             const uint32_t* __restrict__ slot, const float* __restrict__ part, int subb, int nv,
                             int acc_stride, int64_t cap, float* __restrict__ accum) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= K) return;
  const int4 r = tile_rect[g];
  if (!(r.y >= r.x && r.w >= r.z)) return;
  const int n = (r.y - r.x + 1) * (r.w - r.z + 1);
  const uint64_t b = pfx[g];
  float acc = 0.f;
  for (int i = 0; i < n && b + i < (uint64_t)cap; ++i) {
    const uint32_t j = slot[b + i];
    if (lane < nv && j < (uint64_t)cap)
      for (int sidx = 0; sidx < subb; ++sidx) acc += part[((int64_t)j * subb + sidx) * nv + lane];
  }
  if (lane < nv) accum[g * acc_stride + lane] = acc;
}

struct PreBwdArgs {
  Fs4dCloud c;  // snapshot
  Fs4dCloud g;  // output grads (SoA, zero-initialised by the host driver)
  double R[9], tv[3], campos[3];
  double fx, fy, lowpass;
  int H, W, D, acc_stride, sh_degree;
  const uint32_t* order;      // depth order (viewspace outputs in depth order), or null: source order
  const int4* tile_rect;      // culled rows: (0, -1, 0, -1) (source-order mode zeroes their gradients)
  const uint32_t* counters;
  const float* accum;
  const uint32_t* clamp_mask;
  int32_t* vs_index;
  float* vs_norm;
};

__device__ __forceinline__ double sigmoid_db(double x) {
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  double e = exp(x);
  return e / (1.0 + e);
}

// One thread per visible Gaussian (depth rank r).  fp64 throughout, mirroring
// rasterizer.py:395-451 and gaussians.py:156-218.
// One visible Gaussian (depth rank r) or, in source-order mode, row r.
// sh_in / sh_out: this Gaussian's SH row and SH-gradient row -- global
// memory in depth-order mode, the warp's shared-memory staging rows in
// source-order mode (the kernel moves them with coalesced loads / stores).
__device__ __forceinline__ void preprocess_bwd_one(const PreBwdArgs& a, int64_t r, const float* sh_in, float* sh_out) {
  int64_t i;
  if (a.order) {
    if (r >= (int64_t)a.counters[CNT_VISIBLE]) return;
    i = a.order[r];
  } else {  // source order, no viewspace outputs: culled rows get their zero gradients here
    if (r >= a.c.K) return;
    i = r;
    const int4 t = a.tile_rect[i];
    if (t.y < t.x) {
      for (int k = 0; k < 3; ++k) a.g.positions[3 * i + k] = a.g.log_scales[3 * i + k] = a.g.colors_raw[3 * i + k] = 0.f;
      for (int k = 0; k < 4; ++k) a.g.rotations[4 * i + k] = 0.f;
      a.g.opacity_logits[i] = 0.f;
      for (int c = 0; c < a.c.D; ++c) a.g.features[(int64_t)a.c.D * i + c] = 0.f;
      const int nsh = ((a.sh_degree + 1) * (a.sh_degree + 1) - 1) * 3;
      if (sh_out)
        for (int c = 0; c < nsh; ++c) sh_out[c] = 0.f;
      if (a.vs_norm) a.vs_norm[i] = -1.f;  // dense source-indexed norms: culled
      return;
    }
  }
  const float* acc = a.accum + i * a.acc_stride;
  const double dcol[3] = {acc[0], acc[1], acc[2]};
  const double ddep = acc[3], dop = acc[4];
  const double dk00 = acc[5], dk01 = acc[6], dk11 = acc[7];
  const double dmx = acc[8], dmy = acc[9];

  const float* P = a.c.positions + 3 * i;
  const float* Q = a.c.rotations + 4 * i;
  const float* LS = a.c.log_scales + 3 * i;
  const double X = P[0], Y = P[1], Z = P[2];
  const double* R = a.R;
  const double x = R[0] * X + R[1] * Y + R[2] * Z + a.tv[0];
  const double y = R[3] * X + R[4] * Y + R[5] * Z + a.tv[1];
  const double z = R[6] * X + R[7] * Y + R[8] * Z + a.tv[2];

  // covariance (gaussians.py:187-194)
  const double q0 = Q[0], q1 = Q[1], q2 = Q[2], q3 = Q[3];
  const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  // one reciprocal per divisor (fp64; differs from true division by <= 1 ulp,
  // far below the fp32 outputs' resolution) instead of an IEEE divide each
  const double iqn = 1.0 / qn;
  const double qu[4] = {q0 * iqn, q1 * iqn, q2 * iqn, q3 * iqn};
  const double qw = qu[0], qx = qu[1], qy = qu[2], qz = qu[3];
  double Rq[9];
  Rq[0] = 1 - 2 * (qy * qy + qz * qz);
  Rq[1] = 2 * (qx * qy - qw * qz);
  Rq[2] = 2 * (qx * qz + qw * qy);
  Rq[3] = 2 * (qx * qy + qw * qz);
  Rq[4] = 1 - 2 * (qx * qx + qz * qz);
  Rq[5] = 2 * (qy * qz - qw * qx);
  Rq[6] = 2 * (qx * qz - qw * qy);
  Rq[7] = 2 * (qy * qz + qw * qx);
  Rq[8] = 1 - 2 * (qx * qx + qy * qy);
  const double s[3] = {exp((double)LS[0]), exp((double)LS[1]), exp((double)LS[2])};
  const double Dg[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
  double Sig[9];
  for (int rr = 0; rr < 3; ++rr)
    for (int cc = 0; cc < 3; ++cc)
      Sig[3 * rr + cc] = (Rq[3 * rr] * s[0]) * (Rq[3 * cc] * s[0]) + (Rq[3 * rr + 1] * s[1]) * (Rq[3 * cc + 1] * s[1]) +
                         (Rq[3 * rr + 2] * s[2]) * (Rq[3 * cc + 2] * s[2]);

  // projection Jacobian and cov2d (rasterizer.py:141-152)
  const double fx = a.fx, fy = a.fy;
  const double iz = 1.0 / z, iz2 = iz * iz;
  const double j00 = fx * iz, j02 = -fx * x * iz2;
  const double j11 = fy * iz, j12 = -fy * y * iz2;
  double M[6];
  for (int k = 0; k < 3; ++k) {
    M[k] = j00 * R[k] + j02 * R[6 + k];
    M[3 + k] = j11 * R[3 + k] + j12 * R[6 + k];
  }
  double MS[6];
  for (int rr = 0; rr < 2; ++rr)
    for (int k = 0; k < 3; ++k)
      MS[3 * rr + k] = M[3 * rr] * Sig[k] + M[3 * rr + 1] * Sig[3 + k] + M[3 * rr + 2] * Sig[6 + k];
  const double ca = MS[0] * M[0] + MS[1] * M[1] + MS[2] * M[2] + a.lowpass;
  const double cb = MS[0] * M[3] + MS[1] * M[4] + MS[2] * M[5];
  const double cc2 = MS[3] * M[3] + MS[4] * M[4] + MS[5] * M[5] + a.lowpass;
  const double det = ca * cc2 - cb * cb;
  const double idet = 1.0 / det;
  const double C00 = cc2 * idet, C01 = -cb * idet, C11 = ca * idet;

  // d_cov2d = -C dConic C  (rasterizer.py:396), dConic symmetric with dxy off-diagonal
  // T1 = dConic C
  const double t00 = dk00 * C00 + dk01 * C01, t01 = dk00 * C01 + dk01 * C11;
  const double t10 = dk01 * C00 + dk11 * C01, t11 = dk01 * C01 + dk11 * C11;
  const double g00 = -(C00 * t00 + C01 * t10), g01 = -(C00 * t01 + C01 * t11);
  const double g10 = -(C01 * t00 + C11 * t10), g11 = -(C01 * t01 + C11 * t11);
  const double G[4] = {g00, g01, g10, g11};
  const double S2[4] = {2 * g00, g01 + g10, g10 + g01, 2 * g11};  // sym = G + G^T

  // d_Mm = sym @ Mm @ Sigma ; d_sigma = Mm^T G Mm ; d_J = d_Mm @ R^T (rasterizer.py:412-415)
  double dM[6];
  for (int rr = 0; rr < 2; ++rr)
    for (int k = 0; k < 3; ++k)
      dM[3 * rr + k] = S2[2 * rr] * MS[k] + S2[2 * rr + 1] * MS[3 + k];
  double dS[9];
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q)
      dS[3 * p + q] = M[p] * (G[0] * M[q] + G[1] * M[3 + q]) + M[3 + p] * (G[2] * M[q] + G[3] * M[3 + q]);
  double dJ[6];
  for (int rr = 0; rr < 2; ++rr)
    for (int k = 0; k < 3; ++k)
      dJ[3 * rr + k] = dM[3 * rr] * R[3 * k] + dM[3 * rr + 1] * R[3 * k + 1] + dM[3 * rr + 2] * R[3 * k + 2];

  // camera-space gradient (rasterizer.py:417-426)
  const double iz3 = iz2 * iz;
  double dcam[3];
  dcam[0] = dJ[2] * (-fx * iz2) + dmx * fx * iz;
  dcam[1] = dJ[5] * (-fy * iz2) + dmy * fy * iz;
  dcam[2] = dJ[0] * (-fx * iz2) + dJ[2] * (2.0 * fx * x * iz3) + dJ[4] * (-fy * iz2) + dJ[5] * (2.0 * fy * y * iz3) +
            dmx * (-fx * x * iz2) + dmy * (-fy * y * iz2) + ddep;
  double dpos[3];
  for (int k = 0; k < 3; ++k) dpos[k] = dcam[0] * R[k] + dcam[1] * R[3 + k] + dcam[2] * R[6 + k];

  // covariance_backward (gaussians.py:203-218)
  double dR[9];
  {
    double SS[9];
    for (int p = 0; p < 9; ++p) SS[p] = dS[p] + dS[3 * (p % 3) + p / 3];
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q)
        dR[3 * p + q] = (SS[3 * p] * Rq[q] + SS[3 * p + 1] * Rq[3 + q] + SS[3 * p + 2] * Rq[6 + q]) * Dg[q];
  }
  double dls[3];
  for (int k = 0; k < 3; ++k) {
    double v = 0;
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) v += Rq[3 * p + k] * dS[3 * p + q] * Rq[3 * q + k];
    dls[k] = 2.0 * Dg[k] * v;
  }
  const double* g = dR;
  double dqu[4];
  dqu[0] = 2 * (-qz * g[1] + qy * g[2] + qz * g[3] - qx * g[5] - qy * g[6] + qx * g[7]);
  dqu[1] = 2 * (qy * g[1] + qz * g[2] + qy * g[3] - 2 * qx * g[4] - qw * g[5] + qz * g[6] + qw * g[7] - 2 * qx * g[8]);
  dqu[2] = 2 * (-2 * qy * g[0] + qx * g[1] + qw * g[2] + qx * g[3] + qz * g[5] - qw * g[6] + qz * g[7] - 2 * qy * g[8]);
  dqu[3] = 2 * (-2 * qz * g[0] - qw * g[1] + qx * g[2] + qw * g[3] - 2 * qz * g[4] + qy * g[5] + qx * g[6] + qy * g[7]);
  const double inner = dqu[0] * qu[0] + dqu[1] * qu[1] + dqu[2] * qu[2] + dqu[3] * qu[3];

  // colour gate and SH (build extension)
  const uint32_t gate = a.clamp_mask[i];
  double dcg[3];
  for (int k = 0; k < 3; ++k) dcg[k] = (gate >> k) & 1u ? dcol[k] : 0.0;
  const int n_sh = (a.sh_degree + 1) * (a.sh_degree + 1) - 1;
  if (n_sh > 0 && a.c.sh_rest) {
    double vx = X - a.campos[0], vy = Y - a.campos[1], vz = Z - a.campos[2];
    double dn = sqrt(vx * vx + vy * vy + vz * vz);
    dn = dn > 0 ? dn : 1.0;
    const double idn = 1.0 / dn;
    const double ux = vx * idn, uy = vy * idn, uz = vz * idn;
    const float* S = sh_in;
    float* GS = sh_out;
    double ddir[3] = {0, 0, 0};
    sh_visit<double>(a.sh_degree, ux, uy, uz, [&](int k, double Yk, double dYx, double dYy, double dYz) {
      double gk = 0;
      for (int c = 0; c < 3; ++c) {
        GS[3 * k + c] = (float)(Yk * dcg[c]);
        gk += S[3 * k + c] * dcg[c];
      }
      ddir[0] += gk * dYx;
      ddir[1] += gk * dYy;
      ddir[2] += gk * dYz;
    });
    const double dot = ddir[0] * ux + ddir[1] * uy + ddir[2] * uz;
    dpos[0] += (ddir[0] - dot * ux) * idn;
    dpos[1] += (ddir[1] - dot * uy) * idn;
    dpos[2] += (ddir[2] - dot * uz) * idn;
  }

  const double o = sigmoid_db((double)a.c.opacity_logits[i]);
  for (int k = 0; k < 3; ++k) {
    a.g.positions[3 * i + k] = (float)dpos[k];
    a.g.log_scales[3 * i + k] = (float)dls[k];
    a.g.colors_raw[3 * i + k] = (float)dcg[k];
  }
  for (int k = 0; k < 4; ++k) a.g.rotations[4 * i + k] = (float)((dqu[k] - inner * qu[k]) * iqn);
  a.g.opacity_logits[i] = (float)(dop * o * (1.0 - o));
  for (int c = 0; c < a.D; ++c) a.g.features[(int64_t)a.D * i + c] = acc[10 + c];
  if (a.vs_index) a.vs_index[r] = (int32_t)i;
  // depth-ordered: entry r of the visible list; source order: dense per Gaussian
  if (a.vs_norm) a.vs_norm[a.order ? r : i] = (float)hypot(dmx * 0.5 * a.W, dmy * 0.5 * a.H);
}

__global__ void __launch_bounds__(128) k_preprocess_bwd(PreBwdArgs a) {
  extern __shared__ float s_sh[];  // source-order mode: [4 warps][2][32 rows * n_sh * 3]
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int rowf = ((a.sh_degree + 1) * (a.sh_degree + 1) - 1) * 3;
  const bool staged = !a.order && rowf > 0 && a.c.sh_rest && a.g.sh_rest;
  if (!staged) {
    const int64_t i = a.order ? (r < (int64_t)a.counters[CNT_VISIBLE] ? a.order[r] : 0) : r;
    preprocess_bwd_one(a, r, rowf > 0 && a.c.sh_rest ? a.c.sh_rest + (int64_t)rowf * i : nullptr,
                       rowf > 0 && a.g.sh_rest ? a.g.sh_rest + (int64_t)rowf * i : nullptr);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* win = s_sh + warp * 2 * 32 * rowf;
  float* wout = win + 32 * rowf;
  const int64_t g0 = r - lane;
  const int64_t nrows = g0 < a.c.K ? min((int64_t)32, a.c.K - g0) : 0;
  const int64_t nf = nrows * rowf;
  const float* src = a.c.sh_rest + g0 * rowf;
  float* dst = a.g.sh_rest + g0 * rowf;
  const bool vec = nrows == 32 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (vec) {
    for (int e = lane; e < nf / 4; e += 32)
      reinterpret_cast<float4*>(win)[e] = __ldg(reinterpret_cast<const float4*>(src) + e);
  } else {
    for (int e = lane; e < nf; e += 32) win[e] = src[e];
  }
  __syncwarp();
  preprocess_bwd_one(a, r, win + lane * rowf, wout + lane * rowf);
  __syncwarp();
  if (vec) {
    for (int e = lane; e < nf / 4; e += 32) reinterpret_cast<float4*>(dst)[e] = reinterpret_cast<const float4*>(wout)[e];
  } else {
    for (int e = lane; e < nf; e += 32) dst[e] = wout[e];
  }
}

static int blend_bwd_subb() {
  static const int subb = [] {
    const char* e = getenv("FS4D_BLEND_BWD_SUB");
    const int v = e ? atoi(e) : 2;  // measured (configs[4]): 1 -> 285 us, 2 -> 275 us, 4 -> 307 us
    return v == 1 || v == 4 ? v : 2;
  }();
  return subb;
}

// the deterministic variant keeps a [warps][B][values] shared tile of warp
// sums, which fits for 2 or 4 row-split CTAs per tile (not 1)
static int det_subb() { return blend_bwd_subb() == 4 ? 4 : 2; }

static void launch_blend_bwd_det(int dc, int ntiles, const BwdArgs& a, cudaStream_t s) {
#define FS4D_BWD2D(D, SB) k_blend_bwd2<D, 2, SB, true><<<ntiles * SB, kTilePixels / 2 / SB, 0, s>>>(a)
#define FS4D_BWD2D_DC(SB)             \
  switch (dc) {                       \
    case 0: FS4D_BWD2D(0, SB); break;  \
    case 4: FS4D_BWD2D(4, SB); break;  \
    case 8: FS4D_BWD2D(8, SB); break;  \
    default: FS4D_BWD2D(16, SB); break; \
  }
  if (det_subb() == 4) {
    FS4D_BWD2D_DC(4)
  } else {
    FS4D_BWD2D_DC(2)
  }
#undef FS4D_BWD2D_DC
#undef FS4D_BWD2D
}

static void launch_blend_bwd(int dc, int ntiles, const BwdArgs& a, cudaStream_t s) {
  // pixels per thread of the replay (FS4D_BLEND_BWD_PX = 1, 2 or 4)
  static const int px = [] {
    const char* e = getenv("FS4D_BLEND_BWD_PX");
    const int v = e ? atoi(e) : 2;  // measured: 1 -> 416 us, 2 -> 342 us, 4 -> 620 us (configs[4])
    return v == 1 || v == 4 ? v : 2;
  }();
  if (px == 1 || dc > 16) {
    switch (dc) {
      case 0: k_blend_bwd<0><<<ntiles, kTilePixels, 0, s>>>(a); break;
      case 4: k_blend_bwd<4><<<ntiles, kTilePixels, 0, s>>>(a); break;
      case 8: k_blend_bwd<8><<<ntiles, kTilePixels, 0, s>>>(a); break;
      case 16: k_blend_bwd<16><<<ntiles, kTilePixels, 0, s>>>(a); break;
      case 32: k_blend_bwd<32><<<ntiles, kTilePixels, 0, s>>>(a); break;
      default: k_blend_bwd<64><<<ntiles, kTilePixels, 0, s>>>(a); break;
    }
  } else if (px == 2) {
    // CTAs per tile (FS4D_BLEND_BWD_SUB = 1, 2 or 4)
    const int subb = blend_bwd_subb();
#define FS4D_BWD2(D, SB) k_blend_bwd2<D, 2, SB><<<ntiles * SB, kTilePixels / 2 / SB, 0, s>>>(a)
#define FS4D_BWD2_DC(SB)            \
  switch (dc) {                     \
    case 0: FS4D_BWD2(0, SB); break;  \
    case 4: FS4D_BWD2(4, SB); break;  \
    case 8: FS4D_BWD2(8, SB); break;  \
    default: FS4D_BWD2(16, SB); break; \
  }
    if (subb == 4) {
      FS4D_BWD2_DC(4)
    } else if (subb == 2) {
      FS4D_BWD2_DC(2)
    } else {
      FS4D_BWD2_DC(1)
    }
#undef FS4D_BWD2_DC
#undef FS4D_BWD2
  } else {
    switch (dc) {
      case 0: k_blend_bwd2<0, 4, 1><<<ntiles, kTilePixels / 4, 0, s>>>(a); break;
      case 4: k_blend_bwd2<4, 4, 1><<<ntiles, kTilePixels / 4, 0, s>>>(a); break;
      case 8: k_blend_bwd2<8, 4, 1><<<ntiles, kTilePixels / 4, 0, s>>>(a); break;
      default: k_blend_bwd2<16, 4, 1><<<ntiles, kTilePixels / 4, 0, s>>>(a); break;
    }
  }
}

// deterministic-mode scratch: partials, per-Gaussian slots and offsets
size_t render_bwd_det_bytes(const RenderLayout& L) {
  const int64_t K = L.K > 0 ? L.K : 1, cap = L.cap > 0 ? L.cap : 1;
  const int nv = 10 + (L.D > 16 ? 16 : L.D);
  size_t o = 0;
  o = align_up(o + (size_t)cap * 4 /*subb*/ * nv * 4, 256);  // part (up to 4 row-split CTAs)
  o = align_up(o + (size_t)cap * 4, 256);                     // slot
  o = align_up(o + (size_t)K * 4, 256);                       // counts
  o = align_up(o + (size_t)K * 8, 256);                       // offsets
  return o + scan_scratch_bytes(K);
}

int render_backward(const Fs4dCloud& snap, const Fs4dCamera& cam, const Fs4dRasterConfig& cfg,
                    const RenderLayout& L, void* ws, const Fs4dImageGrads& up, Fs4dCloud& grads,
                    int32_t* vs_index, float* vs_norm, void* det_ws, size_t det_bytes, cudaStream_t s) {
  const int64_t K = L.K;
  const int D = cfg.with_features ? L.D : 0;
  if (det_ws) {
    if (D > 16) return fail(FS4D_ERR_CONFIG, "the deterministic backward supports D <= 16 feature channels");
    if (det_bytes < render_bwd_det_bytes(L)) return fail(FS4D_ERR_CONFIG, "deterministic workspace too small");
  }
  float* accum = at<float>(ws, L.accum);
  cudaMemsetAsync(accum, 0, (size_t)K * L.acc_stride * 4, s);
  // Viewspace outputs requested: visit the visible rows in depth order (the
  // order ProjectedGaussians reports them in) and zero the culled rows up
  // front.  Not requested (training): source order, no global depth sort,
  // the kernel writes the culled rows' zeros itself.
  const bool depth_ordered = vs_index != nullptr;
  const int n_sh = (snap.sh_degree + 1) * (snap.sh_degree + 1) - 1;
  if (depth_ordered) {
  // zero the outputs: culled rows keep zero gradients (rasterizer.py:432-441)
  cudaMemsetAsync(grads.positions, 0, (size_t)K * 3 * 4, s);
  cudaMemsetAsync(grads.rotations, 0, (size_t)K * 4 * 4, s);
  cudaMemsetAsync(grads.log_scales, 0, (size_t)K * 3 * 4, s);
  cudaMemsetAsync(grads.opacity_logits, 0, (size_t)K * 4, s);
  cudaMemsetAsync(grads.colors_raw, 0, (size_t)K * 3 * 4, s);
  if (grads.features && snap.D > 0) cudaMemsetAsync(grads.features, 0, (size_t)K * snap.D * 4, s);
  if (grads.sh_rest && n_sh > 0) cudaMemsetAsync(grads.sh_rest, 0, (size_t)K * n_sh * 3 * 4, s);
  }

  BwdArgs b;
  b.H = L.H;
  b.W = L.W;
  b.ntx = L.ntx;
  b.D = D;
  b.acc_stride = L.acc_stride;
  b.nvals = 10 + D;
  b.alpha_cap = (float)cfg.alpha_cap;
  b.alpha_skip = (float)cfg.alpha_skip;
  b.stop = (float)cfg.stop_transmittance;
  b.bg0 = (float)cfg.background[0];
  b.bg1 = (float)cfg.background[1];
  b.bg2 = (float)cfg.background[2];
  b.ranges = at<uint2>(ws, L.ranges);
  b.tperm = L.ntiles <= 65536 ? at<int32_t>(ws, L.tperm) : nullptr;
  b.pvals = at<uint32_t>(ws, L.pvals0);
  b.xy = at<float4>(ws, L.xy);
  b.conic_o = at<float4>(ws, L.conic_o);
  b.pix_rect = at<int4>(ws, L.pix_rect);
  b.rgbz = at<float4>(ws, L.rgbz);
  b.features = snap.features;
  b.tfinal = at<float>(ws, L.tfinal);
  b.last = at<int32_t>(ws, L.last);
  b.dC = up.d_color;
  b.dD = up.d_depth;
  b.dF = D > 0 ? up.d_feature : nullptr;
  b.dA = up.d_alpha;
  b.accum = accum;
  b.part = nullptr;
  int dc = D <= 0 ? 0 : D <= 4 ? 4 : D <= 8 ? 8 : D <= 16 ? 16 : D <= 32 ? 32 : 64;
  if (L.ntiles > 0 && det_ws) {
    StageTimer st(FS4D_STAGE_BLEND_BWD, s);
    const int64_t cap = L.cap > 0 ? L.cap : 1;
    char* d = (char*)det_ws;
    size_t o = 0;
    auto take = [&](size_t bytes) {
      void* at_ = d + o;
      o = align_up(o + bytes, 256);
      return at_;
    };
    b.part = (float*)take((size_t)cap * 4 * b.nvals * 4);
    uint32_t* slot = (uint32_t*)take((size_t)cap * 4);
    uint32_t* cnt = (uint32_t*)take((size_t)(K > 0 ? K : 1) * 4);
    uint64_t* pfx = (uint64_t*)take((size_t)(K > 0 ? K : 1) * 8);
    launch_blend_bwd_det(dc, L.ntiles, b, s);
    if (K > 0) {
      k_det_counts<<<(unsigned)ceil_div(K, 256), 256, 0, s>>>(at<int4>(ws, L.tile_rect), K, cnt);
      exclusive_scan_u32_to_u64(cnt, pfx, K, nullptr, nullptr, d + o, s);
      k_det_slots<<<L.ntiles, 256, 0, s>>>(at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.pvals0), L.ntx,
                                           at<int4>(ws, L.tile_rect), pfx, cap, slot);
      k_det_gather<<<(unsigned)ceil_div(K, 8), 256, 0, s>>>(at<int4>(ws, L.tile_rect), K, pfx, slot, b.part,
                                                            det_subb(), b.nvals, L.acc_stride, cap, accum);
    }
  } else if (L.ntiles > 0) {
    StageTimer st(FS4D_STAGE_BLEND_BWD, s);
    launch_blend_bwd(dc, L.ntiles, b, s);
  }

  PreBwdArgs p;
  p.c = snap;
  p.g = grads;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) p.R[3 * r + k] = cam.T[4 * r + k];
    p.tv[r] = cam.T[4 * r + 3];
  }
  for (int k = 0; k < 3; ++k) p.campos[k] = -(p.R[k] * p.tv[0] + p.R[3 + k] * p.tv[1] + p.R[6 + k] * p.tv[2]);
  p.fx = cam.K[0];
  p.fy = cam.K[4];
  p.lowpass = cfg.lowpass;
  p.H = L.H;
  p.W = L.W;
  p.D = D;
  p.acc_stride = L.acc_stride;
  p.sh_degree = snap.sh_degree;
  p.order = depth_ordered ? depth_order(L, ws, s) : nullptr;  // viewspace statistics come in depth order
  p.tile_rect = at<int4>(ws, L.tile_rect);
  p.counters = at<uint32_t>(ws, L.counters);
  p.accum = accum;
  p.clamp_mask = at<uint32_t>(ws, L.clamp_mask);
  p.vs_index = vs_index;
  p.vs_norm = vs_norm;
  if (K > 0) {
    StageTimer st(FS4D_STAGE_PREPROCESS_BWD, s);
    const size_t sh_smem = p.order ? 0 : (size_t)4 * 2 * 32 * (size_t)(n_sh * 3) * 4;
    static size_t sh_attr = 0;
    if (sh_smem > sh_attr) {
      cudaFuncSetAttribute(k_preprocess_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_smem);
      sh_attr = sh_smem;
    }
    k_preprocess_bwd<<<(unsigned)ceil_div(K, 128), 128, sh_smem, s>>>(p);
  }
  return check_launch("render_bwd");
}

}  // namespace fs4d
