// Forward rasterizer: project -> stable depth sort -> tile binning -> blend.
//
// Reference: rasterizer.render (rasterizer.py:264-303) and the functions it
// calls.  Stage map:
//   k_preprocess      project()            rasterizer.py:117-185 (fp64, per Gaussian)
//   radix + tie fixup np.argsort(z, stable) rasterizer.py:163
//   k_tile_count/scan/k_emit/radix/k_ranges   bin_tiles()  rasterizer.py:188-207
//   k_blend           _tile_alphas + _composite_weights + tile matmuls
//                                          rasterizer.py:215-261, 284-303
#include <stdlib.h>

#include "render_common.cuh"
#include "sh.cuh"

namespace fs4d {

struct PreArgs {
  Fs4dCloud c;
  double R[9], tv[3], campos[3];
  double fx, fy, cx, cy;
  int H, W, ntx, nty;
  double z_near, lowpass;
  int with_features;
  float4* xy;  // (u hi, v hi, u lo, v lo)
  float4* conic_o;
  int4* pix_rect;
  int4* tile_rect;
  float4* rgbz;
  float4* cov_r;
  double* z64;
  uint32_t* dkeys;
  uint32_t* dvals;
  uint32_t* clamp_mask;
  uint32_t* counters;
  uint32_t* tcnt;  // per-tile pair counts (zeroed by the host), filled by the fused histogram
  int32_t* status;
};

__device__ __forceinline__ double sigmoid_d(double x) {
  // gaussians.py:25-31 (sign-split stable form)
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  double e = exp(x);
  return e / (1.0 + e);
}

// One Gaussian of k_preprocess; returns its inclusive tile rectangle
// ((0, -1, 0, -1) when culled / out of range).
__device__ __forceinline__ int4 preprocess_one(const PreArgs& a, int64_t i, const float* __restrict__ sh_row,
                                               bool async_sh = false) {
  if (i >= a.c.K) return make_int4(0, -1, 0, -1);
  a.dvals[i] = (uint32_t)i;
  a.dkeys[i] = 0xFFFFFFFFu;  // culled sentinel sorts last
  a.tile_rect[i] = make_int4(0, -1, 0, -1);

  // ---- finite checks, field order of rasterizer.py:120-127 ----
  const float* P = a.c.positions + 3 * i;
  const float* Q = a.c.rotations + 4 * i;
  const float* LS = a.c.log_scales + 3 * i;
  const float* CR = a.c.colors_raw + 3 * i;
  float p0 = P[0], p1 = P[1], p2 = P[2];
  float q0 = Q[0], q1 = Q[1], q2 = Q[2], q3 = Q[3];
  float s0 = LS[0], s1 = LS[1], s2 = LS[2];
  float ol = a.c.opacity_logits[i];
  float cr0 = CR[0], cr1 = CR[1], cr2 = CR[2];
  bool bad = false;
  if (!(isfinite(p0) && isfinite(p1) && isfinite(p2))) { flag_bad_field(a.status, FS4D_FIELD_POSITIONS, i); bad = true; }
  if (!(isfinite(q0) && isfinite(q1) && isfinite(q2) && isfinite(q3))) { flag_bad_field(a.status, FS4D_FIELD_ROTATIONS, i); bad = true; }
  if (!(isfinite(s0) && isfinite(s1) && isfinite(s2))) { flag_bad_field(a.status, FS4D_FIELD_LOG_SCALES, i); bad = true; }
  if (!isfinite(ol)) { flag_bad_field(a.status, FS4D_FIELD_OPACITY, i); bad = true; }
  if (!(isfinite(cr0) && isfinite(cr1) && isfinite(cr2))) { flag_bad_field(a.status, FS4D_FIELD_COLORS, i); bad = true; }
  {
    const float* F = a.c.features + (int64_t)a.c.D * i;
    bool fb = false;
    if ((a.c.D & 3) == 0 && (reinterpret_cast<uintptr_t>(a.c.features) & 15) == 0) {
      for (int k = 0; k < a.c.D; k += 4) {  // one 16 B load per 4 channels
        const float4 f = __ldg(reinterpret_cast<const float4*>(F + k));
        fb |= !(isfinite(f.x) && isfinite(f.y) && isfinite(f.z) && isfinite(f.w));
      }
    } else {
      for (int k = 0; k < a.c.D; ++k) fb |= !isfinite(F[k]);
    }
    if (fb) { flag_bad_field(a.status, FS4D_FIELD_FEATURES, i); bad = true; }
  }
  const int n_sh = (a.c.sh_degree + 1) * (a.c.sh_degree + 1) - 1;
  if (n_sh > 0 && a.c.sh_rest) {
    if (async_sh) {  // the warp's cp.async copies of its SH rows (issued before the field loads above)
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
    }
    const float* S = sh_row;  // this Gaussian's SH row, staged in shared memory by its warp
    bool sb = false;
    for (int k = 0; k < n_sh * 3; ++k) sb |= !isfinite(S[k]);
    if (sb) { flag_bad_field(a.status, FS4D_FIELD_SH, i); bad = true; }
  }
  if (bad) return make_int4(0, -1, 0, -1);

  // ---- camera space (rasterizer.py:131-140) ----
  const double X = p0, Y = p1, Z = p2;
  const double x = a.R[0] * X + a.R[1] * Y + a.R[2] * Z + a.tv[0];
  const double y = a.R[3] * X + a.R[4] * Y + a.R[5] * Z + a.tv[1];
  const double z = a.R[6] * X + a.R[7] * Y + a.R[8] * Z + a.tv[2];
  if (!(z > a.z_near)) return make_int4(0, -1, 0, -1);
  const double u = a.fx * x / z + a.cx;
  const double v = a.fy * y / z + a.cy;

  // ---- 3-d covariance (gaussians.py:140-194) ----
  const double qn = sqrt((double)q0 * q0 + (double)q1 * q1 + (double)q2 * q2 + (double)q3 * q3);
  if (qn < 1e-12) {
    if (a.status) {
      atomicMin(&a.status[FS4D_ST_DEGEN_INDEX], (int32_t)i);
      raise_status(a.status, FS4D_ERR_DEGENERATE);
    }
    return make_int4(0, -1, 0, -1);
  }
  const double qw = q0 / qn, qx = q1 / qn, qy = q2 / qn, qz = q3 / qn;
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
  const double sc[3] = {exp((double)s0), exp((double)s1), exp((double)s2)};
  double RS[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) RS[3 * r + k] = Rq[3 * r + k] * sc[k];
  double Sig[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      Sig[3 * r + cc] = RS[3 * r] * RS[3 * cc] + RS[3 * r + 1] * RS[3 * cc + 1] + RS[3 * r + 2] * RS[3 * cc + 2];

  // ---- EWA projection (rasterizer.py:141-158) ----
  const double j00 = a.fx / z, j02 = -a.fx * x / (z * z);
  const double j11 = a.fy / z, j12 = -a.fy * y / (z * z);
  double M[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    M[k] = j00 * a.R[k] + j02 * a.R[6 + k];
    M[3 + k] = j11 * a.R[3 + k] + j12 * a.R[6 + k];
  }
  double MS[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      MS[3 * r + k] = M[3 * r] * Sig[k] + M[3 * r + 1] * Sig[3 + k] + M[3 * r + 2] * Sig[6 + k];
  double ca = MS[0] * M[0] + MS[1] * M[1] + MS[2] * M[2];
  double cb = MS[0] * M[3] + MS[1] * M[4] + MS[2] * M[5];
  double cc = MS[3] * M[3] + MS[4] * M[4] + MS[5] * M[5];
  ca += a.lowpass;
  cc += a.lowpass;
  const double mid = 0.5 * (ca + cc);
  const double det = ca * cc - cb * cb;
  const double eig = mid + sqrt(fmax(mid * mid - det, 0.0));
  const double radius = ceil(3.0 * sqrt(eig));

  // ---- offscreen cull (rasterizer.py:160-162) ----
  const bool on = (u + radius >= 0) && (u - radius <= a.W - 1) && (v + radius >= 0) && (v - radius <= a.H - 1);
  if (!on) return make_int4(0, -1, 0, -1);

  // ---- kept: conic, activations, footprints ----
  const double inv = 1.0 / det;
  const double c00 = cc * inv, c01 = -cb * inv, c11 = ca * inv;
  // rasterizer.py:165-171 divides each entry by det; match that rounding
  const double c00r = cc / det, c01r = -cb / det, c11r = ca / det;
  (void)c00; (void)c01; (void)c11;
  const float opac = (float)sigmoid_d((double)ol);

  double col[3] = {cr0, cr1, cr2};
  if (n_sh > 0 && a.c.sh_rest) {
    double dx = X - a.campos[0], dy = Y - a.campos[1], dz = Z - a.campos[2];
    double dn = sqrt(dx * dx + dy * dy + dz * dz);
    dn = dn > 0 ? dn : 1.0;
    const float* S = sh_row;
    sh_visit<double>(a.c.sh_degree, dx / dn, dy / dn, dz / dn, [&](int k, double Yk, double, double, double) {
      col[0] += Yk * S[3 * k + 0];
      col[1] += Yk * S[3 * k + 1];
      col[2] += Yk * S[3 * k + 2];
    });
  }
  uint32_t gate = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (col[k] > 0.0 && col[k] < 1.0) gate |= 1u << k;
    col[k] = fmin(fmax(col[k], 0.0), 1.0);
  }
  a.clamp_mask[i] = gate;

  // pixel footprint |j - u| <= r  <=>  ceil(u - r) <= j <= floor(u + r)  (rasterizer.py:227)
  int px0 = (int)fmax(ceil(u - radius), 0.0), px1 = (int)fmin(floor(u + radius), (double)(a.W - 1));
  int py0 = (int)fmax(ceil(v - radius), 0.0), py1 = (int)fmin(floor(v + radius), (double)(a.H - 1));
  // inclusive tile rectangle (rasterizer.py:198-201)
  const int tx0 = (int)fmin(fmax(floor((u - radius) / kTile), 0.0), (double)(a.ntx - 1));
  const int tx1 = (int)fmin(fmax(floor((u + radius) / kTile), 0.0), (double)(a.ntx - 1));
  const int ty0 = (int)fmin(fmax(floor((v - radius) / kTile), 0.0), (double)(a.nty - 1));
  const int ty1 = (int)fmin(fmax(floor((v + radius) / kTile), 0.0), (double)(a.nty - 1));

  {
    const float uh = (float)u, vh = (float)v;
    a.xy[i] = make_float4(uh, vh, (float)(u - (double)uh), (float)(v - (double)vh));
  }
  a.conic_o[i] = make_float4((float)c00r, (float)c01r, (float)c11r, opac);
  a.pix_rect[i] = make_int4(px0, px1, py0, py1);
  a.tile_rect[i] = make_int4(tx0, tx1, ty0, ty1);
  a.rgbz[i] = make_float4((float)col[0], (float)col[1], (float)col[2], (float)z);
  a.cov_r[i] = make_float4((float)ca, (float)cb, (float)cc, (float)radius);
  a.z64[i] = z;
  a.dkeys[i] = __float_as_uint((float)z);  // z > 0: IEEE bits order as unsigned
  atomicAdd(&a.counters[CNT_VISIBLE], 1u);
  return make_int4(tx0, tx1, ty0, ty1);
}

// Projection of every Gaussian (preprocess_one) fused with the per-tile pair
// histogram bin_tiles needs (rasterizer.py:188-207): block-aggregated in
// shared memory, one global atomic per (block, touched tile).
// The warp's 32 SH rows ([K, n_sh, 3], 180 B each at SH3) are copied into
// shared memory with coalesced 16 B loads first (a thread reading its own
// row 180 B apart from its neighbours' was the kernel's load-issue cost).
#ifdef FS4D_PRE_MINB  // A/B knob: minimum resident blocks per SM (caps registers)
__global__ void __launch_bounds__(256, FS4D_PRE_MINB) k_preprocess(PreArgs a) {
#else
__global__ void __launch_bounds__(256) k_preprocess(PreArgs a) {
#endif
  // dynamic shared memory: [8 warps][32 rows * n_sh * 3 floats] of SH rows,
  // then the block's tile histogram sized to this frame's tile count (a
  // fixed 24 KB array capped the kernel at 3 blocks per SM)
  extern __shared__ float4 s_sh4[];
  const int rowf_all = ((a.c.sh_degree + 1) * (a.c.sh_degree + 1) - 1) * 3;
  uint32_t* h = reinterpret_cast<uint32_t*>(s_sh4) + 8 * 32 * rowf_all;
  const bool smem = a.ntx * a.nty <= kHistTilesSmem;
  if (smem)
    for (int b = threadIdx.x; b < a.ntx * a.nty; b += blockDim.x) h[b] = 0;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rowf = ((a.c.sh_degree + 1) * (a.c.sh_degree + 1) - 1) * 3;
  float* wsh = reinterpret_cast<float*>(s_sh4) + warp * 32 * rowf;
  bool async_sh = false;
  if (rowf > 0 && a.c.sh_rest) {
    const int64_t g0 = i - lane;
    const int64_t nrows = min((int64_t)32, a.c.K - g0);
    const float* src = a.c.sh_rest + g0 * rowf;
    const int64_t nf = nrows * rowf;
    if (nrows == 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      // 32 rows of any width are a multiple of 16 B in total.  Asynchronous
      // 16-byte copies (cp.async): all of a lane's ~11 rows in flight at once
      // with no registers held (a load -> store loop waited on each load)
      // The wait is deferred into preprocess_one, after its field loads are
      // issued: the SH rows and the other fields share one memory latency.
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(wsh));
      for (int e = lane; e < nf / 4; e += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * e),
                     "l"(reinterpret_cast<const float4*>(src) + e)
                     : "memory");
      async_sh = true;
    } else {
      for (int e = lane; e < nf; e += 32) wsh[e] = src[e];
      __syncwarp();
    }
  }
  const int4 t = preprocess_one(a, i, wsh + lane * rowf, async_sh);
  __syncthreads();  // the block's tile histogram was zeroed above
  for (int ty = t.z; ty <= t.w; ++ty)
    for (int tx = t.x; tx <= t.y; ++tx) {
      const int b = ty * a.ntx + tx;
      if (smem) atomicAdd(&h[b], 1u);
      else atomicAdd(&a.tcnt[b], 1u);
    }
  __syncthreads();
  if (smem)
    for (int b = threadIdx.x; b < a.ntx * a.nty; b += blockDim.x)
      if (h[b]) atomicAdd(&a.tcnt[b], h[b]);
}

// Equal fp32 keys are re-ordered by the exact fp64 depth, ties by source
// index, so the order equals np.argsort(z64, kind="stable") (rasterizer.py:163).
__global__ void k_depth_tie_fixup(const uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                  const double* __restrict__ z64, int64_t K, const uint32_t* counters) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t M = counters[CNT_VISIBLE];
  if (r >= M) return;
  const uint32_t key = keys[r];
  if (r > 0 && keys[r - 1] == key) return;        // not a run start
  if (r + 1 >= M || keys[r + 1] != key) return;   // run of length 1
  int64_t e = r + 1;
  while (e < M && keys[e] == key) ++e;
  for (int64_t a = r + 1; a < e; ++a) {  // insertion sort of the (tiny) run
    uint32_t va = vals[a];
    double za = z64[va];
    int64_t b = a - 1;
    while (b >= r) {
      uint32_t vb = vals[b];
      double zb = z64[vb];
      if (zb < za || (zb == za && vb < va)) break;
      vals[b + 1] = vb;
      --b;
    }
    vals[b + 1] = va;
  }
}

// 16-byte global -> shared copy that bypasses registers (cp.async, L2 only)
__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst_smem))),
               "l"(src)
               : "memory");
}

struct BlendArgs {
  int H, W, ntx, D, c0;
  float alpha_cap, alpha_skip, stop;
  float bg0, bg1, bg2;
  const uint2* ranges;
  const int32_t* tperm;  // tiles by decreasing pair count (launch order), or null
  const uint32_t* pvals;
  const float4* xy;
  const float4* conic_o;
  const int4* pix_rect;
  const float4* rgbz;
  const float* features;  // [K, D] snapshot features
  float* out_color;
  float* out_depth;
  float* out_feature;
  float* out_alpha;
  int32_t* out_ncontrib;
  float* tfinal;
  int32_t* last;
};

// One CTA per 16x16 tile, one pixel per thread, Gaussians staged through
// shared memory in batches of 256 (front to back).  DC = feature channels
// handled by this launch ([c0, c0+DC)); the first launch also composites
// colour, depth and alpha.
// SUB > 1 splits a tile's rows over SUB CTAs (each streams the whole depth-
// ordered list but composites 16/SUB rows): shorter critical path for the
// densest tiles, sharper warp-row culling.
#ifdef FS4D_BLEND_TRACE
// debug: per-CTA (globaltimer start, end, smid, batches) of the last k_blend launch
__device__ unsigned long long g_blend_trace[8192][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
extern "C" int fs4d_debug_blend_trace(unsigned long long* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, g_blend_trace, sizeof(g_blend_trace));
}
#endif

template <int DC, int SUB, bool FIRST>
#ifdef FS4D_BLEND_MINB  // A/B knob: minimum resident CTAs per SM (caps registers)
__global__ void __launch_bounds__(kTilePixels / SUB, FS4D_BLEND_MINB) k_blend(BlendArgs a) {
#else  // (no minimum: ptxas settles at 72 registers; an explicit 1 lets it take 112 and costs ~9%)
__global__ void __launch_bounds__(kTilePixels / SUB) k_blend(BlendArgs a) {
#endif
#ifdef FS4D_BLEND_TRACE
  const unsigned long long t_start = gtimer();
  unsigned nbatch = 0;
#endif
  constexpr int NT = kTilePixels / SUB;  // threads = pixels = Gaussians per batch
  // the staged batch as ONE shared array: 16-byte rows [4 + DC/4][NT] -- the
  // scaled conic (gauss_power), the pixel rectangle, rgb + depth, the strip-cull constants, then the
  // feature quads (channel-quad-major: conflict-free staging stores,
  // broadcast reads) -- and the tile-relative means (8 bytes each) after
  // them.  Reads of Gaussian k are [k * 16 + constant] / [k * 8 + constant]
  // off one base (with separate arrays ptxas rebuilt each array's
  // shared-window address inside the compositing loop)
  constexpr int kRows = 4 + (DC > 0 ? DC / 4 : 0);
  __shared__ __align__(16) float4 s_g[kRows * NT + NT / 2];
  float4* const s_cs = s_g;
  int4* const s_pr = reinterpret_cast<int4*>(s_g + NT);
  float4* const s_rgbz = s_g + 2 * NT;
  float4* const s_sc = s_g + 3 * NT;  // strip-cull constants (strip_consts)
  float4* const s_f4 = s_g + 4 * NT;
  float2* const s_xy = reinterpret_cast<float2*>(s_g + kRows * NT);
  // per-warp ballot masks of the staged batch (shared, not a local array)
  __shared__ unsigned s_mask[NT / 32][NT / 32];

  const int tile = a.tperm ? a.tperm[blockIdx.x / SUB] : blockIdx.x / SUB, sub = blockIdx.x % SUB;
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  const int row0 = ty * kTile + sub * (kTile / SUB);
  const int col = tx * kTile + (threadIdx.x & (kTile - 1));
  const int row = row0 + (threadIdx.x / kTile);
  const bool inside = col < a.W && row < a.H;
  const uint2 rg = a.ranges[tile];
  constexpr bool first = FIRST;  // the launch with c0 == 0 also composites colour, depth, alpha
  const int lane = threadIdx.x & 31;
  const int wrow0 = row0 + (threadIdx.x >> 5) * 2;  // this warp's two pixel rows
  const int tcol0 = tx * kTile;
  // pixel and means relative to the tile origin (tile_rel_mean)
  const float ox = (float)tcol0, oy = (float)(ty * kTile);
  const float fc = (float)(col - tcol0), fr = (float)(row - ty * kTile);

  // accumulators as float2 pairs: every update is one FFMA2 (two fp32 FMAs,
  // bit-identical to the scalar FMAs) -- halves the blend's FMA issue slots
  float T = 1.f;
  float2 acc_rg = make_float2(0.f, 0.f), acc_bz = make_float2(0.f, 0.f);
  float2 accf2[DC > 0 ? DC / 2 : 1];
#pragma unroll
  for (int c = 0; c < (DC > 0 ? DC / 2 : 1); ++c) accf2[c] = make_float2(0.f, 0.f);
  int ncontrib = 0, last = -1;
  bool done = !inside || !(1.f >= a.stop);  // rasterizer.py:252: contrib needs T_exc >= stop
  const int nf = DC > 0 ? min(DC, a.D - a.c0) : 0;
  const bool vec_ok = DC >= 4 && nf == DC && (a.D & 3) == 0 && (a.c0 & 3) == 0;

  // the next batch's Gaussian index is loaded one batch ahead (its latency
  // hides behind this batch's compositing instead of preceding the record
  // loads); the records that need no transform (pixel rectangle, rgb +
  // depth, feature quads) go global -> shared with cp.async, no registers
  uint32_t g_next = rg.x + threadIdx.x < rg.y ? a.pvals[rg.x + threadIdx.x] : 0u;
  for (uint32_t b = rg.x; b < rg.y; b += NT) {
    if (__syncthreads_count(done) == NT) break;
#ifdef FS4D_BLEND_TRACE
    ++nbatch;
#endif
    const uint32_t j = b + threadIdx.x;
    const uint32_t g = g_next;
    if (j + NT < rg.y) g_next = a.pvals[j + NT];
    if (j < rg.y) {
      cp_async16(s_pr + threadIdx.x, a.pix_rect + g);
      cp_async16(s_rgbz + threadIdx.x, a.rgbz + g);
      s_xy[threadIdx.x] = tile_rel_mean(a.xy[g], ox, oy);
      const float4 cog = a.conic_o[g];
      s_cs[threadIdx.x] = scaled_conic(cog);
      s_sc[threadIdx.x] = strip_consts(cog, a.alpha_skip);
      if (DC > 0) {
        const float* src = a.features + (int64_t)g * a.D + a.c0;
        if (vec_ok) {
#pragma unroll
          for (int c = 0; c < DC; c += 4) cp_async16(s_f4 + (c / 4) * NT + threadIdx.x, src + c);
        } else {
          for (int c = 0; c < DC; c += 4) {
            float v[4];
            for (int i = 0; i < 4; ++i) v[i] = c + i < nf ? src[c + i] : 0.f;
            s_f4[(c / 4) * NT + threadIdx.x] = make_float4(v[0], v[1], v[2], v[3]);
          }
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int cnt = min((uint32_t)NT, rg.y - b);
    // warp-level culling: one ballot per 32 staged Gaussians keeps those whose
    // pixel footprint touches this warp's two pixel rows; the per-thread loop
    // then walks only the set bits, in depth order
    const int wid = threadIdx.x >> 5;
#pragma unroll
    for (int m = 0; m < NT / 32; ++m) {
      const int kk = m * 32 + lane;
      bool hit = false;
      if (kk < cnt) {
        const int4 pr = s_pr[kk];
        hit = pr.w >= wrow0 && pr.z <= wrow0 + 1 && pr.y >= tcol0 && pr.x <= tcol0 + kTile - 1;
        if (hit) {
          const float2 mr = s_xy[kk];
          hit = strip_hits_c<2>(pr, make_float2(mr.x + ox, mr.y + oy), s_sc[kk], wrow0, tcol0);
        }
      }
      const unsigned msk = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) s_mask[wid][m] = msk;
    }
    __syncwarp();
    if (!done) {
#pragma unroll 1
      for (int m = 0; m < NT / 32 && !done; ++m) {
        unsigned bits = s_mask[wid][m];
        // groups of BK Gaussians: the alphas of a group are independent of T
        // (instruction-level parallelism across the smem loads and ex2), only
        // the compositing below is a serial chain -- same decisions, same order
#ifndef FS4D_BLEND_BK
#define FS4D_BLEND_BK 3  // measured blend stage (round 2, tools/gpu_final.sh): 3 -> 86.8 us, 4 -> 89.5, 5 -> 90.2, 6 -> 93.0
#endif
        constexpr int BK = FS4D_BLEND_BK;
        while (bits) {
          int kk[BK];
          float alv[BK];
          bool live[BK];
#pragma unroll
          for (int j = 0; j < BK; ++j) {
            kk[j] = bits ? m * 32 + __ffs(bits) - 1 : 0;
            live[j] = bits != 0;
            bits &= bits - 1;
          }
#pragma unroll
          for (int j = 0; j < BK; ++j) {
            const int k = kk[j];
            const int4 pr = s_pr[k];
            const float2 mm = s_xy[k];
            const float4 cs = s_cs[k];
            const float dx = fc - mm.x, dy = fr - mm.y;
            const float pw = gauss_power(cs, dx, dy);
            const float al = fminf(cs.w * fast_exp2(pw), a.alpha_cap);
            live[j] = live[j] && !(col < pr.x || col > pr.y || row < pr.z || row > pr.w) && !(pw < kPowSkip) &&
                      !(al < a.alpha_skip);
            alv[j] = al;
          }
#pragma unroll
          for (int j = 0; j < BK; ++j) {
            // (T < stop always sets done right after the update below, and
            // done starts true when 1 < stop: no pre-check needed here)
            if (!live[j] || done) continue;
            const int k = kk[j];
            const float al = alv[j];
            const float w = al * T;
            const float2 w2 = make_float2(w, w);
            if (first) {
              const float4 cz = s_rgbz[k];
              acc_rg = __ffma2_rn(w2, make_float2(cz.x, cz.y), acc_rg);
              acc_bz = __ffma2_rn(w2, make_float2(cz.z, cz.w), acc_bz);
            }
            if (DC > 0) {
#pragma unroll
              for (int c = 0; c < DC; c += 4) {
                const float4 fv = s_f4[(c / 4) * NT + k];
                accf2[c / 2] = __ffma2_rn(w2, make_float2(fv.x, fv.y), accf2[c / 2]);
                accf2[c / 2 + 1] = __ffma2_rn(w2, make_float2(fv.z, fv.w), accf2[c / 2 + 1]);
              }
            }
            T *= (1.f - al);
            ++ncontrib;
            last = (int)(b + k);
            if (T < a.stop) done = true;
          }
          if (done) break;
        }
      }
    }
  }
#ifdef FS4D_BLEND_TRACE
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < 8192) {
    g_blend_trace[blockIdx.x][0] = t_start;
    g_blend_trace[blockIdx.x][1] = gtimer();
    g_blend_trace[blockIdx.x][2] = smid();
    g_blend_trace[blockIdx.x][3] = nbatch;
  }
#endif
  if (!inside) return;
  const int64_t pix = (int64_t)row * a.W + col;
  if (first) {
    a.out_color[3 * pix + 0] = acc_rg.x + T * a.bg0;
    a.out_color[3 * pix + 1] = acc_rg.y + T * a.bg1;
    a.out_color[3 * pix + 2] = acc_bz.x + T * a.bg2;
    a.out_depth[pix] = acc_bz.y;
    a.out_alpha[pix] = 1.f - T;
    if (a.out_ncontrib) a.out_ncontrib[pix] = ncontrib;
    a.tfinal[pix] = T;
    a.last[pix] = last;
  }
  if (DC > 0) {
    float* dst = a.out_feature + pix * a.D + a.c0;
    if (vec_ok) {
#pragma unroll
      for (int c = 0; c < DC; c += 4)
        *reinterpret_cast<float4*>(dst + c) =
            make_float4(accf2[c / 2].x, accf2[c / 2].y, accf2[c / 2 + 1].x, accf2[c / 2 + 1].y);
    } else {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (c < nf) dst[c] = (c & 1) ? accf2[c / 2].y : accf2[c / 2].x;
    }
  }
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
template <int SUB>
static void launch_blend_sub(int dc, int ntiles, const BlendArgs& a, cudaStream_t s) {
  const int grid = ntiles * SUB, nt = kTilePixels / SUB;
  if (a.c0 == 0) {
    switch (dc) {
      case 0: k_blend<0, SUB, true><<<grid, nt, 0, s>>>(a); break;
      case 4: k_blend<4, SUB, true><<<grid, nt, 0, s>>>(a); break;
      case 8: k_blend<8, SUB, true><<<grid, nt, 0, s>>>(a); break;
      case 16: k_blend<16, SUB, true><<<grid, nt, 0, s>>>(a); break;
      default:  // (SUB 1: 256 pixels per CTA, slices capped at 16 channels -- blend_max_dc)
        if constexpr (SUB > 1) k_blend<32, SUB, true><<<grid, nt, 0, s>>>(a);
        break;
    }
  } else {  // further feature-channel slices of a D > 32 map
    switch (dc) {
      case 4: k_blend<4, SUB, false><<<grid, nt, 0, s>>>(a); break;
      case 8: k_blend<8, SUB, false><<<grid, nt, 0, s>>>(a); break;
      case 16: k_blend<16, SUB, false><<<grid, nt, 0, s>>>(a); break;
      default:
        if constexpr (SUB > 1) k_blend<32, SUB, false><<<grid, nt, 0, s>>>(a);
        break;
    }
  }
}

static int blend_sub() {
  static const int sub = getenv("FS4D_BLEND_SUB") ? atoi(getenv("FS4D_BLEND_SUB")) : 2;
  return sub;
}
// widest feature slice of one blend launch: the 256-thread variant (SUB 1)
// stages 256 Gaussians per batch and fits 16 channels in 48 KB of shared memory
static int blend_max_dc() { return blend_sub() == 1 ? 16 : 32; }

static void launch_blend(int dc, int ntiles, const BlendArgs& a, cudaStream_t s) {
  // (two pixels per thread was measured slower: 157-165 vs 150 us)
  const int sub = blend_sub();
  if (sub == 4) launch_blend_sub<4>(dc, ntiles, a, s);
  else if (sub == 1) launch_blend_sub<1>(dc, ntiles, a, s);
  else launch_blend_sub<2>(dc, ntiles, a, s);
}

int render_forward(const Fs4dCloud& snap, const Fs4dCamera& cam, const Fs4dRasterConfig& cfg,
                   const RenderLayout& L, void* ws, Fs4dImages& out, int32_t* status, cudaStream_t s) {
  const int64_t K = L.K;
  uint32_t* counters = at<uint32_t>(ws, L.counters);
  cudaMemsetAsync(counters, 0, CNT_WORDS * 4, s);
  // tile counts, append cursors, offsets and ranges are contiguous: one memset
  cudaMemsetAsync(at<char>(ws, L.tcnt), 0, L.ranges + (size_t)L.ntiles * 8 - L.tcnt, s);

  PreArgs p;
  p.c = snap;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) p.R[3 * r + k] = cam.T[4 * r + k];
    p.tv[r] = cam.T[4 * r + 3];
  }
  for (int k = 0; k < 3; ++k)  // camera centre C = -R^T t
    p.campos[k] = -(p.R[k] * p.tv[0] + p.R[3 + k] * p.tv[1] + p.R[6 + k] * p.tv[2]);
  p.fx = cam.K[0];
  p.fy = cam.K[4];
  p.cx = cam.K[2];
  p.cy = cam.K[5];
  p.H = L.H;
  p.W = L.W;
  p.ntx = L.ntx;
  p.nty = L.nty;
  p.z_near = cfg.z_near;
  p.lowpass = cfg.lowpass;
  p.with_features = cfg.with_features;
  p.xy = at<float4>(ws, L.xy);
  p.conic_o = at<float4>(ws, L.conic_o);
  p.pix_rect = at<int4>(ws, L.pix_rect);
  p.tile_rect = at<int4>(ws, L.tile_rect);
  p.rgbz = at<float4>(ws, L.rgbz);
  p.cov_r = at<float4>(ws, L.cov_r);
  p.z64 = at<double>(ws, L.z64);
  p.dkeys = at<uint32_t>(ws, L.dkeys0);
  p.dvals = at<uint32_t>(ws, L.dvals0);
  p.clamp_mask = at<uint32_t>(ws, L.clamp_mask);
  p.counters = counters;
  p.tcnt = at<uint32_t>(ws, L.tcnt);
  p.status = status;
  {
    StageTimer st(FS4D_STAGE_PREPROCESS, s);
    const int ntl = p.ntx * p.nty;
    const size_t sh_smem = (size_t)8 * 32 * (((snap.sh_degree + 1) * (snap.sh_degree + 1) - 1) * 3) * 4 +
                           (size_t)(ntl <= kHistTilesSmem ? ntl : 0) * 4;
    static size_t sh_attr = 0;
    if (sh_smem > sh_attr) {
      cudaFuncSetAttribute(k_preprocess, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_smem);
      sh_attr = sh_smem;
    }
    if (K > 0) k_preprocess<<<(unsigned)ceil_div(K, 256), 256, sh_smem, s>>>(p);
  }

  // tile binning + per-tile depth order (no global sort on the frame path)
  {
    StageTimer st(FS4D_STAGE_BINNING, s);
    bin_tiles_device(L, ws, p.tile_rect, p.dkeys, p.z64, counters, status, s);
  }

  // blend
  BlendArgs b;
  b.H = L.H;
  b.W = L.W;
  b.ntx = L.ntx;
  b.D = cfg.with_features ? L.D : 0;
  b.alpha_cap = (float)cfg.alpha_cap;
  b.alpha_skip = (float)cfg.alpha_skip;
  b.stop = (float)cfg.stop_transmittance;
  b.bg0 = (float)cfg.background[0];
  b.bg1 = (float)cfg.background[1];
  b.bg2 = (float)cfg.background[2];
  b.ranges = at<uint2>(ws, L.ranges);
  b.tperm = L.ntiles <= 65536 ? at<int32_t>(ws, L.tperm) : nullptr;  // written by k_tile_scan_check
  b.pvals = at<uint32_t>(ws, L.pvals0);
  b.xy = p.xy;
  b.conic_o = p.conic_o;
  b.pix_rect = p.pix_rect;
  b.rgbz = p.rgbz;
  b.features = snap.features;
  b.out_color = out.color;
  b.out_depth = out.depth;
  b.out_feature = out.feature;
  b.out_alpha = out.alpha;
  b.out_ncontrib = out.n_contrib;
  b.tfinal = at<float>(ws, L.tfinal);
  b.last = at<int32_t>(ws, L.last);
  if (L.ntiles > 0) {
    StageTimer st(FS4D_STAGE_BLEND, s);
    int c0 = 0;
    do {
      int rem = b.D - c0;
      int dc = rem <= 0 ? 0 : rem <= 4 ? 4 : rem <= 8 ? 8 : rem <= 16 ? 16 : blend_max_dc();
      b.c0 = c0;
      launch_blend(dc, L.ntiles, b, s);
      c0 += dc;
    } while (c0 < b.D);
  }
  return check_launch("render_fwd");
}

// ---------------------------------------------------------------------------
// record export (ProjectedGaussians / tile lists)
// ---------------------------------------------------------------------------
__global__ void k_export_projected(const uint32_t* __restrict__ order, const uint32_t* counters, int64_t K,
                                   const float4* xy, const float4* conic_o, const float4* rgbz, const float4* cov_r,
                                   const int4* tile_rect, Fs4dProjected o) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)counters[CNT_VISIBLE] || r >= K) return;
  const uint32_t i = order[r];
  const float4 m4 = xy[i];
  const float2 m = make_float2(m4.x + m4.z, m4.y + m4.w);
  const float4 co = conic_o[i], cz = rgbz[i], cv = cov_r[i];
  if (o.mean2d) { o.mean2d[2 * r] = m.x; o.mean2d[2 * r + 1] = m.y; }
  if (o.cov2d) { o.cov2d[3 * r] = cv.x; o.cov2d[3 * r + 1] = cv.y; o.cov2d[3 * r + 2] = cv.z; }
  if (o.conic) { o.conic[3 * r] = co.x; o.conic[3 * r + 1] = co.y; o.conic[3 * r + 2] = co.z; }
  if (o.view_depth) o.view_depth[r] = cz.w;
  if (o.radius) o.radius[r] = cv.w;
  if (o.color) { o.color[3 * r] = cz.x; o.color[3 * r + 1] = cz.y; o.color[3 * r + 2] = cz.z; }
  if (o.opacity) o.opacity[r] = co.w;
  if (o.source_index) o.source_index[r] = (int32_t)i;
  if (o.tiles_touched) {
    int4 t = tile_rect[i];
    o.tiles_touched[r] = (t.y - t.x + 1) * (t.w - t.z + 1);
  }
}

// Global stable depth order of the visible set (np.argsort(z, stable),
// rasterizer.py:163) for the record's consumers that need it
// (ProjectedGaussians export, viewspace statistics of the backward):
// radix sort of the fp32 depth bits + fp64 tie fix-up + inverse permutation.
// Idempotent: re-sorting an already sorted sequence is stable.
__global__ void k_rank_of(const uint32_t* __restrict__ order, int64_t K, int32_t* __restrict__ rank_of) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < K) rank_of[order[r]] = (int32_t)r;
}

const uint32_t* depth_order(const RenderLayout& L, void* ws, cudaStream_t s, bool with_rank) {
  const int64_t K = L.K;
  uint32_t* dk[2] = {at<uint32_t>(ws, L.dkeys0), at<uint32_t>(ws, L.dkeys1)};
  uint32_t* dv[2] = {at<uint32_t>(ws, L.dvals0), at<uint32_t>(ws, L.dvals1)};
  StageTimer st(FS4D_STAGE_DEPTH_SORT, s);
  const int df = radix_sort_pairs(dk, dv, K, nullptr, 0, 32, at<void>(ws, L.scratch), s);
  if (df != 0 && K > 0) {  // keep the sorted sequence in buffer 0 so repeated calls are stable
    cudaMemcpyAsync(dk[0], dk[1], (size_t)K * 4, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(dv[0], dv[1], (size_t)K * 4, cudaMemcpyDeviceToDevice, s);
  }
  if (K > 0) {
    k_depth_tie_fixup<<<(unsigned)ceil_div(K, 256), 256, 0, s>>>(dk[0], dv[0], at<double>(ws, L.z64), K,
                                                                 at<uint32_t>(ws, L.counters));
    if (with_rank) k_rank_of<<<(unsigned)ceil_div(K, 256), 256, 0, s>>>(dv[0], K, at<int32_t>(ws, L.rank_of));
  }
  return dv[0];
}

int render_export_projected(const RenderLayout& L, void* ws, Fs4dProjected& out, cudaStream_t s) {
  const uint32_t* dv = depth_order(L, ws, s);
  if (L.K > 0)
    k_export_projected<<<(unsigned)ceil_div(L.K, 256), 256, 0, s>>>(
        dv, at<uint32_t>(ws, L.counters), L.K, at<float4>(ws, L.xy), at<float4>(ws, L.conic_o),
        at<float4>(ws, L.rgbz), at<float4>(ws, L.cov_r), at<int4>(ws, L.tile_rect), out);
  return check_launch("render_export_projected");
}

__global__ void k_export_pairs(const uint32_t* __restrict__ pvals, const int32_t* __restrict__ rank_of,
                               const uint32_t* counters, int32_t* out, int64_t max_pairs) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)counters[CNT_PAIRS_CLAMPED] || p >= max_pairs) return;
  out[p] = rank_of[pvals[p]];
}

int render_export_tiles(const RenderLayout& L, void* ws, int32_t* ranges, int32_t* rows, int64_t max_pairs,
                        cudaStream_t s) {
  if (ranges) cudaMemcpyAsync(ranges, at<void>(ws, L.ranges), (size_t)L.ntiles * 8, cudaMemcpyDeviceToDevice, s);
  if (rows && max_pairs > 0) {
    depth_order(L, ws, s);  // rank_of
    k_export_pairs<<<(unsigned)ceil_div(max_pairs, 256), 256, 0, s>>>(
        at<uint32_t>(ws, L.pvals0), at<int32_t>(ws, L.rank_of), at<uint32_t>(ws, L.counters), rows, max_pairs);
  }
  return check_launch("render_export_tiles");
}

}  // namespace fs4d
