// Deformation forward, fast path:  HexPlane gather kernel + tcgen05 MLP kernel.
//
//   k_hexplane_latent  hexplane.query_with_cache (hexplane.py:118-142): one
//                      warp per 32 Gaussians; lanes first compute their own
//                      Gaussian's 6*levels bilinear cells in fp64 (once, into
//                      shared memory), then sweep the 32 Gaussians with lane =
//                      channel so every corner fetch is a coalesced 128 B row.
//   k_mlp_tc           every MLP stack of deformation.py:105-136 for a tile of
//                      128 Gaussians on the 5th-gen tensor cores: operands in
//                      shared memory (K-major, no-swizzle core-matrix layout),
//                      fp32 accumulators in TMEM (tcgen05.mma kind::f16,
//                      M=128), 3-term bf16 split (hi*hi + hi*lo + lo*hi, rel.
//                      error ~1e-5) so fp32 parity holds; the epilogue of each
//                      layer (tcgen05.ld -> bias -> ReLU -> split -> st.shared)
//                      produces the next layer's A operand in place, and the
//                      last epilogues add the raw-space deltas straight into
//                      the snapshot (deformation.py:126-133).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdlib.h>
#include <string.h>

#include "tc_common.cuh"

namespace fs4d {


// ---------------------------------------------------------------------------
// HexPlane latent
// ---------------------------------------------------------------------------
#ifndef FS4D_GATHER_WARPS
#define FS4D_GATHER_WARPS 4
#endif
constexpr int kGatherWarps = FS4D_GATHER_WARPS;
constexpr int kGatherMaxLevels = 4;

__global__ void __launch_bounds__(kGatherWarps * 32) k_hexplane_latent(TcPlan p, int64_t K, const float* __restrict__ pos,
                                                                         float* __restrict__ latent) {
  __shared__ int s_base[kGatherWarps][kGatherMaxLevels * 6][32];
  __shared__ float s_fa[kGatherWarps][kGatherMaxLevels * 6][32];
  __shared__ float s_fb[kGatherWarps][kGatherMaxLevels * 6][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g0 = ((int64_t)blockIdx.x * kGatherWarps + warp) * 32;
  if (g0 >= K) return;
  const int L = p.L;
  if (!p.enable_grid) {
    for (int j = 0; j < 32 && g0 + j < K; ++j)
      for (int c = lane; c < L; c += 32) latent[(g0 + j) * L + c] = 0.f;
    return;
  }
  // lane j: bilinear cells of Gaussian g0 + j (fp64 coordinates, hexplane.py:84-110)
  {
    const int64_t k = g0 + lane;
    double c[4] = {0.0, 0.0, 0.0, p.t};
    if (k < K) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double raw = ((double)pos[3 * k + a] - p.lo[a]) / p.span[a];
        c[a] = fmin(fmax(raw, 0.0), 1.0);
      }
    }
    for (int l = 0; l < p.levels; ++l)
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int ra = p.res[l][q][0], rb = p.res[l][q][1];
        const double u = c[plane_axis0(q)] * (ra - 1), v = c[plane_axis1(q)] * (rb - 1);
        int i0 = (int)floor(u), j0 = (int)floor(v);
        i0 = min(max(i0, 0), ra - 2);
        j0 = min(max(j0, 0), rb - 2);
        s_base[warp][l * 6 + q][lane] = (i0 * rb + j0) * p.C;
        s_fa[warp][l * 6 + q][lane] = (float)(u - i0);
        s_fb[warp][l * 6 + q][lane] = (float)(v - j0);
      }
  }
  __syncwarp();
  const int C = p.C;
  for (int j = 0; j < 32; ++j) {
    const int64_t k = g0 + j;
    if (k >= K) break;
    for (int l = 0; l < p.levels; ++l) {
      for (int ch = lane; ch < C; ch += 32) {
        float prod = 1.f;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const int rb = p.res[l][q][1];
          const float* pl = p.planes[l][q] + s_base[warp][l * 6 + q][j] + ch;
          const float fa = s_fa[warp][l * 6 + q][j], fb = s_fb[warp][l * 6 + q][j];
          const float p00 = __ldg(pl), p01 = __ldg(pl + C);
          const float p10 = __ldg(pl + rb * C), p11 = __ldg(pl + rb * C + C);
          prod *= (1.f - fa) * (1.f - fb) * p00 + fa * (1.f - fb) * p10 + (1.f - fa) * fb * p01 + fa * fb * p11;
        }
        latent[k * L + l * C + ch] = prod;
      }
    }
  }
}

// 32-channel planes: lane = (Gaussian j%4, channel quad) so one warp
// instruction fetches four corner rows as float4 (4 x 128 B) and interpolates
// 4 channels per lane; 8x fewer load/FMA instructions than lane = channel.
template <int LEVELS>
__global__ void __launch_bounds__(kGatherWarps * 32) k_hexplane_latent_c32(TcPlan p, int64_t K,
                                                                             const float* __restrict__ pos,
                                                                             float* __restrict__ latent) {
  __shared__ int s_base[kGatherWarps][LEVELS * 6][32];
  __shared__ float2 s_f[kGatherWarps][LEVELS * 6][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g0 = ((int64_t)blockIdx.x * kGatherWarps + warp) * 32;
  if (g0 >= K) return;
  {
    const int64_t k = g0 + lane;
    double c[4] = {0.0, 0.0, 0.0, p.t};
    if (k < K) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double raw = ((double)pos[3 * k + a] - p.lo[a]) / p.span[a];
        c[a] = fmin(fmax(raw, 0.0), 1.0);
      }
    }
#pragma unroll
    for (int l = 0; l < LEVELS; ++l)
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int ra = p.res[l][q][0], rb = p.res[l][q][1];
        const double u = c[plane_axis0(q)] * (ra - 1), v = c[plane_axis1(q)] * (rb - 1);
        int i0 = (int)floor(u), j0 = (int)floor(v);
        i0 = min(max(i0, 0), ra - 2);
        j0 = min(max(j0, 0), rb - 2);
        s_base[warp][l * 6 + q][lane] = (i0 * rb + j0) * 32;
        s_f[warp][l * 6 + q][lane] = make_float2((float)(u - i0), (float)(v - j0));
      }
  }
  __syncwarp();
  const int sub = lane >> 3, ch = (lane & 7) * 4;
  for (int j0 = 0; j0 < 32; j0 += 4) {
    const int j = j0 + sub;
    const int64_t k = g0 + j;
#pragma unroll
    for (int l = 0; l < LEVELS; ++l) {
      float4 prod = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int rs = p.res[l][q][1] * 32;
        const float* pl = p.planes[l][q] + s_base[warp][l * 6 + q][j] + ch;
        const float2 f = s_f[warp][l * 6 + q][j];
        const float w00 = (1.f - f.x) * (1.f - f.y), w10 = f.x * (1.f - f.y);
        const float w01 = (1.f - f.x) * f.y, w11 = f.x * f.y;
        const float4 a = __ldg(reinterpret_cast<const float4*>(pl));
        const float4 b = __ldg(reinterpret_cast<const float4*>(pl + 32));
        const float4 c = __ldg(reinterpret_cast<const float4*>(pl + rs));
        const float4 d = __ldg(reinterpret_cast<const float4*>(pl + rs + 32));
        // hexplane.py:105-106 order: (1-fa)(1-fb)p00 + fa(1-fb)p10 + (1-fa)fb p01 + fa fb p11
        prod.x *= w00 * a.x + w10 * c.x + w01 * b.x + w11 * d.x;
        prod.y *= w00 * a.y + w10 * c.y + w01 * b.y + w11 * d.y;
        prod.z *= w00 * a.z + w10 * c.z + w01 * b.z + w11 * d.z;
        prod.w *= w00 * a.w + w10 * c.w + w01 * b.w + w11 * d.w;
      }
      if (k < K) *reinterpret_cast<float4*>(latent + k * 64 + l * 32 + ch) = prod;
    }
  }
}

#ifndef PLANE_LD
#define PLANE_LD __ldg
#endif
// Same gather, with the three time planes of each level read as 1-D lerps of
// the per-frame time rows (k_pack_tc): 2 corner rows instead of 4 for half
// of the planes, and those rows (72 KB at configs[1]) stay L1/L2-hot.  The
// kernel is bound by L2->SM bytes, so this halves the time planes' share.
//
// IMG: instead of fp32 rows, write each Gaussian's latent as bf16 hi / lo
// (the tcgen05 A-operand split) in one 256-byte row [hi 64 x bf16 | lo 64 x
// bf16]: every row is whole 32-byte sectors whatever the visiting order (the
// core-matrix image itself interleaves row pairs in a sector, which under the
// Morton order turns into partial-sector writes and ECC read-modify-writes),
// and the MLP's epilogue threads move the rows into its operand image with
// asynchronous 16-byte copies, never touching them in registers.
// Minimum resident CTAs per SM: 9 (56 registers, as ptxas picks unbounded,
// but scheduled for that occupancy) measured 69.8 -> 65.8 us, twice; 10 (48
// registers) 72 us, 12 spills; an explicit 1 lets ptxas take 118 registers.
#ifndef FS4D_GATHER_MINB
#define FS4D_GATHER_MINB 9
#endif
template <int LEVELS, bool IMG = false>
__global__ void __launch_bounds__(kGatherWarps * 32, FS4D_GATHER_MINB) k_hexplane_latent_c32t(TcPlan p, int64_t K,
                                                                              const float* __restrict__ pos,
                                                                              const float* __restrict__ rows,
                                                                              float* __restrict__ latent,
                                                                              uint8_t* __restrict__ img = nullptr) {
  __shared__ int s_base[kGatherWarps][LEVELS * 6][32];
  __shared__ float2 s_f[kGatherWarps][LEVELS * 6][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g0 = ((int64_t)blockIdx.x * kGatherWarps + warp) * 32;
  if (g0 >= K) return;
  // slot g0 + lane visits Gaussian kg (the optional locality order)
  const int64_t kg = g0 + lane < K ? (p.order ? (int64_t)p.order[g0 + lane] : g0 + lane) : K;
  {
    const int64_t k = kg;
    double c[3] = {0.0, 0.0, 0.0};
    if (k < K) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double raw = ((double)pos[3 * k + a] - p.lo[a]) / p.span[a];
        c[a] = fmin(fmax(raw, 0.0), 1.0);
      }
    }
#pragma unroll
    for (int l = 0; l < LEVELS; ++l)
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int ra = p.res[l][q][0], rb = p.res[l][q][1];
        const double u = c[plane_axis0(q)] * (ra - 1);
        int i0 = (int)floor(u);
        i0 = min(max(i0, 0), ra - 2);
        if (q == 2 || q == 4 || q == 5) {
          s_base[warp][l * 6 + q][lane] = i0 * 32;
          s_f[warp][l * 6 + q][lane] = make_float2((float)(u - i0), 0.f);
        } else {
          const double v = c[plane_axis1(q)] * (rb - 1);
          int j0 = (int)floor(v);
          j0 = min(max(j0, 0), rb - 2);
          s_base[warp][l * 6 + q][lane] = (i0 * rb + j0) * 32;
          s_f[warp][l * 6 + q][lane] = make_float2((float)(u - i0), (float)(v - j0));
        }
      }
  }
  __syncwarp();
  const int sub = lane >> 3, ch = (lane & 7) * 4;
  for (int j0 = 0; j0 < 32; j0 += 4) {
    const int j = j0 + sub;
    const int64_t k = __shfl_sync(0xffffffffu, kg, j);
#pragma unroll
    for (int l = 0; l < LEVELS; ++l) {
      float4 prod = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float2 f = s_f[warp][l * 6 + q][j];
        if (q == 2 || q == 4 || q == 5) {
          const int tq = q == 2 ? 0 : (q == 4 ? 1 : 2);
          const float* rp = rows + p.row_off[l][tq] + s_base[warp][l * 6 + q][j] + ch;
          const float4 a = __ldg(reinterpret_cast<const float4*>(rp));
          const float4 c = __ldg(reinterpret_cast<const float4*>(rp + 32));
          const float wa = 1.f - f.x;
          prod.x *= wa * a.x + f.x * c.x;
          prod.y *= wa * a.y + f.x * c.y;
          prod.z *= wa * a.z + f.x * c.z;
          prod.w *= wa * a.w + f.x * c.w;
        } else {
          const int rs = p.res[l][q][1] * 32;
          const float* pl = p.planes[l][q] + s_base[warp][l * 6 + q][j] + ch;
          const float w00 = (1.f - f.x) * (1.f - f.y), w10 = f.x * (1.f - f.y);
          const float w01 = (1.f - f.x) * f.y, w11 = f.x * f.y;
          const float4 a = PLANE_LD(reinterpret_cast<const float4*>(pl));
          const float4 b = PLANE_LD(reinterpret_cast<const float4*>(pl + 32));
          const float4 c = PLANE_LD(reinterpret_cast<const float4*>(pl + rs));
          const float4 d = PLANE_LD(reinterpret_cast<const float4*>(pl + rs + 32));
          prod.x *= w00 * a.x + w10 * c.x + w01 * b.x + w11 * d.x;
          prod.y *= w00 * a.y + w10 * c.y + w01 * b.y + w11 * d.y;
          prod.z *= w00 * a.z + w10 * c.z + w01 * b.z + w11 * d.z;
          prod.w *= w00 * a.w + w10 * c.w + w01 * b.w + w11 * d.w;
        }
      }
      if (k < K) {
        if (IMG) {  // bf16 hi | lo row (8 lanes x 8 B = one 64 B run per level and half)
          const uint32_t h01 = cvt_bf16x2(prod.x, prod.y), h23 = cvt_bf16x2(prod.z, prod.w);
          const uint32_t l01 =
              cvt_bf16x2(prod.x - __uint_as_float(h01 << 16), prod.y - __uint_as_float(h01 & 0xFFFF0000u));
          const uint32_t l23 =
              cvt_bf16x2(prod.z - __uint_as_float(h23 << 16), prod.w - __uint_as_float(h23 & 0xFFFF0000u));
          uint8_t* rowp = img + k * 256 + (l * 32 + ch) * 2;
          *reinterpret_cast<uint2*>(rowp) = make_uint2(h01, h23);
          *reinterpret_cast<uint2*>(rowp + 128) = make_uint2(l01, l23);
        } else {
          *reinterpret_cast<float4*>(latent + k * 64 + l * 32 + ch) = prod;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// weight packing: fp32 [out,in] -> bf16 hi/lo K-major core-matrix operands
// ---------------------------------------------------------------------------
struct TcSrc {
  const float* w;  // [rows, in] row-major
  int rows, in, row0;
};
struct TcOperand {
  int N, KT, off, nsrc;
  TcSrc src[4];
};
struct TcBias {
  int n, off, nsrc;
  const float* b[4];
  int len[4], at[4];
};
struct TcRowOp {
  const float* plane;  // [Ra, Rb, 32]
  int Ra, Rb, j0, off; // off: float offset into the rows region
  float fb;
};
struct TcPackArgs {
  TcOperand op[FS4D_MAX_TRUNK + 12];
  int nop;
  TcBias bias[FS4D_MAX_TRUNK + 8];
  int nbias;
  TcRowOp row[FS4D_MAX_LEVELS * 3];
  int nrow;
  float* rows;
  uint8_t* blob;
};

// reserved for the time rows in every blob (fixed so workspace sizing does
// not depend on the field): sum over levels of 3 * Ra * 32 floats
constexpr int kTimeRowBytes = 256 * 1024;
constexpr int kTimeQ[3] = {2, 4, 5};  // planes (x,t), (y,t), (z,t) of PLANE_AXES

__global__ void k_pack_tc(TcPackArgs a) {
  const int o = blockIdx.y;
  if (o < a.nop) {
    const TcOperand& op = a.op[o];
    __nv_bfloat16* hi = reinterpret_cast<__nv_bfloat16*>(a.blob + op.off);
    __nv_bfloat16* lo = reinterpret_cast<__nv_bfloat16*>(a.blob + op.off + op.N * op.KT * 2);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < op.N * op.KT; e += gridDim.x * blockDim.x) {
      const int r = e / op.KT, k = e % op.KT;
      float v = 0.f;
      for (int s = 0; s < op.nsrc; ++s) {
        const TcSrc& S = op.src[s];
        if (r >= S.row0 && r < S.row0 + S.rows && k < S.in) v = S.w[(r - S.row0) * S.in + k];
      }
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
      const int off = core_off(r, k, op.KT) / 2;
      hi[off] = h;
      lo[off] = l;
    }
  } else if (o >= a.nop + a.nbias) {
    const TcRowOp& r = a.row[o - a.nop - a.nbias];
    float* dst = a.rows + r.off;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r.Ra * 32; e += gridDim.x * blockDim.x) {
      const int i = e >> 5, c = e & 31;
      const float* src = r.plane + ((int64_t)i * r.Rb + r.j0) * 32 + c;
      dst[e] = (1.f - r.fb) * src[0] + r.fb * src[32];
    }
  } else {
    const TcBias& b = a.bias[o - a.nop];
    float* dst = reinterpret_cast<float*>(a.blob + b.off);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < b.n; e += gridDim.x * blockDim.x) {
      float v = 0.f;
      for (int s = 0; s < b.nsrc; ++s)
        if (e >= b.at[s] && e < b.at[s] + b.len[s]) v = b.b[s][e - b.at[s]];
      dst[e] = v;
    }
  }
}

struct TcArgs {
  TcPlan p;
  int64_t K;
  const float* latent;
  const uint8_t* lat_img;  // two-slot kernel: [K][hi 64 | lo 64] bf16 latent rows (gather IMG output)
  const uint8_t* blob;
  const float* pos;
  const float* rot;
  const float* ls;
  const float* op;
  const float* feat;
  float* o_pos;
  float* o_rot;
  float* o_ls;
  float* o_op;
  float* o_feat;
  uint8_t* cache;  // deform_with_cache activation images (tc_common.cuh), or null
};

// the same 8 values into a cached row image in global memory
__device__ __forceinline__ void cache_split8(uint8_t* img, int KT, int r, int k0, const float* v) {
  uint4 h, l;
  split8(v, h, l);
  const int off = core_off(r, k0, KT);
  *reinterpret_cast<uint4*>(img + off) = h;
  *reinterpret_cast<uint4*>(img + kTcRows * KT * 2 + off) = l;
}

// the bias column block (1, 0, ..., 0) at column `at` of a cached image
__device__ __forceinline__ void cache_ones(uint8_t* img, int KT, int r, int at) {
  const int off = core_off(r, at, KT);
  *reinterpret_cast<uint4*>(img + off) = make_uint4(0x3F80u, 0u, 0u, 0u);
  *reinterpret_cast<uint4*>(img + kTcRows * KT * 2 + off) = make_uint4(0u, 0u, 0u, 0u);
}

// one accumulator region [col, col+n) -> bias -> (relu) -> split -> A operand
// columns [k0, k0+n).  Two threads share a row: `half` takes the even or odd
// 8-column chunks.
__device__ __forceinline__ void epilogue_to_operand(uint32_t tmem_row, int col, int n, const float* bias, bool relu,
                                                    uint8_t* a_base, int KT, int k0, int r, int half,
                                                    uint8_t* cimg = nullptr, int cKT = 0, int ck0 = 0) {
  for (int c = 8 * half; c < n; c += 16) {
    float v[8];
    tmem_ld8(tmem_row + col + c, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] += bias[c + i];
      if (relu) v[i] = fmaxf(v[i], 0.f);
    }
    store_split8(a_base, KT, r, k0 + c, v);
    if (cimg) cache_split8(cimg, cKT, r, ck0 + c, v);
  }
}

// NCH 8-column TMEM chunks at taddr0 + 16 i (one thread's half of a stage),
// all issued before a single tcgen05.wait::ld: one TMEM round trip per stage
// instead of one per chunk.  The empty asm ties keep every use after the wait.
template <int NCH, int STRIDE = 16>
__device__ __forceinline__ void tmem_ld_batch(uint32_t taddr0, float (&v)[NCH][8]) {
  uint32_t r[NCH][8];
#pragma unroll
  for (int i = 0; i < NCH; ++i)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[i][0]), "=r"(r[i][1]), "=r"(r[i][2]), "=r"(r[i][3]), "=r"(r[i][4]), "=r"(r[i][5]),
                   "=r"(r[i][6]), "=r"(r[i][7])
                 : "r"(taddr0 + (uint32_t)STRIDE * i));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    asm volatile("" : "+r"(r[i][0]), "+r"(r[i][1]), "+r"(r[i][2]), "+r"(r[i][3]), "+r"(r[i][4]), "+r"(r[i][5]),
                 "+r"(r[i][6]), "+r"(r[i][7]));
#pragma unroll
    for (int j = 0; j < 8; ++j) v[i][j] = __uint_as_float(r[i][j]);
  }
}

// bias -> relu -> bf16 hi/lo of one loaded chunk into an A operand (+ optional cached image)
__device__ __forceinline__ void chunk_to_operand(float (&v)[8], const float* bias, uint8_t* a_base, int KT, int k0,
                                                 int r, uint8_t* cimg = nullptr, int cKT = 0, int ck0 = 0) {
  const float4 b0 = *reinterpret_cast<const float4*>(bias), b1 = *reinterpret_cast<const float4*>(bias + 4);
  const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};  // 32-byte aligned bias chunk
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i] + bv[i], 0.f);
  store_split8(a_base, KT, r, k0, v);
  if (cimg) cache_split8(cimg, cKT, r, ck0, v);
}

// ---------------------------------------------------------------------------
// warp-specialised variant: warps 0-7 run the epilogues (two threads per TMEM
// lane), warp 8 only issues MMAs.  Epilogue threads never block on each other:
// after each operand chunk they arrive on `opbar` (count 256) and move on;
// the MMA warp waits on it, issues, and commits to `accbar`, which the
// epilogue threads wait on only when they need the accumulators.  The cloud
// rows a tile updates are prefetched at its start.
// ---------------------------------------------------------------------------
constexpr int kTcEpiThreads = 256;
constexpr int kTcWsThreads = kTcEpiThreads + 32;


constexpr int kTcProducerThreads = 128;  // fused variant: 4 HexPlane producer warps
constexpr int kTcFusedThreads = kTcWsThreads + kTcProducerThreads;

// Producer warp pw of the fused kernel: gathers the latent of tile rows
// [32 pw, 32 pw + 32) straight into the bf16 hi/lo A operand Xs.  Lane j first
// selects its own Gaussian's 12 bilinear cells in fp64 (hexplane.py:84-110)
// and keeps them in registers; then, four Gaussians per step, lanes
// (Gaussian j%4, channel quad) fetch float4 corner rows (hexplane.py:118-142).
__device__ __forceinline__ void produce_latent(const TcArgs& a, int64_t tile, uint8_t* Xs, int pw, int lane) {
  const TcPlan& p = a.p;
  const int r0 = pw * 32;
  const int64_t kl = tile * kTcRows + r0 + lane;
  int base[12];
  float fa[12], fb[12];
  {
    double c[4] = {0.0, 0.0, 0.0, p.t};
    if (kl < a.K) {
#pragma unroll
      for (int q = 0; q < 3; ++q) c[q] = fmin(fmax(((double)a.pos[3 * kl + q] - p.lo[q]) / p.span[q], 0.0), 1.0);
    }
#pragma unroll
    for (int l = 0; l < 2; ++l)
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int ra = p.res[l][q][0], rb = p.res[l][q][1];
        const double u = c[plane_axis0(q)] * (ra - 1), v = c[plane_axis1(q)] * (rb - 1);
        int i0 = (int)floor(u), j0 = (int)floor(v);
        i0 = min(max(i0, 0), ra - 2);
        j0 = min(max(j0, 0), rb - 2);
        base[l * 6 + q] = (i0 * rb + j0) * 32;
        fa[l * 6 + q] = (float)(u - i0);
        fb[l * 6 + q] = (float)(v - j0);
      }
  }
  const int sub = lane >> 3, ch = (lane & 7) * 4;
  for (int j0 = 0; j0 < 32; j0 += 4) {
    const int j = j0 + sub, row = r0 + j;
    const bool ok = p.enable_grid && tile * kTcRows + row < a.K;
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      float4 prod = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int idx = l * 6 + q;
        const int b = __shfl_sync(0xffffffffu, base[idx], j);
        const float f0 = __shfl_sync(0xffffffffu, fa[idx], j), f1 = __shfl_sync(0xffffffffu, fb[idx], j);
        if (ok) {
          const int rs = p.res[l][q][1] * 32;
          const float* pl = p.planes[l][q] + b + ch;
          const float w00 = (1.f - f0) * (1.f - f1), w10 = f0 * (1.f - f1), w01 = (1.f - f0) * f1, w11 = f0 * f1;
          const float4 c00 = __ldg(reinterpret_cast<const float4*>(pl));
          const float4 c01 = __ldg(reinterpret_cast<const float4*>(pl + 32));
          const float4 c10 = __ldg(reinterpret_cast<const float4*>(pl + rs));
          const float4 c11 = __ldg(reinterpret_cast<const float4*>(pl + rs + 32));
          prod.x *= w00 * c00.x + w10 * c10.x + w01 * c01.x + w11 * c11.x;
          prod.y *= w00 * c00.y + w10 * c10.y + w01 * c01.y + w11 * c11.y;
          prod.z *= w00 * c00.z + w10 * c10.z + w01 * c01.z + w11 * c11.z;
          prod.w *= w00 * c00.w + w10 * c10.w + w01 * c01.w + w11 * c11.w;
        }
      }
      if (!ok) prod = make_float4(0.f, 0.f, 0.f, 0.f);
      const float v[4] = {prod.x, prod.y, prod.z, prod.w};
      __nv_bfloat16 h[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        h[i] = __float2bfloat16_rn(v[i]);
        lo[i] = __float2bfloat16_rn(v[i] - __bfloat162float(h[i]));
      }
      const int off = core_off(row, l * 32 + ch, 64);
      *reinterpret_cast<uint2*>(Xs + off) = *reinterpret_cast<const uint2*>(h);
      *reinterpret_cast<uint2*>(Xs + kTcRows * 64 * 2 + off) = *reinterpret_cast<const uint2*>(lo);
    }
  }
}

#ifdef FS4D_MLP_TRACE
// debug timeline of CTA 0 (tools/mlp_trace.sh): clock64 << 4 | event
// (MMA warp: 1 operand ready, 2 commit; epilogue thread 0: 3 acc ready, 4 signal)
// (two-slot kernel: who = 2 * slot + {0 MMA, 1 epilogue})
__device__ long long g_mlp_trace[4][512];
__device__ int g_mlp_n[4];
#define MLP_TRACE(who, ev)                                                           \
  if (blockIdx.x == 0) {                                                             \
    const int i_ = g_mlp_n[who]++;                                                   \
    if (i_ < 512) g_mlp_trace[who][i_] = ((long long)clock64() << 4) | (ev);         \
  }
#else
#define MLP_TRACE(who, ev)
#endif

template <bool FUSED, bool CACHE>
__global__ void __launch_bounds__(FUSED ? kTcFusedThreads : kTcWsThreads, 1) k_mlp_tc_ws(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // one operand barrier per hand-off slot of a tile (a thread may run ahead by
  // one slot, so slots must not share a barrier); parity = tile iteration
  constexpr int kSlots = FS4D_MAX_TRUNK + 16;
  __shared__ __align__(8) uint64_t accbar_s, opbar_s[kSlots], xfull_s[2], xempty_s[2];
  __shared__ uint32_t tmem_base_sh;
  const TcPlan& p = a.p;
  uint8_t* W = smem;
  const int wbytes = (p.fwd_bytes + 1023) & ~1023;
  // X: [128 x 64] hi + lo (32 KB) -- two of them in the fused kernel (the
  // producers fill tile i+1's while tile i runs); E: [128 x 128] hi + lo (64 KB)
  uint8_t* Xb[2] = {smem + wbytes, smem + wbytes + (FUSED ? kTcRows * 64 * 4 : 0)};
  uint8_t* E = Xb[1] + kTcRows * 64 * 4;
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool mma_warp = warp == kTcEpiThreads / 32;
  const bool producer = FUSED && warp > kTcEpiThreads / 32;

  if (CACHE && blockIdx.x == 0 && tid == 0) {
    CacheHeader* h = reinterpret_cast<CacheHeader*>(a.cache);
    h->magic = kCacheMagic;
    h->K = a.K;
    h->t = p.t;
  }
  for (int e = tid; e < p.fwd_bytes / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(W)[e] = __ldg(reinterpret_cast<const uint4*>(a.blob) + e);
  const uint32_t accbar = smem_u32(&accbar_s), opbar = smem_u32(&opbar_s[0]);
  const uint32_t xfull = smem_u32(&xfull_s[0]), xempty = smem_u32(&xempty_s[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(accbar));
    for (int j = 0; j < kSlots; ++j)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(opbar + 8 * j), "r"(kTcEpiThreads));
    for (int j = 0; j < 2; ++j) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(xfull + 8 * j), "r"(kTcProducerThreads));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(xempty + 8 * j));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sW = smem_u32(W), sE = smem_u32(E);
  const int64_t ntiles = ceil_div(a.K, kTcRows);

  if (producer) {
    // ------------------------------------------------------------ producers
    uint32_t iter = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
      const int s = iter & 1;
      if (iter >= 2) mbar_wait(xempty + 8 * s, ((iter >> 1) - 1) & 1);
      produce_latent(a, tile, Xb[s], warp - kTcEpiThreads / 32 - 1, tid & 31);
      fence_async_smem();
      mbar_arrive(xfull + 8 * s);
    }
  } else if (mma_warp) {
    // ------------------------------------------------------------ MMA issuer
    // the whole warp runs the issue code (uniform descriptors); an elected
    // lane issues each tcgen05.mma / commit
    uint32_t iter = 0;
    int slot = 0;
    const bool leader = (tid & 31) == 0;
    auto wait_op = [&]() {
      mbar_wait(opbar + 8 * slot, iter & 1);
      ++slot;
      tc_fence_after();
      if (leader) MLP_TRACE(0, 1);
    };
    auto commit = [&]() {
      mma_commit_w(accbar);
      if (leader) MLP_TRACE(0, 2);
    };
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
      slot = 0;
      const int s = FUSED ? (iter & 1) : 0;
      const uint32_t sX = smem_u32(Xb[s]);
      for (int l = 0; l < p.depth; ++l) {
        if (FUSED && l == 0) {  // producers filled X with the latent
          mbar_wait(xfull + 8 * s, (iter >> 1) & 1);
          tc_fence_after();
        } else {
          wait_op();  // X holds the latent / previous trunk output
        }
        gemm_bf16x3_w(tmem + 128, sX, 64, 0, sW + p.off_trunk[l], 64, 0, 64, 4, false);
        commit();
      }
      for (int c = 0; c < 64; c += 16) {  // hidden chunk c -> extractor-0 K step
        wait_op();
        gemm_bf16x3_w(tmem, sX, 64, c, sW + p.off_ext0, 64, c, 128, 1, c > 0);
      }
      commit();
      for (int b = 0; b < 4; ++b) {  // e1 of branch b -> extractor-1
        wait_op();
        gemm_bf16x3_w(tmem + 32 * b, sE, 128, 32 * b, sW + p.off_ext1[b], 32, 0, 32, 2, false);
      }
      commit();
      for (int b = 0; b < 4; ++b) {  // e2 of branch b -> head b and F_feat layer-0 K slice
        wait_op();
        gemm_bf16x3_w(tmem + 128 + 16 * b, sE, 128, 32 * b, sW + p.off_head[b], 32, 0, 16, 2, false);
        if (p.enable_feat) gemm_bf16x3_w(tmem + 192, sE, 128, 32 * b, sW + p.off_f1, 128, 32 * b, 32, 2, b > 0);
      }
      commit();
      if (p.enable_feat) {
        wait_op();  // FF in X
        gemm_bf16x3_w(tmem, sX, 32, 0, sW + p.off_f2, 32, 0, p.DP, 2, false);
        commit();
      }
      wait_op();  // tile finished: TMEM and X free for the next tile
      if (FUSED && leader) mbar_arrive(xempty + 8 * s);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogues
    const int row = tid & (kTcRows - 1), half = tid / kTcRows;
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float* bias_f = reinterpret_cast<const float*>(W);
    uint32_t ph = 0;
    auto wait_acc = [&]() {
      mbar_wait(accbar, ph);
      ph ^= 1;
      tc_fence_after();
      if (tid == 0) MLP_TRACE(1, 3);
    };
    int slot = 0;
    auto signal = [&]() {
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(opbar + 8 * slot);
      ++slot;
      if (tid == 0) MLP_TRACE(1, 4);
    };
    float4 lat[8];
    auto load_latent = [&](int64_t t) {
      if (FUSED) return;
      const int64_t kk = t * kTcRows + row;
      const float4* src = reinterpret_cast<const float4*>(a.latent + (kk < a.K ? kk : 0) * 64 + 32 * half);
#pragma unroll
      for (int c = 0; c < 8; ++c) lat[c] = (t < ntiles && kk < a.K) ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    load_latent(blockIdx.x);
    uint32_t iter = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
      slot = 0;
      uint8_t* X = Xb[FUSED ? (iter & 1) : 0];
      const int64_t k = tile * kTcRows + row;
      const bool valid = k < a.K;
      // prefetch the cloud values this thread updates at the end of the tile
      float cv[7];
      float fv[16];
#pragma unroll
      for (int q = 0; q < 7; ++q) cv[q] = 0.f;
      if (valid) {
        if (half == 0) {
#pragma unroll
          for (int q = 0; q < 3; ++q) cv[q] = a.pos[3 * k + q];
#pragma unroll
          for (int q = 0; q < 4; ++q) cv[3 + q] = a.rot[4 * k + q];
        } else {
#pragma unroll
          for (int q = 0; q < 3; ++q) cv[q] = a.ls[3 * k + q];
          cv[3] = a.op[k];
        }
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int c = 8 * half + 16 * (q / 8) + (q % 8);
        fv[q] = (valid && p.enable_feat && c < p.D && p.DP <= 32) ? a.feat[(int64_t)p.D * k + c] : 0.f;
      }
      uint8_t* ct = CACHE ? a.cache + kCacheHeader + tile * (int64_t)kCacheTileBytes : nullptr;
      if (CACHE) {
        if (half == 0) {
          cache_ones(ct + kCacheLat, kCacheKtLat, row, 64);
          cache_ones(ct + kCacheHid, kCacheKtHid, row, 64);
          cache_ones(ct + kCacheFF, kCacheKtFF, row, 32);
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b) cache_ones(ct + kCacheE1 + b * kCacheE1Bytes, kCacheKtE1, row, 32);
        }
      }
      if (!FUSED) {
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          float v[8] = {lat[c].x, lat[c].y, lat[c].z, lat[c].w, lat[c + 1].x, lat[c + 1].y, lat[c + 1].z, lat[c + 1].w};
          store_split8(X, 64, row, 32 * half + 4 * c, v);
          if (CACHE) cache_split8(ct + kCacheLat, kCacheKtLat, row, 32 * half + 4 * c, v);
        }
        load_latent(tile + gridDim.x);
        signal();
      }
      for (int l = 0; l < p.depth; ++l) {
        wait_acc();
        const float* tb = bias_f + p.off_b_trunk[l] / 4;
        if (l + 1 < p.depth) {
          epilogue_to_operand(tmem_row, 128, 64, tb, true, X, 64, 0, row, half);
          signal();
        } else {
          float v[4][8];
          tmem_ld_batch<4>(tmem_row + 128 + 8 * half, v);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = 16 * i + 8 * half;
            chunk_to_operand(v[i], tb + c, X, 64, c, row, CACHE ? ct + kCacheHid : nullptr, kCacheKtHid, c);
            signal();
          }
        }
      }
      {
        wait_acc();
        float v[8][8];
        tmem_ld_batch<8>(tmem_row + 8 * half, v);
        const float* eb = bias_f + p.off_b_ext0 / 4;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int c = 32 * b + 16 * i + 8 * half;
            chunk_to_operand(v[2 * b + i], eb + c, E, 128, c, row, CACHE ? ct + kCacheE1 + b * kCacheE1Bytes : nullptr,
                             kCacheKtE1, c - 32 * b);
          }
          signal();
        }
      }
      {
        wait_acc();
        float v[8][8];
        tmem_ld_batch<8>(tmem_row + 8 * half, v);
        const float* eb = bias_f + p.off_b_ext1 / 4;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int c = 32 * b + 16 * i + 8 * half;
            chunk_to_operand(v[2 * b + i], eb + c, E, 128, c, row, CACHE ? ct + kCacheE2 : nullptr, kCacheKtE2, c);
          }
          signal();
        }
      }
      wait_acc();
      {
        const float* hb = bias_f + p.off_b_head / 4;
        float d0[4], d1[4];
        tmem_ld4(tmem_row + 128 + 32 * half, d0);
        tmem_ld4(tmem_row + 144 + 32 * half, d1);
        if (valid) {
          if (half == 0) {
#pragma unroll
            for (int q = 0; q < 3; ++q) a.o_pos[3 * k + q] = cv[q] + d0[q] + hb[q];
#pragma unroll
            for (int q = 0; q < 4; ++q) a.o_rot[4 * k + q] = cv[3 + q] + d1[q] + hb[16 + q];
          } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) a.o_ls[3 * k + q] = cv[q] + d0[q] + hb[32 + q];
            a.o_op[k] = cv[3] + d1[0] + hb[48];
          }
        }
      }
      if (p.enable_feat) {
        epilogue_to_operand(tmem_row, 192, 32, bias_f + p.off_b_f1 / 4, true, X, 32, 0, row, half,
                            CACHE ? ct + kCacheFF : nullptr, kCacheKtFF, 0);
        signal();
        wait_acc();
        const float* fb = bias_f + p.off_b_f2 / 4;
        // the first two 16-column chunks use the prefetched fv[] with static
        // indices (no local-memory array); wider feature maps re-read the cloud
#pragma unroll
        for (int qc = 0; qc < 2; ++qc) {
          const int c = 8 * half + 16 * qc;
          if (c >= p.DP) break;
          float v[8];
          tmem_ld8(tmem_row + c, v);
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (c + i < p.D) {
                const float base = p.DP <= 32 ? fv[8 * qc + i] : a.feat[(int64_t)p.D * k + c + i];
                a.o_feat[(int64_t)p.D * k + c + i] = base + v[i] + fb[c + i];
              }
            }
          }
        }
        for (int c = 8 * half + 32; c < p.DP; c += 16) {
          float v[8];
          tmem_ld8(tmem_row + c, v);
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + i < p.D) a.o_feat[(int64_t)p.D * k + c + i] = a.feat[(int64_t)p.D * k + c + i] + v[i] + fb[c + i];
          }
        }
      }
      signal();  // tile done
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------------------
// two-slot variant: two independent tile pipelines per CTA ("slots"), each
// with its own 8 epilogue warps, its own MMA-issuing warp, TMEM columns
// [256 s, 256 s + 256) and one 64 KB operand region in which X (latent,
// hidden, FF; KT 64/32) and E (e1, e2; KT 128) alias -- every write into the
// region follows the wait for the accumulators that are products of the MMAs
// reading its previous contents, so the alias is race-free.  The weights are
// staged once per CTA and shared.  While one slot's epilogue converts
// accumulators, the other slot's MMAs run: tensor pipe and epilogue issue
// overlap instead of alternating (the single-slot chain leaves both idle half
// of the time).  Epilogue warps 0-7 serve slot 0, 8-15 slot 1 (warp % 4 still
// selects the TMEM lane quarter); warps 16 / 17 issue the MMAs of slot 0 / 1
// (tcgen05.commit tracks the issuing thread's MMAs only, so each slot's
// commits see its own MMAs).  Slot s of CTA c takes tiles c + G (2 i + s).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void prefetch_l2(const void* ptr) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}

// operand hand-offs per group of this many chunks / branches (1, 2 or 4):
// fewer, larger hand-offs when the other slot keeps the tensor pipe busy
#ifndef FS4D_MLP_HAND
#define FS4D_MLP_HAND 1
#endif
constexpr int kMlpHand = FS4D_MLP_HAND;
constexpr int kTc2Threads = 2 * kTcWsThreads;
constexpr int kMaxDynSmemBytes = 232448 - 2048;  // 227 KB opt-in, less the kernel's static barriers
constexpr int kTc2Region = kTcRows * 128 * 4;  // E hi + lo: 64 KB
constexpr int kTc2LatOff = kTc2Region / 2;      // the TMA latent image: upper 32 KB of the region
constexpr int kTc2Hand = FS4D_MAX_TRUNK + 16;  // operand hand-offs per tile (upper bound)

struct Tc2Bars {
  uint64_t acc[2], op[2][kTc2Hand], x[2], rfree[2];
};

// TMA: one 8-column block (16 bytes) of 128 latent rows -> 2 KB of shared
// memory, rows contiguous: i.e. one K-adjacent column of core matrices
__device__ __forceinline__ void tma_lat_block(uint32_t dst, const CUtensorMap* map, int c0, int row0, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(row0), "r"(bar)
      : "memory");
}

// MMA issue of slot SL.  Everything the descriptors depend on is a compile-
// time constant, a kernel parameter or a shared-memory symbol address
// (TMEM: this CTA owns all 512 columns, so slot SL starts at column 256 SL;
// the kernel checks the allocator agrees), so ptxas keeps the descriptor
// arithmetic on the uniform datapath instead of moving every operand with
// R2UR under the elected lane (measured ~100 cycles per MMA issue that way).
template <int SL>
__device__ __forceinline__ void mlp2_issue(const TcArgs& a, const CUtensorMap* tmap, Tc2Bars& bars,
                                           const uint8_t* smem) {
  const TcPlan& p = a.p;
  const uint32_t tmem = (uint32_t)(kTmemCols * SL);
  const uint32_t sW = smem_u32(smem);
  const uint32_t sR = sW + (uint32_t)((p.fwd_bytes + 1023) & ~1023) + (uint32_t)(SL * kTc2Region);
  const uint32_t accbar = smem_u32(&bars.acc[SL]), opbar = smem_u32(&bars.op[SL][0]);
  const uint32_t xbar = smem_u32(&bars.x[SL]), rbar = smem_u32(&bars.rfree[SL]);
  const bool leader = (threadIdx.x & 31) == 0;
  const int64_t ntiles = ceil_div(a.K, kTcRows);
  // the latent rows of tile t -> the upper half of the region by TMA: 16
  // column blocks of [128 rows x 16 B] (8 hi, then 8 lo), i.e. the K-major
  // no-swizzle operand with K-adjacent core matrices 2 KB apart (LBO 2048,
  // SBO 128); rows past K are zero-filled by the TMA unit.  The upper half is
  // free as soon as a tile's head / F_feat-0 MMAs have read e2 (FF, the last
  // operand, lives in the lower 16 KB), so the next tile's latent streams in
  // during the F_feat epilogue and the F_feat-1 MMAs.
  const uint32_t sLat = sR + (uint32_t)kTc2LatOff;
  auto load_x = [&](int64_t t) {
    if (leader) {
      mbar_expect_tx(xbar, kTcRows * 64 * 4);
#pragma unroll 1
      for (int cb = 0; cb < 16; ++cb) tma_lat_block(sLat + 2048 * cb, tmap, 8 * cb, (int)(t * kTcRows), xbar);
    }
    __syncwarp();
  };
  if (blockIdx.x + (int64_t)gridDim.x * SL < ntiles) load_x(blockIdx.x + (int64_t)gridDim.x * SL);
  const TcOpnd xA{sLat, (uint32_t)(kTcRows * 64 * 2), 2048u, 128u, 4096u, false};
  uint32_t iter = 0;
  int slot = 0;
  auto wait_op = [&]() {
    mbar_wait(opbar + 8 * slot, iter & 1);
    ++slot;
    tc_fence_after();
    if (leader) MLP_TRACE(2 * SL, 1);
  };
  auto commit = [&]() {
    mma_commit_w(accbar);
    if (leader) MLP_TRACE(2 * SL, 2);
  };
  for (int64_t tile = blockIdx.x + (int64_t)gridDim.x * SL; tile < ntiles; tile += 2 * (int64_t)gridDim.x, ++iter) {
    slot = 0;
    for (int l = 0; l < p.depth; ++l) {
      if (l == 0) {  // the TMA-loaded latent (column-block-major image)
        mbar_wait(xbar, iter & 1);
        tc_fence_after();
        gemm3_w(tmem + 128, xA, opnd_k(sW + p.off_trunk[0], 64, 64, 0), 64, 4, false);
      } else {
        wait_op();  // previous trunk output (64 columns, row-group-major)
        gemm_bf16x3_w(tmem + 128, sR, 64, 0, sW + p.off_trunk[l], 64, 0, 64, 4, false);
      }
      commit();
    }
    for (int c = 0; c < 64; c += 16) {  // hidden chunk c -> extractor-0 K step
      if ((c / 16) % kMlpHand == 0) wait_op();
      gemm_bf16x3_w(tmem, sR, 64, c, sW + p.off_ext0, 64, c, 128, 1, c > 0);
    }
    commit();
    for (int b = 0; b < 4; ++b) {  // e1 of branch b -> extractor-1
      if (b % kMlpHand == 0) wait_op();
      gemm_bf16x3_w(tmem + 32 * b, sR, 128, 32 * b, sW + p.off_ext1[b], 32, 0, 32, 2, false);
    }
    commit();
    for (int b = 0; b < 4; ++b) {  // e2 of branch b -> head b and F_feat layer-0 K slice
      if (b % kMlpHand == 0) wait_op();
      gemm_bf16x3_w(tmem + 128 + 16 * b, sR, 128, 32 * b, sW + p.off_head[b], 32, 0, 16, 2, false);
      if (p.enable_feat) gemm_bf16x3_w(tmem + 192, sR, 128, 32 * b, sW + p.off_f1, 128, 32 * b, 32, 2, b > 0);
    }
    commit();
    // e2 read: the upper half of the region is free once these MMAs complete
    mma_commit_w(rbar);
    {
      const int64_t next = tile + 2 * (int64_t)gridDim.x;
      if (next < ntiles) {
        mbar_wait(rbar, iter & 1);
        load_x(next);
      }
    }
    if (p.enable_feat) {
      wait_op();  // FF in X
      gemm_bf16x3_w(tmem, sR, 32, 0, sW + p.off_f2, 32, 0, p.DP, 2, false);
      commit();
    }
    wait_op();  // tile finished: the epilogue is done with TMEM
    __syncwarp();
  }
}

template <bool CACHE>
__global__ void __launch_bounds__(kTc2Threads, 1) k_mlp_tc_2s(TcArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) Tc2Bars bars;
  __shared__ uint32_t tmem_base_sh;
  const TcPlan& p = a.p;
  uint8_t* W = smem;
  const int wbytes = (p.fwd_bytes + 1023) & ~1023;
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool mma_warp = warp >= 2 * (kTcEpiThreads / 32);
  const int sl = mma_warp ? warp - 2 * (kTcEpiThreads / 32) : warp / (kTcEpiThreads / 32);
  uint8_t* R = smem + wbytes + sl * kTc2Region;

  if (CACHE && blockIdx.x == 0 && tid == 0) {
    CacheHeader* h = reinterpret_cast<CacheHeader*>(a.cache);
    h->magic = kCacheMagic;
    h->K = a.K;
    h->t = p.t;
  }
  for (int e = tid; e < p.fwd_bytes / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(W)[e] = __ldg(reinterpret_cast<const uint4*>(a.blob) + e);
  const uint32_t accbar = smem_u32(&bars.acc[sl]), opbar = smem_u32(&bars.op[sl][0]);
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars.acc[s])));
      for (int j = 0; j < kTc2Hand; ++j)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars.op[s][j])), "r"(kTcEpiThreads / 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars.x[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars.rfree[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(2 * kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int64_t ntiles = ceil_div(a.K, kTcRows);
  const int64_t first = blockIdx.x + (int64_t)gridDim.x * sl, step = 2 * (int64_t)gridDim.x;

  if (tmem_base_sh != 0u) __trap();  // the issuers assume the CTA owns TMEM from column 0
  if (mma_warp) {
    if (sl == 0)
      mlp2_issue<0>(a, &tmap, bars, smem);
    else
      mlp2_issue<1>(a, &tmap, bars, smem);
  } else {
    // ------------------------------------------------------------ epilogues (slot sl)
    const uint32_t tmem = tmem_base_sh + (uint32_t)(kTmemCols * sl);
    const int etid = tid & (kTcEpiThreads - 1);
    const int row = etid & (kTcRows - 1), half = etid / kTcRows;
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float* bias_f = reinterpret_cast<const float*>(W);
    uint32_t ph = 0;
    auto wait_acc = [&]() {
      mbar_wait(accbar, ph);
      ph ^= 1;
      tc_fence_after();
      if (etid == 0) MLP_TRACE(2 * sl + 1, 3);
    };
    int slot = 0;
    // one arrival per warp (count 8): each thread fences its own operand
    // writes, __syncwarp orders the warp's writes before lane 0's release
    // arrive -- 8 instead of 256 serialised arrivals on the barrier word
    auto signal = [&]() {
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(opbar + 8 * slot);
      ++slot;
      if (etid == 0) MLP_TRACE(2 * sl + 1, 4);
    };
    // desynchronise the slots: slot 1 starts once slot 0's first tile is
    // half-way through its chain (its extractor-0 accumulators are ready), so
    // one slot's exposed latencies overlap the other's work instead of both
    // stalling together
    if (sl == 1 && ntiles > 1) {
      mbar_wait(smem_u32(&bars.acc[0]), 0);  // trunk of slot 0's first tile
      mbar_wait(smem_u32(&bars.acc[0]), 1);  // extractor 0 of it
    }
    for (int64_t tile = first; tile < ntiles; tile += step) {
      slot = 0;
      const int64_t k = tile * kTcRows + row;
      const bool valid = k < a.K;
      uint8_t* ct = CACHE ? a.cache + kCacheHeader + tile * (int64_t)kCacheTileBytes : nullptr;
      if (CACHE) {
        if (half == 0) {
          cache_ones(ct + kCacheLat, kCacheKtLat, row, 64);
          cache_ones(ct + kCacheHid, kCacheKtHid, row, 64);
          cache_ones(ct + kCacheFF, kCacheKtFF, row, 32);
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b) cache_ones(ct + kCacheE1 + b * kCacheE1Bytes, kCacheKtE1, row, 32);
        }
      }
      // the cloud values this thread updates at the end of the tile, loaded
      // now so their latency hides behind the tile's MMA chain (and the other
      // slot's work): position + rotation (half 0) or scales + opacity (half
      // 1), and for D = 16 this thread's 8 feature channels as two float4
      float cv[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) cv[q] = 0.f;
      if (valid) {
        if (half == 0) {
#pragma unroll
          for (int q = 0; q < 3; ++q) cv[q] = __ldg(a.pos + 3 * k + q);
#pragma unroll
          for (int q = 0; q < 4; ++q) cv[3 + q] = __ldg(a.rot + 4 * k + q);
        } else {
#pragma unroll
          for (int q = 0; q < 3; ++q) cv[q] = __ldg(a.ls + 3 * k + q);
          cv[3] = __ldg(a.op + k);
        }
      }
      const bool feat16 = p.enable_feat && p.D == 16 &&
                          ((reinterpret_cast<uintptr_t>(a.feat) | reinterpret_cast<uintptr_t>(a.o_feat)) & 15) == 0;
      float4 fq0 = make_float4(0.f, 0.f, 0.f, 0.f), fq1 = fq0;
      if (feat16 && valid) {
        const float4* fr = reinterpret_cast<const float4*>(a.feat + 16 * k + 8 * half);
        fq0 = __ldg(fr);
        fq1 = __ldg(fr + 1);
      } else if (p.enable_feat && valid) {
        prefetch_l2(a.feat + (int64_t)p.D * k);
      }
      for (int l = 0; l < p.depth; ++l) {
        wait_acc();
        if (CACHE && l == 0) {
          // the latent image into the cache (KT 72, row-group-major) from the
          // TMA image (column-block-major); the slot's 256 epilogue threads
          // meet at a named barrier before any of them overwrites the region
          // with the hidden layer
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = 16 * i + 8 * half;
            const int so = kTc2LatOff + (c >> 3) * 2048 + row * 16, co = core_off(row, c, kCacheKtLat);
            *reinterpret_cast<uint4*>(ct + kCacheLat + co) = *reinterpret_cast<const uint4*>(R + so);
            *reinterpret_cast<uint4*>(ct + kCacheLat + kTcRows * kCacheKtLat * 2 + co) =
                *reinterpret_cast<const uint4*>(R + kTcRows * 64 * 2 + so);
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + sl), "r"(kTcEpiThreads) : "memory");
        }
        const float* tb = bias_f + p.off_b_trunk[l] / 4;
        if (l + 1 < p.depth) {
          epilogue_to_operand(tmem_row, 128, 64, tb, true, R, 64, 0, row, half);
          signal();
        } else {
          float v[4][8];
          tmem_ld_batch<4>(tmem_row + 128 + 8 * half, v);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = 16 * i + 8 * half;
            chunk_to_operand(v[i], tb + c, R, 64, c, row, CACHE ? ct + kCacheHid : nullptr, kCacheKtHid, c);
            if ((i + 1) % kMlpHand == 0) signal();
          }
        }
      }
      wait_acc();  // extractor 0 -> e1 (KT 128), two TMEM batches of two branches
      {
        const float* eb = bias_f + p.off_b_ext0 / 4;
#pragma unroll
        for (int bb = 0; bb < 4; bb += 2) {
          float v[4][8];
          tmem_ld_batch<4>(tmem_row + 32 * bb + 8 * half, v);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int b = bb + j;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int c = 32 * b + 16 * i + 8 * half;
              chunk_to_operand(v[2 * j + i], eb + c, R, 128, c, row,
                               CACHE ? ct + kCacheE1 + b * kCacheE1Bytes : nullptr, kCacheKtE1, c - 32 * b);
            }
            if ((b + 1) % kMlpHand == 0) signal();
          }
        }
      }
      wait_acc();  // extractor 1 -> e2
      {
        const float* eb = bias_f + p.off_b_ext1 / 4;
#pragma unroll
        for (int bb = 0; bb < 4; bb += 2) {
          float v[4][8];
          tmem_ld_batch<4>(tmem_row + 32 * bb + 8 * half, v);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int b = bb + j;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int c = 32 * b + 16 * i + 8 * half;
              chunk_to_operand(v[2 * j + i], eb + c, R, 128, c, row, CACHE ? ct + kCacheE2 : nullptr, kCacheKtE2, c);
            }
            if ((b + 1) % kMlpHand == 0) signal();
          }
        }
      }
      wait_acc();
      {
        const float* hb = bias_f + p.off_b_head / 4;
        float d0[4], d1[4];
        tmem_ld4(tmem_row + 128 + 32 * half, d0);
        tmem_ld4(tmem_row + 144 + 32 * half, d1);
        if (valid) {
          if (half == 0) {
#pragma unroll
            for (int q = 0; q < 3; ++q) a.o_pos[3 * k + q] = cv[q] + d0[q] + hb[q];
#pragma unroll
            for (int q = 0; q < 4; ++q) a.o_rot[4 * k + q] = cv[3 + q] + d1[q] + hb[16 + q];
          } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) a.o_ls[3 * k + q] = cv[q] + d0[q] + hb[32 + q];
            a.o_op[k] = cv[3] + d1[0] + hb[48];
          }
        }
      }
      if (feat16) {
        epilogue_to_operand(tmem_row, 192, 32, bias_f + p.off_b_f1 / 4, true, R, 32, 0, row, half,
                            CACHE ? ct + kCacheFF : nullptr, kCacheKtFF, 0);
        signal();
        wait_acc();
        const float* fb = bias_f + p.off_b_f2 / 4 + 8 * half;
        float v[8];
        tmem_ld8(tmem_row + 8 * half, v);
        if (valid) {
          const float4 b0 = *reinterpret_cast<const float4*>(fb), b1 = *reinterpret_cast<const float4*>(fb + 4);
          float4* o = reinterpret_cast<float4*>(a.o_feat + 16 * k + 8 * half);
          o[0] = make_float4(fq0.x + v[0] + b0.x, fq0.y + v[1] + b0.y, fq0.z + v[2] + b0.z, fq0.w + v[3] + b0.w);
          o[1] = make_float4(fq1.x + v[4] + b1.x, fq1.y + v[5] + b1.y, fq1.z + v[6] + b1.z, fq1.w + v[7] + b1.w);
        }
      } else if (p.enable_feat) {
        float fv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int c = 8 * half + 16 * (q / 8) + (q % 8);
          fv[q] = (valid && c < p.D && p.DP <= 32) ? a.feat[(int64_t)p.D * k + c] : 0.f;
        }
        epilogue_to_operand(tmem_row, 192, 32, bias_f + p.off_b_f1 / 4, true, R, 32, 0, row, half,
                            CACHE ? ct + kCacheFF : nullptr, kCacheKtFF, 0);
        signal();
        wait_acc();
        const float* fb = bias_f + p.off_b_f2 / 4;
#pragma unroll
        for (int qc = 0; qc < 2; ++qc) {
          const int c = 8 * half + 16 * qc;
          if (c >= p.DP) break;
          float v[8];
          tmem_ld8(tmem_row + c, v);
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (c + i < p.D) {
                const float base = p.DP <= 32 ? fv[8 * qc + i] : a.feat[(int64_t)p.D * k + c + i];
                a.o_feat[(int64_t)p.D * k + c + i] = base + v[i] + fb[c + i];
              }
            }
          }
        }
        for (int c = 8 * half + 32; c < p.DP; c += 16) {
          float v[8];
          tmem_ld8(tmem_row + c, v);
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + i < p.D) a.o_feat[(int64_t)p.D * k + c + i] = a.feat[(int64_t)p.D * k + c + i] + v[i] + fb[c + i];
          }
        }
      }
      signal();  // tile done
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(0u), "r"(2 * kTmemCols));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool tc_path_ok(const Fs4dDeformNet& n, const Fs4dHexPlane& f) {
  if (n.width != 64 || n.latent_dim != 64 || n.feature_dim > 64 || n.depth < 1 || n.depth > FS4D_MAX_TRUNK)
    return false;
  if (n.enable_grid && !(f.levels * f.channels == 64 && f.levels <= kGatherMaxLevels)) return false;
  return true;
}

static int build_plan(const Fs4dDeformNet& n, const Fs4dHexPlane& f, double t, TcPlan& p, TcPackArgs* pk) {
  memset(&p, 0, sizeof(p));
  p.depth = n.depth;
  p.D = n.feature_dim;
  p.DP = (n.feature_dim + 15) / 16 * 16;
  if (p.DP == 0) p.DP = 16;
  p.enable_feat = n.enable_feature_update;
  p.enable_grid = n.enable_grid;
  p.levels = f.levels;
  p.C = f.channels;
  p.L = 64;
  for (int l = 0; l < FS4D_MAX_LEVELS; ++l)
    for (int q = 0; q < 6; ++q) {
      p.res[l][q][0] = f.res[l][q][0];
      p.res[l][q][1] = f.res[l][q][1];
      p.planes[l][q] = f.planes[l][q];
    }
  for (int a = 0; a < 3; ++a) {
    p.lo[a] = f.aabb[a];
    p.span[a] = f.aabb[3 + a] - f.aabb[a];
  }
  p.order = f.order;
  p.t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  int off = 0, nop = 0, nb = 0;
  auto operand = [&](int N, int KT) {
    int at = off;
    off += N * KT * 2 * 2;
    return at;
  };
  auto src = [](const Fs4dLinear& l, int row0) {
    TcSrc s;
    s.w = l.weight;
    s.rows = l.out_dim;
    s.in = l.in_dim;
    s.row0 = row0;
    return s;
  };
  for (int l = 0; l < n.depth; ++l) {
    p.off_trunk[l] = operand(64, 64);
    if (pk) pk->op[nop++] = TcOperand{64, 64, p.off_trunk[l], 1, {src(n.trunk[l], 0)}};
  }
  p.off_ext0 = operand(128, 64);
  if (pk)
    pk->op[nop++] = TcOperand{128, 64, p.off_ext0, 4,
                              {src(n.ext[0][0], 0), src(n.ext[1][0], 32), src(n.ext[2][0], 64), src(n.ext[3][0], 96)}};
  for (int b = 0; b < 4; ++b) {
    p.off_ext1[b] = operand(32, 32);
    if (pk) pk->op[nop++] = TcOperand{32, 32, p.off_ext1[b], 1, {src(n.ext[b][1], 0)}};
  }
  for (int b = 0; b < 4; ++b) {
    p.off_head[b] = operand(16, 32);
    if (pk) pk->op[nop++] = TcOperand{16, 32, p.off_head[b], 1, {src(n.head[b], 0)}};
  }
  p.off_f1 = operand(32, 128);
  if (pk) pk->op[nop++] = TcOperand{32, 128, p.off_f1, 1, {src(n.feat[0], 0)}};
  p.off_f2 = operand(p.DP, 32);
  if (pk) pk->op[nop++] = TcOperand{p.DP, 32, p.off_f2, 1, {src(n.feat[1], 0)}};
  auto bias = [&](int len) {
    int at = off;
    off += (len * 4 + 15) / 16 * 16;
    return at;
  };
  for (int l = 0; l < n.depth; ++l) {
    p.off_b_trunk[l] = bias(64);
    if (pk) pk->bias[nb++] = TcBias{64, p.off_b_trunk[l], 1, {n.trunk[l].bias}, {64}, {0}};
  }
  p.off_b_ext0 = bias(128);
  if (pk)
    pk->bias[nb++] = TcBias{128, p.off_b_ext0, 4, {n.ext[0][0].bias, n.ext[1][0].bias, n.ext[2][0].bias, n.ext[3][0].bias},
                            {32, 32, 32, 32}, {0, 32, 64, 96}};
  p.off_b_ext1 = bias(128);
  if (pk)
    pk->bias[nb++] = TcBias{128, p.off_b_ext1, 4, {n.ext[0][1].bias, n.ext[1][1].bias, n.ext[2][1].bias, n.ext[3][1].bias},
                            {32, 32, 32, 32}, {0, 32, 64, 96}};
  p.off_b_head = bias(64);
  if (pk)
    pk->bias[nb++] = TcBias{64, p.off_b_head, 4, {n.head[0].bias, n.head[1].bias, n.head[2].bias, n.head[3].bias},
                            {3, 4, 3, 1}, {0, 16, 32, 48}};
  p.off_b_f1 = bias(32);
  if (pk) pk->bias[nb++] = TcBias{32, p.off_b_f1, 1, {n.feat[0].bias}, {32}, {0}};
  p.off_b_f2 = bias(p.DP);
  if (pk) pk->bias[nb++] = TcBias{p.DP, p.off_b_f2, 1, {n.feat[1].bias}, {p.D}, {0}};
  // backward-only images after everything the forward kernel stages
  p.fwd_bytes = (off + 15) / 16 * 16;
  off = p.fwd_bytes;
  const int hoff[4] = {0, 3, 7, 10};
  for (int b = 0; b < 4; ++b) {
    p.off_headT[b] = operand(16, 32);
    if (pk) pk->op[nop++] = TcOperand{16, 32, p.off_headT[b], 1, {src(n.head[b], hoff[b])}};
  }
  p.blob_bytes = (off + 15) / 16 * 16;
  p.off_rows = (p.blob_bytes + 255) / 256 * 256;
  p.ws_bytes = p.off_rows + kTimeRowBytes;
  // time rows (only for the 32-channel gather; Rb >= 2 guaranteed by the field)
  int nrow = 0, rfl = 0;
  p.rows_ok = n.enable_grid && f.channels == 32 && f.levels == 2;
  for (int l = 0; p.rows_ok && l < f.levels; ++l)
    for (int tq = 0; tq < 3; ++tq) {
      const int q = kTimeQ[tq], Ra = f.res[l][q][0], Rb = f.res[l][q][1];
      if ((rfl + Ra * 32) * 4 > kTimeRowBytes || Rb < 2) {
        p.rows_ok = 0;
        break;
      }
      const double v = p.t * (Rb - 1);  // hexplane.py:99-101 on the time axis
      int j0 = (int)floor(v);
      j0 = j0 < 0 ? 0 : (j0 > Rb - 2 ? Rb - 2 : j0);
      p.row_off[l][tq] = rfl;
      if (pk) pk->row[nrow++] = TcRowOp{f.planes[l][q], Ra, Rb, j0, rfl, (float)(v - j0)};
      rfl += Ra * 32;
    }
  if (!p.rows_ok) nrow = 0;
  if (pk) {
    pk->nop = nop;
    pk->nbias = nb;
    pk->nrow = nrow;
  }
  // shared memory: weights + X + E must fit
  const int smem = ((p.fwd_bytes + 1023) & ~1023) + kTcRows * 64 * 4 + kTcRows * 128 * 4;
  if (smem > 227 * 1024) return fail(FS4D_ERR_CONFIG, "tcgen05 MLP weights exceed shared memory");
  return FS4D_OK;
}

#ifdef FS4D_MLP_TRACE
extern "C" int fs4d_debug_mlp_trace(long long* out, int* n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_mlp_trace, sizeof(long long) * 2048);
  cudaMemcpyFromSymbol(n, g_mlp_n, sizeof(int) * 4);
  int z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_mlp_n, z, sizeof(z));
  return 0;
}
#endif

// Field-only plan: the standalone HexPlane query / query_backward
// (hexplane.py:113-187) reuse the deformation's gather and scatter kernels
// with latent rows of levels * channels floats.
int tc_field_plan(const Fs4dHexPlane& f, double t, TcPlan& p) {
  memset(&p, 0, sizeof(p));
  if (f.levels < 1 || f.levels > kGatherMaxLevels)
    return fail(FS4D_ERR_CONFIG, "hexplane query supports 1.." + std::to_string(kGatherMaxLevels) + " levels");
  if (f.channels < 1) return fail(FS4D_ERR_CONFIG, "hexplane channels must be positive");
  p.enable_grid = 1;
  p.levels = f.levels;
  p.C = f.channels;
  p.L = f.levels * f.channels;
  for (int l = 0; l < f.levels; ++l)
    for (int q = 0; q < 6; ++q) {
      p.res[l][q][0] = f.res[l][q][0];
      p.res[l][q][1] = f.res[l][q][1];
      p.planes[l][q] = f.planes[l][q];
      if (f.res[l][q][0] < 2 || f.res[l][q][1] < 2) return fail(FS4D_ERR_CONFIG, "plane resolutions must be >= 2");
      if (!f.planes[l][q]) return fail(FS4D_ERR_CONFIG, "null plane");
    }
  for (int a = 0; a < 3; ++a) {
    p.lo[a] = f.aabb[a];
    p.span[a] = f.aabb[3 + a] - f.aabb[a];
    if (!(p.span[a] > 0.0)) return fail(FS4D_ERR_CONFIG, "aabb must have hi > lo");
  }
  p.order = f.order;
  p.t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);  // hexplane.py:90
  return FS4D_OK;
}

int hexplane_query(const Fs4dHexPlane& f, const float* pos, int64_t K, double t, float* latent, cudaStream_t s) {
  TcPlan p;
  int rc = tc_field_plan(f, t, p);
  if (rc) return rc;
  if (K == 0) return FS4D_OK;
  const unsigned gblocks = (unsigned)ceil_div(K, kGatherWarps * 32);
  if (p.C == 32 && p.levels == 2)
    k_hexplane_latent_c32<2><<<gblocks, kGatherWarps * 32, 0, s>>>(p, K, pos, latent);
  else
    k_hexplane_latent<<<gblocks, kGatherWarps * 32, 0, s>>>(p, K, pos, latent);
  return check_launch("hexplane_query");
}

int tc_build_plan(const Fs4dDeformNet& n, const Fs4dHexPlane& f, double t, TcPlan& p) {
  return build_plan(n, f, t, p, nullptr);
}

int tc_pack(const Fs4dDeformNet& n, const Fs4dHexPlane& f, double t, TcPlan& p, uint8_t* blob, cudaStream_t s) {
  static thread_local TcPackArgs pk;  // large: keep off the stack (host-side, filled per call; per host thread)
  int rc = build_plan(n, f, t, p, &pk);
  if (rc) return rc;
  pk.blob = blob;
  pk.rows = reinterpret_cast<float*>(blob + p.off_rows);
  k_pack_tc<<<dim3(16, pk.nop + pk.nbias + pk.nrow), 256, 0, s>>>(pk);
  return check_launch("deform_tc_pack");
}

bool tc_bwd_ok(const Fs4dDeformNet& n, const Fs4dHexPlane& f) {
  return tc_path_ok(n, f) && n.depth == 1 && n.enable_grid && n.enable_feature_update && n.feature_dim > 0 &&
         n.feature_dim <= 16 && f.levels * f.channels == 64;
}

size_t tc_cache_bytes(const Fs4dDeformNet& n, const Fs4dHexPlane& f, int64_t K) {
  if (!tc_bwd_ok(n, f)) return 0;
  return (size_t)kCacheHeader + (size_t)ceil_div(K, kTcRows) * kCacheTileBytes;
}

size_t tc_workspace_bytes(const Fs4dDeformNet& n, int64_t K) {
  Fs4dHexPlane f;
  memset(&f, 0, sizeof(f));
  TcPlan p;
  build_plan(n, f, 0.0, p, nullptr);
  // forward: latent [K, 64] (fp32 rows, or per-tile operand images of the same
  // size rounded up to whole tiles); backward: d_latent [K, 64] + one
  // weight-gradient partial per SM
  return (size_t)p.ws_bytes + (size_t)ceil_div(K, kTcRows) * kTcRows * 64 * 4 + (size_t)kNumSMs * kPartStride * 4 + 512 +
         (size_t)kTimeParts * kTimePartFloats * 4;
}

// 2-D tensor map over the [K][hi 64 | lo 64] bf16 latent rows: box of 8
// elements (one 16-byte column block) x 128 rows.  The encode entry point comes
// from the driver through the runtime (no -lcuda); maps are cached per
// (address, K) since the workspace rarely moves.
static int lat_tensor_map(const void* base, int64_t K, CUtensorMap* out) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(FS4D_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  thread_local const void* last_base = nullptr;
  thread_local int64_t last_K = -1;
  thread_local CUtensorMap last;
  if (base != last_base || K != last_K) {
    const cuuint64_t dims[2] = {128, (cuuint64_t)K};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {8, (cuuint32_t)kTcRows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&last, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FS4D_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    last_base = base;
    last_K = K;
  }
  *out = last;
  return FS4D_OK;
}

int deform_forward_tc(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                      Fs4dCloud& snap, void* ws, uint8_t* cache, cudaStream_t s) {
  TcPlan p;
  uint8_t* blob = (uint8_t*)ws;
  int rc = tc_pack(net, field, t, p, blob, s);
  if (rc) return rc;
  float* latent = (float*)((char*)ws + p.ws_bytes);
  const int64_t K = cloud.K;
  if (K == 0) return FS4D_OK;
  // The fused variant (HexPlane gather as 4 producer warps inside the MLP
  // kernel, latent never leaves shared memory) is correct but measured slower
  // on B200 (355 vs 228 us at configs[1]): 4 producer warps per SM expose far
  // less memory-level parallelism than the stand-alone gather at full
  // occupancy.  It stays opt-in (FS4D_FUSED_GATHER=1).
  const bool fused = !cache && getenv("FS4D_FUSED_GATHER") && (!p.enable_grid || (p.C == 32 && p.levels == 2));
  const unsigned gblocks = (unsigned)ceil_div(K, kGatherWarps * 32);
  const bool time_rows = p.rows_ok && !getenv("FS4D_NO_TIME_ROWS");
  // two tile pipelines per CTA whenever the weights + two 64 KB regions fit
  // (depth-1 trunk: 94 + 128 KB) and the gather can emit operand images;
  // FS4D_MLP_SLOTS=1 keeps the single-slot kernel
  const int smem2 = ((p.fwd_bytes + 1023) & ~1023) + 2 * kTc2Region;
  static const bool one_slot = getenv("FS4D_MLP_SLOTS") && atoi(getenv("FS4D_MLP_SLOTS")) == 1;
  const bool two_slot = !fused && !one_slot && time_rows && smem2 <= kMaxDynSmemBytes;
  // two-slot path: bf16 hi|lo latent rows (256 B per Gaussian, the size of
  // the fp32 rows) in the latent workspace
  uint8_t* img = reinterpret_cast<uint8_t*>(latent);
  StageTimer st_gather(fused ? -1 : FS4D_STAGE_DEFORM_GATHER, s);
  if (!fused) {
    // FS4D_GATHER_CARVEOUT (A/B knob): shared-memory carveout preference in
    // percent -- fewer resident CTAs for a larger L1 (the plane corners
    // neighbouring Gaussians share)
    static const int carve = getenv("FS4D_GATHER_CARVEOUT") ? atoi(getenv("FS4D_GATHER_CARVEOUT")) : -1;
    static bool carve_set = false;
    if (carve >= 0 && !carve_set) {
      cudaFuncSetAttribute(k_hexplane_latent_c32t<2, true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
      carve_set = true;
    }
    if (two_slot)
      k_hexplane_latent_c32t<2, true><<<gblocks, kGatherWarps * 32, 0, s>>>(
          p, K, cloud.positions, reinterpret_cast<const float*>(blob + p.off_rows), nullptr, img);
    else if (time_rows)
      k_hexplane_latent_c32t<2><<<gblocks, kGatherWarps * 32, 0, s>>>(
          p, K, cloud.positions, reinterpret_cast<const float*>(blob + p.off_rows), latent);
    else if (p.enable_grid && p.C == 32 && p.levels == 2)
      k_hexplane_latent_c32<2><<<gblocks, kGatherWarps * 32, 0, s>>>(p, K, cloud.positions, latent);
    else
      k_hexplane_latent<<<gblocks, kGatherWarps * 32, 0, s>>>(p, K, cloud.positions, latent);
  }
  st_gather.stop();
  StageTimer st_mlp(FS4D_STAGE_DEFORM_MLP, s);
  TcArgs a;
  a.p = p;
  a.K = K;
  a.latent = latent;
  a.lat_img = img;
  a.blob = blob;
  a.pos = cloud.positions;
  a.rot = cloud.rotations;
  a.ls = cloud.log_scales;
  a.op = cloud.opacity_logits;
  a.feat = cloud.features;
  a.o_pos = snap.positions;
  a.o_rot = snap.rotations;
  a.o_ls = snap.log_scales;
  a.o_op = snap.opacity_logits;
  a.o_feat = snap.features;
  a.cache = cache;
  const int smem = ((p.fwd_bytes + 1023) & ~1023) + kTcRows * 64 * 4 * (fused ? 2 : 1) + kTcRows * 128 * 4;
  const int64_t ntiles = ceil_div(K, kTcRows);
  static const int grid_cap = getenv("FS4D_MLP_GRID") ? atoi(getenv("FS4D_MLP_GRID")) : kNumSMs;
  const int grid = (int)(ntiles < grid_cap ? ntiles : grid_cap);
  if (two_slot) {
    CUtensorMap tmap;
    rc = lat_tensor_map(img, K, &tmap);
    if (rc) return rc;
    // as few CTAs as keep the same number of tile rounds per slot: the
    // makespan is ceil(ntiles / (2 grid)) rounds either way, and the SMs this
    // frees run other frames' kernels (1563 tiles: 6 rounds on 131 CTAs
    // instead of 148)
    const int64_t rounds = ceil_div(ntiles, 2 * (int64_t)grid_cap);
    const int64_t g2 = ceil_div(ntiles, 2 * rounds);
    const int grid2 = (int)(g2 < grid_cap ? g2 : grid_cap);
    if (cache) {
      cudaFuncSetAttribute(k_mlp_tc_2s<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
      k_mlp_tc_2s<true><<<grid2, kTc2Threads, smem2, s>>>(a, tmap);
    } else {
      cudaFuncSetAttribute(k_mlp_tc_2s<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
      k_mlp_tc_2s<false><<<grid2, kTc2Threads, smem2, s>>>(a, tmap);
    }
    return check_launch("deform_tc_2s");
  }
  if (fused) {
    cudaFuncSetAttribute(k_mlp_tc_ws<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mlp_tc_ws<true, false><<<grid, kTcFusedThreads, smem, s>>>(a);
  } else if (cache) {
    cudaFuncSetAttribute(k_mlp_tc_ws<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mlp_tc_ws<false, true><<<grid, kTcWsThreads, smem, s>>>(a);
  } else {
    // (a two-slot variant -- two tiles in flight per SM, branch-wise
    // extractors, one epilogue thread per row -- was measured slower on B200,
    // 220 vs 179 us at configs[1]: the chain is bound by epilogue issue, not
    // by MMA latency, and halving the threads per tile lengthens it.)
    // (a variant with four epilogue threads per row, 16 epilogue warps, was
    // measured equal -- 95.6 vs 95.1 us -- so the epilogue is not starved of
    // warps either; kept out.)
    cudaFuncSetAttribute(k_mlp_tc_ws<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mlp_tc_ws<false, false><<<grid, kTcWsThreads, smem, s>>>(a);
  }
  return check_launch("deform_tc");
}

}  // namespace fs4d
