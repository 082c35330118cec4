// Deformation backward, fast path (deformation.deform_backward,
// deformation.py:139-183; numerics.mlp_backward, numerics.py:78-105;
// hexplane.query_backward, hexplane.py:145-187).
//
//   k_mlp_bwd_tc     one persistent CTA per SM walks tiles of 128 Gaussians.
//                    The activations come from the deform_with_cache images
//                    (cp.async.bulk straight into shared memory); every
//                    input-gradient GEMM (dX = dY * W) and weight-gradient
//                    GEMM (dW^T += X^T * dY, K = the tile's Gaussians) runs on
//                    tcgen05 with the 3-term bf16 split.  The weight gradients
//                    of all 15 layers stay resident in TMEM (384 fp32 columns)
//                    for the CTA's whole tile range; the bias gradient of a
//                    layer rides its weight-gradient MMA as the cached
//                    constant-1 input column (lane `in`), except the heads and
//                    F_feat layer 0 (whose inputs fill all 128 lanes), which
//                    are reduced by the epilogue warps.  Epilogue warps (two
//                    threads per Gaussian) apply the ReLU masks, split the
//                    gradients into the next GEMM's operand image and write
//                    dL/dlatent [K, 64].
//   k_reduce_tc_wgrads  sums the per-CTA partials into the [out, in] / [out]
//                    gradient buffers of DeformationNet.param_arrays().
//   k_hexplane_bwd   plane scatter + position gradient from dL/dlatent.
#include <stdlib.h>
#include <string.h>

#include "tc_common.cuh"

namespace fs4d {

__constant__ int c_axes_bwd[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};  // hexplane.py:16

constexpr int kBwdEpiThreads = 256;
constexpr int kBwdThreads = kBwdEpiThreads + 32;
constexpr int kBwdTmemCols = 512;

// TMEM columns: resident weight-gradient accumulators, then per-tile scratch
constexpr int kDwTrunk = 0, kDwExt0 = 64, kDwExt1 = 192, kDwHead = 320, kDwF1 = 336, kDwF2 = 368;
constexpr int kScr = kDwCols;  // 128 scratch columns

// shared-memory regions after the weight blob (bytes).  Phase F (F_feat and
// heads), phase B (branches, one at a time) and the trunk phase reuse space.
constexpr int kRE2 = 0, kRFF = 65536, kRGZ = 86016, kRGD = 94208, kRGFF = 102400;
constexpr int kRHid = 0, kRE1 = 36864, kRGE2 = 57344, kRGE1 = 73728;
constexpr int kRLat = 36864, kRGH = 73728;
constexpr int kRBytes = 118784 + 2048;  // + slack for M = 128 MN-major reads of narrower images

// ReLU gate of 16 consecutive columns c0.. of row r: bit i set iff value > 0
__device__ __forceinline__ uint32_t relu_bits16(const uint8_t* img, int KT, int r, int c0) {
  const uint4 a = *reinterpret_cast<const uint4*>(img + core_off(r, c0, KT));
  const uint4 b = *reinterpret_cast<const uint4*>(img + core_off(r, c0 + 8, KT));
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t lo = w[i] & 0xFFFFu, hi = w[i] >> 16;
    if (lo != 0 && !(lo & 0x8000u)) m |= 1u << (2 * i);
    if (hi != 0 && !(hi & 0x8000u)) m |= 1u << (2 * i + 1);
  }
  return m;
}

// warp sum of v[i] for every i, added by lane 0 into this warp's own shared
// accumulators (one slot row per warp, summed in warp order at the end: the
// bias gradients are reproducible bit for bit)
template <int N>
__device__ __forceinline__ void warp_sum_to_smem(const float* v, float* dst, int lane) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    float s = v[i];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) dst[i] += s;
  }
}

struct BwdArgs {
  TcPlan p;
  int64_t K;
  const uint8_t* blob;
  const uint8_t* cache;
  const float* g_pos;
  const float* g_rot;
  const float* g_ls;
  const float* g_op;
  const float* g_feat;
  float* dlat;   // [K, 64]
  float* wpart;  // [grid][kPartStride]
  int32_t* status;
};

__global__ void __launch_bounds__(kBwdThreads, 1) k_mlp_bwd_tc(BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t accbar_s, ldbar_s;
  __shared__ uint32_t tmem_base_sh;
  // per-warp bias-gradient accumulators: head biases [0, 16), F_feat layer-0
  // biases [16, 48) of each epilogue warp
  __shared__ float sbias_w[kBwdEpiThreads / 32][64];
  const TcPlan& p = a.p;
  const int wbytes = (p.blob_bytes + 1023) & ~1023;
  uint8_t* W = smem;
  uint8_t* R = smem + wbytes;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the MMA warp runs the issue code warp-wide (uniform descriptors, one
  // elected lane issues); TMA bulk copies stay single-lane
  const bool issuer = warp == kBwdEpiThreads / 32;
  const bool epi = tid < kBwdEpiThreads;

  for (int e = tid; e < p.blob_bytes / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(W)[e] = __ldg(reinterpret_cast<const uint4*>(a.blob) + e);
  for (int e = tid; e < (kBwdEpiThreads / 32) * 64; e += blockDim.x) (&sbias_w[0][0])[e] = 0.f;
  const uint32_t accbar = smem_u32(&accbar_s), ldbar = smem_u32(&ldbar_s);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(accbar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ldbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const CacheHeader* h = reinterpret_cast<const CacheHeader*>(a.cache);
    if (blockIdx.x == 0 && (h->magic != kCacheMagic || h->K != a.K || h->t != p.t))
      raise_status(a.status, FS4D_ERR_CONTRACT);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kBwdTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sW = smem_u32(W), sR = smem_u32(R);
  auto sync_all = [&]() {
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };

  // operand views that do not depend on the tile
  const TcOpnd wF2 = opnd_mn(sW + p.off_f2, p.DP, 32, 0);  // N = 32 inputs, K = D outputs
  const int row = tid & (kTcRows - 1), half = (tid >> 7) & 1;
  const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);

  const int64_t ntiles = ceil_div(a.K, kTcRows);
  bool first = true;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint8_t* ct = a.cache + kCacheHeader + tile * (int64_t)kCacheTileBytes;
    const int64_t k = tile * kTcRows + row;
    const bool valid = k < a.K;
    const bool acc = !first;
    // ------------------------------------------------ phase F: F_feat + heads
    if (issuer) {
      if (lane == 0) mbar_expect_tx(ldbar, 65536 + 20480);
      if (lane == 0) bulk_g2s(sR + kRE2, ct + kCacheE2, 65536, ldbar);
      if (lane == 0) bulk_g2s(sR + kRFF, ct + kCacheFF, 20480, ldbar);
    }
    if (epi) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = 8 * half + i;
        v[i] = (valid && c < p.D) ? a.g_feat[(int64_t)p.D * k + c] : 0.f;
      }
      store_split8(R + kRGZ, 16, row, 8 * half, v);
      // delta gradients in head order: position 3, rotation 4, scale 3, opacity 1
      if (half == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) v[i] = valid ? a.g_pos[3 * k + i] : 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) v[3 + i] = valid ? a.g_rot[4 * k + i] : 0.f;
        v[7] = valid ? a.g_ls[3 * k] : 0.f;
      } else {
        v[0] = valid ? a.g_ls[3 * k + 1] : 0.f;
        v[1] = valid ? a.g_ls[3 * k + 2] : 0.f;
        v[2] = valid ? a.g_op[k] : 0.f;
#pragma unroll
        for (int i = 3; i < 8; ++i) v[i] = 0.f;
      }
      store_split8(R + kRGD, 16, row, 8 * half, v);
      warp_sum_to_smem<8>(v, sbias_w[warp] + 8 * half, lane);
    }
    sync_all();
    if (issuer) {
      mbar_wait(ldbar, 0);
      tc_fence_after();
      // dL/dFF = dL/dz * W_f2 (numerics.py:102), dW_f2^T += FF^T dL/dz
      gemm3_w(tmem + kScr, opnd_k(sR + kRGZ, 128, 16, 0), wF2, 32, 1, false);
      gemm3_w(tmem + kDwF2, opnd_mn(sR + kRFF, 128, kCacheKtFF, 0), opnd_mn(sR + kRGZ, 128, 16, 0), p.DP, 8, acc);
      mma_commit_w(accbar);
    }
    uint64_t m2 = 0;  // ReLU gates of this thread's E2 columns: bit 16b+i = column 32b + 16 half + i
    if (epi) {
      mbar_wait(accbar, 0);
      tc_fence_after();
      mbar_wait(ldbar, 0);
      float g[16];
      tmem_ld16(tmem_row + kScr + 16 * half, g);
      const uint32_t mf = relu_bits16(R + kRFF, kCacheKtFF, row, 16 * half);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (!((mf >> i) & 1u)) g[i] = 0.f;
      store_split8(R + kRGFF, 32, row, 16 * half, g);
      store_split8(R + kRGFF, 32, row, 16 * half + 8, g + 8);
      warp_sum_to_smem<16>(g, sbias_w[warp] + 16 + 16 * half, lane);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        m2 |= (uint64_t)relu_bits16(R + kRE2, kCacheKtE2, row, 32 * b + 16 * half) << (16 * b);
    }
    sync_all();
    auto issue_ge2 = [&](int b) {
      // dL/de2_b = dL/dFF * W_f1[:, 32b:32b+32] + dL/ddelta_b * W_head_b (deformation.py:157-177)
      gemm3_w(tmem + kScr, opnd_k(sR + kRGFF, 128, 32, 0), opnd_mn(sW + p.off_f1, 32, 128, 32 * b), 32, 2, false);
      gemm3_w(tmem + kScr, opnd_k(sR + kRGD, 128, 16, 0), opnd_mn(sW + p.off_headT[b], 16, 32, 0), 32, 1, true);
    };
    if (issuer) {
      const TcOpnd e2 = opnd_mn(sR + kRE2, 128, kCacheKtE2, 0);
      gemm3_w(tmem + kDwF1, e2, opnd_mn(sR + kRGFF, 128, 32, 0), 32, 8, acc);
      gemm3_w(tmem + kDwHead, e2, opnd_mn(sR + kRGD, 128, 16, 0), 16, 8, acc);
      issue_ge2(0);
      mma_commit_w(accbar);
      mbar_wait(accbar, 1);  // E2 no longer read: load the hidden layer and branch 0's e1
      if (lane == 0) mbar_expect_tx(ldbar, 36864 + kCacheE1Bytes);
      if (lane == 0) bulk_g2s(sR + kRHid, ct + kCacheHid, 36864, ldbar);
      if (lane == 0) bulk_g2s(sR + kRE1, ct + kCacheE1, kCacheE1Bytes, ldbar);
    }
    auto epi_ge2 = [&](int b) {
      float g[16];
      tmem_ld16(tmem_row + kScr + 16 * half, g);
      const uint32_t m = (uint32_t)(m2 >> (16 * b)) & 0xFFFFu;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (!((m >> i) & 1u)) g[i] = 0.f;
      store_split8(R + kRGE2, 32, row, 16 * half, g);
      store_split8(R + kRGE2, 32, row, 16 * half + 8, g + 8);
    };
    if (epi) {
      mbar_wait(accbar, 1);
      tc_fence_after();
      epi_ge2(0);
    }
    sync_all();
    // ------------------------------------------------ phase B: one branch at a time
    for (int b = 0; b < 4; ++b) {
      if (issuer) {
        mbar_wait(ldbar, (1 + b) & 1);
        tc_fence_after();
        // dL/de1_b = dL/de2_b * W_ext1_b; dW_ext1_b^T += e1_b^T dL/de2_b
        gemm3_w(tmem + kScr + 32, opnd_k(sR + kRGE2, 128, 32, 0), opnd_mn(sW + p.off_ext1[b], 32, 32, 0), 32, 2, false);
        gemm3_w(tmem + kDwExt1 + 32 * b, opnd_mn(sR + kRE1, 128, kCacheKtE1, 0), opnd_mn(sR + kRGE2, 128, 32, 0), 32, 8,
              acc);
        if (b < 3) issue_ge2(b + 1);
        mma_commit_w(accbar);
      }
      if (epi) {
        mbar_wait(accbar, (2 + b) & 1);
        tc_fence_after();
        mbar_wait(ldbar, (1 + b) & 1);
        float g[16];
        tmem_ld16(tmem_row + kScr + 32 + 16 * half, g);
        const uint32_t m = relu_bits16(R + kRE1, kCacheKtE1, row, 16 * half);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (!((m >> i) & 1u)) g[i] = 0.f;
        store_split8(R + kRGE1, 32, row, 16 * half, g);
        store_split8(R + kRGE1, 32, row, 16 * half + 8, g + 8);
        if (b < 3) epi_ge2(b + 1);
      }
      sync_all();
      if (issuer) {
        // dL/dhidden += dL/de1_b * W_ext0_b; dW_ext0_b^T += hidden^T dL/de1_b
        gemm3_w(tmem + kScr + 64, opnd_k(sR + kRGE1, 128, 32, 0), opnd_mn(sW + p.off_ext0, 128, 64, 0, 32 * b), 64, 2,
              b > 0);
        gemm3_w(tmem + kDwExt0 + 32 * b, opnd_mn(sR + kRHid, 128, kCacheKtHid, 0), opnd_mn(sR + kRGE1, 128, 32, 0), 32,
              8, acc);
        if (b < 3) {
          if (lane == 0) mbar_expect_tx(ldbar, kCacheE1Bytes);
          if (lane == 0) bulk_g2s(sR + kRE1, ct + kCacheE1 + (b + 1) * kCacheE1Bytes, kCacheE1Bytes, ldbar);
        }
      }
    }
    // ------------------------------------------------ trunk
    if (issuer) {
      mma_commit_w(accbar);
      mbar_wait(accbar, 0);
      if (lane == 0) mbar_expect_tx(ldbar, 36864);
      if (lane == 0) bulk_g2s(sR + kRLat, ct + kCacheLat, 36864, ldbar);
    }
    if (epi) {
      mbar_wait(accbar, 0);
      tc_fence_after();
      const uint32_t m0 = relu_bits16(R + kRHid, kCacheKtHid, row, 32 * half);
      const uint32_t m1 = relu_bits16(R + kRHid, kCacheKtHid, row, 32 * half + 16);
      float g[16];
      tmem_ld16(tmem_row + kScr + 64 + 32 * half, g);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (!((m0 >> i) & 1u)) g[i] = 0.f;
      store_split8(R + kRGH, 64, row, 32 * half, g);
      store_split8(R + kRGH, 64, row, 32 * half + 8, g + 8);
      tmem_ld16(tmem_row + kScr + 64 + 32 * half + 16, g);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (!((m1 >> i) & 1u)) g[i] = 0.f;
      store_split8(R + kRGH, 64, row, 32 * half + 16, g);
      store_split8(R + kRGH, 64, row, 32 * half + 24, g + 8);
    }
    sync_all();
    if (issuer) {
      mbar_wait(ldbar, 1);
      tc_fence_after();
      // dL/dlatent = dL/dh0 * W_trunk; dW_trunk^T += latent^T dL/dh0
      gemm3_w(tmem + kScr, opnd_k(sR + kRGH, 128, 64, 0), opnd_mn(sW + p.off_trunk[0], 64, 64, 0), 64, 4, false);
      gemm3_w(tmem + kDwTrunk, opnd_mn(sR + kRLat, 128, kCacheKtLat, 0), opnd_mn(sR + kRGH, 128, 64, 0), 64, 8, acc);
      mma_commit_w(accbar);
    }
    if (epi) {
      mbar_wait(accbar, 1);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float g[16];
        tmem_ld16(tmem_row + kScr + 32 * half + 16 * h, g);
        if (valid) {
          float4* dst = reinterpret_cast<float4*>(a.dlat + k * 64 + 32 * half + 16 * h);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
        }
      }
    }
    sync_all();
    first = false;
  }
  // resident weight gradients -> this CTA's partial, [column][lane]
  if (epi) {
    float* part = a.wpart + (int64_t)blockIdx.x * kPartStride;
    for (int c = (kDwCols / 2) * half; c < (kDwCols / 2) * (half + 1); c += 16) {
      float v[16];
      tmem_ld16(tmem_row + c, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) part[(c + i) * kTcRows + row] = v[i];
    }
    if (tid < 48) {
      float sb = 0.f;
#pragma unroll
      for (int w = 0; w < kBwdEpiThreads / 32; ++w) sb += sbias_w[w][tid];
      part[kDwCols * kTcRows + tid] = sb;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kBwdTmemCols));
}

// ---------------------------------------------------------------------------
// partial reduction into DeformationNet gradient buffers
// ---------------------------------------------------------------------------
struct DwMap {
  float* gw;  // [out, in]
  float* gb;  // [out]
  int out, in, col0, lane0, bias_lane, bias_tail;
};
constexpr int kNumDwMaps = 15;
struct DwReduceArgs {
  DwMap m[kNumDwMaps];
  const float* wpart;
  int nparts;
  int accumulate;
};

// 32 consecutive gradient entries per block iteration; the 8 warps split the
// partials (warp g sums parts g, g+8, ... in two interleaved chains) so each
// thread has ~nparts/8 independent coalesced loads in flight instead of one
// serial chain of nparts; the 8 warp sums are added in a fixed order
// (run-to-run deterministic).
constexpr int kRedGroups = 8;
__device__ __forceinline__ float sum_parts(const float* wpart, int64_t stride, int nparts, int src, int g) {
  float s0 = 0.f, s1 = 0.f;
  int q = g;
  for (; q + kRedGroups < nparts; q += 2 * kRedGroups) {
    s0 += wpart[(int64_t)q * stride + src];
    s1 += wpart[(int64_t)(q + kRedGroups) * stride + src];
  }
  if (q < nparts) s0 += wpart[(int64_t)q * stride + src];
  return s0 + s1;
}

__global__ void __launch_bounds__(32 * kRedGroups) k_reduce_tc_wgrads(DwReduceArgs a) {
  __shared__ float part[kRedGroups][33];
  const DwMap& m = a.m[blockIdx.y];
  const int nw = m.out * m.in, ne = nw + m.out;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int e0 = blockIdx.x * 32; e0 < ne; e0 += gridDim.x * 32) {
    const int e = e0 + lane;
    int src = 0;
    float* dst = nullptr;
    if (e < nw) {
      const int o = e / m.in, i = e % m.in;
      src = (m.col0 + o) * kTcRows + m.lane0 + i;
      dst = m.gw + e;
    } else if (e < ne) {
      const int o = e - nw;
      src = m.bias_lane >= 0 ? (m.col0 + o) * kTcRows + m.bias_lane : kDwCols * kTcRows + m.bias_tail + o;
      dst = m.gb + o;
    }
    part[g][lane] = dst ? sum_parts(a.wpart, kPartStride, a.nparts, src, g) : 0.f;
    __syncthreads();
    if (g == 0 && dst) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kRedGroups; ++w) s += part[w][lane];
      *dst = a.accumulate ? *dst + s : s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// HexPlane backward (hexplane.py:145-187): one warp per Gaussian, lanes over
// channels; prefix/suffix products, 4-corner scatter, bilinear derivatives.
// ---------------------------------------------------------------------------
struct HexBwdArgs {
  TcPlan p;
  int64_t K;
  const float* pos;
  const float* dlat;
  const float* g_pos;
  float* cg_pos;
  float* gplanes[FS4D_MAX_LEVELS][6];
  int accumulate;
  // deterministic mode: int64 fixed-point accumulators per plane (integer
  // adds commute, so the scatter order no longer matters) and the scale of
  // each plane (det_scales)
  unsigned long long* dacc[FS4D_MAX_LEVELS][6];
  const double* dscale;
};

// v * scale rounded to an integer and added to a two's-complement int64 cell
__device__ __forceinline__ void det_add(unsigned long long* cell, float v, double scale) {
  const long long q = __double2ll_rn((double)v * scale);
  if (q) atomicAdd(cell, (unsigned long long)q);
}

constexpr int kHexBwdWarps = 8;

template <bool DET = false>
__global__ void __launch_bounds__(kHexBwdWarps * 32) k_hexplane_bwd(HexBwdArgs a) {
  const TcPlan& p = a.p;
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * kHexBwdWarps + (threadIdx.x >> 5);
  if (k >= a.K) return;
  const int C = p.C;
  double c[4] = {0.0, 0.0, 0.0, p.t};
  bool inside[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double raw = ((double)a.pos[3 * k + q] - p.lo[q]) / p.span[q];
    inside[q] = raw > 0.0 && raw < 1.0;
    c[q] = fmin(fmax(raw, 0.0), 1.0);
  }
  float dco[4] = {0.f, 0.f, 0.f, 0.f};
  for (int l = 0; l < p.levels; ++l) {
    int base[6], rs[6];
    float fa[6], fb[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int ra = p.res[l][q][0], rb = p.res[l][q][1];
      const double u = c[c_axes_bwd[q][0]] * (ra - 1), v = c[c_axes_bwd[q][1]] * (rb - 1);
      int i0 = (int)floor(u), j0 = (int)floor(v);
      i0 = min(max(i0, 0), ra - 2);
      j0 = min(max(j0, 0), rb - 2);
      base[q] = (i0 * rb + j0) * C;
      rs[q] = rb * C;
      fa[q] = (float)(u - i0);
      fb[q] = (float)(v - j0);
    }
    float sa[6], sb[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sa[q] = sb[q] = 0.f;
    for (int ch = lane; ch < C; ch += 32) {
      float s[6], d_a[6], d_b[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float* pl = p.planes[l][q] + base[q] + ch;
        const float p00 = __ldg(pl), p01 = __ldg(pl + C), p10 = __ldg(pl + rs[q]), p11 = __ldg(pl + rs[q] + C);
        s[q] = (1.f - fa[q]) * (1.f - fb[q]) * p00 + fa[q] * (1.f - fb[q]) * p10 + (1.f - fa[q]) * fb[q] * p01 +
               fa[q] * fb[q] * p11;
        d_a[q] = (1.f - fb[q]) * (p10 - p00) + fb[q] * (p11 - p01);
        d_b[q] = (1.f - fa[q]) * (p01 - p00) + fa[q] * (p11 - p10);
      }
      float pre[6], suf[6];
      pre[0] = 1.f;
#pragma unroll
      for (int q = 1; q < 6; ++q) pre[q] = pre[q - 1] * s[q - 1];
      suf[5] = 1.f;
#pragma unroll
      for (int q = 4; q >= 0; --q) suf[q] = suf[q + 1] * s[q + 1];
      const float up = a.dlat[k * p.L + l * C + ch];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float coef = up * pre[q] * suf[q];
        if (coef != 0.f) {
          if (DET) {
            unsigned long long* gp = a.dacc[l][q] + base[q] + ch;
            const double sc = a.dscale[l * 6 + q];
            det_add(gp, coef * (1.f - fa[q]) * (1.f - fb[q]), sc);
            det_add(gp + rs[q], coef * fa[q] * (1.f - fb[q]), sc);
            det_add(gp + C, coef * (1.f - fa[q]) * fb[q], sc);
            det_add(gp + rs[q] + C, coef * fa[q] * fb[q], sc);
          } else {
            float* gp = a.gplanes[l][q] + base[q] + ch;
            red_add(gp, coef * (1.f - fa[q]) * (1.f - fb[q]));
            red_add(gp + rs[q], coef * fa[q] * (1.f - fb[q]));
            red_add(gp + C, coef * (1.f - fa[q]) * fb[q]);
            red_add(gp + rs[q] + C, coef * fa[q] * fb[q]);
          }
        }
        sa[q] += coef * d_a[q];
        sb[q] += coef * d_b[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        sa[q] += __shfl_xor_sync(0xffffffffu, sa[q], off);
        sb[q] += __shfl_xor_sync(0xffffffffu, sb[q], off);
      }
      dco[c_axes_bwd[q][0]] += sa[q] * (float)(p.res[l][q][0] - 1);
      dco[c_axes_bwd[q][1]] += sb[q] * (float)(p.res[l][q][1] - 1);
    }
  }
  if (lane < 3) {
    const float d = inside[lane] ? (float)((double)dco[lane] / p.span[lane]) : 0.f;
    a.cg_pos[3 * k + lane] = (a.accumulate ? a.cg_pos[3 * k + lane] : 0.f) + (a.g_pos ? a.g_pos[3 * k + lane] : 0.f) + d;
  }
}

// 32-channel, 2-level planes (configs[1..4]).  One warp per 32 Gaussians:
// lane j first selects Gaussian j's 12 bilinear cells in fp64 (kept in
// registers, fetched by shuffle), then four Gaussians at a time lanes
// (Gaussian, channel quad) fetch float4 corner rows.  The three time planes
// of a level share one t row pair for every Gaussian, so their scatter is
// reduced per CTA in shared memory over the spatial index only ([Ra][32]
// per plane, the (1-fb, fb) split applied once at the flush); the spatial
// planes scatter with red.global.add.v4.f32.
constexpr int kHexC32Warps = 8;
struct HexC32Args {
  HexBwdArgs h;
  const float* rows;  // the frame's time rows (k_pack_tc), or null: bilinear time-plane gathers
  int toff[2][3];  // offsets (floats) of the time-plane accumulators inside a CTA's partial
  int tfloats;
  float* tpart;    // [grid][tfloats] per-CTA time-plane partials (global, zeroed by the host)
  unsigned long long* tpart_i;  // deterministic mode: the same partials in int64 fixed point
};

__host__ __device__ __forceinline__ bool is_time_plane(int q) { return q == 2 || q == 4 || q == 5; }


// Time planes: every Gaussian of a frame hits the same t row pair, so their
// gradients collapse onto Ra spatial rows per plane.  They accumulate with
// fire-and-forget red.global.add.v4 into a per-CTA partial (no cross-CTA
// contention; a shared-memory float atomic is a CAS loop on sm_100), reduced
// by k_time_partials afterwards.
#ifndef FS4D_HEX_BWD_MINB
#define FS4D_HEX_BWD_MINB 2  // measured: 1 -> 248 us, 2 -> 240 us (128 registers, small spill)
#endif
template <bool DET = false>
__global__ void __launch_bounds__(kHexC32Warps * 32, FS4D_HEX_BWD_MINB) k_hexplane_bwd_c32(HexC32Args A) {
  const HexBwdArgs& a = A.h;
  const TcPlan& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* tacc = DET ? nullptr : A.tpart + (int64_t)blockIdx.x * A.tfloats;
  unsigned long long* tacc_i = DET ? A.tpart_i + (int64_t)blockIdx.x * A.tfloats : nullptr;
  // the shared t cell of each level (hexplane.py:95-110 on the time axis)
  int tj0[2];
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int rt = p.res[l][2][1];
    const double v = p.t * (rt - 1);
    int j0 = (int)floor(v);
    j0 = min(max(j0, 0), rt - 2);
    tj0[l] = j0;
  }
  const int sub = lane >> 3, ch = (lane & 7) * 4;
  const int64_t nchunks = ceil_div(a.K, 32);
  for (int64_t chunk = (int64_t)blockIdx.x * kHexC32Warps + warp; chunk < nchunks;
       chunk += (int64_t)gridDim.x * kHexC32Warps) {
    const int64_t g0 = chunk * 32;
    // lane j: cells of Gaussian g0 + j (fp64 coordinates, hexplane.py:84-110)
    int cell[12];  // spatial planes: element offset of corner 00; time planes: i0
    float fa[12], fb[12];
    uint32_t inside = 0;
    {
      const int64_t kl = g0 + lane;
      double c[4] = {0.0, 0.0, 0.0, p.t};
      if (kl < a.K) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double raw = ((double)a.pos[3 * kl + q] - p.lo[q]) / p.span[q];
          if (raw > 0.0 && raw < 1.0) inside |= 1u << q;
          c[q] = fmin(fmax(raw, 0.0), 1.0);
        }
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
          cell[l * 6 + q] = is_time_plane(q) ? i0 : (i0 * rb + j0) * 32;
          fa[l * 6 + q] = (float)(u - i0);
          fb[l * 6 + q] = (float)(v - j0);
        }
    }
    for (int jj = 0; jj < 32; jj += 4) {
      const int j = jj + sub;
      const int64_t k = g0 + j;
      const bool ok = k < a.K;
      float dco[3] = {0.f, 0.f, 0.f};
      // issue this Gaussian's upstream latent gradient and position-gradient
      // loads before the plane gathers so their latency overlaps them
      float4 up_l[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
      float gpos_in = 0.f, cpos_in = 0.f;
      if (ok) {
        up_l[0] = __ldg(reinterpret_cast<const float4*>(a.dlat + k * 64 + ch));
        up_l[1] = __ldg(reinterpret_cast<const float4*>(a.dlat + k * 64 + 32 + ch));
        if ((lane & 7) < 3) {
          gpos_in = a.g_pos[3 * k + (lane & 7)];
          if (a.accumulate) cpos_in = a.cg_pos[3 * k + (lane & 7)];
        }
      }
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        float4 s[6], da[6], db[6];
        float w_a[6], w_b[6];
        int cb[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const int idx = l * 6 + q;
          const int rb = p.res[l][q][1];
          const int cj = __shfl_sync(0xffffffffu, cell[idx], j);
          w_a[q] = __shfl_sync(0xffffffffu, fa[idx], j);
          w_b[q] = __shfl_sync(0xffffffffu, fb[idx], j);
          cb[q] = cj;
          const int base = is_time_plane(q) ? (cj * rb + tj0[l]) * 32 : cj;
          const int rs = rb * 32;
          const float f0 = w_a[q], f1 = w_b[q];
          if (is_time_plane(q) && A.rows) {
            // the frame's time row of this plane (the t lerp done once per
            // frame by k_pack_tc, as in the forward gather): two float4 loads
            float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
            if (ok) {
              const float* rp = A.rows + p.row_off[l][q == 2 ? 0 : (q == 4 ? 1 : 2)] + cj * 32 + ch;
              r0 = __ldg(reinterpret_cast<const float4*>(rp));
              r1 = __ldg(reinterpret_cast<const float4*>(rp + 32));
            }
            const float g0 = 1.f - f0;
            s[q] = make_float4(g0 * r0.x + f0 * r1.x, g0 * r0.y + f0 * r1.y, g0 * r0.z + f0 * r1.z,
                               g0 * r0.w + f0 * r1.w);
            da[q] = make_float4(r1.x - r0.x, r1.y - r0.y, r1.z - r0.z, r1.w - r0.w);
            db[q] = make_float4(0.f, 0.f, 0.f, 0.f);  // time axis: no position gradient
            continue;
          }
          float4 c00 = make_float4(0.f, 0.f, 0.f, 0.f), c01 = c00, c10 = c00, c11 = c00;
          if (ok) {
            const float* pl = p.planes[l][q] + base + ch;
            c00 = __ldg(reinterpret_cast<const float4*>(pl));
            c01 = __ldg(reinterpret_cast<const float4*>(pl + 32));
            c10 = __ldg(reinterpret_cast<const float4*>(pl + rs));
            c11 = __ldg(reinterpret_cast<const float4*>(pl + rs + 32));
          }
          const float w00 = (1.f - f0) * (1.f - f1), w10 = f0 * (1.f - f1), w01 = (1.f - f0) * f1, w11 = f0 * f1;
          s[q] = make_float4(w00 * c00.x + w10 * c10.x + w01 * c01.x + w11 * c11.x,
                             w00 * c00.y + w10 * c10.y + w01 * c01.y + w11 * c11.y,
                             w00 * c00.z + w10 * c10.z + w01 * c01.z + w11 * c11.z,
                             w00 * c00.w + w10 * c10.w + w01 * c01.w + w11 * c11.w);
          // hexplane.py:179-183 bilinear derivatives along a and b
          da[q] = make_float4((1.f - f1) * (c10.x - c00.x) + f1 * (c11.x - c01.x),
                              (1.f - f1) * (c10.y - c00.y) + f1 * (c11.y - c01.y),
                              (1.f - f1) * (c10.z - c00.z) + f1 * (c11.z - c01.z),
                              (1.f - f1) * (c10.w - c00.w) + f1 * (c11.w - c01.w));
          db[q] = make_float4((1.f - f0) * (c01.x - c00.x) + f0 * (c11.x - c10.x),
                              (1.f - f0) * (c01.y - c00.y) + f0 * (c11.y - c10.y),
                              (1.f - f0) * (c01.z - c00.z) + f0 * (c11.z - c10.z),
                              (1.f - f0) * (c01.w - c00.w) + f0 * (c11.w - c10.w));
        }
        if (!ok) continue;
        const float4 up = up_l[l];
        // product of the other five planes via prefix / suffix (hexplane.py:131-139)
        float4 pre[6], suf[6];
        pre[0] = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
        for (int q = 1; q < 6; ++q)
          pre[q] = make_float4(pre[q - 1].x * s[q - 1].x, pre[q - 1].y * s[q - 1].y, pre[q - 1].z * s[q - 1].z,
                               pre[q - 1].w * s[q - 1].w);
        suf[5] = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
        for (int q = 4; q >= 0; --q)
          suf[q] = make_float4(suf[q + 1].x * s[q + 1].x, suf[q + 1].y * s[q + 1].y, suf[q + 1].z * s[q + 1].z,
                               suf[q + 1].w * s[q + 1].w);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const float4 cf = make_float4(up.x * pre[q].x * suf[q].x, up.y * pre[q].y * suf[q].y,
                                        up.z * pre[q].z * suf[q].z, up.w * pre[q].w * suf[q].w);
          const float f0 = w_a[q], f1 = w_b[q];
          if (DET) {
            const double sc = a.dscale[l * 6 + q];
            auto add4 = [&](unsigned long long* c, float wgt) {
              det_add(c, cf.x * wgt, sc);
              det_add(c + 1, cf.y * wgt, sc);
              det_add(c + 2, cf.z * wgt, sc);
              det_add(c + 3, cf.w * wgt, sc);
            };
            if (is_time_plane(q)) {
              unsigned long long* acc = tacc_i + A.toff[l][q == 2 ? 0 : (q == 4 ? 1 : 2)] + cb[q] * 32 + ch;
              add4(acc, 1.f - f0);
              add4(acc + 32, f0);
            } else {
              const int rs = p.res[l][q][1] * 32;
              unsigned long long* gp = a.dacc[l][q] + cb[q] + ch;
              add4(gp, (1.f - f0) * (1.f - f1));
              add4(gp + rs, f0 * (1.f - f1));
              add4(gp + 32, (1.f - f0) * f1);
              add4(gp + rs + 32, f0 * f1);
            }
          } else if (is_time_plane(q)) {
            float* acc = tacc + A.toff[l][q == 2 ? 0 : (q == 4 ? 1 : 2)] + cb[q] * 32 + ch;
            const float g0 = 1.f - f0;
            red_add_v4(acc, cf.x * g0, cf.y * g0, cf.z * g0, cf.w * g0);
            red_add_v4(acc + 32, cf.x * f0, cf.y * f0, cf.z * f0, cf.w * f0);
          } else {
            const int rs = p.res[l][q][1] * 32;
            float* gp = a.gplanes[l][q] + cb[q] + ch;
            const float w00 = (1.f - f0) * (1.f - f1), w10 = f0 * (1.f - f1), w01 = (1.f - f0) * f1, w11 = f0 * f1;
            red_add_v4(gp, cf.x * w00, cf.y * w00, cf.z * w00, cf.w * w00);
            red_add_v4(gp + rs, cf.x * w10, cf.y * w10, cf.z * w10, cf.w * w10);
            red_add_v4(gp + 32, cf.x * w01, cf.y * w01, cf.z * w01, cf.w * w01);
            red_add_v4(gp + rs + 32, cf.x * w11, cf.y * w11, cf.z * w11, cf.w * w11);
          }
          const float sa = cf.x * da[q].x + cf.y * da[q].y + cf.z * da[q].z + cf.w * da[q].w;
          const float sb = cf.x * db[q].x + cf.y * db[q].y + cf.z * db[q].z + cf.w * db[q].w;
          dco[plane_axis0(q)] += sa * (float)(p.res[l][q][0] - 1);
          if (plane_axis1(q) < 3) dco[plane_axis1(q)] += sb * (float)(p.res[l][q][1] - 1);
        }
      }
#pragma unroll
      for (int off = 1; off < 8; off <<= 1)
#pragma unroll
        for (int q = 0; q < 3; ++q) dco[q] += __shfl_xor_sync(0xffffffffu, dco[q], off);
      const uint32_t ins = __shfl_sync(0xffffffffu, inside, j);
      if (ok && (lane & 7) < 3) {
        const int q = lane & 7;
        const float dq = q == 0 ? dco[0] : (q == 1 ? dco[1] : dco[2]);
        const float d = ((ins >> q) & 1u) ? (float)((double)dq / p.span[q]) : 0.f;
        a.cg_pos[3 * k + q] = cpos_in + gpos_in + d;
      }
    }
  }

}

// Sum the per-CTA time-plane partials (fixed order) and spread each spatial
// row onto the t rows j0 / j0 + 1 with the frame's t weights (hexplane.py:95-110).
struct TimeReduceArgs {
  const float* tpart;
  const unsigned long long* tpart_i;  // deterministic mode (int64 fixed point), or null
  const double* dscale;
  int nparts, tfloats;
  int toff[2][3], ra[2][3], rb[2][3], tj0[2];
  float tfb[2];
  float* gp[2][3];
};
__global__ void __launch_bounds__(32 * kRedGroups) k_time_partials(TimeReduceArgs a) {
  __shared__ float part[kRedGroups][33];
  __shared__ long long ipart[kRedGroups][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  if (a.tpart_i) {  // exact integer sums over the CTAs
    long long acc = 0;
    if (e < a.tfloats)
      for (int q = g; q < a.nparts; q += kRedGroups) acc += (long long)a.tpart_i[(int64_t)q * a.tfloats + e];
    ipart[g][lane] = acc;
  } else {
    part[g][lane] = e < a.tfloats ? sum_parts(a.tpart, a.tfloats, a.nparts, e, g) : 0.f;
  }
  __syncthreads();
  if (g != 0 || e >= a.tfloats) return;
  int l = 0, t = 0;
  for (int ll = 0; ll < 2; ++ll)
    for (int tt = 0; tt < 3; ++tt)
      if (e >= a.toff[ll][tt]) l = ll, t = tt;
  float v = 0.f;
  if (a.tpart_i) {
    long long acc = 0;
#pragma unroll
    for (int w = 0; w < kRedGroups; ++w) acc += ipart[w][lane];
    v = (float)((double)acc / a.dscale[l * 6 + (t == 0 ? 2 : (t == 1 ? 4 : 5))]);
  } else {
#pragma unroll
    for (int w = 0; w < kRedGroups; ++w) v += part[w][lane];
  }
  if (v == 0.f) return;
  const int loc = e - a.toff[l][t], i = loc >> 5, c = loc & 31, rb = a.rb[l][t];
  float* gp = a.gp[l][t];
  gp[(i * rb + a.tj0[l]) * 32 + c] += v * (1.f - a.tfb[l]);
  gp[(i * rb + a.tj0[l] + 1) * 32 + c] += v * a.tfb[l];
}

// ---------------------------------------------------------------------------
// deterministic mode: fixed-point scale per plane and the conversion back
// ---------------------------------------------------------------------------
// out[slot] = max |x| over a [rows, stride] block's columns [col0, col0+ncols)
// (non-negative floats order as their bit patterns: an integer atomicMax,
// independent of the order)
__global__ void k_det_maxabs(const float* __restrict__ x, int64_t rows, int stride, int col0, int ncols,
                             unsigned int* __restrict__ out) {
  float m = 0.f;
  const int64_t n = rows * ncols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = fabsf(x[(e / ncols) * stride + col0 + e % ncols]);
    m = v > m ? v : m;  // NaN-safe: comparisons with NaN are false
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// Plane (l, q): every Gaussian's coefficient is dlat * (product of the other
// five interpolated planes), each interpolation a convex combination of the
// plane's values, so the L1 mass the plane can receive is at most
// B = K * C * max|dlat_l| * prod_{q' != q} max|plane_{l,q'}|.  With
// scale = 2^(62 - ceil(log2 B)) every partial sum fits in int64 and the
// rounding unit is ~B * 2^-62.
__global__ void k_det_scales(const unsigned int* __restrict__ maxima, int levels, int64_t K, int C,
                             double* __restrict__ scale) {
  const int i = threadIdx.x;
  if (i >= levels * 6) return;
  const int l = i / 6, q = i % 6;
  double b = (double)K * C * (double)__uint_as_float(maxima[l]);
  for (int r = 0; r < 6; ++r)
    if (r != q) b *= (double)__uint_as_float(maxima[levels + l * 6 + r]);
  int e = 0;
  if (b > 0.0 && isfinite(b)) {
    frexp(b, &e);  // b <= 2^e
    scale[i] = ldexp(1.0, 62 - e);
  } else {
    scale[i] = 1.0;
  }
}

struct DetConvArgs {
  const unsigned long long* acc[FS4D_MAX_LEVELS * 6];
  float* dst[FS4D_MAX_LEVELS * 6];
  int64_t n[FS4D_MAX_LEVELS * 6];
  int64_t block_start[FS4D_MAX_LEVELS * 6 + 1];
  int nplanes;
  const double* scale;
  int scale_idx[FS4D_MAX_LEVELS * 6];
};

// dst[i] += acc[i] / scale, plane by plane (block ranges per plane)
__global__ void k_det_to_float(const __grid_constant__ DetConvArgs a) {
  int pl = 0;
  while (pl + 1 < a.nplanes && a.block_start[pl + 1] <= (int64_t)blockIdx.x) ++pl;
  const int64_t i = ((int64_t)blockIdx.x - a.block_start[pl]) * blockDim.x + threadIdx.x;
  if (i >= a.n[pl]) return;
  const long long v = (long long)a.acc[pl][i];
  if (v) a.dst[pl][i] += (float)((double)v / a.scale[a.scale_idx[pl]]);
}

// ---------------------------------------------------------------------------
// host driver (after deform_backward's pass-through and plane-gradient reset)
// ---------------------------------------------------------------------------
int tc_field_plan(const Fs4dHexPlane& f, double t, TcPlan& p);

// hexplane.query_backward (hexplane.py:145-187): plane gradients (written,
// or added with accumulate) and position gradients (zero on clamped axes).
int hexplane_query_backward(const Fs4dHexPlane& f, const float* pos, int64_t K, double t, const float* dlat,
                            Fs4dHexPlane& g, float* dpos, int accumulate, cudaStream_t s) {
  TcPlan p;
  int rc = tc_field_plan(f, t, p);
  if (rc) return rc;
  for (int l = 0; l < f.levels; ++l)
    for (int q = 0; q < 6; ++q) {
      if (!g.planes[l][q]) return fail(FS4D_ERR_CONFIG, "null plane gradient buffer");
      if (!accumulate)
        cudaMemsetAsync(g.planes[l][q], 0, (size_t)f.res[l][q][0] * f.res[l][q][1] * f.channels * 4, s);
    }
  if (K == 0) return FS4D_OK;
  HexBwdArgs h;
  memset(&h, 0, sizeof(h));
  h.p = p;
  h.K = K;
  h.pos = pos;
  h.dlat = dlat;
  h.g_pos = nullptr;
  h.cg_pos = dpos;
  for (int l = 0; l < FS4D_MAX_LEVELS; ++l)
    for (int q = 0; q < 6; ++q) h.gplanes[l][q] = l < f.levels ? g.planes[l][q] : nullptr;
  h.accumulate = accumulate;
  k_hexplane_bwd<false><<<(unsigned)ceil_div(K, kHexBwdWarps), kHexBwdWarps * 32, 0, s>>>(h);
  return check_launch("hexplane_query_backward");
}

static inline size_t det_align(size_t x, size_t a) { return (x + a - 1) / a * a; }

// deterministic-mode scratch of deform_backward_tc: maxima, scales, the int64
// plane accumulators and the int64 per-CTA time partials
size_t deform_bwd_det_bytes(const Fs4dHexPlane& f) {
  size_t o = 256 + 512;  // maxima (u32) + scales (double)
  int64_t tf = 0;        // time-plane partial floats of the 32-channel, 2-level kernel
  for (int l = 0; l < f.levels; ++l)
    for (int q = 0; q < 6; ++q) {
      o += det_align((size_t)f.res[l][q][0] * f.res[l][q][1] * f.channels * 8, 256);
      if (f.levels == 2 && f.channels == 32 && (q == 2 || q == 4 || q == 5)) tf += (int64_t)f.res[l][q][0] * 32;
    }
  return o + (size_t)kNumSMs * FS4D_HEX_BWD_MINB * (size_t)tf * 8;
}

int deform_backward_tc(const Fs4dCloud& cloud, const Fs4dHexPlane& field, const Fs4dDeformNet& net, double t,
                       const uint8_t* cache, const Fs4dCloud& sg, Fs4dCloud& cg, Fs4dDeformNet& ng,
                       Fs4dHexPlane* pg, int accumulate, void* ws, int32_t* status, void* det_ws,
                       size_t det_bytes, cudaStream_t s) {
  if (det_ws && det_bytes < deform_bwd_det_bytes(field))
    return fail(FS4D_ERR_CONFIG, "deterministic deform workspace too small");
  TcPlan p;
  uint8_t* blob = (uint8_t*)ws;
  int rc = tc_pack(net, field, t, p, blob, s);
  if (rc) return rc;
  const int64_t K = cloud.K;
  char* base = (char*)ws + p.ws_bytes;
  float* dlat = (float*)base;
  float* wpart = (float*)(base + ((size_t)K * 64 * 4 + 255) / 256 * 256);
  const int64_t ntiles = ceil_div(K, kTcRows);
  const int grid = (int)(ntiles < kNumSMs ? ntiles : kNumSMs);
  if (K > 0) {
    BwdArgs a;
    a.p = p;
    a.K = K;
    a.blob = blob;
    a.cache = cache;
    a.g_pos = sg.positions;
    a.g_rot = sg.rotations;
    a.g_ls = sg.log_scales;
    a.g_op = sg.opacity_logits;
    a.g_feat = sg.features;
    a.dlat = dlat;
    a.wpart = wpart;
    a.status = status;
    const int smem = ((p.blob_bytes + 1023) & ~1023) + kRBytes;
    if (smem > 227 * 1024) return fail(FS4D_ERR_CONFIG, "tcgen05 backward exceeds shared memory");
    cudaFuncSetAttribute(k_mlp_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mlp_bwd_tc<<<grid, kBwdThreads, smem, s>>>(a);

    HexBwdArgs h;
    memset(&h, 0, sizeof(h));
    h.p = p;
    h.K = K;
    h.pos = cloud.positions;
    h.dlat = dlat;
    h.g_pos = sg.positions;
    h.cg_pos = cg.positions;
    for (int l = 0; l < FS4D_MAX_LEVELS; ++l)
      for (int q = 0; q < 6; ++q) h.gplanes[l][q] = l < field.levels ? pg->planes[l][q] : nullptr;
    h.accumulate = accumulate;
    const bool det = det_ws != nullptr;
    unsigned long long* det_tpart = nullptr;
    DetConvArgs dconv;
    int64_t dblocks = 0;
    if (det) {
      // bounds -> scales -> zeroed int64 accumulators (all stream-ordered)
      char* d = (char*)det_ws;
      unsigned int* maxima = (unsigned int*)d;
      double* scales = (double*)(d + 256);
      cudaMemsetAsync(maxima, 0, 256, s);
      for (int l = 0; l < p.levels; ++l) {
        k_det_maxabs<<<kNumSMs * 2, 256, 0, s>>>(dlat, K, 64, l * p.C, p.C, maxima + l);
        for (int q = 0; q < 6; ++q)
          k_det_maxabs<<<kNumSMs, 256, 0, s>>>(field.planes[l][q], (int64_t)p.res[l][q][0] * p.res[l][q][1], p.C,
                                                0, p.C, maxima + p.levels + l * 6 + q);
      }
      k_det_scales<<<1, 64, 0, s>>>(maxima, p.levels, K, p.C, scales);
      h.dscale = scales;
      size_t o = 256 + 512;
      memset(&dconv, 0, sizeof(dconv));
      dconv.scale = scales;
      for (int l = 0; l < p.levels; ++l)
        for (int q = 0; q < 6; ++q) {
          const int64_t n = (int64_t)p.res[l][q][0] * p.res[l][q][1] * p.C;
          h.dacc[l][q] = (unsigned long long*)(d + o);
          o += det_align((size_t)n * 8, 256);
          cudaMemsetAsync(h.dacc[l][q], 0, (size_t)n * 8, s);
        }
      det_tpart = (unsigned long long*)(d + o);
      (void)dblocks;
    }
    HexC32Args hc;
    hc.h = h;
    hc.tpart_i = det_tpart;
    hc.rows = p.rows_ok && !getenv("FS4D_NO_TIME_ROWS") ? reinterpret_cast<const float*>(blob + p.off_rows) : nullptr;
    int tf = 0;
    for (int l = 0; l < 2 && p.levels == 2; ++l)
      for (int qi = 0; qi < 3; ++qi) {
        hc.toff[l][qi] = tf;
        tf += p.res[l][qi == 0 ? 2 : (qi == 1 ? 4 : 5)][0] * 32;
      }
    hc.tfloats = tf;
    hc.tpart = wpart + (size_t)kNumSMs * kPartStride + 128;
    if (p.C == 32 && p.levels == 2 && tf <= kTimePartFloats && !getenv("FS4D_HEX_BWD_GENERIC")) {
      const int64_t nblk = ceil_div(ceil_div(K, 32), kHexC32Warps);
      const int nres = kNumSMs * FS4D_HEX_BWD_MINB;  // resident 256-thread CTAs
      const int grid = (int)(nblk < nres ? nblk : nres);
      if (det) {
        cudaMemsetAsync(hc.tpart_i, 0, (size_t)grid * tf * 8, s);
        k_hexplane_bwd_c32<true><<<grid, kHexC32Warps * 32, 0, s>>>(hc);
      } else {
        cudaMemsetAsync(hc.tpart, 0, (size_t)grid * tf * 4, s);
        k_hexplane_bwd_c32<false><<<grid, kHexC32Warps * 32, 0, s>>>(hc);
      }
      TimeReduceArgs tr;
      tr.tpart = hc.tpart;
      tr.tpart_i = det ? hc.tpart_i : nullptr;
      tr.dscale = h.dscale;
      tr.nparts = grid;
      tr.tfloats = tf;
      for (int l = 0; l < 2; ++l) {
        const int rt = p.res[l][2][1];
        const double v = p.t * (rt - 1);
        int j0 = (int)floor(v);
        j0 = j0 < 0 ? 0 : (j0 > rt - 2 ? rt - 2 : j0);
        tr.tj0[l] = j0;
        tr.tfb[l] = (float)(v - j0);
        for (int qi = 0; qi < 3; ++qi) {
          const int q = qi == 0 ? 2 : (qi == 1 ? 4 : 5);
          tr.toff[l][qi] = hc.toff[l][qi];
          tr.ra[l][qi] = p.res[l][q][0];
          tr.rb[l][qi] = p.res[l][q][1];
          tr.gp[l][qi] = h.gplanes[l][q];
        }
      }
      k_time_partials<<<(unsigned)ceil_div(tf, 32), 32 * kRedGroups, 0, s>>>(tr);
      if (det) {  // spatial planes: int64 -> fp32 (the time planes went through k_time_partials)
        int np = 0;
        for (int l = 0; l < 2; ++l)
          for (int q = 0; q < 6; ++q) {
            if (is_time_plane(q)) continue;
            dconv.acc[np] = h.dacc[l][q];
            dconv.dst[np] = h.gplanes[l][q];
            dconv.n[np] = (int64_t)p.res[l][q][0] * p.res[l][q][1] * 32;
            dconv.scale_idx[np] = l * 6 + q;
            dconv.block_start[np] = dblocks;
            dblocks += ceil_div(dconv.n[np], 256);
            ++np;
          }
        dconv.block_start[np] = dblocks;
        dconv.nplanes = np;
        k_det_to_float<<<(unsigned)dblocks, 256, 0, s>>>(dconv);
      }
    } else if (det) {
      k_hexplane_bwd<true><<<(unsigned)ceil_div(K, kHexBwdWarps), kHexBwdWarps * 32, 0, s>>>(h);
      int np = 0;
      for (int l = 0; l < p.levels; ++l)
        for (int q = 0; q < 6; ++q) {
          dconv.acc[np] = h.dacc[l][q];
          dconv.dst[np] = h.gplanes[l][q];
          dconv.n[np] = (int64_t)p.res[l][q][0] * p.res[l][q][1] * p.C;
          dconv.scale_idx[np] = l * 6 + q;
          dconv.block_start[np] = dblocks;
          dblocks += ceil_div(dconv.n[np], 256);
          ++np;
        }
      dconv.block_start[np] = dblocks;
      dconv.nplanes = np;
      k_det_to_float<<<(unsigned)dblocks, 256, 0, s>>>(dconv);
    } else {
      k_hexplane_bwd<false><<<(unsigned)ceil_div(K, kHexBwdWarps), kHexBwdWarps * 32, 0, s>>>(h);
    }
  }
  DwReduceArgs r;
  memset(&r, 0, sizeof(r));
  int n = 0;
  auto map = [&](Fs4dLinear& g, int col0, int lane0, int bias_lane, int bias_tail) {
    DwMap& m = r.m[n++];
    m.gw = g.weight;
    m.gb = g.bias;
    m.out = g.out_dim;
    m.in = g.in_dim;
    m.col0 = col0;
    m.lane0 = lane0;
    m.bias_lane = bias_lane;
    m.bias_tail = bias_tail;
  };
  const int hoff[4] = {0, 3, 7, 10};
  map(ng.trunk[0], kDwTrunk, 0, 64, 0);
  for (int b = 0; b < 4; ++b) map(ng.ext[b][0], kDwExt0 + 32 * b, 0, 64, 0);
  for (int b = 0; b < 4; ++b) map(ng.ext[b][1], kDwExt1 + 32 * b, 0, 32, 0);
  for (int b = 0; b < 4; ++b) map(ng.head[b], kDwHead + hoff[b], 32 * b, -1, hoff[b]);
  map(ng.feat[0], kDwF1, 0, -1, 16);
  map(ng.feat[1], kDwF2, 0, 32, 0);
  for (int i = 0; i < n; ++i)
    if (!r.m[i].gw || !r.m[i].gb) return fail(FS4D_ERR_CONFIG, "missing net gradient buffer");
  r.wpart = wpart;
  r.nparts = K > 0 ? grid : 0;
  r.accumulate = accumulate;
  int max_ne = 0;
  for (int i = 0; i < n; ++i) max_ne = max_ne > r.m[i].out * (r.m[i].in + 1) ? max_ne : r.m[i].out * (r.m[i].in + 1);
  k_reduce_tc_wgrads<<<dim3((unsigned)ceil_div(max_ne, 32), n), 32 * kRedGroups, 0, s>>>(r);
  return check_launch("deform_bwd_tc");
}

}  // namespace fs4d
