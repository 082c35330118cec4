// tcgen05 building blocks shared by the deformation forward (deform_tc.cu) and
// backward (deform_bwd_tc.cu) kernels.
//
// Operand images.  Every matrix the tensor cores read lives in shared memory
// as a "row image": R rows x KT columns of bf16, split hi/lo (hi block, then
// the lo block R*KT*2 bytes later), in the no-swizzle core-matrix layout
//   byte(r, k) = (r/8)*KT*16 + (k/8)*128 + (r%8)*16 + (k%8)*2.
// Read K-major (rows = M or N, columns = K):  LBO = 128, SBO = KT*16.
// Read MN-major (rows = K, columns = M or N): LBO = KT*16, SBO = 128 and the
// transpose bit of the instruction descriptor (verified on B200 by
// tools/probe_mn_major.cu).  The same image therefore serves a layer's
// forward GEMM (activations as A), its weight-gradient GEMM (activations as
// MN-major A, gradients as MN-major B, K = Gaussians) and its input-gradient
// GEMM (weights as MN-major B, K = output channels) without any transpose.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"

namespace fs4d {

struct TcPlan {
  int depth, D, DP, enable_feat, enable_grid;
  int levels, C, L;
  int res[FS4D_MAX_LEVELS][6][2];
  const float* planes[FS4D_MAX_LEVELS][6];
  const int32_t* order;  // optional Gaussian visiting order (Fs4dHexPlane.order)
  double lo[3], span[3];
  double t;
  // packed blob offsets (bytes)
  int off_trunk[FS4D_MAX_TRUNK], off_ext0, off_ext1[4], off_head[4], off_f1, off_f2;
  int off_headT[4];  // head b weights placed at rows hoff[b].. of a 16-row image (backward)
  int off_b_trunk[FS4D_MAX_TRUNK], off_b_ext0, off_b_ext1, off_b_head, off_b_f1, off_b_f2;
  // per-frame time rows of the (x,t),(y,t),(z,t) planes (all Gaussians share
  // t, so those bilinear lookups collapse to 1-D lerps between two rows of
  // R[i] = (1-fb) P[i][j0] + fb P[i][j0+1]); float offsets from off_rows
  int rows_ok, off_rows, row_off[FS4D_MAX_LEVELS][3];
  int blob_bytes;  // packed weights (what the kernels stage in shared memory)
  int ws_bytes;    // blob + time rows: start of the next workspace region (256-aligned)
  int fwd_bytes;   // prefix the forward kernel stages in shared memory
};

constexpr int kTcRows = 128;       // M tile (TMEM lanes)
constexpr int kTcThreads = 256;    // two threads per row (column halves)
constexpr int kTmemCols = 256;

__host__ __device__ inline int core_off(int r, int k, int KT) {
  return (r >> 3) * (KT * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// no-swizzle shared-memory matrix descriptor (sm_100 version bit 46)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, M = 128; bits 15/16
// select MN-major A/B
__device__ __forceinline__ uint32_t idesc_bf16(int N, bool a_mn = false, bool b_mn = false) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Warp-wide variants: every lane executes the call with identical (uniform)
// descriptors and one elected lane issues -- the descriptor arithmetic then
// stays on the uniform datapath instead of going through one divergent lane
// (measured ~90 cycles per MMA issue that way).
__device__ __forceinline__ void mma_bf16_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

// A[M=128][KT] (hi block then lo block at +128*KT*2 bytes) times B[N][KT]
// (hi, lo) into TMEM columns [col, col+N): hi*hi + hi*lo + lo*hi, K steps of 16.
// A columns [a_k0, a_k0 + 16*ksteps) against B columns [b_k0, ...); the first
// MMA overwrites the accumulator unless `accumulate` is set.
__device__ __forceinline__ void gemm_bf16x3(uint32_t tmem_d, uint32_t a_base, int a_kt, int a_k0, uint32_t b_base,
                                            int b_kt, int b_k0, int N, int ksteps, bool accumulate) {
  const uint32_t id = idesc_bf16(N);
  const uint32_t a_lo = a_base + kTcRows * a_kt * 2, b_lo = b_base + N * b_kt * 2;
  const uint32_t a_sbo = a_kt * 16, b_sbo = b_kt * 16;
#pragma unroll 1
  for (int s = 0; s < ksteps; ++s) {
    const uint32_t ak = (uint32_t)(((a_k0 >> 3) + 2 * s) * 128), bk = (uint32_t)(((b_k0 >> 3) + 2 * s) * 128);
    const uint64_t ah = sdesc(a_base + ak, 128, a_sbo), al = sdesc(a_lo + ak, 128, a_sbo);
    const uint64_t bh = sdesc(b_base + bk, 128, b_sbo), bl = sdesc(b_lo + bk, 128, b_sbo);
    mma_bf16(tmem_d, ah, bh, id, (s > 0 || accumulate) ? 1u : 0u);
    mma_bf16(tmem_d, ah, bl, id, 1u);
    mma_bf16(tmem_d, al, bh, id, 1u);
  }
}

// warp-wide gemm_bf16x3 (all 32 lanes call it; one elected lane issues)
__device__ __forceinline__ void gemm_bf16x3_w(uint32_t tmem_d, uint32_t a_base, int a_kt, int a_k0, uint32_t b_base,
                                              int b_kt, int b_k0, int N, int ksteps, bool accumulate) {
  const uint32_t id = idesc_bf16(N);
  const uint32_t a_lo = a_base + kTcRows * a_kt * 2, b_lo = b_base + N * b_kt * 2;
  const uint32_t a_sbo = a_kt * 16, b_sbo = b_kt * 16;
#pragma unroll
  for (int s = 0; s < ksteps; ++s) {
    const uint32_t ak = (uint32_t)(((a_k0 >> 3) + 2 * s) * 128), bk = (uint32_t)(((b_k0 >> 3) + 2 * s) * 128);
    const uint64_t ah = sdesc(a_base + ak, 128, a_sbo), al = sdesc(a_lo + ak, 128, a_sbo);
    const uint64_t bh = sdesc(b_base + bk, 128, b_sbo), bl = sdesc(b_lo + bk, 128, b_sbo);
    mma_bf16_w(tmem_d, ah, bh, id, (s > 0 || accumulate) ? 1u : 0u);
    mma_bf16_w(tmem_d, ah, bl, id, 1u);
    mma_bf16_w(tmem_d, al, bh, id, 1u);
  }
}

// General operand view of a row image for the backward GEMMs.
struct TcOpnd {
  uint32_t base;   // shared address of the first core matrix used (hi block)
  uint32_t lo;     // byte distance hi -> lo block
  uint32_t lbo, sbo, kstep;  // descriptor strides; bytes per K step of 16
  bool mn;
};

// rows = M/N, columns = K: columns [k0, ...) of an R x KT image
__device__ __forceinline__ TcOpnd opnd_k(uint32_t img, int R, int KT, int k0) {
  return TcOpnd{img + (uint32_t)((k0 >> 3) * 128), (uint32_t)(R * KT * 2), 128u, (uint32_t)(KT * 16), 256u, false};
}

// rows = K, columns = M/N: columns [c0, ...) and rows [k0, ...) of an R x KT image
__device__ __forceinline__ TcOpnd opnd_mn(uint32_t img, int R, int KT, int c0, int k0 = 0) {
  return TcOpnd{img + (uint32_t)((c0 >> 3) * 128 + (k0 >> 3) * KT * 16), (uint32_t)(R * KT * 2), (uint32_t)(KT * 16),
                128u, (uint32_t)(2 * KT * 16), true};
}

__device__ __forceinline__ void gemm3(uint32_t tmem_d, const TcOpnd& A, const TcOpnd& B, int N, int ksteps,
                                      bool accumulate) {
  const uint32_t id = idesc_bf16(N, A.mn, B.mn);
#pragma unroll 1
  for (int s = 0; s < ksteps; ++s) {
    const uint32_t ao = A.base + s * A.kstep, bo = B.base + s * B.kstep;
    const uint64_t ah = sdesc(ao, A.lbo, A.sbo), al = sdesc(ao + A.lo, A.lbo, A.sbo);
    const uint64_t bh = sdesc(bo, B.lbo, B.sbo), bl = sdesc(bo + B.lo, B.lbo, B.sbo);
    mma_bf16(tmem_d, ah, bh, id, (s > 0 || accumulate) ? 1u : 0u);
    mma_bf16(tmem_d, ah, bl, id, 1u);
    mma_bf16(tmem_d, al, bh, id, 1u);
  }
}

// warp-wide gemm3 (all 32 lanes call it; one elected lane issues)
__device__ __forceinline__ void gemm3_w(uint32_t tmem_d, const TcOpnd& A, const TcOpnd& B, int N, int ksteps,
                                      bool accumulate) {
  const uint32_t id = idesc_bf16(N, A.mn, B.mn);
#pragma unroll
  for (int s = 0; s < ksteps; ++s) {
    const uint32_t ao = A.base + s * A.kstep, bo = B.base + s * B.kstep;
    const uint64_t ah = sdesc(ao, A.lbo, A.sbo), al = sdesc(ao + A.lo, A.lbo, A.sbo);
    const uint64_t bh = sdesc(bo, B.lbo, B.sbo), bl = sdesc(bo + B.lo, B.lbo, B.sbo);
    mma_bf16_w(tmem_d, ah, bh, id, (s > 0 || accumulate) ? 1u : 0u);
    mma_bf16_w(tmem_d, ah, bl, id, 1u);
    mma_bf16_w(tmem_d, al, bh, id, 1u);
  }
}

// v = hi + lo with hi = bf16_rn(v), lo = bf16_rn(v - hi) (v - hi is exact in
// fp32).  Pairs go through cvt.rn.bf16x2.f32 (one packed convert per two
// values); bit-identical to per-element __float2bfloat16_rn.
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo_elem, float hi_elem) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
  return d;
}

__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = cvt_bf16x2(v[2 * i], v[2 * i + 1]);
    const float h0 = __uint_as_float(h[i] << 16), h1 = __uint_as_float(h[i] & 0xFFFF0000u);
    l[i] = cvt_bf16x2(v[2 * i] - h0, v[2 * i + 1] - h1);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// store 8 consecutive values (k0..k0+7) of row r into an A operand (hi, lo) with KT columns
__device__ __forceinline__ void store_split8(uint8_t* a_base, int KT, int r, int k0, const float* v) {
  uint4 h, l;
  split8(v, h, l);
  const int off = core_off(r, k0, KT);
  *reinterpret_cast<uint4*>(a_base + off) = h;
  *reinterpret_cast<uint4*>(a_base + kTcRows * KT * 2 + off) = l;
}

// ---------------------------------------------------------------------------
// activation cache of deform_with_cache (deformation.py:105-136) for the tc
// backward: per tile of 128 Gaussians, the row images the backward GEMMs read.
// Images feeding a weight-gradient GEMM carry one extra 8-column block whose
// first column is 1 (the bias gradient rides the same MMA as lane `in`).
// ---------------------------------------------------------------------------
constexpr int kCacheKtLat = 72, kCacheKtHid = 72, kCacheKtE1 = 40, kCacheKtE2 = 128, kCacheKtFF = 40;
constexpr int kCacheLat = 0;
constexpr int kCacheHid = kCacheLat + kTcRows * kCacheKtLat * 4;
constexpr int kCacheE1 = kCacheHid + kTcRows * kCacheKtHid * 4;  // + b * kCacheE1Bytes
constexpr int kCacheE1Bytes = kTcRows * kCacheKtE1 * 4;
constexpr int kCacheE2 = kCacheE1 + 4 * kCacheE1Bytes;
constexpr int kCacheFF = kCacheE2 + kTcRows * kCacheKtE2 * 4;
constexpr int kCacheTileBytes = kCacheFF + kTcRows * kCacheKtFF * 4;
constexpr int kCacheHeader = 256;

struct CacheHeader {
  uint32_t magic;
  uint32_t pad;
  int64_t K;
  double t;
};
constexpr uint32_t kCacheMagic = 0xF54DCAC1u;

// weight-gradient accumulators of the tc backward: TMEM columns [0, 384)
// (fp32, lane = input channel), plus 48 bias sums kept in shared memory; one
// partial per CTA, [column][lane] then the bias tail.
constexpr int kDwCols = 384;
// per-CTA time-plane gradient partials of the HexPlane backward (deform_bwd_tc.cu)
// plane axes (x,y),(x,z),(x,t),(y,z),(y,t),(z,t) (hexplane.py:16) as
// compile-time values inside unrolled loops (a __constant__ table index makes
// the coordinate array dynamically indexed, i.e. local memory)
__host__ __device__ __forceinline__ constexpr int plane_axis0(int q) { return q < 3 ? 0 : (q < 5 ? 1 : 2); }
__host__ __device__ __forceinline__ constexpr int plane_axis1(int q) { return q == 0 ? 1 : (q == 1 || q == 3 ? 2 : 3); }
constexpr int kTimeParts = 2 * 148;
constexpr int kTimePartFloats = 256 * 1024 / 4;  // upper bound of sum_l 3 * Ra * 32 (= kTimeRowBytes / 4)
constexpr int kPartStride = kDwCols * kTcRows + 64;

bool tc_path_ok(const Fs4dDeformNet& n, const Fs4dHexPlane& f);
bool tc_bwd_ok(const Fs4dDeformNet& n, const Fs4dHexPlane& f);
int tc_build_plan(const Fs4dDeformNet& n, const Fs4dHexPlane& f, double t, TcPlan& p);
int tc_pack(const Fs4dDeformNet& n, const Fs4dHexPlane& f, double t, TcPlan& p, uint8_t* blob, cudaStream_t s);

}  // namespace fs4d
