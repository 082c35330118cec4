// Training-step glue around the render path:
//   * masked photometric L1 + depth L1 and their upstream gradients
//     (training.py:300-338);
//   * generic L1 (semantic.py:171-181 feature_loss / _backward);
//   * Adam over the flat parameter buffer, one segment per reference
//     parameter array (numerics.py:119-159, training.py:431-442);
//   * HexPlane total variation loss + gradient (hexplane.py:190-222);
//   * corner-aligned bilinear resize and its adjoint (semantic.py:82-123);
//   * the pointwise feature decoder, its backward, and a fused
//     decode -> feature-L1 -> backward pass (semantic.py:126-181).
//
// Everything here is HBM-bound elementwise / stencil / small-reduction work:
// grid-stride or persistent grids sized in multiples of the SM count,
// coalesced channel-fastest accesses, fixed-order (deterministic) reductions
// where the reference's result feeds a parameter update.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace fs4d {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float sign1(float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); }

// Block-wide sum of one double per thread (kThreads threads); result valid in thread 0.
__device__ __forceinline__ double block_sum_d(double v) {
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();  // red may still be read by a previous call
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

__device__ __forceinline__ int64_t block_sum_i(int64_t v) {
  __shared__ long long red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, (long long)v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

}  // namespace

// ===========================================================================
// masked photometric L1 (training.py:300-338)
// ===========================================================================
constexpr int kPhotoBlocks = kNumSMs * 4;

struct PhotoPartial {
  double sum_rgb, sum_d;
  long long n_rgb, n_d;
};

__global__ void __launch_bounds__(kThreads) k_photo_sums(const float* __restrict__ c, const float* __restrict__ img,
                                                        const uint8_t* __restrict__ mask,
                                                        const float* __restrict__ dep,
                                                        const float* __restrict__ dep_t,
                                                        const float* __restrict__ alpha, int64_t px,
                                                        PhotoPartial* __restrict__ part) {
  double s_rgb = 0.0, s_d = 0.0;
  long long n_rgb = 0, n_d = 0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < px; i += (int64_t)gridDim.x * kThreads) {
    const bool m = mask ? mask[i] != 0 : true;
    if (!m) continue;
    n_rgb += 3;
    s_rgb += (double)(fabsf(c[3 * i] - img[3 * i]) + fabsf(c[3 * i + 1] - img[3 * i + 1]) +
                      fabsf(c[3 * i + 2] - img[3 * i + 2]));
    if (dep && alpha[i] >= 0.5f) {
      n_d += 1;
      s_d += (double)fabsf(dep[i] - dep_t[i]);
    }
  }
  s_rgb = block_sum_d(s_rgb);
  s_d = block_sum_d(s_d);
  n_rgb = block_sum_i(n_rgb);
  n_d = block_sum_i(n_d);
  if (threadIdx.x == 0) part[blockIdx.x] = PhotoPartial{s_rgb, s_d, n_rgb, n_d};
}

__global__ void __launch_bounds__(kThreads) k_photo_grads(const float* __restrict__ c, const float* __restrict__ img,
                                                         const uint8_t* __restrict__ mask,
                                                         const float* __restrict__ dep,
                                                         const float* __restrict__ dep_t,
                                                         const float* __restrict__ alpha, int64_t px,
                                                         const PhotoPartial* __restrict__ part, int n_part,
                                                         double lam_rgb, double lam_d, float* __restrict__ dc,
                                                         float* __restrict__ dd, double* __restrict__ terms,
                                                         double* __restrict__ loss) {
  __shared__ long long n_tot[2];
  // fixed-order reduction of the block partials (thread t takes partials t,
  // t + 256, ...; then the fixed block tree): deterministic, and parallel --
  // one thread walking all partials was a serial chain of n_part loads
  double a = 0.0, b = 0.0;
  long long na = 0, nb = 0;
  for (int i = threadIdx.x; i < n_part; i += kThreads) {
    a += part[i].sum_rgb;
    b += part[i].sum_d;
    na += part[i].n_rgb;
    nb += part[i].n_d;
  }
  a = block_sum_d(a);
  b = block_sum_d(b);
  na = block_sum_i(na);
  nb = block_sum_i(nb);
  if (threadIdx.x == 0) {
    n_tot[0] = na, n_tot[1] = nb;
    const double rgb = na ? a / (double)na : 0.0, dterm = nb ? b / (double)nb : 0.0;
    if (blockIdx.x == 0 && terms) {
      terms[0] = rgb;
      terms[1] = dterm;
      terms[2] = (double)na;
      terms[3] = (double)nb;
    }
    if (blockIdx.x == 0 && loss) atomicAdd(loss, lam_rgb * rgb + (dep ? lam_d * dterm : 0.0));  // lanes share it
  }
  __syncthreads();
  const float g_rgb = n_tot[0] ? (float)(lam_rgb / (double)n_tot[0]) : 0.f;
  const float g_d = n_tot[1] ? (float)(lam_d / (double)n_tot[1]) : 0.f;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < px; i += (int64_t)gridDim.x * kThreads) {
    const float m = (mask ? mask[i] != 0 : true) ? 1.f : 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) dc[3 * i + k] = g_rgb * sign1(c[3 * i + k] - img[3 * i + k]) * m;
    if (dd) {
      const float dm = (m != 0.f && alpha[i] >= 0.5f) ? 1.f : 0.f;
      dd[i] = g_d * sign1(dep[i] - dep_t[i]) * dm;
    }
  }
}

size_t photometric_workspace_bytes(int, int) { return sizeof(PhotoPartial) * kPhotoBlocks; }

int photometric_loss_grad(const float* c, const float* img, const uint8_t* mask, const float* dep,
                          const float* dep_t, const float* alpha, int H, int W, double lam_rgb, double lam_d,
                          float* dc, float* dd, double* terms, double* loss, void* ws, cudaStream_t s) {
  const int64_t px = (int64_t)H * W;
  auto* part = (PhotoPartial*)ws;
  k_photo_sums<<<kPhotoBlocks, kThreads, 0, s>>>(c, img, mask, dep, dep_t, alpha, px, part);
  k_photo_grads<<<kPhotoBlocks, kThreads, 0, s>>>(c, img, mask, dep, dep_t, alpha, px, part, kPhotoBlocks, lam_rgb,
                                                  lam_d, dc, dd, terms, loss);
  return check_launch("photometric_loss_grad");
}

// ===========================================================================
// generic L1 (semantic.py:171-181)
// ===========================================================================
__global__ void __launch_bounds__(kThreads) k_l1(const float* __restrict__ p, const float* __restrict__ t, int64_t n,
                                                float scale, double dscale, float* __restrict__ g,
                                                double* __restrict__ loss) {
  double acc = 0.0;
  float part = 0.f;
  int cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const float d = p[i] - t[i];
    if (g) g[i] = scale * sign1(d);
    part += fabsf(d);
    if (++cnt == 64) {  // bound the fp32 partial's length
      acc += part;
      part = 0.f;
      cnt = 0;
    }
  }
  acc += part;
  if (loss) {
    const double s = block_sum_d(acc);
    if (threadIdx.x == 0) atomicAdd(loss, s * dscale);
  }
}

int l1(const float* p, const float* t, int64_t n, double scale, float* g, double* loss, cudaStream_t s) {
  if (n <= 0) return FS4D_OK;
  const int blocks = (int)std::min<int64_t>(ceil_div(n, kThreads), kNumSMs * 4);
  k_l1<<<blocks, kThreads, 0, s>>>(p, t, n, (float)scale, scale, g, loss);
  return check_launch("l1");
}

// ===========================================================================
// Adam over segments of a flat buffer (numerics.py:137-159)
// ===========================================================================
constexpr int kAdamChunk = kThreads * 16;  // elements per block
constexpr int kStAdamDone = 19;            // status word: finished-block counter

struct AdamTable {
  int n;
  int64_t block_start[FS4D_MAX_ADAM_SEGMENTS + 1];
  Fs4dAdamSegment seg[FS4D_MAX_ADAM_SEGMENTS];
  int32_t slot[FS4D_MAX_ADAM_SEGMENTS];  // table entry -> caller's segment index (step count / status)
};

__device__ __forceinline__ int adam_segment_of(const AdamTable& T, int64_t b) {
  int lo = 0, hi = T.n - 1;  // last segment with block_start <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (T.block_start[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads) k_adam_check(const __grid_constant__ AdamTable T,
                                                        const float* __restrict__ g, int32_t* __restrict__ status) {
  const int s = adam_segment_of(T, blockIdx.x);
  const Fs4dAdamSegment& S = T.seg[s];
  const int64_t lo = S.offset + (blockIdx.x - T.block_start[s]) * (int64_t)kAdamChunk;
  const int64_t hi = min(lo + kAdamChunk, S.offset + S.count);
  int bad = 0;
#pragma unroll 4
  for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) bad += isfinite(g[i]) ? 0 : 1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) {
    atomicAdd(&status[FS4D_ST_ADAM_BAD_COUNT], bad);
    atomicMin(&status[FS4D_ST_ADAM_BAD_SEG], T.slot[s]);
    raise_status(status, FS4D_ERR_NUMERIC);
  }
}

__global__ void __launch_bounds__(kThreads) k_adam_apply(const __grid_constant__ AdamTable T, float* __restrict__ p,
                                                        const float* __restrict__ g, float* __restrict__ m,
                                                        float* __restrict__ v, int32_t* __restrict__ steps,
                                                        int32_t* __restrict__ status) {
  // non-finite gradient (or a failed render gated in by fs4d_status_merge):
  // nothing is touched
  if (status[FS4D_ST_ADAM_BAD_SEG] != 0x7FFFFFFF) return;
  __shared__ float s_coef[4];
  const int s = adam_segment_of(T, blockIdx.x);
  const Fs4dAdamSegment& S = T.seg[s];
  if (threadIdx.x == 0) {
    // AdamState.step_count += 1 (numerics.py:154); beta^step by binary
    // powering in fp64 (~2 log2(step) multiplies, a few hundred cycles, where
    // the libm pow() call stalled every block for microseconds)
    int e = steps[T.slot[s]] + 1;
    double p1 = 1.0, p2 = 1.0, b1d = S.beta1, b2d = S.beta2;
    while (e) {
      if (e & 1) p1 *= b1d, p2 *= b2d;
      b1d *= b1d;
      b2d *= b2d;
      e >>= 1;
    }
    s_coef[0] = (float)(1.0 / (1.0 - p1));
    s_coef[1] = (float)(1.0 / (1.0 - p2));
  }
  __syncthreads();
  const float b1 = (float)S.beta1, b2 = (float)S.beta2, c1 = (float)(1.0 - S.beta1), c2 = (float)(1.0 - S.beta2);
  const float rbc1 = s_coef[0], rbc2 = s_coef[1], lr = (float)S.lr, eps = (float)S.eps;
  const int64_t lo = S.offset + (blockIdx.x - T.block_start[s]) * (int64_t)kAdamChunk;
  const int64_t hi = min(lo + kAdamChunk, S.offset + S.count);
  auto upd = [&](float gi, float& mi, float& vi, float& pi) {
    mi = b1 * mi + c1 * gi;
    vi = b2 * vi + c2 * gi * gi;
    const float mh = mi * rbc1, vh = vi * rbc2;
    pi = pi - lr * mh / (sqrtf(vh) + eps);
  };
  // float4 body (segment offsets are 64-byte aligned by FlatGrads / FlatAdam;
  // checked), scalar tail
  int64_t i0 = lo;
  if ((lo & 3) == 0 && ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                         reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0) {
    const int64_t n4 = (hi - lo) >> 2;
#pragma unroll 2
    for (int64_t q = threadIdx.x; q < n4; q += kThreads) {
      const int64_t i = lo + 4 * q;
      const float4 gq = *reinterpret_cast<const float4*>(g + i);
      float4 mq = *reinterpret_cast<const float4*>(m + i), vq = *reinterpret_cast<const float4*>(v + i);
      float4 pq = *reinterpret_cast<const float4*>(p + i);
      upd(gq.x, mq.x, vq.x, pq.x);
      upd(gq.y, mq.y, vq.y, pq.y);
      upd(gq.z, mq.z, vq.z, pq.z);
      upd(gq.w, mq.w, vq.w, pq.w);
      *reinterpret_cast<float4*>(m + i) = mq;
      *reinterpret_cast<float4*>(v + i) = vq;
      *reinterpret_cast<float4*>(p + i) = pq;
    }
    i0 = lo + 4 * n4;
  }
  for (int64_t i = i0 + threadIdx.x; i < hi; i += kThreads) {
    float mi = m[i], vi = v[i], pi = p[i];
    upd(g[i], mi, vi, pi);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
  }
  // the last block to finish advances every segment's step count
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned ticket = atomicAdd((unsigned*)&status[kStAdamDone], 1u);
    if (ticket == gridDim.x - 1) {
      for (int i = 0; i < T.n; ++i) steps[T.slot[i]] += 1;
      status[kStAdamDone] = 0;
    }
  }
}

int adam_step(float* p, const float* g, float* m, float* v, int32_t* steps, const Fs4dAdamSegment* segs, int n,
              const int32_t* active, int32_t* status, cudaStream_t s) {
  // inactive segments (arrays without a gradient this iteration,
  // training.py:513-515) are left out of the table: neither their
  // parameters, moments nor step counts change
  AdamTable T;
  int64_t blocks = 0;
  int nt = 0;
  for (int i = 0; i < n; ++i) {
    if (active && !active[i]) continue;
    T.seg[nt] = segs[i];
    T.slot[nt] = i;
    T.block_start[nt] = blocks;
    blocks += ceil_div(segs[i].count, kAdamChunk);
    ++nt;
  }
  T.n = nt;
  T.block_start[nt] = blocks;
  if (blocks == 0) return FS4D_OK;
  if (blocks > 0x7FFFFFFF) return fail(FS4D_ERR_CONFIG, "adam buffer too large");
  k_adam_check<<<(unsigned)blocks, kThreads, 0, s>>>(T, g, status);
  k_adam_apply<<<(unsigned)blocks, kThreads, 0, s>>>(T, p, g, m, v, steps, status);
  return check_launch("adam_step");
}

// ===========================================================================
// dst = src[0] + src[1] + ... (fixed order): the training step's per-lane
// gradient buffers summed in one pass (instead of one read-modify-write of
// dst per lane)
// ===========================================================================
constexpr int kMaxSumSrc = 8;
struct SumArgs {
  const float* src[kMaxSumSrc];
  int nsrc;
  float* dst;
  int64_t n;
  int accumulate;
};

__global__ void __launch_bounds__(kThreads) k_sum_buffers(SumArgs a) {
  const int64_t n4 = a.n >> 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(a.dst)) & 15) == 0;
  bool svec = vec;
  for (int j = 0; j < a.nsrc; ++j) svec = svec && ((reinterpret_cast<uintptr_t>(a.src[j]) & 15) == 0);
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int64_t tail0 = 0;
  if (svec) {
    for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < n4; q += stride) {
      float4 acc = a.accumulate ? reinterpret_cast<const float4*>(a.dst)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = 0; j < a.nsrc; ++j) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(a.src[j]) + q);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      reinterpret_cast<float4*>(a.dst)[q] = acc;
    }
    tail0 = n4 << 2;
  }
  for (int64_t i = tail0 + (int64_t)blockIdx.x * kThreads + threadIdx.x; i < a.n; i += stride) {
    float acc = a.accumulate ? a.dst[i] : 0.f;
    for (int j = 0; j < a.nsrc; ++j) acc += a.src[j][i];
    a.dst[i] = acc;
  }
}

int sum_buffers(float* dst, const float* const* src, int nsrc, int64_t n, int accumulate, cudaStream_t s) {
  if (nsrc < 0 || nsrc > kMaxSumSrc) return fail(FS4D_ERR_CONFIG, "sum_buffers: 0..8 sources");
  if (n <= 0) return FS4D_OK;
  SumArgs a;
  for (int j = 0; j < nsrc; ++j) a.src[j] = src[j];
  a.nsrc = nsrc;
  a.dst = dst;
  a.n = n;
  a.accumulate = accumulate;
  const int64_t blocks = std::min<int64_t>(ceil_div(ceil_div(n, 4), kThreads), kNumSMs * 8);
  k_sum_buffers<<<(unsigned)blocks, kThreads, 0, s>>>(a);
  return check_launch("sum_buffers");
}

// ===========================================================================
// HexPlane total variation (hexplane.py:190-222)
// ===========================================================================
constexpr int kTvChunk = kThreads * 4;

struct TvPlane {
  const float* p;
  float* g;
  int ra, rb, c;
  float coef;       // 2 * scale / n_pairs
  double inv_pairs; // scale / n_pairs (loss weight)
};
struct TvTable {
  int n, accumulate;
  int64_t block_start[FS4D_MAX_LEVELS * 6 + 1];
  TvPlane pl[FS4D_MAX_LEVELS * 6];
};

__global__ void __launch_bounds__(kThreads) k_tv(const __grid_constant__ TvTable T, double* __restrict__ loss) {
  int s = 0;
  while (s + 1 < T.n && T.block_start[s + 1] <= (int64_t)blockIdx.x) ++s;
  const TvPlane& P = T.pl[s];
  const int64_t row = (int64_t)P.rb * P.c, total = (int64_t)P.ra * row;
  const int64_t e0 = (blockIdx.x - T.block_start[s]) * (int64_t)kTvChunk;
  float part = 0.f;
#pragma unroll
  for (int k = 0; k < kTvChunk / kThreads; ++k) {
    const int64_t e = e0 + k * kThreads + threadIdx.x;
    if (e >= total) break;
    const int64_t a = e / row;
    const int b = (int)((e - a * row) / P.c);
    const float x = __ldg(P.p + e);
    float grad = 0.f;
    if (a + 1 < P.ra) {
      const float d = __ldg(P.p + e + row) - x;
      part += d * d;
      grad -= d;
    }
    if (a > 0) grad += x - __ldg(P.p + e - row);
    if (b + 1 < P.rb) {
      const float d = __ldg(P.p + e + P.c) - x;
      part += d * d;
      grad -= d;
    }
    if (b > 0) grad += x - __ldg(P.p + e - P.c);
    if (P.g) P.g[e] = (T.accumulate ? P.g[e] : 0.f) + P.coef * grad;
  }
  if (loss) {
    const double sum = block_sum_d((double)part);
    if (threadIdx.x == 0) atomicAdd(loss, sum * P.inv_pairs);
  }
}

int tv_loss_grad(const Fs4dHexPlane& f, Fs4dHexPlane* gr, double scale, int accumulate, double* loss,
                 cudaStream_t s) {
  TvTable T;
  T.n = 0;
  T.accumulate = accumulate;
  int64_t blocks = 0;
  for (int l = 0; l < f.levels; ++l)
    for (int q = 0; q < 6; ++q) {
      const int ra = f.res[l][q][0], rb = f.res[l][q][1], c = f.channels;
      const double n_pairs = ((double)(ra - 1) * rb + (double)ra * (rb - 1)) * c;
      TvPlane& P = T.pl[T.n];
      P.p = f.planes[l][q];
      P.g = gr ? gr->planes[l][q] : nullptr;
      P.ra = ra, P.rb = rb, P.c = c;
      P.coef = n_pairs > 0 ? (float)(2.0 * scale / n_pairs) : 0.f;
      P.inv_pairs = n_pairs > 0 ? scale / n_pairs : 0.0;
      T.block_start[T.n++] = blocks;
      blocks += ceil_div((int64_t)ra * rb * c, kTvChunk);
    }
  T.block_start[T.n] = blocks;
  if (blocks == 0) return FS4D_OK;
  k_tv<<<(unsigned)blocks, kThreads, 0, s>>>(T, loss);
  return check_launch("tv_loss_grad");
}

// ===========================================================================
// corner-aligned bilinear resize (semantic.py:82-123)
// ===========================================================================
// _axis_weights (semantic.py:82-90): pos = o*(n_in-1)/(n_out-1) (0.5*(n_in-1)
// for a single output), lo = clip(floor(pos), 0, max(n_in-2, 0)), frac = pos-lo.
__device__ __forceinline__ int axis_lo(int o, int n_in, int n_out, float* frac) {
  const double pos = n_out == 1 ? 0.5 * (double)(n_in - 1) : (double)o * (double)(n_in - 1) / (double)(n_out - 1);
  int lo = (int)floor(pos);
  lo = max(0, min(lo, max(n_in - 2, 0)));
  if (frac) *frac = (float)(pos - (double)lo);
  return lo;
}
__device__ __forceinline__ int axis_hi(int o, int n_in, int n_out) { return min(axis_lo(o, n_in, n_out, nullptr) + 1, n_in - 1); }

// first output index whose lo (hi_side=false) or hi (hi_side=true) index is >= target (both are monotone)
__device__ __forceinline__ int axis_lower_bound(int target, bool hi_side, int n_in, int n_out) {
  int a = 0, b = n_out;
  while (a < b) {
    const int mid = (a + b) >> 1;
    const int v = hi_side ? axis_hi(mid, n_in, n_out) : axis_lo(mid, n_in, n_out, nullptr);
    if (v < target) a = mid + 1;
    else b = mid;
  }
  return a;
}

__global__ void __launch_bounds__(kThreads) k_resize(const float* __restrict__ in, int hi, int wi, int C,
                                                    float* __restrict__ out, int ho, int wo) {
  const int64_t n = (int64_t)ho * wo * C;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < n; e += (int64_t)gridDim.x * kThreads) {
    const int c = (int)(e % C);
    const int64_t pix = e / C;
    const int xo = (int)(pix % wo), yo = (int)(pix / wo);
    float yf, xf;
    const int y0 = axis_lo(yo, hi, ho, &yf), x0 = axis_lo(xo, wi, wo, &xf);
    const int y1 = min(y0 + 1, hi - 1), x1 = min(x0 + 1, wi - 1);
    const float r0 = in[((int64_t)y0 * wi + x0) * C + c] * (1.f - yf) + in[((int64_t)y1 * wi + x0) * C + c] * yf;
    const float r1 = in[((int64_t)y0 * wi + x1) * C + c] * (1.f - yf) + in[((int64_t)y1 * wi + x1) * C + c] * yf;
    out[e] = r0 * (1.f - xf) + r1 * xf;
  }
}

// Adjoint along one axis as a gather: d_in[.., i, ..] = sum over outputs o with
// lo(o) == i of (1-f(o)) d_out[.., o, ..] + sum over o with hi(o) == i of f(o) d_out.
// axis 1 (x): d_out [A, n_out, C] -> d_in [A, n_in, C]; the same kernel serves
// axis 0 (y) with C' = wi*C and A = 1.
__global__ void __launch_bounds__(kThreads) k_resize_adj(const float* __restrict__ d_out, int A, int n_out, int C,
                                                        float* __restrict__ d_in, int n_in) {
  const int64_t n = (int64_t)A * n_in * C;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < n; e += (int64_t)gridDim.x * kThreads) {
    const int c = (int)(e % C);
    const int64_t r = e / C;
    const int i = (int)(r % n_in);
    const int64_t a = r / n_in;
    const float* src = d_out + a * (int64_t)n_out * C + c;
    float acc = 0.f;
    for (int o = axis_lower_bound(i, false, n_in, n_out); o < n_out; ++o) {
      float f;
      if (axis_lo(o, n_in, n_out, &f) != i) break;
      acc += src[(int64_t)o * C] * (1.f - f);
    }
    for (int o = axis_lower_bound(i, true, n_in, n_out); o < n_out; ++o) {
      float f;
      const int lo = axis_lo(o, n_in, n_out, &f);
      if (min(lo + 1, n_in - 1) != i) break;
      acc += src[(int64_t)o * C] * f;
    }
    d_in[e] = acc;
  }
}

// Same gather with one thread per (row a, input index i, chunk of CH channels):
// the two monotone-range searches (fp64 axis positions, exactly those of
// axis_lo) run once per thread instead of once per channel, and the channel
// chunk moves as float4.  Per element the terms are added in the same order
// as k_resize_adj, so the results are identical.  Needs C % 4 == 0 and
// 16-byte aligned buffers.
constexpr int kAdjChunk = 32;
__global__ void __launch_bounds__(kThreads) k_resize_adj_v(const float* __restrict__ d_out, int A, int n_out, int C,
                                                          float* __restrict__ d_in, int n_in) {
  const int nch = (C + kAdjChunk - 1) / kAdjChunk;
  const int64_t n = (int64_t)A * n_in * nch;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < n; t += (int64_t)gridDim.x * kThreads) {
    const int ch = (int)(t % nch);
    const int64_t r = t / nch;
    const int i = (int)(r % n_in);
    const int64_t a = r / n_in;
    const int c0 = ch * kAdjChunk, cn = min(kAdjChunk, C - c0);
    const float* src = d_out + a * (int64_t)n_out * C + c0;
    float4 acc[kAdjChunk / 4];
#pragma unroll
    for (int q = 0; q < kAdjChunk / 4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto add = [&](int o, float w) {
      const float4* row = reinterpret_cast<const float4*>(src + (int64_t)o * C);
#pragma unroll
      for (int q = 0; q < kAdjChunk / 4; ++q)
        if (4 * q < cn) {
          const float4 v = __ldg(row + q);
          acc[q] = make_float4(acc[q].x + v.x * w, acc[q].y + v.y * w, acc[q].z + v.z * w, acc[q].w + v.w * w);
        }
    };
    for (int o = axis_lower_bound(i, false, n_in, n_out); o < n_out; ++o) {
      float f;
      if (axis_lo(o, n_in, n_out, &f) != i) break;
      add(o, 1.f - f);
    }
    for (int o = axis_lower_bound(i, true, n_in, n_out); o < n_out; ++o) {
      float f;
      const int lo = axis_lo(o, n_in, n_out, &f);
      if (min(lo + 1, n_in - 1) != i) break;
      add(o, f);
    }
    float4* dst = reinterpret_cast<float4*>(d_in + (a * n_in + i) * (int64_t)C + c0);
#pragma unroll
    for (int q = 0; q < kAdjChunk / 4; ++q)
      if (4 * q < cn) dst[q] = acc[q];
  }
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads), kNumSMs * 8)); }

int resize_bilinear(const float* in, int hi, int wi, int C, float* out, int ho, int wo, cudaStream_t s) {
  const int64_t n = (int64_t)ho * wo * C;
  if (n == 0) return FS4D_OK;
  k_resize<<<grid_for(n), kThreads, 0, s>>>(in, hi, wi, C, out, ho, wo);
  return check_launch("resize_bilinear");
}

size_t resize_workspace_bytes(int ho, int wi, int C) { return (size_t)ho * wi * C * sizeof(float); }

int resize_bilinear_backward(const float* d_out, int ho, int wo, int C, float* d_in, int hi, int wi, float* rows,
                             cudaStream_t s) {
  // semantic.py:107-123: columns first (d_rows [ho, wi, C]), then rows.
  int64_t n = (int64_t)ho * wi * C;
  if (n == 0 || (int64_t)hi * wi * C == 0) return FS4D_OK;
  const bool vec = C % 4 == 0 && ((reinterpret_cast<uintptr_t>(d_out) | reinterpret_cast<uintptr_t>(d_in) |
                                    reinterpret_cast<uintptr_t>(rows)) & 15) == 0;
  if (vec) {
    k_resize_adj_v<<<grid_for((int64_t)ho * wi * ceil_div(C, kAdjChunk)), kThreads, 0, s>>>(d_out, ho, wo, C, rows, wi);
    k_resize_adj_v<<<grid_for((int64_t)hi * ceil_div((int64_t)wi * C, kAdjChunk)), kThreads, 0, s>>>(rows, 1, ho, wi * C,
                                                                                                  d_in, hi);
    return check_launch("resize_bilinear_backward");
  }
  k_resize_adj<<<grid_for(n), kThreads, 0, s>>>(d_out, ho, wo, C, rows, wi);
  n = (int64_t)hi * wi * C;
  k_resize_adj<<<grid_for(n), kThreads, 0, s>>>(rows, 1, ho, wi * C, d_in, hi);
  return check_launch("resize_bilinear_backward");
}

// ===========================================================================
// pointwise decoder (semantic.py:126-181)
// ===========================================================================
constexpr int kDecPix = 32;    // output pixels per tile
constexpr int kDecMaxAcc = 48; // weight-gradient accumulators per thread: Ct*(N+1) <= 256*48

struct DecShape {
  int hi, wi, N, Ct, ho, wo;
};

static size_t dec_smem_bytes(int N, int Ct) {
  return sizeof(float) * ((size_t)N * (Ct + 1) + Ct + (size_t)kDecPix * (Ct + 1) + (size_t)kDecPix * N);
}

// resized tile r[p][n] for output pixels [pix0, pix0+kDecPix)
__device__ __forceinline__ void dec_resize_tile(const float* __restrict__ in, const DecShape& S, int64_t pix0,
                                                int64_t npix, float* r) {
  for (int e = threadIdx.x; e < kDecPix * S.N; e += blockDim.x) {
    const int p = e / S.N, n = e - p * S.N;
    const int64_t pix = pix0 + p;
    float val = 0.f;
    if (pix < npix) {
      const int xo = (int)(pix % S.wo), yo = (int)(pix / S.wo);
      float yf, xf;
      const int y0 = axis_lo(yo, S.hi, S.ho, &yf), x0 = axis_lo(xo, S.wi, S.wo, &xf);
      const int y1 = min(y0 + 1, S.hi - 1), x1 = min(x0 + 1, S.wi - 1);
      const int N = S.N;
      const float r0 = in[((int64_t)y0 * S.wi + x0) * N + n] * (1.f - yf) + in[((int64_t)y1 * S.wi + x0) * N + n] * yf;
      const float r1 = in[((int64_t)y0 * S.wi + x1) * N + n] * (1.f - yf) + in[((int64_t)y1 * S.wi + x1) * N + n] * yf;
      val = r0 * (1.f - xf) + r1 * xf;
    }
    r[e] = val;
  }
}

__device__ __forceinline__ void dec_load_weights(const float* __restrict__ w, const float* __restrict__ b,
                                                 const DecShape& S, float* wt, float* bs) {
  for (int e = threadIdx.x; e < S.Ct * S.N; e += blockDim.x) {
    const int ct = e / S.N, n = e - ct * S.N;
    wt[n * (S.Ct + 1) + ct] = w[e];  // transposed, padded rows: conflict-free for both uses
  }
  if (bs)
    for (int e = threadIdx.x; e < S.Ct; e += blockDim.x) bs[e] = b[e];
}

__global__ void __launch_bounds__(kThreads) k_decode(const float* __restrict__ in, const float* __restrict__ w,
                                                    const float* __restrict__ b, DecShape S, float* __restrict__ out,
                                                    float* __restrict__ resized) {
  extern __shared__ float sm[];
  float* wt = sm;
  float* bs = wt + S.N * (S.Ct + 1);
  float* r = bs + S.Ct + kDecPix * (S.Ct + 1);
  dec_load_weights(w, b, S, wt, bs);
  const int64_t npix = (int64_t)S.ho * S.wo;
  for (int64_t pix0 = (int64_t)blockIdx.x * kDecPix; pix0 < npix; pix0 += (int64_t)gridDim.x * kDecPix) {
    __syncthreads();
    dec_resize_tile(in, S, pix0, npix, r);
    __syncthreads();
    if (resized)
      for (int e = threadIdx.x; e < kDecPix * S.N; e += blockDim.x)
        if (pix0 + e / S.N < npix) resized[pix0 * S.N + e] = r[e];
    for (int e = threadIdx.x; e < kDecPix * S.Ct; e += blockDim.x) {
      const int p = e / S.Ct, ct = e - p * S.Ct;
      if (pix0 + p >= npix) break;
      float acc = 0.f;  // resized @ W^T, then + b (semantic.py:154)
      for (int n = 0; n < S.N; ++n) acc += r[p * S.N + n] * wt[n * (S.Ct + 1) + ct];
      out[pix0 * S.Ct + e] = acc + bs[ct];
    }
  }
}

// Backward of the decoder over output tiles.  FUSED: d_out is not read but
// computed from the teacher (feature L1, semantic.py:171-181) and the loss is
// accumulated.  Produces d_resized [ho*wo, N] and per-block weight/bias
// gradient partials [grid, Ct*(N+1)] (bias in column N).
template <bool FUSED>
__global__ void __launch_bounds__(kThreads) k_decode_bwd(const float* __restrict__ d_out_or_teacher,
                                                        const float* __restrict__ resized_or_rendered,
                                                        const float* __restrict__ w, const float* __restrict__ b,
                                                        DecShape S, float gscale, double lscale,
                                                        float* __restrict__ d_resized, float* __restrict__ partials,
                                                        double* __restrict__ loss) {
  extern __shared__ float sm[];
  float* wt = sm;
  float* bs = wt + S.N * (S.Ct + 1);
  float* dt = bs + S.Ct;              // [kDecPix][Ct+1]
  float* r = dt + kDecPix * (S.Ct + 1);  // [kDecPix][N]
  dec_load_weights(w, b, S, wt, FUSED ? bs : nullptr);
  const int nacc = S.Ct * (S.N + 1);
  float acc[kDecMaxAcc];
#pragma unroll
  for (int j = 0; j < kDecMaxAcc; ++j) acc[j] = 0.f;
  double lpart = 0.0;
  const int64_t npix = (int64_t)S.ho * S.wo;
  for (int64_t pix0 = (int64_t)blockIdx.x * kDecPix; pix0 < npix; pix0 += (int64_t)gridDim.x * kDecPix) {
    __syncthreads();
    float ltile = 0.f;
    if (FUSED) {
      dec_resize_tile(resized_or_rendered, S, pix0, npix, r);
    } else {
      for (int e = threadIdx.x; e < kDecPix * S.N; e += blockDim.x)
        r[e] = pix0 + e / S.N < npix ? resized_or_rendered[pix0 * S.N + e] : 0.f;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kDecPix * S.Ct; e += blockDim.x) {
      const int p = e / S.Ct, ct = e - p * S.Ct;
      float d = 0.f;
      if (pix0 + p < npix) {
        if (FUSED) {
          float o = 0.f;
          for (int n = 0; n < S.N; ++n) o += r[p * S.N + n] * wt[n * (S.Ct + 1) + ct];
          const float diff = (o + bs[ct]) - d_out_or_teacher[pix0 * S.Ct + e];
          ltile += fabsf(diff);
          d = gscale * sign1(diff);
        } else {
          d = d_out_or_teacher[pix0 * S.Ct + e];
        }
      }
      dt[p * (S.Ct + 1) + ct] = d;
    }
    lpart += ltile;
    __syncthreads();
    // weight / bias gradient partials: thread owns entries j*kThreads + tid of [Ct][N+1]
#pragma unroll
    for (int j = 0; j < kDecMaxAcc; ++j) {
      const int e = j * kThreads + threadIdx.x;
      if (e < nacc) {
        const int ct = e / (S.N + 1), n = e - ct * (S.N + 1);
        float s = 0.f;
        for (int p = 0; p < kDecPix; ++p) s += dt[p * (S.Ct + 1) + ct] * (n < S.N ? r[p * S.N + n] : 1.f);
        acc[j] += s;
      }
    }
    // d_resized = d_out @ W (semantic.py:167)
    for (int e = threadIdx.x; e < kDecPix * S.N; e += blockDim.x) {
      const int p = e / S.N, n = e - p * S.N;
      if (pix0 + p >= npix) break;
      float s = 0.f;
      for (int ct = 0; ct < S.Ct; ++ct) s += dt[p * (S.Ct + 1) + ct] * wt[n * (S.Ct + 1) + ct];
      d_resized[pix0 * S.N + e] = s;
    }
  }
#pragma unroll
  for (int j = 0; j < kDecMaxAcc; ++j) {
    const int e = j * kThreads + threadIdx.x;
    if (e < nacc) partials[(int64_t)blockIdx.x * nacc + e] = acc[j];
  }
  if (FUSED && loss) {
    const double sum = block_sum_d(lpart);
    if (threadIdx.x == 0) atomicAdd(loss, sum * lscale);
  }
}

// fixed-order sum of the per-block partials into d_weight [Ct,N] / d_bias [Ct]
// 32 accumulators per block; the 8 warps split the per-CTA partials (warp g
// sums partials g, g+8, ...) and are combined in a fixed order: deterministic,
// with ~nblk/8 independent loads per thread instead of a serial chain of nblk
__global__ void __launch_bounds__(kThreads) k_decode_reduce(const float* __restrict__ partials, int nblk, int Ct,
                                                           int N, float* __restrict__ dw, float* __restrict__ db,
                                                           int accumulate) {
  constexpr int G = kThreads / 32;
  __shared__ float part[G][33];
  const int nacc = Ct * (N + 1);
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  float s0 = 0.f, s1 = 0.f;
  if (e < nacc) {
    int i = g;
    for (; i + G < nblk; i += 2 * G) {
      s0 += partials[(int64_t)i * nacc + e];
      s1 += partials[(int64_t)(i + G) * nacc + e];
    }
    if (i < nblk) s0 += partials[(int64_t)i * nacc + e];
  }
  part[g][lane] = s0 + s1;
  __syncthreads();
  if (g != 0 || e >= nacc) return;
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < G; ++w) s += part[w][lane];
  const int ct = e / (N + 1), n = e - ct * (N + 1);
  float* dst = n < N ? dw + ct * N + n : db + ct;
  *dst = accumulate ? *dst + s : s;
}

static int dec_grid(const DecShape& S) {
  const int64_t tiles = ceil_div((int64_t)S.ho * S.wo, kDecPix);
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, kNumSMs * 2));
}

struct DecLayout {
  size_t partials, d_resized, rows, total;
};
static DecLayout dec_layout(const DecShape& S) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  DecLayout L;
  L.partials = 0;
  L.d_resized = al((size_t)dec_grid(S) * S.Ct * (S.N + 1) * sizeof(float));
  L.rows = L.d_resized + al((size_t)S.ho * S.wo * S.N * sizeof(float));
  L.total = L.rows + al(resize_workspace_bytes(S.ho, S.wi, S.N));
  return L;
}

size_t decoder_workspace_bytes(int hi, int wi, int N, int ho, int wo, int Ct) {
  return dec_layout(DecShape{hi, wi, N, Ct, ho, wo}).total;
}

static int dec_check(const DecShape& S) {
  if (S.hi <= 0 || S.wi <= 0 || S.N <= 0 || S.Ct <= 0 || S.ho <= 0 || S.wo <= 0)
    return fail(FS4D_ERR_CONFIG, "decoder sizes must be positive");
  if ((int64_t)S.Ct * (S.N + 1) > (int64_t)kThreads * kDecMaxAcc)
    return fail(FS4D_ERR_CONFIG, "decoder Ct*(N+1) above 12288 is not implemented");
  if (dec_smem_bytes(S.N, S.Ct) > 200 * 1024) return fail(FS4D_ERR_CONFIG, "decoder weights exceed shared memory");
  return FS4D_OK;
}

static void dec_set_smem(const void* fn, size_t bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

int decode_features(const float* in, int hi, int wi, int N, const float* w, const float* b, int Ct, int ho, int wo,
                    float* out, float* resized, cudaStream_t s) {
  const DecShape S{hi, wi, N, Ct, ho, wo};
  if (int rc = dec_check(S)) return rc;
  const size_t smem = dec_smem_bytes(N, Ct);
  dec_set_smem((const void*)k_decode, smem);
  k_decode<<<dec_grid(S), kThreads, smem, s>>>(in, w, b, S, out, resized);
  return check_launch("decode_features");
}

static int dec_backward_common(const DecShape& S, const float* d_out_or_teacher, const float* r_or_in,
                               const float* w, const float* b, bool fused, double lam, float* d_rendered,
                               float* dw, float* db, int accumulate, double* loss, void* ws, size_t ws_bytes,
                               cudaStream_t s) {
  if (int rc = dec_check(S)) return rc;
  const DecLayout L = dec_layout(S);
  if (!ws || ws_bytes < L.total) return fail(FS4D_ERR_CONFIG, "decoder workspace too small");
  char* base = (char*)ws;
  float* partials = (float*)(base + L.partials);
  float* d_res = (float*)(base + L.d_resized);
  float* rows = (float*)(base + L.rows);
  const size_t smem = dec_smem_bytes(S.N, S.Ct);
  const int grid = dec_grid(S);
  const double px = (double)S.ho * S.wo;
  if (fused) {
    dec_set_smem((const void*)k_decode_bwd<true>, smem);
    k_decode_bwd<true><<<grid, kThreads, smem, s>>>(d_out_or_teacher, r_or_in, w, b, S, (float)(lam / px), lam / px,
                                                    d_res, partials, loss);
  } else {
    dec_set_smem((const void*)k_decode_bwd<false>, smem);
    k_decode_bwd<false><<<grid, kThreads, smem, s>>>(d_out_or_teacher, r_or_in, w, b, S, 0.f, 0.0, d_res, partials,
                                                     nullptr);
  }
  const int nacc = S.Ct * (S.N + 1);
  k_decode_reduce<<<(unsigned)ceil_div(nacc, 32), kThreads, 0, s>>>(partials, grid, S.Ct, S.N, dw, db,
                                                                          accumulate);
  if (int rc = check_launch("decoder backward")) return rc;
  return resize_bilinear_backward(d_res, S.ho, S.wo, S.N, d_rendered, S.hi, S.wi, rows, s);
}

int decode_features_backward(const float* d_out, const float* resized, const float* w, int hi, int wi, int N, int Ct,
                             int ho, int wo, float* d_rendered, float* dw, float* db, int accumulate, void* ws,
                             size_t ws_bytes, cudaStream_t s) {
  return dec_backward_common(DecShape{hi, wi, N, Ct, ho, wo}, d_out, resized, w, nullptr, false, 0.0, d_rendered,
                             dw, db, accumulate, nullptr, ws, ws_bytes, s);
}

int decoder_feature_loss(const float* rendered, int hi, int wi, int N, const float* w, const float* b, int Ct,
                         const float* teacher, int ho, int wo, double lam, float* d_rendered, float* dw, float* db,
                         int accumulate, double* loss, void* ws, size_t ws_bytes, cudaStream_t s) {
  return dec_backward_common(DecShape{hi, wi, N, Ct, ho, wo}, teacher, rendered, w, b, true, lam, d_rendered, dw, db,
                             accumulate, loss, ws, ws_bytes, s);
}

}  // namespace fs4d
