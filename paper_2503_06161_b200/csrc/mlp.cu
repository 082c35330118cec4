// Stand-alone dense layers and tile replays for the public helper API:
//
//   fs4d_linear_forward / fs4d_linear_backward   numerics.mlp_forward /
//       mlp_backward (numerics.py:56-105), one layer per call, any shape:
//       SIMT fp32 tiled GEMMs (these are API helpers on small ad-hoc
//       stacks; the deformation MLP on the frame path runs on tcgen05 in
//       deform_tc.cu).  Weight / bias gradients are reduced over the batch in
//       fixed-size chunks and then in chunk order: bitwise deterministic.
//   fs4d_render_tile_alphas                       rasterizer._tile_alphas
//       (rasterizer.py:215-234) replayed from a render record with the blend
//       kernel's own arithmetic (pre-scaled conic, ex2, integer footprint).
//   fs4d_composite_weights                        rasterizer._composite_weights
//       (rasterizer.py:244-261) on a [G, P] alpha matrix, fp32, the blend's
//       multiplication order.
#include "render_common.cuh"

namespace fs4d {

constexpr int kGT = 16;         // GEMM tile edge
constexpr int kSplitRows = 4096;  // batch rows per weight-gradient partial

// C(m, n) = sum_k A(m, k) B(k, n) with element strides; ones_col: B(k, N-1) = 1
// (appends the bias-gradient column to the weight gradient).
struct GemmArgs {
  const float* A;
  const float* B;
  int64_t M, N, K;
  int64_t sam, sak, sbk, sbn;
  int ones_col;
  // epilogue (forward layer): + bias[n], pre out, act out
  const float* bias;
  float* C;     // [M, N] (or the split-K partial [split][M][N])
  float* act;   // optional ReLU output [M, N]
  int relu;
  int64_t k_chunk;  // split-K: blockIdx.z covers [z*k_chunk, (z+1)*k_chunk)
};

__global__ void __launch_bounds__(kGT* kGT) k_gemm(GemmArgs a) {
  __shared__ float sA[kGT][kGT + 1];
  __shared__ float sB[kGT][kGT + 1];
  const int tx = threadIdx.x % kGT, ty = threadIdx.x / kGT;
  const int64_t m = (int64_t)blockIdx.y * kGT + ty;
  const int64_t n = (int64_t)blockIdx.x * kGT + tx;
  const int64_t k_lo = (int64_t)blockIdx.z * a.k_chunk;
  const int64_t k_hi = min(a.K, k_lo + a.k_chunk);
  float acc = 0.f;
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += kGT) {
    {
      const int64_t mm = (int64_t)blockIdx.y * kGT + ty, kk = k0 + tx;
      sA[ty][tx] = (mm < a.M && kk < k_hi) ? a.A[mm * a.sam + kk * a.sak] : 0.f;
    }
    {
      const int64_t kk = k0 + ty, nn = (int64_t)blockIdx.x * kGT + tx;
      float v = 0.f;
      if (kk < k_hi && nn < a.N) v = (a.ones_col && nn == a.N - 1) ? 1.f : a.B[kk * a.sbk + nn * a.sbn];
      sB[ty][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kGT; ++j) acc = fmaf(sA[ty][j], sB[j][tx], acc);
    __syncthreads();
  }
  if (m >= a.M || n >= a.N) return;
  const int64_t o = (int64_t)blockIdx.z * a.M * a.N + m * a.N + n;
  if (a.bias) acc += a.bias[n];
  a.C[o] = acc;
  if (a.act) a.act[m * a.N + n] = a.relu ? fmaxf(acc, 0.f) : acc;
}

// g = dy * (pre > 0) for ReLU layers (numerics.py:99), copied otherwise
__global__ void k_relu_gate(const float* __restrict__ dy, const float* __restrict__ pre, int64_t n, int relu,
                            float* __restrict__ g) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    g[i] = (relu && !(pre[i] > 0.f)) ? 0.f : dy[i];
}

// ordered sum of the split-K partials [S][out][in+1] -> dW [out, in], db [out]
__global__ void k_reduce_dw(const float* __restrict__ part, int S, int out, int in, float* __restrict__ dw,
                            float* __restrict__ db, int accumulate) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = (int64_t)out * (in + 1);
  if (e >= ne) return;
  float s = 0.f;
  for (int z = 0; z < S; ++z) s += part[(int64_t)z * ne + e];
  const int o = (int)(e / (in + 1)), i = (int)(e % (in + 1));
  float* dst = i < in ? dw + (int64_t)o * in + i : db + o;
  *dst = accumulate ? *dst + s : s;
}

static dim3 gemm_grid(int64_t M, int64_t N, int64_t splits) {
  return dim3((unsigned)ceil_div(N, kGT), (unsigned)ceil_div(M, kGT), (unsigned)splits);
}

size_t linear_backward_workspace_bytes(int64_t B, int in, int out) {
  const int64_t S = B > 0 ? ceil_div(B, kSplitRows) : 1;
  return align_up((size_t)B * out * 4, 256) + (size_t)S * out * (in + 1) * 4 + 256;
}

int linear_forward(const float* x, int64_t B, const Fs4dLinear& L, float* pre, float* y, cudaStream_t s) {
  if (B == 0) return FS4D_OK;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.A = x;
  a.B = L.weight;
  a.M = B;
  a.N = L.out_dim;
  a.K = L.in_dim;
  a.sam = L.in_dim;
  a.sak = 1;
  a.sbk = 1;
  a.sbn = L.in_dim;
  a.bias = L.bias;
  a.C = pre;
  a.act = y;
  a.relu = L.relu;
  a.k_chunk = a.K > 0 ? a.K : 1;
  k_gemm<<<gemm_grid(a.M, a.N, 1), kGT * kGT, 0, s>>>(a);
  return check_launch("linear_forward");
}

int linear_backward(const float* x, const float* pre, int64_t B, const Fs4dLinear& L, const float* dy, float* dx,
                    float* dw, float* db, int accumulate, void* ws, cudaStream_t s) {
  const int in = L.in_dim, out = L.out_dim;
  float* g = (float*)ws;
  const int64_t S = B > 0 ? ceil_div(B, kSplitRows) : 1;
  float* part = (float*)((char*)ws + align_up((size_t)B * out * 4, 256));
  if (B > 0) {
    const int64_t n = B * out;
    k_relu_gate<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8), 256, 0, s>>>(dy, pre, n, L.relu, g);
    // dW | db = g^T [x | 1]: split over batch chunks, reduced in chunk order
    GemmArgs w;
    memset(&w, 0, sizeof(w));
    w.A = g;
    w.B = x;
    w.M = out;
    w.N = in + 1;
    w.K = B;
    w.sam = 1;
    w.sak = out;
    w.sbk = in;
    w.sbn = 1;
    w.ones_col = 1;
    w.C = part;
    w.k_chunk = kSplitRows;
    k_gemm<<<gemm_grid(w.M, w.N, S), kGT * kGT, 0, s>>>(w);
    if (dx) {  // dx = g W
      GemmArgs d;
      memset(&d, 0, sizeof(d));
      d.A = g;
      d.B = L.weight;
      d.M = B;
      d.N = in;
      d.K = out;
      d.sam = out;
      d.sak = 1;
      d.sbk = in;
      d.sbn = 1;
      d.C = dx;
      d.k_chunk = out;
      k_gemm<<<gemm_grid(d.M, d.N, 1), kGT * kGT, 0, s>>>(d);
    }
  } else {
    cudaMemsetAsync(part, 0, (size_t)out * (in + 1) * 4, s);
  }
  const int64_t ne = (int64_t)out * (in + 1);
  k_reduce_dw<<<(unsigned)ceil_div(ne, 256), 256, 0, s>>>(part, (int)(B > 0 ? S : 1), out, in, dw, db, accumulate);
  return check_launch("linear_backward");
}

// ---------------------------------------------------------------------------
// tile replays
// ---------------------------------------------------------------------------
struct TileAlphaArgs {
  const float4* xy;
  const float4* conic_o;
  const int4* pix_rect;
  const int32_t* src;
  int64_t G;
  int x0, y0, nx, ny;
  float alpha_cap, alpha_skip;
  float *alpha, *g2d, *a_raw;
};

// the blend kernel's per-pair test, element by element (render_fwd.cu k_blend)
__global__ void k_tile_alphas(TileAlphaArgs a) {
  const int P = a.nx * a.ny;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.G * P) return;
  const int64_t r = e / P;
  const int p = (int)(e % P);
  const int col = a.x0 + p % a.nx, row = a.y0 + p / a.nx;
  const int i = a.src[r];
  // relative to the 16-pixel tile origin, exactly as the blend stages it
  const int ox = col & ~(kTile - 1), oy = row & ~(kTile - 1);
  const float2 mm = tile_rel_mean(a.xy[i], (float)ox, (float)oy);
  const float4 cs = scaled_conic(a.conic_o[i]);
  const int4 pr = a.pix_rect[i];
  const float dx = (float)(col - ox) - mm.x, dy = (float)(row - oy) - mm.y;
  const float pw = gauss_power(cs, dx, dy);
  const bool in_rect = !(col < pr.x || col > pr.y || row < pr.z || row > pr.w);
  const bool live = in_rect && !(pw < kPowSkip);
  const float g = live ? fast_exp2(pw) : 0.f;
  const float raw = cs.w * g;
  float al = fminf(raw, a.alpha_cap);
  if (!live || al < a.alpha_skip) al = 0.f;
  a.alpha[e] = al;
  a.g2d[e] = g;
  a.a_raw[e] = raw;
}

// one thread per pixel column, the blend's front-to-back order
__global__ void k_composite_weights(const float* __restrict__ alpha, int64_t G, int64_t P, float stop,
                                    float* __restrict__ t_exc, uint8_t* __restrict__ contrib, float* __restrict__ w,
                                    float* __restrict__ t_final) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  float T = 1.f, tf = 1.f;
  for (int64_t g = 0; g < G; ++g) {
    const float al = alpha[g * P + p];
    const bool c = !(T < stop);
    t_exc[g * P + p] = T;
    contrib[g * P + p] = c;
    w[g * P + p] = c ? al * T : 0.f;
    T *= (1.f - al);
    if (c) tf = T;
  }
  t_final[p] = tf;
}

int render_tile_alphas(const RenderLayout& L, void* ws, const int32_t* src, int64_t G, int x0, int y0, int nx, int ny,
                       float alpha_cap, float alpha_skip, float* alpha, float* g2d, float* a_raw, cudaStream_t s) {
  TileAlphaArgs a;
  a.xy = at<float4>(ws, L.xy);
  a.conic_o = at<float4>(ws, L.conic_o);
  a.pix_rect = at<int4>(ws, L.pix_rect);
  a.src = src;
  a.G = G;
  a.x0 = x0;
  a.y0 = y0;
  a.nx = nx;
  a.ny = ny;
  a.alpha_cap = alpha_cap;
  a.alpha_skip = alpha_skip;
  a.alpha = alpha;
  a.g2d = g2d;
  a.a_raw = a_raw;
  const int64_t n = G * nx * ny;
  if (n > 0) k_tile_alphas<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(a);
  return check_launch("tile_alphas");
}

int composite_weights(const float* alpha, int64_t G, int64_t P, float stop, float* t_exc, uint8_t* contrib, float* w,
                      float* t_final, cudaStream_t s) {
  if (P > 0) k_composite_weights<<<(unsigned)ceil_div(P, 128), 128, 0, s>>>(alpha, G, P, stop, t_exc, contrib, w, t_final);
  return check_launch("composite_weights");
}

}  // namespace fs4d
