// Fused L1 RGB + feature loss and the upstream image gradients that feed
// fs4d_render_bwd (training.py:302-338 with an all-ones mask,
// semantic.py:171-181 applied at render resolution).  One pass over the
// rendered images: the loss partials are reduced per block and added to a
// device double, the gradients are written element-wise (sign(0) = 0 as
// np.sign).
#include "common.cuh"

namespace fs4d {

__device__ __forceinline__ float sgn(float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); }

__global__ void __launch_bounds__(256) k_l1_loss_grad(const float* __restrict__ c, const float* __restrict__ ct,
                                                      const float* __restrict__ f, const float* __restrict__ ft,
                                                      int64_t n_rgb, int64_t n_feat, float g_rgb, float g_feat,
                                                      float* __restrict__ dc, float* __restrict__ df, double* loss) {
  __shared__ double red[8];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // float4 main part (16-byte aligned tensors), scalar tail
  auto pass = [&](const float* x, const float* y, float* g, int64_t n, float gs) {
    float part = 0.f;
    int64_t n4 = 0;
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(g)) & 15) == 0) {
      n4 = n >> 2;
      for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 a = reinterpret_cast<const float4*>(x)[q], b = reinterpret_cast<const float4*>(y)[q];
        const float d0 = a.x - b.x, d1 = a.y - b.y, d2 = a.z - b.z, d3 = a.w - b.w;
        reinterpret_cast<float4*>(g)[q] = make_float4(gs * sgn(d0), gs * sgn(d1), gs * sgn(d2), gs * sgn(d3));
        part += fabsf(d0) + fabsf(d1) + fabsf(d2) + fabsf(d3);
      }
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const float d = x[i] - y[i];
      g[i] = gs * sgn(d);
      part += fabsf(d);
    }
    return (double)part * gs;
  };
  acc += pass(c, ct, dc, n_rgb, g_rgb);
  if (n_feat > 0) acc += pass(f, ft, df, n_feat, g_feat);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && loss) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    atomicAdd(loss, s);
  }
}

int l1_loss_grad(const float* color, const float* color_target, const float* feature, const float* feature_target,
                 int H, int W, int D, double w_rgb, double w_feat, float* d_color, float* d_feature, double* loss,
                 cudaStream_t s) {
  const int64_t px = (int64_t)H * W;
  const float g_rgb = (float)(w_rgb / (3.0 * (double)px));
  const float g_feat = (float)(w_feat / (double)px);
  k_l1_loss_grad<<<kNumSMs * 4, 256, 0, s>>>(color, color_target, feature, feature_target, px * 3, px * D, g_rgb,
                                             g_feat, d_color, d_feature, loss);
  return check_launch("l1_loss_grad");
}

}  // namespace fs4d
