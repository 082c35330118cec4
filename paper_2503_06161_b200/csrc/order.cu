// Spatially coherent visiting order of a cloud (fs4d_locality_order): the
// Morton code of each Gaussian's position inside the field's aabb, then a
// stable LSD radix sort (scan_sort.cu).  The HexPlane gather / scatter
// kernels visit Gaussians in this order so that the 32 Gaussians of a warp
// share plane cells and corner rows come from L1 instead of L2.
#include "scan_sort.cuh"

namespace fs4d {

__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3FFu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void __launch_bounds__(256) k_morton(const float* __restrict__ pos, int64_t K, double lo0, double lo1,
                                                double lo2, double sp0, double sp1, double sp2,
                                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const double lo[3] = {lo0, lo1, lo2}, sp[3] = {sp0, sp1, sp2};
  uint32_t code = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double u = ((double)pos[3 * i + a] - lo[a]) / sp[a];
    u = fmin(fmax(u, 0.0), 1.0);  // NaN -> 0 (fmax ignores NaN)
    const uint32_t q = (uint32_t)fmin(u * 1024.0, 1023.0);
    code |= spread10(q) << a;
  }
  keys[i] = code;
  vals[i] = (uint32_t)i;
}

struct OrderLayout {
  size_t keys0, keys1, vals1, scratch, total;
};
static OrderLayout order_layout(int64_t K) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  OrderLayout L;
  L.keys0 = 0;
  L.keys1 = al(4 * (size_t)K);
  L.vals1 = L.keys1 + al(4 * (size_t)K);
  L.scratch = L.vals1 + al(4 * (size_t)K);
  L.total = L.scratch + al(radix_scratch_bytes(K));
  return L;
}

size_t locality_order_workspace_bytes(int64_t K) { return order_layout(K).total; }

int locality_order(const float* pos, int64_t K, const double* aabb, int32_t* order, void* ws, size_t ws_bytes,
                   cudaStream_t s) {
  const OrderLayout L = order_layout(K);
  if (!ws || ws_bytes < L.total) return fail(FS4D_ERR_CONFIG, "locality order workspace too small");
  if (K == 0) return FS4D_OK;
  char* b = (char*)ws;
  uint32_t* keys[2] = {(uint32_t*)(b + L.keys0), (uint32_t*)(b + L.keys1)};
  uint32_t* vals[2] = {(uint32_t*)order, (uint32_t*)(b + L.vals1)};
  double sp[3];
  for (int a = 0; a < 3; ++a) sp[a] = aabb[3 + a] - aabb[a] > 0 ? aabb[3 + a] - aabb[a] : 1.0;
  k_morton<<<(unsigned)ceil_div(K, 256), 256, 0, s>>>(pos, K, aabb[0], aabb[1], aabb[2], sp[0], sp[1], sp[2],
                                                        keys[0], vals[0]);
  const int res = radix_sort_pairs(keys, vals, K, nullptr, 0, 30, b + L.scratch, s);
  if (res == 1) cudaMemcpyAsync(order, vals[1], 4 * (size_t)K, cudaMemcpyDeviceToDevice, s);
  return check_launch("locality_order");
}

}  // namespace fs4d
