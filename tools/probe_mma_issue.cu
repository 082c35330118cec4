// Microbenchmark: issue cost of tcgen05.mma (kind::f16, M=128, no-swizzle
// K-major operands in shared memory) from one warp, the way the MLP issues
// them (gemm_bf16x3_w: elected lane, uniform descriptors).  Prints cycles to
// issue 96 MMAs and cycles until their commit lands, for N = 16 .. 256.
// build/run on the box: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2503_06161_b200/csrc -I include tools/probe_mma_issue.cu -o /tmp/probe && /tmp/probe
#include <cstdio>
#include "tc_common.cuh"
using namespace fs4d;

template <int N>
__global__ void probe(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 * 64 * 4 + 256 * 64 * 4) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t sA = smem_u32(smem), sB = sA + 128 * 64 * 4;
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    // 32 gemm steps x 3 MMAs = 96 MMAs, K = 16 each
#pragma unroll 1
    for (int g = 0; g < 8; ++g) gemm_bf16x3_w(0, sA, 64, 0, sB, 64, 0, N, 4, false);
    long long t1 = clock64();
    mma_commit_w(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), r & 1);
    long long t2 = clock64();
    if (threadIdx.x == 0 && r == reps - 1) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

template <int N>
void run() {
  long long* d;
  cudaMalloc(&d, 16);
  const int smem = 128 * 64 * 4 + 256 * 64 * 4;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<1, 32, smem>>>(d, 4);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d: issue 96 MMAs %6lld cycles (%5.1f/MMA), complete %6lld cycles (%5.1f/MMA) err=%s\n", N, h[0],
         h[0] / 96.0, h[1], h[1] / 96.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16>();
  run<32>();
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
