// Probe: does a K-major no-swizzle core-matrix image read back as an MN-major
// tcgen05 operand when LBO/SBO are swapped?  Computes D[i][o] = sum_g X[g][i] Y[g][o]
// with X [128 x KTA], Y [128 x KTB] stored in the row(g)-major image used by
// deform_tc.cu, both operands MN-major (idesc bits 15/16).  Prints max error for
// each (LBO, SBO) assignment.   nvcc -gencode arch=compute_100a,code=sm_100a -o probe probe_mn_major.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int KTA = 72, KTB = 40, NB = 32;

__host__ __device__ inline int core_off(int r, int k, int KT) {
  return (r >> 3) * (KT * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}
__device__ inline uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void k_probe(const __nv_bfloat16* X, const __nv_bfloat16* Y, float* D, int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * KTA * 2 + 4096;
  for (int e = threadIdx.x; e < 128 * KTA; e += blockDim.x) {
    const int g = e / KTA, f = e % KTA;
    *reinterpret_cast<__nv_bfloat16*>(sA + core_off(g, f, KTA)) = X[e];
  }
  for (int e = threadIdx.x; e < 128 * KTB; e += blockDim.x) {
    const int g = e / KTB, f = e % KTB;
    *reinterpret_cast<__nv_bfloat16*>(sB + core_off(g, f, KTB)) = Y[e];
  }
  const uint32_t b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(NB >> 3) << 17) |
                        ((uint32_t)(128 >> 4) << 24);
    uint32_t lboA, sboA, lboB, sboB;
    if (variant == 0) { lboA = KTA * 16; sboA = 128; lboB = KTB * 16; sboB = 128; }
    else { lboA = 128; sboA = KTA * 16; lboB = 128; sboB = KTB * 16; }
    for (int s = 0; s < 8; ++s) {  // K = 128 rows g, 16 per MMA = two 8-row blocks
      const uint32_t ka = variant == 0 ? 2 * s * KTA * 16 : 2 * s * KTA * 16;
      const uint32_t kb = variant == 0 ? 2 * s * KTB * 16 : 2 * s * KTB * 16;
      const uint64_t da = sdesc(smem_u32(sA) + ka, lboA, sboA), db = sdesc(smem_u32(sB) + kb, lboB, sboB);
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}\n" ::"r"(b)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < NB; ++c) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(trow + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[(warp * 32 + lane) * NB + c] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  std::vector<__nv_bfloat16> hx(128 * KTA), hy(128 * KTB);
  std::vector<float> fx(128 * KTA), fy(128 * KTB);
  srand(1);
  for (int i = 0; i < 128 * KTA; ++i) { hx[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fx[i] = __bfloat162float(hx[i]); }
  for (int i = 0; i < 128 * KTB; ++i) { hy[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); fy[i] = __bfloat162float(hy[i]); }
  __nv_bfloat16 *dx, *dy;
  float* dd;
  cudaMalloc(&dx, hx.size() * 2);
  cudaMalloc(&dy, hy.size() * 2);
  cudaMalloc(&dd, 128 * NB * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, hy.data(), hy.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 128 * KTA * 2 + 4096 + 128 * KTB * 2 + 4096;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dd, 0, 128 * NB * 4);
    k_probe<<<1, 128, smem>>>(dx, dy, dd, variant);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hd(128 * NB);
    cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < KTA; ++i)
      for (int o = 0; o < NB; ++o) {
        double ref = 0;
        for (int g = 0; g < 128; ++g) ref += (double)fx[g * KTA + i] * fy[g * KTB + o];
        maxerr = fmax(maxerr, fabs(ref - hd[i * NB + o]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("variant %d (%s): err=%s max_abs_err=%g (max |ref| %g) D[0][0]=%g\n", variant,
           variant == 0 ? "LBO=KT*16,SBO=128" : "LBO=128,SBO=KT*16", cudaGetErrorString(e), maxerr, maxref, hd[0]);
  }
  return 0;
}
