// Device-wide scan + stable LSD radix sort (see scan_sort.cuh).
#include "scan_sort.cuh"

namespace fs4d {

__device__ __forceinline__ int64_t live_count(const uint32_t* n_dev, int64_t cap) {
  if (!n_dev) return cap;
  int64_t n = (int64_t)(*n_dev);
  return n < cap ? n : cap;
}

// ---------------------------------------------------------------------------
// scan: reduce -> scan of block sums -> apply
// ---------------------------------------------------------------------------
template <typename T>
__device__ T block_exclusive_scan(T v, T* smem_warp, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  T base = warp > 0 ? smem_warp[warp - 1] : T(0);
  if (total) *total = smem_warp[(blockDim.x >> 5) - 1];
  T excl = base + x - v;
  __syncthreads();
  return excl;
}

__global__ void k_scan_reduce(const uint32_t* __restrict__ in, int64_t cap, const uint32_t* n_dev,
                              uint64_t* __restrict__ block_sums) {
  __shared__ uint64_t warp_sums[32];
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kScanChunk;
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  // block reduce
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) warp_sums[warp] = s;
  __syncthreads();
  if (warp == 0) {
    s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) block_sums[blockIdx.x] = s;
  }
}

// single block: exclusive scan of block sums in place, grand total out
__global__ void k_scan_block_sums(uint64_t* block_sums, int nblocks, uint64_t* total) {
  __shared__ uint64_t warp_sums[32];
  uint64_t carry = 0;
  for (int base = 0; base < nblocks; base += blockDim.x) {
    int i = base + threadIdx.x;
    uint64_t v = i < nblocks ? block_sums[i] : 0;
    uint64_t tot;
    uint64_t e = block_exclusive_scan<uint64_t>(v, warp_sums, &tot);
    if (i < nblocks) block_sums[i] = carry + e;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_apply(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, int64_t cap,
                             const uint32_t* n_dev, const uint64_t* __restrict__ block_sums) {
  __shared__ uint64_t warp_sums[32];
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kScanChunk;
  if (base >= n) return;
  // blocked arrangement: thread t owns items [t*IPT, t*IPT+IPT)
  uint32_t v[kScanIPT];
  uint64_t local = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    int64_t i = base + (int64_t)threadIdx.x * kScanIPT + k;
    v[k] = i < n ? in[i] : 0u;
    local += v[k];
  }
  uint64_t excl = block_exclusive_scan<uint64_t>(local, warp_sums, nullptr) + block_sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    int64_t i = base + (int64_t)threadIdx.x * kScanIPT + k;
    if (i < n) out[i] = excl;
    excl += v[k];
  }
}

size_t scan_scratch_bytes(int64_t cap) {
  return (size_t)ceil_div(cap > 0 ? cap : 1, kScanChunk) * sizeof(uint64_t) + 256;
}

void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t cap, const uint32_t* n_dev,
                               uint64_t* total, void* scratch, cudaStream_t stream) {
  if (cap <= 0) {
    cudaMemsetAsync(total, 0, sizeof(uint64_t), stream);
    return;
  }
  int nb = (int)ceil_div(cap, kScanChunk);
  uint64_t* block_sums = (uint64_t*)scratch;
  k_scan_reduce<<<nb, kScanThreads, 0, stream>>>(in, cap, n_dev, block_sums);
  k_scan_block_sums<<<1, 1024, 0, stream>>>(block_sums, nb, total);
  k_scan_apply<<<nb, kScanThreads, 0, stream>>>(in, out, cap, n_dev, block_sums);
}

// ---------------------------------------------------------------------------
// radix sort: per pass  histogram -> per-digit scan over blocks -> stable scatter
// hist layout is digit-major: hist[d * nblocks + b]
// ---------------------------------------------------------------------------
__global__ void k_radix_hist(const uint32_t* __restrict__ keys, int64_t cap, const uint32_t* n_dev,
                             int shift, int nbits, uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[kMaxRadix];
  const int radix = 1 << nbits;
  for (int d = threadIdx.x; d < radix; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kSortChunk;
  const uint32_t mask = (1u << nbits) - 1u;
  if (base < n) {
#pragma unroll
    for (int k = 0; k < kSortIPT; ++k) {
      int64_t i = base + (int64_t)k * kSortThreads + threadIdx.x;
      if (i < n) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < radix; d += blockDim.x) hist[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

// one block per digit: exclusive scan over blocks, digit total out
__global__ void k_radix_scan_digit(uint32_t* __restrict__ hist, int nblocks, uint32_t* __restrict__ totals) {
  __shared__ uint32_t warp_sums[32];
  const int d = blockIdx.x;
  uint32_t* row = hist + (int64_t)d * nblocks;
  uint32_t carry = 0;
  for (int base = 0; base < nblocks; base += blockDim.x) {
    int i = base + threadIdx.x;
    uint32_t v = i < nblocks ? row[i] : 0u;
    uint32_t tot;
    uint32_t e = block_exclusive_scan<uint32_t>(v, warp_sums, &tot);
    if (i < nblocks) row[i] = carry + e;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[d] = carry;
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t cap,
    const uint32_t* n_dev, int shift, int nbits, const uint32_t* __restrict__ hist,
    const uint32_t* __restrict__ totals, int nblocks) {
  // dynamic: digit_base[radix] + warp_cnt[kSortWarps][radix]
  extern __shared__ uint32_t rs_smem[];
  __shared__ uint32_t scan_tmp[32];
  const int radix = 1 << nbits;
  uint32_t* digit_base = rs_smem;
  uint32_t* warp_cnt = rs_smem + radix;  // [warp * radix + d]
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kSortChunk;
  if (base >= n) return;  // uniform per block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t mask = (1u << nbits) - 1u;

  // global base per digit = exclusive scan of totals + this block's offset;
  // thread t owns digits [t*per, t*per + per)
  {
    const int per = (radix + kSortThreads - 1) / kSortThreads;
    uint32_t loc = 0;
    for (int q = 0; q < per; ++q) {
      const int d = threadIdx.x * per + q;
      if (d < radix) loc += totals[d];
    }
    uint32_t e = block_exclusive_scan<uint32_t>(loc, scan_tmp, nullptr);
    for (int q = 0; q < per; ++q) {
      const int d = threadIdx.x * per + q;
      if (d < radix) {
        digit_base[d] = e + hist[(int64_t)d * nblocks + blockIdx.x];
        e += totals[d];
      }
    }
  }
  for (int d = threadIdx.x; d < kSortWarps * radix; d += blockDim.x) warp_cnt[d] = 0;
  __syncthreads();

  // warp w ranks its contiguous sub-chunk in order, 32 items per round
  const int64_t wbase = base + (int64_t)warp * 32 * kSortIPT;
  uint32_t k_reg[kSortIPT], v_reg[kSortIPT], r_reg[kSortIPT];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    int64_t i = wbase + r * 32 + lane;
    bool valid = i < n;
    uint32_t key = valid ? keys_in[i] : 0u;
    uint32_t val = valid ? vals_in[i] : 0u;
    uint32_t d = (key >> shift) & mask;
    unsigned peers = __match_any_sync(0xffffffffu, valid ? d : 0xFFFFFFFFu);
    uint32_t rank = 0;
    if (valid) rank = warp_cnt[warp * radix + d] + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers & lt) == 0) warp_cnt[warp * radix + d] += __popc(peers);
    __syncwarp();
    k_reg[r] = key;
    v_reg[r] = val;
    r_reg[r] = valid ? rank : 0xFFFFFFFFu;
  }
  __syncthreads();
  // exclusive scan across warps per digit
  for (int d = threadIdx.x; d < radix; d += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      uint32_t c = warp_cnt[w * radix + d];
      warp_cnt[w * radix + d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortIPT; ++r) {
    if (r_reg[r] == 0xFFFFFFFFu) continue;
    uint32_t d = (k_reg[r] >> shift) & mask;
    uint32_t pos = digit_base[d] + warp_cnt[warp * radix + d] + r_reg[r];
    keys_out[pos] = k_reg[r];
    vals_out[pos] = v_reg[r];
  }
}

size_t radix_scratch_bytes(int64_t cap) {
  int64_t nb = ceil_div(cap > 0 ? cap : 1, kSortChunk);
  return (size_t)(nb * kMaxRadix + kMaxRadix) * sizeof(uint32_t) + 256;
}

// Digits of at most kMaxRadixBits, passes balanced: 32 bits -> 11+11+10,
// 11 tile bits (1280 tiles) -> one pass.
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                     int begin_bit, int end_bit, void* scratch, cudaStream_t stream) {
  int cur = 0;
  if (cap <= 0 || end_bit <= begin_bit) return cur;
  int nb = (int)ceil_div(cap, kSortChunk);
  uint32_t* hist = (uint32_t*)scratch;
  uint32_t* totals = hist + (int64_t)nb * kMaxRadix;
  const int bits = end_bit - begin_bit;
  const int passes = (bits + kMaxRadixBits - 1) / kMaxRadixBits;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_radix_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((kSortWarps + 1) * kMaxRadix * sizeof(uint32_t)));
    attr_set = true;
  }
  int shift = begin_bit;
  for (int p = 0; p < passes; ++p) {
    const int nbits = (bits - (shift - begin_bit) + (passes - p) - 1) / (passes - p);
    const int radix = 1 << nbits;
    k_radix_hist<<<nb, kSortThreads, 0, stream>>>(keys[cur], cap, n_dev, shift, nbits, hist, nb);
    k_radix_scan_digit<<<radix, 256, 0, stream>>>(hist, nb, totals);
    k_radix_scatter<<<nb, kSortThreads, (kSortWarps + 1) * radix * sizeof(uint32_t), stream>>>(
        keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], cap, n_dev, shift, nbits, hist, totals, nb);
    cur ^= 1;
    shift += nbits;
  }
  return cur;
}

int radix_passes(int bits) { return (bits + kMaxRadixBits - 1) / kMaxRadixBits; }

}  // namespace fs4d
