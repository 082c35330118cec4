// Tile binning (bin_tiles, rasterizer.py:188-207, and the stable depth argsort
// it relies on, rasterizer.py:163).
//
// Option (FS4D_BINNING=depth): depth-ordered emission -- no per-tile sort.
//   depth_order       global stable depth order of the kept Gaussians (radix
//                     sort on fp32 depth bits + exact fp64 tie fix-up,
//                     render_fwd.cu) -- the reference's argsort itself
//   k_depth_counts    blocks of 256 consecutive Gaussians in that order count
//                     their pairs per tile WITHOUT atomics: per warp, one
//                     ballot per tile column / row gives the lanes whose
//                     rectangle covers it, X[tx] & Y[ty] the lanes covering a
//                     tile, popc the count -> table [block][tile]
//   k_depth_scan      per tile, exclusive prefix over the blocks + the tile
//                     offset: the table becomes each block's first slot
//   k_depth_emit      each lane writes its pairs at block base + earlier
//                     warps' counts + popc(lanes before it covering the tile):
//                     every tile list comes out in global depth order, written
//                     once, with no atomics and no sort
// Default (per-tile sort):
//   (per-tile pair counts: fused into k_preprocess, render_fwd.cu)
//   scan              tile offsets (device-wide exclusive scan)
//   k_emit_partition  every (tile, Gaussian) pair lands in its tile's segment;
//                     block-level reservation, order inside a segment arbitrary
//   k_tile_sort       one CTA per tile sorts its segment by (fp32 depth bits,
//                     exact fp64 depth on ties, source index) — the reference's
//                     stable float64 argsort order — with a bitonic network in
//                     shared memory (global memory for oversized tiles) and
//                     writes the tile range and the sorted source indices.
#include <limits.h>
#include <stdlib.h>
#include <string.h>

#include "render_common.cuh"

namespace fs4d {

#ifdef FS4D_SORT_TRACE
// debug timeline of the densest tile's CTA (tools/sort_trace.sh)
__device__ long long g_sort_trace[32];  // [0, 16): the densest tile's CTA, [16, 32): CTA FS4D_SORT_TRACE2
#ifndef FS4D_SORT_TRACE2
#define FS4D_SORT_TRACE2 700
#endif
#define SORT_TRACE(i)                                                     \
  if (trace_me && threadIdx.x == 0) g_sort_trace[(blockIdx.x ? 16 : 0) + (i)] = clock64();
extern "C" int fs4d_debug_sort_trace(long long* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, g_sort_trace, sizeof(long long) * 32);
}
#else
#define SORT_TRACE(i)
#endif

constexpr int kHistMaxTiles = 5888;   // shared-memory histogram capacity (23 KB; configs[3] has 5120 tiles)
constexpr int kTileScanThreads = 1024;
constexpr int kWarpTile = 32;           // tiles below this many pairs are sorted by one warp (k_tile_sort)
constexpr int kSortSmemKeys = 8192;   // per-tile keys sorted in shared memory (64 KB)
#ifndef FS4D_TILE_SORT_THREADS
#define FS4D_TILE_SORT_THREADS 512
#endif
constexpr int kTileSortThreads = FS4D_TILE_SORT_THREADS;

__device__ __forceinline__ bool rect_valid(const int4& t) { return t.y >= t.x && t.w >= t.z; }

// key = fp32 depth bits (positive floats order as unsigned) << 32 | source index
// Body shared by k_tile_scan_check and the fused pair partition: every thread
// of a kTileScanThreads block.  `base32` (shared memory, optional) receives
// the offsets saturated at cap as 32-bit values; `toff` (global, optional) the
// 64-bit offsets; `publish` also writes the densest-first tile order, the
// pair total, the capacity check and the status words.
struct TileScanSmem {
  uint64_t wsum[kTileScanThreads / 32];
  uint32_t bcnt[33], bcur[33];
};

__device__ void tile_scan_body(const uint32_t* __restrict__ tcnt, int ntiles, uint64_t* __restrict__ toff,
                               uint32_t* base32, bool publish, uint32_t* counters, int64_t cap, int32_t* status,
                               int32_t* __restrict__ tperm, TileScanSmem& sm) {
  uint64_t* wsum = sm.wsum;
  uint32_t* bcnt = sm.bcnt;
  uint32_t* bcur = sm.bcur;
  const int nthr = blockDim.x, nwarp = nthr >> 5;  // any multiple of 32 up to kTileScanThreads
  const int per = (ntiles + nthr - 1) / nthr;
  const int b0 = threadIdx.x * per;
  uint64_t local = 0;
  for (int q = 0; q < per; ++q)
    if (b0 + q < ntiles) local += tcnt[b0 + q];
  // block-wide exclusive scan of the per-thread sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < nwarp ? wsum[lane] : 0ull;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nwarp) wsum[lane] = wi - w;  // exclusive warp bases
  }
  __syncthreads();
  uint64_t run = wsum[warp] + incl - local;
  for (int q = 0; q < per; ++q)
    if (b0 + q < ntiles) {
      if (toff) toff[b0 + q] = run;
      if (base32) base32[b0 + q] = (uint32_t)(run < (uint64_t)cap ? run : (uint64_t)cap);
      run += tcnt[b0 + q];
    }
  if (!publish) return;
  // launch order for the per-tile kernels: tiles by decreasing count (log2
  // buckets, arbitrary order inside a bucket) so the longest tiles start in
  // the first wave instead of the tail -- the order never affects results
  if (tperm) {
    if (threadIdx.x < 33) bcnt[threadIdx.x] = 0;
    __syncthreads();
    for (int q = 0; q < per; ++q)
      if (b0 + q < ntiles) atomicAdd(&bcnt[32 - __clz(tcnt[b0 + q])], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t r = 0;
      for (int b = 32; b >= 0; --b) {
        bcur[b] = r;
        r += bcnt[b];
        if (b == 32 - __clz(kWarpTile)) counters[CNT_BIG_TILES] = r;  // tiles of >= kWarpTile pairs come first
      }
    }
    __syncthreads();
    for (int q = 0; q < per; ++q)
      if (b0 + q < ntiles) tperm[atomicAdd(&bcur[32 - __clz(tcnt[b0 + q])], 1u)] = b0 + q;
  }
  if ((int)threadIdx.x == nthr - 1) {
    const uint64_t total = run;
    *reinterpret_cast<uint64_t*>(counters + CNT_PAIRS64) = total;
    counters[CNT_PAIRS_CLAMPED] = (uint32_t)(total < (uint64_t)cap ? total : (uint64_t)cap);
    if (status) {
      status[FS4D_ST_N_VISIBLE] = (int32_t)counters[CNT_VISIBLE];
      status[FS4D_ST_PAIRS_LO] = (int32_t)(total & 0xFFFFFFFFu);
      status[FS4D_ST_PAIRS_HI] = (int32_t)(total >> 32);
      if (total > (uint64_t)cap) raise_status(status, FS4D_ERR_CAPACITY);
    }
  }
}

#ifndef FS4D_EMIT_THREADS
#define FS4D_EMIT_THREADS 1024  // measured: 256 -> 22.1 us, 512 -> 21.3, 1024 -> 19.9
#endif
constexpr int kEmitThreads = FS4D_EMIT_THREADS;
// One Gaussian per thread.  The block counts its pairs per tile in shared
// memory, reserves its slice of every touched tile segment with one global
// atomic, and keeps the slice's absolute start (segment offset + reservation,
// 32-bit: pair capacities stay below 2^32) in shared memory, so the emission
// loop is shared-memory atomics + one store per pair (no global load of the
// segment offset on the per-pair critical path).
//
// FUSED (kEmitThreads <= kTileScanThreads, tiles fit in shared memory): the
// tile-offset scan is done by every block into shared memory (1280 counts at
// configs[1]: a few hundred cycles, in parallel) and published by block 0
// (global offsets, densest-first order, pair total, status) -- one launch and
// one serial single-block kernel fewer on the frame's critical path.
template <bool FUSED>
#ifdef FS4D_EMIT_MINB  // A/B knob: minimum resident CTAs per SM
__global__ void __launch_bounds__(kEmitThreads, FS4D_EMIT_MINB) k_emit_partition(
#else
__global__ void __launch_bounds__(kEmitThreads) k_emit_partition(
#endif
const int4* __restrict__ tile_rect,
                                                        const uint32_t* __restrict__ dkeys, int64_t K, int ntx,
                                                        int ntiles, uint64_t* __restrict__ toff,
                                                        uint32_t* __restrict__ tcur, int64_t cap,
                                                        unsigned long long* __restrict__ pkey,
                                                        const uint32_t* __restrict__ tcnt, uint32_t* counters,
                                                        int32_t* status, int32_t* __restrict__ tperm) {
  __shared__ uint32_t cnt[kHistMaxTiles];
  __shared__ uint32_t base[kHistMaxTiles];
  __shared__ TileScanSmem scan_sm;
  const bool smem = FUSED || (ntiles <= kHistMaxTiles && cap <= (int64_t)0xFFFFFFFFu);
  if (smem)
    for (int b = threadIdx.x; b < ntiles; b += blockDim.x) cnt[b] = 0;
  if (FUSED) tile_scan_body(tcnt, ntiles, blockIdx.x == 0 ? toff : nullptr, base, blockIdx.x == 0, counters, cap,
                            status, tperm, scan_sm);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t dk = i < K ? dkeys[i] : 0xFFFFFFFFu;
  const bool kept = dk != 0xFFFFFFFFu;
  int4 t = make_int4(0, -1, 0, -1);
  if (kept) t = tile_rect[i];
  if (smem && kept)
    for (int ty = t.z; ty <= t.w; ++ty)
      for (int tx = t.x; tx <= t.y; ++tx) atomicAdd(&cnt[ty * ntx + tx], 1u);
  __syncthreads();
  if (smem)  // reserve this block's slice of every touched segment: four independent atomics in flight per thread
    for (int b0 = threadIdx.x; b0 < ntiles; b0 += 4 * kEmitThreads) {
      uint32_t c[4], r[4], o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = b0 + j * kEmitThreads;
        c[j] = b < ntiles ? cnt[b] : 0u;
        o[j] = c[j] ? (FUSED ? base[b] : (uint32_t)toff[b]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = c[j] ? atomicAdd(&tcur[b0 + j * kEmitThreads], c[j]) : 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = b0 + j * kEmitThreads;
        if (b < ntiles) {
          if (c[j]) base[b] = o[j] + r[j];
          cnt[b] = 0;
        }
      }
    }
  __syncthreads();
  if (!kept) return;
  const unsigned long long key = ((unsigned long long)dk << 32) | (unsigned long long)i;
  for (int ty = t.z; ty <= t.w; ++ty)
    for (int tx = t.x; tx <= t.y; ++tx) {
      const int b = ty * ntx + tx;
      const uint64_t o = smem ? (uint64_t)(base[b] + atomicAdd(&cnt[b], 1u)) : toff[b] + atomicAdd(&tcur[b], 1u);
      if (o < (uint64_t)cap) pkey[o] = key;
    }
}

// (depth bits, exact fp64 depth, source index) ordering.  The fp64 tie
// break is out of line: inlined, the compiler hoists its two global z64 loads
// above the (almost always taken) early return, and every comparison of the
// per-bucket insertion sorts then waited on an L2 round trip (13k cycles of a
// 25k-cycle dense-tile sort).
__device__ __noinline__ bool key_less_tie(unsigned long long a, unsigned long long b, const double* __restrict__ z64);
__device__ __forceinline__ bool key_less(unsigned long long a, unsigned long long b, const double* __restrict__ z64) {
  const uint32_t ha = (uint32_t)(a >> 32), hb = (uint32_t)(b >> 32);
  if (ha != hb) return ha < hb;
  return key_less_tie(a, b, z64);
}
__device__ __noinline__ bool key_less_tie(unsigned long long a, unsigned long long b, const double* __restrict__ z64) {
  const uint32_t ha = (uint32_t)(a >> 32);
  const uint32_t ia = (uint32_t)a, ib = (uint32_t)b;
  if (ia == ib) return false;
  if (ha == 0xFFFFFFFFu) return ia < ib;  // padding
  const double za = z64[ia], zb = z64[ib];
  if (za != zb) return za < zb;
  return ia < ib;
}

// Bitonic sort of keys[0..n) (virtual +inf padding to a power of two) with
// the all-ascending formulation: every compare-exchange moves the smaller key
// to the lower index, so virtual elements never move into [0, n).
__device__ void bitonic_sort(unsigned long long* keys, int n, const double* __restrict__ z64) {
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int k = 2; k <= p2; k <<= 1) {
    // first step of the merge: compare i with its mirror in the k-block
    for (int q = threadIdx.x; q < p2 / 2; q += blockDim.x) {
      const int blk = q / (k / 2), off = q % (k / 2);
      const int lo = blk * k + off, hi = blk * k + k - 1 - off;
      if (hi < n) {
        const unsigned long long a = keys[lo], b = keys[hi];
        if (key_less(b, a, z64)) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
    }
    __syncthreads();
    for (int j = k / 4; j >= 1; j >>= 1) {
      for (int q = threadIdx.x; q < p2 / 2; q += blockDim.x) {
        const int lo = (q / j) * 2 * j + (q % j), hi = lo + j;
        if (hi < n) {
          const unsigned long long a = keys[lo], b = keys[hi];
          if (key_less(b, a, z64)) {
            keys[lo] = b;
            keys[hi] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kTileSortWarps = kTileSortThreads / 32;
constexpr int kTileSortIPT = kSortSmemKeys / kTileSortThreads;  // 16 items per thread

// Lanes of the warp holding the same 8-bit digit: eight ballots, one per
// digit bit (VOTE + LOP3, ALU latency).  __match_any_sync does the same in one
// instruction but runs on a long variable-latency path (the top short-
// scoreboard stall of this kernel under ncu).
__device__ __forceinline__ unsigned warp_peers8(uint32_t d) {
  unsigned m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

// CTA-wide stable LSD radix sort of up to kSortSmemKeys (depth bits, source
// index) pairs held in registers ("striped": lane l of warp w owns items
// w*32*IPT + r*32 + l), 8-bit digits, shared memory only for counters and the
// exchange buffer.  Then equal-depth-bit runs (rare) are re-ordered by the
// exact fp64 depth and the source index.
__device__ void cta_radix_sort_tile(const unsigned long long* __restrict__ src, int n, const double* __restrict__ z64,
                                    uint32_t* __restrict__ out_vals, unsigned long long* xbuf, uint32_t* wcnt,
                                    uint32_t* dbase) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  // R rounds of 32 items per warp cover n (R <= kTileSortIPT, uniform per CTA)
  const int R = (n + kTileSortThreads - 1) / kTileSortThreads;
  uint32_t key[kTileSortIPT], val[kTileSortIPT];
#pragma unroll
  for (int r = 0; r < kTileSortIPT; ++r) {
    const int q = warp * 32 * R + r * 32 + lane;
    const unsigned long long kv = (r < R && q < n) ? src[q] : 0xFFFFFFFFFFFFFFFFull;
    key[r] = (uint32_t)(kv >> 32);
    val[r] = (uint32_t)kv;
  }
  // digits on which every key of the tile agrees need no pass (e.g. the
  // sign / exponent byte of depths within one octave): AND / OR over the keys
  uint32_t kand = 0xFFFFFFFFu, kor = 0u;
#pragma unroll
  for (int r = 0; r < kTileSortIPT; ++r)
    if (r < R && warp * 32 * R + r * 32 + lane < n) {
      kand &= key[r];
      kor |= key[r];
    }
  kand = __reduce_and_sync(0xffffffffu, kand);
  kor = __reduce_or_sync(0xffffffffu, kor);
  if (lane == 0) {
    dbase[2 * warp] = kand;
    dbase[2 * warp + 1] = kor;
  }
  __syncthreads();
  uint32_t vary = 0u;
  {
    uint32_t ba = 0xFFFFFFFFu, bo = 0u;
    for (int w = 0; w < kTileSortWarps; ++w) {
      ba &= dbase[2 * w];
      bo |= dbase[2 * w + 1];
    }
    vary = ba ^ bo;
  }
  __syncthreads();
  bool sorted_into_xbuf = false;
  for (int shift = 0; shift < 32; shift += 8) {
    if (((vary >> shift) & 0xFFu) == 0u) continue;  // uniform digit (block-uniform branch)
    sorted_into_xbuf = true;
    for (int d = threadIdx.x; d < kTileSortWarps * 256; d += blockDim.x) wcnt[d] = 0;
    __syncthreads();
    uint32_t rank[kTileSortIPT];
#pragma unroll
    for (int r = 0; r < kTileSortIPT; ++r) {
      if (r >= R) break;
      const uint32_t d = (key[r] >> shift) & 0xFFu;
      const unsigned peers = warp_peers8(d);
      rank[r] = wcnt[warp * 256 + d] + __popc(peers & lt);
      __syncwarp();
      if ((peers & lt) == 0) wcnt[warp * 256 + d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // digit totals -> exclusive digit bases; per-digit warp prefixes in place
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kTileSortWarps; ++w) {
        const uint32_t c = wcnt[w * 256 + d];
        wcnt[w * 256 + d] = run;
        run += c;
      }
      dbase[d] = run;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of 256 digit totals by one warp
      uint32_t v[8], s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = dbase[lane * 8 + q];
        s += v[q];
      }
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t run = incl - s;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        dbase[lane * 8 + q] = run;
        run += v[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kTileSortIPT; ++r) {
      if (r >= R) break;
      const uint32_t d = (key[r] >> shift) & 0xFFu;
      const uint32_t pos = dbase[d] + wcnt[warp * 256 + d] + rank[r];
      xbuf[pos] = ((unsigned long long)key[r] << 32) | val[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kTileSortIPT; ++r) {
      if (r >= R) break;
      const unsigned long long kv = xbuf[warp * 32 * R + r * 32 + lane];
      key[r] = (uint32_t)(kv >> 32);
      val[r] = (uint32_t)kv;
    }
  }
  if (!sorted_into_xbuf) {  // all keys equal: the load order is the order
#pragma unroll
    for (int r = 0; r < kTileSortIPT; ++r) {
      const int q = warp * 32 * R + r * 32 + lane;
      if (r < R && q < n) xbuf[q] = ((unsigned long long)key[r] << 32) | val[r];
    }
    __syncthreads();
  }
  // xbuf holds the sorted sequence; fix equal-depth-bit runs, then emit
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const uint32_t k = (uint32_t)(xbuf[q] >> 32);
    const bool start = (q == 0 || (uint32_t)(xbuf[q - 1] >> 32) != k) && q + 1 < n && (uint32_t)(xbuf[q + 1] >> 32) == k;
    if (!start) continue;
    int e = q + 1;
    while (e < n && (uint32_t)(xbuf[e] >> 32) == k) ++e;
    for (int a = q + 1; a < e; ++a) {
      const unsigned long long ka = xbuf[a];
      int b = a - 1;
      while (b >= q && key_less(ka, xbuf[b], z64)) {
        xbuf[b + 1] = xbuf[b];
        --b;
      }
      xbuf[b + 1] = ka;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < n; q += blockDim.x) out_vals[q] = (uint32_t)xbuf[q];
}

// CTA-wide sort of one tile's list by bucketing: each key goes to one of NB
// buckets (NB ~ n, at most 4096) by a monotone map of its depth bits onto the
// tile's [min, max] range, the buckets are laid out by one prefix sum, and the
// few keys of each bucket are put in order by one thread (insertion sort on
// (depth bits, exact fp64 depth, source index) -- the total order the
// reference's stable float64 argsort produces).  One scatter instead of three
// stable 8-bit LSD passes; the order inside a bucket before its sort (shared-
// memory atomics) never matters because the final order is total.  Returns
// false, having written nothing, when some bucket holds more than
// kBucketMax keys (strongly clustered depths); the caller then runs the radix
// sort.
constexpr int kBucketMax = 64;
constexpr int kBucketNB = kTileSortWarps * 256;  // bucket counters reuse the radix sort's warp counters

__device__ bool cta_bucket_sort_tile(const unsigned long long* __restrict__ src, int n, const double* __restrict__ z64,
                                     uint32_t* __restrict__ out_vals, unsigned long long* xbuf, uint32_t* cnt,
                                     uint32_t* red, bool trace_me = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = (n + kTileSortThreads - 1) / kTileSortThreads;
  uint32_t key[kTileSortIPT], val[kTileSortIPT];
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll
  for (int r = 0; r < kTileSortIPT; ++r) {
    const int q = r * kTileSortThreads + threadIdx.x;
    const unsigned long long kv = (r < R && q < n) ? src[q] : 0xFFFFFFFFFFFFFFFFull;
    key[r] = (uint32_t)(kv >> 32);
    val[r] = (uint32_t)kv;
    if (r < R && q < n) {
      kmin = min(kmin, key[r]);
      kmax = max(kmax, key[r]);
    }
  }
  int NB = 32;
  while (NB < n && NB < kBucketNB) NB <<= 1;
  for (int b = threadIdx.x; b < NB; b += kTileSortThreads) cnt[b] = 0;
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0) {
    red[2 * warp] = kmin;
    red[2 * warp + 1] = kmax;
  }
  __syncthreads();
  SORT_TRACE(2)
#pragma unroll 4
  for (int w = 0; w < kTileSortWarps; ++w) {
    kmin = min(kmin, red[2 * w]);
    kmax = max(kmax, red[2 * w + 1]);
  }
  // monotone (non-decreasing) key -> bucket map: fp32 conversion and a
  // positive scale preserve order, truncation keeps it weak
  const float scale = (float)NB / ((float)(kmax - kmin) + 1.0f);
#pragma unroll
  for (int r = 0; r < kTileSortIPT; ++r) {
    if (r >= R) break;
    if (r * kTileSortThreads + (int)threadIdx.x < n) atomicAdd(&cnt[min(NB - 1, (int)((float)(key[r] - kmin) * scale))], 1u);
  }
  __syncthreads();
  SORT_TRACE(3)
  // exclusive scan of the NB counters (E consecutive per thread) + the largest bucket
  const int E = (NB + kTileSortThreads - 1) / kTileSortThreads;
  const int b0 = threadIdx.x * E;
  uint32_t c[kBucketNB / kTileSortThreads > 0 ? kBucketNB / kTileSortThreads : 1];
  uint32_t tsum = 0, tmax = 0;
#pragma unroll
  for (int e = 0; e < (int)(sizeof(c) / sizeof(c[0])); ++e) {
    c[e] = (e < E && b0 + e < NB) ? cnt[b0 + e] : 0u;
    tsum += c[e];
    tmax = max(tmax, c[e]);
  }
  uint32_t incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  tmax = __reduce_max_sync(0xffffffffu, tmax);
  __syncthreads();
  SORT_TRACE(4)  // everyone has read cnt / red
  if (lane == 31) red[warp] = incl;
  if (lane == 0) red[kTileSortWarps + warp] = tmax;
  __syncthreads();
  SORT_TRACE(5)
  uint32_t wbase = 0, bmax = 0;
#pragma unroll 4
  for (int w = 0; w < kTileSortWarps; ++w) {
    if (w < warp) wbase += red[w];
    bmax = max(bmax, red[kTileSortWarps + w]);
  }
#ifdef FS4D_SORT_TRACE
  if (trace_me && threadIdx.x == 0) { const int o = blockIdx.x ? 16 : 0; g_sort_trace[o + 12] = bmax; g_sort_trace[o + 13] = NB; g_sort_trace[o + 14] = n; g_sort_trace[o + 15] = kmax - kmin; }
#endif
  if (bmax > (uint32_t)kBucketMax) return false;  // block-uniform
  {
    uint32_t run = wbase + incl - tsum;
#pragma unroll
    for (int e = 0; e < (int)(sizeof(c) / sizeof(c[0])); ++e)
      if (e < E && b0 + e < NB) {
        cnt[b0 + e] = run;
        run += c[e];
      }
  }
  __syncthreads();
  SORT_TRACE(6)
  // scatter through per-bucket cursors (the bucket starts); afterwards
  // cnt[b] is the end of bucket b, i.e. the start of bucket b + 1
#pragma unroll
  for (int r = 0; r < kTileSortIPT; ++r) {
    if (r >= R) break;
    if (r * kTileSortThreads + (int)threadIdx.x < n) {
      const int b = min(NB - 1, (int)((float)(key[r] - kmin) * scale));
      xbuf[atomicAdd(&cnt[b], 1u)] = ((unsigned long long)key[r] << 32) | val[r];
    }
  }
  __syncthreads();
  SORT_TRACE(7)
  for (int b = threadIdx.x; b < NB; b += kTileSortThreads) {
    const int s0 = b > 0 ? (int)cnt[b - 1] : 0, s1 = (int)cnt[b];
    for (int a = s0 + 1; a < s1; ++a) {
      const unsigned long long ka = xbuf[a];
      int q = a - 1;
      while (q >= s0 && key_less(ka, xbuf[q], z64)) {
        xbuf[q + 1] = xbuf[q];
        --q;
      }
      xbuf[q + 1] = ka;
    }
  }
  __syncthreads();
  SORT_TRACE(8)
  for (int q = threadIdx.x; q < n; q += kTileSortThreads) out_vals[q] = (uint32_t)xbuf[q];
  SORT_TRACE(11)
  return true;
}

// One warp sorts a tile of n < kWarpTile = 32 pairs: a key per lane (+inf
// padding), bitonic network over the lanes with shuffles, under the same
// total order as the CTA sorts.
__device__ __forceinline__ void warp_sort_small_tile(int tile, const unsigned long long* __restrict__ pkey,
                                                     const uint64_t* __restrict__ toff,
                                                     const uint32_t* __restrict__ tcnt, int64_t cap,
                                                     const double* __restrict__ z64, uint32_t* __restrict__ pvals,
                                                     uint2* __restrict__ ranges) {
  const int lane = threadIdx.x & 31;
  const uint64_t off = toff[tile];
  uint64_t end = off + tcnt[tile];
  if (end > (uint64_t)cap) end = (uint64_t)cap;
  const int n = off < end ? (int)(end - off) : 0;
  if (lane == 0) ranges[tile] = make_uint2((uint32_t)off, (uint32_t)(off + n));
  if (n == 0) return;  // warp-uniform
  unsigned long long key = lane < n ? pkey[off + lane] : 0xFFFFFFFFFFFFFFFFull - (unsigned long long)lane;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      // the lower lane of an ascending pair keeps the smaller key
      const bool other_less = key_less(other, key, z64);
      if (lower == up ? other_less : !other_less) key = other;
    }
  }
  if (lane < n) pvals[off + lane] = (uint32_t)key;
}

#ifdef FS4D_SORT_MINB  // A/B knob: minimum resident CTAs per SM
__global__ void __launch_bounds__(kTileSortThreads, FS4D_SORT_MINB) k_tile_sort(
#else
__global__ void __launch_bounds__(kTileSortThreads) k_tile_sort(
#endif
unsigned long long* __restrict__ pkey,
                                                                const uint64_t* __restrict__ toff,
                                                                const uint32_t* __restrict__ tcnt, int ntiles,
                                                                int64_t cap, const double* __restrict__ z64,
                                                                uint32_t* __restrict__ pvals, uint2* __restrict__ ranges,
                                                                const int32_t* __restrict__ tperm,
                                                                const uint32_t* __restrict__ counters, int radix_only) {
  extern __shared__ unsigned long long s_keys[];  // kSortSmemKeys exchange buffer (dynamic, 64 KB)
  __shared__ uint32_t wcnt[kTileSortWarps * 256];
  __shared__ uint32_t dbase[256];
#ifdef FS4D_SORT_TRACE
  if (tperm && (blockIdx.x == 0 || blockIdx.x == FS4D_SORT_TRACE2) && threadIdx.x == 0)
    g_sort_trace[blockIdx.x ? 16 : 0] = clock64();
#endif
  // Tiles of fewer than kWarpTile pairs (the end of the densest-first order,
  // half the tiles of a configs[1] frame) are sorted one per WARP, 16 to a CTA,
  // with a register bitonic network: a CTA-wide sort of a handful of keys cost
  // ~6k cycles of fixed phases and barriers.
  if (tperm) {
    const int nbig = (int)counters[CNT_BIG_TILES];
    if ((int)blockIdx.x >= nbig) {
      const int pos = nbig + ((int)blockIdx.x - nbig) * kTileSortWarps + (int)(threadIdx.x >> 5);
      if (pos < ntiles) warp_sort_small_tile(tperm[pos], pkey, toff, tcnt, cap, z64, pvals, ranges);
      return;
    }
  }
  const int tile = tperm ? tperm[blockIdx.x] : blockIdx.x;
  const uint64_t off = toff[tile];
  uint64_t end = off + tcnt[tile];
  if (end > (uint64_t)cap) end = (uint64_t)cap;  // overflow frame: status already raised
  const int n = off < end ? (int)(end - off) : 0;
  if (threadIdx.x == 0) ranges[tile] = make_uint2((uint32_t)off, (uint32_t)(off + n));
  if (n == 0) return;
  unsigned long long* keys = pkey + off;
  if (n <= kSortSmemKeys) {
    static_assert(kTileSortThreads * kTileSortIPT >= kSortSmemKeys, "bucket sort covers the smem tile size");
#ifdef FS4D_SORT_TRACE
    const bool trace_me = tperm && (blockIdx.x == 0 || blockIdx.x == FS4D_SORT_TRACE2);
    SORT_TRACE(1)
#else
    const bool trace_me = false;
#endif
    if (radix_only || !cta_bucket_sort_tile(keys, n, z64, pvals + off, s_keys, wcnt, dbase, trace_me)) {
      __syncthreads();
      cta_radix_sort_tile(keys, n, z64, pvals + off, s_keys, wcnt, dbase);
    }
  } else {
    bitonic_sort(keys, n, z64);  // oversized tile: in place in global memory (L2-resident)
    for (int q = threadIdx.x; q < n; q += blockDim.x) pvals[off + q] = (uint32_t)keys[q];
  }
}

// Tile offsets for up to a few tens of thousands of tiles in ONE block:
// exclusive scan of the per-tile counts (u64 offsets), the pair total, and
// the capacity check -- one launch instead of a 3-kernel device scan + check.
__global__ void __launch_bounds__(kTileScanThreads) k_tile_scan_check(const uint32_t* __restrict__ tcnt, int ntiles,
                                                                      uint64_t* __restrict__ toff, uint32_t* counters,
                                                                      int64_t cap, int32_t* status,
                                                                      int32_t* __restrict__ tperm) {
  __shared__ TileScanSmem sm;
  tile_scan_body(tcnt, ntiles, toff, nullptr, true, counters, cap, status, tperm, sm);
}

__global__ void k_pairs_check2(uint32_t* counters, int64_t cap, int32_t* status) {
  const uint64_t total = *reinterpret_cast<uint64_t*>(counters + CNT_PAIRS64);
  counters[CNT_PAIRS_CLAMPED] = (uint32_t)(total < (uint64_t)cap ? total : (uint64_t)cap);
  if (status) {
    status[FS4D_ST_N_VISIBLE] = (int32_t)counters[CNT_VISIBLE];
    status[FS4D_ST_PAIRS_LO] = (int32_t)(total & 0xFFFFFFFFu);
    status[FS4D_ST_PAIRS_HI] = (int32_t)(total >> 32);
    if (total > (uint64_t)cap) raise_status(status, FS4D_ERR_CAPACITY);
  }
}

// ---------------------------------------------------------------------------
// depth-ordered emission
// ---------------------------------------------------------------------------
constexpr int kDepthThreads = 256;                 // Gaussians per block (depth order)
constexpr int kDepthWarps = kDepthThreads / 32;
constexpr int kDepthMaxTileAxes = 1024;            // ntx + nty limit (mask table in shared memory)
constexpr int kDepthMaxTilesSmem = 8192;           // emit stages the block's base row in shared memory

// Per warp: masks[tx] = lanes whose tile rectangle covers column tx, and
// masks[ntx + ty] = lanes covering row ty (one ballot per column / row of the
// warp's bounding range; zero elsewhere).  A lane covers tile (tx, ty) iff it
// is in both.
__device__ __forceinline__ void warp_cover_masks(const int4& r, bool live, int ntx, int nty, uint32_t* masks) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < ntx + nty; i += 32) masks[i] = 0u;
  int lo_x = live ? r.x : INT_MAX, hi_x = live ? r.y : -1, lo_y = live ? r.z : INT_MAX, hi_y = live ? r.w : -1;
  lo_x = __reduce_min_sync(0xffffffffu, lo_x);
  hi_x = __reduce_max_sync(0xffffffffu, hi_x);
  lo_y = __reduce_min_sync(0xffffffffu, lo_y);
  hi_y = __reduce_max_sync(0xffffffffu, hi_y);
  __syncwarp();
  for (int tx = lo_x; tx <= hi_x; ++tx) {
    const uint32_t m = __ballot_sync(0xffffffffu, live && r.x <= tx && tx <= r.y);
    if (lane == 0) masks[tx] = m;
  }
  for (int ty = lo_y; ty <= hi_y; ++ty) {
    const uint32_t m = __ballot_sync(0xffffffffu, live && r.z <= ty && ty <= r.w);
    if (lane == 0) masks[ntx + ty] = m;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kDepthThreads) k_depth_counts(const uint32_t* __restrict__ order,
                                                                const uint32_t* __restrict__ counters, int64_t K,
                                                                const int4* __restrict__ tile_rect, int ntx, int nty,
                                                                uint32_t* __restrict__ table) {
  extern __shared__ uint32_t s_masks[];  // [warps][ntx + nty]
  const int warp = threadIdx.x >> 5;
  const int64_t M = counters[CNT_VISIBLE];
  const int64_t r = (int64_t)blockIdx.x * kDepthThreads + threadIdx.x;
  const bool live = r < M && r < K;
  const int4 rect = live ? tile_rect[order[r]] : make_int4(0, -1, 0, -1);
  const int axes = ntx + nty;
  warp_cover_masks(rect, live, ntx, nty, s_masks + warp * axes);
  __syncthreads();
  const int ntiles = ntx * nty;
  uint32_t* row = table + (int64_t)blockIdx.x * ntiles;
  for (int t = threadIdx.x; t < ntiles; t += kDepthThreads) {
    const int ty = t / ntx, tx = t - ty * ntx;
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kDepthWarps; ++w) c += __popc(s_masks[w * axes + tx] & s_masks[w * axes + ntx + ty]);
    row[t] = c;
  }
}

// Column scan of table [nblk][ntiles]: table[b][t] <- toff[t] + sum_{b' < b}
// table[b'][t].  A CTA owns 32 tiles (lane = tile: coalesced rows); its 32
// warps split the blocks into 32 chunks, sum them, and rewrite their chunk
// from the chunk's prefix.
constexpr int kScanColWarps = 32;
__global__ void __launch_bounds__(kScanColWarps * 32) k_depth_scan(uint32_t* __restrict__ table, int64_t nblk,
                                                                   int ntiles, const uint64_t* __restrict__ toff) {
  __shared__ uint32_t s_sum[kScanColWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int64_t per = (nblk + kScanColWarps - 1) / kScanColWarps;
  const int64_t b0 = warp * per, b1 = min(nblk, b0 + per);
  uint32_t sum = 0;
  if (t < ntiles) {
#pragma unroll 8
    for (int64_t b = b0; b < b1; ++b) sum += table[b * ntiles + t];
  }
  s_sum[warp][lane] = sum;
  __syncthreads();
  if (t >= ntiles) return;
  uint32_t run = (uint32_t)toff[t];
  for (int w = 0; w < warp; ++w) run += s_sum[w][lane];
#pragma unroll 8
  for (int64_t b = b0; b < b1; ++b) {
    uint32_t* cell = table + b * ntiles + t;
    const uint32_t c = *cell;
    *cell = run;
    run += c;
  }
}

__global__ void __launch_bounds__(kDepthThreads) k_depth_emit(const uint32_t* __restrict__ order,
                                                              const uint32_t* __restrict__ counters, int64_t K,
                                                              const int4* __restrict__ tile_rect, int ntx, int nty,
                                                              const uint32_t* __restrict__ table, int64_t cap,
                                                              uint32_t* __restrict__ pvals) {
  extern __shared__ uint32_t s_dyn[];  // [warps][ntx + nty] masks, then the block's base row [ntiles]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t M = counters[CNT_VISIBLE];
  const int64_t r = (int64_t)blockIdx.x * kDepthThreads + threadIdx.x;
  const bool live = r < M && r < K;
  const uint32_t g = live ? order[r] : 0u;
  const int4 rect = live ? tile_rect[g] : make_int4(0, -1, 0, -1);
  const int axes = ntx + nty, ntiles = ntx * nty;
  uint32_t* masks = s_dyn;
  warp_cover_masks(rect, live, ntx, nty, masks + warp * axes);
  const uint32_t* row = table + (int64_t)blockIdx.x * ntiles;
  uint32_t* base = s_dyn + kDepthWarps * axes;
  const bool staged = ntiles <= kDepthMaxTilesSmem;
  if (staged)
    for (int t = threadIdx.x; t < ntiles; t += kDepthThreads) base[t] = row[t];
  __syncthreads();
  if (!live) return;
  const uint32_t lt = (1u << lane) - 1u;
  for (int ty = rect.z; ty <= rect.w; ++ty) {
    uint32_t ym[kDepthWarps];
#pragma unroll
    for (int w = 0; w < kDepthWarps; ++w) ym[w] = masks[w * axes + ntx + ty];
    for (int tx = rect.x; tx <= rect.y; ++tx) {
      const int t = ty * ntx + tx;
      uint32_t pos = staged ? base[t] : row[t];
#pragma unroll
      for (int w = 0; w < kDepthWarps; ++w)
        if (w < warp) pos += __popc(masks[w * axes + tx] & ym[w]);
      pos += __popc(masks[warp * axes + tx] & ym[warp] & lt);
      if ((int64_t)pos < cap) pvals[pos] = g;
    }
  }
}

__global__ void k_tile_ranges_from_offsets(const uint64_t* __restrict__ toff, const uint32_t* __restrict__ tcnt,
                                           int ntiles, int64_t cap, uint2* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  uint64_t a = toff[t], e = a + tcnt[t];
  if (a > (uint64_t)cap) a = (uint64_t)cap;
  if (e > (uint64_t)cap) e = (uint64_t)cap;
  ranges[t] = make_uint2((uint32_t)a, (uint32_t)e);
}

// Opt-in (FS4D_BINNING=depth): measured on B200 at configs[1] the global
// depth sort alone (4 radix passes over 200k keys) costs more than the
// per-tile sort path it replaces (binning stage 157 vs 85 us), so the
// per-tile sort stays the default.
bool depth_binning_ok(const RenderLayout& L) {
  static const bool depth = getenv("FS4D_BINNING") && !strcmp(getenv("FS4D_BINNING"), "depth");
  return depth && L.ntx + L.nty <= kDepthMaxTileAxes && L.cap < (int64_t)0xFFFFFFFF;
}

// host: the whole binning stage (counts -> offsets -> partition -> per-tile sort)
void bin_tiles_device(const RenderLayout& L, void* ws, const int4* tile_rect, const uint32_t* dkeys,
                      const double* z64, uint32_t* counters, int32_t* status, cudaStream_t s) {
  const int64_t K = L.K;
  uint32_t* tcnt = at<uint32_t>(ws, L.tcnt);
  uint32_t* tcur = at<uint32_t>(ws, L.tcur);
  uint64_t* toff = at<uint64_t>(ws, L.toff64);
  // tcnt / tcur / ranges were zeroed and tcnt filled by k_preprocess's fused histogram
  const bool fused_scan = K > 0 && kEmitThreads <= kTileScanThreads && L.ntiles <= kHistMaxTiles &&
                          L.cap <= (int64_t)0xFFFFFFFFu && !depth_binning_ok(L);
  if (fused_scan) {
    // (the pair partition below computes and publishes the tile offsets)
  } else if (L.ntiles <= 64 * kTileScanThreads) {
    k_tile_scan_check<<<1, kTileScanThreads, 0, s>>>(tcnt, L.ntiles, toff, counters, L.cap, status,
                                                      at<int32_t>(ws, L.tperm));
  } else {
    exclusive_scan_u32_to_u64(tcnt, toff, L.ntiles, nullptr, reinterpret_cast<uint64_t*>(counters + CNT_PAIRS64),
                              at<void>(ws, L.scratch), s);
    k_pairs_check2<<<1, 1, 0, s>>>(counters, L.cap, status);
  }
  if (depth_binning_ok(L)) {
    const uint32_t* order = depth_order(L, ws, s, false);
    const int64_t nblk = ceil_div(K > 0 ? K : 1, kDepthThreads);
    uint32_t* table = at<uint32_t>(ws, L.dtable);
    const int axes = L.ntx + L.nty;
    const size_t smem_c = (size_t)kDepthWarps * axes * 4;
    const size_t smem_e = smem_c + (L.ntiles <= kDepthMaxTilesSmem ? (size_t)L.ntiles * 4 : 0);
    static size_t attr_c = 0, attr_e = 0;
    if (smem_c > 48 * 1024 && smem_c > attr_c) {
      cudaFuncSetAttribute(k_depth_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c);
      attr_c = smem_c;
    }
    if (smem_e > 48 * 1024 && smem_e > attr_e) {
      cudaFuncSetAttribute(k_depth_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e);
      attr_e = smem_e;
    }
    if (L.ntiles > 0) {
      k_depth_counts<<<(unsigned)nblk, kDepthThreads, smem_c, s>>>(order, counters, K, tile_rect, L.ntx, L.nty, table);
      k_depth_scan<<<(unsigned)ceil_div(L.ntiles, 32), kScanColWarps * 32, 0, s>>>(table, nblk, L.ntiles, toff);
      k_depth_emit<<<(unsigned)nblk, kDepthThreads, smem_e, s>>>(order, counters, K, tile_rect, L.ntx, L.nty, table,
                                                                 L.cap, at<uint32_t>(ws, L.pvals0));
      k_tile_ranges_from_offsets<<<(unsigned)ceil_div(L.ntiles, 256), 256, 0, s>>>(toff, tcnt, L.ntiles, L.cap,
                                                                                  at<uint2>(ws, L.ranges));
    }
    return;
  }
  unsigned long long* pkey = at<unsigned long long>(ws, L.pkey64);
  if (fused_scan)
    k_emit_partition<true><<<(unsigned)ceil_div(K, kEmitThreads), kEmitThreads, 0, s>>>(
        tile_rect, dkeys, K, L.ntx, L.ntiles, toff, tcur, L.cap, pkey, tcnt, counters, status,
        at<int32_t>(ws, L.tperm));
  else if (K > 0)
    k_emit_partition<false><<<(unsigned)ceil_div(K, kEmitThreads), kEmitThreads, 0, s>>>(
        tile_rect, dkeys, K, L.ntx, L.ntiles, toff, tcur, L.cap, pkey, nullptr, nullptr, nullptr, nullptr);
  // FS4D_TILE_SORT=radix: the three-pass LSD radix sort for every tile (A/B)
  static const int radix_only = getenv("FS4D_TILE_SORT") && !strcmp(getenv("FS4D_TILE_SORT"), "radix");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmemKeys * 8);
    attr = true;
  }
  if (L.ntiles > 0)
    k_tile_sort<<<L.ntiles, kTileSortThreads, kSortSmemKeys * 8, s>>>(pkey, toff, tcnt, L.ntiles, L.cap, z64,
                                                                     at<uint32_t>(ws, L.pvals0),
                                                                     at<uint2>(ws, L.ranges),
                                                                     L.ntiles <= 64 * kTileScanThreads
                                                                         ? at<int32_t>(ws, L.tperm)
                                                                         : nullptr,
                                                                     counters, radix_only);
}

}  // namespace fs4d
