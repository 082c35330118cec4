// Device-wide exclusive scan and stable LSD radix sort used by tile binning.
//
// They replace the two order-defining steps of the reference binner:
//   * the global *stable* depth argsort  (rasterizer.py:163, np.argsort kind="stable")
//   * per-tile lists that keep that order (rasterizer.py:202-206)
// Both sorts are stable so ties resolve by source index exactly like NumPy's
// stable argsort.  Element counts may live in device memory (no host sync):
// grids are sized for a capacity and blocks past the live count exit early.
#pragma once
#include "common.cuh"

namespace fs4d {

constexpr int kScanThreads = 256;
constexpr int kScanIPT = 8;
constexpr int kScanChunk = kScanThreads * kScanIPT;

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortIPT = 8;
constexpr int kSortChunk = kSortThreads * kSortIPT;
constexpr int kMaxRadixBits = 8;  // measured: 11-bit digits cost more per pass than they save in passes
constexpr int kMaxRadix = 1 << kMaxRadixBits;

size_t scan_scratch_bytes(int64_t cap);
// out[i] = sum_{j<i} in[j] for i < n; *total = sum of all n.  n = min(*n_dev, cap)
// when n_dev != nullptr, else cap.
void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t cap,
                               const uint32_t* n_dev, uint64_t* total, void* scratch,
                               cudaStream_t stream);

size_t radix_scratch_bytes(int64_t cap);
// Stable sort of (key, value) by key bits [begin_bit, end_bit).  Ping-pongs
// between buffer 0 and 1; returns the index holding the result.
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                     int begin_bit, int end_bit, void* scratch, cudaStream_t stream);
// number of passes (and so ping-pong flips) radix_sort_pairs makes over `bits` key bits
int radix_passes(int bits);

}  // namespace fs4d
