// pxg_prims.cuh — the two data-parallel primitives of the per-pass path, hand-written for
// this library (round 1 called CUB's DeviceScan / DeviceRadixSort here):
//
//   exclusive_sum   int32 exclusive prefix sum of n values (connection slot offsets of every
//                   pixel, and the bin-major histogram of the sort below): tile scan with
//                   warp shuffles -> one-block scan of the tile sums -> add-back.
//   stable_bin_sort stable counting sort of (bin, value) pairs by a small integer bin
//                   (bins < kSortBins): per-tile shared-memory histogram -> exclusive_sum over
//                   the bin-major (bin, tile) matrix -> stable scatter, one warp per tile
//                   walking its elements in order, 32 at a time, ranking equal bins with
//                   __match_any_sync. Pixel order is kept inside every bin, which is what
//                   GammaMatrix::record_contribution's scan-order accumulation needs
//                   (proj/src/proxy.cpp:807-808).
//
// Both are exact integer work and deterministic; the host only enqueues.
#pragma once

#include <cuda_runtime.h>

namespace pxg {

#if defined(__CUDACC__)

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096 values per block

__device__ __forceinline__ int warp_inclusive_sum(int v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) >= d) v += o;
  }
  return v;
}

// Exclusive sum of the block's per-thread values (all threads call); returns this thread's
// exclusive prefix and the block total in `total`. blockDim.x <= 1024.
__device__ __forceinline__ int block_exclusive_sum(int v, int& total) {
  __shared__ int s_warp[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = (blockDim.x + 31) >> 5;
  const int inc = warp_inclusive_sum(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < nwarp ? s_warp[lane] : 0;
    const int wi = warp_inclusive_sum(w);
    s_warp[lane] = wi - w;  // exclusive prefix of the warp sums
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  const int pre = s_warp[warp] + inc - v;
  total = s_warp[32];
  __syncthreads();  // s_warp is reused by the caller's next call
  return pre;
}

// Tile scan: out[i] = exclusive sum within the tile, tile_sum[tile] = the tile's total.
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const int* in, int* out, int* tile_sum, long long n) {
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile + static_cast<long long>(threadIdx.x) * kScanItems;
  int v[kScanItems];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + k;
    v[k] = i < n ? in[i] : 0;
    sum += v[k];
  }
  int total;
  int pre = block_exclusive_sum(sum, total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + k;
    if (i < n) out[i] = pre;
    pre += v[k];
  }
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// One block: exclusive scan of the tile sums in place (any count; chunks of blockDim.x).
__global__ void __launch_bounds__(1024) k_scan_tile_sums(int* tile_sum, int ntiles) {
  int carry = 0;
  for (int b = 0; b < ntiles; b += blockDim.x) {
    const int i = b + threadIdx.x;
    const int v = i < ntiles ? tile_sum[i] : 0;
    int total;
    const int pre = block_exclusive_sum(v, total);
    if (i < ntiles) tile_sum[i] = carry + pre;
    carry += total;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(int* out, const int* tile_pre, long long n) {
  const int add = tile_pre[blockIdx.x];
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + k * kScanThreads + threadIdx.x;
    if (i < n) out[i] += add;
  }
}

inline size_t scan_tiles(long long n) { return static_cast<size_t>((n + kScanTile - 1) / kScanTile); }

// out[i] = in[0] + ... + in[i-1], i < n (in != out). tmp: scan_tiles(n) ints. 3 launches.
inline int exclusive_sum(const int* in, int* out, long long n, int* tmp, cudaStream_t st) {
  if (n <= 0) return 0;
  const int nt = static_cast<int>(scan_tiles(n));
  k_scan_tiles<<<nt, kScanThreads, 0, st>>>(in, out, tmp, n);
  k_scan_tile_sums<<<1, 1024, 0, st>>>(tmp, nt);
  k_scan_add<<<nt, kScanThreads, 0, st>>>(out, tmp, n);
  return 3;
}

// ---------------------------------------------------------------- stable sort by bin
constexpr int kSortBins = 3201;   // gamma bins: 0 = no contribution, 1 + t * 100 + s (32 x 100)
constexpr int kSortTile = 1024;   // elements per tile = one warp's share

// hist[bin * ntiles + tile] = number of elements of the tile in `bin`.
__global__ void __launch_bounds__(256) k_sort_hist(const int* bins, int n, int ntiles, int* hist) {
  __shared__ int s_h[kSortBins];
  const int tile = blockIdx.x;
  for (int b = threadIdx.x; b < kSortBins; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const int lo = tile * kSortTile, hi = min(n, lo + kSortTile);
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&s_h[bins[i]], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < kSortBins; b += blockDim.x) hist[static_cast<size_t>(b) * ntiles + tile] = s_h[b];
}

// Stable scatter: one warp per tile walks its elements in order. `start` is the exclusive sum
// of hist (bin-major), i.e. the destination of the tile's first element of each bin.
__global__ void __launch_bounds__(32) k_sort_scatter(const int* bins, const double* vals, int n, int ntiles,
                                                     const int* start, int* bins_out, double* vals_out) {
  __shared__ int s_next[kSortBins];
  const int tile = blockIdx.x, lane = threadIdx.x;
  for (int b = lane; b < kSortBins; b += 32) s_next[b] = start[static_cast<size_t>(b) * ntiles + tile];
  __syncwarp();
  const int lo = tile * kSortTile, hi = min(n, lo + kSortTile);
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const int i = i0 + lane;
    const bool has = i < hi;
    const int b = has ? bins[i] : -1 - lane;  // absent lanes match nobody
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    if (has) {
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int dst = s_next[b] + rank;
      bins_out[dst] = b;
      vals_out[dst] = vals[i];
    }
    __syncwarp();
    if (has && lane == 31 - __clz(peers)) s_next[b] += __popc(peers);  // the group's last lane advances the bin
    __syncwarp();
  }
}

inline int sort_tiles(int n) { return (n + kSortTile - 1) / kSortTile; }
// ints of scratch stable_bin_sort needs: the histogram, its scan, and the scan's tile sums
inline size_t sort_tmp_ints(int n) {
  const size_t m = static_cast<size_t>(kSortBins) * sort_tiles(n);
  return 2 * m + scan_tiles(static_cast<long long>(m)) + 16;
}

// (bins_out, vals_out) = (bins, vals) stably sorted by bin (0 <= bin < kSortBins).
inline int stable_bin_sort(const int* bins, const double* vals, int n, int* bins_out, double* vals_out, int* tmp,
                           cudaStream_t st) {
  if (n <= 0) return 0;
  const int nt = sort_tiles(n);
  const long long m = static_cast<long long>(kSortBins) * nt;
  int* hist = tmp;
  int* start = tmp + m;
  int* scan_tmp = tmp + 2 * m;
  k_sort_hist<<<nt, 256, 0, st>>>(bins, n, nt, hist);
  const int l = exclusive_sum(hist, start, m, scan_tmp, st);
  k_sort_scatter<<<nt, 32, 0, st>>>(bins, vals, n, nt, start, bins_out, vals_out);
  return 2 + l;
}

#endif  // __CUDACC__

}  // namespace pxg
