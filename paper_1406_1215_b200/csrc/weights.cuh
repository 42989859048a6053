// Weight-array kernels: canonical blocked sum (weights.cpp:21-30) and the
// non-increasing-order contract check (weights.cpp:47-53).
#pragma once

#include "common.cuh"

namespace clg {

constexpr int64_t kSumBlock = 4096;  // weights.cpp:16

// One thread folds one 4096-element block left to right from 0.0, exactly as
// weights.cpp:24-26.  The block's elements are staged through shared memory
// 32 at a time so the global loads stay coalesced (a warp reads 32
// consecutive doubles of one block) while each thread consumes its own row.
__global__ void __launch_bounds__(128) blocked_partials_kernel(const double* __restrict__ x,
                                                               int64_t n, double* __restrict__ part,
                                                               int64_t nblocks) {
  __shared__ double tile[128][33];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t blk0 = static_cast<int64_t>(blockIdx.x) * 128;
  double acc = 0.0;
  for (int k0 = 0; k0 < kSumBlock; k0 += 32) {
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const int row = wid * 32 + rr;
      const int64_t idx = (blk0 + row) * kSumBlock + k0 + lane;
      tile[row][lane] = idx < n ? x[idx] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; ++k) acc = __dadd_rn(acc, tile[t][k]);
    __syncthreads();
  }
  if (blk0 + t < nblocks) part[blk0 + t] = acc;
}

// weights.cpp:27: partials combined left to right from 0.0.  One block:
// the threads stage chunks of partials in shared memory (double-buffered)
// while thread 0 folds the previous chunk in order, so the sequential fold
// waits on shared-memory loads, not on DRAM.
constexpr int kFoldChunk = 2048;
__global__ void __launch_bounds__(256) fold_partials_kernel(const double* __restrict__ part, int64_t nblocks,
                                                            double* __restrict__ out) {
  __shared__ double buf[2][kFoldChunk];
  double total = 0.0;
  const int64_t nchunks = (nblocks + kFoldChunk - 1) / kFoldChunk;
  for (int i = threadIdx.x; i < kFoldChunk; i += blockDim.x)
    if (i < nblocks) buf[0][i] = part[i];
  __syncthreads();
  for (int64_t c = 0; c < nchunks; ++c) {
    const int cur = static_cast<int>(c & 1);
    const int64_t base = c * kFoldChunk;
    if (threadIdx.x == 0) {
      const int m = static_cast<int>(nblocks - base < kFoldChunk ? nblocks - base : kFoldChunk);
      for (int i = 0; i < m; ++i) total = __dadd_rn(total, buf[cur][i]);
    } else if (c + 1 < nchunks) {
      const int64_t nb = base + kFoldChunk;
      for (int i = threadIdx.x - 1; i < kFoldChunk; i += blockDim.x - 1)
        if (nb + i < nblocks) buf[cur ^ 1][i] = part[nb + i];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = total;
}

// First position u with w[u] > w[u-1] (or NaN/negative), else n; `runs`
// counts the maximal runs of bitwise-equal weights.
__global__ void check_sorted_kernel(const double* __restrict__ w, int64_t n,
                                    unsigned long long* first_bad,
                                    unsigned long long* first_negative,
                                    unsigned long long* runs) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned long long starts = 0;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    bool start = false;
    if (i < n) {
      const double x = w[i];
      if (!(x >= 0.0)) atomicMin(first_negative, static_cast<unsigned long long>(i));
      const double y = i > 0 ? w[i - 1] : 0.0;
      if (i > 0 && x > y) atomicMin(first_bad, static_cast<unsigned long long>(i));
      start = i == 0 || __double_as_longlong(x) != __double_as_longlong(y);
    }
    starts += __popc(__ballot_sync(CLG_FULL, start));
  }
  if ((threadIdx.x & 31) == 0 && starts) atomicAdd(runs, starts);
}

// Run-length table of a weight vector with repeated values: run_len[i] =
// (end of the run of bitwise-equal weights containing i) - i, capped at
// INT32_MAX.  The samplers use it to skip the w[v] gather while a chain stays
// inside one run.  Tiles of kRunTile elements; the run crossing a tile's
// right edge is resolved by a galloping search.
constexpr int kRunTile = 2048;
constexpr int kRunThreads = 256;

__global__ void __launch_bounds__(kRunThreads) run_length_kernel(const double* __restrict__ w, int64_t n,
                                                                 int32_t* __restrict__ run_len) {
  constexpr int kPer = kRunTile / kRunThreads;
  __shared__ long long s_w[kRunTile + 1];
  __shared__ long long s_tail;
  __shared__ long long s_warp[kRunThreads / 32];
  __shared__ int32_t s_len[kRunTile];
  const int64_t lo = static_cast<int64_t>(blockIdx.x) * kRunTile;
  const int64_t hi = lo + kRunTile < n ? lo + kRunTile : n;
  const int cnt = static_cast<int>(hi - lo);
  for (int k = threadIdx.x; k <= cnt; k += kRunThreads)
    s_w[k] = lo + k < n ? __double_as_longlong(w[lo + k]) : ~0ll;  // ~0: never equal to a weight (NaN bits)
  if (threadIdx.x == 0) {
    // end of the run of w[hi-1] beyond the tile (galloping + binary search)
    const long long x = __double_as_longlong(w[hi - 1]);
    int64_t good = hi - 1, step = 1, bad = n;
    while (good + step < n) {
      if (__double_as_longlong(w[good + step]) != x) {
        bad = good + step;
        break;
      }
      good += step;
      step <<= 1;
    }
    while (bad - good > 1) {
      const int64_t mid = good + (bad - good) / 2;
      if (__double_as_longlong(w[mid]) == x) good = mid;
      else bad = mid;
    }
    s_tail = bad;
  }
  __syncthreads();
  // thread segment [b, b+kPer): nearest run end at or right of its first element
  const int b = threadIdx.x * kPer;
  long long first_end = LLONG_MAX;
  for (int k = kPer - 1; k >= 0; --k)
    if (b + k < cnt && s_w[b + k + 1] != s_w[b + k]) first_end = lo + b + k + 1;
  // carry = min over threads to the right (exclusive suffix min), seeded by the tail
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl = first_end;
  for (int d = 1; d < 32; d <<= 1) {
    const long long o = __shfl_down_sync(CLG_FULL, incl, d);
    if (lane + d < 32 && o < incl) incl = o;
  }
  if (lane == 0) s_warp[wid] = incl;
  __syncthreads();
  long long carry = __shfl_down_sync(CLG_FULL, incl, 1);
  if (lane == 31) carry = LLONG_MAX;
  for (int x = wid + 1; x < kRunThreads / 32; ++x)
    if (s_warp[x] < carry) carry = s_warp[x];
  if (carry == LLONG_MAX) carry = s_tail;
  for (int k = kPer - 1; k >= 0; --k) {
    if (b + k >= cnt) continue;
    if (s_w[b + k + 1] != s_w[b + k]) carry = lo + b + k + 1;
    const long long d = carry - (lo + b + k);
    s_len[b + k] = d > INT_MAX ? INT_MAX : static_cast<int32_t>(d);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < cnt; k += kRunThreads) run_len[lo + k] = s_len[k];
}

// First index i with sources[i] outside [0,n) (edge_skip.cpp:54).
__global__ void check_sources_kernel(const int64_t* __restrict__ src, int64_t k, int64_t n,
                                     unsigned long long* first_bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    const int64_t u = src[i];
    if (u < 0 || u >= n) atomicMin(first_bad, static_cast<unsigned long long>(i));
  }
}

}  // namespace clg
