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

// weights.cpp:27: partials combined left to right from 0.0.
__global__ void fold_partials_kernel(const double* __restrict__ part, int64_t nblocks,
                                     double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0.0;
  for (int64_t i = 0; i < nblocks; ++i) total = __dadd_rn(total, part[i]);
  *out = total;
}

// First position u with w[u] > w[u-1] (or NaN/negative), else n.
__global__ void check_sorted_kernel(const double* __restrict__ w, int64_t n,
                                    unsigned long long* first_bad,
                                    unsigned long long* first_negative) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = w[i];
    if (!(x >= 0.0)) atomicMin(first_negative, static_cast<unsigned long long>(i));
    if (i > 0 && x > w[i - 1]) atomicMin(first_bad, static_cast<unsigned long long>(i));
  }
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
