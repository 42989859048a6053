// Level-1 UCP partition kernels (partition.cpp:107-203): boundary discovery
// from the exact cumulative costs.  C_u is non-decreasing (c_u >= 1), so
// boundary k is the first node whose partition index reaches k; every node
// compares its own index with its predecessor's and records the k it crosses
// (the same set plan_ucp_oracle's linear scan assigns, partition.cpp:191-200,
// including the empty partitions a dominant node skips).
#pragma once

#include "common.cuh"

namespace clg {

// cost.cpp:53-60
__device__ __forceinline__ int partition_of_dev(double c, double z_bar, int P) {
  const double k = floor(__ddiv_rn(c, z_bar));
  if (k < 0.0) return 0;
  if (k >= static_cast<double>(P)) return P - 1;
  const int i = static_cast<int>(k);
  return i > P - 1 ? P - 1 : i;
}

__global__ void ucp_transitions_kernel(const double* __restrict__ cum, int64_t lo, int64_t hi,
                                       double z_offset, double z_bar, int P,
                                       long long* __restrict__ found) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t u = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < hi; u += stride) {
    const double C = __dadd_rn(cum[u], z_offset);  // finalize_offsets, cost.cpp:48-51
    const int cur = partition_of_dev(C, z_bar, P);
    // C_{lo-1} is bitwise Z_i (partition.cpp:126-130)
    const double Cp = u == lo ? z_offset : __dadd_rn(cum[u - 1], z_offset);
    const int prev = partition_of_dev(Cp, z_bar, P);
    for (int k = prev + 1; k <= cur; ++k) found[k] = u;
  }
}

__global__ void add_offset_kernel(const double* __restrict__ cum, double* __restrict__ out, int64_t lo,
                                  int64_t hi, double z_offset) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t u = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < hi; u += stride)
    out[u] = __dadd_rn(cum[u], z_offset);
}

__global__ void fill_f64_kernel(double* __restrict__ x, int64_t lo, int64_t hi, double v) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t u = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < hi; u += stride) x[u] = v;
}

__global__ void fill_i64_kernel(long long* __restrict__ x, int64_t m, long long v) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < m; u += stride) x[u] = v;
}

}  // namespace clg
