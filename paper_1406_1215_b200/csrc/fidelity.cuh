// Degree-fidelity reporter (the device analogue of degree_histogram +
// compare_distributions, /root/reference/proj/core/src/analysis.cpp:18-85).
//
// expected degree  d_u = max(w_u - w_u*w_u/S, 0)        (analysis.cpp:54-56)
// bins             k = floor(log2(x)), counts of nodes per k for expected
//                  (d_u > 0) and generated (degree > 0) values
// expected_sum is the reference's sequential fold over u, replayed exactly by
// exact_fold.cuh, so mean_expected matches bit for bit.
#pragma once

#include "common.cuh"

namespace clg {

constexpr int kFidBinOff = 1100;  // bins k in [-1100, 1100)
constexpr int kFidBins = 2200;

// floor(log2(x)) for x > 0 as glibc's floor(log2(x)) computes it: the
// exponent, except that values within ~1 ulp of log2-rounding below a power
// of two round up to it (log2 returns the integer).
__device__ __forceinline__ int log2_bin(double x) {
  int e;
  const long long b = __double_as_longlong(x);
  const int ex = static_cast<int>((b >> 52) & 0x7ff);
  if (ex == 0) {
    e = static_cast<int>(floor(log2(x)));  // subnormal: rare, defer to libm
    return e;
  }
  e = ex - 1023;
  const long long man = b & 0x000fffffffffffffLL;
  if (man > 0x000ffffffffff000LL) {  // x within 2^-40 (relative) below 2^(e+1)
    const double l = log2(x);
    return static_cast<int>(floor(l));
  }
  return e;
}

__global__ void fid_expected_kernel(const double* __restrict__ w, int64_t n, double S, double* __restrict__ d,
                                    unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[kFidBins];
  for (int i = threadIdx.x; i < kFidBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += stride) {
    const double wu = w[u];
    double du = S > 0.0 ? __dsub_rn(wu, __ddiv_rn(__dmul_rn(wu, wu), S)) : 0.0;
    if (du < 0.0) du = 0.0;
    d[u] = du;
    if (du > 0.0) {
      int k = log2_bin(du) + kFidBinOff;
      k = k < 0 ? 0 : (k >= kFidBins ? kFidBins - 1 : k);
      atomicAdd(&sh[k], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kFidBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(sh[i]));
}

// Generated degrees (uint32 per node): log2 bins of positive degrees and the
// zero-degree count (hist[kFidBins]).
__global__ void fid_generated_kernel(const uint32_t* __restrict__ deg, int64_t n,
                                     unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[33];
  if (threadIdx.x < 33) sh[threadIdx.x] = 0;
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += stride) {
    const uint32_t x = deg[u];
    atomicAdd(&sh[x ? 31 - __clz(x) : 32], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32 && sh[threadIdx.x]) atomicAdd(&hist[kFidBinOff + threadIdx.x], static_cast<unsigned long long>(sh[threadIdx.x]));
  if (threadIdx.x == 32 && sh[32]) atomicAdd(&hist[kFidBins], static_cast<unsigned long long>(sh[32]));
}

// Undirected degrees of a materialised edge list (degree_histogram's count).
__global__ void edge_degree_kernel(const uint2* __restrict__ e, int64_t m, uint32_t* __restrict__ deg) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 x = e[i];
    atomicAdd(&deg[x.x], 1u);
    atomicAdd(&deg[x.y], 1u);
  }
}

}  // namespace clg
