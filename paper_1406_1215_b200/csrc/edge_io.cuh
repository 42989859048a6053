// Edge persistence in the reference's formats (edge_io.cpp:72-88):
//   binary: "CLGEDGE1", u32 version 1, u32 0, u64 count, then (u64 u, u64 v)
//           little-endian per edge;
//   text:   "u v\n" per edge.
// The device widens uint32 pairs to u64 pairs (binary) or renders decimal
// text (text) chunk by chunk; the host only streams bytes to the file.
#pragma once

#include "common.cuh"

namespace clg {

__global__ void widen_pairs_kernel(const uint2* __restrict__ in, int64_t m,
                                   unsigned long long* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 e = in[i];
    out[2 * i] = e.x;  // the GPU is little-endian, as the format requires
    out[2 * i + 1] = e.y;
  }
}

__device__ __forceinline__ int dec_len(uint32_t x) {
  int l = 1;
  while (x >= 10u) {
    x /= 10u;
    ++l;
  }
  return l;
}

// Text: one thread per edge computes its line length; offsets come from an
// exclusive scan; then each thread writes its digits.
__global__ void text_len_kernel(const uint2* __restrict__ in, int64_t m, int32_t* __restrict__ len) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 e = in[i];
    len[i] = dec_len(e.x) + dec_len(e.y) + 2;
  }
}

__global__ void text_render_kernel(const uint2* __restrict__ in, int64_t m, const int64_t* __restrict__ off,
                                   char* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 e = in[i];
    char* p = out + off[i];
    int lu = dec_len(e.x), lv = dec_len(e.y);
    uint32_t x = e.x;
    for (int k = lu - 1; k >= 0; --k) {
      p[k] = static_cast<char>('0' + x % 10u);
      x /= 10u;
    }
    p[lu] = ' ';
    x = e.y;
    for (int k = lv - 1; k >= 0; --k) {
      p[lu + 1 + k] = static_cast<char>('0' + x % 10u);
      x /= 10u;
    }
    p[lu + 1 + lv] = '\n';
  }
}

}  // namespace clg
