// Shared device helpers for the B200 Chung–Lu generator (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define CLG_FULL 0xffffffffu

namespace clg {

// ---- splitmix64 finaliser (reference rng.hpp:11-16) ----------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Edge hash of the streaming fold's checksum (sum over edges mod 2^64):
// multiply / fold / multiply / fold of the 64-bit key (u << 32) | v.  Not a
// reference function (the reference has no checksum); ten integer
// instructions per edge on the device.  Mirrored by oracle/clgen_oracle.c
// (orc_edge_hash), oracle/ref_driver.cpp and tests/stats.py.
__host__ __device__ __forceinline__ uint64_t edge_hash(uint32_t u, uint32_t v) {
  uint64_t z = ((static_cast<uint64_t>(u) << 32) | v) * 0x9e3779b97f4a7c15ULL;
  z ^= z >> 32;
  z *= 0xd6e8feb86659fd93ULL;
  return z ^ (z >> 32);
}

// rng.hpp:20-22
__host__ __device__ __forceinline__ uint64_t node_rng_key(uint64_t seed, int64_t u) {
  return mix64(seed + static_cast<uint64_t>(u) * 0x9e3779b97f4a7c15ULL);
}

// 64-bit rotate as two 32-bit funnel shifts (SHF.L.W), k in [1, 63] constant
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) {
  const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
  uint32_t nlo, nhi;
  if (k < 32) {
    nhi = __funnelshift_l(lo, hi, k);
    nlo = __funnelshift_l(hi, lo, k);
  } else {
    nhi = __funnelshift_l(hi, lo, k - 32);
    nlo = __funnelshift_l(lo, hi, k - 32);
  }
  return (static_cast<uint64_t>(nhi) << 32) | nlo;
}

// Per-source xoshiro256++ stream, bit-identical to the reference RngStream
// (rng.hpp:26-69).  Four words live in registers of the lane walking u.
struct Xoshiro {
  uint64_t s0, s1, s2, s3;

  __device__ __forceinline__ void seed_key(uint64_t key) {
    uint64_t sm = key;
    uint64_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sm += 0x9e3779b97f4a7c15ULL;
      uint64_t z = sm;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      w[i] = z ^ (z >> 31);
    }
    s0 = w[0]; s1 = w[1]; s2 = w[2]; s3 = w[3];
    if ((s0 | s1 | s2 | s3) == 0) s0 = 1;  // rng.hpp:41
  }

  __device__ __forceinline__ uint64_t next() {
    const uint64_t result = rotl64(s0 + s3, 23) + s0;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return result;
  }

  // xoshiro256+ output (s0 + s3) with the same state transition: used by the
  // counter stream only (its top 53 bits are what the samplers consume).
  __device__ __forceinline__ uint64_t next_plus() {
    const uint64_t result = s0 + s3;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return result;
  }

  // rng.hpp:58-63: (x>>11)*2^-53, exact zeros rejected (loop taken with
  // probability 2^-53 per draw).
  __device__ __forceinline__ double open01() {
    for (;;) {
      const double r = __dmul_rn(static_cast<double>(next() >> 11), 0x1.0p-53);
      if (r > 0.0) return r;
    }
  }
};

// xoroshiro128++ (Blackman & Vigna): the counter stream's per-(unit, lane)
// generator.  128-bit state seeded by two splitmix64 outputs of the stream
// key; all 64 output bits are full quality (the samplers use the top 53 for
// an exponential and the low 11 as acceptance bits).
struct Xoro128 {
  uint64_t s0, s1;

  __device__ __forceinline__ void seed_key(uint64_t key) {
    s0 = mix64(key);
    s1 = mix64(key + 0x9e3779b97f4a7c15ULL);
    if ((s0 | s1) == 0) s0 = 1;
  }

  __device__ __forceinline__ uint64_t next() {
    const uint64_t a = s0;
    uint64_t b = s1;
    const uint64_t result = rotl64(a + b, 17) + a;
    b ^= a;
    s0 = rotl64(a, 49) ^ b ^ (b << 21);
    s1 = rotl64(b, 28);
    return result;
  }

  __device__ __forceinline__ uint64_t next_plus() { return next(); }

  __device__ __forceinline__ double open01() {
    for (;;) {
      const double r = __dmul_rn(static_cast<double>(next() >> 11), 0x1.0p-53);
      if (r > 0.0) return r;
    }
  }
};

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-inclusive scan of an int64 value.
__device__ __forceinline__ int64_t warp_inclusive_scan(int64_t x) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(CLG_FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ int64_t warp_sum(int64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(CLG_FULL, x, o);
  return x;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(CLG_FULL, x, o);
  return x;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Optional per-warp busy interval: slots[2*gw] = start, slots[2*gw+1] = end
// (ns, %globaltimer), gw = global warp id + base.  Used to report the
// level-2 load balance (max/mean per-warp busy time).
struct WarpProf {
  unsigned long long* slots;
  int base;
  __device__ __forceinline__ int gw() const {
    return base + static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  }
};

}  // namespace clg
