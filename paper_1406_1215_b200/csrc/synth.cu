// Device weight synthesis: synth_powerlaw
// (weights.cpp:103-128) + the descending sort of make_weight_sequence
// (weights.cpp:32-55), bit-identical to the host synthesiser, with the
// weights born in HBM.
//
//   draws   The reference draws n values from ONE sequential xoshiro256++
//           stream (RngStream(mix64(seed ^ 0x706c73796e7468)), weights.cpp:17,112).
//           The state update is linear over GF(2), so the state before draw
//           c*2048 is T^(c*2048) s0: the host squares the 256x256 bit matrix
//           T up to T^(2048*2^b), b < 32 (8 KB each), a first kernel composes
//           the matrices picked by the bits of c, and each thread of the draw
//           kernel then steps its own 2048 draws.
//   pow     (a^k + r (b^k - a^k))^(1/k) with glibc pow.  ddpow.cuh evaluates
//           the power in double-double and certifies its rounding; the ~6% of
//           draws it cannot certify are compacted, resolved by the host's libm
//           pow (the reference's own third-party dependency) and scattered
//           back.  No draw is left to device rounding luck.
//   sort    cub radix sort, descending (values only: equal weights are
//           indistinguishable, so the stable label order does not change them).
//   scale   optional: w *= target_mean / (blocked_sum(w) / n), the C4 recipe
//           (SURVEY.md §8(d)); blocked_sum is the context's bit-exact fold.
//
// A zero draw (probability 2^-53 each) makes the reference redraw and shifts
// the rest of the stream; it is detected and reported as CLGEN_ERANGE rather
// than handled.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "../../include/clgen_dev.h"
#include "ddpow.cuh"

int clgen_internal_fail(int code, const char* msg);  // capi.cu

namespace {

constexpr int kChunkLog = 11;
constexpr int64_t kChunk = int64_t(1) << kChunkLog;  // draws per thread
constexpr int kLevels = 32 - kChunkLog + 1;         // chunk-index bits for n < 2^32
constexpr uint64_t kSynthTag = 0x706c73796e7468ULL;  // weights.cpp:17

struct S256 {
  uint64_t s[4];
};

__host__ __device__ inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// xoshiro256++ state update (rng.hpp:47-60); the output function is not linear
// and is applied only when drawing
__host__ __device__ inline void step(S256& x) {
  const uint64_t t = x.s[1] << 17;
  x.s[2] ^= x.s[0];
  x.s[3] ^= x.s[1];
  x.s[1] ^= x.s[2];
  x.s[0] ^= x.s[3];
  x.s[2] ^= t;
  x.s[3] = rotl64(x.s[3], 45);
}

// column j of a matrix = image of the j-th basis state
struct Mat {
  S256 col[256];
};

S256 apply(const Mat& m, const S256& v) {
  S256 r{};
  for (int j = 0; j < 256; ++j)
    if ((v.s[j >> 6] >> (j & 63)) & 1)
      for (int q = 0; q < 4; ++q) r.s[q] ^= m.col[j].s[q];
  return r;
}

void square(const Mat& m, Mat& out) {
  for (int j = 0; j < 256; ++j) out.col[j] = apply(m, m.col[j]);
}

uint64_t mix64_host(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// RngStream(key) seeding (rng.hpp:28-40)
S256 seed_state(uint64_t key) {
  S256 st{};
  uint64_t sm = key;
  bool any = false;
  for (int q = 0; q < 4; ++q) {
    sm += 0x9e3779b97f4a7c15ULL;
    uint64_t z = sm;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    st.s[q] = z ^ (z >> 31);
    any |= st.s[q] != 0;
  }
  if (!any) st.s[0] = 1;
  return st;
}

// T^(kChunk * 2^b), b = 0..kLevels-1 (host, ~20 ms; cached: it does not depend on the seed)
const std::vector<Mat>& jump_matrices() {
  static const std::vector<Mat> mats = [] {
    std::vector<Mat> out(kLevels);
    Mat a{}, b{};
    for (int j = 0; j < 256; ++j) {
      S256 e{};
      e.s[j >> 6] = uint64_t(1) << (j & 63);
      step(e);
      a.col[j] = e;
    }
    for (int i = 0; i < kChunkLog; ++i) {
      square(a, b);
      a = b;
    }
    out[0] = a;
    for (int l = 1; l < kLevels; ++l) square(out[l - 1], out[l]);
    return out;
  }();
  return mats;
}

// state before draw c * kChunk
__global__ void synth_states_kernel(const S256* __restrict__ mats, S256 s0, int64_t chunks, S256* __restrict__ states) {
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= chunks) return;
  S256 v = s0;
  for (int l = 0; l < kLevels; ++l) {
    if (!((c >> l) & 1)) continue;
    const S256* m = mats + size_t(l) * 256;
    S256 r{};
    for (int j = 0; j < 256; ++j) {
      const uint64_t mask = 0 - ((v.s[j >> 6] >> (j & 63)) & 1);
      const ulonglong2 lo = __ldg(reinterpret_cast<const ulonglong2*>(&m[j].s[0]));
      const ulonglong2 hi = __ldg(reinterpret_cast<const ulonglong2*>(&m[j].s[2]));
      r.s[0] ^= lo.x & mask;
      r.s[1] ^= lo.y & mask;
      r.s[2] ^= hi.x & mask;
      r.s[3] ^= hi.y & mask;
    }
    v = r;
  }
  states[c] = v;
}

struct SynthArgs {
  int64_t n;
  double ak, span, inv_k, w_min, w_max;  // x = ak + r * span
  double* out;
  int64_t* flag_idx;
  unsigned long long* flag_count;  // [0] flagged draws, [1] zero draws
  unsigned long long flag_cap;
};

constexpr int kSynthWarps = 4;

// One lane per chunk of kChunk draws; every 32 draws the warp transposes its
// 32x32 tile through shared memory so that each chunk's values leave as one
// 256-byte row.  Uncertified draws leave as their pow ARGUMENT and are listed.
__global__ void __launch_bounds__(kSynthWarps * 32)
synth_draws_kernel(const S256* __restrict__ states, SynthArgs a, clg::dd::ExpCoef cf) {
  __shared__ double tile[kSynthWarps][32][33];
  __shared__ uint32_t fmask[kSynthWarps][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t chunks = (a.n + kChunk - 1) >> kChunkLog;
  const int64_t c0 = (blockIdx.x * int64_t(kSynthWarps) + wid) * 32;  // first chunk of this warp
  if (c0 >= chunks) return;
  const int64_t c = c0 + lane;
  S256 st{};
  if (c < chunks) st = states[c];
  unsigned long long zeros = 0;
  for (int it = 0; it < kChunk / 32; ++it) {
    uint32_t mask = 0;
    const int64_t base = (c << kChunkLog) + it * 32;
#pragma unroll 1
    for (int t = 0; t < 32; ++t) {
      const uint64_t bits = rotl64(st.s[0] + st.s[3], 23) + st.s[0];  // rng.hpp:47-49
      step(st);
      const double r = static_cast<double>(bits >> 11) * 0x1.0p-53;  // open01, rng.hpp:65-69
      double w = 0.0;
      if (c < chunks && base + t < a.n) {
        if (r == 0.0) ++zeros;
        const double x = a.ak + r * a.span;  // no contraction: -fmad=false
        bool sure;
        w = clg::dd::pow_certified(x, a.inv_k, cf, &sure);
        if (sure) {
          w = w < a.w_min ? a.w_min : (a.w_max < w ? a.w_max : w);  // std::clamp
        } else {
          w = x;
          mask |= 1u << t;
        }
      }
      tile[wid][lane][t] = w;
    }
    fmask[wid][lane] = mask;
    __syncwarp();
    for (int row = 0; row < 32; ++row) {
      const int64_t cr = c0 + row;
      if (cr >= chunks) break;
      const int64_t idx = (cr << kChunkLog) + it * 32 + lane;
      const bool live = idx < a.n;
      if (live) a.out[idx] = tile[wid][row][lane];
      const bool fl = live && ((fmask[wid][row] >> lane) & 1);
      const unsigned ball = __ballot_sync(0xffffffffu, fl);
      if (ball) {
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(&a.flag_count[0], static_cast<unsigned long long>(__popc(ball)));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (fl) {
          const unsigned long long slot = at + __popc(ball & ((1u << lane) - 1));
          if (slot < a.flag_cap) a.flag_idx[slot] = idx;
        }
      }
    }
    __syncwarp();
  }
  if (zeros) atomicAdd(&a.flag_count[1], zeros);
}

__global__ void synth_gather_kernel(const double* __restrict__ w, const int64_t* __restrict__ idx, int64_t m,
                                    double* __restrict__ vals) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    vals[i] = w[idx[i]];
}

__global__ void synth_scatter_kernel(double* __restrict__ w, const int64_t* __restrict__ idx, int64_t m,
                                     const double* __restrict__ vals) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    w[idx[i]] = vals[i];
}

__global__ void synth_scale_kernel(double* __restrict__ w, int64_t n, double f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    w[i] = w[i] * f;
}

__global__ void synth_fill_kernel(double* __restrict__ w, int64_t n, double v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    w[i] = v;
}

__global__ void synth_iota_kernel(int64_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) v[i] = i;
}

struct Scratch {
  void* p = nullptr;
  ~Scratch() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 8); }
  template <class T>
  T* as() { return static_cast<T*>(p); }
};

int failf(int code, const char* fmt, const char* what, const char* detail) {
  char buf[384];
  snprintf(buf, sizeof buf, fmt, what, detail);
  return clgen_internal_fail(code, buf);
}

#define SYN_TRY(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) return failf(_e == cudaErrorMemoryAllocation ? CLGEN_ENOMEM : CLGEN_ECUDA, \
                                        "synth_powerlaw: %s failed: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

void host_pow(double* vals, int64_t m, double inv_k, double w_min, double w_max) {
  unsigned T = std::thread::hardware_concurrency();
  if (T == 0) T = 1;
  if (m < (1 << 16)) T = 1;
  const int64_t per = (m + T - 1) / T;
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < T; ++t) {
    const int64_t lo = t * per, hi = std::min<int64_t>(m, lo + per);
    if (lo >= hi) break;
    pool.emplace_back([=] {
      for (int64_t i = lo; i < hi; ++i) vals[i] = std::clamp(std::pow(vals[i], inv_k), w_min, w_max);  // weights.cpp:118-122
    });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" int clgen_dev_synth_powerlaw(clgen_dev_ctx* ctx, int64_t n, double gamma, double w_min, double w_max,
                                        uint64_t seed, int sort_desc, double target_mean, double* d_out,
                                        int64_t* n_host_resolved) {
  if (!ctx) return clgen_internal_fail(CLGEN_EINVAL, "null context");
  // the reference's contract (weights.cpp:105-108)
  if (n < 1) return clgen_internal_fail(CLGEN_EINVAL, "synth_powerlaw: n must be >= 1");
  if (!(gamma > 1.0)) return clgen_internal_fail(CLGEN_EINVAL, "synth_powerlaw: gamma must be > 1");
  if (!(w_min > 0.0)) return clgen_internal_fail(CLGEN_EINVAL, "synth_powerlaw: w_min must be > 0");
  if (w_min > w_max) return clgen_internal_fail(CLGEN_EINVAL, "synth_powerlaw: w_min > w_max");
  if (n >= (int64_t(1) << 32)) return clgen_internal_fail(CLGEN_EINVAL, "synth_powerlaw: n exceeds uint32 node ids (n < 2^32)");
  cudaPointerAttributes pa{};
  Scratch own;  // d_out == NULL: synthesise into scratch and install as the context's weights
  const bool install = d_out == nullptr;
  if (install) {
    pa.device = clgen_dev_device(ctx);
    SYN_TRY(cudaSetDevice(pa.device));
    SYN_TRY(own.alloc(sizeof(double) * n));
    d_out = own.as<double>();
  } else {
    if (cudaPointerGetAttributes(&pa, d_out) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      return clgen_internal_fail(CLGEN_EINVAL, "synth_powerlaw: output must be device memory");
    }
    SYN_TRY(cudaSetDevice(pa.device));
  }
  cudaStream_t stream = static_cast<cudaStream_t>(clgen_dev_stream(ctx));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pa.device);
  const int wide = sms * 8;
  int64_t resolved = 0;

  if (w_min == w_max) {  // weights.cpp:109-111: no draws consumed
    synth_fill_kernel<<<wide, 256, 0, stream>>>(d_out, n, w_min);
    SYN_TRY(cudaGetLastError());
  } else {
    const double k = 1.0 - gamma;
    const double ak = std::pow(w_min, k), bk = std::pow(w_max, k);
    const int64_t chunks = (n + kChunk - 1) >> kChunkLog;
    const auto& mats = jump_matrices();
    Scratch d_mats, d_states, d_idx, d_cnt, d_vals;
    SYN_TRY(d_mats.alloc(sizeof(Mat) * kLevels));
    SYN_TRY(d_states.alloc(sizeof(S256) * chunks));
    // ~2x the expected 1/16; weights beyond e^+-60 leave the certificate's range (ddpow.cuh): all may be listed
    const bool extreme = std::fabs(std::log(w_min)) > 60.0 || std::fabs(std::log(w_max)) > 60.0;
    const unsigned long long cap = static_cast<unsigned long long>((extreme ? n : n / 8) + 4096);
    SYN_TRY(d_idx.alloc(sizeof(int64_t) * cap));
    SYN_TRY(d_cnt.alloc(2 * sizeof(unsigned long long)));
    SYN_TRY(cudaMemcpyAsync(d_mats.p, mats.data(), sizeof(Mat) * kLevels, cudaMemcpyHostToDevice, stream));
    SYN_TRY(cudaMemsetAsync(d_cnt.p, 0, 2 * sizeof(unsigned long long), stream));
    const S256 s0 = seed_state(mix64_host(seed ^ kSynthTag));
    synth_states_kernel<<<static_cast<unsigned>((chunks + 127) / 128), 128, 0, stream>>>(d_mats.as<S256>(), s0, chunks,
                                                                                         d_states.as<S256>());
    SYN_TRY(cudaGetLastError());
    SynthArgs a{};
    a.n = n;
    a.ak = ak;
    a.span = bk - ak;
    a.inv_k = 1.0 / k;
    a.w_min = w_min;
    a.w_max = w_max;
    a.out = d_out;
    a.flag_idx = d_idx.as<int64_t>();
    a.flag_count = d_cnt.as<unsigned long long>();
    a.flag_cap = cap;
    const int64_t warps = (chunks + 31) / 32;
    synth_draws_kernel<<<static_cast<unsigned>((warps + kSynthWarps - 1) / kSynthWarps), kSynthWarps * 32, 0, stream>>>(
        d_states.as<S256>(), a, clg::dd::make_exp_coef());
    SYN_TRY(cudaGetLastError());
    unsigned long long cnt[2] = {0, 0};
    SYN_TRY(cudaMemcpyAsync(cnt, d_cnt.p, sizeof cnt, cudaMemcpyDeviceToHost, stream));
    SYN_TRY(cudaStreamSynchronize(stream));
    if (cnt[1] != 0)
      return clgen_internal_fail(CLGEN_ERANGE, "synth_powerlaw: a zero draw shifts the reference stream; use the host synthesiser for this seed");
    if (cnt[0] > cap) return clgen_internal_fail(CLGEN_ERANGE, "synth_powerlaw: more uncertified draws than the list holds");
    resolved = static_cast<int64_t>(cnt[0]);
    if (resolved > 0) {
      SYN_TRY(d_vals.alloc(sizeof(double) * resolved));
      synth_gather_kernel<<<wide, 256, 0, stream>>>(d_out, d_idx.as<int64_t>(), resolved, d_vals.as<double>());
      SYN_TRY(cudaGetLastError());
      std::vector<double> vals(static_cast<size_t>(resolved));
      SYN_TRY(cudaMemcpyAsync(vals.data(), d_vals.p, sizeof(double) * resolved, cudaMemcpyDeviceToHost, stream));
      SYN_TRY(cudaStreamSynchronize(stream));
      host_pow(vals.data(), resolved, a.inv_k, w_min, w_max);
      SYN_TRY(cudaMemcpyAsync(d_vals.p, vals.data(), sizeof(double) * resolved, cudaMemcpyHostToDevice, stream));
      synth_scatter_kernel<<<wide, 256, 0, stream>>>(d_out, d_idx.as<int64_t>(), resolved, d_vals.as<double>());
      SYN_TRY(cudaGetLastError());
      SYN_TRY(cudaStreamSynchronize(stream));
    }
  }

  if (sort_desc && w_min != w_max) {
    Scratch alt, tmp;
    SYN_TRY(alt.alloc(sizeof(double) * n));
    cub::DoubleBuffer<double> keys(d_out, alt.as<double>());
    size_t tmp_bytes = 0;
    SYN_TRY(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp_bytes, keys, n, 0, 64, stream));
    SYN_TRY(tmp.alloc(tmp_bytes));
    SYN_TRY(cub::DeviceRadixSort::SortKeysDescending(tmp.p, tmp_bytes, keys, n, 0, 64, stream));
    if (keys.Current() != d_out)
      SYN_TRY(cudaMemcpyAsync(d_out, keys.Current(), sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
    SYN_TRY(cudaStreamSynchronize(stream));
  }

  if (target_mean > 0.0) {
    double S = 0.0;
    const int rc = clgen_dev_blocked_sum_array(ctx, d_out, n, &S);
    if (rc) return rc;
    const double mean = S / static_cast<double>(n);
    synth_scale_kernel<<<wide, 256, 0, stream>>>(d_out, n, target_mean / mean);
    SYN_TRY(cudaGetLastError());
  }
  SYN_TRY(cudaStreamSynchronize(stream));
  if (n_host_resolved) *n_host_resolved = resolved;
  if (install) {
    const int rc = clgen_dev_set_weights(ctx, d_out, n);
    if (rc) return rc;
    SYN_TRY(cudaStreamSynchronize(stream));  // the scratch array is freed on return
  }
  return CLGEN_OK;
}

// make_weight_sequence(w, SortPolicy::sort_desc) (weights.cpp:32-55) on the
// device: a stable descending sort of the weights carrying each position's
// original label (LSD radix sort is stable, like the reference's
// std::stable_sort; a -0.0 sorts after +0.0 here, the reference leaves the two
// in input order).
extern "C" int clgen_dev_sort_desc(clgen_dev_ctx* ctx, double* d_w, int64_t n, int64_t* d_labels) {
  if (!ctx) return clgen_internal_fail(CLGEN_EINVAL, "null context");
  if (n < 0 || (n > 0 && !d_w)) return clgen_internal_fail(CLGEN_EINVAL, "sort_desc: bad argument");
  if (n == 0) return CLGEN_OK;
  cudaPointerAttributes pa{}, pl{};
  if (cudaPointerGetAttributes(&pa, d_w) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
      (d_labels && (cudaPointerGetAttributes(&pl, d_labels) != cudaSuccess || pl.type != cudaMemoryTypeDevice))) {
    cudaGetLastError();
    return clgen_internal_fail(CLGEN_EINVAL, "sort_desc: weights and labels must be device memory");
  }
  SYN_TRY(cudaSetDevice(pa.device));
  cudaStream_t stream = static_cast<cudaStream_t>(clgen_dev_stream(ctx));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pa.device);
  Scratch alt_w, alt_l, tmp;
  SYN_TRY(alt_w.alloc(sizeof(double) * n));
  cub::DoubleBuffer<double> keys(d_w, alt_w.as<double>());
  size_t tmp_bytes = 0;
  if (d_labels) {
    SYN_TRY(alt_l.alloc(sizeof(int64_t) * n));
    synth_iota_kernel<<<sms * 8, 256, 0, stream>>>(d_labels, n);
    SYN_TRY(cudaGetLastError());
    cub::DoubleBuffer<int64_t> vals(d_labels, alt_l.as<int64_t>());
    SYN_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, keys, vals, n, 0, 64, stream));
    SYN_TRY(tmp.alloc(tmp_bytes));
    SYN_TRY(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tmp_bytes, keys, vals, n, 0, 64, stream));
    if (vals.Current() != d_labels)
      SYN_TRY(cudaMemcpyAsync(d_labels, vals.Current(), sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, stream));
  } else {
    SYN_TRY(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp_bytes, keys, n, 0, 64, stream));
    SYN_TRY(tmp.alloc(tmp_bytes));
    SYN_TRY(cub::DeviceRadixSort::SortKeysDescending(tmp.p, tmp_bytes, keys, n, 0, 64, stream));
  }
  if (keys.Current() != d_w)
    SYN_TRY(cudaMemcpyAsync(d_w, keys.Current(), sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
  SYN_TRY(cudaStreamSynchronize(stream));
  return CLGEN_OK;
}
