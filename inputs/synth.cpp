// libclgen_inputs.so - workload input preparation, shared by both bench arms.
// It is neither the product (libclgen_b200.so) nor the checker (oracle/): the
// reference's weight synthesisers, reproduced bit-for-bit so the GPU and the
// CPU reference consume identical FP64 arrays, parallelised for n = 1e9.
//
//   clgen_host_powerlaw_draws  weights.cpp:103-128 (before the descending sort)
//   clgen_host_discrete_powerlaw  C1 recipe: inverse CDF over
//       P(K=k) ∝ k^-gamma on integers [kmin,kmax], same synth stream
//
// The synth stream is one sequential xoshiro256++ sequence
// (RngStream(mix64(seed ^ 0x706c73796e7468)), weights.cpp:17,112), so draws
// are produced by one thread and the inverse CDF (glibc pow) is applied by
// all threads.  Compiled without -march: x86-64 SSE2 double arithmetic, no
// FMA, glibc libm — the same as the reference build.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "clgen_inputs.h"

namespace {

uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t key) {
    uint64_t sm = key;
    bool nonzero = false;
    for (auto& word : s) {
      sm += 0x9e3779b97f4a7c15ULL;
      uint64_t z = sm;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      word = z ^ (z >> 31);
      nonzero |= word != 0;
    }
    if (!nonzero) s[0] = 1;
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double open01() {
    for (;;) {
      const double r = static_cast<double>(next() >> 11) * 0x1.0p-53;
      if (r > 0.0) return r;
    }
  }
};

constexpr uint64_t kSynthTag = 0x706c73796e7468ULL;  // weights.cpp:17

template <class F>
void parallel_for(int64_t n, int threads, F&& f) {
  if (threads <= 1 || n < (1 << 16)) {
    f(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

int hw_threads(int requested) {
  if (requested > 0) return requested;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(h) : 1;
}

}  // namespace

extern "C" {

int clgen_host_powerlaw_draws(int64_t n, double gamma, double w_min, double w_max, uint64_t seed,
                              double* out, int threads) {
  if (n < 1 || !(gamma > 1.0) || !(w_min > 0.0) || w_min > w_max || !out) return -1;
  Xoshiro rng(mix64(seed ^ kSynthTag));
  if (w_min == w_max) {
    for (int64_t i = 0; i < n; ++i) out[i] = w_min;
    return 0;
  }
  for (int64_t i = 0; i < n; ++i) out[i] = rng.open01();  // the sequential stream
  const double k = 1.0 - gamma;
  const double ak = std::pow(w_min, k);
  const double bk = std::pow(w_max, k);
  const double inv_k = 1.0 / k;
  parallel_for(n, hw_threads(threads), [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      double w = std::pow(ak + out[i] * (bk - ak), inv_k);  // weights.cpp:118-122
      w = std::clamp(w, w_min, w_max);
      out[i] = w;
    }
  });
  return 0;
}

int clgen_host_discrete_powerlaw(int64_t n, double gamma, int64_t k_min, int64_t k_max,
                                 uint64_t seed, double* out, int threads) {
  if (n < 1 || !(gamma > 0.0) || k_min < 1 || k_min > k_max || !out) return -1;
  const int64_t m = k_max - k_min + 1;
  std::vector<double> cdf(static_cast<size_t>(m));
  double z = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    z += std::pow(static_cast<double>(k_min + i), -gamma);
    cdf[static_cast<size_t>(i)] = z;
  }
  for (auto& c : cdf) c /= z;
  cdf.back() = 1.0;
  Xoshiro rng(mix64(seed ^ kSynthTag));
  for (int64_t i = 0; i < n; ++i) out[i] = rng.open01();
  parallel_for(n, hw_threads(threads), [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      const auto it = std::lower_bound(cdf.begin(), cdf.end(), out[i]);  // min k: u <= F_k
      out[i] = static_cast<double>(k_min + (it - cdf.begin()));
    }
  });
  return 0;
}

int clgen_host_sort_desc(double* w, int64_t n, int threads) {
  if (n < 0 || (n > 0 && !w)) return -1;
  const int T = hw_threads(threads);
  if (T <= 1 || n < (1 << 20)) {
    std::sort(w, w + n, [](double a, double b) { return a > b; });
    return 0;
  }
  // sort T chunks in parallel, then merge pairwise in parallel rounds
  std::vector<int64_t> cuts;
  const int64_t chunk = (n + T - 1) / T;
  for (int64_t lo = 0; lo < n; lo += chunk) cuts.push_back(lo);
  cuts.push_back(n);
  {
    std::vector<std::thread> pool;
    for (size_t i = 0; i + 1 < cuts.size(); ++i)
      pool.emplace_back([=] { std::sort(w + cuts[i], w + cuts[i + 1], [](double a, double b) { return a > b; }); });
    for (auto& th : pool) th.join();
  }
  while (cuts.size() > 2) {
    std::vector<int64_t> next;
    std::vector<std::thread> pool;
    for (size_t i = 0; i + 1 < cuts.size(); i += 2) {
      next.push_back(cuts[i]);
      if (i + 2 < cuts.size()) {
        const int64_t a = cuts[i], b = cuts[i + 1], c = cuts[i + 2];
        pool.emplace_back([=] { std::inplace_merge(w + a, w + b, w + c, [](double x, double y) { return x > y; }); });
      }
    }
    next.push_back(n);
    for (auto& th : pool) th.join();
    cuts.swap(next);
  }
  return 0;
}

}  // extern "C"
