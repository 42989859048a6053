// Single-pass decoupled-lookback exclusive prefix scan (int32 -> int64).
//
// Tiles of kScanThreads*kScanItems elements are claimed in launch order through
// an atomic ticket, so a tile only ever waits on tiles that are already
// running (forward progress without co-residency assumptions).  Each tile
// publishes its aggregate (flag 1) and, once its predecessor's inclusive
// prefix is known, its inclusive prefix (flag 2).  The value and the flag are
// packed into one 64-bit word (flag in the top 2 bits, value < 2^62), so a
// single relaxed-volatile load observes both consistently.
#pragma once

#include "common.cuh"

namespace clg {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int64_t kScanTile = kScanThreads * kScanItems;

constexpr uint64_t kTileAgg = 1ull << 62;
constexpr uint64_t kTileIncl = 2ull << 62;
constexpr uint64_t kTileValMask = (1ull << 62) - 1;

template <typename InT>
__global__ void __launch_bounds__(kScanThreads) scan_lookback_kernel(
    const InT* __restrict__ in, int64_t* __restrict__ out, int64_t n,
    unsigned long long* tile_state, unsigned long long* ticket, int64_t* total, int64_t init) {
  __shared__ int64_t warp_tot[kScanThreads / 32];
  __shared__ int64_t s_prefix;
  __shared__ unsigned long long s_tile;

  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1ull);
  __syncthreads();
  const int64_t tile = static_cast<int64_t>(s_tile);
  const int64_t base = tile * kScanTile;

  // blocked arrangement: thread t owns items [base + t*I, base + t*I + I)
  int64_t v[kScanItems];
  int64_t run = 0;
  const int64_t my0 = base + static_cast<int64_t>(threadIdx.x) * kScanItems;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = my0 + i;
    const int64_t x = idx < n ? static_cast<int64_t>(in[idx]) : 0;
    v[i] = run;
    run += x;
  }
  // block exclusive scan of per-thread totals
  const int lane = lane_id(), wid = threadIdx.x >> 5;
  const int64_t incl = warp_inclusive_scan(run);
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  int64_t wpre = 0, agg = 0;
#pragma unroll
  for (int k = 0; k < kScanThreads / 32; ++k) {
    const int64_t t = warp_tot[k];
    if (k < wid) wpre += t;
    agg += t;
  }
  const int64_t thread_excl = wpre + incl - run;

  // look-back (thread 0)
  if (threadIdx.x == 0) {
    volatile unsigned long long* st = tile_state;
    int64_t prefix = init;
    if (tile == 0) {
      st[0] = kTileIncl | static_cast<uint64_t>(init + agg);
    } else {
      st[tile] = kTileAgg | static_cast<uint64_t>(agg);
      int64_t exclusive = 0;
      int64_t t = tile - 1;
      for (;;) {
        unsigned long long s;
        do {
          s = st[t];
        } while ((s >> 62) == 0);
        exclusive += static_cast<int64_t>(s & kTileValMask);
        if ((s >> 62) == 2) break;
        --t;
      }
      prefix = exclusive;
      __threadfence();
      st[tile] = kTileIncl | static_cast<uint64_t>(exclusive + agg);
    }
    s_prefix = prefix;
    const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
    if (tile == ntiles - 1 && total) *total = prefix + agg;
  }
  __syncthreads();
  const int64_t off = s_prefix + thread_excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = my0 + i;
    if (idx < n) out[idx] = off + v[i];
  }
}

}  // namespace clg
