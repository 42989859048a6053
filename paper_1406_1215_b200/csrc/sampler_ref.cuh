// Reference-stream Chung–Lu sampler: one lane walks one source chain with the
// reference's own per-node xoshiro256++ stream, so every edge of an unflagged
// node is bit-identical to clgen::edges_from_source
// (/root/reference/proj/core/src/edge_skip.cpp:20-46).
//
// Work distribution: persistent warps; each warp refills idle lanes from a
// warp-local batch of source ids taken from a global queue in index order
// (heaviest sources first, since w is non-increasing — an LPT schedule).
#pragma once

#include "common.cuh"
#include "fastmath.cuh"

namespace clg {

// kWalkPairs (counter stream only): many seeds per launch, per-pair edge counts (statistical tests)
enum WalkMode : int { kWalkCount = 0, kWalkWrite = 1, kWalkFold = 2, kWalkPairs = 3 };

struct RefWalkArgs {
  const double* __restrict__ w;  // non-increasing weights, n entries
  const int32_t* run_len;        // optional run-length table (weights.cuh): w[v..v+run_len[v]) all equal
  int64_t n;
  double S;
  int64_t lo, hi;                // source slots [lo,hi)
  const int64_t* sources;        // optional: slot i walks source sources[i] (create_edges)
  uint64_t seed;
  unsigned long long* queue;     // next unclaimed source (starts at lo)
  // count mode
  int32_t* counts;               // counts[slot-lo]
  // write mode
  const int64_t* offsets;        // offsets[slot-lo]: first output position of the slot
  uint2* pairs;                  // (u,v) as uint32 pairs
  int64_t cap;
  // fold mode
  uint32_t* degree;              // tracked undirected degrees, degree[x >> track_shift]
  int track_shift;
  uint2* ring;                   // optional emission ring (power-of-two capacity)
  unsigned long long ring_mask;
  unsigned long long* ring_head;
  unsigned long long* fold_out;  // [0] edges, [1] checksum
  // guard
  unsigned long long* flag_count;
  int64_t* flagged;              // first flag_cap flagged source ids
  int64_t flag_cap;
  unsigned long long* overflow;  // write mode: slots beyond cap
  // single-pass write mode: slot i owns [offsets[i], offsets[i] + slot_cap[i]);
  // counts[i] receives its exact edge count and slots that did not fit are
  // appended to spill (re-walked later at their final offsets)
  const int32_t* slot_cap;
  int64_t* spill;
  unsigned long long* spill_count;
  WarpProf prof;                 // optional per-warp busy intervals
  // fast math (bit-exact with guarded fallbacks, fastmath.cuh)
  const LogTable* logtab;
  double invS;                   // RN(1/S)
  int refill_min;                // refill idle lanes only when at least this many are idle
  // heavy phase: slots [lo, *heavy_end) are walked one per WARP (every lane
  // runs the same chain, lane 0 emits): no divergence on the longest chains
  const int64_t* heavy_end;      // device scalar (ref_heavy_end_kernel); null: no heavy phase
  unsigned long long* hqueue;    // next unclaimed heavy slot, counted from lo
};

// Skip length exactly as edge_skip.cpp:9-16 computes it, with CUDA's libm.
// `amb` is raised when the ratio lies within 2^-47 (relative) of an integer
// >= 1: only there can glibc's log/log1p (<=1 ulp) and CUDA's (<=1 ulp)
// disagree on the floor.  The survey measured 0 such ratios in 3.9e7
// candidates.
__device__ __forceinline__ int64_t skip_length_ref(double p, double r, bool& amb) {
  const double ratio = __ddiv_rn(log(r), log1p(-p));
  if (!(ratio < 9.0e18)) return INT64_MAX;
  const double fl = floor(ratio);
  const double dlo = ratio - fl;
  const double dhi = (fl + 1.0) - ratio;
  const double tol = ratio * 0x1p-47;
  if ((dlo <= tol && fl >= 1.0) || dhi <= tol) amb = true;
  return static_cast<int64_t>(ratio);
}

// Skip length with the fast guarded ratio; the exact reference expression
// (and its glibc-vs-CUDA ambiguity flag) only inside a 2^-45 band around an
// integer, where the fast ratio (error <= ~2^-48) cannot certify the floor.
// ilp caches 1/log1p(-p) for the p it was computed for (lp_p): consecutive
// candidates with equal weights (C2: always; discrete weights: often) reuse it.
__device__ __forceinline__ int64_t skip_length_fast(double p, double r, bool& amb, const LogTable& T,
                                                    double& lp_p, double& ilp) {
  if (p != lp_p) {
    ilp = rcp_fast(log1m_fast(p, T));
    lp_p = p;
  }
  const double ratio = log_fast(r, T) * ilp;
  const double fl = floor(ratio);
  const double tol = ratio * 0x1p-45;
  if (ratio < 1.0e18 && !((ratio - fl <= tol && fl >= 1.0) || (fl + 1.0) - ratio <= tol))
    return static_cast<int64_t>(ratio);
  return skip_length_ref(p, r, amb);
}

// HEAVY: compiled with the heavy phase (launched only when the first slot's
// weight reaches the heavy threshold; 3 CTAs/SM); the lean variant keeps 64
// registers and 4 CTAs/SM for the gather-bound large runs.
template <int MODE, bool FAST, bool HEAVY>
__global__ void __launch_bounds__(256, HEAVY ? 3 : 4) ref_walk_kernel(RefWalkArgs a) {
  constexpr int64_t kBatch = 32;
  __shared__ LogTable s_tab;
  if (FAST) {
    for (int i = threadIdx.x; i < kLogTable; i += blockDim.x) {
      s_tab.inv_c[i] = a.logtab->inv_c[i];
      s_tab.nlog_inv[i] = a.logtab->nlog_inv[i];
    }
    __syncthreads();
  }
  const double invS = a.invS;
  const int lane = lane_id();
  const unsigned long long t_start = a.prof.slots ? globaltimer_ns() : 0ull;
  const double* __restrict__ w = a.w;
  const int64_t n = a.n;
  const double S = a.S;

  // warp-uniform batch state
  int64_t b_next = 0, b_end = 0;
  bool drained = false;
  // Heavy phase (warp-uniform): while slots remain below heavy_end the warp
  // takes ONE slot and all 32 lanes walk it in lockstep with identical state;
  // lane 0 alone emits.  The chain's latency per candidate is then the
  // dependent instruction chain itself, not 32 diverged chains sharing the
  // issue slot (C1: the ~1000-candidate chains of the heaviest sources were
  // the whole step's critical path).
  const int64_t heavy_end = HEAVY && a.heavy_end ? *a.heavy_end : a.lo;
  bool heavy_phase = HEAVY && heavy_end > a.lo;
  // per-warp ring reservation (fold mode)
  unsigned long long r_next = 0, r_end = 0;

  // lane state
  int64_t u = -1, slot = 0, j = 0, out_pos = 0, out_end = 0;
  int32_t cnt = 0;
  double p = 0.0, wu = 0.0, lp_p = -1.0, ilp = 0.0;
  int64_t run_end = 0;  // w is constant from the last gathered position up to run_end
  bool amb = false;
  Xoshiro rng;
  uint64_t checksum = 0;
  unsigned long long edges_total = 0;

  for (;;) {
    // ---------------------------------------------------------------- refill
    const unsigned need = __ballot_sync(CLG_FULL, u < 0);
    // start of slot `mine` on this lane (edge_skip.cpp:23-30)
    auto start_slot = [&](int64_t mine) {
      slot = mine - a.lo;
      u = a.sources ? a.sources[mine] : mine;
      j = u + 1;
      cnt = 0;
      amb = false;
      wu = w[u];
      if (MODE == kWalkWrite) {
        out_pos = a.offsets[slot];
        out_end = a.slot_cap ? out_pos + a.slot_cap[slot] : a.cap;
      }
      run_end = 0;
      if (j < n && S > 0.0) {
        rng.seed_key(node_rng_key(a.seed, u));
        const double wj = w[j];
        if (a.run_len) run_end = j + a.run_len[j];
        p = fmin(FAST ? div_S(__dmul_rn(wu, wj), S, invS) : __ddiv_rn(__dmul_rn(wu, wj), S), 1.0);
      } else {
        p = 0.0;
      }
    };
    if (HEAVY && heavy_phase) {
      if (need == CLG_FULL) {  // every lane finished the previous heavy slot together
        unsigned long long g = 0;
        if (lane == 0) g = atomicAdd(a.hqueue, 1ull);
        g = __shfl_sync(CLG_FULL, g, 0);
        const int64_t mine = a.lo + static_cast<int64_t>(g);
        if (mine >= heavy_end) {
          heavy_phase = false;
          continue;
        }
        start_slot(mine);
      }
    } else
    // refill when enough lanes are idle (a lone refill would stall the long
    // chains sharing the warp) or when the whole warp is idle
    if (need && !drained && (__popc(need) >= a.refill_min || need == CLG_FULL)) {
      const int want = __popc(need);
      const int r = __popc(need & lanemask_lt());
      const bool me = (need >> lane) & 1u;
      int64_t mine = -1;
      const int64_t take1 = clg::imin64(b_end - b_next, want);
      if (me && r < take1) mine = b_next + r;
      b_next += take1;
      if (want > take1) {
        unsigned long long g = 0;
        if (lane == 0) g = atomicAdd(a.queue, (unsigned long long)kBatch);
        g = __shfl_sync(CLG_FULL, g, 0);
        g += static_cast<unsigned long long>(heavy_end - a.lo);  // the light slots start at heavy_end
        if (static_cast<int64_t>(g) >= a.hi) {
          drained = true;
          b_next = b_end = a.hi;
        } else {
          b_next = static_cast<int64_t>(g);
          b_end = clg::imin64(b_next + kBatch, a.hi);
          const int64_t take2 = clg::imin64(b_end - b_next, want - take1);
          if (me && r >= take1 && r - take1 < take2) mine = b_next + (r - take1);
          b_next += take2;
        }
      }
      if (mine >= 0) start_slot(mine);
    }
    const unsigned live = __ballot_sync(CLG_FULL, u >= 0);
    if (!live) {
      if (drained) break;
      continue;
    }

    // ------------------------------------------------------------------ step
    bool accepted = false;
    int64_t v = 0;
    bool finish = false;
    if (u >= 0) {
      if (!(j < n && p > 0.0)) {
        finish = true;  // edge_skip.cpp:31 loop condition
      } else {
        int64_t delta = 0;
        if (p < 1.0)
          delta = FAST ? skip_length_fast(p, rng.open01(), amb, s_tab, lp_p, ilp) : skip_length_ref(p, rng.open01(), amb);
        if (delta >= n - j) {
          finish = true;  // edge_skip.cpp:34
        } else {
          v = j + delta;
          double q;
          const double r2 = rng.open01();
          if (v < run_end) {
            // same weight as the previous candidate: q = p and q/p = 1 > r2
            q = p;
            accepted = true;
          } else {
            const double wv = w[v];
            if (a.run_len) run_end = v + a.run_len[v];
            const double prod = __dmul_rn(wu, wv);
            q = fmin(FAST ? div_S(prod, S, invS) : __ddiv_rn(prod, S), 1.0);
            accepted = FAST ? accept_ref(r2, q, p) : r2 < __ddiv_rn(q, p);  // edge_skip.cpp:38
          }
          p = q;
          j = v + 1;
        }
      }
    }

    const bool lead = !HEAVY || !heavy_phase || lane == 0;  // heavy phase: 32 identical chains, one emitter
    accepted = accepted && lead;
    if (accepted) {
      ++cnt;
      if (MODE == kWalkWrite) {
        if (out_pos < out_end) {
          a.pairs[out_pos] = make_uint2(static_cast<uint32_t>(u), static_cast<uint32_t>(v));
        } else if (!a.slot_cap) {
          atomicAdd(a.overflow, 1ull);
        }
        ++out_pos;
      } else if (MODE == kWalkFold) {
        checksum += edge_hash(static_cast<uint32_t>(u), static_cast<uint32_t>(v));
        ++edges_total;
        if (a.degree && (v & ((1ll << a.track_shift) - 1)) == 0) atomicAdd(&a.degree[v >> a.track_shift], 1u);
      }
    }
    if (MODE == kWalkFold && a.ring) {
      const unsigned am = __ballot_sync(CLG_FULL, accepted);
      if (am) {
        const unsigned k = __popc(am);
        const unsigned rk = __popc(am & lanemask_lt());
        const unsigned long long rem = r_end - r_next;
        unsigned long long nb = 0;
        if (rem < k) {
          if (lane == 0) nb = atomicAdd(a.ring_head, 2048ull);
          nb = __shfl_sync(CLG_FULL, nb, 0);
        }
        if (accepted) {
          const unsigned long long pos = rk < rem ? r_next + rk : nb + (rk - rem);
          a.ring[pos & a.ring_mask] = make_uint2(static_cast<uint32_t>(u), static_cast<uint32_t>(v));
        }
        if (rem < k) {
          r_next = nb + (k - rem);
          r_end = nb + 2048ull;
        } else {
          r_next += k;
        }
      }
    }
    if (u >= 0 && (finish || !(j < n && p > 0.0))) {
      if (lead) {
        if (MODE == kWalkCount) a.counts[slot] = cnt;
        if (MODE == kWalkWrite && a.slot_cap) {
          a.counts[slot] = cnt;
          if (out_pos > out_end) a.spill[atomicAdd(a.spill_count, 1ull)] = slot;
        }
        if (MODE == kWalkFold && a.degree && (u & ((1ll << a.track_shift) - 1)) == 0 && cnt)
          atomicAdd(&a.degree[u >> a.track_shift], static_cast<uint32_t>(cnt));
        if (amb) {
          const unsigned long long idx = atomicAdd(a.flag_count, 1ull);
          if (static_cast<int64_t>(idx) < a.flag_cap) a.flagged[idx] = u;
        }
      }
      u = -1;
    }
  }

  if (a.prof.slots && lane == 0) {
    const int g = a.prof.gw();
    a.prof.slots[2 * g] = t_start;
    a.prof.slots[2 * g + 1] = globaltimer_ns();
  }
  if (MODE == kWalkFold) {
    checksum = warp_sum_u64(checksum);
    edges_total = warp_sum_u64(edges_total);
    if (lane == 0) {
      atomicAdd(&a.fold_out[0], edges_total);
      atomicAdd(&a.fold_out[1], static_cast<unsigned long long>(checksum));
    }
  }
}

// First slot of [lo, hi) whose weight is below tw (w non-increasing), at most
// lo + cap: the heavy phase of ref_walk_kernel covers [lo, that).
__global__ void ref_heavy_end_kernel(const double* __restrict__ w, int64_t lo, int64_t hi, double tw, int64_t cap,
                                     int64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t a = lo - 1, b = hi;  // w[a] >= tw (or a = lo - 1), w[b] < tw (or b = hi)
  while (b - a > 1) {
    const int64_t m = a + ((b - a) >> 1);
    if (w[m] >= tw) a = m; else b = m;
  }
  *out = b < lo + cap ? b : lo + cap;
}

// Per-slot capacity of the single-pass write: the unclamped expected forward
// degree w_u (S - w_u) / S >= sum_{v>u} min(w_u w_v / S, 1) (sigma_u dropped,
// so it also bounds every source of a create_edges list) plus k_sigma sigma +
// k_const (6 and 8 by default).
__global__ void ref_slot_cap_kernel(const double* __restrict__ w, int64_t n, double S, const int64_t* sources,
                                    int64_t lo, int64_t m, double k_sigma, double k_const,
                                    int32_t* __restrict__ cap) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int64_t u = sources ? sources[lo + i] : lo + i;
    const double wu = w[u];
    const double e = S > 0.0 ? fmax(wu * (S - wu) / S, 0.0) : 0.0;
    double c = ceil(e + k_sigma * sqrt(e) + k_const);
    const double rest = static_cast<double>(n - 1 - u);
    c = fmin(c, rest);
    c = fmin(c, 1.0e9);
    cap[i] = static_cast<int32_t>(c > 0.0 ? c : 0.0);
  }
}

// Moves each fitted slot's edges from its scratch run to its final offset.
// One warp per slot; spilled slots (count > cap) are left to the re-walk.
__global__ void ref_compact_kernel(const uint2* __restrict__ scratch, const int64_t* __restrict__ soff,
                                   const int32_t* __restrict__ cap, const int32_t* __restrict__ counts,
                                   const int64_t* __restrict__ foff, int64_t m, uint2* __restrict__ out,
                                   int64_t out_cap) {
  const int lane = lane_id();
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5 << 5; base < m;
       base += warps * 32) {
    // lane l loads the metadata of slot base + l; the warp then copies slot by slot
    const int64_t mine = base + lane;
    int32_t c = 0, k = 0;
    int64_t s = 0, f = 0;
    if (mine < m) {
      c = counts[mine];
      k = cap[mine];
      s = soff[mine];
      f = foff[mine];
    }
    if (c > k) c = 0;
    for (int l = 0; l < 32; ++l) {
      const int32_t cl = __shfl_sync(CLG_FULL, c, l);
      if (cl == 0) continue;
      const int64_t sl = __shfl_sync(CLG_FULL, s, l);
      const int64_t fl = __shfl_sync(CLG_FULL, f, l);
      for (int32_t x = lane; x < cl; x += 32)
        if (fl + x < out_cap) out[fl + x] = scratch[sl + x];
    }
  }
}

// Spilled slots -> (source, final offset) lists for the re-walk.
__global__ void ref_spill_lists_kernel(const int64_t* __restrict__ spill, const unsigned long long* spill_count,
                                       const int64_t* sources, int64_t lo, const int64_t* __restrict__ foff,
                                       int64_t* __restrict__ src_out, int64_t* __restrict__ off_out) {
  const int64_t k = static_cast<int64_t>(*spill_count);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t slot = spill[i];
    src_out[i] = sources ? sources[lo + slot] : lo + slot;
    off_out[i] = foff[slot];
  }
}

}  // namespace clg
