// Bit-exact parallel replay of a SEQUENTIAL left-to-right FP64 fold
//     s_0 = s0,  s_{k+1} = fl(s_k + x_k),   x_k >= 0,
// which is how the reference accumulates the weight prefix sigma_u and the
// cumulative cost C_u inside each rank block (partition.cpp:115-116,
// cost.cpp:37-43; SPEC.md:97 makes that association part of the contract).
//
// Idea.  While the running sum stays inside one binade
// [2^e, 2^(e+1)) it is an integer multiple M of U = 2^(e-52).  Adding x means
// adding the integer K = floor(x/U) plus a rounding bit that depends only on
// the fraction of x/U (below / exactly half / above) and, for ties, on the
// parity of M + K (round half to even).  So each element is the map
//     M -> M + (M odd ? a1 : a0)
// and such maps are closed under composition — an associative operator that
// a parallel scan can use.  Steps that leave the binade (the sum reaches
// 2^(e+1)) are not of this form; they are replayed sequentially.
//
// Pipeline over tiles of kFoldTile elements:
//   A  approximate tile sums (any association)            fold_tile_sums_kernel
//   B  approximate tile starts -> each tile's binade, or   fold_approx_prefix_kernel
//      DIRTY when a crossing may fall inside it           + fold_tile_fun_kernel
//   C  composite map of each clean tile (ordered block scan)
//   D  one warp walks the tiles in order carrying the EXACT (e, M); a tile
//      whose binade or end check fails is folded element by element
//                                                          fold_spine_kernel
//   E  every clean tile re-derives its elements' exact prefixes from its exact
//      start and writes them (optionally transformed)     fold_emit_kernel
// Correctness never depends on the approximate phase: D verifies every tile.
#pragma once

#include "common.cuh"

namespace clg {

constexpr int kFoldThreads = 256;
constexpr int kFoldItems = 16;
constexpr int64_t kFoldTile = kFoldThreads * kFoldItems;
constexpr int kDirty = 0x7fffffff;
constexpr long long kFnSat = 1ll << 62;
constexpr long long kMaxM = (1ll << 53) - 1;

enum FoldOut : int {
  kFoldNone = 0,      // final value only
  kFoldInclusive = 1, // out[k] = s_{k+1}
  kFoldNodeCost = 2,  // out[k] = node_cost(x_k, s_k, S) (cost.cpp:8-13; s_k = sigma_u)
  kFoldSuffixCost = 3,  // out[src(k)] = (x_k / S) * s_k + 1 (cost.cpp:62-77 with a reversed fold)
};

struct Fn {
  long long a0, a1;  // M -> M + (M & 1 ? a1 : a0)
};

__device__ __forceinline__ long long sat_add(long long a, long long b) {
  const long long s = a + b;
  return s > kFnSat ? kFnSat : s;
}

// f first, then g
__device__ __forceinline__ Fn fn_compose(Fn f, Fn g) {
  Fn h;
  h.a0 = sat_add(f.a0, (f.a0 & 1) ? g.a1 : g.a0);
  h.a1 = sat_add(f.a1, ((1 + f.a1) & 1) ? g.a1 : g.a0);
  return h;
}

__device__ __forceinline__ long long fn_apply(Fn f, long long M) { return M + ((M & 1) ? f.a1 : f.a0); }

// Binade of a non-negative double: s = M * 2^(e-52); e = -1022 covers
// zero and subnormals (U = 2^-1074).
__device__ __forceinline__ void binade_of(double s, int& e, long long& M) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(s));
  const int ex = static_cast<int>((b >> 52) & 0x7ff);
  const unsigned long long man = b & ((1ull << 52) - 1);
  if (ex == 0) {
    e = -1022;
    M = static_cast<long long>(man);
  } else {
    e = ex - 1023;
    M = static_cast<long long>(man | (1ull << 52));
  }
}

__device__ __forceinline__ double from_binade(int e, long long M) {
  if (e == -1022 && M < (1ll << 52)) return __longlong_as_double(M);
  const unsigned long long b =
      (static_cast<unsigned long long>(e + 1023) << 52) | (static_cast<unsigned long long>(M) & ((1ull << 52) - 1));
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ int binade_e(double s) {
  int e;
  long long M;
  binade_of(s, e, M);
  return e;
}

// The map of adding x >= 0 to a running sum in binade e; `bad` is raised when
// x alone reaches 2^(e+1) (the step certainly leaves the binade).
__device__ __forceinline__ Fn elem_fn(double x, int e, bool& bad) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const int exr = static_cast<int>((b >> 52) & 0x7ff);
  unsigned long long mx = b & ((1ull << 52) - 1);
  int ex;
  if (exr == 0) {
    ex = -1074;
  } else {
    mx |= 1ull << 52;
    ex = exr - 1075;
  }
  Fn f{0, 0};
  if (mx == 0) return f;
  const int shift = ex - (e - 52);
  long long K;
  int cls = 0;  // 0 below half, 1 tie, 2 above half
  if (shift >= 0) {
    if (shift > 9) {
      bad = true;
      return Fn{kFnSat, kFnSat};
    }
    K = static_cast<long long>(mx << shift);
  } else {
    const int r = -shift;
    if (r >= 54) {
      K = 0;
    } else {
      K = static_cast<long long>(mx >> r);
      const unsigned long long rem = mx & ((1ull << r) - 1);
      const unsigned long long half = 1ull << (r - 1);
      cls = rem < half ? 0 : (rem == half ? 1 : 2);
    }
  }
  if (K > kMaxM) bad = true;
  const long long up0 = cls == 2 ? 1 : (cls == 1 ? (K & 1) : 0);
  const long long up1 = cls == 2 ? 1 : (cls == 1 ? ((1 + K) & 1) : 0);
  f.a0 = K + up0;
  f.a1 = K + up1;
  return f;
}

__device__ __forceinline__ double node_cost_dev(double w, double sigma, double S) {
  // cost.cpp:8-13, operation by operation (no contraction)
  double e = __dmul_rn(__ddiv_rn(w, S), __dsub_rn(__dsub_rn(S, sigma), w));
  if (e < 0.0) e = 0.0;
  return __dadd_rn(e, 1.0);
}

struct FoldArgs {
  const double* x;       // m inputs (>= 0)
  int64_t m;
  double s0;
  double* tsum;          // [T]
  double* approx;        // [T+1]
  Fn* tfun;              // [T]
  int* tbin;             // [T]
  double* start;         // [T] exact start of each tile
  unsigned char* slow;   // [T] replayed by the spine
  double* final_out;     // exact s_m
  int out_mode;
  double* out;           // [m] (may alias x for kFoldInclusive)
  const double* w;       // kFoldNodeCost: x are the weights, S below
  double S;
  int64_t stride;        // element k is x[src(k) * stride] (1: contiguous)
  int reverse;           // src(k) = reverse ? m - 1 - k : k
};

__device__ __forceinline__ int64_t fold_src(const FoldArgs& a, int64_t k) { return a.reverse ? a.m - 1 - k : k; }
__device__ __forceinline__ double fold_x(const FoldArgs& a, int64_t k) { return a.x[fold_src(a, k) * a.stride]; }
__device__ __forceinline__ void fold_put(const FoldArgs& a, int64_t k, double v) { a.out[fold_src(a, k)] = v; }

__device__ __forceinline__ double emit_value(const FoldArgs& a, double s_excl, double s_incl, double x) {
  if (a.out_mode == kFoldSuffixCost) return __dadd_rn(__dmul_rn(__ddiv_rn(x, a.S), s_excl), 1.0);
  return a.out_mode == kFoldNodeCost ? node_cost_dev(x, s_excl, a.S) : s_incl;
}

__global__ void __launch_bounds__(kFoldThreads) fold_tile_sums_kernel(FoldArgs a) {
  __shared__ double red[kFoldThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kFoldTile;
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < kFoldItems; ++i) {
    const int64_t k = base + i * kFoldThreads + threadIdx.x;
    if (k < a.m) acc += fold_x(a, k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(CLG_FULL, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kFoldThreads / 32; ++k) t += red[k];
    a.tsum[blockIdx.x] = t;
  }
}

// approx[t] = s0 + sum_{j<t} tsum[j] (any association), one CTA.
__global__ void __launch_bounds__(1024) fold_approx_prefix_kernel(FoldArgs a, int64_t T) {
  __shared__ double wsum[32];
  __shared__ double carry;
  if (threadIdx.x == 0) carry = a.s0;
  __syncthreads();
  for (int64_t base = 0; base < T; base += 1024) {
    const int64_t t = base + threadIdx.x;
    const double v = t < T ? a.tsum[t] : 0.0;
    double inc = v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(CLG_FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      double ws = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(CLG_FULL, ws, o);
        if (lane >= o) ws += y;
      }
      wsum[lane] = ws;
    }
    __syncthreads();
    const double before = (wid ? wsum[wid - 1] : 0.0) + inc - v;
    if (t < T) a.approx[t] = carry + before;
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.approx[T] = carry;
}

// Ordered block-inclusive scan of per-thread maps; returns the thread's
// EXCLUSIVE prefix and writes the block total to *total.
__device__ __forceinline__ Fn block_scan_fn(Fn mine, Fn* total) {
  __shared__ Fn wtot[kFoldThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Fn inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Fn y;
    y.a0 = __shfl_up_sync(CLG_FULL, inc.a0, o);
    y.a1 = __shfl_up_sync(CLG_FULL, inc.a1, o);
    if (lane >= o) inc = fn_compose(y, inc);
  }
  Fn exc;
  exc.a0 = __shfl_up_sync(CLG_FULL, inc.a0, 1);
  exc.a1 = __shfl_up_sync(CLG_FULL, inc.a1, 1);
  if (lane == 0) exc = Fn{0, 0};
  if (lane == 31) wtot[wid] = inc;
  __syncthreads();
  Fn wpre{0, 0};
  for (int k = 0; k < wid; ++k) wpre = fn_compose(wpre, wtot[k]);
  Fn tot{0, 0};
  for (int k = 0; k < kFoldThreads / 32; ++k) tot = fn_compose(tot, wtot[k]);
  *total = tot;
  __syncthreads();
  return fn_compose(wpre, exc);
}

// Phase B+C: classify each tile and build its composite map.
__global__ void __launch_bounds__(kFoldThreads) fold_tile_fun_kernel(FoldArgs a) {
  __shared__ int any_bad;
  const int64_t t = blockIdx.x;
  const double lo = a.approx[t], hi = a.approx[t + 1];
  const int e_lo = binade_e(lo - lo * 0x1p-20);
  const int e_hi = binade_e(hi + hi * 0x1p-20);
  if (e_lo != e_hi) {
    if (threadIdx.x == 0) a.tbin[t] = kDirty;
    return;
  }
  const int e = e_lo;
  if (threadIdx.x == 0) any_bad = 0;
  __syncthreads();
  const int64_t my0 = t * kFoldTile + static_cast<int64_t>(threadIdx.x) * kFoldItems;
  bool bad = false;
  Fn f{0, 0};
#pragma unroll
  for (int i = 0; i < kFoldItems; ++i) {
    const int64_t k = my0 + i;
    if (k < a.m) f = fn_compose(f, elem_fn(fold_x(a, k), e, bad));
  }
  if (bad) any_bad = 1;
  Fn tot;
  block_scan_fn(f, &tot);
  if (threadIdx.x == 0) {
    a.tbin[t] = any_bad ? kDirty : e;
    a.tfun[t] = tot;
  }
}

// Ordered warp-inclusive scan of per-lane maps; returns the lane's EXCLUSIVE
// prefix, *total = the composition of all 32.
__device__ __forceinline__ Fn warp_scan_fn(Fn mine, Fn* total) {
  const int lane = threadIdx.x & 31;
  Fn inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Fn y;
    y.a0 = __shfl_up_sync(CLG_FULL, inc.a0, o);
    y.a1 = __shfl_up_sync(CLG_FULL, inc.a1, o);
    if (lane >= o) inc = fn_compose(y, inc);
  }
  Fn exc;
  exc.a0 = __shfl_up_sync(CLG_FULL, inc.a0, 1);
  exc.a1 = __shfl_up_sync(CLG_FULL, inc.a1, 1);
  if (lane == 0) exc = Fn{0, 0};
  total->a0 = __shfl_sync(CLG_FULL, inc.a0, 31);
  total->a1 = __shfl_sync(CLG_FULL, inc.a1, 31);
  return exc;
}

// Phase D: one warp carries the exact running sum across the tiles, 32 tiles
// per step (lane l holds tile t0 + l's binade and composite map).  Every lane
// carries the same (s, e, M).
//  * A batch whose 32 tiles are all clean, all in the running sum's binade,
//    and whose composed map keeps M within the binade is taken in one warp
//    scan of the maps (x >= 0: M is monotone, so the end check covers every
//    intermediate value); each lane reads its tile's exact start off its
//    exclusive prefix.
//  * Otherwise the tiles are taken one by one; a tile that fails its check is
//    replayed, and the replay itself goes 32 elements at a time through the
//    same warp scan of element maps, element by element only for the chunk in
//    which the sum leaves its binade.
__global__ void __launch_bounds__(32) fold_spine_kernel(FoldArgs a, int64_t T) {
  const int lane = threadIdx.x;
  int e;
  long long M;
  double s = a.s0;
  binade_of(s, e, M);
  for (int64_t t0 = 0; t0 < T; t0 += 32) {
    const int64_t tt = t0 + lane;
    int et = kDirty;
    Fn f{0, 0};
    if (tt < T) {
      et = a.tbin[tt];
      f = a.tfun[tt];
    }
    const int cnt = T - t0 < 32 ? static_cast<int>(T - t0) : 32;
    if (cnt == 32 && __all_sync(CLG_FULL, et == e)) {
      Fn tot;
      const Fn pre = warp_scan_fn(f, &tot);
      const long long Mend = fn_apply(tot, M);
      if (Mend <= kMaxM) {
        a.start[tt] = from_binade(e, fn_apply(pre, M));
        a.slow[tt] = 0;
        M = Mend;
        s = from_binade(e, M);
        continue;
      }
    }
    double my_start = 0.0;
    int my_slow = 0;
    for (int j = 0; j < cnt; ++j) {
      const int etj = __shfl_sync(CLG_FULL, et, j);
      Fn fj;
      fj.a0 = __shfl_sync(CLG_FULL, f.a0, j);
      fj.a1 = __shfl_sync(CLG_FULL, f.a1, j);
      if (lane == j) my_start = s;
      bool fast = false;
      if (etj != kDirty && etj == e) {
        const long long M2 = fn_apply(fj, M);
        if (M2 <= kMaxM) {
          M = M2;
          s = from_binade(e, M);
          fast = true;
        }
      }
      if (lane == j) my_slow = fast ? 0 : 1;
      if (!fast) {
        // replay of the tile, 32 elements per chunk
        const int64_t b0 = (t0 + j) * kFoldTile;
        const int64_t b1 = b0 + kFoldTile < a.m ? b0 + kFoldTile : a.m;
        for (int64_t c = b0; c < b1; c += 32) {
          const int64_t k = c + lane;
          const double xk = k < b1 ? fold_x(a, k) : 0.0;
          const int n32 = b1 - c < 32 ? static_cast<int>(b1 - c) : 32;
          // the chunk as one scan of element maps, when it stays in the binade
          bool bad = false;
          const Fn fe = elem_fn(xk, e, bad);
          Fn tot;
          const Fn pre = warp_scan_fn(fe, &tot);
          const long long Mend = fn_apply(tot, M);
          if (!__any_sync(CLG_FULL, bad) && Mend <= kMaxM) {
            const long long Mb = fn_apply(pre, M);
            const double before = from_binade(e, Mb);
            const double after = from_binade(e, fn_apply(fe, Mb));
            if (a.out_mode != kFoldNone && k < b1) fold_put(a, k, emit_value(a, before, after, xk));
            M = Mend;
            s = from_binade(e, M);
            continue;
          }
          double myout = 0.0;
          for (int i = 0; i < n32; ++i) {
            const double xi = __shfl_sync(CLG_FULL, xk, i);
            const double before = s;
            s = __dadd_rn(s, xi);
            if (lane == i) myout = emit_value(a, before, s, xi);
          }
          if (a.out_mode != kFoldNone && k < b1) fold_put(a, k, myout);
          binade_of(s, e, M);
        }
      }
    }
    if (tt < T) {
      a.start[tt] = my_start;
      a.slow[tt] = my_slow;
    }
  }
  if (lane == 0) *a.final_out = s;
}

// Phase E: exact per-element prefixes of every tile the spine did not replay.
__global__ void __launch_bounds__(kFoldThreads) fold_emit_kernel(FoldArgs a) {
  const int64_t t = blockIdx.x;
  if (a.slow[t]) return;
  const int e = a.tbin[t];
  int e0;
  long long M0;
  binade_of(a.start[t], e0, M0);
  const int64_t my0 = t * kFoldTile + static_cast<int64_t>(threadIdx.x) * kFoldItems;
  double xs[kFoldItems];
  bool bad = false;
  Fn f{0, 0};
#pragma unroll
  for (int i = 0; i < kFoldItems; ++i) {
    const int64_t k = my0 + i;
    xs[i] = k < a.m ? fold_x(a, k) : 0.0;
    f = fn_compose(f, elem_fn(xs[i], e, bad));
  }
  Fn tot;
  const Fn pre = block_scan_fn(f, &tot);
  long long M = fn_apply(pre, M0);
#pragma unroll
  for (int i = 0; i < kFoldItems; ++i) {
    const int64_t k = my0 + i;
    if (k >= a.m) break;
    const double before = from_binade(e, M);
    M = fn_apply(elem_fn(xs[i], e, bad), M);
    fold_put(a, k, emit_value(a, before, from_binade(e, M), xs[i]));
  }
}

}  // namespace clg
