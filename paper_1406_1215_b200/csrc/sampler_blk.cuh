// Counter-stream Chung–Lu sampler over weight-class pair blocks.
//
// Law: every pair (u, v>u) is an edge independently with probability
// p_uv = min(w_u w_v / S, 1) — the law of edges_from_source
// (edge_skip.cpp:20-46, p and q at :30,:36, acceptance r < q/p at :38).  The
// random stream is the north star's counter-keyed one, not the reference's
// per-node xoshiro256++: statistically exact, deterministic per seed, and
// independent of the GPU count, the source partition and the launch shape.
//
// Construction (Miller–Hagberg skipping with a constant envelope per block):
//  * the sorted weights are cut into classes [s_k, s_{k+1}) on a geometric
//    grid, w[s_k] <= (1+eps) w[s_{k+1}-1] (<= 2^26 nodes per class, so every
//    block below has fewer than 2^52 positions: exact doubles);
//  * block (A,B), A <= B, holds the pairs u in A, v in B (A = B: u < v).  Its
//    envelope pbar = w[s_A] w[s_B] / S (the generators' FP64 expression on the
//    class maxima) bounds every p_uv inside it, since FP products and
//    quotients are monotone;
//  * sparse blocks (pbar < 1): candidates are a Bernoulli(pbar) process over
//    the block's row-major positions — i.i.d. geometric gaps
//    floor(E / -log1p(-pbar)) + 1, E ~ Exp(1) — each thinned with probability
//    p_uv / pbar.  The class bounds give p_uv / pbar >= hs / 2^11 for the
//    block's sure threshold hs, so ~98.5% of candidates are accepted from 11
//    random bits without reading w; the rest gather w_u, w_v (queued per warp
//    in shared memory, 32 at a time);
//  * dense blocks (pbar >= 1, only pairs with p_uv >= ~0.98): every position
//    is a candidate accepted with probability p_uv;
//  * blocks are cut into chunks of about `chunk_cand` expected candidates
//    (a function of the weights only); a chunk restarts the geometric process
//    (memoryless) from its own keyed streams, one xoroshiro128++ per
//    (chunk, lane).  A launch over sources [lo, hi) claims every chunk whose
//    rows meet [lo, hi) and emits only those rows, so any cover of the
//    sources yields the same graph.
// Per round a warp draws 32 x E gaps (E per lane), places them with one warp
// prefix sum, decodes (row, col) = (position / nb, position % nb) in exact
// double arithmetic, and emits accepted pairs through a per-warp shared-memory
// stage flushed as 16-byte vector stores (ring / fold mode) — the level-2
// balance is the uniform chunk size: a hub's v-range is spread over as many
// blocks and chunks as its expected edge count needs.
#pragma once

#include "common.cuh"
#include "fastmath.cuh"
#include "sampler_ref.cuh"

namespace clg {

constexpr int kClassCap = 1024;                 // classes (incl. the zero class)
constexpr int64_t kClassMaxNodes = 1ll << 26;   // nodes per class (block positions < 2^52)
constexpr uint32_t kBlkDiag = 1u, kBlkDense = 2u;

struct __align__(16) BlockDesc {
  double pbar;      // RN(RN(w[s_A] w[s_B]) / S): envelope (>= every p_uv of the block)
  double inv_mu;    // 1 / -log1p(-pbar) (sparse blocks)
  double inv_nb;    // RN(1 / nb)
  int64_t L;        // chunk length in positions
  int64_t nchunks;  // chunks covering [0, na * nb)
  uint32_t a0, na, b0, nb;
  uint32_t hs;      // sure-accept threshold on the 11 acceptance bits
  uint32_t flags;   // kBlkDiag | kBlkDense
};

// Per-launch view of a block: the first chunk meeting the launch's source
// range and the emission window [x_lo, x_hi) of row-major positions.
struct BlockRange {
  int64_t c_lo, x_lo, x_hi;
};

struct BlkArgs {
  const double* __restrict__ w;
  double S;
  const BlockDesc* __restrict__ blocks;
  const BlockRange* __restrict__ ranges;
  const int64_t* __restrict__ chunk_prefix;  // per block: first launch chunk id
  const uint32_t* __restrict__ chunk_block;  // launch chunk id -> block
  const int64_t* total_chunks;               // device scalar (written by the scan)
  unsigned long long* queue;
  uint64_t seed_mix;
  const LogTable* logtab;
  // outputs
  int32_t* counts;          // per launch chunk (count mode)
  const int64_t* offsets;   // per launch chunk (write mode)
  uint2* pairs;
  int64_t cap;
  uint32_t* degree;
  int track_shift;
  uint2* ring;
  unsigned long long ring_mask;
  unsigned long long* fold_out;
  unsigned long long* overflow;
  WarpProf prof;
};

// Exp(1) by inversion from the top 53 bits of x: E = -log(U),
// U = (x>>11 + 1/2) 2^-53 in (0,1); 128-entry table log + degree-5 log1p,
// absolute error < 2^-50 (statistically exact).
__device__ __forceinline__ double exp_bits(uint64_t x, const LogTable& T) {
  const double u = __dmul_rn(static_cast<double>(x >> 11) + 0.5, 0x1.0p-53);
  const long long bx = __double_as_longlong(u);
  const int ex = static_cast<int>((bx >> 52) & 0x7ff) - 1023;
  const int ti = static_cast<int>((bx >> 45) & (kLogTable - 1));
  const double m = __longlong_as_double((bx & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double t = __fma_rn(m, T.inv_c[ti], -1.0);
  double sp = __fma_rn(t, 1.0 / 5.0, -1.0 / 4.0);
  sp = __fma_rn(t, sp, 1.0 / 3.0);
  sp = __fma_rn(t, sp, -0.5);
  sp = __fma_rn(t, sp, 1.0);
  const double e = static_cast<double>(ex);
  return -__fma_rn(e, 0x1.62e42fefa39efp-1, T.nlog_inv[ti] + __fma_rn(e, 0x1.abc9e3b39803fp-56, t * sp));
}

__device__ __forceinline__ double unit53(uint64_t b) {  // [0,1)
  return static_cast<double>(b >> 11) * 0x1.0p-53;
}

// Bernoulli(a) from a lazily refined uniform R = (h + R')/2048: the 11 bits h
// come with the candidate's gap draw (its low bits, independent of the gap),
// R' (53 bits) is hashed from the candidate's identity only when h alone
// cannot decide, so the decision does not depend on when it is taken.
__device__ __forceinline__ bool lazy_accept(uint32_t h, double a, uint64_t key, uint32_t id) {
  const double s = a * 2048.0;  // exact scaling
  if (static_cast<double>(h + 1u) <= s) return true;
  if (static_cast<double>(h) >= s) return false;
  const uint64_t r = mix64((key ^ 0xd6e8feb86659fd93ULL) + 0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(id) + 1ull));
  return unit53(r) < s - static_cast<double>(h);  // s - h exact (Sterbenz)
}

__device__ __forceinline__ double warp_incl_scan_f64(double x) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(CLG_FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ uint32_t warp_excl_scan_u32(uint32_t x, uint32_t& total) {
  const int lane = lane_id();
  uint32_t s = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(CLG_FULL, s, o);
    if (lane >= o) s += y;
  }
  total = __shfl_sync(CLG_FULL, s, 31);
  return s - x;
}

// (row, col) of row-major position x (exact integer double < 2^52) in a
// block of nb columns: quotient from RN(1/nb), corrected by the exact residual.
__device__ __forceinline__ void decode_pos(double x, double inv_nb, double nb_d, int32_t nb, uint32_t& row,
                                           uint32_t& col) {
  uint32_t r = __double2uint_rz(x * inv_nb);
  int32_t c = __double2int_rz(__fma_rn(-static_cast<double>(r), nb_d, x));
  if (c < 0) {
    c += nb;
    --r;
  } else if (c >= nb) {
    c -= nb;
    ++r;
  }
  row = r;
  col = static_cast<uint32_t>(c);
}

constexpr int kStageCap = 256;  // staged pairs per warp (ring / write modes)
constexpr int kUncCap = 64;     // queued uncertain candidates per warp

__host__ __device__ inline size_t blk_smem_bytes(int threads) {
  return sizeof(LogTable) + static_cast<size_t>(threads / 32) * (kStageCap * sizeof(uint2) + kUncCap * 16);
}

template <int MODE, int E, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) blk_kernel(BlkArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LogTable& s_log = *reinterpret_cast<LogTable*>(smem_raw);
  const int wib = threadIdx.x >> 5;
  uint2* stage = reinterpret_cast<uint2*>(smem_raw + sizeof(LogTable)) + wib * kStageCap;
  uint32_t* qbase = reinterpret_cast<uint32_t*>(smem_raw + sizeof(LogTable) +
                                                (THREADS / 32) * kStageCap * sizeof(uint2)) + wib * 4 * kUncCap;
  uint32_t* qu = qbase;
  uint32_t* qv = qbase + kUncCap;
  uint32_t* qh = qbase + 2 * kUncCap;
  uint32_t* qi = qbase + 3 * kUncCap;
  for (int i = threadIdx.x; i < kLogTable; i += THREADS) {
    s_log.inv_c[i] = a.logtab->inv_c[i];
    s_log.nlog_inv[i] = a.logtab->nlog_inv[i];
  }
  __syncthreads();

  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  const unsigned long long t_start = a.prof.slots ? globaltimer_ns() : 0ull;
  const double* __restrict__ w = a.w;
  const double S = a.S;
  const int64_t total = *a.total_chunks;
  const uint32_t tmask = (1u << a.track_shift) - 1u;
  const bool track = a.degree != nullptr;

  // fold-mode ring: a private circular segment per warp (no reservation atomics)
  uint2* seg = nullptr;
  uint32_t smask = 0, wpos = 0;
  if (MODE == kWalkFold && a.ring) {
    const unsigned nw = gridDim.x * (THREADS >> 5);
    const unsigned gw = blockIdx.x * (THREADS >> 5) + wib;
    const int lcap = 63 - __clzll(static_cast<long long>(a.ring_mask + 1ull));
    const int lnw = nw > 1 ? 32 - __clz(nw - 1) : 0;
    int sl = lcap - lnw;
    sl = sl < 6 ? 6 : (sl > 20 ? 20 : sl);
    if (sl > lcap) sl = lcap;
    smask = (1u << sl) - 1u;
    seg = a.ring + ((static_cast<unsigned long long>(gw) << sl) & a.ring_mask);
  }
  const bool staging = (MODE == kWalkFold && seg != nullptr) || MODE == kWalkWrite;
  uint32_t head = 0, tail = 0;  // stage counters (warp-uniform)
  uint64_t checksum = 0;
  uint32_t edges = 0;           // fold: per lane; count: per lane within the chunk
  int64_t out_pos = 0;          // write mode
  Xoro128 rng;

  // flush 64 staged pairs as one 512-byte burst (ring: 16-byte vectors)
  auto flush64 = [&]() {
    __syncwarp();
    if (MODE == kWalkFold) {
      const uint4 v2 = *reinterpret_cast<const uint4*>(&stage[(tail + 2 * lane) & (kStageCap - 1)]);
      *reinterpret_cast<uint4*>(&seg[(wpos + 2 * lane) & smask]) = v2;
      wpos += 64;
    } else {
      for (int i = lane; i < 64; i += 32) {
        const int64_t p = out_pos + i;
        if (p < a.cap) a.pairs[p] = stage[(tail + i) & (kStageCap - 1)];
        else atomicAdd(a.overflow, 1ull);
      }
      out_pos += 64;
    }
    tail += 64;
    __syncwarp();
  };
  auto flush_rest = [&]() {  // < 64 left
    __syncwarp();
    const uint32_t rem = head - tail;
    for (uint32_t i = lane; i < rem; i += 32) {
      const uint2 e = stage[(tail + i) & (kStageCap - 1)];
      if (MODE == kWalkFold) {
        seg[(wpos + i) & smask] = e;
      } else {
        const int64_t p = out_pos + i;
        if (p < a.cap) a.pairs[p] = e;
        else atomicAdd(a.overflow, 1ull);
      }
    }
    if (MODE == kWalkFold) wpos += rem;
    else out_pos += rem;
    tail = head;
    __syncwarp();
  };
  // emission of up to N pairs per lane (lane-major)
  auto fold_one = [&](uint32_t u, uint32_t v) {
    checksum += mix64((static_cast<uint64_t>(u) << 32) | v);
    if (track) {
      if ((u & tmask) == 0) atomicAdd(&a.degree[u >> a.track_shift], 1u);
      if ((v & tmask) == 0) atomicAdd(&a.degree[v >> a.track_shift], 1u);
    }
  };

  for (;;) {
    unsigned long long qq = 0;
    if (lane == 0) qq = atomicAdd(a.queue, 1ull);
    const int64_t q = static_cast<int64_t>(__shfl_sync(CLG_FULL, qq, 0));
    if (q >= total) break;
    const uint32_t b = __ldg(a.chunk_block + q);
    const BlockDesc d = a.blocks[b];
    const BlockRange r = a.ranges[b];
    const int64_t c = r.c_lo + (q - __ldg(a.chunk_prefix + b));
    const int64_t N = static_cast<int64_t>(d.na) * d.nb;
    const int64_t x0 = c * d.L;
    const int64_t x1 = imin64(x0 + d.L, N);
    const double xend = static_cast<double>(x1);
    const double wlo = static_cast<double>(imax64(x0, r.x_lo));
    const double whi = static_cast<double>(imin64(x1, r.x_hi));
    const uint64_t key = mix64(a.seed_mix ^ (static_cast<uint64_t>(b) | (static_cast<uint64_t>(c) << 20)));
    rng.seed_key(key + 0x632be59bd9b4e019ULL * static_cast<uint64_t>(lane + 1));
    const bool diag = (d.flags & kBlkDiag) != 0;
    const double nb_d = static_cast<double>(d.nb);
    const int32_t nbi = static_cast<int32_t>(d.nb);
    uint32_t qn = 0, qt = 0;  // uncertain queue counters (warp-uniform)
    if (MODE == kWalkWrite) out_pos = a.offsets[q];
    if (MODE == kWalkCount) edges = 0;

    auto emit = [&](const bool* acc, const uint32_t* uu, const uint32_t* vv, int n) {
      uint32_t cnt = 0;
      for (int e = 0; e < n; ++e) cnt += acc[e] ? 1u : 0u;
      if (MODE == kWalkCount) {
        edges += cnt;
        return;
      }
      if (MODE == kWalkFold) {
        edges += cnt;
        for (int e = 0; e < n; ++e)
          if (acc[e]) fold_one(uu[e], vv[e]);
      }
      if (!staging) return;
      uint32_t tot;
      uint32_t pos = head + warp_excl_scan_u32(cnt, tot);
      for (int e = 0; e < n; ++e)
        if (acc[e]) stage[(pos++) & (kStageCap - 1)] = make_uint2(uu[e], vv[e]);
      head += tot;
      while (head - tail >= 64) flush64();
    };
    // decide the queued uncertain candidates (k <= 32): gather w_u, w_v
    auto resolve = [&](uint32_t k) {
      __syncwarp();
      bool acc = false;
      uint32_t u = 0, v = 0;
      if (static_cast<uint32_t>(lane) < k) {
        const uint32_t i = (qt + lane) & (kUncCap - 1);
        u = qu[i];
        v = qv[i];
        const double wu = w[u], wv = w[v];
        const double qv_ = __ddiv_rn(__dmul_rn(wu, wv), S);  // edge_skip.cpp:36
        const double p = qv_ < 1.0 ? qv_ : 1.0;
        acc = lazy_accept(qh[i], __ddiv_rn(p, d.pbar), key, qi[i]);
      }
      qt += k;
      __syncwarp();
      emit(&acc, &u, &v, 1);
    };

    if (!(d.flags & kBlkDense)) {
      // ---- sparse block: geometric gaps, E per lane per round ----
      const double inv_mu = d.inv_mu, inv_nb = d.inv_nb;
      const uint32_t hs = d.hs;
      double base = static_cast<double>(x0);  // next candidate is at >= base
      for (uint32_t rid = 0;; ++rid) {
        double pos[E];
        uint32_t hh[E];
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t x = rng.next();
          const double g = fmin(floor(exp_bits(x, s_log) * inv_mu), 0x1.0p52);
          s += g + 1.0;
          pos[e] = s;
          hh[e] = static_cast<uint32_t>(x) & 2047u;
        }
        const double incl = warp_incl_scan_f64(s);
        const double lb = base + (incl - s) - 1.0;
        const double last = __shfl_sync(CLG_FULL, lb + s, 31);
        bool sure[E];
        uint32_t uu[E], vv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double x = lb + pos[e];
          uint32_t row, col;
          decode_pos(x, inv_nb, nb_d, nbi, row, col);
          const bool ok = x < whi && x >= wlo && (!diag || col > row);
          uu[e] = d.a0 + row;
          vv[e] = d.b0 + col;
          sure[e] = ok && hh[e] < hs;
          const bool unc = ok && !sure[e];
          const unsigned m = __ballot_sync(CLG_FULL, unc);
          if (m) {
            if (unc) {
              const uint32_t i = (qn + __popc(m & lt)) & (kUncCap - 1);
              qu[i] = uu[e];
              qv[i] = vv[e];
              qh[i] = hh[e];
              qi[i] = rid * (32u * E) + static_cast<uint32_t>(lane) * E + e;
            }
            qn += __popc(m);
            if (qn - qt >= 32) resolve(32);
          }
        }
        emit(sure, uu, vv, E);
        if (!(last < xend)) break;
        base = last + 1.0;
      }
    } else {
      // ---- dense block (pbar >= 1): every position is a candidate ----
      const double inv_nb = d.inv_nb;
      const double x0d = static_cast<double>(x0);
      for (double xb = x0d; xb < xend; xb += 32.0) {
        const double x = xb + static_cast<double>(lane);
        uint32_t row, col;
        decode_pos(x, inv_nb, nb_d, nbi, row, col);
        const bool cand = x < xend && (!diag || col > row);
        const uint32_t u = d.a0 + row, v = d.b0 + col;
        bool acc = false;
        if (cand) {
          const double q_ = __ddiv_rn(__dmul_rn(w[u], w[v]), S);
          // the draw is taken for every candidate below 1, emitted or not, so
          // the stream does not depend on the launch's window
          acc = q_ >= 1.0 || unit53(rng.next()) < q_;
          acc = acc && x >= wlo && x < whi;
        }
        emit(&acc, &u, &v, 1);
      }
    }
    if (qn != qt) resolve(qn - qt);
    if (MODE == kWalkCount) {
      const uint32_t ce = static_cast<uint32_t>(warp_sum(static_cast<int64_t>(edges)));
      if (lane == 0) a.counts[q] = static_cast<int32_t>(ce);
    }
    if (MODE == kWalkWrite) flush_rest();
  }

  if (MODE == kWalkFold) {
    if (staging) flush_rest();
    const uint64_t cs = warp_sum_u64(checksum);
    const uint64_t es = warp_sum_u64(static_cast<uint64_t>(edges));
    if (lane == 0) {
      atomicAdd(&a.fold_out[0], static_cast<unsigned long long>(es));
      atomicAdd(&a.fold_out[1], static_cast<unsigned long long>(cs));
    }
  }
  if (a.prof.slots && lane == 0) {
    const int g = a.prof.base + static_cast<int>((blockIdx.x * THREADS + threadIdx.x) >> 5);
    a.prof.slots[2 * g] = t_start;
    a.prof.slots[2 * g + 1] = globaltimer_ns();
  }
}

// ---- class table -------------------------------------------------------------
// Classes on a geometric grid anchored at w[0]: thresholds t_k = w[0] /
// (1+eps)^k; class k holds the positive weights in [t_{k+1}, t_k), cut into
// pieces of at most 2^26 nodes; zero weights form one last class.  Every
// boundary is an independent binary search.  The grid width eps is the
// requested one, doubled until the grid fits the class cap.
struct ClassPlan {
  int64_t z;      // first zero weight (n if none)
  int kg;         // grid cells
  int K;          // classes (incl. the zero class); -1: does not fit
  int Knz;        // positive classes (blocks are over these)
  double eps;     // grid width used
  int64_t nblocks;
  unsigned long long chunks_full;  // chunks of the full source range
  int dense_blocks;
};

// one thread: z, the grid width and the thresholds
__global__ void cls_grid_kernel(const double* __restrict__ w, int64_t n, double eps0, int kcap, double* thr,
                                ClassPlan* plan) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t lo = -1, hi = n;  // first j with w[j] == 0 (w non-negative, non-increasing)
  while (hi - lo > 1) {
    const int64_t m = lo + ((hi - lo) >> 1);
    if (w[m] > 0.0) lo = m; else hi = m;
  }
  const int64_t z = hi;
  plan->z = z;
  plan->kg = 0;
  plan->K = 0;
  if (z == 0) {
    plan->eps = eps0;
    return;
  }
  const double wmax = w[0], wmin = w[z - 1];
  const int zero_class = z < n ? 1 : 0;
  // cells needed, plus room for pieces of oversized classes (n / 2^26 extra)
  const int extra = static_cast<int>(n / kClassMaxNodes) + 1;
  double eps = eps0;
  int kg = -1;
  for (int attempt = 0; attempt < 40; ++attempt, eps *= 2.0) {
    const double cells = ceil(log(wmax / wmin) / log1p(eps)) + 1.0;
    if (cells + zero_class + extra <= kcap) {
      kg = static_cast<int>(cells);
      break;
    }
  }
  plan->eps = eps;
  if (kg < 0) {
    plan->K = -1;
    return;
  }
  plan->kg = kg;
  double t = wmax;
  thr[0] = 0.0;
  for (int k = 1; k < kg; ++k) thr[k] = (t = t / (1.0 + eps));
}

__global__ void cls_bounds_kernel(const double* __restrict__ w, const double* __restrict__ thr,
                                  const ClassPlan* plan, int kcap, int64_t* bounds) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int kg = plan->kg;
  const int64_t z = plan->z;
  if (k > kg || k > kcap) return;
  if (k == 0) { bounds[0] = 0; return; }
  if (k == kg) { bounds[kg] = z; return; }
  const double t = thr[k];
  int64_t lo = -1, hi = z;  // first j in [0, z) with w[j] < t, in (lo, hi]
  while (hi - lo > 1) {
    const int64_t m = lo + ((hi - lo) >> 1);
    if (w[m] < t) hi = m; else lo = m;
  }
  bounds[k] = hi;
}

// one thread: compact non-empty cells into classes (splitting pieces of
// 2^26 nodes), append the zero class
__global__ void cls_compact_kernel(const double* __restrict__ w, int64_t n, const int64_t* __restrict__ bounds,
                                   int kcap, ClassPlan* plan, int64_t* start, double* wfirst, double* wlast) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (plan->K < 0) return;
  const int kg = plan->kg;
  const int64_t z = plan->z;
  int K = 0;
  for (int k = 0; k < kg; ++k) {
    for (int64_t a0 = bounds[k]; a0 < bounds[k + 1]; a0 += kClassMaxNodes) {
      const int64_t b0 = imin64(a0 + kClassMaxNodes, bounds[k + 1]);
      if (K >= kcap) { plan->K = -1; return; }
      start[K] = a0;
      wfirst[K] = w[a0];
      wlast[K] = w[b0 - 1];
      ++K;
    }
  }
  plan->Knz = K;
  if (z < n) {
    if (K >= kcap) { plan->K = -1; return; }
    start[K] = z;
    wfirst[K] = 0.0;
    wlast[K] = 0.0;
    ++K;
  }
  start[K] = n;
  plan->K = K;
}

__host__ __device__ __forceinline__ int64_t tri_index(int A, int B, int K) {  // A <= B < K
  return static_cast<int64_t>(A) * K - static_cast<int64_t>(A) * (A - 1) / 2 + (B - A);
}

// Block descriptors, one thread per (A, B), A <= B < Knz; chunks_full += nchunks.
__global__ void blk_desc_kernel(const int64_t* __restrict__ start, const double* __restrict__ wfirst,
                                const double* __restrict__ wlast, ClassPlan* plan, double S, double chunk_cand,
                                BlockDesc* blocks) {
  const int Knz = plan->K < 0 ? 0 : plan->Knz;
  const int A = blockIdx.y * blockDim.y + threadIdx.y;
  const int B = blockIdx.x * blockDim.x + threadIdx.x;
  if (A >= Knz || B >= Knz || B < A) return;
  BlockDesc d;
  d.a0 = static_cast<uint32_t>(start[A]);
  d.na = static_cast<uint32_t>(start[A + 1] - start[A]);
  d.b0 = static_cast<uint32_t>(start[B]);
  d.nb = static_cast<uint32_t>(start[B + 1] - start[B]);
  d.flags = A == B ? kBlkDiag : 0u;
  const double pbar = __ddiv_rn(__dmul_rn(wfirst[A], wfirst[B]), S);
  d.pbar = pbar;
  d.inv_nb = 1.0 / static_cast<double>(d.nb);
  const int64_t N = static_cast<int64_t>(d.na) * d.nb;
  d.inv_mu = 0.0;
  d.hs = 0;
  int64_t L;
  if (!(pbar > 0.0) || N == 0 || (A == B && d.na < 2)) {
    L = 1;
    d.nchunks = 0;
  } else if (pbar >= 1.0) {
    d.flags |= kBlkDense;
    L = static_cast<int64_t>(chunk_cand);
    d.nchunks = (N + L - 1) / L;
    atomicAdd(&plan->dense_blocks, 1);
  } else {
    d.inv_mu = 1.0 / -log1p(-pbar);
    // smallest p_uv of the block, as the generators compute it, over pbar:
    // p_uv / pbar >= that ratio for every pair (monotone FP ops)
    const double qmin = __ddiv_rn(__dmul_rn(wlast[A], wlast[B]), S);
    const double ratio = __ddiv_rn(qmin < 1.0 ? qmin : 1.0, pbar);
    const double hsd = floor(ratio * 2048.0);
    d.hs = hsd >= 2048.0 ? 2048u : static_cast<uint32_t>(hsd);
    const double Ld = floor(chunk_cand / pbar);
    L = Ld >= static_cast<double>(N) ? N : (Ld < 1.0 ? 1 : static_cast<int64_t>(Ld));
    d.nchunks = (N + L - 1) / L;
  }
  d.L = L;
  blocks[tri_index(A, B, Knz)] = d;
  if (d.nchunks) atomicAdd(&plan->chunks_full, static_cast<unsigned long long>(d.nchunks));
}

// Per launch: the chunks of each block whose rows meet [lo, hi).
__global__ void blk_range_kernel(const BlockDesc* __restrict__ blocks, int64_t nblocks, int64_t lo, int64_t hi,
                                 BlockRange* ranges, int64_t* nchunks) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < nblocks; b += stride) {
    const BlockDesc d = blocks[b];
    const int64_t r0 = imin64(imax64(lo - static_cast<int64_t>(d.a0), 0), d.na);
    const int64_t r1 = imin64(imax64(hi - static_cast<int64_t>(d.a0), 0), d.na);
    BlockRange r{0, r0 * d.nb, r1 * d.nb};
    int64_t cnt = 0;
    if (d.nchunks > 0 && r1 > r0) {
      r.c_lo = r.x_lo / d.L;
      const int64_t c_hi = (r.x_hi + d.L - 1) / d.L;
      cnt = c_hi - r.c_lo;
    }
    ranges[b] = r;
    nchunks[b] = cnt;
  }
}

// chunk -> block map of a launch: one warp per block fills its chunk ids
__global__ void blk_chunk_map_kernel(const int64_t* __restrict__ nchunks, const int64_t* __restrict__ prefix,
                                     int64_t nblocks, uint32_t* chunk_block) {
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int lane = lane_id();
  for (int64_t b = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < nblocks; b += nwarps) {
    const int64_t c = nchunks[b], p = prefix[b];
    for (int64_t i = lane; i < c; i += 32) chunk_block[p + i] = static_cast<uint32_t>(b);
  }
}

}  // namespace clg
