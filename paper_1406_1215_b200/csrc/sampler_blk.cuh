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
constexpr int64_t kClassMaxNodes = (1ll << 26) - 64;  // nodes per class (block positions < 2^52 - 2^27)
constexpr uint32_t kBlkDiag = 1u, kBlkDense = 2u;

struct __align__(16) BlockDesc {
  double pbar;      // RN(RN(w[s_A] w[s_B]) / S): envelope (>= every p_uv of the block)
  double inv_mu;    // 1 / -log1p(-pbar) (sparse blocks)
  double inv_nb;    // RD(1 / nb) (decode_pos)
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
  // kWalkPairs: seeds seed..seed+trials-1 in one launch (launch chunk q of
  // trial t is claim t * total + q), edges counted in pair_counts[u * n + v]
  uint64_t seed;
  int64_t trials;
  uint32_t* pair_counts;
  uint32_t n;
};

// E = -log(U) ~ Exp(1) by inversion, U = ((x >> 12) + 1/2) 2^-52 in (0,1)
// from the top 52 bits of x: y = U 2^52 is built from bits (no int->fp
// conversion), log y = exponent + table log of the reciprocal centre + a
// degree-5 log1p series on |t| <= 2^-8; relative error ~2^-47 (statistically
// exact).  T[i] = {RN(1/c_i), -log RN(1/c_i)}, c_i = 1 + (i + 1/2)/128.
__device__ __forceinline__ double exp52_y(uint64_t x) {  // (x >> 12) + 1/2, exact
  return __longlong_as_double(static_cast<long long>((x >> 12) | 0x4330000000000000ull)) - (0x1.0p52 - 0.5);
}
__device__ __forceinline__ int exp52_index(double y) { return (__double2hiint(y) >> 13) & (kLogTable - 1); }
__device__ __forceinline__ double exp52_tab(double y, double2 tc) {
  const int yh = __double2hiint(y);
  const int be = yh >> 20;  // biased exponent (y >= 1/2)
  const double m = __hiloint2double((yh & 0x000fffff) | 0x3ff00000, __double2loint(y));
  const double t = __fma_rn(m, tc.x, -1.0);
  double sp = __fma_rn(t, 1.0 / 5.0, -1.0 / 4.0);
  sp = __fma_rn(t, sp, 1.0 / 3.0);
  sp = __fma_rn(t, sp, -0.5);
  sp = __fma_rn(t, sp, 1.0);
  const double k = __hiloint2double(0x43380000, 1075 - be) - 0x1.8p52;  // 52 - log2 of y's binade, exact
  return __fma_rn(k, 0x1.62e42fefa39efp-1, __fma_rn(k, 0x1.abc9e3b39803fp-56, -__fma_rn(t, sp, tc.y)));
}
__device__ __forceinline__ double exp52(uint64_t x, const double2* __restrict__ T) {
  const double y = exp52_y(x);
  return exp52_tab(y, T[exp52_index(y)]);
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

// (row, col) of row-major position x (exact integer double < 2^52) in a
// block of nb columns.  The quotient is rounded down twice (inv_nb_rd =
// RD(1/nb), RD product), so it is the true quotient or one less; the exact
// residual x - row nb in [0, 2 nb) settles it.  No int <-> fp conversions:
// the integers are read from the low word of 2^52 + value.
__device__ __forceinline__ void decode_pos(double x, double inv_nb_rd, double nb_d, int32_t nb, uint32_t& row,
                                           uint32_t& col) {
  const double qf = __dadd_rd(__dmul_rd(x, inv_nb_rd), 0x1.0p52);  // 2^52 + floor(q)
  uint32_t r = static_cast<uint32_t>(__double2loint(qf));
  int32_t c = __double2loint(__fma_rn(-(qf - 0x1.0p52), nb_d, x) + 0x1.0p52);
  if (c >= nb) {
    c -= nb;
    ++r;
  }
  row = r;
  col = static_cast<uint32_t>(c);
}

constexpr int kStageCap = 512;  // staged pairs per warp (ring / write modes)
constexpr int kUncCap = 64;     // queued uncertain candidates per warp

__host__ __device__ inline size_t blk_smem_bytes(int threads) {
  return kLogTable * sizeof(double2) +
         static_cast<size_t>(threads / 32) * (kStageCap * sizeof(uint2) + kUncCap * (sizeof(uint2) + 4) + 16);
}

// Per-warp chunk constants needed only on the rare paths (uncertain
// candidates), kept in shared memory instead of registers.
struct WarpChunk {
  uint64_t key;
  double pbar;
};

template <int MODE, int E, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) blk_kernel(BlkArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* s_log = reinterpret_cast<double2*>(smem_raw);
  const int wib = threadIdx.x >> 5;
  unsigned char* wbase = smem_raw + kLogTable * sizeof(double2) +
                         static_cast<size_t>(wib) * (kStageCap * sizeof(uint2) + kUncCap * (sizeof(uint2) + 4) + 16);
  uint2* stage = reinterpret_cast<uint2*>(wbase);
  uint2* quv = reinterpret_cast<uint2*>(wbase + kStageCap * sizeof(uint2));
  uint32_t* qh = reinterpret_cast<uint32_t*>(wbase + kStageCap * sizeof(uint2) + kUncCap * sizeof(uint2));
  WarpChunk& wc = *reinterpret_cast<WarpChunk*>(wbase + kStageCap * sizeof(uint2) + kUncCap * (sizeof(uint2) + 4));
  for (int i = threadIdx.x; i < kLogTable; i += THREADS) s_log[i] = make_double2(a.logtab->inv_c[i], a.logtab->nlog_inv[i]);
  __syncthreads();

  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  const unsigned long long t_start = a.prof.slots ? globaltimer_ns() : 0ull;
  const int64_t total = *a.total_chunks;
  const uint32_t tmask = (1u << a.track_shift) - 1u;
  const bool track = MODE == kWalkFold && a.degree != nullptr;

  // fold-mode ring: a private circular segment per warp (no reservation atomics)
  uint2* seg = nullptr;  // null: fold only
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
  constexpr bool staging = MODE == kWalkWrite || MODE == kWalkFold;  // fold: every edge is staged (fold + ring at flush)
  uint32_t head = 0, tail = 0;  // stage counters (warp-uniform)
  uint64_t checksum = 0;
  uint64_t wedges = 0;          // edges of this warp
  int64_t out_pos = 0;          // write mode
  Xoro128 rng;

  // fold of one staged edge: checksum term and tracked degrees
  auto fold_pair = [&](uint2 e, bool live) {
    checksum += live ? edge_hash(e.x, e.y) : 0ull;
    if (track) {
      const bool tu = live && (e.x & tmask) == 0, tv = live && (e.y & tmask) == 0;
      if (__any_sync(CLG_FULL, tu || tv)) {
        if (tu) atomicAdd(&a.degree[e.x >> a.track_shift], 1u);
        if (tv) atomicAdd(&a.degree[e.y >> a.track_shift], 1u);
      }
    }
  };
  // flush 64 staged pairs.  Fold mode folds them (2 per lane, every lane
  // busy) and writes them into the warp's ring segment as one 512-byte burst
  // of 16-byte vector stores (measured faster here than handing the region to
  // the TMA engine with cp.async.bulk, whose issue/wait serialises on one
  // lane); write mode stores them at the chunk's output offset.
  auto flush64 = [&]() {
    __syncwarp();
    if (MODE == kWalkFold) {
      const uint4 v2 = *reinterpret_cast<const uint4*>(&stage[(tail + 2 * lane) & (kStageCap - 1)]);
      fold_pair(make_uint2(v2.x, v2.y), true);
      fold_pair(make_uint2(v2.z, v2.w), true);
      if (seg) *reinterpret_cast<uint4*>(&seg[(wpos + 2 * lane) & smask]) = v2;
      wpos += 64;
    } else {
#pragma unroll
      for (int i = 0; i < 64; i += 32) {
        const int64_t p = out_pos + i + lane;
        if (p < a.cap) a.pairs[p] = stage[(tail + i + lane) & (kStageCap - 1)];
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
    for (uint32_t i0 = 0; i0 < rem; i0 += 32) {
      const bool live = i0 + lane < rem;
      const uint2 e = stage[(tail + i0 + lane) & (kStageCap - 1)];
      if (MODE == kWalkFold) {
        fold_pair(e, live);
        if (seg && live) seg[(wpos + i0 + lane) & smask] = e;
      } else if (live) {
        const int64_t p = out_pos + i0 + lane;
        if (p < a.cap) a.pairs[p] = e;
        else atomicAdd(a.overflow, 1ull);
      }
    }
    if (MODE == kWalkFold) wpos += rem;
    else out_pos += rem;
    tail = head;
    __syncwarp();
  };
  uint32_t cw = 0;  // edges of the current chunk (warp-uniform)
  // one candidate slot per lane: stage the accepted pairs
  auto emit1 = [&](bool acc, uint32_t u, uint32_t v) {
    if (MODE == kWalkPairs && acc) atomicAdd(&a.pair_counts[static_cast<uint64_t>(u) * a.n + v], 1u);
    const unsigned b = __ballot_sync(CLG_FULL, acc);
    const uint32_t nb = __popc(b);
    if (staging) {
      if (acc) stage[(head + __popc(b & lt)) & (kStageCap - 1)] = make_uint2(u, v);
      head += nb;
    }
    cw += nb;
  };

  for (;;) {
    unsigned long long qq = 0;
    if (lane == 0) qq = atomicAdd(a.queue, 1ull);
    int64_t q = static_cast<int64_t>(__shfl_sync(CLG_FULL, qq, 0));
    uint64_t seed_mix = a.seed_mix;
    if (MODE == kWalkPairs) {
      if (total == 0 || q >= total * a.trials) break;
      const int64_t t = q / total;
      q -= t * total;
      seed_mix = mix64((a.seed + static_cast<uint64_t>(t)) ^ 0x636c67656e626c6bULL);  // as blk_args
    } else if (q >= total) {
      break;
    }
    const uint32_t b = __ldg(a.chunk_block + q);
    const BlockDesc d = a.blocks[b];
    const BlockRange r = a.ranges[b];
    const int64_t c = r.c_lo + (q - __ldg(a.chunk_prefix + b));
    const int64_t N = static_cast<int64_t>(d.na) * d.nb;
    const int64_t x0 = c * d.L;
    const int64_t x1 = imin64(x0 + d.L, N);
    const double xend = static_cast<double>(x1);
    // a chunk cut by the launch's source range emits only the rows inside it
    const bool partial = r.x_lo > x0 || r.x_hi < x1;
    const uint64_t key = mix64(seed_mix ^ (static_cast<uint64_t>(b) | (static_cast<uint64_t>(c) << 20)));
    rng.seed_key(key + 0x632be59bd9b4e019ULL * static_cast<uint64_t>(lane + 1));
    __syncwarp();
    if (lane == 0) {
      wc.key = key;
      wc.pbar = d.pbar;
    }
    __syncwarp();
    const bool diag = (d.flags & kBlkDiag) != 0;
    const double nb_d = static_cast<double>(d.nb);
    const int32_t nbi = static_cast<int32_t>(d.nb);
    uint32_t qn = 0, qt = 0;  // uncertain queue counters (warp-uniform)
    if (MODE == kWalkWrite) out_pos = a.offsets[q];
    cw = 0;
    const double wlo = static_cast<double>(r.x_lo), whi = static_cast<double>(r.x_hi);

    // decide the queued uncertain candidates (k <= 32): gather w_u, w_v
    auto resolve = [&](uint32_t k) {
      __syncwarp();
      bool acc = false;
      uint32_t u = 0, v = 0;
      if (static_cast<uint32_t>(lane) < k) {
        const uint32_t i = (qt + lane) & (kUncCap - 1);
        const uint2 uv = quv[i];
        const uint32_t hid = qh[i];
        u = uv.x;
        v = uv.y;
        const double q_ = __ddiv_rn(__dmul_rn(a.w[u], a.w[v]), a.S);  // edge_skip.cpp:36
        acc = lazy_accept(hid & 2047u, __ddiv_rn(q_ < 1.0 ? q_ : 1.0, wc.pbar), wc.key, hid >> 11);
      }
      qt += k;
      __syncwarp();
      emit1(acc, u, v);
      if (staging)
        while (head - tail >= 64) flush64();
    };

    if (!(d.flags & kBlkDense)) {
      // ---- sparse block: each lane runs its own geometric process over its
      // 1/32 of the chunk (memoryless restart at the lane's first position:
      // no cross-lane dependence), E candidates per iteration ----
      const double inv_mu = d.inv_mu, inv_nb = d.inv_nb;
      const uint32_t hs = d.hs;
      const int64_t ls = (x1 - x0 + 31) >> 5;
      const int64_t lx0 = imin64(x0 + lane * ls, x1);
      const double lend = static_cast<double>(imin64(lx0 + ls, x1));
      double pos = static_cast<double>(lx0) - 1.0;  // last candidate position
      bool live = pos + 1.0 < lend;
      for (uint32_t id = 0; __any_sync(CLG_FULL, live); id += E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t x = rng.next();
          // geometric gap floor(E / mu) + 1 (>= 2^52: past every chunk end)
          pos += __dadd_rd(exp52(x, s_log) * inv_mu, 0x1.0p52) - (0x1.0p52 - 1.0);
          live = live && pos < lend;
          uint32_t row, col;
          decode_pos(pos, inv_nb, nb_d, nbi, row, col);
          bool ok = live && (col > row || !diag);
          if (partial) ok = ok && pos >= wlo && pos < whi;
          const uint32_t u = d.a0 + row, v = d.b0 + col;
          const uint32_t h = static_cast<uint32_t>(x) & 2047u;
          const bool sure = ok && h < hs;
          emit1(sure, u, v);
          const bool unc = ok && !sure;
          const unsigned m = __ballot_sync(CLG_FULL, unc);
          if (m) {
            if (unc) {
              const uint32_t i = (qn + __popc(m & lt)) & (kUncCap - 1);
              quv[i] = make_uint2(u, v);
              qh[i] = h | ((((id + e) << 5 | static_cast<uint32_t>(lane)) & 0x1fffffu) << 11);
            }
            qn += __popc(m);
            if (qn - qt >= 32) resolve(32);
          }
        }
        if (staging)
          while (head - tail >= 64) flush64();
      }
    } else {
      // ---- dense block (pbar >= 1): every position is a candidate ----
      const double inv_nb = d.inv_nb;
      for (double xb = static_cast<double>(x0); xb < xend; xb += 32.0) {
        const double x = xb + static_cast<double>(lane);
        uint32_t row, col;
        decode_pos(x, inv_nb, nb_d, nbi, row, col);
        const bool cand = x < xend && (col > row || !diag);
        const uint32_t u = d.a0 + row, v = d.b0 + col;
        bool acc = false;
        if (cand) {
          const double q_ = __ddiv_rn(__dmul_rn(a.w[u], a.w[v]), a.S);
          // the draw is taken for every candidate below 1, emitted or not, so
          // the stream does not depend on the launch's window
          acc = q_ >= 1.0 || unit53(rng.next()) < q_;
          if (partial) acc = acc && x >= wlo && x < whi;
        }
        emit1(acc, u, v);
        if (staging)
          while (head - tail >= 64) flush64();
      }
    }
    if (qn != qt) resolve(qn - qt);
    if (MODE == kWalkCount && lane == 0) a.counts[q] = static_cast<int32_t>(cw);
    wedges += cw;
    if (MODE == kWalkWrite) flush_rest();
  }

  if (MODE == kWalkFold) {
    flush_rest();
    const uint64_t cs = warp_sum_u64(checksum);
    if (lane == 0) {
      atomicAdd(&a.fold_out[0], static_cast<unsigned long long>(wedges));
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
  d.inv_nb = __drcp_rd(static_cast<double>(d.nb));
  const int64_t N = static_cast<int64_t>(d.na) * d.nb;
  d.inv_mu = 0.0;
  d.hs = 0;
  int64_t L;
  // pbar < 2^-900: below 2^-848 expected edges in the block, treated as empty
  if (!(pbar >= 0x1.0p-900) || N == 0 || (A == B && d.na < 2)) {
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
