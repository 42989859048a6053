// Counter-stream Chung–Lu sampler (the north star's keyed RNG: every draw is a
// function of (seed, u, split, lane, draw index)).  Statistically exact, not
// stream-identical to the
// reference: every pair (u, v>u) appears independently with probability
// min(w_u w_v / S, 1), the law of edges_from_source (edge_skip.cpp:20-46).
//
// Envelope construction.  The destination axis is cut into weight classes
// ("segments") [c_k, c_{k+1}) inside which the sorted weights vary by at most
// a factor (1+eps): w[c_k] <= (1+eps) * w[c_{k+1}-1].  Inside a segment a
// source u proposes candidates as a Bernoulli(pbar) process with the CONSTANT
// envelope pbar = min(w_u w[c_k] / S, 1) — i.i.d. geometric skips, so the skip
// no longer depends on the previous candidate's weight — and thins each
// candidate with probability q/pbar = w_v / w[c_k].  Since that ratio is at
// least w[c_{k+1}-1]/w[c_k] >= 1/(1+eps), a candidate whose accept draw is
// below it is accepted WITHOUT reading w[v]; only the remaining ~eps/2 of the
// candidates gather their weight.  A skip past the segment end restarts at the
// next segment (memorylessness).  Saturated segments (pbar = 1) propose every
// position and accept with probability min(q, 1).
//
// Work units: (source u, v-range [lo,hi), split index s).  Heavy sources are
// split into v-ranges of about kSplitCand expected candidates (level-2
// balance, hub splitting) — a deterministic function of the weights, so the
// edge set does not depend on the GPU count or the schedule.
#pragma once

#include "common.cuh"
#include "fastmath.cuh"
#include "sampler_ref.cuh"

namespace clg {

// 53-bit uniform strictly inside (0,1): (x>>11 + 1/2) * 2^-53.
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
  const uint64_t x = (static_cast<uint64_t>(hi) << 32) | lo;
  return __dmul_rn(static_cast<double>(x >> 11) + 0.5, 0x1.0p-53);
}

struct Segments {
  const int64_t* start;  // K+1 entries, start[K] = n
  const double* wfirst;  // w[start[k]]   (the class envelope)
  const double* sure;    // w[start[k+1]-1] / w[start[k]]  (accept without gather below this)
  const double* em;      // K+1 envelope-mass prefix: em[k+1] = em[k] + wfirst[k] * len_k
  const double* invwf;   // 1 / wfirst[k] (0 for a zero class)
  int K;
  const unsigned short* bucket;  // kBuckets entries: a lower bound of the class of any T in bucket b
  int depth;  // max over buckets of (classes a bucket can reach) - 1: the class of T is within
              // [bucket[b], bucket[b] + depth]
  int nb;     // number of buckets (<= kBuckets)
  double em_end;      // em[K]
  double inv_bucket;  // nb / em[K]
};

constexpr int kBuckets = 8192;  // bucket table capacity

constexpr int kSegSmemMax = 1024;  // classes staged in (dynamic) shared memory per CTA
constexpr double kBandTau = 0.0625;  // hazard envelope below pbar = 1/16

struct CtrWalkArgs {
  const double* __restrict__ w;
  int64_t n;
  double S;
  double invS;             // 1 / S (screens and envelope rates only; pbar itself is w_u w_v / S)
  int64_t lo, hi;          // source range [lo,hi)
  Segments seg;
  // hub splitting: sources [lo, lo+H) are split; unit prefix over them
  int64_t H;
  const int64_t* hub_units;  // H+1 prefix of split counts (hub_units[0] = 0)
  int64_t total_units;       // hub_units[H] + (hi - lo - H)
  unsigned long long* queue; // next unclaimed unit
  // outputs (same meaning as RefWalkArgs)
  int32_t* counts;           // per unit (count mode)
  const int64_t* offsets;    // per unit (write mode)
  uint2* pairs;
  int64_t cap;
  uint32_t* degree;
  int track_shift;
  uint2* ring;
  unsigned long long ring_mask;
  unsigned long long* fold_out;
  unsigned long long* overflow;
  WarpProf prof;
  int refill_min;  // refill idle lanes only when at least this many are idle
};

// Segment holding position j (binary search over start[]).
__device__ __forceinline__ int seg_of(const Segments& s, int64_t j) {
  int a = 0, b = s.K;  // start[a] <= j < start[b]
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (__ldg(s.start + m) <= j) a = m; else b = m;
  }
  return a;
}

__device__ __forceinline__ double pbar_of(double wu, double wv, double S) {
  return __ddiv_rn(__dmul_rn(wu, wv), S);  // the generators' q = w_u w_v / S
}

// First v in [a, b) with w_u w[v] / S < thr (b if none); monotone in v.
__device__ __forceinline__ int64_t first_p_below(const double* __restrict__ w, double wu, double S, int64_t a,
                                                 int64_t b, double thr) {
  int64_t lo = a - 1, hi = b;  // answer in (lo, hi]
  while (hi - lo > 1) {
    const int64_t m = lo + ((hi - lo) >> 1);
    if (pbar_of(wu, w[m], S) < thr) hi = m; else lo = m;
  }
  return hi;
}

__device__ __forceinline__ double unit53(uint64_t b) {  // [0,1)
  return static_cast<double>(b >> 11) * 0x1.0p-53;
}

// Key of the per-unit stream: a bijection of (u, split) mixed with the seed.
__device__ __forceinline__ uint64_t unit_key(uint64_t seed_mix, int64_t u, uint32_t split) {
  return mix64(seed_mix ^ (static_cast<uint64_t>(u) | (static_cast<uint64_t>(split) << 36)));
}



// ---- warp-cooperative processing of heavy units --------------------------
// All 32 lanes work on one unit: round r, lane l takes Poisson events 64r+2l
// and 64r+2l+1 of the unit's hazard process (a warp prefix sum of
// exponential pairs), so positions come out sorted across lanes; duplicates
// are adjacent (neighbour shuffle).  Lane l draws from its own keyed stream
// (unit key, lane), so the draws and hence the edges are a deterministic
// function of (seed, u, split) — the same in the count, write and fold modes.
__device__ __forceinline__ double warp_incl_scan_f64(double x) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(CLG_FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ double bern_gk(double inv_kappa, double z) {
  const double z2 = z * z;
  return inv_kappa * (1.0 + z * 0.5 + z2 * (1.0 / 12.0) - z2 * z2 * (1.0 / 720.0) + z2 * z2 * z2 * (1.0 / 30240.0));
}

// Exp(1) by inversion from the top 53 bits of x, E = -log(U),
// U = (x>>11 + 1/2) 2^-53 in (0,1): table log (128 entries) + degree-5
// log1p, absolute error < 2^-50 (statistically exact).
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

// Bernoulli(a) from a lazily refined uniform R = (h + R')/2048: the 11 bits h
// come with the event's exponential draw (its low bits), R' (53 bits) is
// drawn only when h alone cannot decide (probability 1/2048 per uncertain
// test) from a hash of the event's identity, so the decision does not
// depend on when it is taken (the fold mode defers it by one round).
__device__ __forceinline__ bool lazy_accept(uint32_t h, double a, uint64_t key, uint32_t id) {
  const double s = a * 2048.0;  // exact scaling
  if (static_cast<double>(h + 1u) <= s) return true;
  if (static_cast<double>(h) >= s) return false;
  const uint64_t r = mix64((key ^ 0xd6e8feb86659fd93ULL) + 0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(id) + 1ull));
  return unit53(r) < s - static_cast<double>(h);  // s - h exact (Sterbenz)
}

// Fold-mode sink of one warp: checksum, edge count, tracked degrees and the
// ring store of every emitted edge.  Each warp of the launch owns a private
// circular segment of the ring (no reservation atomics): slot = base +
// (emitted-by-this-warp mod segment).  emit2 takes up to two edges per lane,
// slots assigned lane-major by one ballot pair.
struct FoldSink {
  uint64_t checksum;
  uint32_t edges;   // per lane (< 2^32 over a launch)
  uint2* seg;       // this warp's ring segment (nullptr: no ring)
  uint32_t smask;   // segment length - 1
  uint32_t wpos;    // edges this warp has written (warp-uniform)

  __device__ __forceinline__ void init(const CtrWalkArgs& a) {
    checksum = 0;
    edges = 0;
    seg = nullptr;
    smask = 0;
    wpos = 0;
    if (a.ring) {
      const unsigned nw = gridDim.x * (blockDim.x >> 5);
      const unsigned gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
      const int lcap = 63 - __clzll(static_cast<long long>(a.ring_mask + 1ull));
      const int lnw = nw > 1 ? 32 - __clz(nw - 1) : 0;
      int sl = lcap - lnw;
      sl = sl < 5 ? 5 : (sl > 20 ? 20 : sl);
      if (sl > lcap) sl = lcap;
      smask = (1u << sl) - 1u;
      seg = a.ring + ((static_cast<unsigned long long>(gw) << sl) & a.ring_mask);
    }
  }

  __device__ __forceinline__ void one(const CtrWalkArgs& a, uint32_t u, uint32_t v, uint32_t tmask, uint32_t r) {
    checksum += mix64((static_cast<uint64_t>(u) << 32) | v);
    if (a.degree && (v & tmask) == 0) atomicAdd(&a.degree[v >> a.track_shift], 1u);
    if (seg) seg[(wpos + r) & smask] = make_uint2(u, v);
  }

  __device__ __forceinline__ void emit2(const CtrWalkArgs& a, uint32_t u, uint32_t tmask, unsigned lt, int lane,
                                        bool c0, uint32_t v0, bool c1, uint32_t v1) {
    const unsigned b0 = __ballot_sync(CLG_FULL, c0), b1 = __ballot_sync(CLG_FULL, c1);
    if ((b0 | b1) == 0u) return;
    const unsigned r0 = __popc(b0 & lt) + __popc(b1 & lt);
    edges += (c0 ? 1u : 0u) + (c1 ? 1u : 0u);
    if (c0) one(a, u, v0, tmask, r0);
    if (c1) one(a, u, v1, tmask, r0 + (c0 ? 1u : 0u));
    wpos += __popc(b0) + __popc(b1);
  }

  // warp totals into fold_out[0..1]
  __device__ __forceinline__ void finish(const CtrWalkArgs& a, int lane) {
    const uint64_t c = warp_sum_u64(checksum);
    const uint64_t e = warp_sum_u64(static_cast<uint64_t>(edges));
    if (lane == 0) {
      atomicAdd(&a.fold_out[0], static_cast<unsigned long long>(e));
      atomicAdd(&a.fold_out[1], static_cast<unsigned long long>(c));
    }
  }
};

constexpr int kSideCap = 128;
#ifndef CLG_WIN_REFRESH
#define CLG_WIN_REFRESH 16
#endif
constexpr int kWinRefresh = CLG_WIN_REFRESH;  // slide the 32-class acceptance window when the round reached class kw + this  // per-warp staging of deferred accepts (fold mode)

// Class record staged in shared memory: everything an event needs to map its
// envelope mass T to a position in class k (two 16-byte loads).
struct __align__(16) ClassRec {
  double em;    // envelope mass before class k
  double iwf;   // 1 / wfirst[k] (0 for a zero class)
  uint32_t s0;  // first node of the class (node ids < 2^32 in the counter stream)
  uint32_t s1;  // one past the last node
  double wf;    // wfirst[k]
};

// Class holding position j (binary search over the records).
__device__ __forceinline__ int rec_of(const ClassRec* r, int K, int64_t j) {
  int a = 0, b = K;
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (static_cast<int64_t>(r[m].s0) <= j) a = m; else b = m;
  }
  return a;
}

// Dynamic shared memory of the warp kernel: K+2 class records, the log
// table, the bucket index and the per-warp staging of deferred accepts.
__host__ __device__ inline size_t ctr_warp_smem_bytes(int K, int nb, int threads) {
  return static_cast<size_t>(K + 2) * sizeof(ClassRec) + sizeof(LogTable) +
         ((static_cast<size_t>(nb) * sizeof(unsigned short) + 15) & ~size_t(15)) +
         static_cast<size_t>(threads / 32) * kSideCap * sizeof(uint32_t);
}

// Per-warp unit constants of the warp kernel, kept in shared memory instead
// of registers (read at class-window refreshes and rare slow paths only).
struct WarpUnitConst {
  double c_u, inv_kappa;
  uint64_t ukey;  // unit stream key; lane l's key is ukey + C (l + 1)
};

__device__ __forceinline__ uint64_t lane_key(uint64_t ukey, int lane) {
  return ukey + 0x632be59bd9b4e019ULL * static_cast<uint64_t>(lane + 1);
}

// lazy_accept with the lane's key read from shared memory only when the 11
// bits cannot decide
__device__ __forceinline__ bool lazy_accept_w(uint32_t h, double a, const WarpUnitConst& wc, int lane, uint32_t id) {
  const double s = a * 2048.0;
  if (static_cast<double>(h + 1u) <= s) return true;
  if (static_cast<double>(h) >= s) return false;
  return lazy_accept(h, a, lane_key(wc.ukey, lane), id);
}

template <int MODE, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) ctr_warp_kernel(CtrWalkArgs a, const int64_t* __restrict__ split_pos,
                                                              const LogTable* __restrict__ logtab, uint64_t seed_mix,
                                                              int64_t U_heavy, unsigned long long* queue_heavy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.seg.K;
  const int NB = a.seg.nb;
  ClassRec* s_rec = reinterpret_cast<ClassRec*>(smem_raw);
  LogTable& s_log = *reinterpret_cast<LogTable*>(smem_raw + static_cast<size_t>(K + 2) * sizeof(ClassRec));
  unsigned short* s_bucket = reinterpret_cast<unsigned short*>(reinterpret_cast<unsigned char*>(&s_log) + sizeof(LogTable));
  uint32_t* s_side = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(s_bucket) +
                                                 ((static_cast<size_t>(NB) * sizeof(unsigned short) + 15) & ~size_t(15)));
  for (int i = threadIdx.x; i <= K; i += blockDim.x) {
    ClassRec r;
    r.em = a.seg.em[i];
    r.iwf = i < K ? a.seg.invwf[i] : 0.0;
    r.s0 = static_cast<uint32_t>(a.seg.start[i]);
    r.s1 = i < K ? static_cast<uint32_t>(a.seg.start[i + 1]) : r.s0;
    r.wf = i < K ? a.seg.wfirst[i] : 0.0;
    s_rec[i] = r;
    if (i == K) {  // sentinel past the end: no T reaches it
      r.em = __longlong_as_double(0x7ff0000000000000LL);
      r.iwf = 0.0;
      r.wf = 0.0;
      s_rec[K + 1] = r;
    }
  }
  for (int i = threadIdx.x; i < kLogTable; i += blockDim.x) {
    s_log.inv_c[i] = logtab->inv_c[i];
    s_log.nlog_inv[i] = logtab->nlog_inv[i];
  }
  for (int i = threadIdx.x; i < NB; i += blockDim.x) s_bucket[i] = a.seg.bucket[i];
  __syncthreads();
  const double* __restrict__ g_sure = a.seg.sure;

  const int lane = lane_id();
  uint32_t* side = s_side + (threadIdx.x >> 5) * kSideCap;
  __shared__ WarpUnitConst s_wc[THREADS / 32];
  WarpUnitConst& wc = s_wc[threadIdx.x >> 5];
  const unsigned long long t_start = a.prof.slots ? globaltimer_ns() : 0ull;
  const unsigned lt_mask = lanemask_lt();
  const double* __restrict__ w = a.w;
  const double S = a.S;
  const uint32_t tmask = (1u << a.track_shift) - 1u;
  FoldSink fs;
  fs.init(a);
  Xoro128 rng;

  for (;;) {
    unsigned long long ug = 0;
    if (lane == 0) ug = atomicAdd(queue_heavy, 1ull);
    const int64_t unit = static_cast<int64_t>(__shfl_sync(CLG_FULL, ug, 0));
    if (unit >= U_heavy) break;
    // ---- decode (warp-uniform) ----
    int64_t u, j, vend;
    uint32_t split = 0;
    const int64_t hub_units = a.H > 0 ? a.hub_units[a.H] : 0;
    if (unit < hub_units) {
      int64_t lo_h = 0, hi_h = a.H;
      while (hi_h - lo_h > 1) {
        const int64_t m = (lo_h + hi_h) >> 1;
        if (a.hub_units[m] <= unit) lo_h = m; else hi_h = m;
      }
      u = a.lo + lo_h;
      split = static_cast<uint32_t>(unit - a.hub_units[lo_h]);
      j = split_pos[unit];
      vend = unit + 1 == a.hub_units[lo_h + 1] ? a.n : split_pos[unit + 1];
    } else {
      u = a.lo + a.H + (unit - hub_units);
      j = u + 1;
      vend = a.n;
    }
    const double wu = w[u];
    const uint32_t u32 = static_cast<uint32_t>(u);
    int64_t out_pos = MODE == kWalkWrite ? a.offsets[unit] : 0;
    int32_t cnt = 0;
    // lane streams: key(u, split) mixed with the lane
    const uint64_t ukey = unit_key(seed_mix, u, split);
    rng.seed_key(lane_key(ukey, lane));
    __syncwarp();
    if (lane == 0) wc.ukey = ukey;

    // emission of up to two edges per lane, lane-major (c0 before c1)
    auto emit2 = [&](bool c0, uint32_t v0, bool c1, uint32_t v1) {
      if (MODE == kWalkFold) {
        fs.emit2(a, u32, tmask, lt_mask, lane, c0, v0, c1, v1);
      } else {
        const unsigned b0 = __ballot_sync(CLG_FULL, c0), b1 = __ballot_sync(CLG_FULL, c1);
        const unsigned kk = __popc(b0) + __popc(b1);
        if (MODE == kWalkWrite && kk) {
          const unsigned r0 = __popc(b0 & lt_mask) + __popc(b1 & lt_mask);
          if (c0) {
            const int64_t p = out_pos + r0;
            if (p < a.cap) a.pairs[p] = make_uint2(u32, v0); else atomicAdd(a.overflow, 1ull);
          }
          if (c1) {
            const int64_t p = out_pos + r0 + (c0 ? 1 : 0);
            if (p < a.cap) a.pairs[p] = make_uint2(u32, v1); else atomicAdd(a.overflow, 1ull);
          }
          out_pos += kk;
        }
        cnt += kk;
      }
    };
    // fold mode: deferred accepts are staged per warp in shared memory and
    // folded 32 at a time (one per lane)
    unsigned side_n = 0;
    auto side_push = [&](bool c0, uint32_t v0, bool c1, uint32_t v1) {
      const unsigned b0 = __ballot_sync(CLG_FULL, c0), b1 = __ballot_sync(CLG_FULL, c1);
      if ((b0 | b1) == 0u) return;
      const unsigned r0 = side_n + __popc(b0 & lt_mask) + __popc(b1 & lt_mask);
      if (c0) side[r0] = v0;
      if (c1) side[r0 + (c0 ? 1u : 0u)] = v1;
      side_n += __popc(b0) + __popc(b1);  // <= 31 + 64
      while (side_n >= 32) {
        __syncwarp();
        const uint32_t v = side[lane], vn = side[32 + lane], vm = side[64 + lane];
        __syncwarp();
        side[lane] = vn;  // keep the rest (< 64 entries)
        side[32 + lane] = vm;
        fs.emit2(a, u32, tmask, lt_mask, lane, true, v, false, 0u);
        side_n -= 32;
      }
    };
    auto side_flush = [&]() {
      if (side_n > 0) {  // < 32 entries left
        __syncwarp();
        const bool c = static_cast<unsigned>(lane) < side_n;
        const uint32_t v = side[lane];
        fs.emit2(a, u32, tmask, lt_mask, lane, c, v, false, 0u);
        side_n = 0;
      }
    };
    const uint32_t e_unit = fs.edges;

    if (j < vend && S > 0.0 && wu > 0.0) {
      int64_t vB = j, vsat = j;
      // bands only where the first pair is near or above pbar = 1/16 (the
      // multiply-only screen leaves a 0.1% margin to the exact test)
      if (!(wu * w[j] * a.invS < kBandTau * 0.999)) {
        const double y0 = pbar_of(wu, w[j], S);
        if (y0 >= kBandTau) {
          vB = first_p_below(w, wu, S, j, vend, kBandTau);
          vsat = y0 >= 1.0 ? first_p_below(w, wu, S, j, vB, 1.0) : j;
        }
      }
      // ---- saturated band: every position is an edge (cooperative) ----
      for (int64_t p0 = j; p0 < vsat; p0 += 32) {
        const int64_t v = p0 + lane;
        emit2(v < vsat, static_cast<uint32_t>(v), false, 0u);
      }
      // ---- heavy band [vsat, vB): per class a Bernoulli(pbar_k) process,
      // cooperatively: lane i draws a geometric gap, an integer warp prefix
      // sum places 32 candidates; a gap past the class end restarts at the
      // next class (memoryless) ----
      if (vsat < vB) {
        int64_t jj = vsat;
        int k = rec_of(s_rec, K, jj);
        while (jj < vB) {
          while (static_cast<int64_t>(s_rec[k + 1].s0) <= jj) ++k;
          const int64_t seg_hi = imin64(static_cast<int64_t>(s_rec[k + 1].s0), vB);
          const double wf = s_rec[k].wf;
          const double pb = fmin(pbar_of(wu, wf, S), 1.0);
          if (pb >= 1.0) {
            // envelope 1: every position is a candidate, accepted with q
            for (int64_t p0 = jj; p0 < seg_hi; p0 += 32) {
              const int64_t v = p0 + lane;
              bool acc = false;
              if (v < seg_hi) {
                const double q = pbar_of(wu, w[v], S);
                acc = q >= 1.0 || unit53(rng.next_plus()) < q;
              }
              emit2(acc, static_cast<uint32_t>(v), false, 0u);
            }
            jj = seg_hi;
          } else {
            const double imu = 1.0 / -log1p(-pb);  // geometric gap: floor(E / mu) + 1
            const double sure = g_sure[k];
            for (;;) {
              const double x = unit53(rng.next_plus()) + 0x1.0p-54;  // (0,1)
              const double ratio = -log(x) * imu;
              const int64_t gap = ratio < 4.0e18 ? static_cast<int64_t>(ratio) + 1 : (int64_t(1) << 62);
              const int64_t off = warp_inclusive_scan(gap);  // gaps >= 1: positions strictly increase
              const int64_t v = jj + off - 1;
              const bool valid = off <= seg_hi - jj;
              bool acc = false;
              if (valid) {
                const double r2 = unit53(rng.next_plus());
                acc = r2 < sure || r2 * wf < w[v];
              }
              emit2(acc, static_cast<uint32_t>(v), false, 0u);
              if (!__all_sync(CLG_FULL, valid)) break;
              jj = __shfl_sync(CLG_FULL, v, 31) + 1;
              if (jj >= seg_hi) break;
            }
            jj = seg_hi;
          }
          ++k;
        }
      }
      // ---- hazard envelope [vB, vend), cooperative rounds ----
      // Node ids are < 2^32 here (n <= 2^32 - 1, checked by set_weights).
      if (vB < vend) {
        int k = rec_of(s_rec, K, vB);
        const double ymax = wu * s_rec[k].wf * a.invS;  // any kappa >= -log(1-ymax)/ymax keeps the law
        if (ymax > 0.0) {
          // kappa = -log(1-y)/y = sum_k y^k/(k+1) (y < (1+eps)/16: 16 terms
          // leave < 1e-19); reciprocals by one rcp each
          double kappa = 1.0 / 17.0;
#pragma unroll
          for (int t = 16; t >= 1; --t) kappa = __fma_rn(kappa, ymax, 1.0 / static_cast<double>(t));
          const double inv_c = __drcp_rn(kappa * (wu * a.invS));
          if (lane == 0) {
            wc.c_u = kappa * (wu * a.invS);
            wc.inv_kappa = __drcp_rn(kappa);
          }
          __syncwarp();
          double T0 = s_rec[k].em + s_rec[k].wf * static_cast<double>(vB - static_cast<int64_t>(s_rec[k].s0));
          uint32_t prev_v = static_cast<uint32_t>(vB - 1);
          const uint32_t vend32 = static_cast<uint32_t>(vend);
          // Acceptance of a candidate in class k: R < (w_v / wfirst_k) g_k,
          // g_k = (1/kappa) z/(1-e^-z), z = c_u wfirst_k.  Lane i of the
          // window holds class kw + i: g_k and the sure threshold
          // hs_k = floor(sure_k g_k 2^11) (R < hs_k / 2^11 accepts without
          // reading w_v; R's top 11 bits come with the event's draw).
          int kw = k;
          double g_lane = 0.0;
          uint32_t hs_lane = 0;
          auto refresh = [&]() {
            const int kc = kw + lane;
            if (kc < K) {
              g_lane = bern_gk(wc.inv_kappa, wc.c_u * s_rec[kc].wf);
              hs_lane = static_cast<uint32_t>((__ldg(g_sure + kc) * g_lane) * 2048.0);
            } else {
              g_lane = 0.0;
              hs_lane = 0;
            }
          };
          refresh();
          // count/fold modes resolve an uncertain accept one round later (its
          // w[v] load overlaps the next round); the ordered write pass cannot
          constexpr bool kDefer = MODE != kWalkWrite;
          // one deferred candidate per lane: (position, acceptance bits | event b flag << 16, factor, weight)
          bool pend = false;
          uint32_t pv = 0, ph = 0;
          double pf = 0.0, pw = 0.0;
          uint32_t ev = 0;  // this lane's event serial (2 per round)
          // class of T: bucket lower bound, then at most seg.depth forward
          // steps (two branch-free compares when the table guarantees depth <= 2)
          const bool shallow = a.seg.depth <= 2;
          auto class_of = [&](double T) -> int {
            const double bt = T * a.seg.inv_bucket;
            int kl = s_bucket[bt < static_cast<double>(NB - 1) ? static_cast<int>(bt) : NB - 1];
            if (shallow) {
              const bool c1 = !(T < s_rec[kl + 1].em), c2 = !(T < s_rec[kl + 2].em);
              kl += (c1 ? 1 : 0) + (c2 ? 1 : 0);
            } else {
              while (kl < K && !(T < s_rec[kl + 1].em)) ++kl;
            }
            return kl;
          };
          for (;;) {
            const bool accp = kDefer && pend && lazy_accept_w(ph & 0xffffu, pw * pf, wc, lane, ev - 2 + (ph >> 16));
            const uint32_t pvv = pv;
            pend = false;
            const uint64_t xa = rng.next(), xb = rng.next();
            const double Ea = exp_bits(xa, s_log);
            const double Eb = exp_bits(xb, s_log);
            const uint32_t ha = static_cast<uint32_t>(xa) & 2047u, hb = static_cast<uint32_t>(xb) & 2047u;
            const double incl = warp_incl_scan_f64(Ea + Eb);
            const double Ta = T0 + (incl - Eb) * inv_c;
            const double Tb = T0 + incl * inv_c;
            const int kla = class_of(Ta);
            const int klb = class_of(Tb);
            const double2 eia = *reinterpret_cast<const double2*>(&s_rec[kla].em);
            const uint2 sa = *reinterpret_cast<const uint2*>(&s_rec[kla].s0);
            const double2 eib = *reinterpret_cast<const double2*>(&s_rec[klb].em);
            const uint2 sb = *reinterpret_cast<const uint2*>(&s_rec[klb].s0);
            uint32_t va = sa.x + static_cast<uint32_t>(fmax(Ta - eia.x, 0.0) * eia.y);
            va = va > sa.y - 1 ? sa.y - 1 : va;
            uint32_t vb = sb.x + static_cast<uint32_t>(fmax(Tb - eib.x, 0.0) * eib.y);
            vb = vb > sb.y - 1 ? sb.y - 1 : vb;
            const bool valida = Ta < a.seg.em_end && va < vend32;
            const bool validb = Tb < a.seg.em_end && vb < vend32;
            uint32_t vp = __shfl_up_sync(CLG_FULL, vb, 1);
            if (lane == 0) vp = prev_v;
            const bool propa = valida && va > vp;
            const bool propb = validb && vb > va;
            const int dia = kla - kw, dib = klb - kw;
            uint32_t hsa = __shfl_sync(CLG_FULL, hs_lane, dia & 31);
            uint32_t hsb = __shfl_sync(CLG_FULL, hs_lane, dib & 31);
            const bool acca = propa && ha < hsa && dia < 32;
            const bool accb = propb && hb < hsb && dib < 32;
            // uncertain (or outside the window): acceptance factor f = g_k / wfirst_k
            const bool unca = propa && !acca, uncb = propb && !accb;
            bool acca2 = false, accb2 = false;
            if (__any_sync(CLG_FULL, unca || uncb)) {
              double ga = __shfl_sync(CLG_FULL, g_lane, dia & 31);
              double gb = __shfl_sync(CLG_FULL, g_lane, dib & 31);
              if (unca) {
                if (dia >= 32) {
                  ga = bern_gk(wc.inv_kappa, wc.c_u * s_rec[kla].wf);
                  hsa = static_cast<uint32_t>((__ldg(g_sure + kla) * ga) * 2048.0);
                }
                if (ha < hsa) {
                  acca2 = true;
                } else {
                  const double f = ga * eia.y;
                  if (kDefer) {
                    pend = true;
                    pv = va;
                    ph = ha;
                    pf = f;
                    pw = w[va];  // consumed next round
                  } else {
                    acca2 = lazy_accept_w(ha, w[va] * f, wc, lane, ev);
                  }
                }
              }
              if (uncb) {
                if (dib >= 32) {
                  gb = bern_gk(wc.inv_kappa, wc.c_u * s_rec[klb].wf);
                  hsb = static_cast<uint32_t>((__ldg(g_sure + klb) * gb) * 2048.0);
                }
                if (hb < hsb) {
                  accb2 = true;
                } else {
                  const double f = gb * eib.y;
                  if (kDefer && !pend) {
                    pend = true;
                    pv = vb;
                    ph = hb | (1u << 16);
                    pf = f;
                    pw = w[vb];
                  } else {  // write mode, or a second uncertain event this round (rare): decide now
                    accb2 = lazy_accept_w(hb, w[vb] * f, wc, lane, ev + 1);
                  }
                }
              }
            }
            ev += 2;
            if (MODE == kWalkFold) side_push(accp, pvv, false, 0u);
            else if (MODE == kWalkCount) emit2(accp, pvv, false, 0u);
            emit2(acca || acca2, va, accb || accb2, vb);
            // carry the last lane's second event into the next round
            if (!__all_sync(CLG_FULL, validb)) {
              if (kDefer) {
                const bool lp = pend && lazy_accept_w(ph & 0xffffu, pw * pf, wc, lane, ev - 2 + (ph >> 16));
                if (MODE == kWalkFold) side_push(lp, pv, false, 0u);
                else emit2(lp, pv, false, 0u);
              }
              break;
            }
            T0 = __shfl_sync(CLG_FULL, Tb, 31);
            k = __shfl_sync(CLG_FULL, klb, 31);
            prev_v = __shfl_sync(CLG_FULL, vb, 31);
            if (k - kw >= kWinRefresh) {
              kw = k;
              refresh();
            }
          }
        }
      }
    }
    if (MODE == kWalkCount && lane == 0) a.counts[unit] = cnt;
    if (MODE == kWalkFold) {
      side_flush();
      if (a.degree && (u & ((1ll << a.track_shift) - 1)) == 0) {  // tracked source: its out-edges of this unit
        const uint64_t d = warp_sum_u64(static_cast<uint64_t>(fs.edges - e_unit));
        if (lane == 0 && d) atomicAdd(&a.degree[u >> a.track_shift], static_cast<uint32_t>(d));
      }
    }
  }

  if (a.prof.slots && lane == 0) {
    const int g = a.prof.gw();
    a.prof.slots[2 * g] = t_start;
    a.prof.slots[2 * g + 1] = globaltimer_ns();
  }
  if (MODE == kWalkFold) fs.finish(a, lane);
}

// ---- light units: one lane per unit ----------------------------------------
// Each lane walks one unit's hazard process sequentially (kLaneEvents events
// per loop iteration); idle lanes are refilled from a warp-local batch of the
// unit queue.  Same envelope, acceptance and lazy 11-bit acceptance bits as
// the warp kernel; every draw comes from the unit's own stream, in event
// order, so the count, write and fold modes make identical decisions.
#ifndef CLG_LANE_EVENTS
#define CLG_LANE_EVENTS 4
#endif
constexpr int kLaneEvents = CLG_LANE_EVENTS;  // hazard events per lane iteration (light units)

// lazy_accept with the unit stream key derived from (seed, u) only when the
// 11 bits cannot decide (light units keep no key register)
__device__ __forceinline__ bool lazy_accept_u(uint32_t h, double a, uint64_t seed_mix, uint32_t u, uint32_t id) {
  const double s = a * 2048.0;
  if (static_cast<double>(h + 1u) <= s) return true;
  if (static_cast<double>(h) >= s) return false;
  return lazy_accept(h, a, unit_key(seed_mix, u, 0), id);
}

// Dynamic shared memory of the light-unit kernel: K+2 class records, the log
// table, the bucket index, the float sure bounds and the per-warp staging of
// deferred accepts (u, v).
__host__ __device__ inline size_t ctr_walk_smem_bytes(int K, int nb) {
  return static_cast<size_t>(K + 2) * sizeof(ClassRec) + sizeof(LogTable) +
         ((static_cast<size_t>(nb) * sizeof(unsigned short) + 15) & ~size_t(15)) +
         ((static_cast<size_t>(K) * sizeof(float) + 15) & ~size_t(15)) + (256 / 32) * 64 * sizeof(uint2);
}

template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) ctr_walk_kernel(CtrWalkArgs a, const int64_t* __restrict__ split_pos,
                                                          const LogTable* __restrict__ logtab, uint64_t seed_mix) {
  constexpr int64_t kBatch = 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.seg.K;
  ClassRec* s_rec = reinterpret_cast<ClassRec*>(smem_raw);
  LogTable& s_log = *reinterpret_cast<LogTable*>(smem_raw + static_cast<size_t>(K + 2) * sizeof(ClassRec));
  unsigned short* s_bucket = reinterpret_cast<unsigned short*>(reinterpret_cast<unsigned char*>(&s_log) + sizeof(LogTable));
  float* s_suref = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(s_bucket) +
                                            ((static_cast<size_t>(a.seg.nb) * sizeof(unsigned short) + 15) & ~size_t(15)));
  uint2 (*s_side)[64] = reinterpret_cast<uint2 (*)[64]>(reinterpret_cast<unsigned char*>(s_suref) +
                                                        ((static_cast<size_t>(K) * sizeof(float) + 15) & ~size_t(15)));
  for (int i = threadIdx.x; i < K; i += blockDim.x) s_suref[i] = __double2float_rd(a.seg.sure[i]);
  for (int i = threadIdx.x; i <= K; i += blockDim.x) {
    ClassRec r;
    r.em = a.seg.em[i];
    r.iwf = i < K ? a.seg.invwf[i] : 0.0;
    r.s0 = static_cast<uint32_t>(a.seg.start[i]);
    r.s1 = i < K ? static_cast<uint32_t>(a.seg.start[i + 1]) : r.s0;
    r.wf = i < K ? a.seg.wfirst[i] : 0.0;
    s_rec[i] = r;
    if (i == K) {
      r.em = __longlong_as_double(0x7ff0000000000000LL);
      r.iwf = 0.0;
      r.wf = 0.0;
      s_rec[K + 1] = r;
    }
  }
  for (int i = threadIdx.x; i < kLogTable; i += blockDim.x) {
    s_log.inv_c[i] = logtab->inv_c[i];
    s_log.nlog_inv[i] = logtab->nlog_inv[i];
  }
  const int NB = a.seg.nb;
  for (int i = threadIdx.x; i < NB; i += blockDim.x) s_bucket[i] = a.seg.bucket[i];
  __syncthreads();
  const bool shallow = a.seg.depth <= 2;

  const int lane = lane_id();
  const unsigned lt_mask = lanemask_lt();
  uint2* side = s_side[threadIdx.x >> 5];
  unsigned side_n = 0;
  const unsigned long long t_start = a.prof.slots ? globaltimer_ns() : 0ull;
  const double* __restrict__ w = a.w;
  const double S = a.S;
  const uint32_t tmask = (1u << a.track_shift) - 1u;
  FoldSink fs;
  fs.init(a);

  int64_t b_next = 0, b_end = 0;
  bool drained = false;

  // lane state (light units are plain sources whose hazard envelope starts
  // at u+1: the host routes hubs and sources with a pbar >= 1/16 band to the
  // warp kernel)
  constexpr uint32_t kIdle = 0xffffffffu;
  uint32_t u = kIdle;  // the lane's source (kIdle: none); its unit is u - lo - H + hub_units
  int64_t out_pos = 0;
  int k = 0;
  int32_t cnt = 0;
  uint32_t ev = 0;  // event serial of the unit's hazard process
  // proposals form a Poisson process of rate c_u * wfirst[k] per position,
  // i.e. unit rate in T = c_u * (envelope mass); T is tracked in
  // envelope-mass units (divided by c_u).
  double T = 0.0, inv_c = 0.0, c_u = 0.0, inv_kappa = 0.0;
  // hs = floor(sure_k (2^11 / kappa) (1 - 2^-40)) <= floor(sure_k g_k 2^11)
  // (g_k >= 1/kappa): R < hs/2^11 accepts without w[v] and without g_k
  uint32_t hs = 0;
  uint32_t prev_v = 0;
  bool done = true;  // the lane's unit has no events left
  // software-pipelined accept: an uncertain candidate's weight is loaded in
  // one iteration and compared in the next, so the warp never waits on it
  bool pend = false;
  uint32_t pend_v = 0, pend_h = 0;  // pend_h: acceptance bits | event id << 11
  double pend_f = 0.0, pend_w = 0.0;
  Xoro128 rng;

  auto set_class = [&](int kn) {
    k = kn;
    hs = kn < K ? static_cast<uint32_t>(static_cast<double>(s_suref[kn]) * ((2048.0 * inv_kappa) * (1.0 - 0x1.0p-40)))
                : 0u;
  };
  auto class_of = [&](double t) -> int {
    const double bt = t * a.seg.inv_bucket;
    int kl = s_bucket[bt < static_cast<double>(NB - 1) ? static_cast<int>(bt) : NB - 1];
    if (shallow) {
      const bool c1 = !(t < s_rec[kl + 1].em), c2 = !(t < s_rec[kl + 2].em);
      kl += (c1 ? 1 : 0) + (c2 ? 1 : 0);
    } else {
      while (kl < K && !(t < s_rec[kl + 1].em)) ++kl;
    }
    return kl;
  };
  // fold mode: stage the deferred accept of this iteration; fold 32 at a time
  auto side_push = [&](bool c, uint32_t uu, uint32_t vv) {
    const unsigned b = __ballot_sync(CLG_FULL, c);
    if (b == 0u) return;
    if (c) side[side_n + __popc(b & lt_mask)] = make_uint2(uu, vv);
    side_n += __popc(b);
    if (side_n >= 32) {
      __syncwarp();
      const uint2 e = side[lane], en = side[32 + lane];
      __syncwarp();
      side[lane] = en;
      fs.emit2(a, e.x, tmask, lt_mask, lane, true, e.y, false, 0u);
      side_n -= 32;
    }
  };
  const int64_t hub_units = a.H > 0 ? a.hub_units[a.H] : 0;

  for (;;) {
    const unsigned need = __ballot_sync(CLG_FULL, u == kIdle);
    if (need && !drained && (__popc(need) >= a.refill_min || need == CLG_FULL)) {
      const int want = __popc(need);
      const int r = __popc(need & lt_mask);
      const bool me = (need >> lane) & 1u;
      int64_t mine = -1;
      const int64_t take1 = imin64(b_end - b_next, want);
      if (me && r < take1) mine = b_next + r;
      b_next += take1;
      if (want > take1) {
        unsigned long long g = 0;
        if (lane == 0) g = atomicAdd(a.queue, (unsigned long long)kBatch);
        g = __shfl_sync(CLG_FULL, g, 0);
        if (static_cast<int64_t>(g) >= a.total_units) {
          drained = true;
          b_next = b_end = a.total_units;
        } else {
          b_next = static_cast<int64_t>(g);
          b_end = imin64(b_next + kBatch, a.total_units);
          const int64_t take2 = imin64(b_end - b_next, want - take1);
          if (me && r >= take1 && r - take1 < take2) mine = b_next + (r - take1);
          b_next += take2;
        }
      }
      if (mine >= 0) {
        u = static_cast<uint32_t>(a.lo + a.H + (mine - hub_units));
        cnt = 0;
        ev = 0;
        done = true;
        if (MODE == kWalkWrite) out_pos = a.offsets[mine];
        const double wu = w[u];
        rng.seed_key(unit_key(seed_mix, u, 0));
        const int64_t j = static_cast<int64_t>(u) + 1;
        if (mine < hub_units || (j < a.n && !(wu * w[j] * a.invS < kBandTau * 0.999))) {
          atomicAdd(a.overflow, 1ull << 40);  // plan violation: not a light unit (reported as an error)
        } else if (j < a.n && S > 0.0 && wu > 0.0) {
          const int kb = rec_of(s_rec, K, j);
          // kappa = -log(1-ymax)/ymax from the largest envelope used
          const double ymax = wu * s_rec[kb].wf * a.invS;
          if (ymax > 0.0) {
            double kappa = 1.0 / 17.0;  // -log(1-y)/y, 16 series terms (y < 1/8)
#pragma unroll
            for (int t = 16; t >= 1; --t) kappa = __fma_rn(kappa, ymax, 1.0 / static_cast<double>(t));
            c_u = kappa * (wu * a.invS);
            inv_c = __drcp_rn(c_u);
            inv_kappa = __drcp_rn(kappa);
            T = s_rec[kb].em + s_rec[kb].wf * static_cast<double>(j - static_cast<int64_t>(s_rec[kb].s0));
            prev_v = static_cast<uint32_t>(u);
            set_class(kb);
            done = false;
          }
        }
      }
    }
    const unsigned live = __ballot_sync(CLG_FULL, u != kIdle);
    if (!live) {
      if (drained) break;
      continue;
    }

    bool acc[kLaneEvents];
    uint32_t vv[kLaneEvents];
#pragma unroll
    for (int e = 0; e < kLaneEvents; ++e) {
      acc[e] = false;
      vv[e] = 0;
    }
    bool finish = false;
    // resolve the candidate whose weight was requested last iteration
    const bool acc_prev = pend && lazy_accept_u(pend_h & 2047u, pend_w * pend_f, seed_mix, u, pend_h >> 11);
    const uint32_t v_prev = pend_v;
    pend = false;
    bool pend_new = false;
    int pend_slot = -1;
    uint32_t pv_new = 0, ph_new = 0, pid_new = 0;
    double pf_new = 0.0;
    if (u != kIdle) {
      if (done) {
        finish = true;
      } else {
        // ---- hazard envelope: kLaneEvents events per iteration -----------
#pragma unroll
        for (int e = 0; e < kLaneEvents; ++e) {
          if (finish) break;
          const uint64_t x = rng.next();
          T += exp_bits(x, s_log) * inv_c;
          const uint32_t h = static_cast<uint32_t>(x) & 2047u;
          const uint32_t id = ev++;
          if (!(T < s_rec[k + 1].em)) {
            if (!(T < a.seg.em_end)) finish = true;
            else set_class(class_of(T));
          }
          if (!finish) {
            const ClassRec& rc = s_rec[k];
            uint32_t v_e = rc.s0 + static_cast<uint32_t>(fmax(T - rc.em, 0.0) * rc.iwf);
            v_e = v_e > rc.s1 - 1 ? rc.s1 - 1 : v_e;
            if (v_e > prev_v) {  // a position proposed once however many events hit it
              prev_v = v_e;
              vv[e] = v_e;
              if (h < hs) {
                acc[e] = true;
              } else {
                const double fk = bern_gk(inv_kappa, c_u * rc.wf) * rc.iwf;  // g_k / wfirst_k
                if (!pend_new) {
                  pend_new = true;
                  pend_slot = e;
                  pv_new = v_e;
                  ph_new = h;
                  pid_new = id;
                  pf_new = fk;
                } else {  // second uncertain candidate of the iteration (rare): decide now
                  acc[e] = lazy_accept_u(h, w[v_e] * fk, seed_mix, u, id);
                }
              }
            }
          }
          // the write pass keeps each unit's edges in position order: an
          // undecided event (emitted next iteration) ends this iteration
          if (MODE == kWalkWrite && pend_new) break;
        }
        // the unit ends this iteration: an outstanding candidate must be
        // decided before the lane moves on to another unit
        if (finish && pend_new) {
          const bool acc_p = lazy_accept_u(ph_new, w[pv_new] * pf_new, seed_mix, u, pid_new);
#pragma unroll
          for (int e = 0; e < kLaneEvents; ++e)
            if (e == pend_slot) acc[e] = acc_p;
          pend_new = false;
        }
      }
    }

    // a new uncertain candidate: request its weight now, decide next iteration
    // (the unit cannot finish before that: finishing draws no candidate)
    if (pend_new) {
      pend = true;
      pend_v = pv_new;
      pend_h = ph_new | (pid_new << 11);
      pend_f = pf_new;
      pend_w = w[pv_new];
    }
    // emission: the previous iteration's deferred accept, then this iteration's
    cnt += (acc_prev ? 1 : 0);
#pragma unroll
    for (int e = 0; e < kLaneEvents; ++e) cnt += acc[e] ? 1 : 0;
    const uint32_t u32 = static_cast<uint32_t>(u);
    if (MODE == kWalkWrite) {
      if (acc_prev) {
        if (out_pos < a.cap) a.pairs[out_pos] = make_uint2(u32, v_prev); else atomicAdd(a.overflow, 1ull);
        ++out_pos;
      }
#pragma unroll
      for (int e = 0; e < kLaneEvents; ++e) {
        if (acc[e]) {
          if (out_pos < a.cap) a.pairs[out_pos] = make_uint2(u32, vv[e]); else atomicAdd(a.overflow, 1ull);
          ++out_pos;
        }
      }
    } else if (MODE == kWalkFold) {
      side_push(acc_prev, u32, v_prev);
#pragma unroll
      for (int e = 0; e + 1 < kLaneEvents; e += 2)
        fs.emit2(a, u32, tmask, lt_mask, lane, acc[e], vv[e], acc[e + 1], vv[e + 1]);
      if (kLaneEvents & 1)
        fs.emit2(a, u32, tmask, lt_mask, lane, acc[kLaneEvents - 1], vv[kLaneEvents - 1], false, 0u);
    }
    if (u != kIdle && finish) {
      if (MODE == kWalkCount) a.counts[static_cast<int64_t>(u) - a.lo - a.H + hub_units] = cnt;
      if (MODE == kWalkFold && a.degree && (static_cast<int64_t>(u) & ((1ll << a.track_shift) - 1)) == 0 && cnt)
        atomicAdd(&a.degree[static_cast<int64_t>(u) >> a.track_shift], static_cast<uint32_t>(cnt));
      u = kIdle;
    }
  }

  if (MODE == kWalkFold && side_n > 0) {  // < 32 staged accepts left
    __syncwarp();
    const bool c = static_cast<unsigned>(lane) < side_n;
    const uint2 e = side[lane];
    fs.emit2(a, e.x, tmask, lt_mask, lane, c, e.y, false, 0u);
  }
  if (a.prof.slots && lane == 0) {
    const int g = a.prof.gw();
    a.prof.slots[2 * g] = t_start;
    a.prof.slots[2 * g + 1] = globaltimer_ns();
  }
  if (MODE == kWalkFold) fs.finish(a, lane);
}

// Envelope-expected candidate count of source u over [u+1, n), in closed
// form from the envelope-mass prefix (O(log K) per source): positions in
// classes with w_u wfirst_k / S >= 1 (a prefix of the classes) count 1 each,
// the rest (w_u / S) x envelope mass.  The hub split plan and the heavy/light
// choice use it; both are functions of the weights only.
struct HubExpect {
  double sat;    // saturated positions in [u+1, n)
  double scale;  // w_u / S
  double Ta;     // envelope coordinate where the unsaturated part starts
  int64_t a;     // first unsaturated position (>= u+1)
  double E;      // total expected candidates
};

// envelope coordinate of node p in [0, n]: em[k] + wfirst_k (p - start_k)
__device__ __forceinline__ double env_coord(const Segments& seg, int64_t p) {
  if (p >= seg.start[seg.K]) return seg.em[seg.K];
  const int k = seg_of(seg, p);
  return seg.em[k] + seg.wfirst[k] * static_cast<double>(p - seg.start[k]);
}

__device__ __forceinline__ HubExpect hub_expect(const Segments& seg, double wu, int64_t u, double S) {
  HubExpect h{0.0, 0.0, 0.0, u + 1, 0.0};
  const int64_t n = seg.start[seg.K];
  if (u + 1 >= n || !(wu > 0.0) || !(S > 0.0)) return h;
  int lo = -1, hi = seg.K;  // first class with pbar < 1 in (lo, hi]
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (pbar_of(wu, seg.wfirst[m], S) < 1.0) hi = m; else lo = m;
  }
  const int64_t sks = seg.start[hi];
  h.a = sks > u + 1 ? sks : u + 1;
  h.sat = static_cast<double>(h.a - (u + 1));
  h.scale = wu / S;
  h.Ta = env_coord(seg, h.a);
  h.E = h.sat + h.scale * (seg.em[seg.K] - h.Ta);
  return h;
}

// first position p >= u+1 where the expected count over [u+1, p) reaches t
__device__ __forceinline__ int64_t hub_position(const Segments& seg, const HubExpect& h, int64_t u, double t) {
  const int64_t n = seg.start[seg.K];
  if (t <= h.sat) {
    const int64_t p = u + 1 + static_cast<int64_t>(t);
    return p < h.a ? p : h.a;
  }
  const double T = h.Ta + (t - h.sat) / h.scale;
  if (!(T < seg.em[seg.K])) return n;
  int lo = 0, hi = seg.K;  // em[lo] <= T < em[hi]
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (seg.em[m] <= T) lo = m; else hi = m;
  }
  const double wf = seg.wfirst[lo];
  int64_t p = seg.start[lo] + (wf > 0.0 ? static_cast<int64_t>((T - seg.em[lo]) / wf) : 0);
  if (p > seg.start[lo + 1]) p = seg.start[lo + 1];
  if (p < h.a) p = h.a;
  return p;
}

__device__ __forceinline__ double expected_candidates(const double* __restrict__ w, int64_t n, double S,
                                                      const Segments& seg, const double* __restrict__ seg_mass,
                                                      int64_t u) {
  (void)n;
  (void)seg_mass;
  return hub_expect(seg, w[u], u, S).E;
}

// out[i] = expected_candidates(us[i])
__global__ void expected_candidates_kernel(const double* __restrict__ w, int64_t n, double S, Segments seg,
                                           const double* __restrict__ seg_mass, int64_t lo, int64_t hi, int m,
                                           double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t u = lo + (hi - lo) * static_cast<int64_t>(i) / m;
  out[i] = expected_candidates(w, n, S, seg, seg_mass, u);
}

// ---- segment table -------------------------------------------------------
// Classes on a geometric grid anchored at w[0]: thresholds t_k = w[0] /
// (1+eps)^k (t_0 = +inf); class k holds the positive weights in
// [t_{k+1}, t_k), so w[c_k] < (1+eps) w[c_{k+1}-1] holds by construction;
// empty grid cells are dropped and zero weights form one last class.  Every
// boundary is an independent binary search (one thread per grid cell), so
// the table costs ~log2(n) dependent loads instead of a sequential walk.
__global__ void grid_bounds_kernel(const double* __restrict__ w, int64_t z, const double* __restrict__ thr, int kg,
                                   int64_t* bounds) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > kg) return;
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

// Compact the non-empty grid cells into classes (one thread; kg <= a few
// thousand) and append the zero class [z, n); K_out = number of classes.
__global__ void grid_compact_kernel(const double* __restrict__ w, int64_t n, int64_t z,
                                    const int64_t* __restrict__ bounds, int kg, int kmax, int64_t* start,
                                    double* wfirst, double* sure, int* K_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int K = 0;
  for (int k = 0; k < kg; ++k) {
    const int64_t a = bounds[k], b = bounds[k + 1];
    if (b <= a) continue;
    if (K >= kmax) { *K_out = -1; return; }
    start[K] = a;
    wfirst[K] = w[a];
    sure[K] = w[b - 1] / w[a];
    ++K;
  }
  if (z < n) {
    if (K >= kmax) { *K_out = -1; return; }
    start[K] = z;
    wfirst[K] = 0.0;
    sure[K] = 1.0;
    ++K;
  }
  start[K] = n;
  *K_out = K;
}

// Hub split plan: for source u in [lo, lo+Hmax) the expected candidate count
// over [u+1, n) under the class envelope; split count = ceil(E / cap).
__global__ void hub_splits_kernel(const double* __restrict__ w, int64_t n, double S, int64_t lo, int64_t Hmax,
                                  Segments seg, const double* __restrict__ seg_mass, double cap,
                                  int64_t* splits) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < Hmax; i += stride) {
    const double E = expected_candidates(w, n, S, seg, seg_mass, lo + i);
    const double s = ceil(E / cap);
    splits[i] = s < 1.0 ? 1 : static_cast<int64_t>(s);
  }
}

// Split positions of every hub unit: split s of hub u covers
// [pos(s), pos(s+1)) with pos chosen so each share carries E/splits expected
// candidates (closed form, positions interpolated inside a class).
__global__ void hub_positions_kernel(const double* __restrict__ w, int64_t n, double S, int64_t lo, int64_t H,
                                     Segments seg, const double* __restrict__ seg_mass,
                                     const int64_t* __restrict__ hub_units, int64_t* pos) {
  (void)seg_mass;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += stride) {
    const int64_t u = lo + i;
    const int64_t u0 = hub_units[i], ns = hub_units[i + 1] - u0;
    const HubExpect h = hub_expect(seg, w[u], u, S);
    int64_t prev = u + 1;
    pos[u0] = prev;
    for (int64_t s = 1; s < ns; ++s) {
      int64_t p = hub_position(seg, h, u, h.E * static_cast<double>(s) / static_cast<double>(ns));
      if (p < prev) p = prev;
      if (p > n) p = n;
      pos[u0 + s] = p;
      prev = p;
    }
  }
}

// Envelope-mass prefix em[k], 1/wfirst and the per-class envelope mass
// seg_mass[k] = wfirst[k] * len_k (one thread; K is small).  The hub plan
// balances splits on envelope mass: the samplers' work is proportional to
// proposals, i.e. to envelope mass, and no pass over w is needed.
__global__ void segment_envelope_kernel(Segments seg, double* em, double* invwf, double* seg_mass) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (int k = 0; k < seg.K; ++k) {
    em[k] = acc;
    const double wf = seg.wfirst[k];
    const double m = wf * static_cast<double>(seg.start[k + 1] - seg.start[k]);
    seg_mass[k] = m;
    acc += m;
    invwf[k] = wf > 0.0 ? 1.0 / wf : 0.0;
  }
  em[seg.K] = acc;
}

// bucket[b] = class holding envelope mass just below b * em[K] / kBuckets (a
// lower bound of the class of any T the lookup maps to bucket b, robust to
// the rounding of T * kBuckets / em[K]); depth_out = max over b of the number
// of class boundaries up to just above the bucket end.
__device__ __forceinline__ int class_at(const Segments& seg, double x) {
  int lo = 0, hi = seg.K;  // em[lo] <= x < em[hi] (or hi = K)
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (seg.em[m] <= x) lo = m; else hi = m;
  }
  return lo;
}

__global__ void segment_buckets_kernel(Segments seg, unsigned short* bucket, int* depth_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= seg.nb) return;
  const double E = seg.em[seg.K];
  const double x0 = E * (static_cast<double>(b) / seg.nb), x1 = E * (static_cast<double>(b + 1) / seg.nb);
  const int lo = class_at(seg, x0 - E * 0x1.0p-40);
  const int hi = class_at(seg, x1 + E * 0x1.0p-40);
  bucket[b] = static_cast<unsigned short>(lo);
  atomicMax(depth_out, hi - lo);
}

// First source u in [lo,hi) whose hazard envelope starts at u+1, i.e. that
// passes the light kernel's band screen (u+1 >= n or w[u] w[u+1] / S below
// 1/16 with the 0.1% margin); hi if none.  The predicate is monotone in u
// (w non-increasing).  One warp.
__global__ void first_pure_hazard_kernel(const double* __restrict__ w, int64_t n, int64_t lo0, int64_t hi0,
                                         double invS, long long* out) {
  const int lane = threadIdx.x;
  auto pure = [&](int64_t u) { return u + 1 >= n || w[u] * w[u + 1] * invS < kBandTau * 0.999; };
  int64_t lo = lo0 - 1, hi = hi0;  // answer in (lo, hi]
  while (hi - lo > 1) {
    const int64_t span = hi - lo - 1;
    const int64_t step = (span + 31) / 32;
    const int64_t p = lo + 1 + static_cast<int64_t>(lane) * step;
    const bool ok = p >= hi || pure(p);
    const unsigned m = __ballot_sync(CLG_FULL, ok);
    if (m == 0) {
      lo = lo + 1 + 31 * step;
      continue;
    }
    const int f = __ffs(m) - 1;
    const int64_t pf = lo + 1 + static_cast<int64_t>(f) * step;
    const int64_t nlo = f > 0 ? lo + 1 + static_cast<int64_t>(f - 1) * step : lo;
    hi = pf < hi ? pf : hi;
    lo = nlo;
  }
  if (lane == 0) *out = hi;
}

// First index in [lo,hi) with w < lim (hi if none); w non-increasing.  One warp.
__global__ void first_below_kernel(const double* __restrict__ w, int64_t lo0, int64_t hi0, double lim,
                                   long long* out) {
  const int lane = threadIdx.x;
  int64_t lo = lo0 - 1, hi = hi0;  // answer in (lo, hi]
  while (hi - lo > 1) {
    const int64_t span = hi - lo - 1;
    const int64_t step = (span + 31) / 32;
    const int64_t p = lo + 1 + static_cast<int64_t>(lane) * step;
    const bool below = p >= hi || w[p] < lim;
    const unsigned m = __ballot_sync(CLG_FULL, below);
    if (m == 0) {
      lo = lo + 1 + 31 * step;
      continue;
    }
    const int f = __ffs(m) - 1;
    const int64_t pf = lo + 1 + static_cast<int64_t>(f) * step;
    const int64_t nlo = f > 0 ? lo + 1 + static_cast<int64_t>(f - 1) * step : lo;
    hi = pf < hi ? pf : hi;
    lo = nlo;
  }
  if (lane == 0) *out = hi;
}

}  // namespace clg
