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
//    floor(E2 / -log2(1-pbar)) + 1, E2 = -log2 U — each thinned with probability
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
// Per iteration every lane draws E gaps for its own 1/32 of the chunk's
// positions (independent chains: no warp scan, no cross-lane dependence),
// decodes (row, col) = (position / nb, position % nb) with one FMA rounded
// down and a 32-bit integer residual, and emits accepted pairs through a
// per-warp shared-memory stage flushed as 16-byte vector stores (ring / fold
// mode) — the level-2 balance is the uniform chunk size: a hub's v-range is
// spread over as many blocks and chunks as its expected edge count needs.
#pragma once

#include "common.cuh"
#include "fastmath.cuh"
#include "sampler_ref.cuh"

#include <type_traits>

namespace clg {

constexpr int kClassCap = 1024;                 // classes (incl. the zero class)
constexpr int64_t kClassMaxNodes = (1ll << 26) - 64;  // nodes per class (block positions < 2^52 - 2^27)
constexpr uint32_t kBlkDiag = 1u, kBlkDense = 2u;

struct __align__(16) BlockDesc {
  double pbar;      // RN(RN(w[s_A] w[s_B]) / S): envelope (>= every p_uv of the block)
  double inv_mu;    // 1 / -log2(1 - pbar) (sparse blocks)
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

struct Log2Table;

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
  const Log2Table* logtab;
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

// E2 = -log2(U) ~ Exp(ln 2) by inversion, U = ((x >> 12) + 1/2) 2^-52 in (0,1)
// from the top 52 bits of x: y = U 2^52 is built from bits (no int->fp
// conversion), log2 y = exponent + table log2 of the reciprocal centre + a
// degree-5 log1p series on |t| <= 2^-8 (truncation < 2^-50; statistically
// exact).  Table entry i = {RN(1/c_i), -log2 RN(1/c_i)}, c_i = 1 + (i + 1/2)/128,
// replicated 8 times in shared memory (row i = 128 bytes, copy lane & 7) so a
// 16-byte lookup never meets a bank conflict: the 8 lanes of one LDS.128
// phase read 8 different bank groups whatever their indices.
struct Log2Table {
  double inv_c[kLogTable];
  double nlog2_inv[kLogTable];
};
constexpr int kTabCopies = 8;
constexpr size_t kTabBytes = static_cast<size_t>(kLogTable) * kTabCopies * sizeof(double2);
// log2(e) * {1, -1/2, 1/3, -1/4, 1/5}: constant-bank operands of the series FMAs
__constant__ double kLog2Series[5] = {0x1.71547652b82fep+0, -0x1.71547652b82fep-1, 0x1.ec709dc3a03fdp-2,
                                      -0x1.71547652b82fep-2, 0x1.2776c50ef9bfep-2};

__device__ __forceinline__ double exp52_y(uint64_t x) {  // (x >> 12) + 1/2, exact
  return __longlong_as_double(static_cast<long long>((x >> 12) | 0x4330000000000000ull)) - (0x1.0p52 - 0.5);
}
// tab_lane = table base + 16 * (lane & 7) (bytes)
__device__ __forceinline__ double exp2_52(uint64_t x, const unsigned char* tab_lane) {
  const double y = exp52_y(x);
  const int yh = __double2hiint(y);
  const double2 tc = *reinterpret_cast<const double2*>(tab_lane + ((yh >> 6) & ((kLogTable - 1) << 7)));
  const double m = __hiloint2double((yh & 0x000fffff) | 0x3ff00000, __double2loint(y));
  const double t = __fma_rn(m, tc.x, -1.0);
  double s = __fma_rn(t, kLog2Series[4], kLog2Series[3]);
  s = __fma_rn(t, s, kLog2Series[2]);
  s = __fma_rn(t, s, kLog2Series[1]);
  s = __fma_rn(t, s, kLog2Series[0]);
  const double l2m = __fma_rn(t, s, tc.y);                                         // log2 of y's mantissa
  const double k = __hiloint2double(0x43380000, 1075 - (yh >> 20)) - 0x1.8p52;  // 52 - exponent of y, exact
  return k - l2m;
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

// (row, col) of a row-major position in a block of nb columns.  The position
// travels biased, xb = 2^52 + x (x an integer < 2^52): the low word of xb is
// x mod 2^32.  floor(x RD(1/nb)) — one FMA rounded down onto the integer
// grid of [2^52, 2^53) — is the true quotient or one less (x / nb < 2^26, so
// the 2^-52 relative deficit of RD(1/nb) costs less than one unit); the
// residual x - row nb in [0, 2 nb) is taken in 32-bit integer arithmetic
// (nb <= 2^26) and settles it.  No int <-> fp conversions.
__device__ __forceinline__ void decode_pos(double xb, double inv_nb_rd, uint32_t nb, uint32_t& row, uint32_t& col) {
  const double qf = __fma_rd(xb - 0x1.0p52, inv_nb_rd, 0x1.0p52);
  uint32_t r = static_cast<uint32_t>(__double2loint(qf));
  uint32_t c = static_cast<uint32_t>(__double2loint(xb)) - r * nb;
  if (c >= nb) {
    c -= nb;
    ++r;
  }
  row = r;
  col = c;
}

constexpr int kStageCap = 256;  // staged pairs per warp (ring / write modes)
constexpr int kStageBytes = kStageCap * 8;  // 2048: the per-warp stage is 2048-aligned in shared memory
constexpr int kUncCap = 64;     // queued uncertain candidates per warp
constexpr int kUncRec = 32;     // record: {u, v, h | id << 11, -} + {w_u, w_v} (filled by cp.async)
constexpr size_t kWarpQueue = kUncCap * kUncRec + 16;
constexpr int kHotDeg = 256;  // tracked counters kept per CTA in shared memory (the heaviest tracked nodes)

// shared memory: [pad to 2048][stage: warps x 2048 B][log2 table copies][per warp: uncertain queue + chunk constants]
// [hot tracked-degree counters]
__host__ __device__ inline size_t blk_smem_bytes(int threads) {
  return kStageBytes + static_cast<size_t>(threads / 32) * (kStageBytes + kWarpQueue) + kTabBytes +
         kHotDeg * sizeof(uint32_t);
}

// Per-warp chunk constants needed only on the rare paths (uncertain
// candidates), kept in shared memory instead of registers.
struct WarpChunk {
  uint64_t key;
  double pbar;
};

__device__ __forceinline__ void sts_pair(uint32_t saddr, uint32_t u, uint32_t v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr), "r"(u), "r"(v) : "memory");
}
__device__ __forceinline__ uint2 lds_pair(uint32_t saddr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(saddr) : "memory");
  return r;
}
__device__ __forceinline__ uint4 lds_pair2(uint32_t saddr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(saddr) : "memory");
  return r;
}

template <int MODE, int E, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) blk_kernel(BlkArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NW = THREADS / 32;
  const int wib = threadIdx.x >> 5;
  // the stage of warp w sits at a 2048-aligned shared address, so a slot's
  // address is base | (byte counter & 2047): one LOP3
  unsigned char* sm = smem_raw + ((0u - static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw))) & (kStageBytes - 1));
  const uint32_t stage_s = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + wib * kStageBytes;
  unsigned char* tab = sm + NW * kStageBytes;
  unsigned char* wq = tab + kTabBytes + static_cast<size_t>(wib) * kWarpQueue;
  WarpChunk& wc = *reinterpret_cast<WarpChunk*>(wq + kUncCap * kUncRec);
  // The first kHotDeg tracked counters — the heaviest tracked nodes, w being
  // sorted — are accumulated per CTA in shared memory and added to the global
  // array once at the end: a hub's row fills whole flushes with one node, and
  // same-address global reductions serialise in L2 (C3: node 0 alone took 1e5
  // of them within the 6 ms step).
  uint32_t* s_hot = reinterpret_cast<uint32_t*>(tab + kTabBytes + static_cast<size_t>(NW) * kWarpQueue);
  for (int i = threadIdx.x; i < kHotDeg; i += THREADS) s_hot[i] = 0u;
  for (int i = threadIdx.x; i < kLogTable * kTabCopies; i += THREADS) {
    const int e = i / kTabCopies;
    reinterpret_cast<double2*>(tab)[i] = make_double2(a.logtab->inv_c[e], a.logtab->nlog2_inv[e]);
  }
  __syncthreads();

  const int lane = lane_id();
  const unsigned char* tab_lane = tab + 16 * (lane & (kTabCopies - 1));
  const unsigned lt = lanemask_lt();
  const unsigned long long t_start = a.prof.slots ? globaltimer_ns() : 0ull;
  const int64_t total = *a.total_chunks;
  const uint32_t tmask = (1u << a.track_shift) - 1u;
  const bool track = MODE == kWalkFold && a.degree != nullptr;

  // fold-mode ring: a private circular segment per warp (no reservation atomics)
  uint2* seg = nullptr;  // null: fold only
  uint32_t smask = 0, wpos = 0;
  if (MODE == kWalkFold && a.ring) {
    const unsigned nw = gridDim.x * NW;
    const unsigned gw = blockIdx.x * NW + wib;
    const int lcap = 63 - __clzll(static_cast<long long>(a.ring_mask + 1ull));
    const int lnw = nw > 1 ? 32 - __clz(nw - 1) : 0;
    int sl = lcap - lnw;
    sl = sl < 6 ? 6 : (sl > 20 ? 20 : sl);
    if (sl > lcap) sl = lcap;
    smask = (1u << sl) - 1u;
    seg = a.ring + ((static_cast<unsigned long long>(gw) << sl) & a.ring_mask);
  }
  constexpr bool staging = MODE == kWalkWrite || MODE == kWalkFold;  // fold: every edge is staged (fold + ring at flush)
  uint32_t head = 0, tail = 0;  // stage counters in BYTES (warp-uniform; 8 per pair)
  uint64_t checksum = 0;
  uint64_t wedges = 0;          // edges of this warp
  int64_t out_pos = 0;          // write mode
  Xoro128 rng;

  // fold of one staged edge: checksum term and tracked degrees
  // The tracked-degree array (n >> track_shift counters, 62.5 MB at C4) is
  // reduced into at random while 2 TB/s of ring stores stream through L2:
  // without a hint its lines are evicted between touches and every reduction
  // becomes a DRAM read-modify-write (measured at C4: 959 GB of DRAM reads per
  // step, 20% of the step).  The reductions carry an L2 evict_last policy,
  // made on this rare path so no register is held across the hot loop.
  auto red_degree = [&](uint32_t x) {
    const uint32_t id = x >> a.track_shift;
    if (id < static_cast<uint32_t>(kHotDeg)) {
      // address rebuilt from the stage base on this rare path (no register held for it)
      const uint32_t hot_s = stage_s - (threadIdx.x >> 5) * kStageBytes +
                             static_cast<uint32_t>(NW * kStageBytes + kTabBytes + NW * kWarpQueue) + 4u * id;
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hot_s) : "memory");
      return;
    }
    uint32_t* p = &a.degree[id];
    asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                 " red.global.add.L2::cache_hint.u32 [%0], 1, pol;\n}" ::"l"(p) : "memory");
  };
  auto fold_pair = [&](uint2 e, bool live) {
    checksum += live ? edge_hash(e.x, e.y) : 0ull;
    if (track) {
      if (live && (e.x & tmask) == 0) red_degree(e.x);
      if (live && (e.y & tmask) == 0) red_degree(e.y);
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
      const uint4 v2 = lds_pair2(stage_s | ((tail + 16 * lane) & (kStageBytes - 1)));
      fold_pair(make_uint2(v2.x, v2.y), true);
      fold_pair(make_uint2(v2.z, v2.w), true);
      if (seg) *reinterpret_cast<uint4*>(&seg[(wpos + 2 * lane) & smask]) = v2;
      wpos += 64;
    } else {
      // write mode: the 64 pairs go to pairs[out_pos ..) as 16-byte vector
      // stores of two pairs.  The burst may start on an odd pair: then pair 0 and
      // pair 63 are stored alone and lanes 0..30 store pairs (1+2l, 2+2l), so
      // every vector store stays 16-byte aligned in global memory.
      const uint32_t odd = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(a.pairs) >> 3) + out_pos) & 1u;  // 16-byte parity of the address
      const uint32_t k = odd + 2u * lane;  // first staged pair of this lane's vector
      const int64_t p = out_pos + k;
      if (k + 1u < 64u) {
        const uint2 e0 = lds_pair(stage_s | ((tail + 8 * k) & (kStageBytes - 1)));
        const uint2 e1 = lds_pair(stage_s | ((tail + 8 * (k + 1u)) & (kStageBytes - 1)));
        if (p + 1 < a.cap) {
          *reinterpret_cast<uint4*>(&a.pairs[p]) = make_uint4(e0.x, e0.y, e1.x, e1.y);
        } else {
          if (p < a.cap) a.pairs[p] = e0;
          atomicAdd(a.overflow, p < a.cap ? 1ull : 2ull);
        }
      }
      if (odd && (lane == 0 || lane == 31)) {  // the two single pairs of a misaligned burst
        const uint32_t ks = lane == 0 ? 0u : 63u;
        const int64_t ps = out_pos + ks;
        if (ps < a.cap) a.pairs[ps] = lds_pair(stage_s | ((tail + 8 * ks) & (kStageBytes - 1)));
        else atomicAdd(a.overflow, 1ull);
      }
      out_pos += 64;
    }
    tail += 512;
    __syncwarp();
  };
  auto flush_rest = [&]() {  // < 64 left
    __syncwarp();
    const uint32_t rem = (head - tail) >> 3;
    for (uint32_t i0 = 0; i0 < rem; i0 += 32) {
      const bool live = i0 + lane < rem;
      const uint2 e = lds_pair(stage_s | ((tail + 8 * (i0 + lane)) & (kStageBytes - 1)));
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
  uint32_t cw = 0;  // edges of the current chunk (warp-uniform; staging modes count through head)
  // one candidate slot per lane: stage the accepted pairs
  auto emit1 = [&](bool acc, uint32_t u, uint32_t v) {
    if (MODE == kWalkPairs && acc) atomicAdd(&a.pair_counts[static_cast<uint64_t>(u) * a.n + v], 1u);
    const unsigned b = __ballot_sync(CLG_FULL, acc);
    if (staging) {
      if (acc) sts_pair(stage_s | ((head + 8 * __popc(b & lt)) & (kStageBytes - 1)), u, v);
      head += 8 * __popc(b);
    } else {
      cw += __popc(b);
    }
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
    uint32_t qn = 0, qt = 0;  // uncertain queue counters (warp-uniform)
    if (MODE == kWalkWrite) out_pos = a.offsets[q];
    cw = 0;
    const uint32_t head0 = head;
    // biased window bounds (positions travel as 2^52 + x)
    const double wlo = static_cast<double>(r.x_lo) + 0x1.0p52, whi = static_cast<double>(r.x_hi) + 0x1.0p52;

    // decide the queued uncertain candidates (k <= 32): gather w_u, w_v
    auto resolve = [&](uint32_t k) {
      asm volatile("cp.async.wait_all;" ::: "memory");  // this lane's weight copies have landed
      __syncwarp();
      bool acc = false;
      uint32_t u = 0, v = 0;
      if (static_cast<uint32_t>(lane) < k) {
        const unsigned char* rp = wq + ((qt + lane) & (kUncCap - 1)) * kUncRec;
        const uint4 rec = *reinterpret_cast<const uint4*>(rp);
        const double2 ww = *reinterpret_cast<const double2*>(rp + 16);  // w_u, w_v (cp.async, waited for above)
        const uint32_t hid = rec.z;
        u = rec.x;
        v = rec.y;
        const double q_ = __ddiv_rn(__dmul_rn(ww.x, ww.y), a.S);  // edge_skip.cpp:36
        acc = lazy_accept(hid & 2047u, __ddiv_rn(q_ < 1.0 ? q_ : 1.0, wc.pbar), wc.key, hid >> 11);
      }
      qt += k;
      __syncwarp();
      emit1(acc, u, v);
      if (staging)
        while (head - tail >= 512) flush64();
    };

    if (!(d.flags & kBlkDense)) {
      // ---- sparse block: each lane runs its own geometric process over its
      // 1/32 of the chunk (memoryless restart at the lane's first position:
      // no cross-lane dependence), E candidates per iteration.  The E gap
      // draws (RNG, table log2, series) are independent chains issued
      // together; only the position sum is sequential. ----
      const double inv_mu2 = d.inv_mu, inv_nb = d.inv_nb;
      const uint32_t hs = d.hs, nb = d.nb, a0 = d.a0, b0 = d.b0;
      const int64_t ls = (x1 - x0 + 31) >> 5;
      const int64_t lx0 = imin64(x0 + lane * ls, x1);
      const double lend = static_cast<double>(imin64(lx0 + ls, x1)) + 0x1.0p52;  // biased end of the lane's positions
      double pos = static_cast<double>(lx0) + (0x1.0p52 - 1.0);                 // biased last candidate position
      // Two instances of the loop: the plain one (off-diagonal block, chunk not
      // cut by the launch's source range: almost every chunk) drops the
      // u < v and window tests from every candidate.
      auto sparse_loop = [&](auto plain_tag) {
      constexpr bool PLAIN = decltype(plain_tag)::value;
      for (uint32_t id = 0; __any_sync(CLG_FULL, pos < lend); id += E) {
        double gap[E];
        uint32_t h[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t x = rng.next();
          h[e] = static_cast<uint32_t>(x) & 2047u;
          // geometric gap floor(E2 / mu2) + 1 as a double (>= 2^52: past every chunk end)
          gap[e] = __fma_rd(exp2_52(x, tab_lane), inv_mu2, 0x1.0p52) - (0x1.0p52 - 1.0);
        }
        uint32_t u[E], v[E];
        bool sure[E], unc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          pos += gap[e];
          uint32_t row, col;
          decode_pos(pos, inv_nb, nb, row, col);
          bool ok = pos < lend;
          if (!PLAIN) {
            ok = ok && (col > row || !diag);
            if (partial) ok = ok && pos >= wlo && pos < whi;
          }
          u[e] = a0 + row;
          v[e] = b0 + col;
          sure[e] = ok && h[e] < hs;
          unc[e] = ok && h[e] >= hs;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          emit1(sure[e], u[e], v[e]);
          const unsigned m = __ballot_sync(CLG_FULL, unc[e]);
          if (m) {
            if (unc[e]) {
              unsigned char* rp = wq + ((qn + __popc(m & lt)) & (kUncCap - 1)) * kUncRec;
              *reinterpret_cast<uint4*>(rp) =
                  make_uint4(u[e], v[e], h[e] | ((((id + e) << 5 | static_cast<uint32_t>(lane)) & 0x1fffffu) << 11), 0u);
              // w_u and w_v travel straight into the record (asynchronous 8-byte
              // copies, 64-byte L2 fetches): nothing waits until 32 are queued
              const uint32_t sw = static_cast<uint32_t>(__cvta_generic_to_shared(rp + 16));
              asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], 8;" ::"r"(sw), "l"(a.w + u[e]) : "memory");
              asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], 8;" ::"r"(sw + 8u), "l"(a.w + v[e]) : "memory");
            }
            qn += __popc(m);
            if (qn - qt >= 32) resolve(32);
          }
        }
        if (staging)
          while (head - tail >= 512) flush64();
      }
      };
      if (!diag && !partial) sparse_loop(std::true_type{});
      else sparse_loop(std::false_type{});
    } else {
      // ---- dense block (pbar >= 1): every position is a candidate ----
      const double inv_nb = d.inv_nb;
      const double xend = static_cast<double>(x1) + 0x1.0p52;
      for (double xb = static_cast<double>(x0) + 0x1.0p52; xb < xend; xb += 32.0) {
        const double x = xb + static_cast<double>(lane);
        uint32_t row, col;
        decode_pos(x, inv_nb, d.nb, row, col);
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
          while (head - tail >= 512) flush64();
      }
    }
    if (qn != qt) resolve(qn - qt);
    if (staging) cw = (head - head0) >> 3;
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
  if (track) {  // every warp of the CTA has left its loop: hand the hot counters over
    __syncthreads();
    for (int i = threadIdx.x; i < kHotDeg; i += THREADS)
      if (s_hot[i]) atomicAdd(&a.degree[i], s_hot[i]);
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

// one thread: z, the grid width and the thresholds.  min_block_cand > 0
// (automatic width): starting from eps0 the width is doubled — at most twice
// for this reason — while the blocks would hold fewer than min_block_cand
// expected candidates on average (S / 2 over cells^2 / 2): a small graph cut
// into ~5e5 blocks spends its time on block and chunk set-up, and a chunk
// cannot be larger than its block.
__global__ void cls_grid_kernel(const double* __restrict__ w, int64_t n, double eps0, double min_block_cand, double S,
                                int kcap, double* thr, ClassPlan* plan) {
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
    if (cells + zero_class + extra > kcap) continue;
    if (min_block_cand > 0.0 && attempt < 2 && S / (cells * cells) < min_block_cand) continue;
    kg = static_cast<int>(cells);
    break;
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
    d.inv_mu = 0x1.62e42fefa39efp-1 / -log1p(-pbar);  // 1 / -log2(1 - pbar)
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
