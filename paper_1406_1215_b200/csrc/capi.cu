// C ABI of the B200 Chung–Lu generator (include/clgen_dev.h).
//
// Host orchestration of the device pipeline.  Each entry point validates its
// contract exactly where the reference throws clgen::error, launches the
// sm_100a kernels on the context stream, and synchronises only when a scalar
// result must be returned to the caller.

#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>
#include <type_traits>
#include <string>

#include "../../include/clgen_dev.h"
#include "common.cuh"
#include "exact_fold.cuh"
#include "plan.cuh"
#include "edge_io.cuh"
#include "fidelity.cuh"
#include "sampler_blk.cuh"
#include "sampler_ref.cuh"
#include "scan.cuh"
#include "weights.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(CLGEN_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                  __FILE__, __LINE__);                                                    \
  } while (0)

// Growable device scratch buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Small per-call device scalars (one allocation, zeroed per call).
struct Scalars {
  unsigned long long queue;
  unsigned long long queue_heavy;
  long long heavy_end;
  unsigned long long ticket;
  unsigned long long flag_count;
  unsigned long long overflow;
  unsigned long long fold[2];
  unsigned long long ring_head;
  unsigned long long first_bad;
  unsigned long long first_negative;
  unsigned long long spill;
  unsigned long long spill_flags;
  unsigned long long runs;  // flag counter of the spill re-walk (discarded)
  int64_t total;
  double S;
  double fold_final;
};

constexpr int64_t kFlagCap = 4096;

double env_double(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : dflt;
}

}  // namespace

// spmd.cu reports its (lowest failing rank's) error through the caller's slot
int clgen_internal_fail(int code, const char* msg) { return fail(code, "%s", msg); }

struct clgen_dev_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  double* w = nullptr;
  int64_t n = 0;
  size_t w_bytes = 0;
  // clgen_dev_prefetch_weights: the next weight array, copied on its own stream
  double* w_next = nullptr;
  size_t w_next_bytes = 0;
  const double* next_src = nullptr;
  int64_t next_n = -1;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t next_ready = nullptr;
  cudaEvent_t swap_done = nullptr;  // main-stream work issued before the last swap (it may read w_next's buffer)
  bool swapped = false;
  Scalars* sc = nullptr;     // device
  Scalars* sc_host = nullptr;  // pinned mirror
  int64_t* flagged = nullptr;  // device, kFlagCap
  int64_t last_flagged = 0;
  DevBuf counts, offsets, tiles, pairs, partials, degree, sources, foldtmp, cum, found;
  DevBuf slot_cap, soff, scratch, spill;  // single-pass reference-stream materialisation
  DevBuf run_len;         // run-length table of w (weights.cuh), when runs are long
  bool has_runs = false;
  bool use_runs = env_double("CLGEN_RUN_TABLE", 1.0) != 0.0;
  bool one_pass = env_double("CLGEN_REF_1PASS", 1.0) != 0.0;
  double slot_sigma = env_double("CLGEN_REF_SLOT_SIGMA", 6.0), slot_const = env_double("CLGEN_REF_SLOT_CONST", 8.0);
  int plan_G = 0;  // blocks of the cost profile currently held in `cum`
  // counter stream (sampler_blk.cuh): class table per weights, block table
  // per (weights, S), chunk tables per launch range
  DevBuf cls_thr, cls_bounds, cls_start, cls_wfirst, cls_wlast, cls_plan;
  DevBuf blocks, ranges, blk_cnt, blk_prefix, chunk_block, chunk_total, chunk_counts, chunk_offsets;
  DevBuf keys_a, keys_b, sort_tmp;  // materialised counter output: device sort by (u, v)
  DevBuf probe;                     // small scratch (fidelity histograms)
  DevBuf costs;                     // node_costs_sequential (suffix-form costs)
  clg::ClassPlan plan_host{};
  bool cls_valid = false;
  bool blk_valid = false;
  double blk_S = 0.0;
  int64_t rng_lo = -1, rng_hi = -1;  // launch range the chunk tables hold
  double cls_eps = env_double("CLGEN_CTR_EPS", 0.0);  // 0: automatic (1/128, widened for small graphs)
  double cls_S = -1.0;                                // S the automatic class table was built for
  double chunk_cand = env_double("CLGEN_CTR_CHUNK", 0.0);  // 0: auto (auto_chunk_cand)
  int blk_shape = -1;  // clgen_dev_set_kernel_shape (-1: CLGEN_BLK_SHAPE / default)
  int blk_grid[4][5] = {};
  size_t blk_smem[4][5] = {};
  // optional per-warp busy intervals of the sampler kernels
  bool warp_prof = false;
  DevBuf prof;
  int prof_warps = 0;  // slots used by the last sampler launch(es)
  std::vector<int> prof_launch;  // first slot of each of those launches
  void* host_stage = nullptr;    // pinned staging for edge files
  size_t host_stage_bytes = 0;
  uint64_t seed_mix = 0;
  int walk_blocks[2][2][3] = {};  // [heavy][fast][mode]
  size_t l2_persist_max = 0, l2_window_max = 0;  // device limits (clgen_dev_create)
  bool ref_heavy = true;                         // clgen_dev_set_kernel_shape flag
  size_t l2_carve = 0;                           // persisting carve-out currently set
  bool l2_persist_dirty = false;                 // persisting lines left by a fold launch
  double w0 = 0.0;                // w[0] (host copy, set_weights)
  bool fast_math = true;
  int refill_min = static_cast<int>(env_double("CLGEN_REFILL_MIN", 8.0));
  clg::LogTable* logtab = nullptr;  // device
  clg::Log2Table* logtab2 = nullptr;  // device (counter stream: log2 table)
  // instrumentation: kernels launched by this context, and the duration of
  // the last dominant (sampler) kernel measured with events on the stream
  unsigned long long launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timed = false;
};

namespace {

int set_device(clgen_dev_ctx* c) {
  CUDA_TRY(cudaSetDevice(c->device));
  return CLGEN_OK;
}

// Per-warp profile slots for a launch of `grid` 256-thread CTAs.
clg::WarpProf prof_slots(clgen_dev_ctx* c, int grid, bool first) {
  clg::WarpProf p{nullptr, 0};
  if (!c->warp_prof) return p;
  if (first) {
    c->prof_warps = 0;
    c->prof_launch.clear();
  }
  const int warps = grid * 8;
  c->prof_launch.push_back(c->prof_warps);
  // size for several full-occupancy launches up front: growing the buffer
  // later would free the slots an earlier launch of this call writes into
  if (first && c->prof.ensure(static_cast<size_t>(4 * 64 * c->num_sms) * 2 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    return p;
  }
  if (c->prof.ensure(static_cast<size_t>(c->prof_warps + warps) * 2 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    return p;
  }
  p.slots = c->prof.as<unsigned long long>();
  p.base = c->prof_warps;
  c->prof_warps += warps;
  return p;
}

int reset_scalars(clgen_dev_ctx* c, unsigned long long queue_start) {
  Scalars z;
  std::memset(&z, 0, sizeof z);
  z.queue = queue_start;
  z.first_bad = ~0ull;
  z.first_negative = ~0ull;
  *c->sc_host = z;
  CUDA_TRY(cudaMemcpyAsync(c->sc, c->sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, c->stream));
  return CLGEN_OK;
}

int fetch_scalars(clgen_dev_ctx* c) {
  CUDA_TRY(cudaMemcpyAsync(c->sc_host, c->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return CLGEN_OK;
}

// Persisting L2 lines left by a fold launch (tracked degrees) are given back
// lazily, when a launch of another kind is about to run (the reset is a
// device-wide call; a loop of fold launches never pays it).
void release_persisting_l2(clgen_dev_ctx* c) {
  if (!c->l2_persist_dirty) return;
  cudaCtxResetPersistingL2Cache();
  c->l2_persist_dirty = false;
  cudaGetLastError();
}

template <int MODE, bool FAST, bool HEAVY>
int walk_grid(clgen_dev_ctx* c) {
  int& g = c->walk_blocks[HEAVY][FAST][MODE];
  if (!g) {
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, clg::ref_walk_kernel<MODE, FAST, HEAVY>, 256, 0));
    g = (per_sm > 0 ? per_sm : 1) * c->num_sms;
  }
  return g;
}

template <int MODE>
int launch_walk(clgen_dev_ctx* c, const clg::RefWalkArgs& a_in) {
  release_persisting_l2(c);
  clg::RefWalkArgs a = a_in;
  // Heavy phase (range walks only): slots whose weight — an upper bound of
  // the chain's expected candidates — is at least 4x the average work per
  // lane and at least 256 are walked one per warp; at most 8 per warp.  The
  // heavy-capable kernel is launched only when the heaviest weight reaches
  // the threshold (w is non-increasing, w0 read once by set_weights).
  static const bool heavy_on = env_double("CLGEN_REF_HEAVY", 1.0) != 0.0;
  const double lanes_lean = static_cast<double>(c->num_sms) * 4.0 * 256.0;
  const double tw = std::max(256.0, 4.0 * (0.5 * a.S) / lanes_lean);
  const bool heavy = heavy_on && c->ref_heavy && !a.sources && a.hi > a.lo && a.S > 0.0 && c->w0 >= tw;
  int grid;
  if (heavy) grid = c->fast_math ? walk_grid<MODE, true, true>(c) : walk_grid<MODE, false, true>(c);
  else grid = c->fast_math ? walk_grid<MODE, true, false>(c) : walk_grid<MODE, false, false>(c);
  if (grid < 0) return grid;
  a.prof = prof_slots(c, grid, true);
  CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
  if (heavy) {
    CUDA_TRY(cudaMemsetAsync(&c->sc->queue_heavy, 0, sizeof(unsigned long long), c->stream));
    clg::ref_heavy_end_kernel<<<1, 32, 0, c->stream>>>(c->w, a.lo, a.hi, tw, static_cast<int64_t>(grid) * 64,
                                                       reinterpret_cast<int64_t*>(&c->sc->heavy_end));
    a.heavy_end = reinterpret_cast<const int64_t*>(&c->sc->heavy_end);
    a.hqueue = &c->sc->queue_heavy;
    ++c->launches;
    if (c->fast_math) clg::ref_walk_kernel<MODE, true, true><<<grid, 256, 0, c->stream>>>(a);
    else clg::ref_walk_kernel<MODE, false, true><<<grid, 256, 0, c->stream>>>(a);
  } else {
    if (c->fast_math) clg::ref_walk_kernel<MODE, true, false><<<grid, 256, 0, c->stream>>>(a);
    else clg::ref_walk_kernel<MODE, false, false><<<grid, 256, 0, c->stream>>>(a);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
  c->timed = true;
  ++c->launches;
  return CLGEN_OK;
}

clg::RefWalkArgs walk_args(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, uint64_t seed) {
  clg::RefWalkArgs a;
  std::memset(&a, 0, sizeof a);
  a.w = c->w;
  a.run_len = c->has_runs ? c->run_len.as<int32_t>() : nullptr;
  a.n = c->n;
  a.S = S;
  a.lo = lo;
  a.hi = hi;
  a.seed = seed;
  a.queue = &c->sc->queue;
  a.flag_count = &c->sc->flag_count;
  a.flagged = c->flagged;
  a.flag_cap = kFlagCap;
  a.overflow = &c->sc->overflow;
  a.fold_out = c->sc->fold;
  a.ring_head = &c->sc->ring_head;
  a.logtab = c->logtab;
  a.invS = 1.0 / S;  // host IEEE division: RN(1/S)
  a.refill_min = c->refill_min;
  return a;
}

int check_range(clgen_dev_ctx* c, int64_t lo, int64_t hi) {
  if (lo < 0 || hi > c->n || lo > hi) return fail(CLGEN_EINVAL, "create_edges_range: bad node range");
  return CLGEN_OK;
}

// counts[0..m) -> offsets[0..m) exclusive, total in sc->total.
int launch_scan(clgen_dev_ctx* c, const int32_t* counts, int64_t* offsets, int64_t m) {
  const int64_t ntiles = (m + clg::kScanTile - 1) / clg::kScanTile;
  if (ntiles == 0) {
    CUDA_TRY(cudaMemsetAsync(&c->sc->total, 0, sizeof(int64_t), c->stream));
    return CLGEN_OK;
  }
  CUDA_TRY(c->tiles.ensure(ntiles * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(c->tiles.p, 0, ntiles * sizeof(unsigned long long), c->stream));
  CUDA_TRY(cudaMemsetAsync(&c->sc->ticket, 0, sizeof(unsigned long long), c->stream));
  clg::scan_lookback_kernel<int32_t><<<static_cast<unsigned>(ntiles), clg::kScanThreads, 0, c->stream>>>(
      counts, offsets, m, c->tiles.as<unsigned long long>(), &c->sc->ticket, &c->sc->total, 0);
  CUDA_TRY(cudaGetLastError());
  ++c->launches;
  return CLGEN_OK;
}

// weights.cpp:21-30 on device data d[0..n).
int blocked_sum_impl(clgen_dev_ctx* c, const double* d, int64_t n, double* S) {
  int rc = set_device(c);
  if (rc) return rc;
  if (n == 0) {
    *S = 0.0;
    return CLGEN_OK;
  }
  const int64_t nblocks = (n + clg::kSumBlock - 1) / clg::kSumBlock;
  CUDA_TRY(c->partials.ensure(nblocks * sizeof(double)));
  const unsigned grid = static_cast<unsigned>((nblocks + 127) / 128);
  clg::blocked_partials_kernel<<<grid, 128, 0, c->stream>>>(d, n, c->partials.as<double>(), nblocks);
  CUDA_TRY(cudaGetLastError());
  clg::fold_partials_kernel<<<1, 256, 0, c->stream>>>(c->partials.as<double>(), nblocks, &c->sc->S);
  CUDA_TRY(cudaGetLastError());
  c->launches += 2;
  if ((rc = fetch_scalars(c))) return rc;
  *S = c->sc_host->S;
  return CLGEN_OK;
}

// ---- exact sequential-fold replay (exact_fold.cuh) -------------------------
size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Folds x[0..m) left to right from s0 exactly as a sequential FP64 loop
// would; *final_host receives s_m.  out_mode/out/w/S per clg::FoldOut.
int run_fold(clgen_dev_ctx* c, const double* x, int64_t m, double s0, int out_mode, double* out,
             const double* w, double S, double* final_host, int64_t stride = 1, int reverse = 0) {
  if (m == 0) {
    *final_host = s0;
    return CLGEN_OK;
  }
  const int64_t T = (m + clg::kFoldTile - 1) / clg::kFoldTile;
  const size_t b_tsum = align_up(T * sizeof(double)), b_app = align_up((T + 1) * sizeof(double)),
               b_fun = align_up(T * sizeof(clg::Fn)), b_bin = align_up(T * sizeof(int)),
               b_start = align_up(T * sizeof(double)), b_slow = align_up(T);
  CUDA_TRY(c->foldtmp.ensure(b_tsum + b_app + b_fun + b_bin + b_start + b_slow));
  char* base = c->foldtmp.as<char>();
  clg::FoldArgs a;
  a.x = x;
  a.m = m;
  a.s0 = s0;
  a.tsum = reinterpret_cast<double*>(base);
  a.approx = reinterpret_cast<double*>(base + b_tsum);
  a.tfun = reinterpret_cast<clg::Fn*>(base + b_tsum + b_app);
  a.tbin = reinterpret_cast<int*>(base + b_tsum + b_app + b_fun);
  a.start = reinterpret_cast<double*>(base + b_tsum + b_app + b_fun + b_bin);
  a.slow = reinterpret_cast<unsigned char*>(base + b_tsum + b_app + b_fun + b_bin + b_start);
  a.final_out = &c->sc->fold_final;
  a.out_mode = out_mode;
  a.out = out;
  a.w = w;
  a.S = S;
  a.stride = stride;
  a.reverse = reverse;
  const unsigned g = static_cast<unsigned>(T);
  clg::fold_tile_sums_kernel<<<g, clg::kFoldThreads, 0, c->stream>>>(a);
  clg::fold_approx_prefix_kernel<<<1, 1024, 0, c->stream>>>(a, T);
  clg::fold_tile_fun_kernel<<<g, clg::kFoldThreads, 0, c->stream>>>(a);
  clg::fold_spine_kernel<<<1, 32, 0, c->stream>>>(a, T);
  c->launches += 4;
  if (out_mode != clg::kFoldNone) {
    clg::fold_emit_kernel<<<g, clg::kFoldThreads, 0, c->stream>>>(a);
    ++c->launches;
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(&c->sc_host->fold_final, &c->sc->fold_final, sizeof(double),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *final_host = c->sc_host->fold_final;
  return CLGEN_OK;
}

// cost.cpp:15-22
void block_bounds_host(int64_t n, int P, int rank, int64_t* lo, int64_t* hi) {
  const int64_t q = n / P, r = n % P;
  *lo = static_cast<int64_t>(rank) * q + (rank < r ? rank : r);
  *hi = *lo + q + (rank < r ? 1 : 0);
}

int plan_args_ok(clgen_dev_ctx* c, int G, int g) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (G < 1 || g < 0 || g >= G) return fail(CLGEN_EINVAL, "block_bounds: bad rank/P");
  return set_device(c);
}

int ensure_cum(clgen_dev_ctx* c, int G) {
  CUDA_TRY(c->cum.ensure((c->n > 0 ? c->n : 1) * sizeof(double)));
  c->plan_G = G;
  return CLGEN_OK;
}

int block_weight_impl(clgen_dev_ctx* c, int G, int g, double* bw) {
  int64_t lo, hi;
  block_bounds_host(c->n, G, g, &lo, &hi);
  return run_fold(c, c->w + lo, hi - lo, 0.0, clg::kFoldNone, nullptr, nullptr, 0.0, bw);
}

// block_cumulative (cost.cpp:24-46): c_u from the exact sigma fold, then the
// exact cumulative fold (first element cum = c, i.e. a fold from 0.0).
int block_costs_impl(clgen_dev_ctx* c, int G, int g, double sigma_start, double S, double* z) {
  int64_t lo, hi;
  block_bounds_host(c->n, G, g, &lo, &hi);
  int rc = ensure_cum(c, G);
  if (rc) return rc;
  double* cum = c->cum.as<double>();
  if (hi == lo) {
    *z = 0.0;
    return CLGEN_OK;
  }
  if (S > 0.0) {
    double sigma_end;
    if ((rc = run_fold(c, c->w + lo, hi - lo, sigma_start, clg::kFoldNodeCost, cum + lo, c->w + lo, S,
                       &sigma_end)))
      return rc;
  } else {  // S == 0 degenerates to unit costs (cost.cpp:34-36)
    clg::fill_f64_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(cum, lo, hi, 1.0);
    ++c->launches;
    CUDA_TRY(cudaGetLastError());
  }
  return run_fold(c, cum + lo, hi - lo, 0.0, clg::kFoldInclusive, cum + lo, nullptr, 0.0, z);
}

int block_boundaries_impl(clgen_dev_ctx* c, int G, int g, double z_offset, double z_bar, long long* d_found) {
  int64_t lo, hi;
  block_bounds_host(c->n, G, g, &lo, &hi);
  if (!(z_bar > 0.0)) return fail(CLGEN_EINVAL, "partition_of: Z_bar must be > 0");
  if (hi > lo) {
    const int64_t m = hi - lo;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m + 255) / 256, c->num_sms * 16));
    clg::ucp_transitions_kernel<<<grid, 256, 0, c->stream>>>(c->cum.as<double>(), lo, hi, z_offset, z_bar, G,
                                                           d_found);
    ++c->launches;
    CUDA_TRY(cudaGetLastError());
  }
  return CLGEN_OK;
}

// ---- counter stream (sampler_blk.cuh) ----------------------------------------
// Class table of the weights (no host round trip) and block table for S (one
// synchronisation: the host learns the class and chunk counts to size the
// per-launch tables); both cached until the weights, S or the parameters change.
// Automatic chunk size: S / 2 bounds the expected edge count; about 2^15
// chunks per graph, between 4096 candidates (small graphs keep every warp
// busy) and 262144 (8192 per lane: the lanes of a chunk end within ~2% of
// one another).  A function of S only, so every GPU count and every cover of
// the sources cuts the same chunks.
double auto_chunk_cand(double S) {
  const double c = std::floor(S * 0x1.0p-16);
  return c < 4096.0 ? 4096.0 : (c > 262144.0 ? 262144.0 : c);
}
// Automatic class width: 1/128, doubled (at most twice) while the class-pair
// blocks would average fewer than this many expected candidates.
constexpr double kAutoEps = 0.0078125, kAutoMinBlockCand = 8192.0;

int ensure_blocks(clgen_dev_ctx* c, double S) {
  if (c->blk_valid && c->blk_S == S) return CLGEN_OK;
  const int kcap = clg::kClassCap;
  const bool auto_eps = !(c->cls_eps > 0.0);
  if (auto_eps && c->cls_S != S) c->cls_valid = false;  // the automatic width looks at S
  if (!c->cls_valid) {
    CUDA_TRY(c->cls_thr.ensure((kcap + 2) * sizeof(double)));
    CUDA_TRY(c->cls_bounds.ensure((kcap + 2) * sizeof(int64_t)));
    CUDA_TRY(c->cls_start.ensure((kcap + 2) * sizeof(int64_t)));
    CUDA_TRY(c->cls_wfirst.ensure((kcap + 1) * sizeof(double)));
    CUDA_TRY(c->cls_wlast.ensure((kcap + 1) * sizeof(double)));
    CUDA_TRY(c->cls_plan.ensure(sizeof(clg::ClassPlan)));
    CUDA_TRY(cudaMemsetAsync(c->cls_plan.p, 0, sizeof(clg::ClassPlan), c->stream));
    clg::ClassPlan* dp = c->cls_plan.as<clg::ClassPlan>();
    clg::cls_grid_kernel<<<1, 1, 0, c->stream>>>(c->w, c->n, auto_eps ? kAutoEps : c->cls_eps,
                                                 auto_eps ? kAutoMinBlockCand : 0.0, S, kcap, c->cls_thr.as<double>(), dp);
    c->cls_S = S;
    clg::cls_bounds_kernel<<<(kcap + 256) / 256, 256, 0, c->stream>>>(c->w, c->cls_thr.as<double>(), dp, kcap,
                                                                        c->cls_bounds.as<int64_t>());
    clg::cls_compact_kernel<<<1, 1, 0, c->stream>>>(c->w, c->n, c->cls_bounds.as<int64_t>(), kcap, dp,
                                                    c->cls_start.as<int64_t>(), c->cls_wfirst.as<double>(),
                                                    c->cls_wlast.as<double>());
    c->launches += 3;
    CUDA_TRY(cudaGetLastError());
  }
  clg::ClassPlan* dp = c->cls_plan.as<clg::ClassPlan>();
  CUDA_TRY(cudaMemsetAsync(&dp->chunks_full, 0, sizeof(unsigned long long), c->stream));
  CUDA_TRY(cudaMemsetAsync(&dp->dense_blocks, 0, sizeof(int), c->stream));
  const int64_t nb_max = static_cast<int64_t>(kcap) * (kcap + 1) / 2;
  CUDA_TRY(c->blocks.ensure(nb_max * sizeof(clg::BlockDesc)));
  {
    const dim3 blk(32, 8), grd((kcap + 31) / 32, (kcap + 7) / 8);
    clg::blk_desc_kernel<<<grd, blk, 0, c->stream>>>(c->cls_start.as<int64_t>(), c->cls_wfirst.as<double>(),
                                                     c->cls_wlast.as<double>(), dp, S,
                                                     c->chunk_cand > 0.0 ? c->chunk_cand : auto_chunk_cand(S),
                                                     c->blocks.as<clg::BlockDesc>());
    ++c->launches;
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaMemcpyAsync(&c->plan_host, dp, sizeof(clg::ClassPlan), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->plan_host.K < 0) return fail(CLGEN_EINVAL, "counter stream: weight range too wide for the class table");
  c->plan_host.nblocks = static_cast<int64_t>(c->plan_host.Knz) * (c->plan_host.Knz + 1) / 2;
  c->cls_valid = true;
  c->blk_valid = true;
  c->blk_S = S;
  c->rng_lo = c->rng_hi = -1;
  return CLGEN_OK;
}

// Per launch range [lo, hi): chunks per block, their prefix (total on the
// device) and the chunk -> block map.  No host round trip.
int ensure_range(clgen_dev_ctx* c, int64_t lo, int64_t hi) {
  if (c->rng_lo == lo && c->rng_hi == hi) return CLGEN_OK;
  const int64_t nb = c->plan_host.nblocks;
  const int64_t cf = static_cast<int64_t>(c->plan_host.chunks_full);
  CUDA_TRY(c->ranges.ensure((nb > 0 ? nb : 1) * sizeof(clg::BlockRange)));
  CUDA_TRY(c->blk_cnt.ensure((nb > 0 ? nb : 1) * sizeof(int64_t)));
  CUDA_TRY(c->blk_prefix.ensure((nb > 0 ? nb : 1) * sizeof(int64_t)));
  CUDA_TRY(c->chunk_block.ensure((cf > 0 ? cf : 1) * sizeof(uint32_t)));
  CUDA_TRY(c->chunk_total.ensure(sizeof(int64_t)));
  CUDA_TRY(cudaMemsetAsync(c->chunk_total.p, 0, sizeof(int64_t), c->stream));
  if (nb > 0) {
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((nb + 255) / 256, c->num_sms * 8));
    clg::blk_range_kernel<<<grid, 256, 0, c->stream>>>(c->blocks.as<clg::BlockDesc>(), nb, lo, hi,
                                                       c->ranges.as<clg::BlockRange>(), c->blk_cnt.as<int64_t>());
    ++c->launches;
    CUDA_TRY(cudaGetLastError());
    const int64_t ntiles = (nb + clg::kScanTile - 1) / clg::kScanTile;
    CUDA_TRY(c->tiles.ensure(ntiles * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(c->tiles.p, 0, ntiles * sizeof(unsigned long long), c->stream));
    CUDA_TRY(cudaMemsetAsync(&c->sc->ticket, 0, sizeof(unsigned long long), c->stream));
    clg::scan_lookback_kernel<int64_t><<<static_cast<unsigned>(ntiles), clg::kScanThreads, 0, c->stream>>>(
        c->blk_cnt.as<int64_t>(), c->blk_prefix.as<int64_t>(), nb, c->tiles.as<unsigned long long>(), &c->sc->ticket,
        c->chunk_total.as<int64_t>(), 0);
    const unsigned mgrid = static_cast<unsigned>(std::min<int64_t>((nb + 7) / 8, c->num_sms * 16));
    clg::blk_chunk_map_kernel<<<mgrid, 256, 0, c->stream>>>(c->blk_cnt.as<int64_t>(), c->blk_prefix.as<int64_t>(), nb,
                                                            c->chunk_block.as<uint32_t>());
    c->launches += 2;
    CUDA_TRY(cudaGetLastError());
  }
  c->rng_lo = lo;
  c->rng_hi = hi;
  return CLGEN_OK;
}

clg::BlkArgs blk_args(clgen_dev_ctx* c, double S, uint64_t seed) {
  clg::BlkArgs a;
  std::memset(&a, 0, sizeof a);
  a.w = c->w;
  a.S = S;
  a.blocks = c->blocks.as<clg::BlockDesc>();
  a.ranges = c->ranges.as<clg::BlockRange>();
  a.chunk_prefix = c->blk_prefix.as<int64_t>();
  a.chunk_block = c->chunk_block.as<uint32_t>();
  a.total_chunks = c->chunk_total.as<int64_t>();
  a.queue = &c->sc->queue;
  a.seed_mix = clg::mix64(seed ^ 0x636c67656e626c6bULL);  // "clgenblk" domain tag
  a.seed = seed;
  a.trials = 1;
  a.logtab = c->logtab2;
  a.overflow = &c->sc->overflow;
  a.fold_out = c->sc->fold;
  return a;
}

// The counter-stream kernel: one persistent grid, warps claim chunks.  Block
// shape (CLGEN_BLK_SHAPE or clgen_dev_set_kernel_shape): 256 threads x
// 2 / 3 (default: 80 registers, no spills) / 4 / 5 / 6 CTAs per SM for shape 0 / 1 / 2 / 3 / 4; the
// edge set does not depend on it.
constexpr int kBlkE = 4;  // candidates per lane per loop iteration (an unroll factor)

template <int MODE>
int launch_blk(clgen_dev_ctx* c, const clg::BlkArgs& a_in) {
  static const int env_shape = [] {
    const char* e = std::getenv("CLGEN_BLK_SHAPE");
    const int v = e ? std::atoi(e) : 1;
    return v >= 0 && v <= 4 ? v : 1;
  }();
  const int shape = c->blk_shape >= 0 ? c->blk_shape : env_shape;
  if (MODE != clg::kWalkFold) release_persisting_l2(c);
  clg::BlkArgs a = a_in;
  CUDA_TRY(cudaMemsetAsync(&c->sc->queue, 0, sizeof(unsigned long long), c->stream));
  auto launch = [&](auto kern, int threads) -> int {
    const size_t smem = clg::blk_smem_bytes(threads);
    if (!c->blk_grid[MODE][shape] || c->blk_smem[MODE][shape] != smem) {
      if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      int per_sm = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
      c->blk_grid[MODE][shape] = (per_sm > 0 ? per_sm : 1) * c->num_sms;
      c->blk_smem[MODE][shape] = smem;
    }
    const int g = c->blk_grid[MODE][shape];
    a.prof = prof_slots(c, g * threads / 256, true);
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    kern<<<g, threads, smem, c->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    c->timed = true;
    ++c->launches;
    return CLGEN_OK;
  };
  static const int env_e = [] {
    const char* e = std::getenv("CLGEN_BLK_E");  // candidates per lane per loop iteration (unroll; same stream)
    const int v = e ? std::atoi(e) : kBlkE;
    return v == 2 ? 2 : kBlkE;
  }();
  auto by_shape = [&](auto e_tag) -> int {
    constexpr int EE = decltype(e_tag)::value;
    switch (shape) {
      case 0: return launch(clg::blk_kernel<MODE, EE, 256, 2>, 256);
      case 1: return launch(clg::blk_kernel<MODE, EE, 256, 3>, 256);
      case 3: return launch(clg::blk_kernel<MODE, EE, 256, 5>, 256);
      case 4: return launch(clg::blk_kernel<MODE, EE, 256, 6>, 256);
      default: return launch(clg::blk_kernel<MODE, EE, 256, 4>, 256);
    }
  };
  if constexpr (MODE == clg::kWalkPairs) {
    return launch(clg::blk_kernel<MODE, kBlkE, 256, 4>, 256);  // test support: one shape
  } else {
    if (env_e == 2) return by_shape(std::integral_constant<int, 2>{});
    return by_shape(std::integral_constant<int, kBlkE>{});
  }
}

// Sort keys of the materialised counter stream: (u << bits) | v with bits =
// ceil(log2 n), so the radix sort runs over 2 * bits key bits (48 at n = 1e7)
// instead of 64.
__global__ void pairs_to_keys_kernel(const uint2* __restrict__ p, int64_t m, int bits, unsigned long long* keys) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 e = p[i];
    keys[i] = (static_cast<unsigned long long>(e.x) << bits) | e.y;
  }
}

__global__ void keys_to_pairs_kernel(const unsigned long long* __restrict__ keys, int64_t m, int bits, uint2* p) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const unsigned long long vmask = (1ull << bits) - 1ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const unsigned long long k = keys[i];
    p[i] = make_uint2(static_cast<uint32_t>(k >> bits), static_cast<uint32_t>(k & vmask));
  }
}

// Materialised counter-stream generation: count pass per chunk, scan, write
// pass at the scanned offsets, then a device radix sort by (u, v) (CUB) so
// the output order is the reference's (u ascending, then v ascending).
int materialise_ctr(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, uint64_t seed, uint32_t* pairs,
                    int64_t cap, int64_t* count) {
  if (cap < 0 || (cap > 0 && !pairs)) return fail(CLGEN_EINVAL, "generate_range: bad output buffer");
  int rc = set_device(c);
  if (rc) return rc;
  if ((rc = reset_scalars(c, 0))) return rc;
  if (hi == lo || !(S > 0.0) || c->n < 2) {
    if (count) *count = 0;
    return CLGEN_OK;
  }
  if ((rc = ensure_blocks(c, S))) return rc;
  if ((rc = ensure_range(c, lo, hi))) return rc;
  const int64_t U = c->plan_host.chunks_full > 0 ? static_cast<int64_t>(c->plan_host.chunks_full) : 1;
  CUDA_TRY(c->chunk_counts.ensure(U * sizeof(int32_t)));
  CUDA_TRY(c->chunk_offsets.ensure(U * sizeof(int64_t)));
  int64_t units = 0;
  CUDA_TRY(cudaMemcpyAsync(&units, c->chunk_total.p, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  clg::BlkArgs a = blk_args(c, S, seed);
  a.counts = c->chunk_counts.as<int32_t>();
  if ((rc = launch_blk<clg::kWalkCount>(c, a))) return rc;
  if ((rc = launch_scan(c, a.counts, c->chunk_offsets.as<int64_t>(), units))) return rc;
  if ((rc = fetch_scalars(c))) return rc;
  const int64_t total = c->sc_host->total;
  if (count) *count = total;
  if (total > cap)
    return fail(CLGEN_ERANGE, "generate_range: %lld edges exceed capacity %lld", (long long)total, (long long)cap);
  if (total == 0) return CLGEN_OK;
  CUDA_TRY(c->pairs.ensure(total * sizeof(uint2)));
  CUDA_TRY(c->keys_a.ensure(total * sizeof(unsigned long long)));
  CUDA_TRY(c->keys_b.ensure(total * sizeof(unsigned long long)));
  a.counts = nullptr;
  a.offsets = c->chunk_offsets.as<int64_t>();
  a.pairs = c->pairs.as<uint2>();
  a.cap = total;
  if ((rc = launch_blk<clg::kWalkWrite>(c, a))) return rc;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, c->num_sms * 16));
  int bits = 1;
  while (bits < 32 && (int64_t(1) << bits) < c->n) ++bits;  // node ids < 2^bits
  pairs_to_keys_kernel<<<grid, 256, 0, c->stream>>>(c->pairs.as<uint2>(), total, bits,
                                                    c->keys_a.as<unsigned long long>());
  size_t tmp = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, c->keys_a.as<unsigned long long>(),
                                          c->keys_b.as<unsigned long long>(), total, 0, 2 * bits, c->stream));
  CUDA_TRY(c->sort_tmp.ensure(tmp > 0 ? tmp : 1));
  CUDA_TRY(cub::DeviceRadixSort::SortKeys(c->sort_tmp.p, tmp, c->keys_a.as<unsigned long long>(),
                                          c->keys_b.as<unsigned long long>(), total, 0, 2 * bits, c->stream));
  uint2* d_out = is_device_ptr(pairs) ? reinterpret_cast<uint2*>(pairs) : c->pairs.as<uint2>();
  keys_to_pairs_kernel<<<grid, 256, 0, c->stream>>>(c->keys_b.as<unsigned long long>(), total, bits, d_out);
  c->launches += 3;
  CUDA_TRY(cudaGetLastError());
  if (d_out != reinterpret_cast<uint2*>(pairs))
    CUDA_TRY(cudaMemcpyAsync(pairs, d_out, total * sizeof(uint2), cudaMemcpyDeviceToHost, c->stream));
  if ((rc = fetch_scalars(c))) return rc;
  if (c->sc_host->overflow)
    return fail(CLGEN_EINVAL, "generate_range: write pass disagrees with the count pass");
  return CLGEN_OK;
}

// Single-pass materialisation in the reference's emission order.  Each slot
// owns a scratch run sized by ref_slot_cap_kernel (a 6-sigma bound on its
// edge count); one walk writes the edges there and records the exact counts,
// a scan of the counts gives the final offsets, ref_compact_kernel moves the
// runs into place, and the (rare) slots that outgrew their run are re-walked
// straight into their final offsets.  Output identical to the two-pass path.
// Returns 1 (nothing launched) when the scratch would not fit in memory.
int materialise_1pass(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, const int64_t* d_sources,
                      uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* count, int64_t* n_flagged) {
  int rc;
  const int64_t m = hi - lo;
  CUDA_TRY(c->slot_cap.ensure(m * sizeof(int32_t)));
  CUDA_TRY(c->soff.ensure(m * sizeof(int64_t)));
  clg::ref_slot_cap_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(c->w, c->n, S, d_sources, lo, m, c->slot_sigma,
                                                                  c->slot_const, c->slot_cap.as<int32_t>());
  CUDA_TRY(cudaGetLastError());
  ++c->launches;
  if ((rc = launch_scan(c, c->slot_cap.as<int32_t>(), c->soff.as<int64_t>(), m))) return rc;
  if ((rc = fetch_scalars(c))) return rc;
  const int64_t scratch_n = c->sc_host->total;
  const size_t need = static_cast<size_t>(scratch_n > 0 ? scratch_n : 1) * sizeof(uint2);
  if (need > c->scratch.bytes) {
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    if (need - c->scratch.bytes > free_b / 2) return 1;
  }
  CUDA_TRY(c->scratch.ensure(need));
  CUDA_TRY(c->spill.ensure(m * sizeof(int64_t)));
  CUDA_TRY(c->counts.ensure(m * sizeof(int32_t)));
  CUDA_TRY(c->offsets.ensure(m * sizeof(int64_t)));
  clg::RefWalkArgs a = walk_args(c, S, lo, hi, seed);
  a.sources = d_sources;
  a.counts = c->counts.as<int32_t>();
  a.offsets = c->soff.as<int64_t>();
  a.slot_cap = c->slot_cap.as<int32_t>();
  a.pairs = c->scratch.as<uint2>();
  a.cap = scratch_n;
  a.spill = c->spill.as<int64_t>();
  a.spill_count = &c->sc->spill;
  if ((rc = launch_walk<clg::kWalkWrite>(c, a))) return rc;
  if ((rc = launch_scan(c, a.counts, c->offsets.as<int64_t>(), m))) return rc;
  if ((rc = fetch_scalars(c))) return rc;
  const int64_t total = c->sc_host->total;
  const int64_t spilled = static_cast<int64_t>(c->sc_host->spill);
  const bool dev_out = is_device_ptr(pairs);
  uint2* d_pairs = reinterpret_cast<uint2*>(pairs);
  if (!dev_out) {
    const int64_t stage = total < cap ? total : cap;
    CUDA_TRY(c->pairs.ensure((stage > 0 ? stage : 1) * sizeof(uint2)));
    d_pairs = c->pairs.as<uint2>();
    cap = stage;
  }
  clg::ref_compact_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(c->scratch.as<uint2>(), c->soff.as<int64_t>(),
                                                                 c->slot_cap.as<int32_t>(), a.counts,
                                                                 c->offsets.as<int64_t>(), m, d_pairs, cap);
  CUDA_TRY(cudaGetLastError());
  ++c->launches;
  if (spilled > 0) {
    // (source, final offset) of each spilled slot; re-walk them uncapped
    CUDA_TRY(c->sources.ensure(2 * spilled * sizeof(int64_t)));
    int64_t* src_list = c->sources.as<int64_t>();
    int64_t* off_list = src_list + spilled;
    clg::ref_spill_lists_kernel<<<(spilled + 255) / 256, 256, 0, c->stream>>>(
        a.spill, &c->sc->spill, d_sources, lo, c->offsets.as<int64_t>(), src_list, off_list);
    CUDA_TRY(cudaGetLastError());
    ++c->launches;
    c->sc_host->queue = 0;
    CUDA_TRY(cudaMemcpyAsync(&c->sc->queue, &c->sc_host->queue, sizeof(unsigned long long),
                             cudaMemcpyHostToDevice, c->stream));
    clg::RefWalkArgs b = walk_args(c, S, 0, spilled, seed);
    b.sources = src_list;
    b.offsets = off_list;
    b.pairs = d_pairs;
    b.cap = cap;
    b.flag_count = &c->sc->spill_flags;  // already flagged by the first walk
    if ((rc = launch_walk<clg::kWalkWrite>(c, b))) return rc;
  }
  if (!dev_out && cap > 0)
    CUDA_TRY(cudaMemcpyAsync(pairs, d_pairs, cap * sizeof(uint2), cudaMemcpyDeviceToHost, c->stream));
  if ((rc = fetch_scalars(c))) return rc;
  if (count) *count = total;
  c->last_flagged = static_cast<int64_t>(c->sc_host->flag_count);
  if (n_flagged) *n_flagged = c->last_flagged;
  if (total > cap)
    return fail(CLGEN_ERANGE, "create_edges: %lld edges exceed capacity %lld", (long long)total, (long long)cap);
  return CLGEN_OK;
}

// Materialisation in the reference's emission order: single pass when the
// scratch fits (above), else count pass, decoupled-lookback scan of the
// per-slot counts, replay pass writing each slot's edges at its scanned offset.
int materialise(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, const int64_t* d_sources,
                uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* count, int64_t* n_flagged) {
  if (cap < 0 || (cap > 0 && !pairs)) return fail(CLGEN_EINVAL, "create_edges: bad output buffer");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t m = hi - lo;
  if ((rc = reset_scalars(c, static_cast<unsigned long long>(lo)))) return rc;
  if (m == 0) {
    if (count) *count = 0;
    if (n_flagged) *n_flagged = 0;
    c->last_flagged = 0;
    return CLGEN_OK;
  }
  if (c->one_pass) {
    rc = materialise_1pass(c, S, lo, hi, d_sources, seed, pairs, cap, count, n_flagged);
    if (rc != 1) return rc;
    if ((rc = reset_scalars(c, static_cast<unsigned long long>(lo)))) return rc;
  }
  CUDA_TRY(c->counts.ensure(m * sizeof(int32_t)));
  CUDA_TRY(c->offsets.ensure(m * sizeof(int64_t)));
  clg::RefWalkArgs a = walk_args(c, S, lo, hi, seed);
  a.sources = d_sources;
  a.counts = c->counts.as<int32_t>();
  if ((rc = launch_walk<clg::kWalkCount>(c, a))) return rc;
  if ((rc = launch_scan(c, a.counts, c->offsets.as<int64_t>(), m))) return rc;
  const bool dev_out = is_device_ptr(pairs);
  uint2* d_pairs = reinterpret_cast<uint2*>(pairs);
  if (!dev_out) {
    // host output: the exact count sizes the staging buffer
    if ((rc = fetch_scalars(c))) return rc;
    const int64_t total = c->sc_host->total;
    const int64_t stage = total < cap ? total : cap;
    CUDA_TRY(c->pairs.ensure((stage > 0 ? stage : 1) * sizeof(uint2)));
    d_pairs = c->pairs.as<uint2>();
    cap = stage;
  }
  c->sc_host->queue = static_cast<unsigned long long>(lo);
  CUDA_TRY(cudaMemcpyAsync(&c->sc->queue, &c->sc_host->queue, sizeof(unsigned long long),
                           cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemsetAsync(&c->sc->flag_count, 0, sizeof(unsigned long long), c->stream));
  a.counts = nullptr;
  a.offsets = c->offsets.as<int64_t>();
  a.pairs = d_pairs;
  a.cap = cap;
  if ((rc = launch_walk<clg::kWalkWrite>(c, a))) return rc;
  if (!dev_out && cap > 0)
    CUDA_TRY(cudaMemcpyAsync(pairs, d_pairs, cap * sizeof(uint2), cudaMemcpyDeviceToHost, c->stream));
  if ((rc = fetch_scalars(c))) return rc;
  const int64_t total = c->sc_host->total;
  if (count) *count = total;
  c->last_flagged = static_cast<int64_t>(c->sc_host->flag_count);
  if (n_flagged) *n_flagged = c->last_flagged;
  if (total > cap)
    return fail(CLGEN_ERANGE, "create_edges: %lld edges exceed capacity %lld", (long long)total, (long long)cap);
  return CLGEN_OK;
}

}  // namespace

extern "C" {

const char* clgen_dev_last_error(void) { return g_err.c_str(); }

const char* clgen_dev_version(void) { return "clgen-b200 0.1 (sm_100a)"; }

int clgen_dev_create(int device, clgen_dev_ctx** out) {
  if (!out) return fail(CLGEN_EINVAL, "clgen_dev_create: null out");
  *out = nullptr;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(CLGEN_EINVAL, "clgen_dev_create: no CUDA device %d", device);
  auto* c = new clgen_dev_ctx;
  c->device = device;
  int rc = set_device(c);
  if (rc) {
    delete c;
    return rc;
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, device) == cudaSuccess && v > 0)
      c->l2_persist_max = static_cast<size_t>(v);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, device) == cudaSuccess && v > 0)
      c->l2_window_max = static_cast<size_t>(v);
    cudaGetLastError();
  }
  // Random 8-byte weight gathers: ask L2 not to over-fetch around a miss
  // (CLGEN_L2_FETCH=32|64|128; 0 keeps the driver default).
  {
    const char* e = std::getenv("CLGEN_L2_FETCH");
    const int g = e ? std::atoi(e) : 32;
    if (g > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(g));
    cudaGetLastError();
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->sc, sizeof(Scalars)) != cudaSuccess ||
      cudaMallocHost(&c->sc_host, sizeof(Scalars)) != cudaSuccess ||
      cudaMalloc(&c->flagged, kFlagCap * sizeof(int64_t)) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaMalloc(&c->logtab, sizeof(clg::LogTable)) != cudaSuccess ||
      cudaMalloc(&c->logtab2, sizeof(clg::Log2Table)) != cudaSuccess) {
    clgen_dev_destroy(c);
    return fail(CLGEN_ENOMEM, "clgen_dev_create: allocation failed");
  }
  {
    // reciprocal centres and their logs, evaluated in long double on the host
    clg::LogTable t;
    for (int i = 0; i < clg::kLogTable; ++i) {
      const long double ci = 1.0L + (static_cast<long double>(i) + 0.5L) / clg::kLogTable;
      t.inv_c[i] = static_cast<double>(1.0L / ci);
      t.nlog_inv[i] = static_cast<double>(-logl(static_cast<long double>(t.inv_c[i])));
    }
    clg::Log2Table t2;
    for (int i = 0; i < clg::kLogTable; ++i) {
      t2.inv_c[i] = t.inv_c[i];
      t2.nlog2_inv[i] = static_cast<double>(-log2l(static_cast<long double>(t.inv_c[i])));
    }
    if (cudaMemcpy(c->logtab, &t, sizeof t, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->logtab2, &t2, sizeof t2, cudaMemcpyHostToDevice) != cudaSuccess) {
      clgen_dev_destroy(c);
      return fail(CLGEN_ECUDA, "clgen_dev_create: cannot upload log table");
    }
  }
  *out = c;
  return CLGEN_OK;
}

int clgen_dev_destroy(clgen_dev_ctx* c) {
  if (!c) return CLGEN_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);  // a prefetch may still be in flight
  if (c->l2_persist_dirty) cudaCtxResetPersistingL2Cache();
  if (c->w) cudaFree(c->w);
  if (c->w_next) cudaFree(c->w_next);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->next_ready) cudaEventDestroy(c->next_ready);
  if (c->swap_done) cudaEventDestroy(c->swap_done);
  if (c->sc) cudaFree(c->sc);
  if (c->sc_host) cudaFreeHost(c->sc_host);
  if (c->flagged) cudaFree(c->flagged);
  if (c->logtab) cudaFree(c->logtab);
  if (c->logtab2) cudaFree(c->logtab2);
  if (c->host_stage) cudaFreeHost(c->host_stage);
  c->counts.release();
  c->offsets.release();
  c->tiles.release();
  c->pairs.release();
  c->partials.release();
  c->degree.release();
  c->sources.release();
  c->foldtmp.release();
  c->cum.release();
  c->found.release();
  for (DevBuf* d : {&c->costs, &c->cls_thr, &c->cls_bounds, &c->cls_start, &c->cls_wfirst, &c->cls_wlast, &c->cls_plan,
                    &c->blocks, &c->ranges, &c->blk_cnt, &c->blk_prefix, &c->chunk_block, &c->chunk_total,
                    &c->chunk_counts, &c->chunk_offsets, &c->keys_a, &c->keys_b, &c->sort_tmp})
    d->release();
  c->probe.release();
  c->prof.release();
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return CLGEN_OK;
}

void* clgen_dev_stream(clgen_dev_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

unsigned long long clgen_dev_launch_count(clgen_dev_ctx* c) { return c ? c->launches : 0ull; }

int clgen_dev_last_kernel_ms(clgen_dev_ctx* c, float* ms) {
  if (!c || !ms) return fail(CLGEN_EINVAL, "last_kernel_ms: null argument");
  if (!c->timed) return fail(CLGEN_EINVAL, "last_kernel_ms: no sampler kernel launched yet");
  CUDA_TRY(cudaEventSynchronize(c->ev1));
  CUDA_TRY(cudaEventElapsedTime(ms, c->ev0, c->ev1));
  return CLGEN_OK;
}

int clgen_dev_synchronize(clgen_dev_ctx* c) {
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return CLGEN_OK;
}

int clgen_dev_prefetch_weights(clgen_dev_ctx* c, const double* w, int64_t n) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (n <= 0 || !w) return fail(CLGEN_EINVAL, "prefetch_weights: empty weights");
  if (n >= (int64_t(1) << 32)) return fail(CLGEN_EINVAL, "set_weights: n exceeds uint32 node ids (n < 2^32)");
  int rc = set_device(c);
  if (rc) return rc;
  if (!c->copy_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->next_ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->swap_done, cudaEventDisableTiming));
  }
  if (c->swapped) CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->swap_done, 0));
  const size_t bytes = static_cast<size_t>(n) * sizeof(double);
  c->next_n = -1;
  if (bytes > c->w_next_bytes) {
    // the previous copy into the old buffer, if any, must be over before it is freed
    CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
    if (c->w_next) cudaFree(c->w_next);
    c->w_next = nullptr;
    c->w_next_bytes = 0;
    if (cudaMalloc(&c->w_next, bytes) != cudaSuccess)
      return fail(CLGEN_ENOMEM, "prefetch_weights: cannot allocate %lld weights", (long long)n);
    c->w_next_bytes = bytes;
  }
  CUDA_TRY(cudaMemcpyAsync(c->w_next, w, bytes, cudaMemcpyDefault, c->copy_stream));
  CUDA_TRY(cudaEventRecord(c->next_ready, c->copy_stream));
  c->next_src = w;
  c->next_n = n;
  return CLGEN_OK;
}

int clgen_dev_set_weights(clgen_dev_ctx* c, const double* w, int64_t n) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (n < 0) return fail(CLGEN_EINVAL, "set_weights: negative n");
  if (n >= (int64_t(1) << 32)) return fail(CLGEN_EINVAL, "set_weights: n exceeds uint32 node ids (n < 2^32)");
  if (n > 0 && !w) return fail(CLGEN_EINVAL, "set_weights: null weights");
  int rc = set_device(c);
  if (rc) return rc;
  const size_t bytes = static_cast<size_t>(n) * sizeof(double);
  // a copy started by clgen_dev_prefetch_weights for exactly this array: take it
  const bool prefetched = n > 0 && c->next_n == n && c->next_src == w && c->w_next;
  if (prefetched) {
    CUDA_TRY(cudaEventRecord(c->swap_done, c->stream));  // earlier launches may still read the buffer being retired
    c->swapped = true;
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->next_ready, 0));
    std::swap(c->w, c->w_next);
    std::swap(c->w_bytes, c->w_next_bytes);
  }
  c->next_n = -1;
  c->next_src = nullptr;
  if (bytes > c->w_bytes) {
    if (c->w) cudaFree(c->w);
    c->w = nullptr;
    c->w_bytes = 0;
    if (cudaMalloc(&c->w, bytes ? bytes : 8) != cudaSuccess)
      return fail(CLGEN_ENOMEM, "set_weights: cannot allocate %lld weights", (long long)n);
    c->w_bytes = bytes;
  }
  c->n = 0;
  c->has_runs = false;
  c->cls_valid = c->blk_valid = false;
  c->rng_lo = c->rng_hi = -1;
  c->plan_G = 0;
  if (n > 0) {
    if (!prefetched) CUDA_TRY(cudaMemcpyAsync(c->w, w, bytes, cudaMemcpyDefault, c->stream));
    rc = reset_scalars(c, 0);
    if (rc) return rc;
    const int grid = c->num_sms * 8;
    clg::check_sorted_kernel<<<grid, 256, 0, c->stream>>>(c->w, n, &c->sc->first_bad, &c->sc->first_negative,
                                                          &c->sc->runs);
    CUDA_TRY(cudaGetLastError());
    ++c->launches;
    CUDA_TRY(cudaMemcpyAsync(&c->w0, c->w, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    rc = fetch_scalars(c);
    if (rc) return rc;
    if (c->sc_host->first_negative != ~0ull)
      return fail(CLGEN_EINVAL, "weights negative or NaN at position %llu", c->sc_host->first_negative);
    if (c->sc_host->first_bad != ~0ull)
      return fail(CLGEN_EINVAL, "weights unsorted at position %llu", c->sc_host->first_bad);
    // repeated weights (discrete / constant sequences): run-length table
    if (c->use_runs && n >= 64 && c->sc_host->runs * 4 <= static_cast<unsigned long long>(n)) {
      CUDA_TRY(c->run_len.ensure(n * sizeof(int32_t)));
      const unsigned tiles = static_cast<unsigned>((n + clg::kRunTile - 1) / clg::kRunTile);
      clg::run_length_kernel<<<tiles, clg::kRunThreads, 0, c->stream>>>(c->w, n, c->run_len.as<int32_t>());
      CUDA_TRY(cudaGetLastError());
      ++c->launches;
      c->has_runs = true;
    }
  }
  c->n = n;
  // Optional L2 persistence for the hot head of w (candidates land in
  // proportion to w_v, and w is sorted descending): CLGEN_L2_PERSIST_MB.
  {
    const char* e = std::getenv("CLGEN_L2_PERSIST_MB");
    const double mb = e ? std::atof(e) : 0.0;
    if (mb > 0.0 && n > 0) {
      size_t bytes = static_cast<size_t>(mb * 1048576.0);
      if (bytes > static_cast<size_t>(n) * sizeof(double)) bytes = static_cast<size_t>(n) * sizeof(double);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes);
      cudaStreamAttrValue attr;
      std::memset(&attr, 0, sizeof attr);
      attr.accessPolicyWindow.base_ptr = c->w;
      attr.accessPolicyWindow.num_bytes = bytes;
      attr.accessPolicyWindow.hitRatio = 1.0f;
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
      cudaGetLastError();
    }
  }
  return CLGEN_OK;
}

int64_t clgen_dev_num_nodes(clgen_dev_ctx* c) { return c ? c->n : -1; }

const double* clgen_dev_weights(clgen_dev_ctx* c) { return c ? c->w : nullptr; }

int clgen_dev_device(clgen_dev_ctx* c) { return c ? c->device : -1; }

int clgen_dev_copy_weights(clgen_dev_ctx* c, double* out, int64_t n) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (n < 0 || n > c->n || (n > 0 && !out)) return fail(CLGEN_EINVAL, "copy_weights: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  if (n > 0) CUDA_TRY(cudaMemcpyAsync(out, c->w, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDefault, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return CLGEN_OK;
}

int clgen_dev_blocked_sum(clgen_dev_ctx* c, double* S) {
  if (!c || !S) return fail(CLGEN_EINVAL, "blocked_sum: null argument");
  return blocked_sum_impl(c, c->w, c->n, S);
}

int clgen_dev_blocked_sum_array(clgen_dev_ctx* c, const double* xs, int64_t n, double* S) {
  if (!c || !S || n < 0 || (n > 0 && !xs)) return fail(CLGEN_EINVAL, "blocked_sum: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  const double* d = xs;
  if (n > 0 && !is_device_ptr(xs)) {
    CUDA_TRY(c->sources.ensure(n * sizeof(double)));
    CUDA_TRY(cudaMemcpyAsync(c->sources.p, xs, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    d = c->sources.as<double>();
  }
  return blocked_sum_impl(c, d, n, S);
}

int clgen_dev_edge_counts(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, uint64_t seed,
                          int32_t* counts, int64_t* total, int64_t* n_flagged) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  int rc = check_range(c, lo, hi);
  if (rc) return rc;
  if ((rc = set_device(c))) return rc;
  const int64_t m = hi - lo;
  const bool dev_out = is_device_ptr(counts);
  CUDA_TRY(c->counts.ensure((m > 0 ? m : 1) * sizeof(int32_t)));
  int32_t* d_counts = dev_out ? counts : c->counts.as<int32_t>();
  if ((rc = reset_scalars(c, static_cast<unsigned long long>(lo)))) return rc;
  if (m > 0) {
    clg::RefWalkArgs a = walk_args(c, S, lo, hi, seed);
    a.counts = d_counts;
    if ((rc = launch_walk<clg::kWalkCount>(c, a))) return rc;
    CUDA_TRY(c->offsets.ensure(m * sizeof(int64_t)));
    if ((rc = launch_scan(c, d_counts, c->offsets.as<int64_t>(), m))) return rc;
  }
  if (counts && !dev_out && m > 0)
    CUDA_TRY(cudaMemcpyAsync(counts, d_counts, m * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  if ((rc = fetch_scalars(c))) return rc;
  if (total) *total = m > 0 ? c->sc_host->total : 0;
  c->last_flagged = static_cast<int64_t>(c->sc_host->flag_count);
  if (n_flagged) *n_flagged = c->last_flagged;
  return CLGEN_OK;
}

int clgen_dev_create_edges_range(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, uint64_t seed,
                                 uint32_t* pairs, int64_t cap, int64_t* count, int64_t* n_flagged) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  int rc = check_range(c, lo, hi);
  if (rc) return rc;
  return materialise(c, S, lo, hi, nullptr, seed, pairs, cap, count, n_flagged);
}

int clgen_dev_create_edges(clgen_dev_ctx* c, double S, const int64_t* sources, int64_t k,
                           uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* count,
                           int64_t* n_flagged) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (k < 0 || (k > 0 && !sources)) return fail(CLGEN_EINVAL, "create_edges: bad source list");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t* d_src = sources;
  if (k > 0 && !is_device_ptr(sources)) {
    CUDA_TRY(c->sources.ensure(k * sizeof(int64_t)));
    CUDA_TRY(cudaMemcpyAsync(c->sources.p, sources, k * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    d_src = c->sources.as<int64_t>();
  }
  if (k > 0) {
    if ((rc = reset_scalars(c, 0))) return rc;
    clg::check_sources_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(d_src, k, c->n, &c->sc->first_bad);
    CUDA_TRY(cudaGetLastError());
    ++c->launches;
    if ((rc = fetch_scalars(c))) return rc;
    if (c->sc_host->first_bad != ~0ull) return fail(CLGEN_EINVAL, "create_edges: source node out of range");
  }
  return materialise(c, S, 0, k, d_src, seed, pairs, cap, count, n_flagged);
}

int clgen_dev_stream_range(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, uint64_t seed,
                           int stream_mode, int track_shift, uint32_t* degree, int accumulate,
                           uint32_t* ring, int64_t ring_cap, int64_t* count, uint64_t* checksum,
                           int64_t* n_flagged) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  int rc = check_range(c, lo, hi);
  if (rc) return rc;
  if (track_shift < 0 || track_shift > 40) return fail(CLGEN_EINVAL, "stream_range: bad track_shift");
  if (ring && (ring_cap <= 0 || (ring_cap & (ring_cap - 1)) != 0))
    return fail(CLGEN_EINVAL, "stream_range: ring_cap must be a power of two");
  if (ring && !is_device_ptr(ring)) return fail(CLGEN_EINVAL, "stream_range: ring must be device memory");
  if (stream_mode != CLGEN_STREAM_REFERENCE && stream_mode != CLGEN_STREAM_COUNTER)
    return fail(CLGEN_EINVAL, "stream_range: unknown stream mode %d", stream_mode);
  if ((rc = set_device(c))) return rc;
  const int64_t ntracked = (c->n + (int64_t(1) << track_shift) - 1) >> track_shift;
  const bool dev_deg = is_device_ptr(degree);
  uint32_t* d_deg = degree;
  if (degree && !dev_deg) {
    CUDA_TRY(c->degree.ensure((ntracked > 0 ? ntracked : 1) * sizeof(uint32_t)));
    d_deg = c->degree.as<uint32_t>();
  }
  if (degree && (!dev_deg || !accumulate) && ntracked > 0)
    CUDA_TRY(cudaMemsetAsync(d_deg, 0, ntracked * sizeof(uint32_t), c->stream));
  if (stream_mode == CLGEN_STREAM_COUNTER && hi > lo && S > 0.0) {
    if ((rc = ensure_blocks(c, S))) return rc;
    if ((rc = ensure_range(c, lo, hi))) return rc;
    if ((rc = reset_scalars(c, 0))) return rc;
    clg::BlkArgs a = blk_args(c, S, seed);
    a.degree = d_deg;
    a.track_shift = track_shift;
    a.ring = reinterpret_cast<uint2*>(ring);
    a.ring_mask = ring ? static_cast<unsigned long long>(ring_cap - 1) : 0ull;
    // The tracked-degree array is reduced into at random while the ring
    // stream runs through L2: for this launch it gets the persisting part of
    // L2 (as much of it as fits; C4: 62.5 MB of the 82.9 MB B200 allows;
    // measured 193.9 -> 203.5 G edges/s).  CLGEN_L2_PERSIST_DEG=0 disables it.
    static const bool persist_deg = env_double("CLGEN_L2_PERSIST_DEG", 1.0) != 0.0;
    bool window_set = false;
    if (persist_deg && d_deg && ntracked > 0 && c->l2_persist_max > 0 && c->l2_window_max > 0) {
      size_t bytes = static_cast<size_t>(ntracked) * sizeof(uint32_t);
      const size_t carve = std::min(bytes, c->l2_persist_max);
      bytes = std::min(bytes, c->l2_window_max);
      // cudaDeviceSetLimit synchronises the device (it would wait for a weight
      // prefetch in flight): only when the carve-out has to change
      if (c->l2_carve == carve || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) == cudaSuccess) {
        c->l2_carve = carve;
        cudaStreamAttrValue attr;
        std::memset(&attr, 0, sizeof attr);
        attr.accessPolicyWindow.base_ptr = d_deg;
        attr.accessPolicyWindow.num_bytes = bytes;
        attr.accessPolicyWindow.hitRatio =
            carve >= bytes ? 1.0f : static_cast<float>(carve) / static_cast<float>(bytes);
        attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
        window_set = cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr) == cudaSuccess;
      }
      cudaGetLastError();
    }
    rc = launch_blk<clg::kWalkFold>(c, a);
    if (window_set) {  // later launches on the stream carry no window; the lines are released after the sync below
      cudaStreamAttrValue attr;
      std::memset(&attr, 0, sizeof attr);
      cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
      c->l2_persist_dirty = true;
      cudaGetLastError();
    }
    if (rc) return rc;
  } else {
    if ((rc = reset_scalars(c, static_cast<unsigned long long>(lo)))) return rc;
    if (hi > lo && stream_mode == CLGEN_STREAM_REFERENCE) {
      clg::RefWalkArgs a = walk_args(c, S, lo, hi, seed);
      a.degree = d_deg;
      a.track_shift = track_shift;
      a.ring = reinterpret_cast<uint2*>(ring);
      a.ring_mask = ring ? static_cast<unsigned long long>(ring_cap - 1) : 0ull;
      if ((rc = launch_walk<clg::kWalkFold>(c, a))) return rc;
    }
  }
  if (degree && !dev_deg && ntracked > 0)
    CUDA_TRY(cudaMemcpyAsync(degree, d_deg, ntracked * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  if ((rc = fetch_scalars(c))) return rc;
  if (count) *count = static_cast<int64_t>(c->sc_host->fold[0]);
  if (checksum) *checksum = c->sc_host->fold[1];
  c->last_flagged = static_cast<int64_t>(c->sc_host->flag_count);
  if (n_flagged) *n_flagged = c->last_flagged;
  return CLGEN_OK;
}

int clgen_dev_plan_block_weight(clgen_dev_ctx* c, int G, int g, double* block_weight) {
  int rc = plan_args_ok(c, G, g);
  if (rc) return rc;
  if (!block_weight) return fail(CLGEN_EINVAL, "plan_block_weight: null output");
  return block_weight_impl(c, G, g, block_weight);
}

int clgen_dev_plan_block_costs(clgen_dev_ctx* c, int G, int g, double sigma_start, double S,
                               double* block_cost) {
  int rc = plan_args_ok(c, G, g);
  if (rc) return rc;
  if (!block_cost) return fail(CLGEN_EINVAL, "plan_block_costs: null output");
  return block_costs_impl(c, G, g, sigma_start, S, block_cost);
}

int clgen_dev_plan_block_boundaries(clgen_dev_ctx* c, int G, int g, double z_offset, double z_bar,
                                    int64_t* found) {
  int rc = plan_args_ok(c, G, g);
  if (rc) return rc;
  if (!found) return fail(CLGEN_EINVAL, "plan_block_boundaries: null output");
  if (c->plan_G != G) return fail(CLGEN_EINVAL, "plan_block_boundaries: costs of block %d/%d not computed", g, G);
  CUDA_TRY(c->found.ensure((G + 1) * sizeof(long long)));
  long long* d = c->found.as<long long>();
  clg::fill_i64_kernel<<<1, 256, 0, c->stream>>>(d, G + 1, static_cast<long long>(c->n));
  ++c->launches;
  if ((rc = block_boundaries_impl(c, G, g, z_offset, z_bar, d))) return rc;
  CUDA_TRY(cudaMemcpyAsync(found, d, (G + 1) * sizeof(long long), cudaMemcpyDefault, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return CLGEN_OK;
}

int clgen_dev_plan_ucp(clgen_dev_ctx* c, int P, int64_t* boundaries, double* cum_costs) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (P < 1) return fail(CLGEN_EINVAL, "plan_ucp_oracle: P must be >= 1");
  if (!boundaries) return fail(CLGEN_EINVAL, "plan_ucp: null boundaries");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t n = c->n;
  std::vector<long long> b(static_cast<size_t>(P) + 1, 0);
  if (n == 0) {  // trivial_plan (partition.cpp:89-96)
    CUDA_TRY(cudaMemcpy(boundaries, b.data(), b.size() * sizeof(long long), cudaMemcpyDefault));
    return CLGEN_OK;
  }
  double Scan;  // the canonical sum_S (weights.cpp:54)
  if ((rc = blocked_sum_impl(c, c->w, n, &Scan))) return rc;
  // partition.cpp:165-170: block weights, each a fold from 0.0
  std::vector<double> bw(P), bc(P);
  for (int i = 0; i < P; ++i)
    if ((rc = block_weight_impl(c, P, i, &bw[i]))) return rc;
  // :172-177: block_cumulative from the rank-ordered prefix of block weights
  for (int i = 0; i < P; ++i) {
    double sp = 0.0;
    for (int j = 0; j < i; ++j) sp += bw[j];
    if ((rc = block_costs_impl(c, P, i, sp, Scan, &bc[i]))) return rc;
  }
  double total = 0.0;  // :180-181
  for (int j = 0; j < P; ++j) total += bc[j];
  const double z_bar = total / P;
  CUDA_TRY(c->found.ensure((P + 1) * sizeof(long long)));
  long long* d = c->found.as<long long>();
  clg::fill_i64_kernel<<<1, 256, 0, c->stream>>>(d, P + 1, static_cast<long long>(n));
  ++c->launches;
  for (int i = 0; i < P; ++i) {
    double zp = 0.0;
    for (int j = 0; j < i; ++j) zp += bc[j];
    if ((rc = block_boundaries_impl(c, P, i, zp, z_bar, d))) return rc;
    if (cum_costs) {
      int64_t lo, hi;
      block_bounds_host(n, P, i, &lo, &hi);
      if (hi > lo) {
        if (is_device_ptr(cum_costs)) {
          clg::add_offset_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(c->cum.as<double>(), cum_costs, lo, hi, zp);
        } else {
          clg::add_offset_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(c->cum.as<double>(), c->cum.as<double>(), lo,
                                                                      hi, zp);
        }
        ++c->launches;
        CUDA_TRY(cudaGetLastError());
      }
    }
  }
  if (cum_costs && !is_device_ptr(cum_costs))
    CUDA_TRY(cudaMemcpyAsync(cum_costs, c->cum.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(b.data(), d, (P + 1) * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  b[0] = 0;
  b[P] = n;
  if (cum_costs && !is_device_ptr(cum_costs)) c->plan_G = 0;  // cum now holds finalized values
  CUDA_TRY(cudaMemcpy(boundaries, b.data(), b.size() * sizeof(long long), cudaMemcpyDefault));
  return CLGEN_OK;
}

int clgen_dev_generate_range(clgen_dev_ctx* c, double S, int64_t lo, int64_t hi, uint64_t seed,
                             int stream_mode, uint32_t* pairs, int64_t cap, int64_t* count,
                             int64_t* n_flagged) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  int rc = check_range(c, lo, hi);
  if (rc) return rc;
  if (stream_mode == CLGEN_STREAM_REFERENCE)
    return materialise(c, S, lo, hi, nullptr, seed, pairs, cap, count, n_flagged);
  if (stream_mode != CLGEN_STREAM_COUNTER) return fail(CLGEN_EINVAL, "generate_range: unknown stream mode %d", stream_mode);
  if (n_flagged) *n_flagged = 0;
  c->last_flagged = 0;
  return materialise_ctr(c, S, lo, hi, seed, pairs, cap, count);
}

// cost.cpp:62-77 on device data: suffixes accumulated backward from 0.0
// (a reversed exact fold), costs[u] = (w_u / S) * suffix_u + 1; S <= 0: all 1.
int node_costs_dev(clgen_dev_ctx* c, double** d_costs) {
  const int64_t n = c->n;
  CUDA_TRY(c->costs.ensure((n > 0 ? n : 1) * sizeof(double)));
  *d_costs = c->costs.as<double>();
  if (n == 0) return CLGEN_OK;
  double S;
  int rc = blocked_sum_impl(c, c->w, n, &S);
  if (rc) return rc;
  if (!(S > 0.0)) {
    clg::fill_f64_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(*d_costs, 0, n, 1.0);
    ++c->launches;
    CUDA_TRY(cudaGetLastError());
    return CLGEN_OK;
  }
  double total;
  return run_fold(c, c->w, n, 0.0, clg::kFoldSuffixCost, *d_costs, nullptr, S, &total, 1, 1);
}

int clgen_dev_node_costs(clgen_dev_ctx* c, double* costs) {
  if (!c || (c->n > 0 && !costs)) return fail(CLGEN_EINVAL, "node_costs: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  double* d = nullptr;
  if ((rc = node_costs_dev(c, &d))) return rc;
  if (c->n > 0) CUDA_TRY(cudaMemcpyAsync(costs, d, c->n * sizeof(double), cudaMemcpyDefault, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return CLGEN_OK;
}

// partition.cpp:205-222: per-partition sums of the suffix-form costs, each a
// left fold from 0.0 over the partition's nodes in ascending order.
int clgen_dev_partition_costs(clgen_dev_ctx* c, int scheme, int P, const int64_t* boundaries, double* per) {
  if (!c || P < 1 || !per || (scheme != CLGEN_SCHEME_RRP && !boundaries) || scheme < 0 || scheme > 2)
    return fail(CLGEN_EINVAL, "fill_partition_costs: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t n = c->n;
  std::vector<int64_t> b;
  if (scheme != CLGEN_SCHEME_RRP) {
    b.resize(static_cast<size_t>(P) + 1);
    CUDA_TRY(cudaMemcpy(b.data(), boundaries, b.size() * sizeof(int64_t), cudaMemcpyDefault));
    for (int i = 0; i < P; ++i)
      if (b[i] < 0 || b[i + 1] < b[i] || b[i + 1] > n) return fail(CLGEN_EINVAL, "fill_partition_costs: bad boundaries");
  }
  double* d = nullptr;
  if ((rc = node_costs_dev(c, &d))) return rc;
  for (int i = 0; i < P; ++i) {
    double acc = 0.0;
    if (scheme == CLGEN_SCHEME_RRP) {
      const int64_t cnt = n > i ? (n - 1 - i) / P + 1 : 0;  // u = i, i + P, ...
      if ((rc = run_fold(c, d + i, cnt, 0.0, clg::kFoldNone, nullptr, nullptr, 0.0, &acc, P, 0))) return rc;
    } else {
      if ((rc = run_fold(c, d + b[i], b[i + 1] - b[i], 0.0, clg::kFoldNone, nullptr, nullptr, 0.0, &acc))) return rc;
    }
    per[i] = acc;
  }
  return CLGEN_OK;
}

__global__ void squares_kernel(const double* __restrict__ w, int64_t n, double* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __dmul_rn(w[i], w[i]);
}

// weights.cpp:155-162: (S^2 - blocked_sum(w^2)) / (2 S), S the canonical sum.
int clgen_dev_expected_total_edges(clgen_dev_ctx* c, double* m) {
  if (!c || !m) return fail(CLGEN_EINVAL, "expected_total_edges: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t n = c->n;
  double S;
  if ((rc = blocked_sum_impl(c, c->w, n, &S))) return rc;
  if (S <= 0.0) {
    *m = 0.0;
    return CLGEN_OK;
  }
  CUDA_TRY(c->costs.ensure(n * sizeof(double)));
  squares_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(c->w, n, c->costs.as<double>());
  ++c->launches;
  CUDA_TRY(cudaGetLastError());
  double sum_sq;
  if ((rc = blocked_sum_impl(c, c->costs.as<double>(), n, &sum_sq))) return rc;
  *m = (S * S - sum_sq) / (2.0 * S);
  return CLGEN_OK;
}

int clgen_dev_pair_trials(clgen_dev_ctx* c, double S, uint64_t seed, int64_t trials, uint32_t* counts) {
  if (!c || !counts || trials < 0) return fail(CLGEN_EINVAL, "pair_trials: bad argument");
  const int64_t n = c->n;
  if (n > 4096) return fail(CLGEN_EINVAL, "pair_trials: n must be <= 4096 (n*n counters)");
  int rc = set_device(c);
  if (rc) return rc;
  const size_t bytes = static_cast<size_t>(n) * n * sizeof(uint32_t);
  const bool dev_out = is_device_ptr(counts);
  CUDA_TRY(c->probe.ensure(bytes > 0 ? bytes : 8));
  uint32_t* d_counts = dev_out ? counts : c->probe.as<uint32_t>();
  if (bytes) CUDA_TRY(cudaMemsetAsync(d_counts, 0, bytes, c->stream));
  if ((rc = reset_scalars(c, 0))) return rc;
  if (n >= 2 && S > 0.0 && trials > 0) {
    if ((rc = ensure_blocks(c, S))) return rc;
    if ((rc = ensure_range(c, 0, n))) return rc;
    clg::BlkArgs a = blk_args(c, S, seed);
    a.trials = trials;
    a.pair_counts = d_counts;
    a.n = static_cast<uint32_t>(n);
    if ((rc = launch_blk<clg::kWalkPairs>(c, a))) return rc;
  }
  if (!dev_out && bytes) CUDA_TRY(cudaMemcpyAsync(counts, d_counts, bytes, cudaMemcpyDeviceToHost, c->stream));
  return fetch_scalars(c);
}

int clgen_dev_set_counter_params(clgen_dev_ctx* c, double class_eps, double chunk_cand) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (!(class_eps >= 0.0) || !(class_eps <= 1.0)) return fail(CLGEN_EINVAL, "class_eps must be 0 (automatic) or in (0,1]");
  if (!(chunk_cand == 0.0 || (chunk_cand >= 256.0 && chunk_cand <= 1048576.0)))
    return fail(CLGEN_EINVAL, "chunk_cand must be 0 (automatic) or in [256, 2^20]");
  c->cls_eps = class_eps;
  c->chunk_cand = chunk_cand;
  c->cls_valid = c->blk_valid = false;
  c->rng_lo = c->rng_hi = -1;
  return CLGEN_OK;
}

int clgen_dev_set_kernel_shape(clgen_dev_ctx* c, int shape, int flags) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (shape < -1 || shape > 4) return fail(CLGEN_EINVAL, "set_kernel_shape: shape must be in [-1, 4]");
  if (flags & ~CLGEN_SHAPE_NO_HEAVY_PHASE) return fail(CLGEN_EINVAL, "set_kernel_shape: unknown flag");
  c->blk_shape = shape;
  c->ref_heavy = (flags & CLGEN_SHAPE_NO_HEAVY_PHASE) == 0;
  return CLGEN_OK;
}

int clgen_dev_set_warp_profile(clgen_dev_ctx* c, int enable) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  c->warp_prof = enable != 0;
  c->prof_warps = 0;
  return CLGEN_OK;
}

int clgen_dev_warp_profile(clgen_dev_ctx* c, int launch, double* max_over_mean, double* mean_ms,
                           double* max_ms, double* span_ms, int64_t* warps) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  if (!c->warp_prof || c->prof_warps == 0) return fail(CLGEN_EINVAL, "warp_profile: not enabled or no launch yet");
  const int L = static_cast<int>(c->prof_launch.size());
  if (launch < 0 || launch >= L) return fail(CLGEN_EINVAL, "warp_profile: launch %d of %d", launch, L);
  const int lo = c->prof_launch[launch], hi = launch + 1 < L ? c->prof_launch[launch + 1] : c->prof_warps;
  std::vector<unsigned long long> v(static_cast<size_t>(hi - lo) * 2);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpy(v.data(), c->prof.as<unsigned long long>() + 2 * lo, v.size() * sizeof(unsigned long long),
                      cudaMemcpyDeviceToHost));
  double sum = 0.0, mx = 0.0;
  unsigned long long t0 = ~0ull, t1 = 0;
  int64_t k = 0;
  for (int i = 0; i < hi - lo; ++i) {
    const unsigned long long a = v[2 * i], b = v[2 * i + 1];
    if (b <= a) continue;
    const double d = static_cast<double>(b - a) * 1e-6;
    sum += d;
    mx = d > mx ? d : mx;
    t0 = a < t0 ? a : t0;
    t1 = b > t1 ? b : t1;
    ++k;
  }
  const double mean = k ? sum / static_cast<double>(k) : 0.0;
  if (max_over_mean) *max_over_mean = mean > 0.0 ? mx / mean : 1.0;
  if (mean_ms) *mean_ms = mean;
  if (max_ms) *max_ms = mx;
  if (span_ms) *span_ms = k ? static_cast<double>(t1 - t0) * 1e-6 : 0.0;
  if (warps) *warps = k;
  return CLGEN_OK;
}

int clgen_dev_warp_profile_launches(clgen_dev_ctx* c) {
  return c && c->warp_prof ? static_cast<int>(c->prof_launch.size()) : 0;
}

int clgen_dev_set_fast_math(clgen_dev_ctx* c, int enable) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  c->fast_math = enable != 0;
  return CLGEN_OK;
}

int clgen_dev_counter_plan_info(clgen_dev_ctx* c, int* classes, int64_t* blocks, int64_t* chunks,
                                int* dense_blocks, double* class_eps) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  const bool ok = c->blk_valid;
  if (classes) *classes = ok ? c->plan_host.K : 0;
  if (blocks) *blocks = ok ? c->plan_host.nblocks : 0;
  if (chunks) *chunks = ok ? static_cast<int64_t>(c->plan_host.chunks_full) : 0;
  if (dense_blocks) *dense_blocks = ok ? c->plan_host.dense_blocks : 0;
  if (class_eps) *class_eps = ok ? c->plan_host.eps : 0.0;
  return CLGEN_OK;
}

int clgen_dev_write_edges(clgen_dev_ctx* c, const uint32_t* pairs, int64_t count, int binary,
                          const char* path) {
  if (!c || !path || count < 0 || (count > 0 && !pairs)) return fail(CLGEN_EINVAL, "write_edges: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(CLGEN_EINVAL, "cannot open for writing: %s", path);
  const bool dev_in = is_device_ptr(pairs);
  constexpr int64_t kChunk = int64_t(1) << 23;  // edges per chunk
  const int64_t chunk = count < kChunk ? count : kChunk;
  auto done = [&](int code) {
    std::fclose(f);
    return code;
  };
  bool ok = true;
  if (binary) {  // edge_io.cpp:80-86
    unsigned char head[24] = {'C', 'L', 'G', 'E', 'D', 'G', 'E', '1', 1, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) head[16 + i] = static_cast<unsigned char>((static_cast<uint64_t>(count) >> (8 * i)) & 0xff);
    ok = std::fwrite(head, 1, sizeof head, f) == sizeof head;
  }
  if (count > 0 && ok) {
    const size_t out_bytes = binary ? static_cast<size_t>(chunk) * 16 : static_cast<size_t>(chunk) * 22;
    if (c->pairs.ensure(chunk * sizeof(uint2)) != cudaSuccess || c->sources.ensure(out_bytes) != cudaSuccess ||
        c->counts.ensure(chunk * sizeof(int32_t)) != cudaSuccess ||
        c->offsets.ensure((chunk + 1) * sizeof(int64_t)) != cudaSuccess)
      return done(fail(CLGEN_ENOMEM, "write_edges: cannot allocate staging buffers"));
    if (c->host_stage_bytes < out_bytes) {
      if (c->host_stage) cudaFreeHost(c->host_stage);
      c->host_stage = nullptr;
      c->host_stage_bytes = 0;
      if (cudaMallocHost(&c->host_stage, out_bytes) != cudaSuccess)
        return done(fail(CLGEN_ENOMEM, "write_edges: cannot allocate pinned staging"));
      c->host_stage_bytes = out_bytes;
    }
    for (int64_t base = 0; base < count && ok; base += chunk) {
      const int64_t m = count - base < chunk ? count - base : chunk;
      const uint2* src = reinterpret_cast<const uint2*>(pairs) + base;
      if (!dev_in) {
        if (cudaMemcpyAsync(c->pairs.p, src, m * sizeof(uint2), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
          return done(fail(CLGEN_ECUDA, "write_edges: H2D copy failed"));
        src = c->pairs.as<uint2>();
      }
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m + 255) / 256, c->num_sms * 16));
      size_t bytes = 0;
      if (binary) {
        clg::widen_pairs_kernel<<<grid, 256, 0, c->stream>>>(src, m, c->sources.as<unsigned long long>());
        ++c->launches;
        bytes = static_cast<size_t>(m) * 16;
      } else {
        int32_t* len = c->counts.as<int32_t>();
        int64_t* off = c->offsets.as<int64_t>();
        clg::text_len_kernel<<<grid, 256, 0, c->stream>>>(src, m, len);
        ++c->launches;
        if ((rc = launch_scan(c, len, off, m))) return done(rc);
        if ((rc = fetch_scalars(c))) return done(rc);
        bytes = static_cast<size_t>(c->sc_host->total);
        clg::text_render_kernel<<<grid, 256, 0, c->stream>>>(src, m, off, c->sources.as<char>());
        ++c->launches;
      }
      if (cudaGetLastError() != cudaSuccess ||
          cudaMemcpyAsync(c->host_stage, c->sources.p, bytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
          cudaStreamSynchronize(c->stream) != cudaSuccess)
        return done(fail(CLGEN_ECUDA, "write_edges: device staging failed"));
      ok = std::fwrite(c->host_stage, 1, bytes, f) == bytes;
    }
  }
  if (std::fclose(f) != 0) ok = false;
  if (!ok) return fail(CLGEN_EINVAL, "write failed: %s", path);
  return CLGEN_OK;
}

int clgen_dev_edge_degrees(clgen_dev_ctx* c, const uint32_t* pairs, int64_t m, uint32_t* degree) {
  if (!c || m < 0 || (m > 0 && !pairs) || !degree) return fail(CLGEN_EINVAL, "edge_degrees: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t n = c->n;
  const bool dev_deg = is_device_ptr(degree);
  CUDA_TRY(c->degree.ensure((n > 0 ? n : 1) * sizeof(uint32_t)));
  uint32_t* d = dev_deg ? degree : c->degree.as<uint32_t>();
  if (n > 0) CUDA_TRY(cudaMemsetAsync(d, 0, n * sizeof(uint32_t), c->stream));
  const uint2* e = reinterpret_cast<const uint2*>(pairs);
  if (m > 0 && !is_device_ptr(pairs)) {
    CUDA_TRY(c->pairs.ensure(m * sizeof(uint2)));
    CUDA_TRY(cudaMemcpyAsync(c->pairs.p, pairs, m * sizeof(uint2), cudaMemcpyHostToDevice, c->stream));
    e = c->pairs.as<uint2>();
  }
  if (m > 0) {
    clg::edge_degree_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(e, m, d);
    ++c->launches;
    CUDA_TRY(cudaGetLastError());
  }
  if (!dev_deg && n > 0) CUDA_TRY(cudaMemcpyAsync(degree, d, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return CLGEN_OK;
}

int clgen_dev_fidelity(clgen_dev_ctx* c, const uint32_t* degree, int64_t total_edges, double flag_mass,
                       double* scalars, int* bin_k, double* bin_expected, int64_t* bin_generated,
                       double* bin_rel, int* bin_flagged, int cap, int* nbins) {
  if (!c || !degree || !scalars || !nbins) return fail(CLGEN_EINVAL, "fidelity: bad argument");
  int rc = set_device(c);
  if (rc) return rc;
  const int64_t n = c->n;
  double S;
  if ((rc = blocked_sum_impl(c, c->w, n, &S))) return rc;
  // histograms: [0, kFidBins) expected, [kFidBins, 2 kFidBins + 1) generated (+ zeros)
  const size_t hbytes = (2 * clg::kFidBins + 1) * sizeof(unsigned long long);
  CUDA_TRY(c->probe.ensure(hbytes));
  unsigned long long* h = c->probe.as<unsigned long long>();
  CUDA_TRY(cudaMemsetAsync(h, 0, hbytes, c->stream));
  const uint32_t* deg = degree;
  if (n > 0 && !is_device_ptr(degree)) {
    CUDA_TRY(c->degree.ensure(n * sizeof(uint32_t)));
    CUDA_TRY(cudaMemcpyAsync(c->degree.p, degree, n * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    deg = c->degree.as<uint32_t>();
  }
  double expected_sum = 0.0;
  if (n > 0) {
    CUDA_TRY(c->cum.ensure(n * sizeof(double)));
    c->plan_G = 0;  // cum now holds expected degrees
    double* d = c->cum.as<double>();
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, c->num_sms * 8));
    clg::fid_expected_kernel<<<grid, 256, 0, c->stream>>>(c->w, n, S, d, h);
    clg::fid_generated_kernel<<<grid, 256, 0, c->stream>>>(deg, n, h + clg::kFidBins);
    c->launches += 2;
    CUDA_TRY(cudaGetLastError());
    // analysis.cpp:53-58: expected_sum folded left to right over u
    if ((rc = run_fold(c, d, n, 0.0, clg::kFoldNone, nullptr, nullptr, 0.0, &expected_sum))) return rc;
  }
  std::vector<unsigned long long> hv(2 * clg::kFidBins + 1);
  CUDA_TRY(cudaMemcpy(hv.data(), h, hbytes, cudaMemcpyDeviceToHost));
  const double dn = static_cast<double>(n);
  const double mean_expected = n ? expected_sum / dn : 0.0;
  const double mean_generated = n ? 2.0 * static_cast<double>(total_edges) / dn : 0.0;
  scalars[0] = mean_expected;
  scalars[1] = mean_generated;
  scalars[2] = mean_expected > 0.0 ? std::fabs(mean_generated - mean_expected) / mean_expected
                                   : std::fabs(mean_generated);
  double max_flagged = 0.0;
  int nb = 0;
  for (int i = 0; i < clg::kFidBins; ++i) {
    const unsigned long long ec = hv[i], gc = hv[clg::kFidBins + i];
    if (!ec && !gc) continue;
    const double exp_count = static_cast<double>(ec);
    const bool flagged = exp_count >= flag_mass;
    const double rel = exp_count > 0.0 ? std::fabs(static_cast<double>(gc) - exp_count) / exp_count
                                       : (gc == 0 ? 0.0 : 1.0);
    if (flagged && rel > max_flagged) max_flagged = rel;
    if (nb < cap) {
      if (bin_k) bin_k[nb] = i - clg::kFidBinOff;
      if (bin_expected) bin_expected[nb] = exp_count;
      if (bin_generated) bin_generated[nb] = static_cast<int64_t>(gc);
      if (bin_rel) bin_rel[nb] = rel;
      if (bin_flagged) bin_flagged[nb] = flagged ? 1 : 0;
    }
    ++nb;
  }
  scalars[3] = max_flagged;
  scalars[4] = static_cast<double>(hv[2 * clg::kFidBins]);
  *nbins = nb;
  return CLGEN_OK;
}

int clgen_dev_flagged_nodes(clgen_dev_ctx* c, int64_t* out, int64_t cap, int64_t* n) {
  if (!c) return fail(CLGEN_EINVAL, "null context");
  const int64_t k = c->last_flagged < kFlagCap ? c->last_flagged : kFlagCap;
  const int64_t m = k < cap ? k : cap;
  if (m > 0) {
    CUDA_TRY(cudaMemcpyAsync(out, c->flagged, m * sizeof(int64_t), cudaMemcpyDefault, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  if (n) *n = c->last_flagged;
  return CLGEN_OK;
}

}  // extern "C"
