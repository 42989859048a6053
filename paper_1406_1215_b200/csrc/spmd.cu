// One host thread per GPU: the run_spmd / generate analogue of the reference
// (comm.cpp:204-227, runtime.cpp:46-138) for C and C++ callers that bring no
// communicator of their own.
//
// Every rank owns one clgen_dev_ctx on its GPU, holds all of w
// and computes the canonical S locally (weights.cpp:21-30).  The level-1 UCP
// plan then runs the reference's per-rank phases (partition.cpp:107-157) with
// its collectives carried by NCCL over NVLink:
//   all_reduce_sum / exclusive_scan_sum of block weights and block costs ->
//     ncclAllGather of one double per rank, folded on the host in rank order
//     (never summed inside NCCL, whose reduction order is not the
//     reference's);
//   send/recv_boundary + all_gather_i64 -> ncclAllReduce(MIN) of each rank's
//     found boundaries (n where none).
// Generation of [b_g, b_{g+1}) has no data-path collective; the per-rank edge
// counts and checksums are summed with one ncclAllReduce (uint64, mod 2^64).
// NCCL is loaded at run time (dlopen "libnccl.so.2"), so the library keeps no
// link-time dependency on it.  Ranks mapped to the same device (tests on a
// one-GPU box) cannot share an NCCL communicator; they use an in-process
// host communicator with the same semantics (the reference's InprocGroup,
// comm.cpp:28-184) — the collectives carry a handful of scalars either way.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/clgen_dev.h"

int clgen_internal_fail(int code, const char* msg);  // capi.cu: sets the calling thread's error

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
  decltype(&ncclCommCount) count = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = "cannot load libnccl.so.2";
      return a;
    }
    a.init_all = reinterpret_cast<decltype(a.init_all)>(dlsym(h, "ncclCommInitAll"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.err = reinterpret_cast<decltype(a.err)>(dlsym(h, "ncclGetErrorString"));
    a.version = reinterpret_cast<decltype(a.version)>(dlsym(h, "ncclGetVersion"));
    a.count = reinterpret_cast<decltype(a.count)>(dlsym(h, "ncclCommCount"));
    a.ok = a.init_all && a.all_gather && a.all_reduce && a.destroy && a.err && a.version && a.count;
    if (!a.ok) a.why = "libnccl.so.2 lacks the collective entry points";
    return a;
  }();
  return api;
}

// The three collectives the plan and the fold need.
struct Comm {
  virtual ~Comm() = default;
  virtual int all_gather_f64(double x, double* out) = 0;      // out[G]
  virtual int all_reduce_min_i64(int64_t* v, int k) = 0;      // in place
  virtual int all_reduce_sum_u64(uint64_t* v, int k) = 0;     // in place, mod 2^64
  std::string err;
};

// NCCL on the rank's context stream (device scratch, synchronous results).
struct NcclComm final : Comm {
  ncclComm_t comm;
  cudaStream_t stream;
  int G;
  void* dbuf = nullptr;  // 2 * 8 * max(G, 64) bytes
  NcclComm(ncclComm_t c, cudaStream_t s, int g) : comm(c), stream(s), G(g) {}
  ~NcclComm() override {
    if (dbuf) cudaFree(dbuf);
  }
  int ensure() {
    if (dbuf) return 0;
    if (cudaMalloc(&dbuf, 16 * static_cast<size_t>(std::max(G, 64) + 1)) != cudaSuccess) {
      err = "spmd: cannot allocate NCCL scratch";
      return CLGEN_ENOMEM;
    }
    return 0;
  }
  int done(ncclResult_t r) {
    if (r != ncclSuccess) {
      err = std::string("spmd: NCCL ") + nccl().err(r);
      return CLGEN_ECUDA;
    }
    if (cudaStreamSynchronize(stream) != cudaSuccess) {
      err = "spmd: collective stream failed";
      return CLGEN_ECUDA;
    }
    return 0;
  }
  int all_gather_f64(double x, double* out) override {
    if (int rc = ensure()) return rc;
    double* in = static_cast<double*>(dbuf);
    double* o = in + 1;
    cudaMemcpyAsync(in, &x, sizeof x, cudaMemcpyHostToDevice, stream);
    if (int rc = done(nccl().all_gather(in, o, 1, ncclFloat64, comm, stream))) return rc;
    return cudaMemcpy(out, o, G * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : CLGEN_ECUDA;
  }
  template <class T>
  int reduce(T* v, int k, ncclDataType_t t, ncclRedOp_t op) {
    if (int rc = ensure()) return rc;
    T* d = static_cast<T*>(dbuf);
    cudaMemcpyAsync(d, v, k * sizeof(T), cudaMemcpyHostToDevice, stream);
    if (int rc = done(nccl().all_reduce(d, d, k, t, op, comm, stream))) return rc;
    return cudaMemcpy(v, d, k * sizeof(T), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : CLGEN_ECUDA;
  }
  int all_reduce_min_i64(int64_t* v, int k) override { return reduce(v, k, ncclInt64, ncclMin); }
  int all_reduce_sum_u64(uint64_t* v, int k) override { return reduce(v, k, ncclUint64, ncclSum); }
};

// In-process group for ranks that share a device: slots + a generation barrier.
struct HostGroup {
  int G;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned gen = 0;
  bool poisoned = false;
  std::vector<double> f64;
  std::vector<int64_t> i64;
  std::vector<uint64_t> u64;
  explicit HostGroup(int g) : G(g) {}
  // barrier; returns false when a peer failed
  bool sync() {
    std::unique_lock<std::mutex> lk(m);
    const unsigned my = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my || poisoned; });
    }
    return !poisoned;
  }
  void poison() {
    std::lock_guard<std::mutex> lk(m);
    poisoned = true;
    cv.notify_all();
  }
};

struct HostComm final : Comm {
  HostGroup& grp;
  int g;
  HostComm(HostGroup& gr, int rank) : grp(gr), g(rank) {}
  int fail_peer() {
    err = "spmd: a peer rank failed";
    return CLGEN_EINVAL;
  }
  int all_gather_f64(double x, double* out) override {
    grp.f64[g] = x;
    if (!grp.sync()) return fail_peer();
    std::copy(grp.f64.begin(), grp.f64.begin() + grp.G, out);
    return grp.sync() ? 0 : fail_peer();
  }
  int all_reduce_min_i64(int64_t* v, int k) override {
    std::copy(v, v + k, grp.i64.begin() + static_cast<size_t>(g) * k);
    if (!grp.sync()) return fail_peer();
    for (int i = 0; i < k; ++i)
      for (int r = 0; r < grp.G; ++r) v[i] = std::min(v[i], grp.i64[static_cast<size_t>(r) * k + i]);
    return grp.sync() ? 0 : fail_peer();
  }
  int all_reduce_sum_u64(uint64_t* v, int k) override {
    std::copy(v, v + k, grp.u64.begin() + static_cast<size_t>(g) * k);
    if (!grp.sync()) return fail_peer();
    for (int i = 0; i < k; ++i) {
      uint64_t s = 0;
      for (int r = 0; r < grp.G; ++r) s += grp.u64[static_cast<size_t>(r) * k + i];
      v[i] = s;
    }
    return grp.sync() ? 0 : fail_peer();
  }
};

struct RankOut {
  int rc = 0;
  std::string err;
  double S = 0.0, S_check = 0.0;
  int64_t lo = 0, hi = 0;
  std::vector<int64_t> boundaries;
  int64_t edges = 0, flagged = 0;
  uint64_t checksum = 0;
  double gen_ms = 0.0, kernel_ms = 0.0, plan_ms = 0.0;
  uint64_t tot[3] = {0, 0, 0};
};

// partition.cpp:83-87 / comm.cpp:47-53: left fold from 0.0
double fold(const double* xs, int k) {
  double acc = 0.0;
  for (int j = 0; j < k; ++j) acc += xs[j];
  return acc;
}

// generate_on_rank (runtime.cpp:46-91) for rank g of G.
int rank_body(int g, int G, int device, const double* w, int64_t n, uint64_t seed, int mode, Comm& comm,
              RankOut& out) {
  clgen_dev_ctx* ctx = nullptr;
  int rc = clgen_dev_create(device, &ctx);
  auto bail = [&](int code) {
    out.rc = code;
    out.err = comm.err.empty() ? clgen_dev_last_error() : comm.err;
    if (ctx) clgen_dev_destroy(ctx);
    return code;
  };
  if (rc) return bail(rc);
  if ((rc = clgen_dev_set_weights(ctx, w, n))) return bail(rc);
  if ((rc = clgen_dev_blocked_sum(ctx, &out.S))) return bail(rc);  // canonical S, every rank
  const auto t_plan = std::chrono::steady_clock::now();
  std::vector<double> gathered(static_cast<size_t>(G));
  out.boundaries.assign(static_cast<size_t>(G) + 1, n);
  if (n > 0) {
    double bw = 0.0, z = 0.0;
    if ((rc = clgen_dev_plan_block_weight(ctx, G, g, &bw))) return bail(rc);      // partition.cpp:115-116
    if ((rc = comm.all_gather_f64(bw, gathered.data()))) return bail(rc);
    const double sigma_start = fold(gathered.data(), g);                          // :117
    out.S_check = fold(gathered.data(), G);                                       // runtime.cpp:55-58
    if ((rc = clgen_dev_plan_block_costs(ctx, G, g, sigma_start, out.S, &z))) return bail(rc);  // :119
    if ((rc = comm.all_gather_f64(z, gathered.data()))) return bail(rc);
    const double z_offset = fold(gathered.data(), g);                             // :120
    const double z_bar = fold(gathered.data(), G) / G;                            // :123-124
    if ((rc = clgen_dev_plan_block_boundaries(ctx, G, g, z_offset, z_bar, out.boundaries.data()))) return bail(rc);
    if ((rc = comm.all_reduce_min_i64(out.boundaries.data(), G + 1))) return bail(rc);  // :134-154
  }
  out.boundaries[0] = 0;
  out.boundaries[static_cast<size_t>(G)] = n;
  out.plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_plan).count();
  out.lo = out.boundaries[static_cast<size_t>(g)];
  out.hi = out.boundaries[static_cast<size_t>(g) + 1];
  // timed generation section (runtime.cpp:74-86), count-only fold
  const auto t0 = std::chrono::steady_clock::now();
  if ((rc = clgen_dev_stream_range(ctx, out.S, out.lo, out.hi, seed, mode, 0, nullptr, 0, nullptr, 0, &out.edges,
                                   &out.checksum, &out.flagged)))
    return bail(rc);
  out.gen_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  float kms = 0.0f;
  if (out.hi > out.lo && clgen_dev_last_kernel_ms(ctx, &kms) == CLGEN_OK) out.kernel_ms = kms;
  out.tot[0] = static_cast<uint64_t>(out.edges);
  out.tot[1] = out.checksum;
  out.tot[2] = static_cast<uint64_t>(out.flagged);
  if ((rc = comm.all_reduce_sum_u64(out.tot, 3))) return bail(rc);
  clgen_dev_destroy(ctx);
  return 0;
}

}  // namespace

extern "C" int clgen_spmd_generate(const int* devices, int G, const double* w, int64_t n, uint64_t seed,
                                   int stream_mode, int64_t* boundaries, int64_t* rank_edges,
                                   double* rank_gen_ms, double* rank_kernel_ms, clgen_spmd_report* report) {
  if (G < 1 || !devices || (n > 0 && !w) || n < 0 || !boundaries || !report)
    return clgen_internal_fail(CLGEN_EINVAL, "spmd_generate: bad argument");
  if (stream_mode != CLGEN_STREAM_REFERENCE && stream_mode != CLGEN_STREAM_COUNTER)
    return clgen_internal_fail(CLGEN_EINVAL, "spmd_generate: unknown stream mode");
  std::vector<int> devs(devices, devices + G);
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  const char* force = std::getenv("CLGEN_SPMD_COMM");
  const bool use_nccl = distinct && !(force && std::strcmp(force, "host") == 0);
  std::vector<ncclComm_t> comms;
  int nccl_version = 0;
  if (use_nccl) {
    const NcclApi& api = nccl();
    if (!api.ok) return clgen_internal_fail(CLGEN_ECUDA, ("spmd_generate: " + api.why).c_str());
    comms.resize(static_cast<size_t>(G));
    const ncclResult_t r = api.init_all(comms.data(), G, devs.data());  // one communicator per GPU
    if (r != ncclSuccess)
      return clgen_internal_fail(CLGEN_ECUDA, (std::string("spmd_generate: ncclCommInitAll: ") + api.err(r)).c_str());
    api.version(&nccl_version);
    int cnt = 0;
    api.count(comms[0], &cnt);
    if (cnt != G) return clgen_internal_fail(CLGEN_ECUDA, "spmd_generate: NCCL communicator size mismatch");
  }
  HostGroup grp(G);
  grp.f64.assign(static_cast<size_t>(G), 0.0);
  grp.i64.assign(static_cast<size_t>(G) * (G + 1), 0);
  grp.u64.assign(static_cast<size_t>(G) * 3, 0);
  std::vector<RankOut> outs(static_cast<size_t>(G));
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int g = 0; g < G; ++g) {
    pool.emplace_back([&, g] {
      cudaSetDevice(devs[static_cast<size_t>(g)]);
      Comm* comm = nullptr;
      NcclComm* nc = nullptr;
      HostComm hc(grp, g);
      if (use_nccl) {
        // the collectives run on a stream of this rank's device
        cudaStream_t s = nullptr;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        nc = new NcclComm(comms[static_cast<size_t>(g)], s, G);
        comm = nc;
      } else {
        comm = &hc;
      }
      if (rank_body(g, G, devs[static_cast<size_t>(g)], w, n, seed, stream_mode, *comm, outs[static_cast<size_t>(g)]))
        grp.poison();  // wake peers blocked in the host group (comm.cpp:151-168)
      if (nc) {
        cudaStream_t s = nc->stream;
        delete nc;
        cudaStreamDestroy(s);
      }
    });
  }
  for (auto& t : pool) t.join();
  const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (use_nccl)
    for (auto c : comms) nccl().destroy(c);
  for (int g = 0; g < G; ++g)  // the lowest failing rank's error (comm.cpp:209-226)
    if (outs[static_cast<size_t>(g)].rc)
      return clgen_internal_fail(outs[static_cast<size_t>(g)].rc,
                                 ("rank " + std::to_string(g) + ": " + outs[static_cast<size_t>(g)].err).c_str());
  for (int g = 0; g <= G; ++g) boundaries[g] = outs[0].boundaries[static_cast<size_t>(g)];
  for (int g = 0; g < G; ++g) {
    if (outs[static_cast<size_t>(g)].boundaries != outs[0].boundaries)
      return clgen_internal_fail(CLGEN_EINVAL, "spmd_generate: ranks disagree on the plan");
    if (rank_edges) rank_edges[g] = outs[static_cast<size_t>(g)].edges;
    if (rank_gen_ms) rank_gen_ms[g] = outs[static_cast<size_t>(g)].gen_ms;
    if (rank_kernel_ms) rank_kernel_ms[g] = outs[static_cast<size_t>(g)].kernel_ms;
  }
  report->G = G;
  report->S = outs[0].S;
  report->S_check = outs[0].S_check;
  report->total_edges = static_cast<int64_t>(outs[0].tot[0]);
  report->checksum = outs[0].tot[1];
  report->n_flagged = static_cast<int64_t>(outs[0].tot[2]);
  report->wall_ms = wall;
  double pm = 0.0;
  for (auto& o : outs) pm = std::max(pm, o.plan_ms);
  report->plan_ms = pm;
  report->nccl_version = use_nccl ? nccl_version : 0;
  return CLGEN_OK;
}
