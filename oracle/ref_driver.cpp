// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (clgen core, compiled
// from /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).
// It exposes the reference's own entry points to ctypes so tests, smoke() and
// bench.py's CPU arm can run the real reference on identical inputs:
//
//   make_weight_sequence   weights.cpp:32-55
//   blocked_sum            weights.cpp:21-30
//   synth_powerlaw         weights.cpp:103-128
//   synth_constant         weights.cpp:130-140
//   expected_total_edges   weights.cpp:155-162
//   skip_length            edge_skip.cpp:9-16
//   create_edges(_range)   edge_skip.cpp:50-66   (hot path: edges_from_source :20-46)
//   naive_pair_sampler     edge_skip.cpp:72-91
//   node_cost, block_bounds, block_cumulative, partition_of   cost.cpp:8-60
//   plan_ucp_oracle        partition.cpp:159-203
//   plan_ucp (SPMD)        partition.cpp:107-157 via run_spmd comm.cpp:204-227
//   generate               runtime.cpp:93-138
//
// Every function returns 0 on success and -1 when the reference threw
// clgen::error; the message is available from ref_last_error().

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "clgen/cost.hpp"
#include "clgen/analysis.hpp"
#include "clgen/edge_io.hpp"
#include "clgen/edge_skip.hpp"
#include "clgen/partition.hpp"
#include "clgen/rng.hpp"
#include "clgen/runtime.hpp"
#include "clgen/weights.hpp"

using namespace clgen;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Sink writing (u,v) pairs as uint32 into a caller buffer (the device layout),
// or only counting when the buffer is exhausted / absent.
class PairSink final : public EdgeSink {
 public:
  PairSink(std::uint32_t* out, std::int64_t cap) : out_(out), cap_(cap) {}
  std::int64_t stored = 0;

 private:
  void on_edge(const Edge& e) override {
    if (out_ && stored < cap_) {
      out_[2 * stored] = static_cast<std::uint32_t>(e.u);
      out_[2 * stored + 1] = static_cast<std::uint32_t>(e.v);
      ++stored;
    }
  }
  std::uint32_t* out_;
  std::int64_t cap_;
};

// Order-independent fold: sum of edge_hash(u, v) mod 2^64 (the device fold's
// checksum term, paper_1406_1215_b200/csrc/common.cuh), plus optional per-node
// undirected degree counters.
static std::uint64_t edge_hash(std::uint64_t u, std::uint64_t v) {
  std::uint64_t z = ((u << 32) | v) * 0x9e3779b97f4a7c15ULL;
  z ^= z >> 32;
  z *= 0xd6e8feb86659fd93ULL;
  return z ^ (z >> 32);
}

class FoldSink final : public EdgeSink {
 public:
  FoldSink(std::int64_t* degree) : degree_(degree) {}
  std::uint64_t checksum = 0;

 private:
  void on_edge(const Edge& e) override {
    checksum += edge_hash(static_cast<std::uint64_t>(e.u), static_cast<std::uint64_t>(e.v));
    if (degree_) {
      ++degree_[e.u];
      ++degree_[e.v];
    }
  }
  std::int64_t* degree_;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_mix64(std::uint64_t z) { return mix64(z); }

// First `count` draws of next_open01 for stream (seed,u) (rng.hpp:26-69).
void ref_stream_open01(std::uint64_t seed, std::int64_t u, std::int64_t count, double* out) {
  RngStream rng(seed, u);
  for (std::int64_t i = 0; i < count; ++i) out[i] = rng.next_open01();
}

int ref_blocked_sum(const double* xs, std::int64_t n, double* out) {
  return guard([&] { *out = blocked_sum(std::span<const double>(xs, static_cast<std::size_t>(n))); });
}

int ref_ws_create(const double* w, std::int64_t n, int sort_desc, void** handle) {
  return guard([&] {
    std::vector<double> v(w, w + n);
    auto* ws = new WeightSequence(make_weight_sequence(
        std::move(v), sort_desc ? SortPolicy::sort_desc : SortPolicy::require_sorted));
    *handle = ws;
  });
}

void ref_ws_destroy(void* h) { delete static_cast<WeightSequence*>(h); }

double ref_ws_sum(void* h) { return static_cast<WeightSequence*>(h)->sum_S; }

void ref_ws_weights(void* h, double* out) {
  const auto& ws = *static_cast<WeightSequence*>(h);
  std::memcpy(out, ws.weights.data(), ws.weights.size() * sizeof(double));
}

void ref_ws_labels(void* h, std::int64_t* out) {
  const auto& ws = *static_cast<WeightSequence*>(h);
  std::memcpy(out, ws.orig_labels.data(), ws.orig_labels.size() * sizeof(std::int64_t));
}

std::int64_t ref_ws_size(void* h) { return static_cast<WeightSequence*>(h)->size(); }

int ref_synth_powerlaw(std::int64_t n, double gamma, double wmin, double wmax, std::uint64_t seed,
                       void** handle) {
  return guard([&] { *handle = new WeightSequence(synth_powerlaw(n, gamma, wmin, wmax, seed)); });
}

int ref_synth_constant(std::int64_t n, double d, void** handle) {
  return guard([&] { *handle = new WeightSequence(synth_constant(n, d)); });
}

int ref_expected_total_edges(void* h, double* out) {
  return guard([&] { *out = expected_total_edges(*static_cast<WeightSequence*>(h)); });
}

int ref_skip_length(double p, double r, std::int64_t* out) {
  return guard([&] { *out = skip_length(p, r); });
}

int ref_node_cost(double w, double sigma, double S, double* out) {
  return guard([&] { *out = node_cost(w, sigma, S); });
}

int ref_block_bounds(std::int64_t n, int P, int rank, std::int64_t* lo, std::int64_t* hi) {
  return guard([&] {
    auto b = block_bounds(n, P, rank);
    *lo = b.first;
    *hi = b.second;
  });
}

int ref_partition_of(double c, double zbar, int P, int* out) {
  return guard([&] { *out = partition_of(c, zbar, P); });
}

// Materialise (pairs != NULL) or count edges of create_edges_range.
int ref_create_edges_range(void* h, double S, std::int64_t lo, std::int64_t hi, std::uint64_t seed,
                           std::uint32_t* pairs, std::int64_t cap, std::int64_t* count) {
  return guard([&] {
    PairSink sink(pairs, cap);
    create_edges_range(*static_cast<WeightSequence*>(h), S, lo, hi, seed, sink);
    *count = sink.count();
  });
}

int ref_create_edges(void* h, double S, const std::int64_t* sources, std::int64_t k,
                     std::uint64_t seed, std::uint32_t* pairs, std::int64_t cap,
                     std::int64_t* count) {
  return guard([&] {
    PairSink sink(pairs, cap);
    create_edges(*static_cast<WeightSequence*>(h), S,
                 std::span<const node_t>(sources, static_cast<std::size_t>(k)), seed, sink);
    *count = sink.count();
  });
}

int ref_fold_edges_range(void* h, double S, std::int64_t lo, std::int64_t hi, std::uint64_t seed,
                         std::int64_t* degree, std::int64_t* count, std::uint64_t* checksum) {
  return guard([&] {
    FoldSink sink(degree);
    create_edges_range(*static_cast<WeightSequence*>(h), S, lo, hi, seed, sink);
    *count = sink.count();
    *checksum = sink.checksum;
  });
}

int ref_naive_pair_sampler(void* h, std::uint64_t seed, std::uint32_t* pairs, std::int64_t cap,
                           std::int64_t* count) {
  return guard([&] {
    PairSink sink(pairs, cap);
    naive_pair_sampler(*static_cast<WeightSequence*>(h), seed, sink);
    *count = sink.count();
  });
}

int ref_node_costs_sequential(void* h, double* out) {
  return guard([&] {
    const auto c = node_costs_sequential(*static_cast<WeightSequence*>(h));
    std::copy(c.begin(), c.end(), out);
  });
}

// scheme: 0 naive, 1 ucp, 2 rrp (partition.hpp:15); boundaries unused for rrp
int ref_fill_partition_costs(void* h, int scheme, int P, const std::int64_t* boundaries, double* out) {
  return guard([&] {
    const auto& ws = *static_cast<WeightSequence*>(h);
    PartitionPlan plan;
    plan.scheme = scheme == 2 ? Scheme::rrp : (scheme == 1 ? Scheme::ucp : Scheme::naive);
    plan.procs = P;
    plan.n = ws.size();
    if (scheme == 2) plan.rrp_modulus = P;
    else plan.boundaries.assign(boundaries, boundaries + P + 1);
    fill_partition_costs(plan, ws);
    std::copy(plan.per_partition_cost.begin(), plan.per_partition_cost.end(), out);
  });
}

int ref_plan_ucp_oracle(void* h, int P, std::int64_t* boundaries) {
  return guard([&] {
    auto plan = plan_ucp_oracle(*static_cast<WeightSequence*>(h), P);
    for (int i = 0; i <= P; ++i) boundaries[i] = plan.boundaries[static_cast<std::size_t>(i)];
  });
}

int ref_plan_ucp_spmd(void* h, int P, std::int64_t* boundaries) {
  return guard([&] {
    const auto& ws = *static_cast<WeightSequence*>(h);
    std::vector<PartitionPlan> plans(static_cast<std::size_t>(P));
    run_spmd(P, [&](Communicator& comm) {
      plans[static_cast<std::size_t>(comm.rank())] = plan_ucp(ws, comm);
    });
    for (int i = 0; i <= P; ++i) boundaries[i] = plans[0].boundaries[static_cast<std::size_t>(i)];
  });
}

// The G-blocked C_u array (after finalize_offsets) as plan_ucp_oracle builds
// it: partition.cpp:163-181.
int ref_global_cum_costs(void* h, int P, double* cum_out, double* block_weight_out,
                         double* block_cost_out) {
  return guard([&] {
    const auto& ws = *static_cast<WeightSequence*>(h);
    const node_t n = ws.size();
    std::vector<double> bw(static_cast<std::size_t>(P), 0.0);
    for (int i = 0; i < P; ++i) {
      auto [lo, hi] = block_bounds(n, P, i);
      double acc = 0.0;
      for (node_t u = lo; u < hi; ++u) acc += ws.weights[static_cast<std::size_t>(u)];
      bw[static_cast<std::size_t>(i)] = acc;
    }
    std::vector<CostProfile> profs;
    std::vector<double> bc(static_cast<std::size_t>(P), 0.0);
    for (int i = 0; i < P; ++i) {
      double sp = 0.0;
      for (int j = 0; j < i; ++j) sp += bw[static_cast<std::size_t>(j)];
      profs.push_back(block_cumulative(ws, i, P, sp));
      bc[static_cast<std::size_t>(i)] = profs.back().block_cost;
    }
    for (int i = 0; i < P; ++i) {
      double zp = 0.0;
      for (int j = 0; j < i; ++j) zp += bc[static_cast<std::size_t>(j)];
      finalize_offsets(profs[static_cast<std::size_t>(i)], zp);
      const auto& prof = profs[static_cast<std::size_t>(i)];
      std::memcpy(cum_out + prof.block_lo, prof.cum_costs.data(),
                  prof.cum_costs.size() * sizeof(double));
      if (block_weight_out) block_weight_out[i] = bw[static_cast<std::size_t>(i)];
      if (block_cost_out) block_cost_out[i] = bc[static_cast<std::size_t>(i)];
    }
  });
}

// CPU baseline: generate() with the count-only sink (runtime.cpp:93-138,
// EdgeCounter when out_dir is empty: runtime.cpp:69-72).
int ref_generate_count(void* h, int procs, int scheme, std::uint64_t seed, std::int64_t* total,
                       double* max_gen_wall_ms, double* wall_ms, std::int64_t* boundaries) {
  return guard([&] {
    GenConfig cfg;
    cfg.scheme = scheme == 0 ? Scheme::naive : scheme == 1 ? Scheme::ucp : Scheme::rrp;
    cfg.procs = procs;
    cfg.seed = seed;
    const GenReport rep = generate(*static_cast<WeightSequence*>(h), cfg);
    *total = rep.total_edges;
    double mx = 0.0;
    for (const auto& r : rep.ranks) mx = r.gen_wall_ms > mx ? r.gen_wall_ms : mx;
    *max_gen_wall_ms = mx;
    *wall_ms = rep.wall_ms;
    if (boundaries && !rep.boundaries.empty()) {
      for (std::size_t i = 0; i < rep.boundaries.size(); ++i) boundaries[i] = rep.boundaries[i];
    }
  });
}

// CPU baseline for workloads too large for generate(): time create_edges_range
// over the given node ranges, one std::thread per range, all in parallel
// (the acceptance.cpp:221-254 per-partition pattern). Returns total edges and
// the wall time of the parallel section.
int ref_parallel_ranges_count(void* h, double S, const std::int64_t* ranges, int k,
                              std::uint64_t seed, std::int64_t* total, double* wall_ms) {
  return guard([&] {
    const auto& ws = *static_cast<WeightSequence*>(h);
    std::vector<std::int64_t> counts(static_cast<std::size_t>(k), 0);
    std::vector<std::thread> threads;
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < k; ++i) {
      threads.emplace_back([&, i] {
        try {
          EdgeCounter sink;
          create_edges_range(ws, S, ranges[2 * i], ranges[2 * i + 1], seed, sink);
          counts[static_cast<std::size_t>(i)] = sink.count();
        } catch (...) {
          failed = 1;
        }
      });
    }
    for (auto& t : threads) t.join();
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (failed) throw error("ref_parallel_ranges_count: a worker failed");
    std::int64_t s = 0;
    for (auto c : counts) s += c;
    *total = s;
  });
}

// edge_io.cpp:72-88 write_edges on uint32 pairs (widened to Edge).
int ref_write_edges(const std::uint32_t* pairs, std::int64_t count, int binary, const char* path) {
  return guard([&] {
    std::vector<Edge> edges(static_cast<std::size_t>(count));
    for (std::int64_t i = 0; i < count; ++i) edges[i] = Edge{pairs[2 * i], pairs[2 * i + 1]};
    write_edges(edges, binary ? EdgeFormat::binary : EdgeFormat::text, path);
  });
}

// edge_io.cpp:90-123 read_edges into uint32 pairs (cap entries); *count = records.
int ref_read_edges(const char* path, std::uint32_t* pairs, std::int64_t cap, std::int64_t* count) {
  return guard([&] {
    const auto edges = read_edges(path);
    *count = static_cast<std::int64_t>(edges.size());
    for (std::int64_t i = 0; i < *count && i < cap; ++i) {
      pairs[2 * i] = static_cast<std::uint32_t>(edges[i].u);
      pairs[2 * i + 1] = static_cast<std::uint32_t>(edges[i].v);
    }
  });
}

// analysis.cpp:18-85: degree_histogram + compare_distributions on an edge
// list.  Outputs: scalars[0..4] = mean_expected, mean_generated,
// mean_rel_error, max_flagged_rel_error, zero_degree; per bin (up to cap):
// k, expected_count, generated_count, rel_error, flagged.
int ref_fidelity(void* h, const std::uint32_t* pairs, std::int64_t count, double flag_mass,
                 double* scalars, int* bin_k, double* bin_expected, std::int64_t* bin_generated,
                 double* bin_rel, int* bin_flagged, int cap, int* nbins) {
  return guard([&] {
    const auto& ws = *static_cast<WeightSequence*>(h);
    std::vector<Edge> edges(static_cast<std::size_t>(count));
    for (std::int64_t i = 0; i < count; ++i) edges[i] = Edge{pairs[2 * i], pairs[2 * i + 1]};
    const auto hist = degree_histogram(edges, ws.size());
    const auto rep = compare_distributions(ws, hist, flag_mass);
    scalars[0] = rep.mean_expected;
    scalars[1] = rep.mean_generated;
    scalars[2] = rep.mean_rel_error;
    scalars[3] = rep.max_flagged_rel_error;
    scalars[4] = static_cast<double>(hist.zero_degree);
    int i = 0;
    for (const auto& b : rep.bins) {
      if (i >= cap) break;
      bin_k[i] = b.k;
      bin_expected[i] = b.expected_count;
      bin_generated[i] = b.generated_count;
      bin_rel[i] = b.rel_error;
      bin_flagged[i] = b.flagged ? 1 : 0;
      ++i;
    }
    *nbins = static_cast<int>(rep.bins.size());
  });
}

}  // extern "C"
