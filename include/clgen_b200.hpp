// clgen_b200.hpp — header-only C++ mirror of the reference generator API
// (namespace clgen in /root/reference/proj/core/include/clgen/*.hpp) on top of
// the C ABI in clgen_dev.h.  Same names, argument meaning and error
// behaviour: contract violations throw clgen_b200::error exactly where the
// reference throws clgen::error.  A maintainer switches a caller with
//     #include "clgen_b200.hpp"
//     namespace clgen = clgen_b200;
// and links libclgen_b200.so.
//
//   reference (clgen::)                          here (clgen_b200::)
//   WeightSequence          weights.hpp:14-20     WeightSequence (+ device context)
//   make_weight_sequence    weights.hpp:44        make_weight_sequence
//   blocked_sum             weights.hpp:36        blocked_sum
//   synth_powerlaw / synth_constant  weights.hpp:47-50   same (synthesised on the device)
//   validate / ValidationReport      weights.hpp:22-29,53  same (host)
//   expected_total_edges    weights.hpp:55        expected_total_edges (host, O(n))
//   Edge/EdgeSink/EdgeVector/EdgeCounter  edge_skip.hpp:15-49   same
//   create_edges            edge_skip.hpp:58-59   create_edges
//   create_edges_range      edge_skip.hpp:60-61   create_edges_range
//   serial_cl               edge_skip.hpp:63      serial_cl
//   plan_ucp_oracle         partition.hpp:56      plan_ucp_oracle (device, bit-identical)
//   PartitionPlan           partition.hpp:20-31   PartitionPlan (ucp fields)
//   generate / GenConfig / GenReport  runtime.hpp:16-47, runtime.cpp:93-138
//                                                 generate over clgen_spmd_generate
//                                                 (one host thread per GPU, NCCL)
//
// EdgeSink gains one additive member, emit_bulk: the device
// hands a sink a whole materialised run at once; EdgeVector appends it,
// EdgeCounter only advances its count, any other sink still sees on_edge per
// edge.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "clgen_dev.h"

namespace clgen_b200 {

using node_t = std::int64_t;

struct error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc != CLGEN_OK) throw error(clgen_dev_last_error());
}

// One device context (CUDA device + stream + resident weights).
class Device {
 public:
  explicit Device(int device = 0) {
    clgen_dev_ctx* c = nullptr;
    check(clgen_dev_create(device, &c));
    ctx_.reset(c);
  }
  clgen_dev_ctx* get() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(clgen_dev_ctx* c) const { clgen_dev_destroy(c); }
  };
  std::unique_ptr<clgen_dev_ctx, Del> ctx_;
};

struct WeightSequence {
  std::vector<double> weights;      // non-increasing
  double sum_S = 0.0;               // blocked_sum(weights), computed on the device
  std::vector<node_t> orig_labels;  // sorted position -> original input label
  std::shared_ptr<Device> device;   // owns the device copy of the weights
  // host-side sizing aid (lazily built): expected edges of sources [0, u)
  // in the suffix form of node_costs_sequential (cost.cpp:62-77) minus the 1
  mutable std::vector<double> expected_prefix;

  node_t size() const { return static_cast<node_t>(weights.size()); }
  double expected_edges(node_t lo, node_t hi) const {
    if (expected_prefix.empty()) {
      expected_prefix.assign(weights.size() + 1, 0.0);
      double suffix = 0.0;
      std::vector<double> e(weights.size(), 0.0);
      for (size_t u = weights.size(); u-- > 0;) {
        e[u] = sum_S > 0.0 ? weights[u] / sum_S * suffix : 0.0;
        suffix += weights[u];
      }
      for (size_t u = 0; u < weights.size(); ++u) expected_prefix[u + 1] = expected_prefix[u] + e[u];
    }
    return expected_prefix[static_cast<size_t>(hi)] - expected_prefix[static_cast<size_t>(lo)];
  }
};

enum class SortPolicy { require_sorted, sort_desc };

// weights.cpp:32-55
inline WeightSequence make_weight_sequence(std::vector<double> weights, SortPolicy policy,
                                           int device = 0) {
  WeightSequence ws;
  ws.orig_labels.resize(weights.size());
  std::iota(ws.orig_labels.begin(), ws.orig_labels.end(), node_t{0});
  if (policy == SortPolicy::sort_desc) {
    std::stable_sort(ws.orig_labels.begin(), ws.orig_labels.end(),
                     [&](node_t a, node_t b) { return weights[a] > weights[b]; });
    ws.weights.reserve(weights.size());
    for (node_t label : ws.orig_labels) ws.weights.push_back(weights[label]);
  } else {
    ws.weights = std::move(weights);
  }
  ws.device = std::make_shared<Device>(device);
  // the device validates order (throws "weights unsorted at position u")
  check(clgen_dev_set_weights(ws.device->get(), ws.weights.data(), ws.size()));
  check(clgen_dev_blocked_sum(ws.device->get(), &ws.sum_S));
  return ws;
}

// weights.cpp:103-128: the array is synthesised and sorted on the device
// (clgen_dev_synth_powerlaw, bit-identical to the reference's) and read back
// once for `weights`.  orig_labels is the identity: the synthesiser's draw
// order is not kept (the reference's labels index its unsorted draws).
inline WeightSequence synth_powerlaw(node_t n, double gamma, double w_min, double w_max,
                                     std::uint64_t seed, int device = 0) {
  WeightSequence ws;
  ws.device = std::make_shared<Device>(device);
  check(clgen_dev_synth_powerlaw(ws.device->get(), n, gamma, w_min, w_max, seed, 1, 0.0, nullptr, nullptr));
  ws.weights.resize(static_cast<size_t>(n));
  check(clgen_dev_copy_weights(ws.device->get(), ws.weights.data(), n));
  ws.orig_labels.resize(ws.weights.size());
  std::iota(ws.orig_labels.begin(), ws.orig_labels.end(), node_t{0});
  check(clgen_dev_blocked_sum(ws.device->get(), &ws.sum_S));
  return ws;
}

// weights.cpp:130-140
inline WeightSequence synth_constant(node_t n, double d, int device = 0) {
  if (n < 1) throw error("synth_constant: n must be >= 1");
  if (d < 0.0) throw error("synth_constant: d must be >= 0");
  if (d > 0.0 && d >= static_cast<double>(n))
    throw error("synth_constant: inadmissible (d^2 = " + std::to_string(d * d) + " >= S = " + std::to_string(d * n) + ")");
  return make_weight_sequence(std::vector<double>(static_cast<size_t>(n), d), SortPolicy::require_sorted, device);
}

// weights.hpp:22-29, weights.cpp:142-153 (host: O(n) input statistics)
struct ValidationReport {
  bool is_sorted = false;
  bool admissible = false;  // max w^2 < S; false when S == 0
  node_t n = 0;
  double sum_S = 0.0;
  double max_weight = 0.0;
  node_t zero_weight_count = 0;
};

inline ValidationReport validate(const WeightSequence& ws) {
  ValidationReport rep;
  rep.n = ws.size();
  rep.sum_S = ws.sum_S;
  rep.is_sorted = std::is_sorted(ws.weights.begin(), ws.weights.end(), std::greater<double>{});
  for (double w : ws.weights) {
    rep.max_weight = std::max(rep.max_weight, w);
    if (w == 0.0) ++rep.zero_weight_count;
  }
  rep.admissible = ws.sum_S > 0.0 && rep.max_weight * rep.max_weight < ws.sum_S;
  return rep;
}

// weights.cpp:21-30 on the device (any sequence)
inline double blocked_sum(std::span<const double> xs, int device = 0) {
  Device d(device);
  double s = 0.0;
  check(clgen_dev_blocked_sum_array(d.get(), xs.data(), static_cast<int64_t>(xs.size()), &s));
  return s;
}

// weights.cpp:155-162 (host: O(n) input statistics, not on the device path)
inline double expected_total_edges(const WeightSequence& ws) {
  if (ws.sum_S <= 0.0) return 0.0;
  std::vector<double> sq;
  sq.reserve(ws.weights.size());
  for (double w : ws.weights) sq.push_back(w * w);
  return (ws.sum_S * ws.sum_S - blocked_sum(sq)) / (2.0 * ws.sum_S);
}

// ---- edges (edge_skip.hpp:15-49) -------------------------------------------
struct Edge {
  node_t u = 0;
  node_t v = 0;
  friend bool operator==(const Edge&, const Edge&) = default;
  friend auto operator<=>(const Edge&, const Edge&) = default;
};

class EdgeSink {
 public:
  virtual ~EdgeSink() = default;
  void emit(const Edge& e) {
    on_edge(e);
    ++count_;
  }
  // k (u, v) uint32 pairs in emission order; count() advances by k
  void emit_bulk(const std::uint32_t* pairs, std::int64_t k) {
    on_bulk(pairs, k);
    count_ += k;
  }
  std::int64_t count() const { return count_; }

 private:
  virtual void on_edge(const Edge& e) = 0;
  virtual void on_bulk(const std::uint32_t* pairs, std::int64_t k) {
    for (std::int64_t i = 0; i < k; ++i) on_edge(Edge{pairs[2 * i], pairs[2 * i + 1]});
  }
  std::int64_t count_ = 0;
};

class EdgeVector final : public EdgeSink {
 public:
  std::vector<Edge> edges;

 private:
  void on_edge(const Edge& e) override { edges.push_back(e); }
  void on_bulk(const std::uint32_t* pairs, std::int64_t k) override {
    edges.reserve(edges.size() + static_cast<size_t>(k));
    for (std::int64_t i = 0; i < k; ++i) edges.push_back(Edge{pairs[2 * i], pairs[2 * i + 1]});
  }
};

class EdgeCounter final : public EdgeSink {
 private:
  void on_edge(const Edge&) override {}
  void on_bulk(const std::uint32_t*, std::int64_t) override {}
};

namespace detail {
// Materialise on the device (uint32 pairs, reference emission order) in ONE
// generation call sized from the expected edge count (+6 sigma), then hand
// the run to the sink in bulk.  Only if the realised count exceeds that
// capacity (CLGEN_ERANGE, with the exact count) is the call repeated.
template <class Gen>
std::int64_t run(Gen&& gen, double expected, EdgeSink& sink) {
  std::int64_t cap = static_cast<std::int64_t>(expected * 1.01 + 6.0 * std::sqrt(expected + 1.0)) + 4096;
  std::vector<std::uint32_t> pairs(static_cast<size_t>(2 * cap));
  std::int64_t count = 0, flagged = 0;
  int rc = gen(pairs.data(), cap, &count, &flagged);
  if (rc == CLGEN_ERANGE) {
    cap = count;
    pairs.assign(static_cast<size_t>(2 * std::max<std::int64_t>(cap, 1)), 0u);
    rc = gen(pairs.data(), cap, &count, &flagged);
  }
  check(rc);
  sink.emit_bulk(pairs.data(), count);
  return count;
}
}  // namespace detail

// edge_skip.cpp:60-66
inline std::int64_t create_edges_range(const WeightSequence& ws, double S, node_t lo, node_t hi,
                                       std::uint64_t seed, EdgeSink& sink) {
  const double e = (lo >= 0 && hi <= ws.size() && lo <= hi) ? ws.expected_edges(lo, hi) : 0.0;
  return detail::run(
      [&](std::uint32_t* p, std::int64_t cap, std::int64_t* cnt, std::int64_t* fl) {
        return clgen_dev_create_edges_range(ws.device->get(), S, lo, hi, seed, p, cap, cnt, fl);
      },
      e, sink);
}

// edge_skip.cpp:50-58
inline std::int64_t create_edges(const WeightSequence& ws, double S, std::span<const node_t> sources,
                                 std::uint64_t seed, EdgeSink& sink) {
  double e = 0.0;
  for (node_t u : sources)
    if (u >= 0 && u < ws.size()) e += ws.expected_edges(u, u + 1);
  return detail::run(
      [&](std::uint32_t* p, std::int64_t cap, std::int64_t* cnt, std::int64_t* fl) {
        return clgen_dev_create_edges(ws.device->get(), S, sources.data(),
                                      static_cast<int64_t>(sources.size()), seed, p, cap, cnt, fl);
      },
      e, sink);
}

// edge_skip.cpp:68-70
inline std::int64_t serial_cl(const WeightSequence& ws, std::uint64_t seed, EdgeSink& sink) {
  return create_edges_range(ws, ws.sum_S, 0, ws.size(), seed, sink);
}

// ---- partitions (partition.hpp:20-56) ---------------------------------------
struct PartitionPlan {
  int procs = 1;
  node_t n = 0;
  std::vector<node_t> boundaries;  // n_0..n_P
  node_t partition_size(int i) const {
    if (i < 0 || i >= procs) throw error("partition_size: bad partition index");
    return boundaries[static_cast<size_t>(i) + 1] - boundaries[static_cast<size_t>(i)];
  }
};

// partition.cpp:159-203, computed on the device, bit-identical.
inline PartitionPlan plan_ucp_oracle(const WeightSequence& ws, int P) {
  PartitionPlan plan;
  plan.procs = P;
  plan.n = ws.size();
  plan.boundaries.assign(static_cast<size_t>(std::max(P, 0)) + 1, 0);
  check(clgen_dev_plan_ucp(ws.device->get(), P, plan.boundaries.data(), nullptr));
  return plan;
}

// ---- streaming fold (no reference counterpart) -------------------------------
struct StreamFold {
  std::int64_t edges = 0;
  std::uint64_t checksum = 0;  // sum of edge_hash(u, v) mod 2^64 (clgen_dev.h)
  std::int64_t flagged = 0;
};

inline StreamFold stream_range(const WeightSequence& ws, double S, node_t lo, node_t hi,
                               std::uint64_t seed, bool counter_stream = true) {
  StreamFold f;
  check(clgen_dev_stream_range(ws.device->get(), S, lo, hi, seed,
                               counter_stream ? CLGEN_STREAM_COUNTER : CLGEN_STREAM_REFERENCE, 0,
                               nullptr, 0, nullptr, 0, &f.edges, &f.checksum, &f.flagged));
  return f;
}

// ---- whole runs (runtime.hpp:16-47, runtime.cpp:93-138) ----------------------
// GenConfig / GenReport keep the reference's meaning for the fields that apply
// to the device path: procs = GPUs (one host thread each), the UCP scheme,
// count-only generation (the reference's empty out_dir).
struct GenConfig {
  int procs = 1;
  std::uint64_t seed = 1;
  std::vector<int> devices;      // default: 0 .. procs-1
  bool counter_stream = true;    // false: the bit-exact reference stream
};

struct RankReport {
  int rank = 0;
  node_t n_lo = 0, n_hi = 0;
  std::int64_t edges = 0;
  double gen_wall_ms = 0.0;  // the timed generation section (runtime.cpp:74-86)
  double kernel_ms = 0.0;    // its sampler kernel on the device
};

struct GenReport {
  int procs = 1;
  std::vector<node_t> boundaries;
  std::vector<RankReport> ranks;
  std::int64_t total_edges = 0;
  std::uint64_t checksum = 0;
  std::int64_t flagged = 0;
  double sum_S = 0.0, sum_check = 0.0;
  double wall_ms = 0.0, plan_ms = 0.0;
  int nccl_version = 0;  // 0: in-process host communicator (ranks sharing a GPU)
};

inline GenReport generate(const WeightSequence& ws, const GenConfig& cfg) {
  if (cfg.procs < 1) throw error("generate: procs must be >= 1");
  std::vector<int> devs = cfg.devices;
  if (devs.empty())
    for (int g = 0; g < cfg.procs; ++g) devs.push_back(g);
  if (static_cast<int>(devs.size()) != cfg.procs) throw error("generate: one device per rank");
  GenReport rep;
  rep.procs = cfg.procs;
  rep.boundaries.assign(static_cast<size_t>(cfg.procs) + 1, 0);
  std::vector<std::int64_t> edges(static_cast<size_t>(cfg.procs));
  std::vector<double> gen(static_cast<size_t>(cfg.procs)), kern(static_cast<size_t>(cfg.procs));
  clgen_spmd_report r{};
  check(clgen_spmd_generate(devs.data(), cfg.procs, ws.weights.data(), ws.size(), cfg.seed,
                            cfg.counter_stream ? CLGEN_STREAM_COUNTER : CLGEN_STREAM_REFERENCE,
                            rep.boundaries.data(), edges.data(), gen.data(), kern.data(), &r));
  for (int g = 0; g < cfg.procs; ++g)
    rep.ranks.push_back(RankReport{g, rep.boundaries[static_cast<size_t>(g)], rep.boundaries[static_cast<size_t>(g) + 1],
                                   edges[static_cast<size_t>(g)], gen[static_cast<size_t>(g)], kern[static_cast<size_t>(g)]});
  rep.total_edges = r.total_edges;
  rep.checksum = r.checksum;
  rep.flagged = r.n_flagged;
  rep.sum_S = r.S;
  rep.sum_check = r.S_check;
  rep.wall_ms = r.wall_ms;
  rep.plan_ms = r.plan_ms;
  rep.nccl_version = r.nccl_version;
  return rep;
}

}  // namespace clgen_b200
