// C++ drop-in test: the reference's own call patterns (test_edge_skip.cpp,
// test_partition.cpp) against the clgen_b200:: mirror.  Prints one line per
// check and exits non-zero on failure.  Needs a GPU at run time.
#include <cstdio>
#include <vector>

#include <functional>
#include "clgen_b200.hpp"

namespace clgen = clgen_b200;
using namespace clgen;

static int failures = 0;
#define CHECK(x)                                                  \
  do {                                                            \
    if (!(x)) {                                                   \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x);     \
      ++failures;                                                 \
    }                                                             \
  } while (0)

int main() {
  // test_partition.cpp:134-144: (4,3,2,1), P=2 -> (0,1,4)
  const auto ws = make_weight_sequence({4, 3, 2, 1}, SortPolicy::require_sorted);
  CHECK(ws.sum_S == 10.0);
  CHECK((plan_ucp_oracle(ws, 2).boundaries == std::vector<node_t>{0, 1, 4}));

  // test_edge_skip.cpp:84-96: degenerate cases and contract errors
  const auto four = make_weight_sequence({2, 2, 2, 2}, SortPolicy::require_sorted);
  EdgeVector sink;
  const std::vector<node_t> last{3};
  CHECK(create_edges(four, four.sum_S, last, 1, sink) == 0);
  bool threw = false;
  try {
    const std::vector<node_t> bad{99};
    create_edges(four, four.sum_S, bad, 1, sink);
  } catch (const error&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    make_weight_sequence({1, 2}, SortPolicy::require_sorted);
  } catch (const error&) {
    threw = true;
  }
  CHECK(threw);

  // sort_desc keeps labels (weights.cpp:41-46)
  const auto sd = make_weight_sequence({1, 3, 2}, SortPolicy::sort_desc);
  CHECK((sd.orig_labels == std::vector<node_t>{1, 2, 0}));

  // serial_cl is deterministic, canonical, and equals any disjoint cover
  std::vector<double> w(2000);
  for (size_t i = 0; i < w.size(); ++i) w[i] = 5.0 - 4.0 * static_cast<double>(i) / w.size();
  const auto big = make_weight_sequence(w, SortPolicy::require_sorted);
  EdgeVector a, b, c;
  serial_cl(big, 42, a);
  serial_cl(big, 42, b);
  CHECK(a.edges == b.edges);
  CHECK(a.count() == static_cast<std::int64_t>(a.edges.size()));
  create_edges_range(big, big.sum_S, 0, 700, 42, c);
  create_edges_range(big, big.sum_S, 700, big.size(), 42, c);
  CHECK(c.edges == a.edges);
  for (const Edge& e : a.edges) CHECK(e.u < e.v && e.v < big.size());
  const auto f = stream_range(big, big.sum_S, 0, big.size(), 42, false);
  CHECK(f.edges == a.count());
  EdgeCounter counter;
  CHECK(serial_cl(big, 42, counter) == a.count() && counter.count() == a.count());

  // generate (runtime.cpp:93-138) over one host thread per rank: the plan is
  // plan_ucp_oracle's and the union of the ranks' streams is serial_cl's
  for (int procs : {1, 3}) {
    GenConfig cfg;
    cfg.procs = procs;
    cfg.seed = 42;
    cfg.devices.assign(static_cast<size_t>(procs), 0);  // one GPU: ranks share it
    cfg.counter_stream = false;
    const GenReport rep = generate(big, cfg);
    CHECK(rep.boundaries == plan_ucp_oracle(big, procs).boundaries);
    CHECK(rep.total_edges == a.count());
    CHECK(rep.checksum == f.checksum);
    CHECK(rep.sum_S == big.sum_S);
    std::int64_t sum = 0;
    for (const auto& r : rep.ranks) sum += r.edges;
    CHECK(sum == rep.total_edges);
  }

  // synth_powerlaw (weights.cpp:103-128) on the device.  Known answer from the
  // real reference (tests/golden/edges_pl3000.npz, acceptance.cpp:299 recipe):
  // synth_powerlaw(3000, 2.5, 2, 50, 0xDE7) generates 6974 edges at seed 1234.
  {
    const auto pl = synth_powerlaw(3000, 2.5, 2.0, 50.0, 0xDE7);
    CHECK(pl.size() == 3000);
    CHECK(std::is_sorted(pl.weights.begin(), pl.weights.end(), std::greater<double>{}));
    CHECK(pl.weights.front() <= 50.0 && pl.weights.back() >= 2.0);
    CHECK(pl.sum_S == blocked_sum(pl.weights));
    EdgeCounter cnt;
    CHECK(serial_cl(pl, 1234, cnt) == 6974);
    const auto same = make_weight_sequence(pl.weights, SortPolicy::require_sorted);
    CHECK(same.sum_S == pl.sum_S);
    bool bad = false;
    try {
      synth_powerlaw(10, 1.0, 1.0, 2.0, 1);
    } catch (const error& e) {
      bad = std::string(e.what()).find("gamma must be > 1") != std::string::npos;
    }
    CHECK(bad);
    const auto vr = validate(pl);  // weights.cpp:142-153
    CHECK(vr.is_sorted && vr.admissible && vr.n == 3000 && vr.max_weight == pl.weights.front() &&
          vr.zero_weight_count == 0 && vr.sum_S == pl.sum_S);
    CHECK(!validate(make_weight_sequence({3, 1, 0}, SortPolicy::require_sorted)).admissible);  // 9 >= 4
    const auto k = synth_constant(1000, 5.0);  // weights.cpp:130-140
    CHECK(k.size() == 1000 && k.sum_S == 5000.0);
    bad = false;
    try {
      synth_constant(4, 4.0);
    } catch (const error&) {
      bad = true;
    }
    CHECK(bad);
  }

  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
