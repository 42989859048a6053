/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference clgen hot path (Alam & Khan,
 * arXiv:1406.1215, as implemented in /root/reference/proj/core).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  Pinned against the compiled reference (oracle/_ref) and the
 * reference tests' known answers by tests/test_oracle.py.
 *
 * FP discipline: compiled with -ffp-contract=off and no -march, i.e. the same
 * x86-64 SSE2 double arithmetic and glibc libm (log, log1p, pow, floor) the
 * reference build uses.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- RNG: rng.hpp:11-69 ------------------------------------------------- */

/* rng.hpp:11-16 */
uint64_t orc_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:20-22 */
uint64_t orc_node_rng_key(uint64_t seed, int64_t u) {
  return orc_mix64(seed + (uint64_t)u * 0x9e3779b97f4a7c15ULL);
}

typedef struct { uint64_t s[4]; } orc_rng;

/* rng.hpp:30-42: four splitmix64 steps from the key; all-zero guard. */
static void rng_init_key(orc_rng* g, uint64_t key) {
  uint64_t sm = key;
  int nonzero = 0;
  for (int i = 0; i < 4; ++i) {
    sm += 0x9e3779b97f4a7c15ULL;
    uint64_t z = sm;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    g->s[i] = z ^ (z >> 31);
    nonzero |= g->s[i] != 0;
  }
  if (!nonzero) g->s[0] = 1;
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:44-54 xoshiro256++ */
static inline uint64_t rng_next(orc_rng* g) {
  uint64_t* s = g->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:58-63: (x>>11)*2^-53, exact zeros rejected. */
static inline double rng_open01(orc_rng* g) {
  for (;;) {
    const double r = (double)(rng_next(g) >> 11) * 0x1.0p-53;
    if (r > 0.0) return r;
  }
}

void orc_stream_open01(uint64_t seed, int64_t u, int64_t count, double* out) {
  orc_rng g;
  rng_init_key(&g, orc_node_rng_key(seed, u));
  for (int64_t i = 0; i < count; ++i) out[i] = rng_open01(&g);
}

/* ---- weights.cpp:21-30 blocked_sum ------------------------------------- */
double orc_blocked_sum(const double* xs, int64_t n) {
  double total = 0.0;
  for (int64_t lo = 0; lo < n; lo += 4096) {
    const int64_t hi = lo + 4096 < n ? lo + 4096 : n;
    double part = 0.0;
    for (int64_t k = lo; k < hi; ++k) part += xs[k];
    total += part;
  }
  return total;
}

/* weights.cpp:155-162 expected_total_edges */
double orc_expected_total_edges(const double* w, int64_t n, double S) {
  if (!(S > 0.0)) return 0.0;
  double* sq = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) sq[i] = w[i] * w[i];
  const double ssq = orc_blocked_sum(sq, n);
  free(sq);
  return (S * S - ssq) / (2.0 * S);
}

static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}

/* weights.cpp:103-128 synth_powerlaw, values only (the stable label sort of
 * make_weight_sequence, :41-46, does not change the sorted values).
 * Returns 0, or -1 on a contract violation (:105-108). */
int orc_synth_powerlaw(int64_t n, double gamma, double w_min, double w_max, uint64_t seed,
                       double* out) {
  if (n < 1 || !(gamma > 1.0) || !(w_min > 0.0) || w_min > w_max) return -1;
  orc_rng g;
  rng_init_key(&g, orc_mix64(seed ^ 0x706c73796e7468ULL)); /* weights.cpp:17,112 */
  if (w_min == w_max) {
    for (int64_t i = 0; i < n; ++i) out[i] = w_min;
    return 0;
  }
  const double k = 1.0 - gamma;
  const double ak = pow(w_min, k);
  const double bk = pow(w_max, k);
  for (int64_t i = 0; i < n; ++i) {
    const double u = rng_open01(&g);
    double w = pow(ak + u * (bk - ak), 1.0 / k);
    if (w < w_min) w = w_min; /* std::clamp */
    if (w > w_max) w = w_max;
    out[i] = w;
  }
  qsort(out, (size_t)n, sizeof(double), cmp_desc);
  return 0;
}

/* ---- edge_skip.cpp:9-16 skip_length ------------------------------------ */
/* Returns 0 and writes *out, or -1 on the contract violations of :10-11. */
int orc_skip_length(double p, double r, int64_t* out) {
  if (!(p > 0.0) || !(p <= 1.0)) return -1;
  if (!(r > 0.0) || !(r < 1.0)) return -1;
  if (p >= 1.0) { *out = 0; return 0; }
  const double ratio = log(r) / log1p(-p);
  if (!(ratio < 9.0e18)) { *out = INT64_MAX; return 0; }
  *out = (int64_t)ratio;
  return 0;
}

/* Checksum term of one edge (the device fold's edge_hash, common.cuh; not a
 * reference function): multiply / fold / multiply / fold of (u << 32) | v. */
uint64_t orc_edge_hash(uint64_t u, uint64_t v) {
  uint64_t z = ((u << 32) | v) * 0x9e3779b97f4a7c15ULL;
  z ^= z >> 32;
  z *= 0xd6e8feb86659fd93ULL;
  return z ^ (z >> 32);
}

/* Edge consumer: materialise as uint32 pairs and/or fold into a checksum and
 * undirected degree counters. */
typedef struct {
  uint32_t* pairs;     /* may be NULL */
  int64_t cap;
  int64_t count;
  uint64_t checksum;   /* sum of orc_edge_hash(u, v) mod 2^64 */
  int64_t* degree;     /* may be NULL */
} orc_sink;

static inline void sink_emit(orc_sink* s, int64_t u, int64_t v) {
  if (s->pairs && s->count < s->cap) {
    s->pairs[2 * s->count] = (uint32_t)u;
    s->pairs[2 * s->count + 1] = (uint32_t)v;
  }
  s->checksum += orc_edge_hash((uint64_t)u, (uint64_t)v);
  if (s->degree) { ++s->degree[u]; ++s->degree[v]; }
  ++s->count;
}

/* ---- edge_skip.cpp:20-46 edges_from_source (the hot loop) -------------- */
static int64_t edges_from_source(const double* w, int64_t n, double S, int64_t u, uint64_t seed,
                                 orc_sink* sink) {
  int64_t j = u + 1;
  if (j >= n || !(S > 0.0)) return 0;
  const double w_u = w[u];
  orc_rng g;
  rng_init_key(&g, orc_node_rng_key(seed, u));
  int64_t emitted = 0;
  double p = w_u * w[j] / S;
  if (p > 1.0) p = 1.0;
  while (j < n && p > 0.0) {
    int64_t delta = 0;
    if (p < 1.0) orc_skip_length(p, rng_open01(&g), &delta);
    if (delta >= n - j) break;
    const int64_t v = j + delta;
    double q = w_u * w[v] / S;
    if (q > 1.0) q = 1.0;
    const double r = rng_open01(&g);
    if (r < q / p) {
      sink_emit(sink, u, v);
      ++emitted;
    }
    p = q;
    j = v + 1;
  }
  return emitted;
}

/* edge_skip.cpp:60-66 create_edges_range.  pairs/degree may be NULL.
 * Returns 0 or -1 on a bad range (:62). */
int orc_create_edges_range(const double* w, int64_t n, double S, int64_t lo, int64_t hi,
                           uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* degree,
                           int64_t* count, uint64_t* checksum) {
  if (lo < 0 || hi > n || lo > hi) return -1;
  orc_sink s = {pairs, cap, 0, 0, degree};
  for (int64_t u = lo; u < hi; ++u) edges_from_source(w, n, S, u, seed, &s);
  *count = s.count;
  if (checksum) *checksum = s.checksum;
  return 0;
}

/* edge_skip.cpp:50-58 create_edges over a source list. */
int orc_create_edges(const double* w, int64_t n, double S, const int64_t* sources, int64_t k,
                     uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* count,
                     uint64_t* checksum) {
  orc_sink s = {pairs, cap, 0, 0, NULL};
  for (int64_t i = 0; i < k; ++i) {
    if (sources[i] < 0 || sources[i] >= n) return -1;
    edges_from_source(w, n, S, sources[i], seed, &s);
  }
  *count = s.count;
  if (checksum) *checksum = s.checksum;
  return 0;
}

/* Per-source edge counts (the count pass) for [lo,hi). */
void orc_edge_counts(const double* w, int64_t n, double S, int64_t lo, int64_t hi, uint64_t seed,
                     int64_t* counts) {
  for (int64_t u = lo; u < hi; ++u) {
    orc_sink s = {NULL, 0, 0, 0, NULL};
    edges_from_source(w, n, S, u, seed, &s);
    counts[u - lo] = s.count;
  }
}

/* ---- cost.cpp:8-60 ----------------------------------------------------- */

/* cost.cpp:8-13 */
int orc_node_cost(double w_u, double sigma_u, double S, double* out) {
  if (!(S > 0.0)) return -1;
  double e = (w_u / S) * (S - sigma_u - w_u);
  if (e < 0.0) e = 0.0;
  *out = e + 1.0;
  return 0;
}

/* cost.cpp:15-22 ceil-first split */
int orc_block_bounds(int64_t n, int P, int rank, int64_t* lo, int64_t* hi) {
  if (P < 1 || rank < 0 || rank >= P) return -1;
  const int64_t q = n / P, r = n % P;
  *lo = (int64_t)rank * q + ((int64_t)rank < r ? (int64_t)rank : r);
  *hi = *lo + q + ((int64_t)rank < r ? 1 : 0);
  return 0;
}

/* cost.cpp:53-60 */
int orc_partition_of(double c, double z_bar, int P, int* out) {
  if (!(z_bar > 0.0)) return -1;
  const double k = floor(c / z_bar);
  if (k < 0.0) { *out = 0; return 0; }
  if (k >= (double)P) { *out = P - 1; return 0; }
  const int i = (int)k;
  *out = i > P - 1 ? P - 1 : i;
  return 0;
}

/* cost.cpp:24-46 block_cumulative: local (pre-offset) C_u for rank's block,
 * sigma advanced from sigma_start; returns block_cost (last C or 0). */
double orc_block_cumulative(const double* w, int64_t n, double S, int rank, int P,
                            double sigma_start, double* cum_out) {
  int64_t lo, hi;
  orc_block_bounds(n, P, rank, &lo, &hi);
  const int zero_sum = !(S > 0.0);
  double sigma = sigma_start, cum = 0.0, c;
  for (int64_t u = lo; u < hi; ++u) {
    if (zero_sum) c = 1.0; else orc_node_cost(w[u], sigma, S, &c);
    cum = (u == lo) ? c : cum + c;
    cum_out[u - lo] = cum;
    sigma += w[u];
  }
  return hi > lo ? cum_out[hi - lo - 1] : 0.0;
}

/* partition.cpp:159-203 plan_ucp_oracle.  Writes boundaries[0..P] and, when
 * cum_global != NULL, the finalized C_u (cost.cpp:48-51) for all n nodes and
 * per-block weights/costs.  Returns 0, or -1 for P < 1 (:160). */
int orc_plan_ucp(const double* w, int64_t n, double S, int P, int64_t* boundaries,
                 double* cum_global, double* block_weights, double* block_costs) {
  if (P < 1) return -1;
  if (n == 0) {
    for (int i = 0; i <= P; ++i) boundaries[i] = 0;
    return 0;
  }
  double* bw = (double*)calloc((size_t)P, sizeof(double));
  double* bc = (double*)calloc((size_t)P, sizeof(double));
  double* cum = cum_global ? cum_global : (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < P; ++i) { /* partition.cpp:165-170 */
    int64_t lo, hi;
    orc_block_bounds(n, P, i, &lo, &hi);
    double acc = 0.0;
    for (int64_t u = lo; u < hi; ++u) acc += w[u];
    bw[i] = acc;
  }
  for (int i = 0; i < P; ++i) { /* :172-177, fold_prefix :83-87 */
    int64_t lo, hi;
    orc_block_bounds(n, P, i, &lo, &hi);
    double sp = 0.0;
    for (int j = 0; j < i; ++j) sp += bw[j];
    bc[i] = orc_block_cumulative(w, n, S, i, P, sp, cum + lo);
  }
  for (int i = 0; i < P; ++i) { /* :178 finalize_offsets */
    int64_t lo, hi;
    orc_block_bounds(n, P, i, &lo, &hi);
    double zp = 0.0;
    for (int j = 0; j < i; ++j) zp += bc[j];
    for (int64_t u = lo; u < hi; ++u) cum[u] += zp;
  }
  double total = 0.0; /* :180-181 */
  for (int j = 0; j < P; ++j) total += bc[j];
  const double z_bar = total / P;
  for (int i = 0; i <= P; ++i) boundaries[i] = n;
  boundaries[0] = 0;
  int prev = 0; /* :191-200 linear scan */
  for (int64_t u = 0; u < n; ++u) {
    int cur;
    orc_partition_of(cum[u], z_bar, P, &cur);
    for (int k = prev + 1; k <= cur; ++k) boundaries[k] = u;
    prev = cur;
  }
  boundaries[P] = n;
  if (block_weights) memcpy(block_weights, bw, sizeof(double) * (size_t)P);
  if (block_costs) memcpy(block_costs, bc, sizeof(double) * (size_t)P);
  if (!cum_global) free(cum);
  free(bw);
  free(bc);
  return 0;
}
