/*
 * clgen_dev.h — C ABI of the B200-native Chung–Lu generator.
 *
 * This is the drop-in boundary for the reference's generator entry points
 * (namespace clgen in /root/reference/proj/core).  Plain pointers and sizes
 * only; no exceptions cross it.  Every function returns CLGEN_OK (0) or a
 * negative status; clgen_dev_last_error() returns the calling thread's last
 * message.  The C++ mirror in clgen_b200.hpp turns statuses into
 * clgen::error exceptions exactly where the reference throws.
 *
 * Pointers marked "host or device" are classified with
 * cudaPointerGetAttributes: device pointers are used in place, host pointers
 * are staged through the context's device buffers (copies on the context
 * stream, the call returns when they completed).
 *
 * Threading: one context per host thread / GPU (the run_spmd rank analogue,
 * comm.cpp:204-227).  Contexts share nothing.
 */
#ifndef CLGEN_DEV_H
#define CLGEN_DEV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLGEN_OK 0
#define CLGEN_EINVAL (-1)   /* contract violation: the reference throws clgen::error */
#define CLGEN_ECUDA (-2)    /* CUDA runtime / launch failure */
#define CLGEN_ENOMEM (-3)   /* device allocation failed */
#define CLGEN_ERANGE (-4)   /* output capacity exceeded */

typedef struct clgen_dev_ctx clgen_dev_ctx;

/* Stream modes for the sampler. */
#define CLGEN_STREAM_REFERENCE 0 /* per-node xoshiro256++ (rng.hpp:26-69): bit-exact */
#define CLGEN_STREAM_COUNTER 1   /* keyed xoroshiro128++ per (seed,class-pair block,chunk,lane):
                                    statistical, GPU-count / partition / launch invariant */

const char* clgen_dev_last_error(void);
const char* clgen_dev_version(void);

/* Context on CUDA device `device` with its own non-blocking stream. */
int clgen_dev_create(int device, clgen_dev_ctx** out);
int clgen_dev_destroy(clgen_dev_ctx* ctx);
/* The context stream (cudaStream_t) so callers can time / order work on it. */
void* clgen_dev_stream(clgen_dev_ctx* ctx);
int clgen_dev_synchronize(clgen_dev_ctx* ctx);
/* Instrumentation: kernels this context has launched so far, and the device
 * duration (CUDA events on the context stream) of the last sampler kernel. */
unsigned long long clgen_dev_launch_count(clgen_dev_ctx* ctx);
int clgen_dev_last_kernel_ms(clgen_dev_ctx* ctx, float* ms);

/*
 * Weights: replaces make_weight_sequence(w, SortPolicy::require_sorted)
 * (weights.cpp:32-55).  `w` (host or device) must be non-increasing and
 * non-negative; violations return CLGEN_EINVAL with the reference's message
 * ("weights unsorted at position u").  The context keeps its own device copy.
 * `n` may be 0.  Node ids must fit uint32 (n < 2^32).
 */
int clgen_dev_set_weights(clgen_dev_ctx* ctx, const double* w, int64_t n);
/* Starts copying the NEXT weight array (host, ideally page-locked, or device)
 * into a second device buffer on the context's copy stream and returns at
 * once: the copy overlaps whatever the context is generating.  The next
 * clgen_dev_set_weights call with the same pointer and n takes that copy (it
 * waits for it on the device, swaps the buffers and runs its checks) instead
 * of copying; any other set_weights call ignores it.  The caller keeps `w`
 * unchanged until then.  No reference counterpart: ingestion pipelining. */
int clgen_dev_prefetch_weights(clgen_dev_ctx* ctx, const double* w, int64_t n);
int64_t clgen_dev_num_nodes(clgen_dev_ctx* ctx);
/* Device pointer of the context's weight copy (read-only). */
const double* clgen_dev_weights(clgen_dev_ctx* ctx);
/* CUDA device ordinal of the context. */
int clgen_dev_device(clgen_dev_ctx* ctx);
/* Copies the first n resident weights to `out` (host or device memory). */
int clgen_dev_copy_weights(clgen_dev_ctx* ctx, double* out, int64_t n);

/*
 * Device weight synthesis: replaces synth_powerlaw(n, gamma, w_min, w_max, seed)
 * (weights.cpp:103-128; continuous truncated power law by inverse CDF over the
 * sequential synth stream, weights.cpp:17,112) followed, when `sort_desc` is
 * non-zero, by the descending sort of make_weight_sequence (weights.cpp:32-55;
 * values only).  `d_out` is DEVICE memory for n doubles; its contents equal the
 * reference's array bit for bit: the xoshiro stream is entered at every 2048th
 * draw by GF(2) jump matrices, the inverse CDF's pow is evaluated in
 * double-double with a rounding certificate, and the draws that cannot be
 * certified (about 1/16; their count is returned in `n_host_resolved`) are
 * resolved by the host's libm pow, the reference's own dependency.
 * `target_mean` > 0 then multiplies every weight by target_mean / (blocked_sum / n)
 * (the C4 recipe).  Errors like the reference for n < 1, gamma <= 1,
 * w_min <= 0 or w_min > w_max (CLGEN_EINVAL); CLGEN_ERANGE if the stream holds
 * a zero draw (probability n * 2^-53), which the reference redraws.
 * Pass the result to clgen_dev_set_weights (device pointers are accepted), or
 * pass d_out = NULL: the array is then synthesised into scratch memory on the
 * context's device and installed as the context's weights directly
 * (make_weight_sequence(synth_powerlaw(...)) without a host copy;
 * clgen_dev_copy_weights reads it back).
 */
int clgen_dev_synth_powerlaw(clgen_dev_ctx* ctx, int64_t n, double gamma, double w_min, double w_max,
                             uint64_t seed, int sort_desc, double target_mean, double* d_out,
                             int64_t* n_host_resolved);

/*
 * make_weight_sequence(w, SortPolicy::sort_desc) (weights.cpp:32-55) on the
 * device: sorts the n doubles at `d_w` (DEVICE memory) into non-increasing
 * order in place, stably, and, when `d_labels` (DEVICE memory, n int64) is
 * non-NULL, writes orig_labels: labels[i] = input position of the weight now at
 * i.  Equals the reference's std::stable_sort order, except that a -0.0 sorts
 * after +0.0 (the reference keeps the two in input order).
 */
int clgen_dev_sort_desc(clgen_dev_ctx* ctx, double* d_w, int64_t n, int64_t* d_labels);

/*
 * S = blocked_sum(w) (weights.cpp:21-30): 4096-element blocks folded left to
 * right from 0.0, partials folded left to right.  Bit-identical.
 */
int clgen_dev_blocked_sum(clgen_dev_ctx* ctx, double* S);
/* blocked_sum(span<const double>) of an arbitrary array (host or device). */
int clgen_dev_blocked_sum_array(clgen_dev_ctx* ctx, const double* xs, int64_t n, double* S);

/*
 * Materialised generation: replaces create_edges_range(ws, S, lo, hi, seed,
 * EdgeVector&) (edge_skip.cpp:60-66, hot loop :20-46).  Writes the edges as
 * uint32 (u,v) pairs into `pairs` (host or device, 2*cap uint32) in the
 * reference's emission order (u ascending, then v ascending) and the count to
 * *count.  Returns CLGEN_ERANGE (with *count set) when count > cap.
 * *n_flagged = sources whose skip ratio came within 2^-47 of an integer
 * (where CUDA's and glibc's log/log1p may disagree); their ids are available
 * from clgen_dev_flagged_nodes.  Errors like the reference for
 * lo < 0 || hi > n || lo > hi ("create_edges_range: bad node range").
 */
int clgen_dev_create_edges_range(clgen_dev_ctx* ctx, double S, int64_t lo, int64_t hi,
                                 uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* count,
                                 int64_t* n_flagged);

/*
 * Replaces create_edges(ws, S, sources, seed, sink) (edge_skip.cpp:50-58):
 * the sources (host or device int64, k entries) are walked in list order and
 * their edges written in that order.  Any source outside [0,n) returns
 * CLGEN_EINVAL ("create_edges: source node out of range").
 */
int clgen_dev_create_edges(clgen_dev_ctx* ctx, double S, const int64_t* sources, int64_t k,
                           uint64_t seed, uint32_t* pairs, int64_t cap, int64_t* count,
                           int64_t* n_flagged);

/*
 * Materialised generation with a selectable stream: CLGEN_STREAM_REFERENCE is
 * exactly clgen_dev_create_edges_range; CLGEN_STREAM_COUNTER draws from the
 * counter-based stream (statistically exact, deterministic per seed,
 * independent of GPU count).  Output order: u ascending, then v ascending.
 */
int clgen_dev_generate_range(clgen_dev_ctx* ctx, double S, int64_t lo, int64_t hi, uint64_t seed,
                             int stream_mode, uint32_t* pairs, int64_t cap, int64_t* count,
                             int64_t* n_flagged);

/* Counter-stream tunables: weight-class width (w_first <= (1+class_eps)
 * w_last inside a class; 0 = automatic: 1/128, doubled at most twice while the
 * class-pair blocks would average fewer than 8192 expected candidates; any
 * width is doubled until the classes fit 1024) and the chunk size in expected
 * candidates (0 = automatic: S / 2^16 clamped to [4096, 262144]; explicit
 * range [256, 2^20]).  Automatic values are functions of the weights only.
 * Both are part of the stream definition: changing them changes the
 * generated graph (not its law). */
int clgen_dev_set_counter_params(clgen_dev_ctx* ctx, double class_eps, double chunk_cand);
/* Reference stream arithmetic: 1 (default) = fast guarded FP64 (table log,
 * series log1p, FMA-certified divisions; falls back to the reference
 * expressions near rounding/floor boundaries, so results are identical);
 * 0 = the reference expressions everywhere (validation). */
int clgen_dev_set_fast_math(clgen_dev_ctx* ctx, int enable);
/* Level-2 load-balance evidence: when enabled, the sampler kernels record
 * each warp's busy interval (%globaltimer).  For sampler launch `launch` of
 * the last generation call (0 .. clgen_dev_warp_profile_launches()-1) report max/mean
 * per-warp busy time, mean and max in ms, the span first-start to last-end,
 * and the number of warps. */
int clgen_dev_set_warp_profile(clgen_dev_ctx* ctx, int enable);

/* Kernel schedule (no reference counterpart; the edge set does not depend on
 * it).  shape: counter-stream kernel, 256 threads x 2 / 3 (default) / 4 / 5 /
 * 6 CTAs per SM for shape 0 / 1 / 2 / 3 / 4, -1 = CLGEN_BLK_SHAPE or the
 * default.  flags: CLGEN_SHAPE_NO_HEAVY_PHASE walks every reference-stream
 * slot per lane (by default the heaviest chains are walked one per warp).
 * Used by the schedule-invariance tests. */
#define CLGEN_SHAPE_NO_HEAVY_PHASE 1
int clgen_dev_set_kernel_shape(clgen_dev_ctx* ctx, int shape, int flags);
int clgen_dev_warp_profile_launches(clgen_dev_ctx* ctx);
int clgen_dev_warp_profile(clgen_dev_ctx* ctx, int launch, double* max_over_mean, double* mean_ms,
                           double* max_ms, double* span_ms, int64_t* warps);
/* Size of the counter plan of the last counter-stream call: weight classes
 * (incl. the zero class), class-pair blocks, chunks over all sources, dense
 * blocks (envelope >= 1) and the class width actually used. */
int clgen_dev_counter_plan_info(clgen_dev_ctx* ctx, int* classes, int64_t* blocks, int64_t* chunks,
                                int* dense_blocks, double* class_eps);

/* Statistical-test support for the counter stream: runs the generator over
 * all sources for seeds seed, seed+1, ..., seed+trials-1 in ONE launch (each
 * trial is exactly clgen_dev_stream_range / generate_range with that seed)
 * and counts every edge (u, v) in counts[u * n + v] (uint32, n*n entries,
 * host or device; n <= 4096).  The per-pair frequencies are the law check of
 * acceptance.cpp:80-124. */
int clgen_dev_pair_trials(clgen_dev_ctx* ctx, double S, uint64_t seed, int64_t trials, uint32_t* counts);

/* Count pass only: per-source edge counts (int32, hi-lo entries, host or device). */
int clgen_dev_edge_counts(clgen_dev_ctx* ctx, double S, int64_t lo, int64_t hi, uint64_t seed,
                          int32_t* counts, int64_t* total, int64_t* n_flagged);

/*
 * Streaming generation with fused fold (no materialised edge list):
 * *count = edges, *checksum = sum over edges of edge_hash(u, v) mod 2^64
 * (z = ((u<<32)|v) * 0x9e3779b97f4a7c15; z ^= z>>32; z *= 0xd6e8feb86659fd93;
 * z ^ z>>32 — the fold's own definition, mirrored by the oracle), `degree` (host or device, may be NULL) receives
 * undirected degrees of the tracked nodes x with x % 2^track_shift == 0 at
 * degree[x >> track_shift] (uint32, ceil(n / 2^track_shift) entries; counts
 * are ADDED to the existing contents when `degree` is a device pointer and
 * `accumulate` != 0, else overwritten).  When `ring` (device) is non-NULL
 * every edge is also written into it at (position mod ring_cap); ring_cap is
 * a power of two.  stream_mode selects CLGEN_STREAM_REFERENCE (bit-exact
 * per-node streams) or CLGEN_STREAM_COUNTER.
 */
int clgen_dev_stream_range(clgen_dev_ctx* ctx, double S, int64_t lo, int64_t hi, uint64_t seed,
                           int stream_mode, int track_shift, uint32_t* degree, int accumulate,
                           uint32_t* ring, int64_t ring_cap, int64_t* count, uint64_t* checksum,
                           int64_t* n_flagged);

/*
 * Level-1 uniform-cost partition (UCP) of this context's weights into P
 * consecutive blocks, bit-identical to plan_ucp_oracle(ws, P)
 * (partition.cpp:159-203) and hence to the SPMD plan_ucp (:107-157).  The
 * reference's P-blocked sequential FP64 folds (block weights, sigma_u, C_u)
 * are replayed exactly by a parallel per-binade integer scan.
 * boundaries: P+1 int64 (host or device).  cum_costs (optional, host or
 * device, n doubles) receives the finalized C_u (cost.cpp:48-51).
 * P < 1 returns CLGEN_EINVAL ("plan_ucp_oracle: P must be >= 1").
 */
int clgen_dev_plan_ucp(clgen_dev_ctx* ctx, int P, int64_t* boundaries, double* cum_costs);

/*
 * The same plan split into per-rank device phases for G GPUs (rank g calls
 * them on its own context; the caller performs the collectives between them,
 * folding gathered values in rank order as comm.cpp:39-53 does):
 *   1. block weight of rank block g, a fold from 0.0 (partition.cpp:115-116)
 *   2. block_cumulative from sigma_start (cost.cpp:24-46); returns z_g
 *   3. boundaries found in block g given Z_g and Z_bar: found[0..G] (host or
 *      device int64) receives u for every k crossed inside the block, n
 *      elsewhere; the element-wise MIN over ranks is the plan.
 */
int clgen_dev_plan_block_weight(clgen_dev_ctx* ctx, int G, int g, double* block_weight);
int clgen_dev_plan_block_costs(clgen_dev_ctx* ctx, int G, int g, double sigma_start, double S,
                               double* block_cost);
int clgen_dev_plan_block_boundaries(clgen_dev_ctx* ctx, int G, int g, double z_offset,
                                    double z_bar, int64_t* found);

/* Partition schemes (partition.hpp:15). */
#define CLGEN_SCHEME_NAIVE 0
#define CLGEN_SCHEME_UCP 1
#define CLGEN_SCHEME_RRP 2

/* node_costs_sequential (cost.cpp:62-77): the suffix-form per-node cost
 * (w_u / S) * sum_{v>u} w_v + 1 with the suffix accumulated backward from
 * 0.0, bit-identical (an exact reversed fold); costs: n doubles, host or
 * device. */
int clgen_dev_node_costs(clgen_dev_ctx* ctx, double* costs);
/* fill_partition_costs (partition.cpp:205-222): per-partition expected cost,
 * each a left fold from 0.0 of node_costs_sequential over the partition's
 * nodes (consecutive [b_i, b_{i+1}) for naive/ucp, u = i mod P ascending for
 * rrp), bit-identical.  boundaries: P+1 (host or device; ignored for rrp);
 * per: P doubles (host). */
int clgen_dev_partition_costs(clgen_dev_ctx* ctx, int scheme, int P, const int64_t* boundaries, double* per);
/* expected_total_edges (weights.cpp:155-162): (S^2 - blocked_sum(w^2)) / (2S)
 * with the canonical S, bit-identical; 0 when S <= 0. */
int clgen_dev_expected_total_edges(clgen_dev_ctx* ctx, double* m);

/*
 * Persist edges in the reference's formats (edge_io.cpp:72-88): binary
 * CLGEDGE1 (16-byte header, u64 count, u64 pairs) or text "u v" lines.
 * `pairs` (host or device, uint32 (u,v) pairs, `count` of them) are widened /
 * rendered on the device chunk by chunk and streamed to `path`.  Errors as
 * the reference: "cannot open for writing: <path>", "write failed: <path>".
 */
int clgen_dev_write_edges(clgen_dev_ctx* ctx, const uint32_t* pairs, int64_t count, int binary,
                          const char* path);

/*
 * Degree fidelity, the device analogue of degree_histogram +
 * compare_distributions (analysis.cpp:18-85): `degree` (host or device,
 * uint32, the undirected degree of every node, e.g. clgen_dev_stream_range
 * with track_shift 0 or clgen_dev_edge_degrees) against the expected degree
 * max(w - w^2/S, 0).  scalars[5] = mean_expected (bit-identical: the
 * reference's sequential fold), mean_generated, mean_rel_error,
 * max_flagged_rel_error, zero_degree.  Bins ascending by k = floor(log2 x):
 * up to `cap` of (k, expected_count, generated_count, rel_error, flagged);
 * *nbins = total bins.
 */
int clgen_dev_fidelity(clgen_dev_ctx* ctx, const uint32_t* degree, int64_t total_edges,
                       double flag_mass, double* scalars, int* bin_k, double* bin_expected,
                       int64_t* bin_generated, double* bin_rel, int* bin_flagged, int cap,
                       int* nbins);
/* Undirected degrees of a materialised edge list (uint32 pairs, host or
 * device) into degree[n] (host or device). */
int clgen_dev_edge_degrees(clgen_dev_ctx* ctx, const uint32_t* pairs, int64_t m, uint32_t* degree);

/* Ids of the sources flagged by the last generation call (up to cap). */
int clgen_dev_flagged_nodes(clgen_dev_ctx* ctx, int64_t* out, int64_t cap, int64_t* n);

/*
 * Whole-run SPMD entry, the analogue of generate(ws, GenConfig)
 * (runtime.cpp:93-138) over run_spmd (comm.cpp:204-227): G host threads, one
 * per GPU devices[g], each with its own context.  Every rank copies the
 * (non-increasing) weights w[0..n), computes S itself, runs the level-1 UCP
 * plan (partition.cpp:107-157) with the reference's collectives on NCCL
 * (ncclCommInitAll over the devices; all-gathers of block weights / block
 * costs folded in rank order on the host, MIN all-reduce of the found
 * boundaries), then streams its partition [b_g, b_{g+1}) with the fold
 * (count + checksum; stream_mode as in clgen_dev_stream_range) and the
 * totals are summed with one all-reduce.  Ranks that share a device (tests
 * on a one-GPU box, or CLGEN_SPMD_COMM=host) use an in-process host
 * communicator with the same semantics instead of NCCL.
 * Outputs: boundaries[G+1] (== plan_ucp_oracle(ws, G)); per rank (optional,
 * G entries each): edges, host wall ms and sampler-kernel ms of the timed
 * generation section; and the report below.  Errors: the lowest failing
 * rank's message, prefixed "rank g: ".
 */
typedef struct {
  int G;
  double S;            /* canonical blocked_sum, every rank's */
  double S_check;      /* rank-ordered fold of the block weights (runtime.cpp:55-58) */
  int64_t total_edges;
  uint64_t checksum;   /* sum over all edges of edge_hash(u, v) mod 2^64 */
  int64_t n_flagged;
  double wall_ms;      /* whole SPMD section */
  double plan_ms;      /* max over ranks of the plan (phases + collectives) */
  int nccl_version;    /* 0: the in-process host communicator carried the collectives */
} clgen_spmd_report;

int clgen_spmd_generate(const int* devices, int G, const double* w, int64_t n, uint64_t seed,
                        int stream_mode, int64_t* boundaries, int64_t* rank_edges,
                        double* rank_gen_ms, double* rank_kernel_ms, clgen_spmd_report* report);

#ifdef __cplusplus
}
#endif

#endif /* CLGEN_DEV_H */
