/*
 * clgen_inputs.h - workload input preparation (libclgen_inputs.so, built by
 * inputs/__init__.py).  Shared by both bench arms; not part of the product
 * library, so the reference arm never maps libclgen_b200.so.
 *
 * Not the device hot path: these produce the FP64 weight arrays that both the
 * GPU generator and the CPU baseline consume, bit-identical to the reference
 * synthesisers (weights.cpp:103-140), multi-threaded for n = 1e9.
 * Return 0, or -1 on the reference's contract violations (weights.cpp:105-108).
 */
#ifndef CLGEN_INPUTS_H
#define CLGEN_INPUTS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* synth_powerlaw's draws (weights.cpp:110-125), UNSORTED; sort with
 * clgen_host_sort_desc (or any descending sort: the values are what matter). */
int clgen_host_powerlaw_draws(int64_t n, double gamma, double w_min, double w_max, uint64_t seed,
                              double* out, int threads);

/* Discrete power law P(K=k) ∝ k^-gamma on [k_min,k_max] by inverse CDF on the
 * same synth stream (the C1 recipe); UNSORTED. */
int clgen_host_discrete_powerlaw(int64_t n, double gamma, int64_t k_min, int64_t k_max,
                                 uint64_t seed, double* out, int threads);

/* Parallel descending sort of a double array in place. */
int clgen_host_sort_desc(double* w, int64_t n, int threads);

#ifdef __cplusplus
}
#endif

#endif /* CLGEN_INPUTS_H */
