/* ut_debug.h -- verification entry points of libutrack_b200.so (not part of the
 * reference-facing boundary). Used by the GPU parity tests to check the device
 * primitives exhaustively against the oracle. */
#ifndef UT_DEBUG_H_
#define UT_DEBUG_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Evaluates the device's fp32 noise math on its whole 2^24-point input grid
 * (tracking.cpp:29-36): quantity q = kind % 4: 0 = log(((i)+1) * 2^-24),
 * 1 = cos(2pi_f * i*2^-24), 2 = sin(2pi_f * i*2^-24), 3 = sqrt(-2 log(((i)+1) * 2^-24));
 * kind 0..3 through the fp64-libm path, 4..7 through the table-driven production
 * path. host_out receives 2^24 floats. */
int ut_debug_cr_grid(int kind, int device, float* host_out);
/* Counts results of the step kernel's branch-free fp64 sqrt (kind 0) / division
 * (kind 1) for the particle speed clamp that differ from IEEE __dsqrt_rn /
 * __ddiv_rn over n random operands of the clamp's domain; kind 2 / 3: the
 * likelihood distance sqrt (sqrt_dist) results more than 1 ulp / any ulp away
 * from IEEE over squared distances in [2^-60, 2^31] (x = 0 gives NaN by design: the
 * step then takes its exact path); kind 4: the particle-weight exp
 * (exp_neg) results more than 1 ulp away from libm exp over [-760, 0]. */
int ut_debug_ieee_check(int kind, uint64_t seed, int64_t n, int device, uint64_t* mismatches);
/* n consecutive Philox4x32-10 blocks from block0 (rng.hpp:116-131): 4n words. */
int ut_debug_philox(uint64_t key, uint64_t stream, uint64_t block0, int32_t n, int device, uint32_t* host_out);
struct ut_vecenv;
/* Verification knobs: force_exact != 0 makes every particle set take the exact
 * sequential update path (tracking.cpp:119-143 once per measurement) instead of
 * the merged one; trace_env >= 0 printf's a per-set trace for that env (only
 * in the generic step instance: particle counts other than 256/512/1024 or
 * noise-free configs). */
int ut_debug_set_knobs(struct ut_vecenv* v, int force_exact, int64_t trace_env);
/* Grid-size invariance (the device analogue of the reference's worker-count
 * invariance, test_vecenv.cpp:126-143): runs the step / reset kernels on `ctas`
 * co-resident CTAs (1 .. the default grid; 0 restores the default), which
 * changes every CTA's static env range and the dynamic set schedule. */
int ut_debug_set_grid(struct ut_vecenv* v, int32_t ctas);
/* Per-CTA busy cycles (every phase, not the grid-barrier waits) of the step
 * kernel since phase timing was enabled
 * (ut_vecenv_enable_phase_timing): *n = grid size; out may be NULL to query it.
 * Shows the load balance of the persistent grid. */
int ut_debug_cta_cycles(struct ut_vecenv* v, uint64_t* out, int64_t cap, int64_t* n);
/* sizeof of the ABI structs as compiled: ut_env_config, ut_buffers,
 * ut_host_outputs, ut_benchmark_report (no device needed). */
int ut_debug_abi_sizes(int64_t out[4]);
/* Measured fp64 issue peak of the device: thread-level DFMA per second from 8
 * independent chains per thread on 8 CTAs of 256 threads per SM (best of 5). */
int ut_debug_fp64_peak(int device, double* dfma_per_s);
/* Cycles thread 0 of each CTA spent in each phase of the particle-set loop,
 * summed over CTAs (12 slots: noise, TMA wait, load+predict, stages, shift,
 * weight sums, exact/ESS, resample, store, estimate, tail). Non-zero only in
 * builds with -DUT_SET_PROFILE (A/B diagnostics). */
int ut_debug_set_profile(int device, uint64_t* out, int reset);
/* Which step-kernel instance the handle launches: *full = 1 for the TMA /
 * register-tile instance (P in {256, 512, 1024}, particle noise on), 0 for the
 * generic one; *np = its compile-time particle capacity. */
int ut_debug_instance(struct ut_vecenv* v, int32_t* full, int32_t* np);
/* derive_key (rng.hpp:30-38) evaluated on the device. */
int ut_debug_derive_key(uint64_t a, uint64_t b, uint64_t c, uint64_t d, int device, uint64_t* out);
#ifdef __cplusplus
}
#endif
#endif
