/* ut_oracle.h -- TEST INFRASTRUCTURE. CPU restatement (plain C) of the
 * reference's batched environment step, used ONLY by tests/, smoke() and
 * bench.py's cpu_baseline leg as the checker. Never linked into the product.
 * Pinned against the reference itself (oracle/_ref, reference sources compiled
 * against the Eigen shim): bit-identical serialized state and batch buffers,
 * tests/test_oracle_vs_ref.py. See oracle/README.md.
 */
#ifndef UT_ORACLE_H_
#define UT_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "ut_env.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct uto_vecenv uto_vecenv;

void uto_config_default(ut_env_config* cfg);
int uto_config_finalize(ut_env_config* cfg);
int uto_create(const ut_env_config* cfg, int64_t n_envs, uint64_t seed, int64_t env_index_offset,
               uto_vecenv** out);
void uto_destroy(uto_vecenv* v);
int uto_reset_all(uto_vecenv* v);
int uto_step(uto_vecenv* v, const int32_t* actions);
int uto_step_policy(uto_vecenv* v, int policy, int n_steps);
int uto_refresh_outputs(uto_vecenv* v);
int uto_copy_outputs(uto_vecenv* v, const ut_host_outputs* dst);
int uto_serialize(uto_vecenv* v, int64_t env, double* blob, size_t cap, size_t* len);
int uto_deserialize(uto_vecenv* v, int64_t env, const double* blob, size_t len);
int uto_stats(uto_vecenv* v, double out[UT_N_STATS]);
/* the running episode's evaluation accumulators of env e: sum of agent-target
 * distances, sum of tracking errors, collided | lost<<1 (test hook) */
int uto_eval_acc(uto_vecenv* v, int64_t e, double out[3]);
const char* uto_last_error(void);

/* primitives exposed for unit tests */
void uto_philox_block(uint64_t key, uint64_t stream, uint64_t block, uint32_t out[4]);
uint64_t uto_derive_key(uint64_t a, uint64_t b, uint64_t c, uint64_t d);
float uto_cr_logf(float x);
float uto_cr_cosf(float x);
float uto_cr_sinf(float x);
/* kind 0 log, 1 cos, 2 sin, 3 sqrt(-2 log) over the 2^24 draw grid (ut_debug.h) */
void uto_cr_grid(int kind, float* out);
/* fills out[0..4n) with the predict noise of one particle set starting at u32
 * stream position `pos` (tracking.cpp:24-37) */
void uto_fill_normals(uint64_t key, uint64_t stream, uint64_t pos, int64_t n, float* out);

#ifdef __cplusplus
}
#endif
#endif
