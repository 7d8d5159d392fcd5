// ut_blob.cuh -- batched Environment::serialize_state / deserialize_state
// (env.cpp:550-659) straight from / into the device state store: one CTA per
// env packs (unpacks) the reference blob layout into (from) a contiguous staging
// buffer, so a checkpoint of many envs is one kernel and one bulk copy.
//
// Blob layout of an env with A agents, T targets, P particles (env.cpp:550-593):
//   [0, 5)                 step, episode target speed, env RNG {pos, have_spare, spare}
//   [5, 5+6A)              agents: x, y, z, heading, speed, rudder
//   [.., +8T)              targets: x, y, z, heading, speed, rudder, countdown, cmd
//   [.., +T)               miss streaks
//   then per agent a:      AgentInfo[a][0..A) x 6 fields, then per target t:
//                          9 track words + px, py, vx, vy, w (P each)
#pragma once
#include "ut_kernels.cuh"

namespace ut {

// record field accessors (as in ut_kernels.cuh)
#define AG(f, a) rec[c.o_agent + (f) * c.sA + (a)]
#define TG(f, t) rec[c.o_target + (f) * c.sT + (t)]
#define INFO(f, k) rec[c.o_info + (f) * c.sA * c.sA + (k)]
#define TRK(f, ti) rec[c.o_track + (f) * c.sA * c.sT + (ti)]

__host__ __device__ inline int64_t blob_len(int A, int T, int P) {
  return 5 + 6 * (int64_t)A + 9 * (int64_t)T + (int64_t)A * (6 * A + (int64_t)T * (9 + 5 * (int64_t)P));
}

struct BlobMap {
  int A, T, P;
  int64_t head, per_agent, per_set;
  __device__ BlobMap(const DevConfig& c) : A(c.A), T(c.T), P(c.P) {
    head = 5 + 6 * (int64_t)A + 9 * (int64_t)T;
    per_set = 9 + 5 * (int64_t)P;
    per_agent = 6 * (int64_t)A + T * per_set;
  }
  __device__ int64_t agent(int a) const { return head + a * per_agent; }
  __device__ int64_t set(int a, int t) const { return agent(a) + 6 * (int64_t)A + t * per_set; }
};

// env (e0 + blockIdx.x, strided) -> out + off[i - e0] (off: device prefix sums)
__global__ void pack_blobs_kernel(DevBatch B, int64_t e0, int64_t n, const int64_t* off, double* out) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t e = e0 + i;
    const DevConfig& c = cfg_of(B, e);
    const Rec rec = rec_of(B, e);
    const BlobMap m(c);
    const int A = c.A, T = c.T, P = c.P;
    double* o = out + off[i];
    for (int k = threadIdx.x; k < 5; k += blockDim.x) o[k] = rec[k];  // R_STEP .. R_ENV_SPARE
    for (int k = threadIdx.x; k < 6 * A; k += blockDim.x) o[5 + k] = AG(k % 6, k / 6);
    for (int k = threadIdx.x; k < 8 * T; k += blockDim.x) o[5 + 6 * A + k] = TG(k % 8, k / 8);
    for (int k = threadIdx.x; k < T; k += blockDim.x) o[5 + 6 * A + 8 * T + k] = rec[c.o_miss + k];
    for (int k = threadIdx.x; k < A * 6 * A; k += blockDim.x) {
      const int a = k / (6 * A), r = k % (6 * A);
      o[m.agent(a) + r] = INFO(r % 6, a * c.sA + r / 6);
    }
    for (int k = threadIdx.x; k < A * T * K_NBLOB; k += blockDim.x) {
      const int s = k / K_NBLOB, fl = k % K_NBLOB, a = s / T, t = s % T;
      o[m.set(a, t) + fl] = TRK(fl, a * c.sT + t);
    }
    const int64_t so = set_off(B, e);
    const double* fields[5] = {B.px, B.py, B.vx, B.vy, B.w};
    for (int s = 0; s < A * T; ++s) {
      double* dst = o + m.set(s / T, s % T) + K_NBLOB;
#pragma unroll
      for (int f = 0; f < 5; ++f) {
        const double* src = fields[f] + (so + s) * (int64_t)P;
        for (int k = threadIdx.x; k < P; k += blockDim.x) dst[f * (int64_t)P + k] = src[k];
      }
    }
  }
}

// The inverse, with the reference's integer conversions (env.cpp:595-659):
// counters through (int), flags through != 0, RNG positions through (uint64_t).
__global__ void unpack_blobs_kernel(DevBatch B, int64_t e0, int64_t n, const int64_t* off, const double* in) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t e = e0 + i;
    const DevConfig& c = cfg_of(B, e);
    const Rec rec = rec_of(B, e);
    const BlobMap m(c);
    const int A = c.A, T = c.T, P = c.P;
    const double* b = in + off[i];
    auto as_int = [](double x) { return (double)(int)x; };
    auto as_flag = [](double x) { return x != 0.0 ? 1.0 : 0.0; };
    if (threadIdx.x == 0) {
      rec[R_STEP] = as_int(b[0]);
      rec[R_EP_SPEED] = b[1];
      rec[R_ENV_POS] = (double)(uint64_t)b[2];
      rec[R_ENV_HAVE_SPARE] = as_flag(b[3]);
      rec[R_ENV_SPARE] = b[4];
    }
    for (int k = threadIdx.x; k < 6 * A; k += blockDim.x) {
      const int fl = k % 6;
      AG(fl, k / 6) = fl == V_RUDDER ? as_int(b[5 + k]) : b[5 + k];
    }
    for (int k = threadIdx.x; k < 8 * T; k += blockDim.x) {
      const int fl = k % 8;
      const double x = b[5 + 6 * A + k];
      TG(fl, k / 8) = (fl == V_RUDDER || fl == V_COUNTDOWN) ? as_int(x) : x;
    }
    for (int k = threadIdx.x; k < T; k += blockDim.x) rec[c.o_miss + k] = as_int(b[5 + 6 * A + 8 * T + k]);
    for (int k = threadIdx.x; k < A * 6 * A; k += blockDim.x) {
      const int a = k / (6 * A), r = k % (6 * A), fl = r % 6;
      const double x = b[m.agent(a) + r];
      INFO(fl, a * c.sA + r / 6) = fl == I_AGE ? as_int(x) : fl == I_VALID ? as_flag(x) : x;
    }
    for (int k = threadIdx.x; k < A * T * K_NBLOB; k += blockDim.x) {
      const int s = k / K_NBLOB, fl = k % K_NBLOB, a = s / T, t = s % T;
      const double x = b[m.set(a, t) + fl];
      TRK(fl, a * c.sT + t) = fl == K_AGE                          ? as_int(x)
                              : (fl == K_EVER || fl == K_HAVE_SPARE) ? as_flag(x)
                              : fl == K_POS                          ? (double)(uint64_t)x
                                                                     : x;
      if (fl == 0) TRK(K_ESSOK, a * c.sT + t) = 0.0;  // injected weights have not been vetted
    }
    const int64_t so = set_off(B, e);
    double* fields[5] = {B.px, B.py, B.vx, B.vy, B.w};
    for (int s = 0; s < A * T; ++s) {
      const double* src = b + m.set(s / T, s % T) + K_NBLOB;
#pragma unroll
      for (int f = 0; f < 5; ++f) {
        double* dst = fields[f] + (so + s) * (int64_t)P;
        for (int k = threadIdx.x; k < P; k += blockDim.x) dst[k] = src[f * (int64_t)P + k];
      }
    }
  }
}

#undef AG
#undef TG
#undef INFO
#undef TRK

}  // namespace ut
