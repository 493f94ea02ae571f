// Row-level helpers of the rollout policies (rollout.cu, rnn.cu): TeamLayout
// rows from the env's observation view and masked sampling with the
// Collector's per-row key.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {

// masked_log_probs + sample_masked (actor_critic.hpp:218-262) in double over
// one row's float logits with the row's key fold_in(act_key, (seq_base+t)*R
// + r) (ppo.cpp:249-259).  Shared by both policy paths.
__device__ inline void sample_row(const PolicyStep& s, int64_t r, const float* logits, const uint8_t* legal, int n_act,
                           int* action, float* logp) {
  double mx = -INFINITY;
  for (int i = 0; i < n_act; ++i)
    if (legal[i]) mx = fmax(mx, double(logits[i]));
  double denom = 0.0;
  for (int i = 0; i < n_act; ++i)
    if (legal[i]) denom += exp(double(logits[i]) - mx);
  const double log_denom = log(denom);
  const Key ak{s.act_key[0], s.act_key[1], s.act_key[2], s.act_key[3]};
  const Key kk = fold_in(ak, uint64_t(s.step_index) * uint64_t(s.R_global) + uint64_t(s.row0 + r));
  const double u = uniform_at(kk, 0, 0.0, 1.0);  // prng::uniform1
  double cum = 0.0, lp_pick = 0.0;
  int pick = -1;
  for (int i = 0; i < n_act; ++i) {
    if (!legal[i]) continue;
    const double lp = double(logits[i]) - mx - log_denom;
    pick = i;
    lp_pick = lp;
    cum += exp(lp);
    if (u < cum) break;
  }
  *action = pick;
  *logp = float(lp_pick);
}

// The bf16 path's sampler: the same masked softmax + CDF walk with the same
// per-row key and uniform draw, in float (the bf16 logits already differ
// from the reference's by far more than float rounding).
__device__ __forceinline__ double row_uniform(const PolicyStep& s, int64_t r) {
  const Key ak{s.act_key[0], s.act_key[1], s.act_key[2], s.act_key[3]};
  const Key kk = fold_in(ak, uint64_t(s.step_index) * uint64_t(s.R_global) + uint64_t(s.row0 + r));
  return uniform_at(kk, 0, 0.0, 1.0);  // prng::uniform1
}

__device__ inline void sample_row_f32(double u, const float* logits, const uint8_t* legal, int n_act, int* action,
                               float* logp) {
  float mx = -INFINITY;
  for (int i = 0; i < n_act; ++i)
    if (legal[i]) mx = fmaxf(mx, logits[i]);
  float p[16], denom = 0.0f;
  for (int i = 0; i < n_act; ++i) {
    p[i] = legal[i] ? expf(logits[i] - mx) : 0.0f;
    denom += p[i];
  }
  const float log_denom = logf(denom), inv = 1.0f / denom;
  double cum = 0.0;
  int pick = -1;
  for (int i = 0; i < n_act; ++i) {
    if (!legal[i]) continue;
    pick = i;
    cum += double(p[i] * inv);
    if (u < cum) break;
  }
  *action = pick;
  *logp = logits[pick] - mx - log_denom;
}

// sample_row_f32 with the loops bounded by a compile-time NMAX (>= n_act):
// fully unrolled, the probabilities stay in registers.
// sample_row_n for heads of up to 64 actions without the per-action
// probability array (the exponentials are recomputed: same values, same order)
__device__ __forceinline__ void sample_row_wide(double u, const float* logits, const uint8_t* legal, int n_act,
                                                int* action, float* logp) {
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 64; ++i)
    if (i < n_act && legal[i]) mx = fmaxf(mx, logits[i]);
  float denom = 0.0f;
#pragma unroll
  for (int i = 0; i < 64; ++i) denom += (i < n_act && legal[i]) ? expf(logits[i] - mx) : 0.0f;
  const float log_denom = logf(denom), inv = 1.0f / denom;
  double cum = 0.0;
  int pick = -1;
  bool done = false;
  float lpick = 0.0f;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    if (!(i < n_act && legal[i]) || done) continue;
    pick = i;
    lpick = logits[i];
    cum += double(expf(logits[i] - mx) * inv);
    done = u < cum;
  }
  *action = pick;
  *logp = lpick - mx - log_denom;
}

template <int NMAX>
__device__ __forceinline__ void sample_row_n(double u, const float* logits, const uint8_t* legal, int n_act, int* action,
                                             float* logp) {
  bool lg[NMAX];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    lg[i] = i < n_act && legal[i];
    if (lg[i]) mx = fmaxf(mx, logits[i]);
  }
  float p[NMAX], denom = 0.0f;
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    p[i] = lg[i] ? expf(logits[i] - mx) : 0.0f;
    denom += p[i];
  }
  const float log_denom = logf(denom), inv = 1.0f / denom;
  double cum = 0.0;
  int pick = -1;
  bool done = false;
  float lpick = 0.0f;
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    if (!lg[i] || done) continue;
    pick = i;
    lpick = logits[i];
    cum += double(p[i] * inv);
    done = u < cum;
  }
  *action = pick;
  *logp = lpick - mx - log_denom;
}

// The fp32 path's per-row tail: sample, then the buffer writes.
__device__ inline void sample_and_record(const PolicyStep& s, const RolloutBufs& b, int64_t r, const float* logits,
                                  int n_act, float value) {
  const size_t slot = size_t(s.t) * size_t(s.R) + size_t(r);
  int pick;
  float lp;
  sample_row(s, r, logits, b.legal + slot * n_act, n_act, &pick, &lp);
  b.actions[slot] = pick;
  b.logp[slot] = lp;
  b.value[slot] = value;
}

// write_input / write_legal / agent_active of row r for step t (team.cpp:27-42,
// ppo.cpp:333-360); x receives the in_dim floats.
__device__ inline void fill_row(const PolicyStep& s, const RolloutBufs& b, int64_t r, int in_dim, int n_act, float* x,
                         bool write_buffers) {
  const int64_t e = r / s.A;
  const int a = int(r - e * s.A);
  const float* o = s.env_obs + size_t(r) * s.D;  // [E][A][D] == [R][D]
  for (int k = 0; k < s.D; ++k) x[k] = o[k];
  for (int k = s.D; k < in_dim; ++k) x[k] = 0.0f;
  if (s.A > 1) x[s.D + a] = 1.0f;  // agent one-hot (team.cpp:32)
  if (!write_buffers) return;
  const size_t slot = size_t(s.t) * size_t(s.R) + size_t(r);
  float* bo = b.obs + slot * in_dim;
  for (int k = 0; k < in_dim; ++k) bo[k] = x[k];
  b.resets[slot] = s.prev_finished ? s.prev_finished[e] : uint8_t(1);
  uint8_t* lg = b.legal + slot * n_act;
  if (!s.legal_ready) {  // all-legal envs (env.hpp:71-73), padded to n_act with 0 (team.cpp:40)
    const int na = s.agent_actions[a];
    for (int q = 0; q < n_act; ++q) lg[q] = q < na ? 1 : 0;
  }
  // agent_active: SMAX units are active while alive (smax.cpp:213-216), and an
  // alive unit always has its move actions legal; the others are always active.
  b.active[slot] = (s.family == 1) ? (lg[0] ? 1.0f : 0.0f) : 1.0f;
}

}  // namespace marl_b200
