// IPPO rollout collection (BASELINE configs[4]):
// the reference's Collector::collect (proj/core/src/algo/ppo.cpp:206-323) as
// device kernels around the fused env step.  Per rollout step t:
//
//   policy kernel : TeamLayout::write_input (team.cpp:27-33) of every row
//                   straight from the env's observation view, actor and
//                   critic ff_forward (actor_critic.hpp:49-52), masked
//                   sampling with the per-row key fold_in(act_key,
//                   (seq_base+t)*R + r) (ppo.cpp:249-259, sample_masked
//                   actor_critic.hpp:218-262), and every rollout-buffer
//                   write of the step (obs, resets, legal, active, action,
//                   logp, value).  The action slice of the buffer IS the env
//                   step's action input.
//   env step      : the family's fused step kernel (mpe/smax/overcooked.cu).
//   record kernel : rewards (+ annealed shaped reward) and dones of step t
//                   (ppo.cpp:262-276).
// After the window: the policy kernel in bootstrap mode (critic only,
// ppo.cpp:285-299) and a reverse-scan GAE kernel (actor_critic.hpp:282-299).
//
// Two policy paths:
//   * fp32 (this file, policy_fp32_kernel): one thread per row, weights in
//     shared memory, every dot product accumulated in the reference's order
//     with -fmad=false -- the parity path.
//   * bf16 on the 5th-generation tensor cores (rollout_tc.cu): the three
//     layers of actor+critic as tcgen05.mma with TMEM accumulators -- the
//     throughput path.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {

namespace {

constexpr int kMaxIn = 1024;    // actor input width handled by the fp32 path
constexpr int kMaxWidth = 64;   // torso width handled by the fp32 path
constexpr int kMaxAct = 64;

__device__ __forceinline__ float activate(float v, int relu) {  // act_inplace, nn.hpp:136-138
  return relu ? (v > 0.0f ? v : 0.0f) : tanhf(v);
}

// dense_forward (nn.hpp:108-115) for one row: y = x W^T, then + b, then act.
// matmul_nt accumulates acc += x[i] * w[o][i] in float, i ascending (nn.hpp:42-54).
__device__ __forceinline__ float dot_ref(const float* __restrict__ x, const float* __restrict__ w, int n) {
  float acc = 0.0f;
  for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, __fmul_rn(x[i], w[i]));
  return acc;
}

struct SmemNet {  // the net staged in shared memory, same packing as PolicyNet
  const float *w1, *b1, *w2, *b2, *w3, *b3, *cw1, *cb1, *cw2, *cb2, *cw3, *cb3;
};

__host__ __device__ inline int net_floats(int in, int width, int n_act) {
  return (width * in + width + width * width + width + n_act * width + n_act) +
         (width * in + width + width * width + width + width + 1);
}

}  // namespace

// The per-row tail shared by both policy paths: masked_log_probs +
// sample_masked (actor_critic.hpp:218-262) in double over the row's float
// logits, then the buffer writes.  Returns the sampled action.
__device__ int sample_and_record(const PolicyStep& s, const RolloutBufs& b, int64_t r, const float* logits,
                                 int n_act, float value) {
  const int64_t R = s.R;
  const size_t slot = size_t(s.t) * size_t(R) + size_t(r);
  const uint8_t* legal = b.legal + slot * n_act;
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
  b.actions[slot] = pick;
  b.logp[slot] = float(lp_pick);
  b.value[slot] = value;
  return pick;
}

// write_input / write_legal / agent_active of row r for step t (team.cpp:27-42,
// ppo.cpp:333-360); x receives the in_dim floats.
__device__ void fill_row(const PolicyStep& s, const RolloutBufs& b, int64_t r, int in_dim, int n_act, float* x,
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

namespace {

__global__ void __launch_bounds__(128) policy_fp32_kernel(PolicyNet net, PolicyStep s, RolloutBufs b, int staged) {
  extern __shared__ __align__(16) float smem[];
  const int in = net.in_dim, W = net.width, NA = net.n_act;
  // stage the packed actor+critic parameters (one contiguous device block)
  // when they fit in shared memory; wide inputs (Overcooked's 543) read them
  // through L1 instead
  const int total = net_floats(in, W, NA);
  if (staged) {
    for (int q = threadIdx.x; q < total; q += blockDim.x) smem[q] = __ldg(net.w1 + q);
    __syncthreads();
  }
  SmemNet m;
  m.w1 = staged ? smem : net.w1;
  m.b1 = m.w1 + W * in;
  m.w2 = m.b1 + W;
  m.b2 = m.w2 + W * W;
  m.w3 = m.b2 + W;
  m.b3 = m.w3 + NA * W;
  m.cw1 = m.b3 + NA;
  m.cb1 = m.cw1 + W * in;
  m.cw2 = m.cb1 + W;
  m.cb2 = m.cw2 + W * W;
  m.cw3 = m.cb2 + W;
  m.cb3 = m.cw3 + W;

  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.R) return;
  float x[kMaxIn], h1[kMaxWidth], h2[kMaxWidth];
  fill_row(s, b, r, in, NA, x, !s.bootstrap);
  // critic (the value head of ff_forward on the same row: IPPO critic_in == x)
  for (int o = 0; o < W; ++o) h1[o] = activate(__fadd_rn(dot_ref(x, m.cw1 + o * in, in), m.cb1[o]), net.relu);
  for (int o = 0; o < W; ++o) h2[o] = activate(__fadd_rn(dot_ref(h1, m.cw2 + o * W, W), m.cb2[o]), net.relu);
  const float value = __fadd_rn(dot_ref(h2, m.cw3, W), m.cb3[0]);
  if (s.bootstrap) {
    b.last_value[r] = value;
    return;
  }
  // actor
  for (int o = 0; o < W; ++o) h1[o] = activate(__fadd_rn(dot_ref(x, m.w1 + o * in, in), m.b1[o]), net.relu);
  for (int o = 0; o < W; ++o) h2[o] = activate(__fadd_rn(dot_ref(h1, m.w2 + o * W, W), m.b2[o]), net.relu);
  float logits[kMaxAct];
  for (int j = 0; j < NA; ++j) logits[j] = __fadd_rn(dot_ref(h2, m.w3 + j * W, W), m.b3[j]);
  sample_and_record(s, b, r, logits, NA, value);
}

__global__ void record_kernel(RolloutBufs b, int t, int64_t R, int A, const double* __restrict__ rew,
                              const double* __restrict__ infos, int n_info, int shaped_idx, double shaping,
                              const uint8_t* __restrict__ fin) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double v = rew[r];  // [E][A] == [R]
  if (shaping > 0.0 && shaped_idx >= 0) v += shaping * infos[r * n_info + shaped_idx];
  const size_t slot = size_t(t) * size_t(R) + size_t(r);
  b.rewards[slot] = float(v);
  b.dones[slot] = fin[r / A];
}

// compute_gae (actor_critic.hpp:282-299), one row per thread, float with the
// reference's evaluation order (-fmad=false).
__global__ void gae_kernel(RolloutBufs b, int T, int64_t R, float gamma, float lambda) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  float next_adv = 0.0f, next_value = b.last_value[r];
  for (int t = T - 1; t >= 0; --t) {
    const size_t i = size_t(t) * size_t(R) + size_t(r);
    const float not_done = b.dones[i] ? 0.0f : 1.0f;
    const float v = b.value[i];
    const float delta = b.rewards[i] + gamma * next_value * not_done - v;
    next_adv = delta + gamma * lambda * not_done * next_adv;
    b.adv[i] = next_adv;
    b.vtarg[i] = next_adv + v;
    next_value = v;
  }
}

}  // namespace

void rollout_policy_fp32(const PolicyNet& net, const PolicyStep& s, const RolloutBufs& b, cudaStream_t st) {
  size_t sm = size_t(net_floats(net.in_dim, net.width, net.n_act)) * sizeof(float);
  const int staged = sm <= size_t(160) * 1024;
  if (!staged) sm = 0;
  cudaFuncSetAttribute(policy_fp32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  policy_fp32_kernel<<<unsigned((s.R + 127) / 128), 128, sm, st>>>(net, s, b, staged);
  ++g_launches;
}

void rollout_record(const RolloutBufs& b, int t, int64_t R, int A, const double* env_rewards, const double* env_infos,
                    int n_info, int shaped_idx, double shaping, const uint8_t* env_finished, cudaStream_t st) {
  record_kernel<<<unsigned((R + 255) / 256), 256, 0, st>>>(b, t, R, A, env_rewards, env_infos, n_info, shaped_idx,
                                                           shaping, env_finished);
  ++g_launches;
}

bool rollout_policy_bf16_supported(int in_dim, int n_act, int width) { return false; }
void rollout_policy_bf16(const PolicyNet&, const PolicyNetBf16&, const PolicyStep&, const RolloutBufs&, cudaStream_t) {}
void rollout_pack_bf16(const PolicyNet&, uint16_t*, float*, cudaStream_t) {}

void rollout_gae(const RolloutBufs& b, int T, int64_t R, float gamma, float lambda, cudaStream_t st) {
  gae_kernel<<<unsigned((R + 255) / 256), 256, 0, st>>>(b, T, R, gamma, lambda);
  ++g_launches;
}

}  // namespace marl_b200
