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
//   * bf16 on the 5th-generation tensor cores (policy_tc_kernel below): the three
//     layers of actor+critic as tcgen05.mma with TMEM accumulators -- the
//     throughput path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

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


// ===================================================================== tcgen05
// The bf16 throughput path.  One CTA of 128 threads owns a 128-row tile
// (UMMA M = 128, row r of the tile = TMEM lane r = thread r):
//   L1  D[0:128)   = X[128x32]  . [W1_actor ; W1_critic]^T   (N = 128, K = 32)
//   L2  D[0:64)    = H1a[128x64] . W2_actor^T                 (N = 64,  K = 64)
//       D[64:128)  = H1c[128x64] . W2_critic^T
//   L3  D[128:144) = H2a . W3_actor^T (5 rows, padded to 16)  (N = 16,  K = 64)
//       D[144:160) = H2c . W3_critic^T (1 row, padded)
// Operands are bf16 in shared memory in the UMMA canonical K-major layout
// without swizzle (8-row x 16-byte core matrices; LBO = 128 B between the
// two K halves of a core-matrix pair, SBO = (K/8)*128 B between 8-row
// groups); accumulators are fp32 in TMEM (256 columns allocated).  One
// elected thread issues tcgen05.mma and tcgen05.commit to an mbarrier; every
// thread pulls its row back with tcgen05.ld for the bias + tanh epilogue,
// converts to bf16 and writes the next layer's A operand.  The weights are
// staged once per persistent CTA.
namespace {

constexpr int kTcRows = 128;
constexpr uint32_t kTmemCols = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (n, k) in a K-major no-swizzle canonical [N x K] bf16 tile
__host__ __device__ __forceinline__ uint32_t canon_off(int n, int k, int K) {
  return uint32_t((n >> 3) * ((K >> 3) * 128) + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t umma_desc(const void* tile, int K, int k0) {
  const uint32_t addr = smem_u32(tile) + uint32_t(k0 >> 3) * 128u;  // K slice start
  const uint32_t lbo = 128u, sbo = uint32_t(K >> 3) * 128u;
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // descriptor version 1 (sm_100); base offset 0; layout SWIZZLE_NONE
  return d;
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float tanh_fast(float x) {  // MUFU.TANH: ~2^-11 relative, below bf16's 2^-8
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Row `row` of an activation operand: 16 fp32 values at K offset k0 -> bf16
// into the canonical tile (two 16-byte chunks).
__device__ __forceinline__ void put16(uint8_t* tile, int K, int row, int k0, const float* v) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint4 q;
    q.x = pack_bf16(v[8 * c + 0], v[8 * c + 1]);
    q.y = pack_bf16(v[8 * c + 2], v[8 * c + 3]);
    q.z = pack_bf16(v[8 * c + 4], v[8 * c + 5]);
    q.w = pack_bf16(v[8 * c + 6], v[8 * c + 7]);
    *reinterpret_cast<uint4*>(tile + canon_off(row, k0 + 8 * c, K)) = q;
  }
}

struct TcSmem {  // all tiles 1024-byte aligned
  uint8_t w1[128 * 32 * 2];  // [W1a ; W1c]  (N=128, K=32)
  uint8_t w2a[64 * 64 * 2];
  uint8_t w2c[64 * 64 * 2];
  uint8_t w3a[16 * 64 * 2];
  uint8_t w3c[16 * 64 * 2];
  uint8_t x[kTcRows * 32 * 2];    // layer-1 A operand
  uint8_t ha[kTcRows * 64 * 2];   // actor hidden (A of L2, then of L3)
  uint8_t hc[kTcRows * 64 * 2];   // critic hidden
  float bias[4 * 64 + 2 * 16];
  uint64_t bar;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kTcRows) policy_tc_kernel(PolicyNetBf16 nb, int in_dim, int n_act, PolicyStep s,
                                                            RolloutBufs b) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;

  // one-time: weights (already in canonical layout) + biases, barrier, TMEM
  {
    const uint4* src[5] = {reinterpret_cast<const uint4*>(nb.a1), reinterpret_cast<const uint4*>(nb.a2),
                           reinterpret_cast<const uint4*>(nb.c2), reinterpret_cast<const uint4*>(nb.h3),
                           reinterpret_cast<const uint4*>(nb.hc3)};
    uint4* dst[5] = {reinterpret_cast<uint4*>(S.w1), reinterpret_cast<uint4*>(S.w2a),
                     reinterpret_cast<uint4*>(S.w2c), reinterpret_cast<uint4*>(S.w3a),
                     reinterpret_cast<uint4*>(S.w3c)};
    const int n16[5] = {128 * 32 * 2 / 16, 64 * 64 * 2 / 16, 64 * 64 * 2 / 16, 16 * 64 * 2 / 16, 16 * 64 * 2 / 16};
    for (int m = 0; m < 5; ++m)
      for (int q = tid; q < n16[m]; q += blockDim.x) dst[m][q] = __ldg(src[m] + q);
    for (int q = tid; q < 4 * 64 + 2 * 16; q += blockDim.x) S.bias[q] = __ldg(nb.bias + q);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t tmem = S.tmem_base;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  uint32_t phase = 0;

  const int64_t n_tiles = (s.R + kTcRows - 1) / kTcRows;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r = tile * kTcRows + tid;
    const bool live = r < s.R;
    // ---- layer-1 operand: the TeamLayout row (+ buffer writes)
    {
      float x[32];
      if (live) {
        fill_row(s, b, r, in_dim, n_act, x, !s.bootstrap);
      }
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (!live || k >= in_dim) x[k] = 0.0f;
      put16(S.x, 32, tid, 0, x);
      put16(S.x, 32, tid, 16, x + 16);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 128);
      for (int k = 0; k < 32; k += 16) umma_bf16(tmem + 0, umma_desc(S.x, 32, k), umma_desc(S.w1, 32, k), id, k > 0);
      umma_commit(&S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 1: bias + tanh -> bf16 hidden rows
    for (int c = 0; c < 128; c += 16) {
      float v[16];
      tmem_ld16(tmem + lane_base + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = tanh_fast(v[i] + S.bias[c + i]);
      if (c < 64) put16(S.ha, 64, tid, c, v);
      else put16(S.hc, 64, tid, c - 64, v);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 64);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(S.ha, 64, k), umma_desc(S.w2a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 64, umma_desc(S.hc, 64, k), umma_desc(S.w2c, 64, k), id, k > 0);
      umma_commit(&S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 2
    for (int c = 0; c < 128; c += 16) {
      float v[16];
      tmem_ld16(tmem + lane_base + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = tanh_fast(v[i] + S.bias[128 + c + i]);
      if (c < 64) put16(S.ha, 64, tid, c, v);
      else put16(S.hc, 64, tid, c - 64, v);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 16);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 128, umma_desc(S.ha, 64, k), umma_desc(S.w3a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 144, umma_desc(S.hc, 64, k), umma_desc(S.w3c, 64, k), id, k > 0);
      umma_commit(&S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 3: heads, sampling, buffer writes
    float lg[16], vv[16];
    tmem_ld16(tmem + lane_base + 128u, lg);
    tmem_ld16(tmem + lane_base + 144u, vv);
    tc_fence_before();
    if (live) {
      const float value = vv[0] + S.bias[256 + 16];
      if (s.bootstrap) {
        b.last_value[r] = value;
      } else {
        float logits[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) logits[j] = lg[j] + S.bias[256 + j];
        sample_and_record(s, b, r, logits, n_act, value);
      }
    }
    __syncthreads();  // TMEM columns and operand tiles are reused by the next tile
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

// fp32 parameters -> canonical bf16 operand images + bias block.
__global__ void pack_bf16_kernel(PolicyNet n, uint16_t* img, float* bias) {
  const int in = n.in_dim, NA = n.n_act;
  uint16_t* a1 = img;
  uint16_t* a2 = a1 + 128 * 32;
  uint16_t* c2 = a2 + 64 * 64;
  uint16_t* h3 = c2 + 64 * 64;
  uint16_t* hc3 = h3 + 16 * 64;
  auto bf = [](float v) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    return *reinterpret_cast<const uint16_t*>(&h);
  };
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 128 * 32; q += gridDim.x * blockDim.x) {
    const int row = q / 32, k = q % 32;
    float v = 0.0f;
    if (k < in) v = row < 64 ? n.w1[row * in + k] : n.cw1[(row - 64) * in + k];
    a1[canon_off(row, k, 32) / 2] = bf(v);
  }
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 64 * 64; q += gridDim.x * blockDim.x) {
    const int row = q / 64, k = q % 64;
    a2[canon_off(row, k, 64) / 2] = bf(n.w2[row * 64 + k]);
    c2[canon_off(row, k, 64) / 2] = bf(n.cw2[row * 64 + k]);
  }
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 16 * 64; q += gridDim.x * blockDim.x) {
    const int row = q / 64, k = q % 64;
    h3[canon_off(row, k, 64) / 2] = bf(row < NA ? n.w3[row * 64 + k] : 0.0f);
    hc3[canon_off(row, k, 64) / 2] = bf(row == 0 ? n.cw3[k] : 0.0f);
  }
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 64; q += gridDim.x * blockDim.x) {
    bias[q] = n.b1[q];
    bias[64 + q] = n.cb1[q];
    bias[128 + q] = n.b2[q];
    bias[192 + q] = n.cb2[q];
    if (q < 16) {
      bias[256 + q] = q < NA ? n.b3[q] : 0.0f;
      bias[272 + q] = q == 0 ? n.cb3[0] : 0.0f;
    }
  }
}

}  // namespace

bool rollout_policy_bf16_supported(int in_dim, int n_act, int width) {
  return in_dim <= 32 && n_act <= 16 && width == 64;
}

void rollout_pack_bf16(const PolicyNet& net, uint16_t* images, float* bias, cudaStream_t st) {
  pack_bf16_kernel<<<16, 256, 0, st>>>(net, images, bias);
  ++g_launches;
}

void rollout_policy_bf16(const PolicyNet& net, const PolicyNetBf16& nb, const PolicyStep& s, const RolloutBufs& b,
                         cudaStream_t st) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t sm = sizeof(TcSmem) + 1024;  // + alignment slack
  cudaFuncSetAttribute(policy_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  const int64_t tiles = (s.R + kTcRows - 1) / kTcRows;
  const int64_t grid = std::min<int64_t>(tiles, int64_t(sms) * 2);  // two CTAs (2 x 256 TMEM columns) per SM
  policy_tc_kernel<<<unsigned(grid), kTcRows, sm, st>>>(nb, net.in_dim, net.n_act, s, b);
  ++g_launches;
}

void rollout_gae(const RolloutBufs& b, int T, int64_t R, float gamma, float lambda, cudaStream_t st) {
  gae_kernel<<<unsigned((R + 255) / 256), 256, 0, st>>>(b, T, R, gamma, lambda);
  ++g_launches;
}

}  // namespace marl_b200
