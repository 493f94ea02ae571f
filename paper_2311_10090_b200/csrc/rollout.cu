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
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "engine.h"
#include "tc.cuh"
#include "policy_rows.cuh"

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

__host__ __device__ inline int net_floats(int in, int cin, int width, int n_act) {
  return (width * in + width + width * width + width + n_act * width + n_act) +
         (width * cin + width + width * width + width + width + 1);
}

}  // namespace

namespace {

__global__ void __launch_bounds__(128) policy_fp32_kernel(PolicyNet net, PolicyStep s, RolloutBufs b, int staged) {
  extern __shared__ __align__(16) float smem[];
  const int in = net.in_dim, CI = net.critic_in, W = net.width, NA = net.n_act;
  // stage the packed actor+critic parameters (one contiguous device block)
  // when they fit in shared memory; wide inputs (Overcooked's 543) read them
  // through L1 instead
  const int total = net_floats(in, CI, W, NA);
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
  m.cb1 = m.cw1 + W * CI;
  m.cw2 = m.cb1 + W;
  m.cb2 = m.cw2 + W * W;
  m.cw3 = m.cb2 + W;
  m.cb3 = m.cw3 + W;

  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.R) return;
  float x[kMaxIn], h1[kMaxWidth], h2[kMaxWidth];
  fill_row(s, b, r, in, NA, x, !s.bootstrap);
  // critic: IPPO reads the same row (critic_in == x); MAPPO reads the env's
  // world_state (ppo.cpp:341-346), kept in the buffer's critic_in rows
  const float* xc = x;
  if (s.ws) {
    xc = s.ws + size_t(r / s.A) * CI;
    if (!s.bootstrap) {
      float* bc = b.critic_in + (size_t(s.t) * size_t(s.R) + size_t(r)) * CI;
      for (int k = 0; k < CI; ++k) bc[k] = xc[k];
    }
  }
  for (int o = 0; o < W; ++o) h1[o] = activate(__fadd_rn(dot_ref(xc, m.cw1 + o * CI, CI), m.cb1[o]), net.relu);
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
  size_t sm = size_t(net_floats(net.in_dim, net.critic_in, net.width, net.n_act)) * sizeof(float);
  const int staged = sm <= size_t(160) * 1024;
  if (!staged) sm = 0;
  smem_optin(policy_fp32_kernel);
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
constexpr uint32_t kTmemCols = 128;  // L1 uses 128 columns; L2 and L3 reuse them
constexpr int kSplit = 2;            // threads per row (warps w, w+4, ... share a TMEM lane quarter)

// Shared-memory carve-up of the tcgen05 policy kernel, sized from the actual
// row widths (offsets in bytes from a 1024-aligned base).
struct TcLayout {
  uint32_t w1, w2a, w2c, w3a, w3c, x, ha, hc, obs_in[2], obs_out, legal, resets, active, act, logp, value, u, bias,
      bar, bar_in[2], tmem_slot, total, xc, wc1;
  int kx;       // K of layer 1: round16(in_dim)
  int kc;       // MAPPO: K of the critic's layer 1, round16(critic_in) (its own X tile and W1 image); 0: IPPO
  int nbuf;     // staged observation tiles: 2 (next tile prefetched), 1 (prefetched after the row build), 0 (rows read from L2)
  int has_out;  // the buffer's input rows leave as one staged bulk store (else a coalesced cooperative store)
};
constexpr uint32_t kTcSmemMax = 232448;  // 227 KB opt-in per CTA
constexpr int kTcMaxKx = 192;

__host__ __device__ inline uint32_t up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// K of layer 1: 32 for small rows, round16 up to kTcMaxKx, beyond that (the
// wide-row kernel, K-chunked) round64 -- the W1 image is then chunk-major.
__host__ __device__ inline int tc_kx(int in_dim) {
  return in_dim <= 32 ? 32 : in_dim <= 192 ? (in_dim + 15) / 16 * 16 : (in_dim + 63) / 64 * 64;
}

// mode 3: two staged tiles + staged buffer rows; 2: two tiles; 1: one tile; 0: none
__host__ __device__ inline int tc_kc(int critic_in) { return critic_in > 0 ? (critic_in + 15) / 16 * 16 : 0; }

__host__ __device__ inline TcLayout tc_layout_mode(int D, int in_dim, int n_act, int mode, int critic_in = 0) {
  TcLayout L{};
  L.kx = tc_kx(in_dim);
  L.kc = tc_kc(critic_in);
  L.nbuf = mode >= 2 ? 2 : mode;
  L.has_out = mode == 3;
  uint32_t o = 0;
  auto take = [&o](uint32_t bytes, uint32_t align) {
    o = up(o, align);
    const uint32_t at = o;
    o += bytes;
    return at;
  };
  L.w1 = take(128 * L.kx * 2, 128);
  L.w2a = take(64 * 64 * 2, 128);
  L.w2c = take(64 * 64 * 2, 128);
  L.w3a = take(16 * 64 * 2, 128);
  L.w3c = take(16 * 64 * 2, 128);
  L.x = take(kTcRows * L.kx * 2, 128);
  L.ha = take(kTcRows * 64 * 2, 128);
  L.hc = take(kTcRows * 64 * 2, 128);
  L.xc = L.kc ? take(uint32_t(kTcRows * L.kc * 2), 128) : 0;
  L.wc1 = L.kc ? take(uint32_t(64 * L.kc * 2), 128) : 0;
  L.obs_in[0] = L.nbuf >= 1 ? take(uint32_t(kTcRows * D * 4), 16) : 0;
  L.obs_in[1] = L.nbuf >= 2 ? take(uint32_t(kTcRows * D * 4), 16) : L.obs_in[0];
  L.obs_out = L.has_out ? take(uint32_t(kTcRows * in_dim * 4), 16) : 0;
  L.legal = take(uint32_t(kTcRows * n_act), 16);
  L.resets = take(kTcRows, 16);
  L.active = take(kTcRows * 4, 16);
  L.act = take(kTcRows * 4, 16);
  L.logp = take(kTcRows * 4, 16);
  L.value = take(kTcRows * 4, 16);
  L.u = take(kTcRows * 8, 16);
  L.bias = take((4 * 64 + 2 * 16) * 4, 16);
  L.bar = take(8, 8);
  L.bar_in[0] = take(8, 8);
  L.bar_in[1] = take(8, 8);
  L.tmem_slot = take(4, 4);
  L.total = up(o, 128);
  return L;
}

__host__ __device__ inline TcLayout tc_layout(int D, int in_dim, int n_act, int critic_in = 0) {
  for (int mode = 3; mode > 0; --mode) {
    const TcLayout L = tc_layout_mode(D, in_dim, n_act, mode, critic_in);
    if (L.total <= kTcSmemMax) return L;
  }
  return tc_layout_mode(D, in_dim, n_act, 0, critic_in);
}

// Store a staged tile: one TMA bulk store when it qualifies, else a
// cooperative copy.  Every thread calls it after fence + barrier.
__device__ __forceinline__ void tile_put(void* g, const void* sm, size_t bytes) {
  if (bulk_ok(g, sm, bytes)) {
    if (threadIdx.x == 0) bulk_store_s2g(g, sm, uint32_t(bytes));
  } else {
    const uint8_t* src = static_cast<const uint8_t*>(sm);
    uint8_t* dst = static_cast<uint8_t*>(g);
    for (size_t q = threadIdx.x; q < bytes; q += blockDim.x) dst[q] = src[q];
  }
}

// TMA bulk load global -> shared completing on an mbarrier (expect-tx).
__device__ __forceinline__ void bulk_load_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Issue (thread 0) or perform (everyone, synchronously) the load of a tile's
// env observation rows; returns whether a bulk load is in flight.
__device__ __forceinline__ bool tile_obs_load(const PolicyStep& s, int64_t tile, float* dst, uint64_t* bar) {
  const int64_t r0 = tile * kTcRows;
  const int rows = int(min64(kTcRows, s.R - r0));
  const float* g = s.env_obs + size_t(r0) * s.D;
  const size_t bytes = size_t(rows) * s.D * 4;
  if (((reinterpret_cast<uintptr_t>(g) | bytes) & 15) == 0) {
    if (threadIdx.x == 0) bulk_load_g2s(dst, g, uint32_t(bytes), bar);
    return true;
  }
  for (size_t q = threadIdx.x; q < bytes / 4; q += blockDim.x) dst[q] = __ldg(g + q);
  return false;
}

// KXT = 32: the small-input instance (K, staging mode 3 compile-time); 0: any width.
// SD / SA / SN > 0: the observation width, agent count and action count folded
// to compile-time constants (MPE simple_spread: 18 / 3 / 5) -- the row build,
// legal rows and sampling unroll into registers; 0: read from the step.
// CENT (generic instance only): MAPPO -- the critic's layer 1 reads the env's
// world_state row (s.ws, critic_in wide) from its own X tile and W1 image.
template <int KXT, int SD = 0, int SA = 0, int SN = 0, bool CENT = false>
__global__ void __launch_bounds__(kSplit * kTcRows) policy_tc_kernel(PolicyNetBf16 nb, int in_dim_rt, int n_act_rt,
                                                                     PolicyStep s, RolloutBufs b, int critic_in) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int D = SD ? SD : s.D, AA = SA ? SA : s.A, n_act = SN ? SN : n_act_rt;
  const int in_dim = SD ? SD + (SA > 1 ? SA : 0) : in_dim_rt;
  const TcLayout L = KXT ? tc_layout_mode(D, in_dim, n_act, 3) : tc_layout(D, in_dim, n_act, CENT ? critic_in : 0);
  const int KC = CENT ? L.kc : 0;
  uint8_t* sxc = smem_raw + L.xc;
  uint8_t* wc1 = smem_raw + L.wc1;
  const int KX = KXT ? KXT : L.kx;
  const int NBUF = KXT ? 2 : L.nbuf;
  const bool HAS_OUT = KXT ? true : bool(L.has_out);
  uint8_t* base = smem_raw;
  uint8_t *w1 = base + L.w1, *w2a = base + L.w2a, *w2c = base + L.w2c, *w3a = base + L.w3a, *w3c = base + L.w3c;
  uint8_t *sx = base + L.x, *ha = base + L.ha, *hc = base + L.hc;
  float* obs_in[2] = {reinterpret_cast<float*>(base + L.obs_in[0]), reinterpret_cast<float*>(base + L.obs_in[1])};
  float* obs_out = reinterpret_cast<float*>(base + L.obs_out);
  uint8_t* s_legal = base + L.legal;
  uint8_t* s_resets = base + L.resets;
  float* s_active = reinterpret_cast<float*>(base + L.active);
  int32_t* s_act = reinterpret_cast<int32_t*>(base + L.act);
  float* s_logp = reinterpret_cast<float*>(base + L.logp);
  float* s_value = reinterpret_cast<float*>(base + L.value);
  float* s_bias = reinterpret_cast<float*>(base + L.bias);
  double* s_u = reinterpret_cast<double*>(base + L.u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bar);
  uint64_t* bar_in[2] = {reinterpret_cast<uint64_t*>(base + L.bar_in[0]), reinterpret_cast<uint64_t*>(base + L.bar_in[1])};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L.tmem_slot);
  // kSplit threads per row: part q (warps 4q..4q+3) owns accumulator columns
  // [128q/kSplit, 128(q+1)/kSplit) of every layer (actor 0-63, critic
  // 64-127) and K columns [32q/kSplit, ...) of the input row; part 0 samples,
  // part 1 writes the value.
  // Warps w, w+4, ... read the same TMEM lane quarter.
  const int tid = threadIdx.x & (kTcRows - 1), part = threadIdx.x >> 7, warp = threadIdx.x >> 5;
  const int64_t n_tiles = (s.R + kTcRows - 1) / kTcRows;

  // one-time: barriers, TMEM, weights (already in canonical layout) + biases,
  // and the first tile's observation rows in flight
  if (threadIdx.x == 0) {
    for (uint64_t* m : {bar, bar_in[0], bar_in[1]})
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  {
    const uint4* src[5] = {reinterpret_cast<const uint4*>(nb.a1), reinterpret_cast<const uint4*>(nb.a2),
                           reinterpret_cast<const uint4*>(nb.c2), reinterpret_cast<const uint4*>(nb.h3),
                           reinterpret_cast<const uint4*>(nb.hc3)};
    uint4* dst[5] = {reinterpret_cast<uint4*>(w1), reinterpret_cast<uint4*>(w2a), reinterpret_cast<uint4*>(w2c),
                     reinterpret_cast<uint4*>(w3a), reinterpret_cast<uint4*>(w3c)};
    const int n16[5] = {128 * KX * 2 / 16, 64 * 64 * 2 / 16, 64 * 64 * 2 / 16, 16 * 64 * 2 / 16, 16 * 64 * 2 / 16};
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      uint4 v[8];
      for (int q0 = 0; q0 < n16[m]; q0 += 8 * int(blockDim.x)) {  // 8 loads in flight per thread
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int q = q0 + j * int(blockDim.x) + int(threadIdx.x);
          if (q < n16[m]) v[j] = __ldg(src[m] + q);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int q = q0 + j * int(blockDim.x) + int(threadIdx.x);
          if (q < n16[m]) dst[m][q] = v[j];
        }
      }
    }
    for (int q = threadIdx.x; q < 4 * 64 + 2 * 16; q += blockDim.x) s_bias[q] = __ldg(nb.bias + q);
    if (CENT)
      for (int q = threadIdx.x; q < 64 * KC * 2 / 16; q += blockDim.x)
        reinterpret_cast<uint4*>(wc1)[q] = __ldg(reinterpret_cast<const uint4*>(nb.c1) + q);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
  const bool act_mode = !s.bootstrap;
  uint32_t phase = 0, in_phase[2] = {0, 0};
  bool in_flight[2] = {false, false};
  int cur = 0;
  if (NBUF > 0 && int64_t(blockIdx.x) < n_tiles) in_flight[0] = tile_obs_load(s, blockIdx.x, obs_in[0], bar_in[0]);

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r0 = tile * kTcRows, r = r0 + tid;
    const int rows = int(min64(kTcRows, s.R - r0));
    const bool live = tid < rows;
    const size_t slot0 = size_t(s.t) * size_t(s.R) + size_t(r0);
    // this tile's observation rows have landed; the previous tile's bulk
    // stores have read the staging tiles
    if (in_flight[cur]) {
      mbar_wait(bar_in[cur], in_phase[cur]);
      in_phase[cur] ^= 1;
    }
    if (threadIdx.x == 0) bulk_wait_read<0>();
    __syncthreads();
    // prefetch the next tile's rows into the other buffer (its last reader,
    // the previous tile's row build, finished before the barrier above)
    const int64_t next = tile + gridDim.x;
    if (NBUF == 2)
      in_flight[cur ^ 1] = next < n_tiles ? tile_obs_load(s, next, obs_in[cur ^ 1], bar_in[cur ^ 1]) : false;
    // the tile's env observation rows: staged, or read through L2
    const float* tile_obs = NBUF > 0 ? obs_in[cur] : s.env_obs + size_t(r0) * size_t(D);
    // ---- write_input / write_legal / agent_active (team.cpp:27-42): part q
    // builds K columns [KX q/kSplit, KX (q+1)/kSplit) of the row
    {
      const int64_t e = r < 0x7fffffff ? int64_t(uint32_t(r) / uint32_t(AA)) : r / AA;
      const int a = int(r - e * AA);
      const int k0 = (KX / kSplit) * part;
      auto build = [&](auto load) {
#pragma unroll 2
        for (int kk = 0; kk < KX / kSplit; kk += 8) {
          float x[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = k0 + kk + j;
            x[j] = (live && k < D) ? load(k) : 0.0f;
            if (live && AA > 1 && k == D + a) x[j] = 1.0f;
          }
          if (live && act_mode && HAS_OUT) {
            float* o = obs_out + tid * in_dim;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (k0 + kk + j < in_dim) o[k0 + kk + j] = x[j];
          }
          put8(sx, KX, tid, k0 + kk, x);
        }
      };
      if constexpr (KXT != 0) {  // small rows: every load issued before any store
        const float* so = obs_in[cur] + tid * D;
        float x[KXT / kSplit];
#pragma unroll
        for (int j = 0; j < KXT / kSplit; ++j) {
          const int k = k0 + j;
          x[j] = (live && k < D) ? so[k] : 0.0f;
          if (live && AA > 1 && k == D + a) x[j] = 1.0f;
          // folded instance: the last two K columns carry layer 1's bias (hi / lo
          // bf16 halves in W1's image, pack_bf16_kernel) -- the MMA adds it
          if (SD && live && k >= KXT - 2) x[j] = 1.0f;
        }
        if (live && act_mode) {
          float* o = obs_out + tid * in_dim;
#pragma unroll
          for (int j = 0; j < KXT / kSplit; ++j)
            if (k0 + j < in_dim) o[k0 + j] = x[j];
        }
#pragma unroll
        for (int j = 0; j < KXT / kSplit; j += 8) put8(sx, KXT, tid, k0 + j, x + j);
      } else if (NBUF > 0) {  // staged (shared) rows
        const float* so = obs_in[cur] + tid * D;
        build([&](int k) { return so[k]; });
      } else {  // rows through L2
        const float* go = s.env_obs + size_t(r) * size_t(D);
        build([&](int k) { return __ldg(go + k); });
      }
      if (live && act_mode) {
        if (part == 0) {
          s_resets[tid] = s.prev_finished ? s.prev_finished[e] : uint8_t(1);
          uint8_t* lg = s_legal + tid * n_act;
          if (s.legal_ready) {
            const uint8_t* gl = b.legal + (slot0 + size_t(tid)) * n_act;
            for (int q = 0; q < n_act; ++q) lg[q] = gl[q];
          } else {
            const int na = s.agent_actions[a];
#pragma unroll
            for (int q = 0; q < (SN ? SN : 16); ++q)
              if (q < n_act) lg[q] = q < na ? 1 : 0;
          }
          s_active[tid] = (s.family == 1) ? (lg[0] ? 1.0f : 0.0f) : 1.0f;
        }
      }
    }
    if (CENT) {  // MAPPO critic rows: the env's world_state (ppo.cpp:341-346), part q builds K columns
      // [KC q/kSplit, KC (q+1)/kSplit); the buffer keeps them in critic_in rows
      const int64_t e = r < 0x7fffffff ? int64_t(uint32_t(r) / uint32_t(AA)) : r / AA;
      const float* wsr = s.ws + size_t(e) * size_t(critic_in);
      float* bc = b.critic_in + (slot0 + size_t(tid)) * size_t(critic_in);
      const int kc0 = (KC / kSplit) * part;
      for (int kk = 0; kk < KC / kSplit; kk += 8) {
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kc0 + kk + j;
          x[j] = (live && k < critic_in) ? __ldg(wsr + k) : 0.0f;
          if (live && act_mode && k < critic_in) bc[k] = x[j];
        }
        put8(sxc, KC, tid, kc0 + kk, x);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (act_mode) {  // the input-side buffer rows leave while the MMAs run
      if (HAS_OUT) {
        tile_put(b.obs + slot0 * in_dim, obs_out, size_t(rows) * in_dim * 4);
      } else {  // rebuilt from the tile's observation rows, coalesced
        float* go = b.obs + slot0 * in_dim;
        const int n = rows * in_dim;
        for (int q = threadIdx.x; q < n; q += blockDim.x) {
          const int rr = q / in_dim, k = q - rr * in_dim;
          const int a = int((r0 + rr) % AA);
          go[q] = k < D ? (NBUF > 0 ? tile_obs[rr * D + k] : __ldg(tile_obs + size_t(rr) * D + k))
                        : ((AA > 1 && k == D + a) ? 1.0f : 0.0f);
        }
      }
      if (!s.legal_ready) tile_put(b.legal + slot0 * n_act, s_legal, size_t(rows) * n_act);
      if (threadIdx.x == 0) bulk_commit();
      if (live && part == 0) {  // one element per thread: already coalesced
        b.resets[slot0 + tid] = s_resets[tid];
        b.active[slot0 + tid] = s_active[tid];
      }
    }
    if (NBUF == 1) {  // the single staging tile has been read: prefetch the next tile into it
      __syncthreads();
      in_flight[0] = next < n_tiles ? tile_obs_load(s, next, obs_in[0], bar_in[0]) : false;
    }
    if (threadIdx.x == 0) {
      tc_fence_after();
      if (CENT) {  // actor rows 0-63 of W1 over X; the critic's W1 over the world_state tile
        const uint32_t id = idesc_bf16(128, 64);
        for (int k = 0; k < KX; k += 16) umma_bf16(tmem + 0, umma_desc(sx, KX, k), umma_desc(w1, KX, k), id, k > 0);
        for (int k = 0; k < KC; k += 16) umma_bf16(tmem + 64, umma_desc(sxc, KC, k), umma_desc(wc1, KC, k), id, k > 0);
      } else {
        const uint32_t id = idesc_bf16(128, 128);
        for (int k = 0; k < KX; k += 16) umma_bf16(tmem + 0, umma_desc(sx, KX, k), umma_desc(w1, KX, k), id, k > 0);
      }
      umma_commit(bar);
    }
    // the row's sampling uniform (two Threefry blocks) is drawn by part 1
    // while the layer-1 MMA runs; part 0 samples with it after layer 3
    if (part == 1 && live && act_mode) s_u[tid] = row_uniform(s, r);
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 1: bias + tanh -> bf16 hidden rows
#pragma unroll 1
    for (int c = (128 / kSplit) * part; c < (128 / kSplit) * (part + 1); c += 32) {  // this part's columns
      float v[32];
      tmem_ld32(tmem + lane_base + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = tanh_fast(SD ? v[i] : v[i] + s_bias[c + i]);
      uint8_t* dsth = c < 64 ? ha : hc;
      put16(dsth, 64, tid, c & 63, v);
      put16(dsth, 64, tid, (c & 63) + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 64);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(ha, 64, k), umma_desc(w2a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 64, umma_desc(hc, 64, k), umma_desc(w2c, 64, k), id, k > 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 2
#pragma unroll 1
    for (int c = (128 / kSplit) * part; c < (128 / kSplit) * (part + 1); c += 32) {  // this part's columns
      float v[32];
      tmem_ld32(tmem + lane_base + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = tanh_fast(v[i] + s_bias[128 + c + i]);
      uint8_t* dsth = c < 64 ? ha : hc;
      put16(dsth, 64, tid, c & 63, v);
      put16(dsth, 64, tid, (c & 63) + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 16);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(ha, 64, k), umma_desc(w3a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 16, umma_desc(hc, 64, k), umma_desc(w3c, 64, k), id, k > 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 3: part 0 samples from the actor head, part 1 writes the value
    if (part < 2) {
      float hv[16];
      tmem_ld16(tmem + lane_base + uint32_t(16 * part), hv);  // logits in 0..15 / value in 16
      tc_fence_before();
      if (part == 1) {
        const float value = hv[0] + s_bias[256 + 16];
        if (live) {
          if (act_mode) b.value[slot0 + tid] = value;
          else b.last_value[r] = value;
        }
      } else if (act_mode && live) {
        float logits[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) logits[j] = hv[j] + s_bias[256 + j];
        int pick;
        float lp;
        sample_row_n<SN ? SN : 16>(s_u[tid], logits, s_legal + tid * n_act, n_act, &pick, &lp);
        b.actions[slot0 + tid] = pick;  // one element per thread: coalesced
        b.logp[slot0 + tid] = lp;
      }
    }
    if (NBUF == 2) cur ^= 1;
    __syncthreads();  // TMEM columns and operand tiles are reused by the next tile
  }
  if (threadIdx.x == 0) bulk_wait<0>();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

// ---------------------------------------------------------------- wide rows
// IPPO inputs wider than kTcMaxKx (Overcooked: 520-wide observation rows):
// layer 1 runs K-chunked.  W1's image is chunk-major ([KX/64][128 x 64]
// canonical tiles); per 64-column chunk one TMA bulk load brings the W1 tile
// (mbarrier expect-tx) while the 256 threads build the X chunk straight from
// the observation rows in L2 (two threads per row, 32 columns each, the
// buffer's input row written on the way), and one thread issues the chunk's
// four MMAs into the same TMEM accumulators; W1 and X tiles are double
// buffered across chunks (and tiles) and a buffer is refilled only after the
// chunk two back has been committed.  Layers 2-3, sampling and the buffer
// writes are the staged kernel's.
struct WideLayout {
  uint32_t wbuf[2], xbuf[2], ostage[2], w2a, w2c, w3a, w3c, ha, hc, legal, resets, active, bias, bar, bar_w[2],
      bar_c[2], tmem_slot, total;
};
constexpr int kOsPitch = 72;  // fp32 observation staging rows: the 16-byte-aligned 68-float superset of 64 columns, + 4

// cp.async of SZ bytes (4, 8 or 16), zero-filled beyond src_bytes
template <int SZ>
__device__ __forceinline__ void cpa(void* sdst, const void* gsrc, uint32_t src_bytes) {
  if constexpr (SZ == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(sdst)), "l"(gsrc), "n"(SZ),
                 "r"(src_bytes)
                 : "memory");
}

// The [128 rows x 64 columns] fp32 observation block of chunk c of the tile at
// rb into a staging buffer with 16-byte copies whatever D's alignment: row i's
// columns start at float e = (rb + i) D + 64c, and the 17 copies cover the
// aligned superset [e & ~3, (e & ~3) + 68), so the row's data sits at offset
// e & 3 of its staging row (columns past D belong to the next row: the builder
// masks them).  Copies past the end of the observations (or of R) read nothing
// (zero-filled).  One commit group per call, possibly empty.
__device__ __forceinline__ void stage_obs(float* dst, const float* obs, int64_t R, int D, int64_t rb, int c, int nth) {
  const int nrows = int(rb < R ? min64(kTcRows, R - rb) : 0);
  const int64_t total = R * int64_t(D);
  for (int idx = threadIdx.x; idx < kTcRows * 17; idx += nth) {
    const int row = idx / 17, g = idx - row * 17;
    const int64_t e4 = ((rb + row) * int64_t(D) + 64 * c) & ~int64_t(3), q = e4 + 4 * g;
    int64_t nv = row < nrows ? total - q : 0;
    nv = nv < 0 ? 0 : nv > 4 ? 4 : nv;
    cpa<16>(dst + row * kOsPitch + 4 * g, nv ? obs + q : obs, uint32_t(nv * 4));
  }
}

__host__ __device__ inline WideLayout wide_layout(int n_act) {
  WideLayout L{};
  uint32_t o = 0;
  auto take = [&o](uint32_t bytes, uint32_t align) {
    o = up(o, align);
    const uint32_t at = o;
    o += bytes;
    return at;
  };
  for (int q = 0; q < 2; ++q) L.wbuf[q] = take(128 * 64 * 2, 1024);
  for (int q = 0; q < 2; ++q) L.xbuf[q] = take(kTcRows * 64 * 2, 1024);
  for (int q = 0; q < 2; ++q) L.ostage[q] = take(kTcRows * kOsPitch * 4, 16);
  L.w2a = take(64 * 64 * 2, 128);
  L.w2c = take(64 * 64 * 2, 128);
  L.w3a = take(64 * 64 * 2, 128);  // actor head: up to 64 actions
  L.w3c = take(16 * 64 * 2, 128);
  L.ha = take(kTcRows * 64 * 2, 128);
  L.hc = take(kTcRows * 64 * 2, 128);
  L.legal = take(uint32_t(kTcRows * n_act), 16);
  L.resets = take(kTcRows, 16);
  L.active = take(kTcRows * 4, 16);
  L.bias = take((4 * 64 + 2 * 16 + 64) * 4, 16);
  L.bar = take(8, 8);
  for (int q = 0; q < 2; ++q) L.bar_w[q] = take(8, 8);
  for (int q = 0; q < 2; ++q) L.bar_c[q] = take(8, 8);
  L.tmem_slot = take(4, 4);
  L.total = up(o, 128);
  return L;
}

#ifndef MARL_WIDE_SPLIT
#define MARL_WIDE_SPLIT 4
#endif
constexpr int kSplitW = MARL_WIDE_SPLIT;  // wide kernel: threads per row (more warps for the X build's memory traffic)
__global__ void __launch_bounds__(kSplitW * kTcRows, 1) policy_tc_wide_kernel(PolicyNetBf16 nb, int in_dim, int n_act,
                                                                            PolicyStep s, RolloutBufs b) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const WideLayout L = wide_layout(n_act);
  uint8_t* base = smem_raw;
  uint8_t *w2a = base + L.w2a, *w2c = base + L.w2c, *w3a = base + L.w3a, *w3c = base + L.w3c, *ha = base + L.ha,
          *hc = base + L.hc;
  uint8_t* wbuf[2] = {base + L.wbuf[0], base + L.wbuf[1]};
  uint8_t* xbuf[2] = {base + L.xbuf[0], base + L.xbuf[1]};
  float* ostage[2] = {reinterpret_cast<float*>(base + L.ostage[0]), reinterpret_cast<float*>(base + L.ostage[1])};
  uint8_t* s_legal = base + L.legal;
  uint8_t* s_resets = base + L.resets;
  float* s_active = reinterpret_cast<float*>(base + L.active);
  float* s_bias = reinterpret_cast<float*>(base + L.bias);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bar);
  uint64_t* bar_w[2] = {reinterpret_cast<uint64_t*>(base + L.bar_w[0]), reinterpret_cast<uint64_t*>(base + L.bar_w[1])};
  uint64_t* bar_c[2] = {reinterpret_cast<uint64_t*>(base + L.bar_c[0]), reinterpret_cast<uint64_t*>(base + L.bar_c[1])};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L.tmem_slot);
  const int tid = threadIdx.x & (kTcRows - 1), part = threadIdx.x >> 7, warp = threadIdx.x >> 5,
            lane = threadIdx.x & 31;
  const int64_t n_tiles = (s.R + kTcRows - 1) / kTcRows;
  const int D = s.D, AA = s.A, KX = tc_kx(in_dim), NC = KX / 64;
  const int hn = n_act <= 16 ? 16 : (n_act + 15) / 16 * 16;  // actor head MMA N

  if (threadIdx.x == 0) {
    for (uint64_t* m : {bar, bar_w[0], bar_w[1], bar_c[0], bar_c[1]})
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  {
    const uint4* src[4] = {reinterpret_cast<const uint4*>(nb.a2), reinterpret_cast<const uint4*>(nb.c2),
                           reinterpret_cast<const uint4*>(nb.h3), reinterpret_cast<const uint4*>(nb.hc3)};
    uint4* dst[4] = {reinterpret_cast<uint4*>(w2a), reinterpret_cast<uint4*>(w2c), reinterpret_cast<uint4*>(w3a),
                     reinterpret_cast<uint4*>(w3c)};
    const int n16[4] = {64 * 64 * 2 / 16, 64 * 64 * 2 / 16, 64 * 64 * 2 / 16, 16 * 64 * 2 / 16};
    for (int m = 0; m < 4; ++m)
      for (int q = threadIdx.x; q < n16[m]; q += blockDim.x) dst[m][q] = __ldg(src[m] + q);
    for (int q = threadIdx.x; q < 4 * 64 + 2 * 16 + 64; q += blockDim.x) s_bias[q] = __ldg(nb.bias + q);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
  const bool act_mode = !s.bootstrap;
  uint32_t phase = 0;
  int64_t cc = 0;  // chunks issued by this CTA (buffer cc & 1, its (cc >> 1)-th use)
  // the observation block of chunk cc + 1 streams into staging buffer (cc + 1) & 1
  // while chunk cc is built (cp.async, 16-byte copies)
  auto prefetch = [&](int64_t tl, int c, int q) {
    stage_obs(ostage[q], s.env_obs, s.R, D, tl * kTcRows, c, kSplitW * kTcRows);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch(blockIdx.x, 0, 0);

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r0 = tile * kTcRows, r = r0 + tid;
    const int rows = int(min64(kTcRows, s.R - r0));
    const bool live = tid < rows;
    const size_t slot0 = size_t(s.t) * size_t(s.R) + size_t(r0);
    const int64_t e = r < 0x7fffffff ? int64_t(uint32_t(r) / uint32_t(AA)) : r / AA;
    const int a = int(r - e * AA);
    if (live && act_mode && part == 0) {  // write_legal / agent_active (team.cpp:35-42)
      s_resets[tid] = s.prev_finished ? s.prev_finished[e] : uint8_t(1);
      uint8_t* lg = s_legal + tid * n_act;
      if (s.legal_ready) {
        const uint8_t* gl = b.legal + (slot0 + size_t(tid)) * n_act;
        for (int q = 0; q < n_act; ++q) lg[q] = gl[q];
      } else {
        const int na = s.agent_actions[a];
        for (int q = 0; q < n_act; ++q) lg[q] = q < na ? 1 : 0;
      }
      s_active[tid] = (s.family == 1) ? (lg[0] ? 1.0f : 0.0f) : 1.0f;
    }
    const double u_row = (part == 0 && live && act_mode) ? row_uniform(s, r) : 0.0;  // part 0 samples
    // ---- layer 1, K-chunked
    for (int c = 0; c < NC; ++c, ++cc) {
      const int bs = int(cc & 1);
      // the next chunk's observation block (this tile's, else the next tile's first)
      if (c + 1 < NC)
        prefetch(tile, c + 1, bs ^ 1);
      else
        prefetch(tile + gridDim.x, 0, bs ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this chunk's block has landed (own copies)
      __syncthreads();                                       // (everyone's)
      // the MMAs of chunk cc - 2 read this buffer pair
      if (cc >= 2) mbar_wait(bar_c[bs], uint32_t((cc - 2) >> 1) & 1u);
      if (threadIdx.x == 0)
        bulk_load_g2s(wbuf[bs], nb.a1 + size_t(c) * (128 * 64), 128 * 64 * 2, bar_w[bs]);
      // the chunk's [128 rows x 64 columns] X block, built warp-cooperatively: a
      // warp instruction covers 8 rows x 32 columns (4 lanes x 8 columns per row),
      // so the observation loads and buffer-row stores are 32-byte segments and
      // each lane's bf16 octet is one conflict-free 16-byte canonical store
      for (int it = warp; it < 2 * (kTcRows / 8); it += kSplitW * kTcRows / 32) {
        const int rr = (it >> 1) * 8 + (lane >> 2), k = 64 * c + 32 * (it & 1) + 8 * (lane & 3);
        const bool lv = rr < rows;
        float x[8];
        const float* sv = ostage[bs] + rr * kOsPitch + int(((r0 + rr) * int64_t(D) + 64 * c) & 3) + (k - 64 * c);
        if (k + 8 <= D) {
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = sv[j];  // zero for rows beyond R
        } else {  // past the observation: zeros, then the agent one-hot (TeamLayout::write_input)
          const int ar = lv && AA > 1 ? int((r0 + rr) % AA) : -1;
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = k + j < D ? sv[j] : (k + j == D + ar ? 1.0f : 0.0f);
        }
        if (lv && act_mode) {
          float* br = b.obs + (slot0 + size_t(rr)) * size_t(in_dim);
          if (k + 8 <= in_dim && (in_dim & 1) == 0) {
            float2* b2 = reinterpret_cast<float2*>(br + k);
#pragma unroll
            for (int j = 0; j < 4; ++j) b2[j] = make_float2(x[2 * j], x[2 * j + 1]);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (k + j < in_dim) br[k + j] = x[j];
          }
        }
        put8(xbuf[bs], 64, rr, k - 64 * c, x);
      }
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        mbar_wait(bar_w[bs], uint32_t(cc >> 1) & 1u);
        tc_fence_after();
        const uint32_t id = idesc_bf16(128, 128);
        for (int k = 0; k < 64; k += 16)
          umma_bf16(tmem + 0, umma_desc(xbuf[bs], 64, k), umma_desc(wbuf[bs], 64, k), id, (c > 0 || k > 0) ? 1u : 0u);
        umma_commit(bar_c[bs]);
      }
    }
    if (act_mode) {  // legal rows (when the kernel built them), resets, active
      fence_proxy_async_smem();
      __syncthreads();
      if (!s.legal_ready) tile_put(b.legal + slot0 * n_act, s_legal, size_t(rows) * n_act);
      if (threadIdx.x == 0) bulk_commit();
      if (live && part == 0) {
        b.resets[slot0 + tid] = s_resets[tid];
        b.active[slot0 + tid] = s_active[tid];
      }
    }
    mbar_wait(bar_c[int((cc - 1) & 1)], uint32_t((cc - 1) >> 1) & 1u);  // the tile's last chunk: all of layer 1
    tc_fence_after();
    // ---- epilogue 1 / layer 2 / epilogue 2 / heads: as the staged kernel
#pragma unroll 1
    for (int cl = (128 / kSplitW) * part; cl < (128 / kSplitW) * (part + 1); cl += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + uint32_t(cl), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = tanh_fast(v[i] + s_bias[cl + i]);
      uint8_t* dsth = cl < 64 ? ha : hc;
      put16(dsth, 64, tid, cl & 63, v);
      put16(dsth, 64, tid, (cl & 63) + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 64);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(ha, 64, k), umma_desc(w2a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 64, umma_desc(hc, 64, k), umma_desc(w2c, 64, k), id, k > 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
#pragma unroll 1
    for (int cl = (128 / kSplitW) * part; cl < (128 / kSplitW) * (part + 1); cl += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + uint32_t(cl), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = tanh_fast(v[i] + s_bias[128 + cl + i]);
      uint8_t* dsth = cl < 64 ? ha : hc;
      put16(dsth, 64, tid, cl & 63, v);
      put16(dsth, 64, tid, (cl & 63) + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {  // actor head: TMEM columns 0..hn-1; critic head: 64..79
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, hn);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(ha, 64, k), umma_desc(w3a, 64, k), id, k > 0);
      const uint32_t idc = idesc_bf16(128, 16);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 64, umma_desc(hc, 64, k), umma_desc(w3c, 64, k), idc, k > 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    if (part == 1) {
      float hv[16];
      tmem_ld16(tmem + lane_base + 64u, hv);
      tc_fence_before();
      const float value = hv[0] + s_bias[256 + 16];
      if (live) {
        if (act_mode) b.value[slot0 + tid] = value;
        else b.last_value[r] = value;
      }
    } else if (part == 0 && hn == 16) {
      float hv[16];
      tmem_ld16(tmem + lane_base, hv);
      tc_fence_before();
      if (act_mode && live) {
        float logits[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) logits[j] = hv[j] + s_bias[256 + j];
        int pick;
        float lp;
        sample_row_n<16>(u_row, logits, s_legal + tid * n_act, n_act, &pick, &lp);
        b.actions[slot0 + tid] = pick;
        b.logp[slot0 + tid] = lp;
      }
    } else if (part == 0) {  // up to 64 actions (SMAX 27m_vs_30m: 35)
      float logits[64];
      tmem_ld32(tmem + lane_base, logits);
      tmem_ld32(tmem + lane_base + 32u, logits + 32);
      tc_fence_before();
      if (act_mode && live) {
#pragma unroll
        for (int j = 0; j < 64; ++j) logits[j] += s_bias[288 + j];
        int pick;
        float lp;
        sample_row_wide(u_row, logits, s_legal + tid * n_act, n_act, &pick, &lp);
        b.actions[slot0 + tid] = pick;
        b.logp[slot0 + tid] = lp;
      }
    }
    if (threadIdx.x == 0) bulk_wait_read<0>();  // the legal tile has been read out before it is rebuilt
    __syncthreads();  // TMEM columns and hidden tiles are reused by the next tile
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");  // the last (empty) prefetch
  if (threadIdx.x == 0) bulk_wait<0>();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

// fp32 parameters -> canonical bf16 operand images + bias block.
__global__ void pack_bf16_kernel(PolicyNet n, uint16_t* img, float* bias) {
  const int in = n.in_dim, NA = n.n_act, KX = tc_kx(in);
  uint16_t* a1 = img;
  uint16_t* a2 = a1 + 128 * KX;
  uint16_t* c2 = a2 + 64 * 64;
  uint16_t* h3 = c2 + 64 * 64;
  uint16_t* hc3 = h3 + 64 * 64;
  uint16_t* c1 = hc3 + 16 * 64;  // MAPPO: the critic's W1 over world_state rows
  auto bf = [](float v) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    return *reinterpret_cast<const uint16_t*>(&h);
  };
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 128 * KX; q += gridDim.x * blockDim.x) {
    const int row = q / KX, k = q % KX;
    float v = 0.0f;
    if (k < in && (row < 64 || !n.centralized)) v = row < 64 ? n.w1[row * in + k] : n.cw1[(row - 64) * in + k];
    if (KX == 32 && in <= 30 && k >= 30) {  // layer-1 bias as hi / lo bf16 columns (read only by the folded
      const float bb = row < 64 ? n.b1[row] : n.cb1[row - 64];  // instance, whose X carries 1 there)
      const __nv_bfloat16 hi = __float2bfloat16_rn(bb);
      v = k == 30 ? bb : bb - __bfloat162float(hi);
    }
    if (KX > kTcMaxKx)  // wide rows: [chunk of 64 K][128 rows x 64] canonical tiles
      a1[(k / 64) * (128 * 64) + canon_off(row, k % 64, 64) / 2] = bf(v);
    else
      a1[canon_off(row, k, KX) / 2] = bf(v);
  }
  if (n.centralized) {
    const int CI = n.critic_in, KC = tc_kc(CI);
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 64 * KC; q += gridDim.x * blockDim.x) {
      const int row = q / KC, k = q % KC;
      c1[canon_off(row, k, KC) / 2] = bf(k < CI ? n.cw1[row * CI + k] : 0.0f);
    }
  }
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 64 * 64; q += gridDim.x * blockDim.x) {
    const int row = q / 64, k = q % 64;
    a2[canon_off(row, k, 64) / 2] = bf(n.w2[row * 64 + k]);
    c2[canon_off(row, k, 64) / 2] = bf(n.cw2[row * 64 + k]);
  }
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 64 * 64; q += gridDim.x * blockDim.x) {
    const int row = q / 64, k = q % 64;
    h3[canon_off(row, k, 64) / 2] = bf(row < NA ? n.w3[row * 64 + k] : 0.0f);
    if (row < 16) hc3[canon_off(row, k, 64) / 2] = bf(row == 0 ? n.cw3[k] : 0.0f);
  }
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 64; q += gridDim.x * blockDim.x) {
    bias[q] = n.b1[q];
    bias[64 + q] = n.cb1[q];
    bias[128 + q] = n.b2[q];
    bias[192 + q] = n.cb2[q];
    bias[288 + q] = q < NA ? n.b3[q] : 0.0f;
    if (q < 16) {
      bias[256 + q] = q < NA ? n.b3[q] : 0.0f;
      bias[272 + q] = q == 0 ? n.cb3[0] : 0.0f;
    }
  }
}

}  // namespace

int rollout_tc_kx(int in_dim) { return tc_kx(in_dim); }

bool rollout_policy_bf16_supported(int in_dim, int n_act, int width, int critic_in) {
  if (in_dim > kTcMaxKx)  // wide rows: the K-chunked kernel (IPPO critics)
    return critic_in == 0 && n_act <= 64 && width == 64 && wide_layout(n_act).total <= kTcSmemMax;
  // D <= in_dim: the layout without staged tiles bounds every mode
  return in_dim >= 1 && tc_kx(in_dim) <= kTcMaxKx && tc_kc(critic_in) <= kTcMaxKx && n_act <= 16 && width == 64 &&
         tc_layout_mode(in_dim, in_dim, n_act, 0, critic_in).total <= kTcSmemMax;
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
  if (net.in_dim > kTcMaxKx) {  // wide rows: K-chunked layer 1, one CTA per SM
    const size_t smw = wide_layout(net.n_act).total;
    smem_optin(policy_tc_wide_kernel);
    const int64_t tiles = (s.R + kTcRows - 1) / kTcRows;
    const int64_t grid = cap_grid(std::min<int64_t>(tiles, int64_t(sms)));
    policy_tc_wide_kernel<<<unsigned(grid), kSplitW * kTcRows, smw, st>>>(nb, net.in_dim, net.n_act, s, b);
    ++g_launches;
    return;
  }
  const bool cent = s.ws != nullptr;
  const int ci = cent ? net.critic_in : 0;
  const size_t sm = tc_layout(s.D, net.in_dim, net.n_act, ci).total;
  const TcLayout L = tc_layout(s.D, net.in_dim, net.n_act, ci);
  const bool small = !cent && L.kx == 32 && L.nbuf == 2 && L.has_out;
  // MPE simple_spread (obs 18, 3 agents, 5 actions): the folded instance
  const bool spread = small && s.D == 18 && s.A == 3 && net.n_act == 5 && net.in_dim == 21 &&
                      !std::getenv("MARL_TC_GENERIC");
  auto kern = small ? (spread ? policy_tc_kernel<32, 18, 3, 5> : policy_tc_kernel<32>)
                    : (cent ? policy_tc_kernel<0, 0, 0, 0, true> : policy_tc_kernel<0>);
  smem_optin(kern);
  int per_sm = 1;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  static int smem_sm = 0;
  if (smem_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  }
  // the occupancy API under-reports here (1); count shared memory (1 KB
  // reserved per CTA), threads and TMEM columns directly
  per_sm = int(size_t(smem_sm) / (sm + 1024));
  per_sm = std::max(1, std::min({per_sm, int(512 / kTmemCols), 2048 / (kSplit * kTcRows)}));
  if (const char* f = std::getenv("MARL_TC_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(f)));
  if (const char* f = std::getenv("MARL_TC_FORCE_PER_SM")) per_sm = std::atoi(f);
  if (std::getenv("MARL_TC_DEBUG")) std::fprintf(stderr, "policy_tc: smem %zu per_sm %d\n", sm, per_sm);
  const int64_t tiles = (s.R + kTcRows - 1) / kTcRows;
  const int64_t grid = cap_grid(std::min<int64_t>(tiles, int64_t(sms) * per_sm));
  kern<<<unsigned(grid), kSplit * kTcRows, sm, st>>>(nb, net.in_dim, net.n_act, s, b, ci);
  ++g_launches;
}

void rollout_gae(const RolloutBufs& b, int T, int64_t R, float gamma, float lambda, cudaStream_t st) {
  gae_kernel<<<unsigned((R + 255) / 256), 256, 0, st>>>(b, T, R, gamma, lambda);
  ++g_launches;
}

}  // namespace marl_b200
