// Overcooked kitchens (reference: proj/core/src/envs/overcooked.cpp) as one
// fused sm_100a kernel per batch step.  The transition is a handful of integer
// ops per env; 97% of the bytes are the 27-plane observation rows
// (overcooked.cpp:395-427), so the kernel is organised around storing them at
// HBM speed:
//   * state update: one thread per env (threads 0..E-1 of the block),
//   * observation: the block's [E][2][D] rows are filled from a static
//     layout template in shared memory (planes 10-14 never change), patched
//     with the ~20 dynamic cells per row, and leave as contiguous 16-byte
//     streaming stores of the whole tile.
// All state is integer and trajectories are bit-identical to the reference.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {
namespace {

constexpr int kE = 16;          // envs per block
constexpr int kThreads = 128;
constexpr int kUp = 0, kDown = 1, kLeft = 2, kRight = 3, kStay = 4, kInteract = 5;  // overcooked.cpp:16
constexpr int kNone = 0, kOnion = 1, kPlate = 2, kSoup = 3;                         // overcooked.cpp:21
constexpr int kPlanes = 27;

struct Kitchen {  // KitchenState (overcooked.cpp:131-139), unpacked
  int pos[2], facing[2], held[2];
  int onions[kOcMaxPots], timer[kOcMaxPots];
  uint64_t counters[2];  // 2 bits per counter cell
  int t;
};

__device__ __forceinline__ int dr(int a) { return a == kUp ? -1 : a == kDown ? 1 : 0; }
__device__ __forceinline__ int dc(int a) { return a == kLeft ? -1 : a == kRight ? 1 : 0; }

__device__ __forceinline__ int counter_get(const Kitchen& s, int k) {
  return int((s.counters[k >> 5] >> (2 * (k & 31))) & 3u);
}
__device__ __forceinline__ void counter_set(Kitchen& s, int k, int v) {
  uint64_t& w = s.counters[k >> 5];
  const int sh = 2 * (k & 31);
  w = (w & ~(uint64_t(3) << sh)) | (uint64_t(v) << sh);
}

__device__ __forceinline__ void load(Kitchen& s, const OcConfig& c, const OcState& st, int64_t i, int64_t n) {
  uint32_t a = st.agents[i];
  s.pos[0] = int(a & 0xff);
  s.pos[1] = int((a >> 8) & 0xff);
  s.facing[0] = int((a >> 16) & 3);
  s.facing[1] = int((a >> 18) & 3);
  s.held[0] = int((a >> 20) & 3);
  s.held[1] = int((a >> 22) & 3);
  for (int p = 0; p < c.n_pots; ++p) {
    uint32_t w = st.pots[p * n + i];
    s.onions[p] = int(w & 0xff);
    s.timer[p] = int(w >> 8);
  }
  s.counters[0] = st.counters[i];
  s.counters[1] = c.n_counters > 32 ? st.counters[n + i] : 0;
  s.t = st.t[i];
}

__device__ __forceinline__ void store(const Kitchen& s, const OcConfig& c, const OcState& st, int64_t i, int64_t n) {
  st.agents[i] = uint32_t(s.pos[0]) | (uint32_t(s.pos[1]) << 8) | (uint32_t(s.facing[0]) << 16) |
                 (uint32_t(s.facing[1]) << 18) | (uint32_t(s.held[0]) << 20) | (uint32_t(s.held[1]) << 22);
  for (int p = 0; p < c.n_pots; ++p) st.pots[p * n + i] = uint32_t(s.onions[p]) | (uint32_t(s.timer[p]) << 8);
  st.counters[i] = s.counters[0];
  if (c.n_counters > 32) st.counters[n + i] = s.counters[1];
  st.t[i] = s.t;
}

// OvercookedEnv::reset (overcooked.cpp:193-204): the key is unused.
__device__ __forceinline__ void env_reset(Kitchen& s, const OcConfig& c) {
  s.pos[0] = c.spawn[0];
  s.pos[1] = c.spawn[1];
  s.facing[0] = s.facing[1] = kUp;
  s.held[0] = s.held[1] = kNone;
  for (int p = 0; p < kOcMaxPots; ++p) s.onions[p] = s.timer[p] = 0;
  s.counters[0] = s.counters[1] = 0;
  s.t = 0;
}

__device__ __forceinline__ int pot_index(const OcConfig& c, int cell) {
  int p = 0;  // lower_bound over ascending pot cells (overcooked.cpp:386-389)
  while (p < c.n_pots && c.pot_cells[p] < cell) ++p;
  return p;
}
__device__ __forceinline__ int counter_index(const OcConfig& c, int cell) {
  int k = 0;  // overcooked.cpp:390-393
  while (k < c.n_counters && c.counter_cells[k] < cell) ++k;
  return k;
}

// OvercookedEnv::step (overcooked.cpp:206-313); returns done.
__device__ __forceinline__ bool env_step(Kitchen& s, const OcConfig& c, const Key& key, const int* act,
                                         double& reward, double* shaped, int& deliveries) {
  const int prev0 = s.pos[0], prev1 = s.pos[1];
  for (int p = 0; p < c.n_pots; ++p)
    if (s.onions[p] == 3 && s.timer[p] > 0) s.timer[p] -= 1;
  int want[2] = {s.pos[0], s.pos[1]};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (act[i] > kRight) continue;
    s.facing[i] = act[i];
    int r = s.pos[i] / c.w + dr(act[i]);
    int cc = s.pos[i] % c.w + dc(act[i]);
    if (c.kind[r * c.w + cc] == ' ') want[i] = r * c.w + cc;
  }
  const bool swap = want[0] == prev1 && want[1] == prev0 && want[0] != prev0;
  if (want[0] == want[1] || swap) {
    if (c.random_conflicts && !swap && want[0] != prev0 && want[1] != prev1) {
      int loser = to_unit(block_at(key, 0)) < 0.5 ? 0 : 1;  // bernoulli(key, 0.5), prng.cpp:237-240
      want[loser] = loser == 0 ? prev0 : prev1;
    } else {
      want[0] = prev0;
      want[1] = prev1;
    }
  }
  s.pos[0] = want[0];
  s.pos[1] = want[1];
  shaped[0] = shaped[1] = 0.0;
  deliveries = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (act[i] != kInteract) continue;
    const int r = s.pos[i] / c.w + dr(s.facing[i]);
    const int cc = s.pos[i] % c.w + dc(s.facing[i]);
    const int cell = r * c.w + cc;
    switch (c.kind[cell]) {
      case 'O':
        if (s.held[i] == kNone) s.held[i] = kOnion;
        break;
      case 'D':
        if (s.held[i] == kNone) {
          s.held[i] = kPlate;
          shaped[i] += c.sh_plate;
        }
        break;
      case 'P': {
        const int p = pot_index(c, cell);
        if (s.held[i] == kOnion && s.onions[p] < 3) {
          s.onions[p] += 1;
          s.held[i] = kNone;
          shaped[i] += c.sh_onion;
          if (s.onions[p] == 3) s.timer[p] = c.cook_time;
        } else if (s.held[i] == kPlate && s.onions[p] == 3 && s.timer[p] == 0) {
          s.held[i] = kSoup;
          s.onions[p] = 0;
          shaped[i] += c.sh_soup;
        }
        break;
      }
      case 'S':
        if (s.held[i] == kSoup) {
          s.held[i] = kNone;
          deliveries += 1;
        }
        break;
      case 'X': {
        const int k = counter_index(c, cell);
        const int item = counter_get(s, k);
        if (s.held[i] != kNone && item == kNone) {
          counter_set(s, k, s.held[i]);
          s.held[i] = kNone;
        } else if (s.held[i] == kNone && item != kNone) {
          s.held[i] = item;
          counter_set(s, k, kNone);
        }
        break;
      }
      default:
        break;
    }
  }
  s.t += 1;
  reward = c.delivery_reward * deliveries;
  return s.t >= c.max_steps;
}

// Dynamic cells of encode() (overcooked.cpp:395-427) for agent `me`; the
// static planes come from the template already in the row.
__device__ __forceinline__ void patch_row(float* o, const Kitchen& s, const OcConfig& c, int me) {
  const int cells = c.h * c.w, other = 1 - me;
  o[0 * cells + s.pos[me]] = 1.0f;
  o[1 * cells + s.pos[other]] = 1.0f;
  o[(2 + s.facing[me]) * cells + s.pos[me]] = 1.0f;
  o[(6 + s.facing[other]) * cells + s.pos[other]] = 1.0f;
  for (int p = 0; p < c.n_pots; ++p) {
    const int cell = c.pot_cells[p];
    o[15 * cells + cell] = float(s.onions[p]);
    o[16 * cells + cell] = float(s.timer[p]) / float(c.cook_time);
    if (s.onions[p] == 3 && s.timer[p] == 0) o[17 * cells + cell] = 1.0f;
  }
  if (s.held[me] != kNone) o[(18 + s.held[me] - 1) * cells + s.pos[me]] = 1.0f;
  if (s.held[other] != kNone) o[(21 + s.held[other] - 1) * cells + s.pos[other]] = 1.0f;
  for (int k = 0; k < c.n_counters; ++k) {
    const int item = counter_get(s, k);
    if (item != kNone) o[(24 + item - 1) * cells + c.counter_cells[k]] = 1.0f;
  }
  o[kPlanes * cells] = float(s.t) / float(c.max_steps);
}

// Fill rows [r0, r1) of the tile (rows are (env, agent) pairs) from the template.
__device__ __forceinline__ void fill_rows(float* tile, const float* templ, int D, int nrows,
                                          const uint8_t* env_mask) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r = warp; r < nrows; r += nw) {
    if (env_mask && !env_mask[r >> 1]) continue;
    float* row = tile + size_t(r) * D;
    for (int k = lane; k < D; k += 32) row[k] = templ[k];
  }
}

struct Smem {
  float* templ;  // [D]
  float* tile;   // [kE][2][D]
  double* rew;   // [kE][2]
  double* inf;   // [kE][2][2]  deliveries, shaped_reward
  int32_t* act;  // [kE][2]
  uint8_t* done; // [kE][3]
  uint8_t* fin;  // [kE]
};

__host__ __device__ inline size_t a16(size_t b) { return (b + 15) & ~size_t(15); }
__host__ __device__ inline size_t smem_bytes(int D) {
  return a16(size_t(D) * 4) + a16(size_t(kE) * 2 * D * 4) + a16(kE * 2 * 8) + a16(kE * 4 * 8) +
         a16(kE * 2 * 4) + a16(kE * 3) + a16(kE);
}
__device__ __forceinline__ Smem carve(uint8_t* b, int D) {
  Smem m;
  size_t off = 0;
  m.templ = reinterpret_cast<float*>(b + off); off += a16(size_t(D) * 4);
  m.tile = reinterpret_cast<float*>(b + off); off += a16(size_t(kE) * 2 * D * 4);
  m.rew = reinterpret_cast<double*>(b + off); off += a16(kE * 2 * 8);
  m.inf = reinterpret_cast<double*>(b + off); off += a16(kE * 4 * 8);
  m.act = reinterpret_cast<int32_t*>(b + off); off += a16(kE * 2 * 4);
  m.done = b + off; off += a16(kE * 3);
  m.fin = b + off;
  return m;
}

__global__ void __launch_bounds__(kThreads) oc_reset_kernel(OcConfig c, const float* __restrict__ gtempl,
                                                            OcState st, LaunchCommon lc, Key key, Key carry_parent) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int D = kPlanes * c.h * c.w + 1;
  Smem m = carve(smem, D);
  for (int k = threadIdx.x; k < D; k += blockDim.x) m.templ[k] = gtempl[k];
  const int64_t i0 = int64_t(blockIdx.x) * kE;
  const int nvalid = int(min64(kE, lc.n - i0));
  __syncthreads();
  fill_rows(m.tile, m.templ, D, 2 * nvalid, nullptr);
  __syncthreads();
  if (threadIdx.x < nvalid) {
    const int64_t i = i0 + threadIdx.x;
    const uint64_t g = uint64_t(lc.offset + i);
    Kitchen s;
    env_reset(s, c);
    Key ck = split_child(carry_parent, g);  // vector_env.cpp:55; the reset key itself is unused
    (void)key;
    lc.carry.keys[i] = make_uint4(ck.k0, ck.k1, ck.c0, ck.c1);
    lc.carry.ep_return[i] = 0.0;
    lc.carry.ep_length[i] = 0;
    store(s, c, st, i, lc.n);
    for (int a = 0; a < 2; ++a) patch_row(m.tile + (size_t(threadIdx.x) * 2 + a) * D, s, c, a);
  }
  __syncthreads();
  block_store(lc.v.obs + i0 * 2 * D, m.tile, size_t(nvalid) * 2 * D * 4);
}

template <bool RANDOM>
__global__ void __launch_bounds__(kThreads) oc_step_kernel(OcConfig c, const float* __restrict__ gtempl,
                                                           OcState st, LaunchCommon lc, Key step_key) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (*(volatile int*)lc.err) return;
  const int D = kPlanes * c.h * c.w + 1;
  Smem m = carve(smem, D);
  for (int k = threadIdx.x; k < D; k += blockDim.x) m.templ[k] = gtempl[k];
  const int64_t i0 = int64_t(blockIdx.x) * kE;
  const int nvalid = int(min64(kE, lc.n - i0));
  const int tid = threadIdx.x;
  __syncthreads();
  fill_rows(m.tile, m.templ, D, 2 * nvalid, nullptr);

  Kitchen s;
  Key carry{0, 0, 0, 0};
  double ep_ret = 0.0;
  int ep_len = 0;
  bool done = false;
  const bool mine = tid < nvalid;
  const int64_t i = i0 + tid;
  if (mine) {
    uint4 kw = lc.carry.keys[i];
    carry = Key{kw.x, kw.y, kw.z, kw.w};
    ep_ret = lc.carry.ep_return[i];
    ep_len = lc.carry.ep_length[i];
    load(s, c, st, i, lc.n);
    int act[2];
    if (RANDOM) {  // all six actions always legal (env.hpp:71-73)
      Key ek = split_child(step_key, uint64_t(lc.offset + i));
      act[0] = int(block_at(ek, 0) % 6u);
      act[1] = int(block_at(ek, 1) % 6u);
      m.act[tid * 2] = act[0];
      m.act[tid * 2 + 1] = act[1];
    } else {
      act[0] = lc.v.actions[i * 2];
      act[1] = lc.v.actions[i * 2 + 1];
    }
    double reward, shaped[2];
    int deliveries;
    done = env_step(s, c, split_child(carry, 0), act, reward, shaped, deliveries);
    for (int a = 0; a < 2; ++a) {
      m.rew[tid * 2 + a] = reward;
      m.inf[(tid * 2 + a) * 2 + 0] = double(deliveries);  // Info keys in std::map order
      m.inf[(tid * 2 + a) * 2 + 1] = shaped[a];
      m.done[tid * 3 + a] = done;
    }
    m.done[tid * 3 + 2] = done;
    ep_ret = ep_ret + (reward + reward) / 2.0;  // team_reward, vector_env.cpp:14-18
    ep_len = ep_len + 1;
    lc.v.finished[i] = done;
    lc.v.final_returns[i] = done ? ep_ret : 0.0;
    lc.v.final_lengths[i] = done ? ep_len : 0;
  }
  if (tid < kE) m.fin[tid] = done;
  __syncthreads();  // template rows filled
  if (mine)
    for (int a = 0; a < 2; ++a) patch_row(m.tile + (size_t(tid) * 2 + a) * D, s, c, a);
  // episode stats: threads >= kE contribute nothing
  stats_add(lc.stats, done, ep_len, ep_ret);
  if (__syncthreads_or(done)) {
    // terminal rows of finished envs -> final_obs, then re-render reset rows
    for (int e = 0; e < nvalid; ++e) {
      if (!m.fin[e]) continue;
      float* src = m.tile + size_t(e) * 2 * D;
      float* dst = lc.v.final_obs + (i0 + e) * 2 * D;
      for (int k = tid; k < 2 * D; k += blockDim.x) __stcs(dst + k, src[k]);
    }
    __syncthreads();
    fill_rows(m.tile, m.templ, D, 2 * nvalid, m.fin);
    __syncthreads();
    if (done) {
      env_reset(s, c);
      ep_ret = 0.0;
      ep_len = 0;
      for (int a = 0; a < 2; ++a) patch_row(m.tile + (size_t(tid) * 2 + a) * D, s, c, a);
    }
  }
  if (mine) {
    Key nk = split_child(carry, 2);
    lc.carry.keys[i] = make_uint4(nk.k0, nk.k1, nk.c0, nk.c1);
    lc.carry.ep_return[i] = ep_ret;
    lc.carry.ep_length[i] = ep_len;
    store(s, c, st, i, lc.n);
  }
  __syncthreads();
  block_store(lc.v.obs + i0 * 2 * D, m.tile, size_t(nvalid) * 2 * D * 4);
  block_store(lc.v.rewards + i0 * 2, m.rew, size_t(nvalid) * 2 * 8);
  block_store(lc.v.infos + i0 * 4, m.inf, size_t(nvalid) * 4 * 8);
  block_store(lc.v.dones + i0 * 3, m.done, size_t(nvalid) * 3);
  if (RANDOM) block_store(lc.v.actions + i0 * 2, m.act, size_t(nvalid) * 2 * 4);
}

__global__ void oc_hash_kernel(OcConfig c, OcState st, int64_t n, uint64_t* out) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Kitchen s;
  load(s, c, st, i, n);
  uint64_t h = 1469598103934665603ull;  // overcooked.cpp:348-364
  auto mix = [&h](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  for (int a = 0; a < 2; ++a) {
    mix(uint64_t(s.pos[a]));
    mix(uint64_t(s.facing[a]));
    mix(uint64_t(s.held[a]));
  }
  for (int p = 0; p < c.n_pots; ++p) {
    mix(uint64_t(s.onions[p]));
    mix(uint64_t(s.timer[p]));
  }
  for (int k = 0; k < c.n_counters; ++k) mix(uint64_t(counter_get(s, k)));
  mix(uint64_t(s.t));
  out[i] = h;
}

Key to_key(KeyWords k) { return Key{k.w[0], k.w[1], k.w[2], k.w[3]}; }

}  // namespace

size_t oc_smem_bytes(const OcConfig& c) { return smem_bytes(kPlanes * c.h * c.w + 1); }

void oc_launch_reset_t(const OcConfig& c, const float* templ, const OcState& s, const LaunchCommon& lc,
                       KeyWords key, KeyWords carry_parent) {
  size_t sm = oc_smem_bytes(c);
  cudaFuncSetAttribute(oc_reset_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  unsigned g = unsigned((lc.n + kE - 1) / kE);
  oc_reset_kernel<<<g, kThreads, sm, lc.stream>>>(c, templ, s, lc, to_key(key), to_key(carry_parent));
  ++g_launches;
}

void oc_launch_step_t(const OcConfig& c, const float* templ, const OcState& s, const LaunchCommon& lc,
                      bool random, KeyWords step_key) {
  size_t sm = oc_smem_bytes(c);
  auto fn = random ? oc_step_kernel<true> : oc_step_kernel<false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  unsigned g = unsigned((lc.n + kE - 1) / kE);
  fn<<<g, kThreads, sm, lc.stream>>>(c, templ, s, lc, to_key(step_key));
  ++g_launches;
}

void oc_launch_hash(const OcConfig& c, const OcState& s, int64_t n, uint64_t* out, cudaStream_t st) {
  oc_hash_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(c, s, n, out);
  ++g_launches;
}

}  // namespace marl_b200
