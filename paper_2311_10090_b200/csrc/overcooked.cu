// Overcooked kitchens (reference: proj/core/src/envs/overcooked.cpp) as one
// fused sm_100a kernel per batch step.  The transition is a handful of integer
// ops per env; 97% of the bytes are the 27-plane observation rows
// (overcooked.cpp:395-427), so the kernel is organised around storing them at
// HBM speed:
//   * state update: one lane per env (a warp steps 32 envs in SIMT),
//   * observation: the warp streams the static layout template (planes
//     10-14 never change, the dynamic planes are zero in it) from shared
//     memory into its envs' contiguous [32][2][D] rows with 16-byte stores,
//     then every lane overwrites the ~20 dynamic cells of its own rows.
// All state is integer and trajectories are bit-identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {
namespace {

constexpr int kThreads = 256;    // 8 warps, one env per lane
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
// static planes come from the template already in the row.  CLEAR writes the
// template's 0 back into exactly the cells a patch of the same state set.
template <bool CLEAR = false>
__device__ __forceinline__ void patch_row(float* o, const Kitchen& s, const OcConfig& c, int me) {
  const int cells = c.h * c.w, other = 1 - me;
  const float one = CLEAR ? 0.0f : 1.0f;
  o[0 * cells + s.pos[me]] = one;
  o[1 * cells + s.pos[other]] = one;
  o[(2 + s.facing[me]) * cells + s.pos[me]] = one;
  o[(6 + s.facing[other]) * cells + s.pos[other]] = one;
  for (int p = 0; p < c.n_pots; ++p) {
    const int cell = c.pot_cells[p];
    o[15 * cells + cell] = CLEAR ? 0.0f : float(s.onions[p]);
    o[16 * cells + cell] = CLEAR ? 0.0f : float(s.timer[p]) / float(c.cook_time);
    if (s.onions[p] == 3 && s.timer[p] == 0) o[17 * cells + cell] = one;
  }
  if (s.held[me] != kNone) o[(18 + s.held[me] - 1) * cells + s.pos[me]] = one;
  if (s.held[other] != kNone) o[(21 + s.held[other] - 1) * cells + s.pos[other]] = one;
  for (int wd = 0; wd < 2; ++wd) {  // only the occupied counters: 2 bits per counter, 0 = empty
    const uint64_t w = s.counters[wd];
    for (uint64_t occ = (w | (w >> 1)) & 0x5555555555555555ull; occ; occ &= occ - 1) {
      const int bit = __ffsll((long long)occ) - 1;
      const int item = int((w >> bit) & 3u);
      o[(24 + item - 1) * cells + c.counter_cells[wd * 32 + (bit >> 1)]] = one;
    }
  }
  o[kPlanes * cells] = CLEAR ? 0.0f : float(s.t) / float(c.max_steps);
}

// The same cells as a list: emit(index in the row, value).  Used to build a
// per-env patch list that the whole warp then applies.
template <class F>
__device__ __forceinline__ void patch_cells(const Kitchen& s, const OcConfig& c, int me, F&& emit) {
  const int cells = c.h * c.w, other = 1 - me;
  emit(0 * cells + s.pos[me], 1.0f);
  emit(1 * cells + s.pos[other], 1.0f);
  emit((2 + s.facing[me]) * cells + s.pos[me], 1.0f);
  emit((6 + s.facing[other]) * cells + s.pos[other], 1.0f);
  for (int p = 0; p < c.n_pots; ++p) {
    const int cell = c.pot_cells[p];
    emit(15 * cells + cell, float(s.onions[p]));
    emit(16 * cells + cell, float(s.timer[p]) / float(c.cook_time));
    if (s.onions[p] == 3 && s.timer[p] == 0) emit(17 * cells + cell, 1.0f);
  }
  if (s.held[me] != kNone) emit((18 + s.held[me] - 1) * cells + s.pos[me], 1.0f);
  if (s.held[other] != kNone) emit((21 + s.held[other] - 1) * cells + s.pos[other], 1.0f);
  for (int wd = 0; wd < 2; ++wd) {
    const uint64_t w = s.counters[wd];
    for (uint64_t occ = (w | (w >> 1)) & 0x5555555555555555ull; occ; occ &= occ - 1) {
      const int bit = __ffsll((long long)occ) - 1;
      const int item = int((w >> bit) & 3u);
      emit((24 + item - 1) * cells + c.counter_cells[wd * 32 + (bit >> 1)], 1.0f);
    }
  }
  emit(kPlanes * cells, float(s.t) / float(c.max_steps));
}

// Upper bound of patch entries for one env (both rows).
__host__ __device__ inline int oc_max_patches(const OcConfig& c) { return 2 * (7 + 3 * c.n_pots + c.n_counters); }

// ------------------------------------------------------------ row streaming
// A warp's envs own a contiguous run of observation rows ([N][2][D] f32).
// The static planes of every row are identical (the layout template), so the
// warp streams the template straight from shared memory into the run with
// 16-byte stores, then each lane overwrites the ~20 dynamic cells of its own
// env's two rows (patch_row) after a __syncwarp (which orders the warp's
// global stores).  Nothing is staged per env: shared memory holds only the
// template, in four copies shifted by 0..3 floats so that any 4 consecutive
// template floats starting at any row offset are one aligned LDS.128.
struct Tmpl {
  const float* s[4];  // s[r][i] = templ[(i + r) % D]
  int D;
};

__host__ __device__ inline size_t tmpl_floats(int D) { return (size_t(D) + 3 + 3) & ~size_t(3); }

__device__ __forceinline__ Tmpl stage_template(float* smem, const float* __restrict__ g, int D) {
  const size_t stride = tmpl_floats(D);
  for (int idx = threadIdx.x; idx < 4 * int(stride); idx += blockDim.x) {
    const int r = idx / int(stride), i = idx - r * int(stride);
    smem[idx] = __ldg(g + (i + r) % D);
  }
  __syncthreads();
  Tmpl t;
  for (int r = 0; r < 4; ++r) t.s[r] = smem + r * stride;
  t.D = D;
  return t;
}

// dst: start of a run of whole rows (row offset 0), nfloats = rows * D.
__device__ __forceinline__ void stream_rows(float* __restrict__ dst, const Tmpl& t, int nfloats) {
  const int lane = threadIdx.x & 31, D = t.D;
  int head = int(((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) >> 2);
  head = head < nfloats ? head : nfloats;
  if (lane < head) dst[lane] = t.s[0][lane];
  const int nv = (nfloats - head) >> 2;
  float4* d4 = reinterpret_cast<float4*>(dst + head);
  int k = (head + 4 * lane) % D;  // row offset of this lane's first vector
#pragma unroll 4
  for (int q = lane; q < nv; q += 32) {
    const int r = k & 3;
    d4[q] = *reinterpret_cast<const float4*>(t.s[r] + (k - r));
    k += 128;
    while (k >= D) k -= D;
  }
  for (int q = head + 4 * nv + lane; q < nfloats; q += 32) dst[q] = t.s[0][q % D];
}

__global__ void __launch_bounds__(kThreads) oc_reset_kernel(OcConfig c, const float* __restrict__ gtempl,
                                                            OcState st, LaunchCommon lc, Key key, Key carry_parent) {
  extern __shared__ __align__(16) float smem[];
  const int D = kPlanes * c.h * c.w + 1;
  const Tmpl t = stage_template(smem, gtempl, D);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = int64_t(blockIdx.x) * kThreads + (threadIdx.x & ~31);
  if (w0 >= lc.n) return;  // warp-uniform
  const int wvalid = int(min64(32, lc.n - w0));
  const int64_t i = w0 + lane;
  stream_rows(lc.v.obs + w0 * 2 * D, t, wvalid * 2 * D);
  __syncwarp();
  if (lane < wvalid) {
    const uint64_t g = uint64_t(lc.offset + i);
    Kitchen s;
    env_reset(s, c);
    Key ck = split_child(carry_parent, g);  // vector_env.cpp:55; the reset key itself is unused
    (void)key;
    lc.carry.keys[i] = make_uint4(ck.k0, ck.k1, ck.c0, ck.c1);
    lc.carry.ep_return[i] = 0.0;
    lc.carry.ep_length[i] = 0;
    store(s, c, st, i, lc.n);
    for (int a = 0; a < 2; ++a) patch_row(lc.v.obs + (i * 2 + a) * D, s, c, a);
  }
}

// Observation rows through the async proxy: every warp owns two shared-memory
// buffers, each holding FOUR template rows (two envs; 16*D bytes, a multiple
// of 16 for any layout and 16-byte aligned in global memory at even envs).
// Per pair of envs the two owning lanes patch their rows into a buffer, one
// lane issues a single TMA bulk store (cp.async.bulk.global.shared::cta) of
// the whole 4-row run, and when the buffer comes round again the same lanes
// write the template's zeros back into exactly the cells they patched.  No
// row is ever copied through registers; the TMA engine streams 8.6 KB per
// instruction while the warp steps the next pair.
__host__ __device__ inline size_t oc_tma_smem_floats(int D, int warps, int max_patches) {
  return 4 * tmpl_floats(D) + size_t(warps) * (2 * 4 * D + 32 * 2 * size_t(max_patches) + 32);
}

template <bool RANDOM>
__global__ void __launch_bounds__(kThreads) oc_step_kernel(OcConfig c, const float* __restrict__ gtempl,
                                                           OcState st, LaunchCommon lc, Key step_key, int tma) {
  extern __shared__ __align__(16) float smem[];
  if (*(volatile int*)lc.err) return;
  const int D = kPlanes * c.h * c.w + 1;
  const Tmpl t = stage_template(smem, gtempl, D);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, warps = blockDim.x >> 5;
  const int MP = oc_max_patches(c);
  float* wbase = smem + 4 * tmpl_floats(D) + size_t(wid) * (2 * 4 * D + 32 * 2 * size_t(MP) + 32);
  float* bufs = wbase;                                               // 2 x [4 rows][D]
  uint32_t* p_idx = reinterpret_cast<uint32_t*>(wbase + 2 * 4 * D);  // [32][MP] row-relative cell (+ row * D)
  float* p_val = wbase + 2 * 4 * D + 32 * size_t(MP);               // [32][MP]
  int* p_n = reinterpret_cast<int*>(wbase + 2 * 4 * D + 64 * size_t(MP));  // [32]
  if (tma) {  // both buffers start as four template rows
    for (int idx = lane; idx < 2 * 4 * D; idx += 32) bufs[idx] = t.s[0][idx % D];
    __syncwarp();
  }
  const int64_t nchunks = (lc.end - lc.begin + 31) >> 5;  // begin is a multiple of 32
  for (int64_t chunk = int64_t(blockIdx.x) * warps + wid; chunk < nchunks; chunk += int64_t(gridDim.x) * warps) {
    const int64_t w0 = lc.begin + (chunk << 5);
    const int wvalid = int(min64(32, lc.end - w0));
    const int64_t i = w0 + lane;
    const bool mine = lane < wvalid;

    Kitchen s;
    Key carry{0, 0, 0, 0};
    double ep_ret = 0.0;
    int ep_len = 0;
    bool done = false;
    if (mine) {
      const uint4 kw = lc.carry.keys[i];
      carry = Key{kw.x, kw.y, kw.z, kw.w};
      ep_ret = lc.carry.ep_return[i];
      ep_len = lc.carry.ep_length[i];
      load(s, c, st, i, lc.n);
      int act[2];
      if (RANDOM) {  // all six actions always legal (env.hpp:71-73)
        const Key ek = split_child(step_key, uint64_t(lc.offset + i));
        act[0] = int(block_at(ek, 0) % 6u);
        act[1] = int(block_at(ek, 1) % 6u);
        *reinterpret_cast<int2*>(lc.v.actions + i * 2) = make_int2(act[0], act[1]);
      } else {
        act[0] = lc.v.actions[i * 2];  // caller buffer: only 4-byte alignment is guaranteed
        act[1] = lc.v.actions[i * 2 + 1];
      }
      double reward, shaped[2];
      int deliveries;
      done = env_step(s, c, split_child(carry, 0), act, reward, shaped, deliveries);
      *reinterpret_cast<double2*>(lc.v.rewards + i * 2) = make_double2(reward, reward);
      double2* inf = reinterpret_cast<double2*>(lc.v.infos + i * 4);  // Info keys in std::map order
      inf[0] = make_double2(double(deliveries), shaped[0]);
      inf[1] = make_double2(double(deliveries), shaped[1]);
      lc.v.dones[i * 3 + 0] = done;
      lc.v.dones[i * 3 + 1] = done;
      lc.v.dones[i * 3 + 2] = done;
      ep_ret = ep_ret + (reward + reward) / 2.0;  // team_reward, vector_env.cpp:14-18
      ep_len = ep_len + 1;
      lc.v.finished[i] = done;
      lc.v.final_returns[i] = done ? ep_ret : 0.0;
      lc.v.final_lengths[i] = done ? ep_len : 0;
    }
    stats_add(lc.stats, done, ep_len, ep_ret);

    // terminal observations of finished envs -> final_obs (rare: one env in
    // max_steps), then auto-reset (vector_env.cpp:107-119)
    const unsigned fin = __ballot_sync(0xffffffffu, done);
    if (fin) {
      for (unsigned m = fin; m; m &= m - 1) stream_rows(lc.v.final_obs + (w0 + __ffs(m) - 1) * 2 * D, t, 2 * D);
      __syncwarp();
      if (done) {
        for (int a = 0; a < 2; ++a) patch_row(lc.v.final_obs + (i * 2 + a) * D, s, c, a);
        env_reset(s, c);
        ep_ret = 0.0;
        ep_len = 0;
      }
    }

    // observation rows: every lane lists its env's dynamic cells (both rows,
    // index relative to the env's first row), then per pair of envs the whole
    // warp writes the two lists into a 4-row template buffer (and, two rounds
    // later, writes the template's zeros back), one lane issues the bulk store
    const int pairs = tma ? wvalid >> 1 : 0;
    if (pairs > 0) {
      if (mine) {
        int k = 0;
        for (int a = 0; a < 2; ++a)
          patch_cells(s, c, a, [&](int idx, float v) {
            p_idx[lane * MP + k] = uint32_t(a * D + idx);
            p_val[lane * MP + k] = v;
            ++k;
          });
        p_n[lane] = k;
      }
      __syncwarp();
    }
    for (int p = 0; p < pairs; ++p) {
      float* buf = bufs + (p & 1) * 4 * D;
      if (p >= 2) {  // the buffer's previous store must have read it; undo that pair's cells
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        for (int e2 = 0; e2 < 2; ++e2) {
          const int src = 2 * (p - 2) + e2;
          for (int q = lane; q < p_n[src]; q += 32) buf[e2 * 2 * D + p_idx[src * MP + q]] = 0.0f;
        }
        __syncwarp();
      }
      for (int e2 = 0; e2 < 2; ++e2) {
        const int src = 2 * p + e2;
        for (int q = lane; q < p_n[src]; q += 32) buf[e2 * 2 * D + p_idx[src * MP + q]] = p_val[src * MP + q];
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_store_s2g(lc.v.obs + (w0 + 2 * p) * 2 * D, buf, uint32_t(16 * D));
        bulk_commit();
      }
    }
    if (pairs > 0) {  // leave both buffers as clean template rows for the next chunk
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      for (int p = pairs >= 2 ? pairs - 2 : 0; p < pairs; ++p) {
        float* buf = bufs + (p & 1) * 4 * D;
        for (int e2 = 0; e2 < 2; ++e2) {
          const int src = 2 * p + e2;
          for (int q = lane; q < p_n[src]; q += 32) buf[e2 * 2 * D + p_idx[src * MP + q]] = 0.0f;
        }
      }
      __syncwarp();
    }
    const int direct0 = 2 * pairs;  // envs not covered by a bulk store (odd tail / no TMA)
    if (direct0 < wvalid) {
      stream_rows(lc.v.obs + (w0 + direct0) * 2 * D, t, (wvalid - direct0) * 2 * D);
      __syncwarp();
      if (mine && lane >= direct0)
        for (int a = 0; a < 2; ++a) patch_row(lc.v.obs + (i * 2 + a) * D, s, c, a);
    }
    if (mine) {
      const Key nk = split_child(carry, 2);  // vector_env.cpp:126
      lc.carry.keys[i] = make_uint4(nk.k0, nk.k1, nk.c0, nk.c1);
      lc.carry.ep_return[i] = ep_ret;
      lc.carry.ep_length[i] = ep_len;
      store(s, c, st, i, lc.n);
    }
  }
  if (tma && lane == 0) bulk_wait<0>();  // every bulk store has landed before the CTA retires
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

size_t oc_smem_bytes(const OcConfig& c) { return 4 * tmpl_floats(kPlanes * c.h * c.w + 1) * sizeof(float); }

void oc_launch_reset_t(const OcConfig& c, const float* templ, const OcState& s, const LaunchCommon& lc,
                       KeyWords key, KeyWords carry_parent) {
  size_t sm = oc_smem_bytes(c);
  smem_optin(oc_reset_kernel);
  unsigned g = unsigned((lc.n + kThreads - 1) / kThreads);
  oc_reset_kernel<<<g, kThreads, sm, lc.stream>>>(c, templ, s, lc, to_key(key), to_key(carry_parent));
  ++g_launches;
}

void oc_launch_step_t(const OcConfig& c, const float* templ, const OcState& s, const LaunchCommon& lc,
                      bool random, KeyWords step_key) {
  const int D = kPlanes * c.h * c.w + 1;
  // Persistent grid: as many 8-warp (or fewer, for large layouts) blocks as
  // fit on the device; TMA row buffers when they fit in shared memory.
  static int sms = 0, max_smem = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  int warps = kThreads / 32, tma = 1;
  const int mp = oc_max_patches(c);
  while (warps > 1 && oc_tma_smem_floats(D, warps, mp) * 4 > size_t(max_smem)) --warps;
  size_t sm = oc_tma_smem_floats(D, warps, mp) * 4;
  if (sm > size_t(max_smem)) {  // layout too large for the buffers: plain streaming stores
    tma = 0;
    warps = kThreads / 32;
    sm = oc_smem_bytes(c);
  }
  auto fn = random ? oc_step_kernel<true> : oc_step_kernel<false>;
  smem_optin(fn);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, warps * 32, sm);
  const int64_t chunks = (lc.end - lc.begin + 31) / 32;
  const int64_t want = (chunks + warps - 1) / warps;
  const int64_t cap = int64_t(std::max(per_sm, 1)) * sms;
  fn<<<unsigned(cap_grid(std::min(want, cap))), warps * 32, sm, lc.stream>>>(c, templ, s, lc, to_key(step_key), tma);
  ++g_launches;
}

void oc_launch_hash(const OcConfig& c, const OcState& s, int64_t n, uint64_t* out, cudaStream_t st) {
  oc_hash_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(c, s, n, out);
  ++g_launches;
}

}  // namespace marl_b200
