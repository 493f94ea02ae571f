// MPE particle worlds (reference: proj/core/src/envs/mpe.cpp) as one fused
// sm_100a kernel per batch step: random-action draw, physics, rewards, team
// return bookkeeping, auto-reset and observation rows -- the body of
// VectorEnv::step (vector_env.cpp:95-127) for every env in one launch.
//
// Layout: one thread owns one env; state is structure-of-arrays in HBM
// (component-major [c][N] doubles, so a warp's loads/stores of one component
// are a contiguous 256-byte run).  Observation / reward / done rows are built
// in shared memory and leave the SM as contiguous 16-byte vector stores.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {
namespace {

constexpr int kThreads = 128;
constexpr double kDt = 0.1, kDamping = 0.25, kContactForce = 1e2, kContactMargin = 1e-3,
                 kDefaultSens = 5.0;  // mpe.cpp:13-17
constexpr int kEpisodeSteps = 25;     // mpe.cpp:18

// Static entity tables of mpe.cpp:49-75, agents first, landmarks after.
template <int S>
struct Scen;

template <>
struct Scen<kMpeSpread> {
  static constexpr int A = 3, L = 3, E = 6, DC = 2, D = 18;
  MARL_HD static constexpr double size(int i) { return i < 3 ? 0.15 : 0.05; }
  MARL_HD static constexpr bool movable(int i) { return i < 3; }
  MARL_HD static constexpr bool collide(int i) { return i < 3; }
  MARL_HD static constexpr double accel(int) { return -1; }
  MARL_HD static constexpr double max_speed(int) { return -1; }
  MARL_HD static constexpr bool silent(int) { return true; }
  MARL_HD static constexpr bool adversary(int) { return false; }
  MARL_HD static constexpr int n_actions(int) { return 5; }
  MARL_HD static constexpr int obs_size(int) { return 18; }
};

template <>
struct Scen<kMpeSpeakerListener> {
  static constexpr int A = 2, L = 3, E = 5, DC = 3, D = 11;
  MARL_HD static constexpr double size(int i) { return i < 2 ? 0.075 : 0.04; }
  MARL_HD static constexpr bool movable(int i) { return i == 1; }
  MARL_HD static constexpr bool collide(int) { return false; }
  MARL_HD static constexpr double accel(int) { return -1; }
  MARL_HD static constexpr double max_speed(int) { return -1; }
  MARL_HD static constexpr bool silent(int i) { return i != 0; }
  MARL_HD static constexpr bool adversary(int) { return false; }
  MARL_HD static constexpr int n_actions(int i) { return i == 0 ? DC : 5; }
  MARL_HD static constexpr int obs_size(int i) { return i == 0 ? L : 2 + 2 * L + DC; }
};

template <>
struct Scen<kMpeTag> {
  static constexpr int A = 4, L = 2, E = 6, DC = 2, D = 16;
  MARL_HD static constexpr double size(int i) { return i < 3 ? 0.075 : (i == 3 ? 0.05 : 0.2); }
  MARL_HD static constexpr bool movable(int i) { return i < 4; }
  MARL_HD static constexpr bool collide(int) { return true; }
  MARL_HD static constexpr double accel(int i) { return i < 3 ? 3.0 : (i == 3 ? 4.0 : -1); }
  MARL_HD static constexpr double max_speed(int i) { return i < 3 ? 1.0 : (i == 3 ? 1.3 : -1); }
  MARL_HD static constexpr bool silent(int) { return true; }
  MARL_HD static constexpr bool adversary(int i) { return i < 3; }
  MARL_HD static constexpr int n_actions(int) { return 5; }
  MARL_HD static constexpr int obs_size(int i) { return i < 3 ? 16 : 14; }
};

template <class Sc>
struct Local {  // one env's MpeState (mpe.cpp:31-37) in registers
  double pos[2 * Sc::E];
  double vel[2 * Sc::A];
  double comm[Sc::A * Sc::DC];
  int steps;
  int goal;
};

// log(1 + e^z) (mpe.cpp:39-41).  Contacts are soft with margin 1e-3, so for
// all but touching agents z is hugely negative: e^z < 2^-60 makes log1p(e^z)
// round to e^z itself (the next series term is below half an ulp), and below
// -745 e^z is 0 -- the libm calls are skipped with the same result.
__device__ __forceinline__ double log1p_exp_neg(double z) {  // z <= 0
  if (z < -746.0) return 0.0;
  const double t = exp(z);
  return t < 0x1p-60 ? t : log1p(t);
}
__device__ __forceinline__ double logaddexp0(double z) {
  return z > 0 ? z + log1p_exp_neg(-z) : log1p_exp_neg(z);
}

template <class Sc>
__device__ __forceinline__ double lm(const Local<Sc>& s, int j, int axis) {  // mpe.cpp:287-289
  return s.pos[2 * (Sc::A + j) + axis];
}

// MpeEnv::reset body (mpe.cpp:107-124) from the env's reset key.
template <class Sc, int S>
__device__ __forceinline__ void env_reset(Local<Sc>& s, const Key& key) {
#pragma unroll
  for (int i = 0; i < Sc::E; ++i) {
    Key kid = split_child(key, uint64_t(i));
    double lim = i < Sc::A ? 1.0 : 0.9;
    s.pos[2 * i] = uniform_at(kid, 0, -lim, lim);
    s.pos[2 * i + 1] = uniform_at(kid, 1, -lim, lim);
  }
#pragma unroll
  for (int q = 0; q < 2 * Sc::A; ++q) s.vel[q] = 0.0;
#pragma unroll
  for (int q = 0; q < Sc::A * Sc::DC; ++q) s.comm[q] = 0.0;
  s.steps = 0;
  s.goal = -1;
  if (S == kMpeSpeakerListener) {
    Key kid = split_child(key, uint64_t(Sc::E));
    s.goal = int(block_at(kid, 0) % uint64_t(Sc::L));  // randint1(kid, 0, L), prng.cpp:182-190
  }
}

// observe (mpe.cpp:291-334) for agent i into a zero-padded row of D floats.
template <class Sc, int S>
__device__ __forceinline__ void observe(const Local<Sc>& s, int i, float* o) {
  int k = 0;
  if (S == kMpeSpeakerListener && i == 0) {
#pragma unroll
    for (int j = 0; j < Sc::L; ++j) o[k++] = j == s.goal ? 1.0f : 0.0f;
  } else if (S == kMpeSpeakerListener) {
    o[k++] = float(s.vel[2 * i]);
    o[k++] = float(s.vel[2 * i + 1]);
#pragma unroll
    for (int j = 0; j < Sc::L; ++j) {
      o[k++] = float(lm(s, j, 0) - s.pos[2 * i]);
      o[k++] = float(lm(s, j, 1) - s.pos[2 * i + 1]);
    }
#pragma unroll
    for (int c = 0; c < Sc::DC; ++c) o[k++] = float(s.comm[c]);
  } else {
    o[k++] = float(s.vel[2 * i]);
    o[k++] = float(s.vel[2 * i + 1]);
    o[k++] = float(s.pos[2 * i]);
    o[k++] = float(s.pos[2 * i + 1]);
#pragma unroll
    for (int j = 0; j < Sc::L; ++j) {
      o[k++] = float(lm(s, j, 0) - s.pos[2 * i]);
      o[k++] = float(lm(s, j, 1) - s.pos[2 * i + 1]);
    }
#pragma unroll
    for (int j = 0; j < Sc::A; ++j) {
      if (j == i) continue;
      o[k++] = float(s.pos[2 * j] - s.pos[2 * i]);
      o[k++] = float(s.pos[2 * j + 1] - s.pos[2 * i + 1]);
    }
    if (S == kMpeSpread) {
#pragma unroll
      for (int j = 0; j < Sc::A; ++j) {
        if (j == i) continue;
#pragma unroll
        for (int c = 0; c < Sc::DC; ++c) o[k++] = float(s.comm[j * Sc::DC + c]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < Sc::A; ++j) {
        if (j == i || Sc::adversary(j)) continue;
        o[k++] = float(s.vel[2 * j]);
        o[k++] = float(s.vel[2 * j + 1]);
      }
    }
  }
  for (; k < Sc::D; ++k) o[k] = 0.0f;
}

template <class Sc>
__device__ __forceinline__ bool collides(const Local<Sc>& s, int a, int b) {  // mpe.cpp:342-346
  double dx = s.pos[2 * a] - s.pos[2 * b];
  double dy = s.pos[2 * a + 1] - s.pos[2 * b + 1];
  return sqrt(dx * dx + dy * dy) < Sc::size(a) + Sc::size(b);
}

__device__ __forceinline__ double bound_penalty(double x) {  // mpe.cpp:348-352
  if (x < 0.9) return 0.0;
  if (x < 1.0) return (x - 0.9) * 10.0;
  double e = exp(2.0 * x - 2.0);
  return 10.0 < e ? 10.0 : e;
}

// simple_spread's landmark-coverage term of reward() (mpe.cpp:357-365): the
// same value for every agent, so it is evaluated once per step.
template <class Sc>
__device__ __forceinline__ double spread_cover(const Local<Sc>& s) {
  double rew = 0.0;
#pragma unroll
  for (int j = 0; j < Sc::L; ++j) {
    double best = 1e18;
#pragma unroll
    for (int a = 0; a < Sc::A; ++a) {
      double dx = s.pos[2 * a] - lm(s, j, 0);
      double dy = s.pos[2 * a + 1] - lm(s, j, 1);
      double d = sqrt(dx * dx + dy * dy);
      best = d < best ? d : best;
    }
    rew -= best;
  }
  return rew;
}

// cover: spread_cover(s) for simple_spread (unused otherwise)
template <class Sc, int S>
__device__ __forceinline__ double reward(const Local<Sc>& s, int i, bool coop_prey, double cover) {  // mpe.cpp:354-384
  if (S == kMpeSpread) {
    double rew = cover;
#pragma unroll
    for (int a = 0; a < Sc::A; ++a)
      if (a != i && collides(s, a, i)) rew -= 1.0;
    return rew;
  }
  if (S == kMpeSpeakerListener) {
    double dx = s.pos[2] - s.pos[2 * (Sc::A + s.goal)];
    double dy = s.pos[3] - s.pos[2 * (Sc::A + s.goal) + 1];
    return -(dx * dx + dy * dy);
  }
  double touches = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (collides(s, a, 3)) touches += 1.0;
  if (coop_prey || Sc::adversary(i)) return 10.0 * touches;
  double rew = -10.0 * touches;
  rew -= bound_penalty(fabs(s.pos[2 * i]));
  rew -= bound_penalty(fabs(s.pos[2 * i + 1]));
  return rew;
}

// MpeEnv::step physics (mpe.cpp:137-214), in place.  CONT: box actions, the
// agent's row of kBoxActDim floats (u = (v1 - v2, v3 - v4), comm = v[0:dim_c],
// mpe.cpp:144-166); else discrete ids.
template <class Sc, bool CONT>
__device__ __forceinline__ void physics(Local<Sc>& s, const int* act, const float* actf) {
  double force[2 * Sc::E];
#pragma unroll
  for (int q = 0; q < 2 * Sc::E; ++q) force[q] = 0.0;
#pragma unroll
  for (int i = 0; i < Sc::A; ++i) {
    if (Sc::movable(i)) {
      double u0 = 0.0, u1 = 0.0;
      if (CONT) {
        const float* v = actf + i * kBoxActDim;
        u0 = double(v[1]) - double(v[2]);
        u1 = double(v[3]) - double(v[4]);
      } else {
        int a = act[i];
        if (a == 1) u0 = -1.0;
        if (a == 2) u0 = +1.0;
        if (a == 3) u1 = -1.0;
        if (a == 4) u1 = +1.0;
      }
      constexpr double dflt = kDefaultSens;
      double sens = Sc::accel(i) > 0 ? Sc::accel(i) : dflt;
      force[2 * i] += u0 * sens;
      force[2 * i + 1] += u1 * sens;
    }
    if (!Sc::silent(i)) {
#pragma unroll
      for (int c = 0; c < Sc::DC; ++c)
        s.comm[i * Sc::DC + c] = CONT ? double(actf[i * kBoxActDim + c]) : (c == act[i] ? 1.0 : 0.0);
    }
  }
#pragma unroll
  for (int a = 0; a < Sc::E; ++a) {
#pragma unroll
    for (int b = a + 1; b < Sc::E; ++b) {
      if (!Sc::collide(a) || !Sc::collide(b)) continue;
      double dx = s.pos[2 * a] - s.pos[2 * b];
      double dy = s.pos[2 * a + 1] - s.pos[2 * b + 1];
      double dist = sqrt(dx * dx + dy * dy);
      if (dist < 1e-9) dist = 1e-9;
      double dist_min = Sc::size(a) + Sc::size(b);
      double pen = logaddexp0(-(dist - dist_min) / kContactMargin) * kContactMargin;
      double fx = kContactForce * dx / dist * pen;
      double fy = kContactForce * dy / dist * pen;
      if (Sc::movable(a)) {
        force[2 * a] += fx;
        force[2 * a + 1] += fy;
      }
      if (Sc::movable(b)) {
        force[2 * b] -= fx;
        force[2 * b + 1] -= fy;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < Sc::A; ++i) {
    if (!Sc::movable(i)) continue;
    double v0 = s.vel[2 * i] * (1.0 - kDamping);
    double v1 = s.vel[2 * i + 1] * (1.0 - kDamping);
    v0 += force[2 * i] * kDt;
    v1 += force[2 * i + 1] * kDt;
    if (Sc::max_speed(i) > 0) {
      double speed = sqrt(v0 * v0 + v1 * v1);
      if (speed > Sc::max_speed(i)) {
        v0 = v0 / speed * Sc::max_speed(i);
        v1 = v1 / speed * Sc::max_speed(i);
      }
    }
    s.vel[2 * i] = v0;
    s.vel[2 * i + 1] = v1;
    s.pos[2 * i] += v0 * kDt;
    s.pos[2 * i + 1] += v1 * kDt;
  }
  s.steps += 1;
}

template <class Sc, int S>
__device__ __forceinline__ void load_state(Local<Sc>& s, const MpeState& st, int64_t i, int64_t n) {
#pragma unroll
  for (int q = 0; q < 2 * Sc::E; ++q) s.pos[q] = st.pos[q * n + i];
#pragma unroll
  for (int q = 0; q < 2 * Sc::A; ++q) s.vel[q] = st.vel[q * n + i];
#pragma unroll
  for (int q = 0; q < Sc::A * Sc::DC; ++q) s.comm[q] = (S == kMpeSpeakerListener) ? st.comm[q * n + i] : 0.0;
  s.steps = st.steps[i];
  s.goal = (S == kMpeSpeakerListener) ? st.goal[i] : -1;
}

// Landmarks never move (mpe.cpp:194): their slots are only rewritten on reset.
template <class Sc, int S>
__device__ __forceinline__ void store_state(const Local<Sc>& s, const MpeState& st, int64_t i, int64_t n,
                                            bool landmarks) {
#pragma unroll
  for (int q = 0; q < 2 * Sc::E; ++q)
    if (q < 2 * Sc::A || landmarks) st.pos[q * n + i] = s.pos[q];
#pragma unroll
  for (int q = 0; q < 2 * Sc::A; ++q) st.vel[q * n + i] = s.vel[q];
  if (S == kMpeSpeakerListener) {
#pragma unroll
    for (int q = 0; q < Sc::A * Sc::DC; ++q) st.comm[q * n + i] = s.comm[q];
    st.goal[i] = s.goal;
  }
  st.steps[i] = s.steps;
}

template <int S>
__global__ void __launch_bounds__(kThreads) mpe_reset_kernel(MpeState st, LaunchCommon lc, Key key,
                                                             Key carry_parent) {
  using Sc = Scen<S>;
  constexpr int ROW = Sc::A * Sc::D;
  __shared__ __align__(16) float s_obs[kThreads * ROW];
  const int64_t i0 = int64_t(blockIdx.x) * kThreads;
  const int64_t i = i0 + threadIdx.x;
  const int nvalid = int(min64(kThreads, lc.n - i0));
  if (i < lc.n) {
    const uint64_t g = uint64_t(lc.offset + i);
    Local<Sc> s;
    env_reset<Sc, S>(s, split_child(key, g));  // vector_env.cpp:52,57
    Key c = split_child(carry_parent, g);       // vector_env.cpp:55
    lc.carry.keys[i] = make_uint4(c.k0, c.k1, c.c0, c.c1);
    lc.carry.ep_return[i] = 0.0;
    lc.carry.ep_length[i] = 0;
    store_state<Sc, S>(s, st, i, lc.n, true);
#pragma unroll
    for (int a = 0; a < Sc::A; ++a) observe<Sc, S>(s, a, s_obs + threadIdx.x * ROW + a * Sc::D);
  }
  __syncthreads();
  block_store(lc.v.obs + i0 * ROW, s_obs, size_t(nvalid) * ROW * sizeof(float));
}

template <int S, bool RANDOM, bool CONT>
__global__ void __launch_bounds__(kThreads) mpe_step_kernel(MpeState st, LaunchCommon lc, Key step_key,
                                                            int coop_prey) {
  using Sc = Scen<S>;
  constexpr int A = Sc::A, ROW = A * Sc::D;
  __shared__ __align__(16) float s_obs[kThreads * ROW];
  __shared__ __align__(16) double s_rew[kThreads * A];
  __shared__ __align__(16) int32_t s_act[kThreads * A];
  __shared__ __align__(16) uint8_t s_done[kThreads * (A + 1)];
  __shared__ uint8_t s_fin[kThreads];
  if (*(volatile int*)lc.err) return;  // a pending contract error freezes the batch

  const int64_t i0 = lc.begin + int64_t(blockIdx.x) * kThreads;
  const int64_t i = i0 + threadIdx.x;
  const int nvalid = int(min64(kThreads, lc.end - i0));
  const bool live = i < lc.end;
  float* my_obs = s_obs + threadIdx.x * ROW;

  Local<Sc> s;
  Key carry{0, 0, 0, 0};
  double ep_ret = 0.0;
  int ep_len = 0;
  bool done = false;
  if (live) {
    uint4 kw = lc.carry.keys[i];
    carry = Key{kw.x, kw.y, kw.z, kw.w};
    ep_ret = lc.carry.ep_return[i];
    ep_len = lc.carry.ep_length[i];
    load_state<Sc, S>(s, st, i, lc.n);

    int act[A];
    float actf[CONT ? A * kBoxActDim : 1];
    if (RANDOM && CONT) {
      // box spaces: space.sample(fold_in(env_key, j)) = float(uniform(key, flat, 0, 1))
      // (vector_env.cpp:179-181, spaces.cpp:48-54)
      Key ek = split_child(step_key, uint64_t(lc.offset + i));
#pragma unroll
      for (int j = 0; j < A; ++j) {
        const Key kj = fold_in(ek, uint64_t(j));
#pragma unroll
        for (int k = 0; k < kBoxActDim; ++k)
          actf[j * kBoxActDim + k] = k < Sc::n_actions(j) ? float(uniform_at(kj, uint64_t(k), 0.0, 1.0)) : 0.0f;
      }
      float4* dst = reinterpret_cast<float4*>(lc.v.actions_f + i * A * kBoxActDim);
      if ((A * kBoxActDim) % 4 == 0) {
#pragma unroll
        for (int q = 0; q < A * kBoxActDim / 4; ++q)
          dst[q] = make_float4(actf[4 * q], actf[4 * q + 1], actf[4 * q + 2], actf[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < A * kBoxActDim; ++q) lc.v.actions_f[i * A * kBoxActDim + q] = actf[q];
      }
    } else if (CONT) {
#pragma unroll
      for (int q = 0; q < A * kBoxActDim; ++q) actf[q] = lc.v.actions_f[i * A * kBoxActDim + q];
    } else if (RANDOM) {
      // random_legal_actions (vector_env.cpp:169-187); MPE masks are all-legal
      // (env.hpp:71-73) so the draw is bits(env_key, j) % n_actions.
      Key ek = split_child(step_key, uint64_t(lc.offset + i));
#pragma unroll
      for (int j = 0; j < A; ++j) {
        act[j] = int(block_at(ek, uint64_t(j)) % uint64_t(Sc::n_actions(j)));
        s_act[threadIdx.x * A + j] = act[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < A; ++j) act[j] = lc.v.actions[i * A + j];
    }

    physics<Sc, CONT>(s, act, actf);
    done = s.steps >= kEpisodeSteps;
    double sum = 0.0;
    const double cover = S == kMpeSpread ? spread_cover(s) : 0.0;
#pragma unroll
    for (int j = 0; j < A; ++j) {
      double r = reward<Sc, S>(s, j, coop_prey != 0, cover);
      s_rew[threadIdx.x * A + j] = r;
      sum += r;
      s_done[threadIdx.x * (A + 1) + j] = done;
    }
    s_done[threadIdx.x * (A + 1) + A] = done;
    ep_ret = ep_ret + sum / double(A);  // team_reward, vector_env.cpp:14-18,99
    ep_len = ep_len + 1;
#pragma unroll
    for (int a = 0; a < A; ++a) observe<Sc, S>(s, a, my_obs + a * Sc::D);
    lc.v.finished[i] = done;
    lc.v.final_returns[i] = done ? ep_ret : 0.0;
    lc.v.final_lengths[i] = done ? ep_len : 0;
  }
  s_fin[threadIdx.x] = done;
  stats_add(lc.stats, done, ep_len, ep_ret);

  // Terminal observations leave as whole rows before auto-reset overwrites them.
  if (__syncthreads_or(done)) {
    for (int idx = threadIdx.x; idx < nvalid * ROW; idx += kThreads) {
      int r = idx / ROW;
      if (s_fin[r]) __stcs(lc.v.final_obs + i0 * ROW + idx, s_obs[idx]);
    }
    __syncthreads();
    if (done) {  // vector_env.cpp:107-119: reset with the auto-reset child key
      env_reset<Sc, S>(s, split_child(carry, 1));
#pragma unroll
      for (int a = 0; a < A; ++a) observe<Sc, S>(s, a, my_obs + a * Sc::D);
      ep_ret = 0.0;
      ep_len = 0;
    }
  }
  if (live) {
    Key nk = split_child(carry, 2);  // vector_env.cpp:126
    lc.carry.keys[i] = make_uint4(nk.k0, nk.k1, nk.c0, nk.c1);
    lc.carry.ep_return[i] = ep_ret;
    lc.carry.ep_length[i] = ep_len;
    store_state<Sc, S>(s, st, i, lc.n, done);
  }
  // the block's rows leave as TMA bulk stores (one instruction per tile)
  bulk_tile_fence();
  tile_store(lc.v.obs + i0 * ROW, s_obs, size_t(nvalid) * ROW * sizeof(float));
  tile_store(lc.v.rewards + i0 * A, s_rew, size_t(nvalid) * A * sizeof(double));
  tile_store(lc.v.dones + i0 * (A + 1), s_done, size_t(nvalid) * (A + 1));
  if (RANDOM && !CONT) tile_store(lc.v.actions + i0 * A, s_act, size_t(nvalid) * A * sizeof(int32_t));
  tile_store_drain();
}

// Named CTA barriers (ids 1..4; 0 is __syncthreads) between the two warps of
// the probe kernel: a producer arrives, a consumer waits.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// K consecutive iterations of throughput_probe's loop (vector_env.cpp:202-217)
// in ONE launch: step k's action key is split(parent, t0 + k) (parent =
// fold_in(key, 2)), derived in-kernel; the env's state, carry key and episode
// bookkeeping stay on chip across the K steps.  Every step still writes every
// output view (obs, rewards, dones, actions, finished, final_*), so after the
// launch the views hold step t0 + K - 1's outputs exactly as K separate
// mpe_step_kernel launches leave them.
//
// Small batches (configs[0]: 1024 envs) are latency-bound -- one env's step
// is a dependent chain of Threefry blocks and fp64 sqrt / div / exp -- so the
// step is split over a three-warp pipeline per 32 envs (one env per lane in
// each warp), handing data on through double-buffered shared-memory slots
// guarded by named barriers:
//   KEY  warp, one step ahead: the action draw of random_legal_actions, the
//        carry chain split(carry, 2) and, when the step ends an episode (MPE
//        episodes are exactly 25 steps, so the key warp knows), the
//        auto-reset state from split(carry, 1);
//   SIM  warp: the only true recurrence, physics (mpe.cpp:137-214);
//   POST warp, one step behind: rewards, dones, episode bookkeeping,
//        statistics and every output row (terminal rows before the reset).
// Rows leave straight from registers (no staging).
template <int S, bool CONT>
__global__ void __launch_bounds__(96) mpe_probe_kernel(MpeState st, LaunchCommon lc, Key parent, int coop_prey,
                                                       uint64_t t0, int K) {
  using Sc = Scen<S>;
  constexpr int A = Sc::A, D = Sc::D, ROW = A * D, NAF = CONT ? A * kBoxActDim : 1, NP = 2 * Sc::E,
                NV = 2 * Sc::A, NC = Sc::A * Sc::DC;
  struct KeySlot {  // KEY -> SIM
    float actf[NAF][32];
    int32_t act[A][32];
    double rpos[NP][32];
    int32_t rgoal[32];
    uint32_t done;  // bit lane: the step ends lane's episode
  };
  struct SimSlot {  // SIM -> POST: the post-physics state (+ the reset state when done)
    double pos[NP][32], vel[NV][32], comm[NC][32], rpos[NP][32];
    int32_t goal[32], rgoal[32];
    uint32_t done;
  };
  __shared__ KeySlot kslot[2];
  __shared__ SimSlot sslot[2];
  if (*(volatile int*)lc.err) return;  // a pending contract error freezes the batch
  const int lane = threadIdx.x & 31, role = threadIdx.x >> 5;  // 0 SIM, 1 KEY, 2 POST
  const int64_t i = lc.begin + int64_t(blockIdx.x) * 32 + lane;
  const bool live = i < lc.end;
  // barrier ids: KEY->SIM full 1+b / empty 3+b, SIM->POST full 5+b / empty 7+b

  if (role == 1) {  // ------------------------------------------------ KEY
    Key carry{0, 0, 0, 0};
    int steps = 0;
    if (live) {
      const uint4 kw = lc.carry.keys[i];
      carry = Key{kw.x, kw.y, kw.z, kw.w};
      steps = st.steps[i];
    }
    for (int k = 0; k < K; ++k) {
      const int b = k & 1;
      if (k >= 2) nbar_sync(3 + b, 64);  // SIM has consumed step k - 2's slot
      KeySlot& sl = kslot[b];
      bool done = false;
      if (live) {
        const Key ek = split_child(split_child(parent, t0 + uint64_t(k)), uint64_t(lc.offset + i));
        if (CONT) {  // space.sample(fold_in(env_key, j)) (vector_env.cpp:179-181, spaces.cpp:48-54)
#pragma unroll
          for (int j = 0; j < A; ++j) {
            const Key kj = fold_in(ek, uint64_t(j));
#pragma unroll
            for (int q = 0; q < kBoxActDim; ++q) {
              const float v = q < Sc::n_actions(j) ? float(uniform_at(kj, uint64_t(q), 0.0, 1.0)) : 0.0f;
              sl.actf[j * kBoxActDim + q][lane] = v;
              lc.v.actions_f[i * A * kBoxActDim + j * kBoxActDim + q] = v;
            }
          }
        } else {  // random_legal_actions with all-legal masks (vector_env.cpp:169-187, env.hpp:71-73)
#pragma unroll
          for (int j = 0; j < A; ++j) {
            const int a = int(mod_small(block_at(ek, uint64_t(j)), uint32_t(Sc::n_actions(j))));
            sl.act[j][lane] = a;
            lc.v.actions[i * A + j] = a;
          }
        }
        steps += 1;
        done = steps >= kEpisodeSteps;
        if (done) {  // env->reset(split(carry, 3)[1]) (vector_env.cpp:107-119)
          Local<Sc> r;
          env_reset<Sc, S>(r, split_child(carry, 1));
#pragma unroll
          for (int q = 0; q < NP; ++q) sl.rpos[q][lane] = r.pos[q];
          sl.rgoal[lane] = r.goal;
          steps = 0;
        }
        carry = split_child(carry, 2);  // vector_env.cpp:126
      }
      const unsigned dm = __ballot_sync(0xffffffffu, done);
      if (lane == 0) sl.done = dm;
      nbar_arrive(1 + b, 64);  // slot b holds step k
    }
    if (live) lc.carry.keys[i] = make_uint4(carry.k0, carry.k1, carry.c0, carry.c1);
    return;
  }

  if (role == 0) {  // ------------------------------------------------ SIM
    Local<Sc> s;
    if (live) load_state<Sc, S>(s, st, i, lc.n);
    bool any_reset = false;
    for (int k = 0; k < K; ++k) {
      const int b = k & 1;
      nbar_sync(1 + b, 64);  // KEY's slot b holds step k
      const KeySlot& kl = kslot[b];
      int act[A];
      float actf[NAF];
      if (CONT) {
#pragma unroll
        for (int q = 0; q < NAF; ++q) actf[q] = kl.actf[q][lane];
      } else {
#pragma unroll
        for (int j = 0; j < A; ++j) act[j] = kl.act[j][lane];
      }
      const unsigned dm = kl.done;
      const bool done = (dm >> lane) & 1u;
      double rpos[NP];
      int rgoal = -1;
      if (done) {
#pragma unroll
        for (int q = 0; q < NP; ++q) rpos[q] = kl.rpos[q][lane];
        rgoal = kl.rgoal[lane];
      }
      if (k + 2 < K) nbar_arrive(3 + b, 64);  // KEY may refill slot b (step k + 2)
      if (live) physics<Sc, CONT>(s, act, actf);
      if (k >= 2) nbar_sync(7 + b, 64);  // POST has consumed step k - 2's slot
      SimSlot& sl = sslot[b];
      if (live) {
#pragma unroll
        for (int q = 0; q < NP; ++q) sl.pos[q][lane] = s.pos[q];
#pragma unroll
        for (int q = 0; q < NV; ++q) sl.vel[q][lane] = s.vel[q];
#pragma unroll
        for (int q = 0; q < NC; ++q) sl.comm[q][lane] = s.comm[q];
        sl.goal[lane] = s.goal;
        if (done) {
#pragma unroll
          for (int q = 0; q < NP; ++q) sl.rpos[q][lane] = rpos[q];
          sl.rgoal[lane] = rgoal;
        }
      }
      if (lane == 0) sl.done = dm;
      nbar_arrive(5 + b, 64);  // slot b holds step k's state
      if (live && done) {  // the auto-reset state (vector_env.cpp:107-119)
#pragma unroll
        for (int q = 0; q < NP; ++q) s.pos[q] = rpos[q];
#pragma unroll
        for (int q = 0; q < NV; ++q) s.vel[q] = 0.0;
#pragma unroll
        for (int q = 0; q < NC; ++q) s.comm[q] = 0.0;
        s.steps = 0;
        s.goal = rgoal;
        any_reset = true;
      }
    }
    if (live) store_state<Sc, S>(s, st, i, lc.n, any_reset);
    return;
  }

  // ---------------------------------------------------------------- POST
  double ep_ret = 0.0;
  int ep_len = 0;
  if (live) {
    ep_ret = lc.carry.ep_return[i];
    ep_len = lc.carry.ep_length[i];
  }
  static_assert(ROW % 2 == 0, "observation rows are stored as float2");
  auto put_rows = [&](float* dst, const Local<Sc>& cs) {
    float row[ROW];
#pragma unroll
    for (int a = 0; a < A; ++a) observe<Sc, S>(cs, a, row + a * D);
    float2* d2 = reinterpret_cast<float2*>(dst + i * ROW);
#pragma unroll
    for (int q = 0; q < ROW / 2; ++q) d2[q] = make_float2(row[2 * q], row[2 * q + 1]);
  };
  for (int k = 0; k < K; ++k) {
    const int b = k & 1;
    nbar_sync(5 + b, 64);  // SIM's slot b holds step k's state
    const SimSlot& sl = sslot[b];
    const bool done = (sl.done >> lane) & 1u;
    Local<Sc> s;
    double rpos[NP];
    int rgoal = -1;
    if (live) {
#pragma unroll
      for (int q = 0; q < NP; ++q) s.pos[q] = sl.pos[q][lane];
#pragma unroll
      for (int q = 0; q < NV; ++q) s.vel[q] = sl.vel[q][lane];
#pragma unroll
      for (int q = 0; q < NC; ++q) s.comm[q] = sl.comm[q][lane];
      s.goal = sl.goal[lane];
      if (done) {
#pragma unroll
        for (int q = 0; q < NP; ++q) rpos[q] = sl.rpos[q][lane];
        rgoal = sl.rgoal[lane];
      }
    }
    if (k + 2 < K) nbar_arrive(7 + b, 64);  // SIM may refill slot b (step k + 2)
    if (live) {
      double sum = 0.0;
      const double cover = S == kMpeSpread ? spread_cover(s) : 0.0;
#pragma unroll
      for (int j = 0; j < A; ++j) {
        const double r = reward<Sc, S>(s, j, coop_prey != 0, cover);
        lc.v.rewards[i * A + j] = r;
        sum += r;
        lc.v.dones[i * (A + 1) + j] = done;
      }
      lc.v.dones[i * (A + 1) + A] = done;
      ep_ret = ep_ret + sum / double(A);  // team_reward, vector_env.cpp:14-18,99
      ep_len = ep_len + 1;
      lc.v.finished[i] = done;
      lc.v.final_returns[i] = done ? ep_ret : 0.0;
      lc.v.final_lengths[i] = done ? ep_len : 0;
    }
    stats_add(lc.stats, done, ep_len, ep_ret);
    if (live) {
      if (done) {  // terminal rows, then the reset state's rows
        put_rows(lc.v.final_obs, s);
#pragma unroll
        for (int q = 0; q < NP; ++q) s.pos[q] = rpos[q];
#pragma unroll
        for (int q = 0; q < NV; ++q) s.vel[q] = 0.0;
#pragma unroll
        for (int q = 0; q < NC; ++q) s.comm[q] = 0.0;
        s.goal = rgoal;
        ep_ret = 0.0;
        ep_len = 0;
      }
      put_rows(lc.v.obs, s);
    }
  }
  if (live) {
    lc.carry.ep_return[i] = ep_ret;
    lc.carry.ep_length[i] = ep_len;
  }
}

// state_hash (mpe.cpp:254-269), parity aid.
template <int S>
__global__ void mpe_hash_kernel(MpeState st, int64_t n, uint64_t* out) {
  using Sc = Scen<S>;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Local<Sc> s;
  load_state<Sc, S>(s, st, i, n);
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
#pragma unroll
  for (int q = 0; q < 2 * Sc::E; ++q) mix(__double_as_longlong(s.pos[q]));
#pragma unroll
  for (int q = 0; q < 2 * Sc::A; ++q) mix(__double_as_longlong(s.vel[q]));
#pragma unroll
  for (int q = 0; q < Sc::A * Sc::DC; ++q) mix(__double_as_longlong(s.comm[q]));
  mix(uint64_t(s.steps));
  mix(uint64_t(int64_t(s.goal)));
  out[i] = h;
}

Key to_key(KeyWords k) { return Key{k.w[0], k.w[1], k.w[2], k.w[3]}; }
unsigned grid_for(int64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

int mpe_n_agents(int s) {
  return s == kMpeSpread ? Scen<kMpeSpread>::A : s == kMpeSpeakerListener ? Scen<kMpeSpeakerListener>::A : Scen<kMpeTag>::A;
}
int mpe_obs_dim(int s) {
  return s == kMpeSpread ? Scen<kMpeSpread>::D : s == kMpeSpeakerListener ? Scen<kMpeSpeakerListener>::D : Scen<kMpeTag>::D;
}
int mpe_n_entities(int s) {
  return s == kMpeSpread ? Scen<kMpeSpread>::E : s == kMpeSpeakerListener ? Scen<kMpeSpeakerListener>::E : Scen<kMpeTag>::E;
}
int mpe_dim_c(int s) {
  return s == kMpeSpread ? Scen<kMpeSpread>::DC : s == kMpeSpeakerListener ? Scen<kMpeSpeakerListener>::DC : Scen<kMpeTag>::DC;
}
int mpe_n_actions(int s, int a) {
  return s == kMpeSpread ? Scen<kMpeSpread>::n_actions(a)
         : s == kMpeSpeakerListener ? Scen<kMpeSpeakerListener>::n_actions(a) : Scen<kMpeTag>::n_actions(a);
}
int mpe_obs_size(int s, int a) {
  return s == kMpeSpread ? Scen<kMpeSpread>::obs_size(a)
         : s == kMpeSpeakerListener ? Scen<kMpeSpeakerListener>::obs_size(a) : Scen<kMpeTag>::obs_size(a);
}

void mpe_launch_reset(const MpeConfig& c, const MpeState& s, const LaunchCommon& lc, KeyWords key,
                      KeyWords carry_parent) {
  unsigned g = grid_for(lc.n, kThreads);
  Key k = to_key(key), cp = to_key(carry_parent);
  switch (c.scenario) {
    case kMpeSpread: mpe_reset_kernel<kMpeSpread><<<g, kThreads, 0, lc.stream>>>(s, lc, k, cp); break;
    case kMpeSpeakerListener: mpe_reset_kernel<kMpeSpeakerListener><<<g, kThreads, 0, lc.stream>>>(s, lc, k, cp); break;
    default: mpe_reset_kernel<kMpeTag><<<g, kThreads, 0, lc.stream>>>(s, lc, k, cp); break;
  }
  ++g_launches;
}

void mpe_launch_step(const MpeConfig& c, const MpeState& s, const LaunchCommon& lc, bool random,
                     KeyWords step_key) {
  unsigned g = grid_for(lc.end - lc.begin, kThreads);
  Key k = to_key(step_key);
#define MARL_MPE_STEP(S)                                                                  \
  c.continuous ? (random ? mpe_step_kernel<S, true, true><<<g, kThreads, 0, lc.stream>>>(s, lc, k, c.coop_prey)   \
                         : mpe_step_kernel<S, false, true><<<g, kThreads, 0, lc.stream>>>(s, lc, k, c.coop_prey)) \
               : (random ? mpe_step_kernel<S, true, false><<<g, kThreads, 0, lc.stream>>>(s, lc, k, c.coop_prey)  \
                         : mpe_step_kernel<S, false, false><<<g, kThreads, 0, lc.stream>>>(s, lc, k, c.coop_prey))
  switch (c.scenario) {
    case kMpeSpread: MARL_MPE_STEP(kMpeSpread); break;
    case kMpeSpeakerListener: MARL_MPE_STEP(kMpeSpeakerListener); break;
    default: MARL_MPE_STEP(kMpeTag); break;
  }
#undef MARL_MPE_STEP
  ++g_launches;
}

// K probe steps in one launch (mpe_probe_kernel).
void mpe_launch_probe(const MpeConfig& c, const MpeState& s, const LaunchCommon& lc, KeyWords parent,
                      uint64_t t0, int K) {
  const unsigned g = grid_for(lc.end - lc.begin, 32);
  const Key k = to_key(parent);
#define MARL_MPE_PROBE(S)                                                                        \
  c.continuous ? mpe_probe_kernel<S, true><<<g, 96, 0, lc.stream>>>(s, lc, k, c.coop_prey, t0, K) \
               : mpe_probe_kernel<S, false><<<g, 96, 0, lc.stream>>>(s, lc, k, c.coop_prey, t0, K)
  switch (c.scenario) {
    case kMpeSpread: MARL_MPE_PROBE(kMpeSpread); break;
    case kMpeSpeakerListener: MARL_MPE_PROBE(kMpeSpeakerListener); break;
    default: MARL_MPE_PROBE(kMpeTag); break;
  }
#undef MARL_MPE_PROBE
  ++g_launches;
}

void mpe_launch_hash(const MpeConfig& c, const MpeState& s, int64_t n, uint64_t* out, cudaStream_t st) {
  unsigned g = grid_for(n, 256);
  switch (c.scenario) {
    case kMpeSpread: mpe_hash_kernel<kMpeSpread><<<g, 256, 0, st>>>(s, n, out); break;
    case kMpeSpeakerListener: mpe_hash_kernel<kMpeSpeakerListener><<<g, 256, 0, st>>>(s, n, out); break;
    default: mpe_hash_kernel<kMpeTag><<<g, 256, 0, st>>>(s, n, out); break;
  }
  ++g_launches;
}

}  // namespace marl_b200
