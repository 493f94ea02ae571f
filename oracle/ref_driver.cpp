// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI driver over the UNMODIFIED reference library (`marlcore`, compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python tests and bench.py's CPU arm call the reference's own
// VectorEnv::reset/step (vector_env.cpp:51-129) and throughput_probe
// (vector_env.cpp:191-222) through ctypes, and dumps the flattened per-env
// results in exactly the layout the B200 C-ABI exposes (include/marl_b200.h),
// so golden vectors can be compared buffer-for-buffer.
//
// The only logic here that is not a direct call into the reference is the
// random-legal action stream: vector_env.cpp:169-187 keeps it in an anonymous
// namespace, so it is restated below (legal_uniform: vector_env.cpp:21-32) on
// top of the reference's public prng/Env API.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "marl/errors.hpp"
#include "marl/parallel.hpp"
#include "marl/prng.hpp"
#include "marl/registry.hpp"
#include "marl/vector_env.hpp"

using namespace marl;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const NotFoundError& e) {
    return fail(1, e.what());
  } catch (const SchemaError& e) {
    return fail(2, e.what());
  } catch (const ContractError& e) {
    return fail(3, e.what());
  } catch (const DivergenceError& e) {
    return fail(4, e.what());
  } catch (const std::exception& e) {
    return fail(6, e.what());
  }
}

PrngKey to_key(const uint32_t k[4]) { return PrngKey{k[0], k[1], k[2], k[3]}; }
void from_key(const PrngKey& k, uint32_t* out) {
  out[0] = k.k0;
  out[1] = k.k1;
  out[2] = k.c0;
  out[3] = k.c1;
}

// vector_env.cpp:21-32 (anonymous namespace there).
int legal_uniform(uint64_t raw, const std::vector<uint8_t>& mask) {
  int n_legal = 0;
  for (uint8_t m : mask) n_legal += m ? 1 : 0;
  if (n_legal == 0) throw ContractError("no legal action available");
  int pick = int(raw % uint64_t(n_legal));
  for (size_t a = 0; a < mask.size(); ++a) {
    if (!mask[a]) continue;
    if (pick == 0) return int(a);
    --pick;
  }
  return int(mask.size()) - 1;
}

struct Handle {
  std::shared_ptr<const Env> env;
  std::unique_ptr<VectorEnv> venv;
  BatchedState state;
  int n = 0, A = 0, obs_dim = 0, n_act = 0;
  std::vector<std::string> info_keys;  // sorted (std::map order), episode_* excluded
};

void write_obs(const Handle& h, const AgentMap<Obs>& m, float* out) {
  std::fill(out, out + size_t(h.A) * h.obs_dim, 0.0f);
  for (int a = 0; a < h.A; ++a) {
    const Obs& o = m.value(size_t(a));
    std::copy(o.begin(), o.end(), out + size_t(a) * h.obs_dim);
  }
}

}  // namespace

extern "C" {

const char* mref_last_error() { return g_err.c_str(); }

int mref_create(const char* env_id, const char* cfg_json, int n_envs, void** out) {
  return guarded([&] {
    auto h = std::make_unique<Handle>();
    Config cfg = (cfg_json && *cfg_json) ? Config::parse(cfg_json) : Config::object();
    h->env = make_env(env_id, cfg);
    h->venv = std::make_unique<VectorEnv>(h->env, n_envs);
    h->n = n_envs;
    h->A = h->env->num_agents();
    for (const auto& a : h->env->agents()) {
      h->obs_dim = std::max(h->obs_dim, h->env->observation_space(a).flat_size());
      auto sp = h->env->action_space(a);
      h->n_act = std::max(h->n_act, sp.kind == SpaceDescriptor::Kind::kDiscrete ? sp.n : sp.flat_size());
    }
    *out = h.release();
  });
}

void mref_destroy(void* p) { delete static_cast<Handle*>(p); }

int mref_spec(void* p, int* n_agents, int* obs_dim, int* n_act) {
  auto* h = static_cast<Handle*>(p);
  *n_agents = h->A;
  *obs_dim = h->obs_dim;
  *n_act = h->n_act;
  return 0;
}

int mref_set_threads(int n) {
  return guarded([&] { ThreadPool::global().resize(n); });
}

int mref_reset(void* p, const uint32_t key[4], float* obs, uint32_t* keys, uint64_t* hashes) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    auto [o, st] = h->venv->reset(to_key(key));
    h->state = std::move(st);
    for (int i = 0; i < h->n; ++i) {
      if (obs) write_obs(*h, o[size_t(i)], obs + size_t(i) * h->A * h->obs_dim);
      if (keys) from_key(h->state.keys[size_t(i)], keys + 4 * size_t(i));
      if (hashes) hashes[i] = h->env->state_hash(*h->state.states[size_t(i)]);
    }
  });
}

// Env::world_state of the current batch state (smax.cpp:272-289, mpe.cpp:229-242,
// overcooked.cpp:315-319): [N][W] f32, W = world_state_size().
int mref_world_state(void* p, float* out, int* width) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    const int W = h->env->world_state_size();
    *width = W;
    if (!out) return;
    for (int i = 0; i < h->n; ++i) {
      auto w = h->env->world_state(*h->state.states[size_t(i)]);
      std::copy(w->begin(), w->end(), out + size_t(i) * W);
    }
  });
}

// Legal masks of the current batch state: [N][A][n_act] u8.
int mref_legal(void* p, uint8_t* legal) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    for (int i = 0; i < h->n; ++i)
      for (int a = 0; a < h->A; ++a) {
        auto m = h->env->legal_actions(*h->state.states[size_t(i)], h->env->agents()[size_t(a)]);
        uint8_t* dst = legal + (size_t(i) * h->A + a) * h->n_act;
        std::fill(dst, dst + h->n_act, 0);
        std::copy(m.begin(), m.end(), dst);
      }
  });
}

// random_legal_actions (vector_env.cpp:169-187) for the current state.
int mref_random_actions(void* p, const uint32_t step_key[4], int32_t* actions) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    auto env_keys = prng::split(to_key(step_key), size_t(h->n));
    for (int i = 0; i < h->n; ++i) {
      uint64_t j = 0;
      for (const auto& agent : h->env->agents()) {
        auto mask = h->env->legal_actions(*h->state.states[size_t(i)], agent);
        actions[size_t(i) * h->A + j] = legal_uniform(prng::bits(env_keys[size_t(i)], j), mask);
        ++j;
      }
    }
  });
}

// VectorEnv::step with explicit actions [N][A] i32; every output optional.
// infos: [N][A][n_info] f64 in std::map key order minus episode_*.
}  // extern "C"

namespace {
#define MREF_STEP_OUTS                                                                                     \
  float *obs, double *rewards, uint8_t *dones, uint8_t *finished, float *final_obs, double *final_returns, \
      int32_t *final_lengths, double *infos, int n_info, double *ep_returns, int32_t *ep_lengths,         \
      uint32_t *keys, uint64_t *hashes

void step_and_emit(Handle* h, const std::vector<AgentMap<Action>>& acts, MREF_STEP_OUTS) {
  {
    StepBatchResult r = h->venv->step(h->state, acts);
    for (int i = 0; i < h->n; ++i) {
      size_t ui = size_t(i);
      if (obs) write_obs(*h, r.obs[ui], obs + ui * h->A * h->obs_dim);
      for (int a = 0; a < h->A; ++a) {
        if (rewards) rewards[ui * h->A + a] = r.rewards[ui].value(size_t(a));
        if (dones) dones[ui * (h->A + 1) + a] = r.dones[ui].at(h->env->agents()[size_t(a)]);
        if (infos && n_info > 0) {
          const Info& inf = r.infos[ui].value(size_t(a));
          int k = 0;
          for (const auto& [name, v] : inf) {
            if (name == "episode_return" || name == "episode_length") continue;
            if (k < n_info) infos[(ui * h->A + a) * n_info + k] = v;
            ++k;
          }
        }
      }
      if (dones) dones[ui * (h->A + 1) + h->A] = r.dones[ui].at(kAllAgents);
      if (finished) finished[ui] = r.finished[ui];
      if (final_obs && r.finished[ui])
        write_obs(*h, r.final_obs[ui], final_obs + ui * h->A * h->obs_dim);
      if (final_returns) final_returns[ui] = r.final_returns[ui];
      if (final_lengths) final_lengths[ui] = r.final_lengths[ui];
      if (ep_returns) ep_returns[ui] = r.next.episode_returns[ui];
      if (ep_lengths) ep_lengths[ui] = r.next.episode_lengths[ui];
      if (keys) from_key(r.next.keys[ui], keys + 4 * ui);
      if (hashes) hashes[ui] = h->env->state_hash(*r.next.states[ui]);
    }
    h->state = std::move(r.next);
  }
}
}  // namespace

extern "C" {

// VectorEnv::step with explicit discrete actions [N][A] i32; every output optional.
// infos: [N][A][n_info] f64 in std::map key order minus episode_*.
int mref_step(void* p, const int32_t* actions, MREF_STEP_OUTS) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    std::vector<AgentMap<Action>> acts(size_t(h->n));
    for (int i = 0; i < h->n; ++i)
      for (int a = 0; a < h->A; ++a)
        acts[size_t(i)].emplace(h->env->agents()[size_t(a)], int(actions[size_t(i) * h->A + a]));
    step_and_emit(h, acts, obs, rewards, dones, finished, final_obs, final_returns, final_lengths, infos, n_info,
                  ep_returns, ep_lengths, keys, hashes);
  });
}

// The same with box actions [N][A][dim] f32: agent a's vector is its first
// action_space(a).flat_size() floats.
int mref_step_box(void* p, const float* actions, int dim, MREF_STEP_OUTS) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    std::vector<AgentMap<Action>> acts(size_t(h->n));
    for (int i = 0; i < h->n; ++i)
      for (int a = 0; a < h->A; ++a) {
        const auto& ag = h->env->agents()[size_t(a)];
        const int n = h->env->action_space(ag).flat_size();
        const float* v = actions + (size_t(i) * h->A + a) * size_t(dim);
        acts[size_t(i)].emplace(ag, std::vector<float>(v, v + n));
      }
    step_and_emit(h, acts, obs, rewards, dones, finished, final_obs, final_returns, final_lengths, infos, n_info,
                  ep_returns, ep_lengths, keys, hashes);
  });
}

// random_legal_actions for box spaces: space.sample(fold_in(env_key, j))
// (vector_env.cpp:179-181), [N][A][dim] f32 zero-padded.
int mref_random_actions_box(void* p, const uint32_t step_key[4], int dim, float* actions) {
  auto* h = static_cast<Handle*>(p);
  return guarded([&] {
    auto env_keys = prng::split(to_key(step_key), size_t(h->n));
    for (int i = 0; i < h->n; ++i) {
      uint64_t j = 0;
      for (const auto& agent : h->env->agents()) {
        auto act = h->env->action_space(agent).sample(prng::fold_in(env_keys[size_t(i)], j));
        const auto& v = std::get<std::vector<float>>(act);
        float* o = actions + (size_t(i) * h->A + j) * size_t(dim);
        for (int k = 0; k < dim; ++k) o[k] = k < int(v.size()) ? v[size_t(k)] : 0.0f;
        ++j;
      }
    }
  });
}

// The reference's own benchmark: throughput_probe (vector_env.cpp:191-222).
int mref_probe(const char* env_id, const char* cfg_json, int n_envs, int n_steps,
               const uint32_t key[4], double* seconds, double* cold_seconds) {
  return guarded([&] {
    Config cfg = (cfg_json && *cfg_json) ? Config::parse(cfg_json) : Config::object();
    ThroughputResult r = throughput_probe(env_id, n_envs, n_steps, to_key(key), cfg);
    *seconds = r.seconds;
    *cold_seconds = r.cold_seconds;
  });
}

// Raw PRNG entry points (prng.cpp) for KAT / key-derivation cross checks.
void mref_threefry(uint32_t k0, uint32_t k1, uint32_t x0, uint32_t x1, uint32_t* y) {
  prng::threefry2x32(k0, k1, x0, x1, &y[0], &y[1]);
}
void mref_split(const uint32_t key[4], uint64_t n, uint32_t* out) {
  auto v = prng::split(to_key(key), size_t(n));
  for (size_t i = 0; i < v.size(); ++i) from_key(v[i], out + 4 * i);
}
void mref_fold_in(const uint32_t key[4], uint64_t d, uint32_t* out) {
  from_key(prng::fold_in(to_key(key), d), out);
}
double mref_hypot(double x, double y) { return std::hypot(x, y); }

}  // extern "C"
