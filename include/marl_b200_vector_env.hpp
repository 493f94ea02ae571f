// Reference-side drop-in for marl::VectorEnv over the marl-b200 C-ABI.
//
// A header the REFERENCE's maintainers would add to their tree: a class with
// the exact reset/step signatures of marl::VectorEnv
// (/root/reference/proj/core/include/marl/vector_env.hpp:74-89) that runs the
// batch on a B200 and converts the engine's flat views back into the
// reference's StepBatchResult / AgentMap types, so rollout(), the PPO
// Collector and tests written against VectorEnv run unmodified with
// `using VectorEnv = marl_b200::VectorEnv;`.
//
// Compiles against the reference's headers (marl/vector_env.hpp) and links
// libmarl_b200.so; nothing here is used by the engine itself.  Differences
// from the reference class, both deliberate:
//   * the constructor also takes the env's Config (the C-ABI constructs the
//     device env from id + JSON, registry.cpp:83-97);
//   * BatchedState::states is left empty: the live state stays in HBM, the
//     keys / episode_returns / episode_lengths are filled from the device.
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "marl/errors.hpp"
#include "marl/vector_env.hpp"
#include "marl_b200.h"

namespace marl_b200 {

inline void throw_status(int rc) {  // status -> the reference's exception taxonomy (errors.hpp:9-26)
  if (rc == MARL_OK) return;
  const std::string msg = marl_last_error();
  switch (rc) {
    case MARL_ERR_NOT_FOUND: throw marl::NotFoundError(msg);
    case MARL_ERR_SCHEMA: throw marl::SchemaError(msg);
    case MARL_ERR_CONTRACT: throw marl::ContractError(msg);
    case MARL_ERR_DIVERGENCE: throw marl::DivergenceError(msg);
    default: throw std::runtime_error(msg);
  }
}

class VectorEnv {
 public:
  VectorEnv(std::shared_ptr<const marl::Env> env, int n_envs, const marl::Config& config = marl::Config::object(),
            int device = 0)
      : env_(std::move(env)), n_envs_(n_envs) {
    if (n_envs < 1) throw marl::ContractError("VectorEnv: n_envs must be >= 1");  // vector_env.cpp:45-49
    marl_venv* h = nullptr;
    throw_status(marl_venv_create(env_->id().c_str(), config.dump().c_str(), n_envs, device, &h));
    h_.reset(h, [](marl_venv* p) { marl_venv_destroy(p); });
    throw_status(marl_venv_spec(h, &spec_));
    for (int a = 0; a < spec_.n_agents; ++a) {
      char name[128];
      int32_t obs_size = 0, n_act = 0;
      throw_status(marl_venv_agent(h, a, name, sizeof name, &obs_size, &n_act));
      agents_.emplace_back(name);
      obs_size_.push_back(obs_size);
      n_actions_.push_back(n_act);  // discrete n, or the box's flat size
    }
    for (int k = 0; k < spec_.n_info; ++k) {
      char name[128];
      throw_status(marl_venv_info_name(h, k, name, sizeof name));
      info_names_.emplace_back(name);
    }
  }

  const marl::Env& env() const { return *env_; }
  int n_envs() const { return n_envs_; }

  std::pair<std::vector<marl::AgentMap<marl::Obs>>, marl::BatchedState> reset(const marl::PrngKey& key) const {
    const uint32_t k[4] = {key.k0, key.k1, key.c0, key.c1};
    throw_status(marl_venv_reset(h_.get(), k));
    std::vector<float> obs(size_t(n_envs_) * spec_.n_agents * spec_.obs_dim);
    marl_host_step out{};
    out.obs = obs.data();
    throw_status(marl_venv_download(h_.get(), &out));
    return {unflatten_obs(obs.data()), device_state()};
  }

  // VectorEnv::step (vector_env.cpp:72-129): size checks and the reference's
  // ContractError for mismatched batches, host actions validated like
  // Env::validate_actions (env.cpp:7-14), then one fused device step.
  marl::StepBatchResult step(const marl::BatchedState& state,
                             const std::vector<marl::AgentMap<marl::Action>>& actions) const {
    if (state.keys.size() != size_t(n_envs_) || actions.size() != size_t(n_envs_))
      throw marl::ContractError("VectorEnv::step: batch size mismatch");
    int32_t box = 0;  // > 0: box action spaces (continuous MPE), rows of `box` floats
    throw_status(marl_venv_action_dim(h_.get(), &box));
    std::vector<int32_t> flat(box ? 0 : size_t(n_envs_) * spec_.n_agents);
    std::vector<float> flat_f(box ? size_t(n_envs_) * spec_.n_agents * size_t(box) : 0, 0.0f);
    for (int e = 0; e < n_envs_; ++e)
      for (int a = 0; a < spec_.n_agents; ++a) {
        const marl::Action& act = actions[size_t(e)].at(agents_[size_t(a)]);
        if (box) {  // Env::validate_actions: the vector must have the space's flat size
          const auto* v = std::get_if<std::vector<float>>(&act);
          if (!v || v->size() > size_t(box) || int(v->size()) != n_actions_[size_t(a)])
            throw marl::ContractError(env_->id() + ": action for agent '" + agents_[size_t(a)] +
                                      "' is outside its action space");
          std::copy(v->begin(), v->end(), flat_f.begin() + (size_t(e) * spec_.n_agents + a) * size_t(box));
        } else {
          if (!std::holds_alternative<int>(act))
            throw marl::ContractError(env_->id() + ": action for agent '" + agents_[size_t(a)] +
                                      "' is outside its action space");
          flat[size_t(e) * spec_.n_agents + a] = std::get<int>(act);
        }
      }
    const size_t N = size_t(n_envs_), A = size_t(spec_.n_agents), D = size_t(spec_.obs_dim);
    std::vector<float> obs(N * A * D), final_obs(N * A * D);
    std::vector<double> rewards(N * A), infos(N * A * size_t(spec_.n_info)), final_returns(N);
    std::vector<uint8_t> dones(N * (A + 1)), finished(N);
    std::vector<int32_t> final_lengths(N);
    marl_host_step out{obs.data(), rewards.data(), dones.data(), finished.data(), final_obs.data(),
                       final_returns.data(), final_lengths.data(), infos.data(), nullptr};
    if (box)
      throw_status(marl_venv_step_continuous_host(h_.get(), flat_f.data(), &out));
    else
      throw_status(marl_venv_step_host(h_.get(), flat.data(), &out));

    marl::StepBatchResult r;
    r.obs = unflatten_obs(obs.data());
    r.final_obs.resize(N);
    r.rewards.resize(N);
    r.dones.resize(N);
    r.infos.resize(N);
    for (size_t e = 0; e < N; ++e) {
      for (size_t a = 0; a < A; ++a) {
        const std::string& name = agents_[a];
        r.rewards[e].emplace(name, rewards[e * A + a]);
        r.dones[e].emplace(name, dones[e * (A + 1) + a]);
        marl::Info info;
        for (size_t k = 0; k < info_names_.size(); ++k) info[info_names_[k]] = infos[(e * A + a) * info_names_.size() + k];
        if (finished[e]) {  // vector_env.cpp:107-119 adds the episode record to every agent's infos
          info["episode_return"] = final_returns[e];
          info["episode_length"] = double(final_lengths[e]);
        }
        r.infos[e].emplace(name, std::move(info));
      }
      r.dones[e].emplace(marl::kAllAgents, dones[e * (A + 1) + A]);
      if (finished[e]) r.final_obs[e] = unflatten_row(final_obs.data(), e);
    }
    r.finished = std::move(finished);
    r.final_returns = std::move(final_returns);
    r.final_lengths.assign(final_lengths.begin(), final_lengths.end());
    r.next = device_state();
    return r;
  }

 private:
  marl::AgentMap<marl::Obs> unflatten_row(const float* flat, size_t e) const {
    marl::AgentMap<marl::Obs> m;
    const size_t A = size_t(spec_.n_agents), D = size_t(spec_.obs_dim);
    for (size_t a = 0; a < A; ++a) {
      const float* row = flat + (e * A + a) * D;
      m.emplace(agents_[a], marl::Obs(row, row + obs_size_[a]));  // drop the zero padding to D
    }
    return m;
  }
  std::vector<marl::AgentMap<marl::Obs>> unflatten_obs(const float* flat) const {
    std::vector<marl::AgentMap<marl::Obs>> v;
    v.reserve(size_t(n_envs_));
    for (int e = 0; e < n_envs_; ++e) v.push_back(unflatten_row(flat, size_t(e)));
    return v;
  }
  marl::BatchedState device_state() const {
    marl_views views{};
    throw_status(marl_venv_views(h_.get(), &views));
    throw_status(marl_venv_sync(h_.get()));
    const size_t N = size_t(n_envs_);
    std::vector<uint32_t> keys(N * 4);
    marl::BatchedState s;
    s.keys.resize(N);
    s.episode_returns.resize(N);
    s.episode_lengths.resize(N);
    std::vector<int32_t> lens(N);
    throw_status(marl_copy_device_to_host(keys.data(), views.keys, keys.size() * 4));
    throw_status(marl_copy_device_to_host(s.episode_returns.data(), views.episode_returns, N * 8));
    throw_status(marl_copy_device_to_host(lens.data(), views.episode_lengths, N * 4));
    for (size_t e = 0; e < N; ++e) {
      s.keys[e] = marl::PrngKey{keys[4 * e], keys[4 * e + 1], keys[4 * e + 2], keys[4 * e + 3]};
      s.episode_lengths[e] = lens[e];
    }
    return s;
  }

  std::shared_ptr<const marl::Env> env_;
  int n_envs_;
  std::shared_ptr<marl_venv> h_;
  marl_spec spec_{};
  std::vector<std::string> agents_, info_names_;
  std::vector<int32_t> obs_size_, n_actions_;
};

// rollout(venv, policy, n_steps, key) (vector_env.hpp:91-92, vector_env.cpp:131-165)
// over the adapter: the same loop, checks and TrajectoryBatch as the reference's.
inline marl::TrajectoryBatch rollout(const VectorEnv& venv, const marl::Policy& policy, int n_steps,
                                     const marl::PrngKey& key) {
  if (n_steps < 1) throw marl::ContractError("rollout: n_steps must be >= 1");
  marl::TrajectoryBatch traj;
  traj.n_steps = n_steps;
  traj.n_envs = venv.n_envs();
  traj.obs.reserve(size_t(n_steps));
  auto [obs, state] = venv.reset(key);
  for (int t = 0; t < n_steps; ++t) {
    marl::PolicyOutput pi = policy(obs);
    if (pi.actions.size() != size_t(venv.n_envs()))
      throw marl::ContractError("rollout: policy returned " + std::to_string(pi.actions.size()) +
                                " action maps for " + std::to_string(venv.n_envs()) + " envs");
    if (!pi.log_probs.empty() && pi.log_probs.size() != size_t(venv.n_envs()))
      throw marl::ContractError("rollout: policy log_probs batch size mismatch");
    if (!pi.values.empty() && pi.values.size() != size_t(venv.n_envs()))
      throw marl::ContractError("rollout: policy values batch size mismatch");
    marl::StepBatchResult r = venv.step(state, pi.actions);
    traj.obs.push_back(std::move(obs));
    traj.actions.push_back(std::move(pi.actions));
    traj.rewards.push_back(std::move(r.rewards));
    traj.dones.push_back(std::move(r.dones));
    traj.log_probs.push_back(std::move(pi.log_probs));
    traj.values.push_back(std::move(pi.values));
    obs = std::move(r.obs);
    state = std::move(r.next);
  }
  traj.final_obs = std::move(obs);
  traj.final_state = std::move(state);
  return traj;
}

}  // namespace marl_b200
