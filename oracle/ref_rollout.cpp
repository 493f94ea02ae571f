// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI driver for the IPPO rollout over
// the UNMODIFIED reference library compiled into oracle/_ref.  The reference's
// Collector (proj/core/src/algo/ppo.cpp:178-374) and its Rollout buffer
// (ppo.cpp:159-177) live in an anonymous namespace, so the collect loop is
// restated here line for line (ppo.cpp:189-192 constructor, :206-323 collect,
// :333-360 fill_inputs) on top of the reference's own public building blocks:
// VectorEnv (vector_env.hpp:74-89), TeamLayout (team.cpp:10-42),
// ppo_net_spec / ppo_init_nets (ppo.cpp:80-124), nn::ff_forward
// (actor_critic.hpp:49-52), nn::sample_masked (actor_critic.hpp:247-262) and
// nn::compute_gae (actor_critic.hpp:282-299).  Everything numerical is the
// reference's code; only the loop orchestration is restated.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "marl/algo/actor_critic.hpp"
#include "marl/algo/ppo.hpp"
#include "marl/algo/team.hpp"
#include "marl/errors.hpp"
#include "marl/prng.hpp"
#include "marl/registry.hpp"
#include "marl/vector_env.hpp"

using namespace marl;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Config parse(const char* cfg) { return (cfg && *cfg) ? Config::parse(cfg) : Config::object(); }
PrngKey key_of(const uint32_t k[4]) { return PrngKey{k[0], k[1], k[2], k[3]}; }

PpoNetSpec spec_for(const Env& env, int centralized) {
  PpoConfig pc;  // defaults: fc_width 64, n_fc_layers 2, tanh (ppo.hpp:38-57)
  return ppo_net_spec(env, pc, centralized != 0);  // centralized: the MAPPO critic reads world_state
}
}  // namespace

extern "C" {

const char* mref_rollout_last_error(void) { return g_err.c_str(); }

// ppo_net_spec (ppo.cpp:80-107) and the packed parameter counts.
int mref_ppo_spec(const char* env_id, const char* cfg, int centralized, int* in_dim, int* critic_in, int* n_actions,
                  int* n_actor, int* n_critic) {
  return guarded([&] {
    auto env = make_env(env_id, parse(cfg));
    PpoNetSpec s = spec_for(*env, centralized);
    *critic_in = s.critic_in;
    PpoNets nets = ppo_init_nets(prng::key_from_seed(0), s);
    *in_dim = s.in_dim;
    *n_actions = s.n_actions;
    *n_actor = int(nets.pack_actor().size());
    *n_critic = int(nets.pack_critic().size());
  });
}

// ppo_init_nets(key, spec) (ppo.cpp:109-124), packed in nn::pack order.
int mref_ppo_init(const char* env_id, const char* cfg, int centralized, const uint32_t key[4], float* actor,
                  float* critic) {
  return guarded([&] {
    auto env = make_env(env_id, parse(cfg));
    PpoNets nets = ppo_init_nets(key_of(key), spec_for(*env, centralized));
    auto a = nets.pack_actor(), c = nets.pack_critic();
    std::memcpy(actor, a.data(), a.size() * sizeof(float));
    std::memcpy(critic, c.data(), c.size() * sizeof(float));
  });
}

// Collector(env, cfg, spec, centralized, key) + n_windows x collect(nets, T, w*T, shaping);
// the buffers of the LAST window are returned ([T][R] row-major, R = n_envs * A).
int mref_collect(const char* env_id, const char* cfg, int centralized, float* o_critic_in, int n_envs, int T,
                 int n_windows, const uint32_t key[4],
                 const float* actor, const float* critic, double gamma, double lambda, double shaping,
                 float* o_obs, int32_t* o_actions, float* o_rewards, uint8_t* o_dones, uint8_t* o_resets,
                 float* o_logp, float* o_value, uint8_t* o_legal, float* o_active, float* o_adv, float* o_vtarg,
                 double* o_ep_return_sum, int64_t* o_episodes) {
  return guarded([&] {
    auto env = make_env(env_id, parse(cfg));
    const PpoNetSpec spec = spec_for(*env, centralized);
    PpoNets nets = ppo_init_nets(prng::key_from_seed(0), spec);
    {
      auto a = nets.pack_actor(), c = nets.pack_critic();
      nets.unpack_actor(std::vector<float>(actor, actor + a.size()));
      nets.unpack_critic(std::vector<float>(critic, critic + c.size()));
    }
    const TeamLayout layout = TeamLayout::from_env(*env);
    VectorEnv venv(env, n_envs);
    // Collector constructor, ppo.cpp:189-192
    const PrngKey ckey = key_of(key);
    const PrngKey act_key = prng::fold_in(ckey, 2);
    auto [obs0, state0] = venv.reset(prng::fold_in(ckey, 1));
    std::vector<AgentMap<Obs>> cur_obs = std::move(obs0);
    BatchedState state = std::move(state0);
    const int E = n_envs, A = layout.n_agents(), R = E * A;
    std::vector<uint8_t> prev_finished(size_t(E), 1);
    const int in_dim = spec.in_dim, na = spec.n_actions, cin = spec.critic_in;
    double ep_sum = 0.0;
    int64_t episodes = 0;

    auto fill_inputs = [&](nn::Mat<float>& x, nn::Mat<float>& xc, uint8_t* legal, float* active) {  // ppo.cpp:333-360
      std::vector<float> ws;
      for (int e = 0; e < E; ++e) {
        const auto& st = *state.states[size_t(e)];
        if (centralized) ws = *env->world_state(st);
        for (int a = 0; a < A; ++a) {
          const int r = e * A + a;
          layout.write_input(cur_obs[size_t(e)].at(layout.agents[size_t(a)]), a, &x.a[size_t(r) * size_t(in_dim)]);
          if (centralized)
            std::memcpy(&xc.a[size_t(r) * size_t(cin)], ws.data(), ws.size() * sizeof(float));
          else
            std::memcpy(&xc.a[size_t(r) * size_t(cin)], &x.a[size_t(r) * size_t(in_dim)], size_t(in_dim) * 4);
          if (legal) layout.write_legal(*env, st, a, legal + size_t(r) * size_t(na));
          if (active) active[r] = env->agent_active(st, layout.agents[size_t(a)]) ? 1.0f : 0.0f;
        }
      }
    };

    std::vector<float> rew_buf, val_buf;
    std::vector<uint8_t> don_buf;
    for (int w = 0; w < n_windows; ++w) {
      const int64_t seq_base = int64_t(w) * T;
      std::vector<float> obs(size_t(T) * R * in_dim), crit(size_t(T) * R * cin), rewards(size_t(T) * R),
          logp(size_t(T) * R),
          value(size_t(T) * R), active(size_t(T) * R);
      std::vector<int32_t> actions(size_t(T) * R);
      std::vector<uint8_t> dones(size_t(T) * R), resets(size_t(T) * R), legal(size_t(T) * R * na);
      ep_sum = 0.0;
      episodes = 0;
      for (int t = 0; t < T; ++t) {  // ppo.cpp:229-281
        const size_t base = size_t(t) * size_t(R);
        for (int r = 0; r < R; ++r) resets[base + size_t(r)] = prev_finished[size_t(r / A)];
        nn::Mat<float> x(R, in_dim), xc(R, cin);
        fill_inputs(x, xc, &legal[base * size_t(na)], &active[base]);
        std::memcpy(&obs[base * size_t(in_dim)], x.a.data(), x.a.size() * sizeof(float));
        std::memcpy(&crit[base * size_t(cin)], xc.a.data(), xc.a.size() * sizeof(float));
        nn::Mat<float> logits = nn::ff_forward(nets.actor_ff, x, spec.act);
        nn::Mat<float> values = nn::ff_forward(nets.critic_ff, xc, spec.act);
        std::vector<AgentMap<Action>> acts(static_cast<size_t>(E));
        for (int r = 0; r < R; ++r) {
          auto kk = prng::fold_in(act_key, uint64_t(seq_base + t) * uint64_t(R) + uint64_t(r));
          double lp = 0;
          int a = nn::sample_masked(kk, &logits.a[size_t(r) * size_t(na)], &legal[(base + size_t(r)) * size_t(na)],
                                    na, &lp);
          actions[base + size_t(r)] = a;
          logp[base + size_t(r)] = float(lp);
          value[base + size_t(r)] = values(r, 0);
          acts[size_t(r / A)].emplace(layout.agents[size_t(r % A)], a);
        }
        auto res = venv.step(state, acts);
        for (int r = 0; r < R; ++r) {
          const int e = r / A;
          const auto& agent = layout.agents[size_t(r % A)];
          double rew = res.rewards[size_t(e)].at(agent);
          if (shaping > 0.0) {
            const auto& info = res.infos[size_t(e)].at(agent);
            auto it = info.find("shaped_reward");
            if (it != info.end()) rew += shaping * it->second;
          }
          rewards[base + size_t(r)] = float(rew);
          dones[base + size_t(r)] = res.finished[size_t(e)];
        }
        for (int e = 0; e < E; ++e)
          if (res.finished[size_t(e)]) {
            ep_sum += res.final_returns[size_t(e)];
            ++episodes;
          }
        prev_finished = res.finished;
        cur_obs = std::move(res.obs);
        state = std::move(res.next);
      }
      // bootstrap values, ppo.cpp:285-299
      nn::Mat<float> x(R, in_dim), xc(R, cin);
      fill_inputs(x, xc, nullptr, nullptr);
      nn::Mat<float> lastv = nn::ff_forward(nets.critic_ff, xc, spec.act);
      // GAE per row, ppo.cpp:301-321
      std::vector<float> adv(size_t(T) * R), vtarg(size_t(T) * R);
      std::vector<float> rw(static_cast<size_t>(T)), vl(static_cast<size_t>(T));
      std::vector<uint8_t> dn(static_cast<size_t>(T), 0);
      std::vector<float> a_out, t_out;
      for (int r = 0; r < R; ++r) {
        for (int t = 0; t < T; ++t) {
          const size_t i = size_t(t) * size_t(R) + size_t(r);
          rw[size_t(t)] = rewards[i];
          vl[size_t(t)] = value[i];
          dn[size_t(t)] = dones[i];
        }
        nn::compute_gae<float>(rw, vl, dn, lastv(r, 0), float(gamma), float(lambda), &a_out, &t_out);
        for (int t = 0; t < T; ++t) {
          const size_t i = size_t(t) * size_t(R) + size_t(r);
          adv[i] = a_out[size_t(t)];
          vtarg[i] = t_out[size_t(t)];
        }
      }
      if (w == n_windows - 1) {
        auto cp = [](void* d, const void* s, size_t n) {
          if (d) std::memcpy(d, s, n);
        };
        cp(o_obs, obs.data(), obs.size() * 4);
        cp(o_critic_in, crit.data(), crit.size() * 4);
        cp(o_actions, actions.data(), actions.size() * 4);
        cp(o_rewards, rewards.data(), rewards.size() * 4);
        cp(o_dones, dones.data(), dones.size());
        cp(o_resets, resets.data(), resets.size());
        cp(o_logp, logp.data(), logp.size() * 4);
        cp(o_value, value.data(), value.size() * 4);
        cp(o_legal, legal.data(), legal.size());
        cp(o_active, active.data(), active.size() * 4);
        cp(o_adv, adv.data(), adv.size() * 4);
        cp(o_vtarg, vtarg.data(), vtarg.size() * 4);
        if (o_ep_return_sum) *o_ep_return_sum = ep_sum;
        if (o_episodes) *o_episodes = episodes;
      }
    }
  });
}

// ---------------------------------------------------------------- PPO update
// ppo_init_nets(key, spec) for a recurrent spec (PpoConfig recurrent=true, fc_width, hidden_width).
int mref_ppo_init_rnn(const char* env_id, const char* cfg, int centralized, int fc_width, int hidden_width,
                      const uint32_t key[4], float* actor, float* critic, int* n_actor, int* n_critic) {
  return guarded([&] {
    auto env = make_env(env_id, parse(cfg));
    PpoConfig pc;
    pc.recurrent = true;
    pc.fc_width = fc_width;
    pc.hidden_width = hidden_width;
    PpoNets nets = ppo_init_nets(key_of(key), ppo_net_spec(*env, pc, centralized != 0));
    auto a = nets.pack_actor(), c = nets.pack_critic();
    *n_actor = int(a.size());
    *n_critic = int(c.size());
    if (actor) std::memcpy(actor, a.data(), a.size() * sizeof(float));
    if (critic) std::memcpy(critic, c.data(), c.size() * sizeof(float));
  });
}

// prng::permutation(key, n) (prng.cpp:151-159): the reference's Fisher-Yates.
int mref_permutation(const uint32_t key[4], int n, int32_t* out) {
  return guarded([&] {
    auto p = prng::permutation(key_of(key), n);
    std::memcpy(out, p.data(), p.size() * sizeof(int32_t));
  });
}

// ff_minibatch (ppo.cpp:409-441) + gather_rows (ppo.cpp:382-406), which are
// private to ppo.cpp, restated over the reference's public pieces:
// nn::normalize_advantages, nn::ff_forward, nn::ppo_row_loss, nn::ff_backward,
// nn::pack.  Inputs are a [T][R] rollout buffer (the flat slot s = t*R + r);
// out: the flat gradient (actor then critic) and {loss, pg, v, entropy, kl,
// clip_frac}.
int mref_ff_minibatch(const char* env_id, const char* cfg, int centralized, const float* actor, const float* critic,
                      const float* obs, const float* critic_in, const int32_t* actions, const float* logp,
                      const float* adv, const float* vtarg, const float* value, const float* active,
                      const uint8_t* legal, const int32_t* idx, int M, double clip_eps, double ent_coef,
                      double vf_coef, float* grad_out, double* stats_out) {
  return guarded([&] {
    auto env = make_env(env_id, parse(cfg));
    const PpoNetSpec spec = spec_for(*env, centralized);
    PpoNets nets = ppo_init_nets(prng::key_from_seed(0), spec);
    {
      auto a = nets.pack_actor(), c = nets.pack_critic();
      nets.unpack_actor(std::vector<float>(actor, actor + a.size()));
      nets.unpack_critic(std::vector<float>(critic, critic + c.size()));
    }
    const int in = spec.in_dim, cin = spec.critic_in, na = spec.n_actions;
    const size_t m = size_t(M);
    nn::Mat<float> x(M, in), xc(M, cin);
    nn::PpoRows<float> rows;
    rows.n_actions = na;
    rows.actions.resize(m);
    rows.old_log_probs.resize(m);
    rows.advantages.resize(m);
    rows.value_targets.resize(m);
    rows.old_values.resize(m);
    rows.legal.resize(m * size_t(na));
    rows.weights.resize(m);
    for (size_t i = 0; i < m; ++i) {
      const size_t s = size_t(idx[i]);
      std::memcpy(&x.a[i * size_t(in)], obs + s * size_t(in), size_t(in) * sizeof(float));
      const float* xs = centralized ? critic_in + s * size_t(cin) : obs + s * size_t(in);
      std::memcpy(&xc.a[i * size_t(cin)], xs, size_t(cin) * sizeof(float));
      rows.actions[i] = actions[s];
      rows.old_log_probs[i] = logp[s];
      rows.advantages[i] = adv[s];
      rows.value_targets[i] = vtarg[s];
      rows.old_values[i] = value[s];
      rows.weights[i] = active[s];
      std::memcpy(&rows.legal[i * size_t(na)], legal + s * size_t(na), size_t(na));
    }
    nn::normalize_advantages(rows.advantages, rows.weights);
    nn::FfCache<float> ac, cc;
    auto logits = nn::ff_forward(nets.actor_ff, x, spec.act, &ac);
    auto vmat = nn::ff_forward(nets.critic_ff, xc, spec.act, &cc);
    std::vector<float> values(m);
    for (size_t i = 0; i < m; ++i) values[i] = vmat(int(i), 0);
    nn::PpoLossConfig lcfg{clip_eps, ent_coef, vf_coef};
    auto loss = nn::ppo_row_loss(logits, values, rows, lcfg);
    auto ga = nn::ff_backward(nets.actor_ff, ac, spec.act, loss.dlogits);
    nn::Mat<float> dv(M, 1);
    for (size_t i = 0; i < m; ++i) dv(int(i), 0) = loss.dvalues[i];
    auto gc = nn::ff_backward(nets.critic_ff, cc, spec.act, dv);
    std::vector<float> flat;
    nn::pack(ga, flat);
    nn::pack(gc, flat);
    std::memcpy(grad_out, flat.data(), flat.size() * sizeof(float));
    stats_out[0] = double(loss.loss);
    stats_out[1] = loss.pg_loss;
    stats_out[2] = loss.v_loss;
    stats_out[3] = loss.entropy;
    stats_out[4] = loss.approx_kl;
    stats_out[5] = loss.clip_frac;
  });
}

// The reference's own public trainer: train_ippo / train_mappo (ppo.cpp:518-651)
// with PpoConfig::from_config.  metrics: rows x 12 (ppo.cpp:524-527 columns).
int mref_train(const char* env_id, const char* cfg, const char* ppo_cfg, int centralized, const uint32_t key[4],
               double* metrics, int max_rows, int* n_rows, float* actor, int* actor_cap, float* critic,
               int* critic_cap, int* diverged, int64_t* steps_done) {
  return guarded([&] {
    auto env = make_env(env_id, parse(cfg));
    PpoConfig pc = PpoConfig::from_config(parse(ppo_cfg));
    PpoRunResult res = centralized ? train_mappo(env, pc, key_of(key)) : train_ippo(env, pc, key_of(key));
    const auto& rows = res.metrics.rows;
    *n_rows = int(rows.size());
    for (size_t r = 0; r < rows.size() && int(r) < max_rows; ++r)
      for (size_t c = 0; c < rows[r].size(); ++c) metrics[r * rows[r].size() + c] = rows[r][c];
    auto a = res.nets.pack_actor(), c = res.nets.pack_critic();
    if (int(a.size()) <= *actor_cap) std::memcpy(actor, a.data(), a.size() * sizeof(float));
    if (int(c.size()) <= *critic_cap) std::memcpy(critic, c.data(), c.size() * sizeof(float));
    *actor_cap = int(a.size());  // the true sizes (the caller re-runs with larger buffers if short)
    *critic_cap = int(c.size());
    *diverged = res.diverged ? 1 : 0;
    *steps_done = res.steps_done;
  });
}

}  // extern "C"
