// TEST INFRASTRUCTURE ONLY -- reference-side parity driver for the drop-in
// adapter include/marl_b200_vector_env.hpp: the same reference-style code runs
// through marl_b200::VectorEnv (B200) and the UNMODIFIED marl::VectorEnv (CPU,
// oracle/_ref) and every StepBatchResult field is compared exactly.  Built by
// `make -C oracle adapter` into oracle/_ref/adapter_parity (needs the
// reference headers, so only where /root/reference exists; the binary travels
// to the GPU box prebuilt).  Exit 1 = the engine refused (no GPU), 0 = parity.
#include <cstdio>
#include "marl/registry.hpp"
#include "marl/prng.hpp"
#include "marl_b200_vector_env.hpp"

// Reference-side code written against marl::VectorEnv, switched by one alias.
using VectorEnv = marl_b200::VectorEnv;

int main(int argc, char** argv) {
  marl::Config cfg = {{"ally_units", {"marine", "marine", "marine"}},
                      {"enemy_units", {"marine", "marine", "marine"}}};
  auto env = marl::make_env("SMAX_5m_vs_6m", cfg);
  try {
    VectorEnv venv(env, 64, cfg);
    marl::VectorEnv ref(env, 64);
    auto key = marl::prng::key_from_seed(7);
    auto [o1, s1] = venv.reset(key);
    auto [o2, s2] = ref.reset(key);
    if (o1 != o2 || s1.keys != s2.keys) { std::puts("RESET MISMATCH"); return 3; }
    auto akeys = marl::prng::split(marl::prng::fold_in(key, 2), 40);
    for (int t = 0; t < 40; ++t) {
      std::vector<marl::AgentMap<marl::Action>> acts(64);
      for (int e = 0; e < 64; ++e) {
        auto ek = marl::prng::split(akeys[size_t(t)], 64)[size_t(e)];
        for (int a = 0; a < 3; ++a) {
          auto agent = env->agents()[size_t(a)];
          auto legal = env->legal_actions(*s2.states[size_t(e)], agent);
          std::vector<int> idx;
          for (int q = 0; q < int(legal.size()); ++q) if (legal[size_t(q)]) idx.push_back(q);
          acts[size_t(e)].emplace(agent, idx[size_t(marl::prng::bits(ek, uint64_t(a)) % idx.size())]);
        }
      }
      auto r1 = venv.step(s1, acts);
      auto r2 = ref.step(s2, acts);
      if (r1.obs != r2.obs || r1.rewards != r2.rewards || r1.dones != r2.dones || r1.infos != r2.infos ||
          r1.finished != r2.finished || r1.final_returns != r2.final_returns ||
          r1.final_lengths != r2.final_lengths || r1.next.keys != r2.next.keys) {
        std::printf("STEP %d MISMATCH\n", t);
        return 4;
      }
      for (int e = 0; e < 64; ++e)
        if (r2.finished[size_t(e)] && r1.final_obs[size_t(e)] != r2.final_obs[size_t(e)]) { std::puts("FINAL"); return 5; }
      s1 = r1.next;
      s2 = r2.next;
    }
    // rollout(venv, policy, T, key) (vector_env.cpp:131-165): the adapter's vs the reference's
    // free function, with a policy that reads the observations (stop is always legal in SMAX)
    marl::Policy policy = [&](const std::vector<marl::AgentMap<marl::Obs>>& obs) {
      marl::PolicyOutput out;
      for (const auto& m : obs) {
        marl::AgentMap<marl::Action> a;
        marl::AgentMap<double> lp, v;
        for (size_t q = 0; q < m.size(); ++q) {
          const std::string& agent = m.key(q);
          const marl::Obs& o = m.value(q);
          a.emplace(agent, 4);
          lp.emplace(agent, double(o[0]) - double(o[1]));
          v.emplace(agent, double(o[2]) + 0.5 * double(o[3]));
        }
        out.actions.push_back(std::move(a));
        out.log_probs.push_back(std::move(lp));
        out.values.push_back(std::move(v));
      }
      return out;
    };
    auto t1 = marl_b200::rollout(venv, policy, 30, marl::prng::key_from_seed(11));
    auto t2 = marl::rollout(ref, policy, 30, marl::prng::key_from_seed(11));
    if (t1.obs != t2.obs || t1.actions != t2.actions || t1.rewards != t2.rewards || t1.dones != t2.dones ||
        t1.log_probs != t2.log_probs || t1.values != t2.values || t1.final_obs != t2.final_obs ||
        t1.final_state.keys != t2.final_state.keys || t1.n_steps != t2.n_steps || t1.n_envs != t2.n_envs) {
      std::puts("ROLLOUT MISMATCH");
      return 6;
    }
    std::puts("ADAPTER PARITY OK");
    return 0;
  } catch (const marl::ContractError& e) {
    std::printf("ContractError: %s\n", e.what());
    return 2;
  } catch (const std::runtime_error& e) {  // MARL_ERR_CUDA: no device here, no CPU fallback
    std::printf("runtime_error: %s\n", e.what());
    return 1;
  }
}
