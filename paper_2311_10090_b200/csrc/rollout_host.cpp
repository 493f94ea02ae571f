// The IPPO / MAPPO collector of the C-ABI (marl_rollout_*, include/marl_b200.h):
// the reference's private Collector (proj/core/src/algo/ppo.cpp:178-374)
// around the env step and the policy kernels (rollout.cu, rnn.cu).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "host.h"

using namespace marl_b200;
using namespace mhost;


namespace mhost {

// ppo_net_spec (ppo.cpp:80-107) over TeamLayout::from_env (team.cpp:10-25);
// centralized: the MAPPO critic reads world_state (ppo.cpp:90-97).
void policy_dims(const marl_venv* h, int width, int centralized, int* in_dim, int* critic_in, int* n_act,
                 int* n_actor, int* n_critic) {
  const Env& e = *h->env;
  *in_dim = e.D + (e.A > 1 ? e.A : 0);
  *critic_in = centralized ? h->ws_width : *in_dim;
  *n_act = *std::max_element(e.n_actions.begin(), e.n_actions.end());
  *n_actor = width * *in_dim + width + width * width + width + *n_act * width + *n_act;
  *n_critic = width * *critic_in + width + width * width + width + width + 1;
}

PolicyNet net_of(const marl_rollout* r) {
  PolicyNet n{};
  const int in = r->in_dim, W = r->width, NA = r->n_act;
  n.w1 = r->params;
  n.b1 = n.w1 + W * in;
  n.w2 = n.b1 + W;
  n.b2 = n.w2 + W * W;
  n.w3 = n.b2 + W;
  n.b3 = n.w3 + NA * W;
  n.cw1 = n.b3 + NA;
  n.cb1 = n.cw1 + W * r->critic_in;
  n.cw2 = n.cb1 + W;
  n.cb2 = n.cw2 + W * W;
  n.cw3 = n.cb2 + W;
  n.cb3 = n.cw3 + W;
  n.in_dim = in;
  n.critic_in = r->critic_in;
  n.n_act = NA;
  n.width = W;
  n.relu = r->relu;
  n.centralized = r->centralized;
  return n;
}

PolicyNetBf16 net_bf16_of(const marl_rollout* r) {
  PolicyNetBf16 n{};
  n.a1 = r->images;
  n.a2 = n.a1 + 128 * rollout_tc_kx(r->in_dim);
  n.c2 = n.a2 + 64 * 64;
  n.h3 = n.c2 + 64 * 64;
  n.hc3 = n.h3 + 64 * 64;
  n.c1 = r->centralized ? n.hc3 + 16 * 64 : nullptr;
  n.bias = r->bias;
  return n;
}

// rnn_step of actor and critic for all R rows as SGEMMs (embed, GRU input and
// hidden paths, post, head) around the gate kernel; same arithmetic as the
// per-row kernel up to the GEMMs' summation order.
void rnn_collect_gemm(marl_rollout* r, const PolicyStep& s) {
  cudaStream_t st = r->h->stream;
  const float* critic = rnn_critic_params(r, st);
  const int64_t R = r->R;
  const int in = r->in_dim, CI = r->critic_in, NA = r->n_act, F = r->F, H = r->H;
  rnn_policy_rows(s, r->b, in, CI, NA, H, r->s_xa, r->s_xc, r->h_actor, r->h_critic, r->s_hpeek, st);
  for (int branch = (s.bootstrap ? 1 : 0); branch < 2; ++branch) {
    const int bin = branch == 0 ? in : CI, out = branch == 0 ? NA : 1;
    const RnnWPtrs w = rnn_weights(branch == 0 ? r->params : critic, bin, F, H, out);
    float* h = branch == 0 ? r->h_actor : (s.bootstrap ? r->s_hpeek : r->h_critic);
    const float* x = branch == 0 ? r->s_xa : r->s_xc;
    float* y = branch == 0 ? r->s_ya : r->s_yc;
    gemm_nt(st, R, F, bin, x, bin, w.we, bin, r->s_e, F, 0.0f);
    rnn_bias_act(r->s_e, R, F, w.be, true, r->relu, st);
    gemm_nt(st, R, 3 * H, F, r->s_e, F, w.wx, F, r->s_gx, 3 * H, 0.0f);
    gemm_nt(st, R, 3 * H, H, h, H, w.uh, H, r->s_gh, 3 * H, 0.0f);
    rnn_gates_inplace(R, H, h, r->s_gx, r->s_gh, w.bias6, st);
    gemm_nt(st, R, F, H, h, H, w.wp, H, r->s_p, F, 0.0f);
    rnn_bias_act(r->s_p, R, F, w.bp, true, r->relu, st);
    gemm_nt(st, R, out, F, r->s_p, F, w.wh, F, y, out, 0.0f);
    rnn_bias_act(y, R, out, w.bh, false, r->relu, st);
  }
  rnn_policy_sample(s, r->b, NA, r->s_ya, r->s_yc, st);
}

void run_policy(marl_rollout* r, int t, bool bootstrap, int64_t seq_base) {
  marl_venv* h = r->h;
  const Env& e = *h->env;
  PolicyStep s{};
  s.env_obs = h->v.obs;
  s.prev_finished = r->first ? nullptr : h->v.finished;
  s.agent_actions = r->agent_actions;
  s.A = e.A;
  s.D = e.D;
  s.family = e.family;
  s.R = r->R;
  s.row0 = r->row0;
  s.R_global = r->R_global;
  std::memcpy(s.act_key, r->act_key, 16);
  s.step_index = seq_base + t;
  s.t = t;
  s.bootstrap = bootstrap ? 1 : 0;
  if (r->centralized) {  // Env::world_state of the current states (ppo.cpp:341-346)
    if (marl_venv_world_state(h, r->ws) != MARL_OK) raise(MARL_ERR_CUDA, marl_last_error());
    s.ws = r->ws;
  }
  s.legal_ready = (!bootstrap && e.family == MARL_FAMILY_SMAX) ? 1 : 0;
  if (s.legal_ready)  // Env::legal_actions straight into the buffer slice (team.cpp:35-42)
    smax_launch_legal(e.smax, h->smax, h->n, r->n_act, r->b.legal + size_t(t) * size_t(r->R) * r->n_act, h->stream);
  if (r->recurrent && r->rnn_gemm) {
    rnn_collect_gemm(r, s);
  } else if (r->recurrent) {
    RnnPolicyArgs ra{};
    ra.actor = r->params;
    ra.critic = r->params + r->n_actor;
    ra.h_actor = r->h_actor;
    ra.h_critic = r->h_critic;
    ra.in_dim = r->in_dim;
    ra.critic_in = r->critic_in;
    ra.n_act = r->n_act;
    ra.F = r->F;
    ra.H = r->H;
    ra.relu = r->relu;
    rnn_policy(ra, s, r->b, h->stream);
  } else if (r->precision == 1) {
    rollout_policy_bf16(net_of(r), net_bf16_of(r), s, r->b, h->stream);
  } else {
    rollout_policy_fp32(net_of(r), s, r->b, h->stream);
  }
  after_launch();
}

}  // namespace

extern "C" {

int marl_rollout_policy_spec(const marl_venv* h, int width, int n_layers, int relu, int centralized,
                             marl_policy_spec* out) {
  return guarded([&] {
    if (!h || !out) raise(MARL_ERR_CONTRACT, "marl_rollout_policy_spec: NULL argument");
    if (n_layers != 2) raise(MARL_ERR_SCHEMA, "rollout: the B200 policy kernels implement n_fc_layers = 2");
    if (width < 1 || width > 64) raise(MARL_ERR_SCHEMA, "rollout: fc_width must be in [1, 64]");
    *out = marl_policy_spec{};
    policy_dims(h, width, centralized, &out->in_dim, &out->critic_in, &out->n_actions, &out->n_actor_params,
                &out->n_critic_params);
    out->width = width;
    out->n_layers = n_layers;
    out->relu = relu;
    out->rows_per_env = h->env->A;
  });
}

}  // extern "C"

namespace mhost {
// hidden > 0: the recurrent policy (RnnBranch, fc width `width`, GRU `hidden`)
marl_rollout* rollout_create_impl(marl_venv* h, int T, int width, int n_layers, int relu, int centralized,
                                         int precision, int hidden) {
    if (!h) raise(MARL_ERR_CONTRACT, "marl_rollout_create: NULL argument");
    if (T < 1) raise(MARL_ERR_CONTRACT, "rollout: n_rollout_steps must be >= 1");
    marl_policy_spec ps{};
    if (marl_rollout_policy_spec(h, width, hidden > 0 ? 2 : n_layers, relu, centralized, &ps) != MARL_OK)
      raise(MARL_ERR_SCHEMA, marl_last_error());
    if (hidden > 0) {
      if (precision != 0) raise(MARL_ERR_SCHEMA, "rollout: the recurrent policy runs in fp32 (precision 0)");
      if (hidden > 128) raise(MARL_ERR_SCHEMA, "rollout: hidden_width must be in [1, 128]");
      ps.n_actor_params = rnn_branch_params(ps.in_dim, width, hidden, ps.n_actions);
      ps.n_critic_params = rnn_branch_params(ps.critic_in, width, hidden, 1);
    }
    if (h->env->continuous)
      raise(MARL_ERR_SCHEMA, "rollout: the PPO policy is categorical; box action spaces are not supported");
    if (ps.critic_in > 1024) raise(MARL_ERR_SCHEMA, "rollout: critic input wider than 1024");
    if (ps.in_dim > 1024 || ps.n_actions > 64) raise(MARL_ERR_SCHEMA, "rollout: input wider than 1024 or > 64 actions");
    if (precision == 1 && !rollout_policy_bf16_supported(ps.in_dim, ps.n_actions, width, centralized ? ps.critic_in : 0))
      raise(MARL_ERR_SCHEMA, "rollout: the tcgen05 bf16 policy needs in_dim (and the MAPPO critic's world_state) <= "
                             "192 and n_actions <= 16 (wider IPPO rows: <= 1024 with n_actions <= 64), fc_width == 64");
    if (precision != 0 && precision != 1) raise(MARL_ERR_SCHEMA, "rollout: precision must be 0 (fp32) or 1 (bf16)");
    set_device(h);
    auto r = std::make_unique<marl_rollout>();
    r->h = h;
    r->T = T;
    const Env& e = *h->env;
    r->R = h->n * e.A;
    r->row0 = h->off * e.A;
    r->R_global = h->gn * e.A;
    r->in_dim = ps.in_dim;
    r->critic_in = ps.critic_in;
    r->centralized = centralized ? 1 : 0;
    r->n_act = ps.n_actions;
    r->width = width;
    r->relu = relu;
    r->precision = precision;
    r->n_actor = ps.n_actor_params;
    r->n_critic = ps.n_critic_params;
    for (size_t k = 0; k < e.info_names.size(); ++k)
      if (e.info_names[k] == "shaped_reward") r->shaped_idx = int(k);
    const size_t TR = size_t(T) * size_t(r->R);
    Arena& ar = r->arena;
    ar.add(&r->b.obs, TR * size_t(r->in_dim));
    ar.add(&r->b.actions, TR);
    ar.add(&r->b.rewards, TR);
    ar.add(&r->b.dones, TR);
    ar.add(&r->b.resets, TR);
    ar.add(&r->b.logp, TR);
    ar.add(&r->b.value, TR);
    ar.add(&r->b.legal, TR * size_t(r->n_act));
    ar.add(&r->b.active, TR);
    ar.add(&r->b.adv, TR);
    ar.add(&r->b.vtarg, TR);
    ar.add(&r->b.last_value, size_t(r->R));
    if (r->centralized) {
      ar.add(&r->b.critic_in, TR * size_t(r->critic_in));
      ar.add(&r->ws, size_t(h->n) * size_t(r->critic_in));
    }
    ar.add(&r->params, size_t(r->n_actor + r->n_critic));
    ar.add(&r->images, size_t(128 * rollout_tc_kx(ps.in_dim) + 2 * 64 * 64 + 64 * 64 + 16 * 64 +
                              (centralized ? 64 * ((ps.critic_in + 15) / 16 * 16) : 0)));
    ar.add(&r->bias, size_t(4 * 64 + 2 * 16 + 64));
    ar.add(&r->agent_actions, size_t(e.A));
    if (hidden > 0) {
      r->recurrent = 1;
      r->F = width;
      r->H = hidden;
      for (float** q : {&r->h_actor, &r->h_critic, &r->h0_actor, &r->h0_critic})
        ar.add(q, size_t(r->R) * size_t(hidden));
      ar.add(&r->critic_al, size_t(r->n_critic));
      const char* mode = std::getenv("MARL_RNN_COLLECT");
      r->rnn_gemm = mode ? std::string(mode) == "gemm" : r->R >= 4096;
      if (r->rnn_gemm) {
        const size_t R = size_t(r->R);
        ar.add(&r->s_xa, R * r->in_dim);
        ar.add(&r->s_xc, R * r->critic_in);
        ar.add(&r->s_e, R * width);
        ar.add(&r->s_p, R * width);
        ar.add(&r->s_gx, R * 3 * hidden);
        ar.add(&r->s_gh, R * 3 * hidden);
        ar.add(&r->s_ya, R * r->n_act);
        ar.add(&r->s_yc, R);
        ar.add(&r->s_hpeek, R * hidden);
      }
    }
    ar.commit();
    cuda_check(cudaMemcpy(r->agent_actions, e.n_actions.data(), size_t(e.A) * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    return r.release();
}
}  // namespace mhost

extern "C" {

int marl_rollout_create(marl_venv* h, int T, int width, int n_layers, int relu, int centralized, int precision,
                        marl_rollout** out) {
  return guarded([&] {
    if (!out) raise(MARL_ERR_CONTRACT, "marl_rollout_create: NULL argument");
    *out = rollout_create_impl(h, T, width, n_layers, relu, centralized, precision, 0);
  });
}

int marl_rollout_set_params(marl_rollout* r, const float* actor, const float* critic) {
  return guarded([&] {
    if (!r || !actor || !critic) raise(MARL_ERR_CONTRACT, "marl_rollout_set_params: NULL argument");
    set_device(r->h);
    cuda_check(cudaMemcpy(r->params, actor, size_t(r->n_actor) * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    cuda_check(cudaMemcpy(r->params + r->n_actor, critic, size_t(r->n_critic) * 4, cudaMemcpyHostToDevice),
               "cudaMemcpy");
    if (r->precision == 1) {
      rollout_pack_bf16(net_of(r), r->images, r->bias, r->h->stream);
      after_launch();
    }
    r->has_params = true;
  });
}

// Collector constructor (ppo.cpp:189-192): reset with fold_in(key, 1), act_key
// = fold_in(key, 2), every row starts an episode.
int marl_rollout_begin(marl_rollout* r, const uint32_t key[4]) {
  return guarded([&] {
    if (!r || !key) raise(MARL_ERR_CONTRACT, "marl_rollout_begin: NULL argument");
    uint32_t rk[4];
    marl_prng_fold_in(key, 1, rk);
    if (marl_venv_reset(r->h, rk) != MARL_OK) raise(MARL_ERR_CUDA, marl_last_error());
    marl_prng_fold_in(key, 2, r->act_key);
    if (r->recurrent) {  // fresh Collector: zero hidden states (ppo.cpp:194-198)
      cuda_check(cudaMemset(r->h_actor, 0, size_t(r->R) * size_t(r->H) * 4), "cudaMemset");
      cuda_check(cudaMemset(r->h_critic, 0, size_t(r->R) * size_t(r->H) * 4), "cudaMemset");
    }
    r->begun = true;
    r->first = true;
  });
}

}  // extern "C"


extern "C" {

int marl_rollout_collect(marl_rollout* r, int64_t seq_base, double gamma, double lambda, double shaping) {
  return guarded([&] {
    if (!r) raise(MARL_ERR_CONTRACT, "marl_rollout_collect: NULL rollout");
    collect_impl(r, seq_base, gamma, lambda, [shaping](int64_t) { return shaping; });
  });
}

int marl_rollout_get_views(marl_rollout* r, marl_rollout_views* o) {
  return guarded([&] {
    if (!r || !o) raise(MARL_ERR_CONTRACT, "marl_rollout_get_views: NULL argument");
    o->obs = r->b.obs;
    o->actions = r->b.actions;
    o->rewards = r->b.rewards;
    o->dones = r->b.dones;
    o->resets = r->b.resets;
    o->logp = r->b.logp;
    o->value = r->b.value;
    o->legal = r->b.legal;
    o->active = r->b.active;
    o->adv = r->b.adv;
    o->vtarg = r->b.vtarg;
    o->last_value = r->b.last_value;
    o->critic_in = r->b.critic_in;
    o->critic_dim = r->critic_in;
    o->T = r->T;
    o->R = r->R;
    o->in_dim = r->in_dim;
    o->n_actions = r->n_act;
  });
}

int marl_rollout_destroy(marl_rollout* r) {
  return guarded([&] {
    if (!r) return;
    set_device(r->h);
    cudaStreamSynchronize(r->h->stream);
    delete r;
  });
}

}  // extern "C"

