// Internal header of the host side of the C-ABI (not installed): the error
// and config helpers, the resolved env description, the device arena, the
// handle structs behind the opaque C types (marl_venv, marl_rollout,
// marl_ppo) and the functions the host translation units share:
//   venv.cpp         registry, env configs, VectorEnv entry points
//   rollout_host.cpp the IPPO / MAPPO collector (marl_rollout_*)
//   ppo_host.cpp     the trainer (marl_ppo_*), NCCL and cuBLAS loaders
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "common.cuh"
#include "engine.h"
#include "marl_b200.h"

namespace mhost {
using nlohmann::json;
using namespace marl_b200;

extern thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(MARL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MARL_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const json::exception& e) {
    g_err = std::string("config is not valid JSON: ") + e.what();
    return MARL_ERR_SCHEMA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MARL_ERR_INTERNAL;
  }
}

// ---------------------------------------------------------------------------
// Strict typed config reader, same contract as marl::ConfigView
// (config.hpp:19-110): every key read is recorded, leftovers are SchemaError.
class ConfigView {
 public:
  ConfigView(const json& cfg, std::string ctx) : cfg_(cfg), ctx_(std::move(ctx)) {
    if (!cfg_.is_object() && !cfg_.is_null()) raise(MARL_ERR_SCHEMA, ctx_ + ": expected a JSON object");
  }
  bool has(const std::string& k) const { return cfg_.is_object() && cfg_.contains(k); }
  int64_t get_int64(const std::string& k, int64_t dflt) {
    seen_.insert(k);
    if (!has(k)) return dflt;
    const json& v = cfg_.at(k);
    if (!v.is_number_integer() && !v.is_number_unsigned()) bad(k, "integer");
    return v.get<int64_t>();
  }
  int get_int(const std::string& k, int dflt) {
    seen_.insert(k);
    if (!has(k)) return dflt;
    const json& v = cfg_.at(k);
    if (!v.is_number_integer() && !v.is_number_unsigned()) bad(k, "integer");
    return v.get<int>();
  }
  double get_double(const std::string& k, double dflt) {
    seen_.insert(k);
    if (!has(k)) return dflt;
    const json& v = cfg_.at(k);
    if (!v.is_number()) bad(k, "number");
    return v.get<double>();
  }
  bool get_bool(const std::string& k, bool dflt) {
    seen_.insert(k);
    if (!has(k)) return dflt;
    const json& v = cfg_.at(k);
    if (!v.is_boolean()) bad(k, "boolean");
    return v.get<bool>();
  }
  std::string get_string(const std::string& k, const std::string& dflt) {
    seen_.insert(k);
    if (!has(k)) return dflt;
    const json& v = cfg_.at(k);
    if (!v.is_string()) bad(k, "string");
    return v.get<std::string>();
  }
  std::vector<std::string> get_string_list(const std::string& k) {
    seen_.insert(k);
    std::vector<std::string> out;
    if (!has(k)) return out;
    const json& v = cfg_.at(k);
    if (!v.is_array()) raise(MARL_ERR_SCHEMA, ctx_ + ": key '" + k + "' must be an array of strings");
    for (const auto& e : v) {
      if (!e.is_string()) raise(MARL_ERR_SCHEMA, ctx_ + ": key '" + k + "' must be an array of strings");
      out.push_back(e.get<std::string>());
    }
    return out;
  }
  json get_object(const std::string& k) {
    seen_.insert(k);
    if (!has(k)) return json::object();
    const json& v = cfg_.at(k);
    if (!v.is_object()) raise(MARL_ERR_SCHEMA, ctx_ + ": key '" + k + "' must be an object");
    return v;
  }
  void check_no_extras() const {
    if (!cfg_.is_object()) return;
    for (const auto& it : cfg_.items())
      if (!seen_.count(it.key())) raise(MARL_ERR_SCHEMA, ctx_ + ": unknown key '" + it.key() + "'");
  }

 private:
  [[noreturn]] void bad(const std::string& k, const char* type) const {
    raise(MARL_ERR_SCHEMA, ctx_ + ": key '" + k + "' must be a " + type);
  }
  json cfg_;
  std::string ctx_;
  std::set<std::string> seen_;
};

// ---------------------------------------------------------------------------
struct Env {  // resolved make_env(id, config)
  std::string id;
  int family = 0;
  int A = 0, D = 0, n_info = 0, max_steps = 0;
  bool cooperative = false;
  std::vector<std::string> agents, info_names;
  std::vector<int> obs_size, n_actions;  // n_actions: discrete n, or the box's flat size
  bool continuous = false;               // box action spaces (continuous MPE)
  MpeConfig mpe{};
  SmaxConfig smax{};
  OcConfig oc{};
  std::vector<float> oc_templ;
};

// ---------------------------------------------------------------------------
struct Arena {  // one device allocation per handle, carved 256-byte aligned
  uint8_t* base = nullptr;
  size_t size = 0, used = 0;
  std::vector<std::pair<void**, size_t>> reqs;
  template <class T>
  void add(T** p, size_t count) {
    reqs.push_back({reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)});
  }
  void commit() {
    size = 0;
    for (auto& r : reqs) size += (r.second + 255) & ~size_t(255);
    cuda_check(cudaMalloc(&base, size), "cudaMalloc");
    cuda_check(cudaMemset(base, 0, size), "cudaMemset");
    size_t off = 0;
    for (auto& r : reqs) {
      *r.first = base + off;
      off += (r.second + 255) & ~size_t(255);
    }
  }
  ~Arena() {
    if (base) cudaFree(base);
  }
};

}  // namespace mhost

// the handle structs behind the C-ABI's opaque types (global namespace)
using namespace marl_b200;
using mhost::Arena;
using mhost::Env;

struct marl_venv {
  std::unique_ptr<Env> env;
  int device = 0;
  int64_t n = 0, off = 0, gn = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool has_state = false;
  Arena arena;
  StepViews v{};
  Carry carry{};
  unsigned long long* stats = nullptr;
  int* err = nullptr;
  int32_t* n_actions_dev = nullptr;
  int32_t* ws_seg = nullptr;  // world_state gather segments: [src offsets | lengths] (MPE, Overcooked)
  int ws_nseg = 0, ws_width = 0;
  MpeState mpe{};
  SmaxState smax{};
  OcState oc{};
  float* oc_templ = nullptr;
  std::vector<int32_t> host_actions_scratch;
  cudaStream_t copy_stream = nullptr;  // host-buffer steps: D2H of finished chunks
  cudaEvent_t chunk_ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

struct marl_rollout {
  marl_venv* h = nullptr;
  int T = 0;
  int64_t R = 0, R_global = 0, row0 = 0;
  int in_dim = 0, n_act = 0, width = 64, relu = 0, precision = 0;
  int critic_in = 0, centralized = 0;
  float* ws = nullptr;  // [E][critic_in] world_state scratch (MAPPO)
  int n_actor = 0, n_critic = 0, shaped_idx = -1;
  Arena arena;
  RolloutBufs b{};
  float* params = nullptr;     // packed actor | critic (fp32, nn::pack order)
  float* critic_al = nullptr;  // recurrent: a 16-byte-aligned copy of the critic's parameters (rnn_critic_params)
  uint16_t* images = nullptr;  // bf16 UMMA operand images (tcgen05 path)
  float* bias = nullptr;
  int32_t* agent_actions = nullptr;
  uint32_t act_key[4] = {0, 0, 0, 0};
  bool has_params = false, begun = false, first = true;
  // recurrent (GRU) policy: embed F, hidden H (ppo.hpp:52-53); carried hidden
  // states and their copy at the window start (Rollout::h0_*, ppo.cpp:175, 219-222)
  int recurrent = 0, F = 0, H = 0;
  float *h_actor = nullptr, *h_critic = nullptr, *h0_actor = nullptr, *h0_critic = nullptr;
  // GEMM-structured acting step (R >= 4096 rows, or MARL_RNN_COLLECT=gemm|rows)
  bool rnn_gemm = false;
  float *s_xa = nullptr, *s_xc = nullptr, *s_e = nullptr, *s_gx = nullptr, *s_gh = nullptr, *s_p = nullptr,
        *s_ya = nullptr, *s_yc = nullptr, *s_hpeek = nullptr;
};

namespace mhost {
// The recurrent critic's parameters for the 3xTF32 GEMMs: params + n_actor
// when that is 16-byte aligned, else a fresh aligned copy (the GEMMs' staging
// falls back to 4-byte copies on a misaligned weight operand: 25-30 % slower)
inline const float* rnn_critic_params(marl_rollout* r, cudaStream_t st) {
  const float* c = r->params + r->n_actor;
  if (reinterpret_cast<uintptr_t>(c) % 16 == 0 || !r->critic_al) return c;
  cuda_check(cudaMemcpyAsync(r->critic_al, c, size_t(r->n_critic) * 4, cudaMemcpyDeviceToDevice, st),
             "cudaMemcpyAsync (aligned critic)");
  return r->critic_al;
}

struct PpoCfg {  // PpoConfig (ppo.hpp:30-55) with its defaults
  int64_t total_timesteps = 1000000;
  int n_envs = 16, n_rollout_steps = 128;
  double lr = 5e-4;
  bool anneal_lr = true;
  int update_epochs = 5, n_minibatches = 2;
  double gamma = 0.99, gae_lambda = 1.0, clip_eps = 0.3, ent_coef = 0.01, vf_coef = 1.0, max_grad_norm = 0.5;
  std::string activation = "tanh";
  bool recurrent = false;
  int n_fc_layers = 2, fc_width = 64, hidden_width = 128;
  bool shaped_rewards = true;
};
}  // namespace mhost

using mhost::PpoCfg;

struct marl_ppo {
  marl_venv* h = nullptr;
  marl_rollout* ro = nullptr;
  PpoCfg cfg;
  int centralized = 0, precision = 0;
  int64_t n_updates = 0, update = 0, adam_t = 0, batch = 0, per = 0;
  uint32_t train_key[4] = {0, 0, 0, 0};
  double last_mean_return = 0.0;
  int64_t window_episodes = 0;
  double window_return = 0.0;
  bool begun = false, collected = false;
  Arena arena;
  int P = 0, Pa = 0, Pc = 0, grid_a = 0, grid_c = 0;
  bool tc = false;  // minibatch step on tcgen05 (bf16 precision, IPPO width 64, input <= 191)
  uint16_t* obs_bf = nullptr;      // [T*R][kx] bf16 observation rows of the window (tcgen05 step)
  PpoRowRec* rows_rec = nullptr;   // [T*R] their loss-input records
  float *m = nullptr, *v = nullptr, *grad = nullptr, *snapshot = nullptr, *gpart_a = nullptr, *gpart_c = nullptr;
  double *spart_a = nullptr, *spart_c = nullptr, *adv_part = nullptr, *adv_part2 = nullptr, *metrics = nullptr;
  PpoMbStats* mbst = nullptr;
  int32_t* perm = nullptr;
  uint8_t* perm_scratch = nullptr;
  size_t perm_scratch_bytes = 0;
  int* flags = nullptr;  // [0] diverged, [1] illegal stored action
  // data-parallel update over env shards: the global permutation's rows this
  // shard owns; sums all-reduced through `hook` (a callback or native NCCL)
  bool sharded = false;
  int64_t R_local = 0, R_global = 0, row0 = 0;
  int32_t *cmp_tmp = nullptr, *cmp_out = nullptr;
  int64_t* cmp_count = nullptr;
  uint8_t* cmp_scratch = nullptr;
  size_t cmp_scratch_bytes = 0;
  double* adv_g = nullptr;      // [4] advantage sums (all-reduced)
  int64_t* ep_dev = nullptr;    // [3] episode statistics (all-reduced)
  marl_allreduce_fn hook = nullptr;
  void* hook_ctx = nullptr;
  void* nccl_comm = nullptr;
  // recurrent update (rnn_minibatch, ppo.cpp:444-509): BPTT caches for one minibatch
  bool recurrent = false;
  RnnCache rca{}, rcc{};
  int32_t* rnn_flat = nullptr;
  int64_t rnn_chunk = 0;  // rows per BPTT chunk (caches sized for it)
  int rnn_blocks = 0;     // loss partial blocks of the last minibatch
  float *rnn_h = nullptr, *rnn_gx = nullptr, *rnn_gh = nullptr, *rnn_dh = nullptr, *rnn_ones = nullptr;
  // wide-input fp32 update (ff_minibatch as a GEMM chain, minibatch_grad_wide):
  // per branch the gathered rows, both hidden layers and the head's output and
  // gradient, one [M][W] pair for the backward's layer gradients
  float2* adv_gath = nullptr;  // [per] the minibatch's gathered (adv, active): the variance pass reads them in order
  const float* rnn_critic_w = nullptr;  // the critic's (aligned) parameters for this minibatch
  bool wide = false;
  float* wx[2] = {nullptr, nullptr};  // [M][ldx]: the actor's rows, the critic's (== wx[0] for IPPO)
  int wldx[2] = {0, 0};
  // [M][2W], actor columns then critic columns: hidden layers and their gradients
  float *wh1 = nullptr, *wh2 = nullptr, *wd1 = nullptr, *wd2 = nullptr;
  float *wy[2] = {nullptr, nullptr}, *wdy[2] = {nullptr, nullptr};  // head outputs / gradients [M][out]
  float *wq[2] = {nullptr, nullptr};  // aligned parameter copies
  float *w1s = nullptr, *wbias = nullptr, *wg1 = nullptr;  // stacked W1 [2W][ldx], biases [4W], dW1 [2W][in]
  float* wpart = nullptr;  // column-sum partials
  ~marl_ppo();
};

namespace mhost {

// venv.cpp
void set_device(const marl_venv* h);
LaunchCommon common(marl_venv* h);
void after_launch();
void require_state(const marl_venv* h);
void check_device_error(marl_venv* h);
// d_actions: [N][A] int32 ids, or [N][A][kBoxActDim] floats for box action spaces
void launch_step(marl_venv* h, bool random, const uint32_t* step_key, const void* d_actions, int64_t begin = 0,
                 int64_t end = -1);
void download_range(marl_venv* h, const marl_host_step* o, int64_t b, int64_t e, cudaStream_t st);
void step_to_host(marl_venv* h, bool random, const uint32_t* step_key, const void* d_actions,
                  const marl_host_step* o);
void download(marl_venv* h, const marl_host_step* o);

// rollout_host.cpp
void policy_dims(const marl_venv* h, int width, int centralized, int* in_dim, int* critic_in, int* n_act,
                 int* n_actor, int* n_critic);
PolicyNet net_of(const marl_rollout* r);
PolicyNetBf16 net_bf16_of(const marl_rollout* r);
void run_policy(marl_rollout* r, int t, bool bootstrap, int64_t seq_base);
// hidden > 0: the recurrent policy (RnnBranch, fc width `width`, GRU `hidden`)
marl_rollout* rollout_create_impl(marl_venv* h, int T, int width, int n_layers, int relu, int centralized,
                                  int precision, int hidden);

// ppo_host.cpp: row-major GEMM helpers over the 3xTF32 tcgen05 kernel (gemm_tc.cu)
void gemm_nt(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta);
void gemm_nn(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta);
void gemm_tn(cudaStream_t st, int O, int I, int64_t K, const float* D, int ldd, const float* X, int ldx, float* G,
             float beta);
void colsum(cudaStream_t st, int O, int64_t K, const float* D, int ldd, const float* ones, float* g, float beta);

// Collector::collect(nets, T, seq_base, shaping_at) (ppo.cpp:206-323);
// shaping(seq) is the annealed shaped-reward weight of batch step seq.
template <class Shaping>
void collect_impl(marl_rollout* r, int64_t seq_base, double gamma, double lambda, Shaping shaping) {
  if (!r->begun) raise(MARL_ERR_CONTRACT, "rollout: call begin() before collect()");
  if (!r->has_params) raise(MARL_ERR_CONTRACT, "rollout: call set_params() before collect()");
  marl_venv* h = r->h;
  set_device(h);
  const Env& e = *h->env;
  if (r->recurrent) {  // ro.h0_* = the hidden states at the window start (ppo.cpp:219-222)
    const size_t bytes = size_t(r->R) * size_t(r->H) * 4;
    cuda_check(cudaMemcpyAsync(r->h0_actor, r->h_actor, bytes, cudaMemcpyDeviceToDevice, h->stream), "D2D");
    cuda_check(cudaMemcpyAsync(r->h0_critic, r->h_critic, bytes, cudaMemcpyDeviceToDevice, h->stream), "D2D");
  }
  for (int t = 0; t < r->T; ++t) {
    run_policy(r, t, false, seq_base);
    launch_step(h, false, nullptr, r->b.actions + size_t(t) * size_t(r->R));
    rollout_record(r->b, t, r->R, e.A, h->v.rewards, h->v.infos, e.n_info, r->shaped_idx, shaping(seq_base + t),
                   h->v.finished, h->stream);
    after_launch();
    r->first = false;
  }
  run_policy(r, r->T, true, seq_base);  // bootstrap values (ppo.cpp:285-299)
  rollout_gae(r->b, r->T, r->R, float(gamma), float(lambda), h->stream);
  after_launch();
}

}  // namespace mhost
