/* marl-b200: C-ABI of the B200-native batched multi-agent env engine.
 *
 * Drop-in boundary for the reference's batched hot path, marl::VectorEnv
 * (/root/reference/proj/core/include/marl/vector_env.hpp:74-89,
 *  /root/reference/proj/core/src/vector_env.cpp:45-129) and the env registry
 * that feeds it (registry.hpp:16-28).  Plain pointers and sizes only; no C++
 * or torch types cross this boundary.
 *
 * Data model (per handle, N local envs, A agents, D = max obs size):
 *   the reference's per-env AgentMap<...> dictionaries (agent_map.hpp:14-65)
 *   are flattened to fixed-width arrays in agent order:
 *     obs, final_obs    [N][A][D] f32   (rows of smaller agents zero-padded)
 *     rewards           [N][A]    f64
 *     dones             [N][A+1]  u8    (per agent, then "__all__")
 *     finished          [N]       u8    (dones["__all__"])
 *     final_returns     [N]       f64,  final_lengths [N] i32
 *     infos             [N][A][n_info] f64 (fields in std::map key order,
 *                                  see marl_venv_info_name; episode_return /
 *                                  episode_length live in final_returns /
 *                                  final_lengths)
 *     actions           [N][A]    i32
 *     keys              [N][4]    u32   (k0, k1, c0, c1 of the carry key)
 *     episode_returns   [N] f64, episode_lengths [N] i32
 * All view pointers are DEVICE pointers owned by the handle and valid until
 * the next call on it.  final_obs rows are written only where finished.
 *
 * Threading: one caller thread per handle; work is queued on the handle's
 * CUDA stream and is asynchronous until marl_venv_sync / a *_host call.
 *
 * Errors: every call returns a status (the reference's exception taxonomy,
 * errors.hpp:9-26); the message of the last failure on the calling thread is
 * marl_last_error().  Device-side action validation (marl_venv_step) reports
 * at the next synchronising call; the rejected batch leaves the state as it
 * was, like the reference's ContractError from Env::validate_actions
 * (env.cpp:7-14).
 */
#ifndef MARL_B200_H
#define MARL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum marl_status {
  MARL_OK = 0,
  MARL_ERR_NOT_FOUND = 1,   /* NotFoundError   (errors.hpp:9-12)  */
  MARL_ERR_SCHEMA = 2,      /* SchemaError     (errors.hpp:14-17) */
  MARL_ERR_CONTRACT = 3,    /* ContractError   (errors.hpp:19-22) */
  MARL_ERR_DIVERGENCE = 4,  /* DivergenceError (errors.hpp:24-27) */
  MARL_ERR_CUDA = 5,
  MARL_ERR_INTERNAL = 6
};

enum marl_family { MARL_FAMILY_MPE = 0, MARL_FAMILY_SMAX = 1, MARL_FAMILY_OVERCOOKED = 2 };

typedef struct marl_venv marl_venv;

typedef struct {
  int32_t family;       /* marl_family */
  int32_t n_agents;     /* Env::num_agents (env.hpp:46) */
  int32_t obs_dim;      /* max observation_space(agent).flat_size() */
  int32_t n_actions;    /* max action_space(agent).n */
  int32_t n_info;       /* f64 info fields per agent */
  int32_t max_steps;    /* Env::max_steps (env.hpp:59) */
  int32_t cooperative;  /* Env::cooperative (env.hpp:62) */
  int32_t device;
  int64_t n_envs;       /* local envs of this handle */
  int64_t global_offset;/* global index of local env 0 */
  int64_t global_n;     /* envs in the whole (possibly multi-GPU) batch */
} marl_spec;

typedef struct { /* device pointers, see the data model above */
  float* obs;
  double* rewards;
  uint8_t* dones;
  uint8_t* finished;
  float* final_obs;
  double* final_returns;
  int32_t* final_lengths;
  double* infos;
  int32_t* actions;
  uint32_t* keys;
  double* episode_returns;
  int32_t* episode_lengths;
} marl_views;

/* Host destinations for *_host / download calls; NULL = skip.  final_obs is
 * valid where finished (vector_env.hpp:31): when it points into mapped pinned
 * memory (cudaHostAlloc / torch pin_memory) the device writes only the
 * finished rows into it, else the whole view is copied. */
typedef struct {
  float* obs;
  double* rewards;
  uint8_t* dones;
  uint8_t* finished;
  float* final_obs;
  double* final_returns;
  int32_t* final_lengths;
  double* infos;
  int32_t* actions;
} marl_host_step;

/* ---- registry (registry.hpp:16-28) ----------------------------------- */

/* Number of env ids this engine implements; id i via marl_registered_env.
 * Replaces registered_envs() (registry.cpp:99-106). */
int marl_registered_count(void);
const char* marl_registered_env(int i);

/* make_env(env_id, config) alone (registry.cpp:83-97): resolve and validate
 * the id and config and report the env's spec (n_envs fields zero) without
 * touching a GPU.  Same errors as marl_venv_create. */
int marl_env_describe(const char* env_id, const char* config_json, marl_spec* out);
int marl_env_agent(const char* env_id, const char* config_json, int i, char* name, size_t cap,
                   int32_t* obs_size, int32_t* n_actions);

/* ---- lifecycle: make_env + VectorEnv ctor ------------------------------ */

/* make_env(env_id, config) (registry.cpp:83-97) + VectorEnv(env, n_envs)
 * (vector_env.cpp:45-49) on CUDA device `device`.  config_json may be NULL or
 * "" for the defaults; unknown keys are SchemaError (config.hpp:78-83). */
int marl_venv_create(const char* env_id, const char* config_json, int64_t n_envs, int device,
                     marl_venv** out);

/* Shard constructor for multi-GPU batches: this handle owns global envs
 * [global_offset, global_offset + n_local) of a global_n-env batch; per-env
 * keys derive from global indices (vector_env.cpp:52,55,171), so any sharding
 * reproduces the single-device trajectories bit for bit. */
int marl_venv_create_shard(const char* env_id, const char* config_json, int64_t n_local,
                           int64_t global_offset, int64_t global_n, int device, marl_venv** out);

int marl_venv_destroy(marl_venv* h);

/* Queue work on an external cudaStream_t (e.g. the framework's current
 * stream) instead of the handle's own stream. */
int marl_venv_set_stream(marl_venv* h, void* cuda_stream);

/* ---- spaces / metadata (env.hpp:43-82) --------------------------------- */

int marl_venv_spec(const marl_venv* h, marl_spec* out);
/* agents()[i], observation_space(agent).flat_size(), action_space(agent).n */
int marl_venv_agent(const marl_venv* h, int i, char* name, size_t cap, int32_t* obs_size,
                    int32_t* n_actions);
int marl_venv_info_name(const marl_venv* h, int k, char* name, size_t cap);
int marl_venv_id(const marl_venv* h, char* name, size_t cap); /* Env::id() */

/* ---- hot path ----------------------------------------------------------- */

/* VectorEnv::reset(key) (vector_env.cpp:51-70): reset keys split(key, N)[g],
 * carry keys split(fold_in(key, 1), N)[g]; writes obs + carry views. */
int marl_venv_reset(marl_venv* h, const uint32_t key[4]);

/* VectorEnv::step(state, actions) (vector_env.cpp:72-129) with caller actions
 * in DEVICE memory, [N][A] i32.  Step, team-return bookkeeping, auto-reset
 * with the per-env child keys, all in one kernel. */
int marl_venv_step(marl_venv* h, const int32_t* d_actions);

/* One step of throughput_probe's loop (vector_env.cpp:214-217):
 * random_legal_actions(state, step_key) (vector_env.cpp:169-187) fused into
 * the step kernel.  The drawn actions land in views.actions. */
int marl_venv_step_random(marl_venv* h, const uint32_t step_key[4]);

/* n_steps consecutive iterations of throughput_probe's loop (vector_env.cpp:
 * 202-217): iteration k draws random-legal actions with
 * split(parent, t0 + k)[g] -- parent = fold_in(key, 2), the probe's
 * action-key parent -- and steps.  The same outputs as n_steps calls of
 * marl_venv_step_random with those keys (the views hold the last step's);
 * MPE runs all n_steps in one kernel launch with the env state in registers. */
int marl_venv_probe_steps(marl_venv* h, const uint32_t parent[4], uint64_t t0, int n_steps);

/* Host-buffer variants (the end-to-end path): host actions are validated on
 * the host exactly like Env::validate_actions, copied in, stepped, and the
 * requested outputs copied back; returns after the copies complete. */
int marl_venv_step_host(marl_venv* h, const int32_t* h_actions, const marl_host_step* out);
int marl_venv_step_random_host(marl_venv* h, const uint32_t step_key[4], const marl_host_step* out);
/* Copy the current views to host memory (synchronising). */
int marl_venv_download(marl_venv* h, const marl_host_step* out);

int marl_venv_views(marl_venv* h, marl_views* out);
/* Box action spaces (MPE continuous_actions, mpe.cpp:91-99): actions are [N][A][action_dim] f32,
 * agent a's first n_actions[a] entries in [0, 1] (SpaceDescriptor::contains, spaces.cpp:36-46),
 * the rest padding.  action_dim = 0 for discrete envs.  marl_venv_step_random draws
 * space.sample(fold_in(env_key, j)) (vector_env.cpp:179-181) into the f32 action view. */
int marl_venv_action_dim(const marl_venv* h, int32_t* out);
int marl_venv_actions_f32(marl_venv* h, float** out);                 /* device [N][A][action_dim] */
int marl_venv_step_continuous(marl_venv* h, const float* d_actions);  /* VectorEnv::step, device */
int marl_venv_step_continuous_host(marl_venv* h, const float* h_actions, const marl_host_step* out);
/* Synchronous copy of `bytes` from a device pointer (e.g. a marl_views field)
 * to host memory: lets C/C++ callers without the CUDA runtime read views
 * (used by the reference-side adapter include/marl_b200_vector_env.hpp). */
int marl_copy_device_to_host(void* dst, const void* src, size_t bytes);

/* Env::legal_actions (env.hpp:71-73; smax.cpp:195-211) for the current
 * state: d_out [N][A][n_actions] u8 (device). */
int marl_venv_legal(marl_venv* h, uint8_t* d_out);
/* Env::world_state (smax.cpp:272-289, mpe.cpp:229-242, overcooked.cpp:315-319)
 * of the current per-env states -- the MAPPO critic input: d_out [N][W] f32
 * (device), W from marl_venv_world_state_size (Env::world_state_size). */
int marl_venv_world_state_size(const marl_venv* h, int32_t* out);
int marl_venv_world_state(marl_venv* h, float* d_out);
/* Env::state_hash (mpe.cpp:254-269, smax.cpp:312-337, overcooked.cpp:348-364)
 * of the current per-env states: d_out [N] u64 (device). */
int marl_venv_state_hash(marl_venv* h, uint64_t* d_out);

/* Episode statistics accumulated over finished episodes since the last
 * clear: out[0] episodes, out[1] sum of final_lengths, out[2] sum of
 * final_returns in 2^-24 fixed point (exact, order-independent -> identical
 * totals for any GPU count; reduce across ranks with one integer allreduce). */
int marl_venv_episode_stats(marl_venv* h, int64_t out[3], int clear);

int marl_venv_sync(marl_venv* h);

/* ---- IPPO rollout collection (config 5) -------------------------------
 * The reference's Collector (proj/core/src/algo/ppo.cpp:178-374, private):
 * per step the actor/critic feed-forward nets (ff_forward,
 * actor_critic.hpp:49-52) over the TeamLayout rows (team.cpp:27-33), masked
 * sampling with per-row keys fold_in(act_key, (seq_base+t)*R + r)
 * (ppo.cpp:249-259), the env step, and the rollout buffer; then bootstrap
 * values and GAE (ppo.cpp:285-321).  Buffers are [T][R] (R = envs x agents),
 * device-resident, valid until the next collect. */
typedef struct marl_rollout marl_rollout;

typedef struct {
  int32_t in_dim;           /* PpoNetSpec::in_dim: padded obs + agent one-hot (ppo.cpp:80-107) */
  int32_t critic_in;        /* PpoNetSpec::critic_in: in_dim (IPPO) or world_state_size (MAPPO) */
  int32_t n_actions;        /* PpoNetSpec::n_actions (padded action head) */
  int32_t width, n_layers, relu;
  int32_t n_actor_params;   /* floats in PpoNets::pack_actor() order (nn::pack, nn.hpp:326-341) */
  int32_t n_critic_params;
  int32_t rows_per_env;     /* agents */
} marl_policy_spec;

typedef struct { /* device pointers, [T][R] row-major */
  float* obs;        /* [T][R][in_dim] */
  int32_t* actions;
  float* rewards;
  uint8_t* dones;
  uint8_t* resets;
  float* logp;
  float* value;
  uint8_t* legal;    /* [T][R][n_actions] */
  float* active;
  float* adv;
  float* vtarg;
  float* last_value; /* [R] */
  float* critic_in;  /* [T][R][critic_dim] MAPPO critic rows (NULL for IPPO: the critic reads obs) */
  int32_t critic_dim;
  int32_t T;
  int64_t R;
  int32_t in_dim, n_actions;
} marl_rollout_views;

/* ppo_net_spec(env, cfg, centralized) for fc_width/n_fc_layers/activation;
 * centralized = 1 is train_mappo's critic on Env::world_state (ppo.hpp:99). */
int marl_rollout_policy_spec(const marl_venv* h, int width, int n_layers, int relu, int centralized,
                             marl_policy_spec* out);
/* precision 0: fp32 in the reference's accumulation order (parity path);
 * precision 1: bf16 operands, fp32 accumulation on tcgen05 tensor cores. */
int marl_rollout_create(marl_venv* h, int T, int width, int n_layers, int relu, int centralized, int precision,
                        marl_rollout** out);
/* Host parameters in PpoNets::pack_actor()/pack_critic() order. */
int marl_rollout_set_params(marl_rollout* r, const float* actor, const float* critic);
/* Collector constructor (ppo.cpp:189-192): reset(fold_in(key,1)), act_key = fold_in(key,2). */
int marl_rollout_begin(marl_rollout* r, const uint32_t key[4]);
/* Collector::collect(nets, T, seq_base, shaping) (ppo.cpp:206-323) + GAE. Asynchronous. */
int marl_rollout_collect(marl_rollout* r, int64_t seq_base, double gamma, double lambda, double shaping);
int marl_rollout_get_views(marl_rollout* r, marl_rollout_views* out);
int marl_rollout_destroy(marl_rollout* r);

/* ---------------------------------------------------------------- PPO update
 * train_ippo / train_mappo (ppo.hpp:96-99, ppo.cpp:518-651) with the rollout
 * above and the minibatch update on the device:
 * PpoConfig JSON (ppo.cpp:38-62, same keys, defaults and SchemaErrors),
 * ppo_init_nets (ppo.cpp:109-124), permutation minibatches (prng.cpp:151-159),
 * ff_minibatch + ppo_row_loss + ff_backward (ppo.cpp:409-441,
 * actor_critic.hpp:340-412), clip_global_norm + Adam (nn.hpp:417-452), the
 * DivergenceError rollback (ppo.cpp:630-634) and the per-update metrics row.
 * Feed-forward and recurrent (GRU) policies. */
typedef struct marl_ppo marl_ppo;
/* n_envs in the config must equal the VectorEnv's env count. precision as marl_rollout_create. */
int marl_ppo_create(marl_venv* h, const char* ppo_config_json, int centralized, int precision, marl_ppo** out);
/* ppo_init_nets(key, spec) for a feed-forward spec into host arrays (no device needed) */
int marl_ppo_init_nets(int in_dim, int critic_in, int n_actions, int fc_width, int n_fc_layers, const uint32_t key[4],
                       float* actor, float* critic);
int marl_ppo_begin(marl_ppo* p, const uint32_t key[4]);  /* nets fold_in(key,10), collector fold_in(key,11) */
int marl_ppo_n_updates(const marl_ppo* p, int64_t* out);  /* total_timesteps / (n_envs * n_rollout_steps) */
/* 1 when the minibatch step runs on tcgen05 (precision bf16, IPPO, width 64,
 * input <= 191, <= 16 actions), 0 on the fp32 CUDA-core kernels */
int marl_ppo_tensor_core_update(const marl_ppo* p, int* out);
int marl_ppo_param_counts(const marl_ppo* p, int32_t* n_actor, int32_t* n_critic);
/* recurrent=true: RnnBranch nets (embed fc_width, GRU hidden_width, post, head; actor_critic.hpp:74-200)
 * trained by rnn_minibatch (ppo.cpp:444-509), fp32; ppo_init_nets for that spec into host arrays: */
int marl_ppo_init_rnn(int in_dim, int critic_in, int n_actions, int fc_width, int hidden_width, const uint32_t key[4],
                      float* actor, float* critic);
int marl_ppo_set_params(marl_ppo* p, const float* actor, const float* critic);
int marl_ppo_get_params(marl_ppo* p, float* actor, float* critic);
int marl_ppo_rollout(marl_ppo* p, marl_rollout** out);  /* borrowed: views of the current window */
int marl_ppo_collect(marl_ppo* p);
/* row[12] = {step, update, mean_return, n_episodes, loss, pg_loss, v_loss, entropy, approx_kl,
 * clip_frac, grad_norm, lr} (ppo.cpp:524-527); diverged = 1 after a DivergenceError rollback. */
int marl_ppo_update(marl_ppo* p, double row[12], int* diverged);
int marl_ppo_step(marl_ppo* p, double row[12], int* diverged);  /* collect + update */
/* ff_minibatch's gradient (actor | critic, nn::pack order) and {loss, pg, v, entropy, kl, clip_frac}
 * for device slot indices d_idx[M] over the current window, no optimizer step. */
int marl_ppo_minibatch_grad(marl_ppo* p, const int32_t* d_idx, int64_t M, float* grad_out, double* stats_out);
int marl_ppo_destroy(marl_ppo* p);
/* Data-parallel update over env shards (marl_venv_create_shard; n_envs = the global count): every
 * rank draws the same global permutation, keeps the minibatch rows it owns and sums advantage
 * statistics, gradient, loss sums and episode counts over the ranks -- the single-device update's
 * arithmetic, split by rows.  The exchange is an in-place SUM all-reduce: either a callback (the
 * stream is synchronised before the call; return 0 with the sums in place) or native NCCL. */
enum { MARL_DTYPE_F32 = 0, MARL_DTYPE_F64 = 1, MARL_DTYPE_I64 = 2 };
typedef int (*marl_allreduce_fn)(void* ctx, void* dev_buf, int64_t count, int dtype, void* stream);
int marl_ppo_set_allreduce(marl_ppo* p, marl_allreduce_fn fn, void* ctx);
int marl_nccl_unique_id(uint8_t out[128]);
int marl_ppo_set_nccl(marl_ppo* p, const uint8_t id[128], int rank, int world);
/* prng::permutation(key, n) (prng.cpp:151-159) into device memory d_out[n] on `device`. */
int marl_ppo_permutation(const uint32_t key[4], int64_t n, int32_t* d_out, int device);

/* ---- the reference's own benchmark --------------------------------------- */

/* throughput_probe(env_id, n_envs, n_steps, key, config) (vector_env.cpp:
 * 191-222) on `device`: cold = reset + one warm-up step (action_keys[T]),
 * warm = T steps with action_keys = split(fold_in(key, 2), T + 1), timed
 * with CUDA events.  sps = n_envs * n_steps / seconds. */
int marl_throughput_probe(const char* env_id, const char* config_json, int64_t n_envs,
                          int n_steps, const uint32_t key[4], int device, double* seconds,
                          double* cold_seconds);

/* ---- keys (prng.hpp:21-57), host-side helpers ------------------------- */
void marl_prng_key_from_seed(uint64_t seed, uint32_t out[4]);
void marl_prng_split(const uint32_t key[4], uint64_t n, uint32_t* out /* [n][4] */);
void marl_prng_fold_in(const uint32_t key[4], uint64_t data, uint32_t out[4]);
uint64_t marl_prng_bits(const uint32_t key[4], uint64_t index);
void marl_threefry2x32(uint32_t k0, uint32_t k1, uint32_t x0, uint32_t x1, uint32_t out[2]);

/* ---- tensor-core GEMM ---------------------------------------------------
 * The recurrent policy's contractions (embed / GRU / post / head and their
 * BPTT weight gradients; nn.hpp:42-70 matmul_nt / matmul_nn / matmul_tn over
 * the RnnBranch of actor_critic.hpp:74-200), exposed for reuse and testing:
 * C[M x N] = beta*C + A . B'^T, A(m, k) = A[m*sam + k*sak],
 * B'(n, k) = B[n*sbn + k*sbk], C(m, n) = C[m*ldc + n]; fp32 in and out,
 * fp32-accurate 3xTF32 on tcgen05, deterministic; device pointers, enqueued
 * on `stream` (a cudaStream_t, NULL = default). */
int marl_gemm_f32(int64_t M, int N, int64_t K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn,
                  int64_t sbk, float* C, int64_t ldc, float beta, void* stream);

/* ---- diagnostics ------------------------------------------------------ */
const char* marl_last_error(void);
uint64_t marl_launch_count(void); /* kernels launched by this library */
/* Test knob: cap the grid of every persistent (grid-stride / tile-loop) kernel
 * at `ctas` CTAs (0 = no cap) so small inputs exercise the steady state of the
 * loops; returns the previous cap.  No reference counterpart. */
int marl_set_grid_cap(int ctas);
const char* marl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MARL_B200_H */
