// Internal interface between the C-ABI host layer (venv.cpp, g++) and the
// per-family CUDA launchers (mpe.cu, smax.cu, overcooked.cu, nvcc).  Plain
// structs of device pointers and sizes; no CUDA types beyond cudaStream_t.
#pragma once
#include <cuda_runtime.h>

#include <functional>

#include <cstdint>

namespace marl_b200 {

struct KeyWords {
  uint32_t w[4];
};

// Outputs of one VectorEnv::step (vector_env.hpp:22-36), flattened:
// obs/final_obs [N][A][D] f32, rewards [N][A] f64, dones [N][A+1] u8,
// finished [N] u8, final_returns [N] f64, final_lengths [N] i32,
// infos [N][A][n_info] f64, actions [N][A] i32.
struct StepViews {
  float* obs;
  double* rewards;
  uint8_t* dones;
  uint8_t* finished;
  float* final_obs;
  double* final_returns;
  int32_t* final_lengths;
  double* infos;
  int32_t* actions;
  float* actions_f;  // [N][A][kBoxActDim] box actions (continuous MPE), else null
};

// Box action rows (continuous MPE, mpe.cpp:91-99): every agent's flat vector
// padded to the widest (movement: 5 floats in [0, 1]; speaker: dim_c floats).
constexpr int kBoxActDim = 5;

// BatchedState carry (vector_env.hpp:13-20) beside the env-specific state.
struct Carry {
  uint4* keys;         // [N] per-env carry key
  double* ep_return;   // [N]
  int32_t* ep_length;  // [N]
};

struct LaunchCommon {
  int64_t n;            // local envs (also the stride of every [component][N] state array)
  int64_t offset;       // global index of local env 0
  int64_t begin, end;   // the step kernels process local envs [begin, end) (a chunk of the batch)
  Carry carry;
  StepViews v;
  unsigned long long* stats;  // [3] episode statistics (see stats_add)
  int* err;                   // [4] device error record
  cudaStream_t stream;
};

// ---------------------------------------------------------------- MPE
enum MpeScenario { kMpeSpread = 0, kMpeSpeakerListener = 1, kMpeTag = 2 };

struct MpeState {
  double* pos;    // [2E][N]
  double* vel;    // [2A][N]
  double* comm;   // [A*dim_c][N] (speaker_listener only)
  int32_t* steps; // [N]
  int32_t* goal;  // [N] (speaker_listener only)
};

struct MpeConfig {
  int scenario;
  int coop_prey;
  int continuous;  // box action spaces (continuous_actions, mpe.cpp:398)
};

int mpe_obs_dim(int scenario);
int mpe_n_agents(int scenario);
int mpe_n_entities(int scenario);
int mpe_dim_c(int scenario);
int mpe_n_actions(int scenario, int agent);
int mpe_obs_size(int scenario, int agent);

// reset_key = key, carry_parent = fold_in(key, 1) (vector_env.cpp:52-55).
void mpe_launch_reset(const MpeConfig& c, const MpeState& s, const LaunchCommon& lc, KeyWords key,
                      KeyWords carry_parent);
// random: actions drawn in-kernel from split(step_key, N_global)[g]
// (vector_env.cpp:169-187); else read from lc.v.actions.
void mpe_launch_step(const MpeConfig& c, const MpeState& s, const LaunchCommon& lc, bool random,
                     KeyWords step_key);
void mpe_launch_probe(const MpeConfig& c, const MpeState& s, const LaunchCommon& lc, KeyWords parent,
                      uint64_t t0, int K);
void mpe_launch_hash(const MpeConfig& c, const MpeState& s, int64_t n, uint64_t* out,
                     cudaStream_t st);

// --------------------------------------------------------------- SMAX
constexpr int kSmaxMaxUnits = 64;

struct SmaxConfig {
  int na, ne;
  int enemy_controlled;
  int random_types;  // smacv2_*: units per team with per-episode random types (smax.cpp:88-93)
  int max_steps;
  double map;
  double jitter;
  int8_t type[kSmaxMaxUnits];     // per unit
  double stats[6][7];             // health damage cooldown speed sight range radius
  void* dev_params = nullptr;     // device copy of the derived constants (smax_prepare)
  void* host_params = nullptr;    // host copy (passed by value to the one-thread-per-env kernel)
};

// Upload / free the derived per-unit constants for a config (once per handle).
void smax_prepare(SmaxConfig& c);
void smax_release(SmaxConfig& c);

struct SmaxState {
  double* x;          // [U][N]
  double* y;          // [U][N]
  double* health;     // [U][N]
  double* cooldown;   // [U][N]
  uint32_t* mem;      // [U][N] prev_action | ai_target<<8 | ai_sweep<<16 (bytes, see smax.cu)
  int32_t* t;         // [N]
};

void smax_launch_reset(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc,
                       KeyWords key, KeyWords carry_parent);
void smax_launch_step(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, bool random,
                      KeyWords step_key);
void smax_launch_legal(const SmaxConfig& c, const SmaxState& s, int64_t n, int n_act,
                       uint8_t* out, cudaStream_t st);
void smax_launch_hash(const SmaxConfig& c, const SmaxState& s, int64_t n, uint64_t* out,
                      cudaStream_t st);

// --------------------------------------------------------- Overcooked
constexpr int kOcMaxCells = 256;
constexpr int kOcMaxPots = 8;
constexpr int kOcMaxCounters = 64;

struct OcConfig {
  int h, w;
  char kind[kOcMaxCells];
  int spawn[2];
  int n_pots, n_counters;
  int pot_cells[kOcMaxPots];
  int counter_cells[kOcMaxCounters];
  int max_steps, cook_time, random_conflicts;
  double delivery_reward, sh_onion, sh_plate, sh_soup;
};

struct OcState {
  uint32_t* agents;   // [N] pos0 | pos1<<8 | facing0<<16 | facing1<<18 | held0<<20 | held1<<22
  uint32_t* pots;     // [P][N] onions | timer<<8
  uint64_t* counters; // [C/32][N] 2 bits per counter cell (C <= 64 -> up to 2 words)
  int32_t* t;         // [N]
};

// templ: [27*h*w+1] f32 static planes of encode() (overcooked.cpp:404-413).
void oc_launch_reset_t(const OcConfig& c, const float* templ, const OcState& s, const LaunchCommon& lc,
                       KeyWords key, KeyWords carry_parent);
void oc_launch_step_t(const OcConfig& c, const float* templ, const OcState& s, const LaunchCommon& lc,
                      bool random, KeyWords step_key);
void oc_launch_hash(const OcConfig& c, const OcState& s, int64_t n, uint64_t* out,
                    cudaStream_t st);

// ------------------------------------------------------ IPPO rollout (C5)
// Collector::collect (ppo.cpp:206-323) buffers, [T][R] row-major with
// R = envs x agents (TeamLayout rows, team.cpp:27-33).
struct RolloutBufs {
  float* obs;          // [T][R][in_dim] actor input (IPPO critic input is the same row)
  int32_t* actions;    // [T][R]  (slice t doubles as the env step's [E][A] action input)
  float* rewards;      // [T][R]
  uint8_t* dones;      // [T][R]
  uint8_t* resets;     // [T][R]
  float* logp;         // [T][R]
  float* value;        // [T][R]
  uint8_t* legal;      // [T][R][n_act]
  float* active;       // [T][R]
  float* adv;          // [T][R]
  float* vtarg;        // [T][R]
  float* last_value;   // [R]  bootstrap values after the window (ppo.cpp:285-299)
  float* critic_in;    // [T][R][critic_in] centralised (MAPPO) critic rows, else null
};

// Feed-forward actor and critic (ff_forward, actor_critic.hpp:49-52) with two
// activated torso layers: pointers into the packed fp32 parameters in
// nn::pack order (torso w,b per layer, then head w,b; w is [out][in]).
struct PolicyNet {
  const float *w1, *b1, *w2, *b2, *w3, *b3;
  const float *cw1, *cb1, *cw2, *cb2, *cw3, *cb3;
  int in_dim, n_act, width, relu;
  int critic_in;  // == in_dim (IPPO) or world_state_size (MAPPO, ppo.cpp:90-100)
  int centralized;  // 1: the critic reads world_state rows (MAPPO)
};

// bf16 operand images for the tcgen05 path (K-major, no swizzle, UMMA
// canonical layout); built once per parameter upload.
struct PolicyNetBf16 {
  const uint16_t* a1;   // [128 x kx] : actor W1 rows 0..63, critic W1 rows 64..127, K padded to kx = round16(in)
  const uint16_t* a2;   // [64 x 64]  actor W2
  const uint16_t* c2;   // [64 x 64]  critic W2
  const uint16_t* h3;   // [64 x 64]  actor head (rows 0..n_act-1), zero padded (narrow kernels read rows 0..15)
  const uint16_t* hc3;  // [16 x 64]  critic head (row 0), zero padded
  const uint16_t* c1;   // [64 x kc]  MAPPO critic W1 over world_state rows, K padded to kc = round16(critic_in); else null
  const float* bias;    // [64 b1a | 64 b1c | 64 b2a | 64 b2c | 16 b3a | 16 b3c | 64 b3a (heads up to 64)]
};

struct PolicyStep {
  const float* env_obs;        // [E][A][D] current observations
  const uint8_t* prev_finished;  // [E] or null: every row starts an episode (Collector ctor)
  const int32_t* agent_actions;  // [A] device: per-agent action count (legal padding, team.cpp:35-42)
  int A, D, family;
  int64_t R, row0, R_global;   // local rows, global index of local row 0, global rows
  uint32_t act_key[4];         // Collector act_key = fold_in(key, 2) (ppo.cpp:192)
  int64_t step_index;          // seq_base + t
  int t;
  int bootstrap;               // 1: critic only -> last_value (ppo.cpp:285-299)
  const float* ws;             // [E][critic_in] world_state rows (MAPPO critic input) or null (IPPO)
  int legal_ready;             // 1: bufs.legal slice t already filled by the env's legal kernel
};

void rollout_policy_fp32(const PolicyNet& net, const PolicyStep& s, const RolloutBufs& b, cudaStream_t st);
bool rollout_policy_bf16_supported(int in_dim, int n_act, int width, int critic_in = 0);  // critic_in > 0: MAPPO
int rollout_tc_kx(int in_dim);  // K of the tcgen05 policy's layer 1: round16(in_dim), <= 192
void rollout_policy_bf16(const PolicyNet& net, const PolicyNetBf16& nb, const PolicyStep& s, const RolloutBufs& b,
                         cudaStream_t st);
void rollout_pack_bf16(const PolicyNet& net, uint16_t* images, float* bias, cudaStream_t st);
// rewards / dones of step t from the env's views (ppo.cpp:262-276)
void rollout_record(const RolloutBufs& b, int t, int64_t R, int A, const double* env_rewards,
                    const double* env_infos, int n_info, int shaped_idx, double shaping,
                    const uint8_t* env_finished, cudaStream_t st);
// GAE per row (compute_gae, actor_critic.hpp:282-299)
void rollout_gae(const RolloutBufs& b, int T, int64_t R, float gamma, float lambda, cudaStream_t st);

// Env::world_state (smax.cpp:272-289): 18 floats per unit + t/max_steps.
void smax_launch_world_state(const SmaxConfig& c, const SmaxState& s, int64_t n, float* out, cudaStream_t st);
// world_state as a gather from the observation view: MPE concatenates every
// agent's unpadded row (mpe.cpp:229-242), Overcooked is agent 0's row
// (overcooked.cpp:315-319).  seg_src/seg_len: [n_seg] (offset in the env's
// [A][D] obs block, length), written back to back.
// final_obs rows of the finished envs of [0, n) from device `src` into the
// device-accessible (mapped pinned) host buffer `dst`; `row` floats per env.
void launch_gather_finished_rows(const uint8_t* finished, int64_t n, const float* src, float* dst, int64_t row,
                                 cudaStream_t st);
void launch_obs_gather(const float* obs, int64_t n, int row_floats, const int32_t* seg_src, const int32_t* seg_len,
                       int n_seg, int width, float* out, cudaStream_t st);

// ------------------------------------------------------------ recurrent policy
struct PpoMbStats;
// RnnBranch (actor_critic.hpp:74-200): embed in->F, GRU F->H, post H->F, head.
inline int rnn_branch_params(int in, int F, int H, int out) {
  return F * in + F + 3 * H * F + 3 * H * H + 6 * H + F * H + F + out * F + out;
}

struct RnnPolicyArgs {
  const float *actor, *critic;  // packed branches (nn::pack order)
  float *h_actor, *h_critic;    // [R][H] carried hidden states (ppo.cpp:194-198)
  int in_dim, critic_in, n_act, F, H, relu;
};
void rnn_policy(const RnnPolicyArgs& a, const PolicyStep& s, const RolloutBufs& b, cudaStream_t st);

// rnn_seq_forward caches of one branch over K = T*M (t, row) entries, k = t*M + i
struct RnnCache {
  float *x, *y, *e, *h, *z, *r, *c, *ah, *p, *hn;  // forward
  float *dy, *dzp, *daz, *dar, *dac, *dah, *dze;   // backward deltas
};
inline size_t rnn_cache_floats(int in, int F, int H, int out) {
  return size_t(in) + 2 * size_t(out) + 4 * size_t(F) + 10 * size_t(H);
}

struct RnnSeqArgs {
  const float *actor, *critic;
  const float *h0_actor, *h0_critic;  // [R][H] hidden at the window start (ppo.cpp:219-222)
  const int32_t* rows;                // [M] minibatch rows
  int64_t M;
  int T;
  int64_t R;
  int in_dim, critic_in, n_act, F, H, relu;
  const float* obs;          // [T][R][in_dim]
  const float* critic_rows;  // [T][R][critic_in] (MAPPO) or null
  const uint8_t* resets;     // [T][R]
  RnnCache ca, cc;
};
// GEMM-structured update: per time step t, over the M rows of a chunk.
struct RnnWPtrs {  // the branch's matrices / biases in RnnBranch pack order
  const float *we, *be, *wx, *uh, *bias6, *wp, *bp, *wh, *bh;  // wx = [Wz;Wr;Wn], uh = [Uz;Ur;Un]
};
RnnWPtrs rnn_weights(const float* p, int in, int F, int H, int out);
struct RnnStepArgs {
  int t;
  int64_t M, R;
  int in, H;
  const int32_t* rows;
  const uint8_t* resets;
  const float* src;  // [T][R][in] input rows
  const float* h0;   // [R][H] hidden at the window start
  float* h;          // [M][H] running hidden
  float* x;          // cache x_t     [M][in]
  float *hprev, *z, *r, *c, *ah, *hn;  // caches at step t [M][H]
  float* hnext;       // gates: also write step t+1's h_prev (apply_reset at t+1) here; null: no
  const float* dhp;   // gru_bwd: the post layer's dh share of step t (carry > 0)
  int carry;          // gru_bwd: 0 g = dhs; 1 g = dhp; 2 g = (reset at t+1 ? 0 : dhs) + dhp
  struct {
    const float *bzx, *brx, *bnx, *bzh, *brh, *bnh;
  } w;
};
void rnn_step_gather(const RnnStepArgs& a, cudaStream_t s);
// x[t][i][:] = src[t][rows[i]][:] for every t < T at once (the non-recurrent part of sq_gather)
void rnn_seq_x_gather(const int32_t* rows, int64_t Mc, int T, int64_t R, int in, const float* src, float* x,
                      cudaStream_t s);
// GEMM-structured acting step of the collector (many rows)
void rnn_policy_rows(const PolicyStep& s, const RolloutBufs& b, int in, int CI, int NA, int H, float* xa, float* xc,
                     float* ha, float* hc, float* hc_peek, cudaStream_t st);
void rnn_gates_inplace(int64_t M, int H, float* h, const float* gx, const float* gh, const float* b6, cudaStream_t st);
void rnn_policy_sample(const PolicyStep& s, const RolloutBufs& b, int NA, const float* ya, const float* yc,
                       cudaStream_t st);
void rnn_bias_act(float* y, int64_t M, int N, const float* b, bool act, int relu, cudaStream_t s);
void rnn_gates(const RnnStepArgs& a, const float* gx, const float* gh, cudaStream_t s);
void rnn_act_grad(float* g, const float* y, int64_t n, int relu, cudaStream_t s);
void rnn_gru_bwd(const RnnStepArgs& a, const float* dhs, float* d4, float* dh, cudaStream_t s);

// flat[k = t*M + i] = t*R + rows[i] (the loss rows of rnn_minibatch, ppo.cpp:472-477)
void rnn_flat_slots(const int32_t* rows, int64_t M, int T, int64_t R, int32_t* flat, cudaStream_t st);
// ppo_row_loss over the K flat rows from the cached head outputs -> ca.dy, cc.dy;
// per-block loss sums -> spart_a / spart_c [blocks][6]
int rnn_loss_blocks(int64_t K);
void rnn_loss(const RnnSeqArgs& a, const int32_t* flat, int64_t K, const RolloutBufs& b, const PpoMbStats* st,
              double clip_eps, double ent_coef, double vf_coef, double* spart_a, double* spart_c, int* err,
              cudaStream_t s);

// ------------------------------------------------------------ PPO update
// train_ppo_impl's minibatch loop (ppo.cpp:588-628) over a RolloutBufs.
constexpr int kPpoMaxAct = 64;

struct PpoMbStats {  // normalize_advantages over one minibatch (actor_critic.hpp:416-433)
  double mean, std, total_w;
  int normalize;
};

struct PpoBranchArgs {  // one branch (actor or critic) of one minibatch
  const float* params;   // the branch's packed parameters (nn::pack order)
  float* gpart;          // [grid][P] per-CTA gradient partials
  double* spart;         // [grid][6] per-CTA loss sums
  const int32_t* idx;    // minibatch slots (t*R + r)
  int64_t M;
  const float* x;        // input rows: obs (actor, IPPO critic) or critic_in (MAPPO critic)
  const int32_t* actions;
  const float *old_logp, *adv, *vtarg, *old_value, *active;
  const uint8_t* legal;
  const PpoMbStats* st;
  int* err;              // stored action illegal -> ContractError (actor_critic.hpp:366)
  int in, W, out, relu, TR, staged;
  double clip_eps, ent_coef, vf_coef;
};

struct PpoApplyArgs {
  float *params, *grad, *m, *v;  // whole flat vector: actor | critic
  int P;
  const double *actor_stats, *critic_stats;
  int n_actor_parts, n_critic_parts;
  const PpoMbStats* st;
  double vf_coef, ent_coef;
  float max_norm, lr, beta1, beta2, eps, c1, c2;
  double* metrics;   // [8]: loss, pg, v, entropy, kl, clip_frac, grad_norm, counted
  int* diverged;     // sticky DivergenceError flag
};

// The tcgen05 minibatch step (ppo_tc.cu): actor + critic of an IPPO net with
// input <= 191, width 64, <= 16 actions, bf16 operands, fp32 TMEM accumulators.
struct PpoTcArgs {
  const float *actor, *critic;  // packed fp32 parameters (current)
  float *gpart_a, *gpart_c;     // [grid][Pa], [grid][Pc]
  double *spart_a, *spart_c;    // [grid][6]
  const int32_t* idx;
  int64_t M;
  const uint16_t* obs_bf;     // [T*R][kx] bf16 rows (ppo_tc_pack)
  const struct PpoRowRec* rec;  // [T*R] loss-input records (ppo_tc_pack)
  const PpoMbStats* st;
  int* err;
  int in, kx, n_act, relu;
  double clip_eps, ent_coef, vf_coef;
};
int ppo_tc_kx(int in_dim);  // round16(in + 1): the bf16 row width incl. the bias column
// One slot's loss inputs for the tcgen05 step (32 bytes, one gather per row).
struct PpoRowRec {
  float active, adv, logp, vtarg, value;
  int32_t action;
  uint32_t legal;  // bit j: action j legal (n_act <= 16)
  uint32_t pad;
};
struct PpoTcPack {
  const float* obs;  // [rows][in]
  const float *active, *adv, *old_logp, *vtarg, *old_value;
  const int32_t* actions;
  const uint8_t* legal;  // [rows][n_act]
  int64_t rows;
  int in, kx, n_act;
  uint16_t* obs_bf;  // [rows][kx]
  PpoRowRec* rec;    // [rows]
};
// the window's rows for the tcgen05 step (bf16 observations, column kx-1 = 1,
// and the loss-input records), once per update
void ppo_tc_pack(const PpoTcPack& p, cudaStream_t s);
bool ppo_tc_supported(int in_dim, int critic_in, int width, int n_act);
int ppo_tc_grid(int64_t M);
void ppo_update_tc(const PpoTcArgs& a, int grid, cudaStream_t s);

size_t ppo_perm_scratch_bytes(int64_t n);
// prng::permutation(key, n) (prng.cpp:151-159) into out[n] on the device.
void ppo_permutation(KeyWords key, int64_t n, int32_t* out, void* scratch, size_t scratch_bytes, cudaStream_t st);
int ppo_stat_blocks(int64_t M);
// g: device double[4] scratch; allreduce (optional): sum g[0:2) then g[2:3) over the data-parallel ranks
// rec (optional): read adv / active from the tcgen05 step's packed records
void ppo_adv_stats(const RolloutBufs& b, const int32_t* idx, int64_t M, double* part, double* part2, double* g,
                   PpoMbStats* st, cudaStream_t s, const std::function<void(double*, int)>& allreduce,
                   const PpoRowRec* rec = nullptr, float2* gath = nullptr);
// sharded update: the global minibatch slots this shard owns, as local slots (order kept), count -> d_count
size_t ppo_compact_scratch_bytes(int64_t M);
void ppo_shard_compact(const int32_t* idx, int64_t M, int64_t Rg, int64_t row0, int64_t Rl, int32_t* tmp,
                       int32_t* out, int64_t* d_count, void* scratch, size_t scratch_bytes, cudaStream_t s);
void ppo_stats_fold(double* spart, int nparts, cudaStream_t s);
void ppo_branch_geometry(int in, int W, int out, int* TR, int* staged, size_t* smem);
int ppo_branch_grid(int in, int W, int out, int64_t M);
void ppo_branch(PpoBranchArgs a, bool actor, int grid, cudaStream_t s);
void ppo_grad_reduce(const float* part, int nparts, int P, float* grad, cudaStream_t s);
// out[m][0..in) = x[idx[m]][0..in), rows of out `ldo` floats apart (ff_minibatch's gather)
void ppo_gather_rows(const float* x, const int32_t* idx, int64_t M, int in, float* out, int ldo, cudaStream_t s);
// The wide-input fp32 update (ppo_wide.cu, ppo_host.cpp minibatch_grad_wide).
struct WideStage {
  const float *pa, *pc;  // the branches' parameters (nn::pack order)
  int64_t Pa, Pc;
  float *qa, *qc;  // their 16-byte aligned copies
  int W, in_a, in_c, ldx;
  float* w1s;   // [2W][ldx] stacked layer-1 matrices (null: not stacked)
  float* bias;  // [4W] b1a | b1c | b2a | b2c
};
void wide_stage(const WideStage& s, cudaStream_t st);
// y[m][c] = act(y[m][c] + b[c]) over [M][N]
void wide_bias_act(float* y, int64_t M, int N, const float* b, int relu, cudaStream_t st);
// d *= act'(h) in place (h null: unchanged), then column sums of d: columns
// c < split to dst0[c], the rest to dst1[c - split]; part: wide_part_floats(M, N)
void wide_grad_colsum(float* d, const float* h, int64_t M, int N, int relu, float* part, int split, float* dst0,
                      float* dst1, cudaStream_t st);
int64_t wide_part_floats(int64_t M, int N);
void ppo_clip_adam(const PpoApplyArgs& a, cudaStream_t s);

// ------------------------------------------------------------ common
// Device-side Env::validate_actions (env.cpp:7-14): n_actions per agent.
void launch_validate(const int32_t* actions, int64_t n, int A, const int32_t* n_actions_dev,
                     int* err, cudaStream_t st);
// Box spaces (SpaceDescriptor::contains, spaces.cpp:36-46): the first
// flat_size[a] floats of every [kBoxActDim] row finite and in [0, 1].
void launch_validate_box(const float* actions, int64_t n, int A, const int32_t* flat_size_dev, int* err,
                         cudaStream_t st);

// Kernel launches issued by this library since load (evidence counter).
extern unsigned long long g_launches;

// gemm_tc.cu: C[M x N] = beta C + A . B'^T with A(m, k) = A[m*sam + k*sak] and
// B'(n, k) = B[n*sbn + k*sbk] (fp32-accurate 3xTF32 on tcgen05); column sums
// g[o] = beta g[o] + sum_k D[k*ldd + o] (fixed-order reduction).
cudaError_t tc_gemm(cudaStream_t st, int64_t M, int N, int64_t K, const float* A, int64_t sam, int64_t sak,
                    const float* B, int64_t sbn, int64_t sbk, float* C, int64_t ldc, float beta);
cudaError_t tc_colsum(cudaStream_t st, int O, int64_t K, const float* D, int64_t ldd, float* g, float beta);

// Test knob (marl_set_grid_cap): upper bound on the grid of every persistent
// (grid-stride / tile-loop) kernel, so small parity inputs drive each CTA or
// warp through several iterations of its loop.  0 = no cap (the default).
extern int g_grid_cap;
inline int64_t cap_grid(int64_t g) { return g_grid_cap > 0 && g > g_grid_cap ? int64_t(g_grid_cap) : g; }

}  // namespace marl_b200
