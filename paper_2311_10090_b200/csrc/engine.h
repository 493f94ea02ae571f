// Internal interface between the C-ABI host layer (venv.cpp, g++) and the
// per-family CUDA launchers (mpe.cu, smax.cu, overcooked.cu, nvcc).  Plain
// structs of device pointers and sizes; no CUDA types beyond cudaStream_t.
#pragma once
#include <cuda_runtime.h>

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
};

// BatchedState carry (vector_env.hpp:13-20) beside the env-specific state.
struct Carry {
  uint4* keys;         // [N] per-env carry key
  double* ep_return;   // [N]
  int32_t* ep_length;  // [N]
};

struct LaunchCommon {
  int64_t n;            // local envs
  int64_t offset;       // global index of local env 0
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
void mpe_launch_hash(const MpeConfig& c, const MpeState& s, int64_t n, uint64_t* out,
                     cudaStream_t st);

// --------------------------------------------------------------- SMAX
constexpr int kSmaxMaxUnits = 64;

struct SmaxConfig {
  int na, ne;
  int enemy_controlled;
  int max_steps;
  double map;
  double jitter;
  int8_t type[kSmaxMaxUnits];     // per unit
  double stats[6][7];             // health damage cooldown speed sight range radius
  void* dev_params = nullptr;     // device copy of the derived constants (smax_prepare)
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

// ------------------------------------------------------------ common
// Device-side Env::validate_actions (env.cpp:7-14): n_actions per agent.
void launch_validate(const int32_t* actions, int64_t n, int A, const int32_t* n_actions_dev,
                     int* err, cudaStream_t st);

// Kernel launches issued by this library since load (evidence counter).
extern unsigned long long g_launches;

}  // namespace marl_b200
