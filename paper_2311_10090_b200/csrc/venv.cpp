// Host side of the C-ABI (include/marl_b200.h): the env registry and strict
// config schema of the reference (registry.cpp, config.hpp, the per-env
// factories), handle / device-buffer management, and the VectorEnv call
// sequence around the fused CUDA kernels.  Nothing here computes env
// dynamics: every reset/step is a kernel launch (mpe.cu, smax.cu,
// overcooked.cu); a missing GPU is a MARL_ERR_CUDA, never a CPU fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "common.cuh"
#include "engine.h"
#include "host.h"
#include "marl_b200.h"

using nlohmann::json;
using namespace marl_b200;
using namespace mhost;

namespace mhost {
thread_local std::string g_err;
}  // namespace mhost

namespace mhost {



// ---------------------------------------------------------------------------
// Registry (registry.cpp:39-66): the ids this engine implements, plus the
// reference's reserved ids and the ids it registers outside the hot path.
const char* kSmaxScenarios[] = {"2s3z",          "3s5z",           "5m_vs_6m",        "10m_vs_11m",
                                "27m_vs_30m",    "3s5z_vs_3s6z",   "3s_vs_5z",        "6h_vs_8z",
                                "smacv2_5_units", "smacv2_10_units", "smacv2_20_units"};
const char* kLayoutNames[] = {"cramped_room", "asymmetric_advantages", "coordination_ring",
                              "forced_coordination", "counter_circuit"};
const char* kLayoutText[] = {  // overcooked.cpp:28-58
    "XXPXX\nO  2O\nX1  X\nXDXSX\n",
    "XXXXXXXXX\nO XSXOX S\nX   P 1 X\nX 2 P   X\nXXXDXDXXX\n",
    "XXXPX\nX 1 P\nD2X X\nO   X\nXOSXX\n",
    "XXXPX\nO X1P\nO2X X\nD X X\nXXXSX\n",
    "XXXPPXXX\nX 1    X\nD XXXX S\nX     2X\nXXXOOXXX\n"};
const char* kReserved[] = {"MPE_simple_v3",           "MPE_simple_adversary_v3", "MPE_simple_crypto_v3",
                           "MPE_simple_push_v3",      "MPE_simple_reference_v3", "MPE_simple_world_comm_v3"};
const char* kOffPath[] = {"switch_riddle_v0", "bandit_v0", "STORM_ipd_v0", "STORM_matching_pennies_v0",
                          "coin_game_v0", "hanabi_v0"};

const std::vector<std::string>& registered() {
  static std::vector<std::string> ids = [] {
    std::vector<std::string> v = {"MPE_simple_spread_v3", "MPE_simple_speaker_listener_v4", "MPE_simple_tag_v3"};
    for (const char* s : kSmaxScenarios) v.push_back(std::string("SMAX_") + s);
    for (const char* l : kLayoutNames) v.push_back(std::string("overcooked_") + l + "_v0");
    std::sort(v.begin(), v.end());
    return v;
  }();
  return ids;
}

const char* kTypeNames[6] = {"marine", "stalker", "zealot", "hydralisk", "zergling", "marauder"};
const double kDefaultStats[6][7] = {  // smax.cpp:26-33
    {45.0, 6.0, 0.61, 3.15, 9.0, 5.0, 0.375},    {160.0, 13.0, 1.34, 4.13, 9.0, 6.0, 0.625},
    {150.0, 16.0, 0.86, 3.15, 9.0, 0.1, 0.5},    {80.0, 12.0, 0.59, 3.15, 9.0, 5.0, 0.625},
    {35.0, 5.0, 0.497, 4.13, 9.0, 0.1, 0.375},   {125.0, 10.0, 1.07, 3.15, 9.0, 6.0, 0.5625}};
const char* kStatKeys[7] = {"health", "damage", "cooldown", "speed", "sight", "range", "radius"};

std::vector<int8_t> roster(int m, int s, int z, int h, int l) {  // smax.cpp:43-51
  std::vector<int8_t> out;
  for (int i = 0; i < s; ++i) out.push_back(1);
  for (int i = 0; i < z; ++i) out.push_back(2);
  for (int i = 0; i < m; ++i) out.push_back(0);
  for (int i = 0; i < h; ++i) out.push_back(3);
  for (int i = 0; i < l; ++i) out.push_back(4);
  return out;
}


void make_mpe(Env& e, const std::string& scen, const json& cfg) {  // mpe.cpp:45-79, 396-402
  int s = scen == "simple_spread" ? kMpeSpread : scen == "simple_speaker_listener" ? kMpeSpeakerListener : kMpeTag;
  ConfigView v(cfg, "MPE " + scen);
  bool continuous = v.get_bool("continuous_actions", false);
  bool coop = s == kMpeTag ? v.get_bool("cooperative_prey_reward", false) : false;
  v.check_no_extras();
  e.family = MARL_FAMILY_MPE;
  e.mpe.scenario = s;
  e.mpe.coop_prey = coop;
  e.mpe.continuous = continuous ? 1 : 0;
  e.continuous = continuous;
  e.A = mpe_n_agents(s);
  e.D = mpe_obs_dim(s);
  e.max_steps = 25;
  e.cooperative = s != kMpeTag || coop;  // mpe.cpp:103-105
  if (s == kMpeSpread) e.agents = {"agent_0", "agent_1", "agent_2"};
  else if (s == kMpeSpeakerListener) e.agents = {"speaker_0", "listener_0"};
  else e.agents = {"adversary_0", "adversary_1", "adversary_2", "agent_0"};
  for (int a = 0; a < e.A; ++a) {
    e.obs_size.push_back(mpe_obs_size(s, a));
    e.n_actions.push_back(mpe_n_actions(s, a));
  }
}

std::vector<int8_t> parse_roster(const Env& e, const std::vector<std::string>& names, const char* key) {
  std::vector<int8_t> out;
  for (const auto& n : names) {
    int t = -1;
    for (int q = 0; q < 6; ++q)
      if (n == kTypeNames[q]) t = q;
    if (t < 0) raise(MARL_ERR_SCHEMA, e.id + ": " + key + " has unknown unit type '" + n + "'");
    out.push_back(int8_t(t));
  }
  return out;
}

void make_smax(Env& e, const std::string& scen, const json& cfg) {  // smax.cpp:65-146
  std::vector<int8_t> ally, enemy;
  int random_types = 0;
  if (scen == "2s3z") ally = roster(0, 2, 3, 0, 0);
  else if (scen == "3s5z") ally = roster(0, 3, 5, 0, 0);
  else if (scen == "5m_vs_6m") { ally = roster(5, 0, 0, 0, 0); enemy = roster(6, 0, 0, 0, 0); }
  else if (scen == "10m_vs_11m") { ally = roster(10, 0, 0, 0, 0); enemy = roster(11, 0, 0, 0, 0); }
  else if (scen == "27m_vs_30m") { ally = roster(27, 0, 0, 0, 0); enemy = roster(30, 0, 0, 0, 0); }
  else if (scen == "3s5z_vs_3s6z") { ally = roster(0, 3, 5, 0, 0); enemy = roster(0, 3, 6, 0, 0); }
  else if (scen == "3s_vs_5z") { ally = roster(0, 3, 0, 0, 0); enemy = roster(0, 0, 0, 0, 5); }
  else if (scen == "6h_vs_8z") { ally = roster(0, 0, 0, 6, 0); enemy = roster(0, 0, 0, 0, 8); }
  else if (scen == "smacv2_5_units") random_types = 5;
  else if (scen == "smacv2_10_units") random_types = 10;
  else if (scen == "smacv2_20_units") random_types = 20;
  else raise(MARL_ERR_NOT_FOUND, "unknown smax scenario: " + scen);
  if (enemy.empty()) enemy = ally;

  ConfigView v(cfg, e.id);
  SmaxConfig& c = e.smax;
  c.max_steps = v.get_int("max_steps", 100);
  c.map = v.get_double("map_size", 32.0);
  c.enemy_controlled = v.get_bool("enemy_controlled", false);
  c.jitter = v.get_double("spawn_jitter", 0.5);
  auto ao = v.get_string_list("ally_units");
  auto eo = v.get_string_list("enemy_units");
  json stats_cfg = v.get_object("unit_stats");
  v.check_no_extras();
  if (c.max_steps < 1) raise(MARL_ERR_SCHEMA, e.id + ": max_steps must be >= 1");
  if (c.map < 4.0) raise(MARL_ERR_SCHEMA, e.id + ": map_size must be >= 4");
  if (c.jitter < 0.0) raise(MARL_ERR_SCHEMA, e.id + ": spawn_jitter must be >= 0");
  for (int t = 0; t < 6; ++t)
    for (int k = 0; k < 7; ++k) c.stats[t][k] = kDefaultStats[t][k];
  ConfigView sv(stats_cfg, e.id + ".unit_stats");
  for (int t = 0; t < 6; ++t) {
    if (!sv.has(kTypeNames[t])) continue;
    ConfigView uv(sv.get_object(kTypeNames[t]), e.id + ".unit_stats." + kTypeNames[t]);
    double* st = c.stats[t];
    for (int k = 0; k < 7; ++k) st[k] = uv.get_double(kStatKeys[k], st[k]);
    uv.check_no_extras();
    if (st[0] <= 0 || st[2] <= 0 || st[4] <= 0 || st[6] <= 0 || st[1] < 0 || st[3] < 0 || st[5] < 0)
      raise(MARL_ERR_SCHEMA, e.id + ": invalid unit_stats for " + kTypeNames[t]);
  }
  sv.check_no_extras();
  if (!ao.empty()) ally = parse_roster(e, ao, "ally_units");
  if (!eo.empty()) enemy = parse_roster(e, eo, "enemy_units");
  if (!ao.empty() || !eo.empty()) {
    if (random_types > 0 && (ao.empty() || eo.empty()))
      raise(MARL_ERR_SCHEMA, e.id + ": random-type scenarios need both ally_units and enemy_units");
    random_types = 0;
  }
  c.random_types = random_types;
  if (random_types > 0) {  // smax.cpp:144-146: both teams have random_types units
    ally.assign(size_t(random_types), 0);
    enemy.assign(size_t(random_types), 0);
  }
  c.na = int(ally.size());
  c.ne = int(enemy.size());
  if (c.na < 1 || c.ne < 1) raise(MARL_ERR_SCHEMA, e.id + ": both teams need at least one unit");
  if (c.na + c.ne > kSmaxMaxUnits)
    raise(MARL_ERR_SCHEMA, e.id + ": the B200 engine supports at most 64 units per battle");
  for (int u = 0; u < c.na; ++u) c.type[u] = ally[size_t(u)];
  for (int u = 0; u < c.ne; ++u) c.type[c.na + u] = enemy[size_t(u)];
  e.family = MARL_FAMILY_SMAX;
  const int n = c.na + c.ne;
  e.A = c.na + (c.enemy_controlled ? c.ne : 0);
  e.D = 10 + 17 * (n - 1);
  e.n_info = 3;
  e.info_names = {"alive", "battle_won", "draw"};
  e.max_steps = c.max_steps;
  e.cooperative = !c.enemy_controlled;
  for (int i = 0; i < c.na; ++i) e.agents.push_back("ally_" + std::to_string(i));
  if (c.enemy_controlled)
    for (int i = 0; i < c.ne; ++i) e.agents.push_back("enemy_" + std::to_string(i));
  for (int a = 0; a < e.A; ++a) {
    e.obs_size.push_back(e.D);
    e.n_actions.push_back(5 + (a < c.na ? c.ne : c.na));
  }
}

void parse_layout(Env& e, const std::string& text) {  // overcooked.cpp:70-129
  const std::string ctx = e.id;
  std::vector<std::string> rows;
  std::string line;
  for (char ch : text) {
    if (ch == '\n') {
      if (!line.empty()) rows.push_back(line);
      line.clear();
    } else {
      line += ch;
    }
  }
  if (!line.empty()) rows.push_back(line);
  if (rows.size() < 3) raise(MARL_ERR_SCHEMA, ctx + ": layout needs at least 3 rows");
  OcConfig& c = e.oc;
  c.h = int(rows.size());
  c.w = int(rows[0].size());
  for (const auto& r : rows)
    if (int(r.size()) != c.w) raise(MARL_ERR_SCHEMA, ctx + ": layout rows must all have the same width");
  if (c.h * c.w > kOcMaxCells) raise(MARL_ERR_SCHEMA, ctx + ": the B200 engine supports layouts of at most 256 cells");
  c.spawn[0] = c.spawn[1] = -1;
  c.n_pots = c.n_counters = 0;
  for (int r = 0; r < c.h; ++r)
    for (int q = 0; q < c.w; ++q) {
      char ch = rows[size_t(r)][size_t(q)];
      int cell = r * c.w + q;
      switch (ch) {
        case 'X': case 'O': case 'D': case 'P': case 'S':
          c.kind[cell] = ch;
          if (ch == 'P') {
            if (c.n_pots == kOcMaxPots) raise(MARL_ERR_SCHEMA, ctx + ": the B200 engine supports at most 8 pots");
            c.pot_cells[c.n_pots++] = cell;
          }
          if (ch == 'X') {
            if (c.n_counters == kOcMaxCounters) raise(MARL_ERR_SCHEMA, ctx + ": the B200 engine supports at most 64 counters");
            c.counter_cells[c.n_counters++] = cell;
          }
          break;
        case ' ':
          c.kind[cell] = ' ';
          break;
        case '1': case '2': {
          int idx = ch - '1';
          if (c.spawn[idx] != -1) raise(MARL_ERR_SCHEMA, ctx + ": duplicate spawn digit in layout");
          c.spawn[idx] = cell;
          c.kind[cell] = ' ';
          break;
        }
        default:
          raise(MARL_ERR_SCHEMA, ctx + ": unknown layout character '" + std::string(1, ch) + "'");
      }
    }
  if (c.spawn[0] < 0 || c.spawn[1] < 0) raise(MARL_ERR_SCHEMA, ctx + ": layout needs spawn digits 1 and 2");
  for (char need : {'P', 'O', 'D', 'S'}) {
    bool found = false;
    for (int q = 0; q < c.h * c.w; ++q) found |= c.kind[q] == need;
    if (!found) raise(MARL_ERR_SCHEMA, ctx + ": layout needs at least one of each P, O, D, S");
  }
  for (int r = 0; r < c.h; ++r)
    for (int q = 0; q < c.w; ++q)
      if ((r == 0 || q == 0 || r == c.h - 1 || q == c.w - 1) && c.kind[r * c.w + q] == ' ')
        raise(MARL_ERR_SCHEMA, ctx + ": layout border must be walls/stations, not floor");
}

void make_overcooked(Env& e, int layout, const json& cfg) {  // overcooked.cpp:163-179
  ConfigView v(cfg, e.id);
  std::string text = v.get_string("layout", "");
  if (text.empty()) text = kLayoutText[layout];
  OcConfig& c = e.oc;
  c.max_steps = v.get_int("max_steps", 400);
  c.cook_time = v.get_int("cook_time", 20);
  c.delivery_reward = v.get_double("delivery_reward", 20.0);
  c.sh_onion = v.get_double("shaping_onion", 3.0);
  c.sh_plate = v.get_double("shaping_plate", 3.0);
  c.sh_soup = v.get_double("shaping_soup", 5.0);
  c.random_conflicts = v.get_bool("random_conflict_resolution", false);
  v.check_no_extras();
  if (c.max_steps < 1) raise(MARL_ERR_SCHEMA, "overcooked: max_steps must be >= 1");
  if (c.cook_time < 1) raise(MARL_ERR_SCHEMA, "overcooked: cook_time must be >= 1");
  if (c.cook_time >= (1 << 24)) raise(MARL_ERR_SCHEMA, "overcooked: cook_time must be < 2^24 on the B200 engine");
  parse_layout(e, text);
  e.family = MARL_FAMILY_OVERCOOKED;
  e.A = 2;
  e.D = 27 * c.h * c.w + 1;
  e.n_info = 2;
  e.info_names = {"deliveries", "shaped_reward"};
  e.max_steps = c.max_steps;
  e.cooperative = true;
  e.agents = {"agent_0", "agent_1"};
  e.obs_size = {e.D, e.D};
  e.n_actions = {6, 6};
  // static planes of encode(), overcooked.cpp:404-413
  const int cells = c.h * c.w;
  e.oc_templ.assign(size_t(e.D), 0.0f);
  for (int q = 0; q < cells; ++q) {
    int plane = c.kind[q] == 'X' ? 10 : c.kind[q] == 'O' ? 11 : c.kind[q] == 'D' ? 12
              : c.kind[q] == 'P' ? 13 : c.kind[q] == 'S' ? 14 : -1;
    if (plane >= 0) e.oc_templ[size_t(plane * cells + q)] = 1.0f;
  }
}

std::unique_ptr<Env> make_env(const std::string& id, const char* cfg_json) {  // registry.cpp:83-97
  json cfg = (cfg_json && *cfg_json) ? json::parse(cfg_json) : json::object();
  auto e = std::make_unique<Env>();
  e->id = id;
  if (id == "MPE_simple_spread_v3") make_mpe(*e, "simple_spread", cfg);
  else if (id == "MPE_simple_speaker_listener_v4") make_mpe(*e, "simple_speaker_listener", cfg);
  else if (id == "MPE_simple_tag_v3") make_mpe(*e, "simple_tag", cfg);
  else if (id.rfind("SMAX_", 0) == 0 && std::find(registered().begin(), registered().end(), id) != registered().end())
    make_smax(*e, id.substr(5), cfg);
  else {
    for (int l = 0; l < 5; ++l)
      if (id == std::string("overcooked_") + kLayoutNames[l] + "_v0") {
        make_overcooked(*e, l, cfg);
        return e;
      }
    for (const char* r : kReserved)
      if (id == r) raise(MARL_ERR_NOT_FOUND, "env id '" + id + "' is reserved but has no implementation yet");
    for (const char* r : kOffPath)
      if (id == r)
        raise(MARL_ERR_NOT_FOUND, "env id '" + id + "' exists in the reference but is outside the B200 "
                                  "batched hot path (see DESIGN.md)");
    raise(MARL_ERR_NOT_FOUND, "unknown env id '" + id + "' (see registered_envs())");
  }
  return e;
}


}  // namespace


namespace mhost {

void set_device(const marl_venv* h) { cuda_check(cudaSetDevice(h->device), "cudaSetDevice"); }

LaunchCommon common(marl_venv* h) {
  LaunchCommon lc;
  lc.n = h->n;
  lc.offset = h->off;
  lc.begin = 0;
  lc.end = h->n;
  lc.carry = h->carry;
  lc.v = h->v;
  lc.stats = h->stats;
  lc.err = h->err;
  lc.stream = h->stream;
  return lc;
}

void after_launch() { cuda_check(cudaGetLastError(), "kernel launch"); }

void require_state(const marl_venv* h) {
  if (!h->has_state) raise(MARL_ERR_CONTRACT, "VectorEnv::step: call reset() before step()");
}

// Surface (and clear) a device-side validation failure.
void check_device_error(marl_venv* h) {
  int rec[4];
  cuda_check(cudaMemcpyAsync(rec, h->err, sizeof rec, cudaMemcpyDeviceToHost, h->stream), "cudaMemcpyAsync");
  cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
  if (rec[0] == 0) return;
  const int A = h->env->A;
  const int64_t idx = rec[1];
  const int zero[4] = {0, 0x7fffffff, 0, 0};
  cuda_check(cudaMemcpy(h->err, zero, sizeof zero, cudaMemcpyHostToDevice), "cudaMemcpy");
  raise(MARL_ERR_CONTRACT, h->env->id + ": action for agent '" + h->env->agents[size_t(idx % A)] + "' of env " +
                               std::to_string(idx / A) + " is outside its action space");
}

// d_actions: [N][A] int32 ids, or [N][A][kBoxActDim] floats for box action spaces
void launch_step(marl_venv* h, bool random, const uint32_t* step_key, const void* d_actions, int64_t begin,
                 int64_t end) {
  require_state(h);
  LaunchCommon lc = common(h);
  lc.begin = begin;
  lc.end = end < 0 ? h->n : end;
  KeyWords k{};
  if (step_key) std::memcpy(k.w, step_key, 16);
  if (!random) {
    if (h->env->continuous)
      lc.v.actions_f = static_cast<float*>(const_cast<void*>(d_actions));
    else
      lc.v.actions = static_cast<int32_t*>(const_cast<void*>(d_actions));
  }
  switch (h->env->family) {
    case MARL_FAMILY_MPE: mpe_launch_step(h->env->mpe, h->mpe, lc, random, k); break;
    case MARL_FAMILY_SMAX: smax_launch_step(h->env->smax, h->smax, lc, random, k); break;
    default: oc_launch_step_t(h->env->oc, h->oc_templ, h->oc, lc, random, k); break;
  }
  after_launch();
}

// Rows [b, e) of every requested output view -> the host buffers, on stream st.
// The device address of a host pointer into mapped pinned memory (cudaHostAlloc
// / pin_memory under unified addressing), else null.
float* mapped_device_ptr(void* host) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
  return static_cast<float*>(at.devicePointer);
}

void download_range(marl_venv* h, const marl_host_step* o, int64_t b, int64_t e, cudaStream_t st) {
  const Env& E = *h->env;
  const size_t A = size_t(E.A), D = size_t(E.D), rows = size_t(e - b);
  auto cp = [&](void* dst, const void* src, size_t row_bytes) {
    if (dst)
      cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + size_t(b) * row_bytes,
                                 static_cast<const uint8_t*>(src) + size_t(b) * row_bytes, rows * row_bytes,
                                 cudaMemcpyDeviceToHost, st),
                 "cudaMemcpyAsync D2H");
  };
  cp(o->obs, h->v.obs, A * D * 4);
  cp(o->rewards, h->v.rewards, A * 8);
  cp(o->dones, h->v.dones, A + 1);
  cp(o->finished, h->v.finished, 1);
  // final_obs is valid where finished (vector_env.hpp:31): a mapped pinned
  // destination receives only the finished rows, written by the device
  float* fo_dev = o->final_obs ? mapped_device_ptr(o->final_obs) : nullptr;
  if (fo_dev)
    launch_gather_finished_rows(h->v.finished + b, int64_t(rows), h->v.final_obs + size_t(b) * A * D,
                                fo_dev + size_t(b) * A * D, int64_t(A * D), st);
  else
    cp(o->final_obs, h->v.final_obs, A * D * 4);
  cp(o->final_returns, h->v.final_returns, 8);
  cp(o->final_lengths, h->v.final_lengths, 4);
  if (E.n_info) cp(o->infos, h->v.infos, A * size_t(E.n_info) * 8);
  cp(o->actions, h->v.actions, A * 4);
}

// A step whose outputs go to host buffers: the batch runs as up to four env
// chunks on the compute stream and each chunk's rows are copied back on a
// second stream as soon as its kernel finishes, so the PCIe transfer of one
// chunk overlaps the step of the next (the step is per-env independent, so
// chunking changes nothing in the results).
void step_to_host(marl_venv* h, bool random, const uint32_t* step_key, const void* d_actions,
                  const marl_host_step* o) {
  const int64_t n = h->n;
  const int K = n >= 32768 ? 4 : 1;
  if (K == 1) {
    launch_step(h, random, step_key, d_actions);
    download_range(h, o, 0, n, h->stream);
    cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    return;
  }
  if (!h->copy_stream) {
    cuda_check(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& ev : h->chunk_ev) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  }
  int64_t b = 0;
  for (int c = 0; c < K; ++c) {
    const int64_t e = c == K - 1 ? n : std::min(n, ((n * (c + 1) / K) + 255) / 256 * 256);
    if (e <= b) continue;
    launch_step(h, random, step_key, d_actions, b, e);
    cuda_check(cudaEventRecord(h->chunk_ev[c], h->stream), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(h->copy_stream, h->chunk_ev[c], 0), "cudaStreamWaitEvent");
    download_range(h, o, b, e, h->copy_stream);
    b = e;
  }
  cuda_check(cudaStreamSynchronize(h->copy_stream), "cudaStreamSynchronize");
  cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
}

void download(marl_venv* h, const marl_host_step* o) {
  const Env& e = *h->env;
  const size_t N = size_t(h->n), A = size_t(e.A), D = size_t(e.D);
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    if (dst) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream), "cudaMemcpyAsync D2H");
  };
  cp(o->obs, h->v.obs, N * A * D * 4);
  cp(o->rewards, h->v.rewards, N * A * 8);
  cp(o->dones, h->v.dones, N * (A + 1));
  cp(o->finished, h->v.finished, N);
  cp(o->final_obs, h->v.final_obs, N * A * D * 4);
  cp(o->final_returns, h->v.final_returns, N * 8);
  cp(o->final_lengths, h->v.final_lengths, N * 4);
  if (e.n_info) cp(o->infos, h->v.infos, N * A * size_t(e.n_info) * 8);
  cp(o->actions, h->v.actions, N * A * 4);
  cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
}

void create(const char* env_id, const char* cfg, int64_t n_local, int64_t offset, int64_t global_n, int device,
            marl_venv** out) {
  if (!env_id) raise(MARL_ERR_CONTRACT, "env_id is NULL");
  if (n_local < 1) raise(MARL_ERR_CONTRACT, "VectorEnv: n_envs must be >= 1");
  if (offset < 0 || global_n < offset + n_local) raise(MARL_ERR_CONTRACT, "VectorEnv: shard range outside the global batch");
  if (global_n > (int64_t(1) << 40)) raise(MARL_ERR_CONTRACT, "VectorEnv: global batch too large");
  auto h = std::make_unique<marl_venv>();
  h->env = make_env(env_id, cfg);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    raise(MARL_ERR_CUDA, "no CUDA device available: the B200 engine has no CPU fallback");
  if (device < 0 || device >= ndev) raise(MARL_ERR_CONTRACT, "device index out of range");
  h->device = device;
  h->n = n_local;
  h->off = offset;
  h->gn = global_n;
  set_device(h.get());
  cuda_check(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  h->own_stream = true;
  const Env& e = *h->env;
  const size_t N = size_t(n_local), A = size_t(e.A), D = size_t(e.D);
  Arena& ar = h->arena;
  ar.add(&h->v.obs, N * A * D);
  ar.add(&h->v.final_obs, N * A * D);
  ar.add(&h->v.rewards, N * A);
  ar.add(&h->v.dones, N * (A + 1));
  ar.add(&h->v.finished, N);
  ar.add(&h->v.final_returns, N);
  ar.add(&h->v.final_lengths, N);
  ar.add(&h->v.infos, N * A * size_t(std::max(e.n_info, 1)));
  ar.add(&h->v.actions, N * A);
  if (e.continuous) ar.add(&h->v.actions_f, N * A * size_t(kBoxActDim));
  ar.add(&h->carry.keys, N);
  ar.add(&h->carry.ep_return, N);
  ar.add(&h->carry.ep_length, N);
  ar.add(&h->stats, 3);
  ar.add(&h->err, 4);
  ar.add(&h->n_actions_dev, A);
  ar.add(&h->ws_seg, 2 * A);
  if (e.family == MARL_FAMILY_MPE) {
    int s = e.mpe.scenario;
    ar.add(&h->mpe.pos, N * 2 * size_t(mpe_n_entities(s)));
    ar.add(&h->mpe.vel, N * 2 * A);
    ar.add(&h->mpe.comm, N * A * size_t(mpe_dim_c(s)));
    ar.add(&h->mpe.steps, N);
    ar.add(&h->mpe.goal, N);
  } else if (e.family == MARL_FAMILY_SMAX) {
    size_t U = size_t(e.smax.na + e.smax.ne);
    ar.add(&h->smax.x, N * U);
    ar.add(&h->smax.y, N * U);
    ar.add(&h->smax.health, N * U);
    ar.add(&h->smax.cooldown, N * U);
    ar.add(&h->smax.mem, N * U);
    ar.add(&h->smax.t, N);
  } else {
    ar.add(&h->oc.agents, N);
    ar.add(&h->oc.pots, N * size_t(std::max(e.oc.n_pots, 1)));
    ar.add(&h->oc.counters, N * 2);
    ar.add(&h->oc.t, N);
    ar.add(&h->oc_templ, D);
  }
  ar.commit();
  const int zero[4] = {0, 0x7fffffff, 0, 0};
  cuda_check(cudaMemcpy(h->err, zero, sizeof zero, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(h->n_actions_dev, e.n_actions.data(), A * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  {  // world_state segments (mpe.cpp:229-242: every agent's row; overcooked.cpp:315-319: agent 0's)
    std::vector<int32_t> seg;
    if (e.family == MARL_FAMILY_MPE) {
      for (int a = 0; a < e.A; ++a) seg.push_back(a * e.D);
      for (int a = 0; a < e.A; ++a) seg.push_back(e.obs_size[size_t(a)]);
      h->ws_nseg = e.A;
    } else if (e.family == MARL_FAMILY_OVERCOOKED) {
      seg = {0, e.D};
      h->ws_nseg = 1;
    }
    h->ws_width = 0;
    for (int k = 0; k < h->ws_nseg; ++k) h->ws_width += seg[size_t(h->ws_nseg + k)];
    if (e.family == MARL_FAMILY_SMAX) h->ws_width = 18 * (e.smax.na + e.smax.ne) + 1;  // smax.cpp:161
    if (!seg.empty())
      cuda_check(cudaMemcpy(h->ws_seg, seg.data(), seg.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  }
  if (e.family == MARL_FAMILY_SMAX) smax_prepare(h->env->smax);
  if (e.family == MARL_FAMILY_OVERCOOKED)
    cuda_check(cudaMemcpy(h->oc_templ, e.oc_templ.data(), D * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  *out = h.release();
}

void copy_name(const std::string& s, char* dst, size_t cap) {
  if (!dst || cap == 0) return;
  std::snprintf(dst, cap, "%s", s.c_str());
}

}  // namespace

extern "C" {

const char* marl_last_error(void) { return g_err.c_str(); }
uint64_t marl_launch_count(void) { return g_launches; }
int marl_set_grid_cap(int ctas) {
  const int old = g_grid_cap;
  g_grid_cap = ctas > 0 ? ctas : 0;
  return old;
}
const char* marl_version(void) { return "marl-b200 0.1 (sm_100a)"; }

int marl_gemm_f32(int64_t M, int N, int64_t K, const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn,
                  int64_t sbk, float* C, int64_t ldc, float beta, void* stream) {
  return guarded([&] {
    if ((M > 0 && N > 0) && (!A || !B || !C)) raise(MARL_ERR_CONTRACT, "marl_gemm_f32: NULL operand");
    if (M < 0 || N < 0 || K < 0 || N > 65535) raise(MARL_ERR_CONTRACT, "marl_gemm_f32: bad shape");
    cuda_check(tc_gemm(static_cast<cudaStream_t>(stream), M, N, K, A, sam, sak, B, sbn, sbk, C, ldc, beta), "tc_gemm");
  });
}

int marl_registered_count(void) { return int(registered().size()); }
const char* marl_registered_env(int i) {
  return (i >= 0 && i < int(registered().size())) ? registered()[size_t(i)].c_str() : nullptr;
}

int marl_env_describe(const char* env_id, const char* config_json, marl_spec* o) {
  return guarded([&] {
    if (!env_id) raise(MARL_ERR_CONTRACT, "env_id is NULL");
    auto e = make_env(env_id, config_json);
    std::memset(o, 0, sizeof *o);
    o->family = e->family;
    o->n_agents = e->A;
    o->obs_dim = e->D;
    o->n_actions = *std::max_element(e->n_actions.begin(), e->n_actions.end());
    o->n_info = e->n_info;
    o->max_steps = e->max_steps;
    o->cooperative = e->cooperative;
    o->device = -1;
  });
}

int marl_env_agent(const char* env_id, const char* config_json, int i, char* name, size_t cap, int32_t* obs_size,
                   int32_t* n_actions) {
  return guarded([&] {
    if (!env_id) raise(MARL_ERR_CONTRACT, "env_id is NULL");
    auto e = make_env(env_id, config_json);
    if (i < 0 || i >= e->A) raise(MARL_ERR_CONTRACT, "agent index out of range");
    copy_name(e->agents[size_t(i)], name, cap);
    if (obs_size) *obs_size = e->obs_size[size_t(i)];
    if (n_actions) *n_actions = e->n_actions[size_t(i)];
  });
}

int marl_venv_create(const char* env_id, const char* config_json, int64_t n_envs, int device, marl_venv** out) {
  return guarded([&] { create(env_id, config_json, n_envs, 0, n_envs, device, out); });
}

int marl_venv_create_shard(const char* env_id, const char* config_json, int64_t n_local, int64_t global_offset,
                           int64_t global_n, int device, marl_venv** out) {
  return guarded([&] { create(env_id, config_json, n_local, global_offset, global_n, device, out); });
}

int marl_venv_destroy(marl_venv* h) {
  return guarded([&] {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    if (h->env && h->env->family == MARL_FAMILY_SMAX) smax_release(h->env->smax);
    if (h->copy_stream) {
      cudaStreamSynchronize(h->copy_stream);
      cudaStreamDestroy(h->copy_stream);
      for (auto ev : h->chunk_ev) cudaEventDestroy(ev);
    }
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
  });
}

int marl_venv_set_stream(marl_venv* h, void* s) {
  return guarded([&] {
    set_device(h);
    cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = static_cast<cudaStream_t>(s);
    h->own_stream = false;
  });
}

int marl_venv_spec(const marl_venv* h, marl_spec* o) {
  return guarded([&] {
    const Env& e = *h->env;
    o->family = e.family;
    o->n_agents = e.A;
    o->obs_dim = e.D;
    o->n_actions = *std::max_element(e.n_actions.begin(), e.n_actions.end());
    o->n_info = e.n_info;
    o->max_steps = e.max_steps;
    o->cooperative = e.cooperative;
    o->device = h->device;
    o->n_envs = h->n;
    o->global_offset = h->off;
    o->global_n = h->gn;
  });
}

int marl_venv_agent(const marl_venv* h, int i, char* name, size_t cap, int32_t* obs_size, int32_t* n_actions) {
  return guarded([&] {
    const Env& e = *h->env;
    if (i < 0 || i >= e.A) raise(MARL_ERR_CONTRACT, "agent index out of range");
    copy_name(e.agents[size_t(i)], name, cap);
    if (obs_size) *obs_size = e.obs_size[size_t(i)];
    if (n_actions) *n_actions = e.n_actions[size_t(i)];
  });
}

int marl_venv_info_name(const marl_venv* h, int k, char* name, size_t cap) {
  return guarded([&] {
    if (k < 0 || k >= h->env->n_info) raise(MARL_ERR_CONTRACT, "info index out of range");
    copy_name(h->env->info_names[size_t(k)], name, cap);
  });
}

int marl_venv_id(const marl_venv* h, char* name, size_t cap) {
  return guarded([&] { copy_name(h->env->id, name, cap); });
}

int marl_venv_reset(marl_venv* h, const uint32_t key[4]) {
  return guarded([&] {
    set_device(h);
    Key k{key[0], key[1], key[2], key[3]};
    Key cp = fold_in(k, 1);  // vector_env.cpp:55
    KeyWords kw{{k.k0, k.k1, k.c0, k.c1}}, cw{{cp.k0, cp.k1, cp.c0, cp.c1}};
    LaunchCommon lc = common(h);
    const int zero[4] = {0, 0x7fffffff, 0, 0};
    cuda_check(cudaMemcpyAsync(h->err, zero, sizeof zero, cudaMemcpyHostToDevice, h->stream), "cudaMemcpyAsync");
    switch (h->env->family) {
      case MARL_FAMILY_MPE: mpe_launch_reset(h->env->mpe, h->mpe, lc, kw, cw); break;
      case MARL_FAMILY_SMAX: smax_launch_reset(h->env->smax, h->smax, lc, kw, cw); break;
      default: oc_launch_reset_t(h->env->oc, h->oc_templ, h->oc, lc, kw, cw); break;
    }
    after_launch();
    h->has_state = true;
  });
}

int marl_venv_step(marl_venv* h, const int32_t* d_actions) {
  return guarded([&] {
    set_device(h);
    require_state(h);
    if (!d_actions) raise(MARL_ERR_CONTRACT, "VectorEnv::step: actions is NULL");
    if (h->env->continuous)
      raise(MARL_ERR_CONTRACT, h->env->id + ": box action spaces take float actions (marl_venv_step_continuous)");
    launch_validate(d_actions, h->n, h->env->A, h->n_actions_dev, h->err, h->stream);
    after_launch();
    launch_step(h, false, nullptr, d_actions);
  });
}

int marl_venv_step_random(marl_venv* h, const uint32_t step_key[4]) {
  return guarded([&] {
    if (!h || !step_key) raise(MARL_ERR_CONTRACT, "marl_venv_step_random: NULL argument");
    set_device(h);
    launch_step(h, true, step_key, nullptr);
  });
}

int marl_venv_probe_steps(marl_venv* h, const uint32_t parent[4], uint64_t t0, int n_steps) {
  return guarded([&] {
    if (!h || !parent) raise(MARL_ERR_CONTRACT, "marl_venv_probe_steps: NULL argument");
    if (n_steps < 0) raise(MARL_ERR_CONTRACT, "marl_venv_probe_steps: n_steps must be >= 0");
    set_device(h);
    require_state(h);
    if (n_steps == 0) return;
    Key p{parent[0], parent[1], parent[2], parent[3]};
    if (h->env->family == MARL_FAMILY_MPE) {
      // one launch for all K steps (state and carry in registers across them)
      LaunchCommon lc = common(h);
      lc.begin = 0;
      lc.end = h->n;
      KeyWords k{};
      std::memcpy(k.w, parent, 16);
      mpe_launch_probe(h->env->mpe, h->mpe, lc, k, t0, n_steps);
      after_launch();
      return;
    }
    for (int t = 0; t < n_steps; ++t) {
      Key sk = split_child(p, t0 + uint64_t(t));
      uint32_t s[4] = {sk.k0, sk.k1, sk.c0, sk.c1};
      launch_step(h, true, s, nullptr);
    }
  });
}

int marl_venv_step_host(marl_venv* h, const int32_t* h_actions, const marl_host_step* out) {
  return guarded([&] {
    if (!h || !h_actions) raise(MARL_ERR_CONTRACT, "marl_venv_step_host: NULL argument");
    set_device(h);
    require_state(h);
    const Env& e = *h->env;
    if (e.continuous)
      raise(MARL_ERR_CONTRACT, e.id + ": box action spaces take float actions (marl_venv_step_continuous_host)");
    const int64_t total = h->n * e.A;
    for (int64_t q = 0; q < total; ++q) {  // Env::validate_actions, env.cpp:7-14
      int a = int(q % e.A);
      if (h_actions[q] < 0 || h_actions[q] >= e.n_actions[size_t(a)])
        raise(MARL_ERR_CONTRACT, e.id + ": action for agent '" + e.agents[size_t(a)] + "' of env " +
                                     std::to_string(q / e.A) + " is outside its action space");
    }
    cuda_check(cudaMemcpyAsync(h->v.actions, h_actions, size_t(total) * 4, cudaMemcpyHostToDevice, h->stream),
               "cudaMemcpyAsync H2D");
    if (out) {
      step_to_host(h, false, nullptr, h->v.actions, out);
    } else {
      launch_step(h, false, nullptr, h->v.actions);
      cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    }
  });
}

int marl_venv_step_random_host(marl_venv* h, const uint32_t step_key[4], const marl_host_step* out) {
  return guarded([&] {
    if (!h || !step_key) raise(MARL_ERR_CONTRACT, "marl_venv_step_random_host: NULL argument");
    set_device(h);
    require_state(h);
    if (out) {
      step_to_host(h, true, step_key, nullptr, out);
    } else {
      launch_step(h, true, step_key, nullptr);
      cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    }
  });
}

// ---- box action spaces (continuous MPE, mpe.cpp:91-99, 144-166)
int marl_venv_action_dim(const marl_venv* h, int32_t* out) {
  return guarded([&] {
    if (!h || !out) raise(MARL_ERR_CONTRACT, "marl_venv_action_dim: NULL argument");
    *out = h->env->continuous ? kBoxActDim : 0;
  });
}

int marl_venv_actions_f32(marl_venv* h, float** out) {
  return guarded([&] {
    if (!h || !out) raise(MARL_ERR_CONTRACT, "marl_venv_actions_f32: NULL argument");
    *out = h->v.actions_f;
  });
}

int marl_venv_step_continuous(marl_venv* h, const float* d_actions) {
  return guarded([&] {
    set_device(h);
    require_state(h);
    if (!d_actions) raise(MARL_ERR_CONTRACT, "VectorEnv::step: actions is NULL");
    if (!h->env->continuous) raise(MARL_ERR_CONTRACT, h->env->id + ": discrete action spaces take int32 actions");
    launch_validate_box(d_actions, h->n, h->env->A, h->n_actions_dev, h->err, h->stream);
    after_launch();
    launch_step(h, false, nullptr, d_actions);
  });
}

int marl_venv_step_continuous_host(marl_venv* h, const float* h_actions, const marl_host_step* out) {
  return guarded([&] {
    set_device(h);
    require_state(h);
    const Env& e = *h->env;
    if (!h_actions) raise(MARL_ERR_CONTRACT, "VectorEnv::step: actions is NULL");
    if (!e.continuous) raise(MARL_ERR_CONTRACT, e.id + ": discrete action spaces take int32 actions");
    const int64_t rows = h->n * e.A;
    for (int64_t q = 0; q < rows; ++q) {  // Env::validate_actions -> SpaceDescriptor::contains (spaces.cpp:36-46)
      const int a = int(q % e.A);
      for (int k = 0; k < e.n_actions[size_t(a)]; ++k) {
        const float v = h_actions[q * kBoxActDim + k];
        if (!(v >= 0.0f && v <= 1.0f) || !std::isfinite(v))
          raise(MARL_ERR_CONTRACT, e.id + ": action for agent '" + e.agents[size_t(a)] + "' of env " +
                                       std::to_string(q / e.A) + " is outside its action space");
      }
    }
    cuda_check(cudaMemcpyAsync(h->v.actions_f, h_actions, size_t(rows) * kBoxActDim * 4, cudaMemcpyHostToDevice,
                               h->stream),
               "cudaMemcpyAsync H2D");
    if (out) {
      step_to_host(h, false, nullptr, h->v.actions_f, out);
    } else {
      launch_step(h, false, nullptr, h->v.actions_f);
      cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    }
  });
}

int marl_venv_download(marl_venv* h, const marl_host_step* out) {
  return guarded([&] {
    set_device(h);
    download(h, out);
    check_device_error(h);
  });
}

int marl_copy_device_to_host(void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    if (bytes && (!dst || !src)) raise(MARL_ERR_CONTRACT, "marl_copy_device_to_host: NULL pointer");
    if (bytes) cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  });
}

int marl_venv_views(marl_venv* h, marl_views* o) {
  return guarded([&] {
    o->obs = h->v.obs;
    o->rewards = h->v.rewards;
    o->dones = h->v.dones;
    o->finished = h->v.finished;
    o->final_obs = h->v.final_obs;
    o->final_returns = h->v.final_returns;
    o->final_lengths = h->v.final_lengths;
    o->infos = h->v.infos;
    o->actions = h->v.actions;
    o->keys = reinterpret_cast<uint32_t*>(h->carry.keys);
    o->episode_returns = h->carry.ep_return;
    o->episode_lengths = h->carry.ep_length;
  });
}

int marl_venv_legal(marl_venv* h, uint8_t* d_out) {
  return guarded([&] {
    set_device(h);
    require_state(h);
    const Env& e = *h->env;
    const int n_act = *std::max_element(e.n_actions.begin(), e.n_actions.end());
    if (e.family == MARL_FAMILY_SMAX) {
      smax_launch_legal(e.smax, h->smax, h->n, n_act, d_out, h->stream);
    } else {  // default all-legal masks (env.hpp:71-73), padded with zeros
      std::vector<uint8_t> row(size_t(e.A) * n_act, 0);
      for (int a = 0; a < e.A; ++a)
        for (int q = 0; q < e.n_actions[size_t(a)]; ++q) row[size_t(a) * n_act + q] = 1;
      cuda_check(cudaMemcpy2DAsync(d_out, row.size(), row.data(), 0, row.size(), size_t(h->n),
                                   cudaMemcpyHostToDevice, h->stream), "cudaMemcpy2DAsync");
      cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    }
    after_launch();
  });
}

int marl_venv_world_state_size(const marl_venv* h, int32_t* out) {
  return guarded([&] {
    if (!h || !out) raise(MARL_ERR_CONTRACT, "marl_venv_world_state_size: NULL argument");
    *out = h->ws_width;
  });
}

// Env::world_state of every env's current state (the MAPPO critic input,
// ppo.cpp:341-346): d_out [N][world_state_size] f32 (device).
int marl_venv_world_state(marl_venv* h, float* d_out) {
  return guarded([&] {
    set_device(h);
    require_state(h);
    if (!d_out) raise(MARL_ERR_CONTRACT, "marl_venv_world_state: NULL output");
    const Env& e = *h->env;
    if (e.family == MARL_FAMILY_SMAX)
      smax_launch_world_state(e.smax, h->smax, h->n, d_out, h->stream);
    else
      launch_obs_gather(h->v.obs, h->n, e.A * e.D, h->ws_seg, h->ws_seg + h->ws_nseg, h->ws_nseg, h->ws_width, d_out,
                        h->stream);
    after_launch();
  });
}

int marl_venv_state_hash(marl_venv* h, uint64_t* d_out) {
  return guarded([&] {
    set_device(h);
    require_state(h);
    const Env& e = *h->env;
    switch (e.family) {
      case MARL_FAMILY_MPE: mpe_launch_hash(e.mpe, h->mpe, h->n, d_out, h->stream); break;
      case MARL_FAMILY_SMAX: smax_launch_hash(e.smax, h->smax, h->n, d_out, h->stream); break;
      default: oc_launch_hash(e.oc, h->oc, h->n, d_out, h->stream); break;
    }
    after_launch();
  });
}

int marl_venv_episode_stats(marl_venv* h, int64_t out[3], int clear) {
  return guarded([&] {
    set_device(h);
    unsigned long long s[3];
    cuda_check(cudaMemcpyAsync(s, h->stats, sizeof s, cudaMemcpyDeviceToHost, h->stream), "cudaMemcpyAsync");
    if (clear) cuda_check(cudaMemsetAsync(h->stats, 0, sizeof s, h->stream), "cudaMemsetAsync");
    cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    for (int q = 0; q < 3; ++q) out[q] = int64_t(s[q]);
  });
}

int marl_venv_sync(marl_venv* h) {
  return guarded([&] {
    set_device(h);
    cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    check_device_error(h);
  });
}

int marl_throughput_probe(const char* env_id, const char* config_json, int64_t n_envs, int n_steps,
                          const uint32_t key[4], int device, double* seconds, double* cold_seconds) {
  marl_venv* h = nullptr;
  int rc = marl_venv_create(env_id, config_json, n_envs, device, &h);
  if (rc) return rc;
  rc = guarded([&] {
    if (n_steps < 1) raise(MARL_ERR_CONTRACT, "throughput_probe: n_steps must be >= 1");
    Key k{key[0], key[1], key[2], key[3]};
    Key parent = fold_in(k, 2);  // vector_env.cpp:202
    auto action_key = [&](uint64_t t) { return split_child(parent, t); };
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    cudaEventRecord(e0, h->stream);
    if (int r = marl_venv_reset(h, key)) raise(r, g_err);
    Key wk = action_key(uint64_t(n_steps));
    uint32_t w[4] = {wk.k0, wk.k1, wk.c0, wk.c1};
    if (int r = marl_venv_step_random(h, w)) raise(r, g_err);
    cudaEventRecord(e1, h->stream);
    const uint32_t pw[4] = {parent.k0, parent.k1, parent.c0, parent.c1};
    if (int r = marl_venv_probe_steps(h, pw, 0, n_steps)) raise(r, g_err);
    cudaEventRecord(e2, h->stream);
    cuda_check(cudaEventSynchronize(e2), "cudaEventSynchronize");
    float cold_ms = 0, warm_ms = 0;
    cudaEventElapsedTime(&cold_ms, e0, e1);
    cudaEventElapsedTime(&warm_ms, e1, e2);
    *cold_seconds = cold_ms * 1e-3;
    *seconds = std::max(warm_ms * 1e-3, 1e-9);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
  });
  marl_venv_destroy(h);
  return rc;
}

void marl_prng_key_from_seed(uint64_t seed, uint32_t out[4]) {  // prng.cpp:116-118
  out[0] = uint32_t(seed & 0xffffffffu);
  out[1] = uint32_t(seed >> 32);
  out[2] = out[3] = 0;
}
void marl_prng_split(const uint32_t key[4], uint64_t n, uint32_t* out) {
  Key k{key[0], key[1], key[2], key[3]};
  for (uint64_t i = 0; i < n; ++i) {
    Key c = split_child(k, i);
    out[4 * i] = c.k0;
    out[4 * i + 1] = c.k1;
    out[4 * i + 2] = c.c0;
    out[4 * i + 3] = c.c1;
  }
}
void marl_prng_fold_in(const uint32_t key[4], uint64_t d, uint32_t out[4]) {
  Key c = fold_in(Key{key[0], key[1], key[2], key[3]}, d);
  out[0] = c.k0;
  out[1] = c.k1;
  out[2] = c.c0;
  out[3] = c.c1;
}
uint64_t marl_prng_bits(const uint32_t key[4], uint64_t index) {
  return block_at(Key{key[0], key[1], key[2], key[3]}, index);
}
void marl_threefry2x32(uint32_t k0, uint32_t k1, uint32_t x0, uint32_t x1, uint32_t out[2]) {
  threefry2x32(k0, k1, x0, x1, out[0], out[1]);
}

}  // extern "C"

