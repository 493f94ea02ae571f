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
#include "marl_b200.h"

using nlohmann::json;
using namespace marl_b200;

namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void raise(int code, const std::string& msg) { throw Error(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
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

}  // namespace

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

namespace {

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
void launch_step(marl_venv* h, bool random, const uint32_t* step_key, const void* d_actions, int64_t begin = 0,
                 int64_t end = -1) {
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
const char* marl_version(void) { return "marl-b200 0.1 (sm_100a)"; }

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
    set_device(h);
    launch_step(h, true, step_key, nullptr);
  });
}

int marl_venv_step_host(marl_venv* h, const int32_t* h_actions, const marl_host_step* out) {
  return guarded([&] {
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

// ------------------------------------------------------ IPPO rollout (C5)
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

namespace {

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
  return n;
}

PolicyNetBf16 net_bf16_of(const marl_rollout* r) {
  PolicyNetBf16 n{};
  n.a1 = r->images;
  n.a2 = n.a1 + 128 * 32;
  n.c2 = n.a2 + 64 * 64;
  n.h3 = n.c2 + 64 * 64;
  n.hc3 = n.h3 + 16 * 64;
  n.bias = r->bias;
  return n;
}

void gemm_nt(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta);

// rnn_step of actor and critic for all R rows as SGEMMs (embed, GRU input and
// hidden paths, post, head) around the gate kernel; same arithmetic as the
// per-row kernel up to the GEMMs' summation order.
void rnn_collect_gemm(marl_rollout* r, const PolicyStep& s) {
  cudaStream_t st = r->h->stream;
  const int64_t R = r->R;
  const int in = r->in_dim, CI = r->critic_in, NA = r->n_act, F = r->F, H = r->H;
  rnn_policy_rows(s, r->b, in, CI, NA, H, r->s_xa, r->s_xc, r->h_actor, r->h_critic, r->s_hpeek, st);
  for (int branch = (s.bootstrap ? 1 : 0); branch < 2; ++branch) {
    const int bin = branch == 0 ? in : CI, out = branch == 0 ? NA : 1;
    const RnnWPtrs w = rnn_weights(branch == 0 ? r->params : r->params + r->n_actor, bin, F, H, out);
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

// hidden > 0: the recurrent policy (RnnBranch, fc width `width`, GRU `hidden`)
static marl_rollout* rollout_create_impl(marl_venv* h, int T, int width, int n_layers, int relu, int centralized,
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
    if (centralized && precision == 1)
      raise(MARL_ERR_SCHEMA, "rollout: the tcgen05 bf16 policy serves IPPO; use precision 0 for MAPPO");
    if (ps.critic_in > 1024) raise(MARL_ERR_SCHEMA, "rollout: critic input wider than 1024");
    if (ps.in_dim > 1024 || ps.n_actions > 64) raise(MARL_ERR_SCHEMA, "rollout: input wider than 1024 or > 64 actions");
    if (precision == 1 && !rollout_policy_bf16_supported(ps.in_dim, ps.n_actions, width))
      raise(MARL_ERR_SCHEMA, "rollout: the tcgen05 bf16 policy needs in_dim <= 32, n_actions <= 16, fc_width == 64");
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
    ar.add(&r->images, size_t(128 * 32 + 2 * 64 * 64 + 2 * 16 * 64));
    ar.add(&r->bias, size_t(4 * 64 + 2 * 16));
    ar.add(&r->agent_actions, size_t(e.A));
    if (hidden > 0) {
      r->recurrent = 1;
      r->F = width;
      r->H = hidden;
      for (float** q : {&r->h_actor, &r->h_critic, &r->h0_actor, &r->h0_critic})
        ar.add(q, size_t(r->R) * size_t(hidden));
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

extern "C++" {
namespace {
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
}  // namespace
}  // extern "C++"

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
    for (int t = 0; t < n_steps; ++t) {
      Key sk = action_key(uint64_t(t));
      uint32_t s[4] = {sk.k0, sk.k1, sk.c0, sk.c1};
      if (int r = marl_venv_step_random(h, s)) raise(r, g_err);
    }
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

// ====================================================================== PPO
// train_ippo / train_mappo (ppo.cpp:518-651) around the device update
// (ppo.cu): PpoConfig::from_config + validate (ppo.cpp:18-62), ppo_init_nets
// (ppo.cpp:109-124) on the host, and the update loop with its metrics row.
namespace {

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

PpoCfg parse_ppo_config(const char* text) {
  json j = (text && *text) ? json::parse(text) : json::object();
  ConfigView v(j, "ppo config");
  PpoCfg c;
  c.total_timesteps = v.get_int64("total_timesteps", c.total_timesteps);
  c.n_envs = v.get_int("n_envs", c.n_envs);
  c.n_rollout_steps = v.get_int("n_rollout_steps", c.n_rollout_steps);
  c.lr = v.get_double("lr", c.lr);
  c.anneal_lr = v.get_bool("anneal_lr", c.anneal_lr);
  c.update_epochs = v.get_int("update_epochs", c.update_epochs);
  c.n_minibatches = v.get_int("n_minibatches", c.n_minibatches);
  c.gamma = v.get_double("gamma", c.gamma);
  c.gae_lambda = v.get_double("gae_lambda", c.gae_lambda);
  c.clip_eps = v.get_double("clip_eps", c.clip_eps);
  c.ent_coef = v.get_double("ent_coef", c.ent_coef);
  c.vf_coef = v.get_double("vf_coef", c.vf_coef);
  c.max_grad_norm = v.get_double("max_grad_norm", c.max_grad_norm);
  c.activation = v.get_string("activation", c.activation);
  c.recurrent = v.get_bool("recurrent", c.recurrent);
  c.n_fc_layers = v.get_int("n_fc_layers", c.n_fc_layers);
  c.fc_width = v.get_int("fc_width", c.fc_width);
  c.hidden_width = v.get_int("hidden_width", c.hidden_width);
  c.shaped_rewards = v.get_bool("shaped_rewards", c.shaped_rewards);
  v.check_no_extras();
  auto bad = [](const std::string& what) { raise(MARL_ERR_SCHEMA, "ppo config: " + what); };
  if (c.total_timesteps < 0) bad("total_timesteps must be >= 0");
  if (c.n_envs <= 0) bad("n_envs must be positive");
  if (c.n_rollout_steps <= 0) bad("n_rollout_steps must be positive");
  if (c.lr <= 0) bad("lr must be positive");
  if (c.update_epochs <= 0) bad("update_epochs must be positive");
  if (c.n_minibatches <= 0) bad("n_minibatches must be positive");
  if (c.gamma < 0 || c.gamma > 1) bad("gamma must lie in [0, 1]");
  if (c.gae_lambda < 0 || c.gae_lambda > 1) bad("gae_lambda must lie in [0, 1]");
  if (c.clip_eps <= 0 || c.clip_eps >= 1) bad("clip_eps must lie in (0, 1)");
  if (c.ent_coef < 0) bad("ent_coef must be >= 0");
  if (c.vf_coef < 0) bad("vf_coef must be >= 0");
  if (c.max_grad_norm <= 0) bad("max_grad_norm must be positive");
  if (c.activation != "tanh" && c.activation != "relu") bad("activation must be 'tanh' or 'relu'");
  if (c.n_fc_layers <= 0) bad("n_fc_layers must be positive");
  if (c.fc_width <= 0) bad("fc_width must be positive");
  if (c.hidden_width <= 0) bad("hidden_width must be positive");
  return c;
}

Key key4(const uint32_t k[4]) { return Key{k[0], k[1], k[2], k[3]}; }
void put_key(const Key& k, uint32_t out[4]) {
  out[0] = k.k0;
  out[1] = k.k1;
  out[2] = k.c0;
  out[3] = k.c1;
}

// prng::normal (prng.cpp:161-175): Box-Muller over the key's blocks.
std::vector<double> host_normal(const Key& key, size_t n) {
  constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi
  std::vector<double> out(n);
  const size_t pairs = (n + 1) / 2;
  for (size_t p = 0; p < pairs; ++p) {
    const double u1 = double((block_at(key, 2 * p) >> 11) + 1) * 0x1.0p-53;
    const double u2 = to_unit(block_at(key, 2 * p + 1));
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * kPi * u2;
    out[2 * p] = r * std::cos(theta);
    if (2 * p + 1 < n) out[2 * p + 1] = r * std::sin(theta);
  }
  return out;
}

// nn::orthogonal (nn.hpp:457-486): modified Gram-Schmidt on a big x small
// normal draw; the smaller dimension is orthonormal, scaled by gain.
void host_orthogonal(const Key& key, int rows, int cols, float gain, float* w) {
  const int big = std::max(rows, cols), small = std::min(rows, cols);
  auto draws = host_normal(key, size_t(big) * size_t(small));
  std::vector<std::vector<double>> q(size_t(small), std::vector<double>(size_t(big), 0.0));
  for (int c = 0; c < small; ++c)
    for (int r = 0; r < big; ++r) q[size_t(c)][size_t(r)] = draws[size_t(r) * size_t(small) + size_t(c)];
  for (int c = 0; c < small; ++c) {
    auto& col = q[size_t(c)];
    for (int prev = 0; prev < c; ++prev) {
      const auto& pv = q[size_t(prev)];
      double dot = 0.0;
      for (int r = 0; r < big; ++r) dot += col[size_t(r)] * pv[size_t(r)];
      for (int r = 0; r < big; ++r) col[size_t(r)] -= dot * pv[size_t(r)];
    }
    double nrm = 0.0;
    for (double x : col) nrm += x * x;
    nrm = std::sqrt(nrm);
    if (!(nrm > 1e-12)) raise(MARL_ERR_CONTRACT, "nn: orthogonal: degenerate draw");
    for (double& x : col) x /= nrm;
  }
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      const double x = rows >= cols ? q[size_t(c)][size_t(r)] : q[size_t(r)][size_t(c)];
      w[size_t(r) * size_t(cols) + size_t(c)] = float(double(gain) * x);
    }
}

// ff_init (actor_critic.hpp:36-46) packed: torso layer l = dense_init(fold_in(
// fold_in(key,1), l), W, in_l, sqrt 2) with zero bias, head = dense_init(
// fold_in(key,2), out, W, head_gain).
void host_ff_init(const Key& key, int in, int n_layers, int W, int out, float head_gain, float* dst) {
  const Key torso = fold_in(key, 1);
  const float g = float(std::sqrt(2.0));
  int prev = in;
  for (int l = 0; l < n_layers; ++l) {
    host_orthogonal(fold_in(torso, uint64_t(l)), W, prev, g, dst);
    dst += size_t(W) * size_t(prev);
    std::fill(dst, dst + W, 0.0f);
    dst += W;
    prev = W;
  }
  host_orthogonal(fold_in(key, 2), out, W, head_gain, dst);
  dst += size_t(out) * size_t(W);
  std::fill(dst, dst + out, 0.0f);
}

// rnn_init (actor_critic.hpp:82-90) packed: embed = dense(fold_in(fold_in(k,1),0)),
// gru_init(fold_in(k,2)) (nn.hpp:508-517), post = dense(fold_in(fold_in(k,3),0)),
// head = dense(fold_in(k,4), head_gain); biases zero.
void host_rnn_init(const Key& key, int in, int F, int H, int out, float head_gain, float* dst) {
  const float g = float(std::sqrt(2.0));
  host_orthogonal(fold_in(fold_in(key, 1), 0), F, in, g, dst);
  dst += size_t(F) * size_t(in);
  std::fill(dst, dst + F, 0.0f);
  dst += F;
  const Key kg = fold_in(key, 2);
  for (int j = 0; j < 3; ++j) {
    host_orthogonal(fold_in(kg, uint64_t(j)), H, F, 1.0f, dst);
    dst += size_t(H) * size_t(F);
  }
  for (int j = 3; j < 6; ++j) {
    host_orthogonal(fold_in(kg, uint64_t(j)), H, H, 1.0f, dst);
    dst += size_t(H) * size_t(H);
  }
  std::fill(dst, dst + 6 * H, 0.0f);
  dst += 6 * H;
  host_orthogonal(fold_in(fold_in(key, 3), 0), F, H, g, dst);
  dst += size_t(F) * size_t(H);
  std::fill(dst, dst + F, 0.0f);
  dst += F;
  host_orthogonal(fold_in(key, 4), out, F, head_gain, dst);
  dst += size_t(out) * size_t(F);
  std::fill(dst, dst + out, 0.0f);
}

}  // namespace

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
  bool tc = false;  // minibatch step on tcgen05 (bf16 precision, the C5 shape)
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
  ~marl_ppo();
};

namespace {

// (definition below, after the NCCL loader)
// NCCL, loaded at run time (the process's libnccl.so.2 -- torch's, when torch
// is loaded -- so the library has no link-time NCCL dependency).
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      x.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (x.lib) break;
    }
    if (!x.lib) return x;
    x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(x.lib, "ncclGetUniqueId"));
    x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(x.lib, "ncclCommInitRank"));
    x.all_reduce = reinterpret_cast<decltype(x.all_reduce)>(dlsym(x.lib, "ncclAllReduce"));
    x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(x.lib, "ncclCommDestroy"));
    x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(x.lib, "ncclGetErrorString"));
    return x;
  }();
  if (!n.lib || !n.comm_init_rank || !n.all_reduce || !n.get_unique_id)
    raise(MARL_ERR_CUDA, "NCCL (libnccl.so.2) is not loadable in this process");
  return n;
}

// cuBLAS SGEMM / SGEMV for the recurrent update's per-step GEMMs (plain
// library GEMMs), loaded at run time like NCCL (torch's copy when loaded).
struct Blas {
  void* lib = nullptr;
  void* handle = nullptr;
  int (*create)(void**) = nullptr;
  int (*set_stream)(void*, cudaStream_t) = nullptr;
  int (*sgemm)(void*, int, int, int, int, int, const float*, const float*, int, const float*, int, const float*,
               float*, int) = nullptr;
  int (*sgemv)(void*, int, int, int, const float*, const float*, int, const float*, int, const float*, float*,
               int) = nullptr;
};

Blas& blas(cudaStream_t st) {
  static Blas b = [] {
    Blas x;
    for (const char* name : {"libcublas.so.12", "libcublas.so"}) {
      x.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (x.lib) break;
    }
    if (!x.lib) return x;
    x.create = reinterpret_cast<decltype(x.create)>(dlsym(x.lib, "cublasCreate_v2"));
    x.set_stream = reinterpret_cast<decltype(x.set_stream)>(dlsym(x.lib, "cublasSetStream_v2"));
    x.sgemm = reinterpret_cast<decltype(x.sgemm)>(dlsym(x.lib, "cublasSgemm_v2"));
    x.sgemv = reinterpret_cast<decltype(x.sgemv)>(dlsym(x.lib, "cublasSgemv_v2"));
    if (x.create && x.create(&x.handle) != 0) x.handle = nullptr;
    return x;
  }();
  if (!b.handle || !b.sgemm || !b.sgemv || !b.set_stream)
    raise(MARL_ERR_CUDA, "cuBLAS (libcublas.so.12) is not loadable in this process");
  b.set_stream(b.handle, st);
  return b;
}
constexpr int kOpN = 0, kOpT = 1;

// Row-major GEMMs on column-major cuBLAS.
// C[M x N] = A[M x K] . B[N x K]^T (+ beta C)
void gemm_nt(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta) {
  const float one = 1.0f;
  if (blas(st).sgemm(blas(st).handle, kOpT, kOpN, N, int(M), K, &one, B, ldb, A, lda, &beta, C, ldc) != 0)
    raise(MARL_ERR_CUDA, "cublasSgemm failed");
}
// C[M x N] = A[M x K] . B[K x N] (+ beta C)
void gemm_nn(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta) {
  const float one = 1.0f;
  if (blas(st).sgemm(blas(st).handle, kOpN, kOpN, N, int(M), K, &one, B, ldb, A, lda, &beta, C, ldc) != 0)
    raise(MARL_ERR_CUDA, "cublasSgemm failed");
}
// G[O x I] = D[K x O]^T . X[K x I] (+ beta G): matmul_tn summed over all rows
void gemm_tn(cudaStream_t st, int O, int I, int64_t K, const float* D, int ldd, const float* X, int ldx, float* G,
             float beta) {
  const float one = 1.0f;
  if (blas(st).sgemm(blas(st).handle, kOpN, kOpT, I, O, int(K), &one, X, ldx, D, ldd, &beta, G, I) != 0)
    raise(MARL_ERR_CUDA, "cublasSgemm failed");
}
// g[O] = sum_k D[k][o] (+ beta g): the bias gradients
void colsum(cudaStream_t st, int O, int64_t K, const float* D, int ldd, const float* ones, float* g, float beta) {
  const float one = 1.0f;
  if (blas(st).sgemv(blas(st).handle, kOpN, O, int(K), &one, D, ldd, ones, 1, &beta, g, 1) != 0)
    raise(MARL_ERR_CUDA, "cublasSgemv failed");
}

// the native hook: an in-place NCCL sum on the trainer's stream (no host sync)
int nccl_hook(void* ctx, void* buf, int64_t count, int dtype, void* stream) {
  const Nccl& n = nccl();
  const ncclDataType_t t = dtype == MARL_DTYPE_F32 ? ncclFloat32 : dtype == MARL_DTYPE_F64 ? ncclFloat64 : ncclInt64;
  const ncclResult_t r = n.all_reduce(buf, buf, size_t(count), t, ncclSum, static_cast<ncclComm_t>(ctx),
                                      static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : int(r);
}

}  // namespace

marl_ppo::~marl_ppo() {
  if (nccl_comm) nccl().comm_destroy(static_cast<ncclComm_t>(nccl_comm));
  if (ro) marl_rollout_destroy(ro);
}

namespace {

// Sum `count` values at device `buf` over the data-parallel ranks.  A user
// hook sees the stream already synchronised and must return with the sum in
// place; the native NCCL hook is stream-ordered.
void allreduce(marl_ppo* p, void* buf, int64_t count, int dtype) {
  if (!p->hook) return;
  cudaStream_t st = p->h->stream;
  if (p->hook != nccl_hook) cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  const int rc = p->hook(p->hook_ctx, buf, count, dtype, st);
  if (rc != 0) raise(MARL_ERR_CUDA, "ppo: all-reduce hook failed (" + std::to_string(rc) + ")");
}

PpoBranchArgs branch_args(marl_ppo* p, bool actor, const int32_t* idx, int64_t M) {
  marl_rollout* r = p->ro;
  PpoBranchArgs a{};
  a.params = actor ? r->params : r->params + r->n_actor;
  a.gpart = actor ? p->gpart_a : p->gpart_c;
  a.spart = actor ? p->spart_a : p->spart_c;
  a.idx = idx;
  a.M = M;
  a.x = (!actor && r->centralized) ? r->b.critic_in : r->b.obs;
  a.actions = r->b.actions;
  a.old_logp = r->b.logp;
  a.adv = r->b.adv;
  a.vtarg = r->b.vtarg;
  a.old_value = r->b.value;
  a.active = r->b.active;
  a.legal = r->b.legal;
  a.st = p->mbst;
  a.err = p->flags + 1;
  a.in = actor ? r->in_dim : r->critic_in;
  a.W = r->width;
  a.out = actor ? r->n_act : 1;
  a.relu = r->relu;
  a.clip_eps = p->cfg.clip_eps;
  a.ent_coef = p->cfg.ent_coef;
  a.vf_coef = p->cfg.vf_coef;
  return a;
}

// ff_minibatch's gradient (ppo.cpp:409-441) into p->grad (actor | critic).
// global: idx are slots of the GLOBAL rollout (t*R_global + r); a sharded
// trainer keeps the ones it owns and all-reduces the sums.
void minibatch_grad(marl_ppo* p, const int32_t* idx, int64_t M, bool global = false) {
  cudaStream_t st = p->h->stream;
  if (global && p->sharded) {
    ppo_shard_compact(idx, M, p->R_global, p->row0, p->R_local, p->cmp_tmp, p->cmp_out, p->cmp_count,
                      p->cmp_scratch, p->cmp_scratch_bytes, st);
    after_launch();
    int64_t m_local = 0;
    cuda_check(cudaMemcpyAsync(&m_local, p->cmp_count, 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    idx = p->cmp_out;
    M = m_local;
  }
  std::function<void(double*, int)> red;
  if (p->hook) red = [p](double* g, int n) { allreduce(p, g, n, MARL_DTYPE_F64); };
  ppo_adv_stats(p->ro->b, idx, M, p->adv_part, p->adv_part2, p->adv_g, p->mbst, st, red);
  if (p->tc) {
    const marl_rollout* r = p->ro;
    PpoTcArgs a{};
    a.actor = r->params;
    a.critic = r->params + r->n_actor;
    a.gpart_a = p->gpart_a;
    a.gpart_c = p->gpart_c;
    a.spart_a = p->spart_a;
    a.spart_c = p->spart_c;
    a.idx = idx;
    a.M = M;
    a.obs = r->b.obs;
    a.actions = r->b.actions;
    a.old_logp = r->b.logp;
    a.adv = r->b.adv;
    a.vtarg = r->b.vtarg;
    a.old_value = r->b.value;
    a.active = r->b.active;
    a.legal = r->b.legal;
    a.st = p->mbst;
    a.err = p->flags + 1;
    a.in = r->in_dim;
    a.n_act = r->n_act;
    a.relu = r->relu;
    a.clip_eps = p->cfg.clip_eps;
    a.ent_coef = p->cfg.ent_coef;
    a.vf_coef = p->cfg.vf_coef;
    ppo_update_tc(a, p->grid_a, st);
  } else {
    ppo_branch(branch_args(p, true, idx, M), true, p->grid_a, st);
    ppo_branch(branch_args(p, false, idx, M), false, p->grid_c, st);
  }
  ppo_grad_reduce(p->gpart_a, p->grid_a, p->Pa, p->grad, st);
  ppo_grad_reduce(p->gpart_c, p->grid_c, p->Pc, p->grad + p->Pa, st);
  after_launch();
  if (p->hook) {  // the data-parallel exchange: gradient and loss sums over the ranks
    ppo_stats_fold(p->spart_a, p->grid_a, st);
    ppo_stats_fold(p->spart_c, p->grid_c, st);
    after_launch();
    allreduce(p, p->grad, p->P, MARL_DTYPE_F32);
    allreduce(p, p->spart_a, 6, MARL_DTYPE_F64);
    allreduce(p, p->spart_c, 6, MARL_DTYPE_F64);
  }
}

// rnn_seq_forward with cache (actor_critic.hpp:130-158) of one branch over
// the Mc rows of a chunk: per step, the gather / reset kernel, SGEMMs for
// embed, the GRU's input and hidden paths ([Wz;Wr;Wn] and [Uz;Ur;Un] as one
// GEMM each), post and head, with the gate arithmetic in one kernel.
void rnn_chunk_forward(marl_ppo* p, int branch, const int32_t* rows, int64_t Mc) {
  marl_rollout* r = p->ro;
  cudaStream_t st = p->h->stream;
  const RnnCache& c = branch == 0 ? p->rca : p->rcc;
  const int in = branch == 0 ? r->in_dim : r->critic_in, out = branch == 0 ? r->n_act : 1, F = r->F, H = r->H;
  const RnnWPtrs w = rnn_weights(branch == 0 ? r->params : r->params + r->n_actor, in, F, H, out);
  RnnStepArgs a{};
  a.M = Mc;
  a.R = r->R;
  a.in = in;
  a.H = H;
  a.rows = rows;
  a.resets = r->b.resets;
  a.src = (branch == 1 && r->centralized) ? r->b.critic_in : r->b.obs;
  a.h0 = branch == 0 ? r->h0_actor : r->h0_critic;
  a.h = p->rnn_h;
  a.w.bzx = w.bias6;
  a.w.brx = w.bias6 + H;
  a.w.bnx = w.bias6 + 2 * H;
  a.w.bzh = w.bias6 + 3 * H;
  a.w.brh = w.bias6 + 4 * H;
  a.w.bnh = w.bias6 + 5 * H;
  for (int t = 0; t < r->T; ++t) {
    const size_t k0 = size_t(t) * size_t(Mc);
    a.t = t;
    a.x = c.x + k0 * in;
    a.hprev = c.h + k0 * H;
    a.z = c.z + k0 * H;
    a.r = c.r + k0 * H;
    a.c = c.c + k0 * H;
    a.ah = c.ah + k0 * H;
    a.hn = c.hn + k0 * H;
    rnn_step_gather(a, st);
    float* e = c.e + k0 * F;
    gemm_nt(st, Mc, F, in, a.x, in, w.we, in, e, F, 0.0f);
    rnn_bias_act(e, Mc, F, w.be, true, r->relu, st);
    gemm_nt(st, Mc, 3 * H, F, e, F, w.wx, F, p->rnn_gx, 3 * H, 0.0f);
    gemm_nt(st, Mc, 3 * H, H, a.hprev, H, w.uh, H, p->rnn_gh, 3 * H, 0.0f);
    rnn_gates(a, p->rnn_gx, p->rnn_gh, st);
    float* pp = c.p + k0 * F;
    gemm_nt(st, Mc, F, H, a.hn, H, w.wp, H, pp, F, 0.0f);
    rnn_bias_act(pp, Mc, F, w.bp, true, r->relu, st);
    float* y = c.y + k0 * out;
    gemm_nt(st, Mc, out, F, pp, F, w.wh, F, y, out, 0.0f);
    rnn_bias_act(y, Mc, out, w.bh, false, r->relu, st);
  }
  after_launch();
}

// rnn_seq_backward (actor_critic.hpp:164-196) of one branch over a chunk, then
// its weight gradients (matmul_tn over every (t, row)) into G in pack order.
void rnn_chunk_backward(marl_ppo* p, int branch, const int32_t* rows, int64_t Mc, float* G, bool accumulate) {
  marl_rollout* r = p->ro;
  cudaStream_t st = p->h->stream;
  const RnnCache& c = branch == 0 ? p->rca : p->rcc;
  const int in = branch == 0 ? r->in_dim : r->critic_in, out = branch == 0 ? r->n_act : 1, F = r->F, H = r->H;
  const RnnWPtrs w = rnn_weights(branch == 0 ? r->params : r->params + r->n_actor, in, F, H, out);
  const int T = r->T;
  const int64_t Kc = int64_t(T) * Mc;
  RnnStepArgs a{};
  a.M = Mc;
  a.R = r->R;
  a.in = in;
  a.H = H;
  a.rows = rows;
  a.resets = r->b.resets;
  float* dh = p->rnn_dh;
  float* d4 = c.daz;  // [Kc][4H] = daz | dar | dac | dah
  for (int t = T - 1; t >= 0; --t) {
    const size_t k0 = size_t(t) * size_t(Mc);
    a.t = t;
    a.hprev = c.h + k0 * H;
    a.z = c.z + k0 * H;
    a.r = c.r + k0 * H;
    a.c = c.c + k0 * H;
    a.ah = c.ah + k0 * H;
    // head and post: dzp = (dy . Wh) * act'(p); dh_step = dzp . Wp + dh
    float* dzp = c.dzp + k0 * F;
    gemm_nn(st, Mc, F, out, c.dy + k0 * out, out, w.wh, F, dzp, F, 0.0f);
    rnn_act_grad(dzp, c.p + k0 * F, Mc * F, r->relu, st);
    gemm_nn(st, Mc, H, F, dzp, F, w.wp, H, dh, H, t == T - 1 ? 0.0f : 1.0f);
    // gru_backward: gates, carry dh = g*z, then dx and the gate paths of dh
    float* d4t = d4 + k0 * 4 * H;
    rnn_gru_bwd(a, dh, d4t, dh, st);
    float* dze = c.dze + k0 * F;
    gemm_nn(st, Mc, F, 3 * H, d4t, 4 * H, w.wx, F, dze, F, 0.0f);
    rnn_act_grad(dze, c.e + k0 * F, Mc * F, r->relu, st);
    gemm_nn(st, Mc, H, 2 * H, d4t, 4 * H, w.uh, H, dh, H, 1.0f);
    gemm_nn(st, Mc, H, H, d4t + 3 * H, 4 * H, w.uh + 2 * H * H, H, dh, H, 1.0f);
    rnn_cut(a, dh, st);
  }
  const float beta = accumulate ? 1.0f : 0.0f;
  const float* ones = p->rnn_ones;
  gemm_tn(st, F, in, Kc, c.dze, F, c.x, in, G, beta);  // embed
  G += size_t(F) * in;
  colsum(st, F, Kc, c.dze, F, ones, G, beta);
  G += F;
  gemm_tn(st, 3 * H, F, Kc, d4, 4 * H, c.e, F, G, beta);  // wz, wr, wn
  G += size_t(3) * H * F;
  gemm_tn(st, 2 * H, H, Kc, d4, 4 * H, c.h, H, G, beta);  // uz, ur
  G += size_t(2) * H * H;
  gemm_tn(st, H, H, Kc, d4 + 3 * H, 4 * H, c.h, H, G, beta);  // un
  G += size_t(H) * H;
  colsum(st, 3 * H, Kc, d4, 4 * H, ones, G, beta);  // bzx, brx, bnx
  G += 3 * H;
  colsum(st, 2 * H, Kc, d4, 4 * H, ones, G, beta);  // bzh, brh
  G += 2 * H;
  colsum(st, H, Kc, d4 + 3 * H, 4 * H, ones, G, beta);  // bnh
  G += H;
  gemm_tn(st, F, H, Kc, c.dzp, F, c.hn, H, G, beta);  // post
  G += size_t(F) * H;
  colsum(st, F, Kc, c.dzp, F, ones, G, beta);
  G += F;
  gemm_tn(st, out, F, Kc, c.dy, out, c.p, F, G, beta);  // head
  G += size_t(out) * F;
  colsum(st, out, Kc, c.dy, out, ones, G, beta);
  after_launch();
}

// rnn_minibatch's gradient (ppo.cpp:444-509): rnn_seq_forward with cache over
// the rows' whole sequences, ppo_row_loss over the [t][i] rows, rnn_seq_backward,
// and the weight gradients summed over every (t, row) in nn::pack order.
void minibatch_grad_rnn(marl_ppo* p, const int32_t* rows, int64_t M) {
  marl_rollout* r = p->ro;
  cudaStream_t st = p->h->stream;
  const int T = r->T;
  const int64_t K = int64_t(T) * M;
  // advantage statistics over the whole minibatch's [t][i] rows
  rnn_flat_slots(rows, M, T, r->R, p->rnn_flat, st);
  ppo_adv_stats(r->b, p->rnn_flat, K, p->adv_part, p->adv_part2, p->adv_g, p->mbst, st, {});
  // then the rows in chunks whose BPTT caches fit the budget; gradients and
  // per-block loss sums accumulate over the chunks
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(M, p->rnn_chunk));
  int blocks_done = 0;
  for (int64_t c0 = 0; c0 < M; c0 += chunk) {
    const int64_t Mc = std::min<int64_t>(chunk, M - c0), Kc = int64_t(T) * Mc;
    int32_t* flat_c = p->rnn_flat + K;  // the chunk's own [t][i] slots
    rnn_flat_slots(rows + c0, Mc, T, r->R, flat_c, st);
    // rnn_seq_forward with cache, both branches
    for (int branch = 0; branch < 2; ++branch) rnn_chunk_forward(p, branch, rows + c0, Mc);
    RnnSeqArgs la{};  // the loss reads the cached head outputs of both branches
    la.M = Mc;
    la.T = T;
    la.n_act = r->n_act;
    la.ca = p->rca;
    la.cc = p->rcc;
    rnn_loss(la, flat_c, Kc, r->b, p->mbst, p->cfg.clip_eps, p->cfg.ent_coef, p->cfg.vf_coef,
             p->spart_a + size_t(blocks_done) * 6, p->spart_c + size_t(blocks_done) * 6, p->flags + 1, st);
    blocks_done += rnn_loss_blocks(Kc);
    // rnn_seq_backward + the weight gradients, accumulated over the chunks
    float* G = p->grad;
    for (int branch = 0; branch < 2; ++branch) {
      rnn_chunk_backward(p, branch, rows + c0, Mc, G, c0 > 0);
      G += branch == 0 ? r->n_actor : 0;
    }
    after_launch();
  }
  p->rnn_blocks = blocks_done;
}

// clip_global_norm + adam_update for one minibatch (ppo.cpp:605-608).
void minibatch_apply(marl_ppo* p, double lr_u, double* metrics_slot) {
  p->adam_t += 1;
  const float b1 = 0.9f, b2 = 0.999f;  // AdamState defaults (nn.hpp:408-414)
  PpoApplyArgs a{};
  a.params = p->ro->params;
  a.grad = p->grad;
  a.m = p->m;
  a.v = p->v;
  a.P = p->P;
  a.actor_stats = p->spart_a;
  a.critic_stats = p->spart_c;
  a.n_actor_parts = p->hook ? 1 : (p->recurrent ? p->rnn_blocks : p->grid_a);  // folded + all-reduced into row 0
  a.n_critic_parts = p->hook ? 1 : (p->recurrent ? p->rnn_blocks : p->grid_c);
  a.st = p->mbst;
  a.vf_coef = p->cfg.vf_coef;
  a.ent_coef = p->cfg.ent_coef;
  a.max_norm = float(p->cfg.max_grad_norm);
  a.lr = float(lr_u);
  a.beta1 = b1;
  a.beta2 = b2;
  a.eps = 1e-8f;
  a.c1 = 1.0f - std::pow(b1, float(p->adam_t));
  a.c2 = 1.0f - std::pow(b2, float(p->adam_t));
  a.metrics = metrics_slot;
  a.diverged = p->flags;
  ppo_clip_adam(a, p->h->stream);
  after_launch();
}

void ppo_collect_impl(marl_ppo* p) {
  marl_venv* h = p->h;
  int64_t s[3];
  if (marl_venv_episode_stats(h, s, 1) != MARL_OK) raise(MARL_ERR_CUDA, marl_last_error());
  const double half = 0.5 * double(p->cfg.total_timesteps);
  const double n_envs = double(p->cfg.n_envs);
  const bool shaped = p->cfg.shaped_rewards;
  auto shaping_at = [half, n_envs, shaped](int64_t seq) {  // ppo.cpp:572-576
    if (!shaped) return 0.0;
    const double done = double(seq) * n_envs;
    return std::max(0.0, 1.0 - done / std::max(half, 1.0));
  };
  collect_impl(p->ro, p->update * p->cfg.n_rollout_steps, p->cfg.gamma, p->cfg.gae_lambda, shaping_at);
  if (marl_venv_episode_stats(h, s, 1) != MARL_OK) raise(MARL_ERR_CUDA, marl_last_error());
  if (p->hook) {  // episodes finished on every shard
    cuda_check(cudaMemcpy(p->ep_dev, s, sizeof s, cudaMemcpyHostToDevice), "cudaMemcpy");
    allreduce(p, p->ep_dev, 3, MARL_DTYPE_I64);
    cuda_check(cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    cuda_check(cudaMemcpy(s, p->ep_dev, sizeof s, cudaMemcpyDeviceToHost), "cudaMemcpy");
  }
  p->window_episodes = s[0];
  p->window_return = double(s[2]) / 16777216.0;  // stats keep returns in 2^-24 fixed point
  p->collected = true;
}

void ppo_update_impl(marl_ppo* p, double row[12], int* diverged) {
  marl_rollout* r = p->ro;
  cudaStream_t st = p->h->stream;
  const PpoCfg& c = p->cfg;
  const double lr_u = c.anneal_lr ? c.lr * (1.0 - double(p->update) / double(std::max<int64_t>(p->n_updates, 1)))
                                  : c.lr;
  const int n_mb_total = c.update_epochs * c.n_minibatches;
  cuda_check(cudaMemcpyAsync(p->snapshot, r->params, size_t(p->P) * 4, cudaMemcpyDeviceToDevice, st), "cudaMemcpy");
  cuda_check(cudaMemsetAsync(p->flags, 0, 2 * sizeof(int), st), "cudaMemset");
  cuda_check(cudaMemsetAsync(p->metrics, 0, size_t(n_mb_total) * 8 * sizeof(double), st), "cudaMemset");
  int k = 0;
  for (int epoch = 0; epoch < c.update_epochs; ++epoch) {
    uint32_t pk[4];
    put_key(fold_in(key4(p->train_key), uint64_t(p->update) * uint64_t(c.update_epochs) + uint64_t(epoch)), pk);
    KeyWords kw{};
    std::memcpy(kw.w, pk, 16);
    ppo_permutation(kw, p->batch, p->perm, p->perm_scratch, p->perm_scratch_bytes, st);
    after_launch();
    for (int mb = 0; mb < c.n_minibatches; ++mb, ++k) {
      if (p->recurrent)  // whole row sequences (ppo.cpp:594-601)
        minibatch_grad_rnn(p, p->perm + size_t(mb) * size_t(p->per), p->per);
      else
        minibatch_grad(p, p->perm + size_t(mb) * size_t(p->per), p->per, true);
      minibatch_apply(p, lr_u, p->metrics + size_t(k) * 8);
    }
  }
  std::vector<double> m(size_t(n_mb_total) * 8);
  int flags[2];
  cuda_check(cudaMemcpyAsync(m.data(), p->metrics, m.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(flags, p->flags, sizeof flags, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  if (flags[1]) raise(MARL_ERR_CONTRACT, "nn: ppo_row_loss: stored action not legal");
  double sums[7] = {0, 0, 0, 0, 0, 0, 0};
  int n_mb = 0;
  for (int q = 0; q < n_mb_total; ++q) {
    if (m[size_t(q) * 8 + 7] != 1.0) break;  // minibatches after a DivergenceError never ran
    for (int j = 0; j < 7; ++j) sums[j] += m[size_t(q) * 8 + j];
    ++n_mb;
  }
  if (flags[0]) {  // roll back to the last completed update (ppo.cpp:630-634)
    cuda_check(cudaMemcpyAsync(r->params, p->snapshot, size_t(p->P) * 4, cudaMemcpyDeviceToDevice, st), "cudaMemcpy");
  }
  if (r->precision == 1) {
    rollout_pack_bf16(net_of(r), r->images, r->bias, st);
    after_launch();
  }
  const int64_t steps_per_update = int64_t(c.n_envs) * int64_t(c.n_rollout_steps);
  if (p->window_episodes > 0) p->last_mean_return = p->window_return / double(p->window_episodes);
  const double inv = n_mb > 0 ? 1.0 / double(n_mb) : 0.0;
  row[0] = double((p->update + 1) * steps_per_update);
  row[1] = double(p->update);
  row[2] = p->last_mean_return;
  row[3] = double(p->window_episodes);
  for (int j = 0; j < 7; ++j) row[4 + j] = sums[j] * inv;
  row[11] = lr_u;
  *diverged = flags[0];
  p->update += 1;
  p->collected = false;
}

}  // namespace

extern "C" {

int marl_ppo_create(marl_venv* h, const char* ppo_config_json, int centralized, int precision, marl_ppo** out) {
  return guarded([&] {
    if (!h || !out) raise(MARL_ERR_CONTRACT, "marl_ppo_create: NULL argument");
    PpoCfg c = parse_ppo_config(ppo_config_json);
    if (c.recurrent && precision != 0)
      raise(MARL_ERR_SCHEMA, "ppo: recurrent policies run in fp32 (precision 0)");
    if (c.recurrent && h->n != h->gn) raise(MARL_ERR_CONTRACT, "ppo: the recurrent update runs on an unsharded VectorEnv");
    if (int64_t(c.n_envs) != h->gn)
      raise(MARL_ERR_CONTRACT, "ppo: n_envs must equal the VectorEnv's (global) env count");
    set_device(h);
    auto p = std::make_unique<marl_ppo>();
    p->h = h;
    p->cfg = c;
    p->centralized = centralized ? 1 : 0;
    p->precision = precision;
    p->ro = rollout_create_impl(h, c.n_rollout_steps, c.fc_width, c.n_fc_layers, c.activation == "relu", centralized,
                                precision, c.recurrent ? c.hidden_width : 0);
    p->recurrent = c.recurrent;
    marl_rollout* r = p->ro;
    if (r->n_act > kPpoMaxAct) raise(MARL_ERR_SCHEMA, "ppo: more than 64 actions");
    const int64_t steps_per_update = int64_t(c.n_envs) * int64_t(c.n_rollout_steps);
    p->n_updates = c.total_timesteps / steps_per_update;
    p->R_local = r->R;
    p->R_global = r->R_global;
    p->row0 = r->row0;
    p->sharded = r->R != r->R_global;
    p->batch = int64_t(c.n_rollout_steps) * r->R_global;  // the permutation spans the global rollout
    if (c.recurrent) {  // minibatches of whole row sequences (ppo.cpp:548-552, 594-596)
      p->batch = r->R_global;
      if (p->batch % c.n_minibatches != 0)
        raise(MARL_ERR_SCHEMA, "ppo: recurrent minibatches need n_envs*n_agents (" + std::to_string(p->batch) +
                                   ") divisible by n_minibatches (" + std::to_string(c.n_minibatches) + ")");
    } else if (p->batch % c.n_minibatches != 0) {
      raise(MARL_ERR_SCHEMA, "ppo: batch size (" + std::to_string(p->batch) + ") must be divisible by n_minibatches (" +
                                 std::to_string(c.n_minibatches) + ")");
    }
    if (p->batch >= (int64_t(1) << 31)) raise(MARL_ERR_SCHEMA, "ppo: batch (n_rollout_steps * rows) must be < 2^31");
    p->per = p->batch / c.n_minibatches;
    p->Pa = r->n_actor;
    p->Pc = r->n_critic;
    p->P = p->Pa + p->Pc;
    // precision 1: the minibatch step runs on tcgen05 where the shape allows
    // (MARL_PPO_UPDATE_FP32=1 forces the fp32 CUDA-core path)
    p->tc = precision == 1 && !centralized && ppo_tc_supported(r->in_dim, r->critic_in, r->width, r->n_act) &&
            !std::getenv("MARL_PPO_UPDATE_FP32");
    int64_t rnn_K = 0, rnn_Kc = 0;
    if (p->recurrent) {
      // BPTT caches for a chunk of rows: at most a quarter of the free HBM (or MARL_RNN_CACHE_MB)
      rnn_K = int64_t(c.n_rollout_steps) * p->per;
      const size_t per_row = size_t(c.n_rollout_steps) * 4 *
                             (rnn_cache_floats(r->in_dim, r->F, r->H, r->n_act) +
                              rnn_cache_floats(r->critic_in, r->F, r->H, 1));
      size_t free_b = 0, total_b = 0;
      cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      size_t budget = free_b / 4;
      if (const char* mb = std::getenv("MARL_RNN_CACHE_MB")) budget = size_t(std::atoll(mb)) << 20;
      p->rnn_chunk = std::max<int64_t>(1, std::min<int64_t>(p->per, int64_t(budget / per_row)));
      rnn_Kc = int64_t(c.n_rollout_steps) * p->rnn_chunk;
      int64_t nchunks = (p->per + p->rnn_chunk - 1) / p->rnn_chunk;
      p->grid_a = p->grid_c = int(std::min<int64_t>(int64_t(1) << 30, rnn_loss_blocks(rnn_Kc) * nchunks));
    } else if (p->tc) {
      p->grid_a = p->grid_c = ppo_tc_grid(p->per);
    } else {
      p->grid_a = ppo_branch_grid(r->in_dim, r->width, r->n_act, p->per);
      p->grid_c = ppo_branch_grid(r->critic_in, r->width, 1, p->per);
    }
    p->perm_scratch_bytes = ppo_perm_scratch_bytes(p->batch);
    const int nb = ppo_stat_blocks(p->per);
    Arena& ar = p->arena;
    ar.add(&p->m, size_t(p->P));
    ar.add(&p->v, size_t(p->P));
    ar.add(&p->grad, size_t(p->P));
    ar.add(&p->snapshot, size_t(p->P));
    // per-CTA gradient partials of the feed-forward kernels (the recurrent path
    // accumulates straight into the gradient)
    ar.add(&p->gpart_a, p->recurrent ? 1 : size_t(p->grid_a) * size_t(p->Pa));
    ar.add(&p->gpart_c, p->recurrent ? 1 : size_t(p->grid_c) * size_t(p->Pc));
    ar.add(&p->spart_a, size_t(p->grid_a) * 6);
    ar.add(&p->spart_c, size_t(p->grid_c) * 6);
    ar.add(&p->adv_part, size_t(std::max(nb, ppo_stat_blocks(rnn_K))) * 2);
    ar.add(&p->adv_part2, size_t(std::max(nb, ppo_stat_blocks(rnn_K))));
    if (p->recurrent) {
      ar.add(&p->rnn_flat, size_t(rnn_K + rnn_Kc));  // the minibatch's slots, then one chunk's
      const int F = r->F, H = r->H;
      for (int br = 0; br < 2; ++br) {
        RnnCache& cc = br == 0 ? p->rca : p->rcc;
        const int in = br == 0 ? r->in_dim : r->critic_in, out = br == 0 ? r->n_act : 1;
        const size_t K = size_t(rnn_Kc);
        ar.add(&cc.x, K * in);
        ar.add(&cc.y, K * out);
        ar.add(&cc.dy, K * out);
        for (float** q : {&cc.e, &cc.p, &cc.dzp, &cc.dze}) ar.add(q, K * F);
        for (float** q : {&cc.h, &cc.z, &cc.r, &cc.c, &cc.ah, &cc.hn}) ar.add(q, K * H);
        ar.add(&cc.daz, K * 4 * H);  // [K][4H]: daz | dar | dac | dah
      }
      const size_t Mc = size_t(p->rnn_chunk);
      ar.add(&p->rnn_h, Mc * H);
      ar.add(&p->rnn_dh, Mc * H);
      ar.add(&p->rnn_gx, Mc * 3 * H);
      ar.add(&p->rnn_gh, Mc * 3 * H);
      ar.add(&p->rnn_ones, size_t(rnn_Kc));
    }
    ar.add(&p->metrics, size_t(c.update_epochs) * size_t(c.n_minibatches) * 8);
    ar.add(&p->mbst, 1);
    ar.add(&p->perm, size_t(p->batch));
    ar.add(&p->perm_scratch, p->perm_scratch_bytes);
    ar.add(&p->flags, 2);
    ar.add(&p->adv_g, 4);
    ar.add(&p->ep_dev, 3);
    if (p->sharded) {
      p->cmp_scratch_bytes = ppo_compact_scratch_bytes(p->per);
      ar.add(&p->cmp_tmp, size_t(p->per));
      ar.add(&p->cmp_out, size_t(p->per));
      ar.add(&p->cmp_count, 1);
      ar.add(&p->cmp_scratch, p->cmp_scratch_bytes);
    }
    ar.commit();
    if (p->recurrent) {
      std::vector<float> ones(size_t(rnn_Kc), 1.0f);
      cuda_check(cudaMemcpy(p->rnn_ones, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    }
    *out = p.release();
  });
}

// ppo_init_nets(key, spec) (ppo.cpp:109-124) on the host, nn::pack order
// (feed-forward spec; no device needed).
int marl_ppo_init_nets(int in_dim, int critic_in, int n_actions, int fc_width, int n_fc_layers, const uint32_t key[4],
                       float* actor, float* critic) {
  return guarded([&] {
    if (!key || !actor || !critic) raise(MARL_ERR_CONTRACT, "marl_ppo_init_nets: NULL argument");
    if (in_dim < 1 || critic_in < 1 || n_actions < 1 || fc_width < 1 || n_fc_layers < 1)
      raise(MARL_ERR_CONTRACT, "marl_ppo_init_nets: dimensions must be positive");
    const Key k = key4(key);
    host_ff_init(fold_in(k, 1), in_dim, n_fc_layers, fc_width, n_actions, 0.01f, actor);
    host_ff_init(fold_in(k, 2), critic_in, n_fc_layers, fc_width, 1, 1.0f, critic);
  });
}

// train_ppo_impl's setup (ppo.cpp:522-570): nets from fold_in(key, 10), the
// Collector on fold_in(key, 11), the minibatch permutations on fold_in(key, 12).
int marl_ppo_begin(marl_ppo* p, const uint32_t key[4]) {
  return guarded([&] {
    if (!p || !key) raise(MARL_ERR_CONTRACT, "marl_ppo_begin: NULL argument");
    const Key k = key4(key);
    uint32_t k10[4], k11[4];
    put_key(fold_in(k, 10), k10);
    put_key(fold_in(k, 11), k11);
    put_key(fold_in(k, 12), p->train_key);
    std::vector<float> a(size_t(p->Pa)), c(size_t(p->Pc));
    const marl_rollout* r = p->ro;
    if (p->recurrent) {  // ppo_init_nets, recurrent spec (ppo.cpp:112-118)
      host_rnn_init(fold_in(key4(k10), 1), r->in_dim, r->F, r->H, r->n_act, 0.01f, a.data());
      host_rnn_init(fold_in(key4(k10), 2), r->critic_in, r->F, r->H, 1, 1.0f, c.data());
    } else if (marl_ppo_init_nets(r->in_dim, r->critic_in, r->n_act, r->width, p->cfg.n_fc_layers, k10, a.data(),
                                  c.data()) != MARL_OK) {
      raise(MARL_ERR_CONTRACT, marl_last_error());
    }
    if (marl_rollout_set_params(p->ro, a.data(), c.data()) != MARL_OK) raise(MARL_ERR_CUDA, marl_last_error());
    if (marl_rollout_begin(p->ro, k11) != MARL_OK) raise(MARL_ERR_CUDA, marl_last_error());
    set_device(p->h);
    cuda_check(cudaMemset(p->m, 0, size_t(p->P) * 4), "cudaMemset");
    cuda_check(cudaMemset(p->v, 0, size_t(p->P) * 4), "cudaMemset");
    p->update = 0;
    p->adam_t = 0;
    p->last_mean_return = 0.0;
    p->begun = true;
    p->collected = false;
  });
}

int marl_ppo_param_counts(const marl_ppo* p, int32_t* n_actor, int32_t* n_critic) {
  return guarded([&] {
    if (!p || !n_actor || !n_critic) raise(MARL_ERR_CONTRACT, "marl_ppo_param_counts: NULL argument");
    *n_actor = p->Pa;
    *n_critic = p->Pc;
  });
}

// rnn_init-based ppo_init_nets for a recurrent spec (ppo.cpp:112-118), host arrays.
int marl_ppo_init_rnn(int in_dim, int critic_in, int n_actions, int fc_width, int hidden_width, const uint32_t key[4],
                      float* actor, float* critic) {
  return guarded([&] {
    if (!key || !actor || !critic) raise(MARL_ERR_CONTRACT, "marl_ppo_init_rnn: NULL argument");
    const Key k = key4(key);
    host_rnn_init(fold_in(k, 1), in_dim, fc_width, hidden_width, n_actions, 0.01f, actor);
    host_rnn_init(fold_in(k, 2), critic_in, fc_width, hidden_width, 1, 1.0f, critic);
  });
}

int marl_ppo_n_updates(const marl_ppo* p, int64_t* out) {
  return guarded([&] {
    if (!p || !out) raise(MARL_ERR_CONTRACT, "marl_ppo_n_updates: NULL argument");
    *out = p->n_updates;
  });
}

int marl_ppo_set_params(marl_ppo* p, const float* actor, const float* critic) {
  return guarded([&] {
    if (!p) raise(MARL_ERR_CONTRACT, "marl_ppo_set_params: NULL handle");
    if (marl_rollout_set_params(p->ro, actor, critic) != MARL_OK) raise(MARL_ERR_CONTRACT, marl_last_error());
  });
}

int marl_ppo_get_params(marl_ppo* p, float* actor, float* critic) {
  return guarded([&] {
    if (!p || !actor || !critic) raise(MARL_ERR_CONTRACT, "marl_ppo_get_params: NULL argument");
    set_device(p->h);
    cuda_check(cudaStreamSynchronize(p->h->stream), "cudaStreamSynchronize");
    cuda_check(cudaMemcpy(actor, p->ro->params, size_t(p->Pa) * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
    cuda_check(cudaMemcpy(critic, p->ro->params + p->Pa, size_t(p->Pc) * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  });
}

int marl_ppo_rollout(marl_ppo* p, marl_rollout** out) {
  return guarded([&] {
    if (!p || !out) raise(MARL_ERR_CONTRACT, "marl_ppo_rollout: NULL argument");
    *out = p->ro;
  });
}

// Collector::collect for the current update (ppo.cpp:587-588).
int marl_ppo_collect(marl_ppo* p) {
  return guarded([&] {
    if (!p) raise(MARL_ERR_CONTRACT, "marl_ppo_collect: NULL handle");
    if (!p->begun) raise(MARL_ERR_CONTRACT, "ppo: call begin() first");
    ppo_collect_impl(p);
  });
}

// The update epochs over the collected window (ppo.cpp:590-636); row = the
// metrics row {step, update, mean_return, n_episodes, loss, pg_loss, v_loss,
// entropy, approx_kl, clip_frac, grad_norm, lr} (ppo.cpp:524-527, 641-645).
int marl_ppo_update(marl_ppo* p, double row[12], int* diverged) {
  return guarded([&] {
    if (!p || !row || !diverged) raise(MARL_ERR_CONTRACT, "marl_ppo_update: NULL argument");
    if (!p->collected) raise(MARL_ERR_CONTRACT, "ppo: call collect() before update()");
    set_device(p->h);
    ppo_update_impl(p, row, diverged);
  });
}

int marl_ppo_step(marl_ppo* p, double row[12], int* diverged) {
  return guarded([&] {
    if (!p || !row || !diverged) raise(MARL_ERR_CONTRACT, "marl_ppo_step: NULL argument");
    if (!p->begun) raise(MARL_ERR_CONTRACT, "ppo: call begin() first");
    ppo_collect_impl(p);
    ppo_update_impl(p, row, diverged);
  });
}

// One minibatch's flat gradient (actor | critic) and loss statistics
// {loss, pg, v, entropy, kl, clip_frac} without the optimizer step:
// ff_minibatch (ppo.cpp:409-441) over the current buffer.  d_idx: device slots.
int marl_ppo_minibatch_grad(marl_ppo* p, const int32_t* d_idx, int64_t M, float* grad_out, double* stats_out) {
  return guarded([&] {
    if (!p || !d_idx || !grad_out || !stats_out) raise(MARL_ERR_CONTRACT, "marl_ppo_minibatch_grad: NULL argument");
    if (M < 1 || M > p->per) raise(MARL_ERR_CONTRACT, "ppo: minibatch size must be in [1, batch / n_minibatches]");
    set_device(p->h);
    cudaStream_t st = p->h->stream;
    cuda_check(cudaMemsetAsync(p->flags, 0, 2 * sizeof(int), st), "cudaMemset");
    minibatch_grad(p, d_idx, M);
    std::vector<double> sa(size_t(p->grid_a) * 6), sc(size_t(p->grid_c) * 6);
    PpoMbStats ms{};
    int flags[2];
    cuda_check(cudaMemcpyAsync(grad_out, p->grad, size_t(p->P) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(sa.data(), p->spart_a, sa.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(sc.data(), p->spart_c, sc.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(&ms, p->mbst, sizeof ms, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(flags, p->flags, sizeof flags, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    if (flags[1]) raise(MARL_ERR_CONTRACT, "nn: ppo_row_loss: stored action not legal");
    double s[6] = {0, 0, 0, 0, 0, 0}, vt = 0.0;
    for (int c = 0; c < p->grid_a; ++c)
      for (int j = 0; j < 6; ++j) s[j] += sa[size_t(c) * 6 + j];
    for (int c = 0; c < p->grid_c; ++c) vt += sc[size_t(c) * 6 + 1];
    const double tw = ms.total_w;
    if (tw > 0.0) {
      stats_out[0] = double(float((s[0] + p->cfg.vf_coef * vt - p->cfg.ent_coef * s[2]) / tw));
      stats_out[1] = s[0] / tw;
      stats_out[2] = vt / tw;
      stats_out[3] = s[2] / tw;
      stats_out[4] = s[3] / tw;
      stats_out[5] = s[4] / tw;
    } else {
      for (int j = 0; j < 6; ++j) stats_out[j] = 0.0;
    }
  });
}

// Data-parallel update: sum the update's exchanges (advantage sums, gradient,
// loss sums, episode counts) over the ranks with a caller-supplied all-reduce.
int marl_ppo_set_allreduce(marl_ppo* p, marl_allreduce_fn fn, void* ctx) {
  return guarded([&] {
    if (!p) raise(MARL_ERR_CONTRACT, "marl_ppo_set_allreduce: NULL handle");
    p->hook = fn;
    p->hook_ctx = ctx;
  });
}

int marl_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    if (!out) raise(MARL_ERR_CONTRACT, "marl_nccl_unique_id: NULL argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId");
    ncclUniqueId id;
    const ncclResult_t r = nccl().get_unique_id(&id);
    if (r != ncclSuccess) raise(MARL_ERR_CUDA, std::string("ncclGetUniqueId: ") + nccl().error_string(r));
    std::memcpy(out, &id, 128);
  });
}

// The native exchange: an NCCL communicator over `world` ranks (one GPU each)
// whose all-reduces are stream-ordered with the update kernels.
int marl_ppo_set_nccl(marl_ppo* p, const uint8_t id[128], int rank, int world) {
  return guarded([&] {
    if (!p || !id) raise(MARL_ERR_CONTRACT, "marl_ppo_set_nccl: NULL argument");
    if (world < 1 || rank < 0 || rank >= world) raise(MARL_ERR_CONTRACT, "marl_ppo_set_nccl: bad rank / world");
    set_device(p->h);
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = nccl().comm_init_rank(&comm, world, uid, rank);
    if (r != ncclSuccess) raise(MARL_ERR_CUDA, std::string("ncclCommInitRank: ") + nccl().error_string(r));
    if (p->nccl_comm) nccl().comm_destroy(static_cast<ncclComm_t>(p->nccl_comm));
    p->nccl_comm = comm;
    p->hook = nccl_hook;
    p->hook_ctx = comm;
  });
}

int marl_ppo_destroy(marl_ppo* p) {
  return guarded([&] {
    if (!p) return;
    set_device(p->h);
    cudaStreamSynchronize(p->h->stream);
    delete p;
  });
}

// prng::permutation(key, n) (prng.cpp:151-159) into device memory.
int marl_ppo_permutation(const uint32_t key[4], int64_t n, int32_t* d_out, int device) {
  return guarded([&] {
    if (!key || (!d_out && n > 0)) raise(MARL_ERR_CONTRACT, "marl_ppo_permutation: NULL argument");
    if (n < 0) raise(MARL_ERR_CONTRACT, "permutation: n must be >= 0");
    if (n >= (int64_t(1) << 31)) raise(MARL_ERR_CONTRACT, "permutation: n must be < 2^31");
    if (n == 0) return;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    const size_t bytes = ppo_perm_scratch_bytes(n);
    void* scratch = nullptr;
    cuda_check(cudaMalloc(&scratch, bytes), "cudaMalloc");
    KeyWords kw{};
    std::memcpy(kw.w, key, 16);
    ppo_permutation(kw, n, d_out, scratch, bytes, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    cudaFree(scratch);
    cuda_check(e, "permutation");
  });
}

}  // extern "C"
