// SMAX unit combat (reference: proj/core/src/envs/smax.cpp) as one fused
// sm_100a kernel per batch step: random-legal ally actions, the built-in
// heuristic enemy, 8 physics ticks with simultaneous fire and Gauss-Seidel
// separation, win/draw resolution, shaped rewards, infos, auto-reset and the
// observation rows (VectorEnv::step body, vector_env.cpp:95-127).
//
// Exactness: every fp64 op is the reference's, in its order (-fmad=false).
// The reference evaluates ~250 glibc hypot() per 3m step, but almost all are
// only compared against a threshold; those are decided from dx^2+dy^2 outside
// a 2e-12 relative band (dist_le in common.cuh) and by a glibc-exact hypot
// inside it, and the hypot *values* the reference uses (separation pushes,
// nearest-target search) come from the glibc-exact kernel -- so trajectories
// are bit-identical to the reference at a fraction of its fp64 cost.
//
// Layout: one thread owns one env; unit state is [unit][N] structure of
// arrays in HBM; per-unit and per-type-pair constants sit in shared memory
// (uniform-index broadcast reads).  Small fixed rosters (<= 17 units) are
// compile-time specialisations with the whole state in registers; larger or
// overridden rosters use the dynamic-size instantiation.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {
namespace {

constexpr double kDt = 1.0 / 16.0;  // smax.cpp:17
constexpr int kTicks = 8;           // smax.cpp:18
constexpr double kSepTol = 1e-6;    // smax.cpp:19
constexpr int kNorth = 0, kSouth = 1, kEast = 2, kWest = 3, kStop = 4, kAttackBase = 5;
constexpr int kMaxU = kSmaxMaxUnits;

// Per-handle constants, precomputed on the host from SmaxConfig and staged
// into shared memory by every block.
struct Params {
  int na, ne, n, A, controlled, max_steps;
  double map, jitter;
  int8_t type[kMaxU];
  double hmax[kMaxU], dmg[kMaxU], cdmax[kMaxU], spdt[kMaxU], rad[kMaxU], hi[kMaxU];
  Thresh sight[kMaxU];
  Thresh reach[6][6];  // range + radius (shooter type) + radius (target type), smax.cpp:499
  Thresh rsum[6][6];   // fl(ra + rb), smax.cpp:551
  Thresh otol[6][6];   // fl(ra + rb) - 1e-6, the max_overlap tolerance, smax.cpp:565,576
};

template <int NA_, int NE_>
struct Fixed {
  static constexpr int CAP = NA_ + NE_;
  static constexpr int UNROLL = NA_ + NE_;  // fully unrolled: state stays in registers
  __device__ __forceinline__ constexpr int na() const { return NA_; }
  __device__ __forceinline__ constexpr int ne() const { return NE_; }
  __device__ __forceinline__ constexpr int n() const { return NA_ + NE_; }
};
struct Dyn {
  static constexpr int CAP = kMaxU;
  static constexpr int UNROLL = 1;  // runtime-sized loops, state in local memory
  int na_, ne_;
  __device__ __forceinline__ int na() const { return na_; }
  __device__ __forceinline__ int ne() const { return ne_; }
  __device__ __forceinline__ int n() const { return na_ + ne_; }
};

template <class Dm>
struct Units {  // one env's SmaxState (smax.cpp:53-61); winner is -1 between steps
  double x[Dm::CAP], y[Dm::CAP], h[Dm::CAP], cd[Dm::CAP];
  int pa[Dm::CAP];  // prev_action
  int tg[Dm::CAP];  // ai_target
  int sw[Dm::CAP];  // ai_sweep
  int t;
  int winner;
};

__device__ __forceinline__ double dclamp(double v, double lo, double hi) {  // std::clamp
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

template <class Dm>
__device__ __forceinline__ bool in_range(const Params& P, const Units<Dm>& s, int a, int b) {
  const Thresh& r = P.reach[P.type[a]][P.type[b]];  // smax.cpp:497-501
  return dist_le(s.x[a] - s.x[b], s.y[a] - s.y[b], r.r, r.r2lo, r.r2hi);
}

template <class Dm>
__device__ __forceinline__ bool sees(const Params& P, const Units<Dm>& s, int a, int b) {
  const Thresh& r = P.sight[a];  // center_dist(a, b) <= sight(a), smax.cpp:383,613
  return dist_le(s.x[a] - s.x[b], s.y[a] - s.y[b], r.r, r.r2lo, r.r2hi);
}

// separate (smax.cpp:542-567) and max_overlap (smax.cpp:569-580).
template <class Dm>
__device__ __forceinline__ bool overlap_within_tol(const Params& P, const Units<Dm>& s, const Dm& d) {
#pragma unroll(Dm::UNROLL)
  for (int a = 0; a < d.n(); ++a) {
    if (s.h[a] <= 0.0) continue;
#pragma unroll(Dm::UNROLL)
    for (int b = a + 1; b < d.n(); ++b) {
      if (s.h[b] <= 0.0) continue;
      const Thresh& T = P.otol[P.type[a]][P.type[b]];
      double dx = s.x[a] - s.x[b], dy = s.y[a] - s.y[b];
      double d2 = dx * dx + dy * dy;
      if (d2 > T.r2hi) continue;                 // surely sum - d <= tol
      if (d2 < T.r2lo) return false;             // surely sum - d > tol
      double sum = P.rsum[P.type[a]][P.type[b]].r;
      if (!(sum - hypot_glibc(dx, dy) <= kSepTol)) return false;
    }
  }
  return true;
}

template <class Dm>
__device__ __forceinline__ void separate(const Params& P, Units<Dm>& s, const Dm& d, bool to_fixpoint) {
  for (int pass = 0; pass < (to_fixpoint ? 256 : 1); ++pass) {
#pragma unroll(Dm::UNROLL)
    for (int a = 0; a < d.n(); ++a) {
      if (s.h[a] <= 0.0) continue;
#pragma unroll(Dm::UNROLL)
      for (int b = a + 1; b < d.n(); ++b) {
        if (s.h[b] <= 0.0) continue;
        const Thresh& R = P.rsum[P.type[a]][P.type[b]];
        double dx = s.x[b] - s.x[a], dy = s.y[b] - s.y[a];
        double d2 = dx * dx + dy * dy;
        if (d2 > R.r2hi) continue;  // hypot(dx,dy) > ra+rb: overlap <= 0
        double dd = hypot_glibc(dx, dy);
        double overlap = R.r - dd;
        if (overlap <= 0.0) continue;
        double nx = 1.0, ny = 0.0;
        if (dd > 1e-12) {
          nx = dx / dd;
          ny = dy / dd;
        }
        double push = 0.5 * overlap;
        double ra = P.rad[a], rb = P.rad[b];
        s.x[a] = dclamp(s.x[a] - nx * push, ra, P.hi[a]);
        s.y[a] = dclamp(s.y[a] - ny * push, ra, P.hi[a]);
        s.x[b] = dclamp(s.x[b] + nx * push, rb, P.hi[b]);
        s.y[b] = dclamp(s.y[b] + ny * push, rb, P.hi[b]);
      }
    }
    if (!to_fixpoint || overlap_within_tol(P, s, d)) break;
  }
}

// SmaxEnv::reset (smax.cpp:163-193) with fixed-roster cluster spawns
// (spawn_clusters / place_jittered, smax.cpp:448-454,481-492).
template <class Dm>
__device__ __forceinline__ void env_reset(const Params& P, Units<Dm>& s, const Dm& d, const Key& key) {
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    const bool ally = u < d.na();
    const int i = ally ? u : u - d.na();
    double bx = ally ? 0.25 * P.map - 1.5 * (i / 5) : 0.75 * P.map + 1.5 * (i / 5);
    double by = 0.5 * P.map + 1.5 * (i % 5 - 2);
    if (P.jitter > 0.0) {
      bx += uniform_at(fold_in(key, 3000 + 2 * uint64_t(u)), 0, -P.jitter, P.jitter);
      by += uniform_at(fold_in(key, 3001 + 2 * uint64_t(u)), 0, -P.jitter, P.jitter);
    }
    s.x[u] = dclamp(bx, P.rad[u], P.hi[u]);
    s.y[u] = dclamp(by, P.rad[u], P.hi[u]);
    s.h[u] = P.hmax[u];
    s.cd[u] = 0.0;
    s.pa[u] = kStop;
    s.tg[u] = -1;
    s.sw[u] = -1;
  }
  s.t = 0;
  s.winner = -1;
  separate(P, s, d, true);
}

// Legal-action count and the pick-th legal action (smax.cpp:195-211 with
// legal_uniform, vector_env.cpp:21-32).  Legal order: moves 0-3, stop, then
// attacks on living opponents in range.
template <class Dm>
__device__ __forceinline__ int random_legal(const Params& P, const Units<Dm>& s, const Dm& d, int u,
                                            const Key& ek, int j) {
  if (s.h[u] <= 0.0) return kStop;  // only stop is legal: bits % 1 == 0
  const bool ally = u < d.na();
  const int opp0 = ally ? d.na() : 0, opp_n = ally ? d.ne() : d.na();
  uint64_t att = 0;  // bitmask of attackable opponents
  int n_att = 0;
#pragma unroll(Dm::UNROLL)
  for (int k = 0; k < opp_n; ++k) {
    int o = opp0 + k;
    if (s.h[o] > 0.0 && in_range(P, s, u, o)) {
      att |= uint64_t(1) << k;
      ++n_att;
    }
  }
  int pick = int(mod_small(block_at(ek, uint64_t(j)), uint32_t(kAttackBase + n_att)));
  if (pick < kAttackBase) return pick;
  pick -= kAttackBase;
  for (int k = 0; k < 64; ++k) {
    if (att & (uint64_t(1) << k)) {
      if (pick == 0) return kAttackBase + k;
      --pick;
    }
  }
  return kStop;  // unreachable
}

// heuristic_action (smax.cpp:374-419) on the pre-step state.
template <class Dm>
__device__ __forceinline__ int heuristic(const Params& P, const Units<Dm>& s, const Dm& d, int u,
                                         int& target, int& sweep) {
  if (s.h[u] <= 0.0) return kStop;
  const int team = u < d.na() ? 0 : 1;
  const int opp0 = team == 0 ? d.na() : 0, opp_n = team == 0 ? d.ne() : d.na();
  bool keep = false;
  if (target >= 0 && target < opp_n) {
#pragma unroll(Dm::UNROLL)
    for (int k = 0; k < opp_n; ++k)
      if (k == target) keep = s.h[opp0 + k] > 0.0 && sees(P, s, u, opp0 + k);
  }
  if (!keep) {
    target = -1;
#pragma unroll(Dm::UNROLL)
    for (int k = 0; k < opp_n; ++k) {
      if (target >= 0) continue;
      int o = opp0 + k;
      if (s.h[o] > 0.0 && sees(P, s, u, o) && in_range(P, s, u, o)) target = k;
    }
    if (target < 0) {
      double best = 0.0;
#pragma unroll(Dm::UNROLL)
      for (int k = 0; k < opp_n; ++k) {
        int o = opp0 + k;
        if (!(s.h[o] > 0.0 && sees(P, s, u, o))) continue;
        double dd = hypot_glibc(s.x[u] - s.x[o], s.y[u] - s.y[o]);
        if (target < 0 || dd < best) {
          target = k;
          best = dd;
        }
      }
    }
  }
  if (target >= 0) {
    double xo = 0.0, yo = 0.0;
    bool in_reach = false;
#pragma unroll(Dm::UNROLL)
    for (int k = 0; k < opp_n; ++k)
      if (k == target) {
        xo = s.x[opp0 + k];
        yo = s.y[opp0 + k];
        in_reach = in_range(P, s, u, opp0 + k);
      }
    if (in_reach) return kAttackBase + target;
    double dx = xo - s.x[u];
    double dy = yo - s.y[u];
    if (fabs(dx) >= fabs(dy)) return dx > 0 ? kEast : kWest;
    return dy > 0 ? kNorth : kSouth;
  }
  if (sweep < 0) sweep = team == 0 ? kEast : kWest;
  if (s.x[u] <= 1.0) sweep = kEast;
  if (s.x[u] >= P.map - 1.0) sweep = kWest;
  return sweep;
}

// simulate_tick (smax.cpp:503-537).
template <class Dm>
__device__ __forceinline__ void tick(const Params& P, Units<Dm>& s, const Dm& d, const int* act,
                                     bool final_tick) {
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u)
    if (s.h[u] > 0.0) {
      double v = s.cd[u] - kDt;
      s.cd[u] = (0.0 < v) ? v : 0.0;  // std::max(0.0, v)
    }
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    if (s.h[u] <= 0.0 || act[u] > kWest) continue;
    const double dxs = act[u] == kEast ? 1.0 : act[u] == kWest ? -1.0 : 0.0;  // kDirX
    const double dys = act[u] == kNorth ? 1.0 : act[u] == kSouth ? -1.0 : 0.0;  // kDirY
    s.x[u] = dclamp(s.x[u] + P.spdt[u] * dxs, P.rad[u], P.hi[u]);
    s.y[u] = dclamp(s.y[u] + P.spdt[u] * dys, P.rad[u], P.hi[u]);
  }
  // simultaneous fire against the tick-start health snapshot
  double h0[Dm::CAP];
  bool fire[Dm::CAP];
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) h0[u] = s.h[u];
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    fire[u] = false;
    if (h0[u] <= 0.0 || act[u] < kAttackBase) continue;
    const int opp0 = u < d.na() ? d.na() : 0;
    const int o = opp0 + (act[u] - kAttackBase);
    double ho = 0.0;
    bool rng = false;
#pragma unroll(Dm::UNROLL)
    for (int q = 0; q < d.n(); ++q)
      if (q == o) {
        ho = h0[q];
        if (ho > 0.0) rng = in_range(P, s, u, q);
      }
    if (ho <= 0.0 || !rng) continue;
    if (s.cd[u] > 0.0) continue;
    fire[u] = true;
    s.cd[u] = P.cdmax[u];
  }
#pragma unroll(Dm::UNROLL)
  for (int o = 0; o < d.n(); ++o) {
    double damage = 0.0;
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) {
      if (!fire[u]) continue;
      const int opp0 = u < d.na() ? d.na() : 0;
      if (opp0 + (act[u] - kAttackBase) == o) damage += P.dmg[u];
    }
    if (damage > 0.0) {
      double v = h0[o] - damage;
      s.h[o] = (0.0 < v) ? v : 0.0;
    }
  }
  separate(P, s, d, final_tick);
}

template <class Dm>
__device__ __forceinline__ double pool(const Params& P, const Units<Dm>& s, const Dm& d, int team) {
  double total = 0.0;  // smax.cpp:365-372
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    if ((u < d.na()) != (team == 0)) continue;
    total += s.h[u] / P.hmax[u];
    total += s.h[u] > 0.0 ? 1.0 : 0.0;
  }
  return total;
}

// observe (smax.cpp:601-634) for agent `me` into a row of D floats.
template <class Dm>
__device__ __forceinline__ void observe(const Params& P, const Units<Dm>& s, const Dm& d, int me, float* o) {
  const int D = 10 + 17 * (d.n() - 1);
  if (s.h[me] <= 0.0) {
    for (int k = 0; k < D; ++k) o[k] = 0.0f;
    return;
  }
  const double sight = P.sight[me].r;
  int k = 0;
  o[k++] = float(s.h[me] / P.hmax[me]);
  o[k++] = float(s.cd[me] / P.cdmax[me]);
  o[k++] = float(s.x[me] / P.map);
  o[k++] = float(s.y[me] / P.map);
#pragma unroll(Dm::UNROLL)
  for (int q = 0; q < 6; ++q) o[k++] = q == P.type[me] ? 1.0f : 0.0f;
  const bool me_ally = me < d.na();
#pragma unroll(Dm::UNROLL)
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) {
      const bool same = (u < d.na()) == me_ally;
      if (pass == 0 ? (u == me || !same) : same) continue;
      if (!(s.h[u] > 0.0 && sees(P, s, me, u))) {
#pragma unroll(Dm::UNROLL)
        for (int q = 0; q < 17; ++q) o[k + q] = 0.0f;
        k += 17;
        continue;
      }
      o[k++] = 1.0f;
      o[k++] = float((s.x[u] - s.x[me]) / sight);
      o[k++] = float((s.y[u] - s.y[me]) / sight);
      o[k++] = float(s.h[u] / P.hmax[u]);
      o[k++] = float(s.cd[u] / P.cdmax[u]);
#pragma unroll(Dm::UNROLL)
      for (int q = 0; q < 6; ++q) o[k++] = q == P.type[u] ? 1.0f : 0.0f;
      const int bucket = s.pa[u] <= kStop ? s.pa[u] : kStop + 1;  // smax.cpp:589
#pragma unroll(Dm::UNROLL)
      for (int q = 0; q < 6; ++q) o[k++] = q == bucket ? 1.0f : 0.0f;
    }
  }
}

template <class Dm>
__device__ __forceinline__ void load_units(Units<Dm>& s, const SmaxState& st, const Dm& d, int64_t i, int64_t n) {
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    s.x[u] = st.x[u * n + i];
    s.y[u] = st.y[u * n + i];
    s.h[u] = st.health[u * n + i];
    s.cd[u] = st.cooldown[u * n + i];
    uint32_t m = st.mem[u * n + i];
    s.pa[u] = int(m & 0xffu);
    s.tg[u] = int(int8_t((m >> 8) & 0xffu));
    s.sw[u] = int(int8_t((m >> 16) & 0xffu));
  }
  s.t = st.t[i];
  s.winner = -1;
}

template <class Dm>
__device__ __forceinline__ void store_units(const Units<Dm>& s, const SmaxState& st, const Dm& d, int64_t i, int64_t n) {
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    st.x[u * n + i] = s.x[u];
    st.y[u * n + i] = s.y[u];
    st.health[u * n + i] = s.h[u];
    st.cooldown[u * n + i] = s.cd[u];
    st.mem[u * n + i] = uint32_t(s.pa[u] & 0xff) | (uint32_t(uint8_t(int8_t(s.tg[u]))) << 8) |
                        (uint32_t(uint8_t(int8_t(s.sw[u]))) << 16);
  }
  st.t[i] = s.t;
}

// Dynamic shared memory carve-up shared by the reset and step kernels.
struct Smem {
  Params* P;
  float* row;      // [T][D]
  double* rew;     // [T][A]
  double* inf;     // [T][A][3]
  int32_t* act;    // [T][A]
  uint8_t* done;   // [T][A+1]
  uint8_t* fin;    // [T]
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ inline size_t smem_bytes(int T, int D, int A) {
  return align16(sizeof(Params)) + align16(size_t(T) * D * 4) + align16(size_t(T) * A * 8) +
         align16(size_t(T) * A * 24) + align16(size_t(T) * A * 4) + align16(size_t(T) * (A + 1)) +
         align16(size_t(T));
}

__device__ __forceinline__ Smem carve(uint8_t* base, int T, int D, int A) {
  Smem m;
  size_t off = 0;
  m.P = reinterpret_cast<Params*>(base + off);
  off += align16(sizeof(Params));
  m.row = reinterpret_cast<float*>(base + off);
  off += align16(size_t(T) * D * 4);
  m.rew = reinterpret_cast<double*>(base + off);
  off += align16(size_t(T) * A * 8);
  m.inf = reinterpret_cast<double*>(base + off);
  off += align16(size_t(T) * A * 24);
  m.act = reinterpret_cast<int32_t*>(base + off);
  off += align16(size_t(T) * A * 4);
  m.done = base + off;
  off += align16(size_t(T) * (A + 1));
  m.fin = base + off;
  return m;
}

__device__ __forceinline__ void stage_params(Params* dst, const Params* src) {
  const int words = int(sizeof(Params) / 4);
  const int* s = reinterpret_cast<const int*>(src);
  int* d = reinterpret_cast<int*>(dst);
  for (int q = threadIdx.x; q < words; q += blockDim.x) d[q] = __ldg(s + q);
  __syncthreads();
}

// Copy agent a's rows of this block's envs from the staging tile to global
// obs rows ([N][A][D] layout: rows of one agent are D floats at stride A*D).
__device__ __forceinline__ void store_agent_rows(float* gobs, const float* tile, int nvalid, int D,
                                                 int A, int a, const uint8_t* mask) {
  for (int idx = threadIdx.x; idx < nvalid * D; idx += blockDim.x) {
    int e = idx / D, k = idx - e * D;
    if (mask && !mask[e]) continue;
    __stcs(gobs + (size_t(e) * A + a) * D + k, tile[idx]);
  }
}

template <class Dm>
struct DimsOf;
template <int NA_, int NE_>
struct DimsOf<Fixed<NA_, NE_>> {
  __device__ static Fixed<NA_, NE_> make(const Params&) { return {}; }
};
template <>
struct DimsOf<Dyn> {
  __device__ static Dyn make(const Params& P) { return Dyn{P.na, P.ne}; }
};

template <class Dm>
__global__ void smax_reset_kernel(const Params* __restrict__ gP, SmaxState st, LaunchCommon lc, Key key,
                                  Key carry_parent) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int T = blockDim.x;
  Smem m = carve(smem, T, 1, 1);  // params only; rows are staged below
  stage_params(m.P, gP);
  const Params& P = *m.P;
  const Dm d = DimsOf<Dm>::make(P);
  const int A = P.A, D = 10 + 17 * (P.n - 1);
  float* tile = reinterpret_cast<float*>(smem + align16(sizeof(Params)));
  const int64_t i0 = int64_t(blockIdx.x) * T, i = i0 + threadIdx.x;
  const int nvalid = int(min64(T, lc.n - i0));
  Units<Dm> s;
  if (i < lc.n) {
    const uint64_t g = uint64_t(lc.offset + i);
    env_reset(P, s, d, split_child(key, g));
    Key c = split_child(carry_parent, g);
    lc.carry.keys[i] = make_uint4(c.k0, c.k1, c.c0, c.c1);
    lc.carry.ep_return[i] = 0.0;
    lc.carry.ep_length[i] = 0;
    store_units(s, st, d, i, lc.n);
  }
  for (int a = 0; a < A; ++a) {
    if (i < lc.n) observe(P, s, d, a, tile + threadIdx.x * D);
    __syncthreads();
    store_agent_rows(lc.v.obs + i0 * A * D, tile, nvalid, D, A, a, nullptr);
    __syncthreads();
  }
}

template <class Dm, bool RANDOM>
__global__ void smax_step_kernel(const Params* __restrict__ gP, SmaxState st, LaunchCommon lc, Key step_key) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (*(volatile int*)lc.err) return;  // a pending contract error freezes the batch
  const int T = blockDim.x;
  // A and D are only known after the params are staged; carve with the
  // host-side maxima passed through gridDim.y-free args below.
  const Params* Pg = gP;
  const int A = Pg->A, n_units = Pg->n, D = 10 + 17 * (n_units - 1);
  Smem m = carve(smem, T, D, A);
  stage_params(m.P, gP);
  const Params& P = *m.P;
  const Dm d = DimsOf<Dm>::make(P);
  const int tid = threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * T, i = i0 + tid;
  const int nvalid = int(min64(T, lc.n - i0));
  const bool live = i < lc.n;

  Units<Dm> s;
  Key carry{0, 0, 0, 0};
  double ep_ret = 0.0;
  int ep_len = 0;
  bool done = false;
  if (live) {
    uint4 kw = lc.carry.keys[i];
    carry = Key{kw.x, kw.y, kw.z, kw.w};
    ep_ret = lc.carry.ep_return[i];
    ep_len = lc.carry.ep_length[i];
    load_units(s, st, d, i, lc.n);

    // ---- actions: agents (allies, plus enemies when controlled), then the
    // built-in controller on the pre-step state (smax.cpp:225-240)
    int act[Dm::CAP];
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) act[u] = kStop;
    if (RANDOM) {
      Key ek = split_child(step_key, uint64_t(lc.offset + i));  // vector_env.cpp:171
#pragma unroll(Dm::UNROLL)
      for (int u = 0; u < (Dm::UNROLL > 1 ? Dm::CAP : A); ++u) {
        if (u >= A) continue;
        act[u] = random_legal(P, s, d, u, ek, u);
        m.act[tid * A + u] = act[u];
      }
    } else {
#pragma unroll(Dm::UNROLL)
      for (int u = 0; u < (Dm::UNROLL > 1 ? Dm::CAP : A); ++u)
        if (u < A) act[u] = lc.v.actions[i * A + u];
    }
    int new_tg[Dm::CAP], new_sw[Dm::CAP];
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) {
      new_tg[u] = s.tg[u];
      new_sw[u] = s.sw[u];
    }
    if (!P.controlled) {
#pragma unroll(Dm::UNROLL)
      for (int u = 0; u < d.n(); ++u) {
        if (u < d.na()) continue;
        int tg = s.tg[u], sw = s.sw[u];
        act[u] = heuristic(P, s, d, u, tg, sw);
        new_tg[u] = tg;
        new_sw[u] = sw;
      }
    }
    const double pool_prev0 = pool(P, s, d, 0), pool_prev1 = pool(P, s, d, 1);
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) {
      s.tg[u] = new_tg[u];
      s.sw[u] = new_sw[u];
    }

    // ---- physics (smax.cpp:242-254)
    for (int k = 0; k < kTicks; ++k) tick(P, s, d, act, k == kTicks - 1);
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) s.pa[u] = act[u];
    s.t += 1;
    int ally_alive = 0, enemy_alive = 0;
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < d.n(); ++u) {
      if (s.h[u] > 0.0) {
        if (u < d.na()) ++ally_alive;
        else ++enemy_alive;
      }
    }
    if (ally_alive == 0 && enemy_alive == 0) s.winner = 2;
    else if (enemy_alive == 0) s.winner = 0;
    else if (ally_alive == 0) s.winner = 1;
    else if (s.t >= P.max_steps) s.winner = 2;
    done = s.winner != -1;

    // ---- reward_map (smax.cpp:352-363), infos and dones (smax.cpp:256-268)
    double ally_r = 0.5 * (pool_prev1 - pool(P, s, d, 1)) / (2.0 * d.ne());
    double enemy_r = 0.5 * (pool_prev0 - pool(P, s, d, 0)) / (2.0 * d.na());
    if (s.winner == 0) ally_r += 0.5;
    if (s.winner == 1) enemy_r += 0.5;
    double sum = 0.0;
    for (int a = 0; a < A; ++a) {
      const int team = a < d.na() ? 0 : 1;
      const double r = team == 0 ? ally_r : enemy_r;
      m.rew[tid * A + a] = r;
      sum += r;
      double alive = 0.0;
#pragma unroll(Dm::UNROLL)
      for (int u = 0; u < (Dm::UNROLL > 1 ? Dm::CAP : A); ++u)
        if (u == a) alive = s.h[u] > 0.0 ? 1.0 : 0.0;
      m.inf[(tid * A + a) * 3 + 0] = alive;
      m.inf[(tid * A + a) * 3 + 1] = s.winner == team ? 1.0 : 0.0;
      m.inf[(tid * A + a) * 3 + 2] = s.winner == 2 ? 1.0 : 0.0;
      m.done[tid * (A + 1) + a] = done;
    }
    m.done[tid * (A + 1) + A] = done;
    ep_ret = ep_ret + sum / double(A);  // vector_env.cpp:14-18,99
    ep_len = ep_len + 1;
    lc.v.finished[i] = done;
    lc.v.final_returns[i] = done ? ep_ret : 0.0;
    lc.v.final_lengths[i] = done ? ep_len : 0;
  }
  m.fin[tid] = done;
  stats_add(lc.stats, done, ep_len, ep_ret);

  // ---- terminal observations -> final_obs, then auto-reset (vector_env.cpp:107-119)
  if (__syncthreads_or(done)) {
    for (int a = 0; a < A; ++a) {
      if (done) observe(P, s, d, a, m.row + tid * D);
      __syncthreads();
      store_agent_rows(lc.v.final_obs + i0 * A * D, m.row, nvalid, D, A, a, m.fin);
      __syncthreads();
    }
    if (done) {
      env_reset(P, s, d, split_child(carry, 1));
      ep_ret = 0.0;
      ep_len = 0;
    }
  }
  if (live) {
    Key nk = split_child(carry, 2);  // vector_env.cpp:126
    lc.carry.keys[i] = make_uint4(nk.k0, nk.k1, nk.c0, nk.c1);
    lc.carry.ep_return[i] = ep_ret;
    lc.carry.ep_length[i] = ep_len;
    store_units(s, st, d, i, lc.n);
  }
  for (int a = 0; a < A; ++a) {
    if (live) observe(P, s, d, a, m.row + tid * D);
    __syncthreads();
    store_agent_rows(lc.v.obs + i0 * A * D, m.row, nvalid, D, A, a, nullptr);
    __syncthreads();
  }
  block_store(lc.v.rewards + i0 * A, m.rew, size_t(nvalid) * A * sizeof(double));
  block_store(lc.v.infos + i0 * A * 3, m.inf, size_t(nvalid) * A * 3 * sizeof(double));
  block_store(lc.v.dones + i0 * (A + 1), m.done, size_t(nvalid) * (A + 1));
  if (RANDOM) block_store(lc.v.actions + i0 * A, m.act, size_t(nvalid) * A * sizeof(int32_t));
}

template <class Dm>
__global__ void smax_legal_kernel(const Params* __restrict__ gP, SmaxState st, int64_t n, int n_act,
                                  uint8_t* out) {
  __shared__ Params sP;
  stage_params(&sP, gP);
  const Dm d = DimsOf<Dm>::make(sP);
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Units<Dm> s;
  load_units(s, st, d, i, n);
  for (int a = 0; a < sP.A; ++a) {  // smax.cpp:195-211
    uint8_t* row = out + (size_t(i) * sP.A + a) * n_act;
    for (int q = 0; q < n_act; ++q) row[q] = 0;
    row[kStop] = 1;
    double ha = 0.0;
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < (Dm::UNROLL > 1 ? Dm::CAP : sP.A); ++u)
      if (u == a) ha = s.h[u];
    if (ha <= 0.0) continue;
    for (int q = 0; q < kStop; ++q) row[q] = 1;
    const int opp0 = a < d.na() ? d.na() : 0, opp_n = a < d.na() ? d.ne() : d.na();
#pragma unroll(Dm::UNROLL)
    for (int u = 0; u < (Dm::UNROLL > 1 ? Dm::CAP : sP.A); ++u) {
      if (u != a) continue;
#pragma unroll(Dm::UNROLL)
      for (int k = 0; k < (Dm::UNROLL > 1 ? Dm::CAP : opp_n); ++k)
        if (k < opp_n && s.h[opp0 + k] > 0.0 && in_range(sP, s, u, opp0 + k)) row[kAttackBase + k] = 1;
    }
  }
}

template <class Dm>
__global__ void smax_hash_kernel(const Params* __restrict__ gP, SmaxState st, int64_t n, uint64_t* out) {
  __shared__ Params sP;
  stage_params(&sP, gP);
  const Dm d = DimsOf<Dm>::make(sP);
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Units<Dm> s;
  load_units(s, st, d, i, n);
  uint64_t h = 1469598103934665603ull;  // smax.cpp:312-337
  auto mix = [&h](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
#pragma unroll(Dm::UNROLL)
  for (int u = 0; u < d.n(); ++u) {
    mix(__double_as_longlong(s.x[u]));
    mix(__double_as_longlong(s.y[u]));
    mix(__double_as_longlong(s.h[u]));
    mix(__double_as_longlong(s.cd[u]));
    mix(uint64_t(uint8_t(sP.type[u])));
    mix(uint64_t(uint16_t(int16_t(s.pa[u]))));
    mix(uint64_t(uint16_t(int16_t(s.tg[u]))));
    mix(uint64_t(uint8_t(int8_t(s.sw[u]))));
  }
  mix(uint64_t(s.t));
  mix(uint64_t(uint8_t(int8_t(-1))));
  out[i] = h;
}

// ------------------------------------------------------------------ host
Key to_key(KeyWords k) { return Key{k.w[0], k.w[1], k.w[2], k.w[3]}; }

Params make_params(const SmaxConfig& c) {
  Params P{};
  P.na = c.na;
  P.ne = c.ne;
  P.n = c.na + c.ne;
  P.A = c.na + (c.enemy_controlled ? c.ne : 0);
  P.controlled = c.enemy_controlled;
  P.max_steps = c.max_steps;
  P.map = c.map;
  P.jitter = c.jitter;
  for (int u = 0; u < P.n; ++u) {
    const double* st = c.stats[c.type[u]];
    P.type[u] = c.type[u];
    P.hmax[u] = st[0];
    P.dmg[u] = st[1];
    P.cdmax[u] = st[2];
    P.spdt[u] = st[3] * kDt;  // st.speed * kDt, smax.cpp:514
    P.rad[u] = st[6];
    P.hi[u] = c.map - st[6];  // map_ - radius, smax.cpp:515
    P.sight[u] = make_thresh(st[4]);
  }
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      P.reach[a][b] = make_thresh(c.stats[a][5] + c.stats[a][6] + c.stats[b][6]);
      double sum = c.stats[a][6] + c.stats[b][6];
      P.rsum[a][b] = make_thresh(sum);
      P.rsum[a][b].r = sum;
      P.otol[a][b] = make_thresh(sum - kSepTol);
    }
  return P;
}

struct Launch {
  int threads;
  size_t smem;
};

// Which compile-time roster a config maps to (0 = dynamic).
int roster_id(const SmaxConfig& c) {
  if (c.na == 3 && c.ne == 3) return 1;
  if (c.na == 5 && c.ne == 5) return 2;
  if (c.na == 5 && c.ne == 6) return 3;
  if (c.na == 3 && c.ne == 5) return 4;
  if (c.na == 8 && c.ne == 8) return 5;
  if (c.na == 8 && c.ne == 9) return 6;
  if (c.na == 6 && c.ne == 8) return 7;
  return 0;
}

Launch pick_launch(const SmaxConfig& c, bool fixed) {
  const int n = c.na + c.ne, A = c.na + (c.enemy_controlled ? c.ne : 0);
  const int D = 10 + 17 * (n - 1);
  int T = fixed ? 128 : 64;
  while (T > 32 && smem_bytes(T, D, A) > 200 * 1024) T /= 2;
  return Launch{T, smem_bytes(T, D, A)};
}

}  // namespace

void smax_prepare(SmaxConfig& c) {
  Params P = make_params(c);
  Params* d = nullptr;
  cudaMalloc(&d, sizeof(Params));
  cudaMemcpy(d, &P, sizeof P, cudaMemcpyHostToDevice);
  c.dev_params = d;
}

void smax_release(SmaxConfig& c) {
  if (c.dev_params) cudaFree(c.dev_params);
  c.dev_params = nullptr;
}

static const Params* device_params(const SmaxConfig& c, cudaStream_t) {
  return static_cast<const Params*>(c.dev_params);
}

template <class Dm>
static void launch_reset_t(const SmaxConfig& c, const Params* dP, const SmaxState& s, const LaunchCommon& lc,
                           Key k, Key cp, bool fixed) {
  Launch L = pick_launch(c, fixed);
  auto fn = smax_reset_kernel<Dm>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.smem));
  unsigned g = unsigned((lc.n + L.threads - 1) / L.threads);
  fn<<<g, L.threads, L.smem, lc.stream>>>(dP, s, lc, k, cp);
}

template <class Dm>
static void launch_step_t(const SmaxConfig& c, const Params* dP, const SmaxState& s, const LaunchCommon& lc,
                          bool random, Key k, bool fixed) {
  Launch L = pick_launch(c, fixed);
  auto fn = random ? smax_step_kernel<Dm, true> : smax_step_kernel<Dm, false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.smem));
  unsigned g = unsigned((lc.n + L.threads - 1) / L.threads);
  fn<<<g, L.threads, L.smem, lc.stream>>>(dP, s, lc, k);
}

#define MARL_SMAX_DISPATCH(FN, ...)                                          \
  switch (roster_id(c)) {                                                    \
    case 1: FN<Fixed<3, 3>>(__VA_ARGS__, true); break;                       \
    case 2: FN<Fixed<5, 5>>(__VA_ARGS__, true); break;                       \
    default: FN<Dyn>(__VA_ARGS__, false); break;                             \
  }

void smax_launch_reset(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, KeyWords key,
                       KeyWords carry_parent) {
  const Params* dP = device_params(c, lc.stream);
  Key k = to_key(key), cp = to_key(carry_parent);
  MARL_SMAX_DISPATCH(launch_reset_t, c, dP, s, lc, k, cp)
  ++g_launches;
}

void smax_launch_step(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, bool random,
                      KeyWords step_key) {
  const Params* dP = device_params(c, lc.stream);
  Key k = to_key(step_key);
  MARL_SMAX_DISPATCH(launch_step_t, c, dP, s, lc, random, k)
  ++g_launches;
}

template <class Dm>
static void launch_legal_t(const Params* dP, const SmaxState& s, int64_t n, int n_act, uint8_t* out,
                           cudaStream_t st, bool) {
  smax_legal_kernel<Dm><<<unsigned((n + 63) / 64), 64, 0, st>>>(dP, s, n, n_act, out);
}
template <class Dm>
static void launch_hash_t(const Params* dP, const SmaxState& s, int64_t n, uint64_t* out, cudaStream_t st,
                          bool) {
  smax_hash_kernel<Dm><<<unsigned((n + 63) / 64), 64, 0, st>>>(dP, s, n, out);
}

void smax_launch_legal(const SmaxConfig& c, const SmaxState& s, int64_t n, int n_act, uint8_t* out,
                       cudaStream_t st) {
  const Params* dP = device_params(c, st);
  MARL_SMAX_DISPATCH(launch_legal_t, dP, s, n, n_act, out, st)
  ++g_launches;
}

void smax_launch_hash(const SmaxConfig& c, const SmaxState& s, int64_t n, uint64_t* out, cudaStream_t st) {
  const Params* dP = device_params(c, st);
  MARL_SMAX_DISPATCH(launch_hash_t, dP, s, n, out, st)
  ++g_launches;
}

}  // namespace marl_b200
