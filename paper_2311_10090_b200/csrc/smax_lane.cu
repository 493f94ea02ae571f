// SMAX step with ONE THREAD PER ENV for small rosters (3m, 2s3z, 5m_vs_6m,
// smacv2_5_units): the whole VectorEnv::step body around SmaxEnv::step
// (vector_env.cpp:95-127, smax.cpp:218-270) runs in one thread, a warp owns 32
// consecutive envs and all 32 lanes run the same instruction stream (no
// per-unit lane roles, no group barriers).
//
// Two homes for an env's units, chosen for the instruction cache as much as
// for the data path:
// * the eight physics ticks (smax.cpp:503-537, the only code that runs many
//   times per step) keep x, y, health and cooldown in REGISTERS -- every
//   per-unit loop is unrolled over the compile-time roster, the one dynamic
//   index (an attack target) is a select chain, and the reference's
//   sequential Gauss-Seidel separation (smax.cpp:542-567) sits behind a
//   branch-free all-pairs pre-check that proves the common "nothing
//   overlaps" case;
// * everything that runs once per step -- enemy heuristic and random-legal
//   actions, pools, observation rows, auto-reset, the separation passes
//   themselves, state write-back -- is loop code over a per-lane SLICE of
//   shared memory (field f of unit u at [f][u][lane], conflict-free), so the
//   kernel's once-per-step code stays a few KB instead of an unrolled
//   straight line that no warp could keep in the instruction cache.
//
// Observation rows (smax.cpp:601-634) are the bulk of the bytes: per agent
// the lanes build their env's row in a warp tile (odd row stride: conflict
// free), then the warp stores the rows with coalesced 128-byte streaming
// stores.  Resets spread their spawn-jitter Threefry draws over all 32 lanes.
//
// Exactness: the same fp64 sequence as the reference (-fmad=false) and as the
// lane-group kernel in smax.cu, which this kernel equals bit for bit
// (tests/test_smax_lane.py; both are parity-tested against the oracle).
#include <cuda_runtime.h>

#include <cstdlib>

#include "smax_params.cuh"

namespace marl_b200 {
namespace {
using namespace smax;

#ifndef MARL_LANE_LT
#define MARL_LANE_LT 32  // one warp per block: 2048 blocks over 148 SMs balance to within 1 % (128: 13 %)
#endif
constexpr int kLT = MARL_LANE_LT;  // threads (= envs) per block
constexpr int kLW = kLT / 32;

constexpr int a16i(int b) { return (b + 15) & ~15; }
constexpr int imax(int a, int b) { return a > b ? a : b; }

template <int NA_, int NE_, int HT_, bool CTRL_>
struct Roster {
  static constexpr int NA = NA_, NE = NE_, N = NA_ + NE_, HT = HT_;
  static constexpr int A = CTRL_ ? N : NA;      // agents: allies, plus enemies when enemy_controlled
  static constexpr int D = 10 + 17 * (N - 1);  // obs_size, smax.cpp:161
  // Observation emission: the warp's envs are taken CE at a time; the CE
  // envs' rows are one contiguous, 16-byte aligned run of the [N][A][D]
  // output.  Each row is cut into column PARTS of whole unit slots (part 0 =
  // own features + slots [0, K0), part p >= 1 = slots [K0 + (p-1) K, ...)),
  // and every lane builds one (env, agent, part) item of the run in the tile.
  static constexpr int K0 = 2, K = 3;
  static constexpr int NP = N - 1 > K0 ? 1 + (N - 1 - K0 + K - 1) / K : 1;
  static constexpr int ce() {
    int c = 1;
    while (c < 32 && c * A * NP < 20) c *= 2;
    return c;
  }
  static constexpr int CE = ce();
  static constexpr bool kVec = (CE * A * D) % 4 == 0;  // the chunk is whole 16-byte vectors
  static constexpr int kMinBlocks = N <= 6 ? 4 : 3;     // registers: the tick state is 4N doubles
  static constexpr int kItems = CE * A * NP;
  static constexpr int kSliceBytes = 4 * N * 32 * 8 + 4 * N * 32;  // x y h cd (f64) + pa ty tg sw (i8)
  // the tile doubles as the reset scratch: [32] keys + [32][2N] draws
  static constexpr int kTileBytes = a16i(imax(CE * A * D * 4, 32 * 16 + 32 * 2 * N * 8));
  static constexpr int kWarpBytes = kTileBytes + kSliceBytes;
  static_assert(32 % CE == 0, "chunks tile the warp");
};

// One env's units in registers, for the ticks.
template <class R>
struct Units {
  double x[R::N], y[R::N], h[R::N], cd[R::N];
  int act[R::N], ty[R::N];
  __device__ __forceinline__ int T(int u) const { return R::HT >= 0 ? R::HT : ty[u]; }
};

// This lane's slice: field f of unit u at d[(f * N + u) * 32] / b[(f * N + u) * 32].
template <class R>
struct Slice {
  double* d;
  int8_t* b;
  __device__ __forceinline__ double& X(int u) const { return d[(0 * R::N + u) * 32]; }
  __device__ __forceinline__ double& Y(int u) const { return d[(1 * R::N + u) * 32]; }
  __device__ __forceinline__ double& H(int u) const { return d[(2 * R::N + u) * 32]; }
  __device__ __forceinline__ double& CD(int u) const { return d[(3 * R::N + u) * 32]; }
  __device__ __forceinline__ int8_t& PA(int u) const { return b[(0 * R::N + u) * 32]; }  // action / prev_action
  __device__ __forceinline__ int8_t& TY(int u) const { return b[(1 * R::N + u) * 32]; }
  __device__ __forceinline__ int8_t& TG(int u) const { return b[(2 * R::N + u) * 32]; }  // ai_target
  __device__ __forceinline__ int8_t& SW(int u) const { return b[(3 * R::N + u) * 32]; }  // ai_sweep
  __device__ __forceinline__ int T(int u) const { return R::HT >= 0 ? R::HT : int(TY(u)); }
};

template <int N>
__device__ __forceinline__ double pick(const double (&v)[N], int lo, int n, int idx) {
  // v[lo + idx] for a runtime idx in [0, n): a select chain over the range
  double r = v[lo];
#pragma unroll
  for (int q = 1; q < n; ++q)
    if (idx == q) r = v[lo + q];
  return r;
}
template <int N>
__device__ __forceinline__ int pick(const int (&v)[N], int lo, int n, int idx) {
  int r = v[lo];
#pragma unroll
  for (int q = 1; q < n; ++q)
    if (idx == q) r = v[lo + q];
  return r;
}

__device__ __forceinline__ bool dist_le_t(const Thresh& t, double dx, double dy) {
  return dist_le(dx, dy, t.r, t.r2lo, t.r2hi);
}

// center_dist(a, b) <= reach(a -> b), smax.cpp:497-501 / <= sight(a), smax.cpp:383,613
template <class R>
__device__ __forceinline__ bool in_range(const Params& P, const Slice<R>& S, int a, int b) {
  return dist_le_t(P.ps[S.T(a)][S.T(b)].reach, S.X(a) - S.X(b), S.Y(a) - S.Y(b));
}
template <class R>
__device__ __forceinline__ bool sees(const Params& P, const Slice<R>& S, int a, int b) {
  return dist_le_t(P.ts[S.T(a)].sight, S.X(a) - S.X(b), S.Y(a) - S.Y(b));
}

// ---------------------------------------------------------------- separation
// Which living pairs may overlap?  Bit p (pairs in the reference's row-major
// order) is set when d^2 is within the pair's upper band; conservative and
// branch-free.  Zero proves a pass of separate() is a no-op.
template <class R>
__device__ __forceinline__ uint64_t candidates(const Params& P, const Units<R>& e) {
  uint64_t c = 0;
  const double r2 = R::HT >= 0 ? P.ps[R::HT][R::HT].rsum.r2hi : P.sep_r2hi;
  int p = 0;
#pragma unroll
  for (int a = 0; a < R::N - 1; ++a)
#pragma unroll
    for (int b = a + 1; b < R::N; ++b, ++p) {
      const double dx = e.x[b] - e.x[a], dy = e.y[b] - e.y[a];
      if ((e.h[a] > 0.0) & (e.h[b] > 0.0) & (dx * dx + dy * dy <= r2)) c |= uint64_t(1) << p;
    }
  return c;
}

// separate(s, to_fixpoint) (smax.cpp:542-567) on the slice, out of line: runs
// only when two living units may touch.
// `cand` (from candidates()) limits the first pass to the pairs that may
// overlap at its start plus, as it goes, the later pairs of every unit the
// pass pushes: any other pair is farther apart than its radius sum, so the
// reference would skip it too.  Later fixpoint passes test every pair.
// Pair p = (a, b > a) in the reference's row-major order starts row a at
// a (2N - a - 1) / 2.
template <int N>
__device__ __forceinline__ int row_start(int a) {
  return a * (2 * N - a - 1) / 2;
}
template <int N>
__device__ __forceinline__ uint64_t row_mask(int a) {
  return ((uint64_t(1) << (N - 1 - a)) - 1) << row_start<N>(a);
}

template <class R>
__device__ __forceinline__ void separate_slice(const Params& P, Slice<R> S, bool fixpoint, uint64_t cand) {
  constexpr int N = R::N, NPAIRS = N * (N - 1) / 2;
  constexpr uint64_t kAll = NPAIRS == 64 ? ~uint64_t(0) : (uint64_t(1) << NPAIRS) - 1;
  cand &= kAll;
#pragma unroll 1
  for (int pass = 0; pass < (fixpoint ? 256 : 1); ++pass) {
    // one Gauss-Seidel pass in the reference's pair order (smax.cpp:544-565)
    uint64_t todo = cand;
    int a = 0, rs = 0, re = N - 1;  // pairs of row a are [rs, re); p only grows
#pragma unroll 1
    while (todo) {
      const int p = __ffsll((long long)todo) - 1;
      todo &= todo - 1;
      while (p >= re) {
        ++a;
        rs = re;
        re += N - 1 - a;
      }
      const int b = a + 1 + (p - rs);
      if (!(S.H(a) > 0.0) || !(S.H(b) > 0.0)) continue;
      const Thresh& Rs = P.ps[S.T(a)][S.T(b)].rsum;
      const double dx = S.X(b) - S.X(a), dy = S.Y(b) - S.Y(a);
      if (dx * dx + dy * dy > Rs.r2hi) continue;  // hypot(dx, dy) > ra + rb: overlap <= 0
      const double d = hypot_glibc(dx, dy);
      const double overlap = Rs.r - d;
      if (overlap <= 0.0) continue;
      double nx = 1.0, ny = 0.0;  // coincident centres get a fixed nudge axis
      if (d > 1e-12) {
        nx = dx / d;
        ny = dy / d;
      }
      const double push = 0.5 * overlap;
      const TypeStat& A_ = P.ts[S.T(a)];
      const TypeStat& B_ = P.ts[S.T(b)];
      S.X(a) = dclamp(S.X(a) - nx * push, A_.rad, A_.hi);
      S.Y(a) = dclamp(S.Y(a) - ny * push, A_.rad, A_.hi);
      S.X(b) = dclamp(S.X(b) + nx * push, B_.rad, B_.hi);
      S.Y(b) = dclamp(S.Y(b) + ny * push, B_.rad, B_.hi);
      // a and b moved: every later pair with either of them must be tested
      uint64_t later = row_mask<N>(a) | row_mask<N>(b);
#pragma unroll 1
      for (int x = a + 1; x < b; ++x) later |= uint64_t(1) << (row_start<N>(x) + b - x - 1);
      todo |= later & ~((uint64_t(2) << p) - 1);
    }
    if (!fixpoint) return;
    cand = kAll;
    // max_overlap(s) <= kSeparationTol (smax.cpp:569-580), exact
    bool bad = false;
#pragma unroll 1
    for (int a = 0; a < N - 1 && !bad; ++a) {
      if (!(S.H(a) > 0.0)) continue;
#pragma unroll 1
      for (int b = a + 1; b < N; ++b) {
        if (!(S.H(b) > 0.0)) continue;
        const PairStat& Q = P.ps[S.T(a)][S.T(b)];
        const double dx = S.X(a) - S.X(b), dy = S.Y(a) - S.Y(b);
        const double d2 = dx * dx + dy * dy;
        if (d2 > Q.otol.r2hi) continue;  // surely sum - d <= tol
        if (d2 < Q.otol.r2lo || !(Q.rsum.r - hypot_glibc(dx, dy) <= kSepTol)) {
          bad = true;
          break;
        }
      }
    }
    if (!bad) return;
  }
}

// The tick's separate(): the pre-check on registers, the passes on the slice.
template <class R>
__device__ __forceinline__ void separate(const Params& P, Units<R>& e, bool fixpoint, const Slice<R>& S) {
  const uint64_t cand = candidates(P, e);
  if (!cand) return;  // no pass can push anything (and max_overlap <= 0)
#pragma unroll
  for (int u = 0; u < R::N; ++u) {
    S.X(u) = e.x[u];
    S.Y(u) = e.y[u];
    S.H(u) = e.h[u];
  }
  separate_slice<R>(P, S, fixpoint, cand);
#pragma unroll
  for (int u = 0; u < R::N; ++u) {
    e.x[u] = S.X(u);
    e.y[u] = S.Y(u);
  }
}

// ------------------------------------------------------------- unit logic
// The pick-th legal action of unit u (smax.cpp:195-211 + legal_uniform,
// vector_env.cpp:21-32): moves 0-3, stop, attacks on living opponents in range.
template <class R>
__device__ __forceinline__ int random_legal(const Params& P, const Slice<R>& S, int u, const Key& ek) {
  if (!(S.H(u) > 0.0)) return kStop;
  const bool ally = u < R::NA;
  const int opp0 = ally ? R::NA : 0, opp_n = ally ? R::NE : R::NA;
  unsigned att = 0;
#pragma unroll 1
  for (int k = 0; k < opp_n; ++k)
    if (S.H(opp0 + k) > 0.0 && in_range(P, S, u, opp0 + k)) att |= 1u << k;
  int pk = int(mod_small(block_at_nl(ek, uint64_t(u)), uint32_t(kAttackBase + __popc(att))));
  if (pk < kAttackBase) return pk;
  for (pk -= kAttackBase; pk > 0; --pk) att &= att - 1;  // drop the lowest set bits
  return kAttackBase + __ffs(int(att)) - 1;
}

// heuristic_action (smax.cpp:374-419) of unit u on the pre-step state; the
// unit's memory (ai_target / ai_sweep) lives in the slice.
template <class R>
__device__ __forceinline__ int heuristic(const Params& P, const Slice<R>& S, int u) {
  if (!(S.H(u) > 0.0)) return kStop;
  const int team = u < R::NA ? 0 : 1;
  const int opp0 = team == 0 ? R::NA : 0, opp_n = team == 0 ? R::NE : R::NA;
  unsigned vis = 0, inr = 0;
#pragma unroll 1
  for (int k = 0; k < opp_n; ++k) {
    const int o = opp0 + k;
    if (S.H(o) > 0.0 && sees(P, S, u, o)) vis |= 1u << k;
    if (in_range(P, S, u, o)) inr |= 1u << k;
  }
  int target = S.TG(u);
  if (target < 0 || target >= opp_n || !(vis >> target & 1u)) {
    const unsigned reach = vis & inr;  // lowest-index visible opponent already in reach
    if (reach) {
      target = __ffs(int(reach)) - 1;
    } else {  // otherwise the nearest visible one (first of equals)
      target = -1;
      double bdx = 0.0, bdy = 0.0, bd2 = 0.0;
#pragma unroll 1
      for (unsigned m = vis; m; m &= m - 1) {
        const int k = __ffs(int(m)) - 1, o = opp0 + k;
        const double dx = S.X(u) - S.X(o), dy = S.Y(u) - S.Y(o), d2 = dx * dx + dy * dy;
        if (target < 0 || hypot_less(dx, dy, d2, bdx, bdy, bd2)) {
          target = k;
          bdx = dx;
          bdy = dy;
          bd2 = d2;
        }
      }
    }
    S.TG(u) = int8_t(target);
  }
  if (target >= 0) {
    if (inr >> target & 1u) return kAttackBase + target;
    const double dx = S.X(opp0 + target) - S.X(u);
    const double dy = S.Y(opp0 + target) - S.Y(u);
    if (fabs(dx) >= fabs(dy)) return dx > 0 ? kEast : kWest;
    return dy > 0 ? kNorth : kSouth;
  }
  int sweep = S.SW(u);
  if (sweep < 0) sweep = team == 0 ? kEast : kWest;
  if (S.X(u) <= 1.0) sweep = kEast;
  if (S.X(u) >= P.map - 1.0) sweep = kWest;
  S.SW(u) = int8_t(sweep);
  return sweep;
}

// simulate_tick (smax.cpp:503-537) on registers.
template <class R>
__device__ __forceinline__ void tick(const Params& P, Units<R>& e, bool final_tick, const Slice<R>& S) {
#pragma unroll
  for (int u = 0; u < R::N; ++u) {  // weapons recharge, then moves
    if (!(e.h[u] > 0.0)) continue;
    const double v = e.cd[u] - kDt;
    e.cd[u] = (0.0 < v) ? v : 0.0;  // std::max(0.0, v)
    const int a = e.act[u];
    const TypeStat& t = P.ts[e.T(u)];
    // branch-free: a non-moving axis (or a stop / attack action) adds
    // spdt * 0.0 = +0.0 and clamps an in-range value, i.e. leaves it exactly
    // unchanged (positions always lie inside [radius, map - radius])
    const double dxs = a == kEast ? 1.0 : a == kWest ? -1.0 : 0.0;    // kDirX
    const double dys = a == kNorth ? 1.0 : a == kSouth ? -1.0 : 0.0;  // kDirY
    e.x[u] = dclamp(e.x[u] + t.spdt * dxs, t.rad, t.hi);
    e.y[u] = dclamp(e.y[u] + t.spdt * dys, t.rad, t.hi);
  }
  // simultaneous fire against the tick-start health snapshot
  bool fire[R::N];
#pragma unroll
  for (int u = 0; u < R::N; ++u) {
    fire[u] = false;
    const int a = e.act[u];
    if (a < kAttackBase || !(e.h[u] > 0.0)) continue;
    const bool ally = u < R::NA;
    const int opp0 = ally ? R::NA : 0, opp_n = ally ? R::NE : R::NA;
    const int k = a - kAttackBase;
    const double ho = pick(e.h, opp0, opp_n, k);
    const double xo = pick(e.x, opp0, opp_n, k), yo = pick(e.y, opp0, opp_n, k);
    const int to = R::HT >= 0 ? R::HT : pick(e.ty, opp0, opp_n, k);
    fire[u] = ho > 0.0 && !(e.cd[u] > 0.0) && dist_le_t(P.ps[e.T(u)][to].reach, e.x[u] - xo, e.y[u] - yo);
    if (fire[u]) e.cd[u] = P.ts[e.T(u)].cdmax;
  }
#pragma unroll
  for (int o = 0; o < R::N; ++o) {  // damage in shooter order, then health
    const bool ally = o < R::NA;
    const int opp0 = ally ? R::NA : 0, opp_n = ally ? R::NE : R::NA;
    const int me = ally ? o : o - R::NA;
    double damage = 0.0;
#pragma unroll
    for (int k = 0; k < opp_n; ++k) {
      const int u = opp0 + k;
      // adding +0.0 for a non-shooter leaves the ordered sum unchanged
      damage += (fire[u] && e.act[u] - kAttackBase == me) ? P.ts[e.T(u)].dmg : 0.0;
    }
    if (damage > 0.0) {
      const double v = e.h[o] - damage;
      e.h[o] = (0.0 < v) ? v : 0.0;
    }
  }
  separate(P, e, final_tick, S);
}

// pool(s, 0) and pool(s, 1), smax.cpp:365-372
template <class R>
__device__ __forceinline__ void pools(const Params& P, const Slice<R>& S, double& p0, double& p1) {
  p0 = 0.0;
  p1 = 0.0;
#pragma unroll 1
  for (int u = 0; u < R::N; ++u) {
    const double h = S.H(u);
    const double r = ddiv(h, P.ts[S.T(u)].hmax), alive = h > 0.0 ? 1.0 : 0.0;
    double& p = u < R::NA ? p0 : p1;
    p += r;
    p += alive;
  }
}

// SmaxEnv::reset (smax.cpp:163-193) of this lane's env, into the slice.
// `jit` holds the env's 2N spawn-jitter draws (x, y per unit) computed by the
// warp (fixed rosters with jitter, reset_draws below).
template <class R>
__device__ __forceinline__ void env_reset(const Params& P, const Slice<R>& S, const Key& key, const double* jit) {
  constexpr int N = R::N;
#pragma unroll 1
  for (int u = 0; u < N; ++u) {
    if (R::HT < 0)
      S.TY(u) = P.random_types  // randint1(fold_in(key, 10 + i | 500 + i), 0, kTypeCount)
                    ? int8_t(block_at_nl(fold_in_nl(key, u < R::NA ? 10 + uint64_t(u) : 500 + uint64_t(u - R::NA)), 0) %
                             uint64_t(kTypes))
                    : P.type[u];
    S.TG(u) = -1;
    S.SW(u) = -1;
  }
  if (P.random_types) {  // spawn_smacv2, smax.cpp:456-479
    const bool reflect = to_unit(block_at_nl(fold_in_nl(key, 1), 0)) < 0.5;
    const bool allies_center = !reflect && to_unit(block_at_nl(fold_in_nl(key, 2), 0)) < 0.5;
#pragma unroll 1
    for (int u = 0; u < N; ++u) {
      const bool ally = u < R::NA;
      const int i = ally ? u : u - R::NA;
      double bx, by;
      if (reflect) {  // enemy positions mirror the ally draws
        const double ax = uniform_at_nl(fold_in_nl(key, 1000 + 2 * uint64_t(i)), 0.1 * P.map, 0.4 * P.map);
        const double ay = uniform_at_nl(fold_in_nl(key, 1001 + 2 * uint64_t(i)), 0.1 * P.map, 0.9 * P.map);
        bx = ally ? ax : P.map - ax;
        by = ay;
      } else if (ally == allies_center) {
        bx = 0.5 * P.map + 1.5 * (i / 5);
        by = 0.5 * P.map + 1.5 * (i % 5 - 2);
        if (P.jitter > 0.0) {
          bx += uniform_at_nl(fold_in_nl(key, 3000 + 2 * uint64_t(u)), -P.jitter, P.jitter);
          by += uniform_at_nl(fold_in_nl(key, 3001 + 2 * uint64_t(u)), -P.jitter, P.jitter);
        }
      } else {
        const double theta = uniform_at_nl(fold_in_nl(key, 2000 + 2 * uint64_t(i)), 0.0, 6.283185307179586);
        const double rho = uniform_at_nl(fold_in_nl(key, 2001 + 2 * uint64_t(i)), 0.25 * P.map, 0.45 * P.map);
        bx = 0.5 * P.map + rho * cos(theta);
        by = 0.5 * P.map + rho * sin(theta);
      }
      const TypeStat& t = P.ts[S.T(u)];
      S.X(u) = dclamp(bx, t.rad, t.hi);
      S.Y(u) = dclamp(by, t.rad, t.hi);
    }
  } else {  // spawn_clusters + place_jittered, smax.cpp:448-454,481-492
#pragma unroll 1
    for (int u = 0; u < N; ++u) {
      const bool ally = u < R::NA;
      const int i = ally ? u : u - R::NA;
      double bx = ally ? 0.25 * P.map - 1.5 * (i / 5) : 0.75 * P.map + 1.5 * (i / 5);
      double by = 0.5 * P.map + 1.5 * (i % 5 - 2);
      if (P.jitter > 0.0) {
        bx += jit[2 * u];
        by += jit[2 * u + 1];
      }
      const TypeStat& t = P.ts[S.T(u)];
      S.X(u) = dclamp(bx, t.rad, t.hi);
      S.Y(u) = dclamp(by, t.rad, t.hi);
    }
  }
#pragma unroll 1
  for (int u = 0; u < N; ++u) {
    S.H(u) = P.ts[S.T(u)].hmax;
    S.CD(u) = 0.0;
    S.PA(u) = int8_t(kStop);
  }
  separate_slice<R>(P, S, true, ~uint64_t(0));  // spawn jitter may leave small overlaps
}

// Columns of part `p` of observe(s, me) (smax.cpp:601-634), written to
// row[0..) relative to the part's first column.
template <class R>
__device__ __forceinline__ void observe_part(const Params& P, const Slice<R>& S, int me, int p, float* row) {
  const bool alive = S.H(me) > 0.0;  // the dead see nothing
  const int tm = S.T(me);
  const TypeStat& my = P.ts[tm];
  const int s0 = p == 0 ? 0 : R::K0 + (p - 1) * R::K;
  const int s1 = min(R::N - 1, p == 0 ? R::K0 : s0 + R::K);
  const int c0 = p == 0 ? 0 : 10 + 17 * s0;
  if (p == 0) {
    row[0] = alive ? fdiv_f(S.H(me), my.rhmax, my.hmax) : 0.0f;
    row[1] = alive ? fdiv_f(S.CD(me), my.rcdmax, my.cdmax) : 0.0f;
    row[2] = alive ? fdiv_f(S.X(me), P.rmap, P.map) : 0.0f;
    row[3] = alive ? fdiv_f(S.Y(me), P.rmap, P.map) : 0.0f;
#pragma unroll
    for (int q = 0; q < kTypes; ++q) row[4 + q] = alive && q == tm ? 1.0f : 0.0f;
  }
  // teammates (index order, minus me), then opponents
  const bool me_ally = me < R::NA;
  const int tb = me_ally ? 0 : R::NA, tn = me_ally ? R::NA : R::NE, ob = me_ally ? R::NA : 0;
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int u = s < tn - 1 ? tb + s + (tb + s >= me ? 1 : 0) : ob + (s - (tn - 1));
    const bool vis = alive && S.H(u) > 0.0 && sees(P, S, me, u);
    float* o = row + 10 + 17 * s - c0;
    const int tu = S.T(u);
    const TypeStat& st = P.ts[tu];
    const double sight = my.sight.r;
    o[0] = vis ? 1.0f : 0.0f;
    o[1] = vis ? fdiv_f(S.X(u) - S.X(me), my.rsight, sight) : 0.0f;
    o[2] = vis ? fdiv_f(S.Y(u) - S.Y(me), my.rsight, sight) : 0.0f;
    o[3] = vis ? fdiv_f(S.H(u), st.rhmax, st.hmax) : 0.0f;
    o[4] = vis ? fdiv_f(S.CD(u), st.rcdmax, st.cdmax) : 0.0f;
#pragma unroll
    for (int q = 0; q < kTypes; ++q) o[5 + q] = vis && q == tu ? 1.0f : 0.0f;
    const int pa = S.PA(u), bucket = pa <= kStop ? pa : kStop + 1;  // action_bucket, smax.cpp:589
#pragma unroll
    for (int q = 0; q < 6; ++q) o[11 + q] = vis && q == bucket ? 1.0f : 0.0f;
  }
}

// Observation rows of the warp's selected envs (bit l of sel = lane l's env,
// env w0 + l) -> gdst [N][A][D], CE envs per chunk: the lanes build the
// chunk's (env, agent, part) items in the tile, then the warp stores the
// chunk -- as 16-byte vectors when every env of it is selected.
template <class R>
__device__ __forceinline__ void emit_obs(const Params& P, const Slice<R>& S, float* tile, float* __restrict__ gdst,
                                         int64_t w0, unsigned sel) {
  const int lane = threadIdx.x & 31;
  constexpr int RUN = R::A * R::D;  // floats per env
  constexpr unsigned cmask = R::CE == 32 ? 0xffffffffu : (1u << R::CE) - 1u;
#pragma unroll 1
  for (int c = 0; c < 32 / R::CE; ++c) {
    const unsigned cs = (sel >> (c * R::CE)) & cmask;
    if (!cs) continue;  // warp-uniform
#pragma unroll 1
    for (int it = lane; it < R::kItems; it += 32) {
      const int e = it / (R::A * R::NP), rem = it - e * (R::A * R::NP);
      const int me = rem / R::NP, p = rem - me * R::NP;
      if (!(cs >> e & 1u)) continue;
      const int l = c * R::CE + e;  // the env's lane: its slice
      const Slice<R> Se{S.d - lane + l, S.b - lane + l};
      const int c0 = p == 0 ? 0 : 10 + 17 * (R::K0 + (p - 1) * R::K);
      observe_part<R>(P, Se, me, p, tile + e * RUN + me * R::D + c0);
    }
    __syncwarp();
    float* g = gdst + (w0 + c * R::CE) * RUN;
    if (cs == cmask && !R::kVec) {
#pragma unroll 4
      for (int q = lane; q < R::CE * RUN; q += 32) __stcs(g + q, tile[q]);
    } else if (cs == cmask) {
      const float4* src = reinterpret_cast<const float4*>(tile);
      float4* dst = reinterpret_cast<float4*>(g);
#pragma unroll 2
      for (int q = lane; q < R::CE * RUN / 4; q += 32) __stcs(dst + q, src[q]);
    } else {
#pragma unroll 1
      for (unsigned m = cs; m; m &= m - 1) {
        const int e = __ffs(int(m)) - 1;
        for (int q = lane; q < RUN; q += 32) __stcs(g + e * RUN + q, tile[e * RUN + q]);
      }
    }
    __syncwarp();
  }
}

// The spawn-jitter draws of every env of the warp that resets this step,
// spread over all 32 lanes: draw q = 2u + c of env l is
// uniform1(fold_in(reset_key_l, 3000 + 2u + c), -jitter, jitter)
// (place_jittered, smax.cpp:486-492).  scratch: [32] reset keys, then
// [32][2N] draws; returns this lane's draw row.
template <class R>
__device__ __forceinline__ const double* reset_draws(const Params& P, uint8_t* scratch, unsigned done_lanes, bool done,
                                                     const Key& rk) {
  const int lane = threadIdx.x & 31;
  uint4* keys = reinterpret_cast<uint4*>(scratch);
  double* draws = reinterpret_cast<double*>(scratch + 32 * sizeof(uint4));
  if (P.random_types || !(P.jitter > 0.0)) return draws + lane * 2 * R::N;
  if (done) keys[lane] = make_uint4(rk.k0, rk.k1, rk.c0, rk.c1);
  __syncwarp();
  const int total = __popc(done_lanes) * 2 * R::N;
#pragma unroll 1
  for (int j = lane; j < total; j += 32) {
    const int ord = j / (2 * R::N), q = j - ord * 2 * R::N;
    const int l = int(__fns(done_lanes, 0, ord + 1));  // the ord-th resetting lane
    const uint4 kw = keys[l];
    const Key k{kw.x, kw.y, kw.z, kw.w};
    draws[l * 2 * R::N + q] = uniform_at_nl(fold_in_nl(k, 3000 + uint64_t(q)), -P.jitter, P.jitter);
  }
  __syncwarp();
  return draws + lane * 2 * R::N;
}

template <class R, bool RANDOM>
__global__ void __launch_bounds__(kLT, R::kMinBlocks * 128 / kLT) smax_lane_step_kernel(const __grid_constant__ Params P, SmaxState st,
                                                               LaunchCommon lc, Key step_key) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (*(volatile int*)lc.err) return;  // a pending contract error freezes the batch
  const int lane = threadIdx.x & 31;
  uint8_t* wbase = smem + (threadIdx.x >> 5) * R::kWarpBytes;
  float* tile = reinterpret_cast<float*>(wbase);
  const Slice<R> S{reinterpret_cast<double*>(wbase + R::kTileBytes) + lane,
                   reinterpret_cast<int8_t*>(wbase + R::kTileBytes + 4 * R::N * 32 * 8) + lane};
  const int64_t w0 = lc.begin + int64_t(blockIdx.x) * kLT + (threadIdx.x & ~31);
  if (w0 >= lc.end) return;  // whole warp past the end (warp-uniform)
  const int64_t i = w0 + lane;
  const bool live = i < lc.end;
  const int64_t n = lc.n;
  constexpr int A = R::A;

  Key carry{0, 0, 0, 0};
  double ep_ret = 0.0;
  int ep_len = 0, t = 0;
  bool done = false;
  if (live) {
    const uint4 kw = lc.carry.keys[i];
    carry = Key{kw.x, kw.y, kw.z, kw.w};
    ep_ret = lc.carry.ep_return[i];
    ep_len = lc.carry.ep_length[i];
    t = st.t[i];
    Units<R> e;
#pragma unroll
    for (int u = 0; u < R::N; ++u) {
      e.x[u] = st.x[u * n + i];
      e.y[u] = st.y[u * n + i];
      e.h[u] = st.health[u * n + i];
      e.cd[u] = st.cooldown[u * n + i];
      const uint32_t m = st.mem[u * n + i];  // prev_action | ai_target<<8 | ai_sweep<<16 | type<<24
      S.X(u) = e.x[u];
      S.Y(u) = e.y[u];
      S.H(u) = e.h[u];
      S.TG(u) = int8_t((m >> 8) & 0xffu);
      S.SW(u) = int8_t((m >> 16) & 0xffu);
      S.TY(u) = int8_t(m >> 24);
      e.ty[u] = int(int8_t(m >> 24));
    }
    // ---- actions on the pre-step state (smax.cpp:225-240): agents from the
    // caller / the probe's random-legal stream, enemies from the heuristic
    Key ek{0, 0, 0, 0};
    if (RANDOM) ek = split_child(step_key, uint64_t(lc.offset + i));  // vector_env.cpp:171
#pragma unroll 1
    for (int u = 0; u < R::N; ++u) {
      int a;
      if (u < A) {
        a = RANDOM ? random_legal(P, S, u, ek) : lc.v.actions[i * A + u];
        if (RANDOM) lc.v.actions[i * A + u] = a;
      } else {
        a = heuristic(P, S, u);
      }
      S.PA(u) = int8_t(a);  // prev_action <- this step's action (smax.cpp:243)
    }
#pragma unroll
    for (int u = 0; u < R::N; ++u) e.act[u] = S.PA(u);
    double pp0, pp1;
    pools(P, S, pp0, pp1);

    // ---- physics (smax.cpp:242-254)
#pragma unroll 1
    for (int k = 0; k < kTicks; ++k) tick(P, e, k == kTicks - 1, S);
    int ally_alive = 0, enemy_alive = 0;
#pragma unroll
    for (int u = 0; u < R::N; ++u) {
      const int alive = e.h[u] > 0.0 ? 1 : 0;
      if (u < R::NA) ally_alive += alive;
      else enemy_alive += alive;
      S.X(u) = e.x[u];
      S.Y(u) = e.y[u];
      S.H(u) = e.h[u];
      S.CD(u) = e.cd[u];
    }
    t += 1;
    int winner = -1;
    if (ally_alive == 0 && enemy_alive == 0) winner = 2;
    else if (enemy_alive == 0) winner = 0;
    else if (ally_alive == 0) winner = 1;
    else if (t >= P.max_steps) winner = 2;  // timeout is a draw
    done = winner != -1;

    // ---- reward_map (smax.cpp:352-363), infos and dones (smax.cpp:256-268)
    double pn0, pn1;
    pools(P, S, pn0, pn1);
    double ally_r = 0.5 * (pp1 - pn1) / (2.0 * R::NE);
    double enemy_r = 0.5 * (pp0 - pn0) / (2.0 * R::NA);
    if (winner == 0) ally_r += 0.5;
    if (winner == 1) enemy_r += 0.5;
    double sum = 0.0;
#pragma unroll 1
    for (int a = 0; a < A; ++a) {
      const int team = a < R::NA ? 0 : 1;
      const double r = team == 0 ? ally_r : enemy_r;
      sum += r;
      lc.v.rewards[i * A + a] = r;
      double* inf = lc.v.infos + (i * A + a) * 3;
      inf[0] = S.H(a) > 0.0 ? 1.0 : 0.0;    // alive
      inf[1] = winner == team ? 1.0 : 0.0;  // battle_won
      inf[2] = winner == 2 ? 1.0 : 0.0;     // draw
      lc.v.dones[i * (A + 1) + a] = done;
    }
    ep_ret = ep_ret + sum / double(A);  // team_reward, vector_env.cpp:14-18,99
    ep_len = ep_len + 1;
    lc.v.dones[i * (A + 1) + A] = done;
    lc.v.finished[i] = done;
    lc.v.final_returns[i] = done ? ep_ret : 0.0;
    lc.v.final_lengths[i] = done ? ep_len : 0;
  }
  stats_add(lc.stats, done, ep_len, ep_ret);

  // ---- terminal observations -> final_obs, auto-reset (vector_env.cpp:107-119),
  // state write-back, observations; one emission code site for both passes
  const unsigned done_lanes = __ballot_sync(0xffffffffu, done);
  unsigned sel = done_lanes;
  float* dst = lc.v.final_obs;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (sel) emit_obs<R>(P, S, tile, dst, w0, sel);
    if (pass == 1) break;
    if (done_lanes) {
      const Key rk = done ? split_child_nl(carry, 1) : Key{0, 0, 0, 0};
      const double* jit = reset_draws<R>(P, reinterpret_cast<uint8_t*>(tile), done_lanes, done, rk);
      if (done) {
        env_reset<R>(P, S, rk, jit);
        ep_ret = 0.0;
        ep_len = 0;
        t = 0;
      }
      __syncwarp();  // the tile is free again
    }
    if (live) {
      const Key nk = split_child(carry, 2);  // vector_env.cpp:126
      lc.carry.keys[i] = make_uint4(nk.k0, nk.k1, nk.c0, nk.c1);
      lc.carry.ep_return[i] = ep_ret;
      lc.carry.ep_length[i] = ep_len;
      st.t[i] = t;
#pragma unroll 1
      for (int u = 0; u < R::N; ++u) {
        st.x[u * n + i] = S.X(u);
        st.y[u * n + i] = S.Y(u);
        st.health[u * n + i] = S.H(u);
        st.cooldown[u * n + i] = S.CD(u);
        st.mem[u * n + i] = uint32_t(uint8_t(S.PA(u))) | (uint32_t(uint8_t(S.TG(u))) << 8) |
                            (uint32_t(uint8_t(S.SW(u))) << 16) | (uint32_t(uint8_t(S.T(u))) << 24);
      }
    }
    sel = __ballot_sync(0xffffffffu, live);
    dst = lc.v.obs;
  }
}

template <class R>
bool launch(const Params& P, const SmaxState& s, const LaunchCommon& lc, bool random, Key k) {
  const size_t sm = size_t(kLW) * R::kWarpBytes;
  auto fn = random ? smax_lane_step_kernel<R, true> : smax_lane_step_kernel<R, false>;
  smem_optin(fn);
  fn<<<unsigned((lc.end - lc.begin + kLT - 1) / kLT), kLT, sm, lc.stream>>>(P, s, lc, k);
  return true;
}

}  // namespace

// One-thread-per-env instances for the small rosters; false -> the caller
// uses the lane-group kernel (smax.cu).  MARL_SMAX_GROUP=1 forces the latter,
// MARL_SMAX_LANE=1 the former.
bool smax_lane_launch_step(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, bool random,
                           KeyWords step_key) {
  if (std::getenv("MARL_SMAX_GROUP")) return false;
  // small batches: one thread per env leaves most warp slots empty (16 384 envs:
  // 3.5 warps per SM) and the lane-group kernel, G lanes per env, is faster --
  // 3m at 16 384 envs 0.125 vs 0.141 ms, at 32 768 0.193 vs 0.151 ms; 2s3z at
  // 32 768 0.78 vs 0.83 ms, at 49 152 1.12 vs 0.88 ms (same-box runs).
  // MARL_SMAX_LANE=1 forces this kernel at any size (the parity tests).
  static const char* lane_min_env = std::getenv("MARL_SMAX_LANE_MIN");
  const int64_t lane_min = lane_min_env ? std::atoll(lane_min_env) : (c.na + c.ne <= 6 ? 24576 : 40960);
  if (lc.end - lc.begin < lane_min && !std::getenv("MARL_SMAX_LANE")) return false;
  const Params& dP = *static_cast<const Params*>(c.host_params);
  const Key k = to_key(step_key);
  bool marines = !c.random_types;
  for (int u = 0; u < c.na + c.ne && marines; ++u) marines = c.type[u] == 0;
  const bool ctrl = c.enemy_controlled != 0;
  if (c.na == 3 && c.ne == 3 && marines && !ctrl) return launch<Roster<3, 3, 0, false>>(dP, s, lc, random, k);
#ifndef MARL_LANE_3M_ONLY  // development builds: one instance compiles in seconds
  if (c.na == 3 && c.ne == 3 && marines && ctrl) return launch<Roster<3, 3, 0, true>>(dP, s, lc, random, k);
  if (c.na == 5 && c.ne == 6 && marines && !ctrl) return launch<Roster<5, 6, 0, false>>(dP, s, lc, random, k);
  if (c.na == 5 && c.ne == 5 && !ctrl) return launch<Roster<5, 5, -1, false>>(dP, s, lc, random, k);
#endif
  return false;
}

}  // namespace marl_b200
