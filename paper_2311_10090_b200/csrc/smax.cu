// SMAX unit combat (reference: proj/core/src/envs/smax.cpp) as one fused
// sm_100a kernel per batch step: random-legal ally actions, the built-in
// heuristic enemy, 8 physics ticks with simultaneous fire and Gauss-Seidel
// separation, win/draw resolution, shaped rewards, infos, auto-reset and the
// observation rows (VectorEnv::step body, vector_env.cpp:95-127).
//
// Execution model: a GROUP of G lanes (G = 8/16/32, inside one warp) owns one
// env; lane l owns units l and l+G (UPL units per lane).  The env's unit
// state (x, y, health, cooldown, action, prev_action, fire flag) lives in
// shared memory for the duration of the step -- every pairwise query (range,
// sight, nearest target, damage gather, overlap) is a lane reading the
// others' entries -- and group-scope __syncwarp / __ballot_sync / __shfl_sync
// separate the phases and carry the ordered reductions.  Per-unit work
// (heuristic enemy, random-legal draw, cooldown, moves, fire, damage,
// health/max-health ratios, observation slots, spawn jitter) runs one unit per
// lane; pair scans are spread evenly over the group's lanes.  The only
// sequential piece is the reference's Gauss-Seidel separation pass
// (smax.cpp:542-567), whose result depends on pair order: a parallel ballot
// first proves the common case "no living pair can overlap" (the pass is then
// a no-op) and only otherwise one lane replays the exact sequential pass.
//
// Exactness: every fp64 op is the reference's, in its order (-fmad=false).
// Threshold tests on glibc hypot() are decided from dx^2+dy^2 outside a 2e-12
// relative band and by the glibc-exact hypot inside it (dist_le, common.cuh);
// so is the nearest-target comparison.  Hypot values that feed arithmetic
// (separation pushes) use the glibc-exact kernel -- trajectories are
// bit-identical to the reference.
//
// HBM layout: unit state is [unit][N] structure of arrays (a warp's lanes for
// one unit read consecutive envs: full 32-byte sectors).  Observation rows of
// a warp's envs are staged in a per-warp shared-memory tile and leave as
// contiguous (16-byte vector when aligned) streaming stores; no block-wide
// barrier sits on the step path, so a group stuck in a long separation
// fixpoint delays only its own warp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "engine.h"
#include "smax_params.cuh"

namespace marl_b200 {
namespace {
using namespace smax;

// One env's unit state during a step (shared memory).
// HT >= 0: every unit of the roster has type HT (fixed single-type rosters such
// as 3m / 5m_vs_6m / 27m_vs_30m): type lookups fold to compile-time constants.
// FU: the roster fills the lane group exactly with two equal teams and only the
// allies are agents (n == CAP, na == ne == A: 3m, 2s3z): unit, team, agent
// counts and the observation width are compile-time constants and the u < n /
// team tests fold.
template <int CAP, int HT = -1, bool FU = false>
struct EnvSm {
  double x[CAP], y[CAP], h[CAP], cd[CAP];
  int act[CAP];
  int8_t pa[CAP];
  int8_t fire[CAP];
  int8_t ty[CAP];  // unit types of this env (the roster, or smacv2's per-episode draw)
  __device__ __forceinline__ int T(int u) const { return HT >= 0 ? HT : int(ty[u]); }
  __device__ __forceinline__ int nu(const Params& P) const { return FU ? CAP : P.n; }
  __device__ __forceinline__ int na(const Params& P) const { return FU ? CAP / 2 : P.na; }
  __device__ __forceinline__ int ne(const Params& P) const { return FU ? CAP / 2 : P.ne; }
};

// A group of G lanes of one warp (G need not be a power of two: a warp holds
// EPW = 32/G groups; the 32 - EPW*G leftover lanes are "dead" and own no env).
template <int G>
struct Grp {
  static constexpr int EPW = 32 / G;
  int gl;         // lane within the group
  int base;       // warp lane of the group's lane 0
  unsigned mask;  // the group's lanes within the warp
  bool dead;
  __device__ __forceinline__ Grp() {
    const int lane = threadIdx.x & 31, slot = lane / G;
    dead = slot >= EPW;
    base = slot * G;
    gl = lane - base;
    mask = dead ? (1u << lane) : G == 32 ? 0xffffffffu : (((1u << G) - 1u) << base);
  }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  __device__ __forceinline__ bool any(bool p) const { return (__ballot_sync(mask, p) & mask) != 0u; }
  __device__ __forceinline__ bool all(bool p) const { return (__ballot_sync(mask, p) & mask) == mask; }
  __device__ __forceinline__ int count(bool p) const { return __popc(__ballot_sync(mask, p) & mask); }
  __device__ __forceinline__ double bcast(double v, int src) const { return __shfl_sync(mask, v, base + src); }
};

template <int CAP, int HT, bool FU>
__device__ __forceinline__ bool in_range(const Params& P, const EnvSm<CAP, HT, FU>& e, int a, int b) {
  const Thresh& r = P.ps[e.T(a)][e.T(b)].reach;  // smax.cpp:497-501
  return dist_le(e.x[a] - e.x[b], e.y[a] - e.y[b], r.r, r.r2lo, r.r2hi);
}

template <int CAP, int HT, bool FU>
__device__ __forceinline__ bool sees(const Params& P, const EnvSm<CAP, HT, FU>& e, int a, int b) {
  const Thresh& r = P.ts[e.T(a)].sight;  // center_dist(a, b) <= sight(a), smax.cpp:383,613
  return dist_le(e.x[a] - e.x[b], e.y[a] - e.y[b], r.r, r.r2lo, r.r2hi);
}

// ------------------------------------------------------------- pair walks
// Pairs (a, b > a) in the reference's row-major order, dealt round-robin to
// the G lanes: lane l visits pair indices l, l+G, l+2G, ...
struct PairIt {
  int a, b, n;
  __device__ __forceinline__ PairIt(int first, int n_) : a(0), b(0), n(n_) {
    int p = first, row = n - 1;
    while (row > 0 && p >= row) {
      p -= row;
      ++a;
      --row;
    }
    b = a + 1 + p;
  }
  __device__ __forceinline__ bool valid() const { return a < n - 1 && b < n; }
  __device__ __forceinline__ void advance(int step) {
    b += step;
    while (b >= n && a < n - 1) {  // row a holds b in [a+1, n)
      ++a;
      b = b - n + a + 1;
    }
  }
};

// ---------------------------------------------------------------- separation
// glibc hypot with the common case inline: finite operands whose ratio and
// magnitudes need none of __hypot's rescaling go straight to its kernel (the
// same operations hypot_glibc performs for them); the rest call it.  Inline
// on the separation path: the out-of-line call spills the caller's live
// registers around every push and every touching-pair test.
__device__ __forceinline__ double hypot_fast(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax <= 0x1p+511 && ay >= 0x1p-511 && ay > ax * 0x1p-54) return hypot_kernel(ax, ay);
  return hypot_glibc(x, y);
}

__device__ __forceinline__ unsigned long long bits_above(int i) { return i >= 63 ? 0ull : ~0ull << (i + 1); }

// Unit bitmask (bit u) of a per-unit predicate held by the owning lanes.
template <int G, int UPL>
__device__ __forceinline__ unsigned long long unit_mask(const Grp<G>& g, const bool* pred) {
  const int base = g.base;
  const unsigned gbits = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  unsigned long long m = 0;
#pragma unroll
  for (int j = 0; j < UPL; ++j)
    m |= (unsigned long long)((__ballot_sync(g.mask, pred[j]) >> base) & gbits) << (G * j);
  return m;
}

// One Gauss-Seidel pass of separate() (smax.cpp:542-567), exact, row-parallel.
// The reference visits pairs (a, b>a) in row-major order and pushes each
// overlapping pair with the positions current at that moment.  Within row a,
// the next pair it pushes is the lowest b (after the last push) that overlaps
// with the CURRENT positions -- nothing moves in between -- so the group tests
// all remaining b of the row at once (one b per lane, exact hypot test), takes
// the lowest hit by ballot, lets b's lane apply the reference push, and
// repeats from there: rounds per row = pushes in the row + 1, and the
// trajectory is the sequential one bit for bit.
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void separation_pass(const Params& P, EnvSm<CAP, HT, FU>& e, const Grp<G>& g,
                                                unsigned long long alive) {
  const int n = e.nu(P);
  for (int a = 0; a < n - 1; ++a) {
    if (!(alive >> a & 1ull)) continue;
    unsigned long long row = alive & bits_above(a);
    const int ta = e.T(a);
    while (row) {  // group-uniform
      bool hit[UPL];
      double hdx[UPL], hdy[UPL], hd[UPL];
      // a's position is read only by lanes that test a pair of the row, and
      // every value read feeds the ballot below, so all reads of x[a], y[a]
      // have completed before b's lane (past the ballot) writes them.
      bool mine = false;
#pragma unroll
      for (int j = 0; j < UPL; ++j) mine |= (row >> (g.gl + G * j) & 1ull) != 0;
      double xa = 0.0, ya = 0.0;
      if (mine) {
        xa = e.x[a];
        ya = e.y[a];
      }
#pragma unroll
      for (int j = 0; j < UPL; ++j) {
        const int b = g.gl + G * j;
        hit[j] = false;
        hdx[j] = hdy[j] = hd[j] = 0.0;
        if (!(row >> b & 1ull)) continue;
        const double dx = e.x[b] - xa, dy = e.y[b] - ya;
        const Thresh& R = P.ps[ta][e.T(b)].rsum;
        if (dx * dx + dy * dy > R.r2hi) continue;  // hypot(dx,dy) > ra+rb: overlap <= 0
        const double dd = hypot_fast(dx, dy);
        hit[j] = R.r - dd > 0.0;
        hdx[j] = dx;
        hdy[j] = dy;
        hd[j] = dd;
      }
      const unsigned long long hits = unit_mask<G, UPL>(g, hit);
      if (!hits) break;
      const int b = __ffsll((long long)hits) - 1;
      if (g.gl == b % G) {  // b's lane applies the reference push
        const int j = b / G;  // which of the lane's units
        double dx = hdx[0], dy = hdy[0], dd = hd[0];
#pragma unroll
        for (int q = 1; q < UPL; ++q)
          if (j == q) {
            dx = hdx[q];
            dy = hdy[q];
            dd = hd[q];
          }
        const double overlap = P.ps[ta][e.T(b)].rsum.r - dd;
        double nx = 1.0, ny = 0.0;  // coincident centres get a fixed nudge axis
        if (dd > 1e-12) {
          nx = dx / dd;
          ny = dy / dd;
        }
        const double push = 0.5 * overlap;
        const TypeStat& A_ = P.ts[ta];
        const TypeStat& B_ = P.ts[e.T(b)];
        e.x[a] = dclamp(xa - nx * push, A_.rad, A_.hi);
        e.y[a] = dclamp(ya - ny * push, A_.rad, A_.hi);
        e.x[b] = dclamp(e.x[b] + nx * push, B_.rad, B_.hi);
        e.y[b] = dclamp(e.y[b] + ny * push, B_.rad, B_.hi);
      }
      g.sync();
      row &= bits_above(b);
    }
  }
}

// This lane's share of the pairs (a, b>a): indices gl, gl+G, ... of the
// reference's row-major pair order.  For G < 32 the (at most ceil((G-1)/2))
// pairs are listed once per kernel in registers; G = 32 walks them.
template <int G>
struct LanePairs {
  static constexpr int MAXP = G < 32 ? (G - 1 + 1) / 2 : 1;
  int np = 0;
  uint16_t ab[MAXP];  // a | b << 8
  __device__ __forceinline__ LanePairs(int gl, int n) {
    if (G >= 32) return;
    int k = 0;
    for (PairIt it(gl, n); it.valid() && k < MAXP; it.advance(G)) ab[k++] = uint16_t(it.a | (it.b << 8));
    np = k;
  }
};

template <int G, class F>
__device__ __forceinline__ bool for_lane_pairs(const LanePairs<G>& lp, int gl, int n, F&& f) {
  // f(a, b) returns true to stop the walk early; returns whether it stopped
  if constexpr (G < 32) {
#pragma unroll
    for (int k = 0; k < LanePairs<G>::MAXP; ++k)
      if (k < lp.np && f(int(lp.ab[k] & 0xff), int(lp.ab[k] >> 8))) return true;
    return false;
  } else {
    for (PairIt it(gl, n); it.valid(); it.advance(G))
      if (f(it.a, it.b)) return true;
    return false;
  }
}

// Does any living pair of this lane's share overlap right now (the exact
// reference test, hypot only inside the rounding band)?  If no pair overlaps
// at the start of a pass, the pass pushes nothing -- so it is skipped.
template <int G, int CAP, int HT, bool FU>
__device__ __forceinline__ bool lane_pairs_overlap(const Params& P, const EnvSm<CAP, HT, FU>& e, const LanePairs<G>& lp,
                                                   int gl) {
  return for_lane_pairs<G>(lp, gl, e.nu(P), [&](int a, int b) {
    if (e.h[a] <= 0.0 || e.h[b] <= 0.0) return false;
    const double dx = e.x[b] - e.x[a], dy = e.y[b] - e.y[a];
    const double d2 = dx * dx + dy * dy;
    if (d2 > P.sep_r2hi) return false;  // farther than any radius sum
    const Thresh& R = P.ps[e.T(a)][e.T(b)].rsum;
    if (d2 > R.r2hi) return false;
    return d2 < R.r2lo || R.r - hypot_fast(dx, dy) > 0.0;
  });
}

// max_overlap(s) <= kSeparationTol restricted to this lane's pairs (smax.cpp:569-580).
template <int G, int CAP, int HT, bool FU>
__device__ __forceinline__ bool lane_pairs_within_tol(const Params& P, const EnvSm<CAP, HT, FU>& e, const LanePairs<G>& lp,
                                                      int gl) {
  return !for_lane_pairs<G>(lp, gl, e.nu(P), [&](int a, int b) {
    if (e.h[a] <= 0.0 || e.h[b] <= 0.0) return false;
    const PairStat& S = P.ps[e.T(a)][e.T(b)];
    const double dx = e.x[a] - e.x[b], dy = e.y[a] - e.y[b];
    const double d2 = dx * dx + dy * dy;
    if (d2 > S.otol.r2hi) return false;      // surely sum - d <= tol
    if (d2 < S.otol.r2lo) return true;       // surely sum - d > tol
    return !(S.rsum.r - hypot_fast(dx, dy) <= kSepTol);
  });
}

// separate(s, to_fixpoint), smax.cpp:542-567.  A pass is a no-op exactly when
// no living pair overlaps, which the parallel pre-check proves in the common
// case (and then max_overlap <= 0 <= tol ends the fixpoint loop as well).
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void separate(const Params& P, EnvSm<CAP, HT, FU>& e, const Grp<G>& g, const LanePairs<G>& lp,
                                         bool fixpoint) {
  unsigned long long alive = 0;
  bool check = true;  // a pair over the tolerance overlaps: after a failed fixpoint test the next
                      // pass is known not to be a no-op, so its pre-check is skipped
  for (int pass = 0; pass < (fixpoint ? 256 : 1); ++pass) {
    if (check && !g.any(lane_pairs_overlap<G>(P, e, lp, g.gl))) break;
    if (pass == 0) {  // health is constant during separation
      bool al[UPL];
#pragma unroll
      for (int j = 0; j < UPL; ++j) al[j] = g.gl + G * j < e.nu(P) && e.h[g.gl + G * j] > 0.0;
      alive = unit_mask<G, UPL>(g, al);
    }
    separation_pass<G, UPL>(P, e, g, alive);
    if (!fixpoint) break;
    if (g.all(lane_pairs_within_tol<G>(P, e, lp, g.gl))) break;
#ifndef MARL_SEP_ALWAYS_CHECK  // A/B knob (development builds, MARL_NVCC_EXTRA)
    check = false;
#endif
  }
}

// ------------------------------------------------------------- unit logic
// Spawn of unit u: spawn_clusters / place_jittered (smax.cpp:448-454,481-492),
// or spawn_smacv2 (smax.cpp:456-479) for the random-type scenarios; the
// unit's type (e.T(u)) is already set.
__device__ __forceinline__ void place_at(double bx, double by, double rad, double hi, double* x, double* y) {
  *x = dclamp(bx, rad, hi);  // place (smax.cpp:481-485)
  *y = dclamp(by, rad, hi);
}

// spawn_smacv2 (smax.cpp:456-479) for unit u: kept out of line (rare, and
// the fixed-roster step kernel's instruction footprint stays as it was).
template <int CAP, int HT, bool FU>
__device__ __noinline__ void spawn_smacv2(const Params& P, EnvSm<CAP, HT, FU>& e, int u, const Key& key) {
  const bool ally = u < e.na(P);
  const int i = ally ? u : u - e.na(P);
  const TypeStat& t = P.ts[e.T(u)];
  if (to_unit(block_at_nl(fold_in_nl(key, 1), 0)) < 0.5) {
    // reflected uniform spawns: enemy i mirrors ally i's draws
    const double ax = uniform_at_nl(fold_in_nl(key, 1000 + 2 * uint64_t(i)), 0.1 * P.map, 0.4 * P.map);
    const double ay = uniform_at_nl(fold_in_nl(key, 1001 + 2 * uint64_t(i)), 0.1 * P.map, 0.9 * P.map);
    place_at(ally ? ax : P.map - ax, ay, t.rad, t.hi, &e.x[u], &e.y[u]);
    return;
  }
  // one team at the center, the other on a ring (a coin decides which)
  const bool allies_center = to_unit(block_at_nl(fold_in_nl(key, 2), 0)) < 0.5;
  if (ally == allies_center) {
    double bx = 0.5 * P.map + 1.5 * (i / 5), by = 0.5 * P.map + 1.5 * (i % 5 - 2);
    if (P.jitter > 0.0) {  // place_jittered (smax.cpp:486-492)
      bx += uniform_at_nl(fold_in_nl(key, 3000 + 2 * uint64_t(u)), -P.jitter, P.jitter);
      by += uniform_at_nl(fold_in_nl(key, 3001 + 2 * uint64_t(u)), -P.jitter, P.jitter);
    }
    place_at(bx, by, t.rad, t.hi, &e.x[u], &e.y[u]);
  } else {
    const double theta = uniform_at_nl(fold_in_nl(key, 2000 + 2 * uint64_t(i)), 0.0, 6.283185307179586);
    const double rho = uniform_at_nl(fold_in_nl(key, 2001 + 2 * uint64_t(i)), 0.25 * P.map, 0.45 * P.map);
    place_at(0.5 * P.map + rho * cos(theta), 0.5 * P.map + rho * sin(theta), t.rad, t.hi, &e.x[u], &e.y[u]);
  }
}

template <int CAP, int HT, bool FU>
__device__ __forceinline__ void spawn_unit(const Params& P, EnvSm<CAP, HT, FU>& e, int u, const Key& key) {
  const TypeStat& t = P.ts[e.T(u)];
  if (P.random_types) {
    spawn_smacv2(P, e, u, key);
  } else {
    const bool ally = u < e.na(P);
    const int i = ally ? u : u - e.na(P);
    double bx = ally ? 0.25 * P.map - 1.5 * (i / 5) : 0.75 * P.map + 1.5 * (i / 5);
    double by = 0.5 * P.map + 1.5 * (i % 5 - 2);
    if (P.jitter > 0.0) {
      bx += uniform_at_nl(fold_in_nl(key, 3000 + 2 * uint64_t(u)), -P.jitter, P.jitter);
      by += uniform_at_nl(fold_in_nl(key, 3001 + 2 * uint64_t(u)), -P.jitter, P.jitter);
    }
    place_at(bx, by, t.rad, t.hi, &e.x[u], &e.y[u]);
  }
  e.h[u] = t.hmax;
  e.cd[u] = 0.0;
  e.pa[u] = int8_t(kStop);
}

// The pick-th legal action of unit u (smax.cpp:195-211 with legal_uniform,
// vector_env.cpp:21-32).  Legal order: moves 0-3, stop, attacks on living
// opponents in range; a dead unit's only legal action is stop.
template <int CAP, int HT, bool FU>
__device__ __forceinline__ int random_legal(const Params& P, const EnvSm<CAP, HT, FU>& e, int u, const Key& ek) {
  if (e.h[u] <= 0.0) return kStop;
  const bool ally = u < e.na(P);
  const int opp0 = ally ? e.na(P) : 0, opp_n = ally ? e.ne(P) : e.na(P);
  uint64_t att = 0;
  for (int k = 0; k < opp_n; ++k) {
    const int o = opp0 + k;
    if (e.h[o] > 0.0 && in_range(P, e, u, o)) att |= uint64_t(1) << k;
  }
  int pick = int(mod_small(block_at_nl(ek, uint64_t(u)), uint32_t(kAttackBase + __popcll(att))));
  if (pick < kAttackBase) return pick;
  for (pick -= kAttackBase; pick > 0; --pick) att &= att - 1;  // drop the lowest set bits
  return kAttackBase + __ffsll((long long)att) - 1;
}

// heuristic_action (smax.cpp:374-419) of unit u on the pre-step state.
template <int CAP, int HT, bool FU>
__device__ __forceinline__ int heuristic(const Params& P, const EnvSm<CAP, HT, FU>& e, int u, int& target, int& sweep) {
  if (e.h[u] <= 0.0) return kStop;
  const int team = u < e.na(P) ? 0 : 1;
  const int opp0 = team == 0 ? e.na(P) : 0, opp_n = team == 0 ? e.ne(P) : e.na(P);
  if (target < 0 || target >= opp_n || !(e.h[opp0 + target] > 0.0 && sees(P, e, u, opp0 + target))) {
    target = -1;
    for (int k = 0; k < opp_n; ++k) {  // lowest-index opponent already in reach
      const int o = opp0 + k;
      if (e.h[o] > 0.0 && sees(P, e, u, o) && in_range(P, e, u, o)) {
        target = k;
        break;
      }
    }
    if (target < 0) {  // otherwise the nearest visible one (first of equals)
      double bdx = 0.0, bdy = 0.0, bd2 = 0.0;
      for (int k = 0; k < opp_n; ++k) {
        const int o = opp0 + k;
        if (!(e.h[o] > 0.0 && sees(P, e, u, o))) continue;
        const double dx = e.x[u] - e.x[o], dy = e.y[u] - e.y[o], d2 = dx * dx + dy * dy;
        if (target < 0 || hypot_less(dx, dy, d2, bdx, bdy, bd2)) {
          target = k;
          bdx = dx;
          bdy = dy;
          bd2 = d2;
        }
      }
    }
  }
  if (target >= 0) {
    const int o = opp0 + target;
    if (in_range(P, e, u, o)) return kAttackBase + target;
    double dx = e.x[o] - e.x[u];
    double dy = e.y[o] - e.y[u];
    if (fabs(dx) >= fabs(dy)) return dx > 0 ? kEast : kWest;
    return dy > 0 ? kNorth : kSouth;
  }
  if (sweep < 0) sweep = team == 0 ? kEast : kWest;
  if (e.x[u] <= 1.0) sweep = kEast;
  if (e.x[u] >= P.map - 1.0) sweep = kWest;
  return sweep;
}

// simulate_tick (smax.cpp:503-537), one unit per lane per phase.
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void tick(const Params& P, EnvSm<CAP, HT, FU>& e, const Grp<G>& g, const LanePairs<G>& lp,
                                     bool final_tick) {
  // weapons recharge, then moves: each lane touches only its own units
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = g.gl + G * j;
    if (u >= e.nu(P) || e.h[u] <= 0.0) continue;
    double v = e.cd[u] - kDt;
    e.cd[u] = (0.0 < v) ? v : 0.0;  // std::max(0.0, v)
    const int a = e.act[u];
    if (a > kWest) continue;
    const TypeStat& t = P.ts[e.T(u)];
    const double dxs = a == kEast ? 1.0 : a == kWest ? -1.0 : 0.0;    // kDirX
    const double dys = a == kNorth ? 1.0 : a == kSouth ? -1.0 : 0.0;  // kDirY
    e.x[u] = dclamp(e.x[u] + t.spdt * dxs, t.rad, t.hi);
    e.y[u] = dclamp(e.y[u] + t.spdt * dys, t.rad, t.hi);
  }
  g.sync();
  // simultaneous fire against the tick-start health snapshot (health is not
  // written until every shooter has been resolved)
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = g.gl + G * j;
    if (u >= e.nu(P)) continue;
    bool fire = false;
    const int a = e.act[u];
    if (a >= kAttackBase && e.h[u] > 0.0) {
      const int o = (u < e.na(P) ? e.na(P) : 0) + (a - kAttackBase);
      fire = e.h[o] > 0.0 && !(e.cd[u] > 0.0) && in_range(P, e, u, o);
      if (fire) e.cd[u] = P.ts[e.T(u)].cdmax;
    }
    e.fire[u] = fire;
  }
  g.sync();
  double newh[UPL];
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int o = g.gl + G * j;
    newh[j] = -1.0;
    if (o >= e.nu(P)) continue;
    // o's shooters are its opponents; `me` is o's index among THEIR opponents
    const int opp0 = o < e.na(P) ? e.na(P) : 0, opp_n = o < e.na(P) ? e.ne(P) : e.na(P);
    const int me = o < e.na(P) ? o : o - e.na(P);
    double damage = 0.0;
    for (int k = 0; k < opp_n; ++k) {  // shooters in unit order
      const int u = opp0 + k;
      if (e.fire[u] && e.act[u] - kAttackBase == me) damage += P.ts[e.T(u)].dmg;
    }
    if (damage > 0.0) {
      double v = e.h[o] - damage;
      newh[j] = (0.0 < v) ? v : 0.0;
    }
  }
  g.sync();
#pragma unroll
  for (int j = 0; j < UPL; ++j)
    if (newh[j] >= 0.0) e.h[g.gl + G * j] = newh[j];
  g.sync();
  separate<G, UPL>(P, e, g, lp, final_tick);
}

// pool(s, 0) and pool(s, 1) (smax.cpp:365-372): the per-unit ratios are one
// division per lane; the sums run in the reference's unit order over
// shuffled values.
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void pools(const Params& P, const EnvSm<CAP, HT, FU>& e, const Grp<G>& g, double& p0, double& p1) {
  double ratio[UPL];
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = g.gl + G * j;
    ratio[j] = u < e.nu(P) ? e.h[u] / P.ts[e.T(u)].hmax : 0.0;
  }
  p0 = 0.0;
  p1 = 0.0;
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    for (int l = 0; l < G; ++l) {
      const int u = l + G * j;
      const double r = g.bcast(ratio[j], l);  // group-uniform loop: every lane shuffles
      if (u >= e.nu(P)) continue;
      const double alive = e.h[u] > 0.0 ? 1.0 : 0.0;
      if (u < e.na(P)) {
        p0 += r;
        p0 += alive;
      } else {
        p1 += r;
        p1 += alive;
      }
    }
  }
}

// Observation slot of unit u in `me`'s row: teammates (index order, minus
// me), then opponents (smax.cpp:628-632).
__device__ __forceinline__ int obs_slot(const Params& P, int me, int u) {
  const bool me_ally = me < P.na, u_ally = u < P.na;
  if (me_ally == u_ally) {
    const int base = me_ally ? 0 : P.na;
    return (u - base) - (u > me ? 1 : 0);
  }
  const int n_team = me_ally ? P.na : P.ne;
  return n_team - 1 + (u_ally ? u : u - P.na);
}

// This lane's part of observe(s, me) (smax.cpp:601-634) into row[D].
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void observe_part(const Params& P, const EnvSm<CAP, HT, FU>& e, int gl, int me, float* row) {
  const bool me_alive = e.h[me] > 0.0;
  const TypeStat& my = P.ts[e.T(me)];
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = gl + G * j;
    if (u >= e.nu(P)) continue;
    if (u == me) {
      float* o = row;
      if (!me_alive) {
#pragma unroll
        for (int k = 0; k < 10; ++k) o[k] = 0.0f;
        continue;
      }
      o[0] = float(e.h[me] / my.hmax);
      o[1] = float(e.cd[me] / my.cdmax);
      o[2] = float(e.x[me] / P.map);
      o[3] = float(e.y[me] / P.map);
#pragma unroll
      for (int q = 0; q < kTypes; ++q) o[4 + q] = q == e.T(me) ? 1.0f : 0.0f;
      continue;
    }
    float* o = row + 10 + 17 * obs_slot(P, me, u);
    if (!(me_alive && e.h[u] > 0.0 && sees(P, e, me, u))) {
#pragma unroll
      for (int q = 0; q < 17; ++q) o[q] = 0.0f;
      continue;
    }
    const TypeStat& st = P.ts[e.T(u)];
    const double sight = my.sight.r;
    o[0] = 1.0f;
    o[1] = float((e.x[u] - e.x[me]) / sight);
    o[2] = float((e.y[u] - e.y[me]) / sight);
    o[3] = float(e.h[u] / st.hmax);
    o[4] = float(e.cd[u] / st.cdmax);
    const int tu = e.T(u);
#pragma unroll
    for (int q = 0; q < kTypes; ++q) o[5 + q] = q == tu ? 1.0f : 0.0f;
    const int bucket = e.pa[u] <= kStop ? e.pa[u] : kStop + 1;  // action_bucket, smax.cpp:589
#pragma unroll
    for (int q = 0; q < 6; ++q) o[11 + q] = q == bucket ? 1.0f : 0.0f;
  }
}

// ---------------------------------------------------------- warp plumbing
struct Plan {  // host-chosen launch shape, passed by value
  int rb;      // agent rows staged per env per round (A when everything fits)
};

__host__ __device__ inline size_t a16(size_t b) { return (b + 15) & ~size_t(15); }

template <int G>
__host__ __device__ inline size_t warp_tile_floats(int D, int rb) {
  return (size_t(Grp<G>::EPW) * rb * D + 3) & ~size_t(3);
}

template <int G, int UPL>
__host__ __device__ inline size_t smem_bytes(int D, int rb) {
  constexpr int EPB = kWarps * Grp<G>::EPW, CAP = G * UPL;
  return a16(sizeof(Params)) + a16(EPB * sizeof(EnvSm<CAP>)) + kWarps * warp_tile_floats<G>(D, rb) * 4;
}

// Copy nfloats from shared to global with one warp: 16-byte vectors when both
// ends are 16-byte aligned, else 4-byte words.
__device__ __forceinline__ void warp_store(float* __restrict__ gdst, const float* src, int nfloats) {
  const int lane = threadIdx.x & 31;
  // scalar head up to the first 16-byte aligned destination, then 16-byte
  // stores (reading the shared source as one or four words per vector)
  int head = int(((16u - (uint32_t(reinterpret_cast<uintptr_t>(gdst)) & 15u)) & 15u) >> 2);
  head = head < nfloats ? head : nfloats;
  if (lane < head) __stcs(gdst + lane, src[lane]);
  const float* s = src + head;
  float4* d4 = reinterpret_cast<float4*>(gdst + head);
  const int nv = (nfloats - head) >> 2;
  if ((reinterpret_cast<uintptr_t>(s) & 15) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(s);
#pragma unroll 1
    for (int q = lane; q < nv; q += 32) __stcs(d4 + q, s4[q]);
  } else {
#pragma unroll 1
    for (int q = lane; q < nv; q += 32) __stcs(d4 + q, make_float4(s[4 * q], s[4 * q + 1], s[4 * q + 2], s[4 * q + 3]));
  }
#pragma unroll 1
  for (int q = head + (nv << 2) + lane; q < nfloats; q += 32) __stcs(gdst + q, src[q]);
}

// All observation rows of the warp's envs -> gdst ([N][A][D]).  Warp-uniform
// call; `active` says whether this lane's group builds rows, `sel` (bitmask
// over the warp's EPW env slots) which envs are stored.
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __noinline__ void emit_obs(const Params& P, const EnvSm<CAP, HT, FU>& e, const Grp<G>& g, bool active,
                                         float* tile, float* __restrict__ gdst, int64_t w0, int wvalid, int rb,
                                         unsigned sel) {
  constexpr int EPW = Grp<G>::EPW;
  const int A = FU ? CAP / 2 : P.A, D = FU ? 10 + 17 * (CAP - 1) : P.D;
  const int wslot = (threadIdx.x & 31) / G;  // >= EPW only on dead lanes, which never build rows
  for (int a0 = 0; a0 < A; a0 += rb) {
    const int rows = min(rb, A - a0);
    if (active)
      for (int r = 0; r < rows; ++r) observe_part<G, UPL>(P, e, g.gl, a0 + r, tile + (size_t(wslot) * rows + r) * D);
    __syncwarp();
    const int run = rows * D;
    if (rows == A && sel == (1u << EPW) - 1u) {  // the warp's rows are one contiguous run
      warp_store(gdst + w0 * A * D, tile, wvalid * run);
    } else {
      for (int s = 0; s < wvalid; ++s)
        if (sel >> s & 1u) warp_store(gdst + ((w0 + s) * A + a0) * D, tile + size_t(s) * run, run);
    }
    __syncwarp();
  }
}

template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void load_env(const Params& P, EnvSm<CAP, HT, FU>& e, const SmaxState& st, int gl, int64_t i,
                                         int64_t n, int* tg, int* sw) {
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = gl + G * j;
    tg[j] = -1;
    sw[j] = -1;
    if (u >= e.nu(P)) continue;
    e.x[u] = st.x[u * n + i];
    e.y[u] = st.y[u * n + i];
    e.h[u] = st.health[u * n + i];
    e.cd[u] = st.cooldown[u * n + i];
    const uint32_t m = st.mem[u * n + i];  // prev_action | ai_target<<8 | ai_sweep<<16 | type<<24
    e.pa[u] = int8_t(m & 0xffu);
    e.ty[u] = int8_t(m >> 24);
    tg[j] = int(int8_t((m >> 8) & 0xffu));
    sw[j] = int(int8_t((m >> 16) & 0xffu));
  }
}

template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __forceinline__ void store_env(const Params& P, const EnvSm<CAP, HT, FU>& e, const SmaxState& st, int gl,
                                          int64_t i, int64_t n, const int* tg, const int* sw) {
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = gl + G * j;
    if (u >= e.nu(P)) continue;
    st.x[u * n + i] = e.x[u];
    st.y[u * n + i] = e.y[u];
    st.health[u * n + i] = e.h[u];
    st.cooldown[u * n + i] = e.cd[u];
    st.mem[u * n + i] = uint32_t(uint8_t(e.pa[u])) | (uint32_t(uint8_t(int8_t(tg[j]))) << 8) |
                        (uint32_t(uint8_t(int8_t(sw[j]))) << 16) | (uint32_t(uint8_t(e.T(u))) << 24);
  }
}

// SmaxEnv::reset (smax.cpp:163-193): spawns (one unit per lane), separation
// to the fixpoint, fresh heuristic memory.
template <int G, int UPL, int CAP, int HT, bool FU>
__device__ __noinline__ void env_reset(const Params& P, EnvSm<CAP, HT, FU>& e, const Grp<G>& g, const Key& key, int* tg,
                                          int* sw) {
#pragma unroll
  for (int j = 0; j < UPL; ++j) {
    const int u = g.gl + G * j;
    tg[j] = -1;
    sw[j] = -1;
    if (u >= e.nu(P)) continue;
    if (P.random_types) {  // randint1(fold_in(key, 10 + i | 500 + i), 0, kTypeCount) (smax.cpp:169-175)
      const uint64_t d = u < e.na(P) ? 10 + uint64_t(u) : 500 + uint64_t(u - e.na(P));
      e.ty[u] = int8_t(block_at_nl(fold_in_nl(key, d), 0) % uint64_t(kTypes));
    } else {
      e.ty[u] = P.type[u];
    }
    spawn_unit(P, e, u, key);
  }
  g.sync();
  const LanePairs<G> lp(g.gl, e.nu(P));  // rare path: built here rather than passed
  separate<G, UPL>(P, e, g, lp, true);
}

struct Smem {
  uint8_t* envs;
  float* tile;  // this warp's staging tile
};

template <int G, int UPL>
__device__ __forceinline__ Smem carve(uint8_t* base, int D, int rb) {
  constexpr int EPB = kWarps * Grp<G>::EPW, CAP = G * UPL;
  Smem m;
  m.envs = base + a16(sizeof(Params));
  float* tiles = reinterpret_cast<float*>(m.envs + a16(EPB * sizeof(EnvSm<CAP>)));
  m.tile = tiles + (threadIdx.x >> 5) * warp_tile_floats<G>(D, rb);
  return m;
}

template <int G, int UPL>
__global__ void __launch_bounds__(kThreads) smax_reset_kernel(const Params* __restrict__ gP, SmaxState st,
                                                              LaunchCommon lc, Key key, Key carry_parent, Plan plan) {
  constexpr int EPW = Grp<G>::EPW, EPB = kWarps * EPW, CAP = G * UPL;
  extern __shared__ __align__(16) uint8_t smem[];
  stage_params(reinterpret_cast<Params*>(smem), gP);
  const Params& P = *reinterpret_cast<const Params*>(smem);
  Smem m = carve<G, UPL>(smem, P.D, plan.rb);
  const Grp<G> g;
  const int slot = (threadIdx.x >> 5) * EPW + (g.dead ? 0 : (threadIdx.x & 31) / G);
  EnvSm<CAP>& e = reinterpret_cast<EnvSm<CAP>*>(m.envs)[slot];
  const int64_t i = int64_t(blockIdx.x) * EPB + slot;
  const int64_t w0 = int64_t(blockIdx.x) * EPB + (threadIdx.x >> 5) * EPW;
  const int wvalid = int(max(int64_t(0), min64(EPW, lc.n - w0)));
  if (wvalid == 0) return;  // whole warp past the end (warp-uniform)
  const bool live = !g.dead && i < lc.n;
  int tg[UPL], sw[UPL];
  if (live) {
    const uint64_t gi = uint64_t(lc.offset + i);
    env_reset<G, UPL>(P, e, g, split_child_nl(key, gi), tg, sw);  // vector_env.cpp:52,57
    if (g.gl == 0) {
      Key c = split_child_nl(carry_parent, gi);  // vector_env.cpp:55
      lc.carry.keys[i] = make_uint4(c.k0, c.k1, c.c0, c.c1);
      lc.carry.ep_return[i] = 0.0;
      lc.carry.ep_length[i] = 0;
      st.t[i] = 0;
    }
    store_env<G, UPL>(P, e, st, g.gl, i, lc.n, tg, sw);
  }
  emit_obs<G, UPL>(P, e, g, live, m.tile, lc.v.obs, w0, wvalid, plan.rb, (1u << EPW) - 1u);
}

template <int G, int UPL, bool RANDOM, int HT, bool FU>
__global__ void __launch_bounds__(kThreads, 4 * 256 / kThreads) smax_step_kernel(const Params* __restrict__ gP, SmaxState st,
                                                             LaunchCommon lc, Key step_key, Plan plan) {
  constexpr int EPW = Grp<G>::EPW, EPB = kWarps * EPW, CAP = G * UPL;
  extern __shared__ __align__(16) uint8_t smem[];
  if (*(volatile int*)lc.err) return;  // a pending contract error freezes the batch
  stage_params(reinterpret_cast<Params*>(smem), gP);
  const Params& P = *reinterpret_cast<const Params*>(smem);
  Smem m = carve<G, UPL>(smem, P.D, plan.rb);
  const Grp<G> g;
  const int slot = (threadIdx.x >> 5) * EPW + (g.dead ? 0 : (threadIdx.x & 31) / G);
  EnvSm<CAP, HT, FU>& e = reinterpret_cast<EnvSm<CAP, HT, FU>*>(m.envs)[slot];
  const int64_t i = lc.begin + int64_t(blockIdx.x) * EPB + slot;
  const int64_t w0 = lc.begin + int64_t(blockIdx.x) * EPB + (threadIdx.x >> 5) * EPW;
  const int wvalid = int(max(int64_t(0), min64(EPW, lc.end - w0)));
  if (wvalid == 0) return;  // whole warp past the end (warp-uniform)
  const bool live = !g.dead && i < lc.end;
  const int A = FU ? CAP / 2 : P.A;

  int tg[UPL], sw[UPL];
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
    load_env<G, UPL>(P, e, st, g.gl, i, lc.n, tg, sw);
    g.sync();

    // ---- actions on the pre-step state (smax.cpp:225-240): agents from the
    // caller / the probe's random-legal stream, enemies from the heuristic
    int act[UPL];
    Key ek{0, 0, 0, 0};
    if (RANDOM) ek = split_child(step_key, uint64_t(lc.offset + i));  // vector_env.cpp:171
#pragma unroll
    for (int j = 0; j < UPL; ++j) {
      const int u = g.gl + G * j;
      act[j] = kStop;
      if (u >= e.nu(P)) continue;
      if (u < A) {
        act[j] = RANDOM ? random_legal(P, e, u, ek) : lc.v.actions[i * A + u];
        if (RANDOM) lc.v.actions[i * A + u] = act[j];
      } else {
        act[j] = heuristic(P, e, u, tg[j], sw[j]);
      }
    }
    double pool_prev0, pool_prev1;
    pools<G, UPL>(P, e, g, pool_prev0, pool_prev1);
    g.sync();  // every lane has read the pre-step state
#pragma unroll
    for (int j = 0; j < UPL; ++j)
      if (g.gl + G * j < e.nu(P)) e.act[g.gl + G * j] = act[j];
    g.sync();

    // ---- physics (smax.cpp:242-254)
    const LanePairs<G> lp(g.gl, e.nu(P));
#pragma unroll 1
    for (int k = 0; k < kTicks; ++k) tick<G, UPL>(P, e, g, lp, k == kTicks - 1);
    int ally_alive = 0, enemy_alive = 0;
#pragma unroll
    for (int j = 0; j < UPL; ++j) {
      const int u = g.gl + G * j;
      const bool alive = u < e.nu(P) && e.h[u] > 0.0;
      ally_alive += g.count(alive && u < e.na(P));
      enemy_alive += g.count(alive && u >= e.na(P));
    }
    t += 1;
    int winner = -1;
    if (ally_alive == 0 && enemy_alive == 0) winner = 2;
    else if (enemy_alive == 0) winner = 0;
    else if (ally_alive == 0) winner = 1;
    else if (t >= P.max_steps) winner = 2;  // timeout is a draw
    done = winner != -1;

    // ---- reward_map (smax.cpp:352-363), infos and dones (smax.cpp:256-268)
    double pool_next0, pool_next1;
    pools<G, UPL>(P, e, g, pool_next0, pool_next1);
    double ally_r = 0.5 * (pool_prev1 - pool_next1) / (2.0 * e.ne(P));
    double enemy_r = 0.5 * (pool_prev0 - pool_next0) / (2.0 * e.na(P));
    if (winner == 0) ally_r += 0.5;
    if (winner == 1) enemy_r += 0.5;
#pragma unroll
    for (int j = 0; j < UPL; ++j) {
      const int a = g.gl + G * j;
      if (a >= A) continue;
      const int team = a < e.na(P) ? 0 : 1;
      lc.v.rewards[i * A + a] = team == 0 ? ally_r : enemy_r;
      double* inf = lc.v.infos + (i * A + a) * 3;
      inf[0] = e.h[a] > 0.0 ? 1.0 : 0.0;   // alive
      inf[1] = winner == team ? 1.0 : 0.0;  // battle_won
      inf[2] = winner == 2 ? 1.0 : 0.0;     // draw
      lc.v.dones[i * (A + 1) + a] = done;
    }
    if (g.gl == 0) {
      double sum = 0.0;
#pragma unroll 1
      for (int a = 0; a < A; ++a) sum += a < e.na(P) ? ally_r : enemy_r;
      ep_ret = ep_ret + sum / double(A);  // team_reward, vector_env.cpp:14-18,99
      ep_len = ep_len + 1;
      lc.v.dones[i * (A + 1) + A] = done;
      lc.v.finished[i] = done;
      lc.v.final_returns[i] = done ? ep_ret : 0.0;
      lc.v.final_lengths[i] = done ? ep_len : 0;
    }
    // prev_action <- this step's actions (smax.cpp:243)
#pragma unroll
    for (int j = 0; j < UPL; ++j)
      if (g.gl + G * j < e.nu(P)) e.pa[g.gl + G * j] = int8_t(e.act[g.gl + G * j]);
    g.sync();
  }
  stats_add(lc.stats, done && g.gl == 0, ep_len, ep_ret);

  // ---- terminal observations -> final_obs, then auto-reset (vector_env.cpp:107-119)
  const unsigned done_lanes = __ballot_sync(0xffffffffu, done && g.gl == 0);
  if (done_lanes) {
    unsigned sel = 0;
    for (int s = 0; s < EPW; ++s) sel |= ((done_lanes >> (s * G)) & 1u) << s;
    emit_obs<G, UPL>(P, e, g, done, m.tile, lc.v.final_obs, w0, wvalid, plan.rb, sel);
    if (done) {
      env_reset<G, UPL>(P, e, g, split_child_nl(carry, 1), tg, sw);
      ep_ret = 0.0;
      ep_len = 0;
      t = 0;
    }
  }
  if (live) {
    if (g.gl == 0) {
      const Key nk = split_child(carry, 2);  // vector_env.cpp:126
      lc.carry.keys[i] = make_uint4(nk.k0, nk.k1, nk.c0, nk.c1);
      lc.carry.ep_return[i] = ep_ret;
      lc.carry.ep_length[i] = ep_len;
      st.t[i] = t;
    }
    store_env<G, UPL>(P, e, st, g.gl, i, lc.n, tg, sw);
  }
  emit_obs<G, UPL>(P, e, g, live, m.tile, lc.v.obs, w0, wvalid, plan.rb, (1u << EPW) - 1u);
}

// ------------------------------------------------- non-hot helper kernels
// Env::legal_actions (smax.cpp:195-211) and state_hash (smax.cpp:312-337):
// one thread per env straight from the HBM state.
__device__ __forceinline__ int g_type(const SmaxState& st, int64_t n, int64_t i, int u) {
  return int(int8_t(st.mem[u * n + i] >> 24));
}

__device__ __forceinline__ bool g_in_range(const Params& P, const SmaxState& st, int64_t n, int64_t i, int a, int b) {
  const Thresh& r = P.ps[g_type(st, n, i, a)][g_type(st, n, i, b)].reach;
  return dist_le(st.x[a * n + i] - st.x[b * n + i], st.y[a * n + i] - st.y[b * n + i], r.r, r.r2lo, r.r2hi);
}

__global__ void smax_legal_kernel(const Params* __restrict__ gP, SmaxState st, int64_t n, int n_act, uint8_t* out) {
  __shared__ __align__(16) Params sP;
  stage_params(&sP, gP);
  const Params& P = sP;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int a = 0; a < P.A; ++a) {
    uint8_t* row = out + (size_t(i) * P.A + a) * n_act;
    for (int q = 0; q < n_act; ++q) row[q] = 0;
    row[kStop] = 1;  // dead units can only wait
    if (st.health[a * n + i] <= 0.0) continue;
    for (int q = 0; q < kStop; ++q) row[q] = 1;
    const int opp0 = a < P.na ? P.na : 0, opp_n = a < P.na ? P.ne : P.na;
    for (int k = 0; k < opp_n; ++k)
      if (st.health[(opp0 + k) * n + i] > 0.0 && g_in_range(P, st, n, i, a, opp0 + k)) row[kAttackBase + k] = 1;
  }
}

__global__ void smax_hash_kernel(const Params* __restrict__ gP, SmaxState st, int64_t n, uint64_t* out) {
  __shared__ __align__(16) Params sP;
  stage_params(&sP, gP);
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t h = 1469598103934665603ull;  // FNV-1a, smax.cpp:312-337
  auto mix = [&h](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  for (int u = 0; u < sP.n; ++u) {
    const uint32_t m = st.mem[u * n + i];
    mix(__double_as_longlong(st.x[u * n + i]));
    mix(__double_as_longlong(st.y[u * n + i]));
    mix(__double_as_longlong(st.health[u * n + i]));
    mix(__double_as_longlong(st.cooldown[u * n + i]));
    mix(uint64_t(uint8_t(m >> 24)));  // type
    mix(uint64_t(uint16_t(int16_t(int8_t(m & 0xffu)))));         // prev_action
    mix(uint64_t(uint16_t(int16_t(int8_t((m >> 8) & 0xffu)))));  // ai_target
    mix(uint64_t(uint8_t((m >> 16) & 0xffu)));                   // ai_sweep
  }
  mix(uint64_t(st.t[i]));
  mix(uint64_t(uint8_t(int8_t(-1))));  // winner of a live state
  out[i] = h;
}

// world_state (smax.cpp:272-289), one thread per env: per unit alive, x/map,
// y/map, health/max, cooldown/max, team, type one-hot, action-bucket one-hot;
// then t/max_steps.
__global__ void smax_world_state_kernel(const Params* __restrict__ gP, SmaxState st, int64_t n, float* out) {
  __shared__ __align__(16) Params sP;
  stage_params(&sP, gP);
  const Params& P = sP;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int W = 18 * P.n + 1;
  float* w = out + size_t(i) * W;
  for (int u = 0; u < P.n; ++u) {
    const int ty = g_type(st, n, i, u);
    const TypeStat& t = P.ts[ty];
    const double h = st.health[u * n + i];
    const int pa = int(st.mem[u * n + i] & 0xffu);
    const int bucket = pa <= kStop ? pa : kStop + 1;
    float* o = w + 18 * u;
    o[0] = h > 0.0 ? 1.0f : 0.0f;
    o[1] = float(st.x[u * n + i] / P.map);
    o[2] = float(st.y[u * n + i] / P.map);
    o[3] = float(h / t.hmax);
    o[4] = float(st.cooldown[u * n + i] / t.cdmax);
    o[5] = float(u < P.na ? 0 : 1);
    for (int q = 0; q < kTypes; ++q) o[6 + q] = q == ty ? 1.0f : 0.0f;
    for (int q = 0; q < 6; ++q) o[12 + q] = q == bucket ? 1.0f : 0.0f;
  }
  w[18 * P.n] = float(double(st.t[i]) / P.max_steps);
}

// ------------------------------------------------------------------ host
// Group shape for a roster of n units: lanes per env (the smallest listed G
// >= n, so few lanes idle) and units per lane.
int shape_id(const SmaxConfig& c) {
  const int n = c.na + c.ne;
  if (const char* f = std::getenv("MARL_SMAX_SHAPE")) {  // tuning override, see MARL_SMAX_SHAPES
    const int v = std::atoi(f);
    const int lanes[8] = {4, 6, 8, 10, 12, 16, 32, 32}, upl[8] = {1, 1, 1, 1, 1, 1, 1, 2};
    if (v >= 0 && v < 8 && lanes[v] * upl[v] >= n) return v;
  }
  return n <= 4 ? 0 : n <= 6 ? 1 : n <= 8 ? 2 : n <= 10 ? 3 : n <= 12 ? 4 : n <= 16 ? 5 : n <= 32 ? 6 : 7;
}

template <int G, int UPL>
Plan make_plan(const SmaxConfig& c, size_t* smem) {
  const int n = c.na + c.ne, A = c.na + (c.enemy_controlled ? c.ne : 0), D = 10 + 17 * (n - 1);
  constexpr int EPW = Grp<G>::EPW;
  int rb = int(kWarpStageBytes / (size_t(EPW) * D * 4));
  rb = rb < 1 ? 1 : rb > A ? A : rb;
  *smem = smem_bytes<G, UPL>(D, rb);
  return Plan{rb};
}

template <int G, int UPL>
void launch_reset_g(const SmaxConfig& c, const Params* dP, const SmaxState& s, const LaunchCommon& lc, Key k, Key cp) {
  size_t sm;
  Plan plan = make_plan<G, UPL>(c, &sm);
  auto fn = smax_reset_kernel<G, UPL>;
  smem_optin(fn);
  constexpr int EPB = kWarps * Grp<G>::EPW;
  fn<<<unsigned((lc.n + EPB - 1) / EPB), kThreads, sm, lc.stream>>>(dP, s, lc, k, cp, plan);
}

template <int G, int UPL>
void launch_step_g(const SmaxConfig& c, const Params* dP, const SmaxState& s, const LaunchCommon& lc, bool random,
                   Key k) {
  size_t sm;
  Plan plan = make_plan<G, UPL>(c, &sm);
  // a fixed roster of marines only (3m, 5m_vs_6m, 27m_vs_30m, ...): the type-folded instance
  bool marines = !c.random_types;
  for (int u = 0; u < c.na + c.ne && marines; ++u) marines = c.type[u] == 0;
  if (std::getenv("MARL_SMAX_GENERIC")) marines = false;
  const bool full = c.na + c.ne == G * UPL && c.na == c.ne && !c.enemy_controlled && !std::getenv("MARL_SMAX_GENERIC");
  auto pick = [&](auto ht, auto fu) {
    return random ? smax_step_kernel<G, UPL, true, decltype(ht)::value, decltype(fu)::value>
                  : smax_step_kernel<G, UPL, false, decltype(ht)::value, decltype(fu)::value>;
  };
  using Marine = std::integral_constant<int, 0>;
  using AnyType = std::integral_constant<int, -1>;
  auto fn = marines ? (full ? pick(Marine{}, std::true_type{}) : pick(Marine{}, std::false_type{}))
                    : (full ? pick(AnyType{}, std::true_type{}) : pick(AnyType{}, std::false_type{}));
  smem_optin(fn);
  constexpr int EPB = kWarps * Grp<G>::EPW;
  fn<<<unsigned((lc.end - lc.begin + EPB - 1) / EPB), kThreads, sm, lc.stream>>>(dP, s, lc, k, plan);
}

#define MARL_SMAX_SHAPES(FN, ...)           \
  switch (shape_id(c)) {                    \
    case 0: FN<4, 1>(__VA_ARGS__); break;   \
    case 1: FN<6, 1>(__VA_ARGS__); break;   \
    case 2: FN<8, 1>(__VA_ARGS__); break;   \
    case 3: FN<10, 1>(__VA_ARGS__); break;  \
    case 4: FN<12, 1>(__VA_ARGS__); break;  \
    case 5: FN<16, 1>(__VA_ARGS__); break;  \
    case 6: FN<32, 1>(__VA_ARGS__); break;  \
    default: FN<32, 2>(__VA_ARGS__); break; \
  }

}  // namespace

void smax_prepare(SmaxConfig& c) {
  Params P = make_params(c);
  Params* d = nullptr;
  cudaMalloc(&d, sizeof(Params));
  cudaMemcpy(d, &P, sizeof P, cudaMemcpyHostToDevice);
  c.dev_params = d;
  c.host_params = new Params(P);
}

void smax_release(SmaxConfig& c) {
  if (c.dev_params) cudaFree(c.dev_params);
  c.dev_params = nullptr;
  delete static_cast<Params*>(c.host_params);
  c.host_params = nullptr;
}

void smax_launch_reset(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, KeyWords key,
                       KeyWords carry_parent) {
  const Params* dP = static_cast<const Params*>(c.dev_params);
  MARL_SMAX_SHAPES(launch_reset_g, c, dP, s, lc, to_key(key), to_key(carry_parent))
  ++g_launches;
}

// smax_lane.cu: one thread per env for the small rosters (false: not covered)
bool smax_lane_launch_step(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, bool random,
                           KeyWords step_key);

void smax_launch_step(const SmaxConfig& c, const SmaxState& s, const LaunchCommon& lc, bool random,
                      KeyWords step_key) {
  if (smax_lane_launch_step(c, s, lc, random, step_key)) {
    ++g_launches;
    return;
  }
  const Params* dP = static_cast<const Params*>(c.dev_params);
  MARL_SMAX_SHAPES(launch_step_g, c, dP, s, lc, random, to_key(step_key))
  ++g_launches;
}

void smax_launch_legal(const SmaxConfig& c, const SmaxState& s, int64_t n, int n_act, uint8_t* out,
                       cudaStream_t st) {
  smax_legal_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(static_cast<const Params*>(c.dev_params), s, n,
                                                                n_act, out);
  ++g_launches;
}

void smax_launch_world_state(const SmaxConfig& c, const SmaxState& s, int64_t n, float* out, cudaStream_t st) {
  smax_world_state_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(static_cast<const Params*>(c.dev_params), s, n,
                                                                     out);
  ++g_launches;
}

void smax_launch_hash(const SmaxConfig& c, const SmaxState& s, int64_t n, uint64_t* out, cudaStream_t st) {
  smax_hash_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(static_cast<const Params*>(c.dev_params), s, n, out);
  ++g_launches;
}

}  // namespace marl_b200
