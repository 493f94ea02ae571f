// SMAX constants and per-handle parameters shared by the step kernels
// (smax.cu: lane-group kernels for any roster; smax_lane.cu: one thread per
// env for small rosters).  Reference: proj/core/src/envs/smax.cpp.
#pragma once
#include <algorithm>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {
namespace smax {

constexpr double kDt = 1.0 / 16.0;  // smax.cpp:17
constexpr int kTicks = 8;           // smax.cpp:18
constexpr double kSepTol = 1e-6;    // smax.cpp:19
constexpr int kNorth = 0, kSouth = 1, kEast = 2, kWest = 3, kStop = 4, kAttackBase = 5;
#ifndef MARL_SMAX_THREADS
#define MARL_SMAX_THREADS 256
#endif
constexpr int kThreads = MARL_SMAX_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kTypes = 6;
constexpr int kWarpStageBytes = 4 * 1024;  // observation staging budget per warp

struct TypeStat {  // per unit type (smax.cpp:26-33), derived on the host
  double hmax, dmg, cdmax, spdt, rad, hi;  // spdt = speed * dt, hi = map - radius
  Thresh sight;
  double rhmax, rcdmax, rsight;  // correctly rounded reciprocals (fdiv_f below)
};
struct PairStat {  // per (type a, type b)
  Thresh reach;  // range(a) + radius(a) + radius(b), smax.cpp:497-501
  Thresh rsum;   // radius(a) + radius(b), smax.cpp:551
  Thresh otol;   // rsum - 1e-6: the max_overlap tolerance, smax.cpp:565,576
};

// Per-handle constants, staged into shared memory by every block (~3 KB).
struct Params {
  int na, ne, n, A, controlled, max_steps, D, n_pairs;
  double map, jitter;
  double sep_r2hi;  // max rsum.r2hi over the roster's type pairs: conservative overlap pre-check
  double rmap, pad2_;
  int random_types;  // smacv2_*: per-episode random unit types and spawns (smax.cpp:169-181, 456-479)
  int pad_;
  int8_t type[kSmaxMaxUnits];
  TypeStat ts[kTypes];
  PairStat ps[kTypes][kTypes];
};
static_assert(sizeof(Params) % 16 == 0, "Params is staged with 16-byte copies");

__device__ __forceinline__ double dclamp(double v, double lo, double hi) {  // std::clamp
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

// uniform1(key, lo, hi) (prng.cpp:169-178) through the out-of-line block.
__device__ __forceinline__ double uniform_at_nl(const Key& k, double lo, double hi) {
  double v = lo + to_unit(block_at_nl(k, 0)) * (hi - lo);
  if (v >= hi) v = nextafter(hi, lo);
  return v;
}

// Is hypot(dxa, dya) < hypot(dxb, dyb)?  Decided from the squared lengths
// outside a 2e-12 relative band (both hypots are within an ulp of the true
// lengths), by the glibc-exact hypot inside it.
__device__ __forceinline__ bool hypot_less(double dxa, double dya, double d2a, double dxb, double dyb, double d2b) {
  if (d2a < d2b * (1.0 - 2e-12)) return true;
  if (d2a > d2b * (1.0 + 2e-12)) return false;
  return hypot_glibc(dxa, dya) < hypot_glibc(dxb, dyb);
}

#ifdef __CUDACC__
// float(a / b) -- the reference's fp64 quotient rounded to float -- from the
// host-rounded reciprocal r = RN(1/b): q = RN(a * r) is within ~1 ulp of the
// exact quotient, so it rounds to the same float as RN(a / b) unless it lies
// within a few ulps of a float rounding midpoint (low 29 mantissa bits near
// 0x10000000); those (probability ~2^-25) and non-finite cases take the exact
// IEEE division.  Bit-identical to float(a / b) for every input.
__device__ __noinline__ inline float fdiv_slow(double a, double b) { return float(a / b); }
__device__ __forceinline__ float fdiv_f(double a, double r, double b) {
  const double q = a * r;
  const uint32_t lo = uint32_t(__double_as_longlong(q)) & 0x1fffffffu;
  if (lo - (0x10000000u - 8u) <= 16u || !(fabs(q) < 1e300)) return fdiv_slow(a, b);
  return __double2float_rn(q);
}
// exact fp64 division kept out of line (one copy of the IEEE division sequence)
__device__ __noinline__ inline double ddiv(double a, double b) { return a / b; }

__device__ __forceinline__ void stage_params(Params* dst, const Params* __restrict__ src) {
  const int words = int(sizeof(Params) / 16);
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
#pragma unroll 1
  for (int q = threadIdx.x; q < words; q += blockDim.x) d[q] = __ldg(s + q);
  __syncthreads();
}

#endif

inline Key to_key(KeyWords k) { return Key{k.w[0], k.w[1], k.w[2], k.w[3]}; }

inline Params make_params(const SmaxConfig& c) {
  Params P{};
  P.na = c.na;
  P.ne = c.ne;
  P.n = c.na + c.ne;
  P.A = c.na + (c.enemy_controlled ? c.ne : 0);
  P.controlled = c.enemy_controlled;
  P.max_steps = c.max_steps;
  P.D = 10 + 17 * (P.n - 1);
  P.n_pairs = P.n * (P.n - 1) / 2;
  P.map = c.map;
  P.jitter = c.jitter;
  P.rmap = 1.0 / c.map;
  for (int u = 0; u < P.n; ++u) P.type[u] = c.type[u];
  P.random_types = c.random_types;
  for (int t = 0; t < kTypes; ++t) {
    const double* st = c.stats[t];  // health damage cooldown speed sight range radius
    TypeStat& T = P.ts[t];
    T.hmax = st[0];
    T.dmg = st[1];
    T.cdmax = st[2];
    T.spdt = st[3] * kDt;  // st.speed * kDt, smax.cpp:514
    T.rad = st[6];
    T.hi = c.map - st[6];  // map_ - radius, smax.cpp:515
    T.sight = make_thresh(st[4]);
    T.rhmax = 1.0 / st[0];
    T.rcdmax = 1.0 / st[2];
    T.rsight = 1.0 / st[4];
  }
  for (int a = 0; a < kTypes; ++a)
    for (int b = 0; b < kTypes; ++b) {
      PairStat& S = P.ps[a][b];
      S.reach = make_thresh(c.stats[a][5] + c.stats[a][6] + c.stats[b][6]);
      const double sum = c.stats[a][6] + c.stats[b][6];
      S.rsum = make_thresh(sum);
      S.otol = make_thresh(sum - kSepTol);
    }
  P.sep_r2hi = 0.0;
  for (int a = 0; a < P.n; ++a)
    for (int b = 0; b < P.n; ++b) P.sep_r2hi = std::max(P.sep_r2hi, P.ps[P.type[a]][P.type[b]].rsum.r2hi);
  if (c.random_types)  // any type pair can meet
    for (int ta = 0; ta < kTypes; ++ta)
      for (int tb = 0; tb < kTypes; ++tb) P.sep_r2hi = std::max(P.sep_r2hi, P.ps[ta][tb].rsum.r2hi);
  return P;
}


}  // namespace smax
}  // namespace marl_b200
