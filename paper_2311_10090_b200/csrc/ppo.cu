// PPO minibatch update on the device: the
// reference's train_ppo_impl inner loop (proj/core/src/algo/ppo.cpp:588-628)
// over the rollout buffer that rollout.cu fills.  Per update epoch:
//
//   permutation   : prng::permutation(perm_key, T*R) (prng.cpp:151-159), the
//                   exact Fisher-Yates result computed in parallel (below).
// Per minibatch (ff_minibatch, ppo.cpp:409-441):
//   adv stats     : normalize_advantages' weighted mean / std over the
//                   minibatch rows (actor_critic.hpp:416-433), double.
//   branch kernel : per 128-row... tile of gathered rows, one CTA runs
//                   ff_forward with cache (actor_critic.hpp:49-52), the
//                   per-row part of ppo_row_loss (actor_critic.hpp:340-412),
//                   ff_backward (actor_critic.hpp:55-61, nn.hpp:119-128,
//                   180-197) and accumulates the weight gradients of its rows;
//                   actor and critic are separate launches (their losses
//                   only meet in the scalar metrics).
//   reduce        : per-CTA gradient partials -> the flat gradient in
//                   nn::pack order (nn.hpp:326-341), fixed CTA order.
//   clip + Adam   : clip_global_norm then adam_update (nn.hpp:417-452) with
//                   the reference's float evaluation order (-fmad=false), and
//                   the DivergenceError checks as a sticky device flag.
//
// Accuracy contract vs the reference: the permutation, row gather and the
// elementwise optimizer math are exact; the gradient sums are reassociated
// (the reference sums rows sequentially in float), so gradients agree to
// float-accumulation tolerance.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {

namespace {

// ------------------------------------------------------------ permutation
// Fisher-Yates (prng.cpp:151-159): for i = n-1 .. 1, swap(out[i], out[j_i])
// with j_i = bits(key, i) % (i+1).  Position i is final after step i, and
// receives the value sitting at position j_i just before step i.  Position
// q is written only by steps k with j_k = q (all k >= q), so with
//   next(i) = the smallest k > i with j_k = j_i          (same group, next)
//   first(q) = the smallest k > q with j_k = q
//   F(k)    = value at position k before step k = first(k) ? F(first(k)) : k
// the result is out[i] = next(i) ? F(next(i)) : j_i, and out[0] = F(0).
// Groups come from one stable radix sort of (j_k, k); chains are short
// (expected O(log n)).
__global__ void perm_draw_kernel(Key key, int64_t n, uint32_t* __restrict__ j, uint32_t* __restrict__ jk,
                                 uint32_t* __restrict__ kv) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t ji = i == 0 ? 0u : uint32_t(block_at(key, uint64_t(i)) % uint64_t(i + 1));
  j[i] = ji;
  if (i > 0) {  // step 0 does not exist
    jk[i - 1] = ji;
    kv[i - 1] = uint32_t(i);
  }
}

__global__ void perm_link_kernel(int64_t m, const uint32_t* __restrict__ ks, const uint32_t* __restrict__ vs,
                                 int32_t* __restrict__ nxt, int32_t* __restrict__ fst) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= m) return;
  const uint32_t q = ks[p], k = vs[p];
  const bool has_next = p + 1 < m && ks[p + 1] == q;
  const int32_t nx = has_next ? int32_t(vs[p + 1]) : -1;
  nxt[k] = nx;
  if (p == 0 || ks[p - 1] != q) fst[q] = (k != q) ? int32_t(k) : nx;
}

__global__ void perm_resolve_kernel(int64_t n, const uint32_t* __restrict__ j, const int32_t* __restrict__ nxt,
                                    const int32_t* __restrict__ fst, int32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t v;
  if (i == 0) {
    v = 0;
  } else {
    v = nxt[i];
    if (v < 0) {
      out[i] = int32_t(j[i]);
      return;
    }
  }
  // chains climb strictly (first(k) > k), so at most n hops; the bound only
  // guards against a corrupted table
  int64_t hops = 0;
  for (int32_t f = fst[v]; f > v && hops < n; f = fst[v], ++hops) v = f;
  out[i] = v;
}

// ------------------------------------------------------- advantage stats
constexpr int kRedThreads = 256;

// Deterministic block sum of one double per thread (fixed tree).
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < nw; ++q) s += sh[q];
  return s;  // valid on thread 0
}

// pass 1: sum(w * adv), sum(w) over the minibatch rows (actor_critic.hpp:418-421)
// adv / active of slot r at [r * stride] (stride 1: the rollout buffer; 8: the
// tcgen05 step's packed 32-byte records, one sector per row)
__global__ void adv_sum_kernel(const float* __restrict__ adv, const float* __restrict__ active, int stride,
                               const int32_t* __restrict__ idx, int64_t M, double* __restrict__ part,
                               float2* __restrict__ gath) {
  __shared__ double sh[32];
  double s = 0.0, n = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < M; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = int64_t(idx[i]) * stride;
    const float a = adv[r], w32 = active[r];
    if (gath) gath[i] = make_float2(a, w32);  // the variance pass reads these contiguously
    const double w = double(w32);
    s += w * double(a);
    n += w;
  }
  s = block_sum(s, sh);
  n = block_sum(n, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = n;
  }
}

// fold the per-block partials (fixed order: thread t takes blocks t, t+256, ...,
// then a fixed tree): g[0] = sum(w * adv), g[1] = sum(w)
constexpr int kFoldThreads = 256;
__global__ void __launch_bounds__(kFoldThreads) adv_fold_kernel(const double* __restrict__ part, int nb,
                                                                double* __restrict__ g) {
  __shared__ double sh[32];
  double s = 0.0, c = 0.0;
  for (int q = threadIdx.x; q < nb; q += kFoldThreads) {
    s += part[2 * q];
    c += part[2 * q + 1];
  }
  s = block_sum(s, sh);
  c = block_sum(c, sh);
  if (threadIdx.x == 0) {
    g[0] = s;
    g[1] = c;
  }
}

// pass 2: sum(w * (adv - mean)^2) (actor_critic.hpp:424-429) with the
// (all-reduced) mean of g
__global__ void adv_var_kernel(const float* __restrict__ adv, const float* __restrict__ active, int stride,
                               const int32_t* __restrict__ idx, int64_t M, const double* __restrict__ g,
                               double* __restrict__ part2, const float2* __restrict__ gath) {
  __shared__ double sh[32];
  const double mean = g[1] > 0.0 ? g[0] / g[1] : 0.0;
  double v = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < M; i += int64_t(gridDim.x) * blockDim.x) {
    float a, w;
    if (gath) {
      const float2 q = gath[i];
      a = q.x, w = q.y;
    } else {
      const int64_t r = int64_t(idx[i]) * stride;
      a = adv[r], w = active[r];
    }
    const double d = double(a) - mean;
    v += double(w) * d * d;
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part2[blockIdx.x] = v;
}

__global__ void __launch_bounds__(kFoldThreads) adv_fold2_kernel(const double* __restrict__ part2, int nb,
                                                                 double* __restrict__ g) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int q = threadIdx.x; q < nb; q += kFoldThreads) v += part2[q];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) g[2] = v;
}

__global__ void adv_final_kernel(const double* __restrict__ g, PpoMbStats* st) {
  if (threadIdx.x != 0) return;
  const double n = g[1];
  st->total_w = n;
  st->normalize = n > 0.0 ? 1 : 0;  // n <= 0: advantages left as they are
  st->mean = n > 0.0 ? g[0] / n : 0.0;
  st->std = n > 0.0 ? sqrt(g[2] / n) : 0.0;
}

// global minibatch slots (t*R_g + r_g) -> this shard's local slots (t*R_l + r_g - row0) or -1
__global__ void shard_map_kernel(const int32_t* __restrict__ idx, int64_t M, int64_t Rg, int64_t row0, int64_t Rl,
                                 int32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const int64_t s = idx[i], t = s / Rg, r = s - t * Rg - row0;
  out[i] = (r >= 0 && r < Rl) ? int32_t(t * Rl + r) : -1;
}

struct NonNegative {
  __device__ __forceinline__ bool operator()(const int32_t x) const { return x >= 0; }
};

// sum the per-CTA loss statistics into row 0 (the sharded path all-reduces that row)
// Column `col` of n per-CTA stat rows summed by one warp: lane-strided, then a
// fixed shuffle tree (valid on lane 0).  clip_adam_kernel folds with the same
// order, so folding first (the data-parallel path) changes nothing at one rank.
__device__ __forceinline__ double warp_fold_col(const double* __restrict__ src, int n, int col) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int c = lane; c < n; c += 32) v += src[size_t(c) * 6 + col];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void stats_fold_kernel(double* __restrict__ sp, int nparts) {
  const int k = threadIdx.x >> 5;  // warp k owns column k
  if (k >= 6) return;
  const double v = warp_fold_col(sp, nparts, k);
  if ((threadIdx.x & 31) == 0) sp[k] = v;
}

// ----------------------------------------------------------- branch kernel
constexpr int kThreads = 256;
constexpr int kStats = 6;  // pg, v_term, entropy, kl, clipped, (spare)

__device__ __forceinline__ float act_fwd(float v, int relu) { return relu ? (v > 0.0f ? v : 0.0f) : tanhf(v); }
// act_grad_from_output (nn.hpp:141-144), applied as grad *= g(y) (nn.hpp:187-188)
__device__ __forceinline__ float act_bwd(float grad, float y, int relu) {
  return __fmul_rn(grad, relu ? (y > 0.0f ? 1.0f : 0.0f) : __fsub_rn(1.0f, __fmul_rn(y, y)));
}

struct Smem {
  const float *w1, *b1, *w2, *b2, *w3, *b3;
  float *x, *h1, *h2, *d1, *d2, *dl;
  int32_t* slot;
  int ldx, ldw, ldo;
};

// One minibatch branch (actor when ACTOR, else critic).  Thread t of the CTA
// serves tile row r = t % TR in the row phases (QP = 256/TR threads share a
// row, splitting its output columns), and owns gradient entries t, t+256, ...
// of the branch in the accumulation phase.  E > 0: those entries accumulate
// in registers (P <= 256*E); E == 0: in the CTA's own partial row in global
// memory (wide inputs: Overcooked, SMAX 27m).
template <bool ACTOR, int E>
__global__ void __launch_bounds__(kThreads) ppo_branch_kernel(PpoBranchArgs a) {
  extern __shared__ __align__(16) float sm[];
  __shared__ double s_stats[kThreads / 32][kStats];
  const int in = a.in, W = a.W, NO = a.out, TR = a.TR, QP = kThreads / TR;
  const int P = W * in + W + W * W + W + NO * W + NO;
  const int t = threadIdx.x, r = t % TR, q = t / TR;
  Smem s;
  float* base = sm;
  if (a.staged) {
    for (int e = t; e < P; e += kThreads) base[e] = __ldg(a.params + e);
    s.w1 = base;
    base += P;
  } else {
    s.w1 = a.params;
  }
  s.b1 = s.w1 + W * in;
  s.w2 = s.b1 + W;
  s.b2 = s.w2 + W * W;
  s.w3 = s.b2 + W;
  s.b3 = s.w3 + NO * W;
  s.ldx = in | 1;
  s.ldw = W | 1;
  s.ldo = NO | 1;
  s.x = base;
  s.h1 = s.x + TR * s.ldx;
  s.h2 = s.h1 + TR * s.ldw;
  s.d1 = s.h2 + TR * s.ldw;
  s.d2 = s.d1 + TR * s.ldw;
  s.dl = s.d2 + TR * s.ldw;
  s.slot = reinterpret_cast<int32_t*>(s.dl + TR * s.ldo);

  const PpoMbStats st = *a.st;
  const double total_w = st.total_w;
  float acc[E > 0 ? E : 1];
#pragma unroll
  for (int k = 0; k < (E > 0 ? E : 1); ++k) acc[k] = 0.0f;
  float* gp = a.gpart + size_t(blockIdx.x) * size_t(P);
  if (E == 0)
    for (int e = t; e < P; e += kThreads) gp[e] = 0.0f;
  double pg = 0.0, vt = 0.0, ent = 0.0, kl = 0.0, clipn = 0.0;

  const int64_t ntiles = (a.M + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * TR;
    const int nv = int(min(int64_t(TR), a.M - i0));
    __syncthreads();  // the previous tile's smem is consumed
    if (t < nv) s.slot[t] = a.idx[i0 + t];
    __syncthreads();
    // gather the tile's input rows (ff_minibatch's memcpy, ppo.cpp:413-420)
    for (int e = t; e < nv * in; e += kThreads) {
      const int rr = e / in, i = e - rr * in;
      s.x[rr * s.ldx + i] = __ldg(a.x + size_t(s.slot[rr]) * size_t(in) + i);
    }
    __syncthreads();
    const bool live = r < nv;
    // torso layer 1 and 2 (dense_forward + act_inplace, nn.hpp:108-115, 136-138)
    if (live)
      for (int o = q; o < W; o += QP) {
        const float* xr = s.x + r * s.ldx;
        const float* wr = s.w1 + o * in;
        float acc1 = 0.0f;
        for (int i = 0; i < in; ++i) acc1 = __fadd_rn(acc1, __fmul_rn(xr[i], wr[i]));
        s.h1[r * s.ldw + o] = act_fwd(__fadd_rn(acc1, s.b1[o]), a.relu);
      }
    __syncthreads();
    if (live)
      for (int o = q; o < W; o += QP) {
        const float* xr = s.h1 + r * s.ldw;
        const float* wr = s.w2 + o * W;
        float acc2 = 0.0f;
        for (int i = 0; i < W; ++i) acc2 = __fadd_rn(acc2, __fmul_rn(xr[i], wr[i]));
        s.h2[r * s.ldw + o] = act_fwd(__fadd_rn(acc2, s.b2[o]), a.relu);
      }
    __syncthreads();
    // linear head
    if (live)
      for (int o = q; o < NO; o += QP) {
        const float* xr = s.h2 + r * s.ldw;
        const float* wr = s.w3 + o * W;
        float acc3 = 0.0f;
        for (int i = 0; i < W; ++i) acc3 = __fadd_rn(acc3, __fmul_rn(xr[i], wr[i]));
        s.dl[r * s.ldo + o] = __fadd_rn(acc3, s.b3[o]);
      }
    __syncthreads();
    // the row's part of ppo_row_loss (actor_critic.hpp:360-402): dy of the head
    if (live && q == 0) {
      const int64_t sl = s.slot[r];
      float* dl = s.dl + r * s.ldo;
      const double w = double(a.active[sl]);
      if (w == 0.0 || total_w <= 0.0) {
        for (int o = 0; o < NO; ++o) dl[o] = 0.0f;
      } else if (ACTOR) {
        const uint8_t* legal = a.legal + size_t(sl) * size_t(NO);
        double lp[kPpoMaxAct];
        double mx = -INFINITY;
        for (int i = 0; i < NO; ++i)
          if (legal[i]) mx = fmax(mx, double(dl[i]));
        double denom = 0.0;
        for (int i = 0; i < NO; ++i)
          if (legal[i]) denom += exp(double(dl[i]) - mx);
        const double log_denom = log(denom);
        for (int i = 0; i < NO; ++i) lp[i] = legal[i] ? double(dl[i]) - mx - log_denom : -1e30;
        const int act = a.actions[sl];
        if (act < 0 || act >= NO || !legal[act] || !(mx > -INFINITY)) atomicExch(a.err, 1);
        const int ac = act < 0 ? 0 : (act >= NO ? NO - 1 : act);
        // normalize_advantages writes T((adv - mean) / (std + 1e-8)) (actor_critic.hpp:430-432)
        float advf = a.adv[sl];
        if (st.normalize) advf = float((double(advf) - st.mean) / (st.std + 1e-8));
        const double adv = double(advf);
        const double ratio = exp(lp[ac] - double(a.old_logp[sl]));
        const double unclipped = ratio * adv;
        const double rho_c = fmin(fmax(ratio, 1.0 - a.clip_eps), 1.0 + a.clip_eps);
        const double clipped = rho_c * adv;
        const double surr = fmin(unclipped, clipped);
        const double dsurr = unclipped <= clipped ? ratio * adv : 0.0;
        double entropy = 0.0;
        for (int i = 0; i < NO; ++i)
          if (legal[i]) entropy -= exp(lp[i]) * lp[i];
        for (int i = 0; i < NO; ++i) {
          if (!legal[i]) {
            dl[i] = 0.0f;
            continue;
          }
          const double pi = exp(lp[i]);
          const double dlogp = (i == ac ? 1.0 : 0.0) - pi;
          const double dH = -pi * (lp[i] + entropy);
          const double g = -dsurr * dlogp - a.ent_coef * dH;
          dl[i] = float(w / total_w * g);
        }
        pg += w * -surr;
        ent += w * entropy;
        kl += w * (ratio - 1.0 - log(ratio));
        clipn += w * (fabs(ratio - 1.0) > a.clip_eps ? 1.0 : 0.0);
      } else {
        const double v = double(dl[0]);
        const double targ = double(a.vtarg[sl]);
        const double v_old = double(a.old_value[sl]);
        const double v_clip = v_old + fmin(fmax(v - v_old, -a.clip_eps), a.clip_eps);
        const double sq = (v - targ) * (v - targ), sq_c = (v_clip - targ) * (v_clip - targ);
        vt += w * (0.5 * fmax(sq, sq_c));
        dl[0] = float(w / total_w * a.vf_coef * (sq >= sq_c ? (v - targ) : 0.0));
      }
    }
    __syncthreads();
    // ff_backward: head dx (matmul_nn, zero dy skipped, nn.hpp:74-88), act grad
    if (live)
      for (int i = q; i < W; i += QP) {
        float g = 0.0f;
        for (int o = 0; o < NO; ++o) {
          const float gv = s.dl[r * s.ldo + o];
          if (gv != 0.0f) g = __fadd_rn(g, __fmul_rn(gv, s.w3[o * W + i]));
        }
        s.d2[r * s.ldw + i] = act_bwd(g, s.h2[r * s.ldw + i], a.relu);
      }
    __syncthreads();
    if (live)
      for (int i = q; i < W; i += QP) {
        float g = 0.0f;
        for (int o = 0; o < W; ++o) {
          const float gv = s.d2[r * s.ldw + o];
          if (gv != 0.0f) g = __fadd_rn(g, __fmul_rn(gv, s.w2[o * W + i]));
        }
        s.d1[r * s.ldw + i] = act_bwd(g, s.h1[r * s.ldw + i], a.relu);
      }
    __syncthreads();
    // weight gradients of the tile: g.w = dy^T x, g.b = sum dy (nn.hpp:124-126)
    const int ob1 = W * in, ow2 = ob1 + W, ob2 = ow2 + W * W, ow3 = ob2 + W, ob3 = ow3 + NO * W;
    auto entry = [&](int e) {
      const float* dy;
      const float* xx = nullptr;
      int ldd, ldx_ = 0, o, i = -1;
      if (e < ob1) {
        o = e / in, i = e - o * in, dy = s.d1, ldd = s.ldw, xx = s.x, ldx_ = s.ldx;
      } else if (e < ow2) {
        o = e - ob1, dy = s.d1, ldd = s.ldw;
      } else if (e < ob2) {
        o = (e - ow2) / W, i = (e - ow2) - o * W, dy = s.d2, ldd = s.ldw, xx = s.h1, ldx_ = s.ldw;
      } else if (e < ow3) {
        o = e - ob2, dy = s.d2, ldd = s.ldw;
      } else if (e < ob3) {
        o = (e - ow3) / W, i = (e - ow3) - o * W, dy = s.dl, ldd = s.ldo, xx = s.h2, ldx_ = s.ldw;
      } else {
        o = e - ob3, dy = s.dl, ldd = s.ldo;
      }
      float sum = 0.0f;
      if (i >= 0) {
        for (int rr = 0; rr < nv; ++rr) sum = __fadd_rn(sum, __fmul_rn(dy[rr * ldd + o], xx[rr * ldx_ + i]));
      } else {
        for (int rr = 0; rr < nv; ++rr) sum = __fadd_rn(sum, dy[rr * ldd + o]);
      }
      return sum;
    };
    if constexpr (E > 0) {
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int e = t + k * kThreads;
        if (e < P) acc[k] = __fadd_rn(acc[k], entry(e));
      }
    } else {
      for (int e = t; e < P; e += kThreads) gp[e] = __fadd_rn(gp[e], entry(e));
    }
  }
  if constexpr (E > 0) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int e = t + k * kThreads;
      if (e < P) gp[e] = acc[k];
    }
  }
  // per-CTA loss statistics in a fixed order
  double v5[kStats] = {pg, vt, ent, kl, clipn, 0.0};
  for (int c = 0; c < kStats; ++c) {
    double v = v5[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) s_stats[t >> 5][c] = v;
  }
  __syncthreads();
  if (t < kStats) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += s_stats[w][t];
    a.spart[size_t(blockIdx.x) * kStats + t] = v;
  }
}

// ------------------------------------------------- register-tiled branch
// The C5 shape (in <= 32, width 64, <= 16 outputs): every layer of the tile is
// a 64-row GEMM computed as 4x4 register micro-tiles with FMA, operands read
// as float4 from shared memory.  Each activation is kept in both layouts --
// feature-major ([k][row], the A operand of the forward / input-gradient
// GEMMs) and row-major ([row][k], the operands of the weight-gradient GEMMs
// dW = dY^T X) -- so every inner-loop load is one LDS.128 feeding 16 FMAs.
// Weight gradients accumulate in registers across the CTA's tiles.  Padded
// rows / inputs / outputs are zero, so they add exact zeros.
constexpr int kTR = 64;   // rows per tile
constexpr int kTW = 64;   // torso width
constexpr int kTIn = 32;  // padded input width
constexpr int kLD = 68;   // padded leading dim of the 64-wide arrays (float4-aligned, bank-shifted)
constexpr int kLDX = 36;  // padded leading dim of x[row][k]

template <int NOP>
struct TiledSmem {
  float x[2][kTR][kLDX], xt[2][kTIn][kLD];  // double-buffered input tile (cp.async gather)
  float h1[kTR][kLD], h1t[kTW][kLD], h2[kTR][kLD], h2t[kTW][kLD];
  float dz2[kTR][kLD], dz2t[kTW][kLD], dz1[kTR][kLD];
  float dl[kTR][NOP + 4], dlt[NOP][kLD];
  float w1t[kTIn][kTW], w2t[kTW][kTW], w2[kTW][kTW], w3[NOP][kTW], w3t[kTW][NOP];
  float b1[kTW], b2[kTW], b3[NOP];
  float bred[4][kTW + 16];  // bias-gradient partials (4 row quarters)
  int32_t slot[3][kTR];     // slots of tiles it, it+1 (gather in flight), it+2 (loading)
  // per-row loss inputs, gathered with the tile: active, (adv | vtarg), (old logp | old value), action, legal words
  float r_active[2][kTR], r_a[2][kTR], r_b[2][kTR];
  int32_t r_act[2][kTR];
  uint32_t r_legal[2][kTR][5];
};

__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(sdst))),
               "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// per-row inputs of the loss, loaded ahead of the tile's forward GEMMs
struct RowIn {
  float active, adv, logp, vtarg, value;
  int action;
  int legal;
};

// c[i][j] += A[k*lda + i] * B[k*ldb + j] over k < K  (MI x NJ register tile)
template <int MI, int NJ>
__device__ __forceinline__ void mm(const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb, int K,
                                   float (&c)[4][4]) {
#pragma unroll 8
  for (int k = 0; k < K; ++k) {
    float av[4], bv[4];
    if (MI == 4) {
      const float4 v = *reinterpret_cast<const float4*>(A + k * lda);
      av[0] = v.x, av[1] = v.y, av[2] = v.z, av[3] = v.w;
    } else {
      av[0] = A[k * lda];
    }
    if (NJ == 4) {
      const float4 v = *reinterpret_cast<const float4*>(B + k * ldb);
      bv[0] = v.x, bv[1] = v.y, bv[2] = v.z, bv[3] = v.w;
    } else {
      bv[0] = B[k * ldb];
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) c[i][j] = fmaf(av[i], bv[j], c[i][j]);
  }
}

__device__ __forceinline__ void zero44(float (&c)[4][4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0f;
}

// store a 4x4 block (rows r0.., cols c0..) row-major and/or feature-major
template <int LDR, int LDT>
__device__ __forceinline__ void put44(float (*rm)[LDR], float (*fm)[LDT], int r0, int c0, const float (&c)[4][4]) {
  if (rm)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(&rm[r0 + i][c0]) = make_float4(c[i][0], c[i][1], c[i][2], c[i][3]);
  if (fm)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(&fm[c0 + j][r0]) = make_float4(c[0][j], c[1][j], c[2][j], c[3][j]);
}

// d(-surr - ent_coef*H)/dz for one actor row, NOP lanes of a warp segment per
// row, lane j = action j (actor_critic.hpp:360-392 in double; the softmax
// sums are tree-reduced over the segment).  Returns the lane's dz.
template <int NOP>
__device__ __forceinline__ float actor_row_grad(const PpoBranchArgs& a, const PpoMbStats& st, double total_w,
                                                const RowIn& ri, bool row_ok, float z, int j, double* pg, double* ent,
                                                double* kl, double* clipn) {
  const int NO = a.out;
  const unsigned full = 0xffffffffu;
  // every lane of the warp runs the shuffles; rows without weight are masked at the end
  const double w = row_ok ? double(ri.active) : 0.0;
  const bool on = w != 0.0 && total_w > 0.0;
  const bool lg = on && j < NO && ri.legal;
  double mx = lg ? double(z) : -INFINITY;
#pragma unroll
  for (int o = NOP / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(full, mx, o, NOP));
  const double e = lg ? exp(double(z) - mx) : 0.0;
  double denom = e;
#pragma unroll
  for (int o = NOP / 2; o > 0; o >>= 1) denom += __shfl_xor_sync(full, denom, o, NOP);
  const double lp = lg ? double(z) - mx - log(denom) : -1e30;
  const int act = on ? ri.action : 0;
  if (on && j == 0 && (act < 0 || act >= NO || !(mx > -INFINITY))) atomicExch(a.err, 1);
  const int ac = act < 0 ? 0 : (act >= NO ? NO - 1 : act);
  const double lp_a = __shfl_sync(full, lp, ac, NOP);
  const int lg_a = __shfl_sync(full, int(lg), ac, NOP);
  if (on && j == 0 && !lg_a) atomicExch(a.err, 1);
  const double pi = lg ? exp(lp) : 0.0;
  double h = lg ? -pi * lp : 0.0;
#pragma unroll
  for (int o = NOP / 2; o > 0; o >>= 1) h += __shfl_xor_sync(full, h, o, NOP);
  if (!on) return 0.0f;
  float advf = ri.adv;
  if (st.normalize) advf = float((double(advf) - st.mean) / (st.std + 1e-8));
  const double adv = double(advf);
  const double ratio = exp(lp_a - double(ri.logp));
  const double unclipped = ratio * adv;
  const double rho_c = fmin(fmax(ratio, 1.0 - a.clip_eps), 1.0 + a.clip_eps);
  const double clipped = rho_c * adv;
  const double dsurr = unclipped <= clipped ? ratio * adv : 0.0;
  if (j == 0) {
    *pg += w * -fmin(unclipped, clipped);
    *ent += w * h;
    *kl += w * (ratio - 1.0 - log(ratio));
    *clipn += w * (fabs(ratio - 1.0) > a.clip_eps ? 1.0 : 0.0);
  }
  if (!lg) return 0.0f;
  const double dlogp = (j == ac ? 1.0 : 0.0) - pi;
  const double dH = -pi * (lp + h);
  return float(w / total_w * (-dsurr * dlogp - a.ent_coef * dH));
}

template <bool ACTOR, int NOP>
__global__ void __launch_bounds__(kThreads, 1) ppo_branch_tiled_kernel(PpoBranchArgs a) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  TiledSmem<NOP>& s = *reinterpret_cast<TiledSmem<NOP>*>(sm_raw);
  __shared__ double s_stats[kThreads / 32][kStats];
  const int in = a.in, NO = a.out, t = threadIdx.x;
  const float* p = a.params;
  const float *W1 = p, *B1 = W1 + kTW * in, *W2 = B1 + kTW, *B2 = W2 + kTW * kTW, *W3 = B2 + kTW,
              *B3 = W3 + NO * kTW;
  // stage the branch: W1^T (zero-padded to 32 inputs), W2 and W2^T, W3 and W3^T (zero rows)
  for (int e = t; e < kTIn * kTW; e += kThreads) {
    const int k = e / kTW, o = e % kTW;
    s.w1t[k][o] = k < in ? __ldg(W1 + o * in + k) : 0.0f;
  }
  for (int e = t; e < kTW * kTW; e += kThreads) {
    const int o = e / kTW, i = e % kTW;
    const float w = __ldg(W2 + e);
    s.w2[o][i] = w;
    s.w2t[i][o] = w;
  }
  for (int e = t; e < NOP * kTW; e += kThreads) {
    const int o = e / kTW, i = e % kTW;
    const float w = o < NO ? __ldg(W3 + o * kTW + i) : 0.0f;
    s.w3[o][i] = w;
    s.w3t[i][o] = w;
  }
  if (t < kTW) {
    s.b1[t] = __ldg(B1 + t);
    s.b2[t] = __ldg(B2 + t);
  }
  if (t < NOP) s.b3[t] = t < NO ? __ldg(B3 + t) : 0.0f;

  const PpoMbStats st = *a.st;
  const double total_w = st.total_w;
  // persistent gradient accumulators: gW2 tile (every thread), gW1 tile
  // (threads 128..255), gW3 tile (threads 0..NOP*16/4-1, 1x4), bias partials
  float g2[4][4], g1[4][4], g3[4][4];
  zero44(g2);
  zero44(g1);
  zero44(g3);
  float gb1 = 0.0f, gb2 = 0.0f, gb3 = 0.0f;
  double pg = 0.0, vt = 0.0, ent = 0.0, kl = 0.0, clipn = 0.0;
  const int rg = t % 16, cg = t / 16;  // 64x64 GEMMs: rows/outs 4*rg.., cols 4*cg..
  const int bo = t % kTW, bq = t / kTW;  // bias sums: output bo over rows 16*bq..

  const int64_t ntiles = (a.M + kTR - 1) / kTR;
  const int64_t G = gridDim.x;
  auto slot_load = [&](int64_t tile, int sb) {
    if (t < kTR) {
      const int64_t i = tile * kTR + t;
      s.slot[sb][t] = (tile < ntiles && i < a.M) ? a.idx[i] : -1;
    }
  };
  // gather of a tile's input rows (ff_minibatch's memcpy, ppo.cpp:413-420) into
  // buffer xb, row-major and feature-major, zero-filled padding, asynchronous
  auto gather = [&](int xb, int sb) {
    for (int e = t; e < kTR * kTIn; e += kThreads) {
      const int r = e / kTIn, k = e % kTIn;
      const int sl = s.slot[sb][r];
      const bool ok = sl >= 0 && k < in;
      const float* src = ok ? a.x + size_t(sl) * size_t(in) + k : a.x;
      cp_async4(&s.x[xb][r][k], src, ok ? 4 : 0);
      cp_async4(&s.xt[xb][k][r], src, ok ? 4 : 0);
    }
    if (t < kTR) {
      const int sl = s.slot[sb][t];
      const int n = sl >= 0 ? 4 : 0;
      const int64_t q = sl >= 0 ? sl : 0;
      cp_async4(&s.r_active[xb][t], a.active + q, n);
      cp_async4(&s.r_a[xb][t], (ACTOR ? a.adv : a.vtarg) + q, n);
      cp_async4(&s.r_b[xb][t], (ACTOR ? a.old_logp : a.old_value) + q, n);
      if (ACTOR) {
        cp_async4(&s.r_act[xb][t], a.actions + q, n);
        const int64_t base = q * NO, w0 = base & ~int64_t(3);
        const int nw = int(((base & 3) + NO + 3) / 4);
#pragma unroll
        for (int w = 0; w < 5; ++w) cp_async4(&s.r_legal[xb][t][w], a.legal + w0 + 4 * w, (n && w < nw) ? 4 : 0);
      }
    }
    cp_async_commit();
  };
  slot_load(blockIdx.x, 0);
  slot_load(blockIdx.x + G, 1);
  __syncthreads();
  gather(0, 0);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++it) {
    const int xb = it & 1, sb = it % 3;
    __syncthreads();  // the previous tile is consumed: its x buffer and slot buffer are free
    gather(xb ^ 1, (it + 1) % 3);  // tile + G (an empty group past the end)
    slot_load(tile + 2 * G, (it + 2) % 3);
    constexpr int kRows = ACTOR ? (kTR * NOP + kThreads - 1) / kThreads : 1;
    cp_async_wait<1>();  // this tile's gather has landed
    __syncthreads();
    const auto& X = s.x[xb];
    const auto& XT = s.xt[xb];
    // this thread's loss rows (staged with the tile)
    RowIn ri[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
      const int r = ACTOR ? t / NOP + q * (kThreads / NOP) : t;
      ri[q] = RowIn{0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0, 0};
      if (r < kTR && s.slot[sb][r] >= 0) {
        ri[q].active = s.r_active[xb][r];
        if (ACTOR) {
          ri[q].adv = s.r_a[xb][r];
          ri[q].logp = s.r_b[xb][r];
          ri[q].action = s.r_act[xb][r];
          const int j = t % NOP;
          if (j < NO) {
            const int b = int((int64_t(s.slot[sb][r]) * NO) & 3) + j;
            ri[q].legal = (s.r_legal[xb][r][b >> 2] >> (8 * (b & 3))) & 0xffu;
          }
        } else {
          ri[q].vtarg = s.r_a[xb][r];
          ri[q].value = s.r_b[xb][r];
        }
      }
    }
    float c[4][4];
    // F1: h1 = act(x W1^T + b1)
    zero44(c);
    mm<4, 4>(&XT[0][4 * rg], kLD, &s.w1t[0][4 * cg], kTW, kTIn, c);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[i][j] = act_fwd(c[i][j] + s.b1[4 * cg + j], a.relu);
    put44<kLD, kLD>(s.h1, s.h1t, 4 * rg, 4 * cg, c);
    __syncthreads();
    // F2: h2 = act(h1 W2^T + b2)
    zero44(c);
    mm<4, 4>(&s.h1t[0][4 * rg], kLD, &s.w2t[0][4 * cg], kTW, kTW, c);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[i][j] = act_fwd(c[i][j] + s.b2[4 * cg + j], a.relu);
    put44<kLD, kLD>(s.h2, s.h2t, 4 * rg, 4 * cg, c);
    __syncthreads();
    // F3: head -> dl (row-major): 4 rows x 1 output per thread
    if (t < 16 * NOP) {
      const int o = t / 16;
      zero44(c);
      mm<4, 1>(&s.h2t[0][4 * rg], kLD, &s.w3t[0][o], NOP, kTW, c);
#pragma unroll
      for (int i = 0; i < 4; ++i) s.dl[4 * rg + i][o] = c[i][0] + s.b3[o];
    }
    __syncthreads();
    // the row's part of ppo_row_loss (actor_critic.hpp:360-402)
    if (ACTOR) {
      constexpr int kSlots = kThreads / NOP;
      const int j = t % NOP;
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        const int r = t / NOP + q * kSlots;
        if (r < kTR) {  // uniform per warp
          const float g = actor_row_grad<NOP>(a, st, total_w, ri[q], s.slot[sb][r] >= 0, s.dl[r][j], j, &pg, &ent,
                                              &kl, &clipn);
          s.dl[r][j] = g;
          s.dlt[j][r] = g;
        }
      }
    } else if (t < kTR) {
      const int r = t;
      const double w = s.slot[sb][r] >= 0 ? double(ri[0].active) : 0.0;
      float g = 0.0f;
      if (w != 0.0 && total_w > 0.0) {
        const double v = double(s.dl[r][0]);
        const double targ = double(ri[0].vtarg);
        const double v_old = double(ri[0].value);
        const double v_clip = v_old + fmin(fmax(v - v_old, -a.clip_eps), a.clip_eps);
        const double sq = (v - targ) * (v - targ), sq_c = (v_clip - targ) * (v_clip - targ);
        vt += w * (0.5 * fmax(sq, sq_c));
        g = float(w / total_w * a.vf_coef * (sq >= sq_c ? (v - targ) : 0.0));
      }
      for (int o = 0; o < NOP; ++o) {
        s.dl[r][o] = o == 0 ? g : 0.0f;
        s.dlt[o][r] = o == 0 ? g : 0.0f;
      }
    }
    __syncthreads();
    // B1: dz2 = (dl W3) * act'(h2)
    zero44(c);
    mm<4, 4>(&s.dlt[0][4 * rg], kLD, &s.w3[0][4 * cg], kTW, NOP, c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 y = *reinterpret_cast<const float4*>(&s.h2[4 * rg + i][4 * cg]);
      c[i][0] = act_bwd(c[i][0], y.x, a.relu);
      c[i][1] = act_bwd(c[i][1], y.y, a.relu);
      c[i][2] = act_bwd(c[i][2], y.z, a.relu);
      c[i][3] = act_bwd(c[i][3], y.w, a.relu);
    }
    put44<kLD, kLD>(s.dz2, s.dz2t, 4 * rg, 4 * cg, c);
    __syncthreads();
    // B2: dz1 = (dz2 W2) * act'(h1)
    zero44(c);
    mm<4, 4>(&s.dz2t[0][4 * rg], kLD, &s.w2[0][4 * cg], kTW, kTW, c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 y = *reinterpret_cast<const float4*>(&s.h1[4 * rg + i][4 * cg]);
      c[i][0] = act_bwd(c[i][0], y.x, a.relu);
      c[i][1] = act_bwd(c[i][1], y.y, a.relu);
      c[i][2] = act_bwd(c[i][2], y.z, a.relu);
      c[i][3] = act_bwd(c[i][3], y.w, a.relu);
    }
    put44<kLD, 1>(s.dz1, nullptr, 4 * rg, 4 * cg, c);
    __syncthreads();
    // weight gradients of the tile (dense_backward: g.w = dy^T x, g.b = sum dy)
    mm<4, 4>(&s.dz2[0][4 * rg], kLD, &s.h1[0][4 * cg], kLD, kTR, g2);
    if (t >= 128) mm<4, 4>(&s.dz1[0][4 * rg], kLD, &X[0][4 * (cg - 8)], kLDX, kTR, g1);
    if (t < 16 * NOP) mm<1, 4>(&s.dl[0][t / 16], NOP + 4, &s.h2[0][4 * rg], kLD, kTR, g3);
    {
      float s1 = 0.0f, s2 = 0.0f;
#pragma unroll 4
      for (int r = 16 * bq; r < 16 * bq + 16; ++r) {
        s1 += s.dz1[r][bo];
        s2 += s.dz2[r][bo];
      }
      gb1 += s1;
      gb2 += s2;
      if (bo < NOP) {
        float s3 = 0.0f;
        for (int r = 16 * bq; r < 16 * bq + 16; ++r) s3 += s.dl[r][bo];
        gb3 += s3;
      }
    }
  }
  cp_async_wait<0>();
  // write the CTA's partial gradient in nn::pack order
  float* gp = a.gpart + size_t(blockIdx.x) * size_t(kTW * in + kTW + kTW * kTW + kTW + NO * kTW + NO);
  float *G1 = gp, *GB1 = G1 + kTW * in, *G2 = GB1 + kTW, *GB2 = G2 + kTW * kTW, *G3 = GB2 + kTW, *GB3 = G3 + NO * kTW;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) G2[(4 * rg + i) * kTW + 4 * cg + j] = g2[i][j];
  if (t >= 128)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * (cg - 8) + j < in) G1[(4 * rg + i) * in + 4 * (cg - 8) + j] = g1[i][j];
  if (t < 16 * NOP && t / 16 < NO)
#pragma unroll
    for (int j = 0; j < 4; ++j) G3[(t / 16) * kTW + 4 * rg + j] = g3[0][j];
  // bias partials of the 4 row quarters, summed in quarter order
  __syncthreads();
  s.bred[bq][bo] = gb1;
  __syncthreads();
  if (t < kTW) GB1[t] = ((s.bred[0][t] + s.bred[1][t]) + s.bred[2][t]) + s.bred[3][t];
  __syncthreads();
  s.bred[bq][bo] = gb2;
  __syncthreads();
  if (t < kTW) GB2[t] = ((s.bred[0][t] + s.bred[1][t]) + s.bred[2][t]) + s.bred[3][t];
  __syncthreads();
  if (bo < NOP) s.bred[bq][bo] = gb3;
  __syncthreads();
  if (t < NO) GB3[t] = ((s.bred[0][t] + s.bred[1][t]) + s.bred[2][t]) + s.bred[3][t];
  double v5[kStats] = {pg, vt, ent, kl, clipn, 0.0};
  for (int cc = 0; cc < kStats; ++cc) {
    double v = v5[cc];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) s_stats[t >> 5][cc] = v;
  }
  __syncthreads();
  if (t < kStats) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += s_stats[w][t];
    a.spart[size_t(blockIdx.x) * kStats + t] = v;
  }
}

// Sum the per-CTA partial rows in CTA order: grad[p] = sum_c part[c][p].
__global__ void grad_reduce_kernel(const float* __restrict__ part, int nparts, int P, float* __restrict__ grad) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += double(part[size_t(c) * size_t(P) + p]);
  grad[p] = float(s);
}

// clip_global_norm + adam_update (nn.hpp:417-452) and the minibatch metrics
// (ppo.cpp:604-611).  One CTA; every float operation in the reference's order.
__global__ void __launch_bounds__(1024) clip_adam_kernel(PpoApplyArgs a) {
  __shared__ double sh[32];
  __shared__ int s_bad;
  __shared__ float s_scale;
  __shared__ int s_clip;
  const int t = threadIdx.x;
  __shared__ double s_st[kStats + 1];
  if (*a.diverged) return;  // an earlier minibatch threw: the update is being rolled back
  // the per-CTA loss sums: warp k < 6 folds actor column k, warp 6 the critic's v term
  // (lane-strided, then a fixed shuffle tree)
  if ((t >> 5) <= kStats) {
    const int k = t >> 5;
    const bool cr = k == kStats;
    const double v = warp_fold_col(cr ? a.critic_stats : a.actor_stats, cr ? a.n_critic_parts : a.n_actor_parts,
                                   cr ? 1 : k);
    if ((t & 31) == 0) s_st[k] = v;
  }
  __syncthreads();
  if (t == 0) {
    double st[kStats];
    for (int k = 0; k < kStats; ++k) st[k] = s_st[k];
    const double vt = s_st[kStats];
    const double tw = a.st->total_w;
    double* m = a.metrics;
    if (tw > 0.0) {
      // ppo_row_loss: loss = sum w*(-surr + vf*v - ent*H) / total_w, stored as T
      const double loss = (st[0] + a.vf_coef * vt - a.ent_coef * st[2]) / tw;
      m[0] = double(float(loss));
      m[1] = st[0] / tw;
      m[2] = vt / tw;
      m[3] = st[2] / tw;
      m[4] = st[3] / tw;
      m[5] = st[4] / tw;
    } else {
      for (int k = 0; k < 6; ++k) m[k] = 0.0;
    }
    s_bad = isfinite(m[0]) ? 0 : 1;  // ppo_row_loss's DivergenceError
  }
  __syncthreads();
  if (s_bad) {  // the reference throws before clipping: nothing is applied or counted
    if (t == 0) {
      *a.diverged = 1;
      a.metrics[7] = 0.0;
    }
    return;
  }
  double sq = 0.0;
  for (int p = t; p < a.P; p += blockDim.x) sq += double(a.grad[p]) * double(a.grad[p]);
  sq = block_sum(sq, sh);
  if (t == 0) {
    const float norm = float(sqrt(sq));  // T(std::sqrt(sq))
    s_clip = norm > a.max_norm ? 1 : 0;
    s_scale = __fdiv_rn(a.max_norm, norm);
    a.metrics[6] = double(norm);
  }
  __syncthreads();
  int bad = 0;
  for (int p = t; p < a.P; p += blockDim.x) {
    float g = a.grad[p];
    if (s_clip) g = __fmul_rn(g, s_scale);
    a.grad[p] = g;
    if (!isfinite(g)) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (bad) {  // adam_update's non-finite gradient DivergenceError
    if (t == 0) {
      *a.diverged = 1;
      a.metrics[7] = 0.0;
    }
    return;
  }
  const float b1 = a.beta1, b2 = a.beta2, eps = a.eps, lr = a.lr, c1 = a.c1, c2 = a.c2;
  const float omb1 = __fsub_rn(1.0f, b1), omb2 = __fsub_rn(1.0f, b2);
  for (int p = t; p < a.P; p += blockDim.x) {
    const float g = a.grad[p];
    const float m = __fadd_rn(__fmul_rn(b1, a.m[p]), __fmul_rn(omb1, g));
    const float v = __fadd_rn(__fmul_rn(b2, a.v[p]), __fmul_rn(__fmul_rn(omb2, g), g));
    a.m[p] = m;
    a.v[p] = v;
    const float mhat = __fdiv_rn(m, c1), vhat = __fdiv_rn(v, c2);
    a.params[p] = __fsub_rn(a.params[p], __fdiv_rn(__fmul_rn(lr, mhat), __fadd_rn(__fsqrt_rn(vhat), eps)));
  }
  if (t == 0) a.metrics[7] = 1.0;  // this minibatch counts (n_mb, ppo.cpp:611)
}

unsigned blocks_for(int64_t n, int th) { return unsigned((n + th - 1) / th); }

}  // namespace

size_t ppo_perm_scratch_bytes(int64_t n) {
  size_t temp = 0;
  const int m = int(std::max<int64_t>(n - 1, 1));
  cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, temp, kb, vb, m);
  const size_t buf = (size_t(std::max<int64_t>(n, 1)) * 4 + 255) & ~size_t(255);
  return 7 * buf + ((temp + 255) & ~size_t(255)) + 256;
}

void ppo_permutation(KeyWords key, int64_t n, int32_t* out, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (n <= 0) return;
  const size_t N = size_t(n);
  auto carve = [&](size_t bytes) {
    uint8_t* p = static_cast<uint8_t*>(scratch);
    const size_t a = (bytes + 255) & ~size_t(255);
    scratch = p + a;
    scratch_bytes -= a;
    return static_cast<void*>(p);
  };
  uint32_t* j = static_cast<uint32_t*>(carve(N * 4));
  uint32_t* k0 = static_cast<uint32_t*>(carve(N * 4));
  uint32_t* k1 = static_cast<uint32_t*>(carve(N * 4));
  uint32_t* v0 = static_cast<uint32_t*>(carve(N * 4));
  uint32_t* v1 = static_cast<uint32_t*>(carve(N * 4));
  int32_t* nxt = static_cast<int32_t*>(carve(N * 4));
  int32_t* fst = static_cast<int32_t*>(carve(N * 4));
  const Key k{key.w[0], key.w[1], key.w[2], key.w[3]};
  perm_draw_kernel<<<blocks_for(n, 256), 256, 0, st>>>(k, n, j, k0, v0);
  ++g_launches;
  if (cudaMemsetAsync(fst, 0xff, N * 4, st) != cudaSuccess) return;
  const int64_t m = n - 1;
  if (m > 0) {
    int end_bit = 1;
    while ((uint64_t(1) << end_bit) <= uint64_t(n - 1)) ++end_bit;
    cub::DoubleBuffer<uint32_t> kb(k0, k1), vb(v0, v1);
    size_t temp = scratch_bytes;
    cub::DeviceRadixSort::SortPairs(scratch, temp, kb, vb, int(m), 0, end_bit, st);
    ++g_launches;
    perm_link_kernel<<<blocks_for(m, 256), 256, 0, st>>>(m, kb.Current(), vb.Current(), nxt, fst);
    ++g_launches;
  }
  perm_resolve_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, j, nxt, fst, out);
  ++g_launches;
}

int ppo_stat_blocks(int64_t M) { return int(std::min<int64_t>(std::max<int64_t>((M + 255) / 256, 1), 1184)); }

void ppo_adv_stats(const RolloutBufs& b, const int32_t* idx, int64_t M, double* part, double* part2, double* g,
                   PpoMbStats* st, cudaStream_t s, const std::function<void(double*, int)>& allreduce,
                   const PpoRowRec* rec, float2* gath) {
  const int nb = ppo_stat_blocks(M);
  const float* adv = rec ? &rec->adv : b.adv;
  const float* active = rec ? &rec->active : b.active;
  const int stride = rec ? int(sizeof(PpoRowRec) / sizeof(float)) : 1;
  adv_sum_kernel<<<nb, kRedThreads, 0, s>>>(adv, active, stride, idx, M, part, gath);
  adv_fold_kernel<<<1, kFoldThreads, 0, s>>>(part, nb, g);
  if (allreduce) allreduce(g, 2);
  adv_var_kernel<<<nb, kRedThreads, 0, s>>>(adv, active, stride, idx, M, g, part2, gath);
  adv_fold2_kernel<<<1, kFoldThreads, 0, s>>>(part2, nb, g);
  if (allreduce) allreduce(g + 2, 1);
  adv_final_kernel<<<1, 32, 0, s>>>(g, st);
  g_launches += 6;
}

size_t ppo_compact_scratch_bytes(int64_t M) {
  size_t temp = 0;
  cub::DeviceSelect::If(nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                        static_cast<int64_t*>(nullptr), int(std::max<int64_t>(M, 1)), NonNegative());
  return temp + 256;
}

void ppo_shard_compact(const int32_t* idx, int64_t M, int64_t Rg, int64_t row0, int64_t Rl, int32_t* tmp,
                       int32_t* out, int64_t* d_count, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  shard_map_kernel<<<blocks_for(std::max<int64_t>(M, 1), 256), 256, 0, s>>>(idx, M, Rg, row0, Rl, tmp);
  size_t temp = scratch_bytes;
  cub::DeviceSelect::If(scratch, temp, static_cast<const int32_t*>(tmp), out, d_count, int(M), NonNegative(), s);
  g_launches += 2;
}

void ppo_stats_fold(double* spart, int nparts, cudaStream_t s) {
  stats_fold_kernel<<<1, 6 * 32, 0, s>>>(spart, nparts);
  ++g_launches;
}

// Tile geometry of a branch: the largest TR in {64, 32, 16, 8} whose smem fits.
void ppo_branch_geometry(int in, int W, int out, int* TR, int* staged, size_t* smem) {
  const int P = W * in + W + W * W + W + out * W + out;
  const int ldx = in | 1, ldw = W | 1, ldo = out | 1;
  const size_t cap = 200 * 1024;
  for (int st = 1; st >= 0; --st)
    for (int tr : {64, 32, 16, 8}) {
      const size_t bytes = size_t(st ? P : 0) * 4 + size_t(tr) * size_t(ldx + 4 * ldw + ldo + 1) * 4;
      if (bytes <= cap) {
        *TR = tr;
        *staged = st;
        *smem = bytes;
        return;
      }
    }
  *TR = 8;
  *staged = 0;
  *smem = size_t(8) * size_t(ldx + 4 * ldw + ldo + 1) * 4;
}

bool ppo_tiled_ok(int in, int W, int out);

int ppo_branch_grid(int in, int W, int out, int64_t M) {
  int TR, staged;
  size_t sm;
  ppo_branch_geometry(in, W, out, &TR, &staged, &sm);
  if (ppo_tiled_ok(in, W, out) && !getenv("MARL_PPO_GENERIC")) {
    TR = kTR;
    sm = 200 * 1024;  // one CTA per SM
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int per_sm = std::max(1, int((228 * 1024) / (sm + 2048)));
  const int64_t tiles = (M + TR - 1) / TR;
  return int(cap_grid(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * std::min(per_sm, 2)))));
}

template <bool ACTOR>
static void launch_branch(PpoBranchArgs a, int grid, size_t sm, cudaStream_t s) {
  const int P = a.W * a.in + a.W + a.W * a.W + a.W + a.out * a.W + a.out;
  auto go = [&](auto kern) {
    smem_optin(kern);
    kern<<<grid, kThreads, sm, s>>>(a);
  };
  if (P <= kThreads * 24)
    go(ppo_branch_kernel<ACTOR, 24>);
  else if (P <= kThreads * 48)
    go(ppo_branch_kernel<ACTOR, 48>);
  else
    go(ppo_branch_kernel<ACTOR, 0>);
  ++g_launches;
}

bool ppo_tiled_ok(int in, int W, int out) { return in <= kTIn && W == kTW && out <= 16; }

template <bool ACTOR, int NOP>
static void launch_tiled(const PpoBranchArgs& a, int grid, cudaStream_t s) {
  const size_t sm = sizeof(TiledSmem<NOP>);
  smem_optin(ppo_branch_tiled_kernel<ACTOR, NOP>);
  ppo_branch_tiled_kernel<ACTOR, NOP><<<grid, kThreads, sm, s>>>(a);
  ++g_launches;
}

void ppo_branch(PpoBranchArgs a, bool actor, int grid, cudaStream_t s) {
  if (ppo_tiled_ok(a.in, a.W, a.out) && !getenv("MARL_PPO_GENERIC")) {
    const int nop = a.out <= 4 ? 4 : a.out <= 8 ? 8 : 16;
    if (actor) {
      if (nop == 4) launch_tiled<true, 4>(a, grid, s);
      else if (nop == 8) launch_tiled<true, 8>(a, grid, s);
      else launch_tiled<true, 16>(a, grid, s);
    } else {
      launch_tiled<false, 4>(a, grid, s);
    }
    return;
  }
  size_t sm;
  ppo_branch_geometry(a.in, a.W, a.out, &a.TR, &a.staged, &sm);
  if (actor)
    launch_branch<true>(a, grid, sm, s);
  else
    launch_branch<false>(a, grid, sm, s);
}

// one warp per row: 8-byte copies when every row start allows them (522-column
// Overcooked rows are 8-byte aligned), 4-byte copies otherwise
template <int V>
__global__ void gather_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ idx, int64_t M, int in,
                                   float* __restrict__ out, int ldo) {
  const int64_t m = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (m >= M) return;
  const int lane = threadIdx.x & 31;
  const float* src = x + size_t(__ldg(idx + m)) * size_t(in);
  float* dst = out + size_t(m) * size_t(ldo);
  if constexpr (V == 2) {
    for (int i = lane; i < in / 2; i += 32)
      reinterpret_cast<float2*>(dst)[i] = __ldg(reinterpret_cast<const float2*>(src) + i);
  } else {
    for (int i = lane; i < in; i += 32) dst[i] = __ldg(src + i);
  }
}

void ppo_gather_rows(const float* x, const int32_t* idx, int64_t M, int in, float* out, int ldo, cudaStream_t s) {
  if (M <= 0) return;
  const unsigned blocks = unsigned((M * 32 + 255) / 256);
  const bool v2 = in % 2 == 0 && ldo % 2 == 0 && reinterpret_cast<uintptr_t>(x) % 8 == 0 &&
                  reinterpret_cast<uintptr_t>(out) % 8 == 0;
  if (v2)
    gather_rows_kernel<2><<<blocks, 256, 0, s>>>(x, idx, M, in, out, ldo);
  else
    gather_rows_kernel<1><<<blocks, 256, 0, s>>>(x, idx, M, in, out, ldo);
  ++g_launches;
}

void ppo_grad_reduce(const float* part, int nparts, int P, float* grad, cudaStream_t s) {
  grad_reduce_kernel<<<blocks_for(P, 256), 256, 0, s>>>(part, nparts, P, grad);
  ++g_launches;
}

void ppo_clip_adam(const PpoApplyArgs& a, cudaStream_t s) {
  clip_adam_kernel<<<1, 1024, 0, s>>>(a);
  ++g_launches;
}

}  // namespace marl_b200
