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
__global__ void adv_sum_kernel(const float* __restrict__ adv, const float* __restrict__ active,
                               const int32_t* __restrict__ idx, int64_t M, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0, n = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < M; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = idx[i];
    const double w = double(active[r]);
    s += w * double(adv[r]);
    n += w;
  }
  s = block_sum(s, sh);
  n = block_sum(n, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = n;
  }
}

__device__ __forceinline__ void mean_of(const double* part, int nb, double* mean, double* n) {
  double s = 0.0, c = 0.0;
  for (int q = 0; q < nb; ++q) {
    s += part[2 * q];
    c += part[2 * q + 1];
  }
  *n = c;
  *mean = c > 0.0 ? s / c : 0.0;
}

// pass 2: sum(w * (adv - mean)^2) (actor_critic.hpp:424-429)
__global__ void adv_var_kernel(const float* __restrict__ adv, const float* __restrict__ active,
                               const int32_t* __restrict__ idx, int64_t M, const double* __restrict__ part, int nb,
                               double* __restrict__ part2) {
  __shared__ double sh[32];
  __shared__ double s_mean;
  if (threadIdx.x == 0) {
    double n;
    mean_of(part, nb, &s_mean, &n);
  }
  __syncthreads();
  const double mean = s_mean;
  double v = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < M; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = idx[i];
    const double d = double(adv[r]) - mean;
    v += double(active[r]) * d * d;
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part2[blockIdx.x] = v;
}

__global__ void adv_final_kernel(const double* __restrict__ part, const double* __restrict__ part2, int nb,
                                 PpoMbStats* st) {
  if (threadIdx.x != 0) return;
  double mean, n;
  mean_of(part, nb, &mean, &n);
  double var = 0.0;
  for (int q = 0; q < nb; ++q) var += part2[q];
  st->total_w = n;
  st->normalize = n > 0.0 ? 1 : 0;  // n <= 0: advantages left as they are
  st->mean = mean;
  st->std = n > 0.0 ? sqrt(var / n) : 0.0;
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
  if (*a.diverged) return;  // an earlier minibatch threw: the update is being rolled back
  if (t == 0) {
    double st[kStats] = {0, 0, 0, 0, 0, 0};
    for (int c = 0; c < a.n_actor_parts; ++c)
      for (int k = 0; k < kStats; ++k) st[k] += a.actor_stats[size_t(c) * kStats + k];
    double vt = 0.0;
    for (int c = 0; c < a.n_critic_parts; ++c) vt += a.critic_stats[size_t(c) * kStats + 1];
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

void ppo_adv_stats(const RolloutBufs& b, const int32_t* idx, int64_t M, double* part, double* part2, PpoMbStats* st,
                   cudaStream_t s) {
  const int nb = ppo_stat_blocks(M);
  adv_sum_kernel<<<nb, kRedThreads, 0, s>>>(b.adv, b.active, idx, M, part);
  adv_var_kernel<<<nb, kRedThreads, 0, s>>>(b.adv, b.active, idx, M, part, nb, part2);
  adv_final_kernel<<<1, 32, 0, s>>>(part, part2, nb, st);
  g_launches += 3;
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

int ppo_branch_grid(int in, int W, int out, int64_t M) {
  int TR, staged;
  size_t sm;
  ppo_branch_geometry(in, W, out, &TR, &staged, &sm);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int per_sm = std::max(1, int((228 * 1024) / (sm + 2048)));
  const int64_t tiles = (M + TR - 1) / TR;
  return int(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * std::min(per_sm, 2))));
}

template <bool ACTOR>
static void launch_branch(PpoBranchArgs a, int grid, size_t sm, cudaStream_t s) {
  const int P = a.W * a.in + a.W + a.W * a.W + a.W + a.out * a.W + a.out;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
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

void ppo_branch(PpoBranchArgs a, bool actor, int grid, cudaStream_t s) {
  size_t sm;
  ppo_branch_geometry(a.in, a.W, a.out, &a.TR, &a.staged, &sm);
  if (actor)
    launch_branch<true>(a, grid, sm, s);
  else
    launch_branch<false>(a, grid, sm, s);
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
