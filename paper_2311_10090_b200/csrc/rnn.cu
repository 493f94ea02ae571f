// Recurrent (GRU) actor / critic: the reference's
// RnnBranch (proj/core/include/marl/algo/actor_critic.hpp:74-200) and
// gru_step / gru_backward (nn.hpp:200-318) on the device, fp32, every dot
// product in the reference's accumulation order (-fmad=false):
//
//   rnn_policy_kernel : Collector::collect's recurrent acting step
//                       (ppo.cpp:228-250): apply_reset, embed, gru_step, post,
//                       head, for actor (then masked sampling) and critic, the
//                       hidden states carried in place; bootstrap mode peeks
//                       the critic without advancing it (ppo.cpp:283-296).
//   rnn_fwd_kernel    : rnn_seq_forward with cache over a minibatch of row
//                       sequences (rnn_minibatch, ppo.cpp:444-509).
//   rnn_loss_kernel   : the per-row part of ppo_row_loss over the [t][i] rows.
//   rnn_bwd_kernel    : rnn_seq_backward (actor_critic.hpp:164-196): BPTT with
//                       the hidden chain cut at the forward's resets; stores the
//                       per-(t, row) deltas.
//   outer_sum_kernel  : the weight gradients sum_k delta[k] (x) input[k] over
//                       all (t, row) (matmul_tn per step + axpy over steps).
// One thread owns one row (sequence); weights are read through L1 (every
// thread of a warp reads the same element).  This is the parity path; the
// caches hold every step of the minibatch, so the host guards its size.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "engine.h"
#include "policy_rows.cuh"

namespace marl_b200 {

namespace {

constexpr int kRnnMaxIn = 1024, kRnnMaxF = 64, kRnnMaxH = 128, kRnnMaxOut = 64;

struct RnnW {  // one branch in RnnBranch pack order (actor_critic.hpp:198-209)
  const float *we, *be, *wz, *wr, *wn, *uz, *ur, *un, *bzx, *brx, *bnx, *bzh, *brh, *bnh, *wp, *bp, *wh, *bh;
};

__device__ RnnW rnn_w(const float* p, int in, int F, int H, int out) {
  RnnW w;
  w.we = p;
  w.be = w.we + F * in;
  w.wz = w.be + F;
  w.wr = w.wz + H * F;
  w.wn = w.wr + H * F;
  w.uz = w.wn + H * F;
  w.ur = w.uz + H * H;
  w.un = w.ur + H * H;
  w.bzx = w.un + H * H;
  w.brx = w.bzx + H;
  w.bnx = w.brx + H;
  w.bzh = w.bnx + H;
  w.brh = w.bzh + H;
  w.bnh = w.brh + H;
  w.wp = w.bnh + H;
  w.bp = w.wp + F * H;
  w.wh = w.bp + F;
  w.bh = w.wh + out * F;
  return w;
}

__device__ __forceinline__ float dotr(const float* __restrict__ x, const float* __restrict__ w, int n) {
  float acc = 0.0f;  // matmul_nt: acc += x[i] * w[i], i ascending (nn.hpp:42-54)
  for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, __fmul_rn(x[i], __ldg(w + i)));
  return acc;
}
__device__ __forceinline__ float actf(float v, int relu) { return relu ? (v > 0.0f ? v : 0.0f) : tanhf(v); }
__device__ __forceinline__ float actg(float g, float y, int relu) {  // grad *= act_grad_from_output(y)
  return __fmul_rn(g, relu ? (y > 0.0f ? 1.0f : 0.0f) : __fsub_rn(1.0f, __fmul_rn(y, y)));
}
__device__ __forceinline__ float sigm(float v) { return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-v))); }

// One recurrent step of one row (rnn_step, actor_critic.hpp:103-111): h is
// updated in place (already reset by the caller); optional cache outputs.
__device__ void rnn_row_step(const RnnW& w, int in, int F, int H, int out, int relu, const float* x, float* h,
                             float* y, float* c_e, float* c_h, float* c_z, float* c_r, float* c_c, float* c_ah,
                             float* c_p) {
  float e[kRnnMaxF], hn[kRnnMaxH], pz[kRnnMaxF];
  for (int o = 0; o < F; ++o) e[o] = actf(__fadd_rn(dotr(x, w.we + o * in, in), __ldg(w.be + o)), relu);
  if (c_h)
    for (int c = 0; c < H; ++c) c_h[c] = h[c];
  for (int c = 0; c < H; ++c) {  // gru_step (nn.hpp:224-262)
    float z = dotr(e, w.wz + c * F, F);
    z = __fadd_rn(z, __fadd_rn(__fadd_rn(__ldg(w.bzx + c), dotr(h, w.uz + c * H, H)), __ldg(w.bzh + c)));
    z = sigm(z);
    float r = dotr(e, w.wr + c * F, F);
    r = __fadd_rn(r, __fadd_rn(__fadd_rn(__ldg(w.brx + c), dotr(h, w.ur + c * H, H)), __ldg(w.brh + c)));
    r = sigm(r);
    const float ah = __fadd_rn(dotr(h, w.un + c * H, H), __ldg(w.bnh + c));
    const float cand =
        tanhf(__fadd_rn(__fadd_rn(dotr(e, w.wn + c * F, F), __ldg(w.bnx + c)), __fmul_rn(r, ah)));
    hn[c] = __fadd_rn(__fmul_rn(z, h[c]), __fmul_rn(__fsub_rn(1.0f, z), cand));
    if (c_z) {
      c_z[c] = z;
      c_r[c] = r;
      c_c[c] = cand;
      c_ah[c] = ah;
    }
  }
  for (int c = 0; c < H; ++c) h[c] = hn[c];
  for (int o = 0; o < F; ++o) pz[o] = actf(__fadd_rn(dotr(h, w.wp + o * H, H), __ldg(w.bp + o)), relu);
  for (int o = 0; o < out; ++o) y[o] = __fadd_rn(dotr(pz, w.wh + o * F, F), __ldg(w.bh + o));
  if (c_e) {
    for (int o = 0; o < F; ++o) c_e[o] = e[o];
    for (int o = 0; o < F; ++o) c_p[o] = pz[o];
  }
}

__global__ void __launch_bounds__(128) rnn_policy_kernel(RnnPolicyArgs a, PolicyStep s, RolloutBufs b) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.R) return;
  const int in = a.in_dim, CI = a.critic_in, F = a.F, H = a.H, NA = a.n_act;
  const RnnW wa = rnn_w(a.actor, in, F, H, NA), wc = rnn_w(a.critic, CI, F, H, 1);
  float x[kRnnMaxIn], h[kRnnMaxH], y[kRnnMaxOut];
  fill_row(s, b, r, in, NA, x, !s.bootstrap);
  const float* xc = x;
  if (s.ws) {
    xc = s.ws + size_t(r / s.A) * CI;
    if (!s.bootstrap) {
      float* bc = b.critic_in + (size_t(s.t) * size_t(s.R) + size_t(r)) * CI;
      for (int k = 0; k < CI; ++k) bc[k] = xc[k];
    }
  }
  // reset_rows = prev_finished of the row's env (ppo.cpp:229-231); the first
  // window's first step resets every row (Collector ctor, ppo.cpp:193)
  const bool reset = s.prev_finished ? s.prev_finished[r / s.A] != 0 : true;
  float xcl[kRnnMaxIn];
  for (int k = 0; k < CI; ++k) xcl[k] = xc[k];
  // critic: bootstrap peeks a copy (ppo.cpp:290-292), acting advances it
  float* hc = a.h_critic + size_t(r) * H;
  for (int c = 0; c < H; ++c) h[c] = reset ? 0.0f : hc[c];
  rnn_row_step(wc, CI, F, H, 1, a.relu, xcl, h, y, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  const float value = y[0];
  if (s.bootstrap) {
    b.last_value[r] = value;
    return;
  }
  for (int c = 0; c < H; ++c) hc[c] = h[c];
  float* ha = a.h_actor + size_t(r) * H;
  for (int c = 0; c < H; ++c) h[c] = reset ? 0.0f : ha[c];
  rnn_row_step(wa, in, F, H, NA, a.relu, x, h, y, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  for (int c = 0; c < H; ++c) ha[c] = h[c];
  sample_and_record(s, b, r, y, NA, value);
}

// ---- update: rnn_seq_forward with cache over M row sequences x T steps.
// Cache layout: [T*M][width] row-major, k = t*M + i (the loss's flat order).
__global__ void __launch_bounds__(128) rnn_fwd_kernel(RnnSeqArgs a, bool actor) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.M) return;
  const int in = actor ? a.in_dim : a.critic_in, F = a.F, H = a.H, out = actor ? a.n_act : 1;
  const RnnW w = rnn_w(actor ? a.actor : a.critic, in, F, H, out);
  const RnnCache& c = actor ? a.ca : a.cc;
  const int64_t row = a.rows[i];
  float h[kRnnMaxH], x[kRnnMaxIn];
  const float* h0 = (actor ? a.h0_actor : a.h0_critic) + size_t(row) * H;
  for (int q = 0; q < H; ++q) h[q] = h0[q];
  for (int t = 0; t < a.T; ++t) {
    const size_t slot = size_t(t) * size_t(a.R) + size_t(row), k = size_t(t) * size_t(a.M) + size_t(i);
    if (a.resets[slot])
      for (int q = 0; q < H; ++q) h[q] = 0.0f;  // apply_reset (actor_critic.hpp:95-101)
    const float* src = (actor || !a.critic_rows) ? a.obs + slot * size_t(a.in_dim) : a.critic_rows + slot * size_t(in);
    for (int q = 0; q < in; ++q) x[q] = src[q];
    for (int q = 0; q < in; ++q) c.x[k * in + q] = x[q];
    rnn_row_step(w, in, F, H, out, a.relu, x, h, c.y + k * out, c.e + k * F, c.h + k * H, c.z + k * H, c.r + k * H,
                 c.c + k * H, c.ah + k * H, c.p + k * F);
    for (int q = 0; q < H; ++q) c.hn[k * H + q] = h[q];
  }
}

// ---- rnn_seq_backward for one row sequence (actor_critic.hpp:164-196)
__global__ void __launch_bounds__(128) rnn_bwd_kernel(RnnSeqArgs a, bool actor) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.M) return;
  const int in = actor ? a.in_dim : a.critic_in, F = a.F, H = a.H, out = actor ? a.n_act : 1;
  const RnnW w = rnn_w(actor ? a.actor : a.critic, in, F, H, out);
  const RnnCache& c = actor ? a.ca : a.cc;
  const int64_t row = a.rows[i];
  float dh[kRnnMaxH], dhs[kRnnMaxH], dp[kRnnMaxF], dzp[kRnnMaxF];
  for (int q = 0; q < H; ++q) dh[q] = 0.0f;
  bool have_dh = false;
  for (int t = a.T - 1; t >= 0; --t) {
    const size_t k = size_t(t) * size_t(a.M) + size_t(i), slot = size_t(t) * size_t(a.R) + size_t(row);
    const float* dy = c.dy + k * out;
    // head: dp = dy . Wh (matmul_nn skips zero dy, nn.hpp:74-88)
    for (int f = 0; f < F; ++f) dp[f] = 0.0f;
    for (int o = 0; o < out; ++o) {
      const float g = dy[o];
      if (g == 0.0f) continue;
      for (int f = 0; f < F; ++f) dp[f] = __fadd_rn(dp[f], __fmul_rn(g, __ldg(w.wh + o * F + f)));
    }
    // post: dz = dp * act'(p); dh_step = dz . Wp  (+ the carried dh)
    const float* pz = c.p + k * F;
    for (int f = 0; f < F; ++f) dzp[f] = actg(dp[f], pz[f], a.relu);
    for (int f = 0; f < F; ++f) c.dzp[k * F + f] = dzp[f];
    for (int q = 0; q < H; ++q) dhs[q] = 0.0f;
    for (int f = 0; f < F; ++f) {
      const float g = dzp[f];
      if (g == 0.0f) continue;
      for (int q = 0; q < H; ++q) dhs[q] = __fadd_rn(dhs[q], __fmul_rn(g, __ldg(w.wp + f * H + q)));
    }
    if (have_dh)
      for (int q = 0; q < H; ++q) dhs[q] = __fadd_rn(dhs[q], dh[q]);
    // gru_backward (nn.hpp:270-318), elementwise part
    float* daz = c.daz + k * H;
    float* dar = c.dar + k * H;
    float* dac = c.dac + k * H;
    float* dah = c.dah + k * H;
    const float *hp = c.h + k * H, *zz = c.z + k * H, *rr = c.r + k * H, *cc = c.c + k * H, *ahh = c.ah + k * H;
    for (int q = 0; q < H; ++q) {
      const float g = dhs[q], z = zz[q], r = rr[q], cd = cc[q];
      const float dz = __fmul_rn(g, __fsub_rn(hp[q], cd));
      const float dc = __fmul_rn(g, __fsub_rn(1.0f, z));
      const float ac = __fmul_rn(dc, __fsub_rn(1.0f, __fmul_rn(cd, cd)));
      dac[q] = ac;
      dah[q] = __fmul_rn(ac, r);
      const float dr = __fmul_rn(ac, ahh[q]);
      dar[q] = __fmul_rn(__fmul_rn(dr, r), __fsub_rn(1.0f, r));
      daz[q] = __fmul_rn(__fmul_rn(dz, z), __fsub_rn(1.0f, z));
      dh[q] = __fmul_rn(g, z);  // the carry path
    }
    // de = daz.Wz + (dar.Wr + dac.Wn); dh_prev = dh_acc + ((daz.Uz + dar.Ur) + dah.Un)
    float de[kRnnMaxF];
    {
      float t0[kRnnMaxF], t1[kRnnMaxF], t2[kRnnMaxF];
      for (int f = 0; f < F; ++f) t0[f] = t1[f] = t2[f] = 0.0f;
      for (int q = 0; q < H; ++q) {
        const float gz = daz[q], gr = dar[q], gc = dac[q];
        if (gz != 0.0f)
          for (int f = 0; f < F; ++f) t0[f] = __fadd_rn(t0[f], __fmul_rn(gz, __ldg(w.wz + q * F + f)));
        if (gr != 0.0f)
          for (int f = 0; f < F; ++f) t1[f] = __fadd_rn(t1[f], __fmul_rn(gr, __ldg(w.wr + q * F + f)));
        if (gc != 0.0f)
          for (int f = 0; f < F; ++f) t2[f] = __fadd_rn(t2[f], __fmul_rn(gc, __ldg(w.wn + q * F + f)));
      }
      for (int f = 0; f < F; ++f) de[f] = __fadd_rn(t0[f], __fadd_rn(t1[f], t2[f]));
    }
    {
      float t0[kRnnMaxH], t1[kRnnMaxH], t2[kRnnMaxH];
      for (int q = 0; q < H; ++q) t0[q] = t1[q] = t2[q] = 0.0f;
      for (int o = 0; o < H; ++o) {
        const float gz = daz[o], gr = dar[o], gh = dah[o];
        if (gz != 0.0f)
          for (int q = 0; q < H; ++q) t0[q] = __fadd_rn(t0[q], __fmul_rn(gz, __ldg(w.uz + o * H + q)));
        if (gr != 0.0f)
          for (int q = 0; q < H; ++q) t1[q] = __fadd_rn(t1[q], __fmul_rn(gr, __ldg(w.ur + o * H + q)));
        if (gh != 0.0f)
          for (int q = 0; q < H; ++q) t2[q] = __fadd_rn(t2[q], __fmul_rn(gh, __ldg(w.un + o * H + q)));
      }
      for (int q = 0; q < H; ++q) dh[q] = __fadd_rn(dh[q], __fadd_rn(__fadd_rn(t0[q], t1[q]), t2[q]));
    }
    // embed: dz_e = de * act'(e)
    const float* ee = c.e + k * F;
    for (int f = 0; f < F; ++f) c.dze[k * F + f] = actg(de[f], ee[f], a.relu);
    if (a.resets[slot])
      for (int q = 0; q < H; ++q) dh[q] = 0.0f;  // no gradient across episode cuts
    have_dh = true;
  }
}

// G[o][i] (+)= sum_k D[k*ldd + o] * X[k*ldx + i]  (X == null: bias, sum_k D)
__global__ void outer_sum_kernel(const float* __restrict__ D, int ldd, const float* __restrict__ X, int ldx,
                                 int64_t K, int O, int I, float* __restrict__ G) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int cols = X ? I : 1;
  if (e >= int64_t(O) * cols) return;
  const int o = int(e / cols), i = int(e % cols);
  float acc = 0.0f;
  if (X) {
    for (int64_t k = 0; k < K; ++k) acc = __fadd_rn(acc, __fmul_rn(D[k * ldd + o], X[k * ldx + i]));
  } else {
    for (int64_t k = 0; k < K; ++k) acc = __fadd_rn(acc, D[k * ldd + o]);
  }
  G[e] = acc;
}

__global__ void flat_slots_kernel(const int32_t* __restrict__ rows, int64_t M, int T, int64_t R,
                                  int32_t* __restrict__ flat) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= int64_t(T) * M) return;
  const int64_t t = k / M, i = k - t * M;
  flat[k] = int32_t(t * R + rows[i]);
}

constexpr int kLossThreads = 128;

// ppo_row_loss (actor_critic.hpp:340-412) of flat row k: the actor's logits and
// the critic's value from the forward caches, the row data from the buffer.
__global__ void __launch_bounds__(kLossThreads) rnn_loss_kernel(RnnSeqArgs a, const int32_t* __restrict__ flat,
                                                                int64_t K, RolloutBufs b, const PpoMbStats* stp,
                                                                double clip_eps, double ent_coef, double vf_coef,
                                                                double* spart_a, double* spart_c, int* err) {
  __shared__ double sh[kLossThreads / 32][5];
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const PpoMbStats st = *stp;
  const double total_w = st.total_w;
  double pg = 0.0, vt = 0.0, ent = 0.0, kl = 0.0, clipn = 0.0;
  const int NA = a.n_act;
  if (k < K) {
    const int64_t sl = flat[k];
    const double w = double(b.active[sl]);
    float* dl = a.ca.dy + k * NA;
    float* dv = a.cc.dy + k;
    if (w == 0.0 || total_w <= 0.0) {
      for (int i = 0; i < NA; ++i) dl[i] = 0.0f;
      *dv = 0.0f;
    } else {
      const float* z = a.ca.y + k * NA;
      const uint8_t* legal = b.legal + size_t(sl) * size_t(NA);
      double lp[kPpoMaxAct];
      double mx = -INFINITY;
      for (int i = 0; i < NA; ++i)
        if (legal[i]) mx = fmax(mx, double(z[i]));
      double denom = 0.0;
      for (int i = 0; i < NA; ++i)
        if (legal[i]) denom += exp(double(z[i]) - mx);
      const double log_denom = log(denom);
      for (int i = 0; i < NA; ++i) lp[i] = legal[i] ? double(z[i]) - mx - log_denom : -1e30;
      const int act = b.actions[sl];
      if (act < 0 || act >= NA || !legal[act] || !(mx > -INFINITY)) atomicExch(err, 1);
      const int ac = act < 0 ? 0 : (act >= NA ? NA - 1 : act);
      float advf = b.adv[sl];
      if (st.normalize) advf = float((double(advf) - st.mean) / (st.std + 1e-8));
      const double adv = double(advf);
      const double ratio = exp(lp[ac] - double(b.logp[sl]));
      const double unclipped = ratio * adv;
      const double rho_c = fmin(fmax(ratio, 1.0 - clip_eps), 1.0 + clip_eps);
      const double clipped = rho_c * adv;
      const double surr = fmin(unclipped, clipped);
      const double dsurr = unclipped <= clipped ? ratio * adv : 0.0;
      double entropy = 0.0;
      for (int i = 0; i < NA; ++i)
        if (legal[i]) entropy -= exp(lp[i]) * lp[i];
      for (int i = 0; i < NA; ++i) {
        if (!legal[i]) {
          dl[i] = 0.0f;
          continue;
        }
        const double pi = exp(lp[i]);
        const double g = -dsurr * ((i == ac ? 1.0 : 0.0) - pi) - ent_coef * (-pi * (lp[i] + entropy));
        dl[i] = float(w / total_w * g);
      }
      pg = w * -surr;
      ent = w * entropy;
      kl = w * (ratio - 1.0 - log(ratio));
      clipn = w * (fabs(ratio - 1.0) > clip_eps ? 1.0 : 0.0);
      const double v = double(a.cc.y[k]), targ = double(b.vtarg[sl]), v_old = double(b.value[sl]);
      const double v_clip = v_old + fmin(fmax(v - v_old, -clip_eps), clip_eps);
      const double sq = (v - targ) * (v - targ), sq_c = (v_clip - targ) * (v_clip - targ);
      vt = w * (0.5 * fmax(sq, sq_c));
      *dv = float(w / total_w * vf_coef * (sq >= sq_c ? (v - targ) : 0.0));
    }
  }
  double v5[5] = {pg, vt, ent, kl, clipn};
  for (int q = 0; q < 5; ++q) {
    double v = v5[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][q] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s5[5] = {0, 0, 0, 0, 0};
    for (int wq = 0; wq < kLossThreads / 32; ++wq)
      for (int q = 0; q < 5; ++q) s5[q] += sh[wq][q];
    double* pa = spart_a + size_t(blockIdx.x) * 6;
    double* pc = spart_c + size_t(blockIdx.x) * 6;
    pa[0] = s5[0], pa[1] = 0.0, pa[2] = s5[2], pa[3] = s5[3], pa[4] = s5[4], pa[5] = 0.0;
    pc[0] = 0.0, pc[1] = s5[1], pc[2] = pc[3] = pc[4] = pc[5] = 0.0;
  }
}

}  // namespace

int rnn_loss_blocks(int64_t K) { return int(std::max<int64_t>((K + kLossThreads - 1) / kLossThreads, 1)); }

void rnn_loss(const RnnSeqArgs& a, const int32_t* flat, int64_t K, const RolloutBufs& b, const PpoMbStats* st,
              double clip_eps, double ent_coef, double vf_coef, double* spart_a, double* spart_c, int* err,
              cudaStream_t s) {
  rnn_loss_kernel<<<rnn_loss_blocks(K), kLossThreads, 0, s>>>(a, flat, K, b, st, clip_eps, ent_coef, vf_coef,
                                                               spart_a, spart_c, err);
  ++g_launches;
}

void rnn_flat_slots(const int32_t* rows, int64_t M, int T, int64_t R, int32_t* flat, cudaStream_t st) {
  const int64_t K = int64_t(T) * M;
  flat_slots_kernel<<<unsigned(std::max<int64_t>((K + 255) / 256, 1)), 256, 0, st>>>(rows, M, T, R, flat);
  ++g_launches;
}

void rnn_policy(const RnnPolicyArgs& a, const PolicyStep& s, const RolloutBufs& b, cudaStream_t st) {
  rnn_policy_kernel<<<unsigned((s.R + 127) / 128), 128, 0, st>>>(a, s, b);
  ++g_launches;
}

void rnn_forward(const RnnSeqArgs& a, bool actor, cudaStream_t st) {
  rnn_fwd_kernel<<<unsigned((a.M + 127) / 128), 128, 0, st>>>(a, actor);
  ++g_launches;
}

void rnn_backward(const RnnSeqArgs& a, bool actor, cudaStream_t st) {
  rnn_bwd_kernel<<<unsigned((a.M + 127) / 128), 128, 0, st>>>(a, actor);
  ++g_launches;
}

void rnn_outer_sum(const float* D, int ldd, const float* X, int ldx, int64_t K, int O, int I, float* G,
                   cudaStream_t st) {
  const int64_t n = int64_t(O) * (X ? I : 1);
  outer_sum_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(D, ldd, X, ldx, K, O, I, G);
  ++g_launches;
}

}  // namespace marl_b200
