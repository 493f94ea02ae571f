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
//   rnn_rows / gate / sample kernels : the same step for many rows as SGEMMs
//                       (issued by the host) around elementwise kernels.
//   update            : rnn_minibatch (ppo.cpp:444-509) GEMM-structured: per
//                       time step over all rows of a chunk, the gather / reset,
//                       gate and activation-gradient kernels below between
//                       SGEMMs for rnn_seq_forward with cache and
//                       rnn_seq_backward (BPTT with the hidden chain cut at the
//                       forward's resets); rnn_loss_kernel is the per-row part
//                       of ppo_row_loss; the weight gradients are one SGEMM per
//                       matrix over every (t, row).  Chunks of rows bound the
//                       caches (the host sizes them to the free HBM).
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

__host__ __device__ RnnW rnn_w(const float* p, int in, int F, int H, int out) {
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

RnnW rnn_w_host(const float* p, int in, int F, int H, int out) { return rnn_w(p, in, F, H, out); }

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

// ---- elementwise kernels of the GEMM-structured update (rnn_seq_forward /
// rnn_seq_backward, one launch per time step over all M rows; the GEMMs
// between them are plain library SGEMMs issued by the host, venv.cpp)
__global__ void sq_gather_kernel(RnnStepArgs a) {  // x_t rows and h_prev_t (apply_reset)
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t M = a.M, in = a.in, H = a.H;
  if (q < M * in) {
    const int64_t i = q / in, j = q - i * in;
    const size_t slot = size_t(a.t) * size_t(a.R) + size_t(a.rows[i]);
    a.x[i * in + j] = a.src[slot * size_t(in) + j];
  }
  if (q < M * H) {
    const int64_t i = q / H, c = q - i * H;
    const size_t slot = size_t(a.t) * size_t(a.R) + size_t(a.rows[i]);
    const float hv = a.t == 0 ? a.h0[size_t(a.rows[i]) * H + c] : a.h[i * H + c];
    const float v = a.resets[slot] ? 0.0f : hv;
    a.hprev[i * H + c] = v;
    a.h[i * H + c] = v;
  }
}

__global__ void bias_act_kernel(float* __restrict__ y, int64_t M, int N, const float* __restrict__ b, int act,
                                int relu) {  // dense_forward's + b, then act_inplace (nn.hpp:108-115)
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= M * N) return;
  const float v = __fadd_rn(y[q], __ldg(b + q % N));
  y[q] = act ? actf(v, relu) : v;
}

// gru_step's elementwise part (nn.hpp:231-260) from gx = e.[Wz;Wr;Wn]^T and
// gh = h.[Uz;Ur;Un]^T
__global__ void gru_gate_kernel(RnnStepArgs a, const float* __restrict__ gx, const float* __restrict__ gh) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int H = a.H;
  if (q >= a.M * H) return;
  const int64_t i = q / H;
  const int c = int(q - i * H);
  const float* gxi = gx + i * 3 * H;
  const float* ghi = gh + i * 3 * H;
  const auto& w = a.w;
  const float z = sigm(__fadd_rn(gxi[c], __fadd_rn(__fadd_rn(__ldg(w.bzx + c), ghi[c]), __ldg(w.bzh + c))));
  const float r = sigm(__fadd_rn(gxi[H + c], __fadd_rn(__fadd_rn(__ldg(w.brx + c), ghi[H + c]), __ldg(w.brh + c))));
  const float ah = __fadd_rn(ghi[2 * H + c], __ldg(w.bnh + c));
  const float cand = tanhf(__fadd_rn(__fadd_rn(gxi[2 * H + c], __ldg(w.bnx + c)), __fmul_rn(r, ah)));
  const float hp = a.hprev[q];
  const float hn = __fadd_rn(__fmul_rn(z, hp), __fmul_rn(__fsub_rn(1.0f, z), cand));
  a.z[q] = z;
  a.r[q] = r;
  a.c[q] = cand;
  a.ah[q] = ah;
  a.hn[q] = hn;
  if (a.hnext) {  // the next step's sq_gather (h part), fused
    a.hnext[q] = a.resets[size_t(a.t + 1) * size_t(a.R) + size_t(a.rows[i])] ? 0.0f : hn;
  } else {
    a.h[q] = hn;
  }
}

__global__ void act_grad_kernel(float* __restrict__ g, const float* __restrict__ y, int64_t n, int relu) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < n) g[q] = actg(g[q], y[q], relu);
}

// gru_backward's elementwise part (nn.hpp:276-289): dhs -> D4 = [daz | dar | dac | dah], dh = g * z
__global__ void gru_bwd_kernel(RnnStepArgs a, const float* __restrict__ dhs, float* __restrict__ d4,
                               float* __restrict__ dh) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int H = a.H;
  if (q >= a.M * H) return;
  const int64_t i = q / H;
  const int c = int(q - i * H);
  float g;
  if (a.carry == 0) {
    g = dhs[q];
  } else if (a.carry == 1) {
    g = a.dhp[q];
  } else {  // the previous step's cut (no gradient across its episode boundary), then + the post layer's share
    const float d = a.resets[size_t(a.t + 1) * size_t(a.R) + size_t(a.rows[i])] ? 0.0f : dhs[q];
    g = __fadd_rn(d, a.dhp[q]);
  }
  const float z = a.z[q], r = a.r[q], cd = a.c[q];
  const float dz = __fmul_rn(g, __fsub_rn(a.hprev[q], cd));
  const float dc = __fmul_rn(g, __fsub_rn(1.0f, z));
  const float ac = __fmul_rn(dc, __fsub_rn(1.0f, __fmul_rn(cd, cd)));
  float* o = d4 + i * 4 * H;
  o[3 * H + c] = ac;                  // dac
  o[2 * H + c] = __fmul_rn(ac, r);    // dah
  o[H + c] = __fmul_rn(__fmul_rn(__fmul_rn(ac, a.ah[q]), r), __fsub_rn(1.0f, r));
  o[c] = __fmul_rn(__fmul_rn(dz, z), __fsub_rn(1.0f, z));
  dh[q] = __fmul_rn(g, z);
}

unsigned nb(int64_t n) { return unsigned(std::max<int64_t>((n + 255) / 256, 1)); }

// The collector's recurrent step for many rows (GEMM-structured): per row the
// TeamLayout input (+ buffer writes), the critic row, and the hidden states
// reset at the env's episode boundary; bootstrap peeks a copy of the critic's.
__global__ void rnn_rows_kernel(PolicyStep s, RolloutBufs b, int in, int CI, int NA, int H, float* __restrict__ xa,
                                float* __restrict__ xc, float* __restrict__ ha, float* __restrict__ hc,
                                float* __restrict__ hc_peek) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.R) return;
  float x[1024];
  fill_row(s, b, r, in, NA, x, !s.bootstrap);
  for (int k = 0; k < in; ++k) xa[size_t(r) * in + k] = x[k];
  const float* src = s.ws ? s.ws + size_t(r / s.A) * CI : x;
  for (int k = 0; k < CI; ++k) xc[size_t(r) * CI + k] = src[k];
  if (s.ws && !s.bootstrap) {
    float* bc = b.critic_in + (size_t(s.t) * size_t(s.R) + size_t(r)) * CI;
    for (int k = 0; k < CI; ++k) bc[k] = src[k];
  }
  const bool reset = s.prev_finished ? s.prev_finished[r / s.A] != 0 : true;
  if (s.bootstrap) {
    for (int c = 0; c < H; ++c) hc_peek[size_t(r) * H + c] = reset ? 0.0f : hc[size_t(r) * H + c];
  } else if (reset) {
    for (int c = 0; c < H; ++c) ha[size_t(r) * H + c] = 0.0f;
    for (int c = 0; c < H; ++c) hc[size_t(r) * H + c] = 0.0f;
  }
}

// gates in place on h (hn = z h + (1 - z) c), no caches: the acting step
__global__ void gru_gate_inplace_kernel(int64_t M, int H, float* __restrict__ h, const float* __restrict__ gx,
                                        const float* __restrict__ gh, const float* __restrict__ b6) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= M * H) return;
  const int64_t i = q / H;
  const int c = int(q - i * H);
  const float* gxi = gx + i * 3 * H;
  const float* ghi = gh + i * 3 * H;
  const float z = sigm(__fadd_rn(gxi[c], __fadd_rn(__fadd_rn(__ldg(b6 + c), ghi[c]), __ldg(b6 + 3 * H + c))));
  const float r = sigm(__fadd_rn(gxi[H + c], __fadd_rn(__fadd_rn(__ldg(b6 + H + c), ghi[H + c]),
                                                      __ldg(b6 + 4 * H + c))));
  const float ah = __fadd_rn(ghi[2 * H + c], __ldg(b6 + 5 * H + c));
  const float cand = tanhf(__fadd_rn(__fadd_rn(gxi[2 * H + c], __ldg(b6 + 2 * H + c)), __fmul_rn(r, ah)));
  h[q] = __fadd_rn(__fmul_rn(z, h[q]), __fmul_rn(__fsub_rn(1.0f, z), cand));
}

__global__ void rnn_sample_kernel(PolicyStep s, RolloutBufs b, int NA, const float* __restrict__ ya,
                                  const float* __restrict__ yc) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.R) return;
  if (s.bootstrap) {
    b.last_value[r] = yc[r];
    return;
  }
  sample_and_record(s, b, r, ya + size_t(r) * NA, NA, yc[r]);
}

}  // namespace

void rnn_policy_rows(const PolicyStep& s, const RolloutBufs& b, int in, int CI, int NA, int H, float* xa, float* xc,
                     float* ha, float* hc, float* hc_peek, cudaStream_t st) {
  rnn_rows_kernel<<<unsigned((s.R + 127) / 128), 128, 0, st>>>(s, b, in, CI, NA, H, xa, xc, ha, hc, hc_peek);
  ++g_launches;
}
void rnn_gates_inplace(int64_t M, int H, float* h, const float* gx, const float* gh, const float* b6, cudaStream_t st) {
  gru_gate_inplace_kernel<<<nb(M * H), 256, 0, st>>>(M, H, h, gx, gh, b6);
  ++g_launches;
}
void rnn_policy_sample(const PolicyStep& s, const RolloutBufs& b, int NA, const float* ya, const float* yc,
                       cudaStream_t st) {
  rnn_sample_kernel<<<unsigned((s.R + 127) / 128), 128, 0, st>>>(s, b, NA, ya, yc);
  ++g_launches;
}

RnnWPtrs rnn_weights(const float* p, int in, int F, int H, int out) {
  const auto w = rnn_w_host(p, in, F, H, out);
  return RnnWPtrs{w.we, w.be, w.wz, w.uz, w.bzx, w.wp, w.bp, w.wh, w.bh};
}

__global__ void seq_x_gather_kernel(const int32_t* __restrict__ rows, int64_t Mc, int T, int64_t R, int in,
                                    const float* __restrict__ src, float* __restrict__ x) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= int64_t(T) * Mc * in) return;
  const int64_t k = q / in, j = q - k * in, t = k / Mc, i = k - t * Mc;
  x[q] = __ldg(src + (size_t(t) * size_t(R) + size_t(__ldg(rows + i))) * size_t(in) + j);
}
void rnn_seq_x_gather(const int32_t* rows, int64_t Mc, int T, int64_t R, int in, const float* src, float* x,
                      cudaStream_t s) {
  seq_x_gather_kernel<<<nb(int64_t(T) * Mc * in), 256, 0, s>>>(rows, Mc, T, R, in, src, x);
  ++g_launches;
}
void rnn_step_gather(const RnnStepArgs& a, cudaStream_t s) {
  sq_gather_kernel<<<nb(a.M * std::max(a.in, a.H)), 256, 0, s>>>(a);
  ++g_launches;
}
void rnn_bias_act(float* y, int64_t M, int N, const float* b, bool act, int relu, cudaStream_t s) {
  bias_act_kernel<<<nb(M * N), 256, 0, s>>>(y, M, N, b, act ? 1 : 0, relu);
  ++g_launches;
}
void rnn_gates(const RnnStepArgs& a, const float* gx, const float* gh, cudaStream_t s) {
  gru_gate_kernel<<<nb(a.M * a.H), 256, 0, s>>>(a, gx, gh);
  ++g_launches;
}
void rnn_act_grad(float* g, const float* y, int64_t n, int relu, cudaStream_t s) {
  act_grad_kernel<<<nb(n), 256, 0, s>>>(g, y, n, relu);
  ++g_launches;
}
void rnn_gru_bwd(const RnnStepArgs& a, const float* dhs, float* d4, float* dh, cudaStream_t s) {
  gru_bwd_kernel<<<nb(a.M * a.H), 256, 0, s>>>(a, dhs, d4, dh);
  ++g_launches;
}

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




}  // namespace marl_b200
