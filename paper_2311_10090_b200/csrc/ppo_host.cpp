// The trainer of the C-ABI (marl_ppo_*, include/marl_b200.h): the reference's
// train_ippo / train_mappo (proj/core/src/algo/ppo.cpp:518-651) around the
// collector and the device update (ppo.cu, ppo_tc.cu, rnn.cu, gemm_tc.cu),
// with the NCCL library loaded at run time.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "host.h"

using namespace marl_b200;
using namespace mhost;

// ====================================================================== PPO
// train_ippo / train_mappo (ppo.cpp:518-651) around the device update
// (ppo.cu): PpoConfig::from_config + validate (ppo.cpp:18-62), ppo_init_nets
// (ppo.cpp:109-124) on the host, and the update loop with its metrics row.
namespace mhost {


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


namespace mhost {

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

// The recurrent path's GEMMs: fp32-accurate 3xTF32 tcgen05 kernels (gemm_tc.cu).
// Row-major C[M x N] = A[M x K] . B[N x K]^T (+ beta C)
void gemm_nt(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta) {
  cuda_check(tc_gemm(st, M, N, K, A, lda, 1, B, ldb, 1, C, ldc, beta), "tc_gemm");
}
// C[M x N] = A[M x K] . B[K x N] (+ beta C)
void gemm_nn(cudaStream_t st, int64_t M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, float beta) {
  cuda_check(tc_gemm(st, M, N, K, A, lda, 1, B, 1, ldb, C, ldc, beta), "tc_gemm");
}
// G[O x I] = D[K x O]^T . X[K x I] (+ beta G): matmul_tn summed over all rows
void gemm_tn(cudaStream_t st, int O, int I, int64_t K, const float* D, int ldd, const float* X, int ldx, float* G,
             float beta) {
  cuda_check(tc_gemm(st, O, I, K, D, 1, ldd, X, 1, ldx, G, I, beta), "tc_gemm");
}
// g[O] = sum_k D[k][o] (+ beta g): the bias gradients (fixed-order reduction)
void colsum(cudaStream_t st, int O, int64_t K, const float* D, int ldd, const float* /*ones*/, float* g, float beta) {
  cuda_check(tc_colsum(st, O, K, D, ldd, g, beta), "tc_colsum");
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

namespace mhost {

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

// Inputs at least this wide (Overcooked's 522 columns, MAPPO world_state rows
// of Overcooked / 27m) run the fp32 update as a GEMM chain: the per-row
// CUDA-core kernel spends most of its time on layer 1's dot products there.
constexpr int kPpoWideIn = 256;

// ff_minibatch (ppo.cpp:409-441) as a GEMM chain on the fp32-accurate 3xTF32
// tensor-core kernels (gemm_tc.cu): per branch gather the rows, dense_forward
// + act_inplace per layer (nn.hpp:108-115, 136-138), ppo_row_loss over the
// minibatch (rnn_loss: the same per-row loss the recurrent path uses), then the
// backward layer by layer with g.w = dy^T x and g.b = sum dy over all rows
// (nn.hpp:124-126) straight into p->grad in nn::pack order.
void minibatch_grad_wide(marl_ppo* p, const int32_t* idx, int64_t M) {
  marl_rollout* r = p->ro;
  cudaStream_t st = p->h->stream;
  const int W = r->width, W2 = 2 * W, relu = r->relu;
  const bool stack = !r->centralized;  // IPPO: both branches read the same rows
  const int in[2] = {r->in_dim, r->critic_in}, out[2] = {r->n_act, 1};
  p->rnn_blocks = rnn_loss_blocks(M);
  WideStage sg{};
  sg.pa = r->params;
  sg.pc = r->params + r->n_actor;
  sg.Pa = p->Pa;
  sg.Pc = p->Pc;
  sg.qa = p->wq[0];
  sg.qc = p->wq[1];
  sg.W = W;
  sg.in_a = in[0];
  sg.in_c = in[1];
  sg.ldx = p->wldx[0];
  sg.w1s = stack ? p->w1s : nullptr;
  sg.bias = p->wbias;
  wide_stage(sg, st);
  struct Ff {  // one branch's layers in nn::pack order (aligned copy / gradient)
    float *w1, *b1, *w2, *b2, *w3, *b3;
  };
  auto ff = [&](float* q, int br) {
    Ff f;
    f.w1 = q;
    f.b1 = f.w1 + size_t(W) * in[br];
    f.w2 = f.b1 + W;
    f.b2 = f.w2 + W * W;
    f.w3 = f.b2 + W;
    f.b3 = f.w3 + out[br] * W;
    return f;
  };
  const Ff q[2] = {ff(p->wq[0], 0), ff(p->wq[1], 1)};
  const Ff g[2] = {ff(p->grad, 0), ff(p->grad + p->Pa, 1)};
  float *h1 = p->wh1, *h2 = p->wh2, *d1 = p->wd1, *d2 = p->wd2;
  if (M > 0) {  // forward with cache, both branches
    for (int br = 0; br < (stack ? 1 : 2); ++br)
      ppo_gather_rows(br == 0 ? r->b.obs : r->b.critic_in, idx, M, in[br], p->wx[br], p->wldx[br], st);
    if (stack) {
      gemm_nt(st, M, W2, in[0], p->wx[0], p->wldx[0], p->w1s, p->wldx[0], h1, W2, 0.0f);
    } else {
      for (int br = 0; br < 2; ++br)
        gemm_nt(st, M, W, in[br], p->wx[br], p->wldx[br], q[br].w1, in[br], h1 + br * W, W2, 0.0f);
    }
    wide_bias_act(h1, M, W2, p->wbias, relu, st);
    for (int br = 0; br < 2; ++br) gemm_nt(st, M, W, W, h1 + br * W, W2, q[br].w2, W, h2 + br * W, W2, 0.0f);
    wide_bias_act(h2, M, W2, p->wbias + W2, relu, st);
    for (int br = 0; br < 2; ++br) {
      gemm_nt(st, M, out[br], W, h2 + br * W, W2, q[br].w3, W, p->wy[br], out[br], 0.0f);
      rnn_bias_act(p->wy[br], M, out[br], q[br].b3, false, relu, st);
    }
  }
  RnnSeqArgs la{};  // ppo_row_loss reads both branches' head outputs
  la.n_act = r->n_act;
  la.ca.y = p->wy[0];
  la.ca.dy = p->wdy[0];
  la.cc.y = p->wy[1];
  la.cc.dy = p->wdy[1];
  rnn_loss(la, idx, M, r->b, p->mbst, p->cfg.clip_eps, p->cfg.ent_coef, p->cfg.vf_coef, p->spart_a, p->spart_c,
           p->flags + 1, st);
  // backward: head, layer 2, layer 1; g.w = dy^T x over all rows, g.b = sum dy
  for (int br = 0; br < 2; ++br) {
    const float* dy = p->wdy[br];
    wide_grad_colsum(p->wdy[br], nullptr, M, out[br], relu, p->wpart, out[br], g[br].b3, nullptr, st);
    if (M == 0) continue;
    gemm_tn(st, out[br], W, M, dy, out[br], h2 + br * W, W2, g[br].w3, 0.0f);
    gemm_nn(st, M, W, out[br], dy, out[br], q[br].w3, W, d2 + br * W, W2, 0.0f);
  }
  wide_grad_colsum(d2, h2, M, W2, relu, p->wpart, W, g[0].b2, g[1].b2, st);
  for (int br = 0; br < 2 && M > 0; ++br) {
    gemm_tn(st, W, W, M, d2 + br * W, W2, h1 + br * W, W2, g[br].w2, 0.0f);
    gemm_nn(st, M, W, W, d2 + br * W, W2, q[br].w2, W, d1 + br * W, W2, 0.0f);
  }
  wide_grad_colsum(d1, h1, M, W2, relu, p->wpart, W, g[0].b1, g[1].b1, st);
  if (M == 0) {
    for (int br = 0; br < 2; ++br)
      for (float* w : {g[br].w1, g[br].w2, g[br].w3})
        cuda_check(cudaMemsetAsync(w, 0, size_t(W) * size_t(w == g[br].w1 ? in[br] : w == g[br].w2 ? W : out[br]) * 4, st),
                   "cudaMemsetAsync");
  } else if (stack) {  // one dW1 product for both branches, then each branch's rows into place
    gemm_tn(st, W2, in[0], M, d1, W2, p->wx[0], p->wldx[0], p->wg1, 0.0f);
    for (int br = 0; br < 2; ++br)
      cuda_check(cudaMemcpyAsync(g[br].w1, p->wg1 + size_t(br) * W * in[0], size_t(W) * in[0] * 4,
                                 cudaMemcpyDeviceToDevice, st),
                 "cudaMemcpyAsync");
  } else {
    for (int br = 0; br < 2; ++br)
      gemm_tn(st, W, in[br], M, d1 + br * W, W2, p->wx[br], p->wldx[br], g[br].w1, 0.0f);
  }
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
  ppo_adv_stats(p->ro->b, idx, M, p->adv_part, p->adv_part2, p->adv_g, p->mbst, st, red,
                p->tc ? p->rows_rec : nullptr, p->adv_gath);
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
    a.obs_bf = p->obs_bf;
    a.rec = p->rows_rec;
    a.st = p->mbst;
    a.err = p->flags + 1;
    a.in = r->in_dim;
    a.kx = ppo_tc_kx(r->in_dim);
    a.n_act = r->n_act;
    a.relu = r->relu;
    a.clip_eps = p->cfg.clip_eps;
    a.ent_coef = p->cfg.ent_coef;
    a.vf_coef = p->cfg.vf_coef;
    ppo_update_tc(a, p->grid_a, st);
  } else if (p->wide) {
    minibatch_grad_wide(p, idx, M);
  } else {
    ppo_branch(branch_args(p, true, idx, M), true, p->grid_a, st);
    ppo_branch(branch_args(p, false, idx, M), false, p->grid_c, st);
  }
  if (!p->wide) {
    ppo_grad_reduce(p->gpart_a, p->grid_a, p->Pa, p->grad, st);
    ppo_grad_reduce(p->gpart_c, p->grid_c, p->Pc, p->grad + p->Pa, st);
  }
  after_launch();
  if (p->hook) {  // the data-parallel exchange: gradient and loss sums over the ranks
    ppo_stats_fold(p->spart_a, p->wide ? p->rnn_blocks : p->grid_a, st);
    ppo_stats_fold(p->spart_c, p->wide ? p->rnn_blocks : p->grid_c, st);
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
  const RnnWPtrs w = rnn_weights(branch == 0 ? r->params : p->rnn_critic_w, in, F, H, out);
  const int T = r->T;
  const int64_t Kc = int64_t(T) * Mc;
  RnnStepArgs a{};
  a.M = Mc;
  a.R = r->R;
  a.in = 0;  // sq_gather: h_prev only (x is gathered for all steps at once)
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
  // everything but the recurrence runs once over all T x Mc (t, row) pairs (a
  // row's result does not depend on how many rows share its GEMM): the x
  // gather, embed, the GRU's input path gx = e.[Wz;Wr;Wn]^T ...
  rnn_seq_x_gather(rows, Mc, T, r->R, in, a.src, c.x, st);
  gemm_nt(st, Kc, F, in, c.x, in, w.we, in, c.e, F, 0.0f);
  rnn_bias_act(c.e, Kc, F, w.be, true, r->relu, st);
  float* gx = c.daz;  // [Kc][3H] inside the backward's [Kc][4H] buffer, unused until then
  gemm_nt(st, Kc, 3 * H, F, c.e, F, w.wx, F, gx, 3 * H, 0.0f);
  // ... the recurrence per step: gh = h_prev.[Uz;Ur;Un]^T and the gates, which
  // also write the next step's h_prev (apply_reset at t+1) ...
  for (int t = 0; t < T; ++t) {
    const size_t k0 = size_t(t) * size_t(Mc);
    a.t = t;
    a.hprev = c.h + k0 * H;
    a.z = c.z + k0 * H;
    a.r = c.r + k0 * H;
    a.c = c.c + k0 * H;
    a.ah = c.ah + k0 * H;
    a.hn = c.hn + k0 * H;
    a.hnext = t + 1 < T ? c.h + (k0 + Mc) * H : nullptr;
    if (t == 0) rnn_step_gather(a, st);
    gemm_nt(st, Mc, 3 * H, H, a.hprev, H, w.uh, H, p->rnn_gh, 3 * H, 0.0f);
    rnn_gates(a, gx + k0 * 3 * H, p->rnn_gh, st);
  }
  // ... then post and head over all pairs
  gemm_nt(st, Kc, F, H, c.hn, H, w.wp, H, c.p, F, 0.0f);
  rnn_bias_act(c.p, Kc, F, w.bp, true, r->relu, st);
  gemm_nt(st, Kc, out, F, c.p, F, w.wh, F, c.y, out, 0.0f);
  rnn_bias_act(c.y, Kc, out, w.bh, false, r->relu, st);
  after_launch();
}

// rnn_seq_backward (actor_critic.hpp:164-196) of one branch over a chunk, then
// its weight gradients (matmul_tn over every (t, row)) into G in pack order.
// D4 = [daz | dar | dah | dac] per (t, row): the hidden path [Uz;Ur;Un] reads
// columns 0..3H-1 as one operand, the input path [Wz;Wr;Wn] reads 0..2H-1 and dac.
void rnn_chunk_backward(marl_ppo* p, int branch, const int32_t* rows, int64_t Mc, float* G, bool accumulate) {
  marl_rollout* r = p->ro;
  cudaStream_t st = p->h->stream;
  const RnnCache& c = branch == 0 ? p->rca : p->rcc;
  const int in = branch == 0 ? r->in_dim : r->critic_in, out = branch == 0 ? r->n_act : 1, F = r->F, H = r->H;
  const RnnWPtrs w = rnn_weights(branch == 0 ? r->params : p->rnn_critic_w, in, F, H, out);
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
  float* d4 = c.daz;
  // head and post over all (t, row) first: dzp = (dy . Wh) * act'(p) and the
  // post layer's share of each step's dh, dzp . Wp -- [Kc][H] aliased onto the
  // front of d4: step t reads its rows [t Mc H, (t+1) Mc H) before writing d4's
  // [4 t Mc H, 4 (t+1) Mc H), and the earlier steps' rows it still needs lie below
  float* dhp = d4;
  gemm_nn(st, Kc, F, out, c.dy, out, w.wh, F, c.dzp, F, 0.0f);
  rnn_act_grad(c.dzp, c.p, Kc * F, r->relu, st);
  gemm_nn(st, Kc, H, F, c.dzp, F, w.wp, H, dhp, H, 0.0f);
  // the recurrence per step: gru_backward (folding in the post share and the
  // previous step's episode cut), then dh_prev += [daz|dar|dah] . [Uz;Ur;Un]
  for (int t = T - 1; t >= 0; --t) {
    const size_t k0 = size_t(t) * size_t(Mc);
    a.t = t;
    a.hprev = c.h + k0 * H;
    a.z = c.z + k0 * H;
    a.r = c.r + k0 * H;
    a.c = c.c + k0 * H;
    a.ah = c.ah + k0 * H;
    a.dhp = dhp + k0 * H;
    a.carry = t == T - 1 ? 1 : 2;
    float* d4t = d4 + k0 * 4 * H;
    rnn_gru_bwd(a, dh, d4t, dh, st);
    gemm_nn(st, Mc, H, 3 * H, d4t, 4 * H, w.uh, H, dh, H, 1.0f);
  }
  // the embed path over all pairs: dze = ([daz|dar] . [Wz;Wr] + dac . Wn) * act'(e)
  gemm_nn(st, Kc, F, 2 * H, d4, 4 * H, w.wx, F, c.dze, F, 0.0f);
  gemm_nn(st, Kc, F, H, d4 + 3 * H, 4 * H, w.wx + size_t(2) * H * F, F, c.dze, F, 1.0f);
  rnn_act_grad(c.dze, c.e, Kc * F, r->relu, st);
  const float beta = accumulate ? 1.0f : 0.0f;
  const float* ones = p->rnn_ones;
  gemm_tn(st, F, in, Kc, c.dze, F, c.x, in, G, beta);  // embed
  G += size_t(F) * in;
  colsum(st, F, Kc, c.dze, F, ones, G, beta);
  G += F;
  gemm_tn(st, 2 * H, F, Kc, d4, 4 * H, c.e, F, G, beta);  // wz, wr
  G += size_t(2) * H * F;
  gemm_tn(st, H, F, Kc, d4 + 3 * H, 4 * H, c.e, F, G, beta);  // wn
  G += size_t(H) * F;
  gemm_tn(st, 3 * H, H, Kc, d4, 4 * H, c.h, H, G, beta);  // uz, ur, un
  G += size_t(3) * H * H;
  colsum(st, 2 * H, Kc, d4, 4 * H, ones, G, beta);  // bzx, brx
  G += 2 * H;
  colsum(st, H, Kc, d4 + 3 * H, 4 * H, ones, G, beta);  // bnx
  G += H;
  colsum(st, 3 * H, Kc, d4, 4 * H, ones, G, beta);  // bzh, brh, bnh
  G += 3 * H;
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
  ppo_adv_stats(r->b, p->rnn_flat, K, p->adv_part, p->adv_part2, p->adv_g, p->mbst, st, {}, nullptr,
                p->adv_gath);
  p->rnn_critic_w = rnn_critic_params(r, st);  // the parameters are fixed within the minibatch
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
  const bool by_rows = p->recurrent || p->wide;  // loss partials of rnn_loss's blocks
  a.n_actor_parts = p->hook ? 1 : (by_rows ? p->rnn_blocks : p->grid_a);  // folded + all-reduced into row 0
  a.n_critic_parts = p->hook ? 1 : (by_rows ? p->rnn_blocks : p->grid_c);
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

// the tcgen05 step gathers bf16 observation rows: convert the window's rows once
void tc_obs(marl_ppo* p) {
  if (!p->tc) return;
  const marl_rollout* r = p->ro;
  PpoTcPack k{};
  k.obs = r->b.obs;
  k.active = r->b.active;
  k.adv = r->b.adv;
  k.old_logp = r->b.logp;
  k.vtarg = r->b.vtarg;
  k.old_value = r->b.value;
  k.actions = r->b.actions;
  k.legal = r->b.legal;
  k.rows = int64_t(r->T) * r->R;
  k.in = r->in_dim;
  k.kx = ppo_tc_kx(r->in_dim);
  k.n_act = r->n_act;
  k.obs_bf = p->obs_bf;
  k.rec = p->rows_rec;
  ppo_tc_pack(k, p->h->stream);
  after_launch();
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
  tc_obs(p);
  const int64_t adam_t0 = p->adam_t;
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
  // AdamState::t counts only the updates adam_update applied (nn.hpp:420-426):
  // minibatch_apply advanced it for every launched minibatch, including those
  // the device skipped after a DivergenceError
  p->adam_t = adam_t0 + n_mb;
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
    } else if (std::max(r->in_dim, r->critic_in) >= kPpoWideIn && !std::getenv("MARL_PPO_ROW_KERNEL")) {
      p->wide = true;  // MARL_PPO_ROW_KERNEL=1 keeps the per-row kernels (A/B knob)
      p->grid_a = p->grid_c = rnn_loss_blocks(p->per);
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
    const bool no_parts = p->recurrent || p->wide;
    ar.add(&p->gpart_a, no_parts ? 1 : size_t(p->grid_a) * size_t(p->Pa));
    ar.add(&p->gpart_c, no_parts ? 1 : size_t(p->grid_c) * size_t(p->Pc));
    if (p->wide) {
      const size_t M = size_t(p->per), W = size_t(r->width);
      for (int br = 0; br < 2; ++br) {
        const int in = br == 0 ? r->in_dim : r->critic_in;
        p->wldx[br] = (in + 3) / 4 * 4;  // 16-byte rows: four-float copies in the GEMMs' staging
        if (br == 0 || centralized) ar.add(&p->wx[br], M * size_t(p->wldx[br]));
        ar.add(&p->wy[br], M * size_t(br == 0 ? r->n_act : 1));
        ar.add(&p->wdy[br], M * size_t(br == 0 ? r->n_act : 1));
        ar.add(&p->wq[br], size_t(br == 0 ? p->Pa : p->Pc));
      }
      for (float** q : {&p->wh1, &p->wh2, &p->wd1, &p->wd2}) ar.add(q, M * 2 * W);
      if (!centralized) {
        ar.add(&p->w1s, 2 * W * size_t(p->wldx[0]));
        ar.add(&p->wg1, 2 * W * size_t(r->in_dim));
      }
      ar.add(&p->wbias, 4 * W);
      ar.add(&p->wpart, size_t(wide_part_floats(p->per, 2 * r->width)));
    }
    ar.add(&p->spart_a, size_t(p->grid_a) * 6);
    ar.add(&p->spart_c, size_t(p->grid_c) * 6);
    ar.add(&p->adv_part, size_t(std::max(nb, ppo_stat_blocks(rnn_K))) * 2);
    ar.add(&p->adv_part2, size_t(std::max(nb, ppo_stat_blocks(rnn_K))));
    ar.add(&p->adv_gath, size_t(std::max<int64_t>(p->per, rnn_K)));  // the minibatch's (adv, active) pairs
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
    if (p->tc) {
      ar.add(&p->obs_bf, size_t(r->T) * size_t(r->R) * size_t(ppo_tc_kx(r->in_dim)));
      ar.add(&p->rows_rec, size_t(r->T) * size_t(r->R));
    }
    ar.add(&p->ep_dev, 3);
    if (p->sharded) {
      p->cmp_scratch_bytes = ppo_compact_scratch_bytes(p->per);
      ar.add(&p->cmp_tmp, size_t(p->per));
      ar.add(&p->cmp_out, size_t(p->per));
      ar.add(&p->cmp_count, 1);
      ar.add(&p->cmp_scratch, p->cmp_scratch_bytes);
    }
    ar.commit();
    if (p->wide && !centralized) p->wx[1] = p->wx[0];  // IPPO: the critic reads the actor's rows
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

int marl_ppo_tensor_core_update(const marl_ppo* p, int* out) {
  return guarded([&] {
    if (!p || !out) raise(MARL_ERR_CONTRACT, "marl_ppo_tensor_core_update: NULL argument");
    *out = p->tc ? 1 : 0;
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
    tc_obs(p);
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
    // with an all-reduce hook, minibatch_grad already folded the per-CTA rows
    // into row 0 (and summed it over the ranks): read that row only
    // (the wide path's loss rows are rnn_loss's blocks of this minibatch)
    const int na = p->hook ? 1 : p->wide ? p->rnn_blocks : p->grid_a;
    const int nc = p->hook ? 1 : p->wide ? p->rnn_blocks : p->grid_c;
    double s[6] = {0, 0, 0, 0, 0, 0}, vt = 0.0;
    for (int c = 0; c < na; ++c)
      for (int j = 0; j < 6; ++j) s[j] += sa[size_t(c) * 6 + j];
    for (int c = 0; c < nc; ++c) vt += sc[size_t(c) * 6 + 1];
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
    if (p->recurrent && fn)
      raise(MARL_ERR_CONTRACT, "ppo: the data-parallel update covers feed-forward policies only (recurrent=true)");
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
    if (p->recurrent)
      raise(MARL_ERR_CONTRACT, "ppo: the data-parallel update covers feed-forward policies only (recurrent=true)");
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
