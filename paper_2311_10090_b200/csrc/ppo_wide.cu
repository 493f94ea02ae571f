// The wide-input fp32 PPO update's staging and elementwise kernels
// (ff_minibatch as a GEMM chain, ppo_host.cpp minibatch_grad_wide).
//
// Both branches' hidden layers sit side by side in [M][2W] buffers (actor
// columns 0..W-1, critic W..2W-1), so each elementwise pass -- bias + act
// (dense_forward + act_inplace, nn.hpp:108-115, 136-138), the activation
// gradient and the bias gradient g.b = sum dy (nn.hpp:124-126) -- is one
// launch for both branches.  The GEMMs themselves are gemm_tc.cu's 3xTF32
// tcgen05 kernels.  Bias gradients are fixed-order reductions (row blocks of
// kWideRows, then a tree over the blocks), so the update is deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {

namespace {

constexpr int kWideRows = 32;  // rows per column-sum block

__device__ __forceinline__ float wide_act(float v, int relu) { return relu ? (v > 0.0f ? v : 0.0f) : tanhf(v); }
__device__ __forceinline__ float wide_act_grad(float g, float y, int relu) {  // grad *= act_grad_from_output(y)
  return __fmul_rn(g, relu ? (y > 0.0f ? 1.0f : 0.0f) : __fsub_rn(1.0f, __fmul_rn(y, y)));
}

// 16-byte aligned copies of both branches' parameters, the stacked layer-1
// matrix [2W][ldx] (IPPO: one product serves both branches) and the stacked
// biases [b1a | b1c | b2a | b2c]
__global__ void wide_stage_kernel(WideStage s) {
  const int W = s.W;
  const int64_t na = s.Pa, nc = s.Pc, nw = s.w1s ? int64_t(2 * W) * s.ldx : 0, nb = 4 * W;
  const int64_t total = na + nc + nw + nb;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    if (e < na) {
      s.qa[e] = __ldg(s.pa + e);
    } else if (e < na + nc) {
      s.qc[e - na] = __ldg(s.pc + (e - na));
    } else if (e < na + nc + nw) {
      const int64_t q = e - na - nc;
      const int o = int(q / s.ldx), i = int(q - int64_t(o) * s.ldx);
      const bool crit = o >= W;
      const int in = crit ? s.in_c : s.in_a;
      const float* w1 = crit ? s.pc : s.pa;
      s.w1s[q] = i < in ? __ldg(w1 + int64_t(o - (crit ? W : 0)) * in + i) : 0.0f;
    } else {
      const int q = int(e - na - nc - nw), layer = q / (2 * W), c = q % (2 * W);
      const bool crit = c >= W;
      const int in = crit ? s.in_c : s.in_a, o = c - (crit ? W : 0);
      const float* p = crit ? s.pc : s.pa;
      const int64_t off = layer == 0 ? int64_t(W) * in : int64_t(W) * in + W + int64_t(W) * W;
      s.bias[q] = __ldg(p + off + o);
    }
  }
}

template <int V>
__global__ void wide_bias_act_kernel(float* __restrict__ y, int64_t n, int N, const float* __restrict__ b, int relu) {
  const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * V;
  if (q >= n) return;
  const int c = int(q % N);
  if constexpr (V == 4) {
    float4 v = *reinterpret_cast<float4*>(y + q);
    v.x = wide_act(__fadd_rn(v.x, __ldg(b + c)), relu);
    v.y = wide_act(__fadd_rn(v.y, __ldg(b + c + 1)), relu);
    v.z = wide_act(__fadd_rn(v.z, __ldg(b + c + 2)), relu);
    v.w = wide_act(__fadd_rn(v.w, __ldg(b + c + 3)), relu);
    *reinterpret_cast<float4*>(y + q) = v;
  } else {
    y[q] = wide_act(__fadd_rn(y[q], __ldg(b + c)), relu);
  }
}

// D = D * act'(H) in place (act_backward, nn.hpp:140-142; skipped when h is
// null) and the column partial sums of the result over a block of kWideRows rows
__global__ void wide_grad_colsum_kernel(float* __restrict__ d, const float* __restrict__ h, int64_t M, int N,
                                        int relu, float* __restrict__ part) {
  const int c = threadIdx.x;
  if (c >= N) return;
  const int64_t r0 = int64_t(blockIdx.x) * kWideRows, r1 = min(M, r0 + kWideRows);
  float s = 0.0f;
  for (int64_t r = r0; r < r1; ++r) {
    float g = d[r * N + c];
    if (h) {
      g = wide_act_grad(g, __ldg(h + r * N + c), relu);
      d[r * N + c] = g;
    }
    s = __fadd_rn(s, g);
  }
  part[int64_t(blockIdx.x) * N + c] = s;
}

// column c's sum over the row blocks in a fixed order (strided per thread,
// then a tree), to dst0[c] for c < split, dst1[c - split] otherwise
__global__ void wide_fold_kernel(const float* __restrict__ part, int nparts, int N, int split, float* dst0,
                                 float* dst1) {
  __shared__ float sh[256];
  const int c = blockIdx.x, t = threadIdx.x;
  float s = 0.0f;
  for (int q = t; q < nparts; q += 256) s = __fadd_rn(s, part[int64_t(q) * N + c]);
  sh[t] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) sh[t] = __fadd_rn(sh[t], sh[t + w]);
    __syncthreads();
  }
  if (t == 0) {
    if (c < split)
      dst0[c] = sh[0];
    else
      dst1[c - split] = sh[0];
  }
}

}  // namespace

int64_t wide_part_floats(int64_t M, int N) { return ((M + kWideRows - 1) / kWideRows + 1) * int64_t(N); }

void wide_stage(const WideStage& s, cudaStream_t st) {
  wide_stage_kernel<<<4 * 148, 256, 0, st>>>(s);
  ++g_launches;
}

void wide_bias_act(float* y, int64_t M, int N, const float* b, int relu, cudaStream_t st) {
  const int64_t n = M * N;
  if (n <= 0) return;
  if (N % 4 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0)
    wide_bias_act_kernel<4><<<unsigned((n / 4 + 255) / 256), 256, 0, st>>>(y, n, N, b, relu);
  else
    wide_bias_act_kernel<1><<<unsigned((n + 255) / 256), 256, 0, st>>>(y, n, N, b, relu);
  ++g_launches;
}

void wide_grad_colsum(float* d, const float* h, int64_t M, int N, int relu, float* part, int split, float* dst0,
                      float* dst1, cudaStream_t st) {
  const int nparts = int(std::max<int64_t>(1, (M + kWideRows - 1) / kWideRows));
  const int tx = (N + 31) / 32 * 32;
  if (M > 0) {
    wide_grad_colsum_kernel<<<unsigned(nparts), tx, 0, st>>>(d, h, M, N, relu, part);
  } else {
    cudaMemsetAsync(part, 0, size_t(N) * 4, st);
  }
  wide_fold_kernel<<<unsigned(N), 256, 0, st>>>(part, nparts, N, split, dst0, dst1);
  g_launches += 2;
}

}  // namespace marl_b200
