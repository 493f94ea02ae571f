// Device-side Env::validate_actions (env.cpp:7-14) for caller-supplied action
// batches: any out-of-space action records a ContractError (lowest flat index
// wins) and freezes the batch -- every step kernel returns immediately while
// err[0] != 0 -- so a rejected batch leaves the state untouched, as the
// reference's exception does.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.h"

namespace marl_b200 {

unsigned long long g_launches = 0;
int g_grid_cap = 0;

namespace {
__global__ void validate_kernel(const int32_t* __restrict__ actions, int64_t total, int A,
                                const int32_t* __restrict__ n_actions, int* err) {
  int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int a = int(idx % A);
  int32_t v = actions[idx];
  if (v < 0 || v >= __ldg(n_actions + a)) {
    atomicMin(err + 1, int(min64(idx, 0x7fffffff)));
    atomicExch(err + 2, v);
    atomicExch(err + 0, 3);
  }
}
}  // namespace

namespace {
__global__ void validate_box_kernel(const float* __restrict__ actions, int64_t total, int A,
                                    const int32_t* __restrict__ flat, int* err) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // (env, agent)
  if (idx >= total) return;
  const int a = int(idx % A), n = __ldg(flat + a);
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const float v = actions[idx * kBoxActDim + k];
    ok = ok && v >= 0.0f && v <= 1.0f && isfinite(v);
  }
  if (!ok) {
    atomicMin(err + 1, int(min64(idx, 0x7fffffff)));
    atomicExch(err + 0, 3);
  }
}
}  // namespace

void launch_validate_box(const float* actions, int64_t n, int A, const int32_t* flat_size_dev, int* err,
                         cudaStream_t st) {
  const int64_t total = n * A;
  validate_box_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(actions, total, A, flat_size_dev, err);
  ++g_launches;
}

void launch_validate(const int32_t* actions, int64_t n, int A, const int32_t* n_actions_dev, int* err,
                     cudaStream_t st) {
  int64_t total = n * A;
  validate_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(actions, total, A, n_actions_dev, err);
  ++g_launches;
}

namespace {
// out[i][*] = the env's obs segments back to back; one warp per env.
__global__ void obs_gather_kernel(const float* __restrict__ obs, int64_t n, int row_floats,
                                  const int32_t* __restrict__ seg_src, const int32_t* __restrict__ seg_len, int n_seg,
                                  int width, float* __restrict__ out) {
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const float* src = obs + size_t(i) * row_floats;
  float* dst = out + size_t(i) * width;
  int off = 0;
  for (int sgm = 0; sgm < n_seg; ++sgm) {
    const int len = seg_len[sgm], from = seg_src[sgm];
    for (int k = lane; k < len; k += 32) dst[off + k] = src[from + k];
    off += len;
  }
}
}  // namespace

void launch_obs_gather(const float* obs, int64_t n, int row_floats, const int32_t* seg_src, const int32_t* seg_len,
                       int n_seg, int width, float* out, cudaStream_t st) {
  obs_gather_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, st>>>(obs, n, row_floats, seg_src, seg_len, n_seg,
                                                                    width, out);
  ++g_launches;
}

}  // namespace marl_b200
