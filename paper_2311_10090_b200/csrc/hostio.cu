// Host-buffer steps: the terminal observations of the envs that finished
// (StepBatchResult::final_obs is "valid where finished", vector_env.hpp:31)
// go straight from HBM into a mapped, pinned host buffer -- one warp per env,
// 16-byte stores over PCIe when the row allows, nothing for the ~95 % of
// envs that did not finish.  The other views are dense and use cudaMemcpy.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace marl_b200 {
namespace {

__global__ void gather_finished_rows_kernel(const uint8_t* __restrict__ finished, int64_t n,
                                            const float* __restrict__ src, float* dst, int64_t row) {
  const int64_t i = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= n || !finished[i]) return;
  const int lane = threadIdx.x & 31;
  const float* s = src + i * row;
  float* d = dst + i * row;
  if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0 && row % 4 == 0) {
    for (int64_t q = lane; q < row / 4; q += 32)
      reinterpret_cast<float4*>(d)[q] = reinterpret_cast<const float4*>(s)[q];
  } else {
    for (int64_t q = lane; q < row; q += 32) d[q] = s[q];
  }
}

}  // namespace

void launch_gather_finished_rows(const uint8_t* finished, int64_t n, const float* src, float* dst, int64_t row,
                                 cudaStream_t st) {
  if (n <= 0) return;
  gather_finished_rows_kernel<<<unsigned((n + 7) / 8), 256, 0, st>>>(finished, n, src, dst, row);
  ++g_launches;
}

}  // namespace marl_b200
