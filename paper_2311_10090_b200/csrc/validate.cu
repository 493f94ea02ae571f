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

void launch_validate(const int32_t* actions, int64_t n, int A, const int32_t* n_actions_dev, int* err,
                     cudaStream_t st) {
  int64_t total = n * A;
  validate_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(actions, total, A, n_actions_dev, err);
  ++g_launches;
}

}  // namespace marl_b200
