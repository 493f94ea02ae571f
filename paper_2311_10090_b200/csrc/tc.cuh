// tcgen05 / TMEM / UMMA helpers shared by the tensor-core kernels (rollout.cu,
// ppo_tc.cu): shared-memory descriptors for the canonical no-swizzle layouts,
// the kind::f16 instruction descriptor, MMA issue / commit, mbarrier waits,
// TMEM loads and bf16 packing.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace marl_b200 {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (n, k) in a K-major no-swizzle canonical [N x K] bf16 tile
__host__ __device__ __forceinline__ uint32_t canon_off(int n, int k, int K) {
  return uint32_t((n >> 3) * ((K >> 3) * 128) + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t desc_raw(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // descriptor version 1 (sm_100); base offset 0; layout SWIZZLE_NONE
  return d;
}

// K-major operand [rows x K] (canon_off layout), the K slice starting at k0.
__device__ __forceinline__ uint64_t umma_desc(const void* tile, int K, int k0) {
  const uint32_t addr = smem_u32(tile) + uint32_t(k0 >> 3) * 128u;  // K slice start
  return desc_raw(addr, 128u, uint32_t(K >> 3) * 128u);
}

// The same [rows x F] canon_off tile read TRANSPOSED, as an MN-major operand
// whose MN index is the feature f (groups of 8 features 128 B apart) and
// whose K index is the row (groups of 8 rows (F/8)*128 B apart); the K slice
// starts at row r0 (a multiple of 16) -- cute's Major-MN INTERLEAVE layout
// ((T,1,m),(8,k)):((1,T,SBO),(1T,LBO)).
__device__ __forceinline__ uint64_t umma_desc_mn(const void* tile, int F, int r0, int f0 = 0) {
  const uint32_t rg = uint32_t(F >> 3) * 128u;
  const uint32_t addr = smem_u32(tile) + uint32_t(r0 >> 3) * rg + uint32_t(f0 >> 3) * 128u;
  return desc_raw(addr, rg, 128u);
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D, M x N; a_mn / b_mn:
// the operand is MN-major (bits 15 / 16).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn = 0, int b_mn = 0) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Wait for the phase with the given parity to complete.  The suspend-time
// hint lets the waiting warps sleep in the barrier unit instead of spinning
// (the spin loop was ~8 % of the policy kernel's issued instructions).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 consecutive fp32 columns of this thread's TMEM lane (two x16 loads, one wait).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float tanh_fast(float x) {  // MUFU.TANH: ~2^-11 relative, below bf16's 2^-8
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 8 fp32 values at K offset k0 (a multiple of 8) -> one 16-byte chunk.
__device__ __forceinline__ void put8(uint8_t* tile, int K, int row, int k0, const float* v) {
  uint4 q;
  q.x = pack_bf16(v[0], v[1]);
  q.y = pack_bf16(v[2], v[3]);
  q.z = pack_bf16(v[4], v[5]);
  q.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(tile + canon_off(row, k0, K)) = q;
}

// Row `row` of an activation operand: 16 fp32 values at K offset k0 -> bf16
// into the canonical tile (two 16-byte chunks).
__device__ __forceinline__ void put16(uint8_t* tile, int K, int row, int k0, const float* v) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint4 q;
    q.x = pack_bf16(v[8 * c + 0], v[8 * c + 1]);
    q.y = pack_bf16(v[8 * c + 2], v[8 * c + 3]);
    q.z = pack_bf16(v[8 * c + 4], v[8 * c + 5]);
    q.w = pack_bf16(v[8 * c + 6], v[8 * c + 7]);
    *reinterpret_cast<uint4*>(tile + canon_off(row, k0 + 8 * c, K)) = q;
  }
}


}  // namespace
}  // namespace marl_b200
