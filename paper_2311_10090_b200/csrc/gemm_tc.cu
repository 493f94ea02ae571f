// fp32-accurate GEMMs on the 5th-generation tensor cores (3xTF32 on tcgen05)
// for the recurrent policy's per-step and BPTT contractions (rollout_host.cpp,
// ppo_host.cpp: the embed / GRU / post / head layers of the reference's
// RnnBranch, actor_critic.hpp:74-200, nn.hpp:200-318, and their weight
// gradients).  These are tall-skinny GEMMs -- rows x (18..1024) x (1..384) --
// bound by HBM, so the tensor pipe has room for the split-precision scheme
// that keeps them at fp32 accuracy:
//     a = a_hi + a_lo   (a_hi = a with its low 13 mantissa bits cleared, an
//                        exact tf32 value; a_lo = a - a_hi, exact in fp32)
//     a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi      (fp32 accumulation in TMEM)
// The dropped a_lo.b_lo term and the tf32 rounding of the lo parts are
// ~2^-22 relative to each product: the same order as fp32 rounding.
//
// One kernel serves every operand layout: C[M x N] (+)= A[M x K] . B'[N x K]^T
// with element strides A(m, k) = A[m*sam + k*sak], B'(n, k) = B[n*sbn + k*sbk],
// so row-major, transposed and "sum over rows" (weight-gradient) forms are the
// same code.  A CTA owns a 128-row M tile and an N tile of up to 128 columns
// (tcgen05.mma.cta_group::1.kind::tf32, M = 128, accumulators in TMEM).  K
// advances in chunks of 16 (32 for split-K grids): four producer warps stream
// the raw fp32 chunks of A and B' into a ring of NS shared-memory stages with
// cp.async (16-, 8- or 4-byte copies by alignment, zero-filled outside the
// matrix) and signal each stage's mbarrier when their copies land; four
// splitter warps turn a landed stage into the hi / lo images in the canonical
// no-swizzle K-major layout (two tile sets, so the split of chunk c + 1
// overlaps the MMAs on chunk c) and free the stage; one thread of a ninth warp
// issues the 3 x KC/8 MMAs per chunk and commits them to the tile set's
// mbarrier; the accumulator rows come back with tcgen05.ld.  No CTA-wide
// barrier inside the K loop (the earlier lockstep kernel, kept behind
// MARL_GEMM_LOCKSTEP=1, synchronised all threads twice per chunk: the
// warp-specialised one is 10-20 % faster on every shape measured,
// scripts/gemm_shapes.py).  Long reductions (the weight
// gradients sum over every (t, row)) split K across CTAs into per-split
// partial tiles folded in a fixed order: results are deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <mutex>

#include "common.cuh"
#include "engine.h"
#include "tc.cuh"

namespace marl_b200 {
namespace {

constexpr int kGemmM = 128;        // rows per CTA (UMMA M)
constexpr int kGemmMaxN = 128;     // columns per CTA (UMMA N <= 256)
constexpr int kGemmThreads = 256;  // two warps per TMEM lane quarter (accumulator rows 32q..32q+31)
constexpr int kGemmWarps = kGemmThreads / 32;
// Two configurations (K elements per chunk KC, CTAs per SM): grids of M x N
// tiles run KC = 16 with two 256-thread CTAs per SM; split-K grids (the weight
// gradients, a few tiles over a very long K) run KC = 32 with one CTA per SM
// and a deeper raw ring (four stages, two tile sets).
template <int KC>
__host__ __device__ constexpr int raw_pitch() { return KC + 4; }  // raw K-contiguous rows, padded against bank conflicts
constexpr int kEpiPitch = 33;  // epilogue staging rows (32 columns + 1 against bank conflicts)

// byte offset of element (r, k) in a K-major no-swizzle canonical [rows x kKC]
// 4-byte tile: 8-row x 16-byte core matrices, K neighbours 128 B apart, 8-row
// groups (kKC/4)*128 B apart
template <int KC>
__host__ __device__ __forceinline__ uint32_t canon4(int r, int k) {
  return uint32_t((r >> 3) * ((KC / 4) * 128) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// kind::tf32 instruction descriptor: tf32 A/B (format 2), fp32 D, K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// K-major operand descriptor of a canonical [rows x kKC] tile, K step k0 (multiple of 8)
template <int KC>
__device__ __forceinline__ uint64_t desc4(const void* tile, int k0) {
  return desc_raw(smem_u32(tile) + uint32_t(k0 >> 2) * 128u, 128u, (KC / 4) * 128u);
}

// cp.async of SZ bytes (4, 8 or 16), zero-filled beyond src_bytes
template <int SZ>
__device__ __forceinline__ void cp_async(void* sdst, const void* gsrc, uint32_t src_bytes) {
  if constexpr (SZ == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(sdst)), "l"(gsrc), "n"(SZ),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// How an operand X(r, k) = X[r*sr + k*sk] is staged: K-contiguous (raw rows
// [r][KC + 4]) with copies of `vec` floats, or rows-contiguous (raw
// [k][rows]) with copies of `vec` floats along r, or element by element.
struct OpLayout {
  const float* X;
  int64_t sr, sk;
  int kind;  // 0: K-contiguous, 1: rows-contiguous, 2: general (raw [r][KC + 4])
  int vec;   // floats per copy (1, 2, 4)
};

struct GemmArgs {
  OpLayout a, b;
  float* C;        // output (split == 1) ...
  float* part;     // ... or [split][M][N] partial tiles (split > 1)
  int64_t M, K, ldc;
  int N, npad;     // columns; npad: MMA N of a tile (a power of two >= 16)
  int nlog;        // log2(npad)
  int ntile;       // columns per N tile
  int split;       // K splits
  int64_t kchunk;  // K elements per split (multiple of the chunk KC)
  float beta;
  uint32_t tmem_cols;
  int ns, nt;      // raw stages, hi/lo tile sets
  uint32_t a_raw, b_raw, a_tile, b_tile;  // bytes
};

__host__ __device__ inline uint32_t raw_bytes(int rows, int kind, int KC) {
  return kind == 1 ? uint32_t(KC) * rows * 4 : uint32_t(rows) * (KC + 4) * 4;
}

// Operand staging code (compile-time, one path per kernel instance so the
// kernel stays small in the instruction cache): 0 K-contiguous with 16-byte
// copies, 1 K-contiguous (or general strides) element by element, 2
// rows-contiguous with 16-byte copies, 3 rows-contiguous element by element.
__host__ __device__ constexpr int lay_kind(int L) { return L >= 2 ? 1 : 0; }
__host__ __device__ constexpr int lay_vec(int L) { return (L == 0 || L == 2) ? 4 : 1; }

// Issue the cp.async copies of chunk [k0, k0 + KC) of rows [r0, r0 + rows)
// (valid rows < rvalid, valid k < K) into a raw stage.  rows = 1 << rlog, so
// every index split is a shift or a mask.
template <int KC, int L, bool DIRECT = false>
__device__ __forceinline__ void fetch(float* raw, const OpLayout& o, int64_t r0, int rlog, int64_t rvalid, int64_t k0,
                                      int64_t K, int tid = threadIdx.x, int nth = kGemmThreads) {
  constexpr int V = lay_vec(L);
  const int rows = 1 << rlog;
  if constexpr (lay_kind(L) == 1) {  // raw[k][r], copies along r
    const int plog = rlog - (V == 4 ? 2 : 0);  // log2(rows / V)
    for (int idx = tid; idx < (KC << plog); idx += nth) {
      const int k = idx >> plog, r = (idx & ((1 << plog) - 1)) * V;
      const int64_t gk = k0 + k, gr = r0 + r;
      int64_t nv = gk < K ? rvalid - gr : 0;
      nv = nv < 0 ? 0 : nv > V ? V : nv;
      const float* src = nv ? o.X + gr * o.sr + gk * o.sk : o.X;
      cp_async<4 * V>(raw + (k << rlog) + r, src, uint32_t(nv * 4));
    }
  } else {  // raw[r][k], copies along k
    constexpr int per_r = KC / V;
    for (int idx = tid; idx < rows * per_r; idx += nth) {
      const int r = idx / per_r, k = (idx % per_r) * V;
      const int64_t gk = k0 + k, gr = r0 + r;
      int64_t nv = gr < rvalid ? K - gk : 0;
      nv = nv < 0 ? 0 : nv > V ? V : nv;
      const float* src = nv ? o.X + gr * o.sr + gk * o.sk : o.X;
      float* dst = DIRECT ? raw + canon4<KC>(r, k) / 4 : raw + r * raw_pitch<KC>() + k;  // DIRECT: V == 4
      cp_async<4 * V>(dst, src, uint32_t(nv * 4));
    }
  }
}

// hi / lo tf32 images of v: hi = v with the low 13 mantissa bits cleared
// (exact in tf32), lo = v - hi (exact in fp32)
__device__ __forceinline__ void split_tf32(float v, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  lo = v - hi;
}

// raw stage -> hi / lo canonical tiles (four K per thread step)
template <int KC, int KIND, bool DIRECT = false>
__device__ __forceinline__ void convert(const float* raw, int rlog, uint8_t* hi, uint8_t* lo, int tid = threadIdx.x,
                                        int nth = kGemmThreads) {
  const int rows = 1 << rlog;
  for (int idx = tid; idx < rows * (KC / 4); idx += nth) {
    const int r = idx & (rows - 1), k = (idx >> rlog) * 4;  // consecutive threads take consecutive rows
    float4 v;
    if constexpr (DIRECT) {  // the raw stage is the canonical image: it serves as hi, only lo is written
      v = *reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(raw) + canon4<KC>(r, k));
      float4 h, l;
      split_tf32(v.x, h.x, l.x);
      split_tf32(v.y, h.y, l.y);
      split_tf32(v.z, h.z, l.z);
      split_tf32(v.w, h.w, l.w);
      *reinterpret_cast<float4*>(lo + canon4<KC>(r, k)) = l;
      continue;
    }
    if (KIND == 1) {  // raw[k][r]
      v = make_float4(raw[(k << rlog) + r], raw[((k + 1) << rlog) + r], raw[((k + 2) << rlog) + r],
                      raw[((k + 3) << rlog) + r]);
    } else {
      v = *reinterpret_cast<const float4*>(raw + r * raw_pitch<KC>() + k);
    }
    float4 h, l;
    split_tf32(v.x, h.x, l.x);
    split_tf32(v.y, h.y, l.y);
    split_tf32(v.z, h.z, l.z);
    split_tf32(v.w, h.w, l.w);
    *reinterpret_cast<float4*>(hi + canon4<KC>(r, k)) = h;
    *reinterpret_cast<float4*>(lo + canon4<KC>(r, k)) = l;
  }
}

template <int KC, int MINB, int AL, int BL>
__global__ void __launch_bounds__(kGemmThreads, MINB) gemm_tf32x3_kernel(GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int mt = blockIdx.x, nt = blockIdx.y, sp = blockIdx.z;
  const int64_t m0 = int64_t(mt) * kGemmM;
  const int n0 = nt * g.ntile;
  const int nvalid = min(g.ntile, g.N - n0);
  const int64_t kb = int64_t(sp) * g.kchunk, ke = min(g.K, kb + g.kchunk);
  const int nch = int((ke - kb + KC - 1) / KC);
  // smem: [tile sets: A hi, A lo, B hi, B lo] x nt, [raw stages: A, B] x ns, 2 barriers, TMEM slot
  const uint32_t set_bytes = 2 * g.a_tile + 2 * g.b_tile, stage_bytes = g.a_raw + g.b_raw;
  uint8_t* raw0 = smem + g.nt * set_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw0 + max(g.ns * stage_bytes, uint32_t(kGemmWarps * 32 * kEpiPitch * 4)));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 2; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + q)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(g.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  OpLayout bo = g.b;
  bo.X = g.b.X + int64_t(n0) * g.b.sr;
  int wstage = 0;           // the stage the next issued chunk lands in
  auto issue = [&](int c) {  // raw chunk c -> stage c % ns (one commit group per call)
    if (c < nch) {
      float* ra = reinterpret_cast<float*>(raw0 + wstage * stage_bytes);
      float* rb = reinterpret_cast<float*>(raw0 + wstage * stage_bytes + g.a_raw);
      const int64_t k0 = kb + int64_t(c) * KC;
      fetch<KC, AL>(ra, g.a, m0, 7, g.M, k0, ke);
      fetch<KC, BL>(rb, bo, 0, g.nlog, nvalid, k0, ke);
    }
    cp_async_commit();
    wstage = wstage + 1 == g.ns ? 0 : wstage + 1;
  };
  for (int c = 0; c < g.ns - 1; ++c) issue(c);
  int rstage = 0;  // the stage chunk c is read from
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = idesc_tf32(kGemmM, g.npad);

  for (int c = 0; c < nch; ++c) {
    issue(c + g.ns - 1);
    // chunk c's copies (this thread's) have landed: at most ns - 1 newer groups pending
    switch (g.ns) {
      case 8: cp_async_wait<7>(); break;
      case 7: cp_async_wait<6>(); break;
      case 6: cp_async_wait<5>(); break;
      case 5: cp_async_wait<4>(); break;
      case 4: cp_async_wait<3>(); break;
      case 3: cp_async_wait<2>(); break;
      default: cp_async_wait<1>(); break;
    }
    const int ts = g.nt == 2 ? (c & 1) : 0;
    uint8_t* set = smem + ts * set_bytes;
    uint8_t *ah = set, *al = set + g.a_tile, *bh = set + 2 * g.a_tile, *bl = set + 2 * g.a_tile + g.b_tile;
    // the MMAs that last read this tile set (chunk c - nt) are done
    if (c >= g.nt) mbar_wait(bar + ts, uint32_t((c - g.nt) / g.nt) & 1u);
    __syncthreads();  // every thread's copies of chunk c are visible
    const uint8_t* stg = raw0 + rstage * stage_bytes;
    rstage = rstage + 1 == g.ns ? 0 : rstage + 1;
    convert<KC, lay_kind(AL)>(reinterpret_cast<const float*>(stg), 7, ah, al);
    convert<KC, lay_kind(BL)>(reinterpret_cast<const float*>(stg + g.a_raw), g.nlog, bh, bl);
    fence_proxy_async_smem();
    __syncthreads();  // tiles complete; the raw stage may be refilled
    if (threadIdx.x == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < KC; kk += 8) {
        const uint32_t acc0 = (c > 0 || kk > 0) ? 1u : 0u;
        umma_tf32(tmem, desc4<KC>(ah, kk), desc4<KC>(bh, kk), idesc, acc0);
        umma_tf32(tmem, desc4<KC>(ah, kk), desc4<KC>(bl, kk), idesc, 1u);
        umma_tf32(tmem, desc4<KC>(al, kk), desc4<KC>(bh, kk), idesc, 1u);
      }
      umma_commit(bar + ts);
    }
  }
  cp_async_wait<0>();
  if (nch > 0) {
    const int last = nch - 1, ts = g.nt == 2 ? (last & 1) : 0;
    mbar_wait(bar + ts, uint32_t(last / g.nt) & 1u);
  }
  tc_fence_after();

  // epilogue: warp w reads accumulator rows 32 (w % 4) .. +31 (its TMEM lane
  // quarter), every (kGemmWarps / 4)-th 32-column block; each block is staged
  // through shared memory (the raw stages are free now) and written back one
  // row (128 B) per instruction
  __syncthreads();
  float* stg = reinterpret_cast<float*>(raw0) + warp * 32 * kEpiPitch;
  const int lane = threadIdx.x & 31, quarter = warp & 3;
  const uint32_t lane_base = uint32_t(quarter * 32) << 16;
  for (int c0 = (warp >> 2) * 32; c0 < g.npad; c0 += 32 * (kGemmWarps / 4)) {
    float v[32];
    if (nch > 0) {
      tmem_ld32(tmem + lane_base + uint32_t(c0), v);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[lane * kEpiPitch + j] = v[j];
    __syncwarp();
    const int col = c0 + lane;
    if (col < nvalid) {
      const int64_t mq = m0 + quarter * 32;
      const int nr = int(min(int64_t(32), g.M - mq));
      if (g.split > 1) {
        float* dst = g.part + (int64_t(sp) * g.M + mq) * g.N + n0 + col;
        for (int rr = 0; rr < nr; ++rr) dst[int64_t(rr) * g.N] = stg[rr * kEpiPitch + lane];
      } else if (g.beta != 0.0f) {  // C += acc: eight independent loads in flight per batch
        float* dst = g.C + mq * g.ldc + n0 + col;
#pragma unroll 1
        for (int r0 = 0; r0 < nr; r0 += 8) {
          float old[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) old[q] = r0 + q < nr ? dst[int64_t(r0 + q) * g.ldc] : 0.0f;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (r0 + q < nr) dst[int64_t(r0 + q) * g.ldc] = old[q] + stg[(r0 + q) * kEpiPitch + lane];
        }
      } else {
        float* dst = g.C + mq * g.ldc + n0 + col;
        for (int rr = 0; rr < nr; ++rr) dst[int64_t(rr) * g.ldc] = stg[rr * kEpiPitch + lane];
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols) : "memory");
}

// Warp-specialised variant (the default; MARL_GEMM_LOCKSTEP=1 selects the
// kernel above): warps 4-7 issue the cp.async
// copies of chunk c into raw stage c % ns and arrive on full[s] when they land
// (cp.async.mbarrier.arrive.noinc); warps 0-3 split a landed stage into the
// hi / lo tile set c % nt, free the stage (empty[s]) and hand the set to the
// MMA warp (tfull[t]); warp 8 issues the chunk's MMAs and commits them to
// tfree[t].  No CTA-wide barrier inside the K loop: copy, split and MMA each
// run as far ahead as their rings allow.
constexpr int kWsThreads = kGemmThreads + 32;
#ifndef MARL_WS_SPLIT
#define MARL_WS_SPLIT 128
#endif
constexpr int kWsSplit = MARL_WS_SPLIT, kWsProd = kGemmThreads - kWsSplit;  // splitter / producer threads
// MARL_WS_DIRECT=1: K-contiguous 16-byte operands feed the MMA straight from
// the raw stage as the hi image (correct: kind::tf32 ignores the low 13
// mantissa bits, test_gemm_tc passes) but slower (Z1 334 -> 365 us: the raw
// stage is held until the MMAs complete, so the ring runs shallower)
#ifndef MARL_WS_DIRECT
#define MARL_WS_DIRECT 0
#endif
constexpr bool kWsDirect = MARL_WS_DIRECT;
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int KC, int MINB, int AL, int BL>
__global__ void __launch_bounds__(kWsThreads, MINB) gemm_ws_kernel(GemmArgs g) {
  // (kWsDirect) K-contiguous 16-byte operands land in the raw stage in canonical
  // layout and feed the MMA as the hi image directly; the stage then lives until
  // the chunk's MMAs complete
  constexpr bool DA = kWsDirect && AL == 0, DB = kWsDirect && BL == 0, DIRECT = DA || DB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int mt = blockIdx.x, nt = blockIdx.y, sp = blockIdx.z;
  const int64_t m0 = int64_t(mt) * kGemmM;
  const int n0 = nt * g.ntile;
  const int nvalid = min(g.ntile, g.N - n0);
  const int64_t kb = int64_t(sp) * g.kchunk, ke = min(g.K, kb + g.kchunk);
  const int nch = int((ke - kb + KC - 1) / KC);
  const uint32_t set_bytes = 2 * g.a_tile + 2 * g.b_tile, stage_bytes = g.a_raw + g.b_raw;
  uint8_t* raw0 = smem + g.nt * set_bytes;
  // barriers: full[8] | empty[8] | tfull[2] | tfree[2], then the TMEM slot
  uint64_t* full = reinterpret_cast<uint64_t*>(raw0 + max(g.ns * stage_bytes, uint32_t(kGemmWarps * 32 * kEpiPitch * 4)));
  uint64_t* empty = full + 8;
  uint64_t* tfull = empty + 8;
  uint64_t* tfree = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfree + 2);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 8; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + q)), "n"(kWsProd) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + q)), "n"(DIRECT ? 1 : kWsSplit)
                   : "memory");
    }
    for (int q = 0; q < 2; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(tfull + q)), "n"(kWsSplit) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(tfree + q)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(g.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (threadIdx.x >= kWsSplit && threadIdx.x < kGemmThreads) {  // producers
    const int tid = threadIdx.x - kWsSplit;
    OpLayout bo = g.b;
    bo.X = g.b.X + int64_t(n0) * g.b.sr;
    for (int c = 0; c < nch; ++c) {
      const int st = c % g.ns;
      if (c >= g.ns) mbar_wait(empty + st, uint32_t(c / g.ns - 1) & 1u);
      float* ra = reinterpret_cast<float*>(raw0 + st * stage_bytes);
      float* rb = reinterpret_cast<float*>(raw0 + st * stage_bytes + g.a_raw);
      const int64_t k0 = kb + int64_t(c) * KC;
      fetch<KC, AL, DA>(ra, g.a, m0, 7, g.M, k0, ke, tid, kWsProd);
      fetch<KC, BL, DB>(rb, bo, 0, g.nlog, nvalid, k0, ke, tid, kWsProd);
      cp_async_arrive(full + st);
    }
    cp_async_wait<0>();
  } else if (threadIdx.x < kWsSplit) {  // splitters
    const int tid = threadIdx.x;
    for (int c = 0; c < nch; ++c) {
      const int st = c % g.ns, ts = g.nt == 2 ? (c & 1) : 0;
      mbar_wait(full + st, uint32_t(c / g.ns) & 1u);
      if (c >= g.nt) mbar_wait(tfree + ts, uint32_t((c - g.nt) / g.nt) & 1u);
      uint8_t* set = smem + ts * set_bytes;
      uint8_t *ah = set, *al = set + g.a_tile, *bh = set + 2 * g.a_tile, *bl = set + 2 * g.a_tile + g.b_tile;
      const uint8_t* stg = raw0 + st * stage_bytes;
      convert<KC, lay_kind(AL), DA>(reinterpret_cast<const float*>(stg), 7, ah, al, tid, kWsSplit);
      convert<KC, lay_kind(BL), DB>(reinterpret_cast<const float*>(stg + g.a_raw), g.nlog, bh, bl, tid, kWsSplit);
      if (!DIRECT) mbar_arrive(empty + st);
      fence_proxy_async_smem();
      mbar_arrive(tfull + ts);
    }
  } else if (threadIdx.x == 256) {  // the MMA issuer
    const uint32_t idesc = idesc_tf32(kGemmM, g.npad);
    for (int c = 0; c < nch; ++c) {
      const int ts = g.nt == 2 ? (c & 1) : 0, st = c % g.ns;
      mbar_wait(tfull + ts, uint32_t(c / g.nt) & 1u);
      tc_fence_after();
      uint8_t* set = smem + ts * set_bytes;
      uint8_t *ah = set, *al = set + g.a_tile, *bh = set + 2 * g.a_tile, *bl = set + 2 * g.a_tile + g.b_tile;
      if (DA) ah = raw0 + st * stage_bytes;
      if (DB) bh = raw0 + st * stage_bytes + g.a_raw;
#pragma unroll
      for (int kk = 0; kk < KC; kk += 8) {
        const uint32_t acc0 = (c > 0 || kk > 0) ? 1u : 0u;
        umma_tf32(tmem, desc4<KC>(ah, kk), desc4<KC>(bh, kk), idesc, acc0);
        umma_tf32(tmem, desc4<KC>(ah, kk), desc4<KC>(bl, kk), idesc, 1u);
        umma_tf32(tmem, desc4<KC>(al, kk), desc4<KC>(bh, kk), idesc, 1u);
      }
      umma_commit(tfree + ts);
      if (DIRECT) umma_commit(empty + st);  // the stage held this chunk's hi images
    }
  }
  if (nch > 0 && warp < 8) {  // the last chunk's MMAs (and so all of them) are done
    const int last = nch - 1, ts = g.nt == 2 ? (last & 1) : 0;
    mbar_wait(tfree + ts, uint32_t(last / g.nt) & 1u);
  }
  tc_fence_after();
  __syncthreads();  // every raw stage is free for the epilogue staging
  if (warp < 8) {
    float* stg = reinterpret_cast<float*>(raw0) + warp * 32 * kEpiPitch;
    const int lane = threadIdx.x & 31, quarter = warp & 3;
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    for (int c0 = (warp >> 2) * 32; c0 < g.npad; c0 += 32 * (kGemmWarps / 4)) {
      float v[32];
      if (nch > 0) {
        tmem_ld32(tmem + lane_base + uint32_t(c0), v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[lane * kEpiPitch + j] = v[j];
      __syncwarp();
      const int col = c0 + lane;
      if (col < nvalid) {
        const int64_t mq = m0 + quarter * 32;
        const int nr = int(min(int64_t(32), g.M - mq));
        if (g.split > 1) {
          float* dst = g.part + (int64_t(sp) * g.M + mq) * g.N + n0 + col;
          for (int rr = 0; rr < nr; ++rr) dst[int64_t(rr) * g.N] = stg[rr * kEpiPitch + lane];
        } else if (g.beta != 0.0f) {
          float* dst = g.C + mq * g.ldc + n0 + col;
#pragma unroll 1
          for (int r0 = 0; r0 < nr; r0 += 8) {
            float old[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) old[q] = r0 + q < nr ? dst[int64_t(r0 + q) * g.ldc] : 0.0f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (r0 + q < nr) dst[int64_t(r0 + q) * g.ldc] = old[q] + stg[(r0 + q) * kEpiPitch + lane];
          }
        } else {
          float* dst = g.C + mq * g.ldc + n0 + col;
          for (int rr = 0; rr < nr; ++rr) dst[int64_t(rr) * g.ldc] = stg[rr * kEpiPitch + lane];
        }
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols) : "memory");
}

// C = beta C + sum over splits of the partial tiles, in split order
__global__ void gemm_fold_kernel(const float* __restrict__ part, int split, int64_t M, int N, float* C, int64_t ldc,
                                 float beta) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  const int64_t m = i / N;
  const int n = int(i - m * N);
  float s = 0.0f;
  for (int q = 0; q < split; ++q) s += part[int64_t(q) * M * N + i];
  float* d = C + m * ldc + n;
  *d = beta != 0.0f ? *d + s : s;
}

// g[o] = beta g[o] + sum_k D[k][o]: fixed-order partial sums over row blocks, then a fold
constexpr int kColRows = 512;
__global__ void colsum_part_kernel(const float* __restrict__ D, int64_t ldd, int O, int64_t K, float* __restrict__ part) {
  const int o = blockIdx.y * blockDim.x + threadIdx.x;
  if (o >= O) return;
  const int64_t k0 = int64_t(blockIdx.x) * kColRows, k1 = min(K, k0 + kColRows);
  float s = 0.0f;
  for (int64_t k = k0; k < k1; ++k) s += __ldg(D + k * ldd + o);
  part[int64_t(blockIdx.x) * O + o] = s;
}
// one CTA per column: strided partial sums, then a fixed-shape tree
__global__ void colsum_fold_kernel(const float* __restrict__ part, int nparts, int O, float* g, float beta) {
  __shared__ float sh[256];
  const int o = blockIdx.x, t = threadIdx.x;
  float s = 0.0f;
  for (int q = t; q < nparts; q += 256) s += part[int64_t(q) * O + o];
  sh[t] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) sh[t] += sh[t + w];
    __syncthreads();
  }
  if (t == 0) g[o] = beta != 0.0f ? g[o] + sh[0] : sh[0];
}

// split-K / column-sum partials: one scratch buffer per stream (grown on
// demand; the stream's earlier kernels are drained before a buffer is freed)
float* scratch(size_t floats, cudaStream_t st, cudaError_t* err) {
  struct Buf {
    float* p = nullptr;
    size_t n = 0;
  };
  static std::map<cudaStream_t, Buf> bufs;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  Buf& x = bufs[st];
  if (x.n < floats) {
    if (x.p) {
      if ((*err = cudaStreamSynchronize(st)) != cudaSuccess) return nullptr;
      cudaFree(x.p);
      x.p = nullptr;
      x.n = 0;
    }
    if ((*err = cudaMalloc(&x.p, floats * sizeof(float))) != cudaSuccess) {
      x.p = nullptr;
      return nullptr;
    }
    x.n = floats;
  }
  return x.p;
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

uint32_t pow2_cols(int n) {
  uint32_t c = 32;
  while (c < uint32_t(n)) c <<= 1;
  return c;
}

OpLayout op_layout(const float* X, int64_t sr, int64_t sk, int rows_per_tile) {
  OpLayout o{X, sr, sk, 2, 1};
  const uintptr_t base = reinterpret_cast<uintptr_t>(X);
  auto widest = [&](int64_t stride) {  // floats per copy keeping every copy aligned
    for (int v : {4, 2}) {
      if (stride % v == 0 && base % (4 * v) == 0) return v;
    }
    return 1;
  };
  if (sk == 1) {
    o.kind = 0;
    o.vec = widest(sr);
  } else if (sr == 1) {
    o.kind = 1;
    o.vec = widest(sk);
    while (o.vec > 1 && rows_per_tile % o.vec) o.vec >>= 1;
  }
  return o;
}

}  // namespace

int lay_code(const OpLayout& o) { return o.kind == 1 ? (o.vec == 4 ? 2 : 3) : (o.kind == 0 && o.vec == 4 ? 0 : 1); }

using GemmKernel = void (*)(GemmArgs);
template <int KC, int MINB, int AL, bool WS>
GemmKernel pick_b(int bl) {
  switch (bl) {
    case 0: return WS ? gemm_ws_kernel<KC, MINB, AL, 0> : gemm_tf32x3_kernel<KC, MINB, AL, 0>;
    case 1: return WS ? gemm_ws_kernel<KC, MINB, AL, 1> : gemm_tf32x3_kernel<KC, MINB, AL, 1>;
    case 2: return WS ? gemm_ws_kernel<KC, MINB, AL, 2> : gemm_tf32x3_kernel<KC, MINB, AL, 2>;
    default: return WS ? gemm_ws_kernel<KC, MINB, AL, 3> : gemm_tf32x3_kernel<KC, MINB, AL, 3>;
  }
}
template <int KC, int MINB, bool WS>
GemmKernel pick_ab(int al, int bl) {
  switch (al) {
    case 0: return pick_b<KC, MINB, 0, WS>(bl);
    case 1: return pick_b<KC, MINB, 1, WS>(bl);
    case 2: return pick_b<KC, MINB, 2, WS>(bl);
    default: return pick_b<KC, MINB, 3, WS>(bl);
  }
}
GemmKernel pick_kernel(bool deep, bool ws, int al, int bl) {
  if (ws) return deep ? pick_ab<32, 1, true>(al, bl) : pick_ab<16, 2, true>(al, bl);
  return deep ? pick_ab<32, 1, false>(al, bl) : pick_ab<16, 2, false>(al, bl);
}

// C[M x N] = beta C + A . B'^T on the tensor cores (see the file comment).
cudaError_t tc_gemm(cudaStream_t st, int64_t M, int N, int64_t K, const float* A, int64_t sam, int64_t sak,
                    const float* B, int64_t sbn, int64_t sbk, float* C, int64_t ldc, float beta) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  GemmArgs g{};
  g.C = C;
  g.M = M;
  g.K = K;
  g.ldc = ldc;
  g.N = N;
  g.beta = beta;
  // N tiles of up to 128 columns; a grid of fewer than two M x N tiles per SM
  // takes 64-column tiles instead (twice the CTAs in flight)
  const int64_t mt0 = (M + kGemmM - 1) / kGemmM;
  // -- unless K is long enough to split: then the split supplies the CTAs and
  // wider tiles re-stage the A operand fewer times (MARL_GEMM_SPLITN64=1: off)
  const bool splits = mt0 * ((N + kGemmMaxN - 1) / kGemmMaxN) < int64_t(sm_count()) && K >= 64 * 128 &&
                      !getenv("MARL_GEMM_SPLITN64");
  const int maxn = (mt0 * ((N + kGemmMaxN - 1) / kGemmMaxN) < 2 * int64_t(sm_count()) && N > 64 && !splits)
                       ? 64
                       : kGemmMaxN;
  const int ntiles = (N + maxn - 1) / maxn;
  g.ntile = ((N + ntiles - 1) / ntiles + 15) / 16 * 16;  // balanced N tiles, multiples of 16
  g.npad = 16;
  g.nlog = 4;
  while (g.npad < g.ntile) {
    g.npad <<= 1;
    ++g.nlog;
  }
  g.tmem_cols = pow2_cols(g.npad);
  g.a = op_layout(A, sam, sak, kGemmM);
  g.b = op_layout(B, sbn, sbk, g.npad);
  if (g.b.kind == 1 && ntiles > 1) {  // every N tile's base must keep the copy alignment
    while (g.b.vec > 1 && (g.ntile % g.b.vec)) g.b.vec >>= 1;
  }
  const int64_t mtiles = (M + kGemmM - 1) / kGemmM;
  // split K when the M x N tiles alone leave SMs idle and K is long
  int split = 1;
  const int64_t tiles = mtiles * ntiles;
  // the warp-specialised kernel; MARL_GEMM_LOCKSTEP=1 runs the lockstep one (A/B knob)
  static const bool ws = getenv("MARL_GEMM_LOCKSTEP") == nullptr;
  // split-K on the deep ring: the default for the warp-specialised kernel (MARL_GEMM_SHALLOW=1: off),
  // opt-in for the lockstep one (MARL_GEMM_DEEP=1)
  const bool deep_env = ws ? getenv("MARL_GEMM_SHALLOW") == nullptr : getenv("MARL_GEMM_DEEP") != nullptr;
  if (tiles < sm_count() && K > 128) {
    const char* ps = getenv("MARL_GEMM_SPLIT_PER_SM");
    const int64_t per_sm = ps ? std::max(1, atoi(ps)) : deep_env ? 1 : 2;
    split = int(std::min<int64_t>(std::max<int64_t>(1, per_sm * sm_count() / tiles), (K + 127) / 128));
    split = std::max(1, std::min(split, 1024));
  }
  // split-K grids (few tiles over a long K: the weight gradients) take the deep
  // configuration; everything else keeps two CTAs per SM (measured: the deep
  // ring on a 1.3-wave grid of 192 tiles is 1.7x slower than several CTAs per SM)
  const bool deep = split > 1 && deep_env;
  const int KC = deep ? 32 : 16;
  const uint32_t budget = deep ? 227 * 1024 - 1024 : 227 * 1024 / 2 - 1024;
  g.a_raw = raw_bytes(kGemmM, g.a.kind, KC);
  g.b_raw = raw_bytes(g.npad, g.b.kind, KC);
  g.a_tile = kGemmM * KC * 4;
  g.b_tile = uint32_t(g.npad) * KC * 4;
  // as many raw stages (latency hiding) and tile sets (split / MMA overlap) as fit
  g.ns = 8;  // prefetch distance ns - 1 chunks: as deep as shared memory allows
  g.nt = 2;
  auto bytes = [&] {  // the epilogue staging (4 warps x 32 x kEpiPitch floats) reuses the raw stages
    const uint32_t raw = std::max<uint32_t>(g.ns * (g.a_raw + g.b_raw), kGemmWarps * 32 * kEpiPitch * 4);
    return g.nt * (2 * g.a_tile + 2 * g.b_tile) + raw + 256;  // + barriers and the TMEM slot
  };
  while (bytes() > budget && g.ns > 2) --g.ns;
  if (bytes() > budget) g.nt = 1;
  while (bytes() > budget && g.ns > 2) --g.ns;
  const size_t smem = bytes();
  g.kchunk = std::max<int64_t>(KC, ((K + split - 1) / split + KC - 1) / KC * KC);
  split = int(std::max<int64_t>(1, (K + g.kchunk - 1) / g.kchunk));
  g.split = split;
  if (split > 1) {
    cudaError_t e = cudaSuccess;
    g.part = scratch(size_t(split) * size_t(M) * size_t(N), st, &e);
    if (!g.part) return e;
  }
  auto kern = pick_kernel(deep, ws, lay_code(g.a), lay_code(g.b));
  smem_optin(kern);
  kern<<<dim3(unsigned(mtiles), unsigned(ntiles), unsigned(split)), ws ? kWsThreads : kGemmThreads, smem, st>>>(g);
  ++g_launches;
  if (split > 1) {
    const int64_t total = M * N;
    gemm_fold_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(g.part, split, M, N, C, ldc, beta);
    ++g_launches;
  }
  return cudaGetLastError();
}

cudaError_t tc_colsum(cudaStream_t st, int O, int64_t K, const float* D, int64_t ldd, float* g, float beta) {
  if (O <= 0) return cudaSuccess;
  const int nparts = int(std::max<int64_t>(1, (K + kColRows - 1) / kColRows));
  cudaError_t e = cudaSuccess;
  float* part = scratch(size_t(nparts) * size_t(O), st, &e);
  if (!part) return e;
  const int tx = std::min(128, (O + 31) / 32 * 32);
  colsum_part_kernel<<<dim3(unsigned(nparts), unsigned((O + tx - 1) / tx)), tx, 0, st>>>(D, ldd, O, K, part);
  colsum_fold_kernel<<<unsigned(O), 256, 0, st>>>(part, nparts, O, g, beta);
  g_launches += 2;
  return cudaGetLastError();
}

}  // namespace marl_b200
