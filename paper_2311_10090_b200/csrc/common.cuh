// Device-side building blocks shared by every env kernel: the reference's
// Threefry-2x32-20 key streams, a glibc-exact hypot, and block-cooperative
// coalesced row stores.  Compiled for sm_100a with -fmad=false so every fp64
// expression is evaluated as written (the reference is built for baseline
// x86-64 without FMA contraction, proj/CMakeLists.txt:7-9).
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>
#include <mutex>
#include <unordered_set>

#define MARL_HD __host__ __device__ __forceinline__
#ifdef __CUDACC__
#define MARL_NOINLINE __noinline__
#else
#define MARL_NOINLINE __attribute__((noinline))
#endif

namespace marl_b200 {

MARL_HD int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// PrngKey (prng.hpp:12-17): cipher key k0,k1 + 64-bit counter base c1:c0.
struct Key {
  uint32_t k0, k1, c0, c1;
};

MARL_HD uint32_t rotl32(uint32_t x, int r) {
#ifdef __CUDA_ARCH__
  return __funnelshift_l(x, x, r);
#else
  return (x << r) | (x >> (32 - r));
#endif
}

// threefry2x32, prng.cpp:93-114 (20 rounds, key injection every 4).
MARL_HD void threefry2x32(uint32_t k0, uint32_t k1, uint32_t x0, uint32_t x1, uint32_t& y0,
                          uint32_t& y1) {
  const uint32_t k2 = 0x1BD11BDAu ^ k0 ^ k1;
  x0 += k0;
  x1 += k1;
#define MARL_R(r) x0 += x1; x1 = rotl32(x1, r); x1 ^= x0;
  MARL_R(13) MARL_R(15) MARL_R(26) MARL_R(6)
  x0 += k1; x1 += k2 + 1u;
  MARL_R(17) MARL_R(29) MARL_R(16) MARL_R(24)
  x0 += k2; x1 += k0 + 2u;
  MARL_R(13) MARL_R(15) MARL_R(26) MARL_R(6)
  x0 += k0; x1 += k1 + 3u;
  MARL_R(17) MARL_R(29) MARL_R(16) MARL_R(24)
  x0 += k1; x1 += k2 + 4u;
  MARL_R(13) MARL_R(15) MARL_R(26) MARL_R(6)
  x0 += k2; x1 += k0 + 5u;
#undef MARL_R
  y0 = x0;
  y1 = x1;
}

// block_at, prng.cpp:76-81: block at counter base + offset, packed (y0<<32)|y1.
MARL_HD uint64_t block_at(const Key& k, uint64_t off) {
  uint64_t ctr = ((uint64_t(k.c1) << 32) | k.c0) + off;
  uint32_t y0, y1;
  threefry2x32(k.k0, k.k1, uint32_t(ctr), uint32_t(ctr >> 32), y0, y1);
  return (uint64_t(y0) << 32) | y1;
}

constexpr uint64_t kSplitBase = uint64_t(1) << 63;           // prng.cpp:84
constexpr uint64_t kFoldBase = kSplitBase + (uint64_t(1) << 62);  // prng.cpp:162

MARL_HD Key key_from_blocks(uint64_t a, uint64_t b) {  // prng.cpp:153-154
  return Key{uint32_t(a >> 32), uint32_t(a), uint32_t(b), uint32_t(b >> 32)};
}

// Child i of prng::split(key, n) (prng.cpp:147-157); O(1) in i, so any shard
// derives its own children without materialising the others.
MARL_HD Key split_child(const Key& k, uint64_t i) {
  return key_from_blocks(block_at(k, kSplitBase + 2 * i), block_at(k, kSplitBase + 2 * i + 1));
}

// prng.cpp:159-167
MARL_HD Key fold_in(const Key& k, uint64_t d) {
  return key_from_blocks(block_at(k, kFoldBase + 2 * d), block_at(k, kFoldBase + 2 * d + 1));
}

// Out-of-line variants (~70 instructions per block) for kernels that derive
// keys at many sites: one copy keeps a large fused kernel inside the
// instruction cache (the SMAX step kernel).
__host__ __device__ MARL_NOINLINE inline uint64_t block_at_nl(const Key& k, uint64_t off) { return block_at(k, off); }
__host__ __device__ MARL_NOINLINE inline Key split_child_nl(const Key& k, uint64_t i) {
  return key_from_blocks(block_at_nl(k, kSplitBase + 2 * i), block_at_nl(k, kSplitBase + 2 * i + 1));
}
__host__ __device__ MARL_NOINLINE inline Key fold_in_nl(const Key& k, uint64_t d) {
  return key_from_blocks(block_at_nl(k, kFoldBase + 2 * d), block_at_nl(k, kFoldBase + 2 * d + 1));
}

MARL_HD double to_unit(uint64_t b) { return double(b >> 11) * 0x1.0p-53; }  // prng.cpp:86-89

// Element j of prng::uniform(key, n, lo, hi) (prng.cpp:169-178).
MARL_HD double uniform_at(const Key& k, uint64_t j, double lo, double hi) {
  double v = lo + to_unit(block_at(k, j)) * (hi - lo);
  if (v >= hi) v = nextafter(hi, lo);
  return v;
}

// x % n for n < 2^16 with 32-bit arithmetic only (three 32-bit remainders):
// x = h*2^32 + l  ->  ((h % n) * 2^16 + l_hi) % n, then (* 2^16 + l_lo) % n.
MARL_HD uint32_t mod_small(uint64_t x, uint32_t n) {
  uint32_t r = uint32_t(x >> 32) % n;
  r = ((r << 16) | (uint32_t(x) >> 16)) % n;
  r = ((r << 16) | (uint32_t(x) & 0xffffu)) % n;
  return r;
}

// glibc >= 2.35 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, the non-FMA
// Borges "MyHypot3" correction) -- the x86-64 libm the reference links
// (smax.cpp:495,550).  Restated from the published algorithm (Borges,
// arXiv:1904.09481) and glibc's scaling thresholds; every operation below is
// an explicit IEEE round-to-nearest op so nvcc cannot contract it.
MARL_HD double hypot_kernel(double ax, double ay) {
#ifdef __CUDA_ARCH__
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
#else
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
#endif
}

// Out of line on purpose: it is the rare exact path behind dist_le and the
// separation push, and inlining it into every unrolled pair loop bloats code.
__host__ __device__ MARL_NOINLINE inline double hypot_glibc(double x, double y) {
  if (!std::isfinite(x) || !std::isfinite(y)) {
    if (std::isinf(x) || std::isinf(y)) return INFINITY;
    return x + y;
  }
  x = std::fabs(x);
  y = std::fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / 0x1p-54) return ax + ay;
    return hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return hypot_kernel(ax, ay);
}

// Exact evaluation of `hypot(dx, dy) <= r` (the form every SMAX range/sight
// test takes, smax.cpp:383,497-501,613) without the hypot in the common case:
// dx^2+dy^2 is within a few ulps of hypot^2 and glibc's hypot is within one
// ulp, so outside a relative band of 2e-12 around r^2 the squared distance
// decides; inside the band the glibc-exact hypot decides.  r2lo/r2hi are
// r^2*(1 -/+ 1e-12), precomputed on the host.
MARL_HD bool dist_le(double dx, double dy, double r, double r2lo, double r2hi) {
  double d2 = dx * dx + dy * dy;
  if (d2 < r2lo) return true;
  if (d2 > r2hi) return false;
  return hypot_glibc(dx, dy) <= r;
}

struct Thresh {  // a distance threshold and its squared decision band
  double r, r2lo, r2hi;
};

MARL_HD Thresh make_thresh(double r) {
  return Thresh{r, r * r * (1.0 - 1e-12), r * r * (1.0 + 1e-12)};
}

#ifdef __CUDACC__
// Copy `bytes` from shared to global memory with the whole block: 16-byte
// vectors when both ends are 16-byte aligned, else 4-byte words, else bytes.
__device__ __forceinline__ void block_store(void* gdst, const void* ssrc, size_t bytes) {
  const uintptr_t g = reinterpret_cast<uintptr_t>(gdst);
  const uintptr_t s = reinterpret_cast<uintptr_t>(ssrc);
  if (((g | s | bytes) & 15) == 0) {
    const int4* src = static_cast<const int4*>(ssrc);
    int4* dst = static_cast<int4*>(gdst);
    for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) __stcs(dst + i, src[i]);
  } else if (((g | s | bytes) & 3) == 0) {
    const int* src = static_cast<const int*>(ssrc);
    int* dst = static_cast<int*>(gdst);
    for (size_t i = threadIdx.x; i < bytes / 4; i += blockDim.x) __stcs(dst + i, src[i]);
  } else {
    const uint8_t* src = static_cast<const uint8_t*>(ssrc);
    uint8_t* dst = static_cast<uint8_t*>(gdst);
    for (size_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  }
}

// ---- TMA bulk copies (cp.async.bulk, sm_90+; the sm_100a async proxy) ----
// shared::cta -> global, `bytes` a multiple of 16, both ends 16-byte aligned.
// One thread issues; completion is tracked per issuing thread with bulk
// groups.  Generic-proxy writes to the source buffer must be ordered before
// the copy with fence_proxy_async_smem() (by the writing threads) plus a
// barrier, the CUTLASS TMA-store-epilogue protocol.
__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until at most N committed groups still READ their shared source.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// Wait until at most N committed groups are incomplete (writes performed).
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Block-wide store of a shared-memory tile: one TMA bulk store issued by
// thread 0 when the tile and its destination qualify (16-byte aligned, size a
// multiple of 16), else the cooperative vector copy.  Call from every thread
// after the tile is complete; the caller fences and synchronises first
// (bulk_tile_fence).  Thread 0 waits for the TMA engine to finish READING the
// tile, so the caller must not overwrite it before the next barrier.
__device__ __forceinline__ bool bulk_ok(const void* gdst, const void* ssrc, size_t bytes) {
  return ((reinterpret_cast<uintptr_t>(gdst) | reinterpret_cast<uintptr_t>(ssrc) | bytes) & 15) == 0 && bytes > 0;
}
__device__ __forceinline__ void bulk_tile_fence() {
  fence_proxy_async_smem();
  __syncthreads();
}
__device__ __forceinline__ void tile_store(void* gdst, const void* ssrc, size_t bytes);

// Per-block episode statistics, folded into 64-bit integer accumulators so the
// totals are exact and order-independent (identical for any grid shape and any
// number of GPUs): [0] finished episodes, [1] sum of lengths, [2] sum of
// returns in 2^-24 fixed point.
__device__ __forceinline__ void stats_add(unsigned long long* stats, bool finished, int length,
                                          double ret) {
  unsigned long long n = finished ? 1ull : 0ull;
  unsigned long long L = finished ? (unsigned long long)(long long)length : 0ull;
  unsigned long long R = finished ? (unsigned long long)__double2ll_rn(ret * 16777216.0) : 0ull;
  for (int o = 16; o > 0; o >>= 1) {
    n += __shfl_xor_sync(0xffffffffu, n, o);
    L += __shfl_xor_sync(0xffffffffu, L, o);
    R += __shfl_xor_sync(0xffffffffu, R, o);
  }
  if ((threadIdx.x & 31) == 0 && n) {
    atomicAdd(stats + 0, n);
    atomicAdd(stats + 1, L);
    atomicAdd(stats + 2, R);
  }
}
__device__ __forceinline__ void tile_store(void* gdst, const void* ssrc, size_t bytes) {
  if (bulk_ok(gdst, ssrc, bytes)) {
    if (threadIdx.x == 0) {
      bulk_store_s2g(gdst, ssrc, uint32_t(bytes));
      bulk_commit();
    }
  } else {
    block_store(gdst, ssrc, bytes);
  }
}
// Thread 0: the tiles issued by tile_store have been read out of shared memory.
__device__ __forceinline__ void tile_store_drain() {
  if (threadIdx.x == 0) bulk_wait_read<0>();
}
#endif

// Let `fn` use the device's whole opt-in shared memory per block.  Launches
// pass their own dynamic size; setting the attribute to ONE value (the
// maximum) instead of each launch's size keeps concurrent host threads from
// racing on it (one thread's smaller value failing another's launch with
// "too many resources requested").  Done once per kernel.
inline void smem_optin(const void* fn) {
  static std::mutex mu;
  static std::unordered_set<const void*> done;
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert(fn).second) return;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, fn);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - int(fa.sharedSizeBytes));
}
template <class F>
inline void smem_optin(F* fn) {
  smem_optin(reinterpret_cast<const void*>(fn));
}

}  // namespace marl_b200
