// The PPO minibatch step on the 5th-generation tensor cores (bf16 operands,
// fp32 accumulation in TMEM): ff_minibatch (proj/core/src/algo/ppo.cpp:409-441)
// for IPPO nets of width 64, input <= 191 (MPE, SMAX 3m / 2s3z / 5m_vs_6m) and
// <= 16 actions, actor and critic in one persistent kernel, one CTA (256
// threads, all 512 TMEM columns) per SM, 128 gathered rows per tile.  The
// input rows are a bf16 copy of the rollout observations made once per update
// (ppo_tc_pack), Kx = round16(in + 1) wide with the constant 1 in column
// Kx-1, gathered into the canonical operand tile by 16-byte cp.async, and
// its loss inputs packed into one 32-byte record per row:
//
//   F1  D[0:128)   = X[128xKx] . [W1a ; W1c]^T                 forward
//   F2  D[0:64)    = H1a . W2a^T,  D[64:128) = H1c . W2c^T
//   F3  D[0:16)    = H2a . W3a^T,  D[16:32)  = H2c . W3c^T
//   --  ppo_row_loss per row (actor_critic.hpp:340-412) -> dL[128x32]
//   B1  D[0:64)    = dLa . W3a,    D[64:128) = dLc . W3c        input gradients
//       + G3  Dg3[128x32] += H2^T . dL   (gW3^T: actor columns 0..15, critic 16)
//   B2  D[0:64)    = dZ2a . W2a,   D[64:128) = dZ2c . W2c
//       + G2  Dg2[128x128] += dZ2^T . H1 (gW2: the two diagonal 64x64 blocks)
//       + Gb  Dgb[128x32]  += dZ2^T . dL (column 31 of dL is 1 -> gb2)
//   G1  Dg1[128xKx] += dZ1^T . X       (gW1 both nets; X column Kx-1 == 1 -> gb1)
//
// Every activation / gradient tile is written once, bf16, in the canonical
// K-major no-swizzle layout [rows x features]; the input-gradient GEMMs read
// the forward weight images and the weight-gradient GEMMs read the activation
// tiles TRANSPOSED through MN-major descriptors (tc.cuh umma_desc_mn), so no
// operand is ever re-laid-out.  Each weight-gradient GEMM is issued with the
// input-gradient GEMM that last needs its activation tile, so dZ2 overwrites
// H2 and dZ1 overwrites H1 in place (two activation tiles, not four).  The
// weight-gradient accumulators live in TMEM for all the CTA's tiles and are
// read out once.  The next tile's rows are gathered while the current tile
// computes (two X buffers when shared memory allows, else after G1).  The row
// loss is evaluated in float (the operands are bf16 already).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "engine.h"
#include "tc.cuh"

namespace marl_b200 {

namespace {

constexpr int kRows = 128;
constexpr int kThr = 256;
constexpr uint32_t kCols = 512;
constexpr int kMaxKx = 192;
constexpr int kSmemMax = 232448;  // 227 KB opt-in per CTA
constexpr int kStat = 6;
constexpr uint32_t kActBytes = kRows * 128 * 2;  // one [128 x 128] bf16 activation tile
constexpr uint32_t kDlBytes = kRows * 32 * 2;

// TMEM columns: ns work regions of 128 (one per tile in flight), then the
// weight-gradient accumulators gW2 128 | gW3 32 | gb2 32 | gW1 Kx.
__host__ __device__ constexpr uint32_t tm_g2(int ns) { return 128u * uint32_t(ns); }
__host__ __device__ constexpr uint32_t tm_g3(int ns) { return tm_g2(ns) + 128u; }
__host__ __device__ constexpr uint32_t tm_gb(int ns) { return tm_g3(ns) + 32u; }
__host__ __device__ constexpr uint32_t tm_g1(int ns) { return tm_gb(ns) + 32u; }

struct UpdLayout {
  uint32_t w1, w2a, w2c, w3a, w3c, x, ha, hb, dl, st_r, slot, bias, gb3w, bar, bar_g, tmem_slot, total;
  int nx;  // X buffers per tile slot (2: the next tile's rows land while this one computes)
  int ns;  // tiles in flight per CTA
};

__host__ __device__ inline uint32_t upd_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline UpdLayout upd_layout(int kx, int nx, int ns) {
  UpdLayout L{};
  uint32_t o = 0;
  auto take = [&o](uint32_t bytes, uint32_t align) {
    o = upd_up(o, align);
    const uint32_t at = o;
    o += bytes;
    return at;
  };
  L.nx = nx;
  L.ns = ns;
  L.w1 = take(128 * kx * 2, 128);
  L.w2a = take(64 * 64 * 2, 128);
  L.w2c = take(64 * 64 * 2, 128);
  L.w3a = take(16 * 64 * 2, 128);
  L.w3c = take(16 * 64 * 2, 128);
  L.x = take(uint32_t(ns * nx) * kRows * kx * 2, 128);
  L.ha = take(uint32_t(ns) * kActBytes, 128);  // H1, then dZ1 (per slot)
  L.hb = take(uint32_t(ns) * kActBytes, 128);  // H2, then dZ2
  L.dl = take(uint32_t(ns) * kDlBytes, 128);
  L.st_r = take(uint32_t(ns) * kRows * sizeof(PpoRowRec), 16);  // the tiles' loss-input records
  L.slot = take(uint32_t(ns) * 3 * kRows * 4, 16);
  L.bias = take((4 * 64 + 2 * 16) * 4, 16);
  L.gb3w = take(8 * 32 * 4, 16);
  L.bar = take(uint32_t(ns) * 8, 8);
  L.bar_g = take(8, 8);
  L.tmem_slot = take(4, 4);
  L.total = upd_up(o, 128);
  return L;
}

// two tiles in flight when TMEM (Kx <= 64) and shared memory allow; two X buffers when they fit
__host__ __device__ inline UpdLayout upd_layout(int kx) {
  for (int ns = 2; ns >= 1; --ns) {
    if (tm_g1(ns) + uint32_t(kx) > kCols) continue;
    for (int nx = 2; nx >= 1; --nx) {
      const UpdLayout L = upd_layout(kx, nx, ns);
      if (L.total <= uint32_t(kSmemMax)) return L;
    }
  }
  return upd_layout(kx, 1, 1);
}

__device__ __forceinline__ void cpa4(void* sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void cpa16(void* sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ float act_f(float v, int relu) { return relu ? fmaxf(v, 0.0f) : tanh_fast(v); }
__device__ __forceinline__ float act_d(float g, float y, int relu) {
  return relu ? (y > 0.0f ? g : 0.0f) : g * (1.0f - y * y);
}

// 16 bf16 values of row `row`, features [f0, f0+16) of a [rows x F] canonical tile
__device__ __forceinline__ void get16(const uint8_t* tile, int F, int row, int f0, float* v) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint4 q = *reinterpret_cast<const uint4*>(tile + canon_off(row, f0 + 8 * c, F));
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      const float2 f = __bfloat1622float2(h);
      v[8 * c + 2 * i] = f.x;
      v[8 * c + 2 * i + 1] = f.y;
    }
  }
}

__device__ __forceinline__ uint16_t bf16_bits(float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  return *reinterpret_cast<const uint16_t*>(&h);
}

// Once per update, for every slot of the window: the observation row as bf16
// [kx] (column kx-1 = 1, the bias column; zero padding between) and the
// row's loss inputs as one 32-byte record (legal actions as a bit mask).
__global__ void pack_rows_kernel(PpoTcPack p) {
  const int chunks = p.kx / 8;
  const int64_t n = p.rows * chunks;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += stride) {
    const int64_t r = e / chunks;
    const int c0 = int(e - r * chunks) * 8;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = c0 + j;
      v[j] = k < p.in ? __ldg(p.obs + r * p.in + k) : (k == p.kx - 1 ? 1.0f : 0.0f);
    }
    uint4 q;
    q.x = pack_bf16(v[0], v[1]);
    q.y = pack_bf16(v[2], v[3]);
    q.z = pack_bf16(v[4], v[5]);
    q.w = pack_bf16(v[6], v[7]);
    reinterpret_cast<uint4*>(p.obs_bf)[e] = q;
  }
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < p.rows; r += stride) {
    PpoRowRec rec;
    rec.active = __ldg(p.active + r);
    rec.adv = __ldg(p.adv + r);
    rec.logp = __ldg(p.old_logp + r);
    rec.vtarg = __ldg(p.vtarg + r);
    rec.value = __ldg(p.old_value + r);
    rec.action = __ldg(p.actions + r);
    uint32_t m = 0;
    for (int j = 0; j < p.n_act; ++j) m |= (__ldg(p.legal + r * p.n_act + j) ? 1u : 0u) << j;
    rec.legal = m;
    rec.pad = 0;
    p.rec[r] = rec;
  }
}

// NS tiles in flight: the phases of tile slots 0..NS-1 alternate, so one
// slot's MMAs run under the other's epilogue; one thread issues every MMA in
// a fixed order (the accumulation order is deterministic).
// RELU: the torso activation folded (0 tanh, the PpoConfig default; 1 relu).
template <int NS, int RELU>
__global__ void __launch_bounds__(kThr, 1) ppo_update_tc_kernel(PpoTcArgs a) {
  constexpr uint32_t cG2 = tm_g2(NS), cG3 = tm_g3(NS), cGb = tm_gb(NS), cG1 = tm_g1(NS);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int in = a.in, NA = a.n_act, KX = a.kx;
  const UpdLayout L = upd_layout(KX);
  uint8_t* base = smem_raw;
  uint8_t *w1 = base + L.w1, *w2a = base + L.w2a, *w2c = base + L.w2c, *w3a = base + L.w3a, *w3c = base + L.w3c,
          *xb = base + L.x;
  PpoRowRec* st_r = reinterpret_cast<PpoRowRec*>(base + L.st_r);
  int32_t* slot = reinterpret_cast<int32_t*>(base + L.slot);
  float* bias = reinterpret_cast<float*>(base + L.bias);
  float* gb3w = reinterpret_cast<float*>(base + L.gb3w);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bar);
  uint64_t* bar_g = reinterpret_cast<uint64_t*>(base + L.bar_g);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L.tmem_slot);
  auto HA = [&](int s) { return base + L.ha + uint32_t(s) * kActBytes; };
  auto HB = [&](int s) { return base + L.hb + uint32_t(s) * kActBytes; };
  auto DL = [&](int s) { return base + L.dl + uint32_t(s) * kDlBytes; };
  const uint32_t xbytes = uint32_t(kRows) * uint32_t(KX) * 2u;
  auto XB = [&](int s, int k) { return xb + uint32_t(s * L.nx + k) * xbytes; };
  const int t = threadIdx.x, row = t & (kRows - 1), part = t >> 7, warp = t >> 5;
  const int64_t ntiles = (a.M + kRows - 1) / kRows;
  const int64_t G = gridDim.x;

  if (t == 0) {
    for (int s = 0; s <= NS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s < NS ? bar + s : bar_g)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // ---- the nets' current parameters -> canonical bf16 operand images
  {
    const float* pa = a.actor;
    const float* pc = a.critic;
    const float *aw1 = pa, *ab1 = aw1 + 64 * in, *aw2 = ab1 + 64, *ab2 = aw2 + 64 * 64, *aw3 = ab2 + 64,
                *ab3 = aw3 + NA * 64;
    const float *cw1 = pc, *cb1 = cw1 + 64 * in, *cw2 = cb1 + 64, *cb2 = cw2 + 64 * 64, *cw3 = cb2 + 64,
                *cb3 = cw3 + 64;
    uint16_t* W1 = reinterpret_cast<uint16_t*>(w1);
    for (int q = t; q < 128 * KX; q += kThr) {
      const int r = q / KX, k = q - r * KX;
      float v = 0.0f;  // the bias column Kx-1 and the padding multiply zero weights
      if (k < in) v = r < 64 ? __ldg(aw1 + r * in + k) : __ldg(cw1 + (r - 64) * in + k);
      W1[canon_off(r, k, KX) / 2] = bf16_bits(v);
    }
    for (int q = t; q < 64 * 64; q += kThr) {
      const int r = q / 64, k = q % 64;
      reinterpret_cast<uint16_t*>(w2a)[canon_off(r, k, 64) / 2] = bf16_bits(__ldg(aw2 + q));
      reinterpret_cast<uint16_t*>(w2c)[canon_off(r, k, 64) / 2] = bf16_bits(__ldg(cw2 + q));
    }
    for (int q = t; q < 16 * 64; q += kThr) {
      const int r = q / 64, k = q % 64;
      reinterpret_cast<uint16_t*>(w3a)[canon_off(r, k, 64) / 2] = bf16_bits(r < NA ? __ldg(aw3 + r * 64 + k) : 0.0f);
      reinterpret_cast<uint16_t*>(w3c)[canon_off(r, k, 64) / 2] = bf16_bits(r == 0 ? __ldg(cw3 + k) : 0.0f);
    }
    if (t < 64) {
      bias[t] = __ldg(ab1 + t);
      bias[64 + t] = __ldg(cb1 + t);
      bias[128 + t] = __ldg(ab2 + t);
      bias[192 + t] = __ldg(cb2 + t);
    }
    if (t < 16) {
      bias[256 + t] = t < NA ? __ldg(ab3 + t) : 0.0f;
      bias[272 + t] = t == 0 ? __ldg(cb3) : 0.0f;
    }
    gb3w[t] = 0.0f;  // 8 warps x 32
  }
  // ---- gather of a tile's rows (cp.async, zero-filled): X straight into its
  // canonical operand buffer, the loss-input records into the slot's staging area
  auto tile_of = [&](int64_t it, int s) { return int64_t(blockIdx.x) + (int64_t(NS) * it + s) * G; };
  auto slot_ok = [&](int64_t tile, int r) { return tile < ntiles && tile * kRows + r < a.M; };
  auto slot_load = [&](int64_t tile, int s, int sb) {
    if (t < kRows) {
      const bool ok = slot_ok(tile, t);
      cpa4(slot + (s * 3 + sb) * kRows + t, ok ? a.idx + tile * kRows + t : a.idx, ok ? 4 : 0);
    }
  };
  auto gather = [&](int64_t tile, int s, int sb, uint8_t* xdst) {
    const int ch = KX / 8;
    const int32_t* sl_of = slot + (s * 3 + sb) * kRows;
    for (int e = t; e < kRows * ch; e += kThr) {
      const int r = e / ch, c = e - r * ch;
      const int sl = slot_ok(tile, r) ? sl_of[r] : -1;
      cpa16(xdst + canon_off(r, 8 * c, KX), sl >= 0 ? a.obs_bf + (size_t(sl) * size_t(KX) + size_t(8 * c)) : a.obs_bf,
            sl >= 0 ? 16 : 0);
    }
    if (t < kRows) {
      const int sl = slot_ok(tile, t) ? sl_of[t] : -1;
      const int n = sl >= 0 ? 4 : 0;
      const int64_t q = sl >= 0 ? sl : 0;
      const uint8_t* src = reinterpret_cast<const uint8_t*>(a.rec + q);
      uint8_t* dst = reinterpret_cast<uint8_t*>(st_r + s * kRows + t);
      cpa16(dst, src, 4 * n);
      cpa16(dst + 16, src + 16, 4 * n);
    }
  };
  for (int s = 0; s < NS; ++s) {
    slot_load(tile_of(0, s), s, 0);
    slot_load(tile_of(1, s), s, 1);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  for (int s = 0; s < NS; ++s) gather(tile_of(0, s), s, 0, XB(s, 0));
  asm volatile("cp.async.commit_group;" ::: "memory");
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
  const PpoMbStats st = *a.st;
  const float inv_tw = st.total_w > 0.0 ? float(1.0 / st.total_w) : 0.0f;
  double pg = 0.0, vt = 0.0, ent = 0.0, kl = 0.0, clipn = 0.0;
  uint32_t phase[NS], phase_g = 0;
#pragma unroll
  for (int s = 0; s < NS; ++s) phase[s] = 0;
  bool g_first = true;

  // one slot's wait on its MMAs
  auto wait_slot = [&](int s) {
    mbar_wait(bar + s, phase[s]);
    phase[s] ^= 1;
    tc_fence_after();
  };
  // the end of an epilogue: operands visible to the MMA, then one thread issues `issue`
  auto hand_off = [&](auto issue) {
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
      issue();
    }
  };
  // bias + activation of the work columns -> a [128 x 128] bf16 tile
  auto epi_fwd = [&](int s, const float* b, uint8_t* dst) {
    const uint32_t cw = 128u * uint32_t(s);
#pragma unroll 1
    for (int c = 64 * part; c < 64 * part + 64; c += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + cw + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_f(v[i] + b[c + i], RELU);
      put16(dst, 128, row, c, v);
      put16(dst, 128, row, c + 16, v + 16);
    }
  };
  // input gradient of the work columns times act'(y), y read from and dZ written over `tile`
  auto epi_bwd = [&](int s, uint8_t* tile) {
    const uint32_t cw = 128u * uint32_t(s);
#pragma unroll 1
    for (int c = 64 * part; c < 64 * part + 64; c += 32) {
      float v[32], y[32];
      tmem_ld32(tmem + lane_base + cw + uint32_t(c), v);
      get16(tile, 128, row, c, y);
      get16(tile, 128, row, c + 16, y + 16);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_d(v[i], y[i], RELU);
      put16(tile, 128, row, c, v);
      put16(tile, 128, row, c + 16, v + 16);
    }
  };

  for (int64_t it = 0; tile_of(it, 0) < ntiles; ++it) {
    const int sb = int(it % 3);
    const int xi = L.nx == 2 ? int(it & 1) : 0;
    // this iteration's rows have landed (generic-proxy cp.async writes -> visible to the MMA's async proxy)
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async_smem();
    __syncthreads();
    tc_fence_after();
    bool live[NS];
    float r_w[NS], r_adv[NS], r_lp[NS], r_vt[NS], r_v[NS];
    int r_act[NS];
    uint32_t r_lg[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      live[s] = slot_ok(tile_of(it, s), row);
      r_w[s] = r_adv[s] = r_lp[s] = r_vt[s] = r_v[s] = 0.0f;
      r_act[s] = 0;
      r_lg[s] = 0;
      if (live[s]) {
        const PpoRowRec& rr = st_r[s * kRows + row];
        r_w[s] = rr.active;
        if (part == 0) {
          r_adv[s] = rr.adv;
          r_lp[s] = rr.logp;
          r_act[s] = rr.action;
          r_lg[s] = rr.legal;
        } else {
          r_vt[s] = rr.vtarg;
          r_v[s] = rr.value;
        }
      }
    }
    if (t == 0) {  // F1 of every slot: D[work s] = X . [W1a ; W1c]^T
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 128);
      for (int s = 0; s < NS; ++s) {
        for (int k = 0; k < KX; k += 16)
          umma_bf16(tmem + 128u * uint32_t(s), umma_desc(XB(s, xi), KX, k), umma_desc(w1, KX, k), id, k > 0);
        umma_commit(bar + s);
      }
    }
    __syncthreads();  // the staging areas are free: the next rows land while these compute
    for (int s = 0; s < NS; ++s) {
      slot_load(tile_of(it + 2, s), s, int((it + 2) % 3));
      if (L.nx == 2) gather(tile_of(it + 1, s), s, int((it + 1) % 3), XB(s, xi ^ 1));
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // ---- F1 epilogue -> H1; F2
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      wait_slot(s);
      epi_fwd(s, bias, HA(s));
      hand_off([&] {
        const uint32_t id = idesc_bf16(128, 64), cw = 128u * uint32_t(s);
        for (int k = 0; k < 64; k += 16) umma_bf16(tmem + cw, umma_desc(HA(s), 128, k), umma_desc(w2a, 64, k), id, k > 0);
        for (int k = 0; k < 64; k += 16)
          umma_bf16(tmem + cw + 64, umma_desc(HA(s), 128, 64 + k), umma_desc(w2c, 64, k), id, k > 0);
        umma_commit(bar + s);
      });
    }
    // ---- F2 epilogue -> H2; F3 (heads)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      wait_slot(s);
      epi_fwd(s, bias + 128, HB(s));
      hand_off([&] {
        const uint32_t id = idesc_bf16(128, 16), cw = 128u * uint32_t(s);
        for (int k = 0; k < 64; k += 16) umma_bf16(tmem + cw, umma_desc(HB(s), 128, k), umma_desc(w3a, 64, k), id, k > 0);
        for (int k = 0; k < 64; k += 16)
          umma_bf16(tmem + cw + 16, umma_desc(HB(s), 128, 64 + k), umma_desc(w3c, 64, k), id, k > 0);
        umma_commit(bar + s);
      });
    }
    // ---- the row's part of ppo_row_loss (part 0 the actor head, part 1 the critic) -> dL; B1 + G3
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      wait_slot(s);
      float hv[16];
      tmem_ld16(tmem + lane_base + 128u * uint32_t(s) + uint32_t(16 * part), hv);
      float d[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) d[j] = 0.0f;
      const double w = double(r_w[s]);
      const bool on = live[s] && w != 0.0 && st.total_w > 0.0;
      if (part == 0) {
        if (on) {
          float z[16], lp[16];
          bool lg[16];
          float mx = -INFINITY;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            z[j] = hv[j] + bias[256 + j];
            lg[j] = j < NA && ((r_lg[s] >> j) & 1u);
            if (lg[j]) mx = fmaxf(mx, z[j]);
          }
          float den = 0.0f;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (lg[j]) den += __expf(z[j] - mx);
          const float lse = __logf(den);
          float H = 0.0f;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            lp[j] = lg[j] ? z[j] - mx - lse : -1e30f;
            if (lg[j]) H -= __expf(lp[j]) * lp[j];
          }
          const int act = r_act[s];
          if (act < 0 || act >= NA || !lg[act < 0 ? 0 : (act >= NA ? 0 : act)]) atomicExch(a.err, 1);
          const int ac = act < 0 ? 0 : (act >= NA ? NA - 1 : act);
          float lpa = 0.0f;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j == ac) lpa = lp[j];
          float advf = r_adv[s];
          if (st.normalize) advf = float((double(advf) - st.mean) / (st.std + 1e-8));
          const float ratio = __expf(lpa - r_lp[s]);
          const float unclipped = ratio * advf;
          const float rho_c = fminf(fmaxf(ratio, 1.0f - float(a.clip_eps)), 1.0f + float(a.clip_eps));
          const float clipped = rho_c * advf;
          const float dsurr = unclipped <= clipped ? ratio * advf : 0.0f;
          const float scale = r_w[s] * inv_tw;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (!lg[j]) continue;
            const float p = __expf(lp[j]);
            const float g = -dsurr * ((j == ac ? 1.0f : 0.0f) - p) - float(a.ent_coef) * (-p * (lp[j] + H));
            d[j] = scale * g;
          }
          pg += w * -double(fminf(unclipped, clipped));
          ent += w * double(H);
          kl += w * (double(ratio) - 1.0 - log(double(ratio)));
          clipn += w * (fabs(double(ratio) - 1.0) > a.clip_eps ? 1.0 : 0.0);
        }
      } else if (on) {
        const float v = hv[0] + bias[272];
        const float v_clip = r_v[s] + fminf(fmaxf(v - r_v[s], -float(a.clip_eps)), float(a.clip_eps));
        const float sq = (v - r_vt[s]) * (v - r_vt[s]), sq_c = (v_clip - r_vt[s]) * (v_clip - r_vt[s]);
        vt += w * double(0.5f * fmaxf(sq, sq_c));
        d[0] = r_w[s] * inv_tw * float(a.vf_coef) * (sq >= sq_c ? (v - r_vt[s]) : 0.0f);
      }
      // gb3: per-warp column sums, each warp owning its own slots (deterministic)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float sum = d[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if ((t & 31) == 0) gb3w[warp * 32 + 16 * part + j] += sum;
      }
      if (part == 1) d[15] = 1.0f;  // dL column 31: the constant of the gb2 GEMM (W3c row 15 is zero)
      put16(DL(s), 32, row, 16 * part, d);
      // B1: dH2 = dL . W3 (the forward head images read MN-major); G3 reads H2 before it is overwritten
      hand_off([&] {
        const uint32_t id = idesc_bf16(128, 64, 0, 1), i3 = idesc_bf16(128, 32, 1, 1), cw = 128u * uint32_t(s);
        umma_bf16(tmem + cw, umma_desc(DL(s), 32, 0), umma_desc_mn(w3a, 64, 0), id, 0);
        umma_bf16(tmem + cw + 64, umma_desc(DL(s), 32, 16), umma_desc_mn(w3c, 64, 0), id, 0);
        for (int r0 = 0; r0 < kRows; r0 += 16)
          umma_bf16(tmem + cG3, umma_desc_mn(HB(s), 128, r0), umma_desc_mn(DL(s), 32, r0), i3,
                    (g_first && s == 0 && r0 == 0) ? 0u : 1u);
        umma_commit(bar + s);
      });
    }
    // ---- dZ2 over H2; B2 + G2 + Gb (they read dZ2 and H1 before H1 is overwritten)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      wait_slot(s);
      epi_bwd(s, HB(s));
      hand_off([&] {
        const uint32_t id = idesc_bf16(128, 64, 0, 1), i2 = idesc_bf16(128, 128, 1, 1), ib = idesc_bf16(128, 32, 1, 1);
        const uint32_t cw = 128u * uint32_t(s);
        for (int k = 0; k < 64; k += 16)
          umma_bf16(tmem + cw, umma_desc(HB(s), 128, k), umma_desc_mn(w2a, 64, k), id, k > 0);
        for (int k = 0; k < 64; k += 16)
          umma_bf16(tmem + cw + 64, umma_desc(HB(s), 128, 64 + k), umma_desc_mn(w2c, 64, k), id, k > 0);
        for (int r0 = 0; r0 < kRows; r0 += 16) {
          const uint32_t acc = (g_first && s == 0 && r0 == 0) ? 0u : 1u;
          umma_bf16(tmem + cG2, umma_desc_mn(HB(s), 128, r0), umma_desc_mn(HA(s), 128, r0), i2, acc);
          umma_bf16(tmem + cGb, umma_desc_mn(HB(s), 128, r0), umma_desc_mn(DL(s), 32, r0), ib, acc);
        }
        umma_commit(bar + s);
      });
    }
    // ---- dZ1 over H1; G1 (the first layer's weight gradient)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      wait_slot(s);
      epi_bwd(s, HA(s));
      hand_off([&] {
        const uint32_t i1 = idesc_bf16(128, KX, 1, 1);
        for (int r0 = 0; r0 < kRows; r0 += 16)
          umma_bf16(tmem + cG1, umma_desc_mn(HA(s), 128, r0), umma_desc_mn(XB(s, xi), KX, r0), i1,
                    (g_first && s == 0 && r0 == 0) ? 0u : 1u);
        if (s == NS - 1) umma_commit(bar_g);
      });
    }
    g_first = false;
    // H1 / X are rewritten by the next iteration only after G1 has read them
    mbar_wait(bar_g, phase_g);
    phase_g ^= 1;
    if (L.nx == 1) {
      tc_fence_after();
      for (int s = 0; s < NS; ++s) gather(tile_of(it + 1, s), s, int((it + 1) % 3), XB(s, 0));
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  tc_fence_after();
  // ---- read the accumulators once: TMEM lane m = output feature m (actor 0..63, critic 64..127)
  const int m = (warp & 3) * 32 + (t & 31);
  const bool critic = m >= 64;
  const int o = m & 63;
  const int Pa = 64 * in + 64 + 64 * 64 + 64 + NA * 64 + NA, Pc = 64 * in + 64 + 64 * 64 + 64 + 64 + 1;
  float* gp = critic ? a.gpart_c + size_t(blockIdx.x) * Pc : a.gpart_a + size_t(blockIdx.x) * Pa;
  float *G1 = gp, *GB1 = G1 + 64 * in, *G2 = GB1 + 64, *GB2 = G2 + 64 * 64, *G3 = GB2 + 64;
  if (!g_first) {
    float v[16];
#pragma unroll 1
    for (int c = 16 * part; c < KX; c += 32) {  // gW1 columns k (Kx-1: gb1)
      tmem_ld16(tmem + lane_base + cG1 + uint32_t(c), v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int k = c + j;
        if (k < in) G1[o * in + k] = v[j];
        if (k == KX - 1) GB1[o] = v[j];
      }
    }
    float w[32];
    tmem_ld32(tmem + lane_base + cG2 + uint32_t((critic ? 64 : 0) + 32 * part), w);  // diagonal block
#pragma unroll
    for (int j = 0; j < 32; ++j) G2[o * 64 + 32 * part + j] = w[j];
    tmem_ld16(tmem + lane_base + cG3 + uint32_t(16 * part), v);  // gW3^T: row m = H2 feature
    if (!critic && part == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < NA) G3[j * 64 + o] = v[j];
    }
    if (critic && part == 1) G3[o] = v[0];
    tmem_ld16(tmem + lane_base + cGb + 16u, v);  // column 31: dZ2^T . 1
    if (part == 0) GB2[o] = v[15];
  } else {
    for (int e = t; e < Pa; e += kThr) a.gpart_a[size_t(blockIdx.x) * Pa + e] = 0.0f;
    for (int e = t; e < Pc; e += kThr) a.gpart_c[size_t(blockIdx.x) * Pc + e] = 0.0f;
  }
  tc_fence_before();
  __syncthreads();
  if (!g_first) {
    if (t < NA) {  // gb3: per-warp sums of the actor warps (part 0 = warps 0..3), warp order
      float sum = 0.0f;
      for (int wq = 0; wq < 4; ++wq) sum += gb3w[wq * 32 + t];
      a.gpart_a[size_t(blockIdx.x) * Pa + (Pa - NA) + t] = sum;
    } else if (t == 32) {
      float sum = 0.0f;
      for (int wq = 4; wq < 8; ++wq) sum += gb3w[wq * 32 + 16];
      a.gpart_c[size_t(blockIdx.x) * Pc + (Pc - 1)] = sum;
    }
  }
  // per-CTA loss statistics (actor: pg, -, entropy, kl, clipped; critic: -, v_term)
  __shared__ double s_stats[kThr / 32][kStat];
  const double v5[kStat] = {pg, vt, ent, kl, clipn, 0.0};
  for (int c = 0; c < kStat; ++c) {
    double v = v5[c];
    for (int q = 16; q > 0; q >>= 1) v += __shfl_down_sync(0xffffffffu, v, q);
    if ((t & 31) == 0) s_stats[warp][c] = v;
  }
  __syncthreads();
  if (t < kStat) {
    double s0 = 0.0;
    for (int wq = 0; wq < kThr / 32; ++wq) s0 += s_stats[wq][t];
    a.spart_a[size_t(blockIdx.x) * kStat + t] = (t == 1) ? 0.0 : s0;
    a.spart_c[size_t(blockIdx.x) * kStat + t] = (t == 1) ? s0 : 0.0;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}

}  // namespace

int ppo_tc_kx(int in_dim) { return (in_dim + 1 + 15) / 16 * 16; }

bool ppo_tc_supported(int in_dim, int critic_in, int width, int n_act) {
  return in_dim >= 1 && ppo_tc_kx(in_dim) <= kMaxKx && critic_in == in_dim && width == 64 && n_act <= 16 &&
         upd_layout(ppo_tc_kx(in_dim)).total <= uint32_t(kSmemMax);
}

int ppo_tc_grid(int64_t M) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = (M + kRows - 1) / kRows;
  return int(cap_grid(std::max<int64_t>(1, std::min<int64_t>(tiles, sms))));
}

void ppo_tc_pack(const PpoTcPack& p, cudaStream_t s) {
  const int64_t n = p.rows * (p.kx / 8);
  if (n <= 0) return;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
  pack_rows_kernel<<<blocks, 256, 0, s>>>(p);
  ++g_launches;
}

void ppo_update_tc(const PpoTcArgs& a, int grid, cudaStream_t s) {
  const UpdLayout L = upd_layout(a.kx);
  const size_t sm = L.total;
  auto kern = L.ns == 2 ? (a.relu ? ppo_update_tc_kernel<2, 1> : ppo_update_tc_kernel<2, 0>)
                        : (a.relu ? ppo_update_tc_kernel<1, 1> : ppo_update_tc_kernel<1, 0>);
  smem_optin(kern);
  kern<<<grid, kThr, sm, s>>>(a);
  ++g_launches;
}

}  // namespace marl_b200
