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
constexpr uint32_t cWork = 0, cG2 = 128, cG3 = 256, cGb = 288, cG1 = 320;  // cG1 + Kx <= 512
constexpr int kMaxKx = 192;
constexpr int kSmemMax = 232448;  // 227 KB opt-in per CTA
constexpr int kStat = 6;

struct UpdLayout {
  uint32_t w1, w2a, w2c, w3a, w3c, x, ha, hb, dl, st_r, slot, bias, gb3w, bar, bar_g, tmem_slot, total;
  int nx;  // X buffers (2: the next tile's rows land while this one computes)
};

__host__ __device__ inline uint32_t upd_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline UpdLayout upd_layout(int kx, int nx) {
  UpdLayout L{};
  uint32_t o = 0;
  auto take = [&o](uint32_t bytes, uint32_t align) {
    o = upd_up(o, align);
    const uint32_t at = o;
    o += bytes;
    return at;
  };
  L.nx = nx;
  L.w1 = take(128 * kx * 2, 128);
  L.w2a = take(64 * 64 * 2, 128);
  L.w2c = take(64 * 64 * 2, 128);
  L.w3a = take(16 * 64 * 2, 128);
  L.w3c = take(16 * 64 * 2, 128);
  L.x = take(uint32_t(nx) * kRows * kx * 2, 128);
  L.ha = take(kRows * 128 * 2, 128);  // H1, then dZ1
  L.hb = take(kRows * 128 * 2, 128);  // H2, then dZ2
  L.dl = take(kRows * 32 * 2, 128);
  L.st_r = take(kRows * sizeof(PpoRowRec), 16);  // the tile's loss-input records
  L.slot = take(3 * kRows * 4, 16);
  L.bias = take((4 * 64 + 2 * 16) * 4, 16);
  L.gb3w = take(8 * 32 * 4, 16);
  L.bar = take(8, 8);
  L.bar_g = take(8, 8);
  L.tmem_slot = take(4, 4);
  L.total = upd_up(o, 128);
  return L;
}

__host__ __device__ inline UpdLayout upd_layout(int kx) {
  const UpdLayout two = upd_layout(kx, 2);
  return two.total <= uint32_t(kSmemMax) ? two : upd_layout(kx, 1);
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

__global__ void __launch_bounds__(kThr, 1) ppo_update_tc_kernel(PpoTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int in = a.in, NA = a.n_act, KX = a.kx;
  const UpdLayout L = upd_layout(KX);
  uint8_t* base = smem_raw;
  uint8_t *w1 = base + L.w1, *w2a = base + L.w2a, *w2c = base + L.w2c, *w3a = base + L.w3a, *w3c = base + L.w3c,
          *xb = base + L.x, *ha = base + L.ha, *hb = base + L.hb, *sdl = base + L.dl;
  PpoRowRec* st_r = reinterpret_cast<PpoRowRec*>(base + L.st_r);
  int32_t* slot = reinterpret_cast<int32_t*>(base + L.slot);
  float* bias = reinterpret_cast<float*>(base + L.bias);
  float* gb3w = reinterpret_cast<float*>(base + L.gb3w);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L.bar);
  uint64_t* bar_g = reinterpret_cast<uint64_t*>(base + L.bar_g);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L.tmem_slot);
  const uint32_t xbytes = uint32_t(kRows) * uint32_t(KX) * 2u;
  const int t = threadIdx.x, row = t & (kRows - 1), part = t >> 7, warp = t >> 5;
  const int64_t ntiles = (a.M + kRows - 1) / kRows;
  const int64_t G = gridDim.x;

  if (t == 0) {
    for (uint64_t* m : {bar, bar_g}) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
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
  // canonical operand buffer, the loss inputs into the staging area
  auto slot_ok = [&](int64_t tile, int r) { return tile < ntiles && tile * kRows + r < a.M; };
  auto slot_load = [&](int64_t tile, int sb) {
    if (t < kRows) {
      const bool ok = slot_ok(tile, t);
      cpa4(slot + sb * kRows + t, ok ? a.idx + tile * kRows + t : a.idx, ok ? 4 : 0);
    }
  };
  auto gather = [&](int64_t tile, int sb, uint8_t* xdst) {
    const int ch = KX / 8;
    for (int e = t; e < kRows * ch; e += kThr) {
      const int r = e / ch, c = e - r * ch;
      const int sl = slot_ok(tile, r) ? slot[sb * kRows + r] : -1;
      cpa16(xdst + canon_off(r, 8 * c, KX), sl >= 0 ? a.obs_bf + (size_t(sl) * size_t(KX) + size_t(8 * c)) : a.obs_bf,
            sl >= 0 ? 16 : 0);
    }
    if (t < kRows) {
      const int sl = slot_ok(tile, t) ? slot[sb * kRows + t] : -1;
      const int n = sl >= 0 ? 4 : 0;
      const int64_t q = sl >= 0 ? sl : 0;
      const uint8_t* src = reinterpret_cast<const uint8_t*>(a.rec + q);
      cpa16(reinterpret_cast<uint8_t*>(st_r + t), src, 4 * n);
      cpa16(reinterpret_cast<uint8_t*>(st_r + t) + 16, src + 16, 4 * n);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  slot_load(blockIdx.x, 0);
  slot_load(blockIdx.x + G, 1);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  gather(blockIdx.x, 0, xb);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
  const PpoMbStats st = *a.st;
  const float inv_tw = st.total_w > 0.0 ? float(1.0 / st.total_w) : 0.0f;
  double pg = 0.0, vt = 0.0, ent = 0.0, kl = 0.0, clipn = 0.0;
  uint32_t phase = 0, phase_g = 0;
  bool g_first = true;
  int it = 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++it) {
    const int sb = it % 3;
    uint8_t* sx = xb + (L.nx == 2 ? uint32_t(it & 1) * xbytes : 0u);
    // this tile's rows have landed (generic-proxy cp.async writes -> visible to the MMA's async proxy)
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async_smem();
    __syncthreads();
    tc_fence_after();
    const bool live = slot_ok(tile, row);
    float r_w = 0.0f, r_adv = 0.0f, r_lp = 0.0f, r_vt = 0.0f, r_v = 0.0f;
    int r_act = 0;
    uint32_t r_lg = 0;
    if (live) {
      const PpoRowRec& rr = st_r[row];
      r_w = rr.active;
      if (part == 0) {
        r_adv = rr.adv;
        r_lp = rr.logp;
        r_act = rr.action;
        r_lg = rr.legal;
      } else {
        r_vt = rr.vtarg;
        r_v = rr.value;
      }
    }
    if (t == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 128);
      for (int k = 0; k < KX; k += 16) umma_bf16(tmem + cWork, umma_desc(sx, KX, k), umma_desc(w1, KX, k), id, k > 0);
      umma_commit(bar);
    }
    __syncthreads();  // the staging area is free
    slot_load(tile + 2 * G, (it + 2) % 3);
    if (L.nx == 2) gather(tile + G, (it + 1) % 3, xb + uint32_t((it + 1) & 1) * xbytes);
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue F1: h1 = act(. + b1), part p owns the net p columns
#pragma unroll 1
    for (int c = 64 * part; c < 64 * part + 64; c += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + cWork + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_f(v[i] + bias[c + i], a.relu);
      put16(ha, 128, row, c, v);
      put16(ha, 128, row, c + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 64);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(ha, 128, k), umma_desc(w2a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 64, umma_desc(ha, 128, 64 + k), umma_desc(w2c, 64, k), id, k > 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
#pragma unroll 1
    for (int c = 64 * part; c < 64 * part + 64; c += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + uint32_t(c), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_f(v[i] + bias[128 + c + i], a.relu);
      put16(hb, 128, row, c, v);
      put16(hb, 128, row, c + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 16);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(hb, 128, k), umma_desc(w3a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 16, umma_desc(hb, 128, 64 + k), umma_desc(w3c, 64, k), id, k > 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- the row's part of ppo_row_loss: part 0 the actor head, part 1 the critic
    {
      float hv[16];
      tmem_ld16(tmem + lane_base + uint32_t(16 * part), hv);
      float d[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) d[j] = 0.0f;
      const double w = double(r_w);
      const bool on = live && w != 0.0 && st.total_w > 0.0;
      if (part == 0) {
        if (on) {
          float z[16], lp[16];
          bool lg[16];
          float mx = -INFINITY;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            z[j] = hv[j] + bias[256 + j];
            lg[j] = j < NA && ((r_lg >> j) & 1u);
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
          const int act = r_act;
          if (act < 0 || act >= NA || !lg[act < 0 ? 0 : (act >= NA ? 0 : act)]) atomicExch(a.err, 1);
          const int ac = act < 0 ? 0 : (act >= NA ? NA - 1 : act);
          float lpa = 0.0f;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j == ac) lpa = lp[j];
          float advf = r_adv;
          if (st.normalize) advf = float((double(advf) - st.mean) / (st.std + 1e-8));
          const float ratio = __expf(lpa - r_lp);
          const float unclipped = ratio * advf;
          const float rho_c = fminf(fmaxf(ratio, 1.0f - float(a.clip_eps)), 1.0f + float(a.clip_eps));
          const float clipped = rho_c * advf;
          const float dsurr = unclipped <= clipped ? ratio * advf : 0.0f;
          const float scale = r_w * inv_tw;
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
        const float v_clip = r_v + fminf(fmaxf(v - r_v, -float(a.clip_eps)), float(a.clip_eps));
        const float sq = (v - r_vt) * (v - r_vt), sq_c = (v_clip - r_vt) * (v_clip - r_vt);
        vt += w * double(0.5f * fmaxf(sq, sq_c));
        d[0] = r_w * inv_tw * float(a.vf_coef) * (sq >= sq_c ? (v - r_vt) : 0.0f);
      }
      // gb3: per-warp column sums, each warp owning its own slots (deterministic)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float s = d[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((t & 31) == 0) gb3w[warp * 32 + 16 * part + j] += s;
      }
      if (part == 1) d[15] = 1.0f;  // dL column 31: the constant of the gb2 GEMM (W3c row 15 is zero)
      tc_fence_before();
      put16(sdl, 32, row, 16 * part, d);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {  // B1: dH2 = dL . W3 (the forward head images read MN-major); G3 reads H2 before it is overwritten
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 64, 0, 1), i3 = idesc_bf16(128, 32, 1, 1);
      umma_bf16(tmem + 0, umma_desc(sdl, 32, 0), umma_desc_mn(w3a, 64, 0), id, 0);
      umma_bf16(tmem + 64, umma_desc(sdl, 32, 16), umma_desc_mn(w3c, 64, 0), id, 0);
      for (int r0 = 0; r0 < kRows; r0 += 16)
        umma_bf16(tmem + cG3, umma_desc_mn(hb, 128, r0), umma_desc_mn(sdl, 32, r0), i3, (g_first && r0 == 0) ? 0u : 1u);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
#pragma unroll 1
    for (int c = 64 * part; c < 64 * part + 64; c += 32) {  // dZ2 over H2, element by element of this row
      float v[32], y[32];
      tmem_ld32(tmem + lane_base + uint32_t(c), v);
      get16(hb, 128, row, c, y);
      get16(hb, 128, row, c + 16, y + 16);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_d(v[i], y[i], a.relu);
      put16(hb, 128, row, c, v);
      put16(hb, 128, row, c + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {  // B2: dH1 = dZ2 . W2; G2 and Gb read dZ2 and H1 before H1 is overwritten
      tc_fence_after();
      const uint32_t id = idesc_bf16(128, 64, 0, 1), i2 = idesc_bf16(128, 128, 1, 1), ib = idesc_bf16(128, 32, 1, 1);
      for (int k = 0; k < 64; k += 16) umma_bf16(tmem + 0, umma_desc(hb, 128, k), umma_desc_mn(w2a, 64, k), id, k > 0);
      for (int k = 0; k < 64; k += 16)
        umma_bf16(tmem + 64, umma_desc(hb, 128, 64 + k), umma_desc_mn(w2c, 64, k), id, k > 0);
      for (int r0 = 0; r0 < kRows; r0 += 16) {
        const uint32_t acc = (g_first && r0 == 0) ? 0u : 1u;
        umma_bf16(tmem + cG2, umma_desc_mn(hb, 128, r0), umma_desc_mn(ha, 128, r0), i2, acc);
        umma_bf16(tmem + cGb, umma_desc_mn(hb, 128, r0), umma_desc_mn(sdl, 32, r0), ib, acc);
      }
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
#pragma unroll 1
    for (int c = 64 * part; c < 64 * part + 64; c += 32) {  // dZ1 over H1
      float v[32], y[32];
      tmem_ld32(tmem + lane_base + uint32_t(c), v);
      get16(ha, 128, row, c, y);
      get16(ha, 128, row, c + 16, y + 16);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_d(v[i], y[i], a.relu);
      put16(ha, 128, row, c, v);
      put16(ha, 128, row, c + 16, v + 16);
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {  // G1: weight gradient of the first layer, accumulated in TMEM across tiles
      tc_fence_after();
      const uint32_t i1 = idesc_bf16(128, KX, 1, 1);
      for (int r0 = 0; r0 < kRows; r0 += 16)
        umma_bf16(tmem + cG1, umma_desc_mn(ha, 128, r0), umma_desc_mn(sx, KX, r0), i1, (g_first && r0 == 0) ? 0u : 1u);
      umma_commit(bar_g);
    }
    g_first = false;
    // H1 / X are rewritten by the next tile only after G1 has read them
    mbar_wait(bar_g, phase_g);
    phase_g ^= 1;
    if (L.nx == 1) {
      tc_fence_after();
      gather(tile + G, (it + 1) % 3, xb);
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
  const int NO = critic ? 1 : NA;
  float *G1 = gp, *GB1 = G1 + 64 * in, *G2 = GB1 + 64, *GB2 = G2 + 64 * 64, *G3 = GB2 + 64;
  (void)NO;
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
      float s = 0.0f;
      for (int wq = 0; wq < 4; ++wq) s += gb3w[wq * 32 + t];
      a.gpart_a[size_t(blockIdx.x) * Pa + (Pa - NA) + t] = s;
    } else if (t == 32) {
      float s = 0.0f;
      for (int wq = 4; wq < 8; ++wq) s += gb3w[wq * 32 + 16];
      a.gpart_c[size_t(blockIdx.x) * Pc + (Pc - 1)] = s;
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
  return int(std::max<int64_t>(1, std::min<int64_t>(tiles, sms)));
}

void ppo_tc_pack(const PpoTcPack& p, cudaStream_t s) {
  const int64_t n = p.rows * (p.kx / 8);
  if (n <= 0) return;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
  pack_rows_kernel<<<blocks, 256, 0, s>>>(p);
  ++g_launches;
}

void ppo_update_tc(const PpoTcArgs& a, int grid, cudaStream_t s) {
  const size_t sm = upd_layout(a.kx).total;
  cudaFuncSetAttribute(ppo_update_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  ppo_update_tc_kernel<<<grid, kThr, sm, s>>>(a);
  ++g_launches;
}

}  // namespace marl_b200
