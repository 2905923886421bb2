#include <cstring>
#include <atomic>
// Self- and cross-attention of the DiT block (PAPER.md P:L118
// "attention is O(T^2 D)"): O_h = softmax(Q_h K_h^T / sqrt(dh)) V_h, no mask, fp32
// online softmax.
//
// attn_tc: one CTA per (128-query tile, head), warp-specialised, sm_100a:
//   warp 0      TMA: Q once; K_j/V_j 128-key blocks into a 2-deep ring
//   warp 1      MMA (one thread): S_j = Q K_j^T -> TMEM (2 S buffers, 128 cols each);
//               O += P_{j-1} V_{j-1} -> TMEM (dh cols).  QK of block j is issued before
//               PV of block j-1 so the tensor core works while softmax runs.
//   warps 4..7  softmax, thread = query row: tcgen05.ld S row, row max, exp2, P (bf16)
//               into a 128B-swizzled SMEM buffer (double-buffered) as the A operand of PV.
//               Lazy rescaling: O (in TMEM) is rescaled only when the row max grows by
//               more than 2^8 over the max in use; otherwise P <= 256 is accumulated with
//               a stale max (exact after the final 1/l normalisation).
// attn_simt: fp32 warp-per-row reference-grade kernel for the fp32 validation build.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdlib>
#include "kernels.h"

namespace df {

bool make_tmap_3d(CUtensorMap* m, const void* base, uint64_t z, uint64_t rows, uint64_t cols, uint32_t box_rows);

template <int DH>
struct AttnCfg {
  static constexpr int ATOMS = DH / 64;           // 64-element (128 B) swizzle atoms along dh
  static constexpr int TILE = 128 * 128;          // bytes of one [128 x 64] bf16 atom tile
  static constexpr int Q_BYTES = ATOMS * TILE;
  static constexpr int KV_BYTES = ATOMS * TILE;   // one K or one V block
  static constexpr int P_BYTES = 2 * TILE;        // [128 q x 128 kv] bf16
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = Q_BYTES;
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;
  static constexpr int OFF_P = OFF_V + 2 * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t S_COL0 = 0;           // S buffers at cols [0,128) and [128,256)
  static constexpr uint32_t O_COL = 256;          // O at cols [256, 256+DH)
};

template <int DH>
__global__ void __launch_bounds__(256, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                   int dh_real, float scale_log2) {
  using Cfg = AttnCfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint8_t* sP = smem + Cfg::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;    // [2]
  uint64_t* kv_empty = bars + 3;   // [2]
  uint64_t* s_full = bars + 5;     // [2]
  uint64_t* s_empty = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;     // [2]
  uint64_t* p_empty = bars + 11;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = warp_id();
  const int lane = lane_id();
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * 128;
  const int nkb = (Nk + 127) / 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 128);
      mbar_init(&p_full[s], 128);
      mbar_init(&p_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, Cfg::Q_BYTES);
#pragma unroll
      for (int a = 0; a < Cfg::ATOMS; ++a) tma_load_3d(sQ + a * Cfg::TILE, &tmQ, q_full, a * 64, q0, h);
      for (int j = 0; j < nkb; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * Cfg::KV_BYTES);
#pragma unroll
        for (int a = 0; a < Cfg::ATOMS; ++a) {
          tma_load_3d(sK + st * Cfg::KV_BYTES + a * Cfg::TILE, &tmK, &kv_full[st], a * 64, j * 128, h);
          tma_load_3d(sV + st * Cfg::KV_BYTES + a * Cfg::TILE, &tmV, &kv_full[st], a * 64, j * 128, h);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(128, DH, false, true);
      mbar_wait(q_full, 0);
      const uint32_t q_addr = smem_u32(sQ);
      for (int j = 0; j <= nkb; ++j) {
        if (j < nkb) {
          const int st = j & 1;
          mbar_wait(&kv_full[st], (j >> 1) & 1);
          mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sK + st * Cfg::KV_BYTES);
          const uint32_t d_s = tmem + Cfg::S_COL0 + st * 128;
#pragma unroll
          for (int k = 0; k < DH / 16; ++k) {
            const uint32_t off = (k >> 2) * Cfg::TILE + (k & 3) * 32;
            tc_mma_bf16(d_s, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024), idesc_qk,
                        k > 0);
          }
          tc_commit(&s_full[st]);
        }
        if (j >= 1) {
          const int jj = j - 1;
          const int pb = jj & 1;
          mbar_wait(&p_full[pb], (jj >> 1) & 1);
          tc_fence_after();
          const uint32_t p_addr = smem_u32(sP + pb * Cfg::P_BYTES);
          const uint32_t v_addr = smem_u32(sV + pb * Cfg::KV_BYTES);
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // 128 keys / 16
            const uint32_t pa = p_addr + (k >> 2) * Cfg::TILE + (k & 3) * 32;
            const uint32_t vb = v_addr + k * 2048;  // 16 key rows x 128 B
            tc_mma_bf16(tmem + Cfg::O_COL, sdesc_sw128(pa, 16, 1024), sdesc_sw128(vb, Cfg::TILE, 1024), idesc_pv,
                        (jj > 0 || k > 0));
          }
          tc_commit(&p_empty[pb]);
          tc_commit(&kv_empty[pb]);
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int r = ew * 32 + lane;  // query row within tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    float s[128];
    for (int j = 0; j < nkb; ++j) {
      const int sb = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      mbar_wait(&s_full[sb], ph);
      tc_fence_after();
      const uint32_t ts = tmem + lane_off + Cfg::S_COL0 + sb * 128;
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(ts + c, s + c);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[sb]);
      const int valid = Nk - j * 128;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        float z = (c < valid) ? s[c] * scale_log2 : -INFINITY;
        s[c] = z;
        mx = fmaxf(mx, z);
      }
      // P buffer sb is free once PV_{j-2} completed
      mbar_wait(&p_empty[sb], ph ^ 1);
      const bool need = mx > m_used + 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_used;
        if (j > 0) {
          // O holds PV_0..PV_{j-1}: wait for PV_{j-1}, then rescale this warp's rows
          mbar_wait(&p_empty[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
          const float alpha = exp2f(m_used - m_new);
          l *= alpha;
          const uint32_t to = tmem + lane_off + Cfg::O_COL;
#pragma unroll
          for (int c = 0; c < DH; c += 32) {
            float o[32];
            tmem_ld32(to + c, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(to + c, o);
          }
          tc_wait_st();
        }
        m_used = m_new;
      }
      // P = exp2(s - m_used) -> bf16, 128B-swizzled K-major [128 rows x 128 keys]
      uint8_t* prow = sP + sb * Cfg::P_BYTES + r * 128;
      float lsum = 0.f;
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) {
        float p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          p[i] = exp2f(s[ch * 8 + i] - m_used);
          lsum += p[i];
        }
        uint4 u;
        u.x = pack_bf16x2(p[0], p[1]);
        u.y = pack_bf16x2(p[2], p[3]);
        u.z = pack_bf16x2(p[4], p[5]);
        u.w = pack_bf16x2(p[6], p[7]);
        const int atom = ch >> 3, c16 = ch & 7;
        *reinterpret_cast<uint4*>(prow + atom * Cfg::TILE + ((c16 ^ (r & 7)) << 4)) = u;
      }
      l += lsum;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
    }
    // final: wait for the last PV, normalise, store O[q, h*dh + c]
    const int jl = nkb - 1;
    mbar_wait(&p_empty[jl & 1], (jl >> 1) & 1);
    tc_fence_after();
    const float inv = 1.0f / l;
    const int q = q0 + r;
    const uint32_t to = tmem + lane_off + Cfg::O_COL;
    bf16* orow = O + size_t(q) * H * dh_real + size_t(h) * dh_real;
#pragma unroll
    for (int c = 0; c < DH; c += 32) {
      float o[32];
      tmem_ld32(to + c, o);
      tc_wait_ld();
      if (q < Nq && c < dh_real) {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] *= inv;
        if (dh_real - c >= 32) {
          store_vec<32>(orow + c, o);
        } else {
          for (int i = 0; i < dh_real - c; ++i) orow[c + i] = __float2bfloat16_rn(o[i]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ attn_tc2: 2 Q tiles / CTA
// Two 128-query tiles of one head share every K/V block (halving L2->SMEM traffic per
// FLOP).  TMEM (512 cols): S0 [0,128), S1 [128,256), O0 [256, 256+DH), O1 [256+DH, ..).
// P_i (bf16, 2 per column) is written by softmax group i over the first 64 columns of
// S_i and consumed from TMEM as the A operand of PV.  MMA issue order per key block j:
//   PV0_j, QK0_{j+1}, PV1_j, QK1_{j+1}
// so the tensor core always has the other tile's work while a softmax group runs, and
// in-order execution guarantees PV_i_j has read P_i before QK_i_{j+1} overwrites S_i.
template <int DH>
struct Attn2Cfg {
  static constexpr int ATOMS = DH / 64;
  static constexpr int TILE = 128 * 128;
  static constexpr int Q_BYTES = ATOMS * TILE;     // one 128-query tile
  static constexpr int KV_BYTES = ATOMS * TILE;    // one K or V block of 128 keys
  static constexpr int KST = 3;                    // K ring depth (K_j is needed one PV earlier than V_j)
  static constexpr int VST = 2;                    // V ring depth
  static constexpr int OFF_Q = 0;                  // Q0, Q1
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * KV_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t O_COL = 256;
};

DF_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int DH, bool POLY, int DBG = 0>
__global__ void __launch_bounds__(384, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                    int dh_real, float scale_log2, int Hs) {
  using Cfg = Attn2Cfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [KST]
  uint64_t* k_empty = bars + 4;   // [KST]
  uint64_t* v_full = bars + 7;    // [VST]
  uint64_t* v_empty = bars + 9;   // [VST]
  uint64_t* s_full = bars + 11;   // [2] per Q tile
  uint64_t* p_full = bars + 13;   // [2] per Q tile
  uint64_t* o_done = bars + 15;   // [2] per Q tile (after the last PV)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  const int warp = warp_id();
  const int lane = lane_id();
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * 256;
  const int nkb = (Nk + 127) / 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < Cfg::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 128);
      mbar_init(&o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * Cfg::Q_BYTES);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int a = 0; a < Cfg::ATOMS; ++a)
          tma_load_3d(sQ + t * Cfg::Q_BYTES + a * Cfg::TILE, &tmQ, q_full, a * 64, q0 + t * 128, h);
      // K runs ahead of V by up to KST blocks; interleave so neither ring starves
      int jk = 0, jv = 0;
      while (jv < nkb) {
        if (jk < nkb && jk <= jv + 1) {
          const int st = jk % Cfg::KST;
          mbar_wait(&k_empty[st], ((jk / Cfg::KST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::KV_BYTES);
#pragma unroll
          for (int a = 0; a < Cfg::ATOMS; ++a)
            tma_load_3d(sK + st * Cfg::KV_BYTES + a * Cfg::TILE, &tmK, &k_full[st], a * 64, jk * 128, h);
          ++jk;
        } else {
          const int st = jv % Cfg::VST;
          mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[st], Cfg::KV_BYTES);
#pragma unroll
          for (int a = 0; a < Cfg::ATOMS; ++a)
            tma_load_3d(sV + st * Cfg::KV_BYTES + a * Cfg::TILE, &tmV, &v_full[st], a * 64, jv * 128, h);
          ++jv;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(128, DH, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_qk = [&](int t, int j) {
        const uint32_t k_addr = smem_u32(sK + (j % Cfg::KST) * Cfg::KV_BYTES);
        const uint32_t qa = q_addr + t * Cfg::Q_BYTES;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = (k >> 2) * Cfg::TILE + (k & 3) * 32;
          tc_mma_bf16(tmem + t * 128, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024), idesc_qk,
                      k > 0);
        }
        tc_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {
        const uint32_t v_addr = smem_u32(sV + (j % Cfg::VST) * Cfg::KV_BYTES);
#pragma unroll
        for (int k = 0; k < 8; ++k)  // 128 keys / 16; P_t = columns k*8.. of S_t
          tc_mma_bf16_ts(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8,
                         sdesc_sw128(v_addr + k * 2048, Cfg::TILE, 1024), idesc_pv, (j > 0 || k > 0));
      };
      auto wait_k = [&](int j) {
        mbar_wait(&k_full[j % Cfg::KST], (j / Cfg::KST) & 1);
        tc_fence_after();
      };
      mbar_wait(q_full, 0);
      wait_k(0);
      issue_qk(0, 0);
      issue_qk(1, 0);
      tc_commit(&k_empty[0]);
      for (int j = 0; j < nkb; ++j) {
        const bool more = j + 1 < nkb;
        mbar_wait(&v_full[j % Cfg::VST], (j / Cfg::VST) & 1);
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        issue_pv(0, j);
        if (!more) tc_commit(&o_done[0]);
        if (more) {
          wait_k(j + 1);
          issue_qk(0, j + 1);
        }
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        issue_pv(1, j);
        tc_commit(&v_empty[j % Cfg::VST]);
        if (!more) tc_commit(&o_done[1]);
        if (more) {
          issue_qk(1, j + 1);
          tc_commit(&k_empty[(j + 1) % Cfg::KST]);
        }
      }
    }
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;        // Q tile of this softmax group (warps 4-7, 8-11)
    const int ew = warp & 3;              // TMEM lane quarter = warp id mod 4
    const int r = ew * 32 + lane;         // query row within the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const uint32_t ts = tmem + lane_off + t * 128;
    const uint32_t to = tmem + lane_off + Cfg::O_COL + t * DH;
    // One TMEM read of S per key block: the 128 logits of this row stay in registers for
    // the max and the exponentials (TMEM reads are 64 B/clk and the tensor core's own operand
    // reads share them; a second pass over S costs as much TMEM bandwidth as the first).
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      if (DBG == 2) {  // profiling knob: tensor + synchronisation only (no softmax)
        tc_fence_before();
        mbar_arrive(&p_full[t]);
        continue;
      }
      const int valid = Nk - j * 128;
      float s[128];
      if (DBG == 4) {
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = float(c & 7) * 0.01f;
      } else {
#pragma unroll
        for (int c = 0; c < 128; c += 32) tmem_ld32(ts + c, s + c);
        tc_wait_ld();
      }
      if (DBG == 6) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = __float_as_uint(s[i]);
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_st16(ts + 16 * q, pk);
        tc_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[t]);
        continue;
      }
      if (DBG == 3) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 128; ++c) acc += s[c];
        l += acc;
        tc_fence_before();
        mbar_arrive(&p_full[t]);
        continue;
      }
      if (valid < 128) {  // ragged last key block (warp-uniform)
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= valid) s[i] = -INFINITY;
      }
      // row max: four independent FMNMX3 chains
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 128; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(s[i + 2 * u], s[i + 2 * u + 1]));
      }
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
      // lazy rescale: the max in use moves only when a row's max exceeds it by > 8 (log2),
      // so p <= 2^8 and the O correction is rare after the first blocks
      const bool need = mx > m_used + 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_used;
        if (j > 0) {
          // s_full for block j implies PV_{j-1} (issued earlier) completed: O_t is stable
          const float alpha = exp2f(m_used - m_new);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < DH; c += 16) {
            float o[16];
            tmem_ld16(to + c, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= alpha;
            tmem_st16(to + c, reinterpret_cast<uint32_t*>(o));
          }
        }
        m_used = m_new;
      }
      // p = 2^(s*scale - m) -> bf16 pairs into the first 64 columns of S (= P_t); FFMA2 for
      // the affine part; with POLY 3/8 of the exponentials on the FMA pipe (polynomial)
      float2 lsum2 = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      const float2 nm2 = make_float2(-m_used, -m_used);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ffma2(make_float2(s[32 * q + 2 * i], s[32 * q + 2 * i + 1]), sc2, nm2);
          float2 p;
          if (DBG == 1) {
            p = ffma2(x, sc2, nm2);
          } else if (POLY && (i & 7) >= 5) {
            p = exp2_poly2(x);
          } else {
            p.x = ex2_approx(x.x);
            p.y = ex2_approx(x.y);
          }
          lsum2 = fadd2(lsum2, p);
          pk[i] = pack_bf16x2(p.x, p.y);
        }
        // columns 16q .. 16q+15 hold keys 32q .. 32q+31 (S is already in registers)
        if (DBG == 5) {
          l += __uint_as_float(pk[0] ^ pk[5] ^ pk[11] ^ pk[15]) * 1e-30f;
        } else {
          tmem_st16(ts + 16 * q, pk);
        }
      }
      l += lsum2.x + lsum2.y;
      tc_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
    }
    mbar_wait(&o_done[t], 0);
    tc_fence_after();
    const float inv = 1.0f / l;
    const int q = q0 + t * 128 + r;
    // heads of a stacked batch: head h belongs to sample h / Hs; token-major rows b*Nq + q
    const int hb = h / Hs, hl = h - hb * Hs;
    bf16* orow = O + (size_t(hb) * Nq + q) * Hs * dh_real + size_t(hl) * dh_real;
#pragma unroll 1
    for (int c = 0; c < DH; c += 32) {
      float o[32];
      tmem_ld32(to + c, o);
      tc_wait_ld();
      if (q < Nq && c < dh_real) {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] *= inv;
        if (dh_real - c >= 32) store_vec<32>(orow + c, o);
        else
          for (int i = 0; i < dh_real - c; ++i) orow[c + i] = __float2bfloat16_rn(o[i]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int g_attn_impl = 2;

template <int DH, bool POLY, int DBG = 0>
static cudaError_t launch_attn2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, bf16* O, int H,
                                int Nq, int Nk, int dh, float scale, cudaStream_t st, int hs) {
  using Cfg = Attn2Cfg<DH>;
  auto kern = attn_tc2_kernel<DH, POLY, DBG>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((Nq + 255) / 256, H);
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O,   (void*)&H,
                  (void*)&Nq, (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs};
  return launch_ex((const void*)kern, grid, dim3(384), Cfg::SMEM, st, args);
}

// p = 2^x for a pair of logits, packed to bf16x2 for P; adds the pair to the row sum.
// EXPM 0: MUFU ex2 (fp32); 1: 3 of 8 pairs by polynomial on the FMA pipe; 2: 1 of 4 pairs;
// 3: one MUFU ex2.bf16x2 per pair (input rounded to bf16: coarser, profiling only).
template <int EXPM>
DF_DEV uint32_t softmax_exp2(float2 x, int i, float2& lsum2) {
  if (EXPM == 3) {
    const uint32_t xb = pack_bf16x2(x.x, x.y);
    uint32_t pb;
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(pb) : "r"(xb));
    lsum2 = fadd2(lsum2, make_float2(__uint_as_float(pb << 16), __uint_as_float(pb & 0xffff0000u)));
    return pb;
  }
  float2 p;
  if ((EXPM == 1 && (i & 7) >= 5) || (EXPM == 2 && (i & 3) == 3)) {
    p = exp2_poly2(x);
  } else {
    p.x = ex2_approx(x.x);
    p.y = ex2_approx(x.y);
  }
  lsum2 = fadd2(lsum2, p);
  return pack_bf16x2(p.x, p.y);
}

// ------------------------------------------------------------------ attn_tc3: 2 threads per query row
// Same tensor-core schedule and TMEM map as attn_tc2 (two 128-query tiles per CTA, S/P/O in
// TMEM, PV0_j, QK0_{j+1}, PV1_j, QK1_{j+1}), but each query row's softmax is shared by two
// threads of two warps with the same TMEM lane quarter: thread (t, hc, r) owns key columns
// [64 hc, 64 hc + 64) of S_t row r and output columns [64 hc, 64 hc + 64) of O_t.  The
// softmax of one tile is on the critical path between its QK and its PV (P aliases S), so
// halving the per-thread chain (and doubling the warps that hide its latencies) shortens
// every key-block period.  The two halves agree on the row max through shared memory: each
// writes its local max rounded UP to fp16 (any common upper bound is a valid stabiliser and
// both threads then compute the same m), one named barrier per tile and block.
// Warps 0-15 softmax (tile = w >> 3, half = (w >> 2) & 1, lane quarter = w & 3), warp 16
// TMA, warp 17 MMA + TMEM allocation.
constexpr int ATTN3_THREADS = 18 * 32;

DF_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
DF_DEV void sts_u16(uint32_t a, unsigned short v) { asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory"); }
DF_DEV unsigned short lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
DF_DEV void sts_f32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory"); }
DF_DEV float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

template <int EXPM>
__global__ void __launch_bounds__(ATTN3_THREADS, 1)
    attn_tc3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                    int dh_real, float scale_log2, int Hs) {
  constexpr int DH = 128;
  using Cfg = Attn2Cfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [KST]
  uint64_t* k_empty = bars + 4;   // [KST]
  uint64_t* v_full = bars + 7;    // [VST]
  uint64_t* v_empty = bars + 9;   // [VST]
  uint64_t* s_full = bars + 11;   // [2] per Q tile
  // P of tile t is published in key quarters (32 keys each; quarter 2 hc + q is written by
  // the 4 warps of half hc, chunk q): PV starts on the first quarter while the rest is
  // still being exponentiated
  uint64_t* p_q = bars + 18;      // [2 tiles][4 quarters], one arrive per warp
  uint64_t* o_done = bars + 15;   // [2] per Q tile (after the last PV)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  __half* red = reinterpret_cast<__half*>(smem + Cfg::OFF_BAR + 256);  // [2 tiles][2 halves][128 rows]

  const int warp = warp_id();
  const int lane = lane_id();
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * 256;
  const int nkb = (Nk + 127) / 128;

  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < Cfg::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      for (int u = 0; u < 4; ++u) mbar_init(&p_q[s * 4 + u], 4);
      mbar_init(&o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 17) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 16) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * Cfg::Q_BYTES);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int a = 0; a < Cfg::ATOMS; ++a)
          tma_load_3d(sQ + t * Cfg::Q_BYTES + a * Cfg::TILE, &tmQ, q_full, a * 64, q0 + t * 128, h);
      int jk = 0, jv = 0;
      while (jv < nkb) {
        if (jk < nkb && jk <= jv + 1) {
          const int st = jk % Cfg::KST;
          mbar_wait(&k_empty[st], ((jk / Cfg::KST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::KV_BYTES);
#pragma unroll
          for (int a = 0; a < Cfg::ATOMS; ++a)
            tma_load_3d(sK + st * Cfg::KV_BYTES + a * Cfg::TILE, &tmK, &k_full[st], a * 64, jk * 128, h);
          ++jk;
        } else {
          const int st = jv % Cfg::VST;
          mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[st], Cfg::KV_BYTES);
#pragma unroll
          for (int a = 0; a < Cfg::ATOMS; ++a)
            tma_load_3d(sV + st * Cfg::KV_BYTES + a * Cfg::TILE, &tmV, &v_full[st], a * 64, jv * 128, h);
          ++jv;
        }
      }
    }
  } else if (warp == 17) {
    // the whole warp runs the schedule (warp-uniform values live in uniform registers and
    // descriptors are base + constant offsets); one elected lane issues each MMA batch
    constexpr uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16(128, DH, false, true);
    const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t dv = sdesc_sw128(smem_u32(sV), Cfg::TILE, 1024);
    auto issue_qk = [&](int t, int j) {
      const uint64_t a0 = dq + uint64_t((t * Cfg::Q_BYTES) >> 4);
      const uint64_t b0 = dk + uint64_t(((j % Cfg::KST) * Cfg::KV_BYTES) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = ((k >> 2) * Cfg::TILE + (k & 3) * 32) >> 4;
          tc_mma_bf16(tmem + t * 128, a0 + off, b0 + off, idesc_qk, k > 0);
        }
        tc_commit(&s_full[t]);
      }
      __syncwarp();
    };
    // PV of tile t, key quarter u (k-steps 2u, 2u+1); quarters are issued in the order
    // 0, 2, 1, 3 (both halves' first chunks first); the first MMA of block 0 overwrites O
    auto issue_pv = [&](int t, int j, int u, bool first) {
      const uint64_t b0 = dv + uint64_t(((j % Cfg::VST) * Cfg::KV_BYTES) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int k = 2 * u + kk;
          tc_mma_bf16_ts(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8, b0 + uint64_t((k * 2048) >> 4), idesc_pv,
                         !(first && kk == 0));
        }
      }
      __syncwarp();
    };
    auto pv_tile = [&](int t, int j, bool last) {
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int u = (n >> 1) | ((n & 1) << 1);  // 0, 2, 1, 3
        mbar_wait(&p_q[t * 4 + u], j & 1);
        tc_fence_after();
        issue_pv(t, j, u, j == 0 && n == 0);
      }
      if (elect_one()) {
        if (t == 1) tc_commit(&v_empty[j % Cfg::VST]);
        if (last) tc_commit(&o_done[t]);
      }
      __syncwarp();
    };
    auto commit1 = [&](uint64_t* bar) {
      if (elect_one()) tc_commit(bar);
      __syncwarp();
    };
    auto wait_k = [&](int j) {
      mbar_wait(&k_full[j % Cfg::KST], (j / Cfg::KST) & 1);
      tc_fence_after();
    };
    mbar_wait(q_full, 0);
    wait_k(0);
    issue_qk(0, 0);
    issue_qk(1, 0);
    commit1(&k_empty[0]);
    for (int j = 0; j < nkb; ++j) {
      const bool more = j + 1 < nkb;
      mbar_wait(&v_full[j % Cfg::VST], (j / Cfg::VST) & 1);
      pv_tile(0, j, !more);
      if (more) {
        wait_k(j + 1);
        issue_qk(0, j + 1);
      }
      pv_tile(1, j, !more);
      if (more) {
        issue_qk(1, j + 1);
        commit1(&k_empty[(j + 1) % Cfg::KST]);
      }
    }
  } else {
    const int t = warp >> 3;              // Q tile
    const int hc = (warp >> 2) & 1;       // key / output column half
    const int ew = warp & 3;              // TMEM lane quarter
    const int r = ew * 32 + lane;         // query row within the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const uint32_t ts = tmem + lane_off + t * 128;
    const uint32_t to = tmem + lane_off + Cfg::O_COL + t * DH + 64 * hc;
    const uint32_t red_own = smem_u32(red + (t * 2 + hc) * 128 + r);
    const uint32_t red_oth = smem_u32(red + (t * 2 + (hc ^ 1)) * 128 + r);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      if (EXPM == 9) {  // profiling only: tensor cores + synchronisation, no softmax (wrong results)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&p_q[t * 4 + 2 * hc]);
          mbar_arrive(&p_q[t * 4 + 2 * hc + 1]);
        }
        continue;
      }
      float s[64];
      tmem_ld32(ts + 64 * hc, s);
      tmem_ld32(ts + 64 * hc + 32, s + 32);
      tc_wait_ld();
      const int valid = Nk - j * 128 - 64 * hc;
      if (valid < 64) {  // ragged last key block (warp-uniform)
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (i >= valid) s[i] = -INFINITY;
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 64; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(s[i + 2 * u], s[i + 2 * u + 1]));
      }
      // both halves must use the same stabiliser: exchange maxima rounded up to fp16
      const __half hm = __float2half_ru(fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2);
      sts_u16(red_own, __half_as_ushort(hm));
      named_bar_sync(1 + t, 256);
      const float mx = fmaxf(__half2float(hm), __half2float(__ushort_as_half(lds_u16(red_oth))));
      const bool need = mx > m_used + 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_used;
        if (j > 0) {
          const float alpha = exp2f(m_used - m_new);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < 64; c += 16) {
            float o[16];
            tmem_ld16(to + c, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= alpha;
            tmem_st16(to + c, reinterpret_cast<uint32_t*>(o));
          }
        }
        m_used = m_new;
      }
      float2 lsum2 = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      const float2 nm2 = make_float2(-m_used, -m_used);
      // keys 64 hc + 32 q .. +32 -> packed P columns 32 hc + 16 q .. +16 (S was read by both
      // halves before the named barrier); chunk 0's store drains while chunk 1 is computed
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2), i, lsum2);
      tmem_st16(ts + 32 * hc, pk);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[32 + 2 * i], s[32 + 2 * i + 1]), sc2, nm2), i, lsum2);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_q[t * 4 + 2 * hc]);
      tmem_st16(ts + 32 * hc + 16, pk);
      l += lsum2.x + lsum2.y;
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_q[t * 4 + 2 * hc + 1]);
    }
    mbar_wait(&o_done[t], 0);
    tc_fence_after();
    // row sum = both halves' partial sums; Q_t's shared memory is free once O_t is final
    float* lred = reinterpret_cast<float*>(sQ + t * Cfg::Q_BYTES);
    lred[hc * 128 + r] = l;
    named_bar_sync(1 + t, 256);
    const float inv = 1.0f / (l + lred[(hc ^ 1) * 128 + r]);
    const int q = q0 + t * 128 + r;
    const int hb = h / Hs, hl = h - hb * Hs;
    bf16* orow = O + (size_t(hb) * Nq + q) * Hs * dh_real + size_t(hl) * dh_real + 64 * hc;
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
      float o[32];
      tmem_ld32(to + c, o);
      tc_wait_ld();
      if (q < Nq) {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] *= inv;
        store_vec<32>(orow + c, o);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int EXPM>
static cudaError_t launch_attn3(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, bf16* O, int H,
                                int Nq, int Nk, int dh, float scale, cudaStream_t st, int hs) {
  using Cfg = Attn2Cfg<128>;
  constexpr int SMEM = Cfg::SMEM + 1024;  // + the fp16 max exchange (1 KB) after the barriers
  static_assert(SMEM <= 232448, "attn_tc3 shared memory");
  auto kern = attn_tc3_kernel<EXPM>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((Nq + 255) / 256, H);
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O,   (void*)&H,
                  (void*)&Nq, (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs};
  return launch_ex((const void*)kern, grid, dim3(ATTN3_THREADS), SMEM, st, args);
}

// ------------------------------------------------------------------ attn_pair: CTA-pair (cta_group::2)
// A cluster of two CTAs runs M = 256 MMAs: query tile t of the pair is 256 rows, 128 in each
// CTA's shared memory and TMEM. Each CTA stages HALF of every K/V block (K: 64 of the 128
// keys, all of dh; V: all 128 keys, 64 of the 128 dh columns), so per SM the shared-memory
// operand reads of QK^T and PV and the TMA writes halve against attn_tc2 (whose SS-mode
// M=128 QK^T alone saturates the 128 B/clk shared-memory port). The leader CTA's MMA thread
// issues for both; ring barriers live on the leader (count 2: its expect_tx + the peer's
// arrive), MMA completions are multicast to both CTAs. Softmax is per CTA over its own 128
// rows, exactly as in attn_tc2 (P written into TMEM, consumed as the A operand of PV).
struct AttnPairCfg {
  static constexpr int DH = 128;
  static constexpr int ATOM = 64 * 128;              // SW128 atom of 64 rows (8 KB)
  static constexpr int Q_BYTES = 2 * 128 * 128;      // one 128-row Q tile (2 dh atoms of 16 KB)
  static constexpr int K_BYTES = 64 * 128 * 2;       // half K block: 64 keys x 128 dh
  static constexpr int V_BYTES = 128 * 64 * 2;       // half V block: 128 keys x 64 dh
  static constexpr int KST = 4;
  static constexpr int VST = 4;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * V_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t O_COL = 256;
};

template <bool POLY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                     int dh_real, float scale_log2, int Hs) {
  using Cfg = AttnPairCfg;
  constexpr int DH = Cfg::DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;                 // [KST]  leader
  uint64_t* k_empty = k_full + Cfg::KST;       // [KST]  both (multicast commit)
  uint64_t* v_full = k_empty + Cfg::KST;       // [VST]  leader
  uint64_t* v_empty = v_full + Cfg::VST;       // [VST]  both
  uint64_t* s_full = v_empty + Cfg::VST;       // [2]    both
  uint64_t* p_full = s_full + 2;               // [2]    leader: 4 softmax warps x 2 CTAs
  uint64_t* o_done = p_full + 2;               // [2]    both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int h = blockIdx.y;
  const int qp = (blockIdx.x >> 1) * 512;      // first query row of the pair
  const int nkb = (Nk + 127) / 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 2);
    for (int s = 0; s < Cfg::KST; ++s) {
      mbar_init(&k_full[s], 2);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::VST; ++s) {
      mbar_init(&v_full[s], 2);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 8);
      mbar_init(&o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // this CTA's rows of tile t: qp + t*256 + rank*128
      if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * Cfg::Q_BYTES);
      else mbar_arrive_cluster(q_full, 0);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int a = 0; a < 2; ++a)
          tma_load_3d_pair(sQ + t * Cfg::Q_BYTES + a * 2 * Cfg::ATOM, &tmQ, q_full, a * 64,
                           qp + t * 256 + int(rank) * 128, h);
      int jk = 0, jv = 0;
      while (jv < nkb) {
        if (jk < nkb && jk <= jv + 2) {
          const int st = jk % Cfg::KST;
          mbar_wait(&k_empty[st], ((jk / Cfg::KST) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&k_full[st], 2 * Cfg::K_BYTES);
          else mbar_arrive_cluster(&k_full[st], 0);
#pragma unroll
          for (int a = 0; a < 2; ++a)  // keys jk*128 + rank*64 .. +64, dh atom a
            tma_load_3d_pair(sK + st * Cfg::K_BYTES + a * Cfg::ATOM, &tmK, &k_full[st], a * 64,
                             jk * 128 + int(rank) * 64, h);
          ++jk;
        } else {
          const int st = jv % Cfg::VST;
          mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&v_full[st], 2 * Cfg::V_BYTES);
          else mbar_arrive_cluster(&v_full[st], 0);
          // keys jv*128 .. +128, dh columns rank*64 .. +64
          tma_load_3d_pair(sV + st * Cfg::V_BYTES, &tmV, &v_full[st], int(rank) * 64, jv * 128, h);
          ++jv;
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(256, DH, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_qk = [&](int t, int j) {
        const uint32_t k_addr = smem_u32(sK + (j % Cfg::KST) * Cfg::K_BYTES);
        const uint32_t qa = q_addr + t * Cfg::Q_BYTES;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          // A: 128 rows per CTA, dh atoms of 16 KB; B: 64 keys per CTA, dh atoms of 8 KB
          tc_mma_bf16_pair(tmem + t * 128, sdesc_sw128(qa + (k >> 2) * 2 * Cfg::ATOM + (k & 3) * 32, 16, 1024),
                           sdesc_sw128(k_addr + (k >> 2) * Cfg::ATOM + (k & 3) * 32, 16, 1024), idesc_qk, k > 0);
        }
        tc_commit_pair(&s_full[t], 0x3);
      };
      auto issue_pv = [&](int t, int j) {
        const uint32_t v_addr = smem_u32(sV + (j % Cfg::VST) * Cfg::V_BYTES);
#pragma unroll
        for (int k = 0; k < 8; ++k)  // 128 keys / 16; P_t = TMEM columns k*8.. of S_t
          tc_mma_bf16_ts_pair(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8,
                              sdesc_sw128(v_addr + k * 2048, Cfg::V_BYTES, 1024), idesc_pv, (j > 0 || k > 0));
      };
      auto wait_k = [&](int j) {
        mbar_wait(&k_full[j % Cfg::KST], (j / Cfg::KST) & 1);
        tc_fence_after();
      };
      mbar_wait(q_full, 0);
      wait_k(0);
      issue_qk(0, 0);
      issue_qk(1, 0);
      tc_commit_pair(&k_empty[0], 0x3);
      for (int j = 0; j < nkb; ++j) {
        const bool more = j + 1 < nkb;
        mbar_wait(&v_full[j % Cfg::VST], (j / Cfg::VST) & 1);
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        issue_pv(0, j);
        if (!more) tc_commit_pair(&o_done[0], 0x3);
        if (more) {
          wait_k(j + 1);
          issue_qk(0, j + 1);
        }
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        issue_pv(1, j);
        tc_commit_pair(&v_empty[j % Cfg::VST], 0x3);
        if (!more) tc_commit_pair(&o_done[1], 0x3);
        if (more) {
          issue_qk(1, j + 1);
          tc_commit_pair(&k_empty[(j + 1) % Cfg::KST], 0x3);
        }
      }
    }
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;        // Q tile of this softmax group (warps 4-7, 8-11)
    const int ew = warp & 3;              // TMEM lane quarter = warp id mod 4
    const int r = ew * 32 + lane;         // query row within this CTA's half of the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const uint32_t ts = tmem + lane_off + t * 128;
    const uint32_t to = tmem + lane_off + Cfg::O_COL + t * DH;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      const int valid = Nk - j * 128;
      float s[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(ts + c, s + c);
      tc_wait_ld();
      if (valid < 128) {  // ragged last key block (warp-uniform)
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= valid) s[i] = -INFINITY;
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 128; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(s[i + 2 * u], s[i + 2 * u + 1]));
      }
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
      const bool need = mx > m_used + 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_used;
        if (j > 0) {
          // s_full for block j implies PV_{j-1} (issued earlier) completed: O_t is stable
          const float alpha = exp2f(m_used - m_new);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < DH; c += 16) {
            float o[16];
            tmem_ld16(to + c, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= alpha;
            tmem_st16(to + c, reinterpret_cast<uint32_t*>(o));
          }
        }
        m_used = m_new;
      }
      float2 lsum2 = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      const float2 nm2 = make_float2(-m_used, -m_used);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ffma2(make_float2(s[32 * q + 2 * i], s[32 * q + 2 * i + 1]), sc2, nm2);
          float2 p;
          if (POLY && (i & 7) >= 5) {
            p = exp2_poly2(x);
          } else {
            p.x = ex2_approx(x.x);
            p.y = ex2_approx(x.y);
          }
          lsum2 = fadd2(lsum2, p);
          pk[i] = pack_bf16x2(p.x, p.y);
        }
        tmem_st16(ts + 16 * q, pk);
      }
      l += lsum2.x + lsum2.y;
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&p_full[t], 0);  // one arrive per warp, on the leader
    }
    mbar_wait(&o_done[t], 0);
    tc_fence_after();
    const float inv = 1.0f / l;
    const int q = qp + t * 256 + int(rank) * 128 + r;
    const int hb = h / Hs, hl = h - hb * Hs;
    bf16* orow = O + (size_t(hb) * Nq + q) * Hs * dh_real + size_t(hl) * dh_real;
#pragma unroll 1
    for (int c = 0; c < DH; c += 32) {
      float o[32];
      tmem_ld32(to + c, o);
      tc_wait_ld();
      if (q < Nq && c < dh_real) {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] *= inv;
        if (dh_real - c >= 32) store_vec<32>(orow + c, o);
        else
          for (int i = 0; i < dh_real - c; ++i) orow[c + i] = __float2bfloat16_rn(o[i]);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// ------------------------------------------------------------------ attn_pair3: CTA pair + 2 threads per row
// attn_pair's tensor-core schedule (M = 256 over a CTA pair: per SM the QK^T shared-memory
// operand reads drop from 8 KB to 6 KB per 64-clock K step and the PV B reads halve, so the
// 128 B/clk shared-memory port stops pacing the MMAs) with attn_tc3's softmax (two threads
// per query row).  The row maxima are exchanged exactly (fp32) through shared memory.
template <int EXPM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ATTN3_THREADS, 1)
    attn_pair3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                      int dh_real, float scale_log2, int Hs) {
  using Cfg = AttnPairCfg;
  constexpr int DH = Cfg::DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;                 // [KST]  leader
  uint64_t* k_empty = k_full + Cfg::KST;       // [KST]  both (multicast commit)
  uint64_t* v_full = k_empty + Cfg::KST;       // [VST]  leader
  uint64_t* v_empty = v_full + Cfg::VST;       // [VST]  both
  uint64_t* s_full = v_empty + Cfg::VST;       // [2]    both
  uint64_t* p_full = s_full + 2;               // [2]    leader: 8 softmax warps x 2 CTAs
  uint64_t* o_done = p_full + 2;               // [2]    both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  uint64_t* p_q = o_done + 3;                  // [2 tiles][4 key quarters] leader: 4 warps x 2 CTAs
  float* red = reinterpret_cast<float*>(smem + Cfg::OFF_BAR + 256);  // [2 tiles][2 halves][128 rows]

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int h = blockIdx.y;
  const int qp = (blockIdx.x >> 1) * 512;      // first query row of the pair
  const int nkb = (Nk + 127) / 128;

  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 2);
    for (int s = 0; s < Cfg::KST; ++s) {
      mbar_init(&k_full[s], 2);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::VST; ++s) {
      mbar_init(&v_full[s], 2);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 16);
      for (int u = 0; u < 4; ++u) mbar_init(&p_q[s * 4 + u], 8);
      mbar_init(&o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 17) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 16) {
    if (lane == 0) {
      if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * Cfg::Q_BYTES);
      else mbar_arrive_cluster(q_full, 0);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int a = 0; a < 2; ++a)
          tma_load_3d_pair(sQ + t * Cfg::Q_BYTES + a * 2 * Cfg::ATOM, &tmQ, q_full, a * 64,
                           qp + t * 256 + int(rank) * 128, h);
      int jk = 0, jv = 0;
      while (jv < nkb) {
        if (jk < nkb && jk <= jv + 2) {
          const int st = jk % Cfg::KST;
          mbar_wait(&k_empty[st], ((jk / Cfg::KST) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&k_full[st], 2 * Cfg::K_BYTES);
          else mbar_arrive_cluster(&k_full[st], 0);
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_3d_pair(sK + st * Cfg::K_BYTES + a * Cfg::ATOM, &tmK, &k_full[st], a * 64,
                             jk * 128 + int(rank) * 64, h);
          ++jk;
        } else {
          const int st = jv % Cfg::VST;
          mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&v_full[st], 2 * Cfg::V_BYTES);
          else mbar_arrive_cluster(&v_full[st], 0);
          tma_load_3d_pair(sV + st * Cfg::V_BYTES, &tmV, &v_full[st], int(rank) * 64, jv * 128, h);
          ++jv;
        }
      }
    }
  } else if (warp == 17) {
    if (leader) {  // whole warp runs the schedule; one elected lane issues each MMA batch
      constexpr uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(256, DH, false, true);
      const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(sV), Cfg::V_BYTES, 1024);
      auto issue_qk = [&](int t, int j) {
        const uint64_t a0 = dq + uint64_t((t * Cfg::Q_BYTES) >> 4);
        const uint64_t b0 = dk + uint64_t(((j % Cfg::KST) * Cfg::K_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            tc_mma_bf16_pair(tmem + t * 128, a0 + uint64_t(((k >> 2) * 2 * Cfg::ATOM + (k & 3) * 32) >> 4),
                             b0 + uint64_t(((k >> 2) * Cfg::ATOM + (k & 3) * 32) >> 4), idesc_qk, k > 0);
          tc_commit_pair(&s_full[t], 0x3);
        }
        __syncwarp();
      };
      // PV per key quarter (order 0, 2, 1, 3), as in attn_tc3
      auto issue_pv = [&](int t, int j, int u, bool first) {
        const uint64_t b0 = dv + uint64_t(((j % Cfg::VST) * Cfg::V_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int k = 2 * u + kk;
            tc_mma_bf16_ts_pair(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8, b0 + uint64_t((k * 2048) >> 4),
                                idesc_pv, !(first && kk == 0));
          }
        }
        __syncwarp();
      };
      auto pv_tile = [&](int t, int j, bool last) {
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          const int u = (n >> 1) | ((n & 1) << 1);
          mbar_wait(&p_q[t * 4 + u], j & 1);
          tc_fence_after();
          issue_pv(t, j, u, j == 0 && n == 0);
        }
        if (elect_one()) {
          if (t == 1) tc_commit_pair(&v_empty[j % Cfg::VST], 0x3);
          if (last) tc_commit_pair(&o_done[t], 0x3);
        }
        __syncwarp();
      };
      auto commit1 = [&](uint64_t* bar) {
        if (elect_one()) tc_commit_pair(bar, 0x3);
        __syncwarp();
      };
      auto wait_k = [&](int j) {
        mbar_wait(&k_full[j % Cfg::KST], (j / Cfg::KST) & 1);
        tc_fence_after();
      };
      mbar_wait(q_full, 0);
      wait_k(0);
      issue_qk(0, 0);
      issue_qk(1, 0);
      commit1(&k_empty[0]);
      for (int j = 0; j < nkb; ++j) {
        const bool more = j + 1 < nkb;
        mbar_wait(&v_full[j % Cfg::VST], (j / Cfg::VST) & 1);
        pv_tile(0, j, !more);
        if (more) {
          wait_k(j + 1);
          issue_qk(0, j + 1);
        }
        pv_tile(1, j, !more);
        if (more) {
          issue_qk(1, j + 1);
          commit1(&k_empty[(j + 1) % Cfg::KST]);
        }
      }
    }
  } else {
    const int t = warp >> 3;              // Q tile
    const int hc = (warp >> 2) & 1;       // key / output column half
    const int ew = warp & 3;              // TMEM lane quarter
    const int r = ew * 32 + lane;         // query row within this CTA's half of the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const uint32_t ts = tmem + lane_off + t * 128;
    const uint32_t to = tmem + lane_off + Cfg::O_COL + t * DH + 64 * hc;
    const uint32_t red_own = smem_u32(red + (t * 2 + hc) * 128 + r);
    const uint32_t red_oth = smem_u32(red + (t * 2 + (hc ^ 1)) * 128 + r);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      if (EXPM == 9) {  // profiling only: tensor cores + synchronisation, no softmax (wrong results)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(&p_q[t * 4 + 2 * hc], 0);
          mbar_arrive_cluster(&p_q[t * 4 + 2 * hc + 1], 0);
        }
        continue;
      }
      float s[64];
      tmem_ld32(ts + 64 * hc, s);
      tmem_ld32(ts + 64 * hc + 32, s + 32);
      tc_wait_ld();
      const int valid = Nk - j * 128 - 64 * hc;
      if (valid < 64) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (i >= valid) s[i] = -INFINITY;
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 64; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(s[i + 2 * u], s[i + 2 * u + 1]));
      }
      const float mloc = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
      sts_f32(red_own, mloc);
      named_bar_sync(1 + t, 256);
      const float mx = fmaxf(mloc, lds_f32(red_oth));
      const bool need = mx > m_used + 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_used;
        if (j > 0) {
          const float alpha = exp2f(m_used - m_new);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < 64; c += 16) {
            float o[16];
            tmem_ld16(to + c, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= alpha;
            tmem_st16(to + c, reinterpret_cast<uint32_t*>(o));
          }
        }
        m_used = m_new;
      }
      float2 lsum2 = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      const float2 nm2 = make_float2(-m_used, -m_used);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2), i, lsum2);
      tmem_st16(ts + 32 * hc, pk);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[32 + 2 * i], s[32 + 2 * i + 1]), sc2, nm2), i, lsum2);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc], 0);  // one arrive per warp, on the leader
      tmem_st16(ts + 32 * hc + 16, pk);
      l += lsum2.x + lsum2.y;
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc + 1], 0);
    }
    mbar_wait(&o_done[t], 0);
    tc_fence_after();
    float* lred = reinterpret_cast<float*>(sQ + t * Cfg::Q_BYTES);  // Q_t is free once O_t is final
    lred[hc * 128 + r] = l;
    named_bar_sync(1 + t, 256);
    const float inv = 1.0f / (l + lred[(hc ^ 1) * 128 + r]);
    const int q = qp + t * 256 + int(rank) * 128 + r;
    const int hb = h / Hs, hl = h - hb * Hs;
    bf16* orow = O + (size_t(hb) * Nq + q) * Hs * dh_real + size_t(hl) * dh_real + 64 * hc;
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
      float o[32];
      tmem_ld32(to + c, o);
      tc_wait_ld();
      if (q < Nq) {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] *= inv;
        store_vec<32>(orow + c, o);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// ------------------------------------------------------------------ attn_pp: persistent CTA pair
// attn_pair3's MMA schedule and softmax, but each CTA pair loops over work items (512 query
// rows of one head; items head-major so consecutive items reuse K/V in L2) instead of one
// item per launch slot: the TMEM allocation and barrier set-up happen once, the next item's
// Q is loaded while the current item's last blocks run (q_empty is committed after its
// last QK), and the next item's QKs start while the softmax warps normalise and store the
// previous O (the first PV of an item waits for o_free, the epilogue's release of O_t).
// Short-key launches (cross-attention, 4 key blocks per item) are dominated by exactly
// these per-item costs.  All barrier phases run on counters that continue across items.
template <int EXPM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ATTN3_THREADS, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                   int dh_real, float scale_log2, int Hs) {
  using Cfg = AttnPairCfg;
  constexpr int DH = Cfg::DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;                 // leader
  uint64_t* q_empty = bars + 1;                // both (multicast commit after the item's last QK)
  uint64_t* k_full = bars + 2;                 // [KST]  leader
  uint64_t* k_empty = k_full + Cfg::KST;       // [KST]  both
  uint64_t* v_full = k_empty + Cfg::KST;       // [VST]  leader
  uint64_t* v_empty = v_full + Cfg::VST;       // [VST]  both
  uint64_t* s_full = v_empty + Cfg::VST;       // [2]    both
  uint64_t* o_done = s_full + 2;               // [2]    both
  uint64_t* o_free = o_done + 2;               // [2]    leader: 8 softmax warps x 2 CTAs
  uint64_t* p_q = o_free + 2;                  // [2][4] leader: 4 warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_q + 8);
  float* red = reinterpret_cast<float*>(smem + Cfg::OFF_BAR + 512);    // [2 tiles][2 halves][128] row max
  float* lred = red + 512;                                              // [2 tiles][2 halves][128] row sum

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nkb = (Nk + 127) / 128;
  const int nqp = (Nq + 511) / 512;
  const int items = nqp * H;
  const int cid = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 2);
    mbar_init(q_empty, 1);
    for (int s = 0; s < Cfg::KST; ++s) {
      mbar_init(&k_full[s], 2);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::VST; ++s) {
      mbar_init(&v_full[s], 2);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&o_done[s], 1);
      mbar_init(&o_free[s], 16);
      for (int u = 0; u < 4; ++u) mbar_init(&p_q[s * 4 + u], 8);
    }
    fence_mbar_init();
  }
  if (warp == 17) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 16) {
    if (lane == 0) {
      int jk = 0, jv = 0;  // running K / V block counters (ring slots and phases)
      int n = 0;           // items done by this pair
      for (int it = cid; it < items; it += npairs, ++n) {
        const int h = it / nqp, qp = (it - h * nqp) * 512;
        if (n > 0) mbar_wait(q_empty, (n - 1) & 1);  // previous item's QKs no longer read Q
        if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * Cfg::Q_BYTES);
        else mbar_arrive_cluster(q_full, 0);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_3d_pair(sQ + t * Cfg::Q_BYTES + a * 2 * Cfg::ATOM, &tmQ, q_full, a * 64,
                             qp + t * 256 + int(rank) * 128, h);
        const int k_end = jk + nkb, v_end = jv + nkb;
        while (jv < v_end) {
          if (jk < k_end && jk <= jv + 2) {
            const int st = jk % Cfg::KST;
            mbar_wait(&k_empty[st], ((jk / Cfg::KST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&k_full[st], 2 * Cfg::K_BYTES);
            else mbar_arrive_cluster(&k_full[st], 0);
            const int kb = jk - (k_end - nkb);
#pragma unroll
            for (int a = 0; a < 2; ++a)
              tma_load_3d_pair(sK + st * Cfg::K_BYTES + a * Cfg::ATOM, &tmK, &k_full[st], a * 64,
                               kb * 128 + int(rank) * 64, h);
            ++jk;
          } else {
            const int st = jv % Cfg::VST;
            mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&v_full[st], 2 * Cfg::V_BYTES);
            else mbar_arrive_cluster(&v_full[st], 0);
            const int vb = jv - (v_end - nkb);
            tma_load_3d_pair(sV + st * Cfg::V_BYTES, &tmV, &v_full[st], int(rank) * 64, vb * 128, h);
            ++jv;
          }
        }
      }
    }
  } else if (warp == 17) {
    if (leader) {  // whole warp runs the schedule; one elected lane issues each MMA batch
      constexpr uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(256, DH, false, true);
      const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(sV), Cfg::V_BYTES, 1024);
      auto issue_qk = [&](int t, int jg) {
        const uint64_t a0 = dq + uint64_t((t * Cfg::Q_BYTES) >> 4);
        const uint64_t b0 = dk + uint64_t(((jg % Cfg::KST) * Cfg::K_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            tc_mma_bf16_pair(tmem + t * 128, a0 + uint64_t(((k >> 2) * 2 * Cfg::ATOM + (k & 3) * 32) >> 4),
                             b0 + uint64_t(((k >> 2) * Cfg::ATOM + (k & 3) * 32) >> 4), idesc_qk, k > 0);
          tc_commit_pair(&s_full[t], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int jg, int u, bool first) {
        const uint64_t b0 = dv + uint64_t(((jg % Cfg::VST) * Cfg::V_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int k = 2 * u + kk;
            tc_mma_bf16_ts_pair(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8, b0 + uint64_t((k * 2048) >> 4),
                                idesc_pv, !(first && kk == 0));
          }
        }
        __syncwarp();
      };
      auto commit1 = [&](uint64_t* bar) {
        if (elect_one()) tc_commit_pair(bar, 0x3);
        __syncwarp();
      };
      auto wait_k = [&](int jg) {
        mbar_wait(&k_full[jg % Cfg::KST], (jg / Cfg::KST) & 1);
        tc_fence_after();
      };
      int g = 0;  // running key-block counter (ring slots, S/P phases)
      int n = 0;
      for (int it = cid; it < items; it += npairs, ++n, g += nkb) {
        auto pv_tile = [&](int t, int j) {
          const int jg = g + j;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int u = (m >> 1) | ((m & 1) << 1);  // quarters 0, 2, 1, 3
            mbar_wait(&p_q[t * 4 + u], jg & 1);
            tc_fence_after();
            issue_pv(t, jg, u, j == 0 && m == 0);
          }
          if (elect_one()) {
            if (t == 1) tc_commit_pair(&v_empty[jg % Cfg::VST], 0x3);
            if (j == nkb - 1) tc_commit_pair(&o_done[t], 0x3);
          }
          __syncwarp();
        };
        mbar_wait(q_full, n & 1);
        wait_k(g);
        issue_qk(0, g);
        issue_qk(1, g);
        commit1(&k_empty[g % Cfg::KST]);
        if (nkb == 1) commit1(q_empty);
        for (int j = 0; j < nkb; ++j) {
          const bool more = j + 1 < nkb;
          mbar_wait(&v_full[(g + j) % Cfg::VST], ((g + j) / Cfg::VST) & 1);
          if (j == 0 && n > 0) {  // O_0 of the previous item has been read out
            mbar_wait(&o_free[0], (n - 1) & 1);
            tc_fence_after();
          }
          pv_tile(0, j);
          if (more) {
            wait_k(g + j + 1);
            issue_qk(0, g + j + 1);
          }
          if (j == 0 && n > 0) {
            mbar_wait(&o_free[1], (n - 1) & 1);
            tc_fence_after();
          }
          pv_tile(1, j);
          if (more) {
            issue_qk(1, g + j + 1);
            commit1(&k_empty[(g + j + 1) % Cfg::KST]);
            if (j + 2 == nkb) commit1(q_empty);  // the item's last QK is issued: Q may be reloaded
          }
        }
      }
    }
  } else {
    const int t = warp >> 3;              // Q tile
    const int hc = (warp >> 2) & 1;       // key / output column half
    const int ew = warp & 3;              // TMEM lane quarter
    const int r = ew * 32 + lane;         // query row within this CTA's half of the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const uint32_t ts = tmem + lane_off + t * 128;
    const uint32_t to = tmem + lane_off + Cfg::O_COL + t * DH + 64 * hc;
    const uint32_t red_own = smem_u32(red + (t * 2 + hc) * 128 + r);
    const uint32_t red_oth = smem_u32(red + (t * 2 + (hc ^ 1)) * 128 + r);
    const uint32_t lred_own = smem_u32(lred + (t * 2 + hc) * 128 + r);
    const uint32_t lred_oth = smem_u32(lred + (t * 2 + (hc ^ 1)) * 128 + r);
    // one loop-carried counter (n); item and block indices are recomputed from it, which
    // keeps the 96-register budget of 18 warps free of spills
    const int my_items = cid < items ? (items - 1 - cid) / npairs + 1 : 0;
    for (int n = 0; n < my_items; ++n) {
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkb; ++j) {
        const int jg = n * nkb + j;
        mbar_wait(&s_full[t], jg & 1);
        tc_fence_after();
        float s[64];
        tmem_ld32(ts + 64 * hc, s);
        tmem_ld32(ts + 64 * hc + 32, s + 32);
        tc_wait_ld();
        const int valid = Nk - j * 128 - 64 * hc;
        if (valid < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i >= valid) s[i] = -INFINITY;
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 64; i += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(s[i + 2 * u], s[i + 2 * u + 1]));
        }
        const float mloc = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
        sts_f32(red_own, mloc);
        named_bar_sync(1 + t, 256);
        const float mx = fmaxf(mloc, lds_f32(red_oth));
        const bool need = mx > m_used + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_used;
          if (j > 0) {
            const float alpha = exp2f(m_used - m_new);
            l *= alpha;
#pragma unroll 1
            for (int c = 0; c < 64; c += 16) {
              float o[16];
              tmem_ld16(to + c, o);
              tc_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= alpha;
              tmem_st16(to + c, reinterpret_cast<uint32_t*>(o));
            }
          }
          m_used = m_new;
        }
        float2 lsum2 = make_float2(0.f, 0.f);
        const float2 sc2 = make_float2(scale_log2, scale_log2);
        const float2 nm2 = make_float2(-m_used, -m_used);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2), i, lsum2);
        tmem_st16(ts + 32 * hc, pk);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[32 + 2 * i], s[32 + 2 * i + 1]), sc2, nm2), i, lsum2);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc], 0);
        tmem_st16(ts + 32 * hc + 16, pk);
        l += lsum2.x + lsum2.y;
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc + 1], 0);
      }
      mbar_wait(&o_done[t], n & 1);
      tc_fence_after();
      sts_f32(lred_own, l);
      named_bar_sync(1 + t, 256);
      const float inv = 1.0f / (l + lds_f32(lred_oth));
      const int it = cid + n * npairs;
      const int h = it / nqp, qp = (it - h * nqp) * 512;
      const int q = qp + t * 256 + int(rank) * 128 + r;
      const int hb = h / Hs, hl = h - hb * Hs;
      bf16* orow = O + (size_t(hb) * Nq + q) * Hs * dh_real + size_t(hl) * dh_real + 64 * hc;
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        float o[32];
        tmem_ld32(to + c, o);
        tc_wait_ld();
        if (q < Nq) {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= inv;
          store_vec<32>(orow + c, o);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&o_free[t], 0);  // O_t may be overwritten by the next item
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

template <int EXPM>
static cudaError_t launch_attn_pp(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh,
                                  float scale, cudaStream_t st, int hs) {
  using Cfg = AttnPairCfg;
  constexpr int SMEM = Cfg::OFF_BAR + 512 + 4096 + 1024;
  static_assert(SMEM <= 232448, "attn_pp shared memory");
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, 128, 128) || !make_tmap_3d(&tk, K, H, Nk, 128, 64) ||
      !make_tmap_3d(&tv, V, H, Nk, 128, 128))
    return cudaErrorInvalidValue;
  auto kern = attn_pp_kernel<EXPM>;
  static int max_pairs = 0;
  if (!max_pairs) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms());
    cfg.blockDim = dim3(ATTN3_THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    max_pairs = n < num_sms() / 2 ? n : num_sms() / 2;
  }
  const int items = ((Nq + 511) / 512) * H;
  dim3 grid(2 * (items < max_pairs ? items : max_pairs));
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O,   (void*)&H,
                  (void*)&Nq, (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs};
  return launch_ex((const void*)kern, grid, dim3(ATTN3_THREADS), SMEM, st, args);
}

DF_DEV void st_release_u32_attn(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
DF_DEV unsigned ld_acquire_u32_attn(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ attn_ppsk: persistent CTA pair + stream-K
// attn_pair3's MMA schedule and softmax, but each CTA pair loops over work units instead of
// one item per launch slot (an item = 512 query rows of one head; items head-major so
// consecutive items reuse K/V in L2): the TMEM allocation and barrier set-up happen once,
// the next unit's Q is loaded while the current unit's last blocks run (q_empty is committed
// after its last QK), and the next unit's QKs start while the softmax warps normalise and
// store the previous O (the first PV of a unit waits for o_free, the epilogue's release of
// O_t).  All barrier phases run on counters that continue across units.
//
// Stream-K (sk.ws set; the image shape's 192 items on 74 pairs would otherwise leave 30
// pairs idle for the last third): the items x key blocks are cut into equal contiguous
// ranges per pair.  An item cut between pair p (its first key blocks, the "head") and
// pair p + 1 (the rest, the "tail") is finished by p + 1: every pair runs its head unit
// first and publishes the unnormalised O, the row max in use m and the half-row sums l
// (fp32) in its workspace slot with an epoch flag; its tail unit then waits for slot
// p - 1, merges O = O_a 2^(m_a - m) + O_b 2^(m_b - m) (m = max), l likewise, and
// normalises.  The split points depend only on the shape and the pair count: deterministic.
constexpr int SK_MAX_PAIRS = 80;
struct AttnSK {
  float* ws;          // [pairs][2 CTAs] slots of SK_SLOT floats
  unsigned* flag;     // [pairs][2 CTAs] epochs
  unsigned epoch;
  // per-pair schedule computed on the host (kernel parameters are read with uniform loads,
  // so the MMA warp's unit loop stays in uniform registers): head item / block count, tail
  // item / first block, whole items [full0, full1)
  short hd_it[SK_MAX_PAIRS], hd_k[SK_MAX_PAIRS], tl_it[SK_MAX_PAIRS], tl_k[SK_MAX_PAIRS];
  short full0[SK_MAX_PAIRS], full1[SK_MAX_PAIRS];
};
constexpr int SK_SLOT = 2 * 2 * 64 * 128 + 2 * 128 + 2 * 2 * 128;  // O [t][hc][64][128], m [t][128], l [t][hc][128]

struct AttnSched {
  int nkb, step;
  int hd_it, hd_k;        // stream-K head unit: item, block count (0 = none)
  int tl_it, tl_k;        // stream-K tail unit: item, first block (0 = none)
  int full0, full1;       // whole items [full0, full1) in steps of `step`
  int state;              // 0: head next, 1: tail next, 2: whole items
  DF_DEV AttnSched(int items, int nkb_, int npairs, int cid, const AttnSK& sk)
      : nkb(nkb_), step(npairs), hd_it(0), hd_k(0), tl_it(0), tl_k(0), full0(cid), full1(items), state(2) {
    if (!sk.ws) return;
    step = 1;
    state = 0;
    hd_it = sk.hd_it[cid], hd_k = sk.hd_k[cid];
    tl_it = sk.tl_it[cid], tl_k = sk.tl_k[cid];
    full0 = sk.full0[cid], full1 = sk.full1[cid];
  }
  DF_DEV bool next(int& it, int& j0, int& j1) {
    if (state == 0) {
      state = 1;
      if (hd_k) {
        it = hd_it, j0 = 0, j1 = hd_k;
        return true;
      }
    }
    if (state == 1) {
      state = 2;
      if (tl_k) {
        it = tl_it, j0 = tl_k, j1 = nkb;
        return true;
      }
    }
    if (full0 >= full1) return false;
    it = full0;
    j0 = 0;
    j1 = nkb;
    full0 += step;
    return true;
  }
};

template <int EXPM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ATTN3_THREADS, 1)
    attn_ppsk_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                   int dh_real, float scale_log2, int Hs, const __grid_constant__ AttnSK sk) {
  using Cfg = AttnPairCfg;
  constexpr int DH = Cfg::DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS/STS, not generic)
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;                 // leader
  uint64_t* q_empty = bars + 1;                // both (multicast commit after the unit's last QK)
  uint64_t* k_full = bars + 2;                 // [KST]  leader
  uint64_t* k_empty = k_full + Cfg::KST;       // [KST]  both
  uint64_t* v_full = k_empty + Cfg::KST;       // [VST]  leader
  uint64_t* v_empty = v_full + Cfg::VST;       // [VST]  both
  uint64_t* s_full = v_empty + Cfg::VST;       // [2]    both
  uint64_t* o_done = s_full + 2;               // [2]    both
  uint64_t* o_free = o_done + 2;               // [2]    leader: 8 softmax warps x 2 CTAs
  uint64_t* p_q = o_free + 2;                  // [2][4] leader: 4 warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_q + 8);
  float* red = reinterpret_cast<float*>(smem + Cfg::OFF_BAR + 512);    // [2 tiles][2 halves][128] row max
  float* lred = red + 512;                                              // [2 tiles][2 halves][128] row sum

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nkb = (Nk + 127) / 128;
  const int nqp = (Nq + 511) / 512;
  const int items = nqp * H;
  const int cid = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const bool use_sk = sk.ws != nullptr;

  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 2);
    mbar_init(q_empty, 1);
    for (int s = 0; s < Cfg::KST; ++s) {
      mbar_init(&k_full[s], 2);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::VST; ++s) {
      mbar_init(&v_full[s], 2);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&o_done[s], 1);
      mbar_init(&o_free[s], 16);
      for (int u = 0; u < 4; ++u) mbar_init(&p_q[s * 4 + u], 8);
    }
    fence_mbar_init();
  }
  if (warp == 17) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 16) {
    if (lane == 0) {
      int jk = 0, jv = 0;  // running K / V block counters (ring slots and phases)
      int n = 0;           // units done by this pair
      AttnSched sc(items, nkb, npairs, cid, sk);
      int it, j0, j1;
      while (sc.next(it, j0, j1)) {
        const int h = it / nqp, qp = (it - h * nqp) * 512;
        if (n > 0) mbar_wait(q_empty, (n - 1) & 1);  // previous unit's QKs no longer read Q
        if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * Cfg::Q_BYTES);
        else mbar_arrive_cluster(q_full, 0);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_3d_pair(sQ + t * Cfg::Q_BYTES + a * 2 * Cfg::ATOM, &tmQ, q_full, a * 64,
                             qp + t * 256 + int(rank) * 128, h);
        const int nb = j1 - j0;
        const int k_end = jk + nb, v_end = jv + nb;
        while (jv < v_end) {
          if (jk < k_end && jk <= jv + 2) {
            const int st = jk % Cfg::KST;
            mbar_wait(&k_empty[st], ((jk / Cfg::KST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&k_full[st], 2 * Cfg::K_BYTES);
            else mbar_arrive_cluster(&k_full[st], 0);
            const int kb = j0 + jk - (k_end - nb);
#pragma unroll
            for (int a = 0; a < 2; ++a)
              tma_load_3d_pair(sK + st * Cfg::K_BYTES + a * Cfg::ATOM, &tmK, &k_full[st], a * 64,
                               kb * 128 + int(rank) * 64, h);
            ++jk;
          } else {
            const int st = jv % Cfg::VST;
            mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&v_full[st], 2 * Cfg::V_BYTES);
            else mbar_arrive_cluster(&v_full[st], 0);
            const int vb = j0 + jv - (v_end - nb);
            tma_load_3d_pair(sV + st * Cfg::V_BYTES, &tmV, &v_full[st], int(rank) * 64, vb * 128, h);
            ++jv;
          }
        }
        ++n;
      }
    }
  } else if (warp == 17) {
    if (leader) {  // whole warp runs the schedule; one elected lane issues each MMA batch
      constexpr uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(256, DH, false, true);
      const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(sV), Cfg::V_BYTES, 1024);
      auto issue_qk = [&](int t, int jg) {
        const uint64_t a0 = dq + uint64_t((t * Cfg::Q_BYTES) >> 4);
        const uint64_t b0 = dk + uint64_t(((jg % Cfg::KST) * Cfg::K_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            tc_mma_bf16_pair(tmem + t * 128, a0 + uint64_t(((k >> 2) * 2 * Cfg::ATOM + (k & 3) * 32) >> 4),
                             b0 + uint64_t(((k >> 2) * Cfg::ATOM + (k & 3) * 32) >> 4), idesc_qk, k > 0);
          tc_commit_pair(&s_full[t], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int jg, int u, bool first) {
        const uint64_t b0 = dv + uint64_t(((jg % Cfg::VST) * Cfg::V_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int k = 2 * u + kk;
            tc_mma_bf16_ts_pair(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8, b0 + uint64_t((k * 2048) >> 4),
                                idesc_pv, !(first && kk == 0));
          }
        }
        __syncwarp();
      };
      auto commit1 = [&](uint64_t* bar) {
        if (elect_one()) tc_commit_pair(bar, 0x3);
        __syncwarp();
      };
      auto wait_k = [&](int jg) {
        mbar_wait(&k_full[jg % Cfg::KST], (jg / Cfg::KST) & 1);
        tc_fence_after();
      };
      int g = 0;  // running key-block counter (ring slots, S/P phases)
      int n = 0;
      AttnSched sc(items, nkb, npairs, cid, sk);
      int it, j0, j1;
      while (sc.next(it, j0, j1)) {
        const int nb = j1 - j0;
        auto pv_tile = [&](int t, int j, int nb_, int g_) {
          const int jg = g_ + j;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int u = (m >> 1) | ((m & 1) << 1);  // quarters 0, 2, 1, 3
            mbar_wait(&p_q[t * 4 + u], jg & 1);
            tc_fence_after();
            issue_pv(t, jg, u, j == 0 && m == 0);
          }
          if (elect_one()) {
            if (t == 1) tc_commit_pair(&v_empty[jg % Cfg::VST], 0x3);
            if (j == nb_ - 1) tc_commit_pair(&o_done[t], 0x3);
          }
          __syncwarp();
        };
        mbar_wait(q_full, n & 1);
        wait_k(g);
        issue_qk(0, g);
        issue_qk(1, g);
        commit1(&k_empty[g % Cfg::KST]);
        if (nb == 1) commit1(q_empty);
        for (int j = 0; j < nb; ++j) {
          const bool more = j + 1 < nb;
          mbar_wait(&v_full[(g + j) % Cfg::VST], ((g + j) / Cfg::VST) & 1);
          if (j == 0 && n > 0) {  // O_0 of the previous unit has been read out
            mbar_wait(&o_free[0], (n - 1) & 1);
            tc_fence_after();
          }
          pv_tile(0, j, nb, g);
          if (more) {
            wait_k(g + j + 1);
            issue_qk(0, g + j + 1);
          }
          if (j == 0 && n > 0) {
            mbar_wait(&o_free[1], (n - 1) & 1);
            tc_fence_after();
          }
          pv_tile(1, j, nb, g);
          if (more) {
            issue_qk(1, g + j + 1);
            commit1(&k_empty[(g + j + 1) % Cfg::KST]);
            if (j + 2 == nb) commit1(q_empty);  // the unit's last QK is issued: Q may be reloaded
          }
        }
        g += nb;
        ++n;
      }
    }
  } else {
    const int t = warp >> 3;              // Q tile
    const int hc = (warp >> 2) & 1;       // key / output column half
    const int ew = warp & 3;              // TMEM lane quarter
    const int r = ew * 32 + lane;         // query row within this CTA's half of the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const uint32_t ts = tmem + lane_off + t * 128;
    const uint32_t to = tmem + lane_off + Cfg::O_COL + t * DH + 64 * hc;
    const uint32_t red_own = smem_u32(red + (t * 2 + hc) * 128 + r);
    const uint32_t red_oth = smem_u32(red + (t * 2 + (hc ^ 1)) * 128 + r);
    const uint32_t lred_own = smem_u32(lred + (t * 2 + hc) * 128 + r);
    const uint32_t lred_oth = smem_u32(lred + (t * 2 + (hc ^ 1)) * 128 + r);
    int g = 0, n = 0;
    AttnSched sc(items, nkb, npairs, cid, sk);
    int it, j0, j1;
    while (sc.next(it, j0, j1)) {
      const int nb = j1 - j0;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        const int jg = g + j;
        mbar_wait(&s_full[t], jg & 1);
        tc_fence_after();
        float s[64];
        tmem_ld32(ts + 64 * hc, s);
        tmem_ld32(ts + 64 * hc + 32, s + 32);
        tc_wait_ld();
        const int valid = Nk - (j0 + j) * 128 - 64 * hc;
        if (valid < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i >= valid) s[i] = -INFINITY;
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 64; i += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u) m4[u] = fmaxf(m4[u], fmaxf(s[i + 2 * u], s[i + 2 * u + 1]));
        }
        const float mloc = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
        sts_f32(red_own, mloc);
        named_bar_sync(1 + t, 256);
        const float mx = fmaxf(mloc, lds_f32(red_oth));
        const bool need = mx > m_used + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_used;
          if (j > 0) {
            const float alpha = exp2f(m_used - m_new);
            l *= alpha;
#pragma unroll 1
            for (int c = 0; c < 64; c += 16) {
              float o[16];
              tmem_ld16(to + c, o);
              tc_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= alpha;
              tmem_st16(to + c, reinterpret_cast<uint32_t*>(o));
            }
          }
          m_used = m_new;
        }
        float2 lsum2 = make_float2(0.f, 0.f);
        const float2 sc2 = make_float2(scale_log2, scale_log2);
        const float2 nm2 = make_float2(-m_used, -m_used);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2), i, lsum2);
        tmem_st16(ts + 32 * hc, pk);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[32 + 2 * i], s[32 + 2 * i + 1]), sc2, nm2), i, lsum2);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc], 0);
        tmem_st16(ts + 32 * hc + 16, pk);
        l += lsum2.x + lsum2.y;
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc + 1], 0);
      }
      mbar_wait(&o_done[t], n & 1);
      tc_fence_after();
      if (use_sk && j1 < nkb) {
        // head unit: publish the unnormalised O (column-major slot: one coalesced 128 B row of
        // lanes per column), the max in use and this half's row sum; the next pair finishes
        float* slot = sk.ws + size_t(cid * 2 + int(rank)) * SK_SLOT;
        float* po = slot + ((t * 2 + hc) * 64) * 128 + r;
#pragma unroll 1
        for (int c = 0; c < 64; c += 32) {
          float o[32];
          tmem_ld32(to + c, o);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) __stcg(po + (c + i) * 128, o[i]);
        }
        if (hc == 0) __stcg(slot + 2 * 2 * 64 * 128 + t * 128 + r, m_used);
        __stcg(slot + 2 * 2 * 64 * 128 + 2 * 128 + (t * 2 + hc) * 128 + r, l);
        __threadfence();
        named_bar_sync(3, 512);  // all 16 softmax warps of this CTA have published
        if (warp == 0 && lane == 0) st_release_u32_attn(sk.flag + cid * 2 + int(rank), sk.epoch);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&o_free[t], 0);
        g += nb;
        ++n;
        continue;
      }
      float sa = 0.f, sb = 1.f;
      const float* pa = nullptr;
      if (use_sk && j0 > 0) {
        // tail unit: merge the previous pair's head partial of this item (same rows: same rank)
        const float* slot = sk.ws + size_t((cid - 1) * 2 + int(rank)) * SK_SLOT;
        if (lane == 0)
          while (ld_acquire_u32_attn(sk.flag + (cid - 1) * 2 + int(rank)) != sk.epoch) __nanosleep(100);
        __syncwarp();
        const float ma = __ldcg(slot + 2 * 2 * 64 * 128 + t * 128 + r);
        const float la = __ldcg(slot + 2 * 2 * 64 * 128 + 2 * 128 + (t * 2 + hc) * 128 + r);
        const float m = fmaxf(ma, m_used);  // both factors <= 1
        sa = exp2f(ma - m);
        sb = exp2f(m_used - m);
        l = la * sa + l * sb;
        pa = slot + ((t * 2 + hc) * 64) * 128 + r;
      }
      sts_f32(lred_own, l);
      named_bar_sync(1 + t, 256);
      const float inv = 1.0f / (l + lds_f32(lred_oth));
      const int h = it / nqp, qp = (it - h * nqp) * 512;
      const int q = qp + t * 256 + int(rank) * 128 + r;
      const int hb = h / Hs, hl = h - hb * Hs;
      bf16* orow = O + (size_t(hb) * Nq + q) * Hs * dh_real + size_t(hl) * dh_real + 64 * hc;
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        float o[32];
        tmem_ld32(to + c, o);
        tc_wait_ld();
        if (pa) {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __ldcg(pa + (c + i) * 128) * sa + o[i] * sb;
        }
        if (q < Nq) {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= inv;
          store_vec<32>(orow + c, o);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&o_free[t], 0);  // O_t may be overwritten by the next unit
      g += nb;
      ++n;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

template <int EXPM>
static cudaError_t launch_attn_ppsk(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh,
                                  float scale, cudaStream_t st, int hs, float* sk_ws, unsigned* sk_flag) {
  using Cfg = AttnPairCfg;
  constexpr int SMEM = Cfg::OFF_BAR + 512 + 4096 + 1024;
  static_assert(SMEM <= 232448, "attn_ppsk shared memory");
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, 128, 128) || !make_tmap_3d(&tk, K, H, Nk, 128, 64) ||
      !make_tmap_3d(&tv, V, H, Nk, 128, 128))
    return cudaErrorInvalidValue;
  auto kern = attn_ppsk_kernel<EXPM>;
  static int max_pairs = 0;
  if (!max_pairs) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms());
    cfg.blockDim = dim3(ATTN3_THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    max_pairs = n < num_sms() / 2 ? n : num_sms() / 2;
  }
  const int items = ((Nq + 511) / 512) * H;
  const int nkb = (Nk + 127) / 128;
  const int pairs = items < max_pairs ? items : max_pairs;
  dim3 grid(2 * pairs);
  // stream-K when whole items would leave > 8 % of the pairs idle on the last round and
  // every pair's share spans at least one whole item (DF_ATTN_SK=0 turns it off)
  static const int sk_env = [] {
    const char* e = getenv("DF_ATTN_SK");
    return e ? atoi(e) : 1;
  }();
  AttnSK sk;
  std::memset(&sk, 0, sizeof(sk));
  const int rounds = (items + pairs - 1) / pairs;
  if (sk_env && sk_ws && sk_flag && items > pairs && items % pairs && nkb >= 8 && pairs <= SK_MAX_PAIRS &&
      items < 32768 && double(items) / (double(rounds) * pairs) < 0.92) {
    static std::atomic<unsigned> epoch{0};
    sk.ws = sk_ws;
    sk.flag = sk_flag;
    sk.epoch = ++epoch;
    if (sk.epoch == 0) sk.epoch = ++epoch;
    const long long total = (long long)items * nkb;
    for (int p = 0; p < pairs; ++p) {  // equal contiguous ranges of items x key blocks
      const long long b = total * p / pairs, e = total * (p + 1) / pairs;
      const int ta = int(b / nkb), ka = int(b % nkb), tb = int(e / nkb), kb = int(e % nkb);
      sk.hd_it[p] = short(tb), sk.hd_k[p] = short(kb);
      sk.tl_it[p] = short(ta), sk.tl_k[p] = short(ka);
      sk.full0[p] = short(ka ? ta + 1 : ta), sk.full1[p] = short(tb);
    }
  }
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O,   (void*)&H,  (void*)&Nq,
                  (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs, (void*)&sk};
  return launch_ex((const void*)kern, grid, dim3(ATTN3_THREADS), SMEM, st, args);
}

template <int EXPM>
static cudaError_t launch_attn_pair3(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk,
                                     int dh, float scale, cudaStream_t st, int hs) {
  using Cfg = AttnPairCfg;
  constexpr int SMEM = Cfg::SMEM + 2048;  // + fp32 max exchange after the barriers
  static_assert(SMEM <= 232448, "attn_pair3 shared memory");
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, 128, 128) || !make_tmap_3d(&tk, K, H, Nk, 128, 64) ||
      !make_tmap_3d(&tv, V, H, Nk, 128, 128))
    return cudaErrorInvalidValue;
  auto kern = attn_pair3_kernel<EXPM>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(2 * ((Nq + 511) / 512), H);
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O,   (void*)&H,
                  (void*)&Nq, (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs};
  return launch_ex((const void*)kern, grid, dim3(ATTN3_THREADS), SMEM, st, args);
}

template <bool POLY>
static cudaError_t launch_attn_pair(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk,
                                    int dh, float scale, cudaStream_t st, int hs) {
  using Cfg = AttnPairCfg;
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, 128, 128) || !make_tmap_3d(&tk, K, H, Nk, 128, 64) ||
      !make_tmap_3d(&tv, V, H, Nk, 128, 128))
    return cudaErrorInvalidValue;
  auto kern = attn_pair_kernel<POLY>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(2 * ((Nq + 511) / 512), H);
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O,   (void*)&H,
                  (void*)&Nq, (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs};
  return launch_ex((const void*)kern, grid, dim3(384), Cfg::SMEM, st, args);
}

template <int DH>
static cudaError_t launch_attn(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh,
                               float scale, cudaStream_t st, int hs, float* sk_ws, unsigned* sk_flag) {
  if constexpr (DH == 128) {
    if (g_attn_impl == 3) {
      static const int poly = [] {
        const char* e = getenv("DF_ATTN_POLY");
        return e ? atoi(e) : 0;
      }();
      return poly ? launch_attn_pair<true>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs)
                  : launch_attn_pair<false>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
    }
  }
  if constexpr (DH == 128) {
    if (g_attn_impl == 7 && dh == 128) {  // persistent + stream-K split of ragged rounds
      static const int poly = [] {
        const char* e = getenv("DF_ATTN_POLY");
        return e ? atoi(e) : 2;
      }();
      return poly == 0 ? launch_attn_ppsk<0>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs, sk_ws, sk_flag)
                       : launch_attn_ppsk<2>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs, sk_ws, sk_flag);
    }
    if (g_attn_impl == 6 && dh == 128) {
      static const int poly = [] {
        const char* e = getenv("DF_ATTN_POLY");
        return e ? atoi(e) : 2;
      }();
      switch (poly) {  // DF_ATTN_POLY: share of exponentials on the FMA pipe (softmax_exp2)
        case 0: return launch_attn_pp<0>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 1: return launch_attn_pp<1>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        default: return launch_attn_pp<2>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
      }
    }
    if (g_attn_impl == 5 && dh == 128) {
      static const int poly = [] {
        const char* e = getenv("DF_ATTN_POLY");
        return e ? atoi(e) : 2;
      }();
      switch (poly) {  // DF_ATTN_POLY: exponential mode (softmax_exp2)
        case 1: return launch_attn_pair3<1>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 2: return launch_attn_pair3<2>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 3: return launch_attn_pair3<3>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 9: return launch_attn_pair3<9>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        default: return launch_attn_pair3<0>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
      }
    }
    if (g_attn_impl == 4 && dh == 128) {
      static const int poly = [] {  // default 2: a quarter of the exponentials on the FMA pipe
        const char* e = getenv("DF_ATTN_POLY");
        return e ? atoi(e) : 2;
      }();
      CUtensorMap tq, tk, tv;
      if (!make_tmap_3d(&tq, Q, H, Nq, DH, 128) || !make_tmap_3d(&tk, K, H, Nk, DH, 128) ||
          !make_tmap_3d(&tv, V, H, Nk, DH, 128))
        return cudaErrorInvalidValue;
      switch (poly) {  // DF_ATTN_POLY: exponential mode (softmax_exp2)
        case 1: return launch_attn3<1>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
        case 2: return launch_attn3<2>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
        case 3: return launch_attn3<3>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
        case 9: return launch_attn3<9>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
        default: return launch_attn3<0>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
      }
    }
  }
  if (g_attn_impl >= 2 || hs != H) {
    CUtensorMap tq, tk, tv;
    if (!make_tmap_3d(&tq, Q, H, Nq, DH, 128) || !make_tmap_3d(&tk, K, H, Nk, DH, 128) ||
        !make_tmap_3d(&tv, V, H, Nk, DH, 128))
      return cudaErrorInvalidValue;
    static const int poly = [] {
      const char* e = getenv("DF_ATTN_POLY");  // 1: 3/8 of the exponentials by polynomial on the FMA pipe
      return e ? atoi(e) : 0;
    }();
    static const int dbg = [] {
      const char* e = getenv("DF_ATTN_DBG");  // profiling only: 1 = FMA instead of ex2, 2 = no softmax (wrong results)
      return e ? atoi(e) : 0;
    }();
    if (dbg == 1) return launch_attn2<DH, false, 1>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
    if (dbg == 2) return launch_attn2<DH, false, 2>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
    if (dbg == 3) return launch_attn2<DH, false, 3>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
    if (dbg == 4) return launch_attn2<DH, false, 4>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
    if (dbg == 5) return launch_attn2<DH, false, 5>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
    if (dbg == 6) return launch_attn2<DH, false, 6>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
    return poly ? launch_attn2<DH, true>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs)
                : launch_attn2<DH, false>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
  }
  using Cfg = AttnCfg<DH>;
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, DH, 128) || !make_tmap_3d(&tk, K, H, Nk, DH, 128) ||
      !make_tmap_3d(&tv, V, H, Nk, DH, 128))
    return cudaErrorInvalidValue;
  auto kern = attn_tc_kernel<DH>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((Nq + 127) / 128, H);
  kern<<<grid, 256, Cfg::SMEM, st>>>(tq, tk, tv, O, H, Nq, Nk, dh, scale * 1.4426950408889634f);
  return cudaGetLastError();
}

cudaError_t attn_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh, int dh_pad,
                    float scale, cudaStream_t st, int heads_per_sample, float* sk_ws, unsigned* sk_flag) {
  static const int impl_env = [] {
    // 1: one Q tile per CTA (round-1 kernel); 2: two Q tiles, one softmax thread per row;
    // 3: CTA pair (cta_group::2); 4: two Q tiles, two softmax threads per row;
    // 5: CTA pair, two softmax threads per row; 6 (default): 5 made persistent over work
    // items; 7: 6 with the stream-K split of ragged rounds (4-7: dh = 128; other head sizes
    // take 2)
    const char* e = getenv("DF_ATTN_IMPL");
    return e ? atoi(e) : 6;
  }();
  g_attn_impl = impl_env;
  const int hs = heads_per_sample > 0 ? heads_per_sample : H;
  if (Nq <= 0) return cudaSuccess;
  if (Nk <= 0 || dh > dh_pad || H % hs) return cudaErrorInvalidValue;
  if (dh_pad == 64) return launch_attn<64>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs, nullptr, nullptr);
  if (dh_pad == 128) return launch_attn<128>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs, sk_ws, sk_flag);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ fp32 SIMT attention
__global__ void attn_simt_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                 const float* __restrict__ V, float* __restrict__ O, int H, int Nq, int Nk, int dh,
                                 float scale, int hs) {
  const int warps = blockDim.x / 32;
  const int q = blockIdx.x * warps + threadIdx.x / 32;
  const int h = blockIdx.y;
  const int lane = threadIdx.x & 31;
  if (q >= Nq) return;
  const float* qr = Q + (size_t(h) * Nq + q) * dh;
  float qv[4], ov[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) qv[i] = (lane + 32 * i < dh) ? qr[lane + 32 * i] : 0.f;
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j < Nk; ++j) {
    const float* kr = K + (size_t(h) * Nk + j) * dh;
    const float* vr = V + (size_t(h) * Nk + j) * dh;
    float part = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < dh) part = fmaf(qv[i], kr[lane + 32 * i], part);
    float sj = warp_sum(part) * scale;
    float mn = fmaxf(m, sj);
    float corr = expf(m - mn), pj = expf(sj - mn);
    l = l * corr + pj;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < dh) ov[i] = ov[i] * corr + pj * vr[lane + 32 * i];
    m = mn;
  }
  const int hb = h / hs, hl = h - hb * hs;
  float* orow = O + (size_t(hb) * Nq + q) * hs * dh + size_t(hl) * dh;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (lane + 32 * i < dh) orow[lane + 32 * i] = ov[i] / l;
}

cudaError_t attn_simt(const float* Q, const float* K, const float* V, float* O, int H, int Nq, int Nk, int dh,
                      float scale, cudaStream_t st, int heads_per_sample) {
  const int hs = heads_per_sample > 0 ? heads_per_sample : H;
  if (Nq <= 0) return cudaSuccess;
  if (Nk <= 0 || dh > 128 || H % hs) return cudaErrorInvalidValue;
  dim3 grid((Nq + 3) / 4, H);
  attn_simt_kernel<<<grid, 128, 0, st>>>(Q, K, V, O, H, Nq, Nk, dh, scale, hs);
  return cudaGetLastError();
}

}  // namespace df
