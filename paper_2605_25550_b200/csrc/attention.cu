#include <cstring>
#include <atomic>
// Self- and cross-attention of the DiT block (PAPER.md P:L118
// "attention is O(T^2 D)"): O_h = softmax(Q_h K_h^T / sqrt(dh)) V_h, no mask, fp32
// online softmax.
//
// attn_pp (dh = 128, default): persistent CTA pairs (cta_group::2, M = 256 per pair), each
//   pair looping over work items of 512 query rows of one head; S, P and O live in TMEM (P is
//   written bf16 over S and fed back as the TS operand of PV); 16 softmax warps (two threads
//   per query row), one TMA warp, one converged MMA warp issuing from one elected lane; lazy
//   rescale (threshold 2^8); a quarter of the exponentials by a polynomial on the FMA pipe.
// attn_tc2 (dh = 64, and dh = 128 under DF_ATTN_IMPL=2 for A/B): two 128-query tiles per
//   CTA sharing every K/V block, one softmax thread per row.
// attn_simt: fp32 warp-per-row reference-grade kernel for the fp32 validation build.
// (Round 1's other variants -- one tile per CTA, the first CTA pair, the non-persistent
// two-thread kernels and the stream-K split of ragged rounds -- were measured slower or no
// faster, and removed.)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdlib>
#include "kernels.h"

namespace df {

bool make_tmap_3d(CUtensorMap* m, const void* base, uint64_t z, uint64_t rows, uint64_t cols, uint32_t box_rows);
bool make_tmap_3d_u8(CUtensorMap* m, const void* base, uint64_t z, uint64_t rows, uint64_t cols, uint32_t box_rows);
bool make_tmap_3d_u8s(CUtensorMap* m, const void* base, uint64_t z, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows);

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

template <int DH>
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
      // the affine part; the exponentials on MUFU
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
          p.x = ex2_approx(x.x);
          p.y = ex2_approx(x.y);
          lsum2 = fadd2(lsum2, p);
          pk[i] = pack_bf16x2(p.x, p.y);
        }
        // columns 16q .. 16q+15 hold keys 32q .. 32q+31 (S is already in registers)
        tmem_st16(ts + 16 * q, pk);
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

template <int DH>
static cudaError_t launch_attn2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, bf16* O, int H,
                                int Nq, int Nk, int dh, float scale, cudaStream_t st, int hs) {
  using Cfg = Attn2Cfg<DH>;
  auto kern = attn_tc2_kernel<DH>;
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
// p = 2^x for a pair (fp32), added to the row sum: the MUFU / polynomial split of softmax_exp2
template <int EXPM>
DF_DEV float2 softmax_exp2f(float2 x, int i, float2& lsum2) {
  float2 p;
  if ((EXPM == 1 && (i & 7) >= 5) || (EXPM == 2 && (i & 3) == 3) || (EXPM == 5 && (i & 1))) {
    p = exp2_poly2(x);
  } else {
    p.x = ex2_approx(x.x);
    p.y = ex2_approx(x.y);
  }
  lsum2 = fadd2(lsum2, p);
  return p;
}
// four fp32 -> e4m3 bytes (RNE, satfinite), a.x in the lowest byte
DF_DEV uint32_t pack_e4m3x4(float2 a, float2 b) {
  const uint32_t lo = __nv_cvt_float2_to_fp8x2(a, __NV_SATFINITE, __NV_E4M3);
  const uint32_t hi = __nv_cvt_float2_to_fp8x2(b, __NV_SATFINITE, __NV_E4M3);
  return lo | (hi << 16);
}

template <int EXPM>
DF_DEV uint32_t softmax_exp2(float2 x, int i, float2& lsum2) {
  if (EXPM == 4) {  // one MUFU ex2.f16x2 per pair (input rounded to f16: |err(x)| <= |x| 2^-11)
    uint32_t xh, ph;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(xh) : "f"(x.y), "f"(x.x));
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(ph) : "r"(xh));
    const float2 p = __half22float2(*reinterpret_cast<const __half2*>(&ph));
    lsum2 = fadd2(lsum2, p);
    return pack_bf16x2(p.x, p.y);
  }
  if (EXPM == 3) {
    const uint32_t xb = pack_bf16x2(x.x, x.y);
    uint32_t pb;
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(pb) : "r"(xb));
    lsum2 = fadd2(lsum2, make_float2(__uint_as_float(pb << 16), __uint_as_float(pb & 0xffff0000u)));
    return pb;
  }
  float2 p;
  if ((EXPM == 1 && (i & 7) >= 5) || (EXPM == 2 && (i & 3) == 3) || (EXPM == 5 && (i & 1))) {
    p = exp2_poly2(x);
  } else {
    p.x = ex2_approx(x.x);
    p.y = ex2_approx(x.y);
  }
  lsum2 = fadd2(lsum2, p);
  return pack_bf16x2(p.x, p.y);
}

// exponential split of the softmax (A/B, read once): DF_ATTN_EXPM = 2 (default: a quarter of the
// pairs by polynomial), 1 (3 of 8), 5 (half), 0 (all MUFU), 4 (MUFU ex2.f16x2), 3 (ex2.bf16x2)
static int attn_expm() {
  const char* e = getenv("DF_ATTN_EXPM");
  const int v = e ? atoi(e) : 2;
  return (v >= 0 && v <= 5) ? v : 2;
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

// ------------------------------------------------------------------ attn_pair: CTA-pair (cta_group::2)
// A cluster of two CTAs runs M = 256 MMAs: query tile t of the pair is 256 rows, 128 in each
// CTA's shared memory and TMEM. Each CTA stages HALF of every K/V block (K: 64 of the 128
// keys, all of dh; V: all 128 keys, 64 of the 128 dh columns), so per SM the shared-memory
// operand reads of QK^T and PV and the TMA writes halve against attn_tc2 (whose SS-mode
// M=128 QK^T alone saturates the 128 B/clk shared-memory port). The leader CTA's MMA thread
// issues for both; ring barriers live on the leader (count 2: its expect_tx + the peer's
// arrive), MMA completions are multicast to both CTAs. Softmax is per CTA over its own 128
// rows, exactly as in attn_tc2 (P written into TMEM, consumed as the A operand of PV).
// QF8 (FP8 modes): 1 (R32) -- Q and K in e4m3: a 128-dh row is one 128-byte SW128 row, so a Q
// tile is one atom column (16 KB) and a half K block 8 KB; QK^T runs as four kind::f8f6f4 MMAs
// (K = 32 bytes each) instead of eight kind::f16 ones.  2 (R33) -- also PV on e4m3: P written
// as e4m3 into TMEM (four keys per 32-bit column, the A operand of a kind::f8f6f4 TS MMA per
// 32-key quarter) and V^T e4m3 [H][dh][keys] (K-major like K: a half V block is 64 dh rows x
// 128 keys = 8 KB); the per-tensor V scale is applied in the O normalisation.
template <int QF8>
struct AttnPairCfgT {
  static constexpr int DH = 128;
  static constexpr int ATOM = 64 * 128;              // SW128 atom of 64 rows (8 KB)
  static constexpr int Q_BYTES = QF8 ? 128 * 128 : 2 * 128 * 128;  // one 128-row Q tile
  static constexpr int K_BYTES = QF8 ? 64 * 128 : 64 * 128 * 2;    // half K block: 64 keys x 128 dh
  static constexpr int V_BYTES = QF8 == 2 ? 64 * 128 : 128 * 64 * 2;  // half V block
  static constexpr int KST = 4;
  static constexpr int VST = 4;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * V_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t O_COL = 256;
};
using AttnPairCfg = AttnPairCfgT<0>;

// ------------------------------------------------------------------ attn_pair3: CTA pair + 2 threads per row
// attn_pair's tensor-core schedule (M = 256 over a CTA pair: per SM the QK^T shared-memory
// operand reads drop from 8 KB to 6 KB per 64-clock K step and the PV B reads halve, so the
// 128 B/clk shared-memory port stops pacing the MMAs) with attn_tc3's softmax (two threads
// per query row).  The row maxima are exchanged exactly (fp32) through shared memory.
// ------------------------------------------------------------------ attn_pp: persistent CTA pair
// attn_pair3's MMA schedule and softmax, but each CTA pair loops over work items (512 query
// rows of one head; items head-major so consecutive items reuse K/V in L2) instead of one
// item per launch slot: the TMEM allocation and barrier set-up happen once, the next item's
// Q is loaded while the current item's last blocks run (q_empty is committed after its
// last QK), and the next item's QKs start while the softmax warps normalise and store the
// previous O (the first PV of an item waits for o_free, the epilogue's release of O_t).
// Short-key launches (cross-attention, 4 key blocks per item) are dominated by exactly
// these per-item costs.  All barrier phases run on counters that continue across items.
template <int EXPM, int QF8 = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ATTN3_THREADS, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                   int dh_real, float scale_log2, int Hs, const float* __restrict__ vscale) {
  using Cfg = AttnPairCfgT<QF8>;
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
          for (int a = 0; a < (QF8 ? 1 : 2); ++a)
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
            for (int a = 0; a < (QF8 ? 1 : 2); ++a)
              tma_load_3d_pair(sK + st * Cfg::K_BYTES + a * Cfg::ATOM, &tmK, &k_full[st], a * 64,
                               kb * 128 + int(rank) * 64, h);
            ++jk;
          } else {
            const int st = jv % Cfg::VST;
            mbar_wait(&v_empty[st], ((jv / Cfg::VST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&v_full[st], 2 * Cfg::V_BYTES);
            else mbar_arrive_cluster(&v_full[st], 0);
            const int vb = jv - (v_end - nkb);
            if (QF8 == 2) tma_load_3d_pair(sV + st * Cfg::V_BYTES, &tmV, &v_full[st], vb * 128, int(rank) * 64, h);
            else tma_load_3d_pair(sV + st * Cfg::V_BYTES, &tmV, &v_full[st], int(rank) * 64, vb * 128, h);
            ++jv;
          }
        }
      }
    }
  } else if (warp == 17) {
    if (leader) {  // whole warp runs the schedule; one elected lane issues each MMA batch
      constexpr uint32_t idesc_qk = QF8 ? idesc_e4m3(256, 128) : idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = QF8 == 2 ? idesc_e4m3(256, DH) : idesc_bf16(256, DH, false, true);
      const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = QF8 == 2 ? sdesc_sw128(smem_u32(sV), 16, 1024) : sdesc_sw128(smem_u32(sV), Cfg::V_BYTES, 1024);
      auto issue_qk = [&](int t, int jg) {
        const uint64_t a0 = dq + uint64_t((t * Cfg::Q_BYTES) >> 4);
        const uint64_t b0 = dk + uint64_t(((jg % Cfg::KST) * Cfg::K_BYTES) >> 4);
        if (elect_one()) {
          if constexpr (QF8) {
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x 32 bytes of each 128-byte e4m3 row
              tc_mma_f8_pair(tmem + t * 128, a0 + uint64_t((k * 32) >> 4), b0 + uint64_t((k * 32) >> 4), idesc_qk,
                             k > 0);
          } else {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            tc_mma_bf16_pair(tmem + t * 128, a0 + uint64_t(((k >> 2) * 2 * Cfg::ATOM + (k & 3) * 32) >> 4),
                             b0 + uint64_t(((k >> 2) * Cfg::ATOM + (k & 3) * 32) >> 4), idesc_qk, k > 0);
          }
          tc_commit_pair(&s_full[t], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int jg, int u, bool first) {
        const uint64_t b0 = dv + uint64_t(((jg % Cfg::VST) * Cfg::V_BYTES) >> 4);
        if (elect_one()) {
          if constexpr (QF8 == 2) {  // keys 32u .. 32u + 31: P columns 8u .., V^T bytes 32u ..
            tc_mma_f8_ts_pair(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + u * 8, b0 + uint64_t((u * 32) >> 4),
                              idesc_pv, !first);
          } else {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int k = 2 * u + kk;
            tc_mma_bf16_ts_pair(tmem + Cfg::O_COL + t * DH, tmem + t * 128 + k * 8, b0 + uint64_t((k * 2048) >> 4),
                                idesc_pv, !(first && kk == 0));
          }
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
        if constexpr (QF8 == 2) {  // P as e4m3 (p <= 2^8 by the lazy rescale): 4 keys per column
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 a = softmax_exp2f<EXPM>(ffma2(make_float2(s[4 * i], s[4 * i + 1]), sc2, nm2), 2 * i, lsum2);
            const float2 b = softmax_exp2f<EXPM>(ffma2(make_float2(s[4 * i + 2], s[4 * i + 3]), sc2, nm2), 2 * i + 1, lsum2);
            pk[i] = pack_e4m3x4(a, b);
          }
          tmem_st8(ts + 16 * hc, pk);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 a = softmax_exp2f<EXPM>(ffma2(make_float2(s[32 + 4 * i], s[32 + 4 * i + 1]), sc2, nm2), 2 * i, lsum2);
            const float2 b = softmax_exp2f<EXPM>(ffma2(make_float2(s[32 + 4 * i + 2], s[32 + 4 * i + 3]), sc2, nm2), 2 * i + 1, lsum2);
            pk[i] = pack_e4m3x4(a, b);
          }
        } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2), i, lsum2);
        tmem_st16(ts + 32 * hc, pk);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = softmax_exp2<EXPM>(ffma2(make_float2(s[32 + 2 * i], s[32 + 2 * i + 1]), sc2, nm2), i, lsum2);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&p_q[t * 4 + 2 * hc], 0);
        if constexpr (QF8 == 2) tmem_st8(ts + 16 * hc + 8, pk);
        else tmem_st16(ts + 32 * hc + 16, pk);
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
      const float inv = (QF8 == 2 ? __ldg(vscale) : 1.0f) / (l + lds_f32(lred_oth));
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

template <int EXPM, int QF8 = 0>
static cudaError_t launch_attn_pp(const void* Q, const void* K, const void* V, bf16* O, int H, int Nq, int Nk, int dh,
                                  float scale, cudaStream_t st, int hs, const float* vscale = nullptr, int ldv = 0) {
  using Cfg = AttnPairCfgT<QF8>;
  constexpr int SMEM = Cfg::OFF_BAR + 512 + 4096 + 1024;
  static_assert(SMEM <= 232448, "attn_pp shared memory");
  CUtensorMap tq, tk, tv;
  const bool ok = QF8 ? (make_tmap_3d_u8(&tq, Q, H, Nq, 128, 128) && make_tmap_3d_u8(&tk, K, H, Nk, 128, 64))
                      : (make_tmap_3d(&tq, Q, H, Nq, 128, 128) && make_tmap_3d(&tk, K, H, Nk, 128, 64));
  // QF8 == 2: V^T e4m3 [H][128 dh][ldv] bytes (keys contiguous, row stride ldv >= Nk, % 16 == 0)
  const bool okv = QF8 == 2 ? make_tmap_3d_u8s(&tv, V, H, 128, Nk, ldv, 64) : make_tmap_3d(&tv, V, H, Nk, 128, 128);
  if (!ok || !okv) return cudaErrorInvalidValue;
  auto kern = attn_pp_kernel<EXPM, QF8>;
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
                  (void*)&Nq, (void*)&Nk, (void*)&dh, (void*)&sl2, (void*)&hs, (void*)&vscale};
  return launch_ex((const void*)kern, grid, dim3(ATTN3_THREADS), SMEM, st, args);
}

// ------------------------------------------------------------------ attn_sk: short keys (cross-attention)
// For 257 <= N_kv <= 512 (the text cross-attention of every config, N_kv = L_txt = 512; SURVEY
// §8(a) a8), where attn_pp's items are only four dependent QK^T -> softmax -> PV links long and
// the two query tiles of an item reach their epilogues together (ncu: 38.5 % tensor-active on
// the image shape).  Structure:
//  * K and V of a head stay resident in shared memory (per CTA of the pair: 4 x 64 keys x dh
//    of K, 4 x 128 keys x 64 dh of V = 128 KB), loaded once per head segment; a block's
//    buffer is refilled for the next head as soon as the old head's last QK / PV that reads it
//    completes, so a head change costs no pipeline drain;
//  * each CTA pair walks a contiguous, balanced range of (head, 256-query tile) units (one
//    query tile in flight, Q double-buffered);
//  * TMEM: S0, S1 (128 columns each: the S ring, depth 2) and O0, O1 (the accumulator of tile
//    n lives in O[n & 1]), so QK^T of block b + 2 is issued right after PV of block b and
//    tile n + 1 accumulates while tile n is normalised and stored;
//  * 16 softmax warps, four threads per query row (each owns 32 key columns of every block;
//    the row max is exchanged through shared memory), so one block's softmax is a short
//    chain; PV of key quarter u starts as soon as the four warps owning it published P;
//  * 4 epilogue warps normalise and store O, off the softmax warps' critical path.
// Lazy rescale (threshold 2^8) and the polynomial quarter of the exponentials as in attn_pp.
constexpr int ATTN_SK_THREADS = 22 * 32;
struct AttnSkCfg {
  static constexpr int DH = 128;
  static constexpr int ATOM = 64 * 128;
  static constexpr int Q_BYTES = 2 * 128 * 128;      // one CTA's 128 query rows (2 dh atoms)
  static constexpr int K_BYTES = 64 * 128 * 2;       // half K block: 64 keys x 128 dh
  static constexpr int V_BYTES = 128 * 64 * 2;       // half V block: 128 keys x 64 dh
  static constexpr int NKB = 4;                      // resident key blocks (N_kv <= 512)
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + NKB * K_BYTES;
  static constexpr int OFF_Q = OFF_V + NKB * V_BYTES;
  static constexpr int OFF_BAR = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_RED = OFF_BAR + 512;       // [2 block parity][4 col group][128 rows] row max
  static constexpr int OFF_LRED = OFF_RED + 4096;     // [2 tile parity][4 col group][128 rows] row sum
  static constexpr int SMEM = OFF_LRED + 4096 + 1024;
  static constexpr uint32_t S_COL = 0;
};

// SD = depth of the S ring in TMEM (S0, S1 + O double-buffered per tile).  A depth-3 ring with
// a single O (QK^T one block further ahead, the tile's epilogue gating the next tile's first PV)
// was measured 13-20 % slower and removed.
template <int EXPM, int SD = 2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ATTN_SK_THREADS, 1)
    attn_sk_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ O, int H, int Nq, int Nk,
                   float scale_log2, int Hs) {
  using Cfg = AttnSkCfg;
  constexpr int DH = Cfg::DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint8_t* sQ = smem + Cfg::OFF_Q;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bars + 0;        // [2]  leader (both CTAs' bytes)
  uint64_t* q_empty = bars + 2;       // [2]  both (commit after the tile's last QK)
  uint64_t* k_full = bars + 4;        // [4]  leader
  uint64_t* k_empty = bars + 8;       // [4]  both (commit after the head segment's last QK of the block)
  uint64_t* v_full = bars + 12;       // [4]  leader
  uint64_t* v_empty = bars + 16;      // [4]  both
  uint64_t* s_full = bars + 20;       // [SD] both
  uint64_t* pv_done = bars + 23;      // [2]  both (per PV block, read only by a rescale)
  uint64_t* o_done = bars + 25;       // [NO] both (tile's last PV)
  uint64_t* o_free = bars + 27;       // [NO] leader: 4 epilogue warps x 2 CTAs
  uint64_t* l_full = bars + 29;       // [2]  local: 16 softmax warps
  uint64_t* p_q = bars + 31;          // [SD S slot][4 quarter] leader: 4 warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 43);
  constexpr int NO = SD == 2 ? 2 : 1;             // O buffers
  constexpr uint32_t O_COL = uint32_t(SD) * 128;  // O after the S ring
  float* red = reinterpret_cast<float*>(smem + Cfg::OFF_RED);
  float* lred = reinterpret_cast<float*>(smem + Cfg::OFF_LRED);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nkb = (Nk + 127) / 128;   // 3 or 4 (host guarantees)
  const int ntq = (Nq + 255) / 256;   // query tiles per head
  const long long U = (long long)ntq * H;
  const int cid = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int u0 = int(U * cid / npairs), u1 = int(U * (cid + 1) / npairs);
  const int T = u1 - u0;              // this pair's tiles
  const int h0 = u0 / ntq;
  auto head_of = [&](int n) { return (u0 + n) / ntq; };
  auto seg_last = [&](int n) { return n == T - 1 || head_of(n) != head_of(n + 1); };

  if (warp == 20 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 2);
      mbar_init(&q_empty[s], 1);
      mbar_init(&pv_done[s], 1);
      mbar_init(&l_full[s], 16);
    }
    for (int s = 0; s < SD; ++s) mbar_init(&s_full[s], 1);
    for (int s = 0; s < NO; ++s) {
      mbar_init(&o_done[s], 1);
      mbar_init(&o_free[s], 8);
    }
    for (int j = 0; j < Cfg::NKB; ++j) {
      mbar_init(&k_full[j], 2);
      mbar_init(&k_empty[j], 1);
      mbar_init(&v_full[j], 2);
      mbar_init(&v_empty[j], 1);
    }
    for (int i = 0; i < 4 * SD; ++i) mbar_init(&p_q[i], 8);
    fence_mbar_init();
  }
  if (warp == 21) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 20) {
    if (lane == 0) {
      auto load_q = [&](int n) {
        const int u = u0 + n, h = u / ntq, qt = u - h * ntq;
        if (n >= 2) mbar_wait(&q_empty[n & 1], ((n - 2) >> 1) & 1);
        if (leader) mbar_arrive_expect_tx(&q_full[n & 1], 2 * Cfg::Q_BYTES);
        else mbar_arrive_cluster(&q_full[n & 1], 0);
#pragma unroll
        for (int a = 0; a < 2; ++a)
          tma_load_3d_pair(sQ + (n & 1) * Cfg::Q_BYTES + a * 2 * Cfg::ATOM, &tmQ, &q_full[n & 1], a * 64,
                           qt * 256 + int(rank) * 128, h);
      };
      int nq = 0;  // next tile whose Q is to be loaded
      for (int n = 0; n < T; ++n) {
        const int h = head_of(n);
        if (n > 0 && h == head_of(n - 1)) continue;
        const int s = h - h0;  // head segment of this pair
        while (nq <= n + 1 && nq < T) load_q(nq++);  // Q of this tile (and the next) first
        for (int j = 0; j < nkb; ++j) {
          if (s > 0) mbar_wait(&k_empty[j], (s - 1) & 1);
          if (leader) mbar_arrive_expect_tx(&k_full[j], 2 * Cfg::K_BYTES);
          else mbar_arrive_cluster(&k_full[j], 0);
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_3d_pair(sK + j * Cfg::K_BYTES + a * Cfg::ATOM, &tmK, &k_full[j], a * 64,
                             j * 128 + int(rank) * 64, h);
          if (s > 0) mbar_wait(&v_empty[j], (s - 1) & 1);
          if (leader) mbar_arrive_expect_tx(&v_full[j], 2 * Cfg::V_BYTES);
          else mbar_arrive_cluster(&v_full[j], 0);
          tma_load_3d_pair(sV + j * Cfg::V_BYTES, &tmV, &v_full[j], int(rank) * 64, j * 128, h);
        }
        // Q of the tiles up to the next head change
        int n_end = n + 1;
        while (n_end < T && head_of(n_end) == h) ++n_end;
        while (nq < n_end + 1 && nq < T) load_q(nq++);
      }
      while (nq < T) load_q(nq++);
    }
  } else if (warp == 21) {
    if (leader) {
      constexpr uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(256, DH, false, true);
      const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(sV), Cfg::V_BYTES, 1024);
      const int nb = T * nkb;
      auto issue_qk = [&](int b) {
        const int n = b / nkb, j = b - n * nkb;
        if (j == 0) mbar_wait(&q_full[n & 1], (n >> 1) & 1);
        mbar_wait(&k_full[j], (head_of(n) - h0) & 1);
        tc_fence_after();
        const uint64_t a0 = dq + uint64_t(((n & 1) * Cfg::Q_BYTES) >> 4);
        const uint64_t b0 = dk + uint64_t((j * Cfg::K_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            tc_mma_bf16_pair(tmem + Cfg::S_COL + (b % SD) * 128,
                             a0 + uint64_t(((k >> 2) * 2 * Cfg::ATOM + (k & 3) * 32) >> 4),
                             b0 + uint64_t(((k >> 2) * Cfg::ATOM + (k & 3) * 32) >> 4), idesc_qk, k > 0);
          tc_commit_pair(&s_full[b % SD], 0x3);
          if (j == nkb - 1) tc_commit_pair(&q_empty[n & 1], 0x3);
          if (seg_last(n)) tc_commit_pair(&k_empty[j], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int b) {
        const int n = b / nkb, j = b - n * nkb;
        if (j == 0 && n >= NO) mbar_wait(&o_free[n % NO], ((n - NO) / NO) & 1);  // O[n % NO] read out
        mbar_wait(&v_full[j], (head_of(n) - h0) & 1);
        const uint64_t b0 = dv + uint64_t((j * Cfg::V_BYTES) >> 4);
        const uint32_t d = tmem + O_COL + (n % NO) * DH;
        const uint32_t pa = tmem + Cfg::S_COL + (b % SD) * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          mbar_wait(&p_q[(b % SD) * 4 + u], (b / SD) & 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const int k = 2 * u + kk;
              tc_mma_bf16_ts_pair(d, pa + k * 8, b0 + uint64_t((k * 2048) >> 4), idesc_pv, (j > 0 || k > 0));
            }
          }
          __syncwarp();
        }
        if (elect_one()) {
          tc_commit_pair(&pv_done[b & 1], 0x3);
          if (j == nkb - 1) tc_commit_pair(&o_done[n % NO], 0x3);
          if (seg_last(n)) tc_commit_pair(&v_empty[j], 0x3);
        }
        __syncwarp();
      };
      for (int b = 0; b < SD && b < nb; ++b) issue_qk(b);
      for (int b = 0; b < nb; ++b) {
        issue_pv(b);
        if (b + SD < nb) issue_qk(b + SD);  // S[b % SD] is free once PV(b) has read P(b) (in-order pipe)
      }
    }
  } else if (warp >= 16) {
    // epilogue: O[n & 1] / l -> bf16 rows of head h
    const int ew = warp & 3;
    const int r = ew * 32 + lane;
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    for (int n = 0; n < T; ++n) {
      mbar_wait(&l_full[n & 1], (n >> 1) & 1);
      mbar_wait(&o_done[n % NO], (n / NO) & 1);
      tc_fence_after();
      const float* lr = lred + (n & 1) * 512 + r;
      const float inv = 1.0f / ((lr[0] + lr[128]) + (lr[256] + lr[384]));
      const int u = u0 + n, h = u / ntq, qt = u - h * ntq;
      const int q = qt * 256 + int(rank) * 128 + r;
      const int hb = h / Hs, hl = h - hb * Hs;
      bf16* orow = O + (size_t(hb) * Nq + q) * Hs * DH + size_t(hl) * DH;
      const uint32_t to = tmem + lane_off + O_COL + (n % NO) * DH;
#pragma unroll 1
      for (int c = 0; c < DH; c += 32) {
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
      if (lane == 0) mbar_arrive_cluster(&o_free[n % NO], 0);
    }
  } else {
    // softmax: warp (cg, ew) owns key columns [32 cg, 32 cg + 32) of rows ew*32 .. ew*32+31
    const int ew = warp & 3, cg = warp >> 2;
    const int r = ew * 32 + lane;
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    int b = 0;
    for (int n = 0; n < T; ++n) {
      float m_used = -INFINITY, l = 0.f;
      const uint32_t to = tmem + lane_off + O_COL + (n % NO) * DH + 32 * cg;
      for (int j = 0; j < nkb; ++j, ++b) {
        const uint32_t ts = tmem + lane_off + Cfg::S_COL + (b % SD) * 128;
        mbar_wait(&s_full[b % SD], (b / SD) & 1);
        tc_fence_after();
        float s[32];
        tmem_ld32(ts + 32 * cg, s);
        tc_wait_ld();
        const int valid = Nk - j * 128 - 32 * cg;
        if (valid < 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i >= valid) s[i] = -INFINITY;
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
#pragma unroll
          for (int v = 0; v < 4; ++v) m4[v] = fmaxf(m4[v], fmaxf(s[i + 2 * v], s[i + 2 * v + 1]));
        }
        float* rb = red + (b & 1) * 512 + r;
        rb[cg * 128] = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
        named_bar_sync(1 + ew, 128);
        const float mx = fmaxf(fmaxf(rb[0], rb[128]), fmaxf(rb[256], rb[384]));
        const bool need = mx > m_used + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_used;
          if (j > 0) {
            // PV(b - 1) must have landed in O before it is rescaled
            mbar_wait(&pv_done[(b - 1) & 1], ((b - 1) >> 1) & 1);
            tc_fence_after();
            const float alpha = exp2f(m_used - m_new);
            l *= alpha;
            float o[32];
            tmem_ld32(to, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(to, o);
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
        tmem_st16(ts + 16 * cg, pk);  // P: keys 32cg.. as bf16 pairs in columns 16cg..16cg+15
        l += lsum2.x + lsum2.y;
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&p_q[(b % SD) * 4 + cg], 0);
      }
      lred[(n & 1) * 512 + cg * 128 + r] = l;
      __syncwarp();
      if (lane == 0) mbar_arrive(&l_full[n & 1]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 21) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

static cudaError_t launch_attn_sk(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk,
                                  float scale, cudaStream_t st, int hs) {
  using Cfg = AttnSkCfg;
  static_assert(Cfg::SMEM <= 232448, "attn_sk shared memory");
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, 128, 128) || !make_tmap_3d(&tk, K, H, Nk, 128, 64) ||
      !make_tmap_3d(&tv, V, H, Nk, 128, 128))
    return cudaErrorInvalidValue;
  auto kern = attn_sk_kernel<2>;
  static int max_pairs = 0;
  if (!max_pairs) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    max_pairs = num_sms() / 2;
  }
  const long long units = (long long)((Nq + 255) / 256) * H;
  const int pairs = units < max_pairs ? int(units) : max_pairs;
  dim3 grid(2 * pairs);
  float sl2 = scale * 1.4426950408889634f;
  void* args[] = {(void*)&tq, (void*)&tk, (void*)&tv, (void*)&O, (void*)&H, (void*)&Nq, (void*)&Nk, (void*)&sl2, (void*)&hs};
  return launch_ex((const void*)kern, grid, dim3(ATTN_SK_THREADS), Cfg::SMEM, st, args);
}

DF_DEV void st_release_u32_attn(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
DF_DEV unsigned ld_acquire_u32_attn(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int DH>
static cudaError_t launch_attn(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh,
                               float scale, cudaStream_t st, int hs) {
  if constexpr (DH == 128) {
    // N_kv in [257, 512] (cross-attention) with long per-pair runs (>= 8 query tiles per CTA
    // pair: the video shape, 69): the K/V-resident short-key kernel, 4-5 % faster in the step;
    // with few tiles per pair (image, 5.2) attn_pp's items are 3 % faster.
    // DF_ATTN_SK=0 / 2 forces attn_pp / attn_sk for A/B.
    static const int sk = [] {
      const char* e = getenv("DF_ATTN_SK");
      return e ? atoi(e) : 1;
    }();
    const long long sk_tiles = (long long)((Nq + 255) / 256) * H;
    if (g_attn_impl != 2 && sk && dh == 128 && Nk > 256 && Nk <= 512 &&
        (sk == 2 || sk_tiles >= 8LL * (num_sms() / 2)))
      return launch_attn_sk(Q, K, V, O, H, Nq, Nk, scale, st, hs);
    if (g_attn_impl != 2) {
      static const int expm = attn_expm();
      switch (expm) {
        case 0: return launch_attn_pp<0>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 1: return launch_attn_pp<1>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 3: return launch_attn_pp<3>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 4: return launch_attn_pp<4>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        case 5: return launch_attn_pp<5>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
        default: return launch_attn_pp<2>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
      }
    }
  }
  CUtensorMap tq, tk, tv;
  if (!make_tmap_3d(&tq, Q, H, Nq, DH, 128) || !make_tmap_3d(&tk, K, H, Nk, DH, 128) ||
      !make_tmap_3d(&tv, V, H, Nk, DH, 128))
    return cudaErrorInvalidValue;
  return launch_attn2<DH>(tq, tk, tv, O, H, Nq, Nk, dh, scale, st, hs);
}

cudaError_t attn_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh, int dh_pad,
                    float scale, cudaStream_t st, int heads_per_sample) {
  static const int impl_env = [] {
    // dh = 128: attn_pp (default; persistent CTA pairs, a quarter of the exponentials on the
    // FMA pipe) or, with DF_ATTN_IMPL=2, attn_tc2 (two query tiles per CTA) for A/B; dh = 64:
    // attn_tc2.  The round-1 variants measured slower were removed.
    const char* e = getenv("DF_ATTN_IMPL");
    return e ? atoi(e) : 6;
  }();
  g_attn_impl = impl_env;
  const int hs = heads_per_sample > 0 ? heads_per_sample : H;
  if (Nq <= 0) return cudaSuccess;
  if (Nk <= 0 || dh > dh_pad || H % hs) return cudaErrorInvalidValue;
  if (dh_pad == 64) return launch_attn<64>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
  if (dh_pad == 128) return launch_attn<128>(Q, K, V, O, H, Nq, Nk, dh, scale, st, hs);
  return cudaErrorInvalidValue;
}

// FP8 modes (R32): self-attention with e4m3 Q and K ([H][N][128] bytes, head-major like the
// bf16 path) and bf16 V; `scale` already carries the two dequantisation scales.  dh = 128.
cudaError_t attn_tc_qf8(const uint8_t* Q8, const uint8_t* K8, const bf16* V, bf16* O, int H, int Nq, int Nk,
                        float scale, cudaStream_t st, int heads_per_sample) {
  const int hs = heads_per_sample > 0 ? heads_per_sample : H;
  if (Nq <= 0) return cudaSuccess;
  if (Nk <= 0 || H % hs) return cudaErrorInvalidValue;
  return launch_attn_pp<2, 1>(Q8, K8, V, O, H, Nq, Nk, 128, scale, st, hs);
}

// R33: QK^T and PV on e4m3 -- Q8, K8 as above, V8T = e4m3 V^T [H][128][ldv] (keys contiguous)
// with the per-tensor dequantisation scale *vscale (device).
cudaError_t attn_tc_f8(const uint8_t* Q8, const uint8_t* K8, const uint8_t* V8T, int ldv, const float* vscale, bf16* O,
                       int H, int Nq, int Nk, float scale, cudaStream_t st, int heads_per_sample) {
  const int hs = heads_per_sample > 0 ? heads_per_sample : H;
  if (Nq <= 0) return cudaSuccess;
  if (Nk <= 0 || H % hs || ldv < Nk || ldv % 16 || !vscale) return cudaErrorInvalidValue;
  return launch_attn_pp<2, 2>(Q8, K8, V8T, O, H, Nq, Nk, 128, scale, st, hs, vscale, ldv);
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
