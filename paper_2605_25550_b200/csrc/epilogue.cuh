// GEMM epilogues of the DiT step.  One thread owns one output
// row m and a chunk of CW consecutive columns [n0, n0+CW) of the raw fp32
// accumulator (acc = A·W^T, bias NOT yet added).  The tcgen05 GEMM calls these on
// registers loaded from TMEM (row-per-thread 32x32b layout); the fp32 validation
// build calls the same functions from a row kernel after a SIMT GEMM.
#pragma once
#include "common.cuh"

namespace df {

enum EpiKind : int {
  EPI_STORE = 0,   // out[m, n] = act(acc + b[n])                   (bf16 or f32)
  EPI_HEADS = 1,   // sections of width d: per-head RMSNorm*gain (+RoPE), head-major out
  EPI_GRES = 2,    // resid[m, n] += gate[n] * (acc + b[n])        (fp32 RMW, gate may be null)
  EPI_SWIGLU = 3,  // interleaved (16 W1 | 16 W3) columns -> out[m, j] = SiLU(a1+b1)*(a3+b3)
  EPI_EULER = 4,   // head: v = acc + b; x_lat[unpatchify(m, n)] += dsig * v (v_out optional)
};
enum ActKind : int { ACT_NONE = 0, ACT_GELU = 1, ACT_SILU = 2 };

struct Epi {
  int kind;
  int M, N;                // GEMM output rows / cols
  const bf16* bias;        // [N] (interleaved for SWIGLU) or null
  // STORE
  int act;
  void* out;
  int ldo;
  // HEADS
  int d, heads, dh, dh_pad, nsec;
  void* sec_out[3];        // head-major [heads][M][dh_pad]
  const bf16* sec_gain[3]; // [d] gains (null -> no norm)
  int sec_rope[3];
  const float2* rope_tab;  // [(Fp*Df2) + (Hp*Dh2) + (Wp*Dw2)] (cos, sin)
  int Fp, Hp, Wp, Df2, Dh2, Dw2;
  float eps;
  // GRES
  float* resid;
  int ldr;
  const float* gate;       // [N] fp32 or null
  // EULER
  float* x_lat;
  float* v_out;
  float dsig;
  int C, pt, ph, pw, Hl, Wl, Fl;  // latent geometry
  int m_base;              // EULER: token index of GEMM row 0 (the head run over one T->D chunk's tokens)
  // batch of samples stacked along M (classifier-free guidance: conditional, negative):
  // rows per sample; HEADS writes sample-major [b][heads][Mper][dh_pad]; EULER with
  // v_batch stores v of sample b at v_batch[b * latent_elems + idx] instead of updating x.
  int Mper;
  float* v_batch;
  // stream-K (CTA-pair GEMM only; null = data-parallel tiles): partial-tile workspace
  // [pairs][2 CTAs][256 cols][128 rows] fp32, one ready flag per (pair, CTA) holding the
  // epoch of the launch that wrote it
  float* sk_ws;
  unsigned* sk_flag;
  unsigned sk_epoch;
  int sk_force;  // host: take stream-K whenever the tile count allows it (tests)
  // FP8 (e4m3) operands (NEXT-4): device pointers to the per-tensor dequantisation scales of
  // A and B; the accumulator is multiplied by *f8_scale[0] * *f8_scale[1] before the epilogue.
  // f8_row (optional): per-row scales of A [M] replace *f8_scale[0] (R29: activations
  // quantised per token row by the producing RMSNorm)
  const float* f8_scale[2];
  const float* f8_row;
};

DF_DEV float bias_at(const Epi& e, int n) { return e.bias ? bf2f(e.bias[n]) : 0.0f; }

// 16-byte vector stores of CW consecutive values (caller guarantees alignment).
template <int CW>
DF_DEV void store_vec(bf16* o, const float* v) {
#pragma unroll
  for (int i = 0; i < CW; i += 8) {
    uint4 u;
    u.x = pack_bf16x2(v[i], v[i + 1]);
    u.y = pack_bf16x2(v[i + 2], v[i + 3]);
    u.z = pack_bf16x2(v[i + 4], v[i + 5]);
    u.w = pack_bf16x2(v[i + 6], v[i + 7]);
    *reinterpret_cast<uint4*>(o + i) = u;
  }
}
template <int CW>
DF_DEV void store_vec(float* o, const float* v) {
#pragma unroll
  for (int i = 0; i < CW; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}


// rope_cs with the token's grid coordinates decoded once: per-axis table rows, indexed
// by the pair number within the head (the f rows cover pairs [0, Df2), h [Df2, Df2+Dh2),
// w the rest; the h and w bases are pre-offset so the pair index is used unchanged)
struct RopeRow {
  const float2* f;
  const float2* h;
  const float2* w;
};
DF_DEV RopeRow rope_row(const Epi& e, int m) {
  const int hw = e.Hp * e.Wp;
  const int f = m / hw, rem = m - f * hw;
  const int hh = rem / e.Wp, ww = rem - hh * e.Wp;
  RopeRow r;
  r.f = e.rope_tab + f * e.Df2;
  r.h = e.rope_tab + e.Fp * e.Df2 + hh * e.Dh2 - e.Df2;
  r.w = e.rope_tab + e.Fp * e.Df2 + e.Hp * e.Dh2 + ww * e.Dw2 - e.Df2 - e.Dh2;
  return r;
}
DF_DEV float2 rope_at(const Epi& e, const RopeRow& r, int pair) {
  return pair < e.Df2 ? r.f[pair] : (pair < e.Df2 + e.Dh2 ? r.h[pair] : r.w[pair]);
}

// EPI_HEADS math on one head: bias, per-head RMSNorm * gain (if the section has a gain),
// RoPE (if the section rotates); m is the token within its sample (RoPE position).
template <int CW>
DF_DEV void heads_math(const Epi& e, int m, int n0, int sec, int hd, float* v) {
#pragma unroll
  for (int i = 0; i < CW; ++i) v[i] += bias_at(e, n0 + i);
  const bf16* g = e.sec_gain[sec];
  if (g) {
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < CW; ++i) ss += v[i] * v[i];
    float inv = rsqrtf(ss / float(CW) + e.eps);
    const bf16* gg = g + hd * e.dh;
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] = v[i] * inv * bf2f(gg[i]);
  }
  if (e.sec_rope[sec]) {
    const RopeRow rr = rope_row(e, m);
#pragma unroll
    for (int p = 0; p < CW / 2; ++p) {
      float2 cs = rope_at(e, rr, p);
      float a = v[2 * p], b = v[2 * p + 1];
      v[2 * p] = a * cs.x - b * cs.y;
      v[2 * p + 1] = a * cs.y + b * cs.x;
    }
  }
}

// heads_math with the head's bias and gain already staged as fp32 (shared memory); same
// arithmetic in the same order.
template <int CW>
DF_DEV void heads_math_s(const Epi& e, int m, int sec, const float* sb, const float* sg, float* v) {
#pragma unroll
  for (int i = 0; i < CW; i += 4) {
    const float4 b4 = *reinterpret_cast<const float4*>(sb + i);
    v[i] += b4.x, v[i + 1] += b4.y, v[i + 2] += b4.z, v[i + 3] += b4.w;
  }
  if (sg) {
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < CW; ++i) ss += v[i] * v[i];
    float inv = rsqrtf(ss / float(CW) + e.eps);
#pragma unroll
    for (int i = 0; i < CW; i += 4) {
      const float4 g4 = *reinterpret_cast<const float4*>(sg + i);
      v[i] = v[i] * inv * g4.x, v[i + 1] = v[i + 1] * inv * g4.y;
      v[i + 2] = v[i + 2] * inv * g4.z, v[i + 3] = v[i + 3] * inv * g4.w;
    }
  }
  if (e.sec_rope[sec]) {
    const RopeRow rr = rope_row(e, m);
#pragma unroll
    for (int p = 0; p < CW / 2; ++p) {
      float2 cs = rope_at(e, rr, p);
      float a = v[2 * p], b = v[2 * p + 1];
      v[2 * p] = a * cs.x - b * cs.y;
      v[2 * p + 1] = a * cs.y + b * cs.x;
    }
  }
}

// Columns are processed in chunks of CW; for EPI_HEADS CW must equal dh.
template <int CW, typename OutT>
DF_DEV void epi_apply(const Epi& e, int m, int n0, float* v) {
  if (m >= e.M) return;
  if (e.kind == EPI_STORE) {
    OutT* o = reinterpret_cast<OutT*>(e.out) + size_t(m) * e.ldo;
    if (n0 + CW <= e.N && (e.ldo & 7) == 0) {
#pragma unroll
      for (int i = 0; i < CW; ++i) {
        float z = v[i] + bias_at(e, n0 + i);
        if (e.act == ACT_GELU) z = gelu_tanh_f(z);
        else if (e.act == ACT_SILU) z = silu_f(z);
        v[i] = z;
      }
      store_vec<CW>(o + n0, v);
      return;
    }
#pragma unroll
    for (int i = 0; i < CW; ++i) {
      int n = n0 + i;
      if (n < e.N) {
        float z = v[i] + bias_at(e, n);
        if (e.act == ACT_GELU) z = gelu_tanh_f(z);
        else if (e.act == ACT_SILU) z = silu_f(z);
        store_val<OutT>(o + n, z);
      }
    }
  } else if (e.kind == EPI_GRES) {
    float* r = e.resid + size_t(m) * e.ldr;
    if (n0 + CW <= e.N && (e.ldr & 3) == 0) {
#pragma unroll
      for (int i = 0; i < CW; i += 4) {
        float4 x = *reinterpret_cast<float4*>(r + n0 + i);
        float g0 = e.gate ? e.gate[n0 + i] : 1.f, g1 = e.gate ? e.gate[n0 + i + 1] : 1.f;
        float g2 = e.gate ? e.gate[n0 + i + 2] : 1.f, g3 = e.gate ? e.gate[n0 + i + 3] : 1.f;
        x.x += g0 * (v[i] + bias_at(e, n0 + i));
        x.y += g1 * (v[i + 1] + bias_at(e, n0 + i + 1));
        x.z += g2 * (v[i + 2] + bias_at(e, n0 + i + 2));
        x.w += g3 * (v[i + 3] + bias_at(e, n0 + i + 3));
        *reinterpret_cast<float4*>(r + n0 + i) = x;
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < CW; ++i) {
      int n = n0 + i;
      if (n < e.N) {
        float z = v[i] + bias_at(e, n);
        r[n] += (e.gate ? e.gate[n] : 1.0f) * z;
      }
    }
  } else if (e.kind == EPI_SWIGLU) {
    // chunk of 32 = 16 gate (W1) columns then 16 up (W3) columns of the same 16 outputs
    OutT* o = reinterpret_cast<OutT*>(e.out) + size_t(m) * e.ldo;
#pragma unroll
    for (int c = 0; c < CW; c += 32) {
      int nb = n0 + c;
      if (nb < e.N) {
        int j0 = (nb >> 5) * 16;
        float w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float a1 = v[c + i] + bias_at(e, nb + i);
          float a3 = v[c + 16 + i] + bias_at(e, nb + 16 + i);
          w[i] = silu_f(a1) * a3;
        }
        store_vec<16>(o + j0, w);
      }
    }
  } else if (e.kind == EPI_HEADS) {
    if (n0 >= e.N) return;
    const int sec = n0 / e.d;
    const int hd = (n0 - sec * e.d) / e.dh;
    const int mper = e.Mper > 0 ? e.Mper : e.M;
    const int bsm = m / mper;     // sample of the stacked batch
    m -= bsm * mper;              // token within the sample (RoPE position, row)
    heads_math<CW>(e, m, n0, sec, hd, v);
    OutT* o = reinterpret_cast<OutT*>(e.sec_out[sec]) + ((size_t(bsm) * e.heads + hd) * mper + m) * e.dh_pad;
    store_vec<CW>(o, v);
  } else if (e.kind == EPI_EULER) {
    // token m = (f*Hp + hh)*Wp + ww ; column p = ((c*pt + i)*ph + j)*pw + k
    m += e.m_base;
    const int mper = e.Mper > 0 ? e.Mper : e.M;
    const int bsm = m / mper;
    m -= bsm * mper;
    int hw = e.Hp * e.Wp;
    int f = m / hw, rem = m - f * hw;
    int hh = rem / e.Wp, ww = rem - hh * e.Wp;
#pragma unroll
    for (int i = 0; i < CW; ++i) {
      int p = n0 + i;
      if (p < e.N) {
        int k = p % e.pw, t = p / e.pw;
        int j = t % e.ph; t /= e.ph;
        int ii = t % e.pt;
        int c = t / e.pt;
        size_t idx = ((size_t(c) * e.Fl + (f * e.pt + ii)) * e.Hl + (hh * e.ph + j)) * e.Wl + (ww * e.pw + k);
        float vel = v[i] + bias_at(e, p);
        if (e.v_batch) {
          e.v_batch[size_t(bsm) * e.C * e.Fl * e.Hl * e.Wl + idx] = vel;
          continue;
        }
        if (e.v_out) e.v_out[idx] = vel;
        e.x_lat[idx] += e.dsig * vel;
      }
    }
  }
}

}  // namespace df
