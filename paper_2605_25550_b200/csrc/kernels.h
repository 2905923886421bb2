// Host-side launchers of the sm_100a kernels (internal to libdf; not the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "epilogue.cuh"

namespace df {

int num_sms();
extern int g_pdl;  // 1: launch the hot kernels with programmatic dependent launch (DF_PDL=1; default off)
// Launch helper: cudaLaunchKernelEx with optional PDL attribute.
cudaError_t launch_ex(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void** args);
extern int g_disable_pair;  // 1: never use the CTA-pair GEMM (tests)

// ---- tensor-core GEMM: out = epilogue(A[M,K] (bf16, row-major, lda) x W[N,K]^T (bf16, ldw)).
// BN in {64, 128, 256}.  Returns cudaError_t of the launch.
// e4m3 (NEXT-4): per-tensor quantiser (3 launches) and the CTA-pair e4m3 GEMM
cudaError_t quant_e4m3(const bf16* x, size_t n, uint8_t* q, float* scale, cudaStream_t st);
// MXFP8 (NEXT-4, R30): OCP MX quantiser (E4M3 elements, 32-element blocks, tiled E8M0 scale
// bytes) and the block-scaled CTA-pair GEMM (kind::mxf8f6f4.block_scale)
cudaError_t mx_quant_e4m3(const bf16* x, int M, int K, uint8_t* q, uint8_t* sf, cudaStream_t st);
// bytes of the tiled E8M0 scales of an [M, K] MXFP8 matrix: (K / 128) * ceil(M / 128) * 512
inline size_t mx_sf_bytes(size_t M, size_t K) { return (K / 128) * ((M + 127) / 128) * 512; }
// RMSNorm + modulation (or gain) with MXFP8 output (R31): codes q [M, d], tiled block scales sf
cudaError_t rmsnorm_mx(const float* x, uint8_t* q, uint8_t* sf, int M, int d, const float* shift, const float* scale,
                       const bf16* gain, float eps, cudaStream_t st);
cudaError_t gemm_mxf8(const uint8_t* qa, const uint8_t* sa, const uint8_t* qb, const uint8_t* sb, int M, int N, int K,
                      void* out, int ldo, int out_f32, cudaStream_t st);
// FP8 modes (R32): self-attention with e4m3 Q, K (scale folded into `scale`) and bf16 V, and the
// quantiser of the head-major bf16 Q / K: q = e4m3(x * inv), inv a power of two
cudaError_t attn_tc_qf8(const uint8_t* Q8, const uint8_t* K8, const bf16* V, bf16* O, int H, int Nq, int Nk,
                        float scale, cudaStream_t st, int heads_per_sample);
cudaError_t qk_e4m3(const bf16* x, size_t n, float inv, uint8_t* q, cudaStream_t st);
// R33: PV on e4m3 too -- V^T e4m3 [H][128][ldv] with the per-tensor power-of-two scale *vscale
cudaError_t attn_tc_f8(const uint8_t* Q8, const uint8_t* K8, const uint8_t* V8T, int ldv, const float* vscale, bf16* O,
                       int H, int Nq, int Nk, float scale, cudaStream_t st, int heads_per_sample);
// head-major bf16 V [H][N][128] -> e4m3 V^T [H][128][ldv] with s = pow2ceil(amax|V| / 448) written
// to vscale[0]; vscale[1] is the amax accumulator (zero on entry, left zero); three PDL launches
cudaError_t v_e4m3t(const bf16* V, int H, int N, int ldv, float* vscale, uint8_t* VT, cudaStream_t st);
// MXFP8 step (R31): the block-scaled GEMM through the TMA-store epilogues of the bf16 path
cudaError_t gemm_mxf8_epi(const uint8_t* qa, const uint8_t* sa, const uint8_t* qw, const uint8_t* sw, int M, int N,
                          int K, const Epi& e, cudaStream_t st);
// FP8 step (R29): e4m3 A with per-row scales x e4m3 W with a per-tensor scale, through the
// bf16 path's TMA-store epilogues (heads / SwiGLU / stores / gated residual)
cudaError_t gemm_e4m3_epi(const uint8_t* qa, const float* a_row, const uint8_t* qw, const float* w_scale, int M, int N,
                          int K, const Epi& e, cudaStream_t st);
// bf16 activation [M, K] -> e4m3 per row with power-of-two row scales (R29); K % 8 == 0
cudaError_t quant_rows_e4m3(const bf16* x, uint8_t* q, float* s, int M, int K, cudaStream_t st);
// RMSNorm (+ modulation or gain) with e4m3 output quantised per row (R29): q[m, :] =
// e4m3(y[m, :] / s[m]), s[m] = amax|y[m, :]| / 448 (1 for a zero row), y in fp32.
cudaError_t rmsnorm_e4m3(const float* x, uint8_t* q, float* s, int M, int d, const float* shift, const float* scale,
                         const bf16* gain, float eps, cudaStream_t st);
cudaError_t gemm_e4m3(const uint8_t* qa, const uint8_t* qb, const float* sa, const float* sb, int M, int N, int K,
                      void* out, int ldo, int out_f32, cudaStream_t st);
cudaError_t gemm_tc(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K, const Epi& epi,
                    int out_f32, cudaStream_t st, int bn = 256);

// ---- SIMT fp32 GEMM: C[M,N] (fp32, ldc) = act(act_in(A) x W^T + bias); A fp32 or bf16.
cudaError_t gemm_simt(const void* A, int a_bf16, int lda, int act_in, const bf16* W, int ldw, float* C, int ldc,
                      int M, int N, int K, const bf16* bias, int act, cudaStream_t st);
// Apply an epilogue to a raw fp32 accumulator tmp[M, N] (fp32 validation build).
cudaError_t epi_rows(const float* tmp, const Epi& epi, int out_f32, cudaStream_t st);

// ---- attention: O[n, h*dh + c] = softmax(Q_h K_h^T * scale) V_h
// Q/K/V head-major [H][Nq|Nk][dh_pad] bf16; O token-major [Nq, H*dh] bf16.
// heads_per_sample (0 = H): H counts the heads of a stacked batch (B = H / heads_per_sample
// samples, sample-major [b][h]); O rows are b*Nq + q with heads_per_sample*dh columns.
cudaError_t attn_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, int H, int Nq, int Nk, int dh, int dh_pad,
                    float scale, cudaStream_t st, int heads_per_sample = 0);
// fp32 validation build: same layout with float and dh_pad == dh.
cudaError_t attn_simt(const float* Q, const float* K, const float* V, float* O, int H, int Nq, int Nk, int dh,
                      float scale, cudaStream_t st, int heads_per_sample = 0);
// x += dsig * (v_u + g (v_c - v_u)) with v_batch = [v_c | v_u]; v_out (optional) gets the guided v
cudaError_t cfg_euler(float* x, const float* v_batch, float* v_out, size_t n, float guidance, float dsig, cudaStream_t st);

// ---- elementwise
// out[m, :] = RMSNorm(x[m, :]) * (1 + scale) + shift     (mode 0; scale/shift fp32 [d])
//           = RMSNorm(x[m, :]) * gain                     (mode 1; gain bf16 [d])
cudaError_t rmsnorm_mod(const float* x, void* out, int out_f32, int M, int d, const float* shift, const float* scale,
                        const bf16* gain, float eps, cudaStream_t st);
// X[n, p] = patchify(concat(x, y))   (bf16 or fp32 out; y [Cy, F, H, W] only for I2V, Cy = 0 otherwise)
cudaError_t patchify(const float* x, const float* y, int Cy, void* X, int out_f32, int C, int F, int H, int W, int pt,
                     int ph, int pw, cudaStream_t st);
// o += oi (bf16 or fp32, n elements)
cudaError_t add_into(void* o, const void* oi, size_t n, int f32, cudaStream_t st);
// The sigma schedule (R13) on the device, in fp64 then rounded to fp32 exactly as the host's
// sigmas_host: s_i = 1 - i/S, sigma_i = shift s_i / (1 + (shift - 1) s_i), i = 0..S.  The
// pipeline workers use it so that no pageable host->device copy (a host-blocking stream sync)
// sits on their enqueue path.
cudaError_t sigma_schedule(float* sig, int S, float shift, cudaStream_t st);
// sinusoid rows s[i, :] = [cos(1000 sig_i w) | sin(1000 sig_i w)], i < S
cudaError_t sinusoid(const float* sig_dev, float* s, int S, int freq_dim, cudaStream_t st);
// mods[l][k][:] = e6[k][:] + M_l[k][:] for k < 6, all layers; head[0..1][:] = head_mod + e
cudaError_t modulations(const float* e6, const float* e, const bf16* const* layer_mod, int layers,
                        const bf16* head_mod, int d, float* mods, float* head, cudaStream_t st);
cudaError_t silu_inplace(float* x, size_t n, cudaStream_t st);

// ---- init / RNG (Philox4x32-10)
// dst element (r, c) of a row-major [rows, ld] matrix gets logical element given by `layout`:
//   layout 0: identity, logical [in=rows, out=cols]            dst[k*ld + n]
//   layout 1: transposed, dst[(row_off + n)*ld + k]            (W^T, K-major)
//   layout 2: swiglu-interleaved transposed: n -> (n/16)*32 + half*16 + n%16
struct InitSpec {
  uint64_t seed;
  uint32_t tid;
  int kind;        // 0 plain (scale a), 1 gain (1 + w)
  float a;         // fp32(sqrt(3) * std)
  int in, out;     // logical shape [in, out]
  int layout;      // 0/1/2 as above
  int ld;          // destination row stride (elements)
  int row_off;     // destination row offset (layouts 1/2), or `half` for layout 2 (0: W1, 1: W3)
};
cudaError_t init_tensor(bf16* dst, const InitSpec& s, cudaStream_t st);
cudaError_t gen_noise(float* x, size_t n, uint64_t seed, cudaStream_t st);
// I2V E stand-in: clip tokens (bf16) and y (fp32) of request `seed` (R27)
cudaError_t gen_image_cond(uint64_t seed, bf16* clip, size_t n_clip, float* y, int Cy, int F, int H, int W,
                           cudaStream_t st);
cudaError_t gen_tokens(int32_t* ids, int n, int vocab, uint64_t seed, cudaStream_t st, uint32_t stream_c3 = 2);

// ---- E / D stand-ins
cudaError_t embed_rows(const int32_t* ids, const bf16* emb, float* z, int L, int dt, cudaStream_t st);
cudaError_t decode_latent(const float* x, float* out, int C, int F, int H, int W, int cdec, const bf16* w1,
                          const bf16* b1, const bf16* w2f, const bf16* b2f, const bf16* w2r, const bf16* b2r,
                          cudaStream_t st);
cudaError_t decode_latent_region(const float* x, float* out, int C, int F, int H, int W, int cdec, const bf16* w1,
                                 const bf16* b1, const bf16* w2f, const bf16* b2f, const bf16* w2r, const bf16* b2r,
                                 int f0, int nf, int p_begin, int p_end, cudaStream_t st);

// ---- handoff helpers
cudaError_t payload_hash(const void* buf, size_t nbytes, size_t word_offset, unsigned long long* out,
                         cudaStream_t st);
cudaError_t delay_ns(uint64_t ns, cudaStream_t st);

}  // namespace df
