// Internal runtime of libdf: per-instance weights, workspaces and the stage
// programs (E stand-in, DiT prologue/step/layer, D stand-in).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <mutex>
#include <atomic>
#include <cuda_runtime.h>
#include "../../include/df.h"
#include "kernels.h"

namespace df {

extern thread_local std::string tls_err;
// Counts launches issued by this library (bench "gpu_launches").
extern std::atomic<uint64_t>* g_launches;

#define DF_TRY(expr)                                                             \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      df::tls_err = std::string(#expr) + ": " + cudaGetErrorString(_e);          \
      return _e;                                                                 \
    }                                                                            \
  } while (0)

// Tensor ids (DESIGN.md parameter table; restated from the doc, not shared with the oracle).
enum : uint32_t {
  T_PATCH_W = 0, T_PATCH_B, T_TXT1_W, T_TXT1_B, T_TXT2_W, T_TXT2_B, T_TEMB1_W, T_TEMB1_B, T_TEMB2_W, T_TEMB2_B,
  T_TMOD_W, T_TMOD_B, T_HEAD_MOD, T_HEAD_W, T_HEAD_B,
  T_IMG1_W = 15, T_IMG1_B, T_IMG2_W, T_IMG2_B,  // image-to-video (NEXT-3) only
  T_LAYER_BASE = 64, T_LAYER_STRIDE = 32,
  L_MOD = 0, L_QKV_W, L_QKV_B, L_G_Q, L_G_K, L_O_W, L_O_B, L_G_N3, L_CQ_W, L_CQ_B, L_CK_W, L_CK_B, L_CV_W, L_CV_B,
  L_G_CQ, L_G_CK, L_CO_W, L_CO_B, L_W1, L_B1, L_W3, L_B3, L_W2, L_B2,
  L_KI_W = 24, L_KI_B, L_VI_W, L_VI_B, L_G_KI,  // image-to-video (NEXT-3) only
  T_ENC_BASE = 1u << 20, E_EMB = 0, E_G_A, E_W1, E_W3, E_W2, E_G_F,
  T_DEC_BASE = 1u << 21, D_W1 = 0, D_B1, D_W2F, D_B2F, D_W2R, D_B2R,
};

struct LayerW {
  bf16 *mod, *qkv_wT, *qkv_b, *g_q, *g_k, *o_wT, *o_b, *g_n3, *cq_wT, *cq_b, *ckv_wT, *ckv_b, *g_cq, *g_ck, *co_wT,
      *co_b, *w13T, *b13, *w2T, *b2;
  bf16 *ckvi_wT = nullptr, *ckvi_b = nullptr, *g_ki = nullptr;  // I2V image-token K | V, K gain
  // FP8 step (R29): e4m3 copies of the three weights fed by a normalised activation, each with
  // its per-tensor scale (device fp32): QKV, cross-Q, MLP up (interleaved W1 | W3)
  uint8_t *qkv_q = nullptr, *cq_q = nullptr, *w13_q = nullptr, *o_q = nullptr, *co_q = nullptr, *w2_q = nullptr;
  float* f8s = nullptr;  // [6]: qkv, cq, w13, o, co, w2
  // MXFP8 step (R31): the same six weights in MXFP8 (codes in the *_q arrays, E8M0 block
  // scales in the tiled layout of mx_quant_e4m3)
  uint8_t *qkv_sf = nullptr, *cq_sf = nullptr, *w13_sf = nullptr, *o_sf = nullptr, *co_sf = nullptr, *w2_sf = nullptr;
  // FP8 modes' self-attention (R32): power-of-two e4m3 scales of Q and K bounding every
  // component (sqrt(dh) * max|gain| / 448, rounded up to a power of two)
  float sq = 1.f, sk = 1.f;
};

// Where a logical tensor lives on the device (for df_weight_bits).
struct TensorLoc {
  uint32_t tid;
  bf16* base;
  int in, out, layout, ld, row_off;
};

struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  cudaError_t reserve(size_t bytes);
  void* take(size_t bytes);
  void release();
};

// Kernel classes timed by the optional per-launch profiler (df_profile / df_kernel_stats).
enum KernelKind : int {
  K_QKV = 0, K_ATTN_SELF, K_O, K_NORM, K_CQ, K_ATTN_CROSS, K_CO, K_UP, K_DOWN, K_HEAD, K_PATCH, K_PROLOGUE,
  K_MISC, K_COUNT
};

// Records a CUDA event pair around each launch of a class; harvested after the stream
// passes them (no host synchronisation on the launch path).
struct Prof {
  std::mutex mu;
  std::vector<cudaEvent_t> pool;
  struct Pending { int kind; cudaEvent_t a, b; double flops, bytes; };
  std::vector<Pending> pending;
  uint64_t count[K_COUNT] = {};
  double ms[K_COUNT] = {}, flops[K_COUNT] = {}, bytes[K_COUNT] = {};
  cudaEvent_t get();
  void reserve(size_t n);  // pre-create events so the launch path never calls cudaEventCreate
  void harvest();   // consumes completed pairs (blocks on each pending pair)
  void reset();
};

// T->D chunk plan over the fp32 latent [C, F, H, W] (R22): a chunk
// is the block of latent rows [h0, h1) of one latent frame f, all C channels (C strided rows
// of (h1 - h0) W floats).  Video: one frame per chunk; image (F = 1): blocks of hb rows.
// Chunk k -> (f, h0, h1) with f = k / nbh.  n = 1 with hb = H, F = 1 is the whole latent.
struct LatentBlocks {
  int C = 0, F = 1, H = 0, W = 0, hb = 0, nbh = 1, n = 1;
  void block(int k, int& f, int& h0, int& h1) const {
    f = k / nbh;
    h0 = (k % nbh) * hb;
    h1 = h0 + hb < H ? h0 + hb : H;
  }
};

// Chunk-wise consumption of the E->T payload by the request prologue (a1): the prompt ctx
// arrives in chunks of rows_per_chunk rows; wait(c) makes the prologue's stream wait for chunk
// c (device-side) before the rows of chunk c are projected.  Chunks past the prompt (negative
// prompt, I2V image tokens) are all waited for before those parts are read.
struct ChunkHook {
  int rows_per_chunk = 0;
  int nchunks = 0;
  float shift = 0.f;        // > 0: the sigma schedule is generated on the device (sigma_schedule)
  cudaError_t (*wait)(void* user, int c) = nullptr;
  void* user = nullptr;
};

// Chunk-wise production of the final latent (a12 -> a14): on the step it is passed to, the
// head + Euler epilogue runs once per latent block of `lb` and done(k) is called right after
// block k is enqueued (the T->D send of chunk k waits on the event it records).
struct BlockHook {
  LatentBlocks lb;
  cudaError_t (*done)(void* user, int k) = nullptr;
  void* user = nullptr;
};

// Per-request conditioning handle (df_cond).
struct Cond {
  int S = 0;
  std::vector<float> sig;   // host sigma schedule, S+1
  float* sig_dev = nullptr;
  void* kc = nullptr;       // [layers][H][L][dhp]
  void* vc = nullptr;
  float* e = nullptr;       // [S, d]
  float* e6 = nullptr;      // [S, 6d]
  Arena mem;
  int device = 0;
  int B = 1;                // 2: classifier-free guidance (conditional, negative prompt)
  float guidance = 1.f;
  void* kci = nullptr;      // I2V: image-token K/V [layers][B][H][L_img][dhp]
  void* vci = nullptr;
  float* y = nullptr;       // I2V: y [C_y, F, H, W] (mask + first-frame latent), per request
};

struct Model {
  df_dit_cfg c{};
  int precision = DF_BF16;
  int device = 0;
  int stage = DF_T;
  uint64_t seed = 0;
  int max_steps = 0;
  // derived
  int N = 0, P = 0, dh = 0, dhp = 0, Fp = 0, Hp = 0, Wp = 0;
  int Pin = 0;              // patch-embedding input width ((C + C_y) pt ph pw)
  Arena wmem, ws, f8mem;
  std::vector<TensorLoc> locs;
  // global DiT weights
  bf16 *patch_wT = nullptr, *patch_b = nullptr, *txt1_wT = nullptr, *txt1_b = nullptr, *txt2_wT = nullptr,
       *txt2_b = nullptr, *temb1_wT = nullptr, *temb1_b = nullptr, *temb2_wT = nullptr, *temb2_b = nullptr,
       *tmod_wT = nullptr, *tmod_b = nullptr, *head_mod = nullptr, *head_wT = nullptr, *head_b = nullptr;
  bf16 *img1_wT = nullptr, *img1_b = nullptr, *img2_wT = nullptr, *img2_b = nullptr;  // I2V image projection
  std::vector<LayerW> Lw;
  // encoder / decoder
  bf16 *emb = nullptr, *g_a = nullptr, *e_w13T = nullptr, *e_w2T = nullptr, *g_f = nullptr;
  bf16 *d1_w = nullptr, *d1_b = nullptr, *d2f_w = nullptr, *d2f_b = nullptr, *d2r_w = nullptr, *d2r_b = nullptr;
  // workspace (T)
  float* r = nullptr;       // residual [N, d]
  void* h = nullptr;        // [N, d] bf16 | f32
  void* q = nullptr;        // [H][N][dhp]
  void* k = nullptr;
  void* v = nullptr;
  void* qc = nullptr;
  void* o = nullptr;        // [N, d]
  void* a = nullptr;        // [N, f]
  void* oi = nullptr;       // I2V: image cross-attention output [N, d]
  void* X = nullptr;        // [N, P]
  float* tmp = nullptr;     // fp32 build: raw GEMM out [N, max(3d, 2f)]
  float* sk_ws = nullptr;   // bf16 build: stream-K partial tiles [SMs/2][2][256][128] fp32
  unsigned* sk_flag = nullptr;  // [SMs] epochs
  float* mods = nullptr;    // [layers][6][d]
  float* headmod = nullptr; // [2][d]
  float2* rope = nullptr;
  float* vbatch = nullptr;  // [2][C,F,H,W] velocities of a CFG batch
  uint8_t* hq = nullptr;    // FP8 step: e4m3 GEMM input [2N, max(d, f)] and its row scales [2N]
  float* hs = nullptr;
  uint8_t* hsf = nullptr;   // MXFP8 step: the GEMM input's tiled E8M0 block scales
  uint8_t* q8 = nullptr;    // FP8 modes: e4m3 Q and K of the self-attention (R32) [B*heads][N][128]
  uint8_t* k8 = nullptr;
  uint8_t* v8t = nullptr;   // FP8 modes: e4m3 V^T [B*heads][128][ldv8] (R33) and its scale (device)
  float* v8s = nullptr;
  int ldv8 = 0;
  // encoder workspace
  float* ez = nullptr;      // [L, d_txt]
  void* ea = nullptr;       // [L, d_txt]
  void* ef = nullptr;       // [L, f_e]
  float* etmp = nullptr;    // [L, 2 f_e]
  std::vector<const bf16*> layer_mods;
  Prof* prof = nullptr;
  int prof_every = 1;       // profile the launches of every prof_every-th denoising step
  int cur_kind = K_MISC;
  double cur_flops = 0, cur_bytes = 0;

  cudaError_t create(const df_dit_cfg& cfg, int precision, int device, int stage, uint64_t seed, int max_steps);
  void destroy();
  bool f32() const { return precision == DF_FP32_VALIDATION; }
  bool fp8() const { return precision == DF_FP8 || precision == DF_MXFP8; }  // e4m3 block GEMMs
  bool mx() const { return precision == DF_MXFP8; }                           // ... with MX block scales
  size_t act_bytes() const { return f32() ? 4 : 2; }

  cudaError_t prepare(const void* ctx_bf16, const float* sig_host, int S, cudaStream_t st, Cond* out,
                      const void* ctx_neg_bf16 = nullptr, float guidance = 1.f, const void* clip_bf16 = nullptr,
                      const float* y = nullptr, const ChunkHook* hook = nullptr);
  bool i2v() const { return c.C_y > 0; }
  cudaError_t step(const Cond& c, int i, float* x, float* v_out, cudaStream_t st, const BlockHook* bh = nullptr);
  cudaError_t layer(const Cond& c, int i, int l, float* r_io, cudaStream_t st);
  cudaError_t encode(const int32_t* ids, void* ctx_bf16, cudaStream_t st);
  cudaError_t decode(const float* x, float* out, cudaStream_t st);
  cudaError_t decode_block(const float* x, float* out, const LatentBlocks& lb, int k, cudaStream_t st);

  // helpers
  cudaError_t gemm(const void* A, int lda, const bf16* W, int ldw, int M, int Nn, int K, const Epi& e, int out_f32,
                   cudaStream_t st);
  cudaError_t attn(const void* Q, const void* K, const void* V, void* O, int Nq, int Nk, cudaStream_t st, int B = 1);
  Epi heads_epi(int M, int nsec, const bf16* bias, void* o0, const bf16* g0, int rope0, void* o1, const bf16* g1,
                int rope1, void* o2, const bf16* g2, int rope2, int Mper = 0) const;
  cudaError_t block(const Cond& c, int i, int l, float* r, cudaStream_t st);
  cudaError_t norm(const float* x, void* out, int M, int dd, const float* shift, const float* scale, const bf16* gain,
                   cudaStream_t st);
  // FP8 step: the normalised activation straight to e4m3 (hq, hs), then an e4m3 GEMM
  cudaError_t norm_f8(const float* x, int M, const float* shift, const float* scale, const bf16* gain, cudaStream_t st);
  cudaError_t attn_qf8(int l, int Nq, int B, cudaStream_t st);
  cudaError_t gemm_f8(const uint8_t* Wq, const float* wscale, const uint8_t* wsf, int M, int Nn, int K, const Epi& e,
                      cudaStream_t st);
  cudaError_t quant_f8(const void* x, int M, int K, cudaStream_t st);  // bf16 activation -> hq / hs
  cudaError_t quantize_weights(cudaStream_t st);
  cudaError_t init_weights(cudaStream_t st);
};

}  // namespace df
