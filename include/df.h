/* df.h — C ABI of the B200-native DisagFusion hot path (arXiv 2605.25550).
 *
 * The library serves the DiT stage of a disaggregated Encoder -> Transformer (DiT)
 * -> Decoder pipeline (§sec:decentral-pipeline) through the paper's
 * asynchronous stage handoff: the encoder's conditioning
 * hidden states move E -> T and the final latent moves T -> D in chunks on a
 * dedicated comm stream with one event per chunk, so a stage never blocks on its
 * downstream neighbour.
 *
 * Conventions (every call):
 *   - returns df_status; nothing throws or aborts across the ABI;
 *   - device pointers are raw CUDA device addresses on the device of the instance
 *     named by the call; `stream` is a cudaStream_t (NULL = legacy default stream);
 *   - "host" pointers are ordinary CPU memory; sizes are in elements unless the
 *     name says bytes;
 *   - ownership: df_init copies its graph; the context owns all weights, work
 *     buffers, receive slots and caches; caller-owned device buffers passed to a
 *     stream-ordered call must stay valid until that stream work completes;
 *   - CUDA errors are sticky: after DF_ERR_CUDA every further call on the
 *     context returns DF_ERR_STATE; df_last_error() has the message.
 *   - the product path has no CPU fallback: df_init fails with DF_ERR_CUDA if no
 *     sm_100 device is present.
 */
#ifndef DF_H_
#define DF_H_
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DF_OK = 0,
  DF_AGAIN = 1,          /* backpressure: request ring full, retry later */
  DF_EMPTY = 2,          /* df_poll: nothing completed within the timeout                     */
  DF_ERR_INVALID = 10,   /* bad argument; no side effects                                      */
  DF_ERR_CAPACITY = 11,  /* Eq. 1 g_E+g_T+g_D > G, or a stage with 0 instances         */
  DF_ERR_NOMEM = 12,
  DF_ERR_DUPLICATE = 13, /* request id reused ("retry deduplication")                  */
  DF_ERR_STATE = 14,     /* wrong lifecycle, or a call after a sticky CUDA error               */
  DF_ERR_CUDA = 20,
  DF_ERR_NCCL = 21
} df_status;

typedef enum { DF_E = 0, DF_T = 1, DF_D = 2 } df_stage;
/* df_graph.precision.  DF_FP8 (NEXT-4, R29): the six GEMMs of every block (QKV, O,
 * cross-Q, cross-O, MLP up, MLP down) take e4m3 operands -- activations quantised per token row
 * with power-of-two scales (by the RMSNorm that produces them, or a row quantiser for the
 * attention and SwiGLU outputs), weights per tensor -- with fp32 accumulation; everything else
 * as DF_BF16.  Needs d >= 256, a head size of 128 and N >= 256 latent tokens (CTA-pair tiles).
 * DF_MXFP8 (NEXT-4, R31): the same six GEMMs on MXFP8 operands (R30: OCP MX, E4M3
 * elements, one E8M0 scale per 32 consecutive k of a row -- activations quantised by the RMSNorm
 * or the MX quantiser, weights at init) through the block-scaled tensor-core GEMM; needs d and
 * the MLP width multiples of 128 and d in {256, 3072, 5120}. */
enum { DF_BF16 = 0, DF_FP32_VALIDATION = 1, DF_FP8 = 2, DF_MXFP8 = 3 };
enum { DF_ASYNC = 0, DF_SYNC = 1, DF_PERMUTE = 2, DF_HASH = 4, DF_LATENT_BLOCKS = 8 }; /* handoff flags */
#define DF_ALL_CHUNKS 0xFFFFFFFFu
#define DF_MAX_INST 32

typedef struct df_ctx df_ctx;
typedef struct { uint64_t lo, hi; } df_req_id;               /* 128-bit request id */

/* DiT shape (the paper fixes none of it). */
typedef struct {
  uint32_t C, F, H, W;          /* latent [C, F, H, W]                                  */
  uint32_t pt, ph, pw;          /* patch                                                */
  uint32_t d, heads, ffn, layers;
  uint32_t d_txt, L_txt;        /* encoder hidden width / text tokens                   */
  uint32_t freq_dim;            /* time sinusoid width (256)                            */
  uint32_t vocab, enc_ffn, dec_width; /* E / D stand-ins (R17)                          */
  float eps, rope_theta;
  uint32_t rope_axes[3];        /* (D_f, D_h, D_w), sum = d/heads                        */
  /* image-to-video conditioning (NEXT-3; R27): C_y > 0 makes the patch embedding
   * read concat(x, y) (y [C_y, F, H, W] fp32: first-frame mask + VAE latent) and adds a
   * cross-attention over L_img image tokens of width d_img per block; 0 = text only. */
  uint32_t C_y, L_img, d_img;
} df_dit_cfg;

/* Stage graph: the fixed chain E -> T -> D with an E:T:D instance ratio. */
typedef struct {
  uint32_t n_inst;
  /* device: CUDA device index in the process that hosts the instance; rank: that
   * process (0 in single-process mode).  Co-location allowed. */
  struct { int32_t device; int32_t stage; int32_t rank; } inst[DF_MAX_INST];
  uint32_t G;                   /* GPU budget for Eq. 1                                  */
  uint64_t chunk_bytes[2];      /* per edge (0: E->T ctx, 1: T->D latent); 0 = whole     */
  uint32_t n_slots;             /* receive slots per consumer per edge, >= 2             */
  uint32_t handoff_mode;        /* DF_ASYNC (default) | DF_SYNC (P:L151 comparison)      */
  uint32_t ring_capacity;       /* request ring, power of two                   */
  uint32_t precision;           /* DF_BF16 | DF_FP32_VALIDATION | DF_FP8 | DF_MXFP8      */
  uint32_t max_steps;           /* largest S a request may ask for                       */
  uint64_t weight_seed;
  float jitter_p;               /* each transfer delayed by jitter_delay_s w.p. p */
  float jitter_delay_s;
  uint64_t jitter_seed;
  df_dit_cfg dit;
  /* One process per GPU (world > 1): every rank passes the same graph with its own
   * `rank`; instances of other ranks are reached through a POSIX shared-memory control
   * plane named shm_name (FAA metadata rings) and CUDA IPC receive slots
   * (the posted destination addresses).  Rank 0 creates the segment. */
  int32_t rank, world;
  char shm_name[64];
  /* Chunk before which an injected delay is placed (0: before the first chunk; clamped to
   * the last).  The delay holds back that chunk and the ones after it, so a consumer that
   * works chunk by chunk is already busy on the earlier ones (handoff-stress tests). */
  uint32_t jitter_chunk;
} df_graph;

/* df_init: validate the graph (Eq. 1), allocate and Philox-initialise every
 * instance's weights, create streams, receive slots and rings, and
 * start one host worker thread per instance.  *out owns everything. */
df_status df_init(const df_graph* g, df_ctx** out);
/* Drains outstanding requests, joins workers, frees all device memory. */
df_status df_finalize(df_ctx* ctx);
const char* df_last_error(const df_ctx* ctx);

/* ------------------------------------------------------------------ serving API */
typedef struct {
  uint32_t steps;               /* Euler steps S (<= max_steps)                          */
  float shift;                  /* sigma-schedule shift                                  */
  uint64_t seed;                /* noise / token seed                                    */
  const int32_t* token_ids;     /* host [L_txt] or NULL (derive from seed); copied       */
  void* out_host;               /* host fp32 [3, 1+4(F-1), 8H, 8W]; caller keeps it alive */
  uint64_t out_bytes;           /*   until df_poll returns this request (MPI Irecv rule)  */
  uint64_t user_tag;
  df_req_id id;                 /* {0,0} = assign one                                    */
  float guidance;               /* classifier-free guidance scale; 0 or 1 = off (NEXT-2). When
                                   on, E also encodes the negative prompt (tokens from the seed's
                                   negative stream or neg_token_ids) and T runs a batch of 2.  */
  const int32_t* neg_token_ids; /* host [L_txt] or NULL; copied                          */
} df_request;
/* Admit a request ("request scheduler inserts the request into the global
 * request buffer").  MT-safe.  DF_AGAIN if the ring is full, DF_ERR_DUPLICATE if
 * the id was seen before. */
df_status df_submit(df_ctx* ctx, const df_request* r, df_req_id* id_out);

typedef struct {
  df_req_id id;
  df_status status;
  uint64_t user_tag;
  int32_t inst[3];              /* E, T, D instance that served it                       */
  double t_submit, t_start[3], t_end[3], t_done; /* seconds, host monotonic clock        */
  float stage_ms[3];            /* device time of E, T, D compute                         */
  float xfer_ms[2];             /* device time of the E->T / T->D transfers (first copy issued
                                   -> last chunk landed)                                 */
  float exposed_ms[2];          /* consumer stall on in-flight data per edge, on the consumer's
                                   clock: sum over chunks c of max(0, A_c - max(R_c, P_c))
                                                             */
  uint64_t hash_src[2], hash_dst[2]; /* payload hash on both sides of each edge  */
  const void* out_view;         /* the decoded fp32 output in THIS process (the D rank's copy  */
  uint64_t out_view_bytes;      /*   in multi-process mode); valid until the next df_poll      */
  float overlap_ms[2];          /* per edge: how long before the last chunk landed the consumer
                                   was already working on chunk 0 (chunk-wise consumption:
                                   the prologue projects ctx rows as they land, D decodes
                                   latent blocks as they land; north_star) */
} df_completion;
/* Pop up to max completions ("final output is returned to the request
 * scheduler").  Blocks up to timeout_ms (-1 forever). DF_EMPTY if none. */
df_status df_poll(df_ctx* ctx, df_completion* out, uint32_t max, uint32_t* n_out, int32_t timeout_ms);

/* Rebalance the E:T:D ratio (Alg. 1 "Apply").  Each instance host keeps its
 * device.  If a stage has at least g_s instances, the first g_s of them receive new
 * requests and the rest drain.  If a stage has fewer, instances of stages with
 * a surplus are re-purposed: taken out of routing, drained (their queued and in-flight
 * work completes; no request is lost), their old stage freed, the new stage created
 * (weights regenerated from the weight seed -- the cold start) and put into service; each
 * move is logged (df_sched_log, action 4, with the drain and cold-start times).  Blocks
 * until done.  DF_ERR_CAPACITY if a g_s < 1 or sum g exceeds the instance hosts (or G);
 * DF_ERR_STATE if re-purposing is needed on a multi-process context. */
df_status df_set_ratio(df_ctx* ctx, uint32_t gE, uint32_t gT, uint32_t gD);

/* ------------------------------------------------------------------ low-level, stream-ordered */
typedef struct df_cond df_cond;   /* per-request conditioning: cross K/V of every layer, e/e6 of every step */
/* Request prologue on T instance t_inst from a device bf16 ctx
 * [L_txt, d_txt]; sigmas = host float[S+1] schedule.  *out is caller-owned. */
/* Classifier-free guidance variant (NEXT-2; "negative prompts"): ctx_neg_dev is the
 * negative prompt's bf16 ctx; every df_dit_step then runs the conditional and negative
 * samples as one batch of 2 and updates x with v = v_u + guidance (v_c - v_u). */
df_status df_dit_prepare_cfg(df_ctx* ctx, int32_t t_inst, const void* ctx_dev, const void* ctx_neg_dev,
                             float guidance, const float* sigmas, uint32_t S, void* stream, df_cond** out);
df_status df_dit_prepare(df_ctx* ctx, int32_t t_inst, const void* ctx_dev, const float* sigmas, uint32_t S,
                         void* stream, df_cond** out);
/* Image-to-video prologue (NEXT-3; "Encoder produces latent tensors"):
 * for a graph with dit.C_y > 0.  clip_dev: device bf16 [L_img, d_img] image tokens; y_dev:
 * device fp32 [C_y, F, H, W] (first-frame mask + VAE latent), copied into the conditioning
 * (the caller may reuse it once the stream passes).  ctx_neg_dev (optional) adds classifier-
 * free guidance as in df_dit_prepare_cfg.  DF_ERR_INVALID for a text-only graph;
 * df_dit_prepare refuses an I2V graph (it has no image inputs). */
df_status df_dit_prepare_i2v(df_ctx* ctx, int32_t t_inst, const void* ctx_dev, const void* clip_dev,
                             const float* y_dev, const void* ctx_neg_dev, float guidance, const float* sigmas,
                             uint32_t S, void* stream, df_cond** out);
/* One denoising step i (a2-a12): x_dev fp32 [C,F,H,W] updated in place,
 * x <- x + (sigma_{i+1} - sigma_i) v; v_dev (optional, fp32 [C,F,H,W]) gets v. */
df_status df_dit_step(df_ctx* ctx, int32_t t_inst, const df_cond* c, uint32_t i, float* x_dev, float* v_dev,
                      void* stream);
/* One block l at step i on a caller residual r_dev fp32 [N, d] (in place) — for
 * per-layer parity at production shapes. */
df_status df_dit_layer(df_ctx* ctx, int32_t t_inst, const df_cond* c, uint32_t i, uint32_t l, float* r_dev,
                       void* stream);
df_status df_cond_release(df_ctx* ctx, df_cond* c);

/* E stand-in: ids_dev int32 [L_txt] -> ctx_dev bf16 [L_txt, d_txt] (the E->T payload). */
df_status df_encode(df_ctx* ctx, int32_t e_inst, const int32_t* ids_dev, void* ctx_dev, void* stream);
/* D stand-in: latent fp32 [C,F,H,W] -> out fp32 [3, 1+4(F-1), 8H, 8W]. */
df_status df_decode(df_ctx* ctx, int32_t d_inst, const float* x_dev, float* out_dev, void* stream);
/* x0 ~ N(0,1) and token ids from a request seed. */
df_status df_noise(df_ctx* ctx, int32_t inst, uint64_t seed, float* x_dev, void* stream);
df_status df_tokens(df_ctx* ctx, int32_t inst, uint64_t seed, int32_t* ids_dev, void* stream);
/* I2V E stand-in (NEXT-3, R27): the image conditioning of request `seed` — clip_dev
 * bf16 [L_img, d_img] and y_dev fp32 [C_y, F, H, W] (device, caller-owned); DF_ERR_INVALID for
 * a text-only graph. */
df_status df_image_cond(df_ctx* ctx, int32_t inst, uint64_t seed, void* clip_dev, float* y_dev, void* stream);

/* Chunked stage handoff: copy bytes from src (device of
 * src_inst) into dst (device of dst_inst) in ceil(bytes/chunk_bytes) chunks (chunk sizes
 * rounded up to 16 bytes, at most 64 chunks) on the library's comm stream after the work
 * already queued on src_stream, one event per chunk.  DF_LATENT_BLOCKS: bytes is the
 * graph's fp32 latent [C,F,H,W] and a chunk is a block of latent rows of one frame (all
 * channels; a video chunk is one latent frame), sized by chunk_bytes (R22).  DF_SYNC also
 * makes src_stream wait for the last chunk.  DF_PERMUTE issues chunks in a seeded random
 * order (tests).  DF_HASH hashes both sides (the destination on the destination's aux
 * stream).  Jitter per the graph's jitter_p / jitter_delay_s / jitter_chunk.  Never blocks
 * the host.  *out is caller-owned. */
typedef struct {
  int32_t src_inst, dst_inst;
  const void* src;
  void* dst;
  uint64_t bytes, chunk_bytes;
  uint32_t flags;
  uint64_t seq;                 /* request sequence number (jitter draw / permutation seed) */
  uint32_t edge;                /* 0: E->T, 1: T->D                                         */
} df_handoff_desc;
typedef struct df_xfer df_xfer;
df_status df_handoff(df_ctx* ctx, const df_handoff_desc* d, void* src_stream, df_xfer** out);
/* Make dst_stream wait for chunk c (or DF_ALL_CHUNKS). Never blocks the host. */
df_status df_handoff_wait(df_ctx* ctx, df_xfer* x, uint32_t chunk, void* dst_stream);
/* Host query: chunks landed so far; hashes {src, dst} once complete (DF_HASH). */
df_status df_handoff_query(df_ctx* ctx, df_xfer* x, uint32_t* chunks_done, uint64_t hash[2]);
df_status df_handoff_release(df_ctx* ctx, df_xfer* x);

/* Payload hash of a device buffer (DESIGN.md §Handoff hash), synchronous. */
df_status df_payload_hash(df_ctx* ctx, int32_t inst, const void* buf_dev, uint64_t nbytes, uint64_t* hash_out);

/* ------------------------------------------------------------------ kernel-level entry points (tests, bench) */
/* Parity check 0: copy the bf16 bits of parameter `tensor_id` (logical [in,out]
 * row-major, DESIGN.md parameter table) of instance inst into host `dst`. */
df_status df_weight_bits(df_ctx* ctx, int32_t inst, uint32_t tensor_id, uint16_t* dst, uint64_t n);
/* out = A[M,K] (bf16) x W[N,K]^T (bf16), fp32 out [M,N]; tensor-core kernel (tc=1), tensor cores
 * with the stream-K schedule (tc=2: uses the workspace of the first T instance, taken when whole-tile
 * waves would leave > 8 % of the CTA pairs idle; DF_ERR_STATE without a T instance), or
 * SIMT (tc=0).  Device pointers; stream-ordered. */
df_status df_op_gemm(df_ctx* ctx, const void* A, const void* W, float* out, int32_t M, int32_t N, int32_t K,
                     int32_t tc, void* stream);
/* FP8 (P:L116 names quantisation as a serving optimisation, the paper fixes
 * no format -- DESIGN.md R28): per-tensor e4m3 quantisation of n bf16 values x (device),
 * s = amax|x| / 448 (1 if every x is 0), q[i] = e4m3 bits of RNE_satfinite(x[i] / s) with the
 * division rounded in fp32.  q: n bytes (device); scale: one fp32 (device, overwritten).
 * Three stream-ordered launches; DF_ERR_INVALID on null pointers. */
df_status df_op_quant_e4m3(df_ctx* ctx, const void* x, uint64_t n, void* q, float* scale, void* stream);
/* out[M,N] = sa * sb * (qa[M,K] . qb[N,K]^T): e4m3 operands (row-major, K contiguous,
 * K % 16 == 0, M and N >= 256), scales sa/sb device fp32 pointers (as df_op_quant_e4m3 writes
 * them), fp32 accumulation on the tensor cores (tcgen05 kind::f8f6f4, CTA pairs), out fp32
 * (out_f32 = 1) or bf16, row stride N.  Device pointers; stream-ordered. */
df_status df_op_gemm_e4m3(df_ctx* ctx, const void* qa, const void* qb, const float* sa, const float* sb, int32_t M,
                          int32_t N, int32_t K, void* out, int32_t out_f32, void* stream);
/* MXFP8 (SURVEY NEXT-4 "MXFP8 block-scaled GEMM"; R30 = OCP Microscaling Formats
 * v1.0, MXFP8 with E4M3 elements): quantise the bf16 matrix x [M, K] (row-major, device,
 * 16-byte aligned, K % 128 == 0) in blocks of 32 consecutive elements of a row:
 * e = floor(log2 max|block|) - 8 clamped to [-127, 127] (-127 for an all-zero block),
 * q[m, k] = e4m3 bits of RNE_satfinite(x[m, k] * 2^-e) (q: M*K bytes, row-major, 16-byte
 * aligned), scale byte e + 127 written to sf in the tiled layout the GEMM loads by TMA:
 * RB = ceil(M / 128) row blocks; the 512-byte atom of (k-group kg = k / 128, row block
 * rb = m / 128) starts at byte (kg * RB + rb) * 512 and holds row m, k-block kb = k / 32 at
 * (m % 32) * 16 + ((m % 128) / 32) * 4 + kb % 4.  sf: (K / 128) * RB * 512 bytes (device;
 * rows [M, 128 RB) get byte 0).  One stream-ordered launch; DF_ERR_INVALID on bad shapes. */
df_status df_op_mx_quant_e4m3(df_ctx* ctx, const void* x, int32_t M, int32_t K, void* q, void* sf, void* stream);
/* out[M,N] = sum_k dec(qa[m,k]) 2^(sa(m,k/32) - 127) * dec(qb[n,k]) 2^(sb(n,k/32) - 127): MXFP8
 * operands as df_op_mx_quant_e4m3 writes them (qa [M,K], qb [N,K] e4m3, sa / sb tiled scale
 * bytes), fp32 accumulation on the tensor cores (tcgen05 kind::mxf8f6f4.block_scale, scale
 * factors staged shared memory -> TMEM by tcgen05.cp, CTA pairs, 256 x 256 tiles), out fp32
 * (out_f32 = 1) or bf16, row stride N.  K % 128 == 0, M and N >= 256.  Device pointers;
 * stream-ordered. */
df_status df_op_gemm_mxf8(df_ctx* ctx, const void* qa, const void* sa, const void* qb, const void* sb, int32_t M,
                          int32_t N, int32_t K, void* out, int32_t out_f32, void* stream);
/* FP8 modes' self-attention (SURVEY NEXT-4 "FP8 ... attention"; R32): q[i] = e4m3 bits of
 * RNE_satfinite(x[i] * inv) for n bf16 values x (device, 16-byte aligned, n % 8 == 0), inv a
 * power of two (the kernels use 1 / s with s = the R32 scale of Q or K); q: n bytes (device). */
df_status df_op_qk_e4m3(df_ctx* ctx, const void* x, uint64_t n, float inv, void* q, void* stream);
/* O[Nq, H*128] = softmax(dec(Q8) dec(K8)^T * scale) V with e4m3 Q8 [H][Nq][128], K8 [H][Nk][128]
 * (head-major bytes; QK^T on the tensor cores as kind::f8f6f4, fp32 S) and bf16 V [H][Nk][128];
 * `scale` carries the two dequantisation scales (s_q s_k / sqrt(dh)).  Device pointers. */
df_status df_op_attention_qf8(df_ctx* ctx, const void* Q8, const void* K8, const void* V, void* O, int32_t H,
                              int32_t Nq, int32_t Nk, float scale, void* stream);
/* DESIGN.md R33: as df_op_attention_qf8 with PV on e4m3 too: V (bf16 [H][Nk][128], device) is
 * quantised per tensor -- s_v = the smallest power of two >= amax|V| / 448, written to vscale[0]
 * (two device floats, zero-initialised before the first call: vscale[1] is an amax accumulator
 * the call leaves zero again) -- and transposed into v8t (e4m3 V^T [H][128][ldv], ldv = Nk rounded up
 * to 64; H * 128 * ldv bytes of device scratch), P is rounded to e4m3 in TMEM and O is scaled
 * by s_v.  Four stream-ordered launches. */
df_status df_op_attention_f8(df_ctx* ctx, const void* Q8, const void* K8, const void* V, void* O, int32_t H,
                             int32_t Nq, int32_t Nk, float scale, void* v8t, float* vscale, void* stream);
/* O[Nq, H*dh] = softmax(Q K^T * scale) V, head-major bf16 Q/K/V [H][N][dh_pad]. */
df_status df_op_attention(df_ctx* ctx, const void* Q, const void* K, const void* V, void* O, int32_t H, int32_t Nq,
                          int32_t Nk, int32_t dh, int32_t dh_pad, float scale, void* stream);
/* out bf16 [M,d] = RMSNorm(x fp32 [M,d]) * (1 + scale) + shift. */
df_status df_op_rmsnorm_mod(df_ctx* ctx, const float* x, void* out, int32_t M, int32_t d, const float* shift,
                            const float* scale, float eps, void* stream);

/* Per-launch timing of the DiT step's kernel classes (bench.py roofline): when
 * enabled, every GEMM / attention / RMSNorm launch of the T instances is bracketed
 * by CUDA events on its own stream (no host sync on the launch path).  Kinds:
 * 0 QKV, 1 self-attn, 2 O-proj, 3 RMSNorm, 4 cross-Q, 5 cross-attn, 6 cross-O,
 * 7 MLP up (SwiGLU), 8 MLP down, 9 head+Euler, 10 patch embed.  enable = n > 1 samples
 * every n-th denoising step (each event pair is a GPU command between two kernels; the
 * unsampled steps run exactly as with profiling off). */
df_status df_profile(df_ctx* ctx, int32_t enable, int32_t reset);
df_status df_kernel_stats(df_ctx* ctx, uint32_t kind, uint64_t* launches, double* total_ms, double* flops,
                          double* bytes);

/* ------------------------------------------------------------------ hybrid instance scheduler
 * Alg. 1 (§sec:hybrid-scheduling): every delta seconds collect per-stage
 * metrics m = {u_s, q_s, d_s}; if the workload changed (modal request key of the recent
 * 25% of the history differs from the rest) apply the predicted ratio (the Eq. 6 planner
 * over measured stage times) and skip the reactive rule; otherwise scale
 * service s out iff u_s > U_high and q_s > Q_high and d_s rises, in iff u_s < U_low and
 * q_s = 0.  Defaults: delta 2 s, U_high 0.8, Q_high 5, U_low 0.2. */
typedef struct { float delta_s, U_high, U_low; uint32_t Q_high; int32_t move_budget; uint32_t G; } df_sched_cfg;
typedef struct { float u[3]; uint32_t q[3]; float d[3]; } df_sched_metrics;
typedef struct {
  double t;                     /* host monotonic seconds                              */
  int32_t action;               /* 0 none, 1 scale-out, 2 scale-in, 3 reconfigure       */
  int32_t stage;                /* for 1/2                                              */
  uint32_t g[3];                /* allocation after the decision                        */
  df_sched_metrics m;
  /* action 4 (re-purpose, logged by df_set_ratio): instance `inst` moved from from_stage
   * to `stage`; drain_ms = time to take it out of routing and let it finish its work,
   * cold_start_ms = time to free its old stage and create the new one (weights regenerated
   * from the weight seed, buffers, worker) -- P:L357 "cold starts" */
  int32_t inst, from_stage;
  float drain_ms, cold_start_ms;
} df_sched_event;
/* Pure functions (no GPU, no context): the Eq. 6 planner (exhaustive; cur/budget limit
 * the L1 instance moves from cur, budget < 0 = unlimited; ties -> fewer GPUs, then
 * larger g_T, then larger g_D), Alg. 1's reactive rule per stage (out[s] in {-1,0,+1};
 * prev NULL = first tick), and the workload-change detector. */
df_status df_plan_ratio(uint32_t G, const double T[3], const uint32_t* cur, int32_t budget, uint32_t out[3]);
df_status df_sched_react(const df_sched_cfg* cfg, const df_sched_metrics* now, const df_sched_metrics* prev,
                         const uint32_t g[3], int32_t out[3]);
int32_t df_sched_changed(const uint32_t* keys, uint32_t n);
/* Controller thread on a live context (single-process). */
df_status df_sched_start(df_ctx* ctx, const df_sched_cfg* cfg);
df_status df_sched_stop(df_ctx* ctx);
df_status df_sched_log(df_ctx* ctx, df_sched_event* out, uint32_t max, uint32_t* n_out);

/* Self-test of the shared-memory metadata ring (no GPU needed): role 0 creates the
 * segment `name` and pushes n records with seq 0..n-1 into instance 0's inbox; role 1
 * attaches and pops n records, returning in *checksum the sum of seq and in *fifo_ok
 * whether they arrived in order.  For the CPU multi-process tests. */
df_status df_ring_selftest(const char* name, int32_t role, uint64_t n, uint64_t* checksum, int32_t* fifo_ok);

/* The chunk plan of a pipeline edge (host logic, no GPU; R22): edge 0 = the E->T
 * payload of `bytes` bytes in whole ctx rows, edge 1 = the fp32 latent in latent blocks, with
 * the graph's chunk_bytes[edge].  Writes up to `max` pieces: chunk k covers `height` rows of
 * `width` bytes starting at byte `off`, rows `pitch` bytes apart (height 1 for byte ranges);
 * *n = the chunk count.  DF_ERR_INVALID on a null argument or an edge other than 0 / 1. */
df_status df_chunk_plan(const df_graph* g, uint32_t edge, uint64_t bytes, uint32_t* n, uint64_t* off,
                        uint64_t* width, uint64_t* height, uint64_t* pitch, uint32_t max);

/* Number of kernel launches this context issued so far (bench "gpu_launches"). */
uint64_t df_launch_count(const df_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DF_H_ */
