#include <chrono>
#include <thread>
// HBM-bound kernels of the DiT step and the request prologue, plus parameter init
// (Philox4x32-10) and the E/D stand-in stages.
//
// rmsnorm_mod (cross pre-norm): one CTA per row, 16-byte loads,
// warp-shuffle + smem reduction, fp32 statistics, bf16 (or fp32) store.  Algorithmic
// traffic per row: 4d bytes read + 2d bytes written (bf16 out).
#include <cmath>
#include "kernels.h"
#include <cuda_fp8.h>

#include <atomic>
#include <mutex>

namespace df {

// ------------------------------------------------------------------ Philox4x32-10
struct U4 {
  uint32_t x, y, z, w;
};
DF_DEV U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return {c0, c1, c2, c3};
}
DF_DEV uint32_t philox_word(uint64_t seed, uint64_t i, uint32_t c2, uint32_t c3) {
  uint64_t b = i >> 2;
  U4 o = philox(uint32_t(b), uint32_t(b >> 32), c2, c3, uint32_t(seed), uint32_t(seed >> 32));
  switch (i & 3) {
    case 0: return o.x;
    case 1: return o.y;
    case 2: return o.z;
    default: return o.w;
  }
}

__global__ void init_tensor_kernel(bf16* __restrict__ dst, InitSpec s, size_t n) {
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < n; t += size_t(gridDim.x) * blockDim.x) {
    // t enumerates destination elements in the order of the destination layout
    size_t k, nn;  // logical (in, out) index
    size_t dst_idx;
    if (s.layout == 0) {
      k = t / s.out;
      nn = t % s.out;
      dst_idx = k * s.ld + nn;
    } else {
      nn = t / s.in;  // destination row order (logical output index)
      k = t % s.in;
      size_t row;
      if (s.layout == 1) row = s.row_off + nn;
      else row = (nn / 16) * 32 + size_t(s.row_off) * 16 + (nn % 16);
      dst_idx = row * s.ld + k;
    }
    uint64_t i = uint64_t(k) * s.out + nn;  // logical row-major index
    uint32_t u = philox_word(s.seed, i, s.tid, 0);
    float r = float(u >> 8) * 5.9604644775390625e-08f;  // 2^-24, exact
    float w = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, r), 1.0f), s.a);
    if (s.kind == 1) w = __fadd_rn(1.0f, w);
    dst[dst_idx] = __float2bfloat16_rn(w);
  }
}

cudaError_t init_tensor(bf16* dst, const InitSpec& s, cudaStream_t st) {
  size_t n = size_t(s.in) * s.out;
  if (!n) return cudaSuccess;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  init_tensor_kernel<<<unsigned(blocks), 256, 0, st>>>(dst, s, n);
  return cudaGetLastError();
}

__global__ void noise_kernel(float* __restrict__ x, size_t n, uint64_t seed) {
  for (size_t j = blockIdx.x * size_t(blockDim.x) + threadIdx.x; j < n; j += size_t(gridDim.x) * blockDim.x) {
    uint64_t blk = j >> 1;
    U4 o = philox(uint32_t(blk), uint32_t(blk >> 32), 0, 1, uint32_t(seed), uint32_t(seed >> 32));
    uint32_t a = (j & 1) ? o.z : o.x;
    uint32_t b = (j & 1) ? o.w : o.y;
    double u1 = (double(a) + 1.0) * 2.3283064365386963e-10;
    double u2 = double(b) * 2.3283064365386963e-10;
    double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    x[j] = float(z);
  }
}
cudaError_t gen_noise(float* x, size_t n, uint64_t seed, cudaStream_t st) {
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  noise_kernel<<<unsigned(blocks), 256, 0, st>>>(x, n, seed);
  return cudaGetLastError();
}

__global__ void tokens_kernel(int32_t* ids, int n, int vocab, uint64_t seed, uint32_t c3) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) ids[j] = int32_t(philox_word(seed, j, 0, c3) % uint32_t(vocab));
}
// stream c3 = 2: prompt tokens; c3 = 4: negative-prompt tokens
// I2V E stand-in (R27): clip [L_img, d_img] bf16 from stream (seed; 0, 5) and
// y [C_y, F, H, W] fp32 (mask channels 0..3 = 1 on frame 0; channels 4.. of frame 0 from
// stream (seed; 0, 6)), each value fp32((2r - 1) * fp32(sqrt 3)) with r = (u >> 8) 2^-24
DF_DEV float unit_uniform(uint32_t u) {
  const float r = float(u >> 8) * 5.9604644775390625e-08f;  // 2^-24, exact
  return __fmul_rn(__fsub_rn(__fmul_rn(2.0f, r), 1.0f), 1.7320508075688772f);
}
__global__ void image_cond_kernel(uint64_t seed, bf16* clip, size_t n_clip, float* y, int Cy, int F, int H, int W) {
  const size_t hw = size_t(H) * W, n_y = size_t(Cy) * F * hw;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_clip + n_y; i += size_t(gridDim.x) * blockDim.x) {
    if (i < n_clip) {
      clip[i] = __float2bfloat16_rn(unit_uniform(philox_word(seed, i, 0, 5)));
    } else {
      const size_t j = i - n_clip;
      const size_t c = j / (size_t(F) * hw), rem = j - c * size_t(F) * hw, f = rem / hw, p = rem - f * hw;
      float v = 0.f;
      if (f == 0) v = c < 4 ? 1.f : unit_uniform(philox_word(seed, (c - 4) * hw + p, 0, 6));
      y[j] = v;
    }
  }
}
cudaError_t gen_image_cond(uint64_t seed, bf16* clip, size_t n_clip, float* y, int Cy, int F, int H, int W,
                           cudaStream_t st) {
  const size_t n = n_clip + size_t(Cy) * F * H * W;
  unsigned blocks = unsigned((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  image_cond_kernel<<<blocks, 256, 0, st>>>(seed, clip, n_clip, y, Cy, F, H, W);
  return cudaGetLastError();
}

cudaError_t gen_tokens(int32_t* ids, int n, int vocab, uint64_t seed, cudaStream_t st, uint32_t stream_c3) {
  tokens_kernel<<<(n + 255) / 256, 256, 0, st>>>(ids, n, vocab, seed, stream_c3);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ RMSNorm (+ modulation)
template <typename OutT>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x, OutT* __restrict__ out, int d,
                                                      const float* __restrict__ shift, const float* __restrict__ scale,
                                                      const bf16* __restrict__ gain, float eps) {
  // one CTA per row; each thread holds up to 8 float4 (d <= 8192)
  pdl_wait();
  pdl_launch_dependents();
  const int row = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * d);
  const int nv = d / 4;
  float4 v[8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int c = threadIdx.x + i * 256;
    if (c < nv) {
      v[i] = xr[c];
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  }
  __shared__ float red[8];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float inv = rsqrtf(tot / float(d) + eps);
  OutT* orow = out + size_t(row) * d;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int c = threadIdx.x + i * 256;
    if (c < nv) {
      float y[4] = {v[i].x * inv, v[i].y * inv, v[i].z * inv, v[i].w * inv};
      int n0 = 4 * c;
      if (gain) {
#pragma unroll
        for (int q = 0; q < 4; ++q) y[q] *= bf2f(gain[n0 + q]);
      } else {
        float4 sc = reinterpret_cast<const float4*>(scale)[c];
        float4 sh = reinterpret_cast<const float4*>(shift)[c];
        y[0] = y[0] * (1.f + sc.x) + sh.x;
        y[1] = y[1] * (1.f + sc.y) + sh.y;
        y[2] = y[2] * (1.f + sc.z) + sh.z;
        y[3] = y[3] * (1.f + sc.w) + sh.w;
      }
      if constexpr (sizeof(OutT) == 2) {
        uint2 u;
        u.x = pack_bf16x2(y[0], y[1]);
        u.y = pack_bf16x2(y[2], y[3]);
        *reinterpret_cast<uint2*>(orow + n0) = u;
      } else {
        *reinterpret_cast<float4*>(orow + n0) = make_float4(y[0], y[1], y[2], y[3]);
      }
    }
  }
}

// One warp per row (d = 128 * VPT): every lane has VPT independent 16-byte loads in flight
// and the reduction is warp shuffles only. The second pass re-reads x (L1 / L2 hits) rather
// than holding the row in registers: at 24 float4 per lane the kernel needed 148 registers,
// 3 CTAs (12 warps) per SM, and sat at 2.5 TB/s; without the row in registers every CTA of
// the grid is resident at once.  Rows of <= 8 float4 per lane stay in registers.
template <int VPT, typename OutT>
__global__ void __launch_bounds__(128, 8) rmsnorm_warp_kernel(const float* __restrict__ x, OutT* __restrict__ out, int M,
                                                           const float* __restrict__ shift,
                                                           const float* __restrict__ scale,
                                                           const bf16* __restrict__ gain, float eps) {
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (row >= M) return;
  constexpr int d = 128 * VPT;
  constexpr bool KEEP = VPT <= 8;
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * d);
  float4 v[KEEP ? VPT : 1];
  float ss = 0.f;
  if constexpr (KEEP) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      v[i] = xr[lane + 32 * i];
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  } else {
    // 8 independent 16-byte loads in flight per lane and chunk
#pragma unroll 1
    for (int b = 0; b < VPT; b += 8) {
      float4 t[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = (b + i < VPT) ? xr[lane + 32 * (b + i)] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += t[i].x * t[i].x + t[i].y * t[i].y + t[i].z * t[i].z + t[i].w * t[i].w;
    }
  }
  ss = warp_sum(ss);
  const float inv = rsqrtf(ss / float(d) + eps);
  OutT* orow = out + size_t(row) * d;
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    const int c = lane + 32 * i;
    float4 t;
    if constexpr (KEEP) t = v[i];
    else t = xr[c];
    float y[4] = {t.x * inv, t.y * inv, t.z * inv, t.w * inv};
    if (gain) {
      const uint2 g = reinterpret_cast<const uint2*>(gain)[c];
      y[0] *= bf_lo(g.x), y[1] *= bf_hi(g.x), y[2] *= bf_lo(g.y), y[3] *= bf_hi(g.y);
    } else {
      const float4 sc = reinterpret_cast<const float4*>(scale)[c];
      const float4 sh = reinterpret_cast<const float4*>(shift)[c];
      y[0] = y[0] * (1.f + sc.x) + sh.x;
      y[1] = y[1] * (1.f + sc.y) + sh.y;
      y[2] = y[2] * (1.f + sc.z) + sh.z;
      y[3] = y[3] * (1.f + sc.w) + sh.w;
    }
    if constexpr (sizeof(OutT) == 2) {
      uint2 u;
      u.x = pack_bf16x2(y[0], y[1]);
      u.y = pack_bf16x2(y[2], y[3]);
      reinterpret_cast<uint2*>(orow)[c] = u;
    } else {
      reinterpret_cast<float4*>(orow)[c] = make_float4(y[0], y[1], y[2], y[3]);
    }
  }
}

// Bulk-copy variant: one elected thread moves the CTA's 4 rows of x into shared memory with
// cp.async.bulk (one mbarrier, no per-thread load instructions in flight), then each warp
// reduces and normalises its row from shared memory.  DF_RMS_IMPL=2 selects it (A/B).
DF_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
template <int VPT, typename OutT>
__global__ void __launch_bounds__(128) rmsnorm_bulk_kernel(const float* __restrict__ x, OutT* __restrict__ out, int M,
                                                          const float* __restrict__ shift,
                                                          const float* __restrict__ scale,
                                                          const bf16* __restrict__ gain, float eps) {
  constexpr int d = 128 * VPT;
  extern __shared__ __align__(128) uint8_t sm[];
  float4* rows = reinterpret_cast<float4*>(sm + 16);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row0 = blockIdx.x * 4;
  const int nrows = min(4, M - row0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, uint32_t(nrows) * d * 4);
    for (int r = 0; r < nrows; ++r) bulk_g2s(rows + r * (d / 4), x + size_t(row0 + r) * d, d * 4, bar);
  }
  __syncthreads();
  if (w >= nrows) return;
  mbar_wait(bar, 0);
  const float4* xr = rows + w * (d / 4);
  float ss = 0.f;
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    const float4 t = xr[lane + 32 * i];
    ss += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
  }
  ss = warp_sum(ss);
  const float inv = rsqrtf(ss / float(d) + eps);
  OutT* orow = out + size_t(row0 + w) * d;
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    const int c = lane + 32 * i;
    const float4 t = xr[c];
    float y[4] = {t.x * inv, t.y * inv, t.z * inv, t.w * inv};
    if (gain) {
      const uint2 g = reinterpret_cast<const uint2*>(gain)[c];
      y[0] *= bf_lo(g.x), y[1] *= bf_hi(g.x), y[2] *= bf_lo(g.y), y[3] *= bf_hi(g.y);
    } else {
      const float4 sc = reinterpret_cast<const float4*>(scale)[c];
      const float4 sh = reinterpret_cast<const float4*>(shift)[c];
      y[0] = y[0] * (1.f + sc.x) + sh.x;
      y[1] = y[1] * (1.f + sc.y) + sh.y;
      y[2] = y[2] * (1.f + sc.z) + sh.z;
      y[3] = y[3] * (1.f + sc.w) + sh.w;
    }
    if constexpr (sizeof(OutT) == 2) {
      uint2 u;
      u.x = pack_bf16x2(y[0], y[1]);
      u.y = pack_bf16x2(y[2], y[3]);
      reinterpret_cast<uint2*>(orow)[c] = u;
    } else {
      reinterpret_cast<float4*>(orow)[c] = make_float4(y[0], y[1], y[2], y[3]);
    }
  }
}

// Persistent streaming variant (the model widths, default): one CTA per SM loops over rows
// r = blockIdx.x + k * gridDim.x.  A producer thread keeps a ring of STAGES rows in shared
// memory filled with one cp.async.bulk per row (mbarrier complete_tx), so every SM always has
// ~STAGES x row bytes of HBM reads in flight; consumer warp w normalises the rows k = w mod NW
// of its CTA from shared memory (two passes over the row: sum of squares, then scale), writes
// the bf16/fp32 row with coalesced stores and hands the stage back.  The one-row-per-warp
// kernel above issues a row's loads, waits, then writes: with the whole grid resident in one
// wave its read and write phases do not overlap and its launch tail is exposed (3.9 TB/s in
// the image step).
constexpr int RMS_NW = 8;  // consumer warps per CTA
template <int VPT>
struct RmsStream {
  static constexpr int ROW = 128 * VPT * 4;                  // bytes of one fp32 row
  static constexpr int STAGES = (200 * 1024) / ROW < 16 ? (200 * 1024) / ROW : 16;
  static constexpr int OFF_BAR = STAGES * ROW;
  static constexpr int SMEM = OFF_BAR + 2 * STAGES * 8 + 128;
};

template <int VPT, typename OutT>
__global__ void __launch_bounds__(32 * (RMS_NW + 1), 1)
    rmsnorm_stream_kernel(const float* __restrict__ x, OutT* __restrict__ out, int M, const float* __restrict__ shift,
                          const float* __restrict__ scale, const bf16* __restrict__ gain, float eps) {
  using Cfg = RmsStream<VPT>;
  constexpr int d = 128 * VPT;
  extern __shared__ __align__(128) uint8_t sm[];
  float4* ring = reinterpret_cast<float4*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + Cfg::OFF_BAR);
  uint64_t* empty = full + Cfg::STAGES;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const int nk = M > int(blockIdx.x) ? (M - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x) : 0;
  if (w == RMS_NW) {  // producer
    if (lane == 0) {
      for (int k = 0; k < nk; ++k) {
        const int s = k % Cfg::STAGES;
        mbar_wait(&empty[s], ((k / Cfg::STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], Cfg::ROW);
        bulk_g2s(ring + size_t(s) * (d / 4), x + (size_t(blockIdx.x) + size_t(k) * gridDim.x) * d, Cfg::ROW, &full[s]);
      }
    }
    return;
  }
  for (int k = w; k < nk; k += RMS_NW) {
    const int s = k % Cfg::STAGES;
    mbar_wait(&full[s], (k / Cfg::STAGES) & 1);
    const float4* xr = ring + size_t(s) * (d / 4);
    float ss = 0.f;
#pragma unroll 8
    for (int i = 0; i < VPT; ++i) {
      const float4 t = xr[lane + 32 * i];
      ss += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / float(d) + eps);
    OutT* orow = out + (size_t(blockIdx.x) + size_t(k) * gridDim.x) * d;
#pragma unroll 8
    for (int i = 0; i < VPT; ++i) {
      const int c = lane + 32 * i;
      const float4 t = xr[c];
      float y[4] = {t.x * inv, t.y * inv, t.z * inv, t.w * inv};
      if (gain) {
        const uint2 g = reinterpret_cast<const uint2*>(gain)[c];
        y[0] *= bf_lo(g.x), y[1] *= bf_hi(g.x), y[2] *= bf_lo(g.y), y[3] *= bf_hi(g.y);
      } else {
        const float4 sc = reinterpret_cast<const float4*>(scale)[c];
        const float4 sh = reinterpret_cast<const float4*>(shift)[c];
        y[0] = y[0] * (1.f + sc.x) + sh.x;
        y[1] = y[1] * (1.f + sc.y) + sh.y;
        y[2] = y[2] * (1.f + sc.z) + sh.z;
        y[3] = y[3] * (1.f + sc.w) + sh.w;
      }
      if constexpr (sizeof(OutT) == 2) {
        uint2 u;
        u.x = pack_bf16x2(y[0], y[1]);
        u.y = pack_bf16x2(y[2], y[3]);
        reinterpret_cast<uint2*>(orow)[c] = u;
      } else {
        reinterpret_cast<float4*>(orow)[c] = make_float4(y[0], y[1], y[2], y[3]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp's reads of the stage are done
  }
}

template <int VPT>
static cudaError_t launch_rms_warp(const float* x, void* out, int out_f32, int M, const float* shift,
                                   const float* scale, const bf16* gain, float eps, cudaStream_t st) {
  void* args[] = {(void*)&x, (void*)&out, (void*)&M, (void*)&shift, (void*)&scale, (void*)&gain, (void*)&eps};
  dim3 grid((M + 3) / 4);
  // DF_RMS_IMPL (A/B): 0 auto (default), 1 warp per row, 2 bulk per CTA, 3 streaming.  Auto
  // streams when every SM has >= 64 rows to stream (video: 161 vs 217 us standalone at
  // 32760 x 5120); at the image shape (28 rows per SM) the one-wave warp-per-row kernel reads
  // the residual the previous GEMM epilogue just left in L2 and is as fast in the step
  // (DESIGN.md §12).
  static const int impl = [] {
    const char* e = getenv("DF_RMS_IMPL");
    return e ? atoi(e) : 0;
  }();
  const int bulk = impl == 2;
  if ((impl == 3 || (impl == 0 && M >= 64 * num_sms())) && VPT >= 16) {
    using Cfg = RmsStream<VPT>;
    const void* kern =
        out_f32 ? (const void*)rmsnorm_stream_kernel<VPT, float> : (const void*)rmsnorm_stream_kernel<VPT, bf16>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute((const void*)rmsnorm_stream_kernel<VPT, float>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)rmsnorm_stream_kernel<VPT, bf16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    const int g = M < num_sms() ? M : num_sms();
    return launch_ex(kern, dim3(g), dim3(32 * (RMS_NW + 1)), Cfg::SMEM, st, args);
  }
  if (bulk) {
    const size_t smem = 16 + size_t(4) * 128 * VPT * 4;
    const void* kern = out_f32 ? (const void*)rmsnorm_bulk_kernel<VPT, float> : (const void*)rmsnorm_bulk_kernel<VPT, bf16>;
    static bool attr = false;
    if (!attr) {  // both output types
      cudaError_t e = cudaFuncSetAttribute((const void*)rmsnorm_bulk_kernel<VPT, float>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)rmsnorm_bulk_kernel<VPT, bf16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      attr = true;
    }
    return launch_ex(kern, grid, dim3(128), smem, st, args);
  }
  if (out_f32) return launch_ex((const void*)rmsnorm_warp_kernel<VPT, float>, grid, dim3(128), 0, st, args);
  return launch_ex((const void*)rmsnorm_warp_kernel<VPT, bf16>, grid, dim3(128), 0, st, args);
}

cudaError_t rmsnorm_mod(const float* x, void* out, int out_f32, int M, int d, const float* shift, const float* scale,
                        const bf16* gain, float eps, cudaStream_t st) {
  if (d % 4 || d > 8192) return cudaErrorInvalidValue;
  if (M <= 0) return cudaSuccess;
  switch (d) {  // the model widths (mid, image, text encoder, video)
    case 256: return launch_rms_warp<2>(x, out, out_f32, M, shift, scale, gain, eps, st);
    case 3072: return launch_rms_warp<24>(x, out, out_f32, M, shift, scale, gain, eps, st);
    case 4096: return launch_rms_warp<32>(x, out, out_f32, M, shift, scale, gain, eps, st);
    case 5120: return launch_rms_warp<40>(x, out, out_f32, M, shift, scale, gain, eps, st);
    default: break;
  }
  void* args[] = {(void*)&x, (void*)&out, (void*)&d, (void*)&shift, (void*)&scale, (void*)&gain, (void*)&eps};
  if (out_f32) return launch_ex((const void*)rmsnorm_kernel<float>, dim3(M), dim3(256), 0, st, args);
  return launch_ex((const void*)rmsnorm_kernel<bf16>, dim3(M), dim3(256), 0, st, args);
}

// ------------------------------------------------------------------ patchify
// I2V: channels c >= C come from y (concat(x, y) along channels, Wan's in_dim = C + C_y)
template <typename OutT>
__global__ void patchify_kernel(const float* __restrict__ x, const float* __restrict__ y, int Cy, OutT* __restrict__ X,
                                int C, int F, int H, int W, int pt, int ph, int pw, size_t total) {
  const int P = (C + Cy) * pt * ph * pw;
  const int Hp = H / ph, Wp = W / pw;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total; t += size_t(gridDim.x) * blockDim.x) {
    int p = int(t % P);
    size_t n = t / P;
    int ww = int(n % Wp), hh = int((n / Wp) % Hp), f = int(n / (size_t(Wp) * Hp));
    int k = p % pw, r = p / pw;
    int j = r % ph;
    r /= ph;
    int i = r % pt;
    int c = r / pt;
    const size_t sp = (size_t(f * pt + i) * H + hh * ph + j) * W + ww * pw + k;
    const float v = c < C ? x[size_t(c) * F * H * W + sp] : y[size_t(c - C) * F * H * W + sp];
    store_val<OutT>(X + t, v);
  }
}
cudaError_t patchify(const float* x, const float* y, int Cy, void* X, int out_f32, int C, int F, int H, int W, int pt,
                     int ph, int pw, cudaStream_t st) {
  if (Cy > 0 && !y) return cudaErrorInvalidValue;
  size_t total = size_t(C + (Cy > 0 ? Cy : 0)) * F * H * W;
  const int cy = Cy > 0 ? Cy : 0;
  unsigned blocks = unsigned((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (out_f32) patchify_kernel<float><<<blocks, 256, 0, st>>>(x, y, cy, (float*)X, C, F, H, W, pt, ph, pw, total);
  else patchify_kernel<bf16><<<blocks, 256, 0, st>>>(x, y, cy, (bf16*)X, C, F, H, W, pt, ph, pw, total);
  return cudaGetLastError();
}

// o += oi elementwise (I2V: text + image cross-attention outputs), in the activation dtype
template <typename T>
__global__ void add_into_kernel(T* __restrict__ o, const T* __restrict__ oi, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float v = load_val(o + i) + load_val(oi + i);
    store_val<T>(o + i, v);
  }
}
cudaError_t add_into(void* o, const void* oi, size_t n, int f32, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  unsigned blocks = unsigned((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (f32) add_into_kernel<float><<<blocks, 256, 0, st>>>((float*)o, (const float*)oi, n);
  else add_into_kernel<bf16><<<blocks, 256, 0, st>>>((bf16*)o, (const bf16*)oi, n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ time conditioning
__global__ void sigma_kernel(float* sig, int S, float shift) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > S) return;
  const double si = 1.0 - double(i) / double(S);
  sig[i] = float(double(shift) * si / (1.0 + (double(shift) - 1.0) * si));
}
cudaError_t sigma_schedule(float* sig, int S, float shift, cudaStream_t st) {
  sigma_kernel<<<(S + 1 + 127) / 128, 128, 0, st>>>(sig, S, shift);
  return cudaGetLastError();
}

__global__ void sinusoid_kernel(const float* sig, float* s, int S, int freq_dim) {
  int i = blockIdx.x;
  int half = freq_dim / 2;
  for (int k = threadIdx.x; k < half; k += blockDim.x) {
    double t = 1000.0 * double(sig[i]);
    double w = pow(10000.0, -double(k) / double(half));
    s[size_t(i) * freq_dim + k] = float(cos(t * w));
    s[size_t(i) * freq_dim + half + k] = float(sin(t * w));
  }
}
cudaError_t sinusoid(const float* sig_dev, float* s, int S, int freq_dim, cudaStream_t st) {
  if (S <= 0) return cudaSuccess;
  sinusoid_kernel<<<S, 128, 0, st>>>(sig_dev, s, S, freq_dim);
  return cudaGetLastError();
}

struct ModPtrs {
  const bf16* p[64];
};
__global__ void modulations_kernel(const float* __restrict__ e6, const float* __restrict__ e, ModPtrs mp, int l0,
                                   int nl, const bf16* __restrict__ head_mod, int d, float* __restrict__ mods,
                                   float* __restrict__ head) {
  int l = blockIdx.y;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 6 * d; t += gridDim.x * blockDim.x) {
    if (l < nl) mods[size_t(l0 + l) * 6 * d + t] = e6[t] + bf2f(mp.p[l][t]);
    if (l == 0 && t < 2 * d && head) head[t] = bf2f(head_mod[t]) + e[t % d];
  }
}
cudaError_t modulations(const float* e6, const float* e, const bf16* const* layer_mod, int layers,
                        const bf16* head_mod, int d, float* mods, float* head, cudaStream_t st) {
  for (int l0 = 0; l0 < layers; l0 += 64) {
    ModPtrs mp;
    int nl = layers - l0 < 64 ? layers - l0 : 64;
    for (int i = 0; i < nl; ++i) mp.p[i] = layer_mod[l0 + i];
    dim3 grid((6 * d + 255) / 256, nl);
    modulations_kernel<<<grid, 256, 0, st>>>(e6, e, mp, l0, nl, head_mod, d, mods, l0 == 0 ? head : nullptr);
  }
  return cudaGetLastError();
}

__global__ void cfg_euler_kernel(float* __restrict__ x, const float* __restrict__ vb, float* __restrict__ v_out,
                                 size_t n, float g, float dsig) {
  pdl_wait();
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float vc = vb[i], vu = vb[n + i];
    const float v = vu + g * (vc - vu);  // classifier-free guidance (NEXT-2)
    if (v_out) v_out[i] = v;
    x[i] += dsig * v;
  }
}
cudaError_t cfg_euler(float* x, const float* v_batch, float* v_out, size_t n, float guidance, float dsig,
                      cudaStream_t st) {
  unsigned b = unsigned((n + 255) / 256);
  if (b > 148 * 8) b = 148 * 8;
  void* args[] = {(void*)&x, (void*)&v_batch, (void*)&v_out, (void*)&n, (void*)&guidance, (void*)&dsig};
  return launch_ex((const void*)cfg_euler_kernel, dim3(b), dim3(256), 0, st, args);
}

__global__ void silu_kernel(float* x, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    x[i] = x[i] / (1.0f + expf(-x[i]));
}
cudaError_t silu_inplace(float* x, size_t n, cudaStream_t st) {
  unsigned b = unsigned((n + 255) / 256);
  if (b > 4096) b = 4096;
  if (n) silu_kernel<<<b, 256, 0, st>>>(x, n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ E stand-in pieces
__global__ void embed_kernel(const int32_t* ids, const bf16* emb, float* z, int L, int dt) {
  int j = blockIdx.x;
  const bf16* er = emb + size_t(ids[j]) * dt;
  for (int c = threadIdx.x; c < dt; c += blockDim.x) z[size_t(j) * dt + c] = bf2f(er[c]);
}
cudaError_t embed_rows(const int32_t* ids, const bf16* emb, float* z, int L, int dt, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  embed_kernel<<<L, 256, 0, st>>>(ids, emb, z, L, dt);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ D stand-in
// One CTA per (latent frame, 8 latent pixels): u = SiLU(x W1 + b1) in smem, then
// o = tanh(u W2 + b2) scattered by the pixel shuffle.
// One CTA per 8 latent pixels of one latent frame; the launch covers frames [f0, f0 + gridDim.y)
// and pixels [p_begin, p_end) of each (a T->D chunk when D decodes chunk by chunk).
__global__ void decode_kernel(const float* __restrict__ x, float* __restrict__ out, int C, int F, int H, int W,
                              int cdec, const bf16* __restrict__ w1, const bf16* __restrict__ b1,
                              const bf16* __restrict__ w2f, const bf16* __restrict__ b2f,
                              const bf16* __restrict__ w2r, const bf16* __restrict__ b2r, int f0, int p_begin,
                              int p_end) {
  extern __shared__ float sh[];  // [8][cdec]
  const int phi = f0 + blockIdx.y;
  const int pix0 = p_begin + blockIdx.x * 8;
  const int HW = H * W;
  const int npix = min(8, p_end - pix0);
  for (int t = threadIdx.x; t < 8 * cdec; t += blockDim.x) {
    int q = t / cdec, u = t % cdec;
    float acc = 0.f;
    if (q < npix) {
      int pix = pix0 + q;
      acc = bf2f(b1[u]);
      for (int c = 0; c < C; ++c) acc += x[(size_t(c) * F + phi) * HW + pix] * bf2f(w1[size_t(c) * cdec + u]);
      acc = acc / (1.0f + expf(-acc));
    }
    sh[q * cdec + u] = acc;
  }
  __syncthreads();
  const int r = phi == 0 ? 1 : 4;
  const int nout = 3 * r * 64;
  const bf16* w2 = phi == 0 ? w2f : w2r;
  const bf16* b2 = phi == 0 ? b2f : b2r;
  const int T = 1 + 4 * (F - 1);
  for (int t = threadIdx.x; t < npix * nout; t += blockDim.x) {
    int q = t / nout, idx = t % nout;
    float acc = bf2f(b2[idx]);
    const float* u = sh + q * cdec;
    for (int k = 0; k < cdec; ++k) acc += u[k] * bf2f(w2[size_t(k) * nout + idx]);
    float o = tanhf(acc);
    int dx = idx & 7, dy = (idx >> 3) & 7, rest = idx >> 6;
    int tau = rest % r, ch = rest / r;
    int tf = phi == 0 ? 0 : 4 * phi - 3 + tau;
    int pix = pix0 + q, y = pix / W, xx = pix % W;
    out[((size_t(ch) * T + tf) * (8 * H) + 8 * y + dy) * (8 * W) + 8 * xx + dx] = o;
  }
}
cudaError_t decode_latent(const float* x, float* out, int C, int F, int H, int W, int cdec, const bf16* w1,
                          const bf16* b1, const bf16* w2f, const bf16* b2f, const bf16* w2r, const bf16* b2r,
                          cudaStream_t st) {
  return decode_latent_region(x, out, C, F, H, W, cdec, w1, b1, w2f, b2f, w2r, b2r, 0, F, 0, H * W, st);
}
cudaError_t decode_latent_region(const float* x, float* out, int C, int F, int H, int W, int cdec, const bf16* w1,
                                 const bf16* b1, const bf16* w2f, const bf16* b2f, const bf16* w2r, const bf16* b2r,
                                 int f0, int nf, int p_begin, int p_end, cudaStream_t st) {
  if (nf <= 0 || p_end <= p_begin) return cudaSuccess;
  dim3 grid((p_end - p_begin + 7) / 8, nf);
  decode_kernel<<<grid, 256, 8 * cdec * sizeof(float), st>>>(x, out, C, F, H, W, cdec, w1, b1, w2f, b2f, w2r, b2r,
                                                             f0, p_begin, p_end);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ handoff hash
DF_DEV unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// acc[0] = running sum, acc[1] = arrival counter; both back to 0 when the kernel ends, so a
// slot is reusable by the next hash on any stream once this one finished.
__global__ void hash_kernel(const uint8_t* __restrict__ buf, size_t nbytes, size_t word_off,
                            unsigned long long* acc, unsigned long long* out) {
  size_t nw = (nbytes + 7) / 8;
  unsigned long long h = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nw; i += size_t(gridDim.x) * blockDim.x) {
    unsigned long long w = 0;
    size_t b0 = i * 8;
    if (b0 + 8 <= nbytes && (reinterpret_cast<uintptr_t>(buf) & 7) == 0) {
      w = *reinterpret_cast<const unsigned long long*>(buf + b0);
    } else {
      for (int k = 0; k < 8; ++k)
        if (b0 + k < nbytes) w |= (unsigned long long)buf[b0 + k] << (8 * k);
    }
    h += splitmix64(w ^ ((word_off + i) * 0x9E3779B97F4A7C15ull));
  }
  // sum mod 2^64 is order-independent: warp reduce, one device atomic per warp; the last
  // block to arrive publishes the total with one store (out may be host-mapped memory)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, h);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(acc + 1, 1ull) == gridDim.x - 1) {
      __threadfence();
      *out = atomicExch(acc, 0ull);
      acc[1] = 0;
    }
  }
}

// Per-device pool of accumulator slots (zeroed once; every hash returns its slot zeroed).
// Slots are handed out round robin: up to kHashSlots hashes may be in flight per device.
static constexpr int kHashSlots = 1024;
static unsigned long long* hash_slots(int dev) {
  static std::mutex mu;
  static unsigned long long* pool[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!pool[dev]) {
    void* p = nullptr;
    if (cudaMalloc(&p, kHashSlots * 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, kHashSlots * 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
    pool[dev] = static_cast<unsigned long long*>(p);
  }
  return pool[dev];
}

cudaError_t payload_hash(const void* buf, size_t nbytes, size_t word_offset, unsigned long long* out,
                         cudaStream_t st) {
  size_t nw = (nbytes + 7) / 8;
  unsigned blocks = unsigned((nw + 255) / 256);
  if (blocks > 296) blocks = 296;
  if (!blocks) return cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  unsigned long long* pool = hash_slots(dev);
  if (!pool) return cudaErrorMemoryAllocation;
  static std::atomic<unsigned> next{0};
  unsigned long long* acc = pool + 2 * (next.fetch_add(1) % kHashSlots);
  hash_kernel<<<blocks, 256, 0, st>>>((const uint8_t*)buf, nbytes, word_offset, acc, out);
  return cudaGetLastError();
}

// Injected transfer delay (P:L142 jitter, R23): a host function on the comm stream, so the
// delay holds back the stream's later copies without occupying an SM (a spinning 1-thread
// kernel had pinned one SM for the whole delay and stalled the persistent kernels' last pair).
static void CUDART_CB delay_host_fn(void* p) {
  std::this_thread::sleep_for(std::chrono::nanoseconds(reinterpret_cast<uintptr_t>(p)));
}
cudaError_t delay_ns(uint64_t ns, cudaStream_t st) {
  if (ns == 0) return cudaSuccess;
  return cudaLaunchHostFunc(st, delay_host_fn, reinterpret_cast<void*>(uintptr_t(ns)));
}

// ---------------------------------------------------------------- e4m3 quantiser (NEXT-4)
// Per-tensor current scaling (R28): s = amax|x| / 448 (1 when x == 0) and
// q = RNE_satfinite_e4m3(x / s), the division correctly rounded in fp32, so x ~= s * q.
// Three stream-ordered launches: amax (one atomicMax per warp on the float bits -- valid for
// non-negative floats), the scale (one thread, in place), the quantisation (8 per thread).
__global__ void __launch_bounds__(256) e4m3_amax_kernel(const bf16* __restrict__ x, size_t n, unsigned* amax) {
  pdl_wait();
  pdl_launch_dependents();
  float m = 0.f;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const size_t n8 = (reinterpret_cast<uintptr_t>(x) & 15) ? 0 : n / 8;
  auto acc = [&](const uint4 u) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      m = fmaxf(m, fabsf(__uint_as_float(w[k] << 16)));
      m = fmaxf(m, fabsf(__uint_as_float(w[k] & 0xFFFF0000u)));
    }
  };
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n8; i += 4 * stride) {  // four 16-byte loads in flight per thread
    const uint4 u0 = __ldg(xv + i), u1 = __ldg(xv + i + stride), u2 = __ldg(xv + i + 2 * stride),
                u3 = __ldg(xv + i + 3 * stride);
    acc(u0), acc(u1), acc(u2), acc(u3);
  }
  for (; i < n8; i += stride) acc(__ldg(xv + i));
  for (size_t i = n8 * 8 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    m = fmaxf(m, fabsf(bf2f(x[i])));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[8];  // block max, then one atomic per block
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmaxf(m, wm[w]);
    if (m > 0.f) atomicMax(amax, __float_as_uint(m));
  }
}
__global__ void e4m3_scale_kernel(float* s) {
  const float a = __uint_as_float(*reinterpret_cast<const unsigned*>(s));
  *s = a > 0.f ? __fdiv_rn(a, 448.f) : 1.f;
}
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d, float s) {
  const uint32_t q0 = __nv_cvt_float_to_fp8(__fdiv_rn(a, s), __NV_SATFINITE, __NV_E4M3);
  const uint32_t q1 = __nv_cvt_float_to_fp8(__fdiv_rn(b, s), __NV_SATFINITE, __NV_E4M3);
  const uint32_t q2 = __nv_cvt_float_to_fp8(__fdiv_rn(c, s), __NV_SATFINITE, __NV_E4M3);
  const uint32_t q3 = __nv_cvt_float_to_fp8(__fdiv_rn(d, s), __NV_SATFINITE, __NV_E4M3);
  return q0 | (q1 << 8) | (q2 << 16) | (q3 << 24);
}
__global__ void __launch_bounds__(256) e4m3_quant_kernel(const bf16* __restrict__ x, size_t n,
                                                         const float* __restrict__ sp, uint8_t* __restrict__ q) {
  const float s = __ldg(sp);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const bool vec = !((reinterpret_cast<uintptr_t>(x) & 15) | (reinterpret_cast<uintptr_t>(q) & 7));
  const size_t n8 = vec ? n / 8 : 0;
  auto cvt = [&](const uint4 u, size_t i) {
    uint2 o;
    o.x = e4m3x4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                 __uint_as_float(u.y & 0xFFFF0000u), s);
    o.y = e4m3x4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u), __uint_as_float(u.w << 16),
                 __uint_as_float(u.w & 0xFFFF0000u), s);
    reinterpret_cast<uint2*>(q)[i] = o;
  };
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n8; i += 4 * stride) {  // four 16-byte loads in flight per thread
    const uint4 u0 = __ldg(xv + i), u1 = __ldg(xv + i + stride), u2 = __ldg(xv + i + 2 * stride),
                u3 = __ldg(xv + i + 3 * stride);
    cvt(u0, i), cvt(u1, i + stride), cvt(u2, i + 2 * stride), cvt(u3, i + 3 * stride);
  }
  for (; i < n8; i += stride) cvt(__ldg(xv + i), i);
  for (size_t i = n8 * 8 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    q[i] = uint8_t(__nv_cvt_float_to_fp8(__fdiv_rn(bf2f(x[i]), s), __NV_SATFINITE, __NV_E4M3));
}
// RMSNorm + modulation (or gain) quantised per row to e4m3 (FP8 step, R29): one warp per row,
// three passes over the row (the row stays in L1/L2): sum of squares; y and its amax; q.  The
// row scale is a power of two (the fp32 amax / 448 rounded up to one), so y / s is an exact
// exponent shift: one multiply per element instead of an IEEE division.
DF_DEV float pow2_ceil(float v) {  // smallest power of two >= v (v > 0; 2^-126 for subnormal v)
  const uint32_t b = __float_as_uint(v);
  const uint32_t e = b >> 23;
  if (e == 0) return __uint_as_float(1u << 23);
  return (b & 0x7FFFFFu) ? __uint_as_float((e + 1) << 23) : v;
}
__device__ __forceinline__ uint32_t e4m3x4_mul(float a, float b, float c, float d, float inv) {
  const uint32_t q0 = __nv_cvt_float_to_fp8(a * inv, __NV_SATFINITE, __NV_E4M3);
  const uint32_t q1 = __nv_cvt_float_to_fp8(b * inv, __NV_SATFINITE, __NV_E4M3);
  const uint32_t q2 = __nv_cvt_float_to_fp8(c * inv, __NV_SATFINITE, __NV_E4M3);
  const uint32_t q3 = __nv_cvt_float_to_fp8(d * inv, __NV_SATFINITE, __NV_E4M3);
  return q0 | (q1 << 8) | (q2 << 16) | (q3 << 24);
}
template <int VPT>
__global__ void __launch_bounds__(128, 8) rmsnorm_e4m3_kernel(const float* __restrict__ x, uint8_t* __restrict__ q,
                                                          float* __restrict__ srow, int M,
                                                          const float* __restrict__ shift,
                                                          const float* __restrict__ scale,
                                                          const bf16* __restrict__ gain, float eps) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  pdl_wait();
  pdl_launch_dependents();
  if (row >= M) return;
  constexpr int d = 128 * VPT;
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * d);
  float ss = 0.f;
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    const float4 t = xr[lane + 32 * i];
    ss += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
  }
  ss = warp_sum(ss);
  const float inv = rsqrtf(ss / float(d) + eps);
  auto modulate = [&](int c, float* y) {
    const float4 t = xr[c];
    y[0] = t.x * inv, y[1] = t.y * inv, y[2] = t.z * inv, y[3] = t.w * inv;
    if (gain) {
      const uint2 g = reinterpret_cast<const uint2*>(gain)[c];
      y[0] *= bf_lo(g.x), y[1] *= bf_hi(g.x), y[2] *= bf_lo(g.y), y[3] *= bf_hi(g.y);
    } else {
      const float4 sc = reinterpret_cast<const float4*>(scale)[c];
      const float4 sh = reinterpret_cast<const float4*>(shift)[c];
      y[0] = y[0] * (1.f + sc.x) + sh.x;
      y[1] = y[1] * (1.f + sc.y) + sh.y;
      y[2] = y[2] * (1.f + sc.z) + sh.z;
      y[3] = y[3] * (1.f + sc.w) + sh.w;
    }
  };
  float am = 0.f;
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    float y[4];
    modulate(lane + 32 * i, y);
    am = fmaxf(am, fmaxf(fmaxf(fabsf(y[0]), fabsf(y[1])), fmaxf(fabsf(y[2]), fabsf(y[3]))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  const float sr = am > 0.f ? pow2_ceil(__fdiv_rn(am, 448.f)) : 1.f;
  const float rs = __uint_as_float((254u << 23) - __float_as_uint(sr));  // exactly 1 / sr (a power of two)
  uint32_t* qr = reinterpret_cast<uint32_t*>(q + size_t(row) * d);
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    float y[4];
    modulate(lane + 32 * i, y);
    qr[lane + 32 * i] = e4m3x4_mul(y[0], y[1], y[2], y[3], rs);
  }
  if (lane == 0) srow[row] = sr;
}

// A bf16 activation [M, K] quantised per row to e4m3 with power-of-two row scales (R29): the
// inputs of the O, cross-O and MLP-down projections (attention and SwiGLU outputs).  One warp
// per row, 8 bf16 per lane per step; pass 1 the row amax, pass 2 the codes (row re-read from L1/L2).
__global__ void __launch_bounds__(256) quant_rows_e4m3_kernel(const bf16* __restrict__ x, uint8_t* __restrict__ q,
                                                             float* __restrict__ srow, int M, int K) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_wait();
  pdl_launch_dependents();
  if (row >= M) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + size_t(row) * K);
  const int n8 = K / 8;
  float am = 0.f;
  for (int i = lane; i < n8; i += 32) {
    const uint4 u = __ldg(xr + i);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      am = fmaxf(am, fmaxf(fabsf(__uint_as_float(w[k] << 16)), fabsf(__uint_as_float(w[k] & 0xFFFF0000u))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  const float sr = am > 0.f ? pow2_ceil(__fdiv_rn(am, 448.f)) : 1.f;
  const float rs = __uint_as_float((254u << 23) - __float_as_uint(sr));
  uint2* qr = reinterpret_cast<uint2*>(q + size_t(row) * K);
  for (int i = lane; i < n8; i += 32) {
    const uint4 u = __ldg(xr + i);
    uint2 o;
    o.x = e4m3x4_mul(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xFFFF0000u), rs);
    o.y = e4m3x4_mul(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u), __uint_as_float(u.w << 16),
                     __uint_as_float(u.w & 0xFFFF0000u), rs);
    qr[i] = o;
  }
  if (lane == 0) srow[row] = sr;
}

cudaError_t quant_rows_e4m3(const bf16* x, uint8_t* q, float* s, int M, int K, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  if (K % 8) return cudaErrorInvalidValue;
  {
    void* args[] = {(void*)&x, (void*)&q, (void*)&s, (void*)&M, (void*)&K};
    cudaError_t e = launch_ex((const void*)quant_rows_e4m3_kernel, dim3((M + 7) / 8), dim3(256), 0, st, args);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t rmsnorm_e4m3(const float* x, uint8_t* q, float* s, int M, int d, const float* shift, const float* scale,
                         const bf16* gain, float eps, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  dim3 grid((M + 3) / 4);
  void* args[] = {(void*)&x, (void*)&q, (void*)&s, (void*)&M, (void*)&shift, (void*)&scale, (void*)&gain, (void*)&eps};
  switch (d) {
    case 256: return launch_ex((const void*)rmsnorm_e4m3_kernel<2>, grid, dim3(128), 0, st, args);
    case 3072: return launch_ex((const void*)rmsnorm_e4m3_kernel<24>, grid, dim3(128), 0, st, args);
    case 5120: return launch_ex((const void*)rmsnorm_e4m3_kernel<40>, grid, dim3(128), 0, st, args);
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t quant_e4m3(const bf16* x, size_t n, uint8_t* q, float* scale, cudaStream_t st) {
  cudaError_t e0 = cudaMemsetAsync(scale, 0, sizeof(float), st);
  if (e0 != cudaSuccess) return e0;
  if (n == 0) {
    e4m3_scale_kernel<<<1, 1, 0, st>>>(scale);
    return cudaGetLastError();
  }
  const size_t per = 256 * 8 * 4;  // four 8-element vectors per thread
  const unsigned grid = unsigned(std::max<size_t>(1, std::min<size_t>((n + per - 1) / per, size_t(num_sms()) * 8)));
  e4m3_amax_kernel<<<grid, 256, 0, st>>>(x, n, reinterpret_cast<unsigned*>(scale));
  e4m3_scale_kernel<<<1, 1, 0, st>>>(scale);
  e4m3_quant_kernel<<<grid, 256, 0, st>>>(x, n, scale, q);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- MXFP8 quantiser (R30)
// OCP MX v1.0 with E4M3 elements: per 32-element block of a row, e = floor(log2 amax) - 8
// (clamped to [-127, 127]; -127 for an all-zero block), q = RNE_satfinite_e4m3(x * 2^-e) --
// the multiply by a power of two is exact in fp32 unless the quotient is below 2^-126, where
// the e4m3 code is 0 either way.  One thread per block (four 16-byte loads, two 16-byte
// stores); the scale byte e + 127 goes to the tiled layout the MXFP8 GEMM loads by TMA:
// atom (kg = kb / 4, rb = row / 128) at byte (kg * RB + rb) * 512, inside it
// (row % 32) * 16 + ((row % 128) / 32) * 4 + kb % 4.  Rows [M, RB * 128) get scale byte 0.
__global__ void __launch_bounds__(256) mx_quant_e4m3_kernel(const bf16* __restrict__ x, int M, int K, int RB,
                                                            uint8_t* __restrict__ q, uint8_t* __restrict__ sf) {
  const int KB = K / 32;
  const long long idx = blockIdx.x * 256ll + threadIdx.x;
  pdl_wait();
  pdl_launch_dependents();
  if (idx >= (long long)RB * 128 * KB) return;
  const int r = int(idx / KB), kb = int(idx - (long long)r * KB);
  const size_t sfo = (size_t(kb >> 2) * RB + (r >> 7)) * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4 + (kb & 3);
  if (r >= M) {
    sf[sfo] = 0;
    return;
  }
  const uint4* xv = reinterpret_cast<const uint4*>(x + size_t(r) * K + size_t(kb) * 32);
  uint4 u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = __ldg(xv + i);
  float v[32];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t w[4] = {u[i].x, u[i].y, u[i].z, u[i].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[8 * i + 2 * k] = __uint_as_float(w[k] << 16);
      v[8 * i + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  }
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(v[i]));
  int e = -127;
  if (amax > 0.f) {
    int ex;
    frexpf(amax, &ex);  // amax = m 2^ex, m in [0.5, 1): floor(log2 amax) = ex - 1
    e = min(127, max(-127, ex - 1 - 8));
  }
  const float inv = scalbnf(1.0f, -e);
  uint32_t o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = e4m3x4_mul(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3], inv);
  uint4* qv = reinterpret_cast<uint4*>(q + size_t(r) * K + size_t(kb) * 32);
  qv[0] = make_uint4(o[0], o[1], o[2], o[3]);
  qv[1] = make_uint4(o[4], o[5], o[6], o[7]);
  sf[sfo] = uint8_t(e + 127);
}

cudaError_t mx_quant_e4m3(const bf16* x, int M, int K, uint8_t* q, uint8_t* sf, cudaStream_t st) {
  if (M <= 0 || K <= 0) return cudaSuccess;
  if (K % 128 || !x || !q || !sf || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(q) & 15))
    return cudaErrorInvalidValue;
  const int RB = (M + 127) / 128;
  const long long n = (long long)RB * 128 * (K / 32);
  void* args[] = {(void*)&x, (void*)&M, (void*)&K, (void*)&RB, (void*)&q, (void*)&sf};
  return launch_ex((const void*)mx_quant_e4m3_kernel, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, args);
}

// RMSNorm + modulation (or gain) quantised to MXFP8 (R31): one warp per row, pass 1 the sum
// of squares, pass 2 y = RMSNorm(x) (1 + scale) + shift (or * gain) in fp32 and, per 32-element
// block (8 lanes x 4 values of one float4 step), R30's scale exponent from the block amax
// (a shuffle over the 8 lanes) and the e4m3 codes; the scale byte goes to the tiled layout.
template <int VPT>
__global__ void __launch_bounds__(128, 8) rmsnorm_mx_kernel(const float* __restrict__ x, uint8_t* __restrict__ q,
                                                        uint8_t* __restrict__ sf, int M, int RB,
                                                        const float* __restrict__ shift,
                                                        const float* __restrict__ scale,
                                                        const bf16* __restrict__ gain, float eps) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  pdl_wait();
  pdl_launch_dependents();
  if (row >= M) return;
  constexpr int d = 128 * VPT;
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * d);
  float ss = 0.f;
#pragma unroll 8
  for (int i = 0; i < VPT; ++i) {
    const float4 t = xr[lane + 32 * i];
    ss += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
  }
  ss = warp_sum(ss);
  const float inv = rsqrtf(ss / float(d) + eps);
  uint32_t* qr = reinterpret_cast<uint32_t*>(q + size_t(row) * d);
  const size_t sf_row = size_t(row >> 7) * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4;
#pragma unroll 4
  for (int i = 0; i < VPT; ++i) {
    const int c = lane + 32 * i;
    const float4 t = xr[c];
    float y[4] = {t.x * inv, t.y * inv, t.z * inv, t.w * inv};
    if (gain) {
      const uint2 g = reinterpret_cast<const uint2*>(gain)[c];
      y[0] *= bf_lo(g.x), y[1] *= bf_hi(g.x), y[2] *= bf_lo(g.y), y[3] *= bf_hi(g.y);
    } else {
      const float4 sc = reinterpret_cast<const float4*>(scale)[c];
      const float4 sh = reinterpret_cast<const float4*>(shift)[c];
      y[0] = y[0] * (1.f + sc.x) + sh.x;
      y[1] = y[1] * (1.f + sc.y) + sh.y;
      y[2] = y[2] * (1.f + sc.z) + sh.z;
      y[3] = y[3] * (1.f + sc.w) + sh.w;
    }
    float am = fmaxf(fmaxf(fabsf(y[0]), fabsf(y[1])), fmaxf(fabsf(y[2]), fabsf(y[3])));
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 1));
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 2));
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 4));
    int e = -127;
    if (am > 0.f) {
      int ex;
      frexpf(am, &ex);
      e = min(127, max(-127, ex - 1 - 8));
    }
    qr[c] = e4m3x4_mul(y[0], y[1], y[2], y[3], scalbnf(1.0f, -e));
    if ((lane & 7) == 0) {
      const int kb = c >> 3;  // 32-element block of this row
      sf[(size_t(kb >> 2) * RB) * 512 + sf_row + (kb & 3)] = uint8_t(e + 127);
    }
  }
}

cudaError_t rmsnorm_mx(const float* x, uint8_t* q, uint8_t* sf, int M, int d, const float* shift, const float* scale,
                       const bf16* gain, float eps, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  if (d % 128) return cudaErrorInvalidValue;
  const int RB = (M + 127) / 128;
  // one warp per row: a persistent TMA-streaming variant (one HBM read of the row, as the bf16
  // norm's at video sizes) measured 2x slower here at both the image and the video shape
  // (51.8 vs 24.7 us, 594 vs 284 us in the MXFP8 step) and was removed
  void* args[] = {(void*)&x, (void*)&q, (void*)&sf, (void*)&M, (void*)&RB, (void*)&shift, (void*)&scale,
                  (void*)&gain, (void*)&eps};
  const dim3 grid((M + 3) / 4);
  switch (d / 128) {
    case 2: return launch_ex((const void*)rmsnorm_mx_kernel<2>, grid, dim3(128), 0, st, args);
    case 24: return launch_ex((const void*)rmsnorm_mx_kernel<24>, grid, dim3(128), 0, st, args);
    case 40: return launch_ex((const void*)rmsnorm_mx_kernel<40>, grid, dim3(128), 0, st, args);
    default: return cudaErrorInvalidValue;
  }
}

// FP8 modes (R32): head-major bf16 Q or K -> e4m3 codes q = RNE_satfinite(x * inv) with inv a
// power of two (exact), 8 elements per thread (one 16-byte load, one 8-byte store).
__global__ void __launch_bounds__(256) qk_e4m3_kernel(const bf16* __restrict__ x, size_t n8, float inv,
                                                      uint8_t* __restrict__ q) {
  pdl_wait();
  pdl_launch_dependents();
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n8; i += stride) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(x) + i);
    uint2 o;
    o.x = e4m3x4_mul(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xFFFF0000u), inv);
    o.y = e4m3x4_mul(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u), __uint_as_float(u.w << 16),
                     __uint_as_float(u.w & 0xFFFF0000u), inv);
    reinterpret_cast<uint2*>(q)[i] = o;
  }
}

cudaError_t qk_e4m3(const bf16* x, size_t n, float inv, uint8_t* q, cudaStream_t st) {
  if (!n) return cudaSuccess;
  if (n % 8 || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(q) & 7))
    return cudaErrorInvalidValue;
  size_t n8 = n / 8;
  const unsigned grid = unsigned(std::min<size_t>((n8 + 255) / 256, size_t(num_sms()) * 8));
  void* args[] = {(void*)&x, (void*)&n8, (void*)&inv, (void*)&q};
  return launch_ex((const void*)qk_e4m3_kernel, dim3(grid), dim3(256), 0, st, args);
}

// R33: V [H][N][128] bf16 -> V^T e4m3 [H][128][ldv] (keys contiguous: the K-major B operand of
// the e4m3 PV MMA) with one per-tensor power-of-two scale s = pow2ceil(fp32(amax|V| / 448)).
// s[0] = the scale from the amax accumulated in s[1]; s[1] is re-zeroed for the next call
__global__ void v_scale_kernel(float* s) {
  pdl_wait();
  pdl_launch_dependents();
  const float a = __uint_as_float(reinterpret_cast<const unsigned*>(s)[1]);
  s[0] = a > 0.f ? pow2_ceil(__fdiv_rn(a, 448.f)) : 1.f;
  reinterpret_cast<unsigned*>(s)[1] = 0u;
}
// one block per (64 keys, head): 64 x 128 bf16 -> e4m3 through a shared [128][64 + 16] tile
__global__ void __launch_bounds__(256) v_e4m3t_kernel(const bf16* __restrict__ V, int N, int ldv,
                                                      const float* __restrict__ sp, uint8_t* __restrict__ VT) {
  __shared__ uint8_t tile[128][80];
  const int h = blockIdx.y, k0 = blockIdx.x * 64;
  pdl_wait();
  pdl_launch_dependents();
  const float inv = __uint_as_float((254u << 23) - __float_as_uint(__ldg(sp)));  // exactly 1 / s
  const int t = threadIdx.x;
  {  // load: thread t -> key k0 + t / 4, dh [32 (t % 4), +32)
    const int k = k0 + (t >> 2), c0 = (t & 3) * 32;
    uint32_t w[16];
    if (k < N) {
      const uint4* src = reinterpret_cast<const uint4*>(V + (size_t(h) * N + k) * 128 + c0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 u = __ldg(src + i);
        w[4 * i] = u.x, w[4 * i + 1] = u.y, w[4 * i + 2] = u.z, w[4 * i + 3] = u.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = 0;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t q2 = __nv_cvt_float2_to_fp8x2(
          make_float2(__uint_as_float(w[i] << 16) * inv, __uint_as_float(w[i] & 0xFFFF0000u) * inv), __NV_SATFINITE,
          __NV_E4M3);
      tile[c0 + 2 * i][t >> 2] = uint8_t(q2 & 0xFF);
      tile[c0 + 2 * i + 1][t >> 2] = uint8_t(q2 >> 8);
    }
  }
  __syncthreads();
  {  // store: thread t -> dh row t / 2, keys [32 (t % 2), +32)
    const int r = t >> 1, kk = (t & 1) * 32;
    if (k0 + kk < N) {
      const uint4* src = reinterpret_cast<const uint4*>(&tile[r][kk]);
      uint4* dst = reinterpret_cast<uint4*>(VT + (size_t(h) * 128 + r) * ldv + k0 + kk);
      dst[0] = src[0];
      dst[1] = src[1];
    }
  }
}

cudaError_t v_e4m3t(const bf16* V, int H, int N, int ldv, float* vscale, uint8_t* VT, cudaStream_t st) {
  if (H <= 0 || N <= 0) return cudaSuccess;
  if (ldv < ((N + 63) / 64) * 64 || ldv % 16 || (reinterpret_cast<uintptr_t>(V) & 15) ||
      (reinterpret_cast<uintptr_t>(VT) & 15))
    return cudaErrorInvalidValue;
  size_t n = size_t(H) * N * 128;
  const int per = 256 * 8 * 4;
  const unsigned grid = unsigned(std::max<size_t>(1, std::min<size_t>((n + per - 1) / per, size_t(num_sms()) * 8)));
  // three PDL launches; vscale[1] (the amax accumulator) is zero on entry and left zero
  unsigned* acc = reinterpret_cast<unsigned*>(vscale) + 1;
  void* a1[] = {(void*)&V, (void*)&n, (void*)&acc};
  cudaError_t e = launch_ex((const void*)e4m3_amax_kernel, dim3(grid), dim3(256), 0, st, a1);
  if (e != cudaSuccess) return e;
  void* a2[] = {(void*)&vscale};
  e = launch_ex((const void*)v_scale_kernel, dim3(1), dim3(1), 0, st, a2);
  if (e != cudaSuccess) return e;
  const float* sp = vscale;
  void* a3[] = {(void*)&V, (void*)&N, (void*)&ldv, (void*)&sp, (void*)&VT};
  return launch_ex((const void*)v_e4m3t_kernel, dim3((N + 63) / 64, H), dim3(256), 0, st, a3);
}

}  // namespace df
