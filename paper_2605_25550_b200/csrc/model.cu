// Stage programs of one instance: parameter init (DESIGN.md parameter table), the
// DiT request prologue / step / block, the E and D stand-ins.
// Each launch is counted for bench.py's "gpu_launches".
#include <atomic>
#include <cmath>
#include <algorithm>
#include <cstring>
#include "runtime.h"

namespace df {

thread_local std::string tls_err;
static std::atomic<uint64_t> g_launch_count{0};
std::atomic<uint64_t>* g_launches = &g_launch_count;

#define DF_L(expr)                                  \
  do {                                              \
    g_launch_count.fetch_add(1, std::memory_order_relaxed); \
    DF_TRY(expr);                                   \
  } while (0)

// ------------------------------------------------------------------ arena
cudaError_t Arena::reserve(size_t bytes) {
  cap = bytes;
  used = 0;
  if (!bytes) return cudaSuccess;
  cudaError_t e = cudaMalloc(&base, bytes);
  if (e != cudaSuccess) base = nullptr;
  return e;
}
void* Arena::take(size_t bytes) {
  size_t off = (used + 255) & ~size_t(255);
  if (off + bytes > cap) return nullptr;
  used = off + bytes;
  return base + off;
}
void Arena::release() {
  if (base) cudaFree(base);
  base = nullptr;
  cap = used = 0;
}

static size_t al(size_t b) { return (b + 255) & ~size_t(255); }

cudaEvent_t Prof::get() {
  if (pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = pool.back();
  pool.pop_back();
  return e;
}
void Prof::reserve(size_t n) {
  std::lock_guard<std::mutex> lk(mu);
  while (pool.size() < n) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    pool.push_back(e);
  }
}
void Prof::harvest() {
  std::lock_guard<std::mutex> lk(mu);
  for (auto& p : pending) {
    float t = 0.f;
    cudaEventSynchronize(p.b);
    if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
      count[p.kind]++;
      ms[p.kind] += t;
      flops[p.kind] += p.flops;
      bytes[p.kind] += p.bytes;
    }
    cudaGetLastError();
    pool.push_back(p.a);
    pool.push_back(p.b);
  }
  pending.clear();
}
void Prof::reset() {
  harvest();
  std::lock_guard<std::mutex> lk(mu);
  for (int k = 0; k < K_COUNT; ++k) count[k] = 0, ms[k] = flops[k] = bytes[k] = 0;
}

// Brackets one launch with profiler events when profiling is on.
struct ProfScope {
  Prof* p;
  cudaStream_t st;
  int kind;
  double fl, by;
  cudaEvent_t a = nullptr;
  ProfScope(Prof* p_, cudaStream_t s, int k, double f, double b) : p(p_), st(s), kind(k), fl(f), by(b) {
    if (p) {
      std::lock_guard<std::mutex> lk(p->mu);
      a = p->get();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (p) {
      std::lock_guard<std::mutex> lk(p->mu);
      cudaEvent_t b = p->get();
      cudaEventRecord(b, st);
      p->pending.push_back({kind, a, b, fl, by});
    }
  }
};

// ------------------------------------------------------------------ create / init
cudaError_t Model::create(const df_dit_cfg& cfg, int prec, int dev, int stg, uint64_t sd, int msteps) {
  c = cfg;
  precision = prec;
  device = dev;
  stage = stg;
  seed = sd;
  max_steps = msteps;
  DF_TRY(cudaSetDevice(device));
  Fp = c.F / c.pt;
  Hp = c.H / c.ph;
  Wp = c.W / c.pw;
  N = Fp * Hp * Wp;
  P = c.C * c.pt * c.ph * c.pw;
  Pin = (c.C + c.C_y) * c.pt * c.ph * c.pw;
  dh = c.d / c.heads;
  dhp = f32() ? dh : (dh <= 64 ? 64 : 128);
  if (fp8() && stage == DF_T && (c.d < 256 || N < 256 || dh != 128 || c.d % 16))
    return cudaErrorInvalidValue;  // the FP8 GEMMs run on CTA-pair tiles with the head-major TMA epilogue
  if (mx() && stage == DF_T && (c.d % 128 || c.ffn % 128 || (c.d != 256 && c.d != 3072 && c.d != 5120)))
    return cudaErrorInvalidValue;  // MX blocks: K % 128 (one scale atom per 128 k); rmsnorm_mx widths
  if (c.d % c.heads || dh > 128 || c.ffn % 16 || c.d % 4 || c.enc_ffn % 16 ||
      c.rope_axes[0] + c.rope_axes[1] + c.rope_axes[2] != uint32_t(dh) ||
      (c.C_y > 0 && (c.L_img == 0 || c.d_img == 0 || c.d_img % 8)))
    return cudaErrorInvalidValue;
  const size_t d = c.d, f = c.ffn, L = c.L_txt, dt = c.d_txt, fe = c.enc_ffn, ab = act_bytes();
  // ---- weights
  size_t wb = 0;
  if (stage == DF_T) {
    wb += al(d * Pin * 2) + al(d * 2) + al(d * dt * 2) + al(d * 2) + al(d * d * 2) + al(d * 2) + al(d * c.freq_dim * 2) +
          al(d * 2) + al(d * d * 2) + al(d * 2) + al(6 * d * d * 2) + al(6 * d * 2) + al(2 * d * 2) + al(P * d * 2) +
          al(P * 2);
    size_t per = al(6 * d * 2) + al(3 * d * d * 2) + al(3 * d * 2) + 3 * al(d * 2) + al(d * d * 2) + al(d * 2) +
                 al(d * d * 2) + al(d * 2) + al(2 * d * d * 2) + al(2 * d * 2) + 2 * al(d * 2) + al(d * d * 2) +
                 al(d * 2) + al(2 * f * d * 2) + al(2 * f * 2) + al(d * f * 2) + al(d * 2);
    wb += per * c.layers;
    if (i2v())  // image projection + per layer image-token K | V and K gain
      wb += al(d * c.d_img * 2) + al(d * 2) + al(d * d * 2) + al(d * 2) +
            size_t(c.layers) * (al(2 * d * d * 2) + al(2 * d * 2) + al(d * 2));
  } else if (stage == DF_E) {
    wb += al(size_t(c.vocab) * dt * 2) + 2 * al(dt * 2) + al(2 * fe * dt * 2) + al(dt * fe * 2);
  } else {
    wb += al(c.C * c.dec_width * 2) + al(c.dec_width * 2) + al(c.dec_width * 192 * 2) + al(192 * 2) +
          al(c.dec_width * 768 * 2) + al(768 * 2);
  }
  DF_TRY(wmem.reserve(wb + 4096));
  auto W = [&](size_t n) { return static_cast<bf16*>(wmem.take(n * 2)); };
  if (stage == DF_T) {
    patch_wT = W(d * Pin); patch_b = W(d);
    txt1_wT = W(d * dt); txt1_b = W(d); txt2_wT = W(d * d); txt2_b = W(d);
    temb1_wT = W(d * c.freq_dim); temb1_b = W(d); temb2_wT = W(d * d); temb2_b = W(d);
    tmod_wT = W(6 * d * d); tmod_b = W(6 * d); head_mod = W(2 * d); head_wT = W(P * d); head_b = W(P);
    Lw.resize(c.layers);
    for (auto& l : Lw) {
      l.mod = W(6 * d); l.qkv_wT = W(3 * d * d); l.qkv_b = W(3 * d); l.g_q = W(d); l.g_k = W(d);
      l.o_wT = W(d * d); l.o_b = W(d); l.g_n3 = W(d); l.cq_wT = W(d * d); l.cq_b = W(d);
      l.ckv_wT = W(2 * d * d); l.ckv_b = W(2 * d); l.g_cq = W(d); l.g_ck = W(d); l.co_wT = W(d * d); l.co_b = W(d);
      l.w13T = W(2 * f * d); l.b13 = W(2 * f); l.w2T = W(d * f); l.b2 = W(d);
    }
    if (i2v()) {
      img1_wT = W(d * c.d_img); img1_b = W(d); img2_wT = W(d * d); img2_b = W(d);
      for (auto& l : Lw) {
        l.ckvi_wT = W(2 * d * d); l.ckvi_b = W(2 * d); l.g_ki = W(d);
      }
    }
    layer_mods.clear();
    for (auto& l : Lw) layer_mods.push_back(l.mod);
  } else if (stage == DF_E) {
    emb = W(size_t(c.vocab) * dt); g_a = W(dt); e_w13T = W(2 * fe * dt); e_w2T = W(dt * fe); g_f = W(dt);
  } else {
    d1_w = W(c.C * c.dec_width); d1_b = W(c.dec_width); d2f_w = W(c.dec_width * 192); d2f_b = W(192);
    d2r_w = W(c.dec_width * 768); d2r_b = W(768);
  }
  if (!wmem.base) return cudaErrorMemoryAllocation;
  // ---- workspace
  size_t wsb = 0;
  const size_t Nn = N;
  if (stage == DF_T) {
    // activations sized for a batch of 2 (classifier-free guidance stacks cond + negative)
    const size_t N2 = 2 * Nn;
    size_t hd = size_t(c.heads) * N2 * dhp * ab;
    wsb = al(N2 * d * 4) + al(N2 * d * ab) + 4 * al(hd) + al(N2 * d * ab) + al(N2 * f * ab) + al(Nn * Pin * ab) +
          (i2v() ? al(N2 * d * ab) : 0) +
          al(size_t(c.layers) * 6 * d * 4) + al(2 * d * 4) + al(size_t(Fp + Hp + Wp) * dh / 2 * 8) +
          al(2 * size_t(c.C) * c.F * c.H * c.W * 4);
    if (fp8()) wsb += al(N2 * std::max(d, f)) + al(N2 * 4);
    if (mx()) wsb += al(mx_sf_bytes(N2, std::max(d, f)));
    if (fp8()) wsb += 2 * al(hd / 2) + al(size_t(2) * c.heads * 128 * ((Nn + 63) / 64 * 64)) + al(64);
    if (f32()) wsb += al(N2 * std::max(3 * d, 2 * f) * 4);
    else wsb += al(size_t(num_sms()) * 128 * 256 * 4) + al(size_t(num_sms()) * 4);  // GEMM stream-K
  } else if (stage == DF_E) {
    wsb = al(L * dt * 4) + al(L * dt * ab) + al(L * fe * ab) + al(L * 2 * fe * 4);
  }
  DF_TRY(ws.reserve(wsb + 4096));
  if (stage == DF_T) {
    const size_t N2 = 2 * Nn;
    size_t hd = size_t(c.heads) * N2 * dhp * ab;
    r = (float*)ws.take(N2 * d * 4);
    h = ws.take(N2 * d * ab);
    q = ws.take(hd); k = ws.take(hd); v = ws.take(hd); qc = ws.take(hd);
    o = ws.take(N2 * d * ab);
    a = ws.take(N2 * f * ab);
    X = ws.take(Nn * Pin * ab);
    if (i2v()) oi = ws.take(N2 * d * ab);
    vbatch = (float*)ws.take(2 * size_t(c.C) * c.F * c.H * c.W * 4);
    if (fp8()) {
      hq = (uint8_t*)ws.take(N2 * std::max(d, f));
      hs = (float*)ws.take(N2 * 4);
    }
    if (fp8()) {
      q8 = (uint8_t*)ws.take(hd / 2);
      k8 = (uint8_t*)ws.take(hd / 2);
      ldv8 = int((Nn + 63) / 64 * 64);
      v8t = (uint8_t*)ws.take(size_t(2) * c.heads * 128 * ldv8);
      v8s = (float*)ws.take(64);
      DF_TRY(cudaMemset(v8s, 0, 64));  // [1]: v_e4m3t's amax accumulator, zero between calls
    }
    if (mx()) {  // rows past M in the last 128-row block keep scale byte 0
      hsf = (uint8_t*)ws.take(mx_sf_bytes(N2, std::max(d, f)));
      DF_TRY(cudaMemset(hsf, 0, mx_sf_bytes(N2, std::max(d, f))));
    }
    mods = (float*)ws.take(size_t(c.layers) * 6 * d * 4);
    headmod = (float*)ws.take(2 * d * 4);
    rope = (float2*)ws.take(size_t(Fp + Hp + Wp) * dh / 2 * 8 + 64);
    if (f32()) {
      tmp = (float*)ws.take(N2 * std::max(3 * d, 2 * f) * 4);
    } else {
      sk_ws = (float*)ws.take(size_t(num_sms()) * 128 * 256 * 4);
      sk_flag = (unsigned*)ws.take(size_t(num_sms()) * 4);
      DF_TRY(cudaMemset(sk_flag, 0, size_t(num_sms()) * 4));
    }
    // zero the head-major buffers once: the dh..dhp padding must stay 0 (TMA reads it)
    DF_TRY(cudaMemset(q, 0, 4 * al(hd)));
    // RoPE table in fp64 -> fp32 (R7): (cos, sin)(pos_a * theta^(-2j/D_a))
    std::vector<float2> tab;
    const int ax[3] = {int(c.rope_axes[0]), int(c.rope_axes[1]), int(c.rope_axes[2])};
    const int npos[3] = {Fp, Hp, Wp};
    for (int a3 = 0; a3 < 3; ++a3)
      for (int p = 0; p < npos[a3]; ++p)
        for (int j = 0; j < ax[a3] / 2; ++j) {
          double phi = double(p) * std::pow(double(c.rope_theta), -2.0 * j / ax[a3]);
          tab.push_back(make_float2(float(std::cos(phi)), float(std::sin(phi))));
        }
    DF_TRY(cudaMemcpy(rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  } else if (stage == DF_E) {
    ez = (float*)ws.take(L * dt * 4);
    ea = ws.take(L * dt * ab);
    ef = ws.take(L * fe * ab);
    etmp = (float*)ws.take(L * 2 * fe * 4);
  }
  DF_TRY(init_weights(0));
  if (fp8() && stage == DF_T) DF_TRY(quantize_weights(0));
  DF_TRY(cudaDeviceSynchronize());
  return cudaSuccess;
}

// FP8 step (R29): per-tensor e4m3 copies of every block GEMM's weight (R28's quantiser on the
// bf16 weights, so the codes are those of the oracle's quantize_per_tensor; W_1 | W_3 jointly).
cudaError_t Model::quantize_weights(cudaStream_t st) {
  const size_t d = c.d, f = c.ffn;
  {  // R32: the self-attention's e4m3 Q / K scales from the qk-norm gains (host copies, once)
    std::vector<uint16_t> g(d);
    auto qscale = [&](const bf16* gain) -> float {
      if (cudaMemcpy(g.data(), gain, d * 2, cudaMemcpyDeviceToHost) != cudaSuccess) return 0.f;
      float gmax = 0.f;
      for (size_t i = 0; i < d; ++i) {
        uint32_t b = uint32_t(g[i]) << 16;
        float v;
        std::memcpy(&v, &b, 4);
        gmax = std::max(gmax, std::fabs(v));
      }
      const float bound = float(std::sqrt(double(dh)) * double(gmax) / 448.0);
      int e;
      const float m = std::frexp(bound, &e);  // bound = m 2^e, m in [0.5, 1)
      return bound > 0.f ? (m == 0.5f ? bound : std::ldexp(1.0f, e)) : 1.f;
    };
    for (auto& l : Lw) {
      l.sq = qscale(l.g_q);
      l.sk = qscale(l.g_k);
      if (l.sq <= 0.f || l.sk <= 0.f) return cudaErrorUnknown;
    }
  }
  if (mx()) {  // MXFP8 step (R31): OCP MX codes + tiled block scales of every block GEMM's weight [N, K]
    const size_t per = al(3 * d * d) + 3 * al(d * d) + 2 * al(2 * f * d) + al(mx_sf_bytes(3 * d, d)) +
                       3 * al(mx_sf_bytes(d, d)) + al(mx_sf_bytes(2 * f, d)) + al(mx_sf_bytes(d, f));
    DF_TRY(f8mem.reserve(per * c.layers + 4096));
    for (auto& l : Lw) {
      l.qkv_q = (uint8_t*)f8mem.take(3 * d * d);
      l.cq_q = (uint8_t*)f8mem.take(d * d);
      l.w13_q = (uint8_t*)f8mem.take(2 * f * d);
      l.o_q = (uint8_t*)f8mem.take(d * d);
      l.co_q = (uint8_t*)f8mem.take(d * d);
      l.w2_q = (uint8_t*)f8mem.take(d * f);
      l.qkv_sf = (uint8_t*)f8mem.take(mx_sf_bytes(3 * d, d));
      l.cq_sf = (uint8_t*)f8mem.take(mx_sf_bytes(d, d));
      l.w13_sf = (uint8_t*)f8mem.take(mx_sf_bytes(2 * f, d));
      l.o_sf = (uint8_t*)f8mem.take(mx_sf_bytes(d, d));
      l.co_sf = (uint8_t*)f8mem.take(mx_sf_bytes(d, d));
      l.w2_sf = (uint8_t*)f8mem.take(mx_sf_bytes(d, f));
      if (!l.w2_sf) return cudaErrorMemoryAllocation;
      DF_L(mx_quant_e4m3(l.qkv_wT, int(3 * d), int(d), l.qkv_q, l.qkv_sf, st));
      DF_L(mx_quant_e4m3(l.cq_wT, int(d), int(d), l.cq_q, l.cq_sf, st));
      DF_L(mx_quant_e4m3(l.w13T, int(2 * f), int(d), l.w13_q, l.w13_sf, st));
      DF_L(mx_quant_e4m3(l.o_wT, int(d), int(d), l.o_q, l.o_sf, st));
      DF_L(mx_quant_e4m3(l.co_wT, int(d), int(d), l.co_q, l.co_sf, st));
      DF_L(mx_quant_e4m3(l.w2T, int(d), int(f), l.w2_q, l.w2_sf, st));
    }
    return cudaSuccess;
  }
  const size_t per = al(3 * d * d) + 3 * al(d * d) + 2 * al(2 * f * d) + al(6 * 4);
  DF_TRY(f8mem.reserve(per * c.layers + 4096));
  for (auto& l : Lw) {
    l.qkv_q = (uint8_t*)f8mem.take(3 * d * d);
    l.cq_q = (uint8_t*)f8mem.take(d * d);
    l.w13_q = (uint8_t*)f8mem.take(2 * f * d);
    l.o_q = (uint8_t*)f8mem.take(d * d);
    l.co_q = (uint8_t*)f8mem.take(d * d);
    l.w2_q = (uint8_t*)f8mem.take(d * f);
    l.f8s = (float*)f8mem.take(6 * 4);
    if (!l.f8s) return cudaErrorMemoryAllocation;
    DF_L(quant_e4m3(l.qkv_wT, 3 * d * d, l.qkv_q, l.f8s + 0, st));
    DF_L(quant_e4m3(l.cq_wT, d * d, l.cq_q, l.f8s + 1, st));
    DF_L(quant_e4m3(l.w13T, 2 * f * d, l.w13_q, l.f8s + 2, st));
    DF_L(quant_e4m3(l.o_wT, d * d, l.o_q, l.f8s + 3, st));
    DF_L(quant_e4m3(l.co_wT, d * d, l.co_q, l.f8s + 4, st));
    DF_L(quant_e4m3(l.w2T, d * f, l.w2_q, l.f8s + 5, st));
  }
  return cudaSuccess;
}

void Model::destroy() {
  cudaSetDevice(device);
  wmem.release();
  ws.release();
  f8mem.release();
}

cudaError_t Model::init_weights(cudaStream_t st) {
  locs.clear();
  const int d = c.d, f = c.ffn, dt = c.d_txt, fe = c.enc_ffn;
  auto go = [&](bf16* dst, uint32_t tid, int kind, double sd, int in, int out, int layout, int ld,
                int row_off) -> cudaError_t {
    InitSpec s;
    s.seed = seed;
    s.tid = tid;
    s.kind = kind;
    s.a = float(std::sqrt(3.0) * sd);
    s.in = in;
    s.out = out;
    s.layout = layout;
    s.ld = ld;
    s.row_off = row_off;
    locs.push_back({tid, dst, in, out, layout, ld, row_off});
    g_launch_count.fetch_add(1, std::memory_order_relaxed);
    return init_tensor(dst, s, st);
  };
  auto lin = [&](bf16* dst, uint32_t tid, int in, int out) {  // W^T, K-major
    return go(dst, tid, 0, 1.0 / std::sqrt(double(in)), in, out, 1, in, 0);
  };
  auto vec = [&](bf16* dst, uint32_t tid, double sd, int n) { return go(dst, tid, 0, sd, 1, n, 0, n, 0); };
  auto gain = [&](bf16* dst, uint32_t tid, int n) { return go(dst, tid, 1, 0.1, 1, n, 0, n, 0); };
  if (stage == DF_T) {
    DF_TRY(lin(patch_wT, T_PATCH_W, Pin, d));
    DF_TRY(vec(patch_b, T_PATCH_B, 0.02, d));
    DF_TRY(lin(txt1_wT, T_TXT1_W, dt, d));
    DF_TRY(vec(txt1_b, T_TXT1_B, 0.02, d));
    DF_TRY(lin(txt2_wT, T_TXT2_W, d, d));
    DF_TRY(vec(txt2_b, T_TXT2_B, 0.02, d));
    DF_TRY(lin(temb1_wT, T_TEMB1_W, c.freq_dim, d));
    DF_TRY(vec(temb1_b, T_TEMB1_B, 0.02, d));
    DF_TRY(lin(temb2_wT, T_TEMB2_W, d, d));
    DF_TRY(vec(temb2_b, T_TEMB2_B, 0.02, d));
    DF_TRY(go(tmod_wT, T_TMOD_W, 0, 0.1 / std::sqrt(double(d)), d, 6 * d, 1, d, 0));
    DF_TRY(vec(tmod_b, T_TMOD_B, 0.02, 6 * d));
    DF_TRY(go(head_mod, T_HEAD_MOD, 0, 0.1, 2, d, 0, d, 0));
    DF_TRY(lin(head_wT, T_HEAD_W, d, P));
    DF_TRY(vec(head_b, T_HEAD_B, 0.02, P));
    if (i2v()) {
      DF_TRY(lin(img1_wT, T_IMG1_W, c.d_img, d));
      DF_TRY(vec(img1_b, T_IMG1_B, 0.02, d));
      DF_TRY(lin(img2_wT, T_IMG2_W, d, d));
      DF_TRY(vec(img2_b, T_IMG2_B, 0.02, d));
    }
    for (int l = 0; l < c.layers; ++l) {
      const uint32_t b = T_LAYER_BASE + T_LAYER_STRIDE * l;
      LayerW& w = Lw[l];
      DF_TRY(go(w.mod, b + L_MOD, 0, 0.1, 6, d, 0, d, 0));
      DF_TRY(lin(w.qkv_wT, b + L_QKV_W, d, 3 * d));
      DF_TRY(vec(w.qkv_b, b + L_QKV_B, 0.02, 3 * d));
      DF_TRY(gain(w.g_q, b + L_G_Q, d));
      DF_TRY(gain(w.g_k, b + L_G_K, d));
      DF_TRY(lin(w.o_wT, b + L_O_W, d, d));
      DF_TRY(vec(w.o_b, b + L_O_B, 0.02, d));
      DF_TRY(gain(w.g_n3, b + L_G_N3, d));
      DF_TRY(lin(w.cq_wT, b + L_CQ_W, d, d));
      DF_TRY(vec(w.cq_b, b + L_CQ_B, 0.02, d));
      DF_TRY(go(w.ckv_wT, b + L_CK_W, 0, 1.0 / std::sqrt(double(d)), d, d, 1, d, 0));
      DF_TRY(vec(w.ckv_b, b + L_CK_B, 0.02, d));
      DF_TRY(go(w.ckv_wT, b + L_CV_W, 0, 1.0 / std::sqrt(double(d)), d, d, 1, d, d));
      DF_TRY(vec(w.ckv_b + d, b + L_CV_B, 0.02, d));
      DF_TRY(gain(w.g_cq, b + L_G_CQ, d));
      DF_TRY(gain(w.g_ck, b + L_G_CK, d));
      DF_TRY(lin(w.co_wT, b + L_CO_W, d, d));
      DF_TRY(vec(w.co_b, b + L_CO_B, 0.02, d));
      DF_TRY(go(w.w13T, b + L_W1, 0, 1.0 / std::sqrt(double(d)), d, f, 2, d, 0));
      DF_TRY(go(w.b13, b + L_B1, 0, 0.02, 1, f, 2, 1, 0));
      DF_TRY(go(w.w13T, b + L_W3, 0, 1.0 / std::sqrt(double(d)), d, f, 2, d, 1));
      DF_TRY(go(w.b13, b + L_B3, 0, 0.02, 1, f, 2, 1, 1));
      DF_TRY(lin(w.w2T, b + L_W2, f, d));
      DF_TRY(vec(w.b2, b + L_B2, 0.02, d));
      if (i2v()) {  // image-token K | V stacked like the text K | V, K gain
        DF_TRY(go(w.ckvi_wT, b + L_KI_W, 0, 1.0 / std::sqrt(double(d)), d, d, 1, d, 0));
        DF_TRY(vec(w.ckvi_b, b + L_KI_B, 0.02, d));
        DF_TRY(go(w.ckvi_wT, b + L_VI_W, 0, 1.0 / std::sqrt(double(d)), d, d, 1, d, d));
        DF_TRY(vec(w.ckvi_b + d, b + L_VI_B, 0.02, d));
        DF_TRY(gain(w.g_ki, b + L_G_KI, d));
      }
    }
  } else if (stage == DF_E) {
    DF_TRY(go(emb, T_ENC_BASE + E_EMB, 0, 1.0, c.vocab, dt, 0, dt, 0));
    DF_TRY(gain(g_a, T_ENC_BASE + E_G_A, dt));
    DF_TRY(go(e_w13T, T_ENC_BASE + E_W1, 0, 1.0 / std::sqrt(double(dt)), dt, fe, 2, dt, 0));
    DF_TRY(go(e_w13T, T_ENC_BASE + E_W3, 0, 1.0 / std::sqrt(double(dt)), dt, fe, 2, dt, 1));
    DF_TRY(lin(e_w2T, T_ENC_BASE + E_W2, fe, dt));
    DF_TRY(gain(g_f, T_ENC_BASE + E_G_F, dt));
  } else {
    const int cd = c.dec_width;
    DF_TRY(go(d1_w, T_DEC_BASE + D_W1, 0, 1.0 / std::sqrt(double(c.C)), c.C, cd, 0, cd, 0));
    DF_TRY(vec(d1_b, T_DEC_BASE + D_B1, 0.02, cd));
    DF_TRY(go(d2f_w, T_DEC_BASE + D_W2F, 0, 1.0 / std::sqrt(double(cd)), cd, 192, 0, 192, 0));
    DF_TRY(vec(d2f_b, T_DEC_BASE + D_B2F, 0.02, 192));
    DF_TRY(go(d2r_w, T_DEC_BASE + D_W2R, 0, 1.0 / std::sqrt(double(cd)), cd, 768, 0, 768, 0));
    DF_TRY(vec(d2r_b, T_DEC_BASE + D_B2R, 0.02, 768));
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ helpers
cudaError_t Model::gemm(const void* A, int lda, const bf16* Wt, int ldw, int M, int Nn, int K, const Epi& e,
                        int out_f32, cudaStream_t st) {
  ProfScope ps(prof, st, cur_kind, 2.0 * M * Nn * K, 0.0);
  if (!f32()) {
    if (sk_ws && !e.sk_ws) {  // offer this instance's stream-K workspace (gemm_tc decides)
      Epi es = e;
      es.sk_ws = sk_ws;
      es.sk_flag = sk_flag;
      DF_L(gemm_tc(static_cast<const bf16*>(A), lda, Wt, ldw, M, Nn, K, es, out_f32, st));
      return cudaSuccess;
    }
    DF_L(gemm_tc(static_cast<const bf16*>(A), lda, Wt, ldw, M, Nn, K, e, out_f32, st));
  } else {
    DF_L(gemm_simt(A, 0, lda, 0, Wt, ldw, tmp, Nn, M, Nn, K, nullptr, ACT_NONE, st));
    DF_L(epi_rows(tmp, e, 1, st));
  }
  return cudaSuccess;
}

cudaError_t Model::attn(const void* Q, const void* K, const void* V, void* O, int Nq, int Nk, cudaStream_t st,
                        int B) {
  const float scale = 1.0f / std::sqrt(float(dh));
  const int Ht = B * int(c.heads);  // a stacked batch is B x heads sample-major heads
  ProfScope ps(prof, st, cur_kind, 4.0 * Nq * double(Nk) * dh * Ht, 0.0);
  if (!f32()) {
    DF_L(attn_tc((const bf16*)Q, (const bf16*)K, (const bf16*)V, (bf16*)O, Ht, Nq, Nk, dh, dhp, scale, st, c.heads));
  } else {
    DF_L(attn_simt((const float*)Q, (const float*)K, (const float*)V, (float*)O, Ht, Nq, Nk, dh, scale, st, c.heads));
  }
  return cudaSuccess;
}

cudaError_t Model::attn_qf8(int l, int Nq, int B, cudaStream_t st) {
  const LayerW& w = Lw[l];
  const int Ht = B * int(c.heads);
  const size_t n = size_t(Ht) * Nq * 128;
  {
    ProfScope ps(prof, st, K_MISC, 0.0, double(n) * 6.0);
    DF_L(qk_e4m3((const bf16*)q, n, 1.0f / w.sq, q8, st));
    DF_L(qk_e4m3((const bf16*)k, n, 1.0f / w.sk, k8, st));
  }
  // DF_ATTN_F8 (A/B): 2 (default) QK^T and PV on e4m3 (R33), 1 QK^T only (R32)
  static const int lvl = [] {
    const char* e = getenv("DF_ATTN_F8");
    return e ? atoi(e) : 2;
  }();
  if (lvl == 2) {
    ProfScope pv(prof, st, K_MISC, 0.0, double(n) * 3.0);
    DF_L(v_e4m3t((const bf16*)v, Ht, Nq, ldv8, v8s, v8t, st));
  }
  ProfScope ps(prof, st, cur_kind, 4.0 * Nq * double(Nq) * dh * Ht, 0.0);
  const float scale = w.sq * w.sk / std::sqrt(float(dh));
  if (lvl == 2) DF_L(attn_tc_f8(q8, k8, v8t, ldv8, v8s, (bf16*)o, Ht, Nq, Nq, scale, st, c.heads));
  else DF_L(attn_tc_qf8(q8, k8, (const bf16*)v, (bf16*)o, Ht, Nq, Nq, scale, st, c.heads));
  return cudaSuccess;
}

static Epi epi_base(int kind, int M, int N) {
  Epi e;
  std::memset(&e, 0, sizeof(e));
  e.kind = kind;
  e.M = M;
  e.N = N;
  return e;
}

Epi Model::heads_epi(int M, int nsec, const bf16* bias, void* o0, const bf16* g0, int rope0, void* o1,
                     const bf16* g1, int rope1, void* o2, const bf16* g2, int rope2, int Mper) const {
  Epi e = epi_base(EPI_HEADS, M, nsec * c.d);
  e.Mper = Mper > 0 ? Mper : M;
  e.bias = bias;
  e.d = c.d;
  e.heads = c.heads;
  e.dh = dh;
  e.dh_pad = dhp;
  e.nsec = nsec;
  e.sec_out[0] = o0; e.sec_gain[0] = g0; e.sec_rope[0] = rope0;
  e.sec_out[1] = o1; e.sec_gain[1] = g1; e.sec_rope[1] = rope1;
  e.sec_out[2] = o2; e.sec_gain[2] = g2; e.sec_rope[2] = rope2;
  e.rope_tab = rope;
  e.Fp = Fp; e.Hp = Hp; e.Wp = Wp;
  e.Df2 = c.rope_axes[0] / 2; e.Dh2 = c.rope_axes[1] / 2; e.Dw2 = c.rope_axes[2] / 2;
  e.eps = c.eps;
  return e;
}

cudaError_t Model::norm_f8(const float* x, int M, const float* shift, const float* scale, const bf16* gain,
                           cudaStream_t st) {
  ProfScope ps(prof, st, K_NORM, 0.0, double(M) * c.d * (4.0 + 1.0));
  if (mx()) DF_L(rmsnorm_mx(x, hq, hsf, M, int(c.d), shift, scale, gain, c.eps, st));
  else DF_L(rmsnorm_e4m3(x, hq, hs, M, int(c.d), shift, scale, gain, c.eps, st));
  return cudaSuccess;
}

cudaError_t Model::quant_f8(const void* x, int M, int K, cudaStream_t st) {
  ProfScope ps(prof, st, K_MISC, 0.0, double(M) * K * 3.0);
  if (mx()) DF_L(mx_quant_e4m3(static_cast<const bf16*>(x), M, K, hq, hsf, st));
  else DF_L(quant_rows_e4m3(static_cast<const bf16*>(x), hq, hs, M, K, st));
  return cudaSuccess;
}

cudaError_t Model::gemm_f8(const uint8_t* Wq, const float* wscale, const uint8_t* wsf, int M, int Nn, int K,
                           const Epi& e, cudaStream_t st) {
  ProfScope ps(prof, st, cur_kind, 2.0 * M * Nn * K, 0.0);
  if (mx()) DF_L(gemm_mxf8_epi(hq, hsf, Wq, wsf, M, Nn, K, e, st));
  else DF_L(gemm_e4m3_epi(hq, hs, Wq, wscale, M, Nn, K, e, st));
  return cudaSuccess;
}

cudaError_t Model::norm(const float* x, void* out, int M, int dd, const float* shift, const float* scale,
                        const bf16* gain, cudaStream_t st) {
  ProfScope ps(prof, st, K_NORM, 0.0, double(M) * dd * (4.0 + act_bytes()));
  DF_L(rmsnorm_mod(x, out, f32() ? 1 : 0, M, dd, shift, scale, gain, c.eps, st));
  return cudaSuccess;
}

// ------------------------------------------------------------------ prologue (a1)
cudaError_t Model::prepare(const void* ctx_bf16, const float* sig_host, int S, cudaStream_t st, Cond* out,
                           const void* ctx_neg_bf16, float guidance, const void* clip_bf16, const float* y_in,
                           const ChunkHook* hook) {
  const int d = c.d, Lt = c.L_txt, dt = c.d_txt, fd = c.freq_dim;
  const int Li = int(c.L_img), di = int(c.d_img);
  if (i2v() != (clip_bf16 != nullptr && y_in != nullptr)) return cudaErrorInvalidValue;  // I2V needs both
  const size_t ab = act_bytes();
  Cond& cd = *out;
  cd.S = S;
  cd.device = device;
  cd.B = ctx_neg_bf16 ? 2 : 1;
  cd.guidance = guidance;
  cd.sig.assign(sig_host, sig_host + S + 1);
  size_t kvb = size_t(c.layers) * cd.B * c.heads * Lt * dhp * ab;
  const size_t kvbi = size_t(c.layers) * cd.B * c.heads * Li * dhp * ab;         // I2V image-token K (V)
  const size_t yel = size_t(c.C_y) * c.F * c.H * c.W;
  const int Lmax = Lt > Li ? Lt : Li;
  size_t need = al((S + 1) * 4) + 2 * al(kvb) + al(size_t(S) * d * 4) + al(size_t(S) * 6 * d * 4) +
                al(size_t(S) * fd * 4) + al(size_t(S) * d * 4) + 2 * al(size_t(Lmax) * d * ab) +
                (f32() ? al(size_t(Lmax) * 2 * d * 4) : 0) + (i2v() ? 2 * al(kvbi) + al(yel * 4) : 0) + 4096;
  if (cd.mem.base && cd.mem.cap >= need) {
    cd.mem.used = 0;  // persistent cache of a T worker: reused in stream order
  } else {
    cd.mem.release();
    DF_TRY(cd.mem.reserve(need));
  }
  cd.sig_dev = (float*)cd.mem.take((S + 1) * 4);
  cd.kc = cd.mem.take(kvb);
  cd.vc = cd.mem.take(kvb);
  cd.e = (float*)cd.mem.take(size_t(S) * d * 4);
  cd.e6 = (float*)cd.mem.take(size_t(S) * 6 * d * 4);
  float* s = (float*)cd.mem.take(size_t(S) * fd * 4);
  float* t1 = (float*)cd.mem.take(size_t(S) * d * 4);
  void* c1 = cd.mem.take(size_t(Lmax) * d * ab);
  void* cp = cd.mem.take(size_t(Lmax) * d * ab);
  float* ptmp = f32() ? (float*)cd.mem.take(size_t(Lmax) * 2 * d * 4) : nullptr;
  cd.kci = cd.vci = nullptr;
  cd.y = nullptr;
  if (i2v()) {
    cd.kci = cd.mem.take(kvbi);
    cd.vci = cd.mem.take(kvbi);
    cd.y = (float*)cd.mem.take(yel * 4);
  }
  if (!cp || (i2v() && !cd.y)) return cudaErrorMemoryAllocation;
  // nothing above or in the time conditioning reads the E->T payload: with a chunk hook this
  // part runs while the payload is still in flight
  if (!f32()) DF_TRY(cudaMemsetAsync(cd.kc, 0, 2 * al(kvb), st));  // dh padding = 0
  if (i2v() && !f32()) DF_TRY(cudaMemsetAsync(cd.kci, 0, 2 * al(kvbi), st));
  if (hook && hook->shift > 0.f) {
    DF_L(sigma_schedule(cd.sig_dev, S, hook->shift, st));  // no pageable copy on a worker's enqueue path
  } else {
    DF_TRY(cudaMemcpyAsync(cd.sig_dev, sig_host, (S + 1) * 4, cudaMemcpyHostToDevice, st));
  }
  // time conditioning for all S steps (R4, R5), fp32 SIMT: the M = S rows are GEMV-like
  DF_L(sinusoid(cd.sig_dev, s, S, fd, st));
  DF_L(gemm_simt(s, 0, fd, ACT_NONE, temb1_wT, fd, t1, d, S, d, fd, temb1_b, ACT_SILU, st));
  DF_L(gemm_simt(t1, 0, d, ACT_NONE, temb2_wT, d, cd.e, d, S, d, d, temb2_b, ACT_NONE, st));
  DF_L(gemm_simt(cd.e, 0, d, ACT_SILU, tmod_wT, d, cd.e6, 6 * d, S, 6 * d, d, tmod_b, ACT_NONE, st));
  // per context b (0: prompt, 1: negative prompt): ctx' = GELU(ctx W1 + b1) W2 + b2, then
  // [K | V] = ctx' [Wck | Wcv]^T per layer, K <- headRMS * g_ck, into sample-major heads.
  // Every operation is row-wise, so rows [r0, r0 + rows) can be projected as soon as they land
  // (bn = 128 keeps a chunk on the one-CTA tiles, whose head-major epilogue takes the row
  // offset through the output pointer and the Lt-row head stride through Mper).
  const size_t per = size_t(cd.B) * c.heads * Lt * dhp * ab;     // one layer
  const size_t per_b = size_t(c.heads) * Lt * dhp * ab;          // one sample of one layer
  auto project = [&](int b, const void* ctxb, int r0, int rows) -> cudaError_t {
    const bool part = rows != Lt;
    const int bn = part ? 128 : 256;
    Epi e1 = epi_base(EPI_STORE, rows, d);
    e1.bias = txt1_b;
    e1.act = ACT_GELU;
    e1.out = (char*)c1 + size_t(r0) * d * ab;
    e1.ldo = d;
    Epi e2 = epi_base(EPI_STORE, rows, d);
    e2.bias = txt2_b;
    e2.out = (char*)cp + size_t(r0) * d * ab;
    e2.ldo = d;
    const bf16* xr = (const bf16*)ctxb + size_t(r0) * dt;
    if (!f32()) {
      DF_L(gemm_tc(xr, dt, txt1_wT, dt, rows, d, dt, e1, 0, st, bn));
      DF_L(gemm_tc((const bf16*)e1.out, d, txt2_wT, d, rows, d, d, e2, 0, st, bn));
    } else {
      DF_L(gemm_simt(ctxb, 1, dt, 0, txt1_wT, dt, ptmp, d, Lt, d, dt, nullptr, ACT_NONE, st));
      DF_L(epi_rows(ptmp, e1, 1, st));
      DF_L(gemm_simt(c1, 0, d, 0, txt2_wT, d, ptmp, d, Lt, d, d, nullptr, ACT_NONE, st));
      DF_L(epi_rows(ptmp, e2, 1, st));
    }
    for (int l = 0; l < c.layers; ++l) {
      char* kl = (char*)cd.kc + l * per + b * per_b + size_t(r0) * dhp * ab;
      char* vl = (char*)cd.vc + l * per + b * per_b + size_t(r0) * dhp * ab;
      Epi e = heads_epi(rows, 2, Lw[l].ckv_b, kl, Lw[l].g_ck, 0, vl, nullptr, 0, nullptr, nullptr, 0,
                        part ? Lt : 0);
      if (!f32()) {
        DF_L(gemm_tc((const bf16*)e2.out, d, Lw[l].ckv_wT, d, rows, 2 * d, d, e, 0, st, bn));
      } else {
        DF_L(gemm_simt(cp, 0, d, 0, Lw[l].ckv_wT, d, ptmp, 2 * d, Lt, 2 * d, d, nullptr, ACT_NONE, st));
        DF_L(epi_rows(ptmp, e, 1, st));
      }
    }
    return cudaSuccess;
  };
  // the prompt, chunk by chunk as it lands (bf16 path) or whole
  const bool chunked = hook && hook->wait && !f32() && hook->rows_per_chunk > 0 && hook->rows_per_chunk < Lt;
  int waited = 0;  // chunks [0, waited) already waited for
  if (chunked) {
    for (int r0 = 0; r0 < Lt; r0 += hook->rows_per_chunk, ++waited) {
      DF_TRY(hook->wait(hook->user, waited));
      DF_TRY(project(0, ctx_bf16, r0, std::min(hook->rows_per_chunk, Lt - r0)));
    }
  }
  if (hook && hook->wait)
    for (; waited < hook->nchunks; ++waited) DF_TRY(hook->wait(hook->user, waited));
  if (!chunked) DF_TRY(project(0, ctx_bf16, 0, Lt));
  if (cd.B == 2) DF_TRY(project(1, ctx_neg_bf16, 0, Lt));
  if (!i2v()) return cudaSuccess;
  DF_TRY(cudaMemcpyAsync(cd.y, y_in, yel * 4, cudaMemcpyDeviceToDevice, st));
  // I2V (NEXT-3, R27): img' = GELU(clip W_i1 + b_i1) W_i2 + b_i2; [Ki | Vi] = img' [Wki | Wvi]^T
  // per layer, Ki <- headRMS * g_ki (the same image conditioning for both CFG samples)
  for (int b = 0; b < cd.B; ++b) {
    Epi i1 = epi_base(EPI_STORE, Li, d);
    i1.bias = img1_b;
    i1.act = ACT_GELU;
    i1.out = c1;
    i1.ldo = d;
    Epi i2 = epi_base(EPI_STORE, Li, d);
    i2.bias = img2_b;
    i2.out = cp;
    i2.ldo = d;
    if (!f32()) {
      DF_L(gemm_tc((const bf16*)clip_bf16, di, img1_wT, di, Li, d, di, i1, 0, st));
      DF_L(gemm_tc((const bf16*)c1, d, img2_wT, d, Li, d, d, i2, 0, st));
    } else {
      DF_L(gemm_simt(clip_bf16, 1, di, 0, img1_wT, di, ptmp, d, Li, d, di, nullptr, ACT_NONE, st));
      DF_L(epi_rows(ptmp, i1, 1, st));
      DF_L(gemm_simt(c1, 0, d, 0, img2_wT, d, ptmp, d, Li, d, d, nullptr, ACT_NONE, st));
      DF_L(epi_rows(ptmp, i2, 1, st));
    }
    const size_t peri = size_t(cd.B) * c.heads * Li * dhp * ab, peri_b = size_t(c.heads) * Li * dhp * ab;
    for (int l = 0; l < c.layers; ++l) {
      void* kl = (char*)cd.kci + l * peri + b * peri_b;
      void* vl = (char*)cd.vci + l * peri + b * peri_b;
      Epi e = heads_epi(Li, 2, Lw[l].ckvi_b, kl, Lw[l].g_ki, 0, vl, nullptr, 0, nullptr, nullptr, 0);
      if (!f32()) {
        DF_L(gemm_tc((const bf16*)cp, d, Lw[l].ckvi_wT, d, Li, 2 * d, d, e, 0, st));
      } else {
        DF_L(gemm_simt(cp, 0, d, 0, Lw[l].ckvi_wT, d, ptmp, 2 * d, Li, 2 * d, d, nullptr, ACT_NONE, st));
        DF_L(epi_rows(ptmp, e, 1, st));
      }
    }
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ one block (a3-a10)
// res holds B x N rows (sample-major); every GEMM runs over all B*N rows, the heads are
// sample-major [b][h][N][dh] so attention treats the batch as B*H heads.
cudaError_t Model::block(const Cond& cd, int i, int l, float* res, cudaStream_t st) {
  const int d = c.d, f = c.ffn, Lt = c.L_txt, B = cd.B, M = B * N;
  const int of = f32() ? 1 : 0;
  const LayerW& w = Lw[l];
  const float* md = mods + size_t(l) * 6 * d;  // sh1, sc1, g1, sh2, sc2, g2
  const size_t per = size_t(B) * c.heads * Lt * dhp * act_bytes();
  // a4: h = RMSNorm(r)(1 + sc1) + sh1  (FP8 step: straight to e4m3 with row scales, R29)
  if (fp8()) DF_TRY(norm_f8(res, M, md + 0 * d, md + 1 * d, nullptr, st));
  else DF_TRY(norm(res, h, M, d, md + 0 * d, md + 1 * d, nullptr, st));
  // a5: q,k,v = heads(h Wqkv + b); qk-RMSNorm * g; RoPE3 on q, k
  {
    Epi e = heads_epi(M, 3, w.qkv_b, q, w.g_q, 1, k, w.g_k, 1, v, nullptr, 0, N);
    cur_kind = K_QKV;
    if (fp8()) DF_TRY(gemm_f8(w.qkv_q, w.f8s + 0, w.qkv_sf, M, 3 * d, d, e, st));
    else DF_TRY(gemm(h, d, w.qkv_wT, d, M, 3 * d, d, e, of, st));
  }
  // a6: self-attention (per sample); FP8 modes: QK^T on e4m3 Q and K (R32)
  cur_kind = K_ATTN_SELF;
  if (fp8()) DF_TRY(attn_qf8(l, N, B, st));
  else DF_TRY(attn(q, k, v, o, N, N, st, B));
  // a7: r += g1 * (o Wo + bo)
  {
    Epi e = epi_base(EPI_GRES, M, d);
    e.bias = w.o_b;
    cur_kind = K_O;
    e.resid = res;
    e.ldr = d;
    e.gate = md + 2 * d;
    if (fp8()) {
      DF_TRY(quant_f8(o, M, d, st));
      DF_TRY(gemm_f8(w.o_q, w.f8s + 3, w.o_sf, M, d, d, e, st));
    } else {
      DF_TRY(gemm(o, d, w.o_wT, d, M, d, d, e, of, st));
    }
  }
  // a8: cross-attention: hc = RMSNorm(r) g_n3; qc = headRMS(hc Wcq + b) g_cq; r += attn Wco + b
  if (fp8()) DF_TRY(norm_f8(res, M, nullptr, nullptr, w.g_n3, st));
  else DF_TRY(norm(res, h, M, d, nullptr, nullptr, w.g_n3, st));
  {
    Epi e = heads_epi(M, 1, w.cq_b, qc, w.g_cq, 0, nullptr, nullptr, 0, nullptr, nullptr, 0, N);
    cur_kind = K_CQ;
    if (fp8()) DF_TRY(gemm_f8(w.cq_q, w.f8s + 1, w.cq_sf, M, d, d, e, st));
    else DF_TRY(gemm(h, d, w.cq_wT, d, M, d, d, e, of, st));
  }
  cur_kind = K_ATTN_CROSS;
  DF_TRY(attn(qc, (const char*)cd.kc + l * per, (const char*)cd.vc + l * per, o, N, Lt, st, B));
  if (i2v()) {  // I2V: + softmax(qc Ki^T / sqrt(dh)) Vi over the image tokens (R27)
    const size_t peri = size_t(B) * c.heads * c.L_img * dhp * act_bytes();
    DF_TRY(attn(qc, (const char*)cd.kci + l * peri, (const char*)cd.vci + l * peri, oi, N, int(c.L_img), st, B));
    DF_L(add_into(o, oi, size_t(M) * d, of, st));
  }
  {
    Epi e = epi_base(EPI_GRES, M, d);
    e.bias = w.co_b;
    cur_kind = K_CO;
    e.resid = res;
    e.ldr = d;
    if (fp8()) {
      DF_TRY(quant_f8(o, M, d, st));
      DF_TRY(gemm_f8(w.co_q, w.f8s + 4, w.co_sf, M, d, d, e, st));
    } else {
      DF_TRY(gemm(o, d, w.co_wT, d, M, d, d, e, of, st));
    }
  }
  // a9: h2 = RMSNorm(r)(1 + sc2) + sh2
  if (fp8()) DF_TRY(norm_f8(res, M, md + 3 * d, md + 4 * d, nullptr, st));
  else DF_TRY(norm(res, h, M, d, md + 3 * d, md + 4 * d, nullptr, st));
  // a10: a = SiLU(h2 W1 + b1) * (h2 W3 + b3);  r += g2 * (a W2 + b2)
  {
    Epi e = epi_base(EPI_SWIGLU, M, 2 * f);
    e.bias = w.b13;
    cur_kind = K_UP;
    e.out = a;
    e.ldo = f;
    if (fp8()) DF_TRY(gemm_f8(w.w13_q, w.f8s + 2, w.w13_sf, M, 2 * f, d, e, st));
    else DF_TRY(gemm(h, d, w.w13T, d, M, 2 * f, d, e, of, st));
  }
  {
    Epi e = epi_base(EPI_GRES, M, d);
    e.bias = w.b2;
    cur_kind = K_DOWN;
    e.resid = res;
    e.ldr = d;
    e.gate = md + 5 * d;
    if (fp8()) {
      DF_TRY(quant_f8(a, M, f, st));
      DF_TRY(gemm_f8(w.w2_q, w.f8s + 5, w.w2_sf, M, d, f, e, st));
    } else {
      DF_TRY(gemm(a, f, w.w2T, f, M, d, f, e, of, st));
    }
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ one step (a2-a12)
cudaError_t Model::step(const Cond& cd, int i, float* x, float* v_out, cudaStream_t st, const BlockHook* bh) {
  if (prof && prof_every > 1 && i % prof_every) {  // sampled profiling: this step runs unbracketed
    Prof* p = prof;
    prof = nullptr;
    cudaError_t e = step(cd, i, x, v_out, st, bh);
    prof = p;
    return e;
  }
  const int d = c.d, B = cd.B, M = B * N;
  const int of = f32() ? 1 : 0;
  DF_L(modulations(cd.e6 + size_t(i) * 6 * d, cd.e + size_t(i) * d, layer_mods.data(), c.layers, head_mod, d, mods,
                   headmod, st));
  // a2: r = patchify(x) Wpe + bpe   (fp32 residual); a CFG batch starts both samples from it
  DF_L(patchify(x, cd.y, int(c.C_y), X, of, c.C, c.F, c.H, c.W, c.pt, c.ph, c.pw, st));  // I2V: concat(x, y)
  {
    Epi e = epi_base(EPI_STORE, N, d);
    e.bias = patch_b;
    cur_kind = K_PATCH;
    e.out = r;
    e.ldo = d;
    DF_TRY(gemm(X, Pin, patch_wT, Pin, N, d, Pin, e, 1, st));
  }
  if (B == 2) DF_TRY(cudaMemcpyAsync(r + size_t(N) * d, r, size_t(N) * d * 4, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < c.layers; ++l) DF_TRY(block(cd, i, l, r, st));
  // a11 + a12: head modulation, projection, unpatchify, Euler update fused in the epilogue
  DF_TRY(norm(r, h, M, d, headmod, headmod + d, nullptr, st));
  {
    Epi e = epi_base(EPI_EULER, M, P);
    e.bias = head_b;
    cur_kind = K_HEAD;
    e.x_lat = x;
    e.v_out = v_out;
    e.dsig = float(double(cd.sig[i + 1]) - double(cd.sig[i]));
    e.C = c.C; e.pt = c.pt; e.ph = c.ph; e.pw = c.pw; e.Hl = c.H; e.Wl = c.W; e.Fl = c.F;
    e.Hp = Hp; e.Wp = Wp;
    e.Mper = N;
    if (B == 2) e.v_batch = vbatch;  // v of both samples; guidance + Euler below
    const bool blocks = bh && bh->done && B == 1 && c.pt == 1 && bh->lb.n > 1;
    if (!blocks) {
      DF_TRY(gemm(h, d, head_wT, d, M, P, d, e, 1, st));
      if (B == 2)
        DF_L(cfg_euler(x, vbatch, v_out, size_t(c.C) * c.F * c.H * c.W, cd.guidance, e.dsig, st));
      if (bh && bh->done)
        for (int k = 0; k < bh->lb.n; ++k) DF_TRY(bh->done(bh->user, k));
    } else {
      // the head + Euler epilogue once per T->D chunk: latent rows [h0, h1) of frame f are the
      // tokens [(f Hp + h0/ph) Wp, (f Hp + h1/ph) Wp) (pt = 1); the chunk's send starts as soon
      // as its block is final (a12 -> a14)
      for (int k = 0; k < bh->lb.n; ++k) {
        int f, h0, h1;
        bh->lb.block(k, f, h0, h1);
        const int m0 = (f * Hp + h0 / c.ph) * Wp, m1 = (f * Hp + (h1 + c.ph - 1) / c.ph) * Wp;
        Epi eb = e;
        eb.M = m1 - m0;
        eb.m_base = m0;
        DF_TRY(gemm((const char*)h + size_t(m0) * d * act_bytes(), d, head_wT, d, m1 - m0, P, d, eb, 1, st));
        DF_TRY(bh->done(bh->user, k));
      }
    }
  }
  return cudaSuccess;
}

cudaError_t Model::layer(const Cond& cd, int i, int l, float* r_io, cudaStream_t st) {
  DF_L(modulations(cd.e6 + size_t(i) * 6 * c.d, cd.e + size_t(i) * c.d, layer_mods.data(), c.layers, head_mod, c.d,
                   mods, headmod, st));
  return block(cd, i, l, r_io, st);
}

// ------------------------------------------------------------------ E stand-in
cudaError_t Model::encode(const int32_t* ids, void* ctx_out, cudaStream_t st) {
  const int Lt = c.L_txt, dt = c.d_txt, fe = c.enc_ffn;
  const int of = f32() ? 1 : 0;
  DF_L(embed_rows(ids, emb, ez, Lt, dt, st));
  DF_L(rmsnorm_mod(ez, ea, of, Lt, dt, nullptr, nullptr, g_a, c.eps, st));
  Epi e1 = epi_base(EPI_SWIGLU, Lt, 2 * fe);
  e1.out = ef;
  e1.ldo = fe;
  Epi e2 = epi_base(EPI_GRES, Lt, dt);
  e2.resid = ez;
  e2.ldr = dt;
  if (!f32()) {
    DF_L(gemm_tc((const bf16*)ea, dt, e_w13T, dt, Lt, 2 * fe, dt, e1, 0, st));
    DF_L(gemm_tc((const bf16*)ef, fe, e_w2T, fe, Lt, dt, fe, e2, 0, st));
  } else {
    DF_L(gemm_simt(ea, 0, dt, 0, e_w13T, dt, etmp, 2 * fe, Lt, 2 * fe, dt, nullptr, ACT_NONE, st));
    DF_L(epi_rows(etmp, e1, 1, st));
    DF_L(gemm_simt(ef, 0, fe, 0, e_w2T, fe, etmp, dt, Lt, dt, fe, nullptr, ACT_NONE, st));
    DF_L(epi_rows(etmp, e2, 1, st));
  }
  // ctx = bf16_RNE(RMSNorm(z) g_f): the payload is bf16 by definition (R21)
  DF_L(rmsnorm_mod(ez, ctx_out, 0, Lt, dt, nullptr, nullptr, g_f, c.eps, st));
  return cudaSuccess;
}

// ------------------------------------------------------------------ D stand-in
cudaError_t Model::decode(const float* x, float* out, cudaStream_t st) {
  DF_L(decode_latent(x, out, c.C, c.F, c.H, c.W, c.dec_width, d1_w, d1_b, d2f_w, d2f_b, d2r_w, d2r_b, st));
  return cudaSuccess;
}

// One T->D chunk (latent rows [h0, h1) of frame f): every latent pixel decodes on its own, so D
// starts on the first chunk that lands (a14).
cudaError_t Model::decode_block(const float* x, float* out, const LatentBlocks& lb, int k, cudaStream_t st) {
  if (lb.n <= 1) return decode(x, out, st);
  int f, h0, h1;
  lb.block(k, f, h0, h1);
  DF_L(decode_latent_region(x, out, c.C, c.F, c.H, c.W, c.dec_width, d1_w, d1_b, d2f_w, d2f_b, d2r_w, d2r_b, f, 1,
                            h0 * int(c.W), h1 * int(c.W), st));
  return cudaSuccess;
}

}  // namespace df
