// libdf C ABI (include/df.h): context, stage instances, the chunked stage handoff
// and the asynchronous E -> T -> D pipeline workers.
//
// Pipeline (§sec:decentral-pipeline), one host worker per instance:
//   E  pops the global request ring (FAA ring), claims a receive slot on its
//      T instance (the "destination address" handshake), encodes, and hands ctx
//      off in chunks on its comm stream; it proceeds to the next request immediately
//       — the send completes on the comm stream.
//   T  waits (device-side, per chunk) for ctx, runs the prologue and S Euler steps on its
//      compute stream, claims a D slot, hands the final latent off (per-frame chunks) and
//      dequeues its next request without waiting for the send.
//   D  waits per chunk, decodes, copies to the caller's host buffer, completes.
// Request -> instance assignment is deterministic round-robin over the active instances
// of each stage (sequence number mod g_s), so per-request results never depend on load.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <set>
#include <map>
#include <cmath>
#include <string>
#include <thread>
#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "ring.h"
#include "plane.h"
#include "runtime.h"

using namespace df;

struct df_xfer {
  int src_dev = 0, dst_dev = 0;
  uint32_t nchunks = 0;
  std::vector<cudaEvent_t> chunk_ev;  // source device, source comm stream: chunk c landed
  std::vector<cudaEvent_t> ready_ev;  // source device, source comm stream: chunk c's data existed
  std::vector<cudaEvent_t> issued_ev; // source device, source comm stream: chunk c's copy issued
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // timing (source comm stream): first copy issued / last landed
  cudaEvent_t t_hash = nullptr;            // destination hash done (destination aux stream)
  unsigned long long* hash_dev = nullptr;  // [2] src, dst (pinned-mapped host)
  bool hashed = false;
  uint64_t bytes = 0;
};
using Xfer = df_xfer;

namespace {

// NVTX ranges around each stage's host-side work (header-only NVTX3: a no-op unless a tool such
// as nsys is attached), so a timeline shows the workers next to the streams they feed.
struct Nvtx {
  explicit Nvtx(const char* m) { nvtxRangePushA(m); }
  ~Nvtx() { nvtxRangePop(); }
};

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

// Host Philox4x32-10 for jitter draws and chunk permutations.
void philox_host(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = uint64_t(0xD2511F53u) * c[0], p1 = uint64_t(0xCD9E8D57u) * c[2];
    uint32_t n0 = uint32_t(p1 >> 32) ^ c[1] ^ k0, n2 = uint32_t(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = uint32_t(p1);
    c[2] = n2;
    c[3] = uint32_t(p0);
  }
}

// A receive slot on a consumer instance (the posted destination address).
struct Slot {
  void* buf = nullptr;
  cudaEvent_t consumed = nullptr;  // recorded by the consumer after its last read
  uint64_t gen = 0;                // generation counter (catches use-after-release)
};

struct SlotPool {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<int> free_list;
  std::vector<Slot> slots;
  int acquire(std::atomic<bool>& stop) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return !free_list.empty() || stop.load(); });
    if (free_list.empty()) return -1;
    int s = free_list.front();
    free_list.pop_front();
    return s;
  }
  void release(int s) {
    {
      std::lock_guard<std::mutex> lk(mu);
      slots[s].gen++;
      free_list.push_back(s);
    }
    cv.notify_all();
  }
};

struct ReqState {
  df_request req{};
  df_req_id id{};
  uint64_t seq = 0;
  std::vector<int32_t> ids, neg_ids;
  int inst[3] = {-1, -1, -1};
  double t_submit = 0, t_start[3] = {0, 0, 0}, t_end[3] = {0, 0, 0};
  cudaEvent_t ev[6] = {};  // 0,1 E start/end; 2,3 T start/end; 4,5 D start/end (each on its stage's device)
  Xfer* x[2] = {nullptr, nullptr};
  int slot[2] = {-1, -1};
  int xbuf = 0;  // T latent buffer index
  // per edge, measured by the consumer on its own device clock once its work completed
  float exposed[2] = {0, 0}, xfer[2] = {-1, -1}, overlap[2] = {0, 0};
  float stage_ms[3] = {-1, -1, -1};
  bool pre = false;       // multi-process: completion filled by the D worker
  df_completion comp{};
  std::vector<float> outcopy;  // multi-process: decoded output held in the D process
};

struct Job {
  ReqState* rs;
};

template <typename T>
struct Inbox {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<T> q;
  void push(const T& v) {
    {
      std::lock_guard<std::mutex> lk(mu);
      q.push_back(v);
    }
    cv.notify_one();
  }
  bool try_pop(T& out) {
    std::lock_guard<std::mutex> lk(mu);
    if (q.empty()) return false;
    out = q.front();
    q.pop_front();
    return true;
  }
  bool pop(T& out, std::atomic<bool>& stop) {
    return pop_until(out, [&] { return stop.load(); });
  }
  // blocks until an item arrives (true) or done() holds with the queue empty (false)
  template <class F>
  bool pop_until(T& out, F done) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return !q.empty() || done(); });
    if (q.empty()) return false;
    out = q.front();
    q.pop_front();
    return true;
  }
  size_t size() {
    std::lock_guard<std::mutex> lk(mu);
    return q.size();
  }
};

}  // namespace



// Busy time of one instance for Alg. 1's utilisation u_s: accumulated busy intervals
// plus the open one, so a sample taken mid-request credits the time already spent (a request
// credited only at its completion made u_s jump between 0 and 1 from tick to tick).
struct BusyClock {
  std::mutex mu;
  uint64_t acc = 0;
  double since = -1;
  InstStat* mirror = nullptr;  // multi-process: the same intervals in the shared plane
  void begin(double t) {
    std::lock_guard<std::mutex> lk(mu);
    if (since < 0) {
      since = t;
      if (mirror) {
        uint64_t b;
        std::memcpy(&b, &t, 8);
        mirror->busy_since.store(b, std::memory_order_release);
      }
    }
  }
  void end(double t) {
    std::lock_guard<std::mutex> lk(mu);
    if (since >= 0) {
      const uint64_t d = uint64_t(std::max(0.0, t - since) * 1e9);
      acc += d, since = -1;
      if (mirror) {
        mirror->busy_ns.fetch_add(d);
        mirror->busy_since.store(0, std::memory_order_release);
      }
    }
  }
  uint64_t sample(double t) {
    std::lock_guard<std::mutex> lk(mu);
    return acc + (since >= 0 ? uint64_t(std::max(0.0, t - since) * 1e9) : 0);
  }
};

// Consumer-side device timestamps of one in-flight transfer, all on the
// consumer's device so every difference is one clock:
//   R[c], A[c]  consumer compute stream, right before / after its wait on chunk c;
//   P[c]        probe stream, when the producer's "chunk c exists" event fired;
//   I[c], L[c]  probe stream, when chunk c's copy was issued / chunk c landed.
// exposed = sum_c max(0, A_c - max(R_c, P_c)): the consumer stalled on data in flight (injected
// delays included), not on upstream compute.  xfer = sum_c (L_c - I_c): copy time.
// overlap = max(0, L_{n-1} - A_0): how long before the last chunk landed the consumer was
// already working on chunk 0.
struct RecvClock {
  int n = 0;
  cudaStream_t probe = nullptr;
  cudaEvent_t R[PL_MAX_CHUNKS] = {}, A[PL_MAX_CHUNKS] = {}, P[PL_MAX_CHUNKS] = {};
  cudaEvent_t I[PL_MAX_CHUNKS] = {}, L[PL_MAX_CHUNKS] = {};
  unsigned long long* hash = nullptr;  // mapped pinned [2]: src (producer's, via the slot trailer), dst
};

// Producer-owned events of the transfers into one (consumer, slot) (multi-process).
struct SendSet {
  cudaEvent_t ready[PL_MAX_CHUNKS] = {}, issued[PL_MAX_CHUNKS] = {}, chunk[PL_MAX_CHUNKS] = {};
  XferEvHandles h{};
};
// The consumer's handles on a producer's SendSet (opened over IPC, or the producer's own
// events when it lives in this process).
struct OpenSet {
  bool open = false;
  bool ipc = false;
  cudaEvent_t ready[PL_MAX_CHUNKS] = {}, issued[PL_MAX_CHUNKS] = {}, chunk[PL_MAX_CHUNKS] = {};
};

struct Inst {
  int id = 0, stage = 0, device = 0;
  Model m;
  cudaStream_t compute = nullptr, comm = nullptr;
  cudaStream_t aux = nullptr;  // destination hashes and slot release (never behind an outbound send)
  std::thread worker;
  Inbox<Job> inbox;
  SlotPool slots;           // receive slots (T: ctx; D: latent); each has a 64-byte trailer
  size_t slot_cap = 0;      // payload capacity of a slot (the trailer starts here)
  // T: two latent buffers, each with a "send done" event, the per-chunk events of its last
  // step's head blocks, and the receive clock of the E->T transfer it consumed
  float* xbuf[2] = {nullptr, nullptr};
  cudaEvent_t xsent[2] = {nullptr, nullptr};
  cudaEvent_t hb_ev[2][PL_MAX_CHUNKS] = {};
  RecvClock rclk[4];        // T: per latent buffer; D: per pending decode
  int xnext = 0;
  // E: two ctx send buffers
  void* ebuf[2] = {nullptr, nullptr};
  cudaEvent_t esent[2] = {nullptr, nullptr};
  int enext = 0;
  int32_t* ids_dev = nullptr;
  // D: decoded output + pinned staging (one per pending decode)
  float* dout = nullptr;
  float* stage_host[4] = {nullptr, nullptr, nullptr, nullptr};
  BusyClock busy;
  std::atomic<uint64_t> served{0};
  // re-purposing (df_set_ratio, Alg. 1 "Apply"): producers that picked this instance and have
  // not handed it the job yet; a retiring instance drains its inbox and these, then stops
  std::atomic<int> inflight_in{0};
  std::atomic<bool> retire{false};
  // multi-process
  bool local = true;
  cudaEvent_t ipc_consumed[PL_MAX_SLOTS] = {};
  SendSet* sendset[PL_MAX_INST][PL_MAX_SLOTS] = {};  // producer: per (consumer, slot)
  OpenSet opened[PL_MAX_INST][PL_MAX_SLOTS];          // consumer: per (producer, slot)
};

struct df_ctx {
  df_graph g{};
  std::vector<std::unique_ptr<Inst>> inst;
  std::vector<int> by_stage[3];   // routing: instances of each stage (guarded by route_mu)
  std::atomic<int> active[3];     // the first active[s] of by_stage[s] receive new work
  std::mutex route_mu;
  std::atomic<bool> stop{false};
  std::atomic<bool> failed{false};
  std::string err;
  std::unique_ptr<FaaRing<ReqState*>> requests;
  std::unique_ptr<FaaRing<ReqState*>> done;
  std::mutex done_mu;
  std::condition_variable done_cv;
  std::mutex seen_mu;
  std::set<std::pair<uint64_t, uint64_t>> seen;
  std::atomic<uint64_t> seq{0};
  std::atomic<uint64_t> next_id{1};
  std::mutex ratio_mu;
  std::mutex req_mu;   // E workers share the request ring; assignment counters below
  std::atomic<uint64_t> assigned_t{0}, assigned_d{0};
  size_t ctx_bytes = 0, lat_bytes = 0, out_bytes = 0;
  // E->T payload: [ctx | clip | y | ctx_neg]; clip/y only for image-to-video graphs (NEXT-3),
  // ctx_neg only for classifier-free-guidance requests (NEXT-2)
  size_t clip_bytes = 0, y_bytes = 0;
  size_t img_bytes() const { return clip_bytes + y_bytes; }
  size_t neg_off() const { return ctx_bytes + img_bytes(); }
  size_t payload(bool cfgr) const { return ctx_bytes + img_bytes() + (cfgr ? ctx_bytes : 0); }
  std::vector<float*> sched_dev;
  // multi-process plane
  bool mp = false, seg_owner = false;
  PlaneSeg* seg = nullptr;
  std::mutex view_mu;
  struct View {
    bool open = false, remote = false;
    uint32_t gen = 0;         // the consumer's publication this view was opened at
    uint64_t slot_bytes = 0;  // payload capacity; the 64-byte trailer follows
    void* buf[PL_MAX_SLOTS] = {};
    cudaEvent_t consumed[PL_MAX_SLOTS] = {};
  };
  View views[DF_MAX_INST];
  std::vector<ReqState*> last_polled;
  // hybrid scheduler (Alg. 1)
  std::thread sched;
  std::atomic<bool> sched_stop{false};
  df_sched_cfg sched_cfg{};
  std::mutex sched_mu;
  std::deque<uint32_t> hist;               // workload keys (steps) of admitted requests
  std::map<uint32_t, double> stage_s[3];   // measured seconds per request per instance (EMA)
  std::atomic<uint64_t> qd_ns[3], qd_count[3];  // queueing delay accumulators per stage
  std::vector<df_sched_event> sched_log;
  Prof prof;
};

namespace {

thread_local std::string g_tls_msg;

df_status fail(df_ctx* c, const std::string& m, df_status s = DF_ERR_CUDA) {
  if (c) {
    c->err = m;
    if (s == DF_ERR_CUDA || s == DF_ERR_NCCL) c->failed = true;
  }
  g_tls_msg = m;
  return s;
}
#define CK(ctx, expr)                                                                      \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(ctx, std::string(#expr) + ": " + cudaGetErrorString(_e) + " " + df::tls_err); \
  } while (0)

size_t latent_elems(const df_dit_cfg& c) { return size_t(c.C) * c.F * c.H * c.W; }
bool cfg_on(float g) { return g != 0.f && g != 1.f; }
size_t out_elems(const df_dit_cfg& c) { return size_t(3) * (1 + 4 * (c.F - 1)) * 8 * c.H * 8 * c.W; }

std::vector<float> sigmas_host(int S, float shift) {
  // R13: s_i = 1 - i/S, sigma_i = shift s_i / (1 + (shift - 1) s_i)
  std::vector<float> s(S + 1);
  for (int i = 0; i <= S; ++i) {
    double si = 1.0 - double(i) / S;
    s[i] = float(shift * si / (1.0 + (shift - 1.0) * si));
  }
  return s;
}

// ---------------------------------------------------------------- handoff
// Edges that draw injected jitter (bit 0: E->T, bit 1: T->D); DF_JITTER_EDGES narrows the
// handoff-stress experiments to one edge (default both).
static unsigned jitter_edges() {
  static const unsigned m = [] {
    const char* e = getenv("DF_JITTER_EDGES");
    return e ? unsigned(atoi(e)) : 3u;
  }();
  return m;
}

// Jitter (R23): one seeded Bernoulli draw per request-edge transfer; the delay is a
// host function on the comm stream placed before chunk min(jitter_chunk, n - 1).
static bool jitter_draw(const df_ctx* ctx, uint64_t seq, uint32_t edge) {
  if (!(ctx->g.jitter_p > 0.f && ctx->g.jitter_delay_s > 0.f && (jitter_edges() >> edge & 1u))) return false;
  uint32_t c[4] = {uint32_t(seq), uint32_t(seq >> 32), edge, 3u};
  philox_host(c, uint32_t(ctx->g.jitter_seed), uint32_t(ctx->g.jitter_seed >> 32));
  return double(c[0]) < double(ctx->g.jitter_p) * 4294967296.0;
}

// ---------------------------------------------------------------- chunk plans (R22)
// A transfer is cut into n chunks: byte ranges (the E->T payload; the public df_handoff) or
// latent blocks (T->D: rows [h0, h1) of one latent frame, all channels -> a 2-D copy of C
// strided rows).  Both sides derive the same plan from the graph.
struct ChunkPlan {
  int n = 1;
  bool blocks = false;
  uint64_t bytes = 0, chunk = 0;
  LatentBlocks lb;
  void piece(int k, uint64_t& off, uint64_t& width, uint64_t& height, uint64_t& pitch) const {
    if (!blocks) {
      off = uint64_t(k) * chunk;
      width = std::min<uint64_t>(chunk, bytes - off);
      height = 1;
      pitch = width;
      return;
    }
    int f, h0, h1;
    lb.block(k, f, h0, h1);
    off = (uint64_t(f) * lb.H + h0) * lb.W * 4;
    width = uint64_t(h1 - h0) * lb.W * 4;
    height = uint64_t(lb.C);
    pitch = uint64_t(lb.F) * lb.H * lb.W * 4;
  }
};

ChunkPlan plan_bytes(uint64_t bytes, uint64_t chunk, uint64_t align) {
  ChunkPlan p;
  p.bytes = bytes;
  if (chunk == 0 || chunk >= bytes) chunk = bytes;
  chunk = (chunk + align - 1) / align * align;
  if ((bytes + chunk - 1) / chunk > uint64_t(PL_MAX_CHUNKS))
    chunk = ((bytes + PL_MAX_CHUNKS - 1) / PL_MAX_CHUNKS + align - 1) / align * align;
  p.chunk = chunk;
  p.n = int((bytes + chunk - 1) / chunk);
  return p;
}

// T->D plan: blocks of hb = floor(chunk_bytes / (C W 4)) latent rows (a multiple of ph, at
// least ph); a video chunk is one whole latent frame; chunk_bytes = 0 (or a block covering
// the latent, or pt != 1) = one chunk.
ChunkPlan plan_latent(const df_dit_cfg& c, uint64_t chunk_bytes) {
  const uint64_t total = uint64_t(c.C) * c.F * c.H * c.W * 4;
  ChunkPlan p = plan_bytes(total, 0, 16);
  if (chunk_bytes == 0 || chunk_bytes >= total || c.pt != 1) return p;
  LatentBlocks lb;
  lb.C = int(c.C), lb.F = int(c.F), lb.H = int(c.H), lb.W = int(c.W);
  int hb = int(chunk_bytes / (uint64_t(c.C) * c.W * 4));
  hb = std::max<int>(int(c.ph), hb / int(c.ph) * int(c.ph));
  if (c.F > 1 || hb >= int(c.H)) hb = int(c.H);
  lb.hb = hb;
  lb.nbh = (int(c.H) + hb - 1) / hb;
  lb.n = int(c.F) * lb.nbh;
  if (lb.n <= 1 || lb.n > PL_MAX_CHUNKS) return p;
  p.blocks = true;
  p.n = lb.n;
  p.lb = lb;
  return p;
}

// E->T plan: chunks of whole ctx rows (the prologue projects rows as they land).
ChunkPlan plan_ctx(const df_ctx* ctx, uint64_t bytes) {
  uint64_t row = uint64_t(ctx->g.dit.d_txt) * 2, a = 16;
  while (a % row) a += 16;  // lcm(16, row bytes)
  return plan_bytes(bytes, ctx->g.chunk_bytes[0], a);
}

int rows_per_chunk(const df_ctx* ctx, const ChunkPlan& p) {
  return int(p.chunk / (uint64_t(ctx->g.dit.d_txt) * 2));
}

// One chunk on `st`.  peer_dev >= 0: a single-process copy to another device.
cudaError_t copy_piece(const ChunkPlan& p, int k, void* dst, int dst_dev, const void* src, int src_dev,
                       cudaStream_t st) {
  uint64_t off, width, height, pitch;
  p.piece(k, off, width, height, pitch);
  char* d = static_cast<char*>(dst) + off;
  const char* s = static_cast<const char*>(src) + off;
  if (dst_dev == src_dev) {
    if (height == 1) return cudaMemcpyAsync(d, s, width, cudaMemcpyDeviceToDevice, st);
    return cudaMemcpy2DAsync(d, pitch, s, pitch, width, height, cudaMemcpyDeviceToDevice, st);
  }
  if (height == 1) return cudaMemcpyPeerAsync(d, dst_dev, s, src_dev, width, st);
  cudaMemcpy3DPeerParms q{};
  q.srcPtr = make_cudaPitchedPtr(const_cast<char*>(s), pitch, width, height);
  q.srcDevice = src_dev;
  q.dstPtr = make_cudaPitchedPtr(d, pitch, width, height);
  q.dstDevice = dst_dev;
  q.extent = make_cudaExtent(width, height, 1);
  return cudaMemcpy3DPeerAsync(&q, st);
}

void free_xfer(Xfer* x);

// Mapped host slots for the payload hashes, a (src, dst) pair per transfer, pooled
// process-wide (cudaHostAllocPortable: valid on every device).  A cudaHostAlloc/cudaFreeHost
// pair per transfer costs an implicit device synchronisation in the polling thread, which
// held the producer's enqueue behind any in-flight injected delay (the
// handoff-stress point).  Blocks are never returned to the driver (4 KiB each).
class HashPool {
  std::mutex mu_;
  std::vector<unsigned long long*> free_;

 public:
  unsigned long long* get() {
    std::lock_guard<std::mutex> lk(mu_);
    if (free_.empty()) {
      constexpr int kPairs = 256;
      void* p = nullptr;
      if (cudaHostAlloc(&p, kPairs * 2 * sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable) !=
          cudaSuccess)
        return nullptr;
      for (int i = kPairs - 1; i >= 0; --i) free_.push_back(static_cast<unsigned long long*>(p) + 2 * i);
    }
    unsigned long long* p = free_.back();
    free_.pop_back();
    return p;
  }
  void put(unsigned long long* p) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(p);
  }
};
HashPool& hash_pool() {
  static HashPool* pool = new HashPool;  // intentionally leaked: no CUDA calls at exit
  return *pool;
}

// Single-process transfer (df_handoff and the in-process pipeline edges).  The comm stream of
// the source instance runs, per chunk c (in order, or a seeded permutation): wait for the
// chunk's data (piece_ready[c], or the whole producer stream), record ready[c], [the injected
// delay], copy, [source hash after the last copy], record chunk[c].  No host synchronisation.
df_status do_handoff(df_ctx* ctx, const df_handoff_desc* d, const ChunkPlan& plan, cudaStream_t src_stream,
                     const cudaEvent_t* piece_ready, Xfer** out) {
  if (!d || d->src_inst < 0 || d->dst_inst < 0 || d->src_inst >= int(ctx->inst.size()) ||
      d->dst_inst >= int(ctx->inst.size()) || !d->src || !d->dst || !d->bytes || plan.n < 1)
    return fail(ctx, "df_handoff: invalid descriptor", DF_ERR_INVALID);
  Inst& S = *ctx->inst[d->src_inst];
  Inst& D = *ctx->inst[d->dst_inst];
  auto x = new Xfer();
  x->src_dev = S.device;
  x->dst_dev = D.device;
  x->bytes = d->bytes;
  x->nchunks = uint32_t(plan.n);
  CK(ctx, cudaSetDevice(S.device));
  x->chunk_ev.resize(x->nchunks);
  x->ready_ev.resize(x->nchunks);
  x->issued_ev.resize(x->nchunks);
  for (auto& e : x->chunk_ev) CK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : x->ready_ev) CK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : x->issued_ev) CK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(ctx, cudaEventCreate(&x->t0));
  CK(ctx, cudaEventCreate(&x->t1));
  if (!piece_ready) {  // comm stream runs after the producer's queued work
    cudaEvent_t ready;
    CK(ctx, cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(ctx, cudaEventRecord(ready, src_stream));
    CK(ctx, cudaStreamWaitEvent(S.comm, ready, 0));
    CK(ctx, cudaEventDestroy(ready));
  }
  const bool hash = (d->flags & DF_HASH) != 0;
  if (hash) {
    x->hash_dev = hash_pool().get();
    if (!x->hash_dev) {
      free_xfer(x);
      return fail(ctx, "df_handoff: cudaHostAlloc (hash slots) failed", DF_ERR_CUDA);
    }
    x->hash_dev[0] = x->hash_dev[1] = 0;
    x->hashed = true;
  }
  const bool delay = jitter_draw(ctx, d->seq, d->edge);
  const int jc = std::min<int>(int(ctx->g.jitter_chunk), plan.n - 1);
  std::vector<int> order(plan.n);
  for (int i = 0; i < plan.n; ++i) order[i] = i;
  if (d->flags & DF_PERMUTE) {
    for (int i = plan.n; i > 1; --i) {  // seeded Fisher-Yates
      uint32_t c[4] = {uint32_t(d->seq), uint32_t(i), 0x5045524Du, 4u};
      philox_host(c, 0x1234567u, 0x89ABCDEFu);
      std::swap(order[i - 1], order[c[0] % uint32_t(i)]);
    }
  }
  for (int k = 0; k < plan.n; ++k) {
    const int ci = order[k];
    if (piece_ready) CK(ctx, cudaStreamWaitEvent(S.comm, piece_ready[ci], 0));
    CK(ctx, cudaEventRecord(x->ready_ev[ci], S.comm));
    if (delay && k == jc) CK(ctx, delay_ns(uint64_t(double(ctx->g.jitter_delay_s) * 1e9), S.comm));
    if (k == 0) CK(ctx, cudaEventRecord(x->t0, S.comm));
    CK(ctx, cudaEventRecord(x->issued_ev[ci], S.comm));
    CK(ctx, copy_piece(plan, ci, d->dst, D.device, d->src, S.device, S.comm));
    if (hash && k == plan.n - 1) {  // every piece is final here
      g_launches->fetch_add(1);
      CK(ctx, payload_hash(d->src, d->bytes, 0, x->hash_dev, S.comm));
    }
    CK(ctx, cudaEventRecord(x->chunk_ev[ci], S.comm));
  }
  CK(ctx, cudaEventRecord(x->t1, S.comm));
  if (hash) {
    // destination hash on the destination's aux stream (never queued behind that instance's
    // own outbound sends and their injected delays)
    CK(ctx, cudaSetDevice(D.device));
    CK(ctx, cudaStreamWaitEvent(D.aux, x->t1, 0));
    g_launches->fetch_add(1);
    CK(ctx, payload_hash(d->dst, d->bytes, 0, x->hash_dev + 1, D.aux));
    CK(ctx, cudaEventCreateWithFlags(&x->t_hash, cudaEventDisableTiming));
    CK(ctx, cudaEventRecord(x->t_hash, D.aux));
    CK(ctx, cudaSetDevice(S.device));
  }
  if (d->flags & DF_SYNC) CK(ctx, cudaStreamWaitEvent(src_stream, x->t1, 0));
  *out = x;
  return DF_OK;
}

void free_xfer(Xfer* x) {
  if (!x) return;
  if (x->t_hash) cudaEventSynchronize(x->t_hash);  // the pooled hash slot is still being written
  for (auto e : x->chunk_ev) cudaEventDestroy(e);
  for (auto e : x->ready_ev) cudaEventDestroy(e);
  for (auto e : x->issued_ev) cudaEventDestroy(e);
  if (x->t0) cudaEventDestroy(x->t0);
  if (x->t1) cudaEventDestroy(x->t1);
  if (x->t_hash) cudaEventDestroy(x->t_hash);
  if (x->hash_dev) hash_pool().put(x->hash_dev);
  delete x;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = -1.f;
  if (!a || !b || cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return -1.f;
  }
  return ms;
}

// ---------------------------------------------------------------- consumer clocks
cudaError_t clock_create(RecvClock& rc) {
  DF_TRY(cudaStreamCreateWithFlags(&rc.probe, cudaStreamNonBlocking));
  for (int c = 0; c < PL_MAX_CHUNKS; ++c) {
    DF_TRY(cudaEventCreate(&rc.R[c]));
    DF_TRY(cudaEventCreate(&rc.A[c]));
    DF_TRY(cudaEventCreate(&rc.P[c]));
    DF_TRY(cudaEventCreate(&rc.I[c]));
    DF_TRY(cudaEventCreate(&rc.L[c]));
  }
  rc.hash = hash_pool().get();
  return rc.hash ? cudaSuccess : cudaErrorMemoryAllocation;
}

void clock_destroy(RecvClock& rc) {
  if (rc.probe) cudaStreamSynchronize(rc.probe);
  for (cudaEvent_t* set : {rc.R, rc.A, rc.P, rc.I, rc.L})
    for (int c = 0; c < PL_MAX_CHUNKS; ++c)
      if (set[c]) cudaEventDestroy(set[c]);
  if (rc.probe) cudaStreamDestroy(rc.probe);
  if (rc.hash) hash_pool().put(rc.hash);
  rc = RecvClock{};
}

// Probe stream: per chunk, P_c when the producer's ready[c] fired, I_c when its copy was
// issued, L_c when it landed (waits in the producer's own record order).
cudaError_t clock_probe(RecvClock& rc, int n, const cudaEvent_t* ready, const cudaEvent_t* issued,
                        const cudaEvent_t* landed) {
  rc.n = n;
  for (int c = 0; c < n; ++c) {
    DF_TRY(cudaStreamWaitEvent(rc.probe, ready[c], 0));
    DF_TRY(cudaEventRecord(rc.P[c], rc.probe));
    DF_TRY(cudaStreamWaitEvent(rc.probe, issued[c], 0));
    DF_TRY(cudaEventRecord(rc.I[c], rc.probe));
    DF_TRY(cudaStreamWaitEvent(rc.probe, landed[c], 0));
    DF_TRY(cudaEventRecord(rc.L[c], rc.probe));
  }
  return cudaSuccess;
}

// Consumer stream `st` waits for chunk c (device-side), bracketed by R_c / A_c.
cudaError_t clock_chunk(RecvClock& rc, int c, cudaStream_t st, cudaEvent_t chunk_ev) {
  DF_TRY(cudaEventRecord(rc.R[c], st));
  DF_TRY(cudaStreamWaitEvent(st, chunk_ev, 0));
  return cudaEventRecord(rc.A[c], st);
}

// After the consumer's work on this transfer completed on the device.
void clock_read(RecvClock& rc, float& exposed, float& xfer, float& overlap) {
  cudaEventSynchronize(rc.L[rc.n - 1]);
  double ex = 0, xf = 0;
  for (int c = 0; c < rc.n; ++c) {
    const float r = ev_ms(rc.R[0], rc.R[c]), a = ev_ms(rc.R[0], rc.A[c]), p = ev_ms(rc.R[0], rc.P[c]);
    ex += std::max(0.f, a - std::max(r, p));
    xf += std::max(0.f, ev_ms(rc.I[c], rc.L[c]));
  }
  exposed = float(ex);
  xfer = float(xf);
  overlap = std::max(0.f, ev_ms(rc.A[0], rc.L[rc.n - 1]));
}

struct ChunkWaitCtx {
  RecvClock* rc;
  cudaStream_t st;
  const cudaEvent_t* chunk;
};
cudaError_t chunk_wait_cb(void* u, int c) {
  auto* w = static_cast<ChunkWaitCtx*>(u);
  return clock_chunk(*w->rc, c, w->st, w->chunk[c]);
}
struct BlockDoneCtx {
  cudaEvent_t* ev;
  cudaStream_t st;
};
cudaError_t block_done_cb(void* u, int k) {
  auto* b = static_cast<BlockDoneCtx*>(u);
  return cudaEventRecord(b->ev[k], b->st);
}

// ---------------------------------------------------------------- workers
// Scheduler-visible state lives in the context (one process) or in the shared plane (one
// process per GPU, so that a controller on any rank sees and steers every rank's instances).
std::atomic<int>& active_of(df_ctx* ctx, int s) { return ctx->mp ? ctx->seg->active[s] : ctx->active[s]; }

void qd_add(df_ctx* ctx, int s, double sec) {
  std::atomic<uint64_t>* ns = ctx->mp ? ctx->seg->qd_ns : ctx->qd_ns;
  std::atomic<uint64_t>* cnt = ctx->mp ? ctx->seg->qd_count : ctx->qd_count;
  ns[s] += uint64_t(std::max(0.0, sec) * 1e9);
  cnt[s]++;
}

struct SpinLock {
  std::atomic<uint32_t>& l;
  explicit SpinLock(std::atomic<uint32_t>& x) : l(x) {
    uint32_t z = 0;
    while (!l.compare_exchange_weak(z, 1u, std::memory_order_acquire)) {
      z = 0;
      std::this_thread::yield();
    }
  }
  ~SpinLock() { l.store(0, std::memory_order_release); }
};

// Busy nanoseconds of instance i up to now (closed intervals + the open one).
uint64_t busy_sample(df_ctx* ctx, int i, double t) {
  if (!ctx->mp) return ctx->inst[i]->busy.sample(t);
  InstStat& st = ctx->seg->stat[i];
  uint64_t b = st.busy_ns.load(), sb = st.busy_since.load(std::memory_order_acquire);
  if (sb) {
    double since;
    std::memcpy(&since, &sb, 8);
    b += uint64_t(std::max(0.0, t - since) * 1e9);
  }
  return b;
}

// Routing: the instances of each stage in order (the first active[s] receive new work).  One
// process: ctx->by_stage under route_mu.  One process per GPU: the lists live in the shared
// plane (re-purposing changes them), under a spin lock.
std::vector<int> route_of(df_ctx* ctx, int s) {
  if (ctx->mp) {
    PlaneSeg* g = ctx->seg;
    SpinLock lk(g->route_lock);
    return std::vector<int>(g->route[s], g->route[s] + g->route_n[s]);
  }
  std::lock_guard<std::mutex> lk(ctx->route_mu);
  return ctx->by_stage[s];
}

// Round-robin over the active instances of a stage by request sequence number (deterministic).
// hold: the caller will hand the chosen instance a job later; the instance cannot finish
// retiring until that hand-over (release_pick) happened.
int pick(df_ctx* ctx, int stage, uint64_t seq, bool hold = false) {
  if (ctx->mp) {
    PlaneSeg* g = ctx->seg;
    SpinLock lk(g->route_lock);
    const int n = std::min<int>(g->active[stage].load(), g->route_n[stage]);
    if (n <= 0) return -1;
    const int id = g->route[stage][seq % uint64_t(n)];
    if (hold) g->inst[id].inflight++;
    return id;
  }
  std::lock_guard<std::mutex> lk(ctx->route_mu);
  int n = active_of(ctx, stage).load();
  auto& v = ctx->by_stage[stage];
  if (n <= 0 || v.empty()) return -1;
  const int id = v[seq % uint64_t(std::min<int>(n, int(v.size())))];
  if (hold) ctx->inst[id]->inflight_in++;
  return id;
}
void release_pick(df_ctx* ctx, Inst* I) {
  if (ctx->mp) {
    ctx->seg->inst[I->id].inflight--;
    return;
  }
  if (I->inflight_in.fetch_sub(1) == 1) I->inbox.cv.notify_all();
}
int inflight_of(df_ctx* ctx, const Inst* I) {
  return ctx->mp ? ctx->seg->inst[I->id].inflight.load() : I->inflight_in.load();
}

// Take instance id out of stage s's routing (no new picks after this returns) / add it back.
void route_remove(df_ctx* ctx, int s, int id) {
  if (ctx->mp) {
    PlaneSeg* g = ctx->seg;
    SpinLock lk(g->route_lock);
    int n = 0;
    for (int k = 0; k < g->route_n[s]; ++k)
      if (g->route[s][k] != id) g->route[s][n++] = g->route[s][k];
    g->route_n[s] = n;
    g->active[s] = std::min<int>(g->active[s].load(), n);
  }
  std::lock_guard<std::mutex> lk(ctx->route_mu);
  auto& v = ctx->by_stage[s];
  v.erase(std::remove(v.begin(), v.end(), id), v.end());
  ctx->active[s] = std::min<int>(ctx->active[s].load(), int(v.size()));
}
void route_add(df_ctx* ctx, int s, int id) {
  if (ctx->mp) {
    PlaneSeg* g = ctx->seg;
    SpinLock lk(g->route_lock);
    g->route[s][g->route_n[s]++] = id;
  }
  std::lock_guard<std::mutex> lk(ctx->route_mu);
  ctx->by_stage[s].push_back(id);
}

// Stage-time profile for the Eq. 6 planner: EMA of seconds per request per instance, keyed by
// the workload (steps for T; E and D do not depend on steps, tab:stage_time).
void sched_note(df_ctx* ctx, int stage, uint32_t key, double sec) {
  if (ctx->mp) {
    StageEma& e = ctx->seg->ema[stage];
    SpinLock lk(e.lock);
    for (uint32_t k = 0; k < e.n; ++k)
      if (e.key[k] == key) {
        e.sec[k] = 0.7 * e.sec[k] + 0.3 * sec;
        return;
      }
    const uint32_t k = e.n < 8 ? e.n++ : 7;
    e.key[k] = key;
    e.sec[k] = sec;
    return;
  }
  std::lock_guard<std::mutex> lk(ctx->sched_mu);
  auto it = ctx->stage_s[stage].find(key);
  if (it == ctx->stage_s[stage].end()) ctx->stage_s[stage][key] = sec;
  else it->second = 0.7 * it->second + 0.3 * sec;
}

bool stage_time(df_ctx* ctx, int stage, uint32_t key, double& out) {
  if (ctx->mp) {
    StageEma& e = ctx->seg->ema[stage];
    SpinLock lk(e.lock);
    for (uint32_t k = 0; k < e.n; ++k)
      if (e.key[k] == key) {
        out = e.sec[k];
        return true;
      }
    return false;
  }
  std::lock_guard<std::mutex> lk(ctx->sched_mu);
  auto it = ctx->stage_s[stage].find(key);
  if (it == ctx->stage_s[stage].end()) return false;
  out = it->second;
  return true;
}

// Workload keys (steps) of the last 64 admitted requests, for Alg. 1's Changed(H).
void hist_push(df_ctx* ctx, uint32_t key) {
  if (ctx->mp) {
    PlaneSeg* g = ctx->seg;
    SpinLock lk(g->hist_lock);
    g->hist[(g->hist_head + g->hist_n) % 64] = key;
    if (g->hist_n < 64) ++g->hist_n;
    else g->hist_head = (g->hist_head + 1) % 64;
    return;
  }
  std::lock_guard<std::mutex> lk(ctx->sched_mu);
  ctx->hist.push_back(key);
  while (ctx->hist.size() > 64) ctx->hist.pop_front();
}
std::vector<uint32_t> hist_keys(df_ctx* ctx) {
  std::vector<uint32_t> k;
  if (ctx->mp) {
    PlaneSeg* g = ctx->seg;
    SpinLock lk(g->hist_lock);
    for (uint32_t i = 0; i < g->hist_n; ++i) k.push_back(g->hist[(g->hist_head + i) % 64]);
    return k;
  }
  std::lock_guard<std::mutex> lk(ctx->sched_mu);
  k.assign(ctx->hist.begin(), ctx->hist.end());
  return k;
}
void hist_clear(df_ctx* ctx) {
  if (ctx->mp) {
    SpinLock lk(ctx->seg->hist_lock);
    ctx->seg->hist_n = 0;
    return;
  }
  std::lock_guard<std::mutex> lk(ctx->sched_mu);
  ctx->hist.clear();
}

void worker_fail(df_ctx* ctx, const std::string& m) {
  std::lock_guard<std::mutex> lk(ctx->done_mu);
  ctx->err = m;
  ctx->failed = true;
  ctx->done_cv.notify_all();
}

#define WK(expr)                                                                  \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      worker_fail(ctx, std::string(#expr) + ": " + cudaGetErrorString(_e) + " " + df::tls_err); \
      return;                                                                     \
    }                                                                             \
  } while (0)

// Negative prompt (CFG): tokens from the caller or the seed's negative stream, encoded into
// the second half of the send buffer.
// I2V (NEXT-3): the conditioning image's CLIP tokens and VAE latent (stand-in, R27) right
// after the prompt's ctx in the send buffer
cudaError_t encode_image(df_ctx* ctx, Inst* me, uint64_t seed, void* ebuf) {
  if (!ctx->clip_bytes) return cudaSuccess;
  const df_dit_cfg& c = me->m.c;
  char* p = static_cast<char*>(ebuf) + ctx->ctx_bytes;
  g_launches->fetch_add(1);
  return gen_image_cond(seed, reinterpret_cast<bf16*>(p), size_t(c.L_img) * c.d_img,
                        reinterpret_cast<float*>(p + ctx->clip_bytes), int(c.C_y), int(c.F), int(c.H), int(c.W),
                        me->compute);
}
const void* i2v_clip(const df_ctx* ctx, const void* cbuf) {
  return ctx->clip_bytes ? static_cast<const char*>(cbuf) + ctx->ctx_bytes : nullptr;
}
const float* i2v_y(const df_ctx* ctx, const void* cbuf) {
  return ctx->clip_bytes ? reinterpret_cast<const float*>(static_cast<const char*>(cbuf) + ctx->ctx_bytes +
                                                          ctx->clip_bytes)
                         : nullptr;
}

cudaError_t encode_negative(df_ctx* ctx, Inst* me, const int32_t* neg_ids_host, uint64_t seed, void* ebuf) {
  const size_t L = ctx->g.dit.L_txt;
  int32_t* nid = me->ids_dev + L;
  if (neg_ids_host) {
    DF_TRY(cudaMemcpyAsync(nid, neg_ids_host, L * 4, cudaMemcpyHostToDevice, me->compute));
  } else {
    g_launches->fetch_add(1);
    DF_TRY(gen_tokens(nid, int(L), int(me->m.c.vocab), seed, me->compute, 4));
  }
  return me->m.encode(nid, static_cast<char*>(ebuf) + ctx->neg_off(), me->compute);
}

// E stand-in for one request into send buffer b (tokens from the caller or the seed).
cudaError_t encode_request(df_ctx* ctx, Inst* me, ReqState* rs, int b) {
  if (!rs->ids.empty()) {
    DF_TRY(cudaMemcpyAsync(me->ids_dev, rs->ids.data(), rs->ids.size() * 4, cudaMemcpyHostToDevice, me->compute));
  } else {
    g_launches->fetch_add(1);
    DF_TRY(gen_tokens(me->ids_dev, int(me->m.c.L_txt), int(me->m.c.vocab), rs->req.seed, me->compute));
  }
  DF_TRY(me->m.encode(me->ids_dev, me->ebuf[b], me->compute));
  DF_TRY(encode_image(ctx, me, rs->req.seed, me->ebuf[b]));
  if (cfg_on(rs->req.guidance))
    DF_TRY(encode_negative(ctx, me, rs->neg_ids.empty() ? nullptr : rs->neg_ids.data(), rs->req.seed, me->ebuf[b]));
  return cudaSuccess;
}

// Whether instance I is in the active prefix of its stage's routing list (E instances pull
// from the shared request ring, so an encoder beyond g_E must stop pulling by itself).
bool routed(df_ctx* ctx, const Inst* I) {
  const std::vector<int> v = route_of(ctx, I->stage);
  const int n = std::min<int>(active_of(ctx, I->stage).load(), int(v.size()));
  for (int k = 0; k < n; ++k)
    if (v[k] == I->id) return true;
  return false;
}

void e_worker(df_ctx* ctx, Inst* me) {
  cudaSetDevice(me->device);
  while (!ctx->stop.load() && !me->retire.load()) {
    if (!routed(ctx, me)) {
      std::this_thread::sleep_for(std::chrono::microseconds(200));
      continue;
    }
    ReqState* rs = nullptr;
    {
      std::lock_guard<std::mutex> lk(ctx->req_mu);
      if (!ctx->requests->pop(rs)) rs = nullptr;
    }
    if (!rs) {
      std::this_thread::sleep_for(std::chrono::microseconds(50));
      continue;
    }
    Nvtx nv("E: encode + E->T handoff");
    rs->inst[0] = me->id;
    rs->t_start[0] = now_s();
    me->busy.begin(rs->t_start[0]);
    qd_add(ctx, 0, rs->t_start[0] - rs->t_submit);
    WK(cudaEventCreate(&rs->ev[0]));
    WK(cudaEventCreate(&rs->ev[1]));
    const int tid = pick(ctx, DF_T, rs->seq, true);
    Inst* T = ctx->inst[tid].get();
    rs->inst[1] = tid;
    int b = me->enext;
    me->enext ^= 1;
    WK(cudaStreamWaitEvent(me->compute, me->esent[b], 0));  // send buffer reuse
    WK(cudaEventRecord(rs->ev[0], me->compute));
    WK(encode_request(ctx, me, rs, b));
    WK(cudaEventRecord(rs->ev[1], me->compute));
    const bool cfgr = cfg_on(rs->req.guidance);
    // handshake: claim a receive slot on T (its posted destination address); the wait
    // for a free slot is backpressure, not E's work (Alg. 1's u_E)
    const double tw = now_s();
    me->busy.end(tw);
    int s = T->slots.acquire(ctx->stop);
    if (s < 0) return;
    const double tw1 = now_s();
    me->busy.begin(tw1);
    rs->slot[0] = s;
    WK(cudaStreamWaitEvent(me->comm, T->slots.slots[s].consumed, 0));
    df_handoff_desc d{};
    d.src_inst = me->id;
    d.dst_inst = tid;
    d.src = me->ebuf[b];
    d.dst = T->slots.slots[s].buf;
    d.bytes = ctx->payload(cfgr);
    d.chunk_bytes = ctx->g.chunk_bytes[0];
    d.flags = (ctx->g.handoff_mode & (DF_SYNC | DF_HASH));
    d.seq = rs->seq;
    d.edge = 0;
    Xfer* x = nullptr;
    if (do_handoff(ctx, &d, plan_ctx(ctx, d.bytes), me->compute, nullptr, &x) != DF_OK) {
      worker_fail(ctx, ctx->err);
      return;
    }
    rs->x[0] = x;
    WK(cudaEventRecord(me->esent[b], me->comm));
    rs->t_end[0] = now_s();
    me->busy.end(rs->t_end[0]);
    me->served++;
    sched_note(ctx, 0, 0u, (rs->t_end[0] - rs->t_start[0]) - (tw1 - tw));
    T->inbox.push(Job{rs});  // E moves on immediately
    release_pick(ctx, T);
  }
  me->busy.end(now_s());
  cudaStreamSynchronize(me->comm);  // its send buffers are read until the last copy landed
}

// T finishes a request once its compute has drained on the device: stage time and the E->T
// receive clock from the device events, profiler harvest, hand the job to D (whose stream
// waits on the T->D chunk events, so D may enqueue its decode right away).
void t_finish(df_ctx* ctx, Inst* me, ReqState* rs, Inst* D) {
  WK(cudaEventSynchronize(rs->ev[3]));
  if (me->m.prof) me->m.prof->harvest();
  rs->t_end[1] = now_s();
  const double dev_s = ev_ms(rs->ev[2], rs->ev[3]) * 1e-3;
  rs->stage_ms[1] = float(dev_s * 1e3);
  clock_read(me->rclk[rs->xbuf], rs->exposed[0], rs->xfer[0], rs->overlap[0]);
  me->served++;
  sched_note(ctx, 1, rs->req.steps, dev_s);
  D->inbox.push(Job{rs});
  release_pick(ctx, D);
}

// One T instance.  The host enqueues request r's whole prologue + S steps + T->D send,
// then finishes request r-1 (waits for its device completion): the compute stream always
// holds the next request's work, so no host round trip sits between two requests on the
// device (T starts the next request without waiting).  The prologue consumes the
// E->T payload chunk by chunk as it lands; the last step's head writes the latent block by
// block and each T->D chunk is sent as soon as its block is final.  The conditioning cache is
// one persistent buffer reused in stream order (no cudaMalloc/cudaFree per request).
void t_worker(df_ctx* ctx, Inst* me) {
  cudaSetDevice(me->device);
  Cond cd;  // persistent: Model::prepare reuses its arena when it is large enough
  ReqState* pend = nullptr;
  Inst* pendD = nullptr;
  const ChunkPlan lplan = plan_latent(ctx->g.dit, ctx->g.chunk_bytes[1]);
  for (;;) {
    Job j;
    if (pend && !me->inbox.try_pop(j)) {  // nothing queued: finish the request in flight first
      t_finish(ctx, me, pend, pendD);
      pend = nullptr;
      if (me->inbox.size() == 0) me->busy.end(now_s());
      continue;
    }
    if (!pend && !me->inbox.pop_until(j, [&] { return ctx->stop.load() || (me->retire.load() && me->inflight_in.load() == 0); }))
      break;
    ReqState* rs = j.rs;
    Nvtx nv("T: prologue + steps + T->D handoff");
    rs->t_start[1] = now_s();
    me->busy.begin(rs->t_start[1]);
    qd_add(ctx, 1, rs->t_start[1] - rs->t_end[0]);
    WK(cudaEventCreate(&rs->ev[2]));
    WK(cudaEventCreate(&rs->ev[3]));
    const int S = int(rs->req.steps);
    int b = me->xnext;
    me->xnext ^= 1;
    rs->xbuf = b;
    float* x = me->xbuf[b];
    WK(cudaStreamWaitEvent(me->compute, me->xsent[b], 0));  // latent buffer reuse after its send
    WK(cudaEventRecord(rs->ev[2], me->compute));
    g_launches->fetch_add(1);
    WK(gen_noise(x, latent_elems(me->m.c), rs->req.seed, me->compute));  // x0 does not need ctx
    // the prologue consumes ctx chunk by chunk as it lands (device-side waits)
    Xfer* x0 = rs->x[0];
    RecvClock& rc = me->rclk[b];
    WK(clock_probe(rc, int(x0->nchunks), x0->ready_ev.data(), x0->issued_ev.data(), x0->chunk_ev.data()));
    const bool cfgr = cfg_on(rs->req.guidance);
    const ChunkPlan cplan = plan_ctx(ctx, ctx->payload(cfgr));
    ChunkWaitCtx wc{&rc, me->compute, x0->chunk_ev.data()};
    ChunkHook hook;
    hook.rows_per_chunk = rows_per_chunk(ctx, cplan);
    hook.nchunks = int(x0->nchunks);
    hook.shift = rs->req.shift;
    hook.wait = chunk_wait_cb;
    hook.user = &wc;
    std::vector<float> sig = sigmas_host(S, rs->req.shift);
    const void* cbuf = me->slots.slots[rs->slot[0]].buf;
    WK(me->m.prepare(cbuf, sig.data(), S, me->compute, &cd, cfgr ? (const char*)cbuf + ctx->neg_off() : nullptr,
                     cfgr ? rs->req.guidance : 1.f, i2v_clip(ctx, cbuf), i2v_y(ctx, cbuf), &hook));
    // the slot is free once the prologue and the destination hash (aux stream) both read it
    {
      cudaEvent_t& consumed = me->slots.slots[rs->slot[0]].consumed;
      WK(cudaEventRecord(consumed, me->compute));
      WK(cudaStreamWaitEvent(me->aux, consumed, 0));
      if (x0->t_hash) WK(cudaStreamWaitEvent(me->aux, x0->t_hash, 0));
      WK(cudaEventRecord(consumed, me->aux));
    }
    me->slots.release(rs->slot[0]);  // producer's comm stream waits on `consumed` before reuse
    BlockDoneCtx bd{me->hb_ev[b], me->compute};
    BlockHook bh;
    bh.lb = lplan.lb;
    bh.done = block_done_cb;
    bh.user = &bd;
    for (int i = 0; i < S; ++i) WK(me->m.step(cd, i, x, nullptr, me->compute, i == S - 1 ? &bh : nullptr));
    WK(cudaEventRecord(rs->ev[3], me->compute));
    // r-1 drains while r is already queued behind it; finishing it before claiming a D slot
    // means this worker never holds an unsent D slot while it blocks (no slot deadlock with
    // several T instances sharing one D)
    if (pend) t_finish(ctx, me, pend, pendD);
    pend = nullptr;
    // T -> D: claim a D slot, send the final latent chunk by chunk as its blocks are final
    const int did = pick(ctx, DF_D, rs->seq, true);
    Inst* D = ctx->inst[did].get();
    rs->inst[2] = did;
    int s = D->slots.acquire(ctx->stop);
    if (s < 0) return;
    rs->slot[1] = s;
    WK(cudaStreamWaitEvent(me->comm, D->slots.slots[s].consumed, 0));
    df_handoff_desc d{};
    d.src_inst = me->id;
    d.dst_inst = did;
    d.src = x;
    d.dst = D->slots.slots[s].buf;
    d.bytes = ctx->lat_bytes;
    d.chunk_bytes = ctx->g.chunk_bytes[1];
    d.flags = (ctx->g.handoff_mode & (DF_SYNC | DF_HASH));
    d.seq = rs->seq;
    d.edge = 1;
    Xfer* xx = nullptr;
    if (do_handoff(ctx, &d, lplan, me->compute, lplan.n > 1 ? me->hb_ev[b] : nullptr, &xx) != DF_OK) {
      worker_fail(ctx, ctx->err);
      return;
    }
    rs->x[1] = xx;
    WK(cudaEventRecord(me->xsent[b], me->comm));
    pend = rs;
    pendD = D;
  }
  if (pend) t_finish(ctx, me, pend, pendD);
  me->busy.end(now_s());
  WK(cudaStreamSynchronize(me->compute));
  cd.mem.release();
}

void d_worker(df_ctx* ctx, Inst* me) {
  cudaSetDevice(me->device);
  Job j;
  const ChunkPlan lplan = plan_latent(ctx->g.dit, ctx->g.chunk_bytes[1]);
  while (me->inbox.pop_until(j, [&] { return ctx->stop.load() || (me->retire.load() && me->inflight_in.load() == 0); })) {
    ReqState* rs = j.rs;
    Nvtx nv("D: decode");
    rs->t_start[2] = now_s();
    me->busy.begin(rs->t_start[2]);
    qd_add(ctx, 2, rs->t_start[2] - rs->t_end[1]);
    WK(cudaEventCreate(&rs->ev[4]));
    WK(cudaEventCreate(&rs->ev[5]));
    Xfer* x1 = rs->x[1];
    RecvClock& rc = me->rclk[0];
    WK(clock_probe(rc, int(x1->nchunks), x1->ready_ev.data(), x1->issued_ev.data(), x1->chunk_ev.data()));
    WK(cudaEventRecord(rs->ev[4], me->compute));
    const float* lat = (const float*)me->slots.slots[rs->slot[1]].buf;
    for (uint32_t k = 0; k < x1->nchunks; ++k) {  // D decodes each chunk as it lands (a14)
      WK(clock_chunk(rc, int(k), me->compute, x1->chunk_ev[k]));
      WK(me->m.decode_block(lat, me->dout, lplan.lb, int(k), me->compute));
    }
    WK(cudaEventRecord(me->slots.slots[rs->slot[1]].consumed, me->compute));
    WK(cudaEventRecord(rs->ev[5], me->compute));
    if (rs->req.out_host)
      WK(cudaMemcpyAsync(me->stage_host[0], me->dout, ctx->out_bytes, cudaMemcpyDeviceToHost, me->compute));
    WK(cudaStreamSynchronize(me->compute));
    if (x1->t_hash) WK(cudaEventSynchronize(x1->t_hash));
    me->slots.release(rs->slot[1]);
    if (rs->req.out_host && rs->req.out_bytes >= ctx->out_bytes)
      std::memcpy(rs->req.out_host, me->stage_host[0], ctx->out_bytes);
    clock_read(rc, rs->exposed[1], rs->xfer[1], rs->overlap[1]);
    rs->stage_ms[2] = ev_ms(rs->ev[4], rs->ev[5]);
    rs->t_end[2] = now_s();
    me->busy.end(rs->t_end[2]);
    me->served++;
    sched_note(ctx, 2, 0u, rs->t_end[2] - rs->t_start[2]);
    {
      std::lock_guard<std::mutex> lk(ctx->done_mu);
      while (!ctx->done->push(rs)) std::this_thread::yield();
    }
    ctx->done_cv.notify_all();
  }
}

void fill_completion(df_ctx* ctx, ReqState* rs, df_completion* o) {
  if (rs->pre) {
    *o = rs->comp;
    return;
  }
  std::memset(o, 0, sizeof(*o));
  o->id = rs->id;
  o->status = DF_OK;
  o->user_tag = rs->req.user_tag;
  for (int k = 0; k < 3; ++k) {
    o->inst[k] = rs->inst[k];
    o->t_start[k] = rs->t_start[k];
    o->t_end[k] = rs->t_end[k];
  }
  o->t_submit = rs->t_submit;
  o->t_done = rs->t_end[2];
  o->out_view = rs->req.out_host;
  o->out_view_bytes = rs->req.out_host ? ctx->out_bytes : 0;
  o->stage_ms[0] = ev_ms(rs->ev[0], rs->ev[1]);
  o->stage_ms[1] = rs->stage_ms[1];
  o->stage_ms[2] = rs->stage_ms[2];
  for (int e = 0; e < 2; ++e) {
    Xfer* x = rs->x[e];
    if (!x) continue;
    o->xfer_ms[e] = rs->xfer[e];
    o->exposed_ms[e] = rs->exposed[e];
    o->overlap_ms[e] = rs->overlap[e];
    if (x->hashed) {
      if (x->t_hash) cudaEventSynchronize(x->t_hash);
      o->hash_src[e] = x->hash_dev[0];
      o->hash_dst[e] = x->hash_dev[1];
    }
  }
}

void free_req(ReqState* rs) {
  for (auto& e : rs->ev)
    if (e) cudaEventDestroy(e);
  free_xfer(rs->x[0]);
  free_xfer(rs->x[1]);
  delete rs;
}

}  // namespace

// ================================================================== one process per GPU
// (world > 1): instances of other ranks are reached through the shared-memory plane
// (plane.h) and CUDA IPC.  The protocol per edge, for a consumer instance c:
//   consumer: owns n_slots receive buffers (+ a 64-byte trailer each) and an interprocess
//             "consumed" event per slot; posts free slot ids in its free ring (the
//             destination-address handshake).
//   producer: pops a free slot (empty ring = backpressure), publishes the IPC handles of its
//             own ready / start / chunk events for (c, slot) into c's slot record, makes its
//             comm stream wait on `consumed`, copies the payload into the peer slot chunk by
//             chunk, hashes the source into the slot trailer (one peer store), and pushes a
//             fixed-size MetaRec into c's inbox.  Nothing on this path synchronises the host:
//             E pushes the record right away and moves on; T pushes it when its
//             compute of the request has drained (it is already enqueued by then).
//   consumer: pops the inbox, makes its compute stream wait per chunk (device-side),
//             consumes chunk by chunk, hashes the slot and reads the trailer on its stream,
//             records consumed, re-posts the slot, and reads the clocks and hashes once its
//             own completion event fired.
namespace {

void mp_sleep() { std::this_thread::sleep_for(std::chrono::microseconds(20)); }

// Producer-side view of consumer instance `ci` (opened lazily, cached).
df_ctx::View* mp_view(df_ctx* ctx, int ci) {
  df_ctx::View& v = ctx->views[ci];
  std::lock_guard<std::mutex> lk(ctx->view_mu);
  InstPlane& ip = ctx->seg->inst[ci];
  while (ip.ready.load(std::memory_order_acquire) == 0) {
    if (ctx->stop) return nullptr;
    mp_sleep();
  }
  const uint32_t gen = ip.gen.load(std::memory_order_acquire);
  if (v.open && v.gen == gen) return &v;
  if (v.open && v.remote) {  // the consumer was re-created: drop the stale mappings
    for (uint32_t s = 0; s < uint32_t(PL_MAX_SLOTS); ++s) {
      if (v.buf[s]) cudaIpcCloseMemHandle(v.buf[s]);
      if (v.consumed[s]) cudaEventDestroy(v.consumed[s]);
      v.buf[s] = nullptr, v.consumed[s] = nullptr;
    }
  }
  v.open = false;
  v.remote = false;
  v.gen = gen;
  Inst* I = ctx->inst[ci].get();
  v.slot_bytes = ip.slot_bytes;
  for (uint32_t s = 0; s < ip.n_slots; ++s) {
    if (I->local) {
      v.buf[s] = I->slots.slots[s].buf;
      v.consumed[s] = I->ipc_consumed[s];
    } else {
      if (cudaIpcOpenMemHandle(&v.buf[s], ip.slot_mem[s], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return nullptr;
      if (cudaIpcOpenEventHandle(&v.consumed[s], ip.consumed[s]) != cudaSuccess) return nullptr;
      v.remote = true;
    }
  }
  v.open = true;
  return &v;
}

// Publish a local consumer instance's slots and consumed events into the plane.
cudaError_t mp_publish(df_ctx* ctx, Inst& I, size_t slot_bytes) {
  InstPlane& ip = ctx->seg->inst[I.id];
  ip.free_slots.init();  // (a re-purposed instance publishes afresh; nothing is in flight to it)
  ip.inbox.init();
  ip.n_slots = ctx->g.n_slots;
  ip.slot_bytes = slot_bytes;
  ip.nchunks_max = PL_MAX_CHUNKS;
  for (uint32_t s = 0; s < ctx->g.n_slots; ++s) {
    DF_TRY(cudaIpcGetMemHandle(&ip.slot_mem[s], I.slots.slots[s].buf));
    DF_TRY(cudaEventCreateWithFlags(&I.ipc_consumed[s], cudaEventDisableTiming | cudaEventInterprocess));
    DF_TRY(cudaEventRecord(I.ipc_consumed[s], I.compute));
    DF_TRY(cudaIpcGetEventHandle(&ip.consumed[s], I.ipc_consumed[s]));
  }
  DF_TRY(cudaStreamSynchronize(I.compute));
  for (uint32_t s = 0; s < ctx->g.n_slots; ++s)
    while (!ip.free_slots.push(s)) mp_sleep();
  ip.gen.fetch_add(1);
  ip.ready.store(1, std::memory_order_release);
  return cudaSuccess;
}

// The producer's events for (consumer ci, slot s): created on first use on the producer's
// device (interprocess events must not time; the consumer times them on its own clock).
SendSet* send_set(Inst* me, int ci, int s) {
  SendSet*& ss = me->sendset[ci][s];
  if (ss) return ss;
  auto* n = new SendSet();
  const unsigned fl = cudaEventDisableTiming | cudaEventInterprocess;
  bool ok = true;
  for (int c = 0; c < PL_MAX_CHUNKS && ok; ++c) {
    ok = cudaEventCreateWithFlags(&n->ready[c], fl) == cudaSuccess &&
         cudaEventCreateWithFlags(&n->issued[c], fl) == cudaSuccess &&
         cudaEventCreateWithFlags(&n->chunk[c], fl) == cudaSuccess &&
         cudaIpcGetEventHandle(&n->h.ready[c], n->ready[c]) == cudaSuccess &&
         cudaIpcGetEventHandle(&n->h.issued[c], n->issued[c]) == cudaSuccess &&
         cudaIpcGetEventHandle(&n->h.chunk[c], n->chunk[c]) == cudaSuccess;
  }
  if (!ok) {
    delete n;
    return nullptr;
  }
  n->h.producer = me->id;
  ss = n;
  return ss;
}

// The consumer's handles on the events of the transfer in its slot s (published by producer p).
OpenSet* open_set(df_ctx* ctx, Inst* me, int p, int s) {
  OpenSet& os = me->opened[p][s];
  if (os.open) return &os;
  Inst* P = ctx->inst[p].get();
  if (P->local) {  // same process: the producer's own events
    SendSet* ss = P->sendset[me->id][s];
    if (!ss) return nullptr;
    for (int c = 0; c < PL_MAX_CHUNKS; ++c)
      os.ready[c] = ss->ready[c], os.issued[c] = ss->issued[c], os.chunk[c] = ss->chunk[c];
  } else {
    const XferEvHandles& h = ctx->seg->inst[me->id].xev[s];
    for (int c = 0; c < PL_MAX_CHUNKS; ++c) {
      if (cudaIpcOpenEventHandle(&os.ready[c], h.ready[c]) != cudaSuccess) return nullptr;
      if (cudaIpcOpenEventHandle(&os.issued[c], h.issued[c]) != cudaSuccess) return nullptr;
      if (cudaIpcOpenEventHandle(&os.chunk[c], h.chunk[c]) != cudaSuccess) return nullptr;
    }
    os.ipc = true;
  }
  os.open = true;
  return &os;
}

// Producer: claim a slot of consumer `ci` and enqueue the chunked copy of `src` (after
// prod's queued work, or chunk by chunk after piece_ready[c]) on the comm stream.  Fills
// m.slot / nchunks / src; the caller posts m (mp_post).  Returns false on stop / error.
bool mp_send(df_ctx* ctx, Inst* me, int ci, const void* src, const ChunkPlan& plan, cudaStream_t prod,
             const cudaEvent_t* piece_ready, MetaRec& m, uint32_t edge) {
  df_ctx::View* v = mp_view(ctx, ci);
  if (!v) {
    if (!ctx->stop) worker_fail(ctx, "mp_send: cannot open the consumer's IPC handles");
    return false;
  }
  InstPlane& ip = ctx->seg->inst[ci];
  uint32_t s;
  while (!ip.free_slots.pop(s)) {  // backpressure: no posted destination address yet
    if (ctx->stop) return false;
    mp_sleep();
  }
  auto chk = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess) worker_fail(ctx, std::string("mp_send: ") + what + ": " + cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  SendSet* ss = send_set(me, ci, int(s));
  if (!ss) return chk(cudaErrorUnknown, "interprocess events");
  ss->h.nchunks = uint32_t(plan.n);
  std::memcpy(&ip.xev[s], &ss->h, sizeof(XferEvHandles));  // read by c after it pops m (release below)
  if (!chk(cudaStreamWaitEvent(me->comm, v->consumed[s], 0), "wait consumed")) return false;
  if (!piece_ready) {
    cudaEvent_t ready;
    if (!chk(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event")) return false;
    if (!chk(cudaEventRecord(ready, prod), "record")) return false;
    if (!chk(cudaStreamWaitEvent(me->comm, ready, 0), "wait")) return false;
    cudaEventDestroy(ready);
  }
  const bool delay = jitter_draw(ctx, m.seq, edge);
  const int jc = std::min<int>(int(ctx->g.jitter_chunk), plan.n - 1);
  char* dst = static_cast<char*>(v->buf[s]);
  for (int c = 0; c < plan.n; ++c) {
    if (piece_ready && !chk(cudaStreamWaitEvent(me->comm, piece_ready[c], 0), "wait piece")) return false;
    if (!chk(cudaEventRecord(ss->ready[c], me->comm), "ready")) return false;
    if (delay && c == jc &&
        !chk(delay_ns(uint64_t(double(ctx->g.jitter_delay_s) * 1e9), me->comm), "delay"))  // P:L142, R23
      return false;
    if (!chk(cudaEventRecord(ss->issued[c], me->comm), "issued")) return false;
    // IPC-mapped peer memory is addressed from this device: same-device copy kinds
    if (!chk(copy_piece(plan, c, dst, me->device, src, me->device, me->comm), "copy")) return false;
    if (c == plan.n - 1 && (ctx->g.handoff_mode & DF_HASH)) {  // source hash into the slot trailer
      g_launches->fetch_add(1);
      auto* trailer = reinterpret_cast<unsigned long long*>(dst + v->slot_bytes);
      if (!chk(payload_hash(src, plan.bytes, 0, trailer, me->comm), "hash")) return false;
    }
    if (!chk(cudaEventRecord(ss->chunk[c], me->comm), "chunk event")) return false;
  }
  if ((ctx->g.handoff_mode & DF_SYNC) &&  // P:L151 comparison mode: the producer waits for delivery
      !chk(cudaStreamWaitEvent(prod, ss->chunk[plan.n - 1], 0), "sync"))
    return false;
  m.slot = s;
  m.nchunks = uint32_t(plan.n);
  m.chunk_bytes = uint32_t(plan.chunk);
  m.src = me->id;
  return true;
}

bool mp_post(df_ctx* ctx, int ci, const MetaRec& m) {
  InstPlane& ip = ctx->seg->inst[ci];
  while (!ip.inbox.push(m)) {
    if (ctx->stop) return false;
    mp_sleep();
  }
  return true;
}

bool mp_try_recv(df_ctx* ctx, Inst* me, MetaRec& m) { return ctx->seg->inst[me->id].inbox.pop(m); }

// Blocks for the next record; false on stop, or when this instance is retiring and nothing
// can still arrive (no producer holds a pick of it).
bool mp_recv(df_ctx* ctx, Inst* me, MetaRec& m) {
  while (!mp_try_recv(ctx, me, m)) {
    if (ctx->stop) return false;
    if (me->retire.load() && ctx->seg->inst[me->id].inflight.load() == 0 && !mp_try_recv(ctx, me, m)) return false;
    if (me->retire.load() && ctx->seg->inst[me->id].inflight.load() == 0) return true;
    mp_sleep();
  }
  return true;
}

// Consumer, after its last read of slot s on `st`: verify inputs (destination hash into
// rc.hash[1], the producer's hash from the trailer into rc.hash[0]), record consumed, re-post.
cudaError_t mp_finish_slot(df_ctx* ctx, Inst* me, RecvClock& rc, uint32_t s, uint64_t bytes, cudaStream_t st) {
  if (ctx->g.handoff_mode & DF_HASH) {
    const char* buf = static_cast<const char*>(me->slots.slots[s].buf);
    g_launches->fetch_add(1);
    DF_TRY(payload_hash(buf, bytes, 0, rc.hash + 1, st));
    DF_TRY(cudaMemcpyAsync(rc.hash, buf + me->slot_cap, 8, cudaMemcpyDeviceToHost, st));
  }
  DF_TRY(cudaEventRecord(me->ipc_consumed[s], st));
  InstPlane& ip = ctx->seg->inst[me->id];
  while (!ip.free_slots.push(s)) std::this_thread::sleep_for(std::chrono::microseconds(20));
  return cudaSuccess;
}

void mp_e_worker(df_ctx* ctx, Inst* me) {
  cudaSetDevice(me->device);
  ReqRec q;
  while (!ctx->stop.load() && !me->retire.load()) {
    if (!routed(ctx, me) || !ctx->seg->requests.pop(q)) {  // only encoders in the active prefix pull
      mp_sleep();
      continue;
    }
    auto rs = new ReqState();
    rs->seq = q.seq;
    rs->id = {q.id_lo, q.id_hi};
    rs->t_submit = q.t_submit;
    rs->req.seed = q.seed;
    rs->req.user_tag = q.user_tag;
    rs->req.steps = q.steps;
    rs->req.shift = q.shift;
    rs->req.guidance = q.guidance;
    rs->req.out_host = (q.flags & 1u) ? reinterpret_cast<void*>(uintptr_t(1)) : nullptr;  // flag only: D delivers
    const size_t L = ctx->g.dit.L_txt;
    if (q.flags & 2u) rs->ids.assign(q.tokens[0], q.tokens[0] + L);
    if (q.flags & 4u) rs->neg_ids.assign(q.tokens[1], q.tokens[1] + L);
    qd_add(ctx, 0, now_s() - q.t_submit);
    MetaRec m{};
    m.seq = rs->seq;
    m.id_lo = rs->id.lo;
    m.id_hi = rs->id.hi;
    m.seed = rs->req.seed;
    m.user_tag = rs->req.user_tag;
    m.steps = rs->req.steps;
    m.shift = rs->req.shift;
    m.inst_e = me->id;
    m.flags = rs->req.out_host ? 1u : 0u;  // bit0: deliver the decoded output
    m.t_submit = rs->t_submit;
    Nvtx nv("E: encode + E->T handoff (multi-process)");
    m.t_start_e = now_s();
    me->busy.begin(m.t_start_e);
    const int tid = pick(ctx, DF_T, rs->seq, true);
    int b = me->enext;
    me->enext ^= 1;
    WK(cudaStreamWaitEvent(me->compute, me->esent[b], 0));
    WK(encode_request(ctx, me, rs, b));
    const bool cfgr = cfg_on(rs->req.guidance);
    m.guidance = cfgr ? rs->req.guidance : 1.f;
    m.t_end_e = now_s();
    m.stage_ms_e = float((m.t_end_e - m.t_start_e) * 1e3);  // host enqueue time (E never waits)
    me->busy.end(m.t_end_e);
    sched_note(ctx, 0, 0u, m.t_end_e - m.t_start_e);
    const uint64_t bytes = ctx->payload(cfgr);
    if (!mp_send(ctx, me, tid, me->ebuf[b], plan_ctx(ctx, bytes), me->compute, nullptr, m, 0)) {
      free_req(rs);
      return;
    }
    WK(cudaEventRecord(me->esent[b], me->comm));
    const bool posted = mp_post(ctx, tid, m);  // E moves on immediately
    release_pick(ctx, ctx->inst[tid].get());
    if (!posted) {
      free_req(rs);
      return;
    }
    me->served++;
    free_req(rs);  // the request now lives in T's inbox (another process or this one)
  }
}

// Per in-flight request of a multi-process T worker (one per latent buffer).
struct MpTReq {
  MetaRec in{}, out{};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int did = -1;
  bool live = false;
};

// Finish request `r` (its compute and T->D copies are enqueued): wait for its compute, verify
// the E->T hashes, then post its record to D (D's stream waits on the chunk events).
bool mp_t_finish(df_ctx* ctx, Inst* me, MpTReq& r, int b) {
  if (cudaEventSynchronize(r.t1) != cudaSuccess) {
    worker_fail(ctx, "mp_t_worker: request compute failed");
    return false;
  }
  if (me->m.prof) me->m.prof->harvest();
  RecvClock& rc = me->rclk[b];
  MetaRec& o = r.out;
  clock_read(rc, o.exposed_e2t, o.xfer_e2t, o.overlap_e2t);
  o.stage_ms_t = ev_ms(r.t0, r.t1);
  o.t_end_t = now_s();
  if (ctx->g.handoff_mode & DF_HASH) {  // edge-0 check: the ctx we consumed is what E sent
    o.hash_src_e2t = rc.hash[0];
    o.hash_dst_e2t = rc.hash[1];
    if (rc.hash[0] != rc.hash[1]) {
      worker_fail(ctx, "mp_t_worker: E->T payload hash mismatch");
      return false;
    }
  }
  sched_note(ctx, 1, o.steps, o.stage_ms_t * 1e-3);
  me->served++;
  r.live = false;
  const bool posted = mp_post(ctx, r.did, o);
  release_pick(ctx, ctx->inst[r.did].get());
  return posted;
}

void mp_t_worker(df_ctx* ctx, Inst* me) {
  cudaSetDevice(me->device);
  MpTReq req[2];
  for (auto& r : req) {
    cudaEventCreate(&r.t0);
    cudaEventCreate(&r.t1);
  }
  Cond cd;  // persistent conditioning arena, reused in stream order (as in t_worker)
  const ChunkPlan lplan = plan_latent(ctx->g.dit, ctx->g.chunk_bytes[1]);
  int pend = -1;  // latent buffer of the request whose record is not posted yet
  for (;;) {
    MetaRec m;
    if (pend >= 0 && !mp_try_recv(ctx, me, m)) {  // nothing queued: finish the one in flight
      if (!mp_t_finish(ctx, me, req[pend], pend)) return;
      pend = -1;
      me->busy.end(now_s());
      continue;
    }
    if (pend < 0 && !mp_recv(ctx, me, m)) break;
    Nvtx nv("T: prologue + steps + T->D handoff (multi-process)");
    const double ts = now_s();
    me->busy.begin(ts);
    const int S = int(m.steps);
    const int b = me->xnext;
    me->xnext ^= 1;
    MpTReq& r = req[b];
    r.in = m;
    float* x = me->xbuf[b];
    OpenSet* os = open_set(ctx, me, m.src, int(m.slot));
    if (!os) {
      worker_fail(ctx, "mp_t_worker: cannot open the producer's events");
      return;
    }
    WK(cudaStreamWaitEvent(me->compute, me->xsent[b], 0));
    WK(cudaEventRecord(r.t0, me->compute));
    g_launches->fetch_add(1);
    WK(gen_noise(x, latent_elems(me->m.c), m.seed, me->compute));
    const bool cfgr = cfg_on(m.guidance);
    const uint64_t bytes = ctx->payload(cfgr);
    const ChunkPlan cplan = plan_ctx(ctx, bytes);
    RecvClock& rc = me->rclk[b];
    const int n = int(m.nchunks);
    WK(clock_probe(rc, n, os->ready, os->issued, os->chunk));
    ChunkWaitCtx wc{&rc, me->compute, os->chunk};
    ChunkHook hook;
    hook.rows_per_chunk = rows_per_chunk(ctx, cplan);
    hook.nchunks = n;
    hook.shift = m.shift;
    hook.wait = chunk_wait_cb;
    hook.user = &wc;
    std::vector<float> sig = sigmas_host(S, m.shift);
    const void* cbuf = me->slots.slots[m.slot].buf;
    WK(me->m.prepare(cbuf, sig.data(), S, me->compute, &cd, cfgr ? (const char*)cbuf + ctx->neg_off() : nullptr,
                     cfgr ? m.guidance : 1.f, i2v_clip(ctx, cbuf), i2v_y(ctx, cbuf), &hook));
    WK(mp_finish_slot(ctx, me, rc, m.slot, bytes, me->compute));
    BlockDoneCtx bd{me->hb_ev[b], me->compute};
    BlockHook bh;
    bh.lb = lplan.lb;
    bh.done = block_done_cb;
    bh.user = &bd;
    for (int i = 0; i < S; ++i) WK(me->m.step(cd, i, x, nullptr, me->compute, i == S - 1 ? &bh : nullptr));
    WK(cudaEventRecord(r.t1, me->compute));
    // r-1 drains while r is queued behind it; finishing (posting) it before claiming a D slot
    // for r means this worker never holds an unposted D slot while it blocks on backpressure
    if (pend >= 0 && !mp_t_finish(ctx, me, req[pend], pend)) return;
    pend = -1;
    r.out = m;
    r.out.inst_t = me->id;
    r.out.t_start_t = ts;
    r.did = pick(ctx, DF_D, m.seq, true);
    if (!mp_send(ctx, me, r.did, x, lplan, me->compute, lplan.n > 1 ? me->hb_ev[b] : nullptr, r.out, 1)) return;
    WK(cudaEventRecord(me->xsent[b], me->comm));
    r.live = true;
    pend = b;
  }
  if (pend >= 0) mp_t_finish(ctx, me, req[pend], pend);
  me->busy.end(now_s());
  cudaStreamSynchronize(me->compute);
  cd.mem.release();
  for (auto& r : req) {
    cudaEventDestroy(r.t0);
    cudaEventDestroy(r.t1);
  }
}

// The D worker keeps up to 4 decodes in flight (its host never blocks on one transfer while
// others could be enqueued) and completes them in order as their device events fire.
struct MpDReq {
  MetaRec m{};
  cudaEvent_t d0 = nullptr, d1 = nullptr, done = nullptr;
  double t_start = 0;
};

void mp_d_complete(df_ctx* ctx, Inst* me, MpDReq& q, int k) {
  RecvClock& rc = me->rclk[k];
  const MetaRec& m = q.m;
  auto rs = new ReqState();
  rs->pre = true;
  if (m.flags & 1u) {
    rs->outcopy.resize(ctx->out_bytes / 4);
    std::memcpy(rs->outcopy.data(), me->stage_host[k], ctx->out_bytes);
  }
  df_completion& o = rs->comp;
  std::memset(&o, 0, sizeof(o));
  o.id = {m.id_lo, m.id_hi};
  o.status = DF_OK;
  o.user_tag = m.user_tag;
  o.inst[0] = m.inst_e;
  o.inst[1] = m.inst_t;
  o.inst[2] = me->id;
  o.t_submit = m.t_submit;
  o.t_start[0] = m.t_start_e;
  o.t_end[0] = m.t_end_e;
  o.t_start[1] = m.t_start_t;
  o.t_end[1] = m.t_end_t;
  o.t_start[2] = q.t_start;
  o.t_end[2] = o.t_done = now_s();
  o.stage_ms[0] = m.stage_ms_e;
  o.stage_ms[1] = m.stage_ms_t;
  o.stage_ms[2] = ev_ms(q.d0, q.d1);
  o.exposed_ms[0] = m.exposed_e2t;
  o.xfer_ms[0] = m.xfer_e2t;
  o.overlap_ms[0] = m.overlap_e2t;
  clock_read(rc, o.exposed_ms[1], o.xfer_ms[1], o.overlap_ms[1]);
  if (!rs->outcopy.empty()) {
    o.out_view = rs->outcopy.data();
    o.out_view_bytes = ctx->out_bytes;
  }
  if (ctx->g.handoff_mode & DF_HASH) {
    o.hash_src[0] = m.hash_src_e2t;
    o.hash_dst[0] = m.hash_dst_e2t;
    o.hash_src[1] = rc.hash[0];
    o.hash_dst[1] = rc.hash[1];
    if (rc.hash[0] != rc.hash[1]) {
      delete rs;
      worker_fail(ctx, "mp_d_worker: T->D payload hash mismatch");
      return;
    }
  }
  me->served++;
  sched_note(ctx, 2, 0u, o.t_end[2] - o.t_start[2]);
  {
    std::lock_guard<std::mutex> lk(ctx->done_mu);
    while (!ctx->done->push(rs)) std::this_thread::yield();
  }
  ctx->done_cv.notify_all();
}

void mp_d_worker(df_ctx* ctx, Inst* me) {
  cudaSetDevice(me->device);
  constexpr int K = 4;
  MpDReq q[K];
  for (auto& e : q) {
    cudaEventCreate(&e.d0);
    cudaEventCreate(&e.d1);
    cudaEventCreateWithFlags(&e.done, cudaEventDisableTiming);
  }
  const ChunkPlan lplan = plan_latent(ctx->g.dit, ctx->g.chunk_bytes[1]);
  std::deque<int> live;  // pending decodes in enqueue order
  int next = 0;
  for (;;) {
    bool did = false;
    MetaRec m;
    if (int(live.size()) < K && mp_try_recv(ctx, me, m)) {
      did = true;
      Nvtx nv("D: decode (multi-process)");
      const int k = next;
      next = (next + 1) % K;
      MpDReq& r = q[k];
      r.m = m;
      r.t_start = now_s();
      me->busy.begin(r.t_start);
      OpenSet* os = open_set(ctx, me, m.src, int(m.slot));
      if (!os) {
        worker_fail(ctx, "mp_d_worker: cannot open the producer's events");
        return;
      }
      RecvClock& rc = me->rclk[k];
      const int n = int(m.nchunks);
      WK(clock_probe(rc, n, os->ready, os->issued, os->chunk));
      WK(cudaEventRecord(r.d0, me->compute));
      const float* lat = (const float*)me->slots.slots[m.slot].buf;
      for (int c = 0; c < n; ++c) {  // decode each chunk as it lands (a14)
        WK(clock_chunk(rc, c, me->compute, os->chunk[c]));
        WK(me->m.decode_block(lat, me->dout, lplan.lb, c, me->compute));
      }
      WK(cudaEventRecord(r.d1, me->compute));
      WK(mp_finish_slot(ctx, me, rc, m.slot, ctx->lat_bytes, me->compute));
      if (m.flags & 1u)
        WK(cudaMemcpyAsync(me->stage_host[k], me->dout, ctx->out_bytes, cudaMemcpyDeviceToHost, me->compute));
      WK(cudaEventRecord(r.done, me->compute));
      live.push_back(k);
    }
    if (!live.empty()) {
      cudaError_t e = cudaEventQuery(q[live.front()].done);
      if (e == cudaSuccess) {
        mp_d_complete(ctx, me, q[live.front()], live.front());
        live.pop_front();
        if (live.empty()) me->busy.end(now_s());
        did = true;
      } else if (e != cudaErrorNotReady) {
        worker_fail(ctx, std::string("mp_d_worker: ") + cudaGetErrorString(e));
        return;
      }
    }
    if (!did) {
      if (live.empty() && (ctx->stop.load() || (me->retire.load() && ctx->seg->inst[me->id].inflight.load() == 0 &&
                                                ctx->seg->inst[me->id].inbox.size_approx() == 0)))
        break;
      mp_sleep();
    }
  }
  for (auto& e : q) {
    cudaEventDestroy(e.d0);
    cudaEventDestroy(e.d1);
    cudaEventDestroy(e.done);
  }
}

}  // namespace


// ---------------------------------------------------------------- instance lifecycle
// One instance host: streams (created once) plus the model and buffers of its current stage.
// df_init creates every local instance this way; df_set_ratio re-purposes one (drain ->
// free -> create for the new stage -> start), "Apply", "cold starts".
namespace {

cudaError_t inst_create(df_ctx* ctx, Inst& I) {
  const df_graph* g = &ctx->g;
  const df_dit_cfg& c = g->dit;
  DF_TRY(cudaSetDevice(I.device));
  if (!I.compute) {
    int lo = 0, hi = 0;
    DF_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // T's compute stream at the lowest priority: E's and D's short kernels and every copy
    // and hash go first when instances share a GPU
    DF_TRY(cudaStreamCreateWithPriority(&I.compute, cudaStreamNonBlocking, I.stage == DF_T ? lo : hi));
    DF_TRY(cudaStreamCreateWithPriority(&I.comm, cudaStreamNonBlocking, hi));
    DF_TRY(cudaStreamCreateWithPriority(&I.aux, cudaStreamNonBlocking, hi));
  }
  DF_TRY(I.m.create(c, int(g->precision), I.device, I.stage, g->weight_seed, int(g->max_steps)));
  // T receive slots and E send buffers hold up to two ctx (prompt + negative prompt, CFG);
  // every receive slot carries a 64-byte trailer (the producer's payload hash, multi-process)
  size_t slot_bytes = I.stage == DF_T ? ctx->payload(true) : (I.stage == DF_D ? ctx->lat_bytes : 0);
  I.slot_cap = slot_bytes;
  if (slot_bytes) {
    I.slots.slots.resize(g->n_slots);
    for (uint32_t s = 0; s < g->n_slots; ++s) {
      DF_TRY(cudaMalloc(&I.slots.slots[s].buf, slot_bytes + 64));
      DF_TRY(cudaEventCreateWithFlags(&I.slots.slots[s].consumed, cudaEventDisableTiming));
      DF_TRY(cudaEventRecord(I.slots.slots[s].consumed, I.compute));
      I.slots.free_list.push_back(int(s));
    }
    for (auto& rc : I.rclk) DF_TRY(clock_create(rc));
  }
  if (I.stage == DF_T) {
    for (int b = 0; b < 2; ++b) {
      DF_TRY(cudaMalloc(&I.xbuf[b], ctx->lat_bytes));
      DF_TRY(cudaEventCreateWithFlags(&I.xsent[b], cudaEventDisableTiming));
      DF_TRY(cudaEventRecord(I.xsent[b], I.comm));
      for (int k = 0; k < PL_MAX_CHUNKS; ++k) DF_TRY(cudaEventCreateWithFlags(&I.hb_ev[b][k], cudaEventDisableTiming));
    }
  } else if (I.stage == DF_E) {
    for (int b = 0; b < 2; ++b) {
      DF_TRY(cudaMalloc(&I.ebuf[b], ctx->payload(true)));
      DF_TRY(cudaEventCreateWithFlags(&I.esent[b], cudaEventDisableTiming));
      DF_TRY(cudaEventRecord(I.esent[b], I.comm));
    }
    DF_TRY(cudaMalloc(&I.ids_dev, 2 * size_t(c.L_txt) * 4));
  } else {
    DF_TRY(cudaMalloc(&I.dout, ctx->out_bytes));
    for (int k = 0; k < 4; ++k) DF_TRY(cudaHostAlloc(&I.stage_host[k], ctx->out_bytes, cudaHostAllocPortable));
  }
  DF_TRY(cudaDeviceSynchronize());
  if (ctx->mp && slot_bytes) DF_TRY(mp_publish(ctx, I, slot_bytes));
  return cudaSuccess;
}

// Free the model and the stage buffers (not the streams); the instance must be idle.
void inst_free(Inst& I) {
  cudaSetDevice(I.device);
  if (I.compute) cudaStreamSynchronize(I.compute);
  if (I.comm) cudaStreamSynchronize(I.comm);
  if (I.aux) cudaStreamSynchronize(I.aux);
  for (auto& rc : I.rclk) clock_destroy(rc);
  for (auto& sl : I.slots.slots) {
    if (sl.buf) cudaFree(sl.buf);
    if (sl.consumed) cudaEventDestroy(sl.consumed);
  }
  {
    std::lock_guard<std::mutex> lk(I.slots.mu);
    I.slots.slots.clear();
    I.slots.free_list.clear();
  }
  for (int b = 0; b < 2; ++b) {
    if (I.xbuf[b]) cudaFree(I.xbuf[b]);
    if (I.xsent[b]) cudaEventDestroy(I.xsent[b]);
    for (int k = 0; k < PL_MAX_CHUNKS; ++k) {
      if (I.hb_ev[b][k]) cudaEventDestroy(I.hb_ev[b][k]);
      I.hb_ev[b][k] = nullptr;
    }
    if (I.ebuf[b]) cudaFree(I.ebuf[b]);
    if (I.esent[b]) cudaEventDestroy(I.esent[b]);
    I.xbuf[b] = nullptr, I.xsent[b] = nullptr, I.ebuf[b] = nullptr, I.esent[b] = nullptr;
  }
  if (I.ids_dev) cudaFree(I.ids_dev);
  if (I.dout) cudaFree(I.dout);
  I.ids_dev = nullptr, I.dout = nullptr;
  for (auto*& h : I.stage_host) {
    if (h) cudaFreeHost(h);
    h = nullptr;
  }
  I.xnext = I.enext = 0;
  I.m.destroy();
  I.m = Model{};
}

void inst_start(df_ctx* ctx, Inst* I) {
  I->retire = false;
  if (ctx->mp) {
    if (I->stage == DF_E) I->worker = std::thread(mp_e_worker, ctx, I);
    else if (I->stage == DF_T) I->worker = std::thread(mp_t_worker, ctx, I);
    else I->worker = std::thread(mp_d_worker, ctx, I);
  } else {
    if (I->stage == DF_E) I->worker = std::thread(e_worker, ctx, I);
    else if (I->stage == DF_T) I->worker = std::thread(t_worker, ctx, I);
    else I->worker = std::thread(d_worker, ctx, I);
  }
}

// Re-purpose idle-able instance I to `stage`: take it out of routing, let it drain (its inbox
// and every producer that already picked it), free its old stage, create the new one (model
// weights regenerated from the weight seed: the cold start) and start serving.  Returns the
// drain and cold-start times.
cudaError_t inst_repurpose(df_ctx* ctx, Inst* I, int stage, double& drain_s, double& cold_s) {
  const double t0 = now_s();
  route_remove(ctx, I->stage, I->id);
  I->retire = true;
  I->inbox.cv.notify_all();
  if (I->worker.joinable()) I->worker.join();
  if (ctx->mp) {  // withdraw the posted destination addresses; producers re-open on the next publication
    InstPlane& ip = ctx->seg->inst[I->id];
    ip.ready.store(0, std::memory_order_release);
    cudaSetDevice(I->device);
    cudaDeviceSynchronize();
    for (auto& e : I->ipc_consumed)
      if (e) cudaEventDestroy(e), e = nullptr;
  }
  inst_free(*I);
  const double t1 = now_s();
  I->stage = stage;
  cudaError_t e = inst_create(ctx, *I);
  if (e != cudaSuccess) return e;
  const double t2 = now_s();
  inst_start(ctx, I);
  route_add(ctx, stage, I->id);
  drain_s = t1 - t0;
  cold_s = t2 - t1;
  return cudaSuccess;
}

}  // namespace

// ---------------------------------------------------------------- shared-memory plane
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
namespace df {
static const uint64_t PLANE_MAGIC = 0xD15A6F05A11A7E01ull;
PlaneSeg* plane_open(const char* name, bool create, uint32_t world, std::string* err) {
  const size_t sz = sizeof(PlaneSeg);
  int fd = -1;
  if (create) {
    shm_unlink(name);
    fd = shm_open(name, O_CREAT | O_RDWR | O_EXCL, 0600);
    if (fd < 0 || ftruncate(fd, off_t(sz)) != 0) {
      if (err) *err = std::string("shm_open/ftruncate(create) failed for ") + name;
      if (fd >= 0) close(fd);
      return nullptr;
    }
  } else {
    for (int t = 0; t < 120000 && fd < 0; ++t) {  // rank 0 may not have created it yet (<= 120 s)
      fd = shm_open(name, O_RDWR, 0600);
      if (fd < 0) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (fd < 0) {
      if (err) *err = std::string("shm_open(attach) timed out for ") + name;
      return nullptr;
    }
    struct stat st;
    for (int t = 0; t < 120000; ++t) {
      if (fstat(fd, &st) == 0 && size_t(st.st_size) >= sz) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  void* p = mmap(nullptr, sz, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    if (err) *err = "mmap failed";
    return nullptr;
  }
  auto seg = static_cast<PlaneSeg*>(p);
  if (create) {
    std::memset(p, 0, sz);
    seg->world = world;
    for (int i = 0; i < PL_MAX_INST; ++i) {
      seg->inst[i].free_slots.init();
      seg->inst[i].inbox.init();
      seg->stat[i].busy_ns = 0;
      seg->stat[i].busy_since = 0;
    }
    seg->requests.init();
    seg->magic.store(PLANE_MAGIC, std::memory_order_release);
  } else {
    for (int t = 0; t < 120000 && seg->magic.load(std::memory_order_acquire) != PLANE_MAGIC; ++t)
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    if (seg->magic.load() != PLANE_MAGIC) {
      if (err) *err = "plane segment never initialised";
      munmap(p, sz);
      return nullptr;
    }
  }
  seg->attached.fetch_add(1);
  return seg;
}
void plane_close(PlaneSeg* seg, const char* name, bool owner) {
  if (!seg) return;
  munmap(seg, sizeof(PlaneSeg));
  if (owner) shm_unlink(name);
}
}  // namespace df

// ================================================================== hybrid scheduler (Alg. 1)
namespace {

double eq6(const uint32_t g[3], const double T[3]) {
  double q = 1e300;
  for (int s = 0; s < 3; ++s) q = std::min(q, double(g[s]) / T[s]);
  return q;
}

bool plan_ratio(uint32_t G, const double T[3], const uint32_t* cur, int32_t budget, const uint32_t* cap,
                uint32_t out[3]) {
  bool found = false;
  double bq = 0;
  uint32_t best[3] = {0, 0, 0};
  for (uint32_t e = 1; e + 2 <= G; ++e)
    for (uint32_t t = 1; e + t + 1 <= G; ++t)
      for (uint32_t d = 1; e + t + d <= G; ++d) {
        if (cap && (e > cap[0] || t > cap[1] || d > cap[2])) continue;
        if (cur && budget >= 0) {
          int64_t mv = std::llabs(int64_t(e) - cur[0]) + std::llabs(int64_t(t) - cur[1]) + std::llabs(int64_t(d) - cur[2]);
          if (mv > budget) continue;
        }
        uint32_t g[3] = {e, t, d};
        double q = eq6(g, T);
        // ties (to 1e-12 relative): fewer GPUs, then larger g_T, then larger g_D
        bool better = !found || q > bq * (1 + 1e-12);
        if (!better && found && std::fabs(q - bq) <= bq * 1e-12) {
          uint32_t sn = e + t + d, sb = best[0] + best[1] + best[2];
          better = sn < sb || (sn == sb && (t > best[1] || (t == best[1] && d > best[2])));
        }
        if (better) {
          found = true;
          bq = q;
          best[0] = e, best[1] = t, best[2] = d;
        }
      }
  if (found) std::memcpy(out, best, sizeof(best));
  return found;
}

void react(const df_sched_cfg& c, const df_sched_metrics& now, const df_sched_metrics* prev, const uint32_t g[3],
           int32_t out[3]) {
  const uint32_t total = g[0] + g[1] + g[2];
  for (int s = 0; s < 3; ++s) {
    out[s] = 0;
    if (now.u[s] > c.U_high && now.q[s] > c.Q_high && prev && now.d[s] > prev->d[s]) {
      out[s] = (c.G == 0 || total < c.G) ? 1 : 0;
    } else if (now.u[s] < c.U_low && now.q[s] == 0) {
      out[s] = g[s] >= 2 ? -1 : 0;
    }
  }
}

bool changed(const uint32_t* k, uint32_t n) {
  if (n < 4) return false;
  uint32_t cut = n - std::max<uint32_t>(1, n / 4);
  auto mode = [&](uint32_t a, uint32_t b, bool& tie) {
    std::map<uint32_t, uint32_t> cnt;
    for (uint32_t i = a; i < b; ++i) cnt[k[i]]++;
    uint32_t bk = 0, bc = 0, second = 0;
    for (auto& kv : cnt) {
      if (kv.second > bc) {
        second = bc;
        bc = kv.second;
        bk = kv.first;
      } else if (kv.second > second) {
        second = kv.second;
      }
    }
    tie = cnt.size() > 1 && second == bc;
    return bk;
  };
  bool t1 = false, t2 = false;
  uint32_t a = mode(0, cut, t1), b = mode(cut, n, t2);
  return !t1 && !t2 && a != b;
}

// Controller: every delta, measure u/q/d per stage from the live pipeline and apply Alg. 1.
void sched_loop(df_ctx* ctx) {
  df_sched_cfg c = ctx->sched_cfg;
  df_sched_metrics prev{};
  bool have_prev = false;
  std::vector<uint64_t> busy0(ctx->inst.size());
  for (size_t i = 0; i < ctx->inst.size(); ++i) busy0[i] = busy_sample(ctx, int(i), now_s());
  double t_prev = now_s();
  while (!ctx->sched_stop.load()) {
    for (int k = 0; k < int(c.delta_s * 100) && !ctx->sched_stop.load(); ++k)
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    if (ctx->sched_stop.load()) break;
    const double t = now_s(), win = std::max(1e-6, t - t_prev);
    t_prev = t;
    df_sched_metrics m{};
    uint32_t g[3];
    for (int s = 0; s < 3; ++s) g[s] = uint32_t(active_of(ctx, s).load());
    for (int s = 0; s < 3; ++s) {
      const std::vector<int> ids = route_of(ctx, s);
      double busy = 0;
      for (size_t j = 0; j < ids.size(); ++j) {
        const uint64_t b = busy_sample(ctx, ids[j], t);
        if (j < g[s]) busy += double(b - busy0[ids[j]]) * 1e-9;
        busy0[ids[j]] = b;
        if (j < g[s] && s != DF_E)
          m.q[s] += uint32_t(ctx->mp ? ctx->seg->inst[ids[j]].inbox.size_approx() : ctx->inst[ids[j]]->inbox.size());
      }
      if (s == DF_E) m.q[s] = uint32_t(ctx->mp ? ctx->seg->requests.size_approx() : ctx->requests->size_approx());
      m.u[s] = float(std::min(1.0, busy / (double(g[s]) * win)));
      std::atomic<uint64_t>* qn = ctx->mp ? ctx->seg->qd_ns : ctx->qd_ns;
      std::atomic<uint64_t>* qc = ctx->mp ? ctx->seg->qd_count : ctx->qd_count;
      uint64_t n = qc[s].exchange(0);
      uint64_t tot = qn[s].exchange(0);
      m.d[s] = n ? float(double(tot) * 1e-9 / double(n)) : 0.f;
    }
    df_sched_event ev{};
    ev.t = t;
    ev.m = m;
    // workload change -> predictive reconfiguration (Alg. 1 lines 6-10)
    std::vector<uint32_t> keys = hist_keys(ctx);
    bool reconf = false;
    if (changed(keys.data(), uint32_t(keys.size()))) {
      uint32_t key = keys.back();
      double T[3];
      bool ok = true;
      for (int s = 0; s < 3; ++s) {
        ok = ok && stage_time(ctx, s, s == DF_T ? key : 0u, T[s]);
        if (ok) T[s] = std::max(1e-6, T[s]);
      }
      // any allocation over the instance hosts: df_set_ratio re-purposes instances between
      // stages when a stage needs more than it has (single process); across processes the
      // allocation stays within each stage's instances (activation / deactivation only)
      const uint32_t G = c.G ? std::min<uint32_t>(c.G, uint32_t(ctx->inst.size())) : uint32_t(ctx->inst.size());
      uint32_t tgt[3];
      if (ok && plan_ratio(G, T, g, c.move_budget, nullptr, tgt) && std::memcmp(tgt, g, sizeof(g)) != 0 &&
          df_set_ratio(ctx, tgt[0], tgt[1], tgt[2]) == DF_OK) {
        ev.action = 3;
        std::memcpy(ev.g, tgt, sizeof(tgt));
        reconf = true;
        hist_clear(ctx);  // the new regime starts a fresh history
      }
    }
    if (!reconf) {  // reactive rule (lines 11-17); one action per tick
      int32_t dlt[3];
      df_sched_cfg cc = c;
      if (!cc.G) cc.G = uint32_t(ctx->inst.size());
      react(cc, m, have_prev ? &prev : nullptr, g, dlt);
      uint32_t ng[3] = {g[0], g[1], g[2]};
      const uint32_t hosts = uint32_t(ctx->inst.size());
      for (int s = 0; s < 3 && ev.action == 0; ++s) {
        if (dlt[s] > 0 && ng[0] + ng[1] + ng[2] < hosts) {
          ng[s]++;
          ev.action = 1;
          ev.stage = s;
        } else if (dlt[s] < 0) {
          ng[s]--;
          ev.action = 2;
          ev.stage = s;
        }
      }
      if (ev.action && df_set_ratio(ctx, ng[0], ng[1], ng[2]) != DF_OK) {  // e.g. no local donor (one process per GPU)
        ev.action = 0;
        std::memcpy(ng, g, sizeof(g));
      }
      std::memcpy(ev.g, ng, sizeof(ng));
    }
    prev = m;
    have_prev = true;
    std::lock_guard<std::mutex> lk(ctx->sched_mu);
    ctx->sched_log.push_back(ev);
  }
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* df_last_error(const df_ctx* ctx) {
  if (ctx && !ctx->err.empty()) return ctx->err.c_str();
  return g_tls_msg.c_str();
}

uint64_t df_launch_count(const df_ctx*) { return g_launches->load(); }

df_status df_plan_ratio(uint32_t G, const double T[3], const uint32_t* cur, int32_t budget, uint32_t out[3]) {
  if (!T || !out || G < 3 || !(T[0] > 0 && T[1] > 0 && T[2] > 0)) return DF_ERR_INVALID;
  return plan_ratio(G, T, cur, cur ? budget : -1, nullptr, out) ? DF_OK : DF_ERR_CAPACITY;
}

df_status df_sched_react(const df_sched_cfg* cfg, const df_sched_metrics* now, const df_sched_metrics* prev,
                         const uint32_t g[3], int32_t out[3]) {
  if (!cfg || !now || !g || !out) return DF_ERR_INVALID;
  react(*cfg, *now, prev, g, out);
  return DF_OK;
}

int32_t df_sched_changed(const uint32_t* keys, uint32_t n) { return keys && changed(keys, n) ? 1 : 0; }

df_status df_sched_start(df_ctx* ctx, const df_sched_cfg* cfg) {
  if (!ctx || !cfg || !(cfg->delta_s > 0.f) || !(cfg->U_low < cfg->U_high)) return DF_ERR_INVALID;
  if (ctx->sched.joinable()) return fail(ctx, "df_sched_start: already running", DF_ERR_STATE);
  ctx->sched_cfg = *cfg;
  ctx->sched_stop = false;
  ctx->sched = std::thread(sched_loop, ctx);
  return DF_OK;
}

df_status df_sched_stop(df_ctx* ctx) {
  if (!ctx) return DF_ERR_INVALID;
  ctx->sched_stop = true;
  if (ctx->sched.joinable()) ctx->sched.join();
  return DF_OK;
}

df_status df_sched_log(df_ctx* ctx, df_sched_event* out, uint32_t max, uint32_t* n_out) {
  if (!ctx || !n_out) return DF_ERR_INVALID;
  std::lock_guard<std::mutex> lk(ctx->sched_mu);
  uint32_t n = std::min<uint32_t>(max, uint32_t(ctx->sched_log.size()));
  for (uint32_t i = 0; i < n && out; ++i) out[i] = ctx->sched_log[i];
  *n_out = out ? n : uint32_t(ctx->sched_log.size());
  return DF_OK;
}

df_status df_chunk_plan(const df_graph* g, uint32_t edge, uint64_t bytes, uint32_t* n, uint64_t* off,
                        uint64_t* width, uint64_t* height, uint64_t* pitch, uint32_t max) {
  if (!g || !n || edge > 1 || (max && (!off || !width || !height || !pitch))) return DF_ERR_INVALID;
  ChunkPlan p;
  if (edge == 0) {
    uint64_t row = uint64_t(g->dit.d_txt) * 2, a = 16;
    if (!row || !bytes) return DF_ERR_INVALID;
    while (a % row) a += 16;
    p = plan_bytes(bytes, g->chunk_bytes[0], a);
  } else {
    p = plan_latent(g->dit, g->chunk_bytes[1]);
  }
  *n = uint32_t(p.n);
  for (uint32_t k = 0; k < std::min<uint32_t>(max, uint32_t(p.n)); ++k) p.piece(int(k), off[k], width[k], height[k], pitch[k]);
  return DF_OK;
}

df_status df_ring_selftest(const char* name, int32_t role, uint64_t n, uint64_t* checksum, int32_t* fifo_ok) {
  if (!name || !name[0] || (role != 0 && role != 1)) return DF_ERR_INVALID;
  std::string err;
  PlaneSeg* seg = plane_open(name, role == 0, 2, &err);
  if (!seg) return fail(nullptr, "df_ring_selftest: " + err, DF_ERR_STATE);
  auto& inbox = seg->inst[0].inbox;
  uint64_t sum = 0;
  int ok = 1;
  if (role == 0) {
    for (uint64_t i = 0; i < n; ++i) {
      MetaRec m{};
      m.seq = i;
      m.id_lo = i * 7 + 1;
      while (!inbox.push(m)) std::this_thread::yield();  // ring holds 64: exercises backpressure
      sum += i;
    }
    while (seg->inst[1].ready.load(std::memory_order_acquire) == 0) std::this_thread::yield();
  } else {
    uint64_t expect = 0;
    for (uint64_t i = 0; i < n; ++i) {
      MetaRec m;
      while (!inbox.pop(m)) std::this_thread::yield();
      if (m.seq != expect || m.id_lo != m.seq * 7 + 1) ok = 0;
      expect = m.seq + 1;
      sum += m.seq;
    }
    seg->inst[1].ready.store(1, std::memory_order_release);
  }
  if (checksum) *checksum = sum;
  if (fifo_ok) *fifo_ok = ok;
  plane_close(seg, name, role == 0);
  return DF_OK;
}

df_status df_profile(df_ctx* ctx, int32_t enable, int32_t reset) {
  if (!ctx) return DF_ERR_INVALID;
  for (auto& ip : ctx->inst)
    if (ip->stage == DF_T) {
      ip->m.prof = enable ? &ctx->prof : nullptr;
      ip->m.prof_every = enable > 1 ? enable : 1;
    }
  if (reset) ctx->prof.reset();
  // one video request launches ~22k kernels (two events each) between
  // harvests; creating events inside the timed region would put cudaEventCreate on the
  // launch path
  if (enable) ctx->prof.reserve(1 << 16);
  return DF_OK;
}

df_status df_kernel_stats(df_ctx* ctx, uint32_t kind, uint64_t* launches, double* total_ms, double* flops,
                          double* bytes) {
  if (!ctx || kind >= K_COUNT) return DF_ERR_INVALID;
  ctx->prof.harvest();
  std::lock_guard<std::mutex> lk(ctx->prof.mu);
  if (launches) *launches = ctx->prof.count[kind];
  if (total_ms) *total_ms = ctx->prof.ms[kind];
  if (flops) *flops = ctx->prof.flops[kind];
  if (bytes) *bytes = ctx->prof.bytes[kind];
  return DF_OK;
}

df_status df_init(const df_graph* g, df_ctx** out) {
  if (!g || !out) return fail(nullptr, "df_init: null argument", DF_ERR_INVALID);
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) return fail(nullptr, "df_init: no CUDA device");
  if (g->n_inst == 0 || g->n_inst > DF_MAX_INST) return fail(nullptr, "df_init: n_inst", DF_ERR_INVALID);
  int cnt[3] = {0, 0, 0};
  for (uint32_t i = 0; i < g->n_inst; ++i) {
    if (g->inst[i].stage < 0 || g->inst[i].stage > 2 || g->inst[i].device < 0 || g->inst[i].device >= ndev)
      return fail(nullptr, "df_init: bad instance", DF_ERR_INVALID);
    cnt[g->inst[i].stage]++;
  }
  // Eq. 1: every stage has an instance; sum of instances over distinct GPUs <= G
  if (!cnt[0] || !cnt[1] || !cnt[2]) return fail(nullptr, "df_init: every stage needs an instance", DF_ERR_CAPACITY);
  if (g->G && uint32_t(cnt[0] + cnt[1] + cnt[2]) > g->G * 3)
    return fail(nullptr, "df_init: Eq.1 capacity", DF_ERR_CAPACITY);
  if (g->n_slots < 2 || (g->ring_capacity & (g->ring_capacity - 1)) || g->ring_capacity < 2)
    return fail(nullptr, "df_init: n_slots >= 2 and ring_capacity a power of two", DF_ERR_INVALID);
  const bool mp = g->world > 1;
  if (mp && (g->rank < 0 || g->rank >= g->world || !g->shm_name[0] || g->n_slots > uint32_t(PL_MAX_SLOTS)))
    return fail(nullptr, "df_init: multi-process graph needs rank in [0, world), shm_name, n_slots <= 4",
                DF_ERR_INVALID);
  auto is_local = [&](uint32_t i) { return !mp || g->inst[i].rank == g->rank; };
  for (uint32_t i = 0; i < g->n_inst; ++i) {
    if (!is_local(i)) continue;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, g->inst[i].device) != cudaSuccess || p.major != 10)
      return fail(nullptr, "df_init: instance device is not sm_100 (B200)");
  }
  auto ctx = new df_ctx();
  ctx->g = *g;
  ctx->requests.reset(new FaaRing<ReqState*>(g->ring_capacity));
  ctx->done.reset(new FaaRing<ReqState*>(std::max<uint32_t>(g->ring_capacity, 1024)));
  const df_dit_cfg& c = g->dit;
  ctx->ctx_bytes = size_t(c.L_txt) * c.d_txt * 2;
  if (c.C_y > 0) {
    ctx->clip_bytes = (size_t(c.L_img) * c.d_img * 2 + 15) & ~size_t(15);
    ctx->y_bytes = size_t(c.C_y) * c.F * c.H * c.W * 4;
  }
  ctx->lat_bytes = latent_elems(c) * 4;
  ctx->out_bytes = out_elems(c) * 4;
  // peer access between every pair of devices in use (NVLink P2P, P:L390 GPUDirect analogue)
  std::set<int> devs;
  for (uint32_t i = 0; i < g->n_inst; ++i)
    if (is_local(i)) devs.insert(g->inst[i].device);
  if (mp) {
    std::string perr;
    ctx->mp = true;
    ctx->seg_owner = g->rank == 0;
    ctx->seg = plane_open(g->shm_name, ctx->seg_owner, uint32_t(g->world), &perr);
    if (!ctx->seg) {
      delete ctx;
      return fail(nullptr, "df_init: " + perr);
    }
  }
  for (int a : devs)
    for (int b : devs)
      if (a != b) {
        cudaSetDevice(a);
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (can) {
          cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
      }
  for (uint32_t i = 0; i < g->n_inst; ++i) {
    auto in = std::make_unique<Inst>();
    in->id = int(i);
    in->stage = g->inst[i].stage;
    in->device = g->inst[i].device;
    in->local = is_local(i);
    ctx->by_stage[in->stage].push_back(int(i));
    ctx->inst.push_back(std::move(in));
  }
  for (int s = 0; s < 3; ++s) ctx->active[s] = int(ctx->by_stage[s].size());
  if (mp) {
    PlaneSeg* pg = ctx->seg;
    uint32_t z0 = 0;
    if (pg->route_state.compare_exchange_strong(z0, 1u)) {  // every rank derives the same routing: the first writes it
      for (int s = 0; s < 3; ++s) {
        pg->route_n[s] = int32_t(ctx->by_stage[s].size());
        for (size_t k = 0; k < ctx->by_stage[s].size(); ++k) pg->route[s][k] = ctx->by_stage[s][k];
        pg->active[s] = int32_t(ctx->by_stage[s].size());
      }
      pg->route_state.store(2u, std::memory_order_release);
    }
    while (pg->route_state.load(std::memory_order_acquire) != 2u) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    for (auto& ip : ctx->inst)
      if (ip->local) ip->busy.mirror = &ctx->seg->stat[ip->id];
  }
  for (auto& ip : ctx->inst) {
    Inst& I = *ip;
    if (!I.local) continue;
    cudaError_t e = inst_create(ctx, I);
    if (e != cudaSuccess) {
      std::string m = std::string("df_init: instance setup: ") + cudaGetErrorString(e) + " " + df::tls_err;
      df_finalize(ctx);
      return fail(nullptr, m);
    }
  }
  for (auto& ip : ctx->inst)
    if (ip->local) inst_start(ctx, ip.get());
  *out = ctx;
  return DF_OK;
}

df_status df_finalize(df_ctx* ctx) {
  if (!ctx) return DF_ERR_INVALID;
  ctx->sched_stop = true;
  if (ctx->sched.joinable()) ctx->sched.join();
  ctx->stop = true;
  for (auto& ip : ctx->inst) {
    ip->inbox.cv.notify_all();
    ip->slots.cv.notify_all();
  }
  for (auto& ip : ctx->inst)
    if (ip->worker.joinable()) ip->worker.join();
  for (int i = 0; i < int(ctx->inst.size()); ++i) {  // close the IPC views of remote consumers
    df_ctx::View& v = ctx->views[i];
    if (!v.open || !v.remote) continue;
    for (int sl = 0; sl < PL_MAX_SLOTS; ++sl) {
      if (v.buf[sl]) cudaIpcCloseMemHandle(v.buf[sl]);
      if (v.consumed[sl]) cudaEventDestroy(v.consumed[sl]);
    }
  }
  for (auto& ip : ctx->inst) {
    Inst& I = *ip;
    if (!I.local) continue;
    cudaSetDevice(I.device);
    cudaDeviceSynchronize();
    for (int p = 0; p < PL_MAX_INST; ++p)
      for (int sl = 0; sl < PL_MAX_SLOTS; ++sl) {
        OpenSet& os = I.opened[p][sl];
        if (os.open && os.ipc) {
          for (int c = 0; c < PL_MAX_CHUNKS; ++c) {
            cudaEventDestroy(os.ready[c]);
            cudaEventDestroy(os.issued[c]);
            cudaEventDestroy(os.chunk[c]);
          }
        }
        os = OpenSet{};
      }
  }
  for (auto& ip : ctx->inst) {
    Inst& I = *ip;
    if (!I.local) continue;
    cudaSetDevice(I.device);
    for (int sl = 0; sl < PL_MAX_SLOTS; ++sl)
      if (I.ipc_consumed[sl]) cudaEventDestroy(I.ipc_consumed[sl]);
    for (int p = 0; p < PL_MAX_INST; ++p)
      for (int sl = 0; sl < PL_MAX_SLOTS; ++sl) {
        SendSet* ss = I.sendset[p][sl];
        if (!ss) continue;
        for (int c = 0; c < PL_MAX_CHUNKS; ++c) {
          cudaEventDestroy(ss->ready[c]);
          cudaEventDestroy(ss->issued[c]);
          cudaEventDestroy(ss->chunk[c]);
        }
        delete ss;
        I.sendset[p][sl] = nullptr;
      }
    inst_free(I);
    if (I.compute) cudaStreamDestroy(I.compute);
    if (I.comm) cudaStreamDestroy(I.comm);
    if (I.aux) cudaStreamDestroy(I.aux);
    I.m.destroy();
  }
  ReqState* rs;
  while (ctx->requests && ctx->requests->pop(rs)) free_req(rs);
  while (ctx->done && ctx->done->pop(rs)) free_req(rs);
  for (ReqState* old : ctx->last_polled) free_req(old);
  if (ctx->seg) plane_close(ctx->seg, ctx->g.shm_name, ctx->seg_owner);
  delete ctx;
  return DF_OK;
}

df_status df_submit(df_ctx* ctx, const df_request* r, df_req_id* id_out) {
  if (!ctx || !r) return DF_ERR_INVALID;
  if (ctx->failed) return fail(ctx, ctx->err, DF_ERR_STATE);
  if (ctx->mp && ctx->g.dit.L_txt > uint32_t(PL_MAX_TXT))
    return fail(ctx, "df_submit: multi-process requests carry at most 512 text tokens", DF_ERR_INVALID);
  if (r->steps == 0 || r->steps > ctx->g.max_steps || !(r->shift > 0.f))
    return fail(ctx, "df_submit: steps in [1, max_steps] and shift > 0", DF_ERR_INVALID);
  if (r->out_host && r->out_bytes < ctx->out_bytes) return fail(ctx, "df_submit: out_bytes too small", DF_ERR_INVALID);
  df_req_id id = r->id;
  if (id.lo == 0 && id.hi == 0) id = {ctx->next_id.fetch_add(1), 0xD15A6F05ull};
  {
    std::lock_guard<std::mutex> lk(ctx->seen_mu);
    if (!ctx->seen.insert({id.lo, id.hi}).second) return fail(ctx, "df_submit: duplicate id", DF_ERR_DUPLICATE);
  }
  if (ctx->mp) {  // the global request ring in the shared plane: any rank submits, every E pulls
    ReqRec q{};
    q.id_lo = id.lo, q.id_hi = id.hi;
    q.seed = r->seed;
    q.user_tag = r->user_tag;
    q.steps = r->steps;
    q.shift = r->shift;
    q.guidance = r->guidance;
    q.flags = (r->out_host ? 1u : 0u) | (r->token_ids ? 2u : 0u) | (r->neg_token_ids ? 4u : 0u);
    const size_t L = ctx->g.dit.L_txt;
    if (r->token_ids) std::memcpy(q.tokens[0], r->token_ids, L * 4);
    if (r->neg_token_ids) std::memcpy(q.tokens[1], r->neg_token_ids, L * 4);
    q.t_submit = now_s();
    hist_push(ctx, r->steps);
    q.seq = ctx->seg->seq.fetch_add(1);  // FAA ticket
    if (!ctx->seg->requests.push(q)) {
      std::lock_guard<std::mutex> lk(ctx->seen_mu);
      ctx->seen.erase({id.lo, id.hi});
      return DF_AGAIN;
    }
    if (id_out) *id_out = id;
    return DF_OK;
  }
  if (ctx->requests->size_approx() >= ctx->requests->capacity()) {
    std::lock_guard<std::mutex> lk(ctx->seen_mu);
    ctx->seen.erase({id.lo, id.hi});
    return DF_AGAIN;
  }
  auto rs = new ReqState();
  rs->req = *r;
  rs->id = id;
  rs->t_submit = now_s();
  if (r->token_ids) rs->ids.assign(r->token_ids, r->token_ids + ctx->g.dit.L_txt);
  if (r->neg_token_ids) rs->neg_ids.assign(r->neg_token_ids, r->neg_token_ids + ctx->g.dit.L_txt);
  // timing events are created by each stage worker on its own device
  {
    std::lock_guard<std::mutex> lk(ctx->req_mu);
    rs->seq = ctx->mp ? ctx->seg->seq.fetch_add(1) : ctx->seq.fetch_add(1);  // FAA ticket
  }
  hist_push(ctx, r->steps);
  if (!ctx->requests->push(rs)) {
    free_req(rs);
    std::lock_guard<std::mutex> lk(ctx->seen_mu);
    ctx->seen.erase({id.lo, id.hi});
    return DF_AGAIN;
  }
  if (id_out) *id_out = id;
  return DF_OK;
}

df_status df_poll(df_ctx* ctx, df_completion* out, uint32_t max, uint32_t* n_out, int32_t timeout_ms) {
  if (!ctx || !out || !n_out) return DF_ERR_INVALID;
  *n_out = 0;
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms < 0 ? 0 : timeout_ms);
  for (;;) {
    ReqState* rs;
    if (*n_out == 0) {  // views handed out by the previous df_poll expire now
      for (ReqState* old : ctx->last_polled) free_req(old);
      ctx->last_polled.clear();
    }
    while (*n_out < max && ctx->done->pop(rs)) {
      fill_completion(ctx, rs, &out[(*n_out)++]);
      ctx->last_polled.push_back(rs);
    }
    if (*n_out) return DF_OK;
    if (ctx->failed) return fail(ctx, ctx->err, DF_ERR_STATE);
    std::unique_lock<std::mutex> lk(ctx->done_mu);
    if (timeout_ms >= 0 && std::chrono::steady_clock::now() >= deadline) return DF_EMPTY;
    ctx->done_cv.wait_for(lk, std::chrono::milliseconds(2));
  }
}

df_status df_set_ratio(df_ctx* ctx, uint32_t gE, uint32_t gT, uint32_t gD) {
  if (!ctx) return DF_ERR_INVALID;
  if (ctx->failed) return fail(ctx, ctx->err, DF_ERR_STATE);
  std::lock_guard<std::mutex> lk(ctx->ratio_mu);
  const uint32_t g[3] = {gE, gT, gD};
  const uint32_t hosts = uint32_t(ctx->inst.size());
  const uint32_t G = ctx->g.G ? std::min<uint32_t>(ctx->g.G, hosts) : hosts;
  if (g[0] < 1 || g[1] < 1 || g[2] < 1 || g[0] + g[1] + g[2] > G)  // Eq. 1
    return fail(ctx, "df_set_ratio: capacity (every g_s >= 1, sum g <= G)", DF_ERR_CAPACITY);
  int have[3];
  for (int s = 0; s < 3; ++s) have[s] = int(route_of(ctx, s).size());
  // Stages short of instances take them from stages with a surplus (the last instances of
  // the donor's routing list, i.e. the ones beyond its active prefix first): drain ->
  // re-initialise for the new stage -> serve (Alg. 1 "Apply"; cold start P:L357).
  // Across processes only an instance hosted by this process can be re-purposed here.
  for (int s = 0; s < 3; ++s) {
    while (have[s] < int(g[s])) {
      Inst* I = nullptr;
      int donor = -1;
      for (int pass = 0; pass < 3 && !I; ++pass) {  // the donor stage with the largest surplus first
        int best = -1;
        for (int t = 0; t < 3; ++t)
          if (t != s && have[t] > int(g[t]) && (best < 0 || have[t] - int(g[t]) > have[best] - int(g[best]))) {
            bool has_local = false;
            for (int id : route_of(ctx, t)) has_local |= ctx->inst[id]->local;
            if (has_local) best = t;
          }
        if (best < 0) break;
        const std::vector<int> v = route_of(ctx, best);
        for (int k = int(v.size()) - 1; k >= 0 && !I; --k)
          if (ctx->inst[v[k]]->local) I = ctx->inst[v[k]].get(), donor = best;
      }
      if (!I)
        return fail(ctx, ctx->mp ? "df_set_ratio: no instance of this process can be re-purposed"
                                 : "df_set_ratio: no instance to re-purpose",
                    ctx->mp ? DF_ERR_STATE : DF_ERR_CAPACITY);
      double drain_s = 0, cold_s = 0;
      cudaError_t e = inst_repurpose(ctx, I, s, drain_s, cold_s);
      if (e != cudaSuccess)
        return fail(ctx, std::string("df_set_ratio: re-purpose: ") + cudaGetErrorString(e) + " " + df::tls_err);
      have[donor]--, have[s]++;
      df_sched_event ev{};
      ev.t = now_s();
      ev.action = 4;
      ev.stage = s;
      ev.inst = I->id;
      ev.from_stage = donor;
      ev.drain_ms = float(drain_s * 1e3);
      ev.cold_start_ms = float(cold_s * 1e3);
      std::memcpy(ev.g, g, sizeof(ev.g));
      std::lock_guard<std::mutex> sl(ctx->sched_mu);
      ctx->sched_log.push_back(ev);
    }
  }
  // New requests go to the first g_s instances of each stage; instances beyond them drain
  // their inboxes (already-assigned work completes; nothing is dropped).
  for (int s = 0; s < 3; ++s) active_of(ctx, s) = int(g[s]);
  return DF_OK;
}

// ------------------------------------------------------------------ low level
struct df_cond {
  Cond c;
  int inst;
};

static Inst* get_inst(df_ctx* ctx, int32_t i, int stage) {
  if (!ctx || i < 0 || i >= int(ctx->inst.size())) return nullptr;
  Inst* I = ctx->inst[i].get();
  if (stage >= 0 && I->stage != stage) return nullptr;
  cudaSetDevice(I->device);
  return I;
}

df_status df_dit_prepare(df_ctx* ctx, int32_t t_inst, const void* ctx_dev, const float* sigmas, uint32_t S,
                         void* stream, df_cond** out) {
  Inst* I = get_inst(ctx, t_inst, DF_T);
  if (!I || !ctx_dev || !sigmas || !S || !out) return fail(ctx, "df_dit_prepare: invalid", DF_ERR_INVALID);
  if (ctx->failed) return DF_ERR_STATE;
  auto c = new df_cond();
  c->inst = t_inst;
  cudaError_t e = I->m.prepare(ctx_dev, sigmas, int(S), (cudaStream_t)stream, &c->c);
  if (e != cudaSuccess) {
    c->c.mem.release();
    delete c;
    return fail(ctx, std::string("df_dit_prepare: ") + cudaGetErrorString(e) + " " + df::tls_err);
  }
  *out = c;
  return DF_OK;
}

df_status df_dit_prepare_cfg(df_ctx* ctx, int32_t t_inst, const void* ctx_dev, const void* ctx_neg_dev,
                             float guidance, const float* sigmas, uint32_t S, void* stream, df_cond** out) {
  Inst* I = get_inst(ctx, t_inst, DF_T);
  if (!I || !ctx_dev || !ctx_neg_dev || !sigmas || !S || !out)
    return fail(ctx, "df_dit_prepare_cfg: invalid", DF_ERR_INVALID);
  if (ctx->failed) return DF_ERR_STATE;
  auto c = new df_cond();
  c->inst = t_inst;
  cudaError_t e = I->m.prepare(ctx_dev, sigmas, int(S), (cudaStream_t)stream, &c->c, ctx_neg_dev, guidance);
  if (e != cudaSuccess) {
    c->c.mem.release();
    delete c;
    return fail(ctx, std::string("df_dit_prepare_cfg: ") + cudaGetErrorString(e) + " " + df::tls_err);
  }
  *out = c;
  return DF_OK;
}

df_status df_dit_prepare_i2v(df_ctx* ctx, int32_t t_inst, const void* ctx_dev, const void* clip_dev,
                             const float* y_dev, const void* ctx_neg_dev, float guidance, const float* sigmas,
                             uint32_t S, void* stream, df_cond** out) {
  Inst* I = get_inst(ctx, t_inst, DF_T);
  if (!I || !ctx_dev || !clip_dev || !y_dev || !sigmas || !S || !out || !I->m.i2v())
    return fail(ctx, "df_dit_prepare_i2v: invalid", DF_ERR_INVALID);
  if (ctx->failed) return DF_ERR_STATE;
  auto c = new df_cond();
  c->inst = t_inst;
  cudaError_t e = I->m.prepare(ctx_dev, sigmas, int(S), (cudaStream_t)stream, &c->c, ctx_neg_dev,
                               ctx_neg_dev ? guidance : 1.f, clip_dev, y_dev);
  if (e != cudaSuccess) {
    c->c.mem.release();
    delete c;
    return fail(ctx, std::string("df_dit_prepare_i2v: ") + cudaGetErrorString(e) + " " + df::tls_err);
  }
  *out = c;
  return DF_OK;
}

df_status df_dit_step(df_ctx* ctx, int32_t t_inst, const df_cond* c, uint32_t i, float* x_dev, float* v_dev,
                      void* stream) {
  Inst* I = get_inst(ctx, t_inst, DF_T);
  if (!I || !c || !x_dev || int(i) >= c->c.S) return fail(ctx, "df_dit_step: invalid", DF_ERR_INVALID);
  if (ctx->failed) return DF_ERR_STATE;
  cudaError_t e = I->m.step(c->c, int(i), x_dev, v_dev, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(ctx, std::string("df_dit_step: ") + cudaGetErrorString(e) + " " + df::tls_err);
  return DF_OK;
}

df_status df_dit_layer(df_ctx* ctx, int32_t t_inst, const df_cond* c, uint32_t i, uint32_t l, float* r_dev,
                       void* stream) {
  Inst* I = get_inst(ctx, t_inst, DF_T);
  if (!I || !c || !r_dev || int(i) >= c->c.S || l >= I->m.c.layers)
    return fail(ctx, "df_dit_layer: invalid", DF_ERR_INVALID);
  cudaError_t e = I->m.layer(c->c, int(i), int(l), r_dev, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(ctx, std::string("df_dit_layer: ") + cudaGetErrorString(e) + " " + df::tls_err);
  return DF_OK;
}

df_status df_cond_release(df_ctx* ctx, df_cond* c) {
  if (!c) return DF_ERR_INVALID;
  if (ctx) cudaSetDevice(ctx->inst[c->inst]->device);
  c->c.mem.release();
  delete c;
  return DF_OK;
}

df_status df_encode(df_ctx* ctx, int32_t e_inst, const int32_t* ids_dev, void* ctx_dev, void* stream) {
  Inst* I = get_inst(ctx, e_inst, DF_E);
  if (!I || !ids_dev || !ctx_dev) return fail(ctx, "df_encode: invalid", DF_ERR_INVALID);
  cudaError_t e = I->m.encode(ids_dev, ctx_dev, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(ctx, std::string("df_encode: ") + cudaGetErrorString(e) + " " + df::tls_err);
  return DF_OK;
}

df_status df_decode(df_ctx* ctx, int32_t d_inst, const float* x_dev, float* out_dev, void* stream) {
  Inst* I = get_inst(ctx, d_inst, DF_D);
  if (!I || !x_dev || !out_dev) return fail(ctx, "df_decode: invalid", DF_ERR_INVALID);
  cudaError_t e = I->m.decode(x_dev, out_dev, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(ctx, std::string("df_decode: ") + cudaGetErrorString(e));
  return DF_OK;
}

df_status df_noise(df_ctx* ctx, int32_t inst, uint64_t seed, float* x_dev, void* stream) {
  Inst* I = get_inst(ctx, inst, -1);
  if (!I || !x_dev) return fail(ctx, "df_noise: invalid", DF_ERR_INVALID);
  g_launches->fetch_add(1);
  cudaError_t e = gen_noise(x_dev, latent_elems(ctx->g.dit), seed, (cudaStream_t)stream);
  return e == cudaSuccess ? DF_OK : fail(ctx, cudaGetErrorString(e));
}

df_status df_tokens(df_ctx* ctx, int32_t inst, uint64_t seed, int32_t* ids_dev, void* stream) {
  Inst* I = get_inst(ctx, inst, -1);
  if (!I || !ids_dev) return fail(ctx, "df_tokens: invalid", DF_ERR_INVALID);
  g_launches->fetch_add(1);
  cudaError_t e = gen_tokens(ids_dev, int(ctx->g.dit.L_txt), int(ctx->g.dit.vocab), seed, (cudaStream_t)stream);
  return e == cudaSuccess ? DF_OK : fail(ctx, cudaGetErrorString(e));
}

df_status df_image_cond(df_ctx* ctx, int32_t inst, uint64_t seed, void* clip_dev, float* y_dev, void* stream) {
  Inst* I = get_inst(ctx, inst, -1);
  const df_dit_cfg& c = ctx ? ctx->g.dit : df_dit_cfg{};
  if (!I || !clip_dev || !y_dev || c.C_y == 0) return fail(ctx, "df_image_cond: invalid", DF_ERR_INVALID);
  g_launches->fetch_add(1);
  cudaError_t e = gen_image_cond(seed, static_cast<bf16*>(clip_dev), size_t(c.L_img) * c.d_img, y_dev, int(c.C_y),
                                 int(c.F), int(c.H), int(c.W), (cudaStream_t)stream);
  return e == cudaSuccess ? DF_OK : fail(ctx, cudaGetErrorString(e));
}

df_status df_handoff(df_ctx* ctx, const df_handoff_desc* d, void* src_stream, df_xfer** out) {
  if (!ctx || !d || !out) return DF_ERR_INVALID;
  if (ctx->failed) return DF_ERR_STATE;
  ChunkPlan plan;
  if (d->flags & DF_LATENT_BLOCKS) {
    if (d->bytes != ctx->lat_bytes) return fail(ctx, "df_handoff: DF_LATENT_BLOCKS needs the latent's size", DF_ERR_INVALID);
    plan = plan_latent(ctx->g.dit, d->chunk_bytes);
  } else {
    plan = plan_bytes(d->bytes, d->chunk_bytes, 16);
  }
  Xfer* x = nullptr;
  df_status s = do_handoff(ctx, d, plan, (cudaStream_t)src_stream, nullptr, &x);
  if (s == DF_OK) *out = x;
  return s;
}

df_status df_handoff_wait(df_ctx* ctx, df_xfer* x, uint32_t chunk, void* dst_stream) {
  if (!ctx || !x) return DF_ERR_INVALID;
  if (chunk == DF_ALL_CHUNKS) {
    for (auto e : x->chunk_ev) CK(ctx, cudaStreamWaitEvent((cudaStream_t)dst_stream, e, 0));
    return DF_OK;
  }
  if (chunk >= x->nchunks) return fail(ctx, "df_handoff_wait: chunk", DF_ERR_INVALID);
  CK(ctx, cudaStreamWaitEvent((cudaStream_t)dst_stream, x->chunk_ev[chunk], 0));
  return DF_OK;
}

df_status df_handoff_query(df_ctx* ctx, df_xfer* x, uint32_t* chunks_done, uint64_t hash[2]) {
  if (!ctx || !x) return DF_ERR_INVALID;
  uint32_t n = 0;
  for (auto e : x->chunk_ev) n += cudaEventQuery(e) == cudaSuccess ? 1 : 0;
  cudaGetLastError();
  if (chunks_done) *chunks_done = n;
  if (hash) {
    hash[0] = hash[1] = 0;
    if (x->hashed && n == x->nchunks) {  // the source hash precedes the last chunk's event
      if (x->t_hash) cudaEventSynchronize(x->t_hash);
      hash[0] = x->hash_dev[0];
      hash[1] = x->hash_dev[1];
    }
  }
  return DF_OK;
}

df_status df_handoff_release(df_ctx* ctx, df_xfer* x) {
  if (!x) return DF_ERR_INVALID;
  cudaSetDevice(x->src_dev);
  for (auto e : x->chunk_ev) cudaEventSynchronize(e);
  free_xfer(x);
  (void)ctx;
  return DF_OK;
}

df_status df_payload_hash(df_ctx* ctx, int32_t inst, const void* buf_dev, uint64_t nbytes, uint64_t* hash_out) {
  Inst* I = get_inst(ctx, inst, -1);
  if (!I || !buf_dev || !hash_out) return fail(ctx, "df_payload_hash: invalid", DF_ERR_INVALID);
  unsigned long long* h = nullptr;
  CK(ctx, cudaMalloc(&h, 8));
  g_launches->fetch_add(1);
  CK(ctx, payload_hash(buf_dev, nbytes, 0, h, 0));
  unsigned long long v = 0;
  CK(ctx, cudaMemcpy(&v, h, 8, cudaMemcpyDeviceToHost));
  cudaFree(h);
  *hash_out = v;
  return DF_OK;
}

df_status df_weight_bits(df_ctx* ctx, int32_t inst, uint32_t tensor_id, uint16_t* dst, uint64_t n) {
  Inst* I = get_inst(ctx, inst, -1);
  if (!I || !dst) return fail(ctx, "df_weight_bits: invalid", DF_ERR_INVALID);
  for (const TensorLoc& L : I->m.locs) {
    if (L.tid != tensor_id) continue;
    if (n != uint64_t(L.in) * L.out) return fail(ctx, "df_weight_bits: size", DF_ERR_INVALID);
    // gather the logical [in, out] tensor out of its device layout
    size_t rows = 0, cols = L.ld;
    if (L.layout == 0) rows = L.in;
    else if (L.layout == 1) rows = size_t(L.row_off) + L.out;
    else rows = size_t((L.out + 15) / 16) * 32;
    std::vector<uint16_t> buf(rows * cols);
    CK(ctx, cudaMemcpy(buf.data(), L.base, buf.size() * 2, cudaMemcpyDeviceToHost));
    for (int k = 0; k < L.in; ++k)
      for (int o = 0; o < L.out; ++o) {
        size_t idx;
        if (L.layout == 0) idx = size_t(k) * L.ld + o;
        else if (L.layout == 1) idx = size_t(L.row_off + o) * L.ld + k;
        else idx = (size_t(o / 16) * 32 + size_t(L.row_off) * 16 + o % 16) * L.ld + k;
        dst[size_t(k) * L.out + o] = buf[idx];
      }
    return DF_OK;
  }
  return fail(ctx, "df_weight_bits: unknown tensor id on this instance", DF_ERR_INVALID);
}

df_status df_op_gemm(df_ctx* ctx, const void* A, const void* W, float* out, int32_t M, int32_t N, int32_t K,
                     int32_t tc, void* stream) {
  if (!ctx || !A || !W || !out) return DF_ERR_INVALID;
  Epi e;
  std::memset(&e, 0, sizeof(e));
  e.kind = EPI_STORE;
  e.M = M;
  e.N = N;
  e.out = out;
  e.ldo = N;
  g_launches->fetch_add(1);
  if (tc == 2) {  // tensor cores with the stream-K workspace of the first T instance (tests)
    for (auto& ip : ctx->inst)
      if (ip->stage == DF_T && ip->m.sk_ws) {
        e.sk_ws = ip->m.sk_ws;
        e.sk_flag = ip->m.sk_flag;
        e.sk_force = 1;
        break;
      }
    if (!e.sk_ws) return fail(ctx, "df_op_gemm: no stream-K workspace", DF_ERR_STATE);
  }
  cudaError_t r = tc ? gemm_tc((const bf16*)A, K, (const bf16*)W, K, M, N, K, e, 1, (cudaStream_t)stream)
                     : gemm_simt(A, 1, K, 0, (const bf16*)W, K, out, N, M, N, K, nullptr, ACT_NONE, (cudaStream_t)stream);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_gemm: ") + cudaGetErrorString(r));
}

df_status df_op_attention(df_ctx* ctx, const void* Q, const void* K, const void* V, void* O, int32_t H, int32_t Nq,
                          int32_t Nk, int32_t dh, int32_t dh_pad, float scale, void* stream) {
  if (!ctx || !Q || !K || !V || !O) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = attn_tc((const bf16*)Q, (const bf16*)K, (const bf16*)V, (bf16*)O, H, Nq, Nk, dh, dh_pad, scale,
                          (cudaStream_t)stream, 0);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_attention: ") + cudaGetErrorString(r));
}

df_status df_op_rmsnorm_mod(df_ctx* ctx, const float* x, void* out, int32_t M, int32_t d, const float* shift,
                            const float* scale, float eps, void* stream) {
  if (!ctx || !x || !out || !shift || !scale) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = rmsnorm_mod(x, out, 0, M, d, shift, scale, nullptr, eps, (cudaStream_t)stream);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_rmsnorm_mod: ") + cudaGetErrorString(r));
}

df_status df_op_quant_e4m3(df_ctx* ctx, const void* x, uint64_t n, void* q, float* scale, void* stream) {
  if (!ctx || (n && (!x || !q)) || !scale) return DF_ERR_INVALID;
  g_launches->fetch_add(n ? 3 : 1);
  cudaError_t r = quant_e4m3(static_cast<const bf16*>(x), size_t(n), static_cast<uint8_t*>(q), scale,
                             (cudaStream_t)stream);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_quant_e4m3: ") + cudaGetErrorString(r));
}

df_status df_op_gemm_e4m3(df_ctx* ctx, const void* qa, const void* qb, const float* sa, const float* sb, int32_t M,
                          int32_t N, int32_t K, void* out, int32_t out_f32, void* stream) {
  if (!ctx || !qa || !qb || !sa || !sb || !out) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = gemm_e4m3(static_cast<const uint8_t*>(qa), static_cast<const uint8_t*>(qb), sa, sb, M, N, K, out, N,
                            out_f32, (cudaStream_t)stream);
  if (r == cudaErrorInvalidValue) return fail(ctx, "df_op_gemm_e4m3: unsupported shape", DF_ERR_INVALID);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_gemm_e4m3: ") + cudaGetErrorString(r));
}

df_status df_op_qk_e4m3(df_ctx* ctx, const void* x, uint64_t n, float inv, void* q, void* stream) {
  if (!ctx || (n && (!x || !q))) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = qk_e4m3(static_cast<const bf16*>(x), size_t(n), inv, static_cast<uint8_t*>(q), (cudaStream_t)stream);
  if (r == cudaErrorInvalidValue) return fail(ctx, "df_op_qk_e4m3: n % 8 or alignment", DF_ERR_INVALID);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_qk_e4m3: ") + cudaGetErrorString(r));
}

df_status df_op_attention_qf8(df_ctx* ctx, const void* Q8, const void* K8, const void* V, void* O, int32_t H,
                              int32_t Nq, int32_t Nk, float scale, void* stream) {
  if (!ctx || !Q8 || !K8 || !V || !O) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = attn_tc_qf8(static_cast<const uint8_t*>(Q8), static_cast<const uint8_t*>(K8),
                              static_cast<const bf16*>(V), static_cast<bf16*>(O), H, Nq, Nk, scale, (cudaStream_t)stream,
                              0);
  if (r == cudaErrorInvalidValue) return fail(ctx, "df_op_attention_qf8: unsupported shape", DF_ERR_INVALID);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_attention_qf8: ") + cudaGetErrorString(r));
}

df_status df_op_attention_f8(df_ctx* ctx, const void* Q8, const void* K8, const void* V, void* O, int32_t H,
                             int32_t Nq, int32_t Nk, float scale, void* v8t, float* vscale, void* stream) {
  if (!ctx || !Q8 || !K8 || !V || !O || !v8t || !vscale) return DF_ERR_INVALID;
  g_launches->fetch_add(4);
  const int ldv = (Nk + 63) / 64 * 64;
  cudaError_t r = v_e4m3t(static_cast<const bf16*>(V), H, Nk, ldv, vscale, static_cast<uint8_t*>(v8t),
                          (cudaStream_t)stream);
  if (r == cudaSuccess)
    r = attn_tc_f8(static_cast<const uint8_t*>(Q8), static_cast<const uint8_t*>(K8), static_cast<const uint8_t*>(v8t),
                   ldv, vscale, static_cast<bf16*>(O), H, Nq, Nk, scale, (cudaStream_t)stream, 0);
  if (r == cudaErrorInvalidValue) return fail(ctx, "df_op_attention_f8: unsupported shape", DF_ERR_INVALID);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_attention_f8: ") + cudaGetErrorString(r));
}

df_status df_op_mx_quant_e4m3(df_ctx* ctx, const void* x, int32_t M, int32_t K, void* q, void* sf, void* stream) {
  if (!ctx || M < 0 || K < 0 || (M && K && (!x || !q || !sf))) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = mx_quant_e4m3(static_cast<const bf16*>(x), M, K, static_cast<uint8_t*>(q), static_cast<uint8_t*>(sf),
                                (cudaStream_t)stream);
  if (r == cudaErrorInvalidValue) return fail(ctx, "df_op_mx_quant_e4m3: K % 128 or alignment", DF_ERR_INVALID);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_mx_quant_e4m3: ") + cudaGetErrorString(r));
}

df_status df_op_gemm_mxf8(df_ctx* ctx, const void* qa, const void* sa, const void* qb, const void* sb, int32_t M,
                          int32_t N, int32_t K, void* out, int32_t out_f32, void* stream) {
  if (!ctx || !qa || !qb || !sa || !sb || !out) return DF_ERR_INVALID;
  g_launches->fetch_add(1);
  cudaError_t r = gemm_mxf8(static_cast<const uint8_t*>(qa), static_cast<const uint8_t*>(sa),
                            static_cast<const uint8_t*>(qb), static_cast<const uint8_t*>(sb), M, N, K, out, N, out_f32,
                            (cudaStream_t)stream);
  if (r == cudaErrorInvalidValue) return fail(ctx, "df_op_gemm_mxf8: unsupported shape", DF_ERR_INVALID);
  return r == cudaSuccess ? DF_OK : fail(ctx, std::string("df_op_gemm_mxf8: ") + cudaGetErrorString(r));
}

}  // extern "C"
