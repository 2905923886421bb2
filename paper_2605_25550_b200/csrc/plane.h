// Cross-process control plane of the stage handoff (one process per GPU).
//
// PAPER.md §sec:decentral-queue: stages are decoupled by fixed-length
// metadata queues with Fetch-and-Add concurrency control and one-sided access; the
// downstream instance posts a destination address before data moves.
// Inside one node the "RDMA-backed queues" become lock-free rings in a POSIX shared-memory
// segment that every rank maps, and the destination addresses become CUDA IPC handles of
// the consumer's receive slots (data plane: the producer copies chunks straight into the
// peer slot over NVLink; one interprocess event per chunk).
//
// Segment layout (all fixed size, lock-free std::atomic words, no pointers):
//   Header        magic, world, global request sequence (FAA), per-instance ready flags
//   InstPlane[i]  for every consumer instance i: slot IPC handles, a per-slot consumed
//                 event (consumer-owned), a free-slot ring (the posted destination
//                 addresses), an inbox ring of fixed-size metadata records, and per slot the
//                 IPC handles of the events of the transfer currently in that slot.
// Events are always owned (created and recorded) by the side whose stream records them: a
// CUDA event can only be recorded on a stream of its own device, while a stream may wait on
// an event of any device.  So the producer creates its per-(consumer, slot) ready / issued /
// chunk events and publishes their handles into the consumer's slot record when it claims the
// slot; the consumer records `consumed`.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <string>
#include <cuda_runtime.h>

namespace df {

constexpr int PL_MAX_INST = 32;
constexpr int PL_MAX_SLOTS = 4;
constexpr int PL_MAX_CHUNKS = 64;
constexpr int PL_RING = 64;  // power of two

// Fixed-length request metadata ("leveraging fixed-length metadata ... O(1)").
struct alignas(8) MetaRec {
  uint64_t seq, id_lo, id_hi, seed, user_tag;
  uint32_t steps, slot, nchunks, chunk_bytes;
  float shift;
  int32_t inst_e, inst_t;
  int32_t src;                                    // producer instance of this edge's transfer
  uint32_t flags;
  double t_submit, t_start_e, t_end_e, t_start_t, t_end_t;  // host CLOCK_MONOTONIC (node-wide)
  float stage_ms_e, stage_ms_t;
  float exposed_e2t, xfer_e2t, overlap_e2t;       // edge 0, measured by T on its own clock
  float guidance;                                 // CFG scale (payload holds 2 ctx when on)
  uint64_t hash_src_e2t, hash_dst_e2t;            // edge 0 hashes (T verified them)
};
static_assert(sizeof(MetaRec) <= 192, "metadata record must stay fixed-size");

// Bounded MPMC ring of fixed-size records with per-cell sequence words (Vyukov); the
// tail/head tickets are claimed by CAS-FAA on shared words.
template <typename T, int CAP>
struct ShmRing {
  struct Cell {
    std::atomic<uint64_t> seq;
    T val;
  };
  alignas(64) std::atomic<uint64_t> head;
  alignas(64) std::atomic<uint64_t> tail;
  Cell cells[CAP];
  void init() {
    head.store(0);
    tail.store(0);
    for (int i = 0; i < CAP; ++i) cells[i].seq.store(uint64_t(i));
  }
  bool push(const T& v) {
    uint64_t pos = tail.load(std::memory_order_relaxed);
    for (;;) {
      Cell& c = cells[pos & (CAP - 1)];
      uint64_t s = c.seq.load(std::memory_order_acquire);
      int64_t dif = int64_t(s) - int64_t(pos);
      if (dif == 0) {
        if (tail.compare_exchange_weak(pos, pos + 1, std::memory_order_relaxed)) {
          c.val = v;
          c.seq.store(pos + 1, std::memory_order_release);
          return true;
        }
      } else if (dif < 0) {
        return false;
      } else {
        pos = tail.load(std::memory_order_relaxed);
      }
    }
  }
  uint64_t size_approx() const {
    const uint64_t t = tail.load(std::memory_order_relaxed), h = head.load(std::memory_order_relaxed);
    return t > h ? t - h : 0;
  }
  bool pop(T& out) {
    uint64_t pos = head.load(std::memory_order_relaxed);
    for (;;) {
      Cell& c = cells[pos & (CAP - 1)];
      uint64_t s = c.seq.load(std::memory_order_acquire);
      int64_t dif = int64_t(s) - int64_t(pos + 1);
      if (dif == 0) {
        if (head.compare_exchange_weak(pos, pos + 1, std::memory_order_relaxed)) {
          out = c.val;
          c.seq.store(pos + CAP, std::memory_order_release);
          return true;
        }
      } else if (dif < 0) {
        return false;
      } else {
        pos = head.load(std::memory_order_relaxed);
      }
    }
  }
};

// Producer-owned events of one transfer (handles published into the consumer's slot record):
// ready[c] = chunk c's data existed (comm stream, after waiting the producer's compute, before
// any injected delay), issued[c] = chunk c's copy is issued (after any delay), chunk[c] =
// chunk c landed.
struct XferEvHandles {
  int32_t producer;                      // instance that published them (consumer caches per producer)
  uint32_t nchunks;
  cudaIpcEventHandle_t ready[PL_MAX_CHUNKS];
  cudaIpcEventHandle_t issued[PL_MAX_CHUNKS];
  cudaIpcEventHandle_t chunk[PL_MAX_CHUNKS];
};

struct InstPlane {
  std::atomic<uint32_t> ready;  // consumer published its handles
  std::atomic<uint32_t> gen;    // bumped each time the consumer (re)publishes (producers re-open their views)
  std::atomic<int32_t> inflight;  // producers (any rank) that picked this instance and have not posted yet
  uint32_t n_slots, nchunks_max;
  uint64_t slot_bytes;          // payload capacity; each slot has a 64-byte trailer after it
  cudaIpcMemHandle_t slot_mem[PL_MAX_SLOTS];
  cudaIpcEventHandle_t consumed[PL_MAX_SLOTS];
  XferEvHandles xev[PL_MAX_SLOTS];       // written by the producer that claimed the slot
  ShmRing<uint32_t, 16> free_slots;      // posted destination addresses (slot index)
  ShmRing<MetaRec, PL_RING> inbox;       // control plane into this consumer
};

// An admitted request in the global request ring (any rank submits, the encoder instances
// of every rank pull; "the request scheduler inserts the request into the global
// request buffer").  Caller token ids travel inside the record.
constexpr int PL_MAX_TXT = 512;
struct ReqRec {
  uint64_t seq, id_lo, id_hi, seed, user_tag;
  uint32_t steps, flags;  // bit0: deliver the decoded output (to the D rank); bit1: tokens; bit2: negative tokens
  float shift, guidance;
  double t_submit;
  int32_t tokens[2][PL_MAX_TXT];
};

// Controller-visible state of one instance, written by the rank that hosts it (Alg. 1's u_s).
struct InstStat {
  std::atomic<uint64_t> busy_ns;     // closed busy intervals
  std::atomic<uint64_t> busy_since;  // bit pattern of the open interval's start (double seconds), 0 = idle
};

// Measured seconds per request per instance for the Eq. 6 planner, per stage and workload key
// (EMA), shared so that the controller sees the stage times of every rank.
struct StageEma {
  std::atomic<uint32_t> lock;
  uint32_t n;
  uint32_t key[8];
  double sec[8];
};

struct PlaneSeg {
  std::atomic<uint64_t> magic;
  std::atomic<uint64_t> seq;             // global request sequence (FAA)
  std::atomic<uint32_t> attached;
  uint32_t world;
  InstPlane inst[PL_MAX_INST];
  // hybrid scheduler state shared by all ranks (one controller, any rank)
  std::atomic<int32_t> active[3];        // g_s: the first active[s] instances of stage s get new work
  // routing shared by every rank (re-purposing changes it): instances of each stage in order
  std::atomic<uint32_t> route_lock, route_state;  // state 0 empty, 1 being written, 2 ready
  int32_t route_n[3];
  int32_t route[3][PL_MAX_INST];
  std::atomic<uint64_t> qd_ns[3], qd_count[3];
  InstStat stat[PL_MAX_INST];
  StageEma ema[3];
  std::atomic<uint32_t> hist_lock;
  uint32_t hist_n, hist_head;
  uint32_t hist[64];                     // workload keys (steps) of the last admitted requests
  ShmRing<ReqRec, PL_RING> requests;
};

// Create (rank 0) or attach to the named segment; returns nullptr on failure.
PlaneSeg* plane_open(const char* name, bool create, uint32_t world, std::string* err);
void plane_close(PlaneSeg* seg, const char* name, bool owner);

}  // namespace df
