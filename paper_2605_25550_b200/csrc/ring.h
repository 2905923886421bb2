// Lock-free bounded MPMC ring with fixed-size slots and FAA tickets — the host
// analogue of the paper's decentralised metadata queues (PAPER.md P:L377-384,
// §sec:decentral-queue: "Fetch-and-Add (FAA) atomic operations for lock-free queue
// concurrency control", O(1) operations on fixed-length metadata).  Per-slot
// sequence words give the readiness check.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <memory>

namespace df {

template <typename T>
class FaaRing {
 public:
  explicit FaaRing(size_t cap_pow2) : cap_(cap_pow2), mask_(cap_pow2 - 1), cells_(new Cell[cap_pow2]) {
    for (size_t i = 0; i < cap_; ++i) cells_[i].seq.store(i, std::memory_order_relaxed);
    head_.store(0);
    tail_.store(0);
  }
  // false = full (backpressure, DF_AGAIN)
  bool push(const T& v) {
    size_t pos = tail_.load(std::memory_order_relaxed);
    for (;;) {
      Cell& c = cells_[pos & mask_];
      size_t seq = c.seq.load(std::memory_order_acquire);
      intptr_t dif = intptr_t(seq) - intptr_t(pos);
      if (dif == 0) {
        if (tail_.compare_exchange_weak(pos, pos + 1, std::memory_order_relaxed)) {
          c.val = v;
          c.seq.store(pos + 1, std::memory_order_release);
          return true;
        }
      } else if (dif < 0) {
        return false;
      } else {
        pos = tail_.load(std::memory_order_relaxed);
      }
    }
  }
  bool pop(T& out) {
    size_t pos = head_.load(std::memory_order_relaxed);
    for (;;) {
      Cell& c = cells_[pos & mask_];
      size_t seq = c.seq.load(std::memory_order_acquire);
      intptr_t dif = intptr_t(seq) - intptr_t(pos + 1);
      if (dif == 0) {
        if (head_.compare_exchange_weak(pos, pos + 1, std::memory_order_relaxed)) {
          out = c.val;
          c.seq.store(pos + mask_ + 1, std::memory_order_release);
          return true;
        }
      } else if (dif < 0) {
        return false;
      } else {
        pos = head_.load(std::memory_order_relaxed);
      }
    }
  }
  size_t size_approx() const {
    size_t t = tail_.load(std::memory_order_relaxed), h = head_.load(std::memory_order_relaxed);
    return t >= h ? t - h : 0;
  }
  size_t capacity() const { return cap_; }

 private:
  struct Cell {
    std::atomic<size_t> seq;
    T val;
  };
  size_t cap_, mask_;
  std::unique_ptr<Cell[]> cells_;
  alignas(64) std::atomic<size_t> head_;
  alignas(64) std::atomic<size_t> tail_;
};

}  // namespace df
