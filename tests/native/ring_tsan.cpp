// ThreadSanitizer stress of the library's lock-free rings (host code only, no GPU):
// df::FaaRing (the in-process request / completion rings, ring.h) and df::ShmRing (the
// cross-process rings of the shared-memory plane, plane.h) under several producer and
// consumer threads.  Checks conservation (every pushed value popped exactly once, per-producer
// FIFO order); tests/test_native.py builds it with -fsanitize=thread and fails on any report.
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>
#include "ring.h"
#include "plane.h"

template <class Ring, class PushFn, class PopFn>
static int stress(Ring& ring, PushFn push, PopFn pop, int producers, int consumers, uint64_t per) {
  std::vector<std::atomic<uint32_t>> seen(size_t(producers) * per);
  for (auto& s : seen) s.store(0);
  std::atomic<uint64_t> popped{0};
  std::vector<std::thread> th;
  for (int p = 0; p < producers; ++p)
    th.emplace_back([&, p] {
      for (uint64_t i = 0; i < per; ++i) {
        const uint64_t v = uint64_t(p) * per + i;
        while (!push(ring, v)) std::this_thread::yield();
      }
    });
  std::atomic<int> fifo_bad{0};
  for (int c = 0; c < consumers; ++c)
    th.emplace_back([&] {
      std::vector<int64_t> last(size_t(producers), -1);
      const uint64_t total = uint64_t(producers) * per;
      while (popped.load() < total) {
        uint64_t v;
        if (!pop(ring, v)) {
          std::this_thread::yield();
          continue;
        }
        popped++;
        seen[v].fetch_add(1);
        const int p = int(v / per);
        const int64_t i = int64_t(v % per);
        if (i <= last[size_t(p)]) fifo_bad++;  // each consumer sees a producer's values in order
        last[size_t(p)] = i;
      }
    });
  for (auto& t : th) t.join();
  int bad = fifo_bad.load();
  for (auto& s : seen) bad += s.load() != 1;
  return bad;
}

int main() {
  int bad = 0;
  {
    df::FaaRing<uint64_t> r(64);
    bad += stress(r, [](df::FaaRing<uint64_t>& q, uint64_t v) { return q.push(v); },
                  [](df::FaaRing<uint64_t>& q, uint64_t& v) { return q.pop(v); }, 4, 3, 20000);
  }
  {
    auto* r = new df::ShmRing<df::MetaRec, df::PL_RING>();
    r->init();
    bad += stress(*r,
                  [](df::ShmRing<df::MetaRec, df::PL_RING>& q, uint64_t v) {
                    df::MetaRec m{};
                    m.seq = v;
                    m.id_lo = v * 7 + 1;
                    return q.push(m);
                  },
                  [&bad](df::ShmRing<df::MetaRec, df::PL_RING>& q, uint64_t& v) {
                    df::MetaRec m;
                    if (!q.pop(m)) return false;
                    v = m.seq;
                    return m.id_lo == m.seq * 7 + 1;  // a torn record would not match
                  },
                  3, 3, 20000);
    delete r;
  }
  std::printf("ring stress: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
  return bad ? 1 : 0;
}
