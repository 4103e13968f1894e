// The stash ring of k_lamb (paper_2106_10207_b200/csrc/cuda/sp_ring.h),
// driven the way the claims lane drives it: regions allocated in FIFO order
// (or not, when the ring is full), freed in the same order in batches, the
// head moved to the oldest live region. Every live region must stay
// disjoint from every other, inside the buffer and congruent to its chunk
// start mod 4.
#include <cstdint>
#include <deque>
#include <random>
#include <vector>

#include "../../paper_2106_10207_b200/csrc/cuda/sp_ring.h"
#include "harness.hpp"

namespace {

struct Region {
  int off, len;
};

bool disjoint(const Region& a, const Region& b) { return a.off + a.len <= b.off || b.off + b.len <= a.off; }

}  // namespace

TEST_CASE("stash ring: wrapped and full is not mistaken for empty") {
  // live [2051, 35447); the next region wraps to [3, 2051), which leaves
  // tail == head: nothing may be allocated until a region is freed
  sp::Ring r{2051, 35447, 18};
  CHECK(sp::ring_alloc(r, 37176, 3, 2048) == 3);
  CHECK(r.tail == r.head);
  CHECK(sp::ring_alloc(r, 37176, 0, 16) == -1);
  CHECK(sp::ring_alloc(r, 37176, 1, 1) == -1);
}

TEST_CASE("stash ring: random claim / free sequences never overlap") {
  for (int seed = 0; seed < 300; ++seed) {
    std::mt19937_64 g((uint64_t)seed);
    const int cap = 4000 + (int)(g() % 40000);
    sp::Ring r{0, 0, 0};
    std::deque<Region> fifo;  // entries in claim order; off -1: not stashed
    size_t handed = 0;        // entries handed to pass 2 (a prefix of fifo)
    std::deque<int> batches;  // sizes of the pass-2 batches in flight
    for (int it = 0; it < 4000; ++it) {
      if (!batches.empty() && g() % 10 < 9) {  // a pass-2 batch finished: free it
        const int nb = batches.front();
        batches.pop_front();
        for (int j = 0; j < nb; ++j) {
          if (fifo.front().off >= 0) --r.live;
          fifo.pop_front();
          --handed;
        }
        for (const Region& e : fifo)
          if (e.off >= 0) {
            r.head = e.off;
            break;
          }
      }
      if (fifo.size() < 32) {  // claim a chunk
        const int len = g() % 5 ? 2048 : 1 + (int)(g() % 2048);
        const long long start = (long long)(g() % 100000000);
        const int off = sp::ring_alloc(r, cap, start, len);
        if (off >= 0) {
          ++r.live;
          CHECK(off + len <= cap);
          CHECK(((off - start) % 4 + 4) % 4 == 0);
          for (const Region& e : fifo)
            if (e.off >= 0 && !disjoint(e, Region{off, len})) {
              CHECK(false && "overlapping stash regions");
              return;
            }
        }
        fifo.push_back(Region{off, len});
      }
      const int want = (int)(g() % 3);  // hand out up to two entries
      int n = 0;
      while (n < want && handed < fifo.size()) {
        ++handed;
        ++n;
      }
      if (n) batches.push_back(n);
    }
  }
}
