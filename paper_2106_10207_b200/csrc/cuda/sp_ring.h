// sp_ring.h — the stash ring of k_lamb (sp_lamb.cuh): one CTA's u buffer in
// shared memory, regions allocated in FIFO order at claim time and freed in
// the same order after pass 2. Plain C++ (host and device), so the
// allocator is unit-tested on the host (tests/cpp/test_ring.cpp).
#pragma once

#if defined(__CUDACC__)
#define SP_HD __host__ __device__ __forceinline__
#else
#define SP_HD inline
#endif

namespace sp {

// Live regions: [head, tail) when tail > head; else (wrapped) [head, end)
// and [0, tail), with tail == head meaning wrapped and full. head is the
// offset of the oldest live region (the caller sets it when that region is
// freed); live counts the regions.
struct Ring {
  int head, tail, live;
};

// A region of len floats at an offset congruent to start mod 4 (so that the
// chunk's 16-byte vectors land on 16-byte words), or -1 if none fits.
SP_HD int ring_alloc(Ring& r, int cap, long long start, int len) {
  const int a0 = (int)(((start % 4) + 4) % 4);
  if (r.live == 0) {
    r.head = r.tail = 0;
    if (a0 + len > cap) return -1;
    r.tail = a0 + len;
    return a0;
  }
  const int x = r.tail + (int)((((start - r.tail) % 4) + 4) % 4);
  if (r.tail > r.head) {  // room at the end, else wrap to the front
    if (x + len <= cap) {
      r.tail = x + len;
      return x;
    }
    if (a0 + len <= r.head) {
      r.tail = a0 + len;
      return a0;
    }
    return -1;
  }
  if (x + len <= r.head) {  // wrapped: between the front part and the oldest region
    r.tail = x + len;
    return x;
  }
  return -1;
}

}  // namespace sp
