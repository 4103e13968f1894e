// sp_lamb.cuh — the LAMB step of the round (K3 + K4) as one cooperative
// persistent kernel: kLambCtasPerSm CTAs of kLambThreads per SM, chunks of
// at most kLambTile elements claimed from one queue.
//
// LAMB needs every tensor's norms ||p||, ||u|| before any element of it can
// be updated, so each element is touched twice: pass 1 (m' = b1 m + (1-b1) g,
// v' = ..., u = m'^/(sqrt(v'^)+eps) + wd p, norm partials) and pass 2
// (p' = p - lr * trust_t * u). Re-reading p, m', v' in pass 2 costs 12 B per
// element of L2 traffic on top of pass 1's 24 + b; the round-1 kernel moved
// 44 B/element through L2 at 6.35 TB/s.
//
// Loads. Pass 1's g, p, m, v of a chunk (and, with the q8 wire, its block
// scales) are fetched by bulk async copies (cp.async.bulk, completion on the
// stage's `full` mbarrier) into one of kLambStages stages in shared memory,
// one iteration ahead. The bytes in flight hold no registers and do not
// depend on the warp count (scripts/micro/tma_stream.cu,
// profiles/r02/tma_stream.txt: ~6 TB/s with 128-1024 threads per SM), where
// register-held loads need 32 warps per SM and every register of them.
//
// Stash. Pass 1 keeps u in a ring buffer in the rest of the CTA's shared
// memory (sp_ring.h), so pass 2 re-reads only p (mostly an L2 hit: it was
// read in pass 1 shortly before) and writes p': 24 + b + 8 B per element.
//
// Replicated mode (every rank steps the whole vector) streams: CTAs claim
// chunks tensor by tensor (largest first) from one queue; a CTA puts u of
// each chunk it claims into its ring and the chunk into a FIFO; a tensor's
// norms are complete as soon as its last chunk is counted (the CTA that
// counts it sums the chunk partials and publishes lr * trust), and from then
// on the CTAs holding chunks of that tensor run their pass 2: up to two
// FIFO entries beside every pass-1 chunk (their loads issued before the
// pass-1 math, which reads only shared memory), and in iterations without
// a pass-1 chunk as many as the stage's four areas hold (p, and m', v' of
// entries without stash, bulk-copied after a proxy fence). No grid-wide
// barrier: a chunk waits only for its own tensor. A chunk for which the
// ring has no room is queued without stash (u recomputed from p, m', v',
// which the same thread stored in pass 1); only with the FIFO full does a
// chunk go to a global overflow list, processed at the end by any CTA.
//
// Warps. kLambDataWarps data warps run the iterations on their own, waiting
// only on the stage's `full` mbarrier and reporting each iteration on its
// `empty` mbarrier; two control warps keep every global round trip off
// them:
//   claims  once iteration i is done, fills the slot of iteration
//           i + kLambStages and issues its bulk copies into the stage i
//           freed, for a chunk claimed two steps earlier whose descriptor
//           it fetched with cp.async; probes the ready word of the FIFO
//           head's tensor while it fills;
//   books   publishes each iteration's norm partial, counts it for its
//           tensor and completes a tensor whose count is full.
// No fences on this path: partials and ready words carry the launch's tag
// in the same 64-bit word as the value (single-copy atomic), so a reader
// that sees the tag sees the value; readers of a partial spin on the tag.
//
// Sharded mode (ZeRO-1 style): the same loop over this
// rank's owned range without pass 2 (it needs every rank's norms); then the
// last CTA to arrive stores this rank's (sum p^2, sum u^2) of every tensor
// into slot [rank][t] of every rank's norm table (NVLink stores), runs the
// cross-rank barrier and releases the grid; pass 2 forms trust_t from the
// world slots in rank order and stores p' into every rank's parameter
// vector.
//
// Norms (deterministic, same bits on every replica and for any grid size):
// per chunk, per-thread fp32 fmaf chains, warp xor tree, warps summed in
// order -> one partial pair per chunk; per tensor the chunk partials are
// summed in fp64 by one warp (lanes strided in chunk order, xor tree).
// Queues and counters live in global memory: the grid is launched
// cooperatively (all CTAs co-resident) and the last CTA out resets them and
// advances the tag (graph-replay safe).
#pragma once

#include "sp_kernels.cuh"
#include "sp_ring.h"

namespace sp {

constexpr int kFifo = 64;  // chunks a CTA holds for pass 2 at once (more: overflow)
constexpr int kDrain = 4;  // pass-2 entries per iteration without a pass-1 chunk
constexpr int kP2Beside = 2;  // pass-2 entries beside a pass-1 chunk (3 and 4 measured slower)
constexpr int kSlots = kLambStages + 2;  // iteration i uses slot i % kSlots
constexpr int kCtlWarp = kLambDataWarps, kBooksWarp = kLambDataWarps + 1;
static_assert(kLambTile <= 6144, "a chunk's q8 scales (block >= 512) fit the 16-float staging window");

struct LambPlan {
  const Chunk* chunks;            // claim order: tensor by tensor, largest first
  int nchunks;
  const int2* tchunk;             // per tensor: chunks [x, y) (empty: none on this rank)
  unsigned long long* partial;    // per chunk: (sum p^2, tag), (sum u^2, tag)
  int* ovf;                       // overflow chunk ids (recomputed at the end)
  int* cnt;                       // counters (below)
  float* trust;                   // per tensor (what sp_round_read(SP_BUF_TRUST) returns)
  float* step_scale;              // per tensor: lr * trust
  int cap;                        // stash floats per CTA
  int T;
  // sharded mode
  int shard;
  double2* table[SP_MAX_RANKS];   // norm table of rank (rank + 1 + k) % world (self last)
  const double2* my_table;        // this rank's [world][T]
  ParamPush push;
  BarrierArgs bar;                // cross-rank barrier (flags, epoch, err)
  unsigned long long* trace;      // SP_LAMB_TRACE builds: per-CTA globaltimer stamps

  __device__ int* head() const { return cnt + 0; }
  __device__ int* ovf_n() const { return cnt + 1; }
  __device__ int* ovf_claim() const { return cnt + 2; }
  __device__ int* arrive() const { return cnt + 3; }
  __device__ int* release_flag() const { return cnt + 4; }
  __device__ int* exited() const { return cnt + 5; }
  __device__ unsigned* tag_word() const { return reinterpret_cast<unsigned*>(cnt + 6); }  // not reset
  __device__ int* done(int t) const { return cnt + 8 + t; }
  // per tensor: (lr * trust bits, tag); tagged, so never reset
  __device__ unsigned long long* ready(int t) const {
    return reinterpret_cast<unsigned long long*>(cnt + ((8 + T + 1) & ~1)) + t;
  }
  __device__ int nreset() const { return 8 + T; }
};

// host: ints of LambPlan::cnt
inline size_t lamb_counter_ints(int T) { return (size_t)((8 + T + 1) & ~1) + 2 * (size_t)T; }

// SP_LAMB_TRACE builds: per CTA kLambTraceStride words: [0, 64) globaltimer
// stamps (LAMB_STAMP), then clock64 stamps of the first 128 iterations
// (LAMB_ITER: 8 per iteration).
constexpr int kLambTraceStride = 64 + 128 * 8;
#ifdef SP_LAMB_TRACE
#define LAMB_STAMP(k)                                                                                      \
  do {                                                                                                     \
    if (threadIdx.x == 0 && pl.trace) pl.trace[(size_t)blockIdx.x * kLambTraceStride + (k)] = globaltimer(); \
  } while (0)
#define LAMB_ITER(it, j)                                                                              \
  do {                                                                                                \
    if (pl.trace && (it) < 128) pl.trace[(size_t)blockIdx.x * kLambTraceStride + 64 + (it) * 8 + (j)] = \
        (unsigned long long)clock64();                                                               \
  } while (0)
#else
#define LAMB_STAMP(k) \
  do {                \
  } while (0)
#define LAMB_ITER(it, j) \
  do {                   \
  } while (0)
#endif

// ------------------------------------------------------------ primitives
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// all but the newest group complete
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// expect `bytes` more of bulk copies on the current phase
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// the producer's arrival (count 1): the phase completes once the expected
// bytes have landed
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// a bulk copy counted on bar
__device__ __forceinline__ void bulk_counted(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  mbar_expect_tx(bar, bytes);
  bulk_g2s(dst, src, bytes, bar);
}

__device__ __forceinline__ unsigned long long tagged(float x, unsigned tag) {
  return ((unsigned long long)tag << 32) | (unsigned long long)__float_as_uint(x);
}

__device__ __forceinline__ float trust_of(double x, double y) {
  const double r1 = sqrt(x), r2 = sqrt(y);
  return (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
}

__device__ __forceinline__ void publish_partial(const LambPlan& pl, int item, float x, float y, unsigned tag) {
  pl.partial[2 * (size_t)item] = tagged(x, tag);
  pl.partial[2 * (size_t)item + 1] = tagged(y, tag);
}

// One partial of this launch (spins until the word carries the tag).
__device__ __forceinline__ float partial_word(const unsigned long long* w, unsigned long long v, unsigned tag) {
  while ((unsigned)(v >> 32) != tag) v = ld_relaxed_u64(w);
  return __uint_as_float((unsigned)v);
}

// fp64 sums of tensor t's chunk partials by the calling warp: lanes strided
// in chunk order with 8 pairs in flight each, then an xor tree (both lanes
// of every pair add the same two operands, so every lane ends with the same
// bits). Depends only on the chunk table.
__device__ __forceinline__ double2 tensor_sums(const LambPlan& pl, int t, unsigned tag) {
  const int lane = threadIdx.x & 31;
  const int2 r = pl.tchunk[t];
  double x = 0.0, y = 0.0;
  for (int q0 = r.x + lane; q0 < r.y; q0 += 8 * 32) {
    unsigned long long v[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = q0 + 32 * j;
      v[j][0] = v[j][1] = (unsigned long long)tag << 32;  // absent: 0.0f with the tag
      if (q < r.y) {
        v[j][0] = ld_relaxed_u64(pl.partial + 2 * (size_t)q);
        v[j][1] = ld_relaxed_u64(pl.partial + 2 * (size_t)q + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = q0 + 32 * j;
      x += (double)partial_word(pl.partial + 2 * (size_t)q, v[j][0], tag);
      y += (double)partial_word(pl.partial + 2 * (size_t)q + 1, v[j][1], tag);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
  return make_double2(x, y);
}

// --------------------------------------------------------------- pass 1
// Thread t handles body vector t of a chunk (a chunk is at most one tile)
// and, for the unaligned edges, head element t (t < head) or tail element
// t - 32 (32 <= t < 32 + tail). Pass 2 uses the same mapping, so each thread
// reads back exactly the stash words (and, for a chunk without stash, the
// m', v') it wrote.

template <int W, bool FP>
__device__ __forceinline__ void p1_vec(const LambArgs& a, const LambScalars& s, int64_t i, float4 g,
                                       float4 p, float4 m, float4 v, float* st, float& pp, float& uu) {
  float4 u;
  lamb_moments(a, s, g.x, p.x, m.x, v.x, u.x);
  lamb_moments(a, s, g.y, p.y, m.y, v.y, u.y);
  lamb_moments(a, s, g.z, p.z, m.z, v.z, u.z);
  lamb_moments(a, s, g.w, p.w, m.w, v.w, u.w);
  *reinterpret_cast<float4*>(a.m + i) = m;
  *reinterpret_cast<float4*>(a.v + i) = v;
  if (st) *reinterpret_cast<float4*>(st) = u;
  pp = __fmaf_rn(p.x, p.x, pp); pp = __fmaf_rn(p.y, p.y, pp);
  pp = __fmaf_rn(p.z, p.z, pp); pp = __fmaf_rn(p.w, p.w, pp);
  uu = __fmaf_rn(u.x, u.x, uu); uu = __fmaf_rn(u.y, u.y, uu);
  uu = __fmaf_rn(u.z, u.z, uu); uu = __fmaf_rn(u.w, u.w, uu);
}

// Pass 1 of a staged chunk. st: the chunk's stash (indexed by element -
// c.start), or nullptr.
template <int W, bool FP>
__device__ __forceinline__ void p1_staged(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                          const unsigned char* stg, int goff, const float* qs, long long qs0,
                                          float* st, float& pp, float& uu) {
  const ChunkSplit sp = split_chunk(c.start, c.len);
  const int t = threadIdx.x;
  const int64_t b0 = sp.start + sp.head;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = b0 + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float gs = load_grad1<W, FP>(a, si);
    const float ps = a.p[si];
    float ms = a.m[si], vs = a.v[si], us;
    lamb_moments(a, s, gs, ps, ms, vs, us);
    a.m[si] = ms;
    a.v[si] = vs;
    if (st) st[si - c.start] = us;
    pp = __fmaf_rn(ps, ps, pp);
    uu = __fmaf_rn(us, us, uu);
  }
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = t + j * kLambDataThreads;  // body vector
    if (v < sp.nbody4) {
      const int64_t i = b0 + 4 * (int64_t)v;
      GradRaw g;
      if constexpr (FP || W == SP_WIRE_FP32) {
        g.f = reinterpret_cast<const float4*>(stg)[v];
      } else if constexpr (W == SP_WIRE_FP16) {
        g.h = *reinterpret_cast<const uint2*>(stg + goff + 8 * v);
      } else {
        g.q = *reinterpret_cast<const uint32_t*>(stg + goff + 4 * v);
        g.s = qs[(i >> a.qshift) - qs0];  // the chunk's q8 scales, staged
      }
      const float4* pmv = reinterpret_cast<const float4*>(stg + kLambStageG);
      p1_vec<W, FP>(a, s, i, grad_finish<W, FP>(a, i, g), pmv[v], pmv[kLambTile / 4 + v],
                    pmv[2 * (kLambTile / 4) + v], st ? st + (i - c.start) : nullptr, pp, uu);
    }
  }
}

// --------------------------------------------------------------- pass 2
__device__ __forceinline__ float4 p2_vec(float neg, float4 p, float4 u) {
  return make_float4(__fmaf_rn(neg, u.x, p.x), __fmaf_rn(neg, u.y, p.y), __fmaf_rn(neg, u.z, p.z),
                     __fmaf_rn(neg, u.w, p.w));
}

__device__ __forceinline__ float4 dir4(const LambArgs& a, const LambScalars& s, float4 p, float4 m,
                                       float4 v) {
  return make_float4(lamb_dir(a, s, p.x, m.x, v.x), lamb_dir(a, s, p.y, m.y, v.y),
                     lamb_dir(a, s, p.z, m.z, v.z), lamb_dir(a, s, p.w, m.w, v.w));
}

// Loads of a pass-2 chunk's body issued ahead of their use: m', v' (no
// stash), or p (p not staged).
struct P2Regs {
  float4 m[kLambVec], v[kLambVec];
};
__device__ __forceinline__ const P2Regs& r0_dummy() {
  static __device__ P2Regs z;
  return z;
}

__device__ __forceinline__ void p2_load_p(const LambArgs& a, long long start, int len, P2Regs& r) {
  const ChunkSplit sp = split_chunk(start, len);
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = threadIdx.x + j * kLambDataThreads;
    if (v < sp.nbody4) r.m[j] = *reinterpret_cast<const float4*>(a.p + sp.start + sp.head + 4 * (int64_t)v);
  }
}

__device__ __forceinline__ void p2_load_mv(const LambArgs& a, long long start, int len, P2Regs& r) {
  const ChunkSplit sp = split_chunk(start, len);
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = threadIdx.x + j * kLambDataThreads;
    if (v < sp.nbody4) {
      const int64_t i = sp.start + sp.head + 4 * (int64_t)v;
      r.m[j] = *reinterpret_cast<const float4*>(a.m + i);
      r.v[j] = *reinterpret_cast<const float4*>(a.v + i);
    }
  }
}

// Pass 2 of a chunk whose body p is staged at ps, or (ps null, stashed)
// already loaded into mv.m (replicated: p' overwrites p). u from the stash,
// or recomputed from m', v' (already loaded into mv when have_mv).
__device__ __forceinline__ void p2_staged(const LambArgs& a, const LambScalars& s, long long start, int len,
                                          const float4* ps, const float* st, float neg, bool have_mv,
                                          const P2Regs& mv) {
  const ChunkSplit sp = split_chunk(start, len);
  const int t = threadIdx.x;
  const int64_t b0 = sp.start + sp.head;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = b0 + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float p = a.p[si];
    const float u = st ? st[si - start] : lamb_dir(a, s, p, a.m[si], a.v[si]);
    a.p[si] = __fmaf_rn(neg, u, p);
  }
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = t + j * kLambDataThreads;
    if (v < sp.nbody4) {
      const int64_t i = b0 + 4 * (int64_t)v;
      const float4 p = ps ? ps[v] : mv.m[j];
      float4 u;
      if (st) u = *reinterpret_cast<const float4*>(st + (i - start));
      else if (have_mv) u = dir4(a, s, p, mv.m[j], mv.v[j]);
      else u = dir4(a, s, p, *reinterpret_cast<const float4*>(a.m + i), *reinterpret_cast<const float4*>(a.v + i));
      *reinterpret_cast<float4*>(a.p + i) = p2_vec(neg, p, u);
    }
  }
}

// p' = p - (lr * trust) * u, u from the stash or recomputed (bit-identical:
// lamb_dir is pass 1's u expression on the stored m', v'), loads issued by
// the thread (sharded pass 2 and the overflow chunks). Replicated: p'
// overwrites p. Sharded: p' goes to every rank's copy, the local one last.
__device__ __forceinline__ void p2_chunk(const LambArgs& a, const LambScalars& s, long long start, int len,
                                         const float* st, float neg, const ParamPush* push) {
  const ChunkSplit sp = split_chunk(start, len);
  const int t = threadIdx.x;
  const int64_t b0 = sp.start + sp.head;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = b0 + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float ps = a.p[si];
    const float us = st ? st[si - start] : lamb_dir(a, s, ps, a.m[si], a.v[si]);
    const float q = __fmaf_rn(neg, us, ps);
    if (push)
      for (int k = 0; k < push->ndst; ++k) push->dst[k][si] = q;
    else
      a.p[si] = q;
  }
#pragma unroll
  for (int jv = 0; jv < kLambVec; ++jv) {
    const int v = t + jv * kLambDataThreads;
    if (v < sp.nbody4) {
      const int64_t i = b0 + 4 * (int64_t)v;
      const float4 p = *reinterpret_cast<const float4*>(a.p + i);
      const float4 u = st ? *reinterpret_cast<const float4*>(st + (i - start))
                          : dir4(a, s, p, *reinterpret_cast<const float4*>(a.m + i),
                                 *reinterpret_cast<const float4*>(a.v + i));
      const float4 q = p2_vec(neg, p, u);
      if (push) {
        const int4 o = make_int4(__float_as_int(q.x), __float_as_int(q.y), __float_as_int(q.z),
                                 __float_as_int(q.w));
        for (int j = 0; j < push->ndst; ++j) st_v4(push->dst[j] + i, o);
      } else {
        *reinterpret_cast<float4*>(a.p + i) = q;
      }
    }
  }
}

// Pass 2 of a FIFO entry with p (and, without stash, m' and v') staged
// (replicated: p' overwrites p).
template <typename E>
__device__ __forceinline__ void p2_drain(const LambArgs& a, const LambScalars& s, const E& e, const float4* ps,
                                         const float4* ms, const float4* vs, const float* st, float neg) {
  const int t = threadIdx.x;
  const int head = (int)(e.b0 - e.start), tail = e.len - head - 4 * e.nb;
  int64_t si = -1;
  if (t < head) si = e.start + t;
  else if (t >= 32 && t - 32 < tail) si = e.b0 + 4 * (int64_t)e.nb + (t - 32);
  if (si >= 0) {
    const float p = a.p[si];
    const float u = st ? st[si - e.start] : lamb_dir(a, s, p, a.m[si], a.v[si]);
    a.p[si] = __fmaf_rn(neg, u, p);
  }
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = t + j * kLambDataThreads;
    if (v < e.nb) {
      const int64_t i = e.b0 + 4 * (int64_t)v;
      const float4 p = ps[v];
      const float4 u = st ? *reinterpret_cast<const float4*>(st + (i - e.start)) : dir4(a, s, p, ms[v], vs[v]);
      *reinterpret_cast<float4*>(a.p + i) = p2_vec(neg, p, u);
    }
  }
}

// Sharded pass 2 of a FIFO entry in two halves: the body loads (p, and m',
// v' without stash), then the update stored to every rank's copy.
struct P2Full {
  float4 p[kLambVec], m[kLambVec], v[kLambVec];
};

template <typename E>
__device__ __forceinline__ void p2_load_full(const LambArgs& a, const E& e, P2Full& r) {
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = threadIdx.x + j * kLambDataThreads;
    if (v < e.nb) {
      const int64_t i = e.b0 + 4 * (int64_t)v;
      r.p[j] = *reinterpret_cast<const float4*>(a.p + i);
      if (e.off < 0) {
        r.m[j] = *reinterpret_cast<const float4*>(a.m + i);
        r.v[j] = *reinterpret_cast<const float4*>(a.v + i);
      }
    }
  }
}

template <typename E>
__device__ __forceinline__ void p2_finish_full(const LambArgs& a, const LambScalars& s, const E& e,
                                               const float* st, float neg, const ParamPush* push, const P2Full& r) {
  const int t = threadIdx.x;
  const int head = (int)(e.b0 - e.start), tail = e.len - head - 4 * e.nb;
  int64_t si = -1;
  if (t < head) si = e.start + t;
  else if (t >= 32 && t - 32 < tail) si = e.b0 + 4 * (int64_t)e.nb + (t - 32);
  if (si >= 0) {
    const float ps = a.p[si];
    const float us = st ? st[si - e.start] : lamb_dir(a, s, ps, a.m[si], a.v[si]);
    const float q = __fmaf_rn(neg, us, ps);
    if (push)
      for (int k = 0; k < push->ndst; ++k) push->dst[k][si] = q;
    else
      a.p[si] = q;
  }
#pragma unroll
  for (int j = 0; j < kLambVec; ++j) {
    const int v = t + j * kLambDataThreads;
    if (v < e.nb) {
      const int64_t i = e.b0 + 4 * (int64_t)v;
      const float4 u = st ? *reinterpret_cast<const float4*>(st + (i - e.start)) : dir4(a, s, r.p[j], r.m[j], r.v[j]);
      const float4 q = p2_vec(neg, r.p[j], u);
      if (push) {
        const int4 o = make_int4(__float_as_int(q.x), __float_as_int(q.y), __float_as_int(q.z),
                                 __float_as_int(q.w));
        for (int k = 0; k < push->ndst; ++k) st_v4(push->dst[k] + i, o);
      } else {
        *reinterpret_cast<float4*>(a.p + i) = q;
      }
    }
  }
}

// -lr * trust of tensor t for the overflow and sharded pass 2 (the same bits
// everywhere: replicated, the published lr * trust; sharded, the world's
// pairs summed in rank order).
__device__ __forceinline__ float neg_of(const LambPlan& pl, const LambScalars& s, int t) {
  if (!pl.shard) return -__ldcg(pl.step_scale + t);
  double x = 0.0, y = 0.0;
  for (int k = 0; k < pl.bar.world; ++k) {
    const double2 q = __ldcg(pl.my_table + (size_t)k * pl.T + t);
    x += q.x;
    y += q.y;
  }
  return -__fmul_rn(s.lr, trust_of(x, y));
}

// Overflow chunks (no FIFO room), recomputed from p, m', v': claimed by any
// CTA once pass 1 is complete everywhere.
__device__ void overflow_pass2(const LambArgs& a, const LambScalars& s, const LambPlan& pl, int* s_k) {
  const ParamPush* push = pl.shard ? &pl.push : nullptr;
  const int novf = __ldcg(pl.ovf_n());
  if (novf == 0) return;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) *s_k = atomicAdd(pl.ovf_claim(), 1);
    __syncthreads();
    const int k = *s_k;
    if (k >= novf) break;
    const Chunk c = pl.chunks[__ldcg(pl.ovf + k)];
    if (threadIdx.x < kLambDataThreads) p2_chunk(a, s, c.start, c.len, nullptr, neg_of(pl, s, c.tensor), push);
  }
}

// ------------------------------------------------------------ the stream
struct FifoEntry {
  long long start;
  long long b0;  // first body element
  int len;
  int off;       // stash offset of element `start` (float index, = start mod 4); -1: recompute
  int tensor;
  int nb;        // body vectors
};

// Claims lane state, in registers (its step is a chain of dependent
// updates; in shared memory each would cost a load round trip).
struct Ctl {
  int fhead, fnext, ftail;  // FIFO: oldest entry, next to hand to pass 2, one past the newest
  Ring ring;                // the stash ring (sp_ring.h)
  int ready_t;              // last tensor seen ready (-1: none)
  float ready_neg;          // its -lr * trust
  int probe_t;              // tensor whose ready word is in flight (-1: none)
  int pdesc[2];             // chunks whose descriptors are in flight to sh.pdesc (>= nchunks: none)
  int claims_done;          // the queue is exhausted for this CTA
};

// Books lane state, in registers.
struct Books {
  int arrived;   // counted in pl.arrive() (every partial of this CTA out)
  int novf;      // chunks this CTA could not stash (trace builds report it)
};

struct StreamShared {
  unsigned long long full[kLambStages];   // stage mbarriers: slot filled and its bulk copies landed
  unsigned long long empty[kLambStages];  // stage mbarriers: every data warp done with the iteration
  float red_p[kSlots][kLambDataWarps], red_u[kSlots][kLambDataWarps];
  Chunk desc[kSlots];            // pass-1 chunk of the iteration
  int idx[kSlots];               // its index (>= nchunks: none)
  int off[kSlots];               // its stash offset (-1: recompute, -2: global overflow)
  int goff[kSlots];              // its first body gradient in the stage's g area
  alignas(16) float qs[kSlots][16];  // q8: the chunk's block scales (an aligned window)
  long long qs0[kSlots];         // q8: block index of qs[.][0]
  FifoEntry e2[kSlots][kDrain];  // pass-2 entries of the iteration (kDrain >= 2)
  int area2[kSlots][kDrain];     // without a pass-1 chunk: each entry's first stage area
  float neg2[kSlots][kDrain];    // their -lr * trust
  int n2[kSlots];
  int stop[kSlots];              // 1: nothing left for this CTA
  FifoEntry fifo[kFifo];
  Chunk pdesc[2];                // descriptors prefetched by cp.async, two steps ahead
  int nfifo;                     // FIFO entries of the loop (sharded pass 2)
  volatile int books_done;       // iterations the books lane has finished
  volatile int iters_done;       // iterations every data warp has finished (claims lane)
  int k, flag;
  unsigned long long epoch;
};

// The four fp32 areas of a stage (g, p, m, v): in iterations without a
// pass-1 chunk they hold pass-2 entries.
__device__ __forceinline__ int stage_area(int k) { return k == 0 ? 0 : kLambStageG + (k - 1) * kLambArea; }

// Claims lane: the bulk copies of chunk ch's body (g, p, m, v, and the
// q8 block scales) into stage stg, counted on bar, for slot q. Wire formats
// narrower than 16 B per vector are fetched as an aligned superset;
// sh.goff[q] is the offset of the chunk's first body gradient in the g area.
template <int W, bool FP>
__device__ __forceinline__ void stage_copies(const LambArgs& a, const Chunk& ch, unsigned char* stg,
                                             unsigned long long* bar, StreamShared& sh, int q) {
  const int64_t b0 = ch.start + ch.head;
  const unsigned nb = (unsigned)ch.nbody4;
  if (nb) {
    const char* gsrc;
    unsigned gbytes;
    int goff = 0;
    if constexpr (FP) {
      gsrc = reinterpret_cast<const char*>(a.g32 + b0);
      gbytes = 16 * nb;
    } else if constexpr (W == SP_WIRE_FP32) {
      gsrc = reinterpret_cast<const char*>(static_cast<const float*>(a.avg) + b0);
      gbytes = 16 * nb;
    } else {
      constexpr int wb = W == SP_WIRE_FP16 ? 2 : 1;  // wire bytes per element
      const int64_t lo = (wb * b0) & ~(int64_t)15, hi = (wb * (b0 + 4 * (int64_t)nb) + 15) & ~(int64_t)15;
      gsrc = static_cast<const char*>(a.avg) + lo;
      gbytes = (unsigned)(hi - lo);
      goff = (int)(wb * b0 - lo);
    }
    sh.goff[q] = goff;
    if constexpr (W == SP_WIRE_Q8 && !FP) {  // the block scales the body needs, 16-byte window
      const int64_t s0 = b0 >> a.qshift, s1 = (b0 + 4 * (int64_t)nb - 1) >> a.qshift;
      const int64_t lo = s0 & ~(int64_t)3;
      const unsigned cnt = (unsigned)((s1 + 1 - lo + 3) & ~(int64_t)3);  // <= 16 (chunk <= 4096, block >= 512)
      sh.qs0[q] = lo;
      bulk_counted(sh.qs[q], a.avg_scale + lo, 4 * cnt, bar);
    }
    mbar_expect_tx(bar, gbytes + 48 * nb);
    bulk_g2s(stg, gsrc, gbytes, bar);
    bulk_g2s(stg + kLambStageG, a.p + b0, 16 * nb, bar);
    bulk_g2s(stg + kLambStageG + kLambArea, a.m + b0, 16 * nb, bar);
    bulk_g2s(stg + kLambStageG + 2 * kLambArea, a.v + b0, 16 * nb, bar);
  }
}

// Claims lane: chunk c (descriptor ch; >= nchunks: none) into slot q with
// its pass 2 queued; its copies issued here too unless the caller did.
template <int W, bool FP>
__device__ __forceinline__ void stream_fill(const LambArgs& a, const LambPlan& pl, Ctl& k, int q, int c,
                                            const Chunk& ch, unsigned char* stg, unsigned long long* bar,
                                            StreamShared& sh, bool copy = true) {
  sh.idx[q] = c;
  if (c >= pl.nchunks) return;
  sh.desc[q] = ch;
  if (copy) stage_copies<W, FP>(a, ch, stg, bar, sh, q);
  const int64_t b0 = ch.start + ch.head;
  const unsigned nb = (unsigned)ch.nbody4;
  int off = -2;
  if (k.ftail - k.fhead < kFifo) {
    off = ring_alloc(k.ring, pl.cap, ch.start, ch.len);
    if (off >= 0) ++k.ring.live;
    FifoEntry& e = sh.fifo[k.ftail % kFifo];
    e.start = ch.start;
    e.b0 = b0;
    e.len = ch.len;
    e.off = off;
    e.tensor = ch.tensor;
    e.nb = (int)nb;
    ++k.ftail;
  }
  sh.off[q] = off;
}

// Books warp, one step: publish this iteration's partial and count it for
// its tensor; the CTA that counts a tensor's last chunk sums the partials
// and publishes trust and the ready word. With no chunk: every count of
// this CTA is done, so it arrives.
__device__ __forceinline__ void books_step(const LambPlan& pl, const LambScalars& s, StreamShared& sh,
                                           unsigned tag, int slot, bool have1, int item, Books& k) {
  const int lane = threadIdx.x & 31;
  int last = -1;
  if (lane == 0) {
    if (have1) {
      const Chunk& c = sh.desc[slot];
      float x = 0.0f, y = 0.0f;
#pragma unroll
      for (int w = 0; w < kLambDataWarps; ++w) {
        x += sh.red_p[slot][w];
        y += sh.red_u[slot][w];
      }
      publish_partial(pl, item, x, y, tag);
      if (sh.off[slot] < 0) ++k.novf;
      if (sh.off[slot] == -2) pl.ovf[atomicAdd(pl.ovf_n(), 1)] = item;
      if (!pl.shard && atomicAdd(pl.done(c.tensor), 1) == c.tchunks - 1) last = c.tensor;
    } else if (!k.arrived && !pl.shard) {  // every write of this CTA's pass 1 is out
      __threadfence();
      atomicAdd(pl.arrive(), 1);
      k.arrived = 1;
#ifdef SP_LAMB_TRACE
      if (pl.trace) {
        pl.trace[(size_t)blockIdx.x * kLambTraceStride + 1] = globaltimer();
        pl.trace[(size_t)blockIdx.x * kLambTraceStride + 4] = k.novf;
      }
#endif
    }
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last >= 0) {
    const double2 t2 = tensor_sums(pl, last, tag);
    if (lane == 0) {
      const float tr = trust_of(t2.x, t2.y);
      const float sc = __fmul_rn(s.lr, tr);
      pl.trust[last] = tr;
      pl.step_scale[last] = sc;
      *pl.ready(last) = tagged(sc, tag);
    }
  }
}

// The chunk loop (both modes). Replicated: pass 2 of ready tensors
// interleaved. Sharded (pl.shard): pass 1 only; the FIFO keeps every
// chunk's entry for the pass 2 after the cross-rank barrier.
template <int W, bool FP>
__device__ void stream_loop(const LambArgs& a, const LambScalars& s, const LambPlan& pl, unsigned char* stages,
                            float* stash, StreamShared& sh, unsigned tag) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  Ctl k{};                           // claims lane
  Books bk{};                        // books lane
  // Registers written by a global atomic or load in one step and read in
  // the next are assigned unconditionally: a conditional assignment
  // compiles to a select, which waits for the value on the spot.
  int pend = pl.nchunks;             // claims: the claim issued one step earlier (in flight)
  unsigned long long probe = 0;      // claims: ready word of k.probe_t (in flight)
  auto claim = [&]() { return atomicAdd(pl.head(), 1); };
  // the descriptor of chunk c into buffer b (one commit group per call,
  // empty for no chunk, so that wait_group counts steps)
  auto fetch_desc = [&](int b, int c) {
    k.pdesc[b] = c;
    if (c < pl.nchunks) {
      cp_async16(&sh.pdesc[b], pl.chunks + c);
      cp_async16(reinterpret_cast<char*>(&sh.pdesc[b]) + 16, reinterpret_cast<const char*>(pl.chunks + c) + 16);
    }
    cp_async_commit();
  };
  // up to maxn FIFO entries of the tensor known ready, in FIFO order, their
  // body p copied into the stage (beside a pass-1 chunk: its p2 area; else
  // the g, p, m, v areas)
  // In an iteration without a pass-1 chunk the five areas of the stage are
  // shared out: p of a stashed entry takes one, p, m', v' of an entry
  // without stash three (m', v' were written by this CTA's threads in pass
  // 1: a proxy fence orders those stores before the bulk copies read them).
  auto pick2 = [&](int q, int maxn, bool p1, unsigned char* stg, unsigned long long* bar) {
    int n = 0, areas = 0;
    bool fenced = false;
    while (n < maxn && k.fnext < k.ftail) {
      const FifoEntry& e = sh.fifo[k.fnext % kFifo];
      if (e.tensor != k.ready_t) break;
      if (p1 && n >= 1 && e.off < 0) break;  // beside a pass-1 chunk, after the first: stashed only
      const int need = (p1 || e.off >= 0) ? 1 : 3;
      if (!p1 && areas + need > kLambStageAreas) break;
      sh.e2[q][n] = e;
      sh.neg2[q][n] = k.ready_neg;
      sh.area2[q][n] = areas;
      if (e.nb && !p1) {
        const unsigned bytes = 16 * (unsigned)e.nb;
        bulk_counted(stg + stage_area(areas), a.p + e.b0, bytes, bar);
        if (need == 3) {
          if (!fenced) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            fenced = true;
          }
          bulk_counted(stg + stage_area(areas + 1), a.m + e.b0, bytes, bar);
          bulk_counted(stg + stage_area(areas + 2), a.v + e.b0, bytes, bar);
        }
      }
      areas += need;
      ++n;
      ++k.fnext;
    }
    sh.n2[q] = n;
  };
  if (wid == kCtlWarp && lane == 0) {
    k.ready_t = -1;
    k.probe_t = -1;
    sh.books_done = 0;
    sh.iters_done = 0;
    for (int q = 0; q < kSlots; ++q) {
      sh.stop[q] = 0;
      sh.n2[q] = 0;
      sh.idx[q] = pl.nchunks;
    }
    for (int st = 0; st < kLambStages; ++st) {
      mbar_init(&sh.full[st], 1);
      mbar_init(&sh.empty[st], kLambDataWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kLambStages; ++q) {
      const int c = claim();
      if (c >= pl.nchunks) k.claims_done = 1;
      stream_fill<W, FP>(a, pl, k, q, c, c < pl.nchunks ? pl.chunks[c] : Chunk{},
                         stages + (size_t)q * kLambStageBytes, &sh.full[q], sh);
      mbar_arrive(&sh.full[q]);
    }
    for (int b = 0; b < 2; ++b) {
      const int c = k.claims_done ? pl.nchunks : claim();
      if (c >= pl.nchunks) k.claims_done = 1;
      fetch_desc(b, c);
    }
    pend = claim();
  }
  __syncthreads();
  if (wid < kLambDataWarps) {
    // Data warps: each runs the iterations on its own, waiting only for the
    // slot and stage of the next one (full) and reporting each one done
    // (empty).
    for (int it = 0;; ++it) {
      const int q = it % kSlots, stage = it % kLambStages;
      const unsigned ph = (unsigned)(it / kLambStages) & 1u;
      if (tid == 0) LAMB_ITER(it, 0);
      mbar_wait(&sh.full[stage], ph);
      if (tid == 0) LAMB_ITER(it, 1);
      const bool stop = sh.stop[q] != 0;
      if (!stop) {
        const int item = sh.idx[q];
        const bool have1 = item < pl.nchunks;
        const int n2 = sh.n2[q];
        float pp = 0.0f, uu = 0.0f;
        const unsigned char* stg = stages + (size_t)stage * kLambStageBytes;
#ifdef SP_LAMB_TRACE
        if (tid == 0 && pl.trace && !have1) {  // iterations without a pass-1 chunk: empty, drain
          unsigned long long* tw = pl.trace + (size_t)blockIdx.x * kLambTraceStride;
          if (tw[7] == 0) tw[7] = globaltimer();
          ++tw[n2 ? 6 : 5];
        }
#endif
        if (have1) {
          // Beside the pass-1 chunk up to two pass-2 entries: the first with
          // its p staged (and m', v' loaded here if it has no stash), the
          // second (stashed) with its p loaded here; these loads are in
          // flight during the pass-1 math, which reads only shared memory.
          P2Full r0;
          P2Regs r1[kP2Beside > 1 ? kP2Beside - 1 : 1];
          if (n2 >= 1) p2_load_full(a, sh.e2[q][0], r0);
#pragma unroll
          for (int j = 1; j < kP2Beside; ++j)
            if (j < n2) p2_load_p(a, sh.e2[q][j].start, sh.e2[q][j].len, r1[j - 1]);
          const int off = sh.off[q];
          p1_staged<W, FP>(a, s, sh.desc[q], stg, sh.goff[q], sh.qs[q], sh.qs0[q], off >= 0 ? stash + off : nullptr,
                           pp, uu);
          if (tid == 0) LAMB_ITER(it, 2);
          if (n2 >= 1) {
            const FifoEntry& e = sh.e2[q][0];
            p2_finish_full(a, s, e, e.off >= 0 ? stash + e.off : nullptr, sh.neg2[q][0], nullptr, r0);
          }
#pragma unroll
          for (int j = 1; j < kP2Beside; ++j)
            if (j < n2) {
              const FifoEntry& e = sh.e2[q][j];
              p2_staged(a, s, e.start, e.len, nullptr, stash + e.off, sh.neg2[q][j], true, r1[j - 1]);
            }
        } else {
          for (int j = 0; j < n2; ++j) {  // pass 2 only: p (and m', v') staged
            const FifoEntry& e = sh.e2[q][j];
            const int ar = sh.area2[q][j];
            p2_drain(a, s, e, reinterpret_cast<const float4*>(stg + stage_area(ar)),
                     e.off >= 0 ? nullptr : reinterpret_cast<const float4*>(stg + stage_area(ar + 1)),
                     e.off >= 0 ? nullptr : reinterpret_cast<const float4*>(stg + stage_area(ar + 2)),
                     e.off >= 0 ? stash + e.off : nullptr, sh.neg2[q][j]);
          }
        }
        if (tid == 0) LAMB_ITER(it, 3);
        pp = warp_sum(pp);
        uu = warp_sum(uu);
        if (lane == 0) {
          sh.red_p[q][wid] = pp;
          sh.red_u[q][wid] = uu;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[stage]);
      if (tid == 0) LAMB_ITER(it, 4);
      if (stop) break;
    }
  } else if (wid == kCtlWarp) {
    // Claims lane: once every data warp is done with iteration it, the slot
    // and stage of iteration it + stages. The whole warp loops (a barrier
    // after the loop needs it converged); lane 0 does the work and returns
    // 1 once it has produced the stop.
    auto claims_step = [&](int it) -> int {
      const int q = it % kSlots, stage = it % kLambStages;
      mbar_wait(&sh.empty[stage], (unsigned)(it / kLambStages) & 1u);
      sh.iters_done = it + 1;  // for the books lane (a counter: it may lag several phases)
      LAMB_ITER(it, 5);
      // the copies of iteration it + stages first: the stage is free, the
      // descriptor was fetched two steps ago
      const int sq = (it + kLambStages) % kSlots;
      const int b = it & 1;
      const int c = k.pdesc[b];
      cp_async_wait_1();
      unsigned char* stg = stages + (size_t)stage * kLambStageBytes;
      if (c < pl.nchunks) stage_copies<W, FP>(a, sh.pdesc[b], stg, &sh.full[stage], sh, sq);
      const int n2 = sh.n2[q];
      if (n2 > 0) {  // free the entries pass 2 just finished and their ring regions
        for (int j = 0; j < n2; ++j) {
          if (sh.fifo[k.fhead % kFifo].off >= 0) --k.ring.live;
          ++k.fhead;
        }
        for (int f = k.fhead; f < k.ftail; ++f)  // the oldest live region
          if (sh.fifo[f % kFifo].off >= 0) {
            k.ring.head = sh.fifo[f % kFifo].off;
            break;
          }
      }
      // the slot was last used by iteration it + stages - kSlots: the books
      // lane must be done with it
      while (sh.books_done < it + kLambStages - kSlots + 1) {
      }
      // the ready word of the FIFO head's tensor, unless known: in flight
      // while the slot is filled
      k.probe_t = -1;
      if (k.fnext < k.ftail && sh.fifo[k.fnext % kFifo].tensor != k.ready_t)
        k.probe_t = sh.fifo[k.fnext % kFifo].tensor;
      probe = ld_relaxed_u64(pl.ready(k.probe_t >= 0 ? k.probe_t : 0));
      stream_fill<W, FP>(a, pl, k, sq, c, sh.pdesc[b], stg, &sh.full[stage], sh, false);
      // the descriptor of the claim issued last step; claim again
      const int cn = k.claims_done ? pl.nchunks : pend;
      if (cn >= pl.nchunks) k.claims_done = 1;
      fetch_desc(b, cn);
      pend = claim();  // past the end once the queue is exhausted: harmless, reset at exit
      const bool p1 = c < pl.nchunks;
      int stop;
      if (pl.shard) {
        sh.n2[sq] = 0;
        stop = p1 ? 0 : 1;
      } else {
        if (k.probe_t >= 0 && (unsigned)(probe >> 32) == tag) {
          k.ready_t = k.probe_t;
          k.ready_neg = -__uint_as_float((unsigned)probe);
        }
        pick2(sq, p1 ? kP2Beside : kDrain, p1, stg, &sh.full[stage]);
        // nothing left: no chunk, no entry now or later; else (an entry's
        // tensor not ready yet) an empty iteration that polls again
        stop = (!p1 && sh.n2[sq] == 0 && k.fnext >= k.ftail) ? 1 : 0;
        if (!p1 && sh.n2[sq] == 0 && !stop) __nanosleep(100);
      }
      sh.stop[sq] = stop;
      LAMB_ITER(it, 6);
      mbar_arrive(&sh.full[stage]);  // iteration it + stages is ready
      LAMB_ITER(it, 7);
      return stop;
    };
    for (int it = 0;; ++it) {
      int brk = 0;
      if (lane == 0) brk = claims_step(it);
      if (__shfl_sync(0xffffffffu, brk, 0)) {
        // the stop is iteration it + stages: keep counting the ones before
        // it for the books lane
        for (int j = it + 1; lane == 0 && j < it + kLambStages; ++j) {
          mbar_wait(&sh.empty[j % kLambStages], (unsigned)(j / kLambStages) & 1u);
          sh.iters_done = j + 1;
        }
        __syncwarp();
        break;
      }
    }
  } else if (wid == kBooksWarp) {
    // Books lane: once iteration it is done, its partial and count.
    for (int it = 0;; ++it) {
      const int q = it % kSlots;
      // wait until every data warp is done with iteration it, or it is the
      // stop (the claims lane sets that flag and stops counting)
      const volatile int* stopq = &sh.stop[q];
      while (!*stopq && sh.iters_done <= it) {
      }
      if (*stopq) break;
      const int item = sh.idx[q];
      books_step(pl, s, sh, tag, q, item < pl.nchunks, item, bk);
      __syncwarp();
      if (lane == 0) sh.books_done = it + 1;
    }
  }
  if (wid == kCtlWarp && lane == 0) sh.nfifo = k.ftail;
  if (wid == kBooksWarp && !pl.shard) {  // the arrive, if no empty iteration made it
    books_step(pl, s, sh, tag, 0, false, pl.nchunks, bk);
  }
}

template <int W, bool FP>
__device__ void stream_replicated(const LambArgs& a, const LambScalars& s, const LambPlan& pl,
                                  unsigned char* stages, float* stash, StreamShared& sh, unsigned tag) {
  stream_loop<W, FP>(a, s, pl, stages, stash, sh, tag);
  LAMB_STAMP(2);
  // overflow chunks need every CTA's pass 1
  if (threadIdx.x == 0)
    while (ld_acquire_gpu(reinterpret_cast<const unsigned*>(pl.arrive())) < gridDim.x) __nanosleep(64);
  __syncthreads();
  overflow_pass2(a, s, pl, &sh.k);
}

// ----------------------------------------------------------- sharded LAMB
template <int W, bool FP>
__device__ void shard_lamb(const LambArgs& a, const LambScalars& s, const LambPlan& pl, unsigned char* stages,
                           float* stash, StreamShared& sh, unsigned tag) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  stream_loop<W, FP>(a, s, pl, stages, stash, sh, tag);
  LAMB_STAMP(1);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sh.flag = atomicAdd(pl.arrive(), 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (sh.flag) {  // the last CTA: every partial of this rank is out
    // this rank's pair of every tensor (zero where it owns no chunk) into
    // slot [rank][t] of every rank's norm table, one warp per tensor
    for (int t = wid; t < pl.T; t += kLambThreads / 32) {
      const double2 q = tensor_sums(pl, t, tag);
      if (lane < pl.push.ndst) pl.table[lane][(size_t)pl.bar.rank * pl.T + t] = q;
    }
    __threadfence_system();
    __syncthreads();
    // cross-rank barrier (k_barrier's protocol)
    if (tid == 0) {
      sh.epoch = *pl.bar.epoch + 1;
      *pl.bar.epoch = sh.epoch;
    }
    __syncthreads();
    const unsigned long long epoch = sh.epoch;
    if (tid < pl.bar.world) {
      st_release_sys(pl.bar.flags[tid] + pl.bar.rank, epoch);
      const unsigned long long* mine = pl.bar.flags[pl.bar.rank] + tid;
      const unsigned long long t0 = globaltimer();
      while (ld_acquire_sys(mine) < epoch) {
        if (globaltimer() - t0 > pl.bar.timeout_ns) {
          atomicExch_system(pl.bar.err, 1);
          break;
        }
      }
    }
    __syncthreads();
    for (int t = tid; t < pl.T; t += kLambThreads) {  // trust of every tensor, rank order
      double x = 0.0, y = 0.0;
      for (int k = 0; k < pl.bar.world; ++k) {
        const double2 q = __ldcg(pl.my_table + (size_t)k * pl.T + t);
        x += q.x;
        y += q.y;
      }
      const float tr = trust_of(x, y);
      pl.trust[t] = tr;
      pl.step_scale[t] = __fmul_rn(s.lr, tr);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(reinterpret_cast<unsigned*>(pl.release_flag()), 1u);
    }
  }
  if (tid == 0)
    while (ld_acquire_gpu(reinterpret_cast<const unsigned*>(pl.release_flag())) == 0u) __nanosleep(32);
  __syncthreads();
  LAMB_STAMP(2);
  // pass 2 of every FIFO entry of this CTA (nothing was picked), the loads
  // of the next entry in flight while the current one is finished
  const int nf = sh.nfifo;
  if (tid < kLambDataThreads && nf > 0) {
    P2Full cur, nxt;
    p2_load_full(a, sh.fifo[0], cur);
    for (int f = 0; f < nf; ++f) {
      const FifoEntry e = sh.fifo[f];
      if (f + 1 < nf) p2_load_full(a, sh.fifo[f + 1], nxt);
      p2_finish_full(a, s, e, e.off >= 0 ? stash + e.off : nullptr, -__ldcg(pl.step_scale + e.tensor), &pl.push,
                     cur);
      cur = nxt;
    }
  }
  overflow_pass2(a, s, pl, &sh.k);
}

// --------------------------------------------------------------- kernel
template <int W, bool FP>
__global__ void __launch_bounds__(kLambThreads, kLambCtasPerSm) k_lamb(LambArgs a, LambPlan pl) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  __shared__ StreamShared sh;
  unsigned char* stages = dyn_smem;
  float* stash = reinterpret_cast<float*>(dyn_smem + (size_t)kLambStages * kLambStageBytes);
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const unsigned tag = __ldcg(pl.tag_word()) + 1u;  // this launch's tag
#ifdef SP_LAMB_TRACE
  if (threadIdx.x == 0 && pl.trace)
    for (int k = 5; k < 8; ++k) pl.trace[(size_t)blockIdx.x * kLambTraceStride + k] = 0;
#endif
  LAMB_STAMP(0);
  if (!pl.shard) stream_replicated<W, FP>(a, s, pl, stages, stash, sh, tag);
  else shard_lamb<W, FP>(a, s, pl, stages, stash, sh, tag);
  LAMB_STAMP(3);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(pl.exited(), 1) == (int)gridDim.x - 1) {  // last CTA out resets the counters
      const int nc = pl.nreset();
      for (int k = 0; k < nc; ++k)
        if (k != 6) pl.cnt[k] = 0;
      *pl.tag_word() = tag;  // the next launch uses tag + 1
      __threadfence();
    }
  }
}

}  // namespace sp
