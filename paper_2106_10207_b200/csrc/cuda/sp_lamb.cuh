// sp_lamb.cuh — the LAMB step of the round (K3 + K4) as one cooperative
// persistent kernel: 1024 / kLambThreads CTAs per SM, chunks claimed
// dynamically from per-window work queues.
//
// LAMB needs every tensor's norms ||p||, ||u|| before any element of it can
// be updated, so each element is touched twice: pass 1 (m' = b1 m + (1-b1) g,
// v' = ..., u = m'^/(sqrt(v'^)+eps) + wd p, norm partials) and pass 2
// (p' = p - lr * trust_t * u). Re-reading p, m', v' in pass 2 costs 12 B per
// element of L2 traffic on top of pass 1's 24 + b, and on B200 the L2 slice
// throughput (~6.3 KB/clk chip-wide, /opt/skills/guides/B300_MICROARCH.md
// "LTS throughput cap") binds hits and misses alike: the round-1 kernel
// moved 44 B/element through L2 at 6.35 TB/s.
//
// Here pass 1 keeps u in shared memory (the "stash": the SM's shared memory
// split over its CTAs, ~57 K floats per SM), so pass 2 re-reads only p (4 B,
// L2-resident: pass 1 loads it with an evict_last hint) and writes p':
// 24 + b + 8 B per element.
//
// Replicated mode (every rank steps the whole vector). Tensors are packed
// into windows that fit half of all stashes (~4.2 M elements on 148 SMs;
// the largest ALBERT-large tensor has 4,194,304). A CTA runs
//     pass1(w0) arrive(w0) | pass1(w1) arrive(w1) wait(w0) pass2(w0) |
//     pass1(w2) arrive(w2) wait(w1) pass2(w1) | ... wait(last) pass2(last)
// alternating the two stash halves, so the barrier of window w is
// split-phase: its wait comes one window of work after its arrive. In pass 1
// CTAs claim chunks from the window's queue (a static split left the
// slowest SMs 1.7x behind the median, profiles/r02/lamb_trace.txt); a CTA
// stashes u of its chunks while its half has room and lists the rest as
// overflow, which pass 2 recomputes from p, m', v' (any CTA, claimed from
// the overflow list). The CTA that finishes the last chunk of a tensor sums
// the tensor's chunk partials and publishes lr * trust.
//
// Sharded mode (ZeRO-1 style): one window, this rank's owned
// range, stashed in the whole buffer. The last finisher of a tensor stores
// this rank's (sum p^2, sum u^2) into slot [rank][t] of every rank's norm
// table (NVLink stores); after the grid barrier CTA 0 runs the cross-rank
// barrier, and pass 2 forms trust_t from the world slots in rank order and
// stores p' into every rank's parameter vector.
//
// Norms (deterministic, same bits on every replica and for any grid size):
// per chunk, per-thread fp32 fmaf chains, warp xor tree, warps summed in
// order -> one float2 partial per chunk; per tensor the chunk partials are
// summed in fp64 by one warp (lanes strided in chunk order, xor tree).
// All barriers and queues are counters in global memory: the grid is
// launched cooperatively (all CTAs co-resident) and the last CTA out resets
// them (graph-replay safe).
#pragma once

#include "sp_kernels.cuh"

namespace sp {

constexpr int kStashList = 32;  // stashed chunks a CTA remembers per window (more: overflow)

struct LambPlan {
  const Chunk* chunks;      // all chunks, window by window, in element order
  const int2* wchunk;       // per window: chunks [x, y)
  const int2* tchunk;       // per tensor: chunks [x, y) (empty: none on this rank)
  float2* partial;          // per chunk (sum p^2, sum u^2)
  int* ovf;                 // per window w: overflow chunk ids at [wchunk[w].x, ...)
  // counters: [0, nwin) queue heads, [nwin, 2 nwin) overflow counts,
  // [2 nwin, 3 nwin) overflow claims, [3 nwin, 4 nwin + 3) arrivals,
  // [4 nwin + 3, 4 nwin + 3 + T) per-tensor finished chunks, then exited
  int* cnt;
  float* trust;             // per tensor (what sp_round_read(SP_BUF_TRUST) returns)
  float* step_scale;        // per tensor: lr * trust
  int nwin;
  int half;                 // floats per stash half (sharded: one window over both halves)
  int T;
  // sharded mode
  int shard;
  double2* table[SP_MAX_RANKS];  // norm table of rank (rank + 1 + k) % world (self last)
  const double2* my_table;       // this rank's [world][T]
  ParamPush push;
  BarrierArgs bar;               // cross-rank barrier (flags, epoch, err)
  unsigned long long* trace;     // SP_LAMB_TRACE builds: per-CTA globaltimer stamps

  __device__ int* head(int w) const { return cnt + w; }
  __device__ int* ovf_n(int w) const { return cnt + nwin + w; }
  __device__ int* ovf_claim(int w) const { return cnt + 2 * nwin + w; }
  __device__ int* arrive(int k) const { return cnt + 3 * nwin + k; }
  __device__ int* done(int t) const { return cnt + 4 * nwin + 3 + t; }
  __device__ int* exited() const { return cnt + 4 * nwin + 3 + T; }
  __device__ int ncounters() const { return 4 * nwin + 4 + T; }
};

#ifdef SP_LAMB_TRACE
#define LAMB_STAMP(k)                                                                         \
  do {                                                                                        \
    if (threadIdx.x == 0 && pl.trace) pl.trace[(size_t)blockIdx.x * 64 + (k)] = globaltimer(); \
  } while (0)
#else
#define LAMB_STAMP(k) \
  do {                \
  } while (0)
#endif

__device__ __forceinline__ void grid_arrive(int* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(c, 1);
  }
}

__device__ __forceinline__ void grid_wait(const int* c, int target) {
  if (threadIdx.x == 0)
    while (ld_acquire_gpu(reinterpret_cast<const unsigned*>(c)) < (unsigned)target) __nanosleep(32);
  __syncthreads();
}

__device__ __forceinline__ float trust_of(double x, double y) {
  const double r1 = sqrt(x), r2 = sqrt(y);
  return (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
}

// --------------------------------------------------------------- pass 1
template <int W, bool FP>
__device__ __forceinline__ void p1_vec(const LambArgs& a, const LambScalars& s, int64_t i, float4 g,
                                       float4 p, float4 m, float4 v, float* st, uint64_t mv_pol,
                                       float& pp, float& uu) {
  float4 u;
  lamb_moments(a, s, g.x, p.x, m.x, v.x, u.x);
  lamb_moments(a, s, g.y, p.y, m.y, v.y, u.y);
  lamb_moments(a, s, g.z, p.z, m.z, v.z, u.z);
  lamb_moments(a, s, g.w, p.w, m.w, v.w, u.w);
  // m', v' are re-read in pass 2 only for chunks that are not stashed
  st_hint_f4(a.m + i, m, mv_pol);
  st_hint_f4(a.v + i, v, mv_pol);
  if (st) *reinterpret_cast<float4*>(st) = u;
  pp = __fmaf_rn(p.x, p.x, pp); pp = __fmaf_rn(p.y, p.y, pp);
  pp = __fmaf_rn(p.z, p.z, pp); pp = __fmaf_rn(p.w, p.w, pp);
  uu = __fmaf_rn(u.x, u.x, uu); uu = __fmaf_rn(u.y, u.y, uu);
  uu = __fmaf_rn(u.z, u.z, uu); uu = __fmaf_rn(u.w, u.w, uu);
}

// Thread t handles body vectors t, t + kLambThreads, ... and, for the
// unaligned edges, head element t (t < head) or tail element t - 32
// (32 <= t < 32 + tail). Pass 2 uses the same mapping, so each thread reads
// back exactly the stash words it wrote. st: the chunk's stash (indexed by
// element - c.start), or nullptr.
template <int W, bool FP>
__device__ __forceinline__ void p1_chunk(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                         float* st, float& pp, float& uu) {
  const ChunkSplit sp = split_chunk(c.start, c.len);
  const int t = threadIdx.x;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = sp.start + sp.head + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float g = load_grad1<W, FP>(a, si);
    const float p = a.p[si];
    float m = a.m[si], v = a.v[si], u;
    lamb_moments(a, s, g, p, m, v, u);
    a.m[si] = m;
    a.v[si] = v;
    if (st) st[si - c.start] = u;
    pp = __fmaf_rn(p, p, pp);
    uu = __fmaf_rn(u, u, uu);
  }
  const int64_t b0 = sp.start + sp.head;
  const uint64_t p_pol = policy_evict_last();  // re-read by pass 2
  const uint64_t mv_pol = st ? policy_evict_first() : p_pol;
  int k = t;
  // kLambVec vectors per thread: every load of the group issued before use
  for (; k + (kLambVec - 1) * kLambThreads < sp.nbody4; k += kLambVec * kLambThreads) {
    GradRaw g[kLambVec];
    float4 p[kLambVec], m[kLambVec], v[kLambVec];
#pragma unroll
    for (int j = 0; j < kLambVec; ++j) g[j] = grad_load<W, FP>(a, b0 + 4 * (int64_t)(k + j * kLambThreads));
#pragma unroll
    for (int j = 0; j < kLambVec; ++j) p[j] = ld_hint_f4(a.p + b0 + 4 * (int64_t)(k + j * kLambThreads), p_pol);
#pragma unroll
    for (int j = 0; j < kLambVec; ++j) m[j] = ld_hint_f4(a.m + b0 + 4 * (int64_t)(k + j * kLambThreads), mv_pol);
#pragma unroll
    for (int j = 0; j < kLambVec; ++j) v[j] = ld_hint_f4(a.v + b0 + 4 * (int64_t)(k + j * kLambThreads), mv_pol);
#pragma unroll
    for (int j = 0; j < kLambVec; ++j) {
      const int64_t i = b0 + 4 * (int64_t)(k + j * kLambThreads);
      p1_vec<W, FP>(a, s, i, grad_finish<W, FP>(a, i, g[j]), p[j], m[j], v[j],
                    st ? st + (i - c.start) : nullptr, mv_pol, pp, uu);
    }
  }
  for (; k < sp.nbody4; k += kLambThreads) {
    const int64_t i = b0 + 4 * (int64_t)k;
    const GradRaw g = grad_load<W, FP>(a, i);
    const float4 p = ld_hint_f4(a.p + i, p_pol);
    const float4 m = ld_hint_f4(a.m + i, mv_pol), v = ld_hint_f4(a.v + i, mv_pol);
    p1_vec<W, FP>(a, s, i, grad_finish<W, FP>(a, i, g), p, m, v, st ? st + (i - c.start) : nullptr, mv_pol, pp, uu);
  }
}

struct LambShared {
  float red_p[2][kLambThreads / 32], red_u[2][kLambThreads / 32];  // by chunk parity
  int2 list[2][kStashList];  // per stash half: (chunk, stash offset) of the stashed chunks
  int nlist[2];
  Chunk desc[2];  // descriptors of this and the next chunk (by parity)
  int idx[2];     // their indices in the window
  int k;
  float neg;
  int t_neg;
  unsigned long long epoch;
};

// Tensor t's last chunk partial is published: warp 0 sums the tensor's
// chunk partials in fp64 (lanes strided in chunk order, then an xor tree;
// every lane ends with the same bits) and publishes lr * trust (replicated)
// or this rank's pair into every rank's norm table (sharded).
__device__ __forceinline__ void finish_tensor(const LambPlan& pl, const LambScalars& s, int t) {
  const int lane = threadIdx.x & 31;
  __threadfence();  // acquire: the other CTAs' partials precede their counts
  const int2 r = pl.tchunk[t];
  double x = 0.0, y = 0.0;
  for (int q = r.x + lane; q < r.y; q += 32) {
    const float2 v = __ldcg(pl.partial + q);
    x += (double)v.x;
    y += (double)v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
  if (pl.shard) {
    if (lane < pl.push.ndst) {
      pl.table[lane][(size_t)pl.bar.rank * pl.T + t] = make_double2(x, y);
      __threadfence_system();
    }
  } else if (lane == 0) {
    const float tr = trust_of(x, y);
    pl.trust[t] = tr;
    pl.step_scale[t] = __fmul_rn(s.lr, tr);
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Pass 1 of window w: claim chunks from the window's queue until it is
// empty. Per chunk: the moments, u into this CTA's stash half while it has
// room (else the chunk goes to the window's overflow list) and the chunk
// partial. One CTA barrier per chunk, and nothing on a chunk's critical
// path waits for a memory round trip: thread 0 claims two chunks ahead and
// copies the next chunk's descriptor into shared memory (cp.async) while
// this chunk runs, and the count of finished chunks of a chunk's tensor
// (whose last finisher completes the tensor's norms, finish_tensor) is
// examined one chunk later.
template <int W, bool FP>
__device__ void pass1(const LambArgs& a, const LambScalars& s, const LambPlan& pl, int w, int h,
                      float* stash, int cap, LambShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int2 wr = pl.wchunk[w];
  const int nw = wr.y - wr.x;
  int used = 0, nlist = 0;  // this half's stash use: the same values in every thread
  int c1 = 0;               // thread 0: index of the next chunk (claimed one chunk ago)
  int pend_t = -1, pend_old = 0, pend_n = 0;  // thread 0: the previous chunk's tensor count
  if (tid == 0) {
    const int c0 = atomicAdd(pl.head(w), 1);
    sh.idx[0] = c0;
    if (c0 < nw) sh.desc[0] = pl.chunks[wr.x + c0];
    c1 = atomicAdd(pl.head(w), 1);
  }
  __syncthreads();
  int parity = 0;
  for (;;) {
    const int item = sh.idx[parity];
    if (item >= nw) break;
    const Chunk c = sh.desc[parity];
    if (tid == 0) {
      if (c1 < nw) {  // the next chunk's descriptor, in flight while this chunk runs
        cp_async16(&sh.desc[parity ^ 1], pl.chunks + wr.x + c1);
        cp_async16(reinterpret_cast<char*>(&sh.desc[parity ^ 1]) + 16,
                   reinterpret_cast<const char*>(pl.chunks + wr.x + c1) + 16);
      }
    }
    const int c2 = tid == 0 ? atomicAdd(pl.head(w), 1) : 0;  // claim after next
    const int ci = wr.x + item;
    const int off = used + (int)((((c.start - used) % 4) + 4) % 4);  // off = start (mod 4)
    const bool stashed = off + c.len <= cap && nlist < kStashList;
    float pp = 0.0f, uu = 0.0f;
    p1_chunk<W, FP>(a, s, c, stashed ? stash + off : nullptr, pp, uu);
    pp = warp_sum(pp);
    uu = warp_sum(uu);
    if (lane == 0) {
      sh.red_p[parity][wid] = pp;
      sh.red_u[parity][wid] = uu;
    }
    if (tid == 0) {
      cp_async_wait_all();
      sh.idx[parity ^ 1] = c1;
      c1 = c2;
    }
    __syncthreads();
    int last_t = -1;
    if (tid == 0) {
      float x = 0.0f, y = 0.0f;
#pragma unroll
      for (int q = 0; q < kLambThreads / 32; ++q) {
        x += sh.red_p[parity][q];
        y += sh.red_u[parity][q];
      }
      pl.partial[ci] = make_float2(x, y);
      if (stashed) sh.list[h][nlist] = make_int2(ci, off);
      else pl.ovf[wr.x + atomicAdd(pl.ovf_n(w), 1)] = ci;
      if (pend_t >= 0 && pend_old == pend_n - 1) last_t = pend_t;
      __threadfence();  // release: the partial precedes the count
      pend_old = atomicAdd(pl.done(c.tensor), 1);
      pend_t = c.tensor;
      pend_n = c.tchunks;
    }
    if (stashed) {
      used = off + c.len;
      ++nlist;
    }
    if (wid == 0) {
      last_t = __shfl_sync(0xffffffffu, last_t, 0);
      if (last_t >= 0) finish_tensor(pl, s, last_t);
    }
    parity ^= 1;
  }
  int last_t = -1;
  if (tid == 0) {
    if (pend_t >= 0 && pend_old == pend_n - 1) last_t = pend_t;
    sh.nlist[h] = nlist;
  }
  if (wid == 0) {
    last_t = __shfl_sync(0xffffffffu, last_t, 0);
    if (last_t >= 0) finish_tensor(pl, s, last_t);
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

__device__ __forceinline__ void p2_store(const LambArgs& a, const ParamPush* push, int64_t i, float4 q,
                                         uint64_t pol) {
  if (push) {
    const int4 o = make_int4(__float_as_int(q.x), __float_as_int(q.y), __float_as_int(q.z),
                             __float_as_int(q.w));
    for (int j = 0; j < push->ndst; ++j) st_v4(push->dst[j] + i, o);
  } else {
    st_hint_f4(a.p + i, q, pol);
  }
}

// p' = p - (lr * trust) * u, u from the stash or recomputed (bit-identical:
// lamb_dir is pass 1's u expression on the stored m', v'). Replicated: p'
// overwrites p. Sharded: p' goes to every rank's copy, the local one last.
__device__ __forceinline__ void p2_chunk(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                         const float* st, float neg, const ParamPush* push) {
  const ChunkSplit sp = split_chunk(c.start, c.len);
  const int t = threadIdx.x;
  const uint64_t drop = policy_evict_first();
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = sp.start + sp.head + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float p = a.p[si];
    const float u = st ? st[si - c.start] : lamb_dir(a, s, p, a.m[si], a.v[si]);
    const float q = __fmaf_rn(neg, u, p);
    if (push)
      for (int k = 0; k < push->ndst; ++k) push->dst[k][si] = q;
    else
      a.p[si] = q;
  }
  const int64_t b0 = sp.start + sp.head;
  int k = t;
  for (; k + kLambThreads < sp.nbody4; k += 2 * kLambThreads) {
    const int64_t i0 = b0 + 4 * (int64_t)k, i1 = i0 + 4 * (int64_t)kLambThreads;
    const float4 p0 = ld_hint_f4(a.p + i0, drop), p1 = ld_hint_f4(a.p + i1, drop);
    float4 u0, u1;
    if (st) {
      u0 = *reinterpret_cast<const float4*>(st + (i0 - c.start));
      u1 = *reinterpret_cast<const float4*>(st + (i1 - c.start));
    } else {
      const float4 m0 = ld_hint_f4(a.m + i0, drop), m1 = ld_hint_f4(a.m + i1, drop);
      const float4 v0 = ld_hint_f4(a.v + i0, drop), v1 = ld_hint_f4(a.v + i1, drop);
      u0 = dir4(a, s, p0, m0, v0);
      u1 = dir4(a, s, p1, m1, v1);
    }
    p2_store(a, push, i0, p2_vec(neg, p0, u0), drop);
    p2_store(a, push, i1, p2_vec(neg, p1, u1), drop);
  }
  if (k < sp.nbody4) {
    const int64_t i = b0 + 4 * (int64_t)k;
    const float4 p = ld_hint_f4(a.p + i, drop);
    const float4 u = st ? *reinterpret_cast<const float4*>(st + (i - c.start))
                        : dir4(a, s, p, ld_hint_f4(a.m + i, drop), ld_hint_f4(a.v + i, drop));
    p2_store(a, push, i, p2_vec(neg, p, u), drop);
  }
}

// -lr * trust of tensor t for pass 2 (uniform; cached in sh.neg).
__device__ __forceinline__ float neg_scale(const LambPlan& pl, const LambScalars& s, int t,
                                           LambShared& sh) {
  if (t != sh.t_neg) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (pl.shard) {
        double x = 0.0, y = 0.0;
        for (int k = 0; k < pl.bar.world; ++k) {
          const double2 q = __ldcg(pl.my_table + (size_t)k * pl.T + t);
          x += q.x;
          y += q.y;
        }
        sh.neg = -__fmul_rn(s.lr, trust_of(x, y));
      } else {
        sh.neg = -__ldcg(pl.step_scale + t);
      }
      sh.t_neg = t;
    }
    __syncthreads();
  }
  return sh.neg;
}

// Pass 2 of window w: this CTA's stashed chunks, then overflow chunks
// claimed from the window's list (complete: every CTA has passed pass 1).
__device__ void pass2(const LambArgs& a, const LambScalars& s, const LambPlan& pl, int w, int h,
                      const float* stash, LambShared& sh) {
  const ParamPush* push = pl.shard ? &pl.push : nullptr;
  const int n = sh.nlist[h];
  for (int k = 0; k < n; ++k) {
    const int2 e = sh.list[h][k];
    const Chunk c = pl.chunks[e.x];
    p2_chunk(a, s, c, stash + e.y, neg_scale(pl, s, c.tensor, sh), push);
  }
  const int2 wr = pl.wchunk[w];
  const int novf = __ldcg(pl.ovf_n(w));
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) sh.k = atomicAdd(pl.ovf_claim(w), 1);
    __syncthreads();
    const int k = sh.k;
    if (k >= novf) break;
    const Chunk c = pl.chunks[__ldcg(pl.ovf + wr.x + k)];
    p2_chunk(a, s, c, nullptr, neg_scale(pl, s, c.tensor, sh), push);
  }
  __syncthreads();  // the next pass 1 reuses this stash half and list
}

// --------------------------------------------------------------- kernel
template <int W, bool FP>
__global__ void __launch_bounds__(kLambThreads, kLambCtasPerSm) k_lamb(LambArgs a, LambPlan pl) {
  extern __shared__ __align__(16) float stash[];
  __shared__ LambShared sh;
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) sh.t_neg = -1;
  LAMB_STAMP(0);
  if (!pl.shard) {
    for (int w = 0; w <= pl.nwin; ++w) {
      if (w < pl.nwin) {
        pass1<W, FP>(a, s, pl, w, w & 1, stash + (w & 1) * pl.half, pl.half, sh);
        LAMB_STAMP(1 + 3 * w);
        grid_arrive(pl.arrive(w));
      }
      if (w >= 1) {
        const int q = w - 1;
        grid_wait(pl.arrive(q), G);
        LAMB_STAMP(2 + 3 * q);
        pass2(a, s, pl, q, q & 1, stash + (q & 1) * pl.half, sh);
        LAMB_STAMP(3 + 3 * q);
      }
    }
  } else {
    // tensors with no chunk on this rank contribute a zero pair
    for (int t = b; t < pl.T; t += G) {
      const int2 r = pl.tchunk[t];
      if (r.y <= r.x && tid < pl.push.ndst) {
        pl.table[tid][(size_t)pl.bar.rank * pl.T + t] = make_double2(0.0, 0.0);
        __threadfence_system();
      }
    }
    pass1<W, FP>(a, s, pl, 0, 0, stash, 2 * pl.half, sh);
    LAMB_STAMP(1);
    grid_arrive(pl.arrive(0));
    if (b == 0) {  // cross-rank barrier (k_barrier's protocol), then release the grid
      grid_wait(pl.arrive(0), G);
      if (tid == 0) {
        sh.epoch = *pl.bar.epoch + 1;
        *pl.bar.epoch = sh.epoch;
      }
      __syncthreads();
      const unsigned long long epoch = sh.epoch;
      if (tid < pl.bar.world) {
        __threadfence_system();
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
      grid_arrive(pl.arrive(1));
    }
    grid_wait(pl.arrive(1), 1);
    LAMB_STAMP(2);
    for (int t = b; t < pl.T; t += G) {  // trust of every tensor, rank order
      if (tid == 0) {
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
    }
    pass2(a, s, pl, 0, 0, stash, sh);
    LAMB_STAMP(3);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(pl.exited(), 1) == G - 1) {  // last CTA out resets every counter
      const int nc = pl.ncounters();
      for (int k = 0; k < nc; ++k) pl.cnt[k] = 0;
      __threadfence();
    }
  }
}

}  // namespace sp
