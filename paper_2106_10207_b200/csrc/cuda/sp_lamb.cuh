// sp_lamb.cuh — the LAMB step of the round (K3 + K4) as one cooperative
// persistent kernel: 1024 / kLambThreads CTAs per SM, static work split.
//
// LAMB needs every tensor's norms ||p||, ||u|| before any element of it can
// be updated, so each element is touched twice: pass 1 (m' = b1 m + (1-b1) g,
// v' = ..., u = m'^/(sqrt(v'^)+eps) + wd p, norm partials) and pass 2
// (p' = p - lr * trust_t * u). Re-reading p, m', v' in pass 2 costs 12 B per
// element of L2 traffic on top of pass 1's 24 + b, and on B200 the L2 slice
// throughput (~6.3 KB/clk chip-wide, /opt/skills/guides/B300_MICROARCH.md
// "LTS throughput cap") is the binding limit for hits and misses alike: the
// round-1 kernel moved 44 B/element through L2 at 6.35 TB/s.
//
// Here pass 1 keeps u in shared memory (the "stash": the SM's shared memory
// split over its CTAs, ~57 K floats per SM), so pass 2 only re-reads p (4 B,
// L2-resident: pass 1 loads it with an evict_last hint) and writes p':
// 24 + b + 8 B per element.
//
// Replicated mode (every rank steps the whole vector). Tensors are packed
// into windows that fit half the stash (~4.2 M elements on 148 SMs; the
// largest ALBERT-large tensor has 4,194,304). Each window's elements are
// split evenly over the CTAs; a CTA runs
//     pass1(w0) arrive(w0) | pass1(w1) arrive(w1) wait(w0) pass2(w0) |
//     pass1(w2) arrive(w2) wait(w1) pass2(w1) | ... wait(last) pass2(last)
// alternating the two stash halves, so the grid barrier of window w is
// split-phase: its wait comes one window of work after its arrive and is
// normally already satisfied. A tensor larger than a window gets a window
// of its own with as many chunks stashed as fit; pass 2 recomputes u for
// the rest from p, m', v'.
//
// Sharded mode (ZeRO-1 style): one window, this rank's owned
// range, stashed up to the whole buffer. After pass 1 every CTA publishes
// the per-tensor rank sums it is responsible for into slot [rank][t] of
// every rank's norm table (NVLink stores), CTA 0 runs the cross-rank
// barrier, and pass 2 forms trust_t from the world slots in rank order and
// stores p' into every rank's parameter vector.
//
// Norms (deterministic, same bits on every replica): per-thread fp32 fmaf
// chains over a run (consecutive chunks of one tensor in one CTA), warp xor
// tree, warps summed in order -> float2 partial per run; per tensor the runs
// are summed in fp64 by a lane-strided warp xor tree. All grid barriers are
// counters in global memory: the grid is launched cooperatively (all CTAs
// co-resident) and the last CTA out resets the counters (graph-replay safe).
#pragma once

#include "sp_kernels.cuh"

namespace sp {

struct LambPlan {
  const Chunk* chunks;
  const int2* wrange;       // [nwin][grid]: chunks [x, y) of CTA b in window w
  const int2* trun;         // per tensor: runs [x, y)
  float2* partial;          // per run
  int* cnt;                 // [0, nbar): barrier counters, [nbar]: CTAs exited
  int nbar;
  float* trust;             // per tensor (what sp_round_read(SP_BUF_TRUST) returns)
  float* step_scale;        // per tensor: lr * trust
  int nwin;
  int half;                 // floats per stash half
  int T;
  // sharded mode
  int shard;
  double2* table[SP_MAX_RANKS];  // norm table of rank (rank + 1 + k) % world (self last)
  const double2* my_table;       // this rank's [world][T]
  ParamPush push;
  BarrierArgs bar;               // cross-rank barrier (flags, epoch, err)
  unsigned long long* trace;     // SP_LAMB_TRACE builds: per-CTA globaltimer stamps
};

#ifdef SP_LAMB_TRACE
#define LAMB_STAMP(k) \
  do {                                                                                    \
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

// fp64 sums of the run partials [r.x, r.y) of one tensor: lanes take runs
// r.x + lane, r.x + lane + 32, ... then an xor tree (every lane ends with the
// same bits: each pairwise add sees the same two operands in both lanes).
__device__ __forceinline__ double2 run_sum_warp(const float2* partial, int2 r) {
  const int lane = threadIdx.x & 31;
  double x = 0.0, y = 0.0;
  for (int q = r.x + lane; q < r.y; q += 32) {
    const float2 v = __ldcg(partial + q);
    x += (double)v.x;
    y += (double)v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
  return make_double2(x, y);
}

__device__ __forceinline__ float trust_of(double x, double y) {
  const double r1 = sqrt(x), r2 = sqrt(y);
  return (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
}

// --------------------------------------------------------------- pass 1
template <int W>
__device__ __forceinline__ void p1_vec(const LambArgs& a, const LambScalars& s, int64_t i, float4 g,
                                       float4 p, float4 m, float4 v, float* st, bool keep,
                                       float& pp, float& uu) {
  float4 u;
  lamb_moments(a, s, g.x, p.x, m.x, v.x, u.x);
  lamb_moments(a, s, g.y, p.y, m.y, v.y, u.y);
  lamb_moments(a, s, g.z, p.z, m.z, v.z, u.z);
  lamb_moments(a, s, g.w, p.w, m.w, v.w, u.w);
  // m', v' are re-read in pass 2 only for chunks that are not stashed
  const uint64_t pol = keep ? policy_evict_last() : policy_evict_first();
  st_hint_f4(a.m + i, m, pol);
  st_hint_f4(a.v + i, v, pol);
  if (st) *reinterpret_cast<float4*>(st) = u;
  pp = __fmaf_rn(p.x, p.x, pp); pp = __fmaf_rn(p.y, p.y, pp);
  pp = __fmaf_rn(p.z, p.z, pp); pp = __fmaf_rn(p.w, p.w, pp);
  uu = __fmaf_rn(u.x, u.x, uu); uu = __fmaf_rn(u.y, u.y, uu);
  uu = __fmaf_rn(u.z, u.z, uu); uu = __fmaf_rn(u.w, u.w, uu);
}

// Thread t handles body vectors t and t + 1024 and, for the unaligned
// edges, head element t (t < head) or tail element t - 32 (32 <= t < 32 +
// tail). Pass 2 uses the same mapping, so each thread reads back exactly the
// stash words it wrote (no barrier between the passes of a chunk).
template <int W>
__device__ __forceinline__ void p1_chunk(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                         float* stash, float& pp, float& uu) {
  const ChunkSplit sp = split_chunk(c.start, c.len);
  const int t = threadIdx.x;
  float* st = c.stash >= 0 ? stash + c.stash : nullptr;  // indexed by element - c.start
  const bool keep = st == nullptr;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = sp.start + sp.head + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float g = load_grad1<W>(a, si);
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
  const uint64_t mv_pol = keep ? p_pol : policy_evict_first();
  int k = t;
  for (; k + kLambThreads < sp.nbody4; k += 2 * kLambThreads) {
    const int64_t i0 = b0 + 4 * (int64_t)k, i1 = i0 + 4 * (int64_t)kLambThreads;
    const float4 g0 = load_grad4<W>(a, i0), g1 = load_grad4<W>(a, i1);
    const float4 p0 = ld_hint_f4(a.p + i0, p_pol), p1 = ld_hint_f4(a.p + i1, p_pol);
    const float4 m0 = ld_hint_f4(a.m + i0, mv_pol), m1 = ld_hint_f4(a.m + i1, mv_pol);
    const float4 v0 = ld_hint_f4(a.v + i0, mv_pol), v1 = ld_hint_f4(a.v + i1, mv_pol);
    p1_vec<W>(a, s, i0, g0, p0, m0, v0, st ? st + (i0 - c.start) : nullptr, keep, pp, uu);
    p1_vec<W>(a, s, i1, g1, p1, m1, v1, st ? st + (i1 - c.start) : nullptr, keep, pp, uu);
  }
  if (k < sp.nbody4) {
    const int64_t i = b0 + 4 * (int64_t)k;
    const float4 g = load_grad4<W>(a, i);
    const float4 p = ld_hint_f4(a.p + i, p_pol);
    const float4 m = ld_hint_f4(a.m + i, mv_pol), v = ld_hint_f4(a.v + i, mv_pol);
    p1_vec<W>(a, s, i, g, p, m, v, st ? st + (i - c.start) : nullptr, keep, pp, uu);
  }
}

// Block reduction of the thread partials of a finished run -> partial[run].
__device__ __forceinline__ void flush_run(float2* partial, int run, float& pp, float& uu,
                                          float* red_p, float* red_u) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pp = warp_sum(pp);
  uu = warp_sum(uu);
  if (lane == 0) {
    red_p[wid] = pp;
    red_u[wid] = uu;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float x = 0.0f, y = 0.0f;
#pragma unroll
    for (int w = 0; w < kLambThreads / 32; ++w) {
      x += red_p[w];
      y += red_u[w];
    }
    partial[run] = make_float2(x, y);
  }
  __syncthreads();
  pp = 0.0f;
  uu = 0.0f;
}

template <int W>
__device__ __forceinline__ void pass1(const LambArgs& a, const LambScalars& s, const LambPlan& pl,
                                      int2 r, float* stash, float* red_p, float* red_u) {
  float pp = 0.0f, uu = 0.0f;
  for (int ci = r.x; ci < r.y; ++ci) {
    const Chunk c = pl.chunks[ci];
    p1_chunk<W>(a, s, c, stash, pp, uu);
    if (c.last) flush_run(pl.partial, c.run, pp, uu, red_p, red_u);
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

// p' = p - (lr * trust) * u, u from the stash or recomputed (bit-identical:
// lamb_dir is pass 1's u expression on the stored m', v'). Replicated: p'
// overwrites p. Sharded: p' goes to every rank's copy, the local one last.
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

__device__ __forceinline__ void p2_chunk(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                         const float* stash, float neg, const ParamPush* push) {
  const ChunkSplit sp = split_chunk(c.start, c.len);
  const int t = threadIdx.x;
  const float* st = c.stash >= 0 ? stash + c.stash : nullptr;  // indexed by element - c.start
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
  if (st) {  // u from the stash: only p is loaded, keep 4 vectors per thread in flight
    for (; k + 3 * kLambThreads < sp.nbody4; k += 4 * kLambThreads) {
      float4 p[4], u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = ld_hint_f4(a.p + b0 + 4 * (int64_t)(k + j * kLambThreads), drop);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        u[j] = *reinterpret_cast<const float4*>(st + (b0 + 4 * (int64_t)(k + j * kLambThreads) - c.start));
#pragma unroll
      for (int j = 0; j < 4; ++j)
        p2_store(a, push, b0 + 4 * (int64_t)(k + j * kLambThreads), p2_vec(neg, p[j], u[j]), drop);
    }
  }
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

// --------------------------------------------------------------- kernel
template <int W>
__global__ void __launch_bounds__(kLambThreads, kLambCtasPerSm) k_lamb(LambArgs a, LambPlan pl) {
  extern __shared__ __align__(16) float stash[];
  __shared__ float red_p[kLambThreads / 32], red_u[kLambThreads / 32];
  __shared__ float s_neg;
  __shared__ int s_t;
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const int G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) s_t = -1;

  // per-chunk scale of pass 2: -lr * trust of the chunk's tensor, formed by
  // warp 0 when the tensor changes; the CTA holding a tensor's first run also
  // publishes trust / step_scale
  auto scale_for = [&](const Chunk& c) {
    if (c.tensor != s_t) {  // uniform: s_t only changes behind the barrier below
      __syncthreads();
      if (tid < 32) {
        float tr;
        if (pl.shard) {
          double x = 0.0, y = 0.0;
          for (int k = 0; k < pl.bar.world; ++k) {
            const double2 q = __ldcg(pl.my_table + (size_t)k * pl.T + c.tensor);
            x += q.x;
            y += q.y;
          }
          tr = trust_of(x, y);
        } else {
          const double2 q = run_sum_warp(pl.partial, pl.trun[c.tensor]);
          tr = trust_of(q.x, q.y);
        }
        if (tid == 0) {
          s_neg = -__fmul_rn(s.lr, tr);
          s_t = c.tensor;
          if (!pl.shard && c.run == pl.trun[c.tensor].x) {
            pl.trust[c.tensor] = tr;
            pl.step_scale[c.tensor] = __fmul_rn(s.lr, tr);
          }
        }
      }
      __syncthreads();
    }
    return s_neg;
  };

  LAMB_STAMP(0);
  if (!pl.shard) {
    for (int w = 0; w <= pl.nwin; ++w) {
      if (w < pl.nwin) {
        pass1<W>(a, s, pl, pl.wrange[(size_t)w * G + b], stash + (w & 1) * pl.half, red_p, red_u);
        LAMB_STAMP(1 + 3 * w);
        grid_arrive(pl.cnt + w);
      }
      if (w >= 1) {
        const int q = w - 1;
        grid_wait(pl.cnt + q, G);
        LAMB_STAMP(2 + 3 * q);
        const int2 r = pl.wrange[(size_t)q * G + b];
        const float* st = stash + (q & 1) * pl.half;
        for (int ci = r.x; ci < r.y; ++ci) {
          const Chunk c = pl.chunks[ci];
          p2_chunk(a, s, c, st, scale_for(c), nullptr);
        }
        __syncthreads();  // the next pass 1 reuses this stash half
        LAMB_STAMP(3 + 3 * q);
      }
    }
  } else {
    const int2 r = pl.wrange[b];
    pass1<W>(a, s, pl, r, stash, red_p, red_u);
    grid_arrive(pl.cnt + 0);
    grid_wait(pl.cnt + 0, G);
    // this rank's per-tensor sums into slot [rank][t] of every rank's table
    for (int t = b; t < pl.T; t += G) {
      if (tid < 32) {
        const double2 q = run_sum_warp(pl.partial, pl.trun[t]);
        if (tid < pl.push.ndst) {
          pl.table[tid][(size_t)pl.bar.rank * pl.T + t] = q;
          __threadfence_system();
        }
      }
    }
    grid_arrive(pl.cnt + 1);
    if (b == 0) {  // cross-rank barrier (k_barrier's protocol), then release the grid
      grid_wait(pl.cnt + 1, G);
      __shared__ unsigned long long epoch;
      if (tid == 0) {
        epoch = *pl.bar.epoch + 1;
        *pl.bar.epoch = epoch;
      }
      __syncthreads();
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
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(pl.cnt + 2, 1);
      }
    }
    grid_wait(pl.cnt + 2, 1);
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
    for (int ci = r.x; ci < r.y; ++ci) {
      const Chunk c = pl.chunks[ci];
      p2_chunk(a, s, c, stash, scale_for(c), &pl.push);
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(pl.cnt + pl.nbar, 1) == G - 1) {  // last CTA out resets the counters
      for (int k = 0; k <= pl.nbar; ++k) pl.cnt[k] = 0;
      __threadfence();
    }
  }
}

}  // namespace sp
