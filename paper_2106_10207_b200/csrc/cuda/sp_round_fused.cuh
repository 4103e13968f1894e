// sp_round_fused.cuh — the whole averaging round as ONE persistent kernel per
// rank: pack + scatter (NVLink), owner reduce + push (NVLink), LAMB pass 1,
// per-tensor trust, LAMB pass 2. Work items flow through an in-order queue:
//
//   S(cell, owner)  pack this rank's local peers' slice of `cell` that
//                   `owner` owns, store it into owner's inbox (posted NVLink
//                   writes), then add 1 to owner's arrived[cell];
//   R(cell)         wait arrived[cell] == world (every source delivered),
//                   average this rank's slice from local HBM, push it into
//                   every rank's avg, then add 1 to each rank's ready[cell];
//   L1(chunk)       wait ready[cell(chunk)] == #owners of the cell, LAMB
//                   moments + norm partials; the chunk that completes a tensor
//                   computes its trust ratio;
//   L2(chunk)       wait the tensor's trust, LAMB update.
//
// Cells are the fixed grid of max(kLambChunk, q8 block) elements. S items of
// all ranks visit owners in rotated order one cell "column" at a time, so
// each owner's cells complete early and in order: reduce and LAMB pass 1
// start while the scatter is still running, and the NVLink exchange overlaps
// the HBM-bound LAMB work. Counters grow by a per-launch epoch (no resets,
// CUDA-graph replay safe). There are no grid barriers and no barrier
// kernels: the data-flow counters also order consecutive rounds (a rank only
// scatters round t+1 after its round-t LAMB consumed every owner's push).
//
// Deadlock freedom: each rank's queue is stage-sorted (S < R < L1 < L2) and
// items are taken in order; an item only waits on items of earlier stages
// (here or on other GPUs, whose kernels run concurrently), so the
// lowest-stage unfinished item anywhere can always proceed.
#pragma once

#include "sp_kernels.cuh"

namespace sp {

enum : unsigned { kStS = 0u, kStR = 1u, kStL1 = 2u, kStL2 = 3u };

__host__ __device__ inline unsigned make_item(unsigned stage, unsigned owner, unsigned idx) {
  return (stage << 30) | (owner << 27) | idx;
}

struct RoundFused {
  const unsigned* items;
  int nitems;
  int* work;
  int* exited;
  unsigned* epoch;   // rounds completed by this rank's kernel
  int* err;          // host-mapped: a peer wait timed out
  unsigned long long timeout_ns;
  int64_t n;
  int64_t npad;
  int cell;
  int world, rank, L;
  int64_t rank_lo[SP_MAX_RANKS + 1];
  const float* src[SP_MAX_LOCAL];     // local peers' fp32 grads (nullptr: skip)
  char* inbox[SP_MAX_RANKS];          // rank k's inbox slot 0 (mapped)
  size_t slot_bytes;
  int npeers;                         // contributing peers, peer order
  int peer[SP_MAX_PEERS];             // their global index (= inbox slot)
  float w[SP_MAX_PEERS];              // normalized weights
  char* avg[SP_MAX_RANKS];            // push order: rank (rank+1+k) % world
  unsigned* ready_of[SP_MAX_RANKS];   // same order as avg: that rank's ready[]
  unsigned* arrived[SP_MAX_RANKS];    // rank k's arrived[] (indexed by rank)
  unsigned* my_ready;                 // this rank's ready[]
  const unsigned char* cell_owners;   // per cell: number of owning ranks
};

__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int4 ld_cg_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Spin (thread 0) until *p reaches target (wraparound-safe), bounded by the
// timeout; returns false on timeout.
__device__ __forceinline__ bool wait_counter(const unsigned* p, unsigned target,
                                             unsigned long long timeout_ns) {
  if ((int)(ld_acquire_sys_u32(p) - target) >= 0) return true;
  const unsigned long long t0 = globaltimer();
  while ((int)(ld_acquire_sys_u32(p) - target) < 0) {
    __nanosleep(100);
    if (globaltimer() - t0 > timeout_ns) return false;
  }
  return true;
}

// ------------------------------------------------------------- S: scatter
template <int W>
__device__ __forceinline__ void fused_scatter(const RoundFused& f, int64_t s, int64_t e, int owner,
                                              float* red) {
  const int tid = threadIdx.x;
  for (int l = 0; l < f.L; ++l) {
    const float* __restrict__ src = f.src[l];
    if (src == nullptr) continue;
    char* slot = f.inbox[owner] + (size_t)(f.rank * f.L + l) * f.slot_bytes;
    if constexpr (W == SP_WIRE_FP32) {
      const int64_t v0 = s / 4, v1 = (e + 3) / 4, nfull = f.n / 4;
      for (int64_t v = v0 + tid; v < v1; v += blockDim.x) {
        float4 x;
        if (v < nfull) {
          x = __ldg(reinterpret_cast<const float4*>(src) + v);
        } else {
          const int64_t q = v * 4;
          x.x = q + 0 < f.n ? src[q + 0] : 0.0f;
          x.y = q + 1 < f.n ? src[q + 1] : 0.0f;
          x.z = q + 2 < f.n ? src[q + 2] : 0.0f;
          x.w = q + 3 < f.n ? src[q + 3] : 0.0f;
        }
        st_v4(slot + v * 16, make_int4(__float_as_int(x.x), __float_as_int(x.y),
                                       __float_as_int(x.z), __float_as_int(x.w)));
      }
    } else if constexpr (W == SP_WIRE_FP16) {
      const int64_t v0 = s / 8, v1 = (e + 7) / 8, nfull = f.n / 8;
      for (int64_t v = v0 + tid; v < v1; v += blockDim.x) {
        float x[8];
        if (v < nfull) {
          const float4 a0 = __ldg(reinterpret_cast<const float4*>(src) + 2 * v);
          const float4 a1 = __ldg(reinterpret_cast<const float4*>(src) + 2 * v + 1);
          x[0] = a0.x; x[1] = a0.y; x[2] = a0.z; x[3] = a0.w;
          x[4] = a1.x; x[5] = a1.y; x[6] = a1.z; x[7] = a1.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = v * 8 + j < f.n ? src[v * 8 + j] : 0.0f;
        }
        int4 o;
        o.x = (int)pack_half2(x[0], x[1]);
        o.y = (int)pack_half2(x[2], x[3]);
        o.z = (int)pack_half2(x[4], x[5]);
        o.w = (int)pack_half2(x[6], x[7]);
        st_v4(slot + v * 16, o);
      }
    } else {  // q8, block 4096 = 256 threads x 16
      float* scales = reinterpret_cast<float*>(slot + f.npad);
      const int64_t b0 = s / 4096, b1 = (e + 4095) / 4096;
      for (int64_t b = b0; b < b1; ++b) {
        const int64_t e0 = b * 4096 + tid * 16;
        float x[16];
        if (e0 + 16 <= f.n) {
          const float4* s4 = reinterpret_cast<const float4*>(src + e0);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 t = __ldg(s4 + k);
            x[4 * k] = t.x; x[4 * k + 1] = t.y; x[4 * k + 2] = t.z; x[4 * k + 3] = t.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) x[j] = e0 + j < f.n ? src[e0 + j] : 0.0f;
        }
        float amax = 0.0f;
#pragma unroll
        for (int j = 0; j < 16; ++j) amax = fmaxf(amax, fabsf(x[j]));
        amax = block_max(amax, red);
        const float inv = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
        uint32_t wq[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t packed = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            packed |= (uint32_t)(q8_code(x[4 * k + j], inv) & 0xff) << (8 * j);
          wq[k] = packed;
        }
        st_v4(slot + e0, make_int4((int)wq[0], (int)wq[1], (int)wq[2], (int)wq[3]));
        if (tid == 0) scales[b] = __fdiv_rn(amax, 127.0f);
      }
    }
  }
}

// -------------------------------------------------------------- R: reduce
template <int W>
__device__ __forceinline__ void fused_reduce(const RoundFused& f, int64_t s, int64_t e, float* red,
                                             float* sc) {
  const int tid = threadIdx.x;
  const char* base = f.inbox[f.rank];
  if constexpr (W == SP_WIRE_FP32 || W == SP_WIRE_FP16) {
    constexpr int VEC = W == SP_WIRE_FP32 ? 4 : 8;
    const int64_t v0 = s / VEC, v1 = (e + VEC - 1) / VEC;
    for (int64_t v = v0 + tid; v < v1; v += blockDim.x) {
      const size_t off = (size_t)v * 16;
      float acc[8];
      {
        const int4 r0 = ld_cg_v4(base + (size_t)f.peer[0] * f.slot_bytes + off);
        if constexpr (W == SP_WIRE_FP16) {
          mul_half8(acc, f.w[0], r0);
        } else {
          acc[0] = __fmul_rn(f.w[0], __int_as_float(r0.x));
          acc[1] = __fmul_rn(f.w[0], __int_as_float(r0.y));
          acc[2] = __fmul_rn(f.w[0], __int_as_float(r0.z));
          acc[3] = __fmul_rn(f.w[0], __int_as_float(r0.w));
        }
      }
      int g = 1;
      for (; g + 4 <= f.npeers; g += 4) {
        int4 r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = ld_cg_v4(base + (size_t)f.peer[g + k] * f.slot_bytes + off);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if constexpr (W == SP_WIRE_FP16) {
            fma_half8(acc, f.w[g + k], r[k]);
          } else {
            acc[0] = __fmaf_rn(f.w[g + k], __int_as_float(r[k].x), acc[0]);
            acc[1] = __fmaf_rn(f.w[g + k], __int_as_float(r[k].y), acc[1]);
            acc[2] = __fmaf_rn(f.w[g + k], __int_as_float(r[k].z), acc[2]);
            acc[3] = __fmaf_rn(f.w[g + k], __int_as_float(r[k].w), acc[3]);
          }
        }
      }
      for (; g < f.npeers; ++g) {
        const int4 r = ld_cg_v4(base + (size_t)f.peer[g] * f.slot_bytes + off);
        if constexpr (W == SP_WIRE_FP16) {
          fma_half8(acc, f.w[g], r);
        } else {
          acc[0] = __fmaf_rn(f.w[g], __int_as_float(r.x), acc[0]);
          acc[1] = __fmaf_rn(f.w[g], __int_as_float(r.y), acc[1]);
          acc[2] = __fmaf_rn(f.w[g], __int_as_float(r.z), acc[2]);
          acc[3] = __fmaf_rn(f.w[g], __int_as_float(r.w), acc[3]);
        }
      }
      int4 o;
      if constexpr (W == SP_WIRE_FP16) {
        o.x = (int)pack_half2(acc[0], acc[1]);
        o.y = (int)pack_half2(acc[2], acc[3]);
        o.z = (int)pack_half2(acc[4], acc[5]);
        o.w = (int)pack_half2(acc[6], acc[7]);
      } else {
        o = make_int4(__float_as_int(acc[0]), __float_as_int(acc[1]), __float_as_int(acc[2]),
                      __float_as_int(acc[3]));
      }
      for (int k = 0; k < f.world; ++k) st_v4(f.avg[k] + off, o);
    }
  } else {  // q8, block 4096
    const int64_t b0 = s / 4096, b1 = (e + 4095) / 4096;
    for (int64_t b = b0; b < b1; ++b) {
      __syncthreads();
      if (tid < f.npeers)
        sc[tid] = __ldcg(reinterpret_cast<const float*>(base + (size_t)f.peer[tid] * f.slot_bytes + f.npad) + b);
      __syncthreads();
      const size_t e0 = (size_t)b * 4096 + tid * 16;
      if (f.npeers == 1) {  // one contributor: codes and scale forwarded unchanged
        const int4 o = ld_cg_v4(base + (size_t)f.peer[0] * f.slot_bytes + e0);
        for (int k = 0; k < f.world; ++k) {
          st_v4(f.avg[k] + e0, o);
          if (tid == 0) reinterpret_cast<float*>(f.avg[k] + f.npad)[b] = sc[0];
        }
        continue;
      }
      float acc[16];
      mul_q8x16(acc, f.w[0], sc[0], ld_cg_v4(base + (size_t)f.peer[0] * f.slot_bytes + e0));
      int g = 1;
      for (; g + 4 <= f.npeers; g += 4) {
        int4 r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = ld_cg_v4(base + (size_t)f.peer[g + k] * f.slot_bytes + e0);
#pragma unroll
        for (int k = 0; k < 4; ++k) fma_q8x16(acc, f.w[g + k], sc[g + k], r[k]);
      }
      for (; g < f.npeers; ++g)
        fma_q8x16(acc, f.w[g], sc[g], ld_cg_v4(base + (size_t)f.peer[g] * f.slot_bytes + e0));
      float amax = 0.0f;
#pragma unroll
      for (int j = 0; j < 16; ++j) amax = fmaxf(amax, fabsf(acc[j]));
      amax = block_max(amax, red);
      const float inv = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
      uint32_t wq[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t packed = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) packed |= (uint32_t)(q8_code(acc[4 * k + j], inv) & 0xff) << (8 * j);
        wq[k] = packed;
      }
      const int4 o = make_int4((int)wq[0], (int)wq[1], (int)wq[2], (int)wq[3]);
      const float scale = __fdiv_rn(amax, 127.0f);
      for (int k = 0; k < f.world; ++k) {
        st_v4(f.avg[k] + e0, o);
        if (tid == 0) reinterpret_cast<float*>(f.avg[k] + f.npad)[b] = scale;
      }
    }
  }
}

#ifndef SP_FUSED_MIN_CTAS
#define SP_FUSED_MIN_CTAS 4
#endif
template <int W>
__global__ void __launch_bounds__(kLambThreads, SP_FUSED_MIN_CTAS) k_round_fused(RoundFused f, LambArgs a, FusedLamb q) {
  __shared__ unsigned s_item, s_epoch;
  __shared__ int s_last;
  __shared__ float s_scale;
  __shared__ float red[32];
  __shared__ float sc[SP_MAX_PEERS];
  __shared__ float red_p[kLambThreads / 32], red_u[kLambThreads / 32];
  __shared__ double dred_p[kLambThreads], dred_u[kLambThreads];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const LambScalars ls{a.hp[0], a.hp[1], a.hp[2]};
  unsigned next = 0;
  if (tid == 0) {
    s_epoch = *f.epoch + 1u;
    next = (unsigned)atomicAdd(f.work, 1);
  }
  __syncthreads();
  const unsigned epoch = s_epoch;
  for (;;) {
    if (tid == 0) s_item = next;
    __syncthreads();
    const unsigned it = s_item;
    __syncthreads();
    if (it >= (unsigned)f.nitems) break;
    if (tid == 0) next = (unsigned)atomicAdd(f.work, 1);
    const unsigned code = f.items[it];
    const unsigned stage = code >> 30, owner = (code >> 27) & 7u, idx = code & ((1u << 27) - 1u);
    if (stage == kStS) {
      const int64_t c0 = (int64_t)idx * f.cell;
      const int64_t s = max(c0, f.rank_lo[owner]);
      const int64_t e = min(min(c0 + f.cell, f.rank_lo[owner + 1]), f.n);
      fused_scatter<W>(f, s, e, (int)owner, red);
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        red_release_sys(f.arrived[owner] + idx, 1u);
      }
    } else if (stage == kStR) {
      if (tid == 0 &&
          !wait_counter(f.arrived[f.rank] + idx, epoch * (unsigned)f.world, f.timeout_ns))
        atomicExch_system(f.err, 1);
      __syncthreads();
      const int64_t c0 = (int64_t)idx * f.cell;
      const int64_t s = max(c0, f.rank_lo[f.rank]);
      const int64_t e = min(min(c0 + f.cell, f.rank_lo[f.rank + 1]), f.n);
      fused_reduce<W>(f, s, e, red, sc);
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        for (int k = 0; k < f.world; ++k) red_release_sys(f.ready_of[k] + idx, 1u);
      }
    } else if (stage == kStL1) {
      const Chunk c = a.chunks[idx];
      const unsigned cellj = (unsigned)(c.start / f.cell);
      if (tid == 0 &&
          !wait_counter(f.my_ready + cellj, epoch * (unsigned)f.cell_owners[cellj], f.timeout_ns))
        atomicExch_system(f.err, 1);
      __syncthreads();
      float pp = 0.0f, uu = 0.0f;
      lamb_pass1<W>(a, ls, c, pp, uu);
      pp = warp_sum(pp);
      uu = warp_sum(uu);
      if (lane == 0) {
        red_p[wid] = pp;
        red_u[wid] = uu;
      }
      __syncthreads();
      if (tid == 0) {
        float sp_ = 0.0f, su = 0.0f;
#pragma unroll
        for (int w = 0; w < kLambThreads / 32; ++w) {
          sp_ += red_p[w];
          su += red_u[w];
        }
        a.partial[idx] = make_float2(sp_, su);
        __threadfence();
        const int2 r = q.tchunks[c.tensor];
        s_last = atomicAdd(q.done + c.tensor, 1) == r.y - r.x - 1;
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        const int2 r = q.tchunks[c.tensor];
        double dp = 0.0, du = 0.0;
        for (int qq = r.x + tid; qq < r.y; qq += kLambThreads) {
          const float2 v = __ldcg(a.partial + qq);
          dp += (double)v.x;
          du += (double)v.y;
        }
        dred_p[tid] = dp;
        dred_u[tid] = du;
        __syncthreads();
        for (int h = kLambThreads / 2; h > 0; h >>= 1) {
          if (tid < h) {
            dred_p[tid] += dred_p[tid + h];
            dred_u[tid] += dred_u[tid + h];
          }
          __syncthreads();
        }
        if (tid == 0) {
          const double r1 = sqrt(dred_p[0]), r2 = sqrt(dred_u[0]);
          const float tr = (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
          q.trust[c.tensor] = tr;
          const_cast<float*>(a.step_scale)[c.tensor] = __fmul_rn(ls.lr, tr);
          q.done[c.tensor] = 0;
          __threadfence();
          st_release_gpu(q.ready + c.tensor, 1u);
        }
      }
    } else {
      const Chunk c = a.chunks[idx];
      if (tid == 0) {
        while (ld_acquire_gpu(q.ready + c.tensor) == 0u) __nanosleep(64);
        s_scale = __ldcg(a.step_scale + c.tensor);
      }
      __syncthreads();
      lamb_pass2(a, ls, c, -s_scale);
    }
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(f.exited, 1) == (int)gridDim.x - 1) {  // last CTA out
      for (int t = 0; t < q.ntensors; ++t) q.ready[t] = 0u;
      *f.work = 0;
      *f.exited = 0;
      *f.epoch = epoch;
      __threadfence();
    }
  }
}

}  // namespace sp
