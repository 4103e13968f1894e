// sp_kernels.cuh — sm_100a kernels of the averaging round.
//
// All kernels are HBM- or NVLink-bound streaming kernels (no tensor cores:
// the round has no contraction). Conventions shared by every kernel:
//   * 128-bit vector loads/stores on 16-byte aligned, zero-padded buffers;
//   * explicit IEEE intrinsics (__fmul_rn, __fmaf_rn, __fdiv_rn, __fsqrt_rn)
//     so no FMA contraction changes a rounding: the CPU oracle
//     (oracle/sp_oracle.c) performs the same operation sequence and the
//     wire codes, averaged parts and LAMB moments are bit-identical;
//   * peers are summed in peer order 0..G-1 (the order groups::run_plan
//     merges classes in, /root/reference/proj/src/groups.cpp:133-144).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sp_round.h"

namespace sp {

// LAMB CTA (sp_lamb.cuh): SP_LAMB_WARPS data warps, each thread one float4
// of a chunk per array, and two control warps (claims, books);
// SP_LAMB_CTAS CTAs per SM; SP_LAMB_STAGES chunks of g, p, m, v staged in
// shared memory by bulk copies (the loads in flight do not hold registers,
// so one CTA of 16 data warps per SM streams at HBM speed); the rest of the
// SM's shared memory is the u stash.
#ifndef SP_LAMB_WARPS
#define SP_LAMB_WARPS 12
#endif
#ifndef SP_LAMB_CTAS
#define SP_LAMB_CTAS 1
#endif
#ifndef SP_LAMB_STAGES
#define SP_LAMB_STAGES 2
#endif
#ifndef SP_LAMB_VEC
#define SP_LAMB_VEC 2
#endif
constexpr int kLambDataWarps = SP_LAMB_WARPS;
constexpr int kLambDataThreads = kLambDataWarps * 32;
constexpr int kLambThreads = kLambDataThreads + 64;
constexpr int kLambCtasPerSm = SP_LAMB_CTAS;
constexpr int kLambStages = SP_LAMB_STAGES;
constexpr int kLambVec = SP_LAMB_VEC;                    // float4 per data thread per array
constexpr int kLambTile = kLambDataThreads * 4 * kLambVec;  // max chunk length
// one stage: g (wire bytes or fp32, plus 16 bytes of slack for an aligned
// superset of a wire range), p, m, v of the pass-1 chunk (an iteration
// without a pass-1 chunk puts pass-2 entries into these four areas instead)
constexpr int kLambArea = kLambTile * 4;  // one fp32 array of a chunk
constexpr int kLambStageG = kLambArea + 16;
constexpr int kLambStageAreas = 4;
constexpr int kLambStageBytes = kLambStageG + 3 * kLambArea;
constexpr int kPad = 16384;         // wire/avg buffers padded to this multiple

struct BarrierArgs {
  unsigned long long* flags[SP_MAX_RANKS];  // flags array of every rank
  unsigned long long* epoch;                // local epoch counter
  int* err;                                 // host-mapped error flag
  int rank, world;
  unsigned long long timeout_ns;
};

// K1 scatters each local peer's packed gradient straight into the inbox of
// the rank that owns each element range (local HBM or a peer GPU over
// NVLink): posted writes only, no pull reads in the exchange. The kernel
// walks a list of ranges (one per owner, possibly one segment of each
// owner's range) in the given order. The host orders them starting with the
// next rank's range and ending with its own, so at any moment the ranks
// write to different owners: all-to-all without incast (4x B200: ~660
// GB/s/dir rotated vs ~400 GB/s when every rank targets the same owner,
// profiles/r01/p2p_bw.txt).
struct PackArgs {
  const float* src[SP_MAX_LOCAL];          // accumulated fp32 grad of local peer l
  void* dst[SP_MAX_LOCAL][SP_MAX_RANKS];   // inbox slot of local peer l on rank k
  int nr;                                  // ranges, in visiting order
  int owner[SP_MAX_RANKS];                 // owner rank of range j
  int64_t lo[SP_MAX_RANKS];                // first unit of range j (vector / q8 block)
  int64_t pref[SP_MAX_RANKS + 1];          // prefix sums of range lengths in units
  int cta0[SP_MAX_RANKS + 1];              // CTAs [cta0[j], cta0[j+1]) work on range j
  int64_t n;                               // valid elements
  int64_t npad;                            // padded elements (multiple of kPad)
  int qblock;                              // q8 block
};

// Ranges are processed concurrently: the CTAs are split across them in
// proportion to their lengths, so a rank streams to every owner at once (the
// all-to-all "spread" pattern, ~666 GB/s/dir on 4x B200) and its local
// range overlaps the NVLink traffic instead of trailing it.
struct RangeSlice {
  int j;          // range
  int64_t first;  // first unit of this CTA
  int64_t stride;
  int64_t end;    // one past the range's last unit (in range-local units)
};

__device__ __forceinline__ RangeSlice cta_slice(const PackArgs& a) {
  int j = 0;
  while (j + 1 < a.nr && (int)blockIdx.x >= a.cta0[j + 1]) ++j;
  RangeSlice s;
  s.j = j;
  const int nct = a.cta0[j + 1] - a.cta0[j];
  s.first = (int64_t)(blockIdx.x - a.cta0[j]) * blockDim.x + threadIdx.x;
  s.stride = (int64_t)nct * blockDim.x;
  s.end = a.pref[j + 1] - a.pref[j];
  return s;
}

struct ReduceArgs {
  const void* src[SP_MAX_PEERS];  // inbox slot of each contributing peer (local)
  float w[SP_MAX_PEERS];          // normalized weight w_g / sum(w), fp32
  void* dst[SP_MAX_RANKS];        // avg buffer of every rank, push order
  int npeers;                     // contributing (nonzero-weight) peers
  int ndst;
  int64_t lo, hi;                 // element range reduced by this launch
  int64_t npad;
  int qblock;
  // device-side weights (accumulation mode): per-peer sample counts published
  // by every rank; the kernel normalizes them exactly like the host would
  const double* dev_w;            // G counts (nullptr: use src/w/npeers)
  const void* all_src[SP_MAX_PEERS];  // inbox slot of every peer
  int G;
  int* err;
};

// Contributing peers of a reduce launch, in peer order. With device weights
// thread 0 computes sum(w) in fp64 in peer order and (float)(w_g / sum), the
// same operations the host normalization uses, so results stay bit-exact.
struct PeerView {
  const void* src[SP_MAX_PEERS];
  float w[SP_MAX_PEERS];
  int np;
};

__device__ __forceinline__ void load_peers(const ReduceArgs& a, PeerView& pv) {
  if (threadIdx.x == 0) {
    if (a.dev_w) {
      double s = 0.0;
      for (int g = 0; g < a.G; ++g) s += a.dev_w[g];
      int np = 0;
      if (s > 0.0) {
        for (int g = 0; g < a.G; ++g) {
          const double w = a.dev_w[g];
          if (w == 0.0) continue;
          pv.src[np] = a.all_src[g];
          pv.w[np] = (float)(w / s);
          ++np;
        }
      } else if (a.err) {
        atomicExch_system(a.err, 2);  // no samples accumulated anywhere
      }
      pv.np = np;
    } else {
      for (int g = 0; g < a.npeers; ++g) {
        pv.src[g] = a.src[g];
        pv.w[g] = a.w[g];
      }
      pv.np = a.npeers;
    }
  }
  __syncthreads();
}

// One LAMB work item: a piece of one tensor, at most kLambTile elements,
// claimed by one CTA in pass 1 (sp_lamb.cuh).
struct alignas(16) Chunk {
  long long start;
  int len;
  int tensor;
  int tchunks;  // chunks of this tensor (in this rank's table)
  int head;     // unaligned leading elements (split_chunk)
  int nbody4;   // 16-byte body vectors
  int tail;     // trailing elements
};

struct LambArgs {
  const void* avg;          // all-gathered averaged gradient, wire format
  const float* avg_scale;   // q8 scales (nullptr otherwise)
  float* p;
  float* m;
  float* v;
  const float* hp;          // device: [lr, 1/(1-b1^t), 1/(1-b2^t)]
  float b1, b2, omb1, omb2, eps, wd;
  int qshift;               // log2(q8 block): scale index = i >> qshift
  // one rank, one peer, fp32/fp16 wire: the pack is fused into pass 1, which
  // reads the fp32 gradient, rounds it to the wire format (the identity
  // average) and also stores the wire values (nullptr: read `avg`)
  const float* g32;
  void* wire_out;
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// L2 eviction-priority policies (createpolicy) and hinted 128-bit accesses.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_hint_f4(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_hint_f4(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p,
                                               unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
               : "=l"(v)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// 8-bit code of x given inv = 127/absmax: rint(x*inv), clamped to +-127.
__device__ __forceinline__ int q8_code(float x, float inv) {
  int q = __float2int_rn(__fmul_rn(x, inv));
  return max(-127, min(127, q));
}

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Block-wide max over blockDim.x threads (multiple of 32, <= 1024).
__device__ __forceinline__ float block_max(float x, float* smem32) {
  x = warp_max(x);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) smem32[wid] = x;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float y = lane < nw ? smem32[lane] : 0.0f;
  y = warp_max(y);
  __syncthreads();
  return y;
}

// 16 values -> 16 packed 8-bit codes, code = clamp(rint(x*inv), +-127).
// Fast path: y = x*inv is rounded to an integer by adding 1.5*2^23 (exact
// RNE for |y| < 2^22) and the code is the low byte of the sum; every caller
// has |x| <= amax and inv = 127/amax, so |y| <= 127*(1+2^-23) < 127.5 and
// the clamp is implied. A non-finite inv (amax < 127/FLT_MAX) takes the
// converting path; the block-uniform branch costs nothing otherwise.
__device__ __forceinline__ int4 quant16(const float* x, float inv) {
  uint32_t w[4];
  if (inv <= 3.0e38f) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = __float_as_uint(__fadd_rn(__fmul_rn(x[4 * k + j], inv), 12582912.0f));
      w[k] = __byte_perm(__byte_perm(t[0], t[1], 0x0040), __byte_perm(t[2], t[3], 0x0040), 0x5410);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t packed = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) packed |= (uint32_t)(q8_code(x[4 * k + j], inv) & 0xff) << (8 * j);
      w[k] = packed;
    }
  }
  return make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
}

// 4 int8 codes (one word) -> 4 exact floats: each byte, biased by 0x80, is
// placed in the mantissa of 2^23 (one PRMT) and 2^23 + 128 is subtracted.
__device__ __forceinline__ float4 dequant4(uint32_t u) {
  const uint32_t b = u ^ 0x80808080u;
  return make_float4(__fsub_rn(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7440)), 8388736.0f),
                     __fsub_rn(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7441)), 8388736.0f),
                     __fsub_rn(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7442)), 8388736.0f),
                     __fsub_rn(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7443)), 8388736.0f));
}

__device__ __forceinline__ float absmax16(const float* x) {
  float m = 0.0f;
#pragma unroll
  for (int j = 0; j < 16; ++j) m = fmaxf(m, fabsf(x[j]));
  return m;
}

// --------------------------------------------------------------- synthetic

__global__ void k_fill_synthetic(float* __restrict__ out, int64_t n,
                                 unsigned long long seed, int peer,
                                 float scale, int64_t every, float mult) {
  const unsigned long long key = seed ^ ((unsigned long long)peer << 40);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long u = splitmix64(key ^ (unsigned long long)i) >> 40;
    float x = __fmul_rn(__fmul_rn((float)(long long)u - 8388608.0f,
                                  1.0f / 8388608.0f),
                        scale);
    if (every > 0 && i % every == 0) x = __fmul_rn(x, mult);
    out[i] = x;
  }
}

// ----------------------------------------------------------------- barrier
// Cross-rank barrier over NVLink between the exchange kernels: rank r stores
// the new epoch into flags_k[r] of every rank k (system-scope release), then
// waits until its own flags[k] >= epoch for all k (acquire). One warp.
// (Folding this wait/signal into the producer/consumer kernels was measured
// slower at N=4: every CTA polls the flags and pays a fence.)

__global__ void k_barrier(BarrierArgs a) {
  __shared__ unsigned long long epoch;
  if (threadIdx.x == 0) {
    epoch = *a.epoch + 1;
    *a.epoch = epoch;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < a.world) {
    __threadfence_system();
    st_release_sys(a.flags[t] + a.rank, epoch);
    const unsigned long long* mine = a.flags[a.rank] + t;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(mine) < epoch) {
      if (globaltimer() - t0 > a.timeout_ns) {
        atomicExch_system(a.err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

// -------------------------------------------------------------- accumulate
// Peers accumulate micro-batch gradients to the target batch (the DeDLOC
// round's first step): acc = g for the first micro-batch of a round, then
// acc = acc + g (one fp32 rounding per add, in call order).

__global__ void __launch_bounds__(256) k_accumulate(float* __restrict__ acc,
                                                    const float* __restrict__ g, int64_t n,
                                                    int overwrite) {
  const int64_t nv = n / 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(g) + v);
    float4* d = reinterpret_cast<float4*>(acc) + v;
    if (overwrite) {
      *d = x;
    } else {
      float4 y = *d;
      y.x = __fadd_rn(y.x, x.x);
      y.y = __fadd_rn(y.y, x.y);
      y.z = __fadd_rn(y.z, x.z);
      y.w = __fadd_rn(y.w, x.w);
      *d = y;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t i = nv * 4 + threadIdx.x;
    acc[i] = overwrite ? g[i] : __fadd_rn(acc[i], g[i]);
  }
}

// Copies this rank's L per-peer sample counts into the count table of every
// rank (NVLink stores; the following barrier orders them).
struct PublishArgs {
  const double* staged;          // L counts (device copy of the host tallies)
  double* table[SP_MAX_RANKS];   // every rank's count table for this buffer
  int world, first, L;
};

__global__ void k_publish_counts(PublishArgs a) {
  const int t = threadIdx.x;
  if (t < a.world * a.L) a.table[t / a.L][a.first + t % a.L] = a.staged[t % a.L];
}

// ------------------------------------------------- group all-reduce (fp64)
// Vector primitives of groups::run_plan on device-resident rows, in the
// reference's own arithmetic (fp64; /root/reference/proj/src/groups.cpp:
// 120 class init w*v, 141-143 merged = 0 + sum in first-seen order, 158
// sum / weight), so the GPU and CPU plans agree bit for bit.

struct VecList {
  const double* src[SP_MAX_PEERS];
  int k;
};

__global__ void k_vec_scale(double* __restrict__ dst, const double* __restrict__ src, double w,
                            int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __dmul_rn(src[i], w);
}

__global__ void k_vec_sum(double* __restrict__ dst, VecList l, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < l.k; ++c) s = __dadd_rn(s, l.src[c][i]);
    dst[i] = s;
  }
}

__global__ void k_vec_div(double* __restrict__ dst, const double* __restrict__ src, double d,
                          int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ddiv_rn(src[i], d);
}

// -------------------------------------------------------------------- pack
// K1. fp32 accumulated gradient -> wire format. blockIdx.y = local peer.

__global__ void __launch_bounds__(256) k_pack_fp32(PackArgs a) {
  const float* __restrict__ src = a.src[blockIdx.y];
  const RangeSlice rs = cta_slice(a);
  const int j = rs.j;
  const int64_t nunits = src ? rs.end : 0;
  const int64_t nfull = a.n / 4;
  for (int64_t w = rs.first; w < nunits; w += rs.stride) {
    const int64_t v = a.lo[j] + w;
    float4 x;
    if (v < nfull) {
      x = __ldg(reinterpret_cast<const float4*>(src) + v);
    } else {
      const int64_t e = v * 4;
      x.x = e + 0 < a.n ? src[e + 0] : 0.0f;
      x.y = e + 1 < a.n ? src[e + 1] : 0.0f;
      x.z = e + 2 < a.n ? src[e + 2] : 0.0f;
      x.w = e + 3 < a.n ? src[e + 3] : 0.0f;
    }
    float* dst = static_cast<float*>(a.dst[blockIdx.y][a.owner[j]]);
    reinterpret_cast<float4*>(dst)[v] = x;
  }
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __halves2half2(__float2half_rn(lo), __float2half_rn(hi));
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float2 unpack_half2(uint32_t u) {
  __half2 h = *reinterpret_cast<__half2*>(&u);
  return __half22float2(h);
}

__global__ void __launch_bounds__(256) k_pack_fp16(PackArgs a) {
  const float* __restrict__ src = a.src[blockIdx.y];
  const RangeSlice rs = cta_slice(a);
  const int j = rs.j;
  const int64_t nunits = src ? rs.end : 0;
  const int64_t nfull = a.n / 8;
  for (int64_t w = rs.first; w < nunits; w += rs.stride) {
    const int64_t v = a.lo[j] + w;
    float x[8];
    if (v < nfull) {
      float4 a0 = __ldg(reinterpret_cast<const float4*>(src) + 2 * v);
      float4 a1 = __ldg(reinterpret_cast<const float4*>(src) + 2 * v + 1);
      x[0] = a0.x; x[1] = a0.y; x[2] = a0.z; x[3] = a0.w;
      x[4] = a1.x; x[5] = a1.y; x[6] = a1.z; x[7] = a1.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t e = v * 8 + j;
        x[j] = e < a.n ? src[e] : 0.0f;
      }
    }
    int4 o;
    o.x = (int)pack_half2(x[0], x[1]);
    o.y = (int)pack_half2(x[2], x[3]);
    o.z = (int)pack_half2(x[4], x[5]);
    o.w = (int)pack_half2(x[6], x[7]);
    char* dst = static_cast<char*>(a.dst[blockIdx.y][a.owner[j]]);
    st_v4(dst + v * 16, o);
  }
}

// Blockwise absmax int8. One CTA (qblock/16 threads) per q8 block; thread t
// owns 16 contiguous elements. Codes at dst[0, npad), scales at dst + npad.
__device__ __forceinline__ void load16(const float* __restrict__ src, int64_t e0, int64_t n, float* x) {
  if (e0 + 16 <= n) {
    const float4* s4 = reinterpret_cast<const float4*>(src + e0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 t = __ldg(s4 + k);
      x[4 * k] = t.x; x[4 * k + 1] = t.y; x[4 * k + 2] = t.z; x[4 * k + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = e0 + j < n ? src[e0 + j] : 0.0f;
  }
}

__global__ void __launch_bounds__(1024) k_pack_q8(PackArgs a) {
  __shared__ float red[32];
  const float* __restrict__ src = a.src[blockIdx.y];
  int j = 0;
  while (j + 1 < a.nr && (int)blockIdx.x >= a.cta0[j + 1]) ++j;
  const int64_t nblk = src ? a.pref[j + 1] - a.pref[j] : 0;
  const int nct = a.cta0[j + 1] - a.cta0[j];
  int8_t* __restrict__ codes = static_cast<int8_t*>(a.dst[blockIdx.y][a.owner[j]]);
  float* __restrict__ scales = reinterpret_cast<float*>(codes + a.npad);
  for (int64_t bb = blockIdx.x - a.cta0[j]; bb < nblk; bb += nct) {
    const int64_t b = a.lo[j] + bb;
    const int64_t e0 = b * a.qblock + threadIdx.x * 16;
    float x[16];
    load16(src, e0, a.n, x);
    const float amax = block_max(absmax16(x), red);
    const float inv = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
    st_v4(codes + e0, quant16(x, inv));
    if (threadIdx.x == 0) scales[b] = __fdiv_rn(amax, 127.0f);
  }
}

// ------------------------------------------------------------------ reduce
// K2. Fused reduce-scatter + weighted average + all-gather: this rank reads
// element range [lo, hi) of every contributing peer's wire buffer (local HBM
// or a peer GPU's HBM over NVLink), accumulates sum_g w_g * x_g in fp32 in
// peer order with fmaf, converts to the wire format and stores the result
// into the avg buffer of every rank.

__global__ void __launch_bounds__(256) k_reduce_fp32(ReduceArgs a) {
  __shared__ PeerView pv;
  load_peers(a, pv);
  if (pv.np == 0) return;
  const int64_t nvec = (a.hi - a.lo + 3) / 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = (a.lo + v * 4) * 4;  // bytes
    // the sum starts from the first contributor's product (no +0 seed), so a
    // single contributor with weight 1 reproduces its values bit for bit
    float acc[4];
    {
      const int4 r0 = ld_nc_v4(static_cast<const char*>(pv.src[0]) + off);
      acc[0] = __fmul_rn(pv.w[0], __int_as_float(r0.x));
      acc[1] = __fmul_rn(pv.w[0], __int_as_float(r0.y));
      acc[2] = __fmul_rn(pv.w[0], __int_as_float(r0.z));
      acc[3] = __fmul_rn(pv.w[0], __int_as_float(r0.w));
    }
    int g = 1;
    for (; g + 4 <= pv.np; g += 4) {
      int4 r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = ld_nc_v4(static_cast<const char*>(pv.src[g + k]) + off);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float w = pv.w[g + k];
        acc[0] = __fmaf_rn(w, __int_as_float(r[k].x), acc[0]);
        acc[1] = __fmaf_rn(w, __int_as_float(r[k].y), acc[1]);
        acc[2] = __fmaf_rn(w, __int_as_float(r[k].z), acc[2]);
        acc[3] = __fmaf_rn(w, __int_as_float(r[k].w), acc[3]);
      }
    }
    for (; g < pv.np; ++g) {
      int4 r = ld_nc_v4(static_cast<const char*>(pv.src[g]) + off);
      const float w = pv.w[g];
      acc[0] = __fmaf_rn(w, __int_as_float(r.x), acc[0]);
      acc[1] = __fmaf_rn(w, __int_as_float(r.y), acc[1]);
      acc[2] = __fmaf_rn(w, __int_as_float(r.z), acc[2]);
      acc[3] = __fmaf_rn(w, __int_as_float(r.w), acc[3]);
    }
    int4 o = make_int4(__float_as_int(acc[0]), __float_as_int(acc[1]),
                       __float_as_int(acc[2]), __float_as_int(acc[3]));
    for (int k = 0; k < a.ndst; ++k) st_v4(static_cast<char*>(a.dst[k]) + off, o);
  }
}

__device__ __forceinline__ void fma_half8(float* acc, float w, int4 r) {
  const uint32_t u[4] = {(uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 f = unpack_half2(u[k]);
    acc[2 * k] = __fmaf_rn(w, f.x, acc[2 * k]);
    acc[2 * k + 1] = __fmaf_rn(w, f.y, acc[2 * k + 1]);
  }
}

__device__ __forceinline__ void mul_half8(float* acc, float w, int4 r) {
  const uint32_t u[4] = {(uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 f = unpack_half2(u[k]);
    acc[2 * k] = __fmul_rn(w, f.x);
    acc[2 * k + 1] = __fmul_rn(w, f.y);
  }
}

__global__ void __launch_bounds__(256) k_reduce_fp16(ReduceArgs a) {
  __shared__ PeerView pv;
  load_peers(a, pv);
  if (pv.np == 0) return;
  const int64_t nvec = (a.hi - a.lo + 7) / 8;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = (a.lo + v * 8) * 2;  // bytes
    float acc[8];
    mul_half8(acc, pv.w[0], ld_nc_v4(static_cast<const char*>(pv.src[0]) + off));
    int g = 1;
    for (; g + 4 <= pv.np; g += 4) {
      int4 r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = ld_nc_v4(static_cast<const char*>(pv.src[g + k]) + off);
#pragma unroll
      for (int k = 0; k < 4; ++k) fma_half8(acc, pv.w[g + k], r[k]);
    }
    for (; g < pv.np; ++g)
      fma_half8(acc, pv.w[g], ld_nc_v4(static_cast<const char*>(pv.src[g]) + off));
    int4 o;
    o.x = (int)pack_half2(acc[0], acc[1]);
    o.y = (int)pack_half2(acc[2], acc[3]);
    o.z = (int)pack_half2(acc[4], acc[5]);
    o.w = (int)pack_half2(acc[6], acc[7]);
    for (int k = 0; k < a.ndst; ++k) st_v4(static_cast<char*>(a.dst[k]) + off, o);
  }
}

__device__ __forceinline__ void fma_q8x16(float* acc, float w, float scale, int4 r) {
  const uint32_t u[4] = {(uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 q = dequant4(u[k]);
    acc[4 * k] = __fmaf_rn(w, __fmul_rn(q.x, scale), acc[4 * k]);
    acc[4 * k + 1] = __fmaf_rn(w, __fmul_rn(q.y, scale), acc[4 * k + 1]);
    acc[4 * k + 2] = __fmaf_rn(w, __fmul_rn(q.z, scale), acc[4 * k + 2]);
    acc[4 * k + 3] = __fmaf_rn(w, __fmul_rn(q.w, scale), acc[4 * k + 3]);
  }
}

__device__ __forceinline__ void mul_q8x16(float* acc, float w, float scale, int4 r) {
  const uint32_t u[4] = {(uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 q = dequant4(u[k]);
    acc[4 * k] = __fmul_rn(w, __fmul_rn(q.x, scale));
    acc[4 * k + 1] = __fmul_rn(w, __fmul_rn(q.y, scale));
    acc[4 * k + 2] = __fmul_rn(w, __fmul_rn(q.z, scale));
    acc[4 * k + 3] = __fmul_rn(w, __fmul_rn(q.w, scale));
  }
}

// q8 blocks of [lo, hi) (lo block aligned), qblock/16 threads per CTA.
// Every thread loads the peers' scales itself (warp-broadcast loads issued
// together with the codes), so the only barriers are the block max's two.
__device__ __forceinline__ float peer_scale(const PeerView& pv, int g, int64_t npad, int64_t b) {
  return __ldg(reinterpret_cast<const float*>(static_cast<const char*>(pv.src[g]) + npad) + b);
}

__global__ void __launch_bounds__(1024) k_reduce_q8(ReduceArgs a) {
  __shared__ float red[32];
  __shared__ PeerView pv;
  load_peers(a, pv);
  if (pv.np == 0) return;
  const int64_t b0 = a.lo / a.qblock;
  const int64_t b1 = (a.hi + a.qblock - 1) / a.qblock;
  if (pv.np == 1) {  // one contributor: its codes and scales, forwarded unchanged
    for (int64_t b = b0 + blockIdx.x; b < b1; b += gridDim.x) {
      const int64_t e0 = b * a.qblock + threadIdx.x * 16;
      const int4 r = ld_nc_v4(static_cast<const char*>(pv.src[0]) + e0);
      const float sc = peer_scale(pv, 0, a.npad, b);
      for (int k = 0; k < a.ndst; ++k) {
        char* d = static_cast<char*>(a.dst[k]);
        st_v4(d + e0, r);
        if (threadIdx.x == 0) reinterpret_cast<float*>(d + a.npad)[b] = sc;
      }
    }
    return;
  }
  for (int64_t b = b0 + blockIdx.x; b < b1; b += gridDim.x) {
    const int64_t e0 = b * a.qblock + threadIdx.x * 16;
    float acc[16];
    mul_q8x16(acc, pv.w[0], peer_scale(pv, 0, a.npad, b),
              ld_nc_v4(static_cast<const char*>(pv.src[0]) + e0));
    int g = 1;
    for (; g + 4 <= pv.np; g += 4) {
      int4 r[4];
      float sc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        r[k] = ld_nc_v4(static_cast<const char*>(pv.src[g + k]) + e0);
        sc[k] = peer_scale(pv, g + k, a.npad, b);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) fma_q8x16(acc, pv.w[g + k], sc[k], r[k]);
    }
    for (; g < pv.np; ++g)
      fma_q8x16(acc, pv.w[g], peer_scale(pv, g, a.npad, b),
                ld_nc_v4(static_cast<const char*>(pv.src[g]) + e0));
    const float amax = block_max(absmax16(acc), red);
    const float inv = amax > 0.0f ? __fdiv_rn(127.0f, amax) : 0.0f;
    const int4 o = quant16(acc, inv);
    const float scale = __fdiv_rn(amax, 127.0f);
    for (int k = 0; k < a.ndst; ++k) {
      char* d = static_cast<char*>(a.dst[k]);
      st_v4(d + e0, o);
      if (threadIdx.x == 0) reinterpret_cast<float*>(d + a.npad)[b] = scale;
    }
  }
}

// -------------------------------------------------------------------- LAMB
// K3 (moments + per-chunk norm partials) and K4 (update). Per element:
//   m' = b1*m + (1-b1)*g          v' = b2*v + (1-b2)*g^2
//   u  = (m'*ibc1) / (sqrt(v'*ibc2) + eps) + wd*p
//   trust_t = ||p||_t / ||u||_t  (1 if either norm is 0)
//   p' = p - (lr*trust_t) * u
// The reference has no optimizer beyond x <- x - lr*g
// (/root/reference/proj/src/sgd.cpp:207-210) and scopes LAMB out
// (/root/reference/SPEC.md:519); this follows You et al. (2019) as cited by
// the paper.

// The averaged gradient of 4 elements in two steps, so that a thread issues
// every load of an iteration before the first dependent store: grad_load
// issues the load (raw wire bits, or the fp32 gradient when the pack is
// fused), grad_finish converts it and, with the fused pack, stores the wire
// values.
struct GradRaw {
  float4 f;    // fp32 gradient (fused pack) or fp32 wire
  uint2 h;     // fp16 wire
  uint32_t q;  // q8 codes
  float s;     // q8 scale
};

// FP: the pack is fused (one rank, one peer, fp32/fp16 wire; a.g32 set).
template <int W, bool FP>
__device__ __forceinline__ GradRaw grad_load(const LambArgs& a, int64_t i) {
  GradRaw r;
  if constexpr (FP) {
    r.f = *reinterpret_cast<const float4*>(a.g32 + i);
    return r;
  }
  if constexpr (W == SP_WIRE_FP32) {
    r.f = *reinterpret_cast<const float4*>(static_cast<const float*>(a.avg) + i);
  } else if constexpr (W == SP_WIRE_FP16) {
    r.h = *reinterpret_cast<const uint2*>(static_cast<const __half*>(a.avg) + i);
  } else {
    r.q = *reinterpret_cast<const uint32_t*>(static_cast<const int8_t*>(a.avg) + i);
    r.s = a.avg_scale[i >> a.qshift];
  }
  return r;
}

template <int W, bool FP>
__device__ __forceinline__ float4 grad_finish(const LambArgs& a, int64_t i, const GradRaw& r) {
  if constexpr (FP) {  // fused pack: the identity average, rounded to the wire format
    static_assert(W != SP_WIRE_Q8, "the q8 pack is never fused");
    if constexpr (W == SP_WIRE_FP32) {
      *reinterpret_cast<float4*>(static_cast<float*>(a.wire_out) + i) = r.f;
      return r.f;
    } else {
      const uint32_t lo = pack_half2(r.f.x, r.f.y), hi = pack_half2(r.f.z, r.f.w);
      *reinterpret_cast<uint2*>(static_cast<__half*>(a.wire_out) + i) = make_uint2(lo, hi);
      const float2 f0 = unpack_half2(lo), f1 = unpack_half2(hi);
      return make_float4(f0.x, f0.y, f1.x, f1.y);
    }
  }
  if constexpr (W == SP_WIRE_FP32) {
    return r.f;
  } else if constexpr (W == SP_WIRE_FP16) {
    const float2 lo = unpack_half2(r.h.x), hi = unpack_half2(r.h.y);
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  } else {
    const float4 q = dequant4(r.q);
    return make_float4(__fmul_rn(q.x, r.s), __fmul_rn(q.y, r.s), __fmul_rn(q.z, r.s), __fmul_rn(q.w, r.s));
  }
}

template <int W, bool FP>
__device__ __forceinline__ float load_grad1(const LambArgs& a, int64_t i) {
  if constexpr (FP) {  // fused pack
    const float x = a.g32[i];
    if constexpr (W == SP_WIRE_FP32) {
      static_cast<float*>(a.wire_out)[i] = x;
      return x;
    } else {
      const __half h = __float2half_rn(x);
      static_cast<__half*>(a.wire_out)[i] = h;
      return __half2float(h);
    }
  }
  if constexpr (W == SP_WIRE_FP32) {
    return static_cast<const float*>(a.avg)[i];
  } else if constexpr (W == SP_WIRE_FP16) {
    return __half2float(static_cast<const __half*>(a.avg)[i]);
  } else {
    return __fmul_rn((float)static_cast<const int8_t*>(a.avg)[i], a.avg_scale[i >> a.qshift]);
  }
}

struct LambScalars {
  float lr, ibc1, ibc2;
};

// IEEE sqrt / division with exact-zero operands kept off the library slow
// path (sqrt(+-0) = +-0; (+-0)/d = +-0 for d > 0), bit-identical results.
// With the 8-bit wire most small gradients average to exactly 0, so m and v
// stay 0 and the slow path would otherwise double the kernel's instructions.
__device__ __forceinline__ float sqrt_rn_z(float x) {
  const bool z = x == 0.0f;
  const float r = __fsqrt_rn(z ? 1.0f : x);
  return z ? x : r;
}

__device__ __forceinline__ float div_rn_z(float a, float b) {
  const bool z = (a == 0.0f) & (b > 0.0f);
  const float r = __fdiv_rn(z ? 1.0f : a, b);
  return z ? a : r;
}

__device__ __forceinline__ void lamb_moments(const LambArgs& a, const LambScalars& s,
                                             float g, float p, float& m, float& v,
                                             float& u) {
  m = __fmaf_rn(a.b1, m, __fmul_rn(a.omb1, g));
  v = __fmaf_rn(a.b2, v, __fmul_rn(a.omb2, __fmul_rn(g, g)));
  const float den = __fadd_rn(sqrt_rn_z(__fmul_rn(v, s.ibc2)), a.eps);
  u = __fmaf_rn(a.wd, p, div_rn_z(__fmul_rn(m, s.ibc1), den));
}

__device__ __forceinline__ float lamb_dir(const LambArgs& a, const LambScalars& s,
                                          float p, float m, float v) {
  const float den = __fadd_rn(sqrt_rn_z(__fmul_rn(v, s.ibc2)), a.eps);
  return __fmaf_rn(a.wd, p, div_rn_z(__fmul_rn(m, s.ibc1), den));
}

// Splits chunk [start, start+len) into a scalar head (until 4-aligned), a
// float4 body and a scalar tail.
struct ChunkSplit {
  int64_t start;
  int head, nbody4, tail;
};

__device__ __forceinline__ ChunkSplit split_chunk(long long start, int len) {
  ChunkSplit s;
  s.start = start;
  int head = (int)((4 - (start & 3)) & 3);
  if (head > len) head = len;
  s.head = head;
  s.nbody4 = (len - head) >> 2;
  s.tail = len - head - 4 * s.nbody4;
  return s;
}

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct ParamPush {
  float* dst[SP_MAX_RANKS];  // every rank's parameter vector, next rank first, self last
  int ndst;
};

}  // namespace sp
