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

constexpr int kLambChunk = 8192;  // elements per LAMB work item (one CTA)
#ifndef SP_LAMB_THREADS
#define SP_LAMB_THREADS 256
#endif
constexpr int kLambThreads = SP_LAMB_THREADS;
constexpr int kPad = 16384;       // wire/avg buffers padded to this multiple

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

struct Chunk {
  long long start;
  int len;
  int tensor;
};

struct LambArgs {
  const void* avg;          // all-gathered averaged gradient, wire format
  const float* avg_scale;   // q8 scales (nullptr otherwise)
  float* p;
  float* m;
  float* v;
  const Chunk* chunks;
  float2* partial;          // per chunk (sum p^2, sum u^2)
  const float* hp;          // device: [lr, 1/(1-b1^t), 1/(1-b2^t)]
  const float* step_scale;  // per tensor lr * trust (update kernel only)
  float b1, b2, omb1, omb2, eps, wd;
  int qshift;               // log2(q8 block): scale index = i >> qshift
  int l2_hints;             // fused LAMB: keep p/m/v of pass 1 in L2 for pass 2
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

template <int W>
__device__ __forceinline__ float4 load_grad4(const LambArgs& a, int64_t i) {
  if constexpr (W != SP_WIRE_Q8) {
    if (a.g32) {  // fused pack
      const float4 x = *reinterpret_cast<const float4*>(a.g32 + i);
      if constexpr (W == SP_WIRE_FP32) {
        *reinterpret_cast<float4*>(static_cast<float*>(a.wire_out) + i) = x;
        return x;
      } else {
        const uint32_t lo = pack_half2(x.x, x.y), hi = pack_half2(x.z, x.w);
        *reinterpret_cast<uint2*>(static_cast<__half*>(a.wire_out) + i) = make_uint2(lo, hi);
        const float2 f0 = unpack_half2(lo), f1 = unpack_half2(hi);
        return make_float4(f0.x, f0.y, f1.x, f1.y);
      }
    }
  }
  if constexpr (W == SP_WIRE_FP32) {
    return *reinterpret_cast<const float4*>(static_cast<const float*>(a.avg) + i);
  } else if constexpr (W == SP_WIRE_FP16) {
    uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __half*>(a.avg) + i);
    float2 lo = unpack_half2(u.x), hi = unpack_half2(u.y);
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  } else {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(static_cast<const int8_t*>(a.avg) + i);
    const float s = a.avg_scale[i >> a.qshift];
    const float4 q = dequant4(u);
    return make_float4(__fmul_rn(q.x, s), __fmul_rn(q.y, s), __fmul_rn(q.z, s), __fmul_rn(q.w, s));
  }
}

template <int W>
__device__ __forceinline__ float load_grad1(const LambArgs& a, int64_t i) {
  if constexpr (W != SP_WIRE_Q8) {
    if (a.g32) {  // fused pack
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

__device__ __forceinline__ ChunkSplit split_chunk(const Chunk& c) {
  ChunkSplit s;
  s.start = c.start;
  int head = (int)((4 - (c.start & 3)) & 3);
  if (head > c.len) head = c.len;
  s.head = head;
  s.nbody4 = (c.len - head) >> 2;
  s.tail = c.len - head - 4 * s.nbody4;
  return s;
}

template <int W>
__global__ void __launch_bounds__(kLambThreads) k_lamb_moments(LambArgs a) {
  __shared__ float red_p[kLambThreads / 32], red_u[kLambThreads / 32];
  const Chunk c = a.chunks[blockIdx.x];
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const ChunkSplit sp = split_chunk(c);
  float pp = 0.0f, uu = 0.0f;
  const int t = threadIdx.x;
  // scalar head and tail
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
    pp = __fmaf_rn(p, p, pp);
    uu = __fmaf_rn(u, u, uu);
  }
  const int64_t b0 = sp.start + sp.head;
  for (int k = t; k < sp.nbody4; k += kLambThreads) {
    const int64_t i = b0 + 4 * (int64_t)k;
    const float4 g = load_grad4<W>(a, i);
    const float4 p = *reinterpret_cast<const float4*>(a.p + i);
    float4 m = *reinterpret_cast<const float4*>(a.m + i);
    float4 v = *reinterpret_cast<const float4*>(a.v + i);
    float4 u;
    lamb_moments(a, s, g.x, p.x, m.x, v.x, u.x);
    lamb_moments(a, s, g.y, p.y, m.y, v.y, u.y);
    lamb_moments(a, s, g.z, p.z, m.z, v.z, u.z);
    lamb_moments(a, s, g.w, p.w, m.w, v.w, u.w);
    *reinterpret_cast<float4*>(a.m + i) = m;
    *reinterpret_cast<float4*>(a.v + i) = v;
    pp = __fmaf_rn(p.x, p.x, pp); pp = __fmaf_rn(p.y, p.y, pp);
    pp = __fmaf_rn(p.z, p.z, pp); pp = __fmaf_rn(p.w, p.w, pp);
    uu = __fmaf_rn(u.x, u.x, uu); uu = __fmaf_rn(u.y, u.y, uu);
    uu = __fmaf_rn(u.z, u.z, uu); uu = __fmaf_rn(u.w, u.w, uu);
  }
  pp = warp_sum(pp);
  uu = warp_sum(uu);
  const int lane = t & 31, wid = t >> 5;
  if (lane == 0) {
    red_p[wid] = pp;
    red_u[wid] = uu;
  }
  __syncthreads();
  if (t == 0) {
    float sp_ = 0.0f, su = 0.0f;
#pragma unroll
    for (int w = 0; w < kLambThreads / 32; ++w) {
      sp_ += red_p[w];
      su += red_u[w];
    }
    a.partial[blockIdx.x] = make_float2(sp_, su);
  }
}

// One CTA per tensor: deterministic fp64 sum of its chunk partials, then
// step_scale[t] = lr * trust_t and trust[t].
__global__ void __launch_bounds__(256) k_lamb_trust(const float2* __restrict__ partial,
                                                    const int2* __restrict__ tchunks,
                                                    const float* __restrict__ hp,
                                                    float* __restrict__ trust,
                                                    float* __restrict__ step_scale) {
  __shared__ double sp_[256], su[256];
  const int2 r = tchunks[blockIdx.x];
  double a = 0.0, b = 0.0;
  for (int c = r.x + threadIdx.x; c < r.y; c += blockDim.x) {
    const float2 q = partial[c];
    a += (double)q.x;
    b += (double)q.y;
  }
  sp_[threadIdx.x] = a;
  su[threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sp_[threadIdx.x] += sp_[threadIdx.x + s];
      su[threadIdx.x] += su[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double r1 = sqrt(sp_[0]), r2 = sqrt(su[0]);
    const float tr = (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
    trust[blockIdx.x] = tr;
    step_scale[blockIdx.x] = __fmul_rn(hp[0], tr);
  }
}

// ------------------------------------------------------------ fused LAMB
// One persistent kernel for K3 + trust + K4. Work items (chunk, pass) are
// handed out in a host-built order through an atomic counter: all pass-1
// chunks in tensor order, with the pass-2 chunks of tensor t inserted `lag`
// items after t's last pass-1 chunk, so pass 2 re-reads p/m/v while they are
// still L2-resident. The CTA finishing the last pass-1 chunk of a tensor
// reduces its chunk partials (fixed order, fp64) into trust[t] and releases
// a ready flag that the tensor's pass-2 CTAs acquire. Items are taken in
// list order and a pass-2 item only waits on earlier pass-1 items, so the
// queue cannot deadlock; the last CTA to exit resets the counters for the
// next launch (CUDA-graph replay safe).

struct FusedLamb {
  const int* items;        // >= 0: pass-1 chunk, < 0: ~chunk for pass 2
  int nitems;
  int* work;               // next item
  int* exited;             // CTAs done
  int* done;               // per tensor: pass-1 chunks finished
  unsigned int* ready;     // per tensor: trust available
  const int2* tchunks;     // per tensor [first, last) chunk
  float* trust;
  int ntensors;
  int final_launch;        // last LAMB launch of the round: clears the trust flags
};

template <int W>
__device__ __forceinline__ void lamb_p1_vec(const LambArgs& a, const LambScalars& s, int64_t i,
                                            float4 g, float4 p, float4 m, float4 v, float& pp,
                                            float& uu) {
  float4 u;
  lamb_moments(a, s, g.x, p.x, m.x, v.x, u.x);
  lamb_moments(a, s, g.y, p.y, m.y, v.y, u.y);
  lamb_moments(a, s, g.z, p.z, m.z, v.z, u.z);
  lamb_moments(a, s, g.w, p.w, m.w, v.w, u.w);
  if (a.l2_hints) {
    const uint64_t keep = policy_evict_last();
    st_hint_f4(a.m + i, m, keep);
    st_hint_f4(a.v + i, v, keep);
  } else {
    *reinterpret_cast<float4*>(a.m + i) = m;
    *reinterpret_cast<float4*>(a.v + i) = v;
  }
  pp = __fmaf_rn(p.x, p.x, pp); pp = __fmaf_rn(p.y, p.y, pp);
  pp = __fmaf_rn(p.z, p.z, pp); pp = __fmaf_rn(p.w, p.w, pp);
  uu = __fmaf_rn(u.x, u.x, uu); uu = __fmaf_rn(u.y, u.y, uu);
  uu = __fmaf_rn(u.z, u.z, uu); uu = __fmaf_rn(u.w, u.w, uu);
}

template <int W>
__device__ __forceinline__ void lamb_pass1(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                           float& pp, float& uu) {
  const ChunkSplit sp = split_chunk(c);
  const int t = threadIdx.x;
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
    pp = __fmaf_rn(p, p, pp);
    uu = __fmaf_rn(u, u, uu);
  }
  const int64_t b0 = sp.start + sp.head;
  int k = t;
  // two independent vectors per iteration: all 8 loads issued before use
  for (; k + kLambThreads < sp.nbody4; k += 2 * kLambThreads) {
    const int64_t i0 = b0 + 4 * (int64_t)k, i1 = i0 + 4 * (int64_t)kLambThreads;
    const float4 g0 = load_grad4<W>(a, i0), g1 = load_grad4<W>(a, i1);
    float4 p0, p1, m0, m1, v0, v1;
    if (a.l2_hints) {
      const uint64_t keep = policy_evict_last();
      p0 = ld_hint_f4(a.p + i0, keep);
      p1 = ld_hint_f4(a.p + i1, keep);
      m0 = ld_hint_f4(a.m + i0, keep);
      m1 = ld_hint_f4(a.m + i1, keep);
      v0 = ld_hint_f4(a.v + i0, keep);
      v1 = ld_hint_f4(a.v + i1, keep);
    } else {
      p0 = *reinterpret_cast<const float4*>(a.p + i0);
      p1 = *reinterpret_cast<const float4*>(a.p + i1);
      m0 = *reinterpret_cast<const float4*>(a.m + i0);
      m1 = *reinterpret_cast<const float4*>(a.m + i1);
      v0 = *reinterpret_cast<const float4*>(a.v + i0);
      v1 = *reinterpret_cast<const float4*>(a.v + i1);
    }
    lamb_p1_vec<W>(a, s, i0, g0, p0, m0, v0, pp, uu);
    lamb_p1_vec<W>(a, s, i1, g1, p1, m1, v1, pp, uu);
  }
  if (k < sp.nbody4) {
    const int64_t i = b0 + 4 * (int64_t)k;
    lamb_p1_vec<W>(a, s, i, load_grad4<W>(a, i), *reinterpret_cast<const float4*>(a.p + i),
                   *reinterpret_cast<const float4*>(a.m + i),
                   *reinterpret_cast<const float4*>(a.v + i), pp, uu);
  }
}

__device__ __forceinline__ float4 lamb_p2_vec(const LambArgs& a, const LambScalars& s, float neg,
                                              float4 p, float4 m, float4 v) {
  p.x = __fmaf_rn(neg, lamb_dir(a, s, p.x, m.x, v.x), p.x);
  p.y = __fmaf_rn(neg, lamb_dir(a, s, p.y, m.y, v.y), p.y);
  p.z = __fmaf_rn(neg, lamb_dir(a, s, p.z, m.z, v.z), p.z);
  p.w = __fmaf_rn(neg, lamb_dir(a, s, p.w, m.w, v.w), p.w);
  return p;
}

__device__ __forceinline__ void lamb_pass2(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                           float neg) {
  const ChunkSplit sp = split_chunk(c);
  const int t = threadIdx.x;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = sp.start + sp.head + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float p = a.p[si];
    a.p[si] = __fmaf_rn(neg, lamb_dir(a, s, p, a.m[si], a.v[si]), p);
  }
  const int64_t b0 = sp.start + sp.head;
  int k = t;
  for (; k + kLambThreads < sp.nbody4; k += 2 * kLambThreads) {
    const int64_t i0 = b0 + 4 * (int64_t)k, i1 = i0 + 4 * (int64_t)kLambThreads;
    if (a.l2_hints) {  // last use of m/v this step: let them go first
      const uint64_t drop = policy_evict_first();
      const float4 p0 = ld_hint_f4(a.p + i0, drop), p1 = ld_hint_f4(a.p + i1, drop);
      const float4 m0 = ld_hint_f4(a.m + i0, drop), m1 = ld_hint_f4(a.m + i1, drop);
      const float4 v0 = ld_hint_f4(a.v + i0, drop), v1 = ld_hint_f4(a.v + i1, drop);
      st_hint_f4(a.p + i0, lamb_p2_vec(a, s, neg, p0, m0, v0), drop);
      st_hint_f4(a.p + i1, lamb_p2_vec(a, s, neg, p1, m1, v1), drop);
      continue;
    }
    const float4 p0 = *reinterpret_cast<const float4*>(a.p + i0);
    const float4 p1 = *reinterpret_cast<const float4*>(a.p + i1);
    const float4 m0 = *reinterpret_cast<const float4*>(a.m + i0);
    const float4 m1 = *reinterpret_cast<const float4*>(a.m + i1);
    const float4 v0 = *reinterpret_cast<const float4*>(a.v + i0);
    const float4 v1 = *reinterpret_cast<const float4*>(a.v + i1);
    *reinterpret_cast<float4*>(a.p + i0) = lamb_p2_vec(a, s, neg, p0, m0, v0);
    *reinterpret_cast<float4*>(a.p + i1) = lamb_p2_vec(a, s, neg, p1, m1, v1);
  }
  if (k < sp.nbody4) {
    const int64_t i = b0 + 4 * (int64_t)k;
    *reinterpret_cast<float4*>(a.p + i) =
        lamb_p2_vec(a, s, neg, *reinterpret_cast<const float4*>(a.p + i),
                    *reinterpret_cast<const float4*>(a.m + i), *reinterpret_cast<const float4*>(a.v + i));
  }
}

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef SP_LAMB_MIN_CTAS
#define SP_LAMB_MIN_CTAS 1
#endif
template <int W>
__global__ void __launch_bounds__(kLambThreads, SP_LAMB_MIN_CTAS) k_lamb_fused(LambArgs a, FusedLamb f) {
  __shared__ int s_item;
  __shared__ int s_last;
  __shared__ float s_scale;
  __shared__ float red_p[kLambThreads / 32], red_u[kLambThreads / 32];
  __shared__ double dred_p[kLambThreads], dred_u[kLambThreads];
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int next = 0;
  if (tid == 0) next = atomicAdd(f.work, 1);
  for (;;) {
    if (tid == 0) s_item = next;
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= f.nitems) break;
    if (tid == 0) next = atomicAdd(f.work, 1);  // in flight while this item runs
    const int code = f.items[it];
    if (code >= 0) {
      const Chunk c = a.chunks[code];
      float pp = 0.0f, uu = 0.0f;
      lamb_pass1<W>(a, s, c, pp, uu);
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
        a.partial[code] = make_float2(sp_, su);
        __threadfence();
        const int2 r = f.tchunks[c.tensor];
        s_last = atomicAdd(f.done + c.tensor, 1) == r.y - r.x - 1;
      }
      __syncthreads();
      if (s_last) {  // every pass-1 chunk of this tensor has published its partial
        __threadfence();
        const int2 r = f.tchunks[c.tensor];
        double dp = 0.0, du = 0.0;
        for (int q = r.x + tid; q < r.y; q += kLambThreads) {
          const float2 v = __ldcg(a.partial + q);
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
          f.trust[c.tensor] = tr;
          const_cast<float*>(a.step_scale)[c.tensor] = __fmul_rn(s.lr, tr);
          f.done[c.tensor] = 0;
          __threadfence();
          st_release_gpu(f.ready + c.tensor, 1u);
        }
      }
    } else {
      const Chunk c = a.chunks[~code];
      if (tid == 0) {
        while (ld_acquire_gpu(f.ready + c.tensor) == 0u) __nanosleep(64);
        s_scale = __ldcg(a.step_scale + c.tensor);
      }
      __syncthreads();
      lamb_pass2(a, s, c, -s_scale);
    }
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(f.exited, 1) == (int)gridDim.x - 1) {  // last CTA out resets the queue
      if (f.final_launch)
        for (int t = 0; t < f.ntensors; ++t) f.ready[t] = 0u;
      *f.work = 0;
      *f.exited = 0;
      __threadfence();
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kLambThreads) k_lamb_update(LambArgs a) {
  const Chunk c = a.chunks[blockIdx.x];
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const float neg = -a.step_scale[c.tensor];
  const ChunkSplit sp = split_chunk(c);
  const int t = threadIdx.x;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = sp.start + sp.head + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float p = a.p[si];
    a.p[si] = __fmaf_rn(neg, lamb_dir(a, s, p, a.m[si], a.v[si]), p);
  }
  const int64_t b0 = sp.start + sp.head;
  for (int k = t; k < sp.nbody4; k += kLambThreads) {
    const int64_t i = b0 + 4 * (int64_t)k;
    float4 p = *reinterpret_cast<const float4*>(a.p + i);
    const float4 m = *reinterpret_cast<const float4*>(a.m + i);
    const float4 v = *reinterpret_cast<const float4*>(a.v + i);
    p.x = __fmaf_rn(neg, lamb_dir(a, s, p.x, m.x, v.x), p.x);
    p.y = __fmaf_rn(neg, lamb_dir(a, s, p.y, m.y, v.y), p.y);
    p.z = __fmaf_rn(neg, lamb_dir(a, s, p.z, m.z, v.z), p.z);
    p.w = __fmaf_rn(neg, lamb_dir(a, s, p.w, m.w, v.w), p.w);
    *reinterpret_cast<float4*>(a.p + i) = p;
  }
}

// ------------------------------------------------------ sharded LAMB (N1)
// ZeRO-1 style step: the owner of [lo, hi) runs pass 1
// (k_lamb_moments) on its range only. Per tensor it sums its chunk partials
// in fp64 (chunk order) and stores the pair into slot [rank][t] of every
// rank's norm table; after a barrier every rank adds the world slots in rank
// order, so all ranks hold identical trust ratios; pass 2 updates the owned
// range and stores p' into every rank's parameter vector over NVLink.

struct ShardNormArgs {
  const float2* partial;
  const int2* tchunks;             // this rank's chunks of tensor t (may be empty)
  double2* table[SP_MAX_RANKS];    // push order: next rank first, self last
  int ndst, rank, T;
  int t0;                          // first sharded tensor (CTA b handles t0 + b)
};

__global__ void __launch_bounds__(256) k_shard_norms(ShardNormArgs a) {
  __shared__ double sx[256], sy[256];
  const int t = a.t0 + blockIdx.x;
  const int2 r = a.tchunks[t];
  double x = 0.0, y = 0.0;
  for (int c = r.x + threadIdx.x; c < r.y; c += blockDim.x) {
    const float2 q = a.partial[c];
    x += (double)q.x;
    y += (double)q.y;
  }
  sx[threadIdx.x] = x;
  sy[threadIdx.x] = y;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      sx[threadIdx.x] += sx[threadIdx.x + h];
      sy[threadIdx.x] += sy[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x < a.ndst) a.table[threadIdx.x][(size_t)a.rank * a.T + t] = make_double2(sx[0], sy[0]);
}

// k_lamb_moments with k_shard_norms folded in (the default sharded chain
// when every tensor is sharded): the CTA finishing a tensor's last owned
// chunk sums the chunk partials in fp64 in k_shard_norms' order and stores
// the pair into slot [rank][t] of every rank's table. Tensors this rank has
// no chunk of get a zero pair. `nchunks` may be 0 (grid 1: zeros only).
template <int W>
__global__ void __launch_bounds__(kLambThreads) k_lamb_moments_shard(LambArgs a, ShardNormArgs na,
                                                                    int* __restrict__ done,
                                                                    int nchunks) {
  __shared__ float red_p[kLambThreads / 32], red_u[kLambThreads / 32];
  __shared__ double dred_p[kLambThreads], dred_u[kLambThreads];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int t = na.t0 + blockIdx.x; t < na.T; t += gridDim.x) {
    const int2 r = na.tchunks[t];
    if (r.y <= r.x && tid < na.ndst) na.table[tid][(size_t)na.rank * na.T + t] = make_double2(0.0, 0.0);
  }
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  // grid-stride over the owned chunks (a grid of one resident wave)
  for (int ci = blockIdx.x; ci < nchunks; ci += gridDim.x) {
    const Chunk c = a.chunks[ci];
    float pp = 0.0f, uu = 0.0f;
    lamb_pass1<W>(a, s, c, pp, uu);
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
      a.partial[ci] = make_float2(sp_, su);
      __threadfence();
      const int2 r = na.tchunks[c.tensor];
      s_last = atomicAdd(done + c.tensor, 1) == r.y - r.x - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int2 r = na.tchunks[c.tensor];
      double x = 0.0, y = 0.0;
      for (int q = r.x + tid; q < r.y; q += kLambThreads) {
        const float2 v = __ldcg(a.partial + q);
        x += (double)v.x;
        y += (double)v.y;
      }
      dred_p[tid] = x;
      dred_u[tid] = y;
      __syncthreads();
      for (int h = kLambThreads / 2; h > 0; h >>= 1) {
        if (tid < h) {
          dred_p[tid] += dred_p[tid + h];
          dred_u[tid] += dred_u[tid + h];
        }
        __syncthreads();
      }
      if (tid < na.ndst)
        na.table[tid][(size_t)na.rank * na.T + c.tensor] = make_double2(dred_p[0], dred_u[0]);
      if (tid == 0) done[c.tensor] = 0;
    }
    __syncthreads();  // red_p / s_last reused by the next chunk
  }
}

__device__ __forceinline__ float trust_from_table(const double2* __restrict__ table, int world, int T,
                                                  int t) {
  double x = 0.0, y = 0.0;
  for (int k = 0; k < world; ++k) {
    const double2 v = __ldcg(table + (size_t)k * T + t);
    x += v.x;
    y += v.y;
  }
  const double r1 = sqrt(x), r2 = sqrt(y);
  return (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
}

// trust[t] = sqrt(sum_k pp[k][t]) / sqrt(sum_k uu[k][t]) over ranks in order
// (1 if either is 0); step_scale[t] = lr * trust[t].
__global__ void k_shard_trust(const double2* __restrict__ table, int world, int T, int t0,
                              const float* __restrict__ hp, float* __restrict__ trust,
                              float* __restrict__ step_scale) {
  for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < world; ++k) {
      const double2 v = __ldcg(table + (size_t)k * T + t);
      x += v.x;
      y += v.y;
    }
    const double r1 = sqrt(x), r2 = sqrt(y);
    const float tr = (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
    trust[t] = tr;
    step_scale[t] = __fmul_rn(hp[0], tr);
  }
}

struct ParamPush {
  float* dst[SP_MAX_RANKS];  // every rank's parameter vector, next rank first, self last
  int ndst;
};

// Pass 2 of the owned chunks: p' = p - lr*trust*u, stored into every rank's
// copy (the local one last, so the local read of p precedes the local write).
__device__ __forceinline__ void lamb_push_chunk(const LambArgs& a, const LambScalars& s, const Chunk& c,
                                                float neg, const ParamPush& d) {
  const ChunkSplit sp = split_chunk(c);
  const int t = threadIdx.x;
  int64_t si = -1;
  if (t < sp.head) si = sp.start + t;
  else if (t >= 32 && t - 32 < sp.tail) si = sp.start + sp.head + 4 * (int64_t)sp.nbody4 + (t - 32);
  if (si >= 0) {
    const float p = a.p[si];
    const float q = __fmaf_rn(neg, lamb_dir(a, s, p, a.m[si], a.v[si]), p);
    for (int k = 0; k < d.ndst; ++k) d.dst[k][si] = q;
  }
  const int64_t b0 = sp.start + sp.head;
  int k = t;
  // two vectors per iteration: all loads in flight before the stores
  for (; k + kLambThreads < sp.nbody4; k += 2 * kLambThreads) {
    const int64_t i0 = b0 + 4 * (int64_t)k, i1 = i0 + 4 * (int64_t)kLambThreads;
    const float4 p0 = *reinterpret_cast<const float4*>(a.p + i0);
    const float4 p1 = *reinterpret_cast<const float4*>(a.p + i1);
    const float4 m0 = *reinterpret_cast<const float4*>(a.m + i0);
    const float4 m1 = *reinterpret_cast<const float4*>(a.m + i1);
    const float4 v0 = *reinterpret_cast<const float4*>(a.v + i0);
    const float4 v1 = *reinterpret_cast<const float4*>(a.v + i1);
    const float4 q0 = lamb_p2_vec(a, s, neg, p0, m0, v0), q1 = lamb_p2_vec(a, s, neg, p1, m1, v1);
    const int4 o0 = make_int4(__float_as_int(q0.x), __float_as_int(q0.y), __float_as_int(q0.z),
                              __float_as_int(q0.w));
    const int4 o1 = make_int4(__float_as_int(q1.x), __float_as_int(q1.y), __float_as_int(q1.z),
                              __float_as_int(q1.w));
    for (int q = 0; q < d.ndst; ++q) {
      st_v4(d.dst[q] + i0, o0);
      st_v4(d.dst[q] + i1, o1);
    }
  }
  if (k < sp.nbody4) {
    const int64_t i = b0 + 4 * (int64_t)k;
    const float4 q = lamb_p2_vec(a, s, neg, *reinterpret_cast<const float4*>(a.p + i),
                                 *reinterpret_cast<const float4*>(a.m + i),
                                 *reinterpret_cast<const float4*>(a.v + i));
    const int4 o = make_int4(__float_as_int(q.x), __float_as_int(q.y), __float_as_int(q.z),
                             __float_as_int(q.w));
    for (int j = 0; j < d.ndst; ++j) st_v4(d.dst[j] + i, o);
  }
}

template <int W>
__global__ void __launch_bounds__(kLambThreads) k_lamb_update_push(LambArgs a, ParamPush d) {
  const Chunk c = a.chunks[blockIdx.x];
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  lamb_push_chunk(a, s, c, -__ldcg(a.step_scale + c.tensor), d);
}

// k_lamb_update_push with k_shard_trust folded in: every CTA forms its
// tensor's trust ratio from the norm table (k_shard_trust's arithmetic), and
// CTAs b, b + grid, ... also write trust / step_scale of tensor b (what
// read_trust() returns). `nchunks` may be 0 (grid 1: trust only).
template <int W>
__global__ void __launch_bounds__(kLambThreads) k_lamb_update_push_trust(
    LambArgs a, ParamPush d, const double2* __restrict__ table, int world, int T, int t0,
    float* __restrict__ trust, float* __restrict__ step_scale, int nchunks) {
  __shared__ float s_neg;
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  if (threadIdx.x == 0) {
    for (int t = t0 + blockIdx.x; t < T; t += gridDim.x) {
      const float tr = trust_from_table(table, world, T, t);
      trust[t] = tr;
      step_scale[t] = __fmul_rn(s.lr, tr);
    }
  }
  for (int ci = blockIdx.x; ci < nchunks; ci += gridDim.x) {  // grid-stride over owned chunks
    const Chunk c = a.chunks[ci];
    if (threadIdx.x == 0) s_neg = -__fmul_rn(s.lr, trust_from_table(table, world, T, c.tensor));
    __syncthreads();
    lamb_push_chunk(a, s, c, s_neg, d);
    __syncthreads();
  }
}

// ------------------------------------------- sharded LAMB, one kernel (N1)
// The chain above (pass 1 -> norms -> barrier -> trust -> pass 2 + push)
// as one persistent kernel over a work queue of this rank's chunks:
//   pass-1 item: moments + chunk partial; the CTA finishing the tensor's
//     last chunk sums the partials in fp64 (k_shard_norms' order), stores the
//     pair into slot [rank][t] of every rank's norm table and release-stores
//     the round's epoch into flag [rank][t] of every rank;
//   pass-2 item: waits for the world flags of its tensor, forms the trust
//     ratio from the world slots in rank order (k_shard_trust's arithmetic),
//     updates the chunk and stores p' into every rank's parameter vector.
// Pass-2 items of tensor t are queued `lag` items after its last pass-1
// item, so the NVLink push of early tensors can overlap the HBM-bound pass 1
// of later ones. Measured (4x B200, profiles/r01/shard_fused.txt): no faster
// than the chain at 268M elements and 1.4-2.5x slower at ALBERT-large size
// (pass-2 items wait on the slowest chunk of their tensor on every rank, and
// the push needs every CTA to keep NVLink busy), so it is opt-in
// (SP_SHARD_FUSED=1) and kept bit-exact by the tests. Items only wait on earlier items of this rank's queue and
// on other GPUs' pass 1, which progresses independently: no deadlock. The
// last CTA out waits for every flag, writes trust / step_scale for all
// tensors (what read_trust() returns) and resets the queue; flags carry
// the epoch, so nothing needs clearing between graph replays.
struct ShardFused {
  const int* items;                         // >= 0 pass-1 chunk, < 0 ~chunk (pass 2 + push)
  int nitems;
  int* work;
  int* exited;
  int* done;                                // per tensor: pass-1 chunks finished
  const int2* tchunks;                      // this rank's chunks of tensor t
  double2* table[SP_MAX_RANKS];             // norm table of rank (rank + 1 + k) % world
  unsigned long long* flags[SP_MAX_RANKS];  // norm flags of the same ranks
  const double2* my_table;                  // [world][T]
  const unsigned long long* my_flags;       // [world][T]
  unsigned long long* epoch;                // local round counter
  float* trust;
  float* step_scale;
  ParamPush push;
  int rank, world, T;
  int* err;
  unsigned long long timeout_ns;
};

__device__ __forceinline__ bool wait_norms(const ShardFused& f, int t, unsigned long long e) {
  const unsigned long long t0 = globaltimer();
  for (int k = 0; k < f.world; ++k)
    while (ld_acquire_sys(f.my_flags + (size_t)k * f.T + t) < e) {
      if (globaltimer() - t0 > f.timeout_ns) {
        atomicExch_system(f.err, 1);
        return false;
      }
      __nanosleep(256);  // hundreds of CTAs may poll: keep them off the memory system
    }
  return true;
}

__device__ __forceinline__ float shard_trust(const ShardFused& f, int t) {
  double x = 0.0, y = 0.0;
  for (int k = 0; k < f.world; ++k) {
    const double2 v = __ldcg(f.my_table + (size_t)k * f.T + t);
    x += v.x;
    y += v.y;
  }
  const double r1 = sqrt(x), r2 = sqrt(y);
  return (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
}

// thread 0..world-1 store the pair, then thread 0 publishes the epoch
__device__ __forceinline__ void publish_norms(const ShardFused& f, int t, double x, double y,
                                              unsigned long long e) {
  if (threadIdx.x < f.world) {
    f.table[threadIdx.x][(size_t)f.rank * f.T + t] = make_double2(x, y);
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x < f.world) st_release_sys(f.flags[threadIdx.x] + (size_t)f.rank * f.T + t, e);
}

template <int W>
__global__ void __launch_bounds__(kLambThreads, 4) k_shard_lamb_fused(LambArgs a,
                                                                                     ShardFused f) {
  __shared__ int s_item, s_last;
  __shared__ float s_neg;
  __shared__ unsigned long long s_epoch;
  __shared__ float red_p[kLambThreads / 32], red_u[kLambThreads / 32];
  __shared__ double dred_p[kLambThreads], dred_u[kLambThreads];
  const LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_epoch = *f.epoch + 1;
  __syncthreads();
  const unsigned long long e = s_epoch;
  // tensors with no chunk on this rank contribute a zero pair
  for (int t = blockIdx.x; t < f.T; t += gridDim.x) {
    const int2 r = f.tchunks[t];
    if (r.y <= r.x) publish_norms(f, t, 0.0, 0.0, e);
    __syncthreads();
  }
  int next = 0;
  if (tid == 0) next = atomicAdd(f.work, 1);
  for (;;) {
    if (tid == 0) s_item = next;
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= f.nitems) break;
    if (tid == 0) next = atomicAdd(f.work, 1);
    const int code = f.items[it];
    if (code >= 0) {
      const Chunk c = a.chunks[code];
      float pp = 0.0f, uu = 0.0f;
      lamb_pass1<W>(a, s, c, pp, uu);
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
        a.partial[code] = make_float2(sp_, su);
        __threadfence();
        const int2 r = f.tchunks[c.tensor];
        s_last = atomicAdd(f.done + c.tensor, 1) == r.y - r.x - 1;
      }
      __syncthreads();
      if (s_last) {  // this rank's partials of the tensor are all in
        __threadfence();
        const int2 r = f.tchunks[c.tensor];
        double dp = 0.0, du = 0.0;
        for (int q = r.x + tid; q < r.y; q += kLambThreads) {
          const float2 v = __ldcg(a.partial + q);
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
        if (tid == 0) f.done[c.tensor] = 0;
        publish_norms(f, c.tensor, dred_p[0], dred_u[0], e);
      }
    } else {
      const Chunk c = a.chunks[~code];
      if (tid == 0) {
        s_neg = wait_norms(f, c.tensor, e) ? -__fmul_rn(s.lr, shard_trust(f, c.tensor)) : 0.0f;
      }
      __syncthreads();
      lamb_push_chunk(a, s, c, s_neg, f.push);
    }
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(f.exited, 1) == (int)gridDim.x - 1) {  // last CTA out
      for (int t = 0; t < f.T; ++t) {
        const float tr = wait_norms(f, t, e) ? shard_trust(f, t) : 1.0f;
        f.trust[t] = tr;
        f.step_scale[t] = __fmul_rn(s.lr, tr);
      }
      *f.work = 0;
      *f.exited = 0;
      *f.epoch = e;
      __threadfence();
    }
  }
}

}  // namespace sp
