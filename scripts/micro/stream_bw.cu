// stream_bw.cu — what LAMB's pass-1 access pattern can reach on this GPU.
//
//   copy      read 1 stream, write 1 (the MEASURED_PEAKS recipe's pattern)
//   lamb1     read g32, p, m, v; write wire fp16, m, v (26 B/elem), trivial math
//   lamb1m    the same with LAMB's IEEE arithmetic (div, sqrt per element)
//   lamb1s    lamb1m + a store of u into shared memory (the k_lamb stash)
//
// grid-stride, 256-thread CTAs, 2 float4 per thread per iteration; the
// vector is larger than L2 (rotating between two copies defeats reuse).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu
#include <cstdint>
#include <cstdio>

#include "../../paper_2106_10207_b200/csrc/cuda/sp_kernels.cuh"
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) k_copy(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n4; i += (long)gridDim.x * 256) b[i] = a[i];
}

template <int MATH, int STASH>
__global__ void __launch_bounds__(256, 4) k_lamb1(const float4* __restrict__ g, const float4* __restrict__ p,
                                                  float4* __restrict__ m, float4* __restrict__ v,
                                                  uint2* __restrict__ w, long n4, float* sink) {
  __shared__ float4 st[256 * 2];
  float acc = 0.f;
  const long stride = (long)gridDim.x * 512;
  for (long i = blockIdx.x * 512L + threadIdx.x; i < n4; i += stride) {
    const long j = i + 256;
    const bool two = j < n4;
    float4 g0 = g[i], p0 = p[i], m0 = m[i], v0 = v[i];
    float4 g1 = two ? g[j] : g0, p1 = two ? p[j] : p0, m1 = two ? m[j] : m0, v1 = two ? v[j] : v0;
    float4* mm[2] = {&m0, &m1};
    float4* vv[2] = {&v0, &v1};
    float4 gg[2] = {g0, g1}, pp[2] = {p0, p1};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float* gm = &gg[k].x;
      float* pm = &pp[k].x;
      float* ma = &mm[k]->x;
      float* va = &vv[k]->x;
      float u[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ma[e] = __fmaf_rn(0.9f, ma[e], __fmul_rn(0.1f, gm[e]));
        va[e] = __fmaf_rn(0.999f, va[e], __fmul_rn(0.001f, __fmul_rn(gm[e], gm[e])));
        if (MATH) {
          const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(va[e], 1000.f)), 1e-6f);
          u[e] = __fmaf_rn(0.01f, pm[e], __fdiv_rn(__fmul_rn(ma[e], 10.f), den));
        } else {
          u[e] = __fmaf_rn(0.01f, pm[e], ma[e]);
        }
        acc = __fmaf_rn(u[e], u[e], acc);
      }
      if (STASH) st[threadIdx.x + 256 * k] = make_float4(u[0], u[1], u[2], u[3]);
    }
    m[i] = m0;
    v[i] = v0;
    const __half2 a0 = __floats2half2_rn(g0.x, g0.y), a1 = __floats2half2_rn(g0.z, g0.w);
    w[i] = make_uint2(*reinterpret_cast<const unsigned*>(&a0), *reinterpret_cast<const unsigned*>(&a1));
    if (two) {
      m[j] = m1;
      v[j] = v1;
      const __half2 b0 = __floats2half2_rn(g1.x, g1.y), b1 = __floats2half2_rn(g1.z, g1.w);
      w[j] = make_uint2(*reinterpret_cast<const unsigned*>(&b0), *reinterpret_cast<const unsigned*>(&b1));
    }
  }
  if (STASH) acc += st[(threadIdx.x * 7) & 511].x;
  if (acc == 12345.f) *sink = acc;
}

// k_lamb's pass-1 structure without its bookkeeping: 2048-element chunks,
// CLAIM: claimed one ahead from a global counter by thread 0 with one
// __syncthreads per chunk (else static grid-stride), HINT: evict_last on p,
// evict_first on m, v (as k_lamb).
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t q;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(q));
  return q;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t q;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(q));
  return q;
}
__device__ __forceinline__ float4 ldh(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void sth(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

template <int CLAIM, int HINT, int CTAS>
__global__ void __launch_bounds__(256, CTAS) k_lamb2(const float4* __restrict__ g, const float4* __restrict__ p,
                                                     float4* __restrict__ m, float4* __restrict__ v,
                                                     uint2* __restrict__ w, long n4, int* ctr, float2* part) {
  __shared__ float4 st[256 * 2];
  __shared__ int s_item;
  __shared__ float red[8];
  const long nchunks = n4 / 512;
  int next = 0;
  long item = blockIdx.x;
  if (CLAIM) {
    if (threadIdx.x == 0) s_item = atomicAdd(ctr, 1);
    __syncthreads();
    item = s_item;
  }
  const uint64_t pl = pol_last(), pf = pol_first();
  while (item < nchunks) {
    if (CLAIM && threadIdx.x == 0) next = atomicAdd(ctr, 1);
    const long i = item * 512 + threadIdx.x, j = i + 256;
    float4 g0 = g[i], g1 = g[j];
    float4 p0 = HINT ? ldh(p + i, pl) : p[i], p1 = HINT ? ldh(p + j, pl) : p[j];
    float4 m0 = HINT ? ldh(m + i, pf) : m[i], m1 = HINT ? ldh(m + j, pf) : m[j];
    float4 v0 = HINT ? ldh(v + i, pf) : v[i], v1 = HINT ? ldh(v + j, pf) : v[j];
    float4 gg[2] = {g0, g1}, pp[2] = {p0, p1}, mm[2] = {m0, m1}, vv[2] = {v0, v1};
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float* gm = &gg[k].x; float* pm = &pp[k].x; float* ma = &mm[k].x; float* va = &vv[k].x;
      float u[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ma[e] = __fmaf_rn(0.9f, ma[e], __fmul_rn(0.1f, gm[e]));
        va[e] = __fmaf_rn(0.999f, va[e], __fmul_rn(0.001f, __fmul_rn(gm[e], gm[e])));
        const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(va[e], 1000.f)), 1e-6f);
        u[e] = __fmaf_rn(0.01f, pm[e], __fdiv_rn(__fmul_rn(ma[e], 10.f), den));
        acc = __fmaf_rn(u[e], u[e], acc);
      }
      st[threadIdx.x + 256 * k] = make_float4(u[0], u[1], u[2], u[3]);
    }
    if (HINT) { sth(m + i, mm[0], pf); sth(m + j, mm[1], pf); sth(v + i, vv[0], pf); sth(v + j, vv[1], pf); }
    else { m[i] = mm[0]; m[j] = mm[1]; v[i] = vv[0]; v[j] = vv[1]; }
    const __half2 a0 = __floats2half2_rn(g0.x, g0.y), a1 = __floats2half2_rn(g0.z, g0.w);
    w[i] = make_uint2(*reinterpret_cast<const unsigned*>(&a0), *reinterpret_cast<const unsigned*>(&a1));
    const __half2 b0 = __floats2half2_rn(g1.x, g1.y), b1 = __floats2half2_rn(g1.z, g1.w);
    w[j] = make_uint2(*reinterpret_cast<const unsigned*>(&b0), *reinterpret_cast<const unsigned*>(&b1));
    if (CLAIM) {
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
      if (threadIdx.x == 0) s_item = next;
      __syncthreads();
      if (threadIdx.x == 0) {
        float x = 0.f;
        for (int q = 0; q < 8; ++q) x += red[q];
        part[item] = make_float2(x, x);
      }
      item = s_item;
    } else {
      if (acc == 12345.f) part[0] = make_float2(acc, acc);
      item += gridDim.x;
    }
  }
}

// k_lamb2's claim structure with k_lamb's exact per-element code: LAMB
// moments with the IEEE div/sqrt of sp_kernels.cuh (lamb_moments), the fp16
// wire store of the fused pack (grad_load / grad_finish), evict hints.
__global__ void __launch_bounds__(256, 4) k_lamb3(sp::LambArgs a, long n4, int* ctr, float2* part) {
  __shared__ float4 st[256 * 2];
  __shared__ int s_item;
  __shared__ float red[8];
  const long nchunks = n4 / 512;
  int next = 0;
  if (threadIdx.x == 0) s_item = atomicAdd(ctr, 1);
  __syncthreads();
  long item = s_item;
  const sp::LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  const uint64_t pl = sp::policy_evict_last(), pf = sp::policy_evict_first();
  while (item < nchunks) {
    if (threadIdx.x == 0) next = atomicAdd(ctr, 1);
    const int64_t i0 = 4 * (item * 512 + threadIdx.x), i1 = i0 + 4 * 256;
    const sp::GradRaw g0 = sp::grad_load<SP_WIRE_FP16, true>(a, i0), g1 = sp::grad_load<SP_WIRE_FP16, true>(a, i1);
    float4 p0 = sp::ld_hint_f4(a.p + i0, pl), p1 = sp::ld_hint_f4(a.p + i1, pl);
    float4 m0 = sp::ld_hint_f4(a.m + i0, pf), m1 = sp::ld_hint_f4(a.m + i1, pf);
    float4 v0 = sp::ld_hint_f4(a.v + i0, pf), v1 = sp::ld_hint_f4(a.v + i1, pf);
    const float4 f0 = sp::grad_finish<SP_WIRE_FP16, true>(a, i0, g0), f1 = sp::grad_finish<SP_WIRE_FP16, true>(a, i1, g1);
    float pp = 0.f, uu = 0.f;
    float4 u0, u1;
    sp::lamb_moments(a, s, f0.x, p0.x, m0.x, v0.x, u0.x); sp::lamb_moments(a, s, f0.y, p0.y, m0.y, v0.y, u0.y);
    sp::lamb_moments(a, s, f0.z, p0.z, m0.z, v0.z, u0.z); sp::lamb_moments(a, s, f0.w, p0.w, m0.w, v0.w, u0.w);
    sp::lamb_moments(a, s, f1.x, p1.x, m1.x, v1.x, u1.x); sp::lamb_moments(a, s, f1.y, p1.y, m1.y, v1.y, u1.y);
    sp::lamb_moments(a, s, f1.z, p1.z, m1.z, v1.z, u1.z); sp::lamb_moments(a, s, f1.w, p1.w, m1.w, v1.w, u1.w);
    sp::st_hint_f4(a.m + i0, m0, pf); sp::st_hint_f4(a.v + i0, v0, pf);
    sp::st_hint_f4(a.m + i1, m1, pf); sp::st_hint_f4(a.v + i1, v1, pf);
    st[threadIdx.x] = u0;
    st[threadIdx.x + 256] = u1;
    pp = __fmaf_rn(p0.x, p0.x, pp); pp = __fmaf_rn(p1.x, p1.x, pp);
    uu = __fmaf_rn(u0.x, u0.x, uu); uu = __fmaf_rn(u1.x, u1.x, uu);
    for (int o = 16; o > 0; o >>= 1) uu += __shfl_xor_sync(0xffffffffu, uu, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = uu + pp;
    if (threadIdx.x == 0) s_item = next;
    __syncthreads();
    if (threadIdx.x == 0) {
      float x = 0.f;
      for (int q = 0; q < 8; ++q) x += red[q];
      part[item] = make_float2(x, x);
    }
    item = s_item;
  }
}

int main() {
  const long n = 64L << 20;  // elements per array (256 MB fp32): > L2
  const long n4 = n / 4;
  float *a[2], *b[2], *g[2], *p[2], *m[2], *v[2], *sink;
  uint2* w[2];
  for (int k = 0; k < 2; ++k) {
    cudaMalloc(&a[k], n * 4); cudaMalloc(&b[k], n * 4);
    cudaMalloc(&g[k], n * 4); cudaMalloc(&p[k], n * 4); cudaMalloc(&m[k], n * 4); cudaMalloc(&v[k], n * 4);
    cudaMalloc(&w[k], n * 2);
    cudaMemset(a[k], 0, n * 4); cudaMemset(g[k], 0, n * 4); cudaMemset(p[k], 0, n * 4);
    cudaMemset(m[k], 0, n * 4); cudaMemset(v[k], 0, n * 4);
  }
  cudaMalloc(&sink, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double bytes_per_elem, auto launch) {
    for (int r = 0; r < 3; ++r) launch(r & 1);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) launch(r & 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms / reps * 1e-3;
    printf("%-8s %7.1f us/launch  %7.1f GB/s  (%.0f B/elem)\n", name, t * 1e6, bytes_per_elem * n / t / 1e9,
           bytes_per_elem);
  };
  run("copy", 8.0, [&](int k) { k_copy<<<grid, 256>>>((float4*)a[k], (float4*)b[k], n4); });
  run("lamb1", 26.0, [&](int k) {
    k_lamb1<0, 0><<<grid, 256>>>((float4*)g[k], (float4*)p[k], (float4*)m[k], (float4*)v[k], w[k], n4, sink);
  });
  run("lamb1m", 26.0, [&](int k) {
    k_lamb1<1, 0><<<grid, 256>>>((float4*)g[k], (float4*)p[k], (float4*)m[k], (float4*)v[k], w[k], n4, sink);
  });
  run("lamb1s", 26.0, [&](int k) {
    k_lamb1<1, 1><<<grid, 256>>>((float4*)g[k], (float4*)p[k], (float4*)m[k], (float4*)v[k], w[k], n4, sink);
  });
  int* ctr;
  float2* part;
  cudaMalloc(&ctr, 64 * sizeof(int));
  cudaMalloc(&part, (n / 2048 + 1) * sizeof(float2));
  for (long nn : {n, 4L << 20}) {
    const long nn4 = nn / 4;
    printf("-- n = %ld elements (k_lamb pass-1 structure, 26 B/elem)\n", nn);
    auto run2 = [&](const char* name, auto kern, int ctas) {
      const int gr = sms * ctas;
      for (int r = 0; r < 3; ++r) {
        cudaMemsetAsync(ctr, 0, 4);
        kern<<<gr, 256>>>((float4*)g[r & 1], (float4*)p[r & 1], (float4*)m[r & 1], (float4*)v[r & 1], w[r & 1], nn4, ctr, part);
      }
      cudaEventRecord(e0);
      const int reps = 20;
      for (int r = 0; r < reps; ++r) {
        cudaMemsetAsync(ctr, 0, 4);
        kern<<<gr, 256>>>((float4*)g[r & 1], (float4*)p[r & 1], (float4*)m[r & 1], (float4*)v[r & 1], w[r & 1], nn4, ctr, part);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / reps * 1e-3;
      printf("%-22s %7.1f us/launch  %7.1f GB/s\n", name, t * 1e6, 26.0 * nn / t / 1e9);
    };
    run2("static    nohint c4", k_lamb2<0, 0, 4>, 4);
    run2("static    hint   c4", k_lamb2<0, 1, 4>, 4);
    run2("claim     nohint c4", k_lamb2<1, 0, 4>, 4);
    run2("claim     hint   c4", k_lamb2<1, 1, 4>, 4);
    run2("claim     hint   c3", k_lamb2<1, 1, 3>, 3);
    run2("claim     nohint c3", k_lamb2<1, 0, 3>, 3);
  }
  {
    float* hp;
    cudaMalloc(&hp, 16);
    const float hph[4] = {1e-3f, 10.f, 1000.f, 0.f};
    cudaMemcpy(hp, hph, 16, cudaMemcpyHostToDevice);
    for (long nn : {n, 17842176L, 4L << 20}) {
      sp::LambArgs la{};
      la.hp = hp; la.b1 = 0.9f; la.b2 = 0.999f; la.omb1 = 0.1f; la.omb2 = 0.001f; la.eps = 1e-6f; la.wd = 0.01f;
      auto go = [&](int k) {
        la.g32 = g[k]; la.p = p[k]; la.m = m[k]; la.v = v[k]; la.wire_out = w[k];
        cudaMemsetAsync(ctr, 0, 4);
        k_lamb3<<<sms * 4, 256>>>(la, nn / 4, ctr, part);
      };
      for (int r = 0; r < 3; ++r) go(r & 1);
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r) go(r & 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / 20 * 1e-3;
      printf("k_lamb math, n=%ld     %7.1f us/launch  %7.1f GB/s (26 B/elem)\n", nn, t * 1e6, 26.0 * nn / t / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
