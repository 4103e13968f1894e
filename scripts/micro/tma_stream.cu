// tma_stream.cu — can LAMB pass 1 stream at HBM speed with its loads
// staged by bulk async copies (cp.async.bulk + mbarrier) instead of
// per-thread loads held in registers? Pass 1 of the fused fp16 round (read
// g fp32, p, m, v; write m', v', fp16 wire), chunks claimed from one
// counter, the CTA's thread 0 issuing the copies S - 1 chunks ahead.
// Compared with k_lamb3 of stream_bw.cu (same math, register loads).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2106_10207_b200/csrc/cuda -o scripts/micro/tma_stream scripts/micro/tma_stream.cu
#include <cstdint>
#include <cstdio>

#include "sp_kernels.cuh"

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int THREADS, int STAGES, int CTAS>
__global__ void __launch_bounds__(THREADS, CTAS) k_tma(sp::LambArgs a, long nchunks, int* ctr, float2* part) {
  constexpr int CH = THREADS * 4;           // elements per chunk: one float4 per thread
  constexpr unsigned ABYTES = CH * 4;       // bytes of one array's chunk
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[STAGES];
  __shared__ long s_item[STAGES];
  __shared__ float red_p[THREADS / 32], red_u[THREADS / 32];
  float4* stage = reinterpret_cast<float4*>(smem);  // [STAGES][4][THREADS] float4: g, p, m, v
  const int tid = threadIdx.x;
  const sp::LambScalars s{a.hp[0], a.hp[1], a.hp[2]};
  long pend = 0;
  auto issue = [&](int st, long c) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&full[st], 4 * ABYTES);
    float4* b = stage + (size_t)st * 4 * THREADS;
    const long e = c * CH;
    bulk_g2s(b + 0 * THREADS, a.g32 + e, ABYTES, &full[st]);
    bulk_g2s(b + 1 * THREADS, a.p + e, ABYTES, &full[st]);
    bulk_g2s(b + 2 * THREADS, a.m + e, ABYTES, &full[st]);
    bulk_g2s(b + 3 * THREADS, a.v + e, ABYTES, &full[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < STAGES; ++st) {
      const long c = atomicAdd(ctr, 1);
      s_item[st] = c;
      if (c < nchunks) issue(st, c);
    }
    pend = atomicAdd(ctr, 1);
  }
  __syncthreads();
  for (int it = 0;; ++it) {
    const int st = it % STAGES;
    const long c = s_item[st];
    if (c >= nchunks) break;
    while (!mbar_try_wait(&full[st], (it / STAGES) & 1)) {
    }
    const float4* b = stage + (size_t)st * 4 * THREADS;
    const int64_t i = c * CH + 4 * tid;
    const sp::GradRaw gr{b[tid], {}, 0, 0.0f};
    const float4 g = sp::grad_finish<SP_WIRE_FP16, true>(a, i, gr);
    float4 p = b[THREADS + tid], m = b[2 * THREADS + tid], v = b[3 * THREADS + tid], u;
    sp::lamb_moments(a, s, g.x, p.x, m.x, v.x, u.x);
    sp::lamb_moments(a, s, g.y, p.y, m.y, v.y, u.y);
    sp::lamb_moments(a, s, g.z, p.z, m.z, v.z, u.z);
    sp::lamb_moments(a, s, g.w, p.w, m.w, v.w, u.w);
    *reinterpret_cast<float4*>(a.m + i) = m;
    *reinterpret_cast<float4*>(a.v + i) = v;
    float pp = 0.f, uu = 0.f;
    pp = __fmaf_rn(p.x, p.x, pp); pp = __fmaf_rn(p.y, p.y, pp);
    pp = __fmaf_rn(p.z, p.z, pp); pp = __fmaf_rn(p.w, p.w, pp);
    uu = __fmaf_rn(u.x, u.x, uu); uu = __fmaf_rn(u.y, u.y, uu);
    uu = __fmaf_rn(u.z, u.z, uu); uu = __fmaf_rn(u.w, u.w, uu);
    pp = sp::warp_sum(pp);
    uu = sp::warp_sum(uu);
    if ((tid & 31) == 0) {
      red_p[tid >> 5] = pp;
      red_u[tid >> 5] = uu;
    }
    __syncthreads();
    if (tid == 0) {
      float x = 0.f, y = 0.f;
      for (int w = 0; w < THREADS / 32; ++w) {
        x += red_p[w];
        y += red_u[w];
      }
      part[c] = make_float2(x, y);
      const long c2 = pend;
      s_item[st] = c2;
      if (c2 < nchunks) issue(st, c2);
      pend = atomicAdd(ctr, 1);
    }
  }
}

int main() {
  const long nmax = 64L << 20;
  float *g[2], *p[2], *m[2], *v[2];
  uint2* w[2];
  for (int k = 0; k < 2; ++k) {
    cudaMalloc(&g[k], nmax * 4); cudaMalloc(&p[k], nmax * 4); cudaMalloc(&m[k], nmax * 4); cudaMalloc(&v[k], nmax * 4);
    cudaMalloc(&w[k], nmax * 2);
    cudaMemset(g[k], 0, nmax * 4); cudaMemset(p[k], 0, nmax * 4);
    cudaMemset(m[k], 0, nmax * 4); cudaMemset(v[k], 0, nmax * 4);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* ctr;
  float2* part;
  cudaMalloc(&ctr, 64);
  cudaMalloc(&part, (nmax / 1024 + 1) * sizeof(float2));
  float* hp;
  cudaMalloc(&hp, 16);
  const float hph[4] = {1e-3f, 10.f, 1000.f, 0.f};
  cudaMemcpy(hp, hph, 16, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto bench = [&](const char* name, auto kern, int threads, int stages, int ctas, long n) {
    const size_t dyn = (size_t)stages * 4 * threads * 16;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    const long nch = n / (threads * 4);
    sp::LambArgs la{};
    la.hp = hp; la.b1 = 0.9f; la.b2 = 0.999f; la.omb1 = 0.1f; la.omb2 = 0.001f; la.eps = 1e-6f; la.wd = 0.01f;
    auto go = [&](int k) {
      la.g32 = g[k]; la.p = p[k]; la.m = m[k]; la.v = v[k]; la.wire_out = w[k];
      cudaMemsetAsync(ctr, 0, 4);
      kern<<<sms * ctas, threads, dyn>>>(la, nch, ctr, part);
    };
    for (int r = 0; r < 3; ++r) go(r & 1);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) go(r & 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms / 20 * 1e-3;
    const long ne = nch * threads * 4;
    printf("%-26s n=%9ld %7.1f us/launch %7.1f GB/s (26 B/elem)  %s\n", name, ne, t * 1e6, 26.0 * ne / t / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (long n : {64L << 20, 17842176L, 4L << 20}) {
    bench("tma t512 s4 c1", k_tma<512, 4, 1>, 512, 4, 1, n);
    bench("tma t512 s3 c1", k_tma<512, 3, 1>, 512, 3, 1, n);
    bench("tma t256 s3 c2", k_tma<256, 3, 2>, 256, 3, 2, n);
    bench("tma t256 s4 c2", k_tma<256, 4, 2>, 256, 4, 2, n);
    bench("tma t128 s4 c4", k_tma<128, 4, 4>, 128, 4, 4, n);
    bench("tma t1024 s3 c1", k_tma<1024, 3, 1>, 1024, 3, 1, n);
    bench("tma t256 s6 c2", k_tma<256, 6, 2>, 256, 6, 2, n);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
