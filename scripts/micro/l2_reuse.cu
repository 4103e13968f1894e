// L2 reuse micro-benchmark: write/read a buffer of X MB in pass A, then read it
// again in pass B (separate kernels, back to back). Reports B's bandwidth for
// default caching and with L2::evict_last on pass A / evict_first on pass B.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void passA(float4* __restrict__ a, size_t n, int hint) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v;
    if (hint) {
      asm volatile("{.reg .b64 pol; createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                   "ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], pol;}" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a + i));
      v.x += 1.f;
      asm volatile("{.reg .b64 pol; createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                   "st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, pol;}" :: "l"(a + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
    } else {
      v = a[i]; v.x += 1.f; a[i] = v;
    }
  }
}
__global__ void passB(const float4* __restrict__ a, size_t n, float* out) {
  float s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = a[i]; s += v.x + v.y + v.z + v.w;
  }
  if (s == 123.456f) *out = s;
}
__global__ void flush(float4* f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = make_float4(0,0,0,0);
}
int main() {
  size_t maxb = 512ull << 20;
  float4 *a, *fl; float* out;
  cudaMalloc(&a, maxb); cudaMalloc(&fl, 512ull << 20); cudaMalloc(&out, 4);
  cudaMemset(a, 0, maxb);
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  int mbs[] = {8, 16, 32, 48, 64, 80, 96, 112, 128, 192, 256};
  for (int hint = 0; hint < 2; ++hint)
  for (int mb : mbs) {
    size_t n = ((size_t)mb << 20) / 16;
    float best_a = 1e9, best_b = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      flush<<<148 * 8, 256>>>(fl, (512ull << 20) / 16);
      cudaEventRecord(e0); passA<<<148 * 8, 256>>>(a, n, hint); cudaEventRecord(e1);
      passB<<<148 * 8, 256>>>(a, n, out); cudaEventRecord(e2); cudaEventSynchronize(e2);
      float ta, tb; cudaEventElapsedTime(&ta, e0, e1); cudaEventElapsedTime(&tb, e1, e2);
      best_a = ta < best_a ? ta : best_a; best_b = tb < best_b ? tb : best_b;
    }
    printf("hint=%d %4d MB  passA(rw) %7.1f GB/s  passB(re-read) %7.1f GB/s\n", hint, mb,
           2.0 * mb * 1.048576e-3 / best_a, mb * 1.048576e-3 / best_b);
  }
  return 0;
}
