// NVLink P2P bandwidth patterns (single process, peer access):
//  write: every GPU pushes `bytes` to every other GPU (all-to-all), kernel stores
//  read:  every GPU pulls `bytes` from every other GPU, kernel loads
//  ce:    cudaMemcpyPeerAsync all-to-all (copy engines)
// Reports per-GPU per-direction GB/s = (ngpu-1)*bytes / time.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int UNROLL>
__global__ void push(int4* const* dst, const int4* src, size_t n16, int ndst) {
  // each CTA streams its slice of src to all destinations
  for (int d = 0; d < ndst; ++d) {
    int4* out = dst[d];
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * UNROLL; i < n16;
         i += (size_t)gridDim.x * blockDim.x * UNROLL) {
      int4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = src[i + u];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) out[i + u] = v[u];
    }
  }
}
template <int UNROLL>
__global__ void pull(int4* dst, int4* const* src, size_t n16, int nsrc) {
  for (int d = 0; d < nsrc; ++d) {
    const int4* in = src[d];
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * UNROLL; i < n16;
         i += (size_t)gridDim.x * blockDim.x * UNROLL) {
      int4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = __ldcg(in + i + u);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) dst[i + u] = v[u];
    }
  }
}
// interleaved destinations: consecutive iterations go to different peers
template <int UNROLL>
__global__ void push_interleaved(int4* const* dst, const int4* src, size_t n16, int ndst) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * UNROLL;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * UNROLL; i < n16; i += stride) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = src[i + u];
    for (int d = 0; d < ndst; ++d) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) dst[d][i + u] = v[u];
    }
  }
}

// every warp streams to destination (warp % ndst): all destinations at once
__global__ void push_spread(int4* const* dst, const int4* src, size_t n16, int ndst) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int d = warp % ndst;
  const int wpd = nwarps / ndst;  // warps per destination
  const int w = warp / ndst;
  int4* out = dst[d];
  for (size_t i = (size_t)w * 32 + lane; i < n16; i += (size_t)wpd * 32) out[i] = src[i];
}

int main(int argc, char** argv) {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  size_t bytes = (argc > 1 ? atol(argv[1]) : 16) << 20;  // per pair
  size_t n16 = bytes / 16;
  printf("gpus=%d bytes/pair=%zu MB\n", ng, bytes >> 20);
  for (int a = 0; a < ng; ++a) { CK(cudaSetDevice(a)); for (int b = 0; b < ng; ++b) if (a != b) cudaDeviceEnablePeerAccess(b, 0); }
  std::vector<int4*> src(ng), inbox(ng);  // inbox[g]: (ng) slots of bytes
  std::vector<int4**> dtab(ng), stab(ng);
  std::vector<cudaStream_t> st(ng);
  std::vector<cudaEvent_t> e0(ng), e1(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&inbox[g], bytes * ng));
    CK(cudaMemset(src[g], 1, bytes));
    CK(cudaStreamCreate(&st[g]));
    cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]);
  }
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    std::vector<int4*> d, s;
    for (int dd = 1; dd < ng; ++dd) { int k = (g + dd) % ng; d.push_back(inbox[k] + (size_t)g * n16); s.push_back(src[k]); }
    CK(cudaMalloc(&dtab[g], sizeof(int4*) * 8)); CK(cudaMalloc(&stab[g], sizeof(int4*) * 8));
    CK(cudaMemcpy(dtab[g], d.data(), sizeof(int4*) * d.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(stab[g], s.data(), sizeof(int4*) * s.size(), cudaMemcpyHostToDevice));
  }
  int active = ng;  // GPUs 0..active-1 launch
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      for (int g = 0; g < ng; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); }
      for (int g = 0; g < active; ++g) { cudaSetDevice(g); cudaEventRecord(e0[g], st[g]); launch(g); cudaEventRecord(e1[g], st[g]); }
      float worst = 0;
      for (int g = 0; g < active; ++g) { cudaSetDevice(g); cudaEventSynchronize(e1[g]); float ms; cudaEventElapsedTime(&ms, e0[g], e1[g]); worst = ms > worst ? ms : worst; }
      if (rep > 0 && worst < best) best = worst;
    }
    CK(cudaGetLastError());
    printf("%-34s %8.1f us  %7.1f GB/s per GPU per direction\n", name, best * 1e3, (ng - 1) * bytes / (best * 1e-3) / 1e9);
  };
  const int sms = 148;
  for (int ai : {1, 2, 4}) { active = ai > ng ? ng : ai;
    printf("-- %d GPU(s) sending concurrently\n", active);
    for (int gr : {2 * sms, 8 * sms}) {
      char nm[64];
      snprintf(nm, 64, "push u1 grid=%d", gr);
      run(nm, [&](int g) { push<1><<<gr, 256, 0, st[g]>>>(dtab[g], src[g], n16, ng - 1); });
      snprintf(nm, 64, "pull u1 grid=%d", gr);
      run(nm, [&](int g) { pull<1><<<gr, 256, 0, st[g]>>>(inbox[g], stab[g], n16, ng - 1); });
    }
    run("push_spread grid=1184", [&](int g) { push_spread<<<8 * sms, 256, 0, st[g]>>>(dtab[g], src[g], n16, ng - 1); });
    run("copy engine memcpyPeerAsync", [&](int g) {
      for (int dd = 1; dd < ng; ++dd) { int k = (g + dd) % ng; cudaMemcpyPeerAsync(inbox[k] + (size_t)g * n16, k, src[g], g, bytes, st[g]); }
    });
  }
  active = ng;
  int grids[] = {2 * sms};
  for (int gr : grids) {
    char nm[64];
    snprintf(nm, 64, "push u1 grid=%d", gr);
    run(nm, [&](int g) { push<1><<<gr, 256, 0, st[g]>>>(dtab[g], src[g], n16, ng - 1); });
    snprintf(nm, 64, "push u4 grid=%d", gr);
    run(nm, [&](int g) { push<4><<<gr, 256, 0, st[g]>>>(dtab[g], src[g], n16, ng - 1); });
    snprintf(nm, 64, "push_interleaved u2 grid=%d", gr);
    run(nm, [&](int g) { push_interleaved<2><<<gr, 256, 0, st[g]>>>(dtab[g], src[g], n16, ng - 1); });
    snprintf(nm, 64, "pull u1 grid=%d", gr);
    run(nm, [&](int g) { pull<1><<<gr, 256, 0, st[g]>>>(inbox[g], stab[g], n16, ng - 1); });
    snprintf(nm, 64, "pull u4 grid=%d", gr);
    run(nm, [&](int g) { pull<4><<<gr, 256, 0, st[g]>>>(inbox[g], stab[g], n16, ng - 1); });
  }
  run("copy engine memcpyPeerAsync", [&](int g) {
    for (int k = 0; k < ng; ++k) if (k != g) cudaMemcpyPeerAsync(inbox[k] + (size_t)g * n16, k, src[g], g, bytes, st[g]);
  });
  return 0;
}
