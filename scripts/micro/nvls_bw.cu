// NVSwitch multicast (NVLS) vs unicast peer stores for the round's all-gather
// pattern, one process driving every visible GPU (no handle passing needed).
//   unicast : GPU g stores its 1/N slice into every other GPU's buffer (the
//             sharded parameter push / replicated average push of the round)
//   multicast: GPU g stores its slice once through the multicast mapping
//             (multimem.st), the switch replicates it to every GPU
// Also: one writer (GPU 0) sending a whole buffer to everyone (the dominant
// owner of a non-uniform split). Reports per-GPU per-direction GB/s on the
// receive side. Every driver call is checked before any kernel runs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvls_bw nvls_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CU(x)                                                              \
  do {                                                                     \
    CUresult e_ = (x);                                                     \
    if (e_ != CUDA_SUCCESS) {                                              \
      const char* s_ = nullptr;                                            \
      cuGetErrorString(e_, &s_);                                           \
      std::printf("%s failed: %s\n", #x, s_ ? s_ : "?");                   \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)
#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::printf("%s failed: %s\n", #x, cudaGetErrorString(e_));          \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

__global__ void mc_store(float4* mc, const float4* src, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  }
}

struct Dst {
  float4* p[8];
  int n;
};

__global__ void uc_store(Dst d, const float4* src, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    for (int k = 0; k < d.n; ++k) d.p[k][i] = v;
  }
}

int main(int argc, char** argv) {
  const size_t want = (argc > 1 ? std::atol(argv[1]) : 64) << 20;  // bytes per GPU buffer
  CU(cuInit(0));
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) {
    std::printf("needs >= 2 GPUs\n");
    return 0;
  }
  if (ng > 8) ng = 8;
  std::vector<CUdevice> dev(ng);
  std::vector<CUcontext> ctx(ng);
  for (int g = 0; g < ng; ++g) {
    CU(cuDeviceGet(&dev[g], g));
    int mc = 0;
    CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[g]));
    if (!mc) {
      std::printf("gpu %d: no multicast support\n", g);
      return 0;
    }
    CU(cuDevicePrimaryCtxRetain(&ctx[g], dev[g]));
  }
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)ng;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = want;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (want + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int g = 0; g < ng; ++g) CU(cuMulticastAddDevice(mc, dev[g]));

  std::vector<CUmemGenericAllocationHandle> mem(ng);
  std::vector<CUdeviceptr> uc(ng), mcva(ng);
  std::vector<CUmemAccessDesc> acc(ng);
  for (int g = 0; g < ng; ++g) {
    acc[g].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[g].location.id = g;
    acc[g].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  for (int g = 0; g < ng; ++g) {
    CU(cuCtxSetCurrent(ctx[g]));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ugran = 0;
    CU(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    if (size % ugran) {
      std::printf("size %zu not a multiple of the allocation granularity %zu\n", size, ugran);
      return 1;
    }
    CU(cuMemCreate(&mem[g], size, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mem[g], 0, size, 0));
  }
  for (int g = 0; g < ng; ++g) {
    CU(cuCtxSetCurrent(ctx[g]));
    CU(cuMemAddressReserve(&uc[g], size, gran, 0, 0));
    CU(cuMemMap(uc[g], size, 0, mem[g], 0));
    CU(cuMemSetAccess(uc[g], size, acc.data(), ng));  // every GPU may store into it
    CU(cuMemAddressReserve(&mcva[g], size, gran, 0, 0));
    CU(cuMemMap(mcva[g], size, 0, mc, 0));
    CU(cuMemSetAccess(mcva[g], size, &acc[g], 1));
  }
  for (int a = 0; a < ng; ++a) {
    CK(cudaSetDevice(a));
    for (int b = 0; b < ng; ++b)
      if (a != b) {
        cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      }
  }
  std::vector<float4*> src(ng);
  std::vector<cudaStream_t> st(ng);
  std::vector<cudaEvent_t> e0(ng), e1(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&src[g], size));
    std::vector<float> h(size / 4);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(g * 1000003 + i % 977);
    CK(cudaMemcpy(src[g], h.data(), size, cudaMemcpyHostToDevice));
    CK(cudaMemset(reinterpret_cast<void*>(uc[g]), 0, size));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  const size_t n16 = size / 16, slice = n16 / ng;
  const int grid = 148 * 4, block = 256;
  auto timed = [&](const char* name, int writers, size_t recv_bytes, auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < writers; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        launch(g);
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0.0f;
      for (int g = 0; g < writers; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        worst = ms > worst ? ms : worst;
      }
      CK(cudaGetLastError());
      if (rep > 0 && worst < best) best = worst;
    }
    std::printf("%-44s %9.1f us  %7.1f GB/s received per GPU\n", name, best * 1e3,
                recv_bytes / (best * 1e-3) / 1e9);
  };
  std::printf("gpus=%d buffer=%zu MB (gran %zu KB)\n", ng, size >> 20, gran >> 10);
  // all-gather: every GPU writes its slice to all; each GPU receives (ng-1) slices
  const size_t ag_recv = (size_t)(ng - 1) * slice * 16;
  timed("all-gather unicast (stores to ng-1 peers)", ng, ag_recv, [&](int g) {
    Dst d{};
    for (int k = 1; k < ng; ++k) d.p[d.n++] = reinterpret_cast<float4*>(uc[(g + k) % ng]) + g * slice;
    uc_store<<<grid, block, 0, st[g]>>>(d, src[g] + g * slice, slice);
  });
  timed("all-gather multicast (multimem.st)", ng, ag_recv, [&](int g) {
    mc_store<<<grid, block, 0, st[g]>>>(reinterpret_cast<float4*>(mcva[g]) + g * slice,
                                        src[g] + g * slice, slice);
  });
  // dominant owner: GPU 0 sends the whole buffer to everyone
  timed("one owner -> all, unicast", 1, size, [&](int g) {
    Dst d{};
    for (int k = 1; k < ng; ++k) d.p[d.n++] = reinterpret_cast<float4*>(uc[k]);
    uc_store<<<grid, block, 0, st[g]>>>(d, src[0], n16);
  });
  timed("one owner -> all, multicast", 1, size, [&](int g) {
    mc_store<<<grid, block, 0, st[g]>>>(reinterpret_cast<float4*>(mcva[0]), src[0], n16);
  });
  // check: after the last run every GPU holds GPU 0's buffer
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    float got[4], want4[4];
    CK(cudaMemcpy(got, reinterpret_cast<void*>(uc[g] + 4096), 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(want4, reinterpret_cast<char*>(src[0]) + 4096, 16, cudaMemcpyDeviceToHost));
    std::printf("gpu %d check: %s\n", g, (got[0] == want4[0] && got[3] == want4[3]) ? "ok" : "MISMATCH");
  }
  return 0;
}
