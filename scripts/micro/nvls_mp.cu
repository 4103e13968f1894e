// Multi-process NVSwitch multicast: the setup sequence the round will need
// when every rank is its own process (one GPU each).
//   rank 0: cuMulticastCreate, export the handle as a POSIX fd, pass it to
//           the other ranks over an abstract Unix socket (SCM_RIGHTS)
//   all   : import, cuMulticastAddDevice(own GPU), barrier, cuMemCreate +
//           cuMulticastBindMem, map the unicast and multicast ranges
//   then  : every rank stores its slice through multimem.st; every rank
//           checks that all slices arrived in its own memory.
// Usage: nvls_mp <world>   (forks one process per GPU; prints one line per rank)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvls_mp nvls_mp.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CU(x)                                                                  \
  do {                                                                         \
    CUresult e_ = (x);                                                         \
    if (e_ != CUDA_SUCCESS) {                                                  \
      const char* s_ = nullptr;                                                \
      cuGetErrorString(e_, &s_);                                               \
      std::printf("rank %d: %s failed: %s\n", rank, #x, s_ ? s_ : "?");       \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__global__ void mc_store(float* mc, size_t first, size_t count, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    const float v = base + (float)(i % 1024);
    asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(mc + first + i), "f"(v) : "memory");
  }
}

static int rank = -1;

static sockaddr_un addr_of(const std::string& name) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  a.sun_path[0] = '\0';  // abstract namespace
  std::memcpy(a.sun_path + 1, name.data(), name.size());
  return a;
}

// rank 0 <-> others: fd hand-off and byte-sized barriers over one socket each
static void send_fd(int sock, int fd) {
  char b = 'f';
  iovec io{&b, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
  if (sendmsg(sock, &m, 0) != 1) std::exit(2);
}

static int recv_fd(int sock) {
  char b;
  iovec io{&b, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  if (recvmsg(sock, &m, 0) != 1) std::exit(3);
  int fd = -1;
  std::memcpy(&fd, CMSG_DATA(CMSG_FIRSTHDR(&m)), sizeof(int));
  return fd;
}

static void put(int s) {
  char b = 'b';
  if (write(s, &b, 1) != 1) std::exit(4);
}
static void get(int s) {
  char b;
  if (read(s, &b, 1) != 1) std::exit(5);
}

int main(int argc, char** argv) {
  const int world = argc > 1 ? std::atoi(argv[1]) : 2;
  const std::string name = "sp-nvls-" + std::to_string(getpid());
  // rank 0 listens before forking, so connects cannot race the bind
  int srv = socket(AF_UNIX, SOCK_STREAM, 0);
  sockaddr_un sa = addr_of(name);
  const socklen_t len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + name.size());
  if (bind(srv, (sockaddr*)&sa, len) || listen(srv, world)) return 6;
  rank = 0;
  for (int r = 1; r < world; ++r)
    if (fork() == 0) {
      rank = r;
      break;
    }
  std::vector<int> peers;  // rank 0: one socket per other rank
  int up = -1;             // others: socket to rank 0
  if (rank == 0) {
    for (int r = 1; r < world; ++r) peers.push_back(accept(srv, nullptr, nullptr));
  } else {
    up = socket(AF_UNIX, SOCK_STREAM, 0);
    if (connect(up, (sockaddr*)&sa, len)) return 7;
  }
  auto barrier = [&]() {
    if (rank == 0) {
      for (int s : peers) get(s);
      for (int s : peers) put(s);
    } else {
      put(up);
      get(up);
    }
  };

  CU(cuInit(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, rank));
  CUcontext ctx;
  CU(cuDevicePrimaryCtxRetain(&ctx, dev));
  CU(cuCtxSetCurrent(ctx));
  cudaSetDevice(rank);

  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = 1;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = gran;  // one granule (512 MB on B200)
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  if (rank == 0) {
    CU(cuMulticastCreate(&mc, &mp));
    int fd = -1;
    CU(cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    for (int s : peers) send_fd(s, fd);
    close(fd);
  } else {
    const int fd = recv_fd(up);
    CU(cuMemImportFromShareableHandle(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    close(fd);
  }
  CU(cuMulticastAddDevice(mc, dev));
  barrier();  // every device added before any memory is bound

  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = rank;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  CU(cuMemCreate(&mem, size, &ap, 0));
  CU(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = rank;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcva = 0;
  CU(cuMemAddressReserve(&uc, size, gran, 0, 0));
  CU(cuMemMap(uc, size, 0, mem, 0));
  CU(cuMemSetAccess(uc, size, &acc, 1));
  CU(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CU(cuMemMap(mcva, size, 0, mc, 0));
  CU(cuMemSetAccess(mcva, size, &acc, 1));
  CU(cuMemsetD8(uc, 0, size));
  CU(cuCtxSynchronize());
  barrier();  // every rank bound and mapped

  const size_t n = size / 4, slice = n / world;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mc_store<<<148 * 4, 256>>>(reinterpret_cast<float*>(mcva), rank * slice, slice, 1000.0f * rank);
  cudaEventRecord(e1);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    std::printf("rank %d: kernel failed\n", rank);
    return 8;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  barrier();  // every rank's stores done (each rank synchronized its kernel)

  std::vector<float> h(n);
  CU(cuMemcpyDtoH(h.data(), uc, size));
  long bad = 0;
  for (int r = 0; r < world; ++r)
    for (size_t i = 0; i < slice; i += 4099)
      bad += h[r * slice + i] != 1000.0f * r + (float)(i % 1024);
  std::printf("rank %d: multicast slice of %zu MB in %.1f us (%.0f GB/s out of this GPU), %s\n", rank,
              slice * 4 >> 20, ms * 1e3, slice * 4.0 / (ms * 1e-3) / 1e9, bad ? "MISMATCH" : "all slices ok");
  std::fflush(stdout);
  barrier();
  if (rank == 0)
    for (int r = 1; r < world; ++r) wait(nullptr);
  return bad ? 1 : 0;
}
