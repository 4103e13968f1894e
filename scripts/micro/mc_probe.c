/* Prints, per visible GPU, whether the driver offers NVSwitch multicast
 * (NVLS, multimem.*) and the shareable-handle types it could be exported
 * with. Build: gcc -O2 mc_probe.c -I/usr/local/cuda/include -lcuda */
#include <cuda.h>
#include <stdio.h>

int main(void) {
  if (cuInit(0) != CUDA_SUCCESS) { printf("cuInit failed\n"); return 1; }
  int n = 0;
  cuDeviceGetCount(&n);
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    cuDeviceGet(&dev, d);
    int mc = -1, fd = -1, fab = -1, vmm = -1;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
    printf("gpu %d: multicast %d posix_fd %d fabric %d vmm %d\n", d, mc, fd, fab, vmm);
  }
  return 0;
}
