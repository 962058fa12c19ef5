// Does this node support NVLink SHARP multicast objects (NVLS)?
//   nvcc -o tools/nvls_check tools/nvls_check.cu -lcuda
#include <cstdio>
#include <cuda.h>
int main() {
  if (cuInit(0) != CUDA_SUCCESS) { printf("cuInit failed\n"); return 1; }
  int n = 0;
  cuDeviceGetCount(&n);
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    cuDeviceGet(&dev, d);
    int mc = -1, fabric = -1, posix = -1;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
    printf("{\"device\": %d, \"multicast\": %d, \"fabric_handles\": %d, \"posix_fd_handles\": %d}\n", d, mc, fabric, posix);
  }
  if (n > 0) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = n;
    prop.size = 2 << 20;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CUresult r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("{\"multicast_granularity\": %zu, \"rc\": %d}\n", gran, (int)r);
    CUmemGenericAllocationHandle h;
    r = cuMulticastCreate(&h, &prop);
    printf("{\"multicast_create_rc\": %d}\n", (int)r);
  }
  return 0;
}
