// probe_multicast.cu — does this B200 expose NVLink SHARP multicast objects (the
// multimem / NVLS path NEXT-4 would use)?  nvcc tools/probe_multicast.cu -lcuda
#include <cstdio>
#include <cuda.h>
int main() {
  cuInit(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  int mc = -1, fab = -1, vmm = -1;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported %d vmm %d fabric_handle %d\n", mc, vmm, fab);
  if (mc == 1) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.size = 2 << 20;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CUresult r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("granularity %zu (rc %d)\n", gran, (int)r);
    CUmemGenericAllocationHandle h;
    r = cuMulticastCreate(&h, &prop);
    printf("cuMulticastCreate(1 device) rc %d\n", (int)r);
    if (r == CUDA_SUCCESS) {
      r = cuMulticastAddDevice(h, dev);
      printf("cuMulticastAddDevice rc %d\n", (int)r);
    }
  }
  return 0;
}
