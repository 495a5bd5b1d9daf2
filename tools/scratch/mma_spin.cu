// does mbarrier polling by many warps slow tcgen05.mma? (experiment)
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace bsde::tc;
template <int MODE>   // 0: others idle at bar.sync, 1: others spin try_wait on an mbarrier, 2: try_wait + nanosleep
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, bar2;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < (128 + 112) * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (t == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before(); __syncthreads(); tc_after();
  const uint32_t tm = slot;
  if (warp == 8) {
    if (t == 256) {
      constexpr uint32_t I = idesc_bf16(128, 112, false, false);
      const unsigned long long t0 = clock64();
      for (int i = 0; i < iters; ++i) gemm(tm, kmaj(sm, 112), kmaj(sm + 128 * 112 * 2, 112), 7, I, false);
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      const unsigned long long t2 = clock64();
      out[0] = t2 - t0;
      mbar_arrive(&bar2);
    }
  } else if (MODE == 1) {
    mbar_wait(&bar2, 0);
  } else if (MODE == 2) {
    while (!mbar_test(&bar2, 0)) __nanosleep(200);
  }
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(tm, 512); }
}
template <int M> void run(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<M><<<1, 288, 64 * 1024>>>(300, d);
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.1f cyc/mma\n", name, h / 2100.0);
}
int main() {
  run<0>("8 warps at bar.sync");
  run<1>("8 warps polling mbarrier try_wait");
  run<2>("8 warps test_wait + nanosleep(200)");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
