// issue rate of tcgen05.mma kind::f16 M=128 for N in {112, 64, 48}, SS and TS (experiment)
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace bsde::tc;
template <int N, int TS>
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < (128 + 112) * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before(); __syncthreads(); tc_after();
  const uint32_t tm = slot;
  if (t == 0) {
    constexpr uint32_t I = idesc_bf16(128, N, false, false);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) gemm_ta(tm, tm + 256, kmaj(sm + 128 * 112 * 2, 112), 7, I, false);
      else gemm(tm, kmaj(sm, 112), kmaj(sm + 128 * 112 * 2, 112), 7, I, false);
    }
    const unsigned long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_before(); __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(tm, 512); }
}
template <int N, int TS> void run() {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<N, TS><<<1, 128, 64 * 1024>>>(200, d);
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d %s: issue %.1f cyc/mma, complete %.1f cyc/mma\n", N, TS ? "TS" : "SS", h[0] / 1400.0, h[1] / 1400.0);
}
int main() {
  run<112, 0>(); run<64, 0>(); run<48, 0>(); run<112, 1>(); run<64, 1>(); run<48, 1>(); run<16, 0>();
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
