// D / A column-offset legality of tcgen05.mma on sm_100a (experiment)
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace bsde::tc;
__global__ void k(int doff, int aoff, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < (128 + 112) * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before(); __syncthreads(); tc_after();
  const uint32_t tm = slot;
  if (aoff >= 0) {
    for (int c = 0; c < 14; ++c) tmem_st4(tm + ((uint32_t)(warp * 32) << 16) + aoff + 4 * c, make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u));
    tmem_wait_st();
  }
  tc_before(); __syncthreads(); tc_after();
  if (t == 0) {
    constexpr uint32_t I = idesc_bf16(128, 112, false, false);
    if (aoff >= 0) gemm_ta(tm + doff, tm + aoff, kmaj(sm + 128 * 112 * 2, 112), 7, I, false);
    else gemm(tm + doff, kmaj(sm, 112), kmaj(sm + 128 * 112 * 2, 112), 7, I, false);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_after();
  float v[16];
  tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + doff + 96, v);
  out[t] = v[15];
  tc_before(); __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(tm, 512); }
}
int main() {
  float* d; cudaMalloc(&d, 512);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int cases[][2] = {{0, -1}, {176, -1}, {288, -1}, {400, -1}, {16, -1}, {0, 112}, {0, 120}, {176, 112}};
  for (auto& c : cases) {
    k<<<1, 128, 64 * 1024>>>(c[0], c[1], d);
    cudaError_t e = cudaDeviceSynchronize();
    float h = -1; if (e == cudaSuccess) cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("D col %3d A col %4d: %s value %.1f (expect 112)\n", c[0], c[1], cudaGetErrorString(e), h);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
