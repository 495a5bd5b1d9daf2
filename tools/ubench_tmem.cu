// ubench_tmem.cu — microbenchmarks that size the epilogue / MMA budget of the
// tcgen05 kernels on the B200 (sm_100a):
//   1. tcgen05.ld.32x32b.x{8,16,32,64} throughput vs the number of loading warps
//   2. back-to-back tcgen05.mma kind::f16 M=128 N=112 K=16 (SS) issue rate
//   3. the same MMA stream while 12 other warps read TMEM
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1910_11623_b200/csrc tools/ubench_tmem.cu -o /tmp/ubench && /tmp/ubench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace bsde::tc;

template <int X>
__device__ __forceinline__ void ldx(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ldx<8>(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(a));
}
template <>
__device__ __forceinline__ void ldx<16>(uint32_t a, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(a));
}
template <>
__device__ __forceinline__ void ldx<32>(uint32_t a, uint32_t* r) {
  ldx<16>(a, r);
  ldx<16>(a + 16, r + 16);
}
__device__ __forceinline__ void ldwait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// nw warps load X columns per instruction, `per_wait` loads between waits
template <int X, int PER_WAIT>
__global__ void __launch_bounds__(512, 1) k_ld(int iters, int nw, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nw) {
    for (int i = 0; i < iters; ++i) {
      uint32_t r[X * PER_WAIT];
#pragma unroll
      for (int j = 0; j < PER_WAIT; ++j)
        ldx<X>(tm + (((i * PER_WAIT + j) * X + 128 * (warp >> 2)) & 511), r + X * j);
      ldwait();
#pragma unroll
      for (int j = 0; j < X * PER_WAIT; ++j) acc += r[j];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  if (acc == 12345) sink[threadIdx.x] = acc;
  tc_before();
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(slot, 512); }
}

// thread 0 issues iters GEMMs of 7 MMAs (M=128, N=112, K=16 each) into cols
// [0,112); warps 4..4+ldw-1 read TMEM cols [256, 512) meanwhile.
__global__ void __launch_bounds__(512, 1) k_mma(int iters, int ldw, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  uint8_t* a = sm;
  uint8_t* b = sm + 128 * 112 * 2;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 112) * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = slot;
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  constexpr uint32_t I = idesc_bf16(128, 112, false, false);
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) gemm(tm, kmaj(a, 112), kmaj(b, 112), 7, I, i > 0);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    done = 1;
  } else if (warp >= 4 && warp < 4 + ldw) {
    const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 256;
    int i = 0;
    while (!done) {
      uint32_t r[32];
      ldx<32>(base + ((i * 32 + 64 * (warp >> 2)) & 255), r);
      ldwait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
      ++i;
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  if (acc == 12345) sink[threadIdx.x] = acc;
  tc_before();
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(slot, 512); }
}

int main_old() {
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 4096);
  unsigned long long c;
  const int iters = 2000;
#define RUN_LD(X, PW)                                                                       \
  for (int nw : {4, 8, 16}) {                                                               \
    k_ld<X, PW><<<1, 512>>>(iters, nw, d_out, sink);                                        \
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);                                       \
    const double bytes = (double)nw * 32 * X * PW * 4 * iters;                              \
    printf("ld 32x32b.x%-2d x%d/wait  warps %2d : %8.1f B/cyc  %6.1f cyc/warp-ld\n", X, PW, nw, \
           bytes / c, (double)c / iters / PW * 1.0);                                        \
  }
  RUN_LD(8, 1) RUN_LD(8, 4) RUN_LD(16, 1) RUN_LD(16, 4) RUN_LD(32, 1) RUN_LD(32, 2)
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ldw : {0, 4, 12}) {
    k_mma<<<1, 512, 64 * 1024>>>(iters, ldw, d_out, sink);
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
    printf("mma M128 N112 K16 SS: %.1f cyc/mma with %d TMEM-reading warps\n", (double)c / (iters * 7), ldw);
  }
  // full-chip: 148 CTAs
  k_mma<<<148, 512, 64 * 1024>>>(iters, 0, d_out, sink);
  cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  printf("mma (148 CTAs): %.1f cyc/mma\n", (double)c / (iters * 7));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// ---- epilogue pattern cost: [ld 4x8 + wait] [16 cvt + 4 STS] [fence.proxy.async] [bar]
template <int PARTS>
__global__ void __launch_bounds__(512, 1) k_epi(int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, q = warp & 3, g = warp >> 2;
  const int row = 32 * q + lane;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = slot + ((uint32_t)(32 * q) << 16) + 8u * g;
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float v[32];
    tmem_ld4x8(tm + ((i & 1) ? 128 : 0), v);
    if (PARTS & 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 u = make_uint4(pack2(v[8 * c], v[8 * c + 1]), pack2(v[8 * c + 2], v[8 * c + 3]),
                             pack2(v[8 * c + 4], v[8 * c + 5]), pack2(v[8 * c + 6], v[8 * c + 7]));
        *reinterpret_cast<uint4*>(sm + (row >> 3) * 1792 + (g + 4 * c) * 128 + (row & 7) * 16) = u;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) acc += __float_as_uint(v[c]);
    }
    if (PARTS & 8) {   // + 4 tcgen05.st.32x32b.x4 of the packed chunks and wait::st
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_st4(tm + 256 + 4 * c + 16 * g, make_uint4(__float_as_uint(v[8 * c]), __float_as_uint(v[8 * c + 1]),
                                                       __float_as_uint(v[8 * c + 2]), __float_as_uint(v[8 * c + 3])));
      tmem_wait_st();
    }
    if (PARTS & 2) fence_async_smem();
    if (PARTS & 4) {
      tc_before();
      __syncthreads();
      tc_after();
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (t == 0) *out = t1 - t0;
  if (acc == 12345) sink[t] = acc;
  tc_before();
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(slot, 512); }
}

void run_epi() {
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 4096);
  unsigned long long c;
  const int iters = 1000;
#define EPI(P, name)                                                                   \
  cudaFuncSetAttribute(k_epi<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
  k_epi<P><<<1, 512, 64 * 1024>>>(iters, d_out, sink);                                 \
  cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);                                    \
  printf("epilogue %-34s %7.1f cyc/iter\n", name, (double)c / iters);
  EPI(0, "ld4x8+wait (+sum)")
  EPI(1, "ld + cvt + STS")
  EPI(3, "ld + cvt + STS + fence.proxy.async")
  EPI(5, "ld + cvt + STS + bar")
  EPI(7, "ld + cvt + STS + fence + bar")
  EPI(4, "ld + bar")
  EPI(9, "ld + cvt + STS + tmem st")
  EPI(15, "ld + cvt + STS + tmem st + fence + bar")
}



// ---- latency of one dependent GEMM stage: issue 7 MMAs (M128 N112 K16), commit,
// every thread waits on the mbarrier, barrier; repeated.  mode 1: A from TMEM.
template <int AT>
__global__ void __launch_bounds__(512, 1) k_mma_lat(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  uint8_t* a = sm;
  uint8_t* b = sm + 128 * 112 * 2;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 112) * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = slot;
  constexpr uint32_t I = idesc_bf16(128, 112, false, false);
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) {
      tc_after();
      if (AT) gemm_ta(tm, tm + 256, kmaj(b, 112), 7, I, false);
      else gemm(tm, kmaj(a, 112), kmaj(b, 112), 7, I, false);
      mma_commit(&bar);
    }
    mbar_wait(&bar, i & 1);
    tc_after();
    tc_before();
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  tc_before();
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(slot, 512); }
}

void run_lat() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 8);
  unsigned long long c;
  cudaFuncSetAttribute(k_mma_lat<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_mma_lat<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_mma_lat<0><<<1, 512, 64 * 1024>>>(200, d_out);
  cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  printf("GEMM stage latency (7 MMAs SS + commit + wait + bar): %.1f cyc\n", (double)c / 200);
  k_mma_lat<1><<<1, 512, 64 * 1024>>>(200, d_out);
  cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  printf("GEMM stage latency (7 MMAs A-in-TMEM + commit + wait + bar): %.1f cyc\n", (double)c / 200);
  k_mma_lat<0><<<148, 512, 64 * 1024>>>(200, d_out);
  cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  printf("GEMM stage latency, 148 CTAs: %.1f cyc\n", (double)c / 200);
}

void run_lat();
int main() {
  main_old();
  run_epi();
  run_lat();
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
