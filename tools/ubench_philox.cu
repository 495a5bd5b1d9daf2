// ubench_philox.cu — Philox4x32-10 + Box-Muller throughput per SM on the B200,
// to size the RNG share of the forward pass (SURVEY §8(d) budget).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1910_11623_b200/csrc tools/ubench_philox.cu -o tools/ubench_philox.bin
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace bsde;

__device__ __forceinline__ void mulhilo_split(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi) {
  asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(a), "r"(b));
  asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(b));
}

template <int MODE, int K>
__global__ void __launch_bounds__(512, 1) k_philox(int iters, uint32_t k0, uint32_t k1,
                                                   unsigned long long* out, uint32_t* sink) {
  uint4 c[K];
#pragma unroll
  for (int j = 0; j < K; ++j) c[j] = make_uint4(threadIdx.x + j, blockIdx.x, 7, 9);
  float acc = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint4 x[K];
#pragma unroll
    for (int j = 0; j < K; ++j) x[j] = make_uint4(c[j].x + i, c[j].y, c[j].z, c[j].w);
    uint32_t a0 = k0, a1 = k1;
    // MODE 3: the forward's per-lane share with the round 0-2 table (fwd_philox_table):
    // 16 IMAD.WIDE per block, i.e. eight full rounds, + Box-Muller
#pragma unroll
    for (int r = (MODE == 3 ? 2 : 0); r < 10; ++r) {
      if (r) { a0 += kPhiloxW0; a1 += kPhiloxW1; }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        uint32_t lo0, hi0, lo1, hi1;
        if (MODE == 1) {
          mulhilo_split(kPhiloxM0, x[j].x, lo0, hi0);
          mulhilo_split(kPhiloxM1, x[j].z, lo1, hi1);
        } else {
          lo0 = kPhiloxM0 * x[j].x; hi0 = __umulhi(kPhiloxM0, x[j].x);
          lo1 = kPhiloxM1 * x[j].z; hi1 = __umulhi(kPhiloxM1, x[j].z);
        }
        x[j] = make_uint4(hi1 ^ x[j].y ^ a0, lo1, hi0 ^ x[j].w ^ a1, lo0);
      }
    }
    if (MODE == 2 || MODE == 3) {   // + the fast Box-Muller map of the tcgen05 kernels
#pragma unroll
      for (int j = 0; j < K; ++j) {
        float z0, z1, z2, z3;
        box_muller_fast(x[j].x, x[j].y, 0.06f, z0, z1);
        box_muller_fast(x[j].z, x[j].w, 0.06f, z2, z3);
        acc += (z0 + z1) + (z2 + z3);
      }
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) acc += __uint_as_float((x[j].x ^ x[j].y ^ x[j].z ^ x[j].w) & 0x3fffffffu);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1.2345f) sink[threadIdx.x] = 1;
}

template <int MODE, int K>
void run(const char* name, int threads) {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4096);
  const int iters = 400;
  k_philox<MODE, K><<<148, threads>>>(iters, 1, 2, d, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_philox<MODE, K><<<148, threads>>>(iters, 1, 2, d, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per_sm = (double)threads * K * iters;
  printf("%-28s threads %3d K %d : %6.3f Philox/cyc/SM (%.1f cyc per warp-Philox), %.3f ms\n", name,
         threads, K, per_sm / c, (double)c / (iters * K) * (threads / 32) / 4.0, ms);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<0, 4>("philox (umulhi, default)", 512);
  run<0, 2>("philox (umulhi, default)", 512);
  run<0, 8>("philox (umulhi, default)", 256);
  run<1, 4>("philox (mul.lo + mul.hi)", 512);
  run<2, 4>("philox + box-muller fast", 512);
  run<2, 2>("philox + box-muller fast", 512);
  run<2, 4>("philox + box-muller fast", 256);
  run<2, 8>("philox + box-muller fast", 256);
  run<2, 4>("philox + box-muller fast", 384);
  run<2, 6>("philox + box-muller fast", 384);
  run<2, 8>("philox + box-muller fast", 512);
  run<3, 4>("philox(8 rounds) + box-muller", 512);
  run<3, 3>("philox(8 rounds) + box-muller", 384);
  run<3, 3>("philox(8 rounds) + box-muller", 416);
  run<2, 3>("philox + box-muller fast", 416);
  // (a polynomial sin/cos instead of MUFU measured 0.76 Philox/cyc/SM at 384
  //  and 512 threads: the map is issue-bound, not MUFU-bound)
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
