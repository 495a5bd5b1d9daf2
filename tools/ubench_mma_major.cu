// ubench_mma_major.cu — back-to-back tcgen05.mma kind::f16 M=128 N=112 K=16 (SS)
// issue rate for each operand-major combination of the adjoint's GEMMs: the chain
// GEMMs read K-major operands, the weight-gradient GEMMs G5 / G7 / G8 (sums over the
// 128 paths of a tile) read both operands MN-major from the tile images
// (tc_common.cuh kmaj / mnmaj).  One CTA and 148 CTAs, one issuing thread; then the
// same stream while 12 other warps load (tcgen05.ld.32x32b.x16 + wait) or store
// (tcgen05.st.32x32b.x4 + wait) TMEM columns outside the accumulator, as the
// adjoint's epilogues do while G5 / G7 / G8 run.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1910_11623_b200/csrc tools/ubench_mma_major.cu -o /tmp/ub_major && /tmp/ub_major
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace bsde::tc;

// MODE 0: A, B K-major; 1: A, B MN-major; 2: A MN-major, B K-major; 3: A K-major, B MN-major
// TRAFFIC 0: none; 1: 12 warps load TMEM; 2: 12 warps store TMEM
template <int MODE, int TRAFFIC>
__global__ void __launch_bounds__(512, 1) k_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  uint8_t* a = sm;                    // 128 x 112 image
  uint8_t* b = sm + 128 * 112 * 2;    // 128 x 112 image
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * 128 * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = slot;
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    constexpr bool amn = MODE == 1 || MODE == 2, bmn = MODE == 1 || MODE == 3;
    constexpr uint32_t I = idesc_bf16(128, 112, amn, bmn);
    const Opnd A = amn ? mnmaj(a, 112) : kmaj(a, 112);
    const Opnd B = bmn ? mnmaj(b, 112) : kmaj(b, 112);
    for (int i = 0; i < iters; ++i) gemm(tm, A, B, 7, I, i > 0);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    done = 1;
  } else if (TRAFFIC && warp >= 4) {   // columns 256..511 of the warp's lane quadrant
    const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 256u + 64u * ((warp >> 2) - 1);
    uint32_t acc = 0;
    while (!done) {
      if (TRAFFIC == 1) {
        float v[16];
        tmem_ld16(base, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += __float_as_uint(v[j]);
      } else {
        tmem_st4(base, make_uint4(acc, acc, acc, acc));
        tmem_wait_st();
        ++acc;
      }
    }
    if (acc == 12345u) out[1] = acc;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
  tc_before();
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(slot, 512); }
}

// one elected lane of a converged warp issues (operands warp-uniform)
__device__ __forceinline__ void mma_el(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// issue time of a burst of n MMAs into an idle tensor pipe (the issuing thread's
// clock around the tcgen05.mma instructions only), then their completion
template <bool WARP>
__global__ void __launch_bounds__(128, 1) k_issue(int n, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  uint8_t* a = sm;
  uint8_t* b = sm + 128 * 112 * 2;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * 128 * 112 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = slot;
  if (WARP ? warp == 0 : threadIdx.x == 0) {
    constexpr uint32_t I = idesc_bf16(128, 112, false, false);
    const uint64_t a0 = sdesc(smem_u32(a), 128u, 112u * 16u), b0 = sdesc(smem_u32(b), 128u, 112u * 16u);
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
      if (WARP) mma_el(tm, a0 + (uint64_t)(16 * (k % 7)), b0 + (uint64_t)(16 * (k % 7)), I, k > 0);
      else mma_bf16(tm, a0 + (uint64_t)(16 * (k % 7)), b0 + (uint64_t)(16 * (k % 7)), I, k > 0);
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 0) { tc_after(); tmem_dealloc(slot, 512); }
}

void run_issue() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 16);
  const int smem = 2 * 128 * 112 * 2;
  cudaFuncSetAttribute(k_issue<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_issue<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int w = 0; w < 2; ++w)
    for (int n : {1, 2, 4, 8, 16, 24}) {
      unsigned long long c[2] = {0, 0};
      for (int rep = 0; rep < 2; ++rep) {
        if (w) k_issue<true><<<1, 128, smem>>>(n, d_out);
        else k_issue<false><<<1, 128, smem>>>(n, d_out);
      }
      cudaMemcpy(c, d_out, 16, cudaMemcpyDeviceToHost);
      printf("%s burst of %2d MMAs into an idle pipe: issue %5llu cycles, complete %5llu cycles\n",
             w ? "warp + elect.sync" : "one thread       ", n, c[0], c[1]);
    }
  cudaFree(d_out);
}

template <int MODE, int TRAFFIC>
void run(const char* name) {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 16);
  const int smem = 2 * 128 * 112 * 2;
  cudaFuncSetAttribute(k_rate<MODE, TRAFFIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 400;
  for (int ctas : {1, 148}) {
    k_rate<MODE, TRAFFIC><<<ctas, 512, smem>>>(iters, d_out);
    unsigned long long c = 0;
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %-12s %3d CTA: %.1f cycles per MMA\n", name,
           TRAFFIC == 0 ? "" : TRAFFIC == 1 ? "+ 12w ld" : "+ 12w st", ctas, (double)c / (iters * 7));
  }
  cudaFree(d_out);
}

int main() {
  run_issue();
  run<0, 0>("A K-major, B K-major");
  run<1, 0>("A MN-major, B MN-major");
  run<2, 0>("A MN-major, B K-major");
  run<3, 0>("A K-major, B MN-major");
  run<0, 1>("A K-major, B K-major");
  run<1, 1>("A MN-major, B MN-major");
  run<0, 2>("A K-major, B K-major");
  run<1, 2>("A MN-major, B MN-major");
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
