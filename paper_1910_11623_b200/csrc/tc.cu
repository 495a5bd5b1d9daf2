// tc.cu — tcgen05 (sm_100a) kernels of the bf16 path: bf16 operands in shared
// memory, fp32 accumulators in tensor memory (TMEM), one CTA of 512 threads per SM.
//
// Thread layout: warp w accesses TMEM lanes 32·(w%4)..+31, so a 128-path tile is
// one path per lane and four threads per path; thread group g = w/4 owns the
// 8-column chunks g, g+4, g+8, g+12 of every 112-column accumulator / operand
// image (loads: 4 × tcgen05.ld.32x32b.x8 and one wait).
//
// Data flow of one iteration:
//  k_pack_tc   fp32 master θ -> per-step bf16 operand images W̃1 [Wp×Dp], W̃2 [Wp×Wp],
//              W̃3 [Dp×Wp] with the biases folded into a constant-1 column
//              (W̃1 row w = e_d makes H1[w] = 1; W̃2/W̃3 take b2/b3 in column w).
//  k_fwd_tc    tile-major rollout: a1 Philox ΔW (fused behind the GEMMs), a2 exact
//              fp32 Euler X, a3 three GEMMs per step, a4 Y update, a5 terminal loss
//              and the scalar adjoint ā; stores the bf16 X_n operand images and the
//              fp16 ΔW_n images for the adjoint (tc_fwd.cuh).
//  k_bwd_tc    step-major adjoint a6 with TMEM-resident per-step weight-gradient
//              accumulators (tc_bwd.cuh).
//
// Citations: Eq. 5, Eq. 7, Eq. 6.
#include <cuda_fp16.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace bsde {
namespace tc {

constexpr int NTH = 512;   // threads per CTA (4 per path)
constexpr float kSqrt2 = 1.41421356237309515f;

// ------------------------------------------------------------------ weight packing
template <int D, int W>
__global__ void k_pack_tc(const float* __restrict__ params, uint8_t* __restrict__ out, int N) {
  using Dm = Dims<D, W>;
  const NetDims nd{D, W};
  constexpr int c1 = Dm::Wp * (Dm::Dp / 8), c2 = Dm::Wp * (Dm::Wp / 8), c3 = Dm::Dp * (Dm::Wp / 8);
  constexpr int per_step = c1 + c2 + c3;
  const int64_t total = (int64_t)N * per_step;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / per_step);
    int r = (int)(i - (int64_t)n * per_step);
    const float* P = params + nd.step_base(n);
    uint8_t* img = out + (size_t)n * Dm::WB;
    float v[8];
    int row, chunk, C;
    if (r < c1) {                       // W̃1 [Wp × Dp]: [W1 | b1], row W = e_D
      C = Dm::Dp; row = r / (C / 8); chunk = r - row * (C / 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = chunk * 8 + e;
        float x = 0.0f;
        if (row < W) x = k < D ? P[nd.off_W1() + row * D + k] : (k == D ? P[nd.off_b1() + row] : 0.0f);
        else if (row == W) x = (k == D) ? 1.0f : 0.0f;
        v[e] = x;
      }
    } else if (r < c1 + c2) {           // W̃2 [Wp × Wp]: [W2 | b2], rows >= W zero
      r -= c1; img += Dm::W1B;
      C = Dm::Wp; row = r / (C / 8); chunk = r - row * (C / 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = chunk * 8 + e;
        float x = 0.0f;
        if (row < W) x = k < W ? P[nd.off_W2() + row * W + k] : (k == W ? P[nd.off_b2() + row] : 0.0f);
        v[e] = x;
      }
    } else {                            // W̃3 [Dp × Wp]: [W3 | b3], rows >= D zero
      r -= c1 + c2; img += Dm::W1B + Dm::W2B;
      C = Dm::Wp; row = r / (C / 8); chunk = r - row * (C / 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = chunk * 8 + e;
        float x = 0.0f;
        if (row < D) x = k < W ? P[nd.off_W3() + row * W + k] : (k == W ? P[nd.off_b3() + row] : 0.0f);
        v[e] = x;
      }
    }
    st_chunk(img, row, chunk, C, v);
  }
}

// Column predicates of this thread's chunks c = g + 4i (g = 0..3) that fold at
// compile time after unrolling: column 8(g+4i)+e is < LIM for every g when
// 8(3+4i)+e < LIM, and for no g when 8(4i)+e >= LIM.
__device__ __forceinline__ bool col_lt(int g, int i, int e, int LIM) {
  return (8 * (3 + 4 * i) + e < LIM) || (8 * (4 * i) + e < LIM && 8 * (g + 4 * i) + e < LIM);
}
// chunk g + 4i exists in an image of NC chunks
__device__ __forceinline__ bool chunk_lt(int g, int i, int NC) {
  return (3 + 4 * i < NC) || (4 * i < NC && g + 4 * i < NC);
}

}  // namespace tc
}  // namespace bsde

#include "tc_fwd.cuh"
#include "tc_bwd.cuh"

namespace bsde {
namespace tc {

// ------------------------------------------------------------------ UMMA self-test
// mode 0: D = A·Bᵀ, A [128×112] and B [112×112] K-major (like the forward GEMMs)
// mode 1: D = A·B,  A [128×112] K-major, B [112(k)×112(n)] MN-major view (like G4/G6)
// mode 2: D = Aᵀ·B, A [128(k)×112(m)], B [128(k)×112(n)], both MN-major (like G5/G7/G8);
//         output rows m >= 112 are undefined.
// mode 3: D = A·Bᵀ as mode 0 with A in tensor memory (like the forward's G2/G3).
__global__ void __launch_bounds__(128, 1) k_umma_test(int mode, const float* A, const float* B,
                                                      float* Dout) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int C = 112;
  uint8_t* aimg = sm;
  uint8_t* bimg = sm + 128 * C * 2 + 256;
  uint64_t* bar = reinterpret_cast<uint64_t*>(bimg + 128 * C * 2 + 256);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int t = threadIdx.x, warp = t >> 5;
  const int brows = mode == 2 ? 128 : 112;
  for (int r = 0; r < 128; ++r)
    if (t < C / 8) {
      float v[8];
      for (int e = 0; e < 8; ++e) v[e] = A[r * C + t * 8 + e];
      st_chunk(aimg, r, t, C, v);
    }
  for (int r = 0; r < brows; ++r)
    if (t < C / 8) {
      float v[8];
      for (int e = 0; e < 8; ++e) v[e] = B[r * C + t * 8 + e];
      st_chunk(bimg, r, t, C, v);
    }
  if (t == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(tslot, 256);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = *tslot;
  if (mode == 3) {   // A into TMEM columns [128, 184): thread t = row t, bf16 pairs
    for (int c = 0; c < C / 8; ++c) {
      uint4 u;
      const float* r = A + t * C + 8 * c;
      u.x = pack2(r[0], r[1]); u.y = pack2(r[2], r[3]); u.z = pack2(r[4], r[5]); u.w = pack2(r[6], r[7]);
      tmem_st4(tm + ((uint32_t)(warp * 32) << 16) + 128 + 4 * c, u);
    }
    tmem_wait_st();
    tc_before();
    __syncthreads();
    tc_after();
  }
  if (t == 0) {
    if (mode == 3) gemm_ta(tm, tm + 128, kmaj(bimg, C), C / 16, idesc_bf16(128, 112, false, false), false);
    if (mode == 0) gemm(tm, kmaj(aimg, C), kmaj(bimg, C), C / 16, idesc_bf16(128, 112, false, false), false);
    if (mode == 1) gemm(tm, kmaj(aimg, C), mnmaj(bimg, C), C / 16, idesc_bf16(128, 112, false, true), false);
    if (mode == 2) gemm(tm, mnmaj(aimg, C), mnmaj(bimg, C), 128 / 16, idesc_bf16(128, 112, true, true), false);
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_after();
  for (int c = 0; c < C / 16; ++c) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c * 16, v);
    for (int e = 0; e < 16; ++e) Dout[t * C + c * 16 + e] = v[e];
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 256);
  }
}

__global__ void k_debug_dw_fast(uint32_t it, int n, int64_t m0, int64_t count, int d, float sdt,
                                uint32_t k0, uint32_t k1, float* out) {
  const int nq = (d + 3) >> 2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count * nq) return;
  const int64_t p = i / nq;
  const int q = (int)(i - p * nq);
  const float4 z = dw4_fast((uint32_t)q, (uint32_t)(m0 + p), (uint32_t)n, it, k0, k1, sdt);
  const float zz[4] = {z.x, z.y, z.z, z.w};
  for (int k = 0; k < 4; ++k)
    if (4 * q + k < d) out[p * d + 4 * q + k] = zz[k];
}

// ------------------------------------------------------------------ dispatch
template <int D, int W>
struct Impl {
  using Dm = Dims<D, W>;
  static size_t fwd_smem() { return FwdSmem<D, W>::BYTES; }
  static size_t bwd_smem() { return Dm::WB + 5 * Dm::ACT + 96; }
  static int ntiles(const PassArgs& a) { return (int)((a.B_local + 127) / 128); }
  static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }
  template <bool CPL, bool MULT>
  static cudaError_t fwd_v(const PassArgs& a, cudaStream_t s) {
    // the Philox round 0-2 table when it fits beside the kernel's own 111 KB (N <= ~200)
    using L = FwdSmem<D, W>;
    const size_t with_tab = (size_t)L::TAB + L::tab_bytes(a.N);
    const bool use_tab = !CPL && with_tab <= 227u * 1024u;
    const size_t smem = use_tab ? with_tab : fwd_smem();
    const auto kern = use_tab ? k_fwd_tc<D, W, CPL, MULT, !CPL> : k_fwd_tc<D, W, CPL, MULT, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nt = ntiles(a), sms = sm_count();
    kern<<<nt < sms ? nt : sms, kFwdThreads, smem, s>>>(a, nt);
    return cudaGetLastError();
  }
  static cudaError_t fwd(const PassArgs& a, cudaStream_t s) {
    const bool mult = a.problem == kBlackScholes;
    if (a.cpl > 1) return mult ? fwd_v<true, true>(a, s) : fwd_v<true, false>(a, s);
    return mult ? fwd_v<false, true>(a, s) : fwd_v<false, false>(a, s);
  }
  template <bool NEEDZ>
  static cudaError_t bwd_z(const PassArgs& a, cudaStream_t s) {
    const size_t smem = bwd_smem();
    cudaError_t e = cudaFuncSetAttribute(k_bwd_tc<D, W, NEEDZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nt = ntiles(a), sms = sm_count();
    const int64_t items = (int64_t)nt * a.N;
    k_bwd_tc<D, W, NEEDZ><<<(int)(items < sms ? items : sms), NTH, smem, s>>>(a, nt, items);
    return cudaGetLastError();
  }
  // dZ needs the recomputed Z only where ∂_z f != 0 (HJB)
  static cudaError_t bwd(const PassArgs& a, cudaStream_t s) {
    return a.problem == kHJB ? bwd_z<true>(a, s) : bwd_z<false>(a, s);
  }
  static cudaError_t pack(const PassArgs& a, cudaStream_t s) {
    constexpr int per = Dm::Wp * (Dm::Dp / 8) + Dm::Wp * (Dm::Wp / 8) + Dm::Dp * (Dm::Wp / 8);
    const int64_t total = (int64_t)a.N * per;
    int grid = (int)((total + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_pack_tc<D, W><<<grid, 256, 0, s>>>(a.params, static_cast<uint8_t*>(const_cast<void*>(a.wpack)), a.N);
    return cudaGetLastError();
  }
};

#define BSDE_TC_DIMS(X) X(100, 110) X(10, 20) X(37, 45)

}  // namespace tc

bool tc_supported(int d, int w) {
#define X(D_, W_) if (d == D_ && w == W_) return true;
  BSDE_TC_DIMS(X)
#undef X
  return false;
}

size_t tc_pack_bytes(int d, int w, int N, int) {
#define X(D_, W_) if (d == D_ && w == W_) return (size_t)N * tc::Dims<D_, W_>::WB;
  BSDE_TC_DIMS(X)
#undef X
  return 16;
}

// X_n operand images (bf16) and ΔW_n images (fp16) have the same size
size_t tc_xstore_bytes(int d, int w, int N, int64_t B_local) {
#define X(D_, W_) \
  if (d == D_ && w == W_) return (size_t)N * (size_t)((B_local + 127) / 128) * tc::Dims<D_, W_>::XB;
  BSDE_TC_DIMS(X)
#undef X
  return 16;
}

cudaError_t launch_fwd_tc(const PassArgs& a, cudaStream_t s) {
#define X(D_, W_) if (a.d == D_ && a.w == W_) return tc::Impl<D_, W_>::fwd(a, s);
  BSDE_TC_DIMS(X)
#undef X
  return cudaErrorNotSupported;
}
cudaError_t launch_bwd_tc(const PassArgs& a, cudaStream_t s) {
#define X(D_, W_) if (a.d == D_ && a.w == W_) return tc::Impl<D_, W_>::bwd(a, s);
  BSDE_TC_DIMS(X)
#undef X
  return cudaErrorNotSupported;
}
cudaError_t launch_pack_weights(const PassArgs& a, cudaStream_t s) {
#define X(D_, W_) if (a.d == D_ && a.w == W_) return tc::Impl<D_, W_>::pack(a, s);
  BSDE_TC_DIMS(X)
#undef X
  return cudaErrorNotSupported;
}

cudaError_t launch_umma_test(int mode, const float* A, const float* B, float* D, cudaStream_t s) {
  const size_t smem = 2 * (128 * 112 * 2 + 256) + 64;
  cudaError_t e = cudaFuncSetAttribute(tc::k_umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tc::k_umma_test<<<1, 128, smem, s>>>(mode, A, B, D);
  return cudaGetLastError();
}

cudaError_t launch_debug_dw_fast(uint32_t it, int n, int64_t m0, int64_t count, int d,
                                 float sqrt_dt, uint32_t k0, uint32_t k1, float* out,
                                 cudaStream_t s) {
  const int64_t th = count * ((d + 3) / 4);
  tc::k_debug_dw_fast<<<(int)((th + 255) / 256), 256, 0, s>>>(it, n, m0, count, d, sqrt_dt, k0, k1,
                                                             out);
  return cudaGetLastError();
}

}  // namespace bsde
