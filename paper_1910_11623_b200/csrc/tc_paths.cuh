// tc_paths.cuh — the Brownian paths of one iteration for the tcgen05 kernels
// (SURVEY §8(a) rows a1, a2): for every (tile, step n) the increments
// ΔW_n = √Δt·z (Philox4x32-10 + Box-Muller, R8) and the Euler states
// X_{n+1} = X_n + √2 ΔW_n (Eq. 5) in exact fp32 registers.
// Outputs, both in the UMMA operand-image layout of one 128-path tile:
//   X_n  as bf16 [128 × Dp] with the constant-1 column d (the forward and adjoint
//        GEMM operand, bulk-copied straight into shared memory),
//   ΔW_n as fp16 [128 × Dp] (relative rounding 2^-12, well inside the bf16
//        operand rounding of R17; consumed by the Y update and dZ),
// and |X_N|² (fp32) per path for the terminal condition.  The paths do not depend
// on θ, so this is one pass shared by the forward and the adjoint kernel.
// Thread layout as in the GEMM kernels: 4 threads per path, each owning the
// 8-column chunks g, g+4, g+8, g+12 (16-byte stores of both images).
#pragma once

namespace bsde {
namespace tc {

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int D, int W>
__global__ void __launch_bounds__(NTH, 1) k_paths_tc(PassArgs a, int ntiles) {
  using Dm = Dims<D, W>;
  constexpr int Dp = Dm::Dp;
  __shared__ float red[4][128];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int q = warp & 3, g = warp >> 2;
  const int row = 32 * q + lane;
  uint8_t* xst = static_cast<uint8_t*>(a.xpack);
  uint8_t* dst = static_cast<uint8_t*>(a.dwpack);
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t mloc = (int64_t)tile * 128 + row;
    const uint32_t mg = (uint32_t)(a.m0 + mloc);
    float X[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) X[i] = a.x0;
    for (int n = 0; n < a.N; ++n) {
      const size_t img = ((size_t)n * ntiles + tile) * Dm::XB;
      const DwGen gen{mg, (uint32_t)n, it, a.k0, a.k1, a.sqrt_dt, g};
      float dw[32];
      gen.run<D, 0, 4>(dw);
      gen.run<D, 4, 8>(dw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (chunk_lt(g, i, Dp / 8)) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = 8 * (g + 4 * i) + e;
            v[e] = col_lt(g, i, e, D) ? X[8 * i + e] : (j == D ? 1.0f : 0.0f);
          }
          st_chunk(xst + img, row, g + 4 * i, Dp, v);   // X_n operand image (bf16)
          uint4 u;
          u.x = pack_h2(dw[8 * i + 0], dw[8 * i + 1]);
          u.y = pack_h2(dw[8 * i + 2], dw[8 * i + 3]);
          u.z = pack_h2(dw[8 * i + 4], dw[8 * i + 5]);
          u.w = pack_h2(dw[8 * i + 6], dw[8 * i + 7]);
          *reinterpret_cast<uint4*>(dst + img + (row >> 3) * (Dp * 16) + (g + 4 * i) * 128 +
                                    (row & 7) * 16) = u;                 // ΔW_n image (fp16)
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) X[i] = fmaf(kSqrt2, dw[i], X[i]);       // a2 (exact fp32)
    }
    float sx = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (col_lt(g, i, e, D)) sx = fmaf(X[8 * i + e], X[8 * i + e], sx);
    red[g][row] = sx;
    __syncthreads();
    if (g == 0 && mloc < a.B_local)
      a.xn2[mloc] = (red[0][row] + red[1][row]) + (red[2][row] + red[3][row]);
    __syncthreads();
  }
}

// ΔW chunk of this thread from the fp16 image (16 bytes -> 8 floats)
__device__ __forceinline__ void unpack_dw(const uint4& u, float* v) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}

}  // namespace tc
}  // namespace bsde
