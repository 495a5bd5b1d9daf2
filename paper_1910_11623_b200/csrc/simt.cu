// simt.cu — fp32 CUDA-core forward and adjoint kernels.
//
// The exact-fp32 path: configs with fp32 operands at small width (config 1),
// any d, w too large for the tcgen05 tiles, and the on-device cross-check of
// the tensor-core kernels.  Same data flow as the tcgen05 path:
//
//  k_fwd_simt  one CTA = TP paths, all N steps ("tile-major"): a1 Philox ΔW,
//              a2 Euler X, a3 Z-net, a4 Y update, a5 terminal loss; stores X_n
//              (for the adjoint) and, for Allen-Cahn, Y_n; ends with the ā
//              recursion (a6 scalar part) and dY0.
//  k_bwd_simt  one CTA = (step n, TP paths) ("step-major"): reloads X_n,
//              regenerates ΔW_n, recomputes the net, and back-propagates
//              dZ_n = ā_{n+1}(ΔW_n - Δt ∂_z f) through it (a6), accumulating
//              the per-step weight gradients with fp32 atomics.
//
// Citations: Eq. 5, Eq. 7, Eq. 6.
#include "kernels.cuh"

namespace bsde {
namespace {

constexpr int TP = 32;    // paths per CTA
constexpr int NT = 256;   // threads per CTA
constexpr float kSqrt2 = 1.41421356237309515f;

__host__ __device__ inline int odd_ld(int K) { return (K & 1) ? K + 2 : K + 1; }

// Ws[j*ld + k] = W[j*K + k]  (rows of a [nout][K] row-major matrix, odd pitch)
__device__ void stage_rows(float* Ws, int ld, const float* __restrict__ W, int nout, int K) {
  for (int idx = threadIdx.x; idx < nout * K; idx += NT) {
    const int j = idx / K, k = idx - j * K;
    Ws[j * ld + k] = __ldg(W + idx);
  }
}
__device__ void stage_copy(float* Ws, const float* __restrict__ W, int count) {
  for (int idx = threadIdx.x; idx < count; idx += NT) Ws[idx] = __ldg(W + idx);
}

// out[p][j] = Σ_k A[p][k] · (TRANS ? Ws[j][k] : Ws[k][j]) for p < TP, j < nout;
// epi(p, j, acc).  A row reads are warp broadcasts; Ws reads are unit-stride in
// j (odd pitch for TRANS), hence bank-conflict free.
template <bool TRANS, typename Epi>
__device__ __forceinline__ void gemm_tp(const float* A, int lda, int K, const float* Ws,
                                        int ldw, int nout, Epi epi) {
  const int jt = min(128, (nout + 31) & ~31);
  const int groups = NT / jt;
  const int g = threadIdx.x / jt;
  const int jl = threadIdx.x - g * jt;
  const int rows = TP / groups;
  if (g >= groups) return;
  for (int j0 = 0; j0 < nout; j0 += jt) {
    const int j = j0 + jl;
    if (j >= nout) continue;
    float acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = 0.0f;
    for (int k = 0; k < K; ++k) {
      const float wv = TRANS ? Ws[j * ldw + k] : Ws[k * ldw + j];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < rows) acc[r] = fmaf(A[(g + r * groups) * lda + k], wv, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r < rows) epi(g + r * groups, j, acc[r]);
  }
}

// G[i][j] += Σ_p L[p][i] R[p][j];  gb[i] += Σ_p L[p][i]   (fp32 atomics)
__device__ void wgrad_tp(const float* L, int ldl, int ni, const float* R, int ldr, int nj,
                         float* G, float* gb) {
  for (int idx = threadIdx.x; idx < ni * nj; idx += NT) {
    const int i = idx / nj, j = idx - i * nj;
    float s = 0.0f;
#pragma unroll 8
    for (int p = 0; p < TP; ++p) s = fmaf(L[p * ldl + i], R[p * ldr + j], s);
    atomicAdd(G + idx, s);
  }
  for (int i = threadIdx.x; i < ni; i += NT) {
    float s = 0.0f;
    for (int p = 0; p < TP; ++p) s += L[p * ldl + i];
    atomicAdd(gb + i, s);
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ΔW_n for the TP paths of this CTA (global index mg0 + p) into dW[p][j].
__device__ void gen_dw(float* dW, int d, int64_t mg0, int64_t valid, int n, uint32_t it,
                       uint32_t k0, uint32_t k1, float sqrt_dt) {
  const int nq = (d + 3) >> 2;
  for (int idx = threadIdx.x; idx < TP * nq; idx += NT) {
    const int p = idx / nq, q = idx - p * nq;
    const float4 z = normals4((uint32_t)q, (uint32_t)(mg0 + p), (uint32_t)n, it, k0, k1);
    const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = 4 * q + i;
      if (j < d) dW[p * d + j] = p < valid ? sqrt_dt * zz[i] : 0.0f;
    }
  }
}

__global__ void __launch_bounds__(NT) k_fwd_simt(PassArgs a) {
  extern __shared__ float sm[];
  const int d = a.d, w = a.w;
  const NetDims nd{d, w};
  const int64_t mloc0 = (int64_t)blockIdx.x * TP;
  const int64_t valid = min((int64_t)TP, a.B_local - mloc0);
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  float* X = sm;
  float* dW = X + TP * d;
  float* Z = dW + TP * d;
  float* H1 = Z + TP * d;
  float* H2 = H1 + TP * w;
  float* Y = H2 + TP * w;
  float* red = Y + TP;
  float* Ws = red + 64;
  const int lw = odd_ld(w), ld_ = odd_ld(d);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int idx = threadIdx.x; idx < TP * d; idx += NT) X[idx] = a.x0;
  if (threadIdx.x < TP) Y[threadIdx.x] = a.params[0];
  __syncthreads();

  for (int n = 0; n < a.N; ++n) {
    const float* P = a.params + nd.step_base(n);
    if (!a.eval) {   // X_n for the adjoint pass (coalesced: the tile is contiguous)
      float* xs = a.Xstore + ((int64_t)n * a.B_local + mloc0) * d;
      for (int idx = threadIdx.x; idx < valid * d; idx += NT) xs[idx] = X[idx];
    }
    gen_dw(dW, d, a.m0 + mloc0, valid, n, it, a.k0, a.k1, a.sqrt_dt);          // a1
    stage_rows(Ws, ld_, P + nd.off_W1(), w, d);
    __syncthreads();
    const float* b1 = P + nd.off_b1();
    gemm_tp<true>(X, d, d, Ws, ld_, w, [&](int p, int j, float v) {            // a3
      H1[p * w + j] = fmaxf(v + __ldg(b1 + j), 0.0f);
    });
    __syncthreads();
    stage_rows(Ws, lw, P + nd.off_W2(), w, w);
    __syncthreads();
    const float* b2 = P + nd.off_b2();
    gemm_tp<true>(H1, w, w, Ws, lw, w, [&](int p, int j, float v) {
      H2[p * w + j] = H1[p * w + j] + fmaxf(v + __ldg(b2 + j), 0.0f);
    });
    __syncthreads();
    stage_rows(Ws, lw, P + nd.off_W3(), d, w);
    __syncthreads();
    const float* b3 = P + nd.off_b3();
    gemm_tp<true>(H2, w, w, Ws, lw, d, [&](int p, int j, float v) {
      Z[p * d + j] = v + __ldg(b3 + j);
    });
    __syncthreads();
    for (int p = warp; p < TP; p += NT / 32) {                                  // a4
      float c = 0.0f, zz = 0.0f;
      for (int j = lane; j < d; j += 32) {
        const float z = Z[p * d + j];
        c = fmaf(z, dW[p * d + j], c);
        zz = fmaf(z, z, zz);
      }
      c = warp_sum(c);
      zz = warp_sum(zz);
      if (lane == 0) {
        const float y = Y[p];
        if (!a.eval && a.problem == kAllenCahn && p < valid)
          a.Ystore[(int64_t)n * a.B_local + mloc0 + p] = y;
        Y[p] = y - driver_f(a.problem, y, zz, a.lam) * a.dt + c;
      }
    }
    for (int idx = threadIdx.x; idx < TP * d; idx += NT) X[idx] = fmaf(kSqrt2, dW[idx], X[idx]);  // a2
    __syncthreads();
  }

  // a5: R = Y_N - g(X_N); loss; ā recursion and dY0 (a6, scalar part)
  float l2 = 0.0f, dy0 = 0.0f;
  for (int p = warp; p < TP; p += NT / 32) {
    float s = 0.0f;
    for (int j = lane; j < d; j += 32) s = fmaf(X[p * d + j], X[p * d + j], s);
    s = warp_sum(s);
    if (lane == 0 && p < valid) {
      const float R = Y[p] - terminal_g(a.problem, s);
      l2 += R * R;
      if (!a.eval) {
        const int64_t m = mloc0 + p;
        a.Rstore[m] = R;
        float ab = 2.0f * R * a.inv_B;
        if (a.problem == kAllenCahn) {
          for (int n = a.N - 1; n >= 0; --n) {
            const float y = a.Ystore[(int64_t)n * a.B_local + m];
            a.abar[(int64_t)n * a.B_local + m] = ab;                 // ā_{n+1}
            ab *= 1.0f - a.dt * driver_dfdy(a.problem, y);
          }
        } else {
          a.abar[m] = ab;                                              // ā_N = ā_n
        }
        dy0 += ab;
      }
    }
  }
  if (lane == 0) { red[warp] = l2; red[32 + warp] = dy0; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double L = 0.0;
    float g0 = 0.0f;
    for (int i = 0; i < NT / 32; ++i) { L += (double)red[i]; g0 += red[32 + i]; }
    atomicAdd(a.loss_acc, L);
    if (!a.eval) atomicAdd(a.grad, g0);
  }
}

__global__ void __launch_bounds__(NT) k_bwd_simt(PassArgs a, int tiles) {
  extern __shared__ float sm[];
  const int d = a.d, w = a.w;
  const NetDims nd{d, w};
  const int n = blockIdx.x / tiles;
  const int tile = blockIdx.x - n * tiles;
  const int64_t mloc0 = (int64_t)tile * TP;
  const int64_t valid = min((int64_t)TP, a.B_local - mloc0);
  const uint32_t it = a.state->it;
  float* X = sm;
  float* dW = X + TP * d;     // ΔW_n, then dZ_n in place
  float* H1 = dW + TP * d;    // H1, then dA1 in place
  float* A2 = H1 + TP * w;    // A2, then dA2 in place
  float* H2 = A2 + TP * w;    // H2, then dH2
  float* ab = H2 + TP * w;    // ā_{n+1} per path
  float* Ws = ab + TP;
  const int lw = odd_ld(w), ld_ = odd_ld(d);
  const float* P = a.params + nd.step_base(n);
  float* G = a.grad + nd.step_base(n);

  const float* xs = a.Xstore + ((int64_t)n * a.B_local + mloc0) * d;
  for (int idx = threadIdx.x; idx < TP * d; idx += NT) X[idx] = idx < valid * d ? xs[idx] : 0.0f;
  if (threadIdx.x < TP) {
    const int p = threadIdx.x;
    float v = 0.0f;
    if (p < valid)
      v = a.problem == kAllenCahn ? a.abar[(int64_t)n * a.B_local + mloc0 + p] : a.abar[mloc0 + p];
    ab[p] = v;
  }
  gen_dw(dW, d, a.m0 + mloc0, valid, n, it, a.k0, a.k1, a.sqrt_dt);
  stage_rows(Ws, ld_, P + nd.off_W1(), w, d);
  __syncthreads();
  // recompute the forward of step n (activation recompute)
  const float* b1 = P + nd.off_b1();
  gemm_tp<true>(X, d, d, Ws, ld_, w, [&](int p, int j, float v) {
    H1[p * w + j] = fmaxf(v + __ldg(b1 + j), 0.0f);
  });
  __syncthreads();
  stage_rows(Ws, lw, P + nd.off_W2(), w, w);
  __syncthreads();
  const float* b2 = P + nd.off_b2();
  gemm_tp<true>(H1, w, w, Ws, lw, w, [&](int p, int j, float v) {
    const float a2 = v + __ldg(b2 + j);
    A2[p * w + j] = a2;
    H2[p * w + j] = H1[p * w + j] + fmaxf(a2, 0.0f);
  });
  __syncthreads();
  stage_rows(Ws, lw, P + nd.off_W3(), d, w);
  __syncthreads();
  const float* b3 = P + nd.off_b3();
  const float zc = -a.dt * driver_dfdz_coef(a.problem, a.lam);   // dZ = ā(ΔW - Δt ∂_z f)
  gemm_tp<true>(H2, w, w, Ws, lw, d, [&](int p, int j, float v) {
    const float z = v + __ldg(b3 + j);
    dW[p * d + j] = ab[p] * fmaf(zc, z, dW[p * d + j]);
  });
  __syncthreads();
  // dW3 += dZᵀ H2 ; db3 += Σ dZ
  wgrad_tp(dW, d, d, H2, w, w, G + nd.off_W3(), G + nd.off_b3());
  stage_copy(Ws, P + nd.off_W3(), d * w);
  __syncthreads();
  // dH2 = dZ W3 ; dA2 = dH2 ⊙ 1[A2 > 0]  (ReLU'(0) = 0, R15)
  gemm_tp<false>(dW, d, d, Ws, w, w, [&](int p, int j, float v) {
    H2[p * w + j] = v;
    A2[p * w + j] = A2[p * w + j] > 0.0f ? v : 0.0f;
  });
  __syncthreads();
  // dW2 += dA2ᵀ H1 ; db2 += Σ dA2
  wgrad_tp(A2, w, w, H1, w, w, G + nd.off_W2(), G + nd.off_b2());
  stage_copy(Ws, P + nd.off_W2(), w * w);
  __syncthreads();
  // dH1 = dH2 + dA2 W2 ; dA1 = dH1 ⊙ 1[A1 > 0]  (A1 > 0 ⟺ H1 > 0)
  gemm_tp<false>(A2, w, w, Ws, w, w, [&](int p, int j, float v) {
    const float dh1 = H2[p * w + j] + v;
    H1[p * w + j] = H1[p * w + j] > 0.0f ? dh1 : 0.0f;
  });
  __syncthreads();
  // dW1 += dA1ᵀ X ; db1 += Σ dA1
  wgrad_tp(H1, w, w, X, d, d, G + nd.off_W1(), G + nd.off_b1());
}

size_t fwd_smem(int d, int w) {
  const size_t ws = (size_t)max(w * odd_ld(d), max(w * odd_ld(w), d * odd_ld(w)));
  return sizeof(float) * ((size_t)TP * (3 * d + 2 * w) + TP + 64 + ws);
}
size_t bwd_smem(int d, int w) {
  const size_t ws = (size_t)max(w * odd_ld(d), max(w * odd_ld(w), d * odd_ld(w)));
  return sizeof(float) * ((size_t)TP * (2 * d + 3 * w) + TP + ws);
}

}  // namespace

cudaError_t launch_fwd_simt(const PassArgs& a, cudaStream_t s) {
  const size_t smem = fwd_smem(a.d, a.w);
  cudaError_t e = cudaFuncSetAttribute(k_fwd_simt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)((a.B_local + TP - 1) / TP);
  k_fwd_simt<<<grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bwd_simt(const PassArgs& a, cudaStream_t s) {
  const size_t smem = bwd_smem(a.d, a.w);
  cudaError_t e = cudaFuncSetAttribute(k_bwd_simt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int tiles = (int)((a.B_local + TP - 1) / TP);
  k_bwd_simt<<<a.N * tiles, NT, smem, s>>>(a, tiles);
  return cudaGetLastError();
}

size_t simt_max_smem(int d, int w) { return fwd_smem(d, w) > bwd_smem(d, w) ? fwd_smem(d, w) : bwd_smem(d, w); }

}  // namespace bsde
