// simt.cu — fp32 CUDA-core forward and adjoint kernels (the fp32-accurate path:
// configs 1, 2, 4 and any d, w <= 127 outside the tcgen05 instantiations).
//
// Same data flow as the tensor-core path, register-tiled FFMA GEMMs:
//  k_pack_simt  fp32 master θ -> per-step transposed/padded weight images
//               W1ᵀ [d][112], W2ᵀ [w][112], W3ᵀ [w][112], W3 [d][112], W2 [w][112]
//               (row pitch LDW = 112 floats, zero padded) so staging is a straight copy.
//  k_fwd_simt   tile-major: a 64-path tile walks all N steps; activations are kept
//               feature-major in shared memory ([feature][64 paths]); every GEMM
//               C[64×nout] = A[64×K]·B[K×nout] gives each thread a 4-path × 8-output
//               block (32 FFMA per 3 LDS.128).  a1 Philox ΔW, a2 Euler X, a3 Z-net,
//               a4 Y update, a5 terminal loss; X_n stored for the adjoint.
//  k_bwd_simt   step-major persistent: each CTA owns a contiguous range of (n, tile)
//               items, recomputes the step-n net, back-propagates dZ_n, and adds the
//               weight-gradient blocks (8×8 per thread, contraction over the 64 paths)
//               into a per-CTA scratch gradient that is flushed with fp32 atomics when
//               the step changes.
//
// Citations: Eq. 5, Eq. 7, Eq. 6.
#include "kernels.cuh"

namespace bsde {
namespace {

constexpr int TP = 64;     // paths per tile
constexpr int TPP = 68;    // row pitch (floats) of the feature-major [k][path] smem buffers:
                           // rows 16 B apart in bank space, so the weight-gradient GEMM's
                           // 16-row float4 loads are conflict-free
constexpr int NT = 256;    // threads per CTA
constexpr int LDW = 112;   // row pitch of the packed weight images (floats); d, w <= 112

struct Pack {
  int d, w;
  int nais = 0;   // + Bᵀ image; the W2 images hold A = -RᵀR - εI (R25)
  __host__ __device__ size_t w1t() const { return 0; }                        // [d][LDW]
  __host__ __device__ size_t w2t() const { return (size_t)d * LDW; }          // [w][LDW]
  __host__ __device__ size_t w3t() const { return (size_t)(d + w) * LDW; }    // [w][LDW]
  __host__ __device__ size_t w3n() const { return (size_t)(d + 2 * w) * LDW; }  // [d][LDW]
  __host__ __device__ size_t w2n() const { return (size_t)(2 * d + 2 * w) * LDW; }  // [w][LDW]
  __host__ __device__ size_t bt() const { return (size_t)(2 * d + 3 * w) * LDW; }    // [d][LDW]
  __host__ __device__ size_t per_step() const { return (size_t)(2 * d + 3 * w + (nais ? d : 0)) * LDW; }
};

// A[i][j] = -Σ_r R[r][i] R[r][j] - ε δ_ij (NAIS-Net, R25; symmetric, so the
// transposed and the plain W2 images are the same matrix)
__device__ __forceinline__ float nais_A(const float* R, int w, int i, int j) {
  float g = 0.0f;
  for (int r = 0; r < w; ++r) g = fmaf(R[r * w + i], R[r * w + j], g);
  return -g - (i == j ? kNaisEps : 0.0f);
}

__global__ void k_pack_simt(const float* __restrict__ params, float* __restrict__ out, int d,
                            int w, int N, int nais) {
  const NetDims nd{d, w, nais};
  const Pack pk{d, w, nais};
  const int64_t per = (int64_t)pk.per_step();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)N * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / per);
    const int64_t r = i - n * per;
    const int row = (int)(r / LDW), col = (int)(r % LDW);
    const float* P = params + nd.step_base(n);
    float v = 0.0f;
    if (row < d) {                                  // W1ᵀ[k][j] = W1[j][k]
      if (col < w) v = P[nd.off_W1() + (int64_t)col * d + row];
    } else if (row < d + w) {                       // W2ᵀ[k][j] = W2[j][k]
      const int k = row - d;
      if (col < w) v = nais ? nais_A(P + nd.off_W2(), w, k, col) : P[nd.off_W2() + (int64_t)col * w + k];
    } else if (row < d + 2 * w) {                   // W3ᵀ[k][j] = W3[j][k]
      const int k = row - d - w;
      if (col < d) v = P[nd.off_W3() + (int64_t)col * w + k];
    } else if (row < 2 * d + 2 * w) {               // W3[i][j]
      const int k = row - d - 2 * w;
      if (col < w) v = P[nd.off_W3() + (int64_t)k * w + col];
    } else if (row < 2 * d + 3 * w) {               // W2[i][j]
      const int k = row - 2 * d - 2 * w;
      if (col < w) v = nais ? nais_A(P + nd.off_W2(), w, k, col) : P[nd.off_W2() + (int64_t)k * w + col];
    } else {                                        // Bᵀ[k][j] = B[j][k] (NAIS)
      const int k = row - 2 * d - 3 * w;
      if (col < w) v = P[nd.off_B() + (int64_t)col * d + k];
    }
    out[i] = v;
  }
}

// copy `floats` (multiple of 4) from global to shared, 16 B per thread-iteration
__device__ __forceinline__ void stage(float* dst, const float* __restrict__ src, int floats) {
  const float4* s = reinterpret_cast<const float4*>(src);
  float4* o = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < floats / 4; i += NT) o[i] = __ldg(s + i);
}

// C[p][j] = Σ_k At[k][p] · Bs[k][j] for p < 64, j < nout (<= LDW).  Thread
// (ty, tx) = (t/16, t%16) owns paths 4ty..4ty+3 and outputs 4tx..4tx+3 and
// 64+4tx..64+4tx+3.  epi(p0, j, float4 values-of-paths p0..p0+3).
template <typename Epi>
__device__ __forceinline__ void gemm_n(const float* At, const float* Bs, int K, int nout, Epi epi) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int p0 = 4 * ty, j0 = 4 * tx, j1 = 64 + 4 * tx;
  float acc[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;
  const bool hi = j1 < nout;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    const float4 a = *reinterpret_cast<const float4*>(At + k * TPP + p0);
    const float4 b0 = *reinterpret_cast<const float4*>(Bs + k * LDW + j0);
    const float4 b1 = hi ? *reinterpret_cast<const float4*>(Bs + k * LDW + j1) : make_float4(0, 0, 0, 0);
    const float av[4] = {a.x, a.y, a.z, a.w};
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int j = (c < 4 ? j0 : j1 - 4) + c;
    if (j < nout) epi(p0, j, make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]));
  }
}

// G[i][j] += Σ_p L[i][p] R[j][p] (feature-major operands, p < 64) into the per-CTA
// scratch gradient, i < ni, j < nj, row pitch ldg; gb[i] += Σ_p L[i][p].
__device__ void gemm_t(const float* L, int ni, const float* R, int nj, float* __restrict__ G,
                       int ldg, float* __restrict__ gb) {
  const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
  int iv[8], jv[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    iv[r] = (r < 4 ? 4 * ti : 64 + 4 * ti - 4) + r;
    jv[r] = (r < 4 ? 4 * tj : 64 + 4 * tj - 4) + r;
  }
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;
  for (int p = 0; p < TP; p += 4) {
    float4 lv[8], rv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      lv[r] = iv[r] < ni ? *reinterpret_cast<const float4*>(L + iv[r] * TPP + p) : make_float4(0, 0, 0, 0);
      rv[r] = jv[r] < nj ? *reinterpret_cast<const float4*>(R + jv[r] * TPP + p) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        acc[r][c] = fmaf(lv[r].x, rv[c].x, acc[r][c]);
        acc[r][c] = fmaf(lv[r].y, rv[c].y, acc[r][c]);
        acc[r][c] = fmaf(lv[r].z, rv[c].z, acc[r][c]);
        acc[r][c] = fmaf(lv[r].w, rv[c].w, acc[r][c]);
      }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (iv[r] < ni && jv[c] < nj) G[iv[r] * ldg + jv[c]] += acc[r][c];
  for (int i = threadIdx.x; i < ni; i += NT) {
    const float4* l = reinterpret_cast<const float4*>(L + i * TPP);
    float s = 0.0f;
#pragma unroll 4
    for (int q = 0; q < TP / 4; ++q) {
      const float4 v = l[q];
      s += (v.x + v.y) + (v.z + v.w);
    }
    if (gb) gb[i] += s;
  }
}

// ΔW_n of the tile into dWs[k][p] (feature-major), zero for paths >= valid.
// ΔW_n of a 64-path tile; coupled paths (cpl > 1): the sum of the cpl increments
// of fine steps n·cpl + j, each √(Δt/cpl)·z (NEXT-3)
__device__ void gen_dw(float* dWs, int d, int64_t mg0, int64_t valid, int n, uint32_t it,
                       uint32_t k0, uint32_t k1, float sqrt_dt_f, int cpl) {
  const int nq = (d + 3) >> 2;
  for (int idx = threadIdx.x; idx < TP * nq; idx += NT) {
    const int q = idx / TP, p = idx - q * TP;   // consecutive threads: consecutive paths
    float zz[4] = {0.f, 0.f, 0.f, 0.f};
    if (p < valid) {
      for (int j = 0; j < cpl; ++j) {
        const float4 z = normals4((uint32_t)q, (uint32_t)(mg0 + p), (uint32_t)(n * cpl + j), it, k0, k1);
        zz[0] += sqrt_dt_f * z.x; zz[1] += sqrt_dt_f * z.y;
        zz[2] += sqrt_dt_f * z.z; zz[3] += sqrt_dt_f * z.w;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (4 * q + i < d) dWs[(4 * q + i) * TPP + p] = zz[i];
  }
}

__device__ __forceinline__ float sum16(float v) {   // over the 16 lanes sharing ty
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(NT, 1) k_fwd_simt(PassArgs a, int ntiles) {
  extern __shared__ __align__(16) float sm[];
  const int d = a.d, w = a.w;
  const NetDims nd{d, w, a.nais};
  const Pack pk{d, w, a.nais};
  float* Xs = sm;                         // [d][64] X_n (fp32 state)
  float* dWs = Xs + d * TPP;              // [d][64]
  float* H1 = dWs + d * TPP;              // [w][64]
  float* H2 = H1 + w * TPP;               // [w][64]
  float* Ws = H2 + w * TPP;               // [K <= max(d, w)][LDW]
  float* Ys = Ws + (d > w ? d : w) * LDW; // [64]
  float* Ps = Ys + TP;                    // [64] prefix products P_{n+1} of the ā factors
  const float* wp = static_cast<const float*>(a.wpack);
  const int t = threadIdx.x, lane = t & 31, ty = t >> 4, tx = t & 15;
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  double lsum = 0.0;
  float dy0 = 0.0f;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t mloc0 = (int64_t)tile * TP;
    const int64_t valid = min((int64_t)TP, a.B_local - mloc0);
    for (int i = t; i < d * TPP; i += NT) Xs[i] = a.x0;
    if (t < TP) { Ys[t] = a.params[0]; Ps[t] = 1.0f; }
    __syncthreads();
    for (int n = 0; n < a.N; ++n) {
      const float* P = a.params + nd.step_base(n);
      const float* W = wp + (size_t)n * pk.per_step();
      if (!a.eval) {   // X_n for the adjoint pass: [n][tile][k][64], coalesced
        float4* xs = reinterpret_cast<float4*>(a.Xstore + ((size_t)n * ntiles + tile) * d * TP);
        for (int i = t; i < d * TP / 4; i += NT)
          xs[i] = *reinterpret_cast<const float4*>(Xs + (i >> 4) * TPP + 4 * (i & 15));
      }
      gen_dw(dWs, d, a.m0 + mloc0, valid, n, it, a.k0, a.k1, a.sqrt_dt_f, a.cpl);  // a1
      stage(Ws, W + pk.w1t(), d * LDW);
      __syncthreads();
      const float* b1 = P + nd.off_b1();
      gemm_n(Xs, Ws, d, w, [&](int p0, int j, float4 v) {                          // a3
        const float b = __ldg(b1 + j);
        *reinterpret_cast<float4*>(H1 + j * TPP + p0) =
            make_float4(fmaxf(v.x + b, 0.f), fmaxf(v.y + b, 0.f), fmaxf(v.z + b, 0.f), fmaxf(v.w + b, 0.f));
      });
      __syncthreads();
      const float* b2 = P + nd.off_b2();
      if (a.nais) {   // NAIS block (R25): first B X + C into H2, then A H1 is added below
        stage(Ws, W + pk.bt(), d * LDW);
        __syncthreads();
        gemm_n(Xs, Ws, d, w, [&](int p0, int j, float4 v) {
          const float b = __ldg(b2 + j);
          *reinterpret_cast<float4*>(H2 + j * TPP + p0) = make_float4(v.x + b, v.y + b, v.z + b, v.w + b);
        });
        __syncthreads();
      }
      stage(Ws, W + pk.w2t(), w * LDW);
      __syncthreads();
      gemm_n(H1, Ws, w, w, [&](int p0, int j, float4 v) {
        // A2 = W2 H1 + b2, or A H1 + (B X + C) for NAIS; H2 = H1 + ReLU(A2)
        const float4 c = a.nais ? *reinterpret_cast<const float4*>(H2 + j * TPP + p0)
                                : make_float4(__ldg(b2 + j), __ldg(b2 + j), __ldg(b2 + j), __ldg(b2 + j));
        const float4 h = *reinterpret_cast<const float4*>(H1 + j * TPP + p0);
        *reinterpret_cast<float4*>(H2 + j * TPP + p0) =
            make_float4(h.x + fmaxf(v.x + c.x, 0.f), h.y + fmaxf(v.y + c.y, 0.f),
                        h.z + fmaxf(v.z + c.z, 0.f), h.w + fmaxf(v.w + c.w, 0.f));
      });
      __syncthreads();
      stage(Ws, W + pk.w3t(), w * LDW);
      __syncthreads();
      const float* b3 = P + nd.off_b3();
      float c4[4] = {0, 0, 0, 0}, z4[4] = {0, 0, 0, 0}, s4[4] = {0, 0, 0, 0};
      gemm_n(H2, Ws, w, d, [&](int p0, int j, float4 v) {                          // a4 partials
        const float b = __ldg(b3 + j);
        const float4 dw = *reinterpret_cast<const float4*>(dWs + j * TPP + p0);
        const float zv[4] = {v.x + b, v.y + b, v.z + b, v.w + b};
        const float wv[4] = {dw.x, dw.y, dw.z, dw.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          c4[r] = fmaf(zv[r], wv[r], c4[r]);
          z4[r] = fmaf(zv[r], zv[r], z4[r]);
          s4[r] += zv[r];
        }
      });
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        c4[r] = sum16(c4[r]);
        z4[r] = sum16(z4[r]);
        s4[r] = sum16(s4[r]);
      }
      if (tx == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int p = 4 * ty + r;
          const float y = Ys[p];
          if (!a.eval && per_step_abar(a.problem)) {
            Ps[p] *= 1.0f - a.dt * driver_dfdy(a.problem, y);
            if (p < valid) a.Pstore[(int64_t)n * a.B_local + mloc0 + p] = Ps[p];
          }
          Ys[p] = y - driver_f(a.problem, y, z4[r], s4[r], a.lam) * a.dt + c4[r];
        }
      }
      for (int i = t; i < d * TPP; i += NT) Xs[i] = x_step(a.problem, Xs[i], dWs[i]);   // a2
      __syncthreads();
    }
    // a5: R = Y_N - g(X_N); loss; ā_N (times P_N) and dY0 = ā_0 = ā_N P_N
    if (t < TP && t < valid) {
      float s = 0.0f;
      for (int k = 0; k < d; ++k) s = fmaf(Xs[k * TPP + t], Xs[k * TPP + t], s);
      const float R = Ys[t] - terminal_g(a.problem, s);
      const int64_t m = mloc0 + t;
      lsum += (double)R * R;
      if (!a.eval) {
        a.Rstore[m] = R;
        float ab = 2.0f * R * a.inv_B;
        if (per_step_abar(a.problem)) ab *= Ps[t];
        a.abar[m] = ab;
        dy0 += ab;
      }
    }
    __syncthreads();
  }
  // block reduction (threads t < 64 carry the sums)
  double lw = lsum;
  float gw = dy0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lw += __shfl_xor_sync(0xffffffffu, lw, o);
    gw += __shfl_xor_sync(0xffffffffu, gw, o);
  }
  __shared__ double lred[2];
  __shared__ float gred[2];
  if (t < 64 && lane == 0) { lred[t >> 5] = lw; gred[t >> 5] = gw; }
  __syncthreads();
  if (t == 0) {
    const double L = lred[0] + lred[1];
    const float g0 = gred[0] + gred[1];
    if (a.lpart) {   // deterministic mode: per-CTA partials, summed in order by k_det_reduce
      a.lpart[blockIdx.x] = L;
      a.y0part[blockIdx.x] = a.eval ? 0.0f : g0;
    } else {
      if (L != 0.0) atomicAdd(a.loss_acc, L);
      if (!a.eval && g0 != 0.0f) atomicAdd(a.grad, g0);
    }
  }
}

__global__ void __launch_bounds__(NT, 1) k_bwd_simt(PassArgs a, int ntiles, int64_t items) {
  extern __shared__ __align__(16) float sm[];
  const int d = a.d, w = a.w;
  const NetDims nd{d, w, a.nais};
  const Pack pk{d, w, a.nais};
  float* Xs = sm;                         // [d][64]
  float* dZ = Xs + d * TPP;               // [d][64]  ΔW_n, then dZ_n in place
  float* H1 = dZ + d * TPP;               // [w][64]
  float* H2 = H1 + w * TPP;               // [w][64]
  float* dH = H2 + w * TPP;               // [w][64]  dH2, then dA1 in place
  float* dA2 = dH + w * TPP;              // [w][64]
  float* Ws = dA2 + w * TPP;              // [K <= max(d, w)][LDW]
  float* ab = Ws + (d > w ? d : w) * LDW; // [64]
  uint8_t* m2 = reinterpret_cast<uint8_t*>(ab + TP);   // [w][64] 1[A2 > 0]
  const float* wp = static_cast<const float*>(a.wpack);
  float* scratch = a.gpart + (size_t)blockIdx.x * nd.step_size();
  const int t = threadIdx.x;
  const uint32_t it = a.state->it;
  const float zc = -a.dt * driver_dfdz_coef(a.problem, a.lam);
  const float zc0 = -a.dt * driver_dfdz_const(a.problem);
  const int64_t i0 = blockIdx.x * items / gridDim.x, i1 = (blockIdx.x + 1) * items / gridDim.x;
  const int64_t P = nd.step_size();
  int cur_n = -1;

  auto flush = [&]() {   // scratch -> gradient of step cur_n (fp32 atomics), then zero
    __syncthreads();
    if (a.dpart) {   // deterministic mode: this CTA's partial of step cur_n (every entry)
      float* G = a.dpart + ((int64_t)blockIdx.x * a.dseg + (cur_n - (int)(i0 / ntiles))) * P;
      for (int64_t i = t; i < P; i += NT) {
        G[i] = scratch[i];
        scratch[i] = 0.0f;
      }
    } else {
      float* G = a.grad + nd.step_base(cur_n);
      for (int64_t i = t; i < P; i += NT) {
        const float v = scratch[i];
        if (v != 0.0f) atomicAdd(G + i, v);
        scratch[i] = 0.0f;
      }
    }
    __syncthreads();
  };
  for (int64_t i = t; i < P; i += NT) scratch[i] = 0.0f;
  __syncthreads();

  for (int64_t item = i0; item < i1; ++item) {
    const int n = (int)(item / ntiles), tile = (int)(item - (int64_t)n * ntiles);
    if (n != cur_n) {
      if (cur_n >= 0) flush();
      cur_n = n;
    }
    const int64_t mloc0 = (int64_t)tile * TP;
    const int64_t valid = min((int64_t)TP, a.B_local - mloc0);
    const float* Pn = a.params + nd.step_base(n);
    const float* W = wp + (size_t)n * pk.per_step();
    {
      const float4* xs = reinterpret_cast<const float4*>(a.Xstore + ((size_t)n * ntiles + tile) * d * TP);
      for (int i = t; i < d * TP / 4; i += NT)
        *reinterpret_cast<float4*>(Xs + (i >> 4) * TPP + 4 * (i & 15)) = __ldg(xs + i);
    }
    if (t < TP) {
      const int64_t m = mloc0 + t;
      ab[t] = t < valid ? (per_step_abar(a.problem) ? a.abar[m] / a.Pstore[(int64_t)n * a.B_local + m] : a.abar[m])
                        : 0.0f;
    }
    gen_dw(dZ, d, a.m0 + mloc0, valid, n, it, a.k0, a.k1, a.sqrt_dt_f, a.cpl);
    stage(Ws, W + pk.w1t(), d * LDW);
    __syncthreads();
    const float* b1 = Pn + nd.off_b1();
    gemm_n(Xs, Ws, d, w, [&](int p0, int j, float4 v) {           // recompute H1
      const float b = __ldg(b1 + j);
      *reinterpret_cast<float4*>(H1 + j * TPP + p0) =
          make_float4(fmaxf(v.x + b, 0.f), fmaxf(v.y + b, 0.f), fmaxf(v.z + b, 0.f), fmaxf(v.w + b, 0.f));
    });
    __syncthreads();
    const float* b2 = Pn + nd.off_b2();
    if (a.nais) {   // NAIS: B X + C into H2 first (R25)
      stage(Ws, W + pk.bt(), d * LDW);
      __syncthreads();
      gemm_n(Xs, Ws, d, w, [&](int p0, int j, float4 v) {
        const float b = __ldg(b2 + j);
        *reinterpret_cast<float4*>(H2 + j * TPP + p0) = make_float4(v.x + b, v.y + b, v.z + b, v.w + b);
      });
      __syncthreads();
    }
    stage(Ws, W + pk.w2t(), w * LDW);
    __syncthreads();
    gemm_n(H1, Ws, w, w, [&](int p0, int j, float4 v) {           // recompute H2, mask of A2
      const float4 c = a.nais ? *reinterpret_cast<const float4*>(H2 + j * TPP + p0)
                              : make_float4(__ldg(b2 + j), __ldg(b2 + j), __ldg(b2 + j), __ldg(b2 + j));
      const float4 h = *reinterpret_cast<const float4*>(H1 + j * TPP + p0);
      const float av[4] = {v.x + c.x, v.y + c.y, v.z + c.z, v.w + c.w};
      *reinterpret_cast<float4*>(H2 + j * TPP + p0) =
          make_float4(h.x + fmaxf(av[0], 0.f), h.y + fmaxf(av[1], 0.f), h.z + fmaxf(av[2], 0.f),
                      h.w + fmaxf(av[3], 0.f));
      uchar4 mk;
      mk.x = av[0] > 0.f; mk.y = av[1] > 0.f; mk.z = av[2] > 0.f; mk.w = av[3] > 0.f;
      *reinterpret_cast<uchar4*>(m2 + j * TP + p0) = mk;
    });
    __syncthreads();
    stage(Ws, W + pk.w3t(), w * LDW);
    __syncthreads();
    const float* b3 = Pn + nd.off_b3();
    gemm_n(H2, Ws, w, d, [&](int p0, int j, float4 v) {           // dZ = ā(ΔW - Δt ∂_z f)
      const float b = __ldg(b3 + j);
      float4 dw = *reinterpret_cast<const float4*>(dZ + j * TPP + p0);
      dw.x = ab[p0] * fmaf(zc, v.x + b, dw.x + zc0);
      dw.y = ab[p0 + 1] * fmaf(zc, v.y + b, dw.y + zc0);
      dw.z = ab[p0 + 2] * fmaf(zc, v.z + b, dw.z + zc0);
      dw.w = ab[p0 + 3] * fmaf(zc, v.w + b, dw.w + zc0);
      *reinterpret_cast<float4*>(dZ + j * TPP + p0) = dw;
    });
    __syncthreads();
    stage(Ws, W + pk.w3n(), d * LDW);
    // dW3 += dZᵀ H2 ; db3 += Σ dZ   (while W3 is being staged)
    gemm_t(dZ, d, H2, w, scratch + nd.off_W3(), w, scratch + nd.off_b3());
    __syncthreads();
    gemm_n(dZ, Ws, d, w, [&](int p0, int j, float4 v) {           // dH2 = dZ W3 ; dA2
      *reinterpret_cast<float4*>(dH + j * TPP + p0) = v;
      const uchar4 mk = *reinterpret_cast<const uchar4*>(m2 + j * TP + p0);
      *reinterpret_cast<float4*>(dA2 + j * TPP + p0) =
          make_float4(mk.x ? v.x : 0.f, mk.y ? v.y : 0.f, mk.z ? v.z : 0.f, mk.w ? v.w : 0.f);
    });
    __syncthreads();
    stage(Ws, W + pk.w2n(), w * LDW);
    // dW2 += dA2ᵀ H1 ; db2 += Σ dA2
    gemm_t(dA2, w, H1, w, scratch + nd.off_W2(), w, scratch + nd.off_b2());
    if (a.nais) gemm_t(dA2, w, Xs, d, scratch + nd.off_B(), d, nullptr);   // B̄ += dA2ᵀ X (R25)
    __syncthreads();
    gemm_n(dA2, Ws, w, w, [&](int p0, int j, float4 v) {          // dA1 = (dH2 + dA2 W2) ⊙ 1[H1 > 0]
      const float4 h = *reinterpret_cast<const float4*>(H1 + j * TPP + p0);
      const float4 g = *reinterpret_cast<const float4*>(dH + j * TPP + p0);
      *reinterpret_cast<float4*>(dH + j * TPP + p0) =
          make_float4(h.x > 0.f ? g.x + v.x : 0.f, h.y > 0.f ? g.y + v.y : 0.f,
                      h.z > 0.f ? g.z + v.z : 0.f, h.w > 0.f ? g.w + v.w : 0.f);
    });
    __syncthreads();
    // dW1 += dA1ᵀ X ; db1 += Σ dA1
    gemm_t(dH, w, Xs, d, scratch + nd.off_W1(), d, scratch + nd.off_b1());
    __syncthreads();
  }
  if (cur_n >= 0) flush();
}

size_t fwd_smem(int d, int w) {
  return sizeof(float) * ((size_t)TPP * (2 * d + 2 * w) + (size_t)(d > w ? d : w) * LDW + 2 * TP + 16);
}
size_t bwd_smem(int d, int w) {
  return sizeof(float) * ((size_t)TPP * (2 * d + 4 * w) + (size_t)(d > w ? d : w) * LDW + TP) +
         (size_t)w * TP;
}
int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

bool simt_supported(int d, int w) { return d <= LDW && w <= LDW && bwd_smem(d, w) <= 227 * 1024; }
size_t simt_max_smem(int d, int w) { return fwd_smem(d, w) > bwd_smem(d, w) ? fwd_smem(d, w) : bwd_smem(d, w); }
size_t simt_pack_bytes(int d, int w, int N, int nais) {
  return (size_t)N * Pack{d, w, nais}.per_step() * sizeof(float);
}
size_t simt_xstore_bytes(int d, int N, int64_t B_local) {
  return (size_t)N * (size_t)((B_local + TP - 1) / TP) * d * TP * sizeof(float);
}
size_t simt_scratch_bytes(int d, int w, int nais) {
  return (size_t)sm_count() * NetDims{d, w, nais}.step_size() * sizeof(float);
}

cudaError_t launch_pack_simt(const PassArgs& a, cudaStream_t s) {
  const int64_t total = (int64_t)a.N * Pack{a.d, a.w, a.nais}.per_step();
  int grid = (int)((total + NT - 1) / NT);
  if (grid > 148 * 16) grid = 148 * 16;
  k_pack_simt<<<grid, NT, 0, s>>>(a.params, static_cast<float*>(const_cast<void*>(a.wpack)), a.d, a.w,
                                  a.N, a.nais);
  return cudaGetLastError();
}

cudaError_t launch_fwd_simt(const PassArgs& a, cudaStream_t s) {
  const size_t smem = fwd_smem(a.d, a.w);
  cudaError_t e = cudaFuncSetAttribute(k_fwd_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int ntiles = (int)((a.B_local + TP - 1) / TP), sms = sm_count();
  k_fwd_simt<<<ntiles < sms ? ntiles : sms, NT, smem, s>>>(a, ntiles);
  return cudaGetLastError();
}

cudaError_t launch_bwd_simt(const PassArgs& a, cudaStream_t s) {
  const size_t smem = bwd_smem(a.d, a.w);
  cudaError_t e = cudaFuncSetAttribute(k_bwd_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int ntiles = (int)((a.B_local + TP - 1) / TP), sms = sm_count();
  const int64_t items = (int64_t)ntiles * a.N;
  k_bwd_simt<<<(int)(items < sms ? items : sms), NT, smem, s>>>(a, ntiles, items);
  return cudaGetLastError();
}

}  // namespace bsde
